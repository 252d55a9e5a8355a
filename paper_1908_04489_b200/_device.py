"""PyTorch plumbing: device selection, raw pointers and streams for the C ABI."""
from __future__ import annotations

import numpy as np
import torch

F64 = torch.float64
I64 = torch.int64


def require_cuda(device=None) -> torch.device:
    """The CUDA device to run on; raises (no CPU fallback) when there is none."""
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1908_04489_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device (got {dev})")
    return dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "device tensor must be contiguous CUDA memory"
    return t.data_ptr()


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def to_device_f64(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=F64).contiguous()
    a = np.ascontiguousarray(x, dtype=np.float64)
    if not a.flags.writeable:
        a = a.copy()
    return torch.from_numpy(a).to(device)


def to_device_i64(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=I64).contiguous()
    a = np.ascontiguousarray(x, dtype=np.int64)
    if not a.flags.writeable:
        a = a.copy()
    return torch.from_numpy(a).to(device)


def to_host_f64(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        return x.detach().to("cpu").numpy()
    return np.asarray(x, dtype=np.float64)
