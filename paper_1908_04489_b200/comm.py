"""NCCL communicator of the C ABI (ucp_comm_*, ucp_allgather_f64,
ucp_allreduce_min_i64) -- the exchange plumbing a non-Python host uses
(SURVEY.md §8b).  The Python solver itself exchanges through
torch.distributed (distributed.py); this wrapper exists to exercise and
document the C entry points from Python.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._device import ptr, stream_ptr

__all__ = ["NcclComm", "COMM_ID_BYTES"]

COMM_ID_BYTES = 128
_c = ctypes
_SIGS = {
    "ucp_comm_unique_id": (_c.c_int, [_c.c_void_p]),
    "ucp_comm_init": (_c.c_int, [_c.c_int, _c.c_int, _c.c_void_p, _c.POINTER(_c.c_void_p)]),
    "ucp_comm_destroy": (_c.c_int, [_c.c_void_p]),
    "ucp_allgather_f64": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_void_p]),
    "ucp_allreduce_min_i64": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_void_p]),
}
_lib.SIGNATURES.update(_SIGS)


def _bind():
    lib = _lib.load()
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


class NcclComm:
    """One rank of an NCCL communicator on the current CUDA device."""

    @staticmethod
    def unique_id() -> bytes:
        lib = _bind()
        buf = (_c.c_ubyte * COMM_ID_BYTES)()
        _lib.check(lib.ucp_comm_unique_id(_c.cast(buf, _c.c_void_p)), "ucp_comm_unique_id")
        return bytes(buf)

    def __init__(self, nranks: int, rank: int, uid: bytes):
        if len(uid) != COMM_ID_BYTES:
            raise ValueError(f"communicator id must be {COMM_ID_BYTES} bytes")
        self.lib = _bind()
        self.nranks, self.rank = int(nranks), int(rank)
        buf = (_c.c_ubyte * COMM_ID_BYTES).from_buffer_copy(uid)
        self.handle = _c.c_void_p()
        _lib.check(self.lib.ucp_comm_init(self.nranks, self.rank, _c.cast(buf, _c.c_void_p), _c.byref(self.handle)),
                   "ucp_comm_init")

    def allgather_(self, buf: torch.Tensor) -> None:
        """In-place all-gather of each rank's chunk of a float64 CUDA tensor."""
        c = buf.numel() // self.nranks
        send = buf.data_ptr() + 8 * self.rank * c
        _lib.check(self.lib.ucp_allgather_f64(self.handle, send, ptr(buf), c, stream_ptr(buf.device)),
                   "ucp_allgather_f64")

    def allreduce_min_(self, t: torch.Tensor) -> None:
        _lib.check(self.lib.ucp_allreduce_min_i64(self.handle, ptr(t), t.numel(), stream_ptr(t.device)),
                   "ucp_allreduce_min_i64")

    def close(self) -> None:
        if self.handle:
            self.lib.ucp_comm_destroy(self.handle)
            self.handle = _c.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass
