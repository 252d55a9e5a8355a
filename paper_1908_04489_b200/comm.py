"""The library's own NCCL communicator (C ABI: ucp_comm_*, ucp_allgather_f64,
ucp_allgatherv_f64, ucp_allreduce_min_i64) as a sharding backend.

The solver's exchanges -- one all-gather of the updated controller per phase,
one MIN all-reduce of the error slots per synchronisation (reference
solver.py:16-20) -- normally run through torch.distributed
(distributed.py).  A process that has no torch.distributed process group (an
MPI or batch-system launch, or a non-Python host driving the same C ABI)
shards the solve with this communicator instead: rank 0 creates the 128-byte
NCCL id, the launcher hands it to every rank, and

    comm = NcclComm(world, rank, uid)
    P.solve(problem, cfg, sharding=comm.sharding())

runs the identical work-balanced plans and exchanges as the torch path --
bitwise the single-GPU result.  NCCL is resolved with dlopen inside the
library (a libnccl already in the process is reused).
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._device import ptr, stream_ptr
from .distributed import Sharding

__all__ = ["NcclComm", "CommSharding", "COMM_ID_BYTES"]

COMM_ID_BYTES = 128
_c = ctypes
_SIGS = {
    "ucp_comm_unique_id": (_c.c_int, [_c.c_void_p]),
    "ucp_comm_init": (_c.c_int, [_c.c_int, _c.c_int, _c.c_void_p, _c.POINTER(_c.c_void_p)]),
    "ucp_comm_destroy": (_c.c_int, [_c.c_void_p]),
    "ucp_allgather_f64": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_void_p]),
    "ucp_allgatherv_f64": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_void_p]),
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
    """One rank of an NCCL communicator on the current CUDA device.  All
    collectives are asynchronous on the current stream (stream order is the
    solver's ordering, as for every other library call)."""

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

    def sharding(self) -> "CommSharding":
        """The solver's Sharding over this communicator."""
        return CommSharding(rank=self.rank, world=self.nranks, comm=self)

    def allgather_(self, buf: torch.Tensor) -> None:
        """In-place all-gather of each rank's equal chunk of a float64 CUDA tensor."""
        c = buf.numel() // self.nranks
        send = buf.data_ptr() + 8 * self.rank * c
        _lib.check(self.lib.ucp_allgather_f64(self.handle, send, ptr(buf), c, stream_ptr(buf.device)),
                   "ucp_allgather_f64")

    def allgatherv_(self, buf: torch.Tensor, bounds) -> None:
        """In-place uneven all-gather: rank r owns buf[bounds[r]:bounds[r+1]]."""
        b = (_c.c_int64 * len(bounds))(*[int(x) for x in bounds])
        _lib.check(self.lib.ucp_allgatherv_f64(self.handle, ptr(buf), b, stream_ptr(buf.device)),
                   "ucp_allgatherv_f64")

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


class CommSharding(Sharding):
    """Sharding whose exchanges run on a library NcclComm instead of a
    torch.distributed process group (same plans, same layout, same bits)."""

    def __init__(self, rank: int, world: int, comm: NcclComm):
        super().__init__(rank=rank, world=world)
        object.__setattr__(self, "comm", comm)

    def allgather_(self, buf: torch.Tensor) -> None:
        if self.world > 1:
            self.comm.allgather_(buf)

    def allgather_uneven_(self, buf: torch.Tensor, bounds: tuple) -> None:
        if self.world > 1:
            self.comm.allgatherv_(buf, bounds)

    def allreduce_min_(self, t: torch.Tensor) -> None:
        if self.world > 1:
            self.comm.allreduce_min_(t)
