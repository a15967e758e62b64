"""NCCL communicators over NVLink for the every-tau weight average (psg_comm_*).

Multi-process (torchrun, one process per GPU): ``Communicator.create(ctx, nranks, rank,
uid)`` with the 128-byte ncclUniqueId broadcast by the launcher (torch.distributed is
only the rendezvous plumbing).  Single process driving several GPUs:
``Communicator.create_all(ctxs)`` (ncclCommInitAll).
"""
from __future__ import annotations

import ctypes
from typing import List, Sequence

from . import _lib

MODES = {"fast": _lib.AVERAGE_FAST, "ordered": _lib.AVERAGE_ORDERED}


def unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _lib.call("psg_comm_unique_id", buf)
    return buf.raw


class Communicator:
    def __init__(self, handle, ctx):
        self.handle = handle
        self.ctx = ctx

    @classmethod
    def create(cls, ctx, nranks: int, rank: int, uid: bytes) -> "Communicator":
        h = ctypes.c_void_p()
        _lib.call("psg_comm_create", ctx.handle, nranks, rank, uid, ctypes.byref(h))
        return cls(h, ctx)

    @classmethod
    def create_all(cls, ctxs: Sequence) -> List["Communicator"]:
        arr = (ctypes.c_void_p * len(ctxs))(*[c.handle.value for c in ctxs])
        out = (ctypes.c_void_p * len(ctxs))()
        _lib.call("psg_comm_create_all", arr, len(ctxs), out)
        return [cls(ctypes.c_void_p(out[i]), ctxs[i]) for i in range(len(ctxs))]

    def close(self) -> None:
        """Destroy the communicator (ncclCommDestroy).  With several communicators per
        process, close them in the same order on every rank, after the nets whose captured
        round graphs use them."""
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.lib().psg_comm_destroy(h)
            except Exception:
                pass
            self.handle = None

    def __del__(self):
        self.close()

    @staticmethod
    def average(comms: Sequence["Communicator"], nets: Sequence, mode: str = "fast") -> None:
        """In-place weights_mean of every net's flat parameters (stream-ordered)."""
        c = (ctypes.c_void_p * len(comms))(*[x.handle.value for x in comms])
        n = (ctypes.c_void_p * len(nets))(*[x.handle.value for x in nets])
        _lib.call("psg_comm_average", c, n, len(nets), MODES[mode])

    @staticmethod
    def average_grads(comms: Sequence["Communicator"], nets: Sequence, mode: str = "fast") -> None:
        """In-place mean of every net's flat gradient buffer (run_naive, schemes.hpp:248)."""
        c = (ctypes.c_void_p * len(comms))(*[x.handle.value for x in comms])
        n = (ctypes.c_void_p * len(nets))(*[x.handle.value for x in nets])
        _lib.call("psg_comm_average_grads", c, n, len(nets), MODES[mode])

    @staticmethod
    def broadcast(comms: Sequence["Communicator"], nets: Sequence, root: int = 0) -> None:
        c = (ctypes.c_void_p * len(comms))(*[x.handle.value for x in comms])
        n = (ctypes.c_void_p * len(nets))(*[x.handle.value for x in nets])
        _lib.call("psg_comm_broadcast", c, n, len(nets), root)


class FlatBuffer:
    """A raw fp32 buffer in HBM (psg_buffer) for the averaging-only sweep."""

    def __init__(self, ctx, n: int):
        self.ctx = ctx
        self.n = n
        h = ctypes.c_void_p()
        _lib.call("psg_buffer_create", ctx.handle, n, ctypes.byref(h))
        self.handle = h

    def fill_uniform(self, seed: int, lo: float = -1.0, hi: float = 1.0) -> None:
        _lib.call("psg_buffer_fill_uniform", self.handle, seed, lo, hi)

    def read(self):
        import numpy as np
        out = np.empty(self.n, np.float32)
        _lib.call("psg_buffer_read", self.handle, out.ctypes.data_as(_lib._F), self.n)
        return out

    def write(self, host) -> None:
        import numpy as np
        a = np.ascontiguousarray(host, np.float32)
        _lib.call("psg_buffer_write", self.handle, a.ctypes.data_as(_lib._F), a.size)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.lib().psg_buffer_destroy(h)
            except Exception:
                pass
            self.handle = None

    @staticmethod
    def average(comms: Sequence[Communicator], bufs: Sequence["FlatBuffer"],
                mode: str = "fast") -> float:
        """Average one buffer per communicator; returns the max device time (ms)."""
        c = (ctypes.c_void_p * len(comms))(*[x.handle.value for x in comms])
        b = (ctypes.c_void_p * len(bufs))(*[x.handle.value for x in bufs])
        ms = ctypes.c_float()
        _lib.call("psg_comm_average_buffer", c, b, len(bufs), MODES[mode], ctypes.byref(ms))
        return ms.value

    @staticmethod
    def average_local(bufs: Sequence["FlatBuffer"]) -> None:
        b = (ctypes.c_void_p * len(bufs))(*[x.handle.value for x in bufs])
        _lib.call("psg_buffer_average_local", b, len(bufs))
