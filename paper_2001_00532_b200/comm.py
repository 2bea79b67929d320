"""NCCL communicators of libspx (spx_comm_init / spx_gather /
spx_reduce_rows; §8(e)): the data-path collectives of the multi-GPU shards.

One communicator per process (one process per GPU under torchrun).  The
128-byte NCCL unique id is created by rank 0 through the C-ABI and broadcast
over the existing torch.distributed process group (its store), which is the
only thing torch.distributed carries; the gathers and reductions themselves
run as NCCL calls on the caller's CUDA stream.  `partition.gather_rows` /
`reduce_partials` route through a `Comm` when one is given and the tensors
are on the GPU, and through torch.distributed otherwise (gloo in the CPU
tests).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib

_DTYPES = {torch.float64: _lib.SPX_F64, torch.float32: _lib.SPX_F32, torch.int32: _lib.SPX_I32}


def available() -> bool:
    return bool(_lib.load().spx_comm_available())


def _stream_ptr(t: torch.Tensor, stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream(t.device)
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dtype(t: torch.Tensor) -> int:
    if t.dtype not in _DTYPES:
        raise TypeError(f"collective on {t.dtype}: only float64, float32 and int32 are supported")
    return _DTYPES[t.dtype]


class Comm:
    """An NCCL communicator created through libspx."""

    def __init__(self, handle: int, nranks: int, rank: int):
        self.handle = ctypes.c_void_p(handle)
        self.nranks = nranks
        self.rank = rank

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _lib.check(_lib.load().spx_comm_unique_id(buf), "spx_comm_unique_id")
        return buf.raw

    @classmethod
    def init(cls, nranks: int, rank: int, uid: bytes) -> "Comm":
        """Join communicator `uid` as `rank` on the current CUDA device."""
        if len(uid) != 128:
            raise ValueError("an NCCL unique id is 128 bytes")
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(uid, 128)
        _lib.check(_lib.load().spx_comm_init(nranks, rank, buf, ctypes.byref(h)), "spx_comm_init")
        return cls(h.value, nranks, rank)

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        """One communicator over the ranks of a torch.distributed group (the
        id travels over the group; every rank's current device is its GPU)."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        box = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0, group=group)
        return cls.init(world, rank, box[0])

    @classmethod
    def single(cls) -> "Comm":
        """A one-rank communicator on the current device."""
        return cls.init(1, 0, cls.unique_id())

    def info(self) -> tuple[int, int]:
        n, r = ctypes.c_int(), ctypes.c_int()
        _lib.check(_lib.load().spx_comm_info(self.handle, ctypes.byref(n), ctypes.byref(r)), "spx_comm_info")
        return n.value, r.value

    def all_gather(self, send: torch.Tensor, recv: torch.Tensor, stream=None) -> torch.Tensor:
        """recv[r*count:(r+1)*count] = rank r's `send` (count = send.numel())."""
        if not (send.is_cuda and recv.is_cuda and send.is_contiguous() and recv.is_contiguous()):
            raise ValueError("all_gather needs contiguous CUDA tensors")
        if send.dtype != recv.dtype or recv.numel() != send.numel() * self.nranks:
            raise ValueError("recv must hold nranks * send.numel() elements of send's dtype")
        _lib.check(_lib.load().spx_gather(self.handle, send.data_ptr(), recv.data_ptr(), send.numel(), _dtype(send),
                                          _stream_ptr(send, stream)), "spx_gather")
        return recv

    def all_reduce(self, t: torch.Tensor, stream=None) -> torch.Tensor:
        """In-place element-wise sum over ranks."""
        if not (t.is_cuda and t.is_contiguous()):
            raise ValueError("all_reduce needs a contiguous CUDA tensor")
        _lib.check(_lib.load().spx_reduce_rows(self.handle, t.data_ptr(), t.data_ptr(), t.numel(), _dtype(t),
                                               _stream_ptr(t, stream)), "spx_reduce_rows")
        return t

    def close(self) -> None:
        if self.handle:
            _lib.check(_lib.load().spx_comm_destroy(self.handle), "spx_comm_destroy")
            self.handle = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
