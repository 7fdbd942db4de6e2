"""Multi-GPU type II: one process per GPU, the rank-K sum
split across GPUs inside the library.

The reference parallelizes exec_nufft2 over host threads: contiguous r-ranges
per worker, each accumulating a partial f, merged in a fixed order
(proj/include/nufft/transforms.hpp:174-197).  Here the workers are GPUs:

* ``NcclComm`` — an NCCL communicator owned by the library (nufft_comm_init;
  NCCL is dlopen'ed by libnufft_b200.so).  ``from_process_group`` bootstraps
  it over an existing torch.distributed group (rank 0's unique id broadcast
  through that group, any backend).
* ``Plan2.execute_multi_device(c, f, comm)`` — nufft_plan2_exec_multi: rank g
  evaluates terms [K g/G, K (g+1)/G), pass 2 writes its partial in bucket
  order in row chunks, each chunk is summed (ncclReduce / ncclAllReduce, fp64)
  on the communicator's stream while the next chunk computes, and the
  receiving ranks un-permute once.
* ``exec_rsplit_torch`` — the same algorithm with the collective supplied by
  torch.distributed (e.g. gloo on CPU tensors): used by the tests, and by
  callers that already own a process group and not an NCCL communicator.
* batch sharding (weak scaling) needs no collective: each rank runs
  ``execute_device`` on its own slice of the batch (``batch_range``).
"""
from __future__ import annotations

import ctypes as C

from ._lib import lib
from .api import _check

UNIQUE_ID_BYTES = 128


def term_range(K: int, world: int, rank: int) -> tuple[int, int]:
    """[r_begin, r_end) of `rank` (nufft_multi_term_range; host-only, no GPU)."""
    a, b = C.c_size_t(), C.c_size_t()
    _check(lib().nufft_multi_term_range(K, world, rank, C.byref(a), C.byref(b)))
    return a.value, b.value


def batch_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice of a batch of transforms owned by `rank` (weak scaling)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return batch * rank // world, batch * (rank + 1) // world


def unique_id() -> bytes:
    buf = (C.c_ubyte * UNIQUE_ID_BYTES)()
    _check(lib().nufft_comm_unique_id(buf))
    return bytes(buf)


class NcclComm:
    """The library's NCCL communicator on one GPU (nufft_comm)."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        if len(uid) != UNIQUE_ID_BYTES:
            raise ValueError("unique id must be 128 bytes")
        buf = (C.c_ubyte * UNIQUE_ID_BYTES).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(lib().nufft_comm_init(buf, nranks, rank, device, C.byref(h)))
        self.handle = h
        self.nranks, self.rank, self.device = nranks, rank, device

    @classmethod
    def from_process_group(cls, rank: int, world: int, device: int, group=None) -> "NcclComm":
        """Rank 0 creates the unique id; every rank receives it through `group`."""
        import torch
        import torch.distributed as dist
        backend = dist.get_backend(group)
        dev = torch.device("cuda", device) if backend == "nccl" else torch.device("cpu")
        t = torch.zeros(UNIQUE_ID_BYTES, dtype=torch.uint8, device=dev)
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(unique_id()), dtype=torch.uint8))
        dist.broadcast(t, src=0, group=group)
        return cls(bytes(t.cpu().numpy().tobytes()), world, rank, device)

    def close(self) -> None:
        if self.handle:
            lib().nufft_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def reduce_chunks_torch(buf, offsets, dst: int | None = 0, group=None):
    """Sum a bucket-order partial across ranks chunk by chunk (the chunks of
    nufft_plan2_reduce_chunks): dist.reduce to `dst`, or dist.all_reduce when
    dst is None.  In place on `buf` (a 1-D tensor)."""
    import torch.distributed as dist
    for q in range(len(offsets) - 1):
        part = buf[int(offsets[q]):int(offsets[q + 1])]
        if part.numel() == 0:
            continue
        if dst is None:
            dist.all_reduce(part, group=group)
        else:
            dist.reduce(part, dst=dst, group=group)
    return buf


def exec_rsplit_torch(plan, c, f, group=None, nchunks: int = 4, dst: int | None = 0):
    """exec_multi's algorithm with a torch.distributed collective (any backend).

    c, f: complex128 CUDA tensors of N (one vector).  Each rank computes the
    bucket-order partial over its terms, the chunks are summed with
    dist.reduce (dst) / dist.all_reduce (dst=None) — on CPU copies when the
    group's backend is not NCCL — and the receiving rank(s) un-permute into f.
    """
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    r0, r1 = term_range(plan.rank(), world, rank)
    fs = torch.empty_like(c)
    plan.execute_terms_sorted_device(c.data_ptr(), fs.data_ptr(), r0, r1,
                                     torch.cuda.current_stream(c.device).cuda_stream)
    on_gpu = dist.get_backend(group) == "nccl"
    buf = fs if on_gpu else fs.cpu()
    reduce_chunks_torch(buf, plan.reduce_chunks(nchunks), dst, group)
    if dst is None or rank == dst:
        if not on_gpu:
            fs.copy_(buf)
        plan.unpermute_device(fs.data_ptr(), f.data_ptr(), 1, torch.cuda.current_stream(c.device).cuda_stream)
    return f


__all__ = ["term_range", "batch_range", "unique_id", "NcclComm", "reduce_chunks_torch", "exec_rsplit_torch",
           "UNIQUE_ID_BYTES"]
