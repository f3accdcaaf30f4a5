"""Data parallelism across GPUs: images shard, one all-reduce.

Each rank (one process per GPU) owns a contiguous slice of the image batch
(`shard_range`) and runs the full forward and backward of those images
locally -- per-image tensors (unary, weight planes, messages, p, q, dtheta,
dw) never leave the GPU. The only exchange is one all-reduce (sum) of the
packed shared-parameter gradient `[sum_b dV_b (L*L floats), sum_b sum(dw_b)]`
(mrf_pack_shared_grads_f32), issued on the compute stream right after the
last backward kernel through the library's C-ABI collective
(mrf_allreduce_grads_f32 over an NCCL communicator built by `NcclComm`;
latency-bound: 1.8 KB at config C4). On CPU (gloo, tests) the same buffer is
all-reduced by torch.distributed.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist


def shard_range(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) slice of `batch` images for `rank`
    (the first batch % world ranks get one extra image)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


class NcclComm:
    """An NCCL communicator over the ranks of the default process group,
    created through the library (mrf_nccl_unique_id / mrf_nccl_comm_init):
    rank 0's unique id travels by torch.distributed broadcast. With one rank
    it needs no process group."""

    def __init__(self, device: torch.device, group=None):
        from . import _lib

        lib = _lib.lib()
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            _lib.check(lib.mrf_nccl_unique_id(uid.data_ptr(), 128))
        if world > 1:
            bdev = device if dist.get_backend(group) == "nccl" else torch.device("cpu")
            t = uid.to(bdev)
            dist.broadcast(t, src=0, group=group)
            uid = t.cpu()
        self.comm = C.c_void_p()
        with torch.cuda.device(device):
            _lib.check(lib.mrf_nccl_comm_init(C.byref(self.comm), world, uid.data_ptr(), rank))
        self.world, self.rank = world, rank

    def allreduce(self, buf: torch.Tensor, stream=None) -> torch.Tensor:
        """In-place sum of a float32 CUDA tensor over the communicator's ranks."""
        from . import _lib

        s = stream if stream is not None else torch.cuda.current_stream(buf.device)
        _lib.check(_lib.lib().mrf_allreduce_grads_f32(self.comm, buf.data_ptr(), buf.numel(), C.c_void_p(s.cuda_stream)))
        return buf

    def close(self):
        from . import _lib

        if self.comm:
            _lib.check(_lib.lib().mrf_nccl_comm_destroy(self.comm))
            self.comm = C.c_void_p()


def allreduce_shared(buf: torch.Tensor, comm: NcclComm | None = None, group=None) -> torch.Tensor:
    """Sum the packed shared gradient over ranks in place: through the
    library's NCCL collective when a communicator is given, else through
    torch.distributed (gloo on CPU); a no-op for one process."""
    if comm is not None:
        return comm.allreduce(buf)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


def unpack_shared(buf: torch.Tensor, labels: int):
    """(dV [L, L], total dw) from a packed shared-gradient buffer."""
    L = labels
    return buf[:L * L].view(L, L), buf[L * L]


class DataParallelStep:
    """One training step of this rank's shard of an MRF batch: forward (K
    iterations, indices kept on the device), backward for the given cost
    gradient, pack of the shared gradient, one all-reduce. Uses the C-ABI
    through api.py (bench.py's step)."""

    def __init__(self, mrf, engine: str, iterations: int, comm: NcclComm | None = None, group=None):
        from . import api

        self.api = api
        self.mrf, self.engine, self.K, self.comm, self.group = mrf, engine, iterations, comm, group
        self.fwd = api._alloc_forward(mrf, iterations)
        dev = mrf.unary.device
        t = mrf.topo
        self.grads = api.GradientSet(torch.empty_like(mrf.unary),
                                     torch.empty((mrf.batch, mrf.labels, mrf.labels), device=dev),
                                     torch.empty((mrf.batch, t.num_dirs // 2, t.nodes), device=dev))
        self.shared = torch.empty(mrf.labels * mrf.labels + 1, device=dev)

    def forward(self, mrf=None, out=None):
        f = self.api.isgmr_forward if self.engine == "isgmr" else self.api.trwp_forward
        return f(mrf or self.mrf, self.K, out=out or self.fwd)

    def backward(self, grad_cost, mrf=None, fwd=None, grads=None):
        b = self.api.isgmr_backward if self.engine == "isgmr" else self.api.trwp_backward
        m, g = mrf or self.mrf, grads or self.grads
        b(m, fwd or self.fwd, grad_cost, out=g)
        self.api.pack_shared_grads(m, g, out=self.shared)
        allreduce_shared(self.shared, self.comm, self.group)
        return g, self.shared

    def step(self, grad_cost, mrf=None, out=None, grads=None):
        f = self.forward(mrf, out)
        return self.backward(grad_cost, mrf, f, grads)
