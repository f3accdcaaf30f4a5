"""Data parallelism across GPUs: images shard, one all-reduce.

Each rank (one process per GPU, torch.distributed over NCCL; gloo on CPU for
tests) owns a contiguous slice of the image batch and runs the full forward
and backward of those images locally -- per-image tensors (unary, weight
planes, messages, p, q, dtheta, dw) never leave the GPU. The only exchange is
one all-reduce (sum) of the packed shared-parameter gradient
`[sum_b dV_b (L*L floats), sum_b sum(dw_b)]`, issued on the compute stream
right after the last backward kernel (latency-bound: 1.8 KB at config C4).
"""
from __future__ import annotations

import os

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


def env_rank_world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def allreduce_shared(buf: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the packed shared gradient over ranks in place (no-op for one rank)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


def unpack_shared(buf: torch.Tensor, labels: int):
    """(dV [L, L], total dw) from a packed shared-gradient buffer."""
    L = labels
    return buf[:L * L].view(L, L), buf[L * L]


class DataParallelStep:
    """One training step of a sharded MRF batch: forward (K iterations,
    indices kept on the device), backward for the given cost gradient, pack
    of the shared gradient, one all-reduce. Uses the C-ABI through api.py."""

    def __init__(self, mrf, engine: str, iterations: int, group=None):
        from . import api

        self.api = api
        self.mrf, self.engine, self.K, self.group = mrf, engine, iterations, group
        self.fwd = api._alloc_forward(mrf, iterations)
        dev = mrf.unary.device
        t = mrf.topo
        self.grads = api.GradientSet(torch.empty_like(mrf.unary),
                                     torch.empty((mrf.batch, mrf.labels, mrf.labels), device=dev),
                                     torch.empty((mrf.batch, t.num_dirs // 2, t.nodes), device=dev))
        self.shared = torch.empty(mrf.labels * mrf.labels + 1, device=dev)

    def forward(self):
        f = self.api.isgmr_forward if self.engine == "isgmr" else self.api.trwp_forward
        return f(self.mrf, self.K, out=self.fwd)

    def backward(self, grad_cost):
        b = self.api.isgmr_backward if self.engine == "isgmr" else self.api.trwp_backward
        b(self.mrf, self.fwd, grad_cost, out=self.grads)
        self.api.pack_shared_grads(self.mrf, self.grads, out=self.shared)
        allreduce_shared(self.shared, self.group)
        return self.grads, self.shared
