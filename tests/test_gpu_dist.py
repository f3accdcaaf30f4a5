"""The data-parallel path on one GPU: the library's NCCL collective
(mrf_allreduce_grads_f32) on a 1-rank communicator created through the C-ABI
(mrf_nccl_unique_id / mrf_nccl_comm_init), and DataParallelStep (bench.py's
step) against per-image device gradients."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1910_10892_b200 import api
from paper_1910_10892_b200 import workloads as WL
from paper_1910_10892_b200.dist import DataParallelStep, NcclComm, unpack_shared
from tests.gpu_util import to_mrf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = NcclComm(torch.device("cuda", 0))
    yield c
    c.close()


def test_allreduce_one_rank_is_identity(comm):
    x = torch.randn(441 + 1, device="cuda")
    y = x.clone()
    comm.allreduce(y)
    torch.cuda.synchronize()
    assert comm.world == 1 and torch.equal(x, y)


def test_data_parallel_step_packs_and_reduces(comm):
    """C4-shaped shard (explicit V, per-edge weights, TRWP): the all-reduced
    shared gradient equals the sum over images of the device dV and dw, and
    each image's dV matches the reference."""
    H, W, L, K = 16, 12, 21, 3
    wl = WL.seg_batch(H, W, L, 3, K=K, first=5)
    pr0 = O.Problem(H, W, L, 4, wl.unary[0], wl.V, 1.0, wl.w_planes[0], 0.5, None)
    mrf = to_mrf(pr0, batch_unary=list(wl.unary), batch_wplanes=list(wl.w_planes))
    dp = DataParallelStep(mrf, "trwp", K, comm=comm)
    gc = torch.randn_like(mrf.unary)
    grads, shared = dp.step(gc)
    torch.cuda.synchronize()
    dv, dw = unpack_shared(shared, L)
    want_dv = grads.pairwise.double().sum(0)
    assert torch.allclose(dv.double(), want_dv, rtol=1e-5, atol=1e-6)
    assert abs(dw.item() - grads.edge_weights.double().sum().item()) <= 1e-4 * max(1.0, abs(dw.item()))
    for b in range(wl.B):
        pr = O.Problem(H, W, L, 4, wl.unary[b], wl.V, 1.0, wl.w_planes[b], 0.5, None)
        ref = O.forward("trwp", pr, K)
        gref = O.backward("trwp", pr, K, ref.p, ref.q, gc[b].cpu().numpy().reshape(-1))
        got = grads.pairwise[b].cpu().numpy().reshape(-1)
        assert np.linalg.norm(got - gref.pairwise) <= 1e-5 * np.linalg.norm(gref.pairwise)
