"""The grouped small-L TRWP-4 forward (fwd_grp.cuh: 8 lanes x 3 labels per
scanline, 4 scanlines per warp; the kernel for 16 < L <= 24, C4's) against
the reference restatement, bit for bit, next to the lane-per-label kernel it
replaces (MRF_FWD_GRP=0). Shapes with a scanline count that is not a multiple
of 4 (partly filled warps), L = 17 / 21 / 24 (one, three and no padding
labels per line), constant and per-edge weights, rho planes, and the cost /
labels aggregation fused into the last sweep."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1910_10892_b200 import workloads as WL

from tests.gpu_util import assert_forward_equal, gpu_forward, to_mrf

CASES = [
    # H, W, L, K, per-edge w, rho planes
    (9, 11, 21, 3, True, False),
    (13, 6, 17, 2, False, False),
    (7, 10, 24, 3, True, True),
    (1, 12, 21, 2, False, True),
    (6, 1, 19, 2, True, False),
    (23, 18, 21, 5, True, True),
]


@pytest.mark.gpu
@pytest.mark.parametrize("grp", ["1", "0"], ids=["grouped", "lane_per_label"])
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}L{c[2]}K{c[3]}{'w' if c[4] else ''}{'r' if c[5] else ''}" for c in CASES])
def test_grouped_small_forward_bit_exact(case, grp, monkeypatch):
    monkeypatch.setenv("MRF_FWD_GRP", grp)
    H, W, L, K, per_edge, rho_pl = case
    un, V, wc, planes = WL.random_problem(H, W, L, 4, seed=H * 31 + W + L, per_edge=per_edge)
    rho = np.random.default_rng(L).uniform(0.2, 1.0, 2 * H * W).astype(np.float32) if rho_pl else None
    pr = O.Problem(H, W, L, 4, un, V, wc, planes, 0.5, rho)
    ref = O.forward("trwp", pr, K)
    f = gpu_forward("trwp", to_mrf(pr), K)
    assert_forward_equal(f, ref)


@pytest.mark.gpu
def test_grouped_small_forward_batch_seg():
    """C4's recipe (seg_batch: -logits, explicit V, 0/1 edge weights) at 6
    images of 40 x 36: every image equal to its own reference run."""
    H, W, L, K, B = 40, 36, 21, 3, 6
    wl = WL.seg_batch(H, W, L, B, K=K, first=5)
    prs = [O.Problem(H, W, L, 4, wl.unary[b], wl.V, 1.0, wl.w_planes[b], 0.5, None) for b in range(B)]
    f = gpu_forward("trwp", to_mrf(prs[0], batch_unary=list(wl.unary), batch_wplanes=list(wl.w_planes)), K)
    for b in range(B):
        assert_forward_equal(f, O.forward("trwp", prs[b], K), b=b)


BWD_CASES = [
    # H, W, L, K, per-edge w, batch
    (9, 11, 21, 3, True, 3),
    (13, 6, 17, 2, False, 2),
    (7, 10, 24, 3, True, 2),
    (1, 12, 21, 2, False, 1),
    (23, 18, 21, 4, True, 2),
]


@pytest.mark.gpu
@pytest.mark.parametrize("grp", ["1", "1u", "0"], ids=["grouped_fused", "grouped", "lane_per_label"])
@pytest.mark.parametrize("case", BWD_CASES, ids=[f"{c[0]}x{c[1]}L{c[2]}K{c[3]}B{c[5]}{'w' if c[4] else ''}" for c in BWD_CASES])
def test_grouped_small_backward(case, grp, monkeypatch):
    """The grouped small-L TRWP-4 backward (bwd_grp.cuh), with the unary
    gradient collected in its direction-0 sweep (default) or by
    dtheta_acc_kernel (MRF_GRP_FUSE=0), against the reference restatement
    within 1e-5 (normwise and elementwise), and bit-identical run to run;
    MRF_BWD_SMALL=1 puts these few-line launches on the small-L kernels,
    MRF_BWD_GRP=0 on the lane-per-label one it replaces."""
    import torch
    from tests.gpu_util import assert_grads_close, gpu_backward
    monkeypatch.setenv("MRF_BWD_SMALL", "1")
    monkeypatch.setenv("MRF_BWD_GRP", grp[0])
    monkeypatch.setenv("MRF_GRP_FUSE", "0" if grp == "1u" else "1")
    H, W, L, K, per_edge, B = case
    uns, pls, prs = [], [], []
    V = wc0 = None
    for b in range(B):  # V and a constant weight are shared by the batch
        un, V0, wc, planes = WL.random_problem(H, W, L, 4, seed=H * 7 + W + L + b, per_edge=per_edge)
        V = V0 if V is None else V
        wc0 = wc if wc0 is None else wc0
        uns.append(un)
        pls.append(planes)
        prs.append(O.Problem(H, W, L, 4, un, V, wc0, planes, 0.5, None))
    mrf = to_mrf(prs[0], batch_unary=uns, batch_wplanes=pls if per_edge else None)
    f = gpu_forward("trwp", mrf, K)
    gcs = np.random.default_rng(L + K).normal(size=(B, H * W * L)).astype(np.float32)
    g = gpu_backward("trwp", mrf, f, gcs)
    for b in range(B):
        ref = O.forward("trwp", prs[b], K)
        assert_forward_equal(f, ref, b=b)
        assert_grads_close(g, O.backward("trwp", prs[b], K, ref.p, ref.q, gcs[b]), b=b)
    g2 = gpu_backward("trwp", mrf, f, gcs)
    assert torch.equal(g.pairwise, g2.pairwise) and torch.equal(g.unary, g2.unary)
    if g.edge_weights is not None:
        assert torch.equal(g.edge_weights, g2.edge_weights)
