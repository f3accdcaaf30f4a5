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
