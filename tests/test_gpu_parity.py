"""GPU parity: libmrf_cuda.so (through the C-ABI) against the CPU checkers.

Forward outputs (messages, cost, labels, p, q) must be bit-identical to the
reference; gradients within GRAD_RTOL (1e-5, normwise) of the reference's
float backward. Mirrors the reference's bit-identity tests
(test_isgmr.cpp:84-96, test_trwp.cpp:73-86, test_autodiff.cpp:86-110) with
"GPU == CPU reference" in place of "1 thread == N threads".
"""
import glob
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1910_10892_b200 import api
from paper_1910_10892_b200 import workloads as WL
from tests.gpu_util import (assert_forward_equal, assert_grads_close, gpu_backward, gpu_forward, to_mrf)

pytestmark = pytest.mark.gpu

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_golden_fixtures(path):
    from tests.golden.make_golden import load

    eng, pr, K, z = load(path)
    mrf = to_mrf(pr)
    f = gpu_forward(eng, mrf, K)
    assert_forward_equal(f, {k: z[k] for k in ("cost", "labels", "messages", "p", "q")})
    g = gpu_backward(eng, mrf, f, z["grad_cost"])
    assert_grads_close(g, {k: z[k] for k in ("g_unary", "g_pairwise", "g_wplanes")})


CASES = [
    # H, W, L, conn, K, per_edge, explicit
    (7, 9, 5, 4, 3, True, True),
    (7, 9, 5, 8, 3, True, True),
    (6, 6, 4, 16, 2, False, True),
    (13, 11, 16, 4, 2, False, False),
    (9, 14, 21, 8, 2, True, True),
    (3, 17, 1, 4, 3, False, True),
    (1, 12, 5, 4, 1, False, True),
    (1, 12, 16, 4, 2, False, False),  # banded TRWP-4 on one row: no vertical line to fuse into
    (2, 9, 24, 4, 2, False, False),
    (12, 1, 7, 8, 2, True, False),
    (10, 12, 32, 4, 2, False, True),
    (8, 9, 33, 4, 2, True, True),
    (6, 10, 64, 8, 2, False, False),
    (5, 7, 128, 4, 2, True, True),
    (6, 5, 192, 4, 2, False, False),
    (4, 6, 256, 4, 2, False, False),
    (4, 5, 256, 8, 1, True, True),
]


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}L{c[2]}c{c[3]}" for c in CASES])
def test_random_problems_bit_exact(engine, case):
    H, W, L, conn, K, per_edge, explicit = case
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=H * 1000 + W * 10 + L, per_edge=per_edge,
                                          explicit=explicit)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    ref = O.forward(engine, pr, K)
    mrf = to_mrf(pr)
    f = gpu_forward(engine, mrf, K)
    assert_forward_equal(f, ref)
    rng = np.random.default_rng(L)
    _, _, gc = O.soft_head(ref.cost, rng.uniform(0.25, max(L - 1.25, 0.3), H * W), L)
    gref = O.backward(engine, pr, K, ref.p, ref.q, gc)
    g = gpu_backward(engine, mrf, f, gc)
    assert_grads_close(g, gref)


WIDE = [
    # H, W, L, conn, K, pairwise (kind, param), per_edge
    (9, 11, 16, 4, 2, ("tl", 3.0), False),
    (7, 13, 64, 8, 2, ("tl", 6.0), True),
    (8, 7, 100, 4, 2, ("tq", 40.0), False),
    (6, 9, 192, 4, 2, ("tl", 15.0), False),
    (5, 6, 256, 4, 3, ("tq", 200.0), False),
    (10, 8, 21, 8, 2, ("tq", 9.0), True),
    (7, 7, 33, 4, 2, ("tl", 16.0), False),
    (6, 8, 40, 4, 2, ("tl", 17.0), False),   # D = 17 > 16: generic banded path
    (6, 8, 12, 4, 2, ("potts", 1.0), False),  # D = 1
]


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
@pytest.mark.parametrize("case", WIDE, ids=[f"{c[5][0]}{c[5][1]:g}L{c[2]}c{c[3]}" for c in WIDE])
def test_wide_band_bit_exact(engine, case):
    """Banded V with D != 2 (truncated linear / quadratic, Potts): the
    wide-band forward (2 < D <= 16) and the generic banded path."""
    H, W, L, conn, K, (kind, prm), per_edge = case
    un, _, wc, planes = WL.random_problem(H, W, L, conn, seed=H * 7 + L, per_edge=per_edge)
    V = {"tl": WL.truncated_linear, "tq": WL.truncated_quadratic}[kind](L, prm) if kind != "potts" else WL.potts(L)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    ref = O.forward(engine, pr, K)
    mrf = to_mrf(pr)
    f = gpu_forward(engine, mrf, K)
    assert_forward_equal(f, ref)
    _, _, gc = O.soft_head(ref.cost, np.random.default_rng(L).uniform(0.25, L - 1.25, H * W), L)
    g = gpu_backward(engine, mrf, f, gc)
    assert_grads_close(g, O.backward(engine, pr, K, ref.p, ref.q, gc))


def test_c5_shaped_integer_ties():
    """C5 recipe (integer TQ denoising, V = min(d^2, 200), w = 25: exact
    arithmetic, maximal ties) on a small grid, both engines."""
    H, W, L = 24, 20, 256
    un = WL.denoise_tq(H, W, L, seed=5)
    V = WL.truncated_quadratic(L, 200.0)
    for engine in ("isgmr", "trwp"):
        pr = O.Problem(H, W, L, 4, un, V, 25.0, None, 0.5, None)
        ref = O.forward(engine, pr, 3)
        f = gpu_forward(engine, to_mrf(pr), 3)
        assert_forward_equal(f, ref)


SMALL_TIES = [
    # H, W, L, conn, K, kind
    (9, 11, 21, 4, 3, "int"),
    (8, 7, 32, 8, 2, "int"),
    (10, 9, 5, 4, 3, "int"),
    (9, 11, 21, 4, 2, "tiny"),
    (7, 8, 16, 4, 2, "huge"),
]


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
@pytest.mark.parametrize("case", SMALL_TIES, ids=[f"{c[5]}L{c[2]}c{c[3]}" for c in SMALL_TIES])
def test_small_label_ties_zeros_and_extremes(engine, case):
    """The dense small-L forward finds the reference's first strict-'<' winner
    as the first candidate equal to the minimum, keyed, for finite |min| >=
    2^-60, and falls back to the scan as written for +-0, tiny and infinite
    minima (fwd_small.cuh). Integer data (-0 unaries, zero V diagonal, integer
    weights: exact ties and exact zeros everywhere), values around 2^-60..2^-90
    and mixed 1e37 / O(1) magnitudes (key differences overflow to +inf) drive
    every branch."""
    H, W, L, conn, K, kind = case
    rng = np.random.default_rng(L * 7 + conn)
    n = H * W * L
    if kind == "int":
        un = -rng.integers(-2, 3, n).astype(np.float32)  # -logits: -0 where the logit is 0
        V = rng.integers(0, 3, (L, L)).astype(np.float32)
        np.fill_diagonal(V, 0.0)
        planes = rng.integers(0, 3, (conn // 2) * H * W).astype(np.float32)
    elif kind == "tiny":
        un = (rng.integers(0, 4, n) * 2.0 ** -88).astype(np.float32) * rng.choice([1, -1], n).astype(np.float32)
        V = (rng.integers(0, 3, (L, L)) * 2.0 ** -89).astype(np.float32)
        np.fill_diagonal(V, 0.0)
        planes = rng.choice([0.5, 1.0, 2.0], (conn // 2) * H * W).astype(np.float32)
    else:
        un = rng.choice([1e37, 0.0, 3.0, -1e37], n).astype(np.float32)
        V = rng.choice([0.0, 1e37, 1.0], (L, L)).astype(np.float32)
        planes = rng.choice([1.0, 3.0], (conn // 2) * H * W).astype(np.float32)
    pr = O.Problem(H, W, L, conn, un, V.reshape(-1), 1.0, planes, 0.5, None)
    ref = O.forward(engine, pr, K)
    f = gpu_forward(engine, to_mrf(pr), K)
    assert_forward_equal(f, ref)


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
@pytest.mark.parametrize("shape", [(11, 9, 21, 4, 2, 3), (7, 10, 21, 4, 3, 2), (7, 10, 5, 8, 3, 3),
                                   (7, 10, 192, 4, 3, 2), (5, 8, 30, 4, 1, 3)],
                         ids=["11x9L21K2", "7x10L21K3", "7x10L5c8K3", "7x10L192K3", "5x8L30K1"])
def test_batch_images_independent(engine, shape):
    """Images of a batch are independent. The odd-K / odd-(H+W) shapes put
    image b >= 1's p and q rows at byte offsets that are not word aligned
    (K*E % 4 != 0, K*E*L % 4 != 0)."""
    H, W, L, conn, K, B = shape
    uns, pls, rhos, refs = [], [], [], []
    V = None
    for b in range(B):
        un, V0, wc, planes = WL.random_problem(H, W, L, conn, seed=50 + b, per_edge=True)
        V = V0 if V is None else V
        rho = np.random.default_rng(b).uniform(0.2, 1.0, (conn // 2) * H * W).astype(np.float32)
        uns.append(un)
        pls.append(planes)
        rhos.append(rho)
        refs.append(O.Problem(H, W, L, conn, un, V, 1.0, planes, 0.5, rho))
    mrf = to_mrf(refs[0], batch_unary=uns, batch_wplanes=pls, batch_rho=rhos if engine == "trwp" else None)
    f = gpu_forward(engine, mrf, K)
    gcs = np.random.default_rng(9).normal(size=(B, H * W * L)).astype(np.float32)
    g = gpu_backward(engine, mrf, f, gcs)
    for b in range(B):
        pr = refs[b] if engine == "trwp" else O.Problem(H, W, L, conn, uns[b], V, 1.0, pls[b], 0.5, None)
        ref = O.forward(engine, pr, K)
        assert_forward_equal(f, ref, b=b)
        gref = O.backward(engine, pr, K, ref.p, ref.q, gcs[b])
        assert_grads_close(g, gref, b=b)
    # shared-parameter pack: sum over the batch of dV, and the total dw
    packed = api.pack_shared_grads(mrf, g).cpu().numpy()
    want = g.pairwise.sum(0).reshape(-1).cpu().numpy()
    assert np.allclose(packed[:-1], want, rtol=1e-5, atol=1e-6)
    assert np.isclose(packed[-1], g.edge_weights.sum().item(), rtol=1e-4)


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
def test_engine_step_api_matches_forward(engine):
    H, W, L, conn, K = 9, 10, 8, 8, 3
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=77)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    mrf = to_mrf(pr)
    eng = (api.IsgmrEngine if engine == "isgmr" else api.TrwpEngine)(mrf, K)
    ref_msgs = []
    for k in range(K):
        eng.step()
        ref_msgs.append(O.forward(engine, pr, k + 1))
        cost, labels = eng.aggregate()
        torch.cuda.synchronize()
        assert np.array_equal(bits_(eng.messages()[0]), bits_(ref_msgs[-1].messages))
        assert np.array_equal(bits_(cost[0]), bits_(ref_msgs[-1].cost))
        assert np.array_equal(labels[0].cpu().numpy().view(np.uint16), ref_msgs[-1].labels)
    assert np.array_equal(eng.p[0].cpu().numpy().reshape(-1), ref_msgs[-1].p)
    assert np.array_equal(eng.q[0].cpu().numpy().reshape(-1), ref_msgs[-1].q)


def bits_(t):
    a = t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
    return np.ascontiguousarray(a).reshape(-1).view(np.uint8)


def test_zero_cost_gradient_gives_zero_gradients():
    """test_autodiff.cpp:44-54."""
    H, W, L, conn, K = 6, 6, 4, 4, 2
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=1, per_edge=True)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    mrf = to_mrf(pr)
    for engine in ("isgmr", "trwp"):
        f = gpu_forward(engine, mrf, K)
        g = gpu_backward(engine, mrf, f, np.zeros(H * W * L, np.float32))
        assert not g.unary.any() and not g.pairwise.any() and not g.edge_weights.any()


@pytest.mark.parametrize("case", [(12, 13, 16, 8, 2, True, True), (9, 11, 192, 4, 3, False, False),
                                  (10, 9, 21, 4, 2, True, True), (8, 10, 100, 4, 2, False, True),
                                  (7, 9, 256, 4, 2, False, False)],
                         ids=["L16c8", "L192band", "L21small", "L100dense", "L256band"])
def test_backward_deterministic_run_to_run(case):
    """test_autodiff.cpp:86-110 analogue: every gradient, dV included, is
    bit-identical run to run (dV: private per-CTA slots reduced in a fixed
    order)."""
    H, W, L, conn, K, per_edge, explicit = case
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=5, per_edge=per_edge, explicit=explicit)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    mrf = to_mrf(pr)
    gc = np.random.default_rng(3).normal(size=H * W * L).astype(np.float32)
    for engine in ("isgmr", "trwp"):
        f = gpu_forward(engine, mrf, K)
        a = gpu_backward(engine, mrf, f, gc)
        for _ in range(3):
            b = gpu_backward(engine, mrf, f, gc)
            assert torch.equal(a.unary, b.unary)
            assert torch.equal(a.edge_weights, b.edge_weights)
            assert torch.equal(a.pairwise, b.pairwise)


def test_invalid_arguments_raise():
    H, W, L, conn = 4, 4, 3, 4
    un, V, wc, _ = WL.random_problem(H, W, L, conn, seed=2)
    mrf = to_mrf(O.Problem(H, W, L, conn, un, V, wc, None, 0.5, None))
    with pytest.raises(ValueError):
        api.isgmr_forward(mrf, 0)
    bad = api.MRF(mrf.topo, mrf.unary, mrf.V, 1.0, 1.5)
    with pytest.raises(ValueError):
        api.trwp_forward(bad, 1)
    x = mrf.unary.clone()
    assert api.check_finite(x)
    x[0, 3, 1] = float("inf")
    assert not api.check_finite(x)


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
def test_c1_full_size_matches_reference(engine):
    """Config C1 (288x384, L=16, 4 dirs, K=5, TL tau=2) at full size against
    the reference library itself (oracle/_ref, all host threads)."""
    if not O.have_ref():
        pytest.skip("reference library not present")
    wl = WL.config("C1")
    pr = O.Problem(wl.H, wl.W, wl.L, wl.conn, wl.unary[0], wl.V, wl.w_const, None, 0.5, None)
    ref = O.forward(engine, pr, wl.K, impl="ref", threads=0)
    mrf = to_mrf(pr)
    f = gpu_forward(engine, mrf, wl.K)
    assert_forward_equal(f, ref)
    gc = np.full(wl.N * wl.L, 1.0 / (wl.N * wl.L), np.float32)
    gref = O.backward(engine, pr, wl.K, ref.p, ref.q, gc, impl="ref", threads=0)
    g = gpu_backward(engine, mrf, f, gc)
    assert_grads_close(g, gref)


@pytest.mark.parametrize("stages", ["3", "4"])
@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
@pytest.mark.parametrize("case", [(6, 9, 192, 4, 3, True), (5, 7, 150, 8, 2, False), (4, 6, 256, 4, 2, False),
                                  (7, 5, 100, 4, 2, True)], ids=["L192c4", "L150c8", "L256c4", "L100c4"])
def test_band2_ring_depths_bit_exact(case, engine, stages, monkeypatch):
    """The banded D == 2 forward at both cp.async ring depths (the launcher
    picks 3 only for launches with many long lines; forced here)."""
    monkeypatch.setenv("MRF_BAND2_STAGES", stages)
    H, W, L, conn, K, per_edge = case
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=L + H, per_edge=per_edge, explicit=False)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    ref = O.forward(engine, pr, K)
    assert_forward_equal(gpu_forward(engine, to_mrf(pr), K), ref)


GAP_CASES = [(7, 9, 5, 4, 3, True, True), (6, 8, 40, 8, 2, False, False), (5, 6, 192, 4, 2, False, False),
             (9, 7, 21, 4, 2, True, True), (4, 5, 256, 8, 1, False, True), (1, 9, 3, 4, 2, False, True)]


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
@pytest.mark.parametrize("case", GAP_CASES, ids=[f"{c[0]}x{c[1]}L{c[2]}c{c[3]}" for c in GAP_CASES])
def test_diagnostic_min_argmin_gap_matches_reference(engine, case):
    """Diagnostic mode (mrf_problem_f32::diag_gap): min_argmin_gap equals the
    reference's ForwardResult::min_argmin_gap (isgmr.hpp:64-68,109-129,
    trwp.hpp:57-59), and messages / indices stay bit-identical."""
    if not O.have_ref():
        pytest.skip("reference library not present")
    H, W, L, conn, K, per_edge, explicit = case
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=H * 31 + L, per_edge=per_edge, explicit=explicit)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    ref = O.forward(engine, pr, K, impl="ref", threads=1)
    mrf = to_mrf(pr)
    f = (api.isgmr_forward if engine == "isgmr" else api.trwp_forward)(mrf, K, diagnostic=True)
    torch.cuda.synchronize()
    assert_forward_equal(f, ref)
    assert f.min_argmin_gap[0].item() == ref.gap
    eng = (api.IsgmrEngine if engine == "isgmr" else api.TrwpEngine)(mrf, 1, diagnostic=True)
    for _ in range(K):
        eng.step()
    assert eng.min_argmin_gap()[0].item() == ref.gap


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
def test_engine_index_store_grows(engine):
    """step() past the initial capacity regrows the device index store (the
    reference's append_iteration); indices of every iteration survive."""
    H, W, L, conn, K = 6, 7, 16, 4, 5
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=8, explicit=False)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    ref = O.forward(engine, pr, K)
    eng = (api.IsgmrEngine if engine == "isgmr" else api.TrwpEngine)(to_mrf(pr), 1)
    for _ in range(K):
        eng.step()
    p, q = eng.indices()
    assert eng.iterations() == K
    assert np.array_equal(p[0].cpu().numpy().reshape(-1), ref.p)
    assert np.array_equal(q[0].cpu().numpy().reshape(-1), ref.q)
    assert np.array_equal(bits_(eng.messages()[0]), bits_(ref.messages))


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
def test_non_finite_unary_rejected_at_the_c_abi(engine):
    """The forward entry points reject NaN / Inf unaries with MRF_EINVAL (the
    reference engines throw std::invalid_argument, isgmr.hpp:32-35,
    trwp.hpp:33-36); engines reject them at construction."""
    H, W, L, conn = 5, 6, 7, 4
    un, V, wc, _ = WL.random_problem(H, W, L, conn, seed=3)
    for bad in (float("nan"), float("inf"), float("-inf")):
        x = un.copy()
        x[17] = bad
        mrf = to_mrf(O.Problem(H, W, L, conn, x, V, wc, None, 0.5, None))
        fwd = api.isgmr_forward if engine == "isgmr" else api.trwp_forward
        with pytest.raises(ValueError, match="non-finite"):
            fwd(mrf, 2)
        with pytest.raises(ValueError, match="non-finite"):
            (api.IsgmrEngine if engine == "isgmr" else api.TrwpEngine)(mrf, 2)
        mrf.assume_finite = True  # caller's promise: no scan, no error
        fwd(mrf, 1)
        torch.cuda.synchronize()



@pytest.mark.parametrize("mode", ["split", "warp"])
@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
@pytest.mark.parametrize("case", [(9, 14, 192, 4, 3, False), (8, 11, 128, 8, 2, True), (10, 13, 16, 4, 3, False),
                                  (7, 9, 100, 4, 2, True), (1, 20, 64, 4, 2, False)],
                         ids=["L192c4", "L128c8", "L16c4", "L100c4", "1x20L64"])
def test_banded_backward_both_kernels(case, engine, mode, monkeypatch):
    """Banded D <= 2 backward through both kernels (the launcher picks one
    warp per line for launches with many lines, the warp-specialised split
    kernel otherwise; forced here), against the reference restatement."""
    monkeypatch.setenv("MRF_BWD_BAND", mode)
    H, W, L, conn, K, per_edge = case
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=L * 3 + H, per_edge=per_edge, explicit=False)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    ref = O.forward(engine, pr, K)
    mrf = to_mrf(pr)
    f = gpu_forward(engine, mrf, K)
    assert_forward_equal(f, ref)
    _, _, gc = O.soft_head(ref.cost, np.random.default_rng(L).uniform(0.25, L - 1.25, H * W), L)
    g = gpu_backward(engine, mrf, f, gc)
    assert_grads_close(g, O.backward(engine, pr, K, ref.p, ref.q, gc))
    g2 = gpu_backward(engine, mrf, f, gc)
    assert torch.equal(g.pairwise, g2.pairwise) and torch.equal(g.unary, g2.unary)


@pytest.mark.parametrize("kernel", [("0",), ("1",)], ids=["small", "small_fused"])
@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
def test_small_label_backward_many_lines(engine, kernel, monkeypatch):
    """The one-warp-per-line small-L backward (bwd_small.cuh: C4's kernel,
    picked for L <= 32 with >= 2368 lines per launch): 30 images of 80 x 80,
    explicit 21 x 21 V, per-edge weights, each image against the reference
    restatement; with and without the fused unary-gradient sweep."""
    monkeypatch.setenv("MRF_SMALL_FUSE", kernel[0])
    H, W, L, conn, K, B = 80, 80, 21, 4, 2, 30
    wl = WL.seg_batch(H, W, L, B, K=K, first=3)
    prs = [O.Problem(H, W, L, conn, wl.unary[b], wl.V, 1.0, wl.w_planes[b], 0.5, None) for b in range(B)]
    mrf = to_mrf(prs[0], batch_unary=list(wl.unary), batch_wplanes=list(wl.w_planes))
    f = gpu_forward(engine, mrf, K)
    gcs = np.random.default_rng(4).normal(size=(B, H * W * L)).astype(np.float32)
    g = gpu_backward(engine, mrf, f, gcs)
    for b in range(0, B, 7):
        ref = O.forward(engine, prs[b], K)
        assert_forward_equal(f, ref, b=b)
        assert_grads_close(g, O.backward(engine, prs[b], K, ref.p, ref.q, gcs[b]), b=b)
    g2 = gpu_backward(engine, mrf, f, gcs)
    assert torch.equal(g.pairwise, g2.pairwise) and torch.equal(g.unary, g2.unary)
