"""GPU parity of the readout / evaluation callers of the path (SURVEY.md §8f
ranks 1-2): the fused soft head (softhead.hpp:22-74) and the energy of a
labelling (potentials.hpp:175-199), against the C restatement and the
reference library itself (oracle/_ref)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1910_10892_b200 import api
from paper_1910_10892_b200 import workloads as WL
from tests.gpu_util import gpu_forward, normwise, to_mrf

pytestmark = pytest.mark.gpu

RTOL = 1e-5  # north_star: FP32 results within 1e-5 relative


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("N,L", [(1, 1), (37, 5), (200, 16), (96, 33), (64, 192), (17, 256)])
def test_soft_head_matches_reference(N, L):
    rng = np.random.default_rng(N * 7 + L)
    cost = rng.uniform(-3.0, 20.0, N * L).astype(np.float32)
    target = rng.uniform(0.0, L - 1, N).astype(np.float32)
    target[::7] = 0.0
    impls = ["oracle"] + (["ref"] if O.have_ref() else [])
    r = api.soft_head(torch.from_numpy(cost).cuda().view(1, N, L), torch.from_numpy(target).cuda().view(1, N),
                      confidence=True)
    disp, grad = r.disparity[0].cpu().numpy(), r.grad_cost[0].cpu().numpy().reshape(-1)
    conf = r.confidence[0].cpu().numpy()
    assert np.allclose(conf.sum(-1), 1.0, rtol=1e-5)
    for impl in impls:
        loss, d_ref, g_ref = O.soft_head(cost, target, L, impl=impl)
        np.testing.assert_allclose(disp, d_ref, rtol=RTOL, atol=1e-5 * L)
        assert abs(r.loss[0].item() - loss) <= RTOL * max(abs(loss), 1e-3)
        assert normwise(grad, g_ref) <= RTOL


def test_soft_head_batch_and_ties():
    """Exact ties (disparity == target) give zero gradient rows; images of a
    batch are independent."""
    B, N, L = 3, 40, 8
    rng = np.random.default_rng(3)
    cost = rng.uniform(0.0, 5.0, (B, N, L)).astype(np.float32)
    cost[:, 0] = 1.0  # uniform row: disparity (L-1)/2 exactly
    target = rng.uniform(0.0, L - 1, (B, N)).astype(np.float32)
    target[:, 0] = (L - 1) / 2
    r = api.soft_head(torch.from_numpy(cost).cuda(), torch.from_numpy(target).cuda())
    g = r.grad_cost.cpu().numpy()
    for b in range(B):
        loss, d_ref, g_ref = O.soft_head(cost[b].reshape(-1), target[b], L)
        assert normwise(g[b], g_ref) <= RTOL
        assert not g[b, 0].any()
        assert abs(r.loss[b].item() - loss) <= RTOL * abs(loss)


def _numpy_energy(H, W, L, conn, un, V, wc, planes, lab):
    """potentials.hpp:175-199 in numpy (double), edges via the even directions."""
    steps = [(0, 1), (1, 0), (1, 1), (1, -1), (1, 2), (1, -2), (2, 1), (2, -1)][: conn // 2]
    un = un.reshape(H * W, L)
    V = V.reshape(L, L)
    e = float(np.sum(un[np.arange(H * W), lab].astype(np.float64)))
    for f, (dh, dw) in enumerate(steps):
        for h in range(H):
            for w in range(W):
                h2, w2 = h + dh, w + dw
                if 0 <= h2 < H and 0 <= w2 < W:
                    n, m = h * W + w, h2 * W + w2
                    we = planes.reshape(conn // 2, H * W)[f, n] if planes is not None else wc
                    e += float(np.float64(we) * np.float64(V[lab[n], lab[m]]))
    return e


@pytest.mark.parametrize("conn,per_edge", [(4, False), (8, True), (16, False)])
def test_energy_matches_reference(conn, per_edge):
    H, W, L = 9, 11, 7
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=conn, per_edge=per_edge)
    lab = np.random.default_rng(conn).integers(0, L, H * W).astype(np.uint16)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    mrf = to_mrf(pr)
    e = api.energy(mrf, torch.from_numpy(lab.view(np.int16)).cuda())[0]
    want = O.ref_energy(pr, lab) if O.have_ref() else _numpy_energy(H, W, L, conn, un, V, wc, planes, lab)
    assert abs(e - want) <= 1e-9 * max(1.0, abs(want))
    assert abs(e - _numpy_energy(H, W, L, conn, un, V, wc, planes, lab)) <= 1e-9 * max(1.0, abs(want))


def test_energy_rejects_out_of_range_label():
    H, W, L = 4, 5, 3
    un, V, wc, _ = WL.random_problem(H, W, L, 4, seed=1)
    mrf = to_mrf(O.Problem(H, W, L, 4, un, V, wc, None, 0.5, None))
    lab = torch.zeros(1, H * W, dtype=torch.int16, device="cuda")
    lab[0, 7] = L
    with pytest.raises(ValueError):
        api.energy(mrf, lab)


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
def test_iterate_energy_on_4_connected_protocol(engine):
    """isgmr/trwp_iterate_energy with an 8-connected problem evaluated on the
    4-connected edge set (mrfmp.cpp:91-94): per iteration, the energy of the
    reference forward's labels."""
    H, W, L, K = 8, 9, 6, 3
    un, V, wc, _ = WL.random_problem(H, W, L, 8, seed=21)
    pr = O.Problem(H, W, L, 8, un, V, wc, None, 0.5, None)
    mrf = to_mrf(pr)
    t4 = api.GridTopology(H, W, 4)
    es = api.iterate_energy(engine, mrf, K, eval_topo=t4)
    for k in range(K):
        ref = O.forward(engine, pr, k + 1)
        want = _numpy_energy(H, W, L, 4, un, V, wc, None, ref.labels.astype(np.int64))
        assert abs(es[k][0] - want) <= 1e-9 * max(1.0, abs(want))


SGM_CASES = [(6, 7, 5, 4, False, True), (9, 8, 16, 8, True, True), (7, 9, 21, 4, True, False), (5, 6, 40, 4, False, False)]


@pytest.mark.parametrize("H,W,L,conn,per_edge,explicit", SGM_CASES)
def test_sgm_matches_reference(H, W, L, conn, per_edge, explicit):
    """mp::sgm_forward (baselines.hpp:31-98): standard bit-exact against the
    reference library; revised == one ISGMR iteration (test_baselines.cpp:58-68)."""
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=H * W + L, per_edge=per_edge, explicit=explicit)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    mrf = to_mrf(pr)
    cost, labels, msgs = api.sgm_forward(mrf, "revised")
    ref = O.forward("isgmr", pr, 1)
    assert np.array_equal(cost[0].cpu().numpy().reshape(-1).view(np.uint32), ref.cost.view(np.uint32))
    assert np.array_equal(msgs[0].cpu().numpy().reshape(-1).view(np.uint32), ref.messages.view(np.uint32))
    assert np.array_equal(labels[0].cpu().numpy().view(np.uint16), ref.labels)
    if not O.have_ref():
        pytest.skip("reference library not present")
    c_ref, l_ref, m_ref = O.ref_sgm_standard(pr)
    cost, labels, msgs = api.sgm_forward(mrf, "standard")
    assert np.array_equal(msgs[0].cpu().numpy().reshape(-1).view(np.uint32), m_ref.view(np.uint32))
    assert np.array_equal(cost[0].cpu().numpy().reshape(-1).view(np.uint32), c_ref.view(np.uint32))
    assert np.array_equal(labels[0].cpu().numpy().view(np.uint16), l_ref)
    c_rev, _ = O.ref_sgm_revised(pr)
    assert np.array_equal(c_rev.view(np.uint32), ref.cost.view(np.uint32))


@pytest.mark.parametrize("variant", ["standard", "revised"])
@pytest.mark.parametrize("H,W,L,conn,per_edge,explicit", [(6, 7, 5, 4, False, True), (9, 8, 16, 8, True, False),
                                                          (7, 9, 21, 4, True, True)])
def test_sgm_iterative_matches_reference(variant, H, W, L, conn, per_edge, explicit):
    """mp::sgm_iterative (baselines.hpp:108-161): every round's cost and
    labels bit-identical to the reference library's."""
    if not O.have_ref():
        pytest.skip("reference library not present")
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=H + W * L, per_edge=per_edge, explicit=explicit)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    K = 4
    got = api.sgm_iterative(to_mrf(pr), K, variant)
    want = O.ref_sgm_iterative(pr, K, variant)
    for k in range(K):
        assert np.array_equal(got[k][0][0].cpu().numpy().reshape(-1).view(np.uint32), want[k][0].view(np.uint32)), k
        assert np.array_equal(got[k][1][0].cpu().numpy().view(np.uint16), want[k][1]), k
