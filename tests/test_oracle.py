"""Pins the C restatement (oracle/mrf_oracle.c) to the reference.

Three anchors, mirroring the reference's own test strategy:
  1. committed golden fixtures produced by the reference library itself
     (tests/golden/make_golden.py);
  2. the reference library compiled from its own sources (oracle/_ref), run on
     fresh seeded inputs -- bit-identical forward AND backward;
  3. the reference's known answers and properties: SPEC.md:197 / :245 hand
     examples, single-label zero messages (test_isgmr.cpp:18), index
     footprint (test_isgmr.cpp:98-109), reparametrisation minimum 0 and heads 0
     (test_isgmr.cpp:51-68), the reference's own FD gradient check
     (test_autodiff.cpp:56-84) and revised SGM == ISGMR K=1
     (test_baselines.cpp:58-68).
"""
import glob
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1910_10892_b200 import workloads as WL

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
need_ref = pytest.mark.skipif(not O.have_ref(), reason="reference library not built here")


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_restatement_matches_golden(path):
    from tests.golden.make_golden import load

    eng, pr, K, z = load(path)
    f = O.forward(eng, pr, K)
    for name in ("cost", "labels", "messages", "p", "q"):
        assert np.array_equal(bits(getattr(f, name)), bits(z[name])), name
    g = O.backward(eng, pr, K, z["p"], z["q"], z["grad_cost"])
    assert np.array_equal(g.unary, z["g_unary"])
    assert np.array_equal(g.pairwise, z["g_pairwise"])
    assert np.array_equal(g.wplanes, z["g_wplanes"])


@need_ref
@pytest.mark.parametrize("H,W", [(1, 1), (1, 7), (5, 1), (3, 5), (4, 6), (7, 7), (12, 9), (16, 16), (2, 13)])
@pytest.mark.parametrize("conn", [4, 8, 16])
def test_restatement_topology_matches_reference(H, W, conn):
    a, b = O.oracle_topology(H, W, conn), O.ref_topology(H, W, conn)
    assert a.total_edges == b.total_edges
    assert np.array_equal(a.edge_index, b.edge_index)
    assert np.array_equal(a.dir_offset, b.dir_offset)
    for r in range(conn):
        assert np.array_equal(a.line_first[r], b.line_first[r])
        assert np.array_equal(a.line_len[r], b.line_len[r])


CASES = [
    # H, W, L, conn, K, per_edge, explicit
    (7, 9, 5, 4, 3, True, True),
    (7, 9, 5, 8, 3, True, True),
    (6, 6, 4, 16, 2, False, True),
    (5, 11, 16, 4, 2, False, False),
    (9, 4, 21, 8, 2, True, True),
    (3, 17, 1, 4, 3, False, True),
    (1, 12, 5, 4, 1, False, True),
    (12, 1, 7, 8, 2, True, False),
]


@need_ref
@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
@pytest.mark.parametrize("case", CASES)
def test_restatement_bit_identical_to_reference(engine, case):
    H, W, L, conn, K, per_edge, explicit = case
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=H * 100 + W + L, per_edge=per_edge, explicit=explicit)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, None)
    a, b = O.forward(engine, pr, K, "oracle"), O.forward(engine, pr, K, "ref")
    for name in ("cost", "labels", "messages", "p", "q"):
        assert np.array_equal(bits(getattr(a, name)), bits(getattr(b, name))), name
    rng = np.random.default_rng(1)
    _, _, gc = O.soft_head(a.cost, rng.uniform(0.25, max(L - 1.25, 0.3), H * W), L, "ref")
    ga, gb = O.backward(engine, pr, K, a.p, a.q, gc, "oracle"), O.backward(engine, pr, K, b.p, b.q, gc, "ref")
    for name in ("unary", "pairwise", "wplanes"):
        assert np.array_equal(getattr(ga, name), getattr(gb, name)), name


@need_ref
def test_restatement_rho_planes_and_threads():
    H, W, L, conn, K = 8, 7, 6, 8, 2
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=3, per_edge=True)
    rho = np.random.default_rng(4).uniform(0.1, 1.0, (conn // 2) * H * W).astype(np.float32)
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, rho)
    a = O.forward("trwp", pr, K, "oracle")
    b = O.forward("trwp", pr, K, "ref", threads=4)
    assert np.array_equal(bits(a.messages), bits(b.messages)) and np.array_equal(a.p, b.p)
    gc = np.random.default_rng(5).normal(size=H * W * L).astype(np.float32)
    ga = O.backward("trwp", pr, K, a.p, a.q, gc, "oracle")
    gb = O.backward("trwp", pr, K, b.p, b.q, gc, "ref", threads=4)
    assert np.array_equal(ga.unary, gb.unary) and np.array_equal(ga.pairwise, gb.pairwise)


def test_known_answer_spec_1x2_potts():
    """1x2 chain, theta_0=(0,2), theta_1=(0,0), Potts w=1, K=1:
    the message into node 1 along E before reparam is (0,1) -> after reparam
    (0,1), p entries (0,0)."""
    un = np.array([0, 2, 0, 0], np.float32)
    pr = O.Problem(1, 2, 2, 4, un, WL.potts(2), 1.0, None, 0.5, None)
    f = O.forward("isgmr", pr, 1)
    m = f.messages.reshape(4, 2, 2)
    assert m[0, 1].tolist() == [0.0, 1.0]
    assert f.p[:2].tolist() == [0, 0]
    # TRWP rho=0.5: min_mu(0.5*theta_0(mu) + [mu != l]) = (0,1)
    f = O.forward("trwp", pr, 1)
    assert f.messages.reshape(4, 2, 2)[0, 1].tolist() == [0.0, 1.0]


def test_single_label_zero_messages():
    un, V, wc, _ = WL.random_problem(4, 5, 1, 8, seed=1)
    pr = O.Problem(4, 5, 1, 8, un, V, wc, None, 0.5, None)
    for eng in ("isgmr", "trwp"):
        f = O.forward(eng, pr, 3)
        assert not f.messages.any()
        assert np.array_equal(f.cost, un)


@pytest.mark.parametrize("conn", [4, 8, 16])
def test_index_footprint(conn):
    H, W, L, K = 5, 8, 3, 2
    edges = sum((H - abs(dh)) * (W - abs(dw)) for dh, dw in
                [(0, 1), (0, -1), (1, 0), (-1, 0), (1, 1), (-1, -1), (1, -1), (-1, 1),
                 (1, 2), (-1, -2), (1, -2), (-1, 2), (2, 1), (-2, -1), (2, -1), (-2, 1)][:conn])
    assert O.total_edges(H, W, conn) == edges
    un, V, wc, _ = WL.random_problem(H, W, L, conn, seed=6)
    f = O.forward("isgmr", O.Problem(H, W, L, conn, un, V, wc, None, 0.5, None), K)
    assert f.p.size + f.q.size == K * edges * (L + 1)


def test_reparam_min_zero_heads_zero():
    H, W, L, conn = 5, 6, 4, 8
    un, V, wc, _ = WL.random_problem(H, W, L, conn, seed=3)
    pr = O.Problem(H, W, L, conn, un, V, wc, None, 0.5, None)
    topo = O.oracle_topology(H, W, conn)
    for eng in ("isgmr", "trwp"):
        m = O.forward(eng, pr, 2).messages.reshape(conn, H * W, L)
        heads = topo.edge_index < 0
        assert not m[heads].any()
        assert np.all(m[~heads].min(axis=1) == 0.0)


@need_ref
@pytest.mark.parametrize("trwp", [False, True])
@pytest.mark.parametrize("conn", [4, 8])
def test_reference_fd_gradient_check_pins_backward(trwp, conn):
    """The reference's own double-precision FD check (test_autodiff.cpp:56-72)
    -- the float restatement above is bit-identical to that backward."""
    err, comps, _ = O.ref_gradient_check(4, 5, 4, conn, 2, trwp, True, 7)
    assert comps > 0 and err < 1e-6


@need_ref
def test_revised_sgm_equals_isgmr_k1():
    """test_baselines.cpp:58-68 (cross-engine golden)."""
    H, W, L, conn = 6, 7, 5, 4
    un, V, wc, _ = WL.random_problem(H, W, L, conn, seed=9)
    pr = O.Problem(H, W, L, conn, un, V, wc, None, 0.5, None)
    cost, msg = O.ref_sgm_revised(pr)
    f = O.forward("isgmr", pr, 1)
    assert np.array_equal(bits(cost), bits(f.cost)) and np.array_equal(bits(msg), bits(f.messages))


def test_soft_head_matches_reference_and_fd():
    rng = np.random.default_rng(41)
    L, N = 4, 3
    cost = rng.uniform(0, 5, N * L).astype(np.float32)
    target = np.array([0.7, 1.9, 2.4], np.float32)
    loss, disp, g = O.soft_head(cost, target, L)
    if O.have_ref():
        l2, d2, g2 = O.soft_head(cost, target, L, impl="ref")
        assert loss == l2 and np.array_equal(disp, d2) and np.array_equal(g, g2)
    h = 1e-2
    for i in range(N * L):
        c1, c2 = cost.copy(), cost.copy()
        c1[i] += h
        c2[i] -= h
        fd = (O.soft_head(c1, target, L)[0] - O.soft_head(c2, target, L)[0]) / (2 * h)
        assert abs(fd - g[i]) < 2e-3
