"""Full-size parity: every BASELINE.json configuration at its own shape,
through the C-ABI, against the reference library itself (oracle/_ref: the
unmodified reference compiled from its sources, all host threads).

Mirrors the reference's bit-identity tests (test_isgmr.cpp:84-96,
test_trwp.cpp:73-86, acceptance.cpp:248-271) with "GPU == reference" in place
of "1 thread == N threads": messages, cost, labels, p and q bit-identical;
gradients within 1e-5 normwise AND elementwise (tests/gpu_util.py).

Iteration counts: C2 (the headline) and C4 run their full K=5; C3 and C5 run
K=2 at full grid size (per-iteration work is identical, and the reference's
C5 K=10 alone would take minutes per engine). Set MRF_PARITY_LOG=<path> to
dump every gradient error measured here as JSON.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1910_10892_b200 import workloads as WL
from tests import gpu_util as GU
from tests.gpu_util import assert_forward_equal, assert_grads_close, gpu_backward, gpu_forward, to_mrf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not O.have_ref():
        pytest.skip("reference library (oracle/_ref) not built")
    yield
    path = os.environ.get("MRF_PARITY_LOG")
    if path:
        with open(path, "w") as f:
            json.dump(GU.GRAD_LOG, f, indent=1)


def _soft_head_grad(cost, L, N, seed):
    """dc from the soft head with a seeded target (GradCheckInstance recipe)."""
    _, _, gc = O.soft_head(cost, np.random.default_rng(seed).uniform(0.25, L - 1.25, N).astype(np.float32), L)
    return gc


def _run(engine, pr, K, tag, grad="head"):
    ref = O.forward(engine, pr, K, impl="ref", threads=0)
    mrf = to_mrf(pr)
    f = gpu_forward(engine, mrf, K)
    assert_forward_equal(f, ref)
    gc = _soft_head_grad(ref.cost, pr.L, pr.N, 7) if grad == "head" else \
        np.full(pr.N * pr.L, 1.0 / (pr.N * pr.L), np.float32)
    g = gpu_backward(engine, mrf, f, gc)
    gref = O.backward(engine, pr, K, ref.p, ref.q, gc, impl="ref", threads=0)
    assert_grads_close(g, gref, tag=tag)


def test_c2_trwp_full_size_k5():
    """C2, the headline: TRWP-4, 375x1242, L=192, K=5 (band2 forward with the
    fused aggregation, warp-specialised backward)."""
    wl = WL.config("C2")
    pr = O.Problem(wl.H, wl.W, wl.L, wl.conn, wl.unary[0], wl.V, wl.w_const, None, 0.5, None)
    _run("trwp", pr, wl.K, "C2")


def test_c3_isgmr8_full_size():
    """C3: ISGMR-8, 500x750, L=128 (band2<4,0,8,1> forward and
    bwd_split<4,0,8,1,...> backward), K=2 at full grid size."""
    wl = WL.config("C3")
    pr = O.Problem(wl.H, wl.W, wl.L, wl.conn, wl.unary[0], wl.V, wl.w_const, None, 0.5, None)
    _run("isgmr", pr, 2, "C3")


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
def test_c5_full_size(engine):
    """C5: 512x512, L=256, integer truncated quadratic (wide-band forward,
    window-mode backward): maximal ties, K=2 at full grid size."""
    wl = WL.config("C5", engine=engine)
    pr = O.Problem(wl.H, wl.W, wl.L, wl.conn, wl.unary[0], wl.V, wl.w_const, None, 0.5, None)
    _run(engine, pr, 2, f"C5-{engine}")


def test_c4_batched_images_full_size():
    """C4: TRWP-4, 512x512, L=21, explicit V, per-edge weights, K=5: three
    images of the seeded batch in ONE batched call, each against the
    reference, plus the shared-gradient pack over the batch."""
    from paper_1910_10892_b200 import api

    wl = WL.config("C4", batch=3)
    prs = [O.Problem(wl.H, wl.W, wl.L, wl.conn, wl.unary[b], wl.V, 1.0, wl.w_planes[b], 0.5, None)
           for b in range(wl.B)]
    mrf = to_mrf(prs[0], batch_unary=list(wl.unary), batch_wplanes=list(wl.w_planes))
    f = gpu_forward("trwp", mrf, wl.K)
    refs = [O.forward("trwp", pr, wl.K, impl="ref", threads=0) for pr in prs]
    gcs = np.stack([_soft_head_grad(r.cost, wl.L, wl.N, 100 + b) for b, r in enumerate(refs)])
    g = gpu_backward("trwp", mrf, f, gcs)
    dv_sum = np.zeros(wl.L * wl.L, np.float64)
    for b, (pr, ref) in enumerate(zip(prs, refs)):
        assert_forward_equal(f, ref, b=b)
        gref = O.backward("trwp", pr, wl.K, ref.p, ref.q, gcs[b], impl="ref", threads=0)
        assert_grads_close(g, gref, b=b, tag="C4")
        dv_sum += gref.pairwise
    packed = api.pack_shared_grads(mrf, g).cpu().numpy()
    assert GU.normwise(packed[:-1], dv_sum) <= GU.GRAD_RTOL


@pytest.mark.parametrize("engine", ["isgmr", "trwp"])
def test_l128_conn8_band2_small(engine):
    """Small case with the C3 instantiation (96 < L <= 128, banded tau=2,
    8 directions) for both engines, against the reference."""
    H, W, L = 12, 17, 128
    un = WL.stereo_like(H, W, L, 31)
    pr = O.Problem(H, W, L, 8, un, WL.truncated_linear(L, 2.0), 1.0, None, 0.5, None)
    _run(engine, pr, 2, f"L128c8-{engine}")
