"""Helpers shared by the GPU parity tests: run libmrf_cuda.so on numpy
problems (reference layouts) and compare with the CPU checkers."""
import numpy as np
import torch

from oracle import oracle as O
from paper_1910_10892_b200 import api


def to_mrf(pr: O.Problem, batch_unary=None, batch_wplanes=None, batch_rho=None):
    """Device MRF for one oracle problem (or a batch of per-image arrays)."""
    dev = torch.device("cuda", 0)
    topo = api.GridTopology(pr.H, pr.W, pr.conn)
    un = np.stack(batch_unary) if batch_unary is not None else pr.unary[None]
    unary = torch.from_numpy(np.ascontiguousarray(un.reshape(un.shape[0], pr.N, pr.L))).to(dev)
    V = torch.from_numpy(pr.V.reshape(pr.L, pr.L).copy()).to(dev)
    R2 = pr.conn // 2
    w = pr.w_const
    if batch_wplanes is not None:
        w = torch.from_numpy(np.stack(batch_wplanes).reshape(-1, R2, pr.N).copy()).to(dev)
    elif pr.w_planes is not None and batch_unary is None:
        w = torch.from_numpy(pr.w_planes.reshape(1, R2, pr.N).copy()).to(dev)
    rho = pr.rho_const
    if batch_rho is not None:
        rho = torch.from_numpy(np.stack(batch_rho).reshape(-1, R2, pr.N).copy()).to(dev)
    elif pr.rho_planes is not None and batch_unary is None:
        rho = torch.from_numpy(pr.rho_planes.reshape(1, R2, pr.N).copy()).to(dev)
    return api.MRF(topo, unary, V, w, rho)


def gpu_forward(engine, mrf, K):
    f = (api.isgmr_forward if engine == "isgmr" else api.trwp_forward)(mrf, K)
    torch.cuda.synchronize()
    return f


def gpu_backward(engine, mrf, fwd, grad_cost):
    gc = torch.from_numpy(np.ascontiguousarray(grad_cost, np.float32).reshape(mrf.unary.shape)).cuda()
    g = (api.isgmr_backward if engine == "isgmr" else api.trwp_backward)(mrf, fwd, gc)
    torch.cuda.synchronize()
    return g


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def assert_forward_equal(f, ref, b=0, what=("cost", "labels", "messages", "p", "q")):
    """Bit-exact comparison of image b of a device ForwardResult with a
    checker Forward (numpy, reference layout)."""
    got = {
        "cost": f.cost[b].cpu().numpy().reshape(-1),
        "labels": f.labels[b].cpu().numpy().view(np.uint16).reshape(-1),
        "messages": f.messages[b].cpu().numpy().reshape(-1),
        "p": f.p[b].cpu().numpy().reshape(-1),
        "q": f.q[b].cpu().numpy().reshape(-1),
    }
    for name in what:
        g, r = got[name], getattr(ref, name) if not isinstance(ref, dict) else ref[name]
        if not np.array_equal(bits(g), bits(r)):
            diff = np.nonzero(bits(g) != bits(r))[0]
            raise AssertionError(f"{name}: {diff.size} differing bytes, first at {diff[:5]}")


def normwise(a, b):
    a = np.asarray(a, np.float64).reshape(-1)
    b = np.asarray(b, np.float64).reshape(-1)
    den = max(np.linalg.norm(b), 1e-30)
    return float(np.linalg.norm(a - b) / den)


# Gradient tolerance stated by north_star: "within 1e-5 relative in FP32".
# Two checks per gradient tensor (scatter/reduction order differs from the
# reference's sequential loops; indices are identical):
#   normwise     ||got - want||_2 / ||want||_2 <= GRAD_RTOL
#   elementwise  |got_i - want_i| <= GRAD_RTOL * |want_i| + GRAD_RTOL * ||want||_inf
# The elementwise atol is scaled to the tensor's largest entry: an element that
# is a cancellation of terms of that size can only be exact to that scale.
GRAD_RTOL = 1e-5

# every comparison made by assert_grads_close (tests that log errors read it)
GRAD_LOG = []


def grad_errors(got, want):
    got = np.asarray(got, np.float64).reshape(-1)
    want = np.asarray(want, np.float64).reshape(-1)
    d = np.abs(got - want)
    inf = float(np.max(np.abs(want))) if want.size else 0.0
    den = np.abs(want) + inf
    return {"normwise": normwise(got, want), "max_abs": float(d.max()) if d.size else 0.0, "want_inf": inf,
            "max_elem_rel": float(np.max(d / np.maximum(den, 1e-30))) if d.size else 0.0}


def assert_grads_close(g, ref, b=0, rtol=GRAD_RTOL, tag=""):
    pairs = [("unary", g.unary[b], ref.unary if not isinstance(ref, dict) else ref["g_unary"]),
             ("pairwise", g.pairwise[b], ref.pairwise if not isinstance(ref, dict) else ref["g_pairwise"]),
             ("wplanes", g.edge_weights[b], ref.wplanes if not isinstance(ref, dict) else ref["g_wplanes"])]
    for name, got, want in pairs:
        got = got.cpu().numpy().reshape(-1)
        want = np.asarray(want).reshape(-1)
        if not np.any(want) and not np.any(got):
            continue
        e = grad_errors(got, want)
        GRAD_LOG.append({"tag": tag, "b": b, "tensor": name, **e})
        assert e["normwise"] <= rtol, f"{name}: normwise rel err {e['normwise']:.3e} > {rtol}"
        # |d| <= rtol (|want| + inf)  <=>  d / (|want| + inf) <= rtol
        assert e["max_elem_rel"] <= rtol, f"{name}: elementwise err {e['max_elem_rel']:.3e} > {rtol} ({e})"
