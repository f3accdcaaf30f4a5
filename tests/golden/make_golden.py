"""Generate the committed golden fixtures from the REFERENCE library itself.

Run in the container that has /root/reference (it builds oracle/_ref from the
reference's own sources and calls its public entry points through the shim):

    python tests/golden/make_golden.py

Each case stores the inputs and the reference's outputs: forward (cost,
labels, messages, p, q) and backward (d unary, d V, d w planes) for a
soft-head cost gradient computed by the reference's own soft_head_backward.
The CPU suite checks the C restatement against these; the GPU suite checks
libmrf_cuda.so against them.
"""
import os
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402
from paper_1910_10892_b200 import workloads as WL  # noqa: E402

CASES = [
    # name, engine, H, W, L, conn, K, per_edge, explicit, rho_planes
    ("isgmr_8c_explicit_planes", "isgmr", 6, 7, 5, 8, 3, True, True, False),
    ("isgmr_4c_tl_const", "isgmr", 9, 11, 8, 4, 2, False, False, False),
    ("trwp_4c_explicit_planes_rho", "trwp", 7, 6, 4, 4, 3, True, True, True),
    ("trwp_8c_tl_const", "trwp", 8, 9, 12, 8, 2, False, False, False),
    ("trwp_4c_seg21", "trwp", 10, 12, 21, 4, 2, True, True, False),
    ("isgmr_16c_explicit", "isgmr", 5, 6, 3, 16, 2, False, True, False),
]


def make(case):
    name, eng, H, W, L, conn, K, per_edge, explicit, rho_pl = case
    un, V, wc, planes = WL.random_problem(H, W, L, conn, seed=zlib.crc32(name.encode()) % 10000, per_edge=per_edge,
                                          explicit=explicit)
    rng = np.random.default_rng(7)
    rho_planes = rng.uniform(0.2, 1.0, (conn // 2) * H * W).astype(np.float32) if rho_pl else None
    pr = O.Problem(H, W, L, conn, un, V, wc, planes, 0.5, rho_planes)
    f = O.forward(eng, pr, K, impl="ref")
    target = rng.uniform(0.25, L - 1.25, H * W).astype(np.float32)
    loss, _, gc = O.soft_head(f.cost, target, L, impl="ref")
    g = O.backward(eng, pr, K, f.p, f.q, gc, impl="ref")
    arrs = dict(engine=np.array(eng), dims=np.array([H, W, L, conn, K]), unary=un, V=V, w_const=np.float32(wc),
                rho_const=np.float32(0.5), target=target, grad_cost=gc, cost=f.cost, labels=f.labels,
                messages=f.messages, p=f.p, q=f.q, g_unary=g.unary, g_pairwise=g.pairwise, g_wplanes=g.wplanes)
    if planes is not None:
        arrs["w_planes"] = planes
    if rho_planes is not None:
        arrs["rho_planes"] = rho_planes
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrs)
    return name


def load(path):
    z = np.load(path)
    H, W, L, conn, K = (int(x) for x in z["dims"])
    pr = O.Problem(H, W, L, conn, z["unary"], z["V"], float(z["w_const"]),
                   z["w_planes"] if "w_planes" in z else None, float(z["rho_const"]),
                   z["rho_planes"] if "rho_planes" in z else None)
    return str(z["engine"]), pr, K, z


if __name__ == "__main__":
    if not O.have_ref():
        O.build()
    for c in CASES:
        print("wrote", make(c))
