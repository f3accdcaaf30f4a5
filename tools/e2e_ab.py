"""A/B of the bench's end-to-end (host-buffer) step: python tools/e2e_ab.py C2 [variant ...]
variants: full, nopack, nofwd (backward only on a fixed forward), nobwd."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1910_10892_b200 import api  # noqa: E402
from paper_1910_10892_b200.dist import DataParallelStep  # noqa: E402
from paper_1910_10892_b200 import workloads as WL  # noqa: E402

wl = WL.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
variants = sys.argv[2:] or ["full"]
dev = torch.device("cuda", 0)
topo = api.GridTopology(wl.H, wl.W, wl.conn)
unary = torch.from_numpy(wl.unary.reshape(wl.B, wl.N, wl.L)).to(dev)
V = torch.from_numpy(wl.V.reshape(wl.L, wl.L)).to(dev)
w = wl.w_const if wl.w_planes is None else torch.from_numpy(wl.w_planes.reshape(wl.B, wl.conn // 2, wl.N)).to(dev)
fwd0 = api.isgmr_forward if wl.engine == "isgmr" else api.trwp_forward
LU = wl.K * topo.total_edges * wl.L


class A:
    e2e_steps = 12


pack0 = api.pack_shared_grads
for v in variants * 2:
    mrf = api.MRF(topo, unary, V, w, wl.rho_const)
    dp = DataParallelStep(mrf, wl.engine, wl.K)
    fwd0(mrf, wl.K, out=dp.fwd)
    if v == "nofwd":
        dp.forward = lambda mrf=None, out=None: dp.fwd
    if v == "nobwd":
        dp.backward = lambda *a, **k: None
    api.pack_shared_grads = (lambda *a, **k: None) if v in ("nopack", "nobwd") else pack0
    r = bench.run_e2e(A, wl, mrf, dp, 1, wl.B, dev, LU, lambda: None)
    print(f"{v:8s} e2e ms/step {r['ms_per_step']:.3f}", flush=True)
