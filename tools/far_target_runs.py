"""How often the backward's main far target changes from one node step to the
next along a scanline (C2, last iteration, direction 0): each change flushes
the POST role's far dV partials. Usage: python tools/far_target_runs.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_10892_b200 import api  # noqa: E402
from paper_1910_10892_b200 import workloads as WL  # noqa: E402

wl = WL.config("C2")
dev = torch.device("cuda", 0)
topo = api.GridTopology(wl.H, wl.W, wl.conn)
unary = torch.from_numpy(wl.unary.reshape(wl.B, wl.N, wl.L)).to(dev)
V = torch.from_numpy(wl.V.reshape(wl.L, wl.L)).to(dev)
mrf = api.MRF(topo, unary, V, wl.w_const, wl.rho_const)
f = api.trwp_forward(mrf, wl.K)
E0 = wl.H * (wl.W - 1)  # direction 0 edges: H lines of W-1
p = f.p[0, wl.K - 1].reshape(-1, wl.L)[:E0].cpu().numpy().astype(np.int32).reshape(wl.H, wl.W - 1, wl.L)
lab = np.arange(wl.L)[None, None, :]
far = np.abs(p - lab) >= 2
tgt = np.where(far, p, -1).max(axis=2)  # common far target (max over far labels)
lo = np.where(far, p, 10**6).min(axis=2)
uniq = (tgt == lo) | (tgt < 0)
chg = (tgt[:, 1:] != tgt[:, :-1]).mean()
print(f"edges/line {wl.W - 1}: single far target {uniq.mean():.3f}, main target changes at {chg:.3f} of steps")
# flushes with a small LRU of far-target partial rows
for cap in (1, 2, 3, 4):
    miss = 0
    for row in tgt:
        lru = []
        for t in row:
            if t < 0:
                continue
            if t in lru:
                lru.remove(t)
            else:
                miss += 1
                if len(lru) == cap:
                    lru.pop(0)
            lru.append(t)
    print(f"LRU of {cap} targets: {miss / tgt.size:.3f} flushes per step")
