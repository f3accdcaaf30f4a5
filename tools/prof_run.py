"""One fwd+bwd of a BASELINE config through the C-ABI (for ncu / nsys-style
launch lists). Usage: python tools/prof_run.py [C1..C5] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1910_10892_b200 import api  # noqa: E402
from paper_1910_10892_b200 import workloads as WL  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    batch = int(os.environ.get("PROF_BATCH", "0")) or None
    wl = WL.config(cfg, batch=batch) if cfg == "C4" else WL.config(cfg)
    dev = torch.device("cuda", 0)
    topo = api.GridTopology(wl.H, wl.W, wl.conn)
    unary = torch.from_numpy(wl.unary.reshape(wl.B, wl.N, wl.L)).to(dev)
    V = torch.from_numpy(wl.V.reshape(wl.L, wl.L)).to(dev)
    w = wl.w_const if wl.w_planes is None else torch.from_numpy(wl.w_planes.reshape(wl.B, wl.conn // 2, wl.N)).to(dev)
    mrf = api.MRF(topo, unary, V, w, wl.rho_const)
    fwd = api.isgmr_forward if wl.engine == "isgmr" else api.trwp_forward
    bwd = api.isgmr_backward if wl.engine == "isgmr" else api.trwp_backward
    gc = torch.full_like(unary, 1.0 / (wl.N * wl.L))
    for _ in range(reps):
        f = fwd(mrf, wl.K)
        bwd(mrf, f, gc)
    torch.cuda.synchronize()
    print("done", cfg)


if __name__ == "__main__":
    main()
