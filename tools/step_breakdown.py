"""Device-time breakdown of one fwd+bwd step (CUDA events between phases and
the library's per-kernel-class launch profiler). Usage:
    python tools/step_breakdown.py [C1..C5] [steps]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1910_10892_b200 import _lib, api  # noqa: E402
from paper_1910_10892_b200 import workloads as WL  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    wl = WL.config(cfg)
    dev = torch.device("cuda", 0)
    topo = api.GridTopology(wl.H, wl.W, wl.conn)
    unary = torch.from_numpy(wl.unary.reshape(wl.B, wl.N, wl.L)).to(dev)
    V = torch.from_numpy(wl.V.reshape(wl.L, wl.L)).to(dev)
    w = wl.w_const if wl.w_planes is None else torch.from_numpy(wl.w_planes.reshape(wl.B, wl.conn // 2, wl.N)).to(dev)
    mrf = api.MRF(topo, unary, V, w, wl.rho_const)
    fwd = api.isgmr_forward if wl.engine == "isgmr" else api.trwp_forward
    bwd = api.isgmr_backward if wl.engine == "isgmr" else api.trwp_backward
    gc = torch.full_like(unary, 1.0 / (wl.N * wl.L))
    out = api._alloc_forward(mrf, wl.K)
    grads = api.GradientSet(torch.empty_like(unary), torch.empty((wl.B, wl.L, wl.L), device=dev),
                            torch.empty((wl.B, wl.conn // 2, wl.N), device=dev))
    for _ in range(2):
        f = fwd(mrf, wl.K, out=out)
        bwd(mrf, f, gc, out=grads)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    _lib.check(_lib.lib().mrf_profiler_enable(1))
    tf = tb = 0.0
    h0 = time.perf_counter()
    for _ in range(steps):
        ev[0].record()
        f = fwd(mrf, wl.K, out=out)
        ev[1].record()
        bwd(mrf, f, gc, out=grads)
        ev[2].record()
        torch.cuda.synchronize()
        tf += ev[0].elapsed_time(ev[1])
        tb += ev[1].elapsed_time(ev[2])
    host = (time.perf_counter() - h0) * 1e3 / steps
    names = ["fwd_sweep", "bwd_sweep", "aggregate", "aux"]
    print(f"{cfg}: fwd call {tf / steps:.2f} ms, bwd call {tb / steps:.2f} ms, host wall {host:.2f} ms per step")
    for c in range(4):
        t = C.c_double()
        n = C.c_int64()
        _lib.check(_lib.lib().mrf_profiler_read(c, C.byref(t), C.byref(n)))
        print(f"  {names[c]:10s} {t.value / steps:8.3f} ms/step  {n.value // steps} launches/step")
    _lib.check(_lib.lib().mrf_profiler_enable(0))


if __name__ == "__main__":
    main()
