"""Host-feed check for bench.py's device-resident step: device time of K
steps (events around each step, as bench.py) against the sum of the
library's per-kernel device times, with and without the forward's finite
scan, and the host time per step() call. A device step much longer than
its kernels means the GPU idled waiting for the host.
    python tools/host_gap.py [C1..C5] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1910_10892_b200 import api  # noqa: E402
from paper_1910_10892_b200 import workloads as WL  # noqa: E402
from paper_1910_10892_b200.dist import DataParallelStep  # noqa: E402


def run(cfg, steps, assume_finite, sync_each=False, flush=False):
    wl = WL.config(cfg)
    dev = torch.device("cuda", 0)
    topo = api.GridTopology(wl.H, wl.W, wl.conn)
    unary = torch.from_numpy(wl.unary.reshape(wl.B, wl.N, wl.L)).to(dev)
    V = torch.from_numpy(wl.V.reshape(wl.L, wl.L)).to(dev)
    w = wl.w_const if wl.w_planes is None else torch.from_numpy(wl.w_planes.reshape(wl.B, wl.conn // 2, wl.N)).to(dev)
    mrf = api.MRF(topo, unary, V, w, wl.rho_const, assume_finite)
    gc = torch.full_like(unary, 1.0 / (wl.N * wl.L))
    dp = DataParallelStep(mrf, wl.engine, wl.K)
    for _ in range(3):
        dp.step(gc)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    host = 0.0
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
    for a, b in evs:
        if flush:
            scratch.fill_(1)
        a.record()
        t0 = time.perf_counter()
        dp.step(gc)
        host += time.perf_counter() - t0
        b.record()
        if sync_each:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    dev_ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    span = evs[0][0].elapsed_time(evs[-1][1]) / steps
    print(f"{cfg} assume_finite={assume_finite} sync_each={sync_each} l2_flush={flush}: device {dev_ms:.3f} ms/step "
          f"(first-to-last span {span:.3f}), host {1e3 * host / steps:.3f} ms per step() call")


if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    run(cfg, steps, False)
    run(cfg, steps, True)
    run(cfg, steps, True, sync_each=True)
    run(cfg, steps, False, flush=True)
    run(cfg, steps, True, flush=True)
