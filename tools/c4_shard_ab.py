"""C4 as one rank of an N-GPU shard sees it (32/N images), timed on one GPU
with each backward kernel choice (MRF_BWD_SMALL unset = library default,
1 = small-L / grouped kernels). Usage: python tools/c4_shard_ab.py [N ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1910_10892_b200 import api  # noqa: E402
from paper_1910_10892_b200 import workloads as WL  # noqa: E402


def run(n):
    wl = WL.config("C4", batch=32 // n)
    dev = torch.device("cuda", 0)
    topo = api.GridTopology(wl.H, wl.W, wl.conn)
    unary = torch.from_numpy(wl.unary.reshape(wl.B, wl.N, wl.L)).to(dev)
    V = torch.from_numpy(wl.V.reshape(wl.L, wl.L)).to(dev)
    w = torch.from_numpy(wl.w_planes.reshape(wl.B, wl.conn // 2, wl.N)).to(dev)
    mrf = api.MRF(topo, unary, V, w, wl.rho_const)
    gc = torch.full_like(unary, 1.0 / (wl.N * wl.L))
    for mode in ("default", "1"):
        if mode == "default":
            os.environ.pop("MRF_BWD_SMALL", None)
        else:
            os.environ["MRF_BWD_SMALL"] = mode
        f = api.trwp_forward(mrf, wl.K)
        for _ in range(2):
            api.trwp_backward(mrf, f, gc)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            api.trwp_backward(mrf, f, gc)
        e1.record()
        torch.cuda.synchronize()
        print(f"N={n} images/rank={wl.B} bwd[{mode}] {e0.elapsed_time(e1) / 5:.2f} ms", flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:] or ["8", "4"]:
        run(int(a))
