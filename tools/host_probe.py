import sys, time, os
sys.path.insert(0, '/root/repo')
import torch
from paper_1910_10892_b200 import api, workloads as WL
wl = WL.config("C2")
dev = torch.device("cuda", 0)
topo = api.GridTopology(wl.H, wl.W, wl.conn)
unary = torch.from_numpy(wl.unary.reshape(wl.B, wl.N, wl.L)).to(dev)
V = torch.from_numpy(wl.V.reshape(wl.L, wl.L)).to(dev)
mrf = api.MRF(topo, unary, V, wl.w_const, wl.rho_const)
gc = torch.full_like(unary, 1.0 / (wl.N * wl.L))
out = api._alloc_forward(mrf, wl.K)
grads = api.GradientSet(torch.empty_like(unary), torch.empty((1, wl.L, wl.L), device=dev), torch.empty((1, 2, wl.N), device=dev))
def step():
    f = api.trwp_forward(mrf, wl.K, out=out)
    api.trwp_backward(mrf, f, gc, out=grads)
for _ in range(3): step()
torch.cuda.synchronize()
for n in (1, 5, 10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter(); e0.record()
    for _ in range(n): step()
    h1 = time.perf_counter(); e1.record(); torch.cuda.synchronize(); h2 = time.perf_counter()
    print(f"n={n}: device {e0.elapsed_time(e1)/n:.2f} ms/step, host enqueue {(h1-h0)*1e3/n:.2f} ms/step, wall {(h2-h0)*1e3/n:.2f}")
