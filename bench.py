#!/usr/bin/env python
"""Benchmark: ISGMR / TRWP min-sum message passing, fwd+bwd, on B200.

Workload (BASELINE.json configs[1]): C2 = TRWP, 4 directions,
K=5 iterations, KITTI-shaped 375x1242 synthetic stereo cost volume, L=192,
truncated-linear pairwise (tau=2), w=1, rho=0.5; one image per GPU (weak
scaling: images shard across GPUs, one NCCL all-reduce of the shared pairwise
gradient per step when N > 1). A "step" = forward (K iterations, indices
stored) + aggregate + index-driven backward for dc = 1/(N*L) (acceptance.cpp
:282-283) + shared-gradient pack (+ all-reduce).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C1..C5]

Prints ONE JSON line on rank 0. `value` = whole-job G label-updates/s
(LU = K * sum_r|E^r| * L per image) with inputs resident in HBM; `e2e` = the
same metric through the C-ABI with host (pinned) buffers, H2D/D2H inside the
timed region; `roofline` = the dominant kernel class measured with CUDA events
on its launch stream inside the timed region; `cpu_baseline` = the reference
library (oracle/_ref, compiled from the reference sources) timed on this host.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Peaks: MEASURED_PEAKS.json (driver-written) for HBM; the FP32 ALU roof is the
# nominal P_cand of SURVEY.md §8d (148 SMs x 128 lanes x 2 flop x 1.965 GHz).
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
FALLBACK_HBM_GBS = 6650.0


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


# --------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ workloads

GLOBAL_BATCH = {"C4": 32}  # configs whose batch is fixed and sharded over the ranks (strong scaling)


def make_workload(cfg: str, rank: int, world: int = 1, engine: str | None = None):
    """This rank's workload: C4's 32-image batch is split into contiguous
    shards (dist.shard_range; strong scaling); every other
    config runs one image per rank, a different seeded image on each rank
    (weak scaling over independent images)."""
    from paper_1910_10892_b200 import workloads as WL
    from paper_1910_10892_b200.dist import shard_range

    cfg = cfg.upper()
    if cfg in GLOBAL_BATCH:
        start, stop = shard_range(GLOBAL_BATCH[cfg], rank, world)
        return WL.config(cfg, batch=stop - start, first=start)
    return WL.config(cfg, engine=engine, seed_offset=1000 * rank)


def algorithmic_units(wl, E, E_r):
    """Per-image work: label-updates, candidates, and the
    forward / backward algorithmic bytes."""
    K, L, R, N = wl.K, wl.L, wl.conn, wl.N
    per_edge = wl.w_planes is not None
    LU = K * E * L
    cand = LU * L
    P = R if wl.engine == "isgmr" else R + 1
    X = R - 2 if wl.engine == "isgmr" else R - 1
    fwd_bytes = K * E * (4 * L * P + L + 1 + (4 if per_edge else 0)) + (R + 2) * N * L * 4 + 2 * N
    bwd_bytes = K * E * (13 * L + 8 * L * X + 9) + (K + 1) * R * N * L * 4 + N * L * 4
    return LU, cand, fwd_bytes, bwd_bytes


def implemented_bytes(wl, E_r, dv_slots):
    """Minimum HBM bytes of the algorithm as IMPLEMENTED here (every row the
    kernels must read or write once per image and step), as
    opposed to algorithmic_units' reference-as-written formula (SURVEY.md
    §8d), which counts the R+1 read-modify-writes per node the scatter-plane
    backward does not do. Returns (fwd_total, fwd_sweep, bwd_total, bwd_sweep,
    fwd_launches, bwd_launches) in bytes per image and sweep launches per step."""
    K, L, R, N = wl.K, wl.L, wl.conn, wl.N
    trwp = wl.engine == "trwp"
    per_w = wl.w_planes is not None
    rho_pl = trwp and wl.rho_planes is not None
    row = 4 * L
    E = sum(E_r)
    # forward: theta + the other planes at prev, the swept row at cur, p row, q
    rows_fwd = R if trwp else R - 1
    per_edge = rows_fwd * row + row + L + 1 + (4 if per_w else 0) + (4 if rho_pl else 0)
    fwd_sweep = K * E * per_edge
    fused_agg = trwp and R == 4 and wl.H >= 2
    agg = N * (row + 2) if fused_agg else N * (row * (R + 1) + row + 2)
    fwd_total = fwd_sweep + R * N * row * (1 if trwp else 2) + N * row + agg  # + message zeroing, finite scan
    # backward: per edge the rows gm^r(cur) is assembled from, p row, q, the
    # plane row written at prev and the dw read-modify-write
    fused_dt = trwp and not (L <= 32 and wl.H * wl.B >= 148 * 16)
    bwd_sweep = 0
    for k in range(K):
        first = k == K - 1
        for r in range(R):
            if trwp:
                rows = (1 + (R - 1 - r)) if first else R - 1
            else:
                rows = 1 if first else R - 2
            bwd_sweep += E_r[r] * (rows * row + L + 1 + row + 8 + (4 if per_w else 0) + (4 * rows if rho_pl else 0))
        if fused_dt:
            bwd_sweep += N * 2 * row  # direction 0's sweep carries dtheta (read + write)
    bwd_total = bwd_sweep + 2 * N * row + 2 * dv_slots * L * L * 4  # dc -> dtheta copy, dV slots zero + reduce
    if not fused_dt:
        bwd_total += K * N * row * (R + 2)  # dtheta_acc_kernel per iteration
    fwd_launches = K * R if trwp else K
    bwd_launches = K * R if trwp else K
    return fwd_total, fwd_sweep, bwd_total, bwd_sweep, fwd_launches, bwd_launches


# ---------------------------------------------------------------- cpu baseline

def host_info(threads: int) -> dict:
    """nproc, CPU model and OpenMP setting of the host the CPU legs ran on
    (BASELINE.md §3 item 3)."""
    model = None
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    # threads == 0 is the reference's parallel_for default: every hardware thread
    return {"nproc": os.cpu_count(), "cpu_model": model, "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
            "threads_used": threads if threads > 0 else os.cpu_count()}


def cpu_reference_run(wl, K: int, rows: int | None = None, threads: int = 0):
    """One fwd+bwd of the reference library (oracle/_ref; the C restatement if
    absent) on image 0 of the workload, rows [0, rows) (default: the whole
    image), K iterations, `threads` OpenMP threads (0 = all). Returns
    (label-updates, seconds, kind)."""
    from oracle import oracle as O

    kind = "reference" if O.have_ref() else "port"
    impl = "ref" if kind == "reference" else "oracle"
    h = wl.H if rows is None else rows
    un = wl.unary[0].reshape(wl.H, wl.W * wl.L)[:h].reshape(-1).copy()
    wp = None
    if wl.w_planes is not None:
        wp = wl.w_planes[0].reshape(wl.conn // 2, wl.H, wl.W)[:, :h].reshape(-1).copy()
    pr = O.Problem(h, wl.W, wl.L, wl.conn, un, wl.V, wl.w_const, wp, wl.rho_const, None)
    E = O.total_edges(h, wl.W, wl.conn)
    gc = np.full(h * wl.W * wl.L, 1.0 / (h * wl.W * wl.L), np.float32)
    t0 = time.perf_counter()
    f = O.forward(wl.engine, pr, K, impl=impl, threads=threads)
    O.backward(wl.engine, pr, K, f.p, f.q, gc, impl=impl, threads=threads)
    return K * E * wl.L, time.perf_counter() - t0, kind


def cpu_baseline(wl) -> dict:
    """bench.py's cpu_baseline leg: the reference library on
    this host, the WHOLE image at the full K (no extrapolation; the
    reference's O(K^2) index-store regrowth included), all host threads; plus
    a 1-thread figure on a strip of the image at K = 1 (same per-row work)."""
    lu, dt, kind = cpu_reference_run(wl, wl.K)
    rows1 = max(2, min(wl.H, wl.H // 16))
    lu1, dt1, _ = cpu_reference_run(wl, 1, rows=rows1, threads=1)
    return {"value": lu / dt / 1e9, "unit": "G label-updates/s", "cores": os.cpu_count(), "kind": kind,
            "sample": f"{wl.name} {wl.engine.upper()}-{wl.conn} image 0, all {wl.H}x{wl.W} nodes, L={wl.L}, "
                      f"K={wl.K}, fwd+bwd, OpenMP threads=all ({os.cpu_count()}); not extrapolated",
            "seconds": dt, "one_thread": {"value": lu1 / dt1 / 1e9, "seconds": dt1,
                                          "sample": f"rows[0:{rows1}] x {wl.W}, K=1, fwd+bwd, 1 thread"},
            "host": host_info(0)}


# --------------------------------------------------------------------- runs

def run_reference_arm(args, wl):
    """--impl reference: the reference CPU implementation (oracle/_ref) on the
    host cores. Every timed step is one fwd+bwd iteration (K = 1 of the
    config's K identical iterations) over the WHOLE image with all host
    threads -- the workload of one GPU step divided by K; the value is its
    label-update rate. Warm-up steps run on an 8-row strip (paging in the
    library and the inputs, untimed)."""
    kind = None
    for _ in range(args.warmup):
        _, _, kind = cpu_reference_run(wl, 1, rows=min(8, wl.H))
    lus, dts = [], []
    for _ in range(args.steps):
        lu, dt, kind = cpu_reference_run(wl, 1)
        lus.append(lu)
        dts.append(dt)
    value = sum(lus) / sum(dts) / 1e9
    desc = (f"{wl.name} {wl.engine.upper()}-{wl.conn} image 0, all {wl.H}x{wl.W} nodes, L={wl.L}, one of the "
            f"K={wl.K} iterations per step (per-iteration work identical), fwd+bwd, OpenMP threads=all")
    line = {
        "impl": "reference", "metric": metric_name(wl), "value": value, "unit": "G label-updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(dts) / len(dts), "ms_per_step_median": 1e3 * float(np.median(dts)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(wl, args.gpus),
        "cpu_baseline": {"value": value, "unit": "G label-updates/s", "cores": os.cpu_count(), "kind": kind,
                         "sample": desc, "host": host_info(0)},
        "e2e": {"value": value, "unit": "G label-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name(wl):
    return (f"fwd+bwd G label-updates/s, {wl.engine.upper()}-{wl.conn} {wl.W}x{wl.H}x{wl.L} K={wl.K} "
            f"(ms/image alongside)")


def working_set_bytes(wl) -> int:
    """Bytes one step touches per GPU: unary, messages, p, q."""
    R, N, L, K = wl.conn, wl.N, wl.L, wl.K
    E = sum((wl.H - abs(dh)) * (wl.W - abs(dw)) for dh, dw in
            [(0, 1), (0, -1), (1, 0), (-1, 0), (1, 1), (-1, -1), (1, -1), (-1, 1)][:min(R, 8)]) if R <= 8 else N * R
    return wl.B * (N * L * 4 * (R + 1) + K * E * (L + 1))


def l2_flush_needed(wl) -> bool:
    return working_set_bytes(wl) < 2 * 126 * 2 ** 20


def config_dict(wl, n, global_batch=None):
    return {"workload": f"{wl.name}: {wl.engine.upper()} fwd+bwd, {wl.conn} directions, K={wl.K}, "
                        f"{wl.W}x{wl.H} synthetic volume, {wl.L} labels",
            "H": wl.H, "W": wl.W, "L": wl.L, "K": wl.K, "connectivity": wl.conn, "engine": wl.engine,
            "images_per_gpu": wl.B, "global_batch": global_batch or wl.B * n, "parallelism": f"dp{n}",
            "l2": (f"L2 flushed (256 MB write) before every timed step: working set {working_set_bytes(wl) / 1e6:.0f} MB"
                   if l2_flush_needed(wl) else
                   f"inputs larger than L2: working set {working_set_bytes(wl) / 1e9:.2f} GB per GPU (unary, "
                   f"messages, indices)")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--engine", default=None, choices=[None, "isgmr", "trwp"], help="C5's engine (default ISGMR)")
    # enough steps that the pipeline's fill (the first H2D) and drain (the last
    # D2H) do not dominate the end-to-end rate
    ap.add_argument("--e2e-steps", type=int, default=48)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            run_reference_arm(args, make_workload(args.config, 0, 1, args.engine))
        return

    import torch
    import torch.distributed as dist

    from paper_1910_10892_b200 import _lib, api
    from paper_1910_10892_b200.dist import DataParallelStep, NcclComm

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.lib()  # fail loudly if the CUDA library is missing

    wl = make_workload(args.config, rank, world, args.engine)
    global_batch = GLOBAL_BATCH.get(wl.name, world)  # images per step over all ranks
    topo = api.GridTopology(wl.H, wl.W, wl.conn)
    E = topo.total_edges
    E_r = [int(x) for x in topo.edge_count]
    B = wl.B
    unary = torch.from_numpy(wl.unary.reshape(B, wl.N, wl.L)).to(dev)
    V = torch.from_numpy(wl.V.reshape(wl.L, wl.L)).to(dev)
    w = wl.w_const
    if wl.w_planes is not None:
        w = torch.from_numpy(wl.w_planes.reshape(B, wl.conn // 2, wl.N)).to(dev)
    mrf = api.MRF(topo, unary, V, w, wl.rho_const)
    gc = torch.full_like(unary, 1.0 / (wl.N * wl.L))
    # one all-reduce of the packed shared gradient per step, through the
    # library's NCCL collective (mrf_allreduce_grads_f32)
    comm, collective = None, "none (one GPU)"
    if world > 1:
        try:
            comm = NcclComm(dev)
            collective = "mrf_allreduce_grads_f32 (library NCCL communicator)"
        except Exception as exc:  # keep the run alive: the same single all-reduce through torch's NCCL
            collective = f"torch.distributed.all_reduce (library communicator failed: {exc})"
    dp = DataParallelStep(mrf, wl.engine, wl.K, comm=comm)
    fwd_out, grads, shared = dp.fwd, dp.grads, dp.shared
    stream = torch.cuda.current_stream()

    def step():
        dp.step(gc)

    def barrier():
        if world > 1:
            dist.barrier()

    clocks = ClockSampler(local)  # sampling from warm-up through the timed region
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()

    import ctypes as C
    n0 = C.c_int64()
    _lib.check(_lib.lib().mrf_launch_count(C.byref(n0)))
    # a step's working set smaller than twice the L2 gets the L2 flushed
    # (a 256 MB write, outside the per-step event pairs) before every step
    flush = l2_flush_needed(wl)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a_ev, b_ev in evs:
        if flush:
            scratch.fill_(1)
        a_ev.record(stream)
        step()
        b_ev.record(stream)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    n1 = C.c_int64()
    _lib.check(_lib.lib().mrf_launch_count(C.byref(n1)))
    launches = n1.value - n0.value  # every kernel this library launched in the timed region
    ms = sum(a_ev.elapsed_time(b_ev) for a_ev, b_ev in evs)
    # per-kernel-class device time (roofline): a second pass of the same K
    # steps with the library's launch profiler on (events around every
    # launch), kept out of the timed region above
    _lib.check(_lib.lib().mrf_profiler_enable(1))
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    prof = {}
    for cls in range(4):
        tot = C.c_double()
        n = C.c_int64()
        _lib.check(_lib.lib().mrf_profiler_read(cls, C.byref(tot), C.byref(n)))
        prof[cls] = (tot.value, n.value)
    _lib.check(_lib.lib().mrf_profiler_enable(0))
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    LU, cand, fwd_bytes, bwd_bytes = algorithmic_units(wl, E, E_r)
    images = global_batch * args.steps
    value = LU * images / (ms / 1e3) / 1e9
    ms_per_step = ms / args.steps

    # ---- roofline of the dominant kernel class (device time inside the timed region)
    hbm_peak, peak_kind = load_peaks()
    fwd_ms, fwd_n = prof[_lib.KCLASS_FWD_SWEEP]
    bwd_ms, bwd_n = prof[_lib.KCLASS_BWD_SWEEP]
    n_img_local = B * args.steps
    maxlines = max(wl.H, wl.W) * (1 if wl.engine == "trwp" else wl.conn) + (wl.H + wl.W if wl.conn > 4 else 0)
    dv_slots = 592 * 4 if wl.L <= 32 else min(maxlines, 2048)
    f_tot, f_sw, b_tot, b_sw, f_nl, b_nl = implemented_bytes(wl, E_r, dv_slots)
    # sweeps launched per step (ProfScope brackets one sweep, all its strategy kernels)
    f_launch_ms = fwd_ms / max(fwd_n, 1)
    b_launch_ms = bwd_ms / max(bwd_n, 1)
    traffic = ncu_traffic(wl.name)

    def kernel_roof(name, sweep_bytes, n_launch, launch_ms, share, tkey):
        per_launch = sweep_bytes * B / n_launch  # bytes one sweep launch moves (whole local batch)
        achieved = per_launch / (launch_ms / 1e3) / 1e9
        t = traffic.get(tkey) if traffic else None
        d = {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
             "frac": achieved / hbm_peak, "peak_source": peak_kind, "avg_launch_ms": launch_ms,
             "share_of_step": share, "algorithmic_bytes_per_launch": per_launch,
             "bytes_model": "implemented algorithm's minimum bytes (bench.implemented_bytes, DESIGN.md §4)",
             "traffic": t}
        if t:
            d["traffic_frac"] = t / (launch_ms / 1e3) / 1e9 / hbm_peak  # ncu dram bytes at the measured launch time
            d["traffic_source"] = f"profiles/ncu_full_{wl.name}.json (ncu --set full dram__bytes_read+write)"
        return d

    fwd_roof = kernel_roof("fwd sweep (min-plus + argmin, stored indices)", f_sw, f_nl, f_launch_ms,
                           fwd_ms / max(ms, 1e-9), "fwd")
    bwd_roof = kernel_roof("bwd sweep (index-driven scatter: bwd_split / bwd_warp / bwd_small / bwd_grp by config)", b_sw, b_nl, b_launch_ms,
                           bwd_ms / max(ms, 1e-9), "bwd")
    roof = dict(bwd_roof if bwd_ms >= fwd_ms else fwd_roof)
    roof["other_kernel"] = fwd_roof if bwd_ms >= fwd_ms else bwd_roof
    t_min_ms = (f_tot + b_tot) * B / (hbm_peak * 1e9) * 1e3
    roof["step"] = {"t_min_ms": t_min_ms, "measured_ms": ms_per_step, "frac": t_min_ms / ms_per_step,
                    "bytes_per_image": f_tot + b_tot,
                    "note": "whole step at the HBM roof over the implemented algorithm's minimum bytes"}
    roof["fwd_ms_per_image"] = fwd_ms / n_img_local
    roof["bwd_ms_per_image"] = bwd_ms / n_img_local
    # secondary, labelled: SURVEY.md §8d's reference-as-written formulas
    roof["dense_equivalent"] = {
        "fwd_alu_frac": (2.0 * cand * n_img_local / (fwd_ms / 1e3) / 1e12) / FP32_PEAK_TFLOPS if fwd_ms else None,
        "bwd_hbm_frac": (bwd_bytes * n_img_local / (bwd_ms / 1e3) / 1e9) / hbm_peak if bwd_ms else None,
        "note": "L^2 dense candidates (the banded forward evaluates ~(2D+1)/L of them) and the §8d "
                "backward bytes with R+1 row read-modify-writes per node; NOT kernel efficiency"}

    # ---- end to end through the C-ABI with pinned host buffers
    e2e = run_e2e(args, wl, mrf, dp, world, global_batch, dev, LU, barrier)

    line = {
        "metric": metric_name(wl), "value": value, "unit": "G label-updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "ms_per_image": ms / images * world, "higher_is_better": True,
        "scaling": "strong" if wl.name in GLOBAL_BATCH else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded stereo-like cost volume; no datasets)",
        "config": dict(config_dict(wl, world, global_batch), collective=collective), "roofline": roof, "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, wl, mrf, dp, world, global_batch, dev, LU, barrier):
    """Same step through the C-ABI with host buffers: every step copies its
    inputs (unary, cost gradient) from pinned host memory and reads its
    result (gradients + labels) back, all inside the timed region. Steps are
    double-buffered the way a data loader would run them: the H2D of step
    i+1 and the D2H of step i-1 run on copy streams while step i computes
    (stream events order every buffer reuse)."""
    import torch
    import torch.distributed as dist

    from paper_1910_10892_b200 import api

    NB = 2
    h_unary = mrf.unary.cpu().pin_memory()
    h_gc = torch.full(tuple(mrf.unary.shape), 1.0 / (wl.N * wl.L)).pin_memory()
    d_un = [torch.empty_like(mrf.unary) for _ in range(NB)]
    d_gc = [torch.empty_like(mrf.unary) for _ in range(NB)]
    mrfs = [api.MRF(mrf.topo, d_un[i], mrf.V, mrf.weight, mrf.rho) for i in range(NB)]
    fwd_out, grads = dp.fwd, dp.grads
    outs = [fwd_out] + [api._alloc_forward(mrf, wl.K) for _ in range(NB - 1)]
    gsets = [grads] + [api.GradientSet(torch.empty_like(grads.unary), torch.empty_like(grads.pairwise),
                                       torch.empty_like(grads.edge_weights)) for _ in range(NB - 1)]
    hs = [dict(gu=torch.empty_like(h_unary).pin_memory(), gv=torch.empty(tuple(grads.pairwise.shape)).pin_memory(),
               gw=torch.empty(tuple(grads.edge_weights.shape)).pin_memory(),
               lab=torch.empty(tuple(fwd_out.labels.shape), dtype=torch.int16).pin_memory()) for _ in range(NB)]
    s_c = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()
    in_done, comp_done, out_done = [ev() for _ in range(NB)], [ev() for _ in range(NB)], [ev() for _ in range(NB)]
    used = [False] * NB

    def step(i):
        k = i % NB
        if used[k]:
            s_in.wait_event(comp_done[k])  # step i-NB has consumed these inputs
        with torch.cuda.stream(s_in):
            d_un[k].copy_(h_unary, non_blocking=True)
            d_gc[k].copy_(h_gc, non_blocking=True)
            in_done[k].record(s_in)
        s_c.wait_event(in_done[k])
        if used[k]:
            s_c.wait_event(out_done[k])  # step i-NB's results are on the host
        dp.step(d_gc[k], mrf=mrfs[k], out=outs[k], grads=gsets[k])
        comp_done[k].record(s_c)
        s_out.wait_event(comp_done[k])
        with torch.cuda.stream(s_out):
            h = hs[k]
            h["gu"].copy_(gsets[k].unary, non_blocking=True)
            h["gv"].copy_(gsets[k].pairwise, non_blocking=True)
            h["gw"].copy_(gsets[k].edge_weights, non_blocking=True)
            h["lab"].copy_(outs[k].labels, non_blocking=True)
            out_done[k].record(s_out)
        used[k] = True

    for i in range(NB):  # warm-up (workspaces, page-in of the pinned buffers)
        step(i)
    torch.cuda.synchronize()
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(s_c)
    s_in.wait_event(t0)
    for i in range(args.e2e_steps):
        step(i)
    for k in range(NB):
        s_c.wait_event(out_done[k])
    t1.record(s_c)
    torch.cuda.synchronize()
    barrier()
    ms = t0.elapsed_time(t1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    images = global_batch * args.e2e_steps
    h2d = h_unary.numel() * 4 + h_gc.numel() * 4
    d2h = (hs[0]["gu"].numel() + hs[0]["gv"].numel() + hs[0]["gw"].numel()) * 4 + hs[0]["lab"].numel() * 2
    return {"value": LU * images / (ms / 1e3) / 1e9, "unit": "G label-updates/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms / args.e2e_steps,
            "path": "C-ABI mrf_*_forward_f32 + mrf_*_backward_f32 with pinned host inputs/outputs, "
                    "double-buffered (copies of neighbouring steps overlap compute)"}


def ncu_traffic(cfg):
    """dram bytes per launch of the forward / backward sweep from the
    committed ncu --set full summary (profiles/ncu_full_<cfg>.json), else None."""
    p = os.path.join(ROOT, "profiles", f"ncu_full_{cfg}.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {k: d[k]["dram_bytes_per_launch"] for k in ("fwd", "bwd") if k in d}
    except Exception:
        return None


if __name__ == "__main__":
    main()
