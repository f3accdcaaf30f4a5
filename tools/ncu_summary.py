"""Summarise ncu reports for profiles/.

    python tools/ncu_summary.py full  <report.ncu-rep> <out.json> [label] [edges] [longest_line_steps]
    python tools/ncu_summary.py launches <launches.csv> <out.json>

`full`: per profiled launch -- duration, SM cycles, instructions, DRAM bytes
read/written, registers, grid, L2 hit rate and the warp-stall breakdown
(from `ncu --set full`), the pipe-utilisation / issue-slot counters, and --
given the launch's edge count and longest line -- warp instructions per edge
and ns per dependent node step. `launches`: the per-launch device-time list of
`ncu --metrics gpu__time_duration.sum --clock-control none --csv`, grouped by
kernel with each kernel's share of the total.
"""
import collections
import csv
import io
import json
import subprocess
import sys


def full(rep, out, label="", edges=0, chain_steps=0):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))

        def num(k):
            try:
                v = float(d.get(k, "nan").replace(",", ""))
            except ValueError:
                return None
            return v * scale.get(units.get(k, ""), 1.0)

        stalls = {}
        for k in hdr:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                v = num(k)
                if v:
                    stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
        # pipe utilisation and issue-slot counters (north_star: the FP32
        # ALU / FMNMX pipe as the forward's roofline, evidenced by ncu)
        pipes = {}
        for k in hdr:
            if (("pipe_" in k and (k.endswith("pct_of_peak_sustained_active") or k.endswith(".sum")))
                    or "issue_active" in k or k.startswith("smsp__inst_executed_pipe_")
                    or k in ("smsp__inst_executed.avg.per_cycle_active", "sm__inst_executed.avg.per_cycle_active",
                             "sm__instruction_throughput.avg.pct_of_peak_sustained_active")):
                v = num(k)
                if v is not None:
                    pipes[k] = v
        res.append({
            "kernel": d.get("Kernel Name"),
            "duration_ms": num("gpu__time_duration.sum"),
            "sm_clock_note": "ncu locks SM clocks to base unless --clock-control none",
            "sm_cycles": num("sm__cycles_elapsed.avg"),
            "instructions": num("smsp__inst_executed.sum"),
            "dram_bytes_read": num("dram__bytes_read.sum"),
            "dram_bytes_write": num("dram__bytes_write.sum"),
            "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
            "registers": num("launch__registers_per_thread"),
            "grid": num("launch__grid_size"),
            "block": num("launch__block_size"),
            "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "stall_samples": dict(sorted(stalls.items(), key=lambda kv: -kv[1])),
            "pipes": pipes,
        })
        if edges:  # per node step: work model of the scanline kernels
            r = res[-1]
            r["edges"] = edges
            if r["instructions"]:
                r["warp_instructions_per_edge"] = r["instructions"] / edges
            if chain_steps and r["duration_ms"]:
                # one node step of the longest line is the dependent chain of a lone warp
                r["longest_line_steps"] = chain_steps
                r["ns_per_chain_step"] = r["duration_ms"] * 1e6 / chain_steps
    with open(out, "w") as f:
        json.dump({"label": label, "report": rep, "launches": res}, f, indent=1)


def launches(path, out):
    text = open(path).read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = collections.defaultdict(list)
    for r in rows[1:]:
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        ms = v / 1e6 if unit == "ns" else v / 1e3 if unit == "us" else v if unit == "ms" else v
        per[r[ik].split("(")[0]].append(ms)
    total = sum(sum(v) for v in per.values())
    summary = {k: {"launches": len(v), "total_ms": sum(v), "avg_ms": sum(v) / len(v), "share": sum(v) / total}
               for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))}
    with open(out, "w") as f:
        json.dump({"source": path, "total_ms": total, "kernels": summary}, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "",
             int(sys.argv[5]) if len(sys.argv) > 5 else 0, int(sys.argv[6]) if len(sys.argv) > 6 else 0)
    else:
        launches(sys.argv[2], sys.argv[3])
