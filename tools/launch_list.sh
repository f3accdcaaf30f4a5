#!/bin/bash
# Per-launch device time + grid of one fwd+bwd: bash tools/launch_list.sh <cfg> <tag>
CFG=${1:-C2}; TAG=${2:-x}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv \
    --log-file gpurun_out/ll_${CFG}_${TAG}.csv python tools/prof_run.py $CFG 1 > /dev/null 2>&1
python - "$CFG" "$TAG" <<'PY'
import csv, sys, collections
cfg, tag = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(f"gpurun_out/ll_{cfg}_{tag}.csv")) if len(r) > 10]
hdr = rows[0]; data = rows[2:] if rows[1][0] == "" else rows[1:]
iN = hdr.index("Kernel Name"); iM = hdr.index("Metric Name"); iV = hdr.index("Metric Value"); iID = hdr.index("ID")
L = collections.OrderedDict()
for r in data:
    L.setdefault(r[iID], {"name": r[iN]})[r[iM]] = r[iV]
agg = collections.OrderedDict()
for d in L.values():
    key = (d["name"][:60], d.get("launch__grid_size"), d.get("launch__block_size"))
    t = float(d["gpu__time_duration.sum"].replace(",", ""))
    a = agg.setdefault(key, [0, 0.0]); a[0] += 1; a[1] += t
tot = sum(a[1] for a in agg.values())
for k, (n, t) in agg.items():
    print(f"{n:4d} x {t/n/1e3:9.1f} us = {t/1e6:8.3f} ms  {100*t/tot:5.1f}%  grid={k[1]} blk={k[2]}  {k[0]}")
print(f"total {tot/1e6:.3f} ms")
PY
