#!/bin/bash
# Profile capture for profiles/ (run under gpurun; one GPU, never multi-rank).
#   bash tools/profile_round.sh <tag>
# 1) launch list of one C2 fwd+bwd (device time per launch, clocks unlocked)
# 2) ncu --set full of the top kernels: first horizontal + vertical forward
#    sweep and backward sweep launches of C2
# 3) the bench line itself (not under ncu)
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2_${TAG}.csv \
    python tools/prof_run.py C2 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:fwd_band2 -s 0 -c 1 -o gpurun_out/ncu_fwdH_C2_${TAG} python tools/prof_run.py C2 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:fwd_band2 -s 2 -c 1 -o gpurun_out/ncu_fwdV_C2_${TAG} python tools/prof_run.py C2 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:bwd_ -s 0 -c 1 -o gpurun_out/ncu_bwdV_C2_${TAG} python tools/prof_run.py C2 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:bwd_ -s 2 -c 1 -o gpurun_out/ncu_bwdH_C2_${TAG} python tools/prof_run.py C2 1 > /dev/null 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C2_${TAG}.json 2> gpurun_out/bench_C2_${TAG}.err
tail -1 gpurun_out/bench_C2_${TAG}.json
