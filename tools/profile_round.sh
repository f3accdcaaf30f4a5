#!/bin/bash
# Profile capture for profiles/ (run under gpurun; one GPU, never multi-rank).
#   bash tools/profile_round.sh <tag>
# 1) launch list of one C2 fwd+bwd (device time per launch, clocks unlocked)
# 2) ncu --set full of the top kernels: first horizontal + vertical forward
#    sweep and backward sweep launches of C2 (the banded-mode instantiation)
# 3) the bench line itself (not under ncu; run first, see below)
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
# the bench line first: a bench run right after the ncu replays measured
# 10-50% slow on the same box (r01e, r01h), never on a fresh one
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C2_${TAG}.json 2> gpurun_out/bench_C2_${TAG}.err
tail -1 gpurun_out/bench_C2_${TAG}.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2_${TAG}.csv \
    python tools/prof_run.py C2 1 > /dev/null 2>&1
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
# forward: directions E, W (horizontal), S, N (vertical) per iteration -> launch 0 = H, 2 = V
$NCU -k regex:fwd_band2_kernel -s 0 -c 1 -o gpurun_out/ncu_fwdH_C2_${TAG} python tools/prof_run.py C2 1 > /dev/null 2>&1
$NCU -k regex:fwd_band2_kernel -s 2 -c 1 -o gpurun_out/ncu_fwdV_C2_${TAG} python tools/prof_run.py C2 1 > /dev/null 2>&1
# backward: directions N, S (vertical), W, E (horizontal), each as 3 launches (banded D<=2,
# window, general; the non-owners exit at once): launch 0 = N (vertical), 6 = W (horizontal)
$NCU -k regex:bwd_split_kernel -s 0 -c 1 -o gpurun_out/ncu_bwdV_C2_${TAG} python tools/prof_run.py C2 1 > /dev/null 2>&1
$NCU -k regex:bwd_split_kernel -s 6 -c 1 -o gpurun_out/ncu_bwdH_C2_${TAG} python tools/prof_run.py C2 1 > /dev/null 2>&1
# summaries for profiles/ (the .ncu-rep files stay on the box: gpurun brings back <= 64 MiB)
for k in fwdH fwdV bwdH bwdV; do
  python tools/ncu_summary.py full gpurun_out/ncu_${k}_C2_${TAG}.ncu-rep gpurun_out/ncu_${k}_C2_${TAG}.json "C2 $k ${TAG}"
done
python tools/ncu_summary.py launches gpurun_out/launches_C2_${TAG}.csv gpurun_out/launches_C2_${TAG}.json
rm -f gpurun_out/*.ncu-rep
