#!/bin/bash
# Profile capture for profiles/ (run under gpurun; one GPU, never multi-rank).
#   bash tools/profile_round.sh <tag> [configs...]     (default: C2 C3 C4 C5 C1)
# 1) the bench line (not under ncu; run first: a bench right after the ncu
#    replays measured 10-50% slow on the same box in round 1)
# 2) the C2 launch list (device time per launch, clocks unlocked)
# 3) per config, ncu --set full of the owning launch of the top kernels,
#    summarised with pipe-utilisation counters and per-edge / per-chain-step
#    models (tools/ncu_summary.py). The .ncu-rep files stay on the box.
set -x
TAG=${1:-r02}
shift
CONFIGS=${@:-C2 C3 C4 C5 C1}
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C2_${TAG}.json 2> gpurun_out/bench_C2_${TAG}.err
tail -1 gpurun_out/bench_C2_${TAG}.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2_${TAG}.csv \
    python tools/prof_run.py C2 1 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_C2_${TAG}.csv gpurun_out/launches_C2_${TAG}.json
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
cap() {  # cap <cfg> <name> <kernel regex> <skip> <edges> <longest line steps>
  local cfg=$1 name=$2 kre=$3 skip=$4 edges=$5 steps=$6
  timeout 600 $NCU -k "regex:$kre" -s $skip -c 1 -o gpurun_out/ncu_${name}_${cfg}_${TAG} python tools/prof_run.py $cfg 1 > /dev/null 2>&1
  python tools/ncu_summary.py full gpurun_out/ncu_${name}_${cfg}_${TAG}.ncu-rep gpurun_out/ncu_${name}_${cfg}_${TAG}.json \
    "$cfg $name $TAG" $edges $steps
  rm -f gpurun_out/ncu_${name}_${cfg}_${TAG}.ncu-rep
}
for CFG in $CONFIGS; do
  export PROF_BATCH=
  [ "$CFG" = C4 ] && export PROF_BATCH=32
  case $CFG in
    C2)  # TRWP-4 375x1242: forward launch 0 = E (horizontal), 2 = S (vertical); backward
         # sweeps N, S, W, E with 3 split-kernel launches each: 0 = N (vertical), 6 = W (horizontal)
      cap C2 fwdH fwd_band2_kernel 0 465375 1241
      cap C2 fwdV fwd_band2_kernel 2 464508 374
      cap C2 bwdV bwd_split_kernel 0 464508 374
      cap C2 bwdH bwd_split_kernel 6 465375 1241 ;;
    C3)  # ISGMR-8 500x750 L=128: one launch per iteration over all directions
      cap C3 fwd fwd_band2_kernel 0 2992504 749
      cap C3 bwd bwd_warp_kernel 0 2992504 749 ;;
    C4)  # TRWP-4 512x512 L=21, B=32: one launch covers the batch
      cap C4 fwd fwd_small_kernel 0 8372224 511
      cap C4 bwd bwd_small_kernel 0 8372224 511 ;;
    C5)  # ISGMR-4 512x512 L=256 TQ: wide-band forward, window-mode backward
      cap C5 fwd fwd_bandw_kernel 0 1046528 511
      cap C5 bwd bwd_split_kernel 0 1046528 511 ;;
    C1)
      cap C1 fwd fwd_band2_kernel 0 441024 383
      cap C1 bwd bwd_warp_kernel 0 441024 383 ;;
  esac
done
