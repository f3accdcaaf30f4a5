#!/bin/bash
# Per-source-line / per-SASS-instruction metrics of one kernel launch (run under gpurun).
#   bash tools/ncu_source.sh <cfg> <name> <kernel regex> <skip>
# writes gpurun_out/src_<name>_<cfg>.{cuda,sass}.csv
cfg=$1; name=$2; kre=$3; skip=$4
mkdir -p gpurun_out
export PROF_BATCH=; [ "$cfg" = C4 ] && export PROF_BATCH=32
ncu --set full --import-source on --clock-control none -k "regex:$kre" -s $skip -c 1 -o /tmp/src_${name}_${cfg} \
  python tools/prof_run.py $cfg 1 > /dev/null 2>&1
ncu -i /tmp/src_${name}_${cfg}.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_${name}_${cfg}.cuda.csv 2>&1
ncu -i /tmp/src_${name}_${cfg}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${name}_${cfg}.sass.csv 2>&1
