#!/bin/bash
# Step-time breakdown of every BASELINE config (C5 both engines): per-kernel
# device time from one fwd+bwd. bash tools/all_configs.sh <tag>
TAG=${1:-x}
for C in C1 C2 C3 C4 C5; do
  echo "== $C"; timeout 300 bash tools/launch_list.sh $C $TAG | tail -14
done
