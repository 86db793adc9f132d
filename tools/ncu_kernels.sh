#!/bin/bash
# ncu --set full captures of find-pipeline kernels (one bench step each).
# usage (under gpurun): bash tools/ncu_kernels.sh TAG [kernel-regex ...]
TAG=${1:-x}; shift
KS=${@:-"k_prefilter_cells k_newton_round1 k_find_rest"}
mkdir -p gpurun_out
for k in $KS; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/${k}_$TAG -f python bench.py --steps 1 --warmup 3 --cpu-sample 1000 > gpurun_out/ncu_${k}_$TAG.log 2>&1
  echo "$k rc=$?"
done
