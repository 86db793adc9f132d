#!/bin/bash
# ncu --set full captures of the find pipeline's kernels (one bench step).
TAG=${1:-x}
for k in k_find_prefilter k_round_next_emit k_round2_emit k_newton_sparse k_newton_round1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/${k}_$TAG -f python bench.py --steps 1 --warmup 3 --cpu-sample 1000 > gpurun_out/ncu_${k}_$TAG.log 2>&1
  echo "$k rc=$?"
done
