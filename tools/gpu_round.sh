#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + full capture.
# usage (under gpurun): bash tools/gpu_round.sh [tag] [what...]
TAG=${1:-r1}; shift
WHAT=${@:-"tests smoke bench ncu"}
mkdir -p gpurun_out
for w in $WHAT; do
  case $w in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu_$TAG.log)" ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" ;;
    bench) timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_$TAG.json ;;
    list)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --cpu-sample 2000 > /dev/null 2>&1; echo "ncu-list rc=$?"
      python tools/launches.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt; cat gpurun_out/launches_$TAG.txt ;;
    ncu)
      bash tools/ncu_kernels.sh $TAG k_newton_stream k_rest_l1 k_prefilter_points ;;
  esac
done
