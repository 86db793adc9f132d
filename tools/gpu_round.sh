#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + full capture.
# usage (under gpurun): bash tools/gpu_round.sh [tag] [what...]
TAG=${1:-r1}; shift
WHAT=${@:-"tests smoke bench ncu"}
mkdir -p gpurun_out
for w in $WHAT; do
  case $w in
    tests) timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" ;;
    bench) timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_$TAG.json ;;
    ncu)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --cpu-sample 2000 > /dev/null 2>&1; echo "ncu-list rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_newton_round1 -s 3 -c 1 \
        -o gpurun_out/newton_$TAG -f python bench.py --steps 1 --warmup 3 --cpu-sample 2000 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?" ;;
  esac
done
