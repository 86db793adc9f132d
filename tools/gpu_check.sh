#!/bin/bash
# Standard GPU check (under gpurun): gpu tests, smoke, bench -> gpurun_out/*_TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider 2>&1 | grep -v "^$" > gpurun_out/pytest_gpu_$TAG.log
echo "pytest: $(tail -1 gpurun_out/pytest_gpu_$TAG.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
    print("value %.4g ms %.4f e2e_ms %.4f frac %.3f kern_ms %.4f" % (d["value"], d["ms_per_step"], d["e2e"]["ms_per_step"], d["roofline"]["frac"], d["roofline"]["kernel_ms"]))
    w = d["work"]; print({k: w[k] for k in ("newton", "iters", "rest_points", "r1_warp_evals", "r1_w2_evals", "iters_r1", "rest_lane_evals", "redo", "setup_ms")})
except Exception as e:
    print("bench parse failed", e)
PY
