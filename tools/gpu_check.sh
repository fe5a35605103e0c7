#!/bin/bash
# One gpurun round trip: GPU parity suite, stage profile, short bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_tile.py --tiles 4 --passes 3 > gpurun_out/prof_tile.log 2>&1
cat gpurun_out/prof_tile.log | tail -12
timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench_quick.log 2> gpurun_out/bench_quick.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.log").read().strip().splitlines()[-1])
print("value", d["value"], "stage_ms", d["stage_ms_per_tile"])
print("roofline", d["roofline"]["stage"], d["roofline"]["frac"], "stream", d["roofline_streaming"]["frac"])
PY
