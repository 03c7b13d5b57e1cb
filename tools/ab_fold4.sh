#!/bin/bash
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_fft.py tests/test_gpu_fixtures.py tests/test_gpu_driver.py tests/test_shard.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1
tail -3 gpurun_out/ab_tests.log
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c4_f4.json 2> gpurun_out/bench_c4_f4.err
python - gpurun_out/bench_c4_f4.json <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print(sys.argv[1], d["ms_per_step"], d["value"], d["roofline"]["phase_s"], d["roofline"]["frac"], d["e2e"]["value"] if d.get("e2e") else None)
PY
