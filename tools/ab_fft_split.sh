#!/bin/bash
# the score update split off the FFT pass (k_fft_fold beside the solve): parity, then C4 timing of both modes
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_fft.py tests/test_gpu_fixtures.py tests/test_gpu_driver.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1
tail -15 gpurun_out/ab_tests.log
TF_FFT_SPLIT=0 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c4_fused.json 2> gpurun_out/bench_c4_fused.err
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
for f in gpurun_out/bench_c4_fused.json gpurun_out/bench_c4.json; do python - "$f" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print(sys.argv[1], d["ms_per_step"], d["value"], d["roofline"]["phase_s"], d["e2e"]["value"] if d.get("e2e") else None)
PY
done
