#!/bin/bash
# the split pass with the next spectrum prefetched into registers (k_lsar_pass_fft_r) against the
# fused kernel with its score phase skipped: parity (incl. the one-rank sharded sweep), then C4 timing
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_fft.py tests/test_gpu_fixtures.py tests/test_gpu_driver.py tests/test_shard.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1
tail -5 gpurun_out/ab_tests.log
TF_FFT_RPF=0 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c4_rpf0.json 2> gpurun_out/bench_c4_rpf0.err
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
for f in gpurun_out/bench_c4_rpf0.json gpurun_out/bench_c4.json; do python - "$f" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print(sys.argv[1], d["ms_per_step"], d["value"], d["roofline"]["phase_s"], d["roofline"]["frac"], d["e2e"]["value"] if d.get("e2e") else None)
PY
done
