#!/bin/bash
# the FFT pass after the state-phase rewrite: parity tests first, then the C4 per-lag timing
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_fft.py tests/test_gpu_fixtures.py tests/test_gpu_driver.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1
tail -5 gpurun_out/ab_tests.log
python tools/fft_pass_time.py 1e9 500 200000 fft > gpurun_out/ab_state.log 2>&1
tail -3 gpurun_out/ab_state.log
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
cut -c1-400 gpurun_out/bench_c4.json
