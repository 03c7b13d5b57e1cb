#!/bin/bash
# A/B of the FFT pass twiddle variants (TF_FFT_TW=0 tables / 1 register powers) at C4,
# the direct pass beside them for the crossover, then the FFT parity tests on the default.
cd "$(dirname "$0")/.."
TF_FFT_TW=0 python tools/fft_pass_time.py 1e9 500 200000 fft > gpurun_out/ab_tw0.log 2>&1
cp gpurun_out/fft_pass_time.json gpurun_out/fft_pass_time_tw0.json 2>/dev/null
TF_FFT_TW=1 python tools/fft_pass_time.py 1e9 500 200000 dmma,fft > gpurun_out/ab_tw1.log 2>&1
python -m pytest tests/test_gpu_fft.py tests/test_gpu_fixtures.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1
tail -4 gpurun_out/ab_tw0.log; tail -30 gpurun_out/ab_tw1.log; tail -3 gpurun_out/ab_tests.log
