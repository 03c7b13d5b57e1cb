#!/bin/bash
# ncu --set full of one k_lsar_pass_fft launch (lag ~150 of a C4-shaped sweep,
# n = 2e8) and the launch list of that sweep; outputs under gpurun_out/
set -e
cd "$(dirname "$0")/.."
export TF_PASS=fft TF_NO_GRAPHS=1
ncu --set full --clock-control none --import-source on -k regex:k_lsar_pass_fft --launch-skip 150 --launch-count 1 \
  -o gpurun_out/ncu_fft_pass -f python tools/fft_pass_time.py 2e8 200 50000 > gpurun_out/ncu_fft.log 2>&1 || true
