#!/bin/bash
# ncu --set full of one launch each of the FFT pass kernels (k_lsar_pass_fft at
# lag ~150, the double-double spectra k_fft_series_dd / k_fft_taps_dd) on a
# C4-shaped sweep (n = 2e8); outputs under gpurun_out/
cd "$(dirname "$0")/.."
export TF_PASS=fft TF_NO_GRAPHS=1
ncu --set full --clock-control none --import-source on -k regex:k_lsar_pass_fft --launch-skip 150 --launch-count 1 \
  -o gpurun_out/ncu_fft_pass -f python tools/fft_pass_time.py 2e8 200 50000 > gpurun_out/ncu_fft.log 2>&1 || true
ncu --set full --clock-control none --import-source on -k regex:"k_fft_series_dd|k_fft_taps_dd" --launch-skip 0 \
  --launch-count 3 -o gpurun_out/ncu_fft_spectra -f python tools/fft_pass_time.py 2e8 200 50000 \
  > gpurun_out/ncu_fft_spectra.log 2>&1 || true
