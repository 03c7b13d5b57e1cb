#!/bin/bash
# DRAM bytes + duration of k_lsar_pass_fft per L2-prefetch variant (TF_FFT_PF)
cd "$(dirname "$0")/.."
export TF_PASS=fft TF_NO_GRAPHS=1
for pf in ${PFS:-0 1 2 3}; do
  TF_FFT_PF=$pf timeout 300 python tools/fft_pass_time.py 1e9 160 50000 > gpurun_out/fft_pf$pf.log 2>&1
  TF_FFT_PF=$pf ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_lsar_pass_fft --launch-skip 100 --launch-count 3 --csv python tools/fft_pass_time.py 2e8 160 50000 \
    > gpurun_out/ncu_fft_pf$pf.csv 2>/dev/null
done
