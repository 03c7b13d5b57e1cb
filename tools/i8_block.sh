#!/bin/bash
# k_i8_gemm launch-order block size (TF_I8_BLOCK): solve time of a C4-shaped sweep
# (n = 2e8, p_bar = 500, c = 2e5) and ncu DRAM bytes / duration of one long-lag launch
cd "$(dirname "$0")/.."
for b in ${BLOCKS:-1 4 8 16}; do
  echo "block $b"
  TF_I8_BLOCK=$b timeout 300 python tools/fft_pass_time.py 2e8 500 200000 fft 2>&1 | grep sweep
  TF_I8_BLOCK=$b TF_NO_GRAPHS=1 ncu --metrics dram__bytes_read.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_i8_gemm --launch-skip 440 --launch-count 1 --csv python tools/fft_pass_time.py 2e8 500 200000 fft 2>/dev/null \
    | grep -E "dram__bytes|lts__t_bytes|gpu__time" | awk -F'","' '{print $(NF-2), $NF}'
done
