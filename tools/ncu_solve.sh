#!/bin/bash
# ncu --set full of the solve kernels at a long lag of a C4-shaped sweep
# (n = 2e8, p_bar = 500, c = 2e5): k_i8_gemm, k_i8_slice, k_svd_minnorm,
# k_pchol_dd (one launch each, ~lag 450); outputs under gpurun_out/
cd "$(dirname "$0")/.."
export TF_NO_GRAPHS=1
for k in k_i8_gemm k_i8_slice k_svd_minnorm k_pchol_dd; do
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 450 --launch-count 1 \
    -o gpurun_out/ncu_$k -f python tools/fft_pass_time.py 2e8 500 200000 fft > gpurun_out/ncu_$k.log 2>&1 || true
done
