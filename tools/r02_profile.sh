#!/bin/bash
# Round-2 evidence run at C4: the bench (no profiler), one ncu --set full launch of
# k_lsar_pass_fft (lag ~ 260), then the ncu launch list of the same bench command.
cd "$(dirname "$0")/.."
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_lsar_pass_fft --launch-skip 200 --launch-count 1 \
  -o gpurun_out/ncu_fft_c4 -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_fft_c4.log 2>&1
if [ "$1" = "list" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 16500 --csv --log-file gpurun_out/c4_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_list.log 2>&1
gzip -f gpurun_out/c4_launches.csv
fi
cut -c1-300 gpurun_out/bench_c4.json
