#!/bin/bash
# Round-2 evidence run at C4: the full GPU suite + smoke, the bench (no profiler), one ncu --set full
# launch each of k_lsar_pass_fft and k_fft_fold (lag ~ 260), then the ncu launch list of the same
# bench command.
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err || exit 1
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_c4_reference.json 2> gpurun_out/bench_c4_reference.err
ncu --set full --clock-control none --import-source on -k regex:k_lsar_pass_fft --launch-skip 200 --launch-count 1 \
  -o gpurun_out/ncu_fft_c4 -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_fft_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fft_fold --launch-skip 200 --launch-count 1 \
  -o gpurun_out/ncu_fold_c4 -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_fold_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 17500 --csv --log-file gpurun_out/c4_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_list.log 2>&1
gzip -f gpurun_out/c4_launches.csv
tail -3 gpurun_out/gputest.log; tail -1 gpurun_out/smoke.log; cut -c1-300 gpurun_out/bench_c4.json; cut -c1-300 gpurun_out/bench_c4_reference.json
