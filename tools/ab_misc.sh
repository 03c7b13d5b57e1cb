#!/bin/bash
cd "$(dirname "$0")/.."
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c4_a.json 2> gpurun_out/bench_c4_a.err
TF_FFT_MINQ=16 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c4_q16.json 2> gpurun_out/bench_c4_q16.err
TF_FFT_MINQ=32 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c4_q32.json 2> gpurun_out/bench_c4_q32.err
for f in gpurun_out/bench_c4_a.json gpurun_out/bench_c4_q16.json gpurun_out/bench_c4_q32.json; do python - "$f" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
print(sys.argv[1], d["ms_per_step"], d["value"], d["roofline"]["phase_s"], d["roofline"]["frac"], d["e2e"]["value"] if d.get("e2e") else None)
PY
done
