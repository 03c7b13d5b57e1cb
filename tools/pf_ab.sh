./tools/bin/pass_bench
python tools/phase_profile.py C2 10000 2>&1 | grep -E "pass|total"
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
