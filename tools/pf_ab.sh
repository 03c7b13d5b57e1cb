python tools/phase_profile.py C2 10000 2>&1 | grep -E "total|solve"
python tools/dbg_solve.py 2>&1 | tail -6
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
