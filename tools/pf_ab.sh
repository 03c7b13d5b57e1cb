python tools/phase_profile.py C2 100000 2>&1 | grep -E "p=|total|sample"
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
