for v in 0 1; do echo "== PST=$v"; TF_QFORM_PST=$v python tools/phase_profile.py C2 100000 2>&1 | grep -E "p=|total|solve"; done
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
