for v in 1 0; do echo "== NO_COND=$v"; TF_NO_COND_GRAPHS=$v python tools/phase_profile.py C2 10000 2>&1 | grep -E "total|solve|p=  2|p=200"; done
python tools/dbg_rh.py 2>&1 | tail -6
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
