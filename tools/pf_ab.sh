for f in 1 4 16 1000; do echo "== F=$f"; TF_HK_F=$f python tools/dbg_rh.py 2>&1 | grep "depth=-"; done
