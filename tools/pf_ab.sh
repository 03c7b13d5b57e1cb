for m in 4 3 6 9; do echo "== GRAM_CTAS=$m"; TF_GRAM_CTAS=$m python tools/phase_profile.py C2 100000 2>&1 | grep -E "total|solve  "; done
