for r in 1 2; do for L in "$@"; do echo "$L $(FBS_LIB=$PWD/$L python scripts/spmv_iso.py 4 2>&1 | tail -1)"; done; done
