for L in "$@"; do for c in c3 c2; do echo "$L $c $(FBS_LIB=$PWD/$L python scripts/prof_cfg.py $c 2>&1 | grep -E 'wall|coarse<PCG>' | tr '\n' ' ')"; done; done
