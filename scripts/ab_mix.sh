# Same-box A/B of (library, environment) pairs on the bench workload:
#   bash scripts/ab_mix.sh "lib.so:VAR=a,VAR2=b" "lib2.so:" ...      (FBS_AB_KERNELS: kernel prefixes to print)
for r in 1 2; do for spec in "$@"; do
L=${spec%%:*}; E=${spec#*:}
env ${E//,/ } FBS_LIB=$PWD/$L python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,os,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
want=os.environ.get('FBS_AB_KERNELS','k_bistoch,k_spmv2,k_tree_lift<PCG>,k_tree_coarse<PCG>,k_tree_level0<PCG>,k_hier_level0<UPDATE>,k_splat,k_grid_sort,k_grid_write,k_grid_neigh,k_pyr_sort,k_slice').split(',')
ks=' '.join('%s=%.1f' % (k[:14], v['avg_us']) for k, v in d['kernels'].items() if any(k.startswith(w) for w in want))
print('$spec', round(d['value'],1), round(d['ms_per_step'],3), ks)"
done; done
