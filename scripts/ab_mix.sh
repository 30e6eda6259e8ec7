# Same-box A/B of (library, environment) pairs on the bench workload:
#   bash scripts/ab_mix.sh "lib.so:VAR=a,VAR2=b" "lib2.so:" ...
for r in 1 2; do for spec in "$@"; do
L=${spec%%:*}; E=${spec#*:}
env ${E//,/ } FBS_LIB=$PWD/$L python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
ks=' '.join('%s=%.1f' % (k[:16], v['avg_us']) for k, v in list(d['kernels'].items())[:8])
print('$spec', round(d['value'],1), round(d['ms_per_step'],3), ks)"
done; done
