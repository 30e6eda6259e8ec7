# Same-box A/B of environment settings on the bench workload: bash scripts/ab_env.sh "VAR=a VAR=b ..."
for r in 1 2; do for kv in $1; do
env $kv python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
ks=' '.join('%s=%.1f' % (k[:16], v['avg_us']) for k, v in list(d['kernels'].items())[:6])
print('$kv', round(d['value'],1), round(d['ms_per_step'],3), ks)"
done; done
