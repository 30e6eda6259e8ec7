# Sweep FBS_PCG_GROUPS x FBS_BPF_OCC on the bench workload: bash scripts/ab_occ.sh "G:OCC ..."
for r in 1 2; do for go in $1; do G=${go%%:*}; O=${go##*:}
FBS_PCG_GROUPS=$G FBS_BPF_OCC=$O python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
ks=' '.join('%s=%.1f' % (k[:16], v['avg_us']) for k, v in list(d['kernels'].items())[:6])
print('G $G occ $O', round(d['value'],1), round(d['ms_per_step'],3), ks)"
done; done
