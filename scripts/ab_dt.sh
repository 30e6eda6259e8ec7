# DT filter timing on the bench frames: bash scripts/ab_dt.sh ["ENV=.. ENV=.."]  (FBS_LIB per entry optional)
for kv in ${1:-"X=0"}; do
env $kv python -c "
import torch, sys
sys.path.insert(0,'.')
import paper_1511_03296_b200 as fbs
from workloads import make
w = make('c5')
rgb = torch.from_numpy(w.rgb).cuda(); x = torch.from_numpy(w.t).cuda()
for _ in range(2): fbs.dt_filter(rgb, x, 16.0, 16.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): fbs.dt_filter(rgb, x, 16.0, 16.0)
e1.record(); torch.cuda.synchronize(); print('$kv', e0.elapsed_time(e1) / 10)
"
done
