for L in paper_1511_03296_b200/alt/libfbs_head.so paper_1511_03296_b200/libfbs.so; do
FBS_LIB=$PWD/$L python -c "
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
e1.record(); torch.cuda.synchronize(); print('$L', e0.elapsed_time(e1) / 10)
"
done
