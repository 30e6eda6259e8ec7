"""Debug: grid build of the ragged-shape test images against the oracle (which arrays differ)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle as O
import paper_1511_03296_b200 as fbs
for (H, W) in [(1, 1), (9, 9), (33, 65), (33, 65), (61, 83)]:
    rng = np.random.default_rng(H * 100 + W)
    rgb = rng.integers(0, 256, (1, H, W, 3), dtype=np.uint8)
    og = O.build_grid(rgb, 8.0, 4.0, 3.0)
    g = fbs.grid_build(torch.from_numpy(rgb).cuda(), 8.0, 4.0, 3.0)
    e = g.export()
    bad = [k for k, a in (("keys", og.keys), ("vid", og.vid), ("m", og.m), ("nbr", og.nbr)) if not np.array_equal(e[k], a)]
    msg = ""
    if "nbr" in bad:
        d = np.nonzero(np.any(e["nbr"] != og.nbr, axis=1))[0]
        msg = f" nbr rows differ: {len(d)} e.g. v={d[:3]} gpu={e['nbr'][d[0]]} ora={og.nbr[d[0]]}"
    print((H, W), "M", g.M, og.M, "bad", bad, msg, flush=True)
