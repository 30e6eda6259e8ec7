"""Refresh the committed measurement evidence under profiles/ from a gpurun_out/ directory:

  gpurun_out/bench.json                 -> profiles/r01_bench.json          (python bench.py)
  gpurun_out/ref.json                   -> profiles/r01_reference.json      (bench.py --impl reference)
  gpurun_out/launches.csv               -> profiles/r01_launches_summary.json (ncu launch list)
  gpurun_out/r01_pcg_iteration.ncu-rep  -> profiles/r01_ncu_<kernel>.json, profiles/traffic.json,
                                           profiles/r01_pcg_iteration.ncu-rep

python scripts/update_profiles.py [gpurun_out] [round tag, default r01]
"""
import json
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_list import load  # noqa: E402
from ncu_summary import summary  # noqa: E402

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
tag = sys.argv[2] if len(sys.argv) > 2 else "r01"
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")

for name, out in (("bench.json", f"{tag}_bench.json"), ("ref.json", f"{tag}_reference.json")):
    p = os.path.join(src, name)
    if os.path.exists(p):
        line = [l for l in open(p).read().splitlines() if l.startswith("{")][-1]
        with open(os.path.join(dst, out), "w") as fh:
            json.dump(json.loads(line), fh, indent=1)
        print("wrote", out)

p = os.path.join(src, "launches.csv")
if os.path.exists(p):
    seq = load(p)
    tot = {}
    for k, us, _ in seq:
        n = k.split("(")[0]
        c, t = tot.get(n, (0, 0.0))
        tot[n] = (c + 1, t + us * 1000.0)
    all_ns = sum(t for _, t in tot.values())
    doc = {"command": "ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv python bench.py "
                      "--steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras",
           "note": "cold-cache serialised per-launch times over the warm-up, timed and profiled passes (3 steps); "
                   "compare shares, not absolutes. Template ids: k_tree_*<0> = PCG, <1> = PDA, <2> = INIT; "
                   "k_hier_level0<0,0> = UPDATE, <1,0> = RESID, <2,0> = RESID0, <0,1> = UPDATE,LAST; a trailing "
                   "false/true is the channel-split flag (K > 1).",
           "total_ns": all_ns, "launches": len(seq),
           "kernels": {k: {"launches": c, "total_ns": t, "share": round(t / all_ns, 4)}
                       for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1])}}
    with open(os.path.join(dst, f"{tag}_launches_summary.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    print("wrote launches summary")

p = os.path.join(src, f"{tag}_pcg_iteration.ncu-rep")
if os.path.exists(p):
    names = {"k_spmv2": "k_spmv2", "void k_hier_level0<0, 0>": "k_hier_level0_UPDATE",
             "void k_tree_lift<0>": "k_tree_lift_PCG", "void k_tree_coarse<0>": "k_tree_coarse_PCG",
             "void k_tree_level0<0>": "k_tree_level0_PCG"}
    keys = {"k_spmv2": "k_spmv2", "k_hier_level0_UPDATE": "k_hier_level0<UPDATE>",
            "k_tree_lift_PCG": "k_tree_lift<PCG>", "k_tree_coarse_PCG": "k_tree_coarse<PCG>",
            "k_tree_level0_PCG": "k_tree_level0<PCG>"}
    traffic = {"_source": "dram__bytes_read.sum + dram__bytes_write.sum of one launch from ncu --set full "
                          "(scripts/prof_pcg.py: one frame group = 4 of the 8 bench frames, PCG iteration 2; "
                          f"profiles/{tag}_ncu_*.json); ncu attributes L2 write-backs late, so writes are "
                          "undercounted for single launches"}

    def mb(v):
        x, unit = v.split()
        return float(x.replace(",", "")) * {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}[unit]

    def short_name(kname):
        base = kname.split("(")[0]
        for k, v in names.items():  # template instances may carry extra flags (e.g. <0, 0, false>)
            if base == k or base.startswith(k[:-1] + ", "):
                return v
        return None

    for rec in summary(p):
        short = short_name(rec["Kernel Name"])
        if not short:
            continue
        with open(os.path.join(dst, f"{tag}_ncu_{short}.json"), "w") as fh:
            json.dump(rec, fh, indent=1)
        traffic[keys[short]] = int(mb(rec["dram__bytes_read.sum"]) + mb(rec["dram__bytes_write.sum"]))
    with open(os.path.join(dst, "traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    shutil.copy(p, os.path.join(dst, f"{tag}_pcg_iteration.ncu-rep"))
    print("wrote ncu summaries + traffic")

p = os.path.join(src, f"{tag}_build_kernels.ncu-rep")
if os.path.exists(p):
    seen = set()
    for rec in summary(p):
        base = rec["Kernel Name"].split("(")[0].replace("void ", "")
        short = base.split("<")[0] + ("_" + base.split("<")[1].rstrip(">").replace(", ", "_") if "<" in base else "")
        if short in seen:
            continue
        seen.add(short)
        with open(os.path.join(dst, f"{tag}_ncu_{short}.json"), "w") as fh:
            json.dump(rec, fh, indent=1)
    shutil.copy(p, os.path.join(dst, f"{tag}_build_kernels.ncu-rep"))
    print("wrote build-kernel summaries:", sorted(seen))

p = os.path.join(src, "gputest.log")
if os.path.exists(p):
    shutil.copy(p, os.path.join(dst, f"{tag}_gputest.log"))
    print("copied gputest.log")
