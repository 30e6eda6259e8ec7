#!/usr/bin/env python
"""bench.py — megapixels/s of the bilateral-space solve (grid build + Alg. 1 + pyramid + splat +
assemble + hierarchical init + 25 PCG iterations + slice) on BASELINE.json configs[4] (batch
scaling: independent 1920×1080 frames, 8 per GPU, sharded over ranks with no collective on the
solve path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fbs|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one rank per GPU, NCCL)

Prints ONE JSON line on rank 0.  `value` = all ranks' pixels ÷ the max-over-ranks device time
of exactly K steps (CUDA events, barrier + synchronize on both sides).  `--impl reference`
times the fp64 oracle (oracle/, the CPU reference of this build) on a bounded sample instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "megapixels/sec solved (grid+PCG+slice); PCG HBM GB/s vs peak; 1/2/4/8 GPUs"
SIGMAS = (8.0, 4.0, 3.0)
LAM = 128.0
ITERS = 25

# Algorithmic bytes per launch of each kernel: fp32 vectors, K = 1, neighbour
# structure 16 B/vertex (8 int8 near offsets + 2 int32 y offsets).  Gathers of neighbour values
# are cache-resident re-reads and are not counted.  M = level-0 vertices, lv = level sizes.
def kernel_bytes(name, M, lv, N):
    up = sum(lv[1:])  # pyramid vertices above level 0
    lv1 = lv[1] if len(lv) > 1 else 0
    table = {
        "k_spmv2": 32 * M,             # nbr 16 + (d,n) 8 + Sc 4 + q write 4
        # r rw 8 + q 4 + mu0 4 (x += αd is done by the next direction pass; w = mask∘r is r itself
        # on a forward solve, so it is not written: DESIGN §5)
        "k_hier_level0<UPDATE>": 16 * M,
        # tord0 4 + r gather 4 per level-0 vertex; csT 4 + mu1 4 + (P w)_1 write 4 + prefix write 8 per level-1 vertex
        "k_tree_lift<PCG>": 8 * M + 20 * lv1,
        # parent0T 4 + r 4 + mu0 4 + (d,n) rw 16 + x rw 8 (level-1 gathers cache-resident)
        "k_tree_level0<PCG>": 36 * M,
        "k_update": 36 * M,            # x rw 8 + r rw 8 + (d,n) 8 + q 4 + mu0 4 + s write 4
        "k_direction2": 20 * M,        # s 4 + (d,n) read 8 + (d,n) write 8
        "k_bistoch": 28 * M,           # nbr 16 + m 4 + n 4 + n write 4
        "k_grid_sort": 4 * N,          # rgb 3 + perm 1 per px (+ 12 B per cell)
        "k_grid_write": 8 * N + 12 * M,  # perm 1 + rgb 3 (heads) + vid 4 per px; key 8 + m 4 per vertex
        "k_grid_neighbours": 24 * M,   # keys 8 + nbr write 16
        "k_splat<true>": 12 * N + 8 * M,  # vid 4 + c 4 + t 4 per px; Sc, b per vertex
        "k_slice": 8 * N,              # vid 4 + x 4 per px
        "k_slice4": 8 * N,             # the same, 4 px per thread
    }
    return table.get(name)


def hbm_peak():
    """(GB/s, source): MEASURED_PEAKS.json's measured copy bandwidth, else the profiling guide's
    fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return 6650.0, "B200_PROFILING.md fallback"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["fbs", "reference"], default="fbs")
    ap.add_argument("--frames-per-gpu", type=int, default=8)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check without CUDA: shard the frames over the ranks (gloo), reduce a fake "
                         "per-rank time with the max-over-ranks path and print what each rank owns")
    return ap.parse_args()


def _free_port() -> int:
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def relaunch(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-exec this script as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1, exactly as the driver would launch it, and pass rank 0's
    JSON line through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def run_dry(args, rank, world) -> int:
    """--dry-run: the multi-rank plumbing of the real arm (shard_frames, reduce_max, rank-0 print)
    over gloo, with rank r reporting a fake device time of 1 + r ms."""
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    frames = shard_frames(rank, args.frames_per_gpu)
    ms = reduce_max(1.0 + rank, world)
    owned = [None] * world
    if world > 1:
        dist.all_gather_object(owned, frames)
    else:
        owned = [frames]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "gpus_requested": args.gpus, "frames": owned,
                          "max_ms": ms, "config": workload_config(args, world)}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms during the timed region."""

    Q = ("uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, uuid: str):
        self.uuid = uuid
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons, n = [], [], set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or (self.uuid and self.uuid not in f[0]):
                continue
            n += 1
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        loaded = [s for s in sm if smax and s > 0.5 * max(smax)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons), "samples": n}


# --------------------------------------------------------------------------- reference arm
def oracle_run(w):
    import oracle as O
    opts = O.SolveOptions(precond=w.precond, init=w.init, mode=w.mode, iters=w.iters, n_bistoch=w.n_bistoch)
    t0 = time.perf_counter()
    O.solve(w.rgb, w.t, w.c, w.sigma_xy, w.sigma_l, w.sigma_uv, w.lam, opts)
    return time.perf_counter() - t0


def _oracle_worker(frame, W, H, barrier, out):
    """One frame of the workload through the oracle in its own process, timed after a barrier so
    that all workers solve concurrently."""
    from threadpoolctl import threadpool_limits
    from workloads import make
    w = make("c5", frames=1, first_frame=frame, W=W, H=H)
    barrier.wait()
    with threadpool_limits(1):
        out[frame] = oracle_run(w)


def oracle_all_cores(frames, W, H):
    """The oracle frame-parallel over host processes (SURVEY.md §8(d) 'all cores'): P frames at
    once, P = min(cores, frames); returns (MP/s over the slowest worker, P, seconds)."""
    import multiprocessing as mp
    P = max(1, min(os.cpu_count() or 1, frames))
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(P)
    out = ctx.Manager().dict()
    procs = [ctx.Process(target=_oracle_worker, args=(f, W, H, barrier, out)) for f in range(P)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join()
    sec = max(out.values())
    return P * W * H / 1e6 / sec, P, sec


def oracle_sample(args, frame, crop):
    """Bounded sample of the workload for the CPU oracle: a crop of one frame."""
    from workloads import make
    W, H = crop
    return make("c5", frames=1, first_frame=frame, W=W, H=H)


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from threadpoolctl import threadpool_limits
    crop = (min(args.width, 960), min(args.height, 540))
    w = oracle_sample(args, 0, crop)
    with threadpool_limits(1):
        for _ in range(args.warmup):
            oracle_run(w)
        times = [oracle_run(w) for _ in range(args.steps)]
    ms = 1e3 * sum(times) / len(times)
    value = w.pixels / 1e6 / (ms / 1e3)
    sample = f"frame 0 of c5_batch cropped to {crop[0]}x{crop[1]} (seed 5000), hier+hier, 25 PCG iters, fp64 oracle"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "MP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world),
            "cpu_baseline": {"value": value, "unit": "MP/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, world=1):
    return {"workload": f"c5_batch: {args.frames_per_gpu} independent {args.width}x{args.height} RGB frames per GPU "
                        f"(300-cell Voronoi + gradients + noise 3, planar depth with 5% outliers), "
                        f"sigma=(8,4,3), lambda=128, Alg.1 x20, hier precond+init, {ITERS} PCG iters, K=1",
            "frames_per_gpu": args.frames_per_gpu, "width": args.width, "height": args.height,
            "parallelism": f"frames sharded over {world} rank(s) (one per GPU), no collective on the solve path",
            "l2": "inputs larger than L2 (rgb+t+c = 11 B/px, 182 MB per GPU-step > 126 MB L2)"}


# --------------------------------------------------------------------------- sharding
def shard_frames(rank: int, per_gpu: int):
    """Frames of configs[4] owned by `rank`: [rank·per_gpu, (rank+1)·per_gpu).
    Frames are independent systems, so no data-path collective is needed."""
    return list(range(rank * per_gpu, (rank + 1) * per_gpu))


def reduce_max(value: float, world: int, device=None) -> float:
    """Max over ranks (device-timed ms), outside the timed region."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------- main arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not (args.impl == "reference" and not args.dry_run):
        return relaunch(args)  # one process per GPU, as the driver's torchrun launch
    if world != args.gpus and args.impl != "reference":
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks")
    if args.dry_run:
        return run_dry(args, rank, world)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_1511_03296_b200 as fbs
    from workloads import make

    F = args.frames_per_gpu
    frames = shard_frames(rank, F)
    w = make("c5", frames=F, first_frame=frames[0], W=args.width, H=args.height)
    rgb_h = torch.from_numpy(w.rgb).pin_memory()
    t_h = torch.from_numpy(w.t).pin_memory()
    c_h = torch.from_numpy(w.c).pin_memory()
    rgb_d, t_d, c_d = rgb_h.to(dev), t_h.to(dev), c_h.to(dev)
    x_d = torch.empty_like(t_d)
    x_h = torch.empty_like(t_h).pin_memory()
    stream = torch.cuda.current_stream()

    def step():
        g = fbs.grid_build(rgb_d, *SIGMAS, n_bistoch=20)
        fbs.solve(g, t_d, c_d, LAM, precond="hier", init="hier", mode="fixed", iters=ITERS, out=x_d)
        g.close()
        return g

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        return reduce_max(v, world, dev)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device time, CUDA events on the launching stream)
    uuid = str(torch.cuda.get_device_properties(dev).uuid) if hasattr(torch.cuda.get_device_properties(dev), "uuid") else ""
    clocks = ClockSampler(uuid)
    clocks.start()
    barrier()
    l0 = fbs.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = fbs.launch_count() - l0
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(ms)
    pixels_all = w.pixels * world
    value = pixels_all / 1e6 / (ms / 1e3 / args.steps)

    # ---- the same step captured once into a CUDA graph and replayed (the build and the FIXED-mode
    # solve only enqueue work, so the whole step is capturable); device time of K replays
    graph_line = None
    try:
        cs = torch.cuda.Stream(dev)
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            step()
        stream.wait_stream(cs)
        torch.cuda.synchronize()
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg):
            step()
        cg.replay()
        torch.cuda.synchronize()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            cg.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        gms = max_over_ranks(g0.elapsed_time(g1))
        graph_line = {"value": pixels_all / 1e6 / (gms / 1e3 / args.steps), "unit": "MP/s",
                      "ms_per_step": gms / args.steps,
                      "note": "grid build + solve + release captured once with torch.cuda.graph and replayed"}
        del cg
    except Exception as exc:  # noqa: BLE001 (reported, not fatal)
        graph_line = {"error": str(exc)[:200]}

    # ---- per-kernel device times over a second pass of the same K steps (events per launch)
    g_info = fbs.grid_build(rgb_d, *SIGMAS, n_bistoch=20)
    M = g_info.M
    info = g_info.info()
    g_info.close()
    fbs.profile_reset()
    fbs.profile_enable(True)
    barrier()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        step()
    p1.record(stream)
    torch.cuda.synchronize()
    fbs.profile_enable(False)
    prof = fbs.profile_report()
    prof_ms = p0.elapsed_time(p1)
    kernels = {k: {"launches": n, "ms_per_step": tot / args.steps, "avg_us": 1e3 * tot / max(n, 1)}
               for k, (n, tot) in sorted(prof.items(), key=lambda kv: -kv[1][1])}
    roof = None
    lv = [int(x) for x in info["level_vertices"]]
    # Frame groups run concurrently on their own streams: the FIXED-mode PCG in G groups (api.cu
    # run_pcg) and Alg. 1 in Gb groups (fbs_grid_build).  A grouped launch covers 1/G of the
    # vertices (on average over the groups) and shares the SMs with the other groups' launches, so
    # its per-launch rate is a lower bound on the kernel's own, and the summed event times of a
    # grouped kernel overstate its share of the step G-fold (wall share ≈ sum / G).
    G = max(1, min(int(os.environ.get("FBS_PCG_GROUPS", "2") or 2), w.frames))
    Gb = max(1, min(int(os.environ.get("FBS_BS_GROUPS", "2") or 2), w.frames))
    PCG_GROUPED = ("k_spmv2", "k_hier_level0<UPDATE>", "k_tree_lift<PCG>", "k_tree_coarse<PCG>", "k_tree_level0<PCG>",
                   "k_hier_level0<UPDATE,LAST>", "k_hier_level0<RESID>", "k_init_scalars")

    def groups_of(k):
        return G if k in PCG_GROUPED else (Gb if k == "k_bistoch" else 1)

    def launch_bytes(k):
        gk = groups_of(k)
        return kernel_bytes(k, M / gk, [x / gk for x in lv], w.pixels)

    for k, v in kernels.items():
        v["frame_groups"] = groups_of(k)
        v["wall_share_ms_per_step"] = v["ms_per_step"] / groups_of(k)
    cand = [(k, v) for k, v in kernels.items() if launch_bytes(k) is not None]
    if cand:
        # the dominant kernel = the largest (wall) share of the step among kernels with a byte model
        kname, kv = max(cand, key=lambda kv_: kv_[1]["wall_share_ms_per_step"])
        bytes_launch = launch_bytes(kname)
        achieved = bytes_launch / (kv["avg_us"] * 1e-6) / 1e9
        peak, peak_src = hbm_peak()
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
                traffic = json.load(fh).get(kname)
        except Exception:
            pass
        gk = groups_of(kname)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kname, "bytes_per_launch": bytes_launch,
                "vertices_per_launch": M / gk, "frame_groups": gk,
                "avg_launch_us": kv["avg_us"],
                "share_of_step": kv["wall_share_ms_per_step"] / (prof_ms / args.steps),
                "peak_source": peak_src}
        if gk > 1:
            roof["note"] = (f"{gk} frame groups run their launches concurrently on {gk} streams; the average "
                            "launch duration includes sharing the SMs with the other groups' launches "
                            "(traffic: one launch of the 4-frame ncu capture, profiles/traffic.json)")
    for k, v in kernels.items():
        b = launch_bytes(k)
        if b is not None:
            v["algorithmic_GBps"] = b / (v["avg_us"] * 1e-6) / 1e9
    def stage_of(name):
        for prefix, st in (("k_axis_bins", "grid_build"), ("k_bin_lut", "grid_build"), ("k_grid_", "grid_build"),
                           ("k_scan_excl", "grid_build"),
                           ("k_bistoch", "bistochastize"),
                           ("k_pyr_", "pyramid"), ("k_tree_top", "pyramid"),
                           ("k_tree_down", "pyramid"), ("k_tree_finish", "pyramid"),
                           ("k_tree_anc_mult", "splat_assemble_init"), ("k_tree_anc", "pyramid"),
                           ("k_splat", "splat_assemble_init"), ("k_assemble", "splat_assemble_init"),
                           ("k_fill_init_w0", "splat_assemble_init"),
                           ("k_tree_lift<PDA>", "splat_assemble_init"),
                           ("k_tree_coarse<PDA>", "splat_assemble_init"), ("k_tree_lift<INIT>", "splat_assemble_init"),
                           ("k_tree_coarse<INIT>", "splat_assemble_init"), ("k_tree_level0<INIT>", "splat_assemble_init"),
                           ("k_spmv2", "pcg"), ("k_update", "pcg"), ("k_direction2", "pcg"), ("k_residual0", "pcg"),
                           ("k_init_scalars", "pcg"), ("k_hier_level0", "pcg"), ("k_tree_", "pcg"),
                           ("k_slice", "slice")):
            if name.startswith(prefix):
                return st
        return "other"

    stages_ms = {}
    for k, v in kernels.items():
        st = stage_of(k)
        stages_ms[st] = stages_ms.get(st, 0.0) + v["ms_per_step"]
    for st in ("grid_build", "bistochastize", "pyramid", "splat_assemble_init", "pcg", "slice"):
        stages_ms.setdefault(st, 0.0)
    # Grouped stages (Alg. 1, PCG) overlap their groups, so their summed launch times exceed their
    # share of the step: their wall times are measured directly, as differences of device-timed
    # calls — grid build with 20 vs 0 Alg. 1 iterations, solve with 25 vs 1 PCG iterations.
    stages_ms["pcg_kernel_time_sum"] = stages_ms.pop("pcg")
    stages_ms["bistochastize_kernel_time_sum"] = stages_ms.pop("bistochastize")

    def dev_time(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        for _ in range(reps):
            fn()
        b_.record(stream)
        torch.cuda.synchronize()
        return a_.elapsed_time(b_) / reps

    def gb(nb):
        def f():
            # without the pyramid, which otherwise runs beside Alg. 1 on a side stream and would
            # hide in the 20-iteration build but not in the 0-iteration one
            gx = fbs.grid_build(rgb_d, *SIGMAS, n_bistoch=nb, build_pyramid=False)
            gx.close()
        return f

    def wall_diff(fa, fb, rounds=5):  # median over interleaved rounds: one round is noisy (±10 %)
        return max(0.0, float(np.median([dev_time(fa) - dev_time(fb) for _ in range(rounds)])))

    bs_wall = wall_diff(gb(20), gb(0))
    g_w = fbs.grid_build(rgb_d, *SIGMAS, n_bistoch=20)

    def sv(iters):
        return lambda: fbs.solve(g_w, t_d, c_d, LAM, precond="hier", init="hier", mode="fixed", iters=iters, out=x_d)

    pcg24 = wall_diff(sv(ITERS), sv(1))
    g_w.close()
    stages_ms["bistochastize_wall"] = bs_wall
    stages_ms["pcg_wall_per_iteration"] = pcg24 / (ITERS - 1)
    it_bytes = sum(kernel_bytes(k, M, lv, w.pixels) for k in
                   ("k_spmv2", "k_hier_level0<UPDATE>", "k_tree_lift<PCG>", "k_tree_level0<PCG>"))
    pcg_iteration_rate = {"algorithmic_bytes": it_bytes, "GBps": it_bytes / (pcg24 / (ITERS - 1) * 1e-3) / 1e9,
                          "frac": it_bytes / (pcg24 / (ITERS - 1) * 1e-3) / 1e9 / hbm_peak()[0],  # of the measured copy bandwidth
                          "note": "one PCG iteration over all frames (both groups): spmv + update + lift + level0 "
                                  "byte models (coarse levels unmodelled) over its wall time, measured as "
                                  "(solve with 25 iterations - solve with 1) / 24, median of 5 interleaved rounds"}
    # SURVEY.md §8(d)'s floor for one hierarchical PCG iteration: s + 4 + 32K B per level-0 vertex
    # (s = 16 B neighbour structure; diag/M⁻¹; x, r, d read+write; q round trip) plus the
    # hierarchy's 2·r·(4K + 4) + 4r with r = Σ_{k≥0} M_k / M (lift + project + μ over all levels,
    # level 0 included: ≈ 1.23 in the survey), K = 1
    r_lv = sum(lv) / max(M, 1)
    floor_bpv = 16 + 4 + 32 + 2 * r_lv * 8 + 4 * r_lv
    t_it = pcg24 / (ITERS - 1) * 1e-3
    pcg_iteration_rate["floor_bytes"] = floor_bpv * M
    pcg_iteration_rate["floor_bytes_per_vertex"] = floor_bpv
    pcg_iteration_rate["modelled_bytes_per_vertex"] = it_bytes / max(M, 1)
    pcg_iteration_rate["floor_GBps"] = floor_bpv * M / t_it / 1e9
    pcg_iteration_rate["floor_frac"] = floor_bpv * M / t_it / 1e9 / hbm_peak()[0]
    pcg_iteration_rate["modelled_over_floor"] = it_bytes / max(floor_bpv * M, 1)
    bistoch_rate = {"algorithmic_bytes": kernel_bytes("k_bistoch", M, lv, w.pixels),
                    "GBps": 20 * kernel_bytes("k_bistoch", M, lv, w.pixels) / (bs_wall * 1e-3) / 1e9 if bs_wall else None,
                    "note": "one Alg. 1 iteration over all frames (all groups) over its wall time, measured as "
                            "(grid build with 20 iterations - grid build with 0) / 20, both without the pyramid"}
    if bistoch_rate["GBps"]:
        bistoch_rate["frac"] = bistoch_rate["GBps"] / hbm_peak()[0]
    # the other stages against their algorithmic bytes (DESIGN §7 byte models; summed launch times,
    # single-stream stages): grid build (sort + write + neighbours) and slice
    stage_rates = {}
    for st, names in (("grid_build", ("k_grid_sort", "k_grid_write", "k_grid_neighbours")), ("slice", ("k_slice4",))):
        ms_ = sum(kernels[n]["ms_per_step"] for n in names if n in kernels)
        by_ = sum(kernel_bytes(n, M, lv, w.pixels) for n in names if n in kernels)
        if ms_ > 0:
            stage_rates[st] = {"ms": ms_, "algorithmic_bytes": by_, "GBps": by_ / (ms_ * 1e-3) / 1e9,
                               "frac": by_ / (ms_ * 1e-3) / 1e9 / hbm_peak()[0]}

    # ---- end to end through the public API with host buffers: every step copies its inputs H2D from
    # pinned memory and its result D2H inside the timed region.  Double-buffered: the H2D of step
    # i+1 and the D2H of step i run on their own streams, overlapping step i's compute (a video
    # pipeline); the timed region ends when the last result is on the host.
    e2e = None
    if not args.no_e2e:
        s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        bufs = [(rgb_d, t_d, c_d, x_d),
                (torch.empty_like(rgb_d), torch.empty_like(t_d), torch.empty_like(c_d), torch.empty_like(x_d))]
        x_hs = [x_h, torch.empty_like(x_h).pin_memory()]
        ev_rgb = [torch.cuda.Event() for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_comp = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def step_on(slot):
            rgb_b, t_b, c_b, x_b = bufs[slot]
            # the grid build needs only the reference image; t and c (72 % of the upload) are
            # waited for just before the solve, so the first step's build overlaps their copy
            stream.wait_event(ev_rgb[slot])
            g = fbs.grid_build(rgb_b, *SIGMAS, n_bistoch=20)
            stream.wait_event(ev_in[slot])
            fbs.solve(g, t_b, c_b, LAM, precond="hier", init="hier", mode="fixed", iters=ITERS, out=x_b)
            g.close()

        def h2d(i):
            # inputs of step i into slot i % 2, once step i − 2 (the slot's last reader) is done
            slot = i % 2
            rgb_b, t_b, c_b, _ = bufs[slot]
            with torch.cuda.stream(s_h2d):
                if i >= 2:
                    s_h2d.wait_event(ev_comp[slot])
                rgb_b.copy_(rgb_h, non_blocking=True)
                ev_rgb[slot].record(s_h2d)
                t_b.copy_(t_h, non_blocking=True)
                c_b.copy_(c_h, non_blocking=True)
                ev_in[slot].record(s_h2d)

        def run_e2e(nsteps):
            # The H2D of step i + 1 is enqueued before step i's compute (the grid build's host
            # synchronisations would otherwise delay it until step i is mostly enqueued), so
            # it overlaps all of step i; the D2H of step i overlaps step i + 1.
            h2d(0)
            for i in range(nsteps):
                slot = i % 2
                x_b = bufs[slot][3]
                if i + 1 < nsteps:
                    h2d(i + 1)
                if i >= 2:
                    stream.wait_event(ev_out[slot])  # the D2H of step i-2 has drained x_b
                step_on(slot)
                ev_comp[slot].record(stream)
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(ev_comp[slot])
                    x_hs[slot].copy_(x_b, non_blocking=True)
                    ev_out[slot].record(s_d2h)
            stream.wait_event(ev_out[(nsteps - 1) % 2])
            if nsteps > 1:
                stream.wait_event(ev_out[(nsteps - 2) % 2])

        run_e2e(2)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s_h2d.wait_event(e0)
        run_e2e(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1))
        h2d = rgb_h.numel() + 4 * t_h.numel() + 4 * c_h.numel()
        e2e = {"value": pixels_all / 1e6 / (ems / 1e3 / args.steps), "unit": "MP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(4 * x_h.numel()),
               "ms_per_step": ems / args.steps,
               "pipelining": "double-buffered: the H2D of step i+1 (enqueued before step i) and the D2H of step i-1 "
                              "run on their own streams while step i computes; each step's grid build waits for its "
                              "reference image only, its solve for t and c"}

    # ---- §8(f) rows on the same GPU (device time, not part of `value`): the domain-transform
    # post-filter of this workload's output, the robust solver per IRLS round on it, and
    # configs[3] (21 channels, 500×375) solved in full vs with the low-rank reduction (ε = 0.01)
    extras = None
    if not args.no_extras and rank == 0:
        def dev_ms(fn, reps=3):
            fn()
            torch.cuda.synchronize()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            for _ in range(reps):
                fn()
            b_.record(stream)
            torch.cuda.synchronize()
            return a_.elapsed_time(b_) / reps

        g_x = fbs.grid_build(rgb_d, *SIGMAS, n_bistoch=20)
        fbs.solve(g_x, t_d, c_d, LAM, precond="hier", init="hier", mode="fixed", iters=ITERS, out=x_d)
        dt_ms = dev_ms(lambda: fbs.dt_filter(rgb_d, x_d, 16.0, 16.0))
        rb_ms = dev_ms(lambda: fbs.solve_robust(g_x, t_d, c_d, LAM, 10.0, 2, precond="hier", init="hier",
                                                mode="fixed", iters=ITERS, out=x_d), reps=2) / 2
        g_x.close()
        w4 = make("c4")
        rgb4, t4, c4 = (torch.from_numpy(a_).to(dev) for a_ in (w4.rgb, w4.t, w4.c))
        g4 = fbs.grid_build(rgb4, w4.sigma_xy, w4.sigma_l, w4.sigma_uv)
        full_ms = dev_ms(lambda: fbs.solve(g4, t4, c4, w4.lam, precond="hier", init="hier", mode="tol", tol=1e-6))
        lr_ms = dev_ms(lambda: fbs.solve(g4, t4, c4, w4.lam, precond="hier", init="hier", mode="tol", tol=1e-6,
                                         lowrank_eps=0.01))
        # the case the reduction is for: 21 channels that are mixtures of 4 underlying maps
        rng4 = np.random.default_rng(21)
        basis = w4.t[:, :4]
        mix = rng4.uniform(0, 1, (21, 4)).astype(np.float32)
        t4r = torch.from_numpy(np.ascontiguousarray(np.einsum("kj,fjhw->fkhw", mix, basis))).to(dev)
        full_r_ms = dev_ms(lambda: fbs.solve(g4, t4r, c4, w4.lam, precond="hier", init="hier", mode="tol",
                                             tol=1e-6))
        lr_r_ms = dev_ms(lambda: fbs.solve(g4, t4r, c4, w4.lam, precond="hier", init="hier", mode="tol",
                                           tol=1e-6, lowrank_eps=0.01))
        g4.close()
        # the reduction at scale: 2 frames of the workload with 21 channels mixed from 4 planar maps,
        # hier+hier fixed 25 — the full solve's channel-split kernels scale with K here, the reduced
        # one solves t_f ≈ 4 live channels (Supp. §4)
        w2 = make("c5", frames=2, W=args.width, H=args.height)
        rng2 = np.random.default_rng(22)
        maps = np.stack([w2.t[:, 0], np.clip(w2.t[:, 0] * 0.5 + 40, 0, 255), 255 - w2.t[:, 0],
                         rng2.uniform(0, 1, w2.t[:, 0].shape).astype(np.float32) * 10], axis=1)
        mix2 = rng2.uniform(0, 1, (21, 4)).astype(np.float32)
        t21 = torch.from_numpy(np.ascontiguousarray(np.einsum("kj,fjhw->fkhw", mix2, maps))).to(dev)
        rgb2, c2 = torch.from_numpy(w2.rgb).to(dev), torch.from_numpy(w2.c).to(dev)
        g2 = fbs.grid_build(rgb2, *SIGMAS, n_bistoch=20)
        big_full_ms = dev_ms(lambda: fbs.solve(g2, t21, c2, LAM, precond="hier", init="hier", mode="fixed", iters=ITERS))
        big_lr_ms = dev_ms(lambda: fbs.solve(g2, t21, c2, LAM, precond="hier", init="hier", mode="fixed", iters=ITERS,
                                             lowrank_eps=0.01))
        g2.close()
        del t21
        # the other BASELINE.json configs as specified (grid build + solve [+ backward for configs[3]]),
        # device time per call; TOL-mode solves include the host's active-count polls
        cfg_rows = {}
        # configs[2] is run both ways BASELINE.json names: fixed 25 (c3) and to tol 1e-6 (c3_tol)
        for name, over in (("c1", {}), ("c2", {}), ("c3", {}), ("c3_tol", {"mode": "tol", "max_iters": 5000}),
                           ("c4", {})):
            wc = make(name.split("_")[0])
            if over:
                import dataclasses
                wc = dataclasses.replace(wc, **over)
            rgbc, tc, cc = (torch.from_numpy(a_).to(dev) for a_ in (wc.rgb, wc.t, wc.c))
            gc_ = torch.from_numpy(wc.g).to(dev) if wc.g is not None else None
            opts = dict(precond=wc.precond, init=wc.init, mode=wc.mode, tol=wc.tol, max_iters=wc.max_iters)
            if wc.mode == "fixed":
                opts["iters"] = wc.iters

            # the pyramid only serves the hierarchical preconditioner / init (Jacobi configs skip it)
            pyr = wc.precond == "hier" or wc.init == "hier"

            def run_cfg():
                gg = fbs.grid_build(rgbc, wc.sigma_xy, wc.sigma_l, wc.sigma_uv, n_bistoch=wc.n_bistoch,
                                    build_pyramid=pyr)
                if gc_ is not None:
                    _, S_ = fbs.solve(gg, tc, cc, wc.lam, keep_system=True, **opts)
                    S_.backward(gc_, tc, cc)
                    S_.close()
                else:
                    fbs.solve(gg, tc, cc, wc.lam, **opts)
                gg.close()

            ms_c = dev_ms(run_cfg)
            graph_ms = None
            if True:  # every step is enqueue-only inside a capture (TOL: a device-side loop): as a CUDA graph
                try:
                    cs2 = torch.cuda.Stream(dev)
                    cs2.wait_stream(stream)
                    with torch.cuda.stream(cs2):
                        run_cfg()
                    stream.wait_stream(cs2)
                    torch.cuda.synchronize()
                    gq = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gq):
                        run_cfg()
                    graph_ms = dev_ms(gq.replay, reps=10)
                    del gq
                except Exception:  # noqa: BLE001
                    graph_ms = None
            gg = fbs.grid_build(rgbc, wc.sigma_xy, wc.sigma_l, wc.sigma_uv, n_bistoch=wc.n_bistoch,
                                build_pyramid=pyr)
            _, S_ = fbs.solve(gg, tc, cc, wc.lam, keep_system=True, **opts)
            pcg_its = int(S_.stats()["iterations"].max())
            S_.close()
            gg.close()
            cfg_rows[name] = {"ms": ms_c, "MP_per_s": wc.pixels / 1e6 / (ms_c / 1e3), "pcg_iterations": pcg_its,
                              "graph_ms": graph_ms,
                              "shape": f"{wc.frames}x{wc.H}x{wc.W}, K={wc.K}",
                              "pyramid_built": pyr,
                              "solver": f"{wc.precond}+{wc.init}, " +
                                        (f"fixed {wc.iters} it" if wc.mode == "fixed" else f"tol {wc.tol:g}") +
                                        (", + backward" if gc_ is not None else "")}
        # configs[4] also to tol 1e-6 ("tol 1e-6 also reported"); TOL mode runs
        # the frames in one group (the host polls the active count)
        def c5_tol():
            gt = fbs.grid_build(rgb_d, *SIGMAS, n_bistoch=20)
            fbs.solve(gt, t_d, c_d, LAM, precond="hier", init="hier", mode="tol", tol=1e-6, out=x_d)
            gt.close()

        tol_ms = dev_ms(c5_tol)
        gt = fbs.grid_build(rgb_d, *SIGMAS, n_bistoch=20)
        _, St = fbs.solve(gt, t_d, c_d, LAM, precond="hier", init="hier", mode="tol", tol=1e-6, keep_system=True)
        tol_its = [int(v) for v in St.stats()["iterations"].ravel()]
        St.close()
        gt.close()
        cfg_rows["c5_tol"] = {"ms": tol_ms, "MP_per_s": w.pixels / 1e6 / (tol_ms / 1e3), "pcg_iterations": tol_its,
                              "shape": f"{F}x{args.height}x{args.width}, K=1", "solver": "hier+hier, tol 1e-06"}
        extras = {"configs": cfg_rows,
                  "dt_post_filter_ms": dt_ms,
                  "dt_post_filter": f"{F} frames x1, sigma'_xy = sigma'_rgb = 16, 3 iterations (PAPER.md:329)",
                  # algorithmic bytes: per pixel 11 (distances: rgb 3, Dx, Dy 8) + 8 (input
                  # copied to the output) + 3 iterations × 2 passes × 12 (value read + write, weight read)
                  "dt_post_filter_rate": {"bytes_per_pixel": 91, "GBps": 91 * w.pixels / (dt_ms / 1e3) / 1e9,
                                          "frac": 91 * w.pixels / (dt_ms / 1e3) / 1e9 / hbm_peak()[0]},
                  "robust_ms_per_irls_round": rb_ms,
                  "robust": f"{F} frames, sigma_gm = 10, hier+hier, {ITERS} PCG iters per round (Supp. Alg. 3)",
                  "configs3_full_solve_ms": full_ms, "configs3_lowrank_solve_ms": lr_ms,
                  "rank4_full_solve_ms": full_r_ms, "rank4_lowrank_solve_ms": lr_r_ms,
                  "rank4": "configs[3]'s grid with 21 channels mixed from 4 of its target maps: full vs eps = 0.01",
                  "rank4_2frames_full_solve_ms": big_full_ms, "rank4_2frames_lowrank_solve_ms": big_lr_ms,
                  "rank4_2frames": f"2 workload frames ({args.width}x{args.height}), 21 channels mixed from 4 maps, "
                                   "hier+hier fixed 25: full vs eps = 0.01 (solve only)",
                  "lowrank": "configs[3] 500x375, K = 21, hier+hier to tol 1e-6: full vs eps = 0.01 (Supp. §4)"}

    # ---- CPU baseline: the oracle as it stands, one frame, host cores (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from threadpoolctl import threadpool_limits
        wf = make("c5", frames=2, first_frame=0, W=args.width, H=args.height)
        with threadpool_limits(1):
            sec = oracle_run(wf)
        cpu = {"value": wf.pixels / 1e6 / sec, "unit": "MP/s", "cores": 1, "kind": "oracle",
               "sample": f"frames 0-1 of the workload ({args.width}x{args.height}), fp64 numpy/scipy oracle, "
                         f"hier+hier, 25 PCG iters, single thread ({sec:.1f} s)"}
        mps_all, P, sec_all = oracle_all_cores(args.frames_per_gpu, args.width, args.height)
        cpu_all = {"value": mps_all, "unit": "MP/s", "cores": P, "kind": "oracle",
                   "sample": f"frames 0-{P - 1} of the workload, one single-threaded oracle process per frame, "
                             f"all solving at once ({sec_all:.1f} s for the slowest)"}
        cpu["all_cores"] = cpu_all

    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "MP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": workload_config(args, world) | {"vertices_per_gpu": M,
                                                   "levels": int(info["levels"])},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "extras": extras,
                "graph": graph_line,
                "clocks": clk, "stages_ms_per_step": stages_ms, "pcg_iteration_rate": pcg_iteration_rate,
                "bistoch_iteration_rate": bistoch_rate, "stage_rates": stage_rates, "kernels": kernels,
                "profiled_ms_per_step": prof_ms / args.steps}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
