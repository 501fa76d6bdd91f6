#!/usr/bin/env python
"""bench.py — throughput of the batched PNCG-IPC tactile step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one pass of the whole hot path for every env
of the rank: tac_step (fixed 50 PNCG iterations, the paper's "tens") +
tac_markers.  Timed window: steps [W, W+K) (default 16-63) from a
checkpoint taken after the W warm-up steps; the per-kernel profile and e2e passes replay the
same window from the same checkpoint.  Workload at N=1: BASELINE configs[2] (C3: 1,024 envs of peg-insertion
trajectories on the 19,800-tet GelSight-Mini-like pad).  N>1 (torchrun): weak scaling,
1,024 envs per GPU with distinct env ids, plus an NCCL all-gather of the marker fields
every step (configs[3], C4).  Timing: CUDA events on the stream, barrier + synchronize
on both sides, max over ranks.  The per-env state (~470 MB/GPU) exceeds the 126 MB L2,
so no L2 flush is needed between steps.

--impl reference times the fp64 CPU oracle (oracle/) on this host as the reference
arm (the paper's code is not available).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FIXED_ITERS = 50
ENVS_PER_GPU = 1024
METRIC = "env-steps/sec (marker fields/sec) at 1/2/4/8 B200; % of HBM roofline"
WORKLOADS = {
    "c3": "C3: 1024 envs/GPU peg-insertion trajectories (press, shear, twist, release), 19,800-tet / 4,278-vertex pad, "
          "8 mm diameter cylinder peg, 7x9 markers",
    "c3u": "C3 on the unstructured pad (jittered interior, random vertex/tet numbering; SURVEY 8f-1)",
    "c5": "C5 stress: 103,680-tet / 19,943-vertex pad, sharp 8x8 mm square peg (face / edge press, slide, twist)",
    "c2": "C2: 1 env, GelSight-Mini-like 19,800-tet pad, R 5 mm icosphere: normal press + shear slide + retract, "
          "50 steps (latency-bound; ms_per_step is the step latency)",
    "c1": "C1: 1 env, 288-tet pad, R 3 mm icosphere pressed 0.5 mm in one step from 0.2 mm above; every bench "
          "step is that solve again from rest (tac_reset to the initial pose inside the timed region; latency)",
}


def make_scene(config, n_envs, n_steps, seed0):
    """The workload of `config` (workloads/ generators; env ids from seed0)."""
    import workloads as w
    if config == "c5":
        return w.scene_c5(n_envs=n_envs, n_steps=n_steps, seed0=20270000 + seed0)
    if config == "c3u":
        return w.scene_c3_unstructured(n_envs=n_envs, n_steps=n_steps, seed0=20260000 + seed0)
    if config == "c2":
        assert n_envs == 1, "C2 is a single-env config"
        return w.scene_c2(steps=n_steps)
    if config == "c1":
        assert n_envs == 1, "C1 is a single-env config"
        s = w.scene_c1()
        s.poses = np.repeat(s.poses[:1], n_steps, axis=0)  # the same press solved every step, from rest
        return s
    return w.scene_c3(n_envs=n_envs, n_steps=n_steps, seed0=20260000 + seed0)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws == 1 and not os.environ.get("TAC_FORCE_DIST"):
        return 0, 0, 1
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    import torch
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return rank, local, ws


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        load = [s for s in sm if s > 300] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if "Active" in v and "Not" not in v:
                    reasons.add(n)
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": float(rows[0][2]), "reasons": sorted(reasons),
                "samples": len(rows)}


# algorithmic work per env-iteration (DESIGN.md §Kernels and roofline): a
# kernel's work in the window = this x the env-iterations it processed (fixed mode: every env
# every iteration; tolerance mode: the envs still iterating)
def kernel_models(nv_free, nt):
    return {
        "elem_grad": ("alu", 350.0 * nt, "flop", "350 flop per tet per env-iteration (SURVEY §8d.2 phase A)"),
        "elem_curv": ("alu", 140.0 * nt, "flop", "140 flop per tet per env-iteration (phase C)"),
        "vert_pre": ("hbm", 84.0 * nv_free, "B", "84 B per free vertex per env-iteration: read u,p,u^; write u,g,D"),
        "dir_reduce": ("hbm", 60.0 * nv_free, "B", "60 B per free vertex per env-iteration: read g,g_prev,p,D"),
        "dir_apply": ("hbm", 72.0 * nv_free, "B", "72 B per free vertex per env-iteration: read g,D,p; write p,g_prev"),
    }


def run_ours(args, rank, local, ws):
    import torch
    import paper_2603_28475_b200 as P
    import workloads as w

    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    from paper_2603_28475_b200.dist import MarkerGather, NativeMarkerGather, env_range
    nsteps = max(64, args.warmup + args.steps)  # warm-up, then the timed window [W, W + K)
    if args.scaling == "strong":  # C4 strong: a fixed total split over the ranks
        e0, e1 = env_range(rank, ws, args.total_envs)
    else:  # weak: a fixed env count per GPU, distinct env ids per rank
        e0, e1 = rank * args.envs, (rank + 1) * args.envs
    E = e1 - e0
    scene = make_scene(args.config, E, nsteps, e0)
    if args.tol is not None:  # tolerance mode (SURVEY §8d.1 timing protocol iii)
        scene.params.fixed_iters = 0
        scene.params.tol_x = args.tol
        scene.params.max_iters = args.max_iters
    else:
        scene.params.fixed_iters = args.iters
    if os.environ.get("TAC_BP_MARGIN"):  # experiments only (candidate margin sweep)
        scene.params.bp_margin = float(os.environ["TAC_BP_MARGIN"])
    sim = P.TacSim.from_scene(scene, device=local)
    poses = torch.tensor(scene.poses, dtype=torch.float32, device=dev).contiguous()  # resident in HBM
    nm = scene.markers.shape[0]
    distributed = ws > 1 or bool(os.environ.get("TAC_FORCE_DIST"))
    # N > 1 (C4): the marker fields of every rank are all-gathered in place every step --
    # through the C ABI (tac_gather_markers: tac_markers into the rank's slot + ncclAllGather
    # on the same stream) unless TAC_TORCH_GATHER selects torch.distributed's all-gather
    native = distributed and not os.environ.get("TAC_TORCH_GATHER")
    mg = NativeMarkerGather(sim, E, nm, 2, rank, ws, dev) if native else MarkerGather(E, nm, 2, rank, ws, dev)
    mk = mg.slot  # this rank's slot of the gather buffer
    gather = mg if distributed else None
    stream = torch.cuda.current_stream()
    # C1: every step solves the same press from rest (tac_reset of the env to its initial pose)
    reset_all = args.config == "c1"
    if reset_all:
        rmask = torch.ones(E, dtype=torch.uint8, device=dev)
        rposes = torch.tensor(scene.init_poses, dtype=torch.float32, device=dev).contiguous()

    def emit_markers():
        if native:
            gather.gather()
            return
        sim.markers(mk)
        if gather is not None:
            gather.gather()

    def one_step(k, pose_k=None, count=False):
        """One step of the hot path for every env of the rank; with `count`, returns its kernel
        launches (tac_last_launch_count, which synchronises in tolerance mode)."""
        if reset_all:
            sim.reset(rmask, rposes)
        sim.step(poses[k] if pose_k is None else pose_k, scene.dt)
        n = sim.last_launch_count() if count else 0
        emit_markers()
        return n + sim.last_launch_count() + (2 if reset_all else 0) if count else 0

    import torch.distributed as dist

    def barrier():
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier()

    def max_over_ranks(x):
        if dist.is_initialized():
            t = torch.tensor([x], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            x = float(t.item())
        return x

    for k in range(args.warmup):
        one_step(k)
    # the state after warm-up: all three timed passes (headline, per-kernel profile, e2e)
    # start from it and run the same window [W, W + K) of the trajectories
    ckpt = sim.checkpoint_save()
    window = range(args.warmup, args.warmup + args.steps)
    barrier()
    clocks = Clocks(local)
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    # headline timed region: device-resident inputs, no per-launch events, no host syncs
    t0.record(stream)
    for k in window:
        one_step(k)
    t1.record(stream)
    barrier()
    cl = clocks.stop()
    ms = max_over_ranks(t0.elapsed_time(t1))
    n_all = args.total_envs if args.scaling == "strong" else ws * E
    value = n_all * args.steps / (ms / 1e3)

    # profiled pass over the same window from the same state: CUDA events around every launch
    # on its stream give each kernel's live per-launch time (roofline, breakdown); the per-step
    # solver statistics of the window are read here (outside the headline timing)
    sim.checkpoint_load(ckpt)
    sim.profile_enable(True)
    sim.profile_read()
    iters_per_step, stats_per_step, flags_per_step = [], [], []
    launches = 0  # kernels of the window (the headline pass runs the same kernels)
    barrier()
    t0.record(stream)
    for k in window:
        launches += one_step(k, count=True)
        it_k, _, fl_k = sim.env_status()
        iters_per_step.append(it_k)
        flags_per_step.append(fl_k)
        stats_per_step.append(sim.env_stats())
    t1.record(stream)
    barrier()
    pms = t0.elapsed_time(t1)
    prof = sim.profile_read()
    sim.profile_enable(False)

    # roofline of the dominant kernel (live CUDA-event timing over the profiled pass)
    nfree = scene.X.shape[0] - len(scene.fixed)
    models = kernel_models(nfree, scene.tets.shape[0])
    # env-iterations of the profiled window (its per-step iteration counts): evaluations for the
    # evaluation kernels; the step's last evaluation computes no direction or curvature (R31)
    its_w = torch.stack(iters_per_step).float()
    env_its = float(its_w.sum())
    env_dirs = float((its_w - 1).clamp(min=0).sum())
    tot = {k: v for k, v in prof.items() if v[1] > 0}
    dom = max(tot, key=lambda k: tot[k][0])
    peaks, src = _peaks()
    share = {k: round(v[0] / pms, 4) for k, v in sorted(tot.items(), key=lambda kv: -kv[1][0])}
    dom_model = dom if dom in models else max((k for k in tot if k in models), key=lambda k: tot[k][0])
    bound, unit_work, wunit, note = models[dom_model]
    n_units = env_its if dom_model in ("elem_grad", "vert_pre", "dir_reduce") else env_dirs
    work = unit_work * n_units / tot[dom_model][1]  # per launch, averaged over the window
    avg_s = tot[dom_model][0] / tot[dom_model][1] / 1e3
    if bound == "hbm":
        achieved = work / avg_s / 1e9
        peak = float(peaks["hbm_gbs"])
        unit = "GB/s"
    else:
        achieved = work / avg_s / 1e12
        peak = 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
        unit = "TFLOP/s"
    roof = {"bound": bound, "kernel": dom_model, "achieved": round(achieved, 3), "peak": round(peak, 1),
            "unit": unit, "frac": round(achieved / peak, 4), "traffic": None,
            "peak_source": f"{src} ({'MEASURED_PEAKS.json hbm_gbs' if bound == 'hbm' else '148 SM x 128 FP32 lanes x 2 flop x sm_max_mhz'})",
            "work_per_launch": work, "work_note": note + f"; {n_units:.0f} env-iterations over "
                                                              f"{tot[dom_model][1]} launches in the window",
            "avg_launch_us": round(avg_s * 1e6, 2),
            "dominant_by_time": dom, "share_of_step": share,
            "timing": f"per-launch CUDA events in a second timed pass of {args.steps} steps ({pms:.1f} ms, "
                      f"{pms / ms:.3f}x the unprofiled pass that gives value)",
            "kernel_ms_total_and_launches": {k: [round(v[0], 3), v[1]] for k, v in tot.items()}}
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            tr = json.load(open(tfile)).get(dom_model)
            if tr:
                roof["traffic"] = tr
        except Exception:
            pass

    # e2e through the public API with host buffers (pinned), copies inside the timed region,
    # the same window from the same state again
    host_poses = torch.tensor(scene.poses, dtype=torch.float32).pin_memory()
    host_mk = torch.empty((E, nm, 2), dtype=torch.float32).pin_memory()
    dpose = torch.empty((E, 7), dtype=torch.float32, device=dev)
    sim.checkpoint_load(ckpt)
    barrier()
    w0 = time.perf_counter()
    for k in window:
        dpose.copy_(host_poses[k], non_blocking=True)
        one_step(k, dpose)
        host_mk.copy_(mk, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    w1 = time.perf_counter()
    e2e_s = max_over_ranks(w1 - w0)
    e2e = {"value": round(n_all * args.steps / e2e_s, 2), "unit": "env-steps/s",
           "h2d_bytes_per_step": E * 7 * 4, "d2h_bytes_per_step": E * nm * 2 * 4,
           "timing": "wall clock, steps [W, W+K) from the post-warm-up checkpoint, pinned poses H2D and marker "
                     "field D2H every step, synchronize per step (result read on host)", "steps": args.steps}

    its = torch.stack(iters_per_step).float().flatten().cpu().numpy()
    stt = torch.stack(stats_per_step).float().reshape(-1, 4)
    fls = torch.stack(flags_per_step).flatten()
    mean_it = float(its.mean())
    # whole-iteration HBM fraction (SURVEY §8d.2 "Reporting" 1): algorithmic bytes of one
    # PNCG iteration of one env (phases A + B + C per free vertex, static mesh amortised)
    b_iter = 180.0 * nfree + 112.0 * scene.tets.shape[0] / E
    hbm_it = {"bytes_per_env_iter": round(b_iter, 1),
              "achieved_gbs": round(value * mean_it * b_iter / 1e9, 1), "peak_gbs": float(peaks["hbm_gbs"]),
              "note": "180 B per free vertex per iteration (read u,p,u^; write u,g,D | read g,g_prev,p,D; write p | "
                      "read u,p) + 112 B per tet of static mesh shared by all envs; env-steps/s x mean iterations"}
    hbm_it["frac"] = round(hbm_it["achieved_gbs"] / hbm_it["peak_gbs"], 4)
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "env-steps/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32 (fp64 per-env reductions and rigid DOFs)",
        "data": "synthetic (seeded generators: workloads/)",
        "config": {"workload": WORKLOADS[args.config],
                   "envs_per_gpu": E, "total_envs": n_all, "iters_per_step": args.iters if args.tol is None else None,
                   "iteration_mode": "fixed" if args.tol is None else f"tolerance (tol_x {args.tol:g} m, max {args.max_iters})",
                   "parallelism": f"env-sharded dp{ws}" + ((" + NCCL all-gather of markers ("
                                  + (("tac_gather_markers, C ABI, " + ("torch's NCCL communicator"
                                      if type(mg.comm).__name__ == "_BorrowedComm" else "own communicator"))
                                     if native else "torch.distributed") + ")") if distributed else ""),
                   "l2": "per-env state ~470 MB/GPU > 126 MB L2 (no flush needed)"},
        "roofline": roof,
        "hbm_iteration": hbm_it,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": cl,
        "solver": {"window": f"steps [{args.warmup}, {args.warmup + args.steps}) of every env (profiled pass from "
                             "the same checkpoint)",
                   "mean_iters": mean_it, "p95_iters": float(np.percentile(its, 95)),
                   "max_iters": float(its.max()), "mean_peak_candidates": float(stt[:, 1].mean()),
                   "max_peak_candidates": int(stt[:, 1].max()), "mean_anchors": float(stt[:, 2].mean()),
                   "max_anchors": int(stt[:, 2].max()),
                   "env_steps_with_anchors": round(float((stt[:, 2] > 0).float().mean()), 4),
                   "mean_rebuilds_per_step": float(stt[:, 3].mean()),
                   "converged_env_steps": int(((fls & 1) != 0).sum()),
                   "overflow_env_steps": int(((fls & 32) != 0).sum()), "nan_env_steps": int(((fls & 12) != 0).sum()),
                   "stagnated_env_steps": int(((fls & 64) != 0).sum())},
    }
    return out, scene, sim


def cpu_baseline(config="c3", iters=FIXED_ITERS, budget_s=12.0):
    """The oracle (fp64, one env per thread on all host cores), the same fixed iteration count,
    on a bounded sample of the bench's workload: 2 x nproc envs (1 for C2), steps until
    ~budget_s of CPU time."""
    import oracle as O
    nproc = os.cpu_count() or 1
    n = 1 if config == "c2" else 2 * nproc
    s = make_scene(config, n, 64, 0)
    s.params.fixed_iters = iters
    o = O.Oracle(s)
    t0 = time.perf_counter()
    steps = 0
    while steps < 64:
        o.step(s.poses[steps], threads=nproc)
        steps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": round(n * steps / dt, 3), "unit": "env-steps/s", "cores": min(nproc, n), "kind": "oracle",
            "sample": f"{config.upper()} workload, {n} envs x {steps} steps (first steps of each trajectory), "
                      f"{iters} iterations/step, fp64 C++ oracle, one env per thread"}


def run_reference(args, rank, ws):
    if rank != 0:
        return None
    import oracle as O
    import workloads as w
    nproc = os.cpu_count() or 1
    n = nproc
    s = w.scene_c3(n_envs=n, n_steps=max(64, args.warmup + args.steps))
    s.params.fixed_iters = FIXED_ITERS
    o = O.Oracle(s)
    for k in range(args.warmup):
        o.step(s.poses[k], threads=nproc)
    t0 = time.perf_counter()
    for k in range(args.warmup, args.warmup + args.steps):
        o.step(s.poses[k], threads=nproc)
    dt = time.perf_counter() - t0
    v = n * args.steps / dt
    return {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "env-steps/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3 peg-insertion trajectories (bounded sample: one env per host core per step)",
                       "envs_per_step": n, "iters_per_step": FIXED_ITERS, "iteration_mode": "fixed"},
            "cpu_baseline": {"value": round(v, 3), "unit": "env-steps/s", "cores": nproc, "kind": "oracle",
                             "sample": f"{n} envs x {args.steps} steps, {FIXED_ITERS} iterations/step"},
            "e2e": {"value": round(v, 3), "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=48, help="timed steps (SURVEY §8d.1: steps 16-63)")
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs", type=int, default=None, help="envs per GPU (default 1024; 256 for c5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--config", default="c3", choices=["c3", "c3u", "c5", "c2", "c1"])
    ap.add_argument("--iters", type=int, default=FIXED_ITERS, help="fixed PNCG iterations per step (headline 50)")
    ap.add_argument("--tol", type=float, default=None, help="tolerance mode: tol_x [m] (SURVEY §8d.1: 1e-7)")
    ap.add_argument("--max-iters", type=int, default=2000, help="tolerance mode iteration cap")
    ap.add_argument("--total-envs", type=int, default=8192, help="strong scaling: envs over all ranks (C4)")
    args = ap.parse_args()
    assert args.warmup >= 1 and args.iters >= 1
    if args.envs is None:
        args.envs = {"c5": 256, "c2": 1, "c1": 1}.get(args.config, ENVS_PER_GPU)
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        ws = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        out = run_reference(args, rank, ws)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    rank, local, ws = _dist()
    out, scene, sim = run_ours(args, rank, local, ws)
    if rank == 0:
        if ws == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args.config, args.iters)
        else:
            out["cpu_baseline"] = None
        print(json.dumps(out), flush=True)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
