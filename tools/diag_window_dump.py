"""Find and dump same-start parity mismatches in converged C3 windows (diagnosis tool).

C3 (1,024 envs) runs in tolerance mode through step max(windows); at each window step the
GPU's start and final states of the sampled envs are compared with the oracle's step from the
same start; every env-step whose gel positions differ by more than --dump-above is saved
(start state, target, GPU final state, GPU flags / iterations) to an .npz for offline study.
Usage: python tools/diag_window_dump.py --bps 16 --envs 0:1024:8 --windows 10,20,30
"""
import argparse
import concurrent.futures as cf
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import workloads as w  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bps", type=int, default=16)
    ap.add_argument("--envs", default="0:1024:8")
    ap.add_argument("--windows", default="10,20,30")
    ap.add_argument("--gpu-tol", type=float, default=3e-10)
    ap.add_argument("--dump-above", type=float, default=1e-6)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    os.environ["TAC_CONTACT_BPS"] = str(a.bps)
    import torch
    import paper_2603_28475_b200 as P
    envs = list(range(*[int(x) for x in a.envs.split(":")]))
    wins = [int(x) for x in a.windows.split(",")]
    s = w.scene_c3(n_envs=1024, n_steps=64)
    pt = w.Params(**s.params.__dict__)
    pt.fixed_iters = 0
    pt.tol_x = a.gpu_tol
    pt.max_iters = 20000
    pt.stagnation = 5000
    p_or = w.Params(**pt.__dict__)
    p_or.tol_x = 1e-11
    sim = P.TacSim.from_scene(s, params=pt)
    poses = torch.tensor(s.poses, dtype=torch.float32, device="cuda").contiguous()
    ex = cf.ThreadPoolExecutor(1)
    jobs = []
    t0 = time.time()
    for k in range(max(wins) + 1):
        if k in wins:
            starts = {e: sim.get_state(e) for e in envs}
        sim.step(poses[k], s.dt)
        if k not in wins:
            continue
        it, pg, fl = sim.env_status()
        it, pg, fl = it.cpu().numpy(), pg.cpu().numpy(), fl.cpu().numpy()
        finals = {e: sim.get_state(e) for e in envs}

        def run(k=k, starts=starts):
            o = O.Oracle(s, params=p_or, init_poses=s.init_poses[envs])
            for j, e in enumerate(envs):
                o.set_state(j, *starts[e])
            o.step(s.poses[k][envs], threads=os.cpu_count() or 1)
            return [(o.get_state(j), o.status_of(j)) for j in range(len(envs))]
        jobs.append((k, starts, finals, it.copy(), pg.copy(), fl.copy(), ex.submit(run)))
        print(f"gpu step {k} done at {time.time() - t0:.0f} s", flush=True)
    n_bad = 0
    summary = []
    for k, starts, finals, it, pg, fl, fut in jobs:
        res = fut.result()
        du = []
        for j, e in enumerate(envs):
            (uo, vo, co, Ro), st = res[j]
            ug, vg, cg, Rg = finals[e]
            d = float(np.abs(ug - uo).max())
            du.append(d)
            stuck = not (st["flags"] & 1) and not (st["flags"] & 64 and st["pg"] <= 1e-10)
            if d > a.dump_above or stuck:
                n_bad += 1
                ut, vt, ct, Rt = starts[e]
                fn = f"gpurun_out/mismatch{a.tag}_bps{a.bps}_k{k}_e{e}.npz"
                np.savez_compressed(fn, u_t=ut, v_t=vt, c_t=ct, R_t=Rt, target=s.poses[k][e].astype(np.float64),
                                    u_gpu=ug, c_gpu=cg, R_gpu=Rg, u_or=uo, c_or=co, R_or=Ro, gpu_iters=it[e],
                                    gpu_flags=fl[e], gpu_pg=pg[e], or_iters=st["iters"], or_flags=st["flags"],
                                    env=e, k=k)
                print(json.dumps(dict(k=k, env=e, du=d, oracle_stuck=stuck, gpu_iters=int(it[e]), gpu_flags=int(fl[e]),
                                      gpu_pg=float(pg[e]), oracle=st)), flush=True)
        summary.append(dict(k=k, worst=max(du), n_over_1e7=int(sum(x > 1e-7 for x in du)), n=len(du)))
        print(json.dumps(summary[-1]), flush=True)
    print(f"mismatches dumped: {n_bad}", flush=True)


if __name__ == "__main__":
    main()
