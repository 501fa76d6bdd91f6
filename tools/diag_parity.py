"""Diagnose converged-parity divergences between the CUDA path and the fp64 oracle on C3.

Measurement / diagnosis tool (not a test): runs C3 at full size (1,024 envs) in tolerance
mode on the GPU for a few steps, keeps the GPU's state of sampled envs after every step,
and for each sampled env
  * runs the oracle along the same targets (independent history),
  * re-runs the oracle's last step from the GPU's own step-start state (same history),
  * evaluates the oracle's fp64 gradient at the GPU's final state (|P g|_disp, energy),
so a divergence can be attributed to a different history, an early stop, or a second
minimiser.  Usage:  python tools/diag_parity.py [--steps 3] [--envs 0,511,1023] [--tol 1e-9]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import workloads as w  # noqa: E402


def pg_disp(o, scene, ev, rho_max):
    """fp64 |P g|_disp (block-Jacobi P = D^-1 per vertex / rigid block) from an oracle eval."""
    free = np.setdiff1d(np.arange(len(scene.X)), scene.fixed)
    g, D = ev["g"], ev["D"]
    m = 0.0
    for v in free:
        m = max(m, np.linalg.norm(np.linalg.solve(D[v], g[v])))
    pc = np.linalg.solve(ev["Drig"][0], ev["grig"][:3])
    pt = np.linalg.solve(ev["Drig"][1], ev["grig"][3:])
    return max(m, np.linalg.norm(pc) + rho_max * np.linalg.norm(pt)), float(np.abs(g[free]).max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--envs", default="0,511,1023")
    ap.add_argument("--tol", type=float, default=1e-9)
    ap.add_argument("--n-envs", type=int, default=1024)
    ap.add_argument("--out", default="gpurun_out/diag_parity.json")
    ap.add_argument("--detail-above", type=float, default=0.0,
                    help="same-start re-run and fp64 residuals only where du_max exceeds this [m]")
    ap.add_argument("--repeat", type=int, default=1, help="GPU runs of the same workload (atomics order varies)")
    a = ap.parse_args()
    import torch
    import paper_2603_28475_b200 as P

    if ":" in a.envs:  # start:stop:step
        envs = list(range(*[int(x) for x in a.envs.split(":")]))
    else:
        envs = [int(x) for x in a.envs.split(",")]
    s = w.scene_c3(n_envs=a.n_envs, n_steps=a.steps)
    s.params.tol_x = a.tol
    s.params.max_iters = 8000
    s.params.stagnation = 3000
    runs = []
    for r in range(a.repeat):
        sim = P.TacSim.from_scene(s)
        gstates = {e: [] for e in envs}
        t0 = time.time()
        for k in range(a.steps):
            sim.step(torch.tensor(s.poses[k], dtype=torch.float32, device="cuda"), s.dt)
            it, pg, fl = sim.env_status()
            torch.cuda.synchronize()
            for e in envs:
                gstates[e].append((sim.get_state(e), int(it[e]), int(fl[e]), float(pg[e])))
            fl_np = fl.cpu().numpy()
            print(f"run {r} gpu step {k}: converged {int((fl_np & 1).sum())}/{a.n_envs}, "
                  f"stagnated {int(((fl_np & 64) != 0).sum())}, failed {int(((fl_np & 44) != 0).sum())}, "
                  f"max iters {int(it.max())}", flush=True)
        print(f"run {r} gpu done in {time.time() - t0:.1f} s", flush=True)
        runs.append(gstates)
        sim.close()
    rho_max = float(np.linalg.norm(s.Y, axis=1).max())
    p_or = w.Params(**s.params.__dict__)
    p_or.tol_x = 1e-11
    o = O.Oracle(s, params=p_or, init_poses=s.init_poses[envs])
    ostates = {e: [] for e in envs}
    for k in range(a.steps):
        o.step(s.poses[k][envs], threads=min(len(envs), os.cpu_count() or 1))
        for j, e in enumerate(envs):
            ostates[e].append((o.get_state(j), o.status_of(j)))
    report = []
    bound = 1e-4 * max(s.extent)
    for r, gstates in enumerate(runs):
        worst = (0.0, None)
        for j, e in enumerate(envs):
            for k in range(a.steps):
                (ug, vg, cg, Rg), itg, flg, pgg = gstates[e][k]
                (uo, vo, co, Ro), sto = ostates[e][k]
                d = np.abs(ug - uo).max(axis=1)
                vmax = int(d.argmax())
                row = dict(run=r, env=e, step=k, gpu_iters=itg, gpu_flags=flg, gpu_pg=pgg, or_iters=sto["iters"],
                           or_flags=sto["flags"], du_max=float(d.max()), u_max=float(np.abs(uo).max()), vert=vmax,
                           vert_X=s.X[vmax].tolist(), u_or_vert=uo[vmax].tolist(), u_gpu_vert=ug[vmax].tolist())
                if row["du_max"] > worst[0]:
                    worst = (row["du_max"], (e, k))
                if k > 0 and (row["du_max"] > a.detail_above or a.detail_above <= 0):
                    # same history: the oracle's step k from the GPU's step-start state
                    (ut, vt, ct, Rt), _, _, _ = gstates[e][k - 1]
                    o1 = O.Oracle(s, params=p_or, init_poses=s.init_poses[[e]])
                    o1.set_state(0, ut, vt, ct, Rt)
                    o1.step(s.poses[k][[e]])
                    uo1, _, co1, Ro1 = o1.get_state(0)
                    row["du_same_start"] = float(np.abs(ug - uo1).max())
                    row["or_same_start_iters"] = o1.status_of(0)["iters"]
                    tgt = s.poses[k][e].astype(np.float64)
                    evg = o1.eval(ut, vt, ct, Rt, ug, cg, Rg, tgt)
                    evo = o1.eval(ut, vt, ct, Rt, uo1, co1, Ro1, tgt)
                    row["E_gpu_final"] = evg["E"]
                    row["E_or_final"] = evo["E"]
                    row["pg_disp_or_at_gpu"], row["gmax_or_at_gpu"] = pg_disp(o1, s, evg, rho_max)
                    row["pg_disp_or_at_or"], row["gmax_or_at_or"] = pg_disp(o1, s, evo, rho_max)
                    row["dmin_gpu"] = o1.dmin(ug, cg, Rg)
                    print(json.dumps(row), flush=True)
                report.append(row)
        n_bad = sum(1 for row in report if row["run"] == r and row["du_max"] > bound)
        print(f"run {r}: worst du_max {worst[0]:.3e} m at (env, step) {worst[1]}; {n_bad} env-steps over the "
              f"{bound:.1e} m bound", flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
