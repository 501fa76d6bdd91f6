"""Which C3 envs stop without converging in tolerance mode, and why (diagnosis tool).

Runs C3 (1,024 envs) in tolerance mode on the GPU, lists the envs flagged stagnated (64) or
at max_iters (2) after each step, and for up to --max-detail of them re-runs the oracle's
step from the GPU's own step-start state: the oracle's iterations / flags, the distance of
the GPU's exit state to the oracle's minimiser, and the oracle's fp64 |P g|_disp at the GPU's
exit state.  Usage: python tools/diag_stagnation.py [--steps 3] [--tol 1e-9]
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
from tools.diag_parity import pg_disp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--tol", type=float, default=1e-9)
    ap.add_argument("--stagnation", type=int, default=3000)
    ap.add_argument("--max-iters", type=int, default=8000)
    ap.add_argument("--max-detail", type=int, default=6)
    ap.add_argument("--out", default="gpurun_out/diag_stagnation.json")
    a = ap.parse_args()
    import torch
    import paper_2603_28475_b200 as P
    s = w.scene_c3(n_envs=1024, n_steps=a.steps)
    s.params.tol_x = a.tol
    s.params.max_iters = a.max_iters
    s.params.stagnation = a.stagnation
    sim = P.TacSim.from_scene(s)
    rho_max = float(np.linalg.norm(s.Y, axis=1).max())
    p_or = w.Params(**s.params.__dict__)
    p_or.tol_x = 1e-11
    prev = {}
    bad = []
    for k in range(a.steps):
        starts = {}
        t0 = time.time()
        sim.step(torch.tensor(s.poses[k], dtype=torch.float32, device="cuda"), s.dt)
        it, pg, fl = sim.env_status()
        fl = fl.cpu().numpy()
        it = it.cpu().numpy()
        pg = pg.cpu().numpy()
        idx = np.nonzero(fl & (2 | 64))[0]
        print(f"step {k} ({time.time() - t0:.1f} s): not converged {idx.tolist()} flags {fl[idx].tolist()} "
              f"iters {it[idx].tolist()} pg {pg[idx].tolist()}", flush=True)
        for e in idx:
            if len(bad) < a.max_detail:
                bad.append((int(e), k, prev.get(int(e)), sim.get_state(int(e)), int(it[e]), int(fl[e]), float(pg[e])))
        # step-start states of the next step (any env may stop without converging there)
        prev = {e: sim.get_state(e) for e in range(1024)} if k + 1 < a.steps else {}
    report = []
    for e, k, start, (ug, vg, cg, Rg), itg, flg, pgg in bad:
        o1 = O.Oracle(s, params=p_or, init_poses=s.init_poses[[e]])
        if start is not None:
            ut, vt, ct, Rt = start
            o1.set_state(0, ut, vt, ct, Rt)
        else:
            ut, vt, ct, Rt = o1.get_state(0)
        o1.set_trace(0, True)
        o1.step(s.poses[k][[e]])
        uo, _, co, Ro = o1.get_state(0)
        st = o1.status_of(0)
        tgt = s.poses[k][e].astype(np.float64)
        evg = o1.eval(ut, vt, ct, Rt, ug, cg, Rg, tgt)
        evo = o1.eval(ut, vt, ct, Rt, uo, co, Ro, tgt)
        tr = o1.trace(0)
        row = dict(env=e, step=k, gpu_iters=itg, gpu_flags=flg, gpu_pg=pgg, or_iters=st["iters"], or_flags=st["flags"],
                   du=float(np.abs(ug - uo).max()), u_max=float(np.abs(uo).max()),
                   E_gpu=evg["E"], E_or=evo["E"], n_cand=evg["n_cand"], n_anchor=evg["n_anchor"],
                   pg_or_at_gpu=pg_disp(o1, s, evg, rho_max)[0], pg_or_at_or=pg_disp(o1, s, evo, rho_max)[0],
                   dc=float(np.abs(cg - co).max()),
                   or_pg_trace=[float(x) for x in tr[tr[:, 2] == 1][:, 8][::50]],
                   or_alpha_trace=[float(x) for x in tr[tr[:, 2] == 1][:, 3][::50]])
        report.append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
