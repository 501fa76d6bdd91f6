"""Diagnose a same-start parity mismatch in a C3 window (diagnosis tool, not a test).

The GPU runs C3 (1,024 envs) in fixed-iteration mode to step k, a tolerance-mode simulator
loads the checkpoint and converges step k; for the listed envs the oracle runs the same step
from the GPU's start state.  Reports per env: iterations and flags on both sides, |u_gpu -
u_or|, the energies of both final states (oracle eval) and the oracle's fp64 |P g|_disp at
both, the pose difference, and the oracle's trace of |P g| and E.
Usage: python tools/diag_window.py --k 12 --envs 22,6 [--bps 8]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import workloads as w  # noqa: E402
from tools.diag_parity import pg_disp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=12)
    ap.add_argument("--envs", default="22,6")
    ap.add_argument("--bps", type=int, default=16)
    ap.add_argument("--gpu-tol", type=float, default=1e-9)
    ap.add_argument("--out", default="gpurun_out/diag_window.json")
    a = ap.parse_args()
    os.environ["TAC_CONTACT_BPS"] = str(a.bps)
    import torch
    import paper_2603_28475_b200 as P
    envs = [int(x) for x in a.envs.split(",")]
    s = w.scene_c3(n_envs=1024, n_steps=64)
    pf = w.Params(**s.params.__dict__)
    pf.fixed_iters = 50
    pt = w.Params(**s.params.__dict__)
    pt.fixed_iters = 0
    pt.tol_x = a.gpu_tol
    pt.max_iters = 20000
    pt.stagnation = 5000
    fixed = P.TacSim.from_scene(s, params=pf)
    tol = P.TacSim.from_scene(s, params=pt)
    poses = torch.tensor(s.poses, dtype=torch.float32, device="cuda").contiguous()
    for k in range(a.k):
        fixed.step(poses[k], s.dt)
    tol.checkpoint_load(fixed.checkpoint_save())
    starts = {e: tol.get_state(e) for e in envs}
    tol.step(poses[a.k], s.dt)
    it, pg, fl = tol.env_status()
    finals = {e: tol.get_state(e) for e in envs}
    p_or = w.Params(**pt.__dict__)
    p_or.tol_x = 1e-11
    rho_max = float(np.linalg.norm(s.Y, axis=1).max())
    rep = []
    for e in envs:
        o = O.Oracle(s, params=p_or, init_poses=s.init_poses[[e]])
        o.set_state(0, *starts[e])
        o.set_trace(0, True)
        o.step(s.poses[a.k][[e]])
        st = o.status_of(0)
        uo, _, co, Ro = o.get_state(0)
        ug, _, cg, Rg = finals[e]
        ut, vt, ct, Rt = starts[e]
        tgt = s.poses[a.k][e].astype(np.float64)
        evg = o.eval(ut, vt, ct, Rt, ug, cg, Rg, tgt)
        evo = o.eval(ut, vt, ct, Rt, uo, co, Ro, tgt)
        tr = o.trace(0)
        acc = tr[tr[:, 2] == 1]
        d = np.abs(ug - uo).max(axis=1)
        v = int(d.argmax())
        # energy along the segment between the two final states (a barrier between two minima?)
        seg = []
        for t in np.linspace(0, 1, 11):
            ui = uo + t * (ug - uo)
            ci = co + t * (cg - co)
            seg.append(o.eval(ut, vt, ct, Rt, ui, ci, Ro if t < 0.5 else Rg, tgt)["E"] - evo["E"])
        row = dict(env=e, k=a.k, gpu_iters=int(it[e]), gpu_flags=int(fl[e]), gpu_pg=float(pg[e]),
                   or_iters=st["iters"], or_flags=st["flags"], or_pg=st["pg"], du=float(d.max()), vert=v,
                   X=s.X[v].tolist(), u_or=uo[v].tolist(), u_gpu=ug[v].tolist(), dc=(cg - co).tolist(),
                   E_gpu=evg["E"], E_or=evo["E"], parts_gpu=evg["parts"].tolist(), parts_or=evo["parts"].tolist(),
                   pg_or_at_gpu=pg_disp(o, s, evg, rho_max)[0], pg_or_at_or=pg_disp(o, s, evo, rho_max)[0],
                   n_anchor=evo["n_anchor"], E_segment=seg, du_start=float(np.abs(ug - ut).max()),
                   or_pg_trace=[float(x) for x in acc[::max(1, len(acc) // 40), 8]],
                   or_E_trace=[float(x) for x in acc[::max(1, len(acc) // 40), 1]])
        rep.append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rep, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
