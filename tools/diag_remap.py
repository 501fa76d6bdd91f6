"""Tail block remapping vs the identity mapping (diagnosis tool, not a test).

The setup of tests/test_gpu_api.py::test_tolerance_tail_block_remap_matches_identity: a
1,024-env C3 simulator with a few envs in contact (the rest at rest) solved in tolerance mode,
twice with the remapped tail (TAC_REMAP_BLOCKS=512) and twice with the identity mapping
(TAC_REMAP_BLOCKS=0).  Prints per env the iterations of each run, the pairwise max |du| and the
oracle's energy and fp64 |P g|_disp at each final state (two different converged states with
equal standing are two minima; a remap bug would show as a non-converged state).
Usage: python tools/diag_remap.py [--k 10] [--envs 5,300,301,777]
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
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--envs", default="5,300,301,777")
    ap.add_argument("--tol", type=float, default=1e-9)
    a = ap.parse_args()
    import torch
    import paper_2603_28475_b200 as P
    acts = [int(x) for x in a.envs.split(",")]
    s = w.scene_c3(n_envs=1024, n_steps=a.k + 2)
    pf = w.Params(**s.params.__dict__)
    pf.fixed_iters = 50
    fixed = P.TacSim.from_scene(s, params=pf)
    poses = torch.tensor(s.poses, dtype=torch.float32, device="cuda").contiguous()
    for j in range(a.k):
        fixed.step(poses[j], s.dt)
    sts = {e: fixed.get_state(e) for e in acts}
    fixed.close()
    pt = w.Params(**s.params.__dict__)
    pt.fixed_iters = 0
    pt.tol_x = a.tol
    pt.max_iters = 6000
    pt.stagnation = 3000
    tgt = torch.tensor(s.init_poses, dtype=torch.float32, device="cuda").contiguous()
    for e in acts:
        tgt[e] = poses[a.k][e]
    runs = []
    for remap in ("512", "0", "512", "0"):
        os.environ["TAC_REMAP_BLOCKS"] = remap
        sim = P.TacSim.from_scene(s, params=pt)
        del os.environ["TAC_REMAP_BLOCKS"]
        sim.reset(torch.ones(1024, dtype=torch.uint8, device="cuda"),
                  torch.tensor(s.init_poses, dtype=torch.float32, device="cuda").contiguous())
        for e in acts:
            sim.set_state(e, *sts[e])
        sim.step(tgt, s.dt)
        it, pg, fl = sim.env_status()
        runs.append(dict(remap=remap, it=it.cpu().numpy()[acts].tolist(), fl=fl.cpu().numpy()[acts].tolist(),
                         pg=pg.cpu().numpy()[acts].tolist(), st={e: sim.get_state(e) for e in acts}))
        sim.close()
        print(json.dumps({k: v for k, v in runs[-1].items() if k != "st"}), flush=True)
    rho = float(np.linalg.norm(s.Y, axis=1).max())
    for e in acts:
        o = O.Oracle(s, init_poses=s.init_poses[[e]])
        ut, vt, ct, Rt = sts[e]
        tg = s.poses[a.k][e].astype(np.float64)
        row = dict(env=e, du=[[float(np.abs(r1["st"][e][0] - r2["st"][e][0]).max()) for r2 in runs] for r1 in runs])
        row["E"] = []
        row["pg_or"] = []
        for r in runs:
            u, _, c, R = r["st"][e]
            ev = o.eval(ut, vt, ct, Rt, u, c, R, tg)
            row["E"].append(ev["E"])
            row["pg_or"].append(pg_disp(o, s, ev, rho)[0])
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
