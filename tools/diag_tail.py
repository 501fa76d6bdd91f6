"""Cost of a tolerance-mode tail iteration (diagnosis tool, not a test).

One env of C3 is solved in tolerance mode from a contact state twice: inside a 1,024-env
simulator whose other envs sit at rest out of contact (they converge in a few iterations, so
almost every iteration of the step serves the one env -- the tail of a tolerance-mode step),
and alone in a 1-env simulator.  Prints iterations and device time per iteration of both.
Usage: python tools/diag_tail.py [--k 24] [--env 5] [--tol 1e-7]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as w  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=24)
    ap.add_argument("--env", type=int, default=5)
    ap.add_argument("--tol", type=float, default=1e-7)
    ap.add_argument("--max-iters", type=int, default=2000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n-active", type=int, default=1, help="envs in contact (the others at rest)")
    ap.add_argument("--only-1024", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2603_28475_b200 as P
    s = w.scene_c3(n_envs=1024, n_steps=64)
    pf = w.Params(**s.params.__dict__)
    pf.fixed_iters = 50
    fixed = P.TacSim.from_scene(s, params=pf)
    poses = torch.tensor(s.poses, dtype=torch.float32, device="cuda").contiguous()
    for k in range(a.k):
        fixed.step(poses[k], s.dt)
    acts = [(a.env + 37 * i) % 1024 for i in range(a.n_active)]
    sts = {e: fixed.get_state(e) for e in acts}
    fixed.close()
    pt = w.Params(**s.params.__dict__)
    pt.fixed_iters = 0
    pt.tol_x = a.tol
    pt.max_iters = a.max_iters
    rows = []
    for n in ((1024,) if a.only_1024 else (1024, 1)):
        init = s.init_poses if n == 1024 else s.init_poses[[a.env]]
        sim = P.TacSim.from_scene(s, params=pt, n_envs=n, init_poses=init)
        j = a.env if n == 1024 else 0
        tgt = torch.tensor(init, dtype=torch.float32, device="cuda").contiguous()  # rest poses: no motion
        for e in (acts if n == 1024 else [a.env]):
            tgt[e if n == 1024 else 0] = poses[a.k][e]
        for rep in range(a.reps):
            mask = torch.ones(n, dtype=torch.uint8, device="cuda")
            sim.reset(mask, torch.tensor(init, dtype=torch.float32, device="cuda").contiguous())
            for e in (acts if n == 1024 else [a.env]):
                sim.set_state(e if n == 1024 else 0, *sts[e])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sim.step(tgt, s.dt)
            e1.record()
            torch.cuda.synchronize()
            it, pg, fl = sim.env_status()
            it = it.cpu().numpy()
            ms = e0.elapsed_time(e1)
            rows.append(dict(n_envs=n, n_active=a.n_active if n > 1 else 1, rep=rep, iters=int(it[j]),
                             max_iters=int(it.max()), max_other=int(np.delete(it, acts).max()) if n > 1 else 0,
                             ms=ms, us_per_iter=1e3 * ms / max(1, int(it.max())), flags=int(fl.cpu().numpy()[j])))
            print(json.dumps(rows[-1]), flush=True)
        sim.close()


if __name__ == "__main__":
    main()
