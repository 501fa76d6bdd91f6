"""Find C3 env-steps that overflow their candidate list in tolerance mode and replay them
(diagnosis tool).  Runs C3 (1,024 envs) in the bench's tolerance mode (tol_x 1e-7 m, 2,000
iterations), keeps every env's step-start state, dumps the start state of each env-step flagged
32 (overflow) and replays it alone with growing fixed iteration budgets to find the iteration
where it goes wrong.  Usage: python tools/diag_overflow.py [--steps 32]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--tol", type=float, default=1e-7)
    ap.add_argument("--max-iters", type=int, default=2000)
    ap.add_argument("--max-cases", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2603_28475_b200 as P
    s = w.scene_c3(n_envs=1024, n_steps=64)
    pt = w.Params(**s.params.__dict__)
    pt.fixed_iters = 0
    pt.tol_x = a.tol
    pt.max_iters = a.max_iters
    sim = P.TacSim.from_scene(s, params=pt)
    poses = torch.tensor(s.poses, dtype=torch.float32, device="cuda").contiguous()
    cases = []
    for k in range(a.steps):
        starts = {e: sim.get_state(e) for e in range(1024)}
        sim.step(poses[k], s.dt)
        it, pg, fl = sim.env_status()
        st = sim.env_stats().cpu().numpy()
        fl = fl.cpu().numpy()
        bad = np.nonzero(fl & 32)[0]
        print(f"step {k}: overflow {bad.tolist()} iters {it.cpu().numpy()[bad].tolist()} "
              f"peak cand {st[bad, 1].tolist()} max iters {int(it.max())}", flush=True)
        for e in bad[:a.max_cases - len(cases)]:
            cases.append((k, int(e), starts[int(e)]))
            ut, vt, ct, Rt = starts[int(e)]
            np.savez_compressed(f"gpurun_out/overflow_k{k}_e{e}.npz", u_t=ut, v_t=vt, c_t=ct, R_t=Rt,
                                target=s.poses[k][e], k=k, env=e)
        if len(cases) >= a.max_cases:
            break
    # replay each case alone: growing fixed budgets from the same start
    o = O.Oracle(s, init_poses=s.init_poses[:1])
    for k, e, (ut, vt, ct, Rt) in cases:
        s1 = w.scene_c3(n_envs=1, n_steps=64)
        s1.init_poses = s.init_poses[[e]]
        rows = []
        for n in (10, 30, 100, 300, 600, 1000, 1500, 2000):
            p1 = w.Params(**pt.__dict__)
            p1.fixed_iters = n
            one = P.TacSim.from_scene(s1, params=p1)
            one.set_state(0, ut, vt, ct, Rt)
            one.step(torch.tensor(s.poses[k][[e]], dtype=torch.float32, device="cuda").contiguous(), s.dt)
            it1, pg1, fl1 = one.env_status()
            stt = one.env_stats().cpu().numpy()[0]
            u, v, c, R = one.get_state(0)
            fin = bool(np.isfinite(u).all() and np.isfinite(c).all() and np.isfinite(R).all())
            dmin = o.dmin(u, c, R) if fin else float("nan")
            rows.append(dict(n=n, flags=int(fl1[0]), pg=float(pg1[0]), peak_cand=int(stt[1]), finite=fin,
                             dmin=dmin, du=float(np.abs(u - ut).max()) if fin else None, c=c.tolist()))
            print(json.dumps(dict(k=k, env=e, **rows[-1])), flush=True)
            one.close()


if __name__ == "__main__":
    main()
