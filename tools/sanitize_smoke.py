"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): C1 press steps
with friction (tolerance mode, device-side loop) and a ragged 5-env peg scene (fixed iterations,
candidate rebuilds, dedup on), markers, checkpoint save/load.  Exits 0 when the run completes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_2603_28475_b200 as P  # noqa: E402
import workloads as w  # noqa: E402
from helpers import c1_press_scene  # noqa: E402


def main():
    s = c1_press_scene(mu_f=1.0, steps=2, depth=0.15e-3)
    s.params.tol_x = 1e-9
    s.params.max_iters = 400
    sim = P.TacSim.from_scene(s)
    for k in range(2):
        sim.step(torch.tensor(s.poses[k], dtype=torch.float32, device="cuda").contiguous(), s.dt)
    sim.markers()
    s2 = w.scene_small_peg(n_envs=5, n_steps=3)
    s2.params.fixed_iters = 20
    s2.params.dedup = 1
    sim2 = P.TacSim.from_scene(s2)
    ck = sim2.checkpoint_save()
    for k in range(3):
        sim2.step(torch.tensor(s2.poses[k], dtype=torch.float32, device="cuda").contiguous(), s2.dt)
    sim2.checkpoint_load(ck)
    sim2.step(torch.tensor(s2.poses[0], dtype=torch.float32, device="cuda").contiguous(), s2.dt)
    m = sim2.markers(ncomp=3)
    torch.cuda.synchronize()
    assert torch.isfinite(m).all()
    print("sanitize smoke ok", sim.env_status()[2].tolist(), sim2.env_status()[2].tolist())


if __name__ == "__main__":
    main()
