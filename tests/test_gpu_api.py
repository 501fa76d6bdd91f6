"""Edge cases of the C ABI on the GPU: reset, capacity overflow, refused
infeasible poses, three-component markers, status flags and per-env statistics."""
import numpy as np
import pytest

import oracle as O
import workloads as w
from helpers import c1_press_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    if not t.cuda.is_available():
        pytest.skip("no CUDA device")
    return t


def _sim(scene, **kw):
    import paper_2603_28475_b200 as P
    return P.TacSim.from_scene(scene, **kw)


def _poses(torch, p):
    return torch.tensor(p, dtype=torch.float32, device="cuda").contiguous()


def test_reset_restores_rest_state_and_pose(torch):
    """tac_reset: masked envs go back to rest (u = v = 0) at the given pose and then
    evolve like fresh envs; unmasked envs are untouched."""
    s = w.scene_small_peg(n_envs=4, n_steps=3)
    s.params.fixed_iters = 40
    sim = _sim(s)
    for k in range(2):
        sim.step(_poses(torch, s.poses[k]), s.dt)
    before = [sim.get_state(e) for e in range(4)]
    mask = torch.tensor([0, 1, 0, 1], dtype=torch.uint8, device="cuda")
    sim.reset(mask, _poses(torch, s.init_poses))
    torch.cuda.synchronize()
    for e in range(4):
        u, v, c, R = sim.get_state(e)
        if e in (1, 3):
            assert np.all(u == 0) and np.all(v == 0)
            assert np.allclose(c, s.init_poses[e][:3], atol=1e-7)
            assert np.allclose(R, O.quat_to_R(s.init_poses[e]), atol=1e-6)
        else:
            for a, b in zip((u, v, c, R), before[e]):
                assert np.array_equal(a, b)
    # a reset env steps like the same env of a fresh simulator
    sim.step(_poses(torch, s.poses[0]), s.dt)
    fresh = _sim(s)
    fresh.step(_poses(torch, s.poses[0]), s.dt)
    m1, m2 = sim.markers().cpu().numpy(), fresh.markers().cpu().numpy()
    scale = max(np.abs(m2[1]).max(), 1e-9)
    assert np.abs(m1[1] - m2[1]).max() <= 1e-4 * scale + 1e-12


def test_candidate_overflow_fails_the_step_and_rolls_back(torch):
    """A candidate capacity far below the contact's needs would drop pairs (the barrier and
    the step bound would no longer see them): the step fails with flag 32 (overflow) and the
    env is rolled back to its step-start state; the call itself succeeds and the fields stay
    finite."""
    s = c1_press_scene(mu_f=1.0, steps=3, depth=0.3e-3)
    s.params.max_candidates = 16
    s.params.fixed_iters = 30
    sim = _sim(s)
    for k in range(3):
        sim.step(_poses(torch, s.poses[k]), s.dt)
        it, pg, fl = sim.env_status()
        assert int(fl[0]) & 32 and not int(fl[0]) & 1
        u, v, c, R = sim.get_state(0)
        assert np.all(u == 0) and np.all(v == 0)  # x^t = rest: every step rolled back
        assert np.allclose(c, s.init_poses[0][:3], atol=1e-9)
    assert torch.isfinite(sim.markers()).all()


def test_initial_intersection_is_refused(torch):
    import paper_2603_28475_b200 as P
    s = w.scene_c1()
    for z in (2.0e-3, 3.0e-3 - 0.1e-3):  # sphere of radius 3 mm 1 mm / 0.1 mm into the pad
        s.init_poses[0, 2] = z
        with pytest.raises(P.TacError, match="intersects|touches"):
            _sim(s)
    s.init_poses[0, 2] = 3.0e-3 + 0.05e-3  # 50 um above: accepted
    _sim(s)


@pytest.mark.parametrize("field,value", [("beta_rule", 4), ("beta_rule", -1), ("precond", 2)])
def test_invalid_solver_switch_is_refused(torch, field, value):
    """tac_create validates the solver switches (include/tac.h: outside their ranges ->
    TAC_EINVAL) instead of running an undefined variant."""
    import paper_2603_28475_b200 as P
    s = w.scene_c1()
    setattr(s.params, field, value)
    with pytest.raises(P.TacError, match="invalid solver parameters"):
        _sim(s)


def test_three_component_markers_match_oracle(torch):
    """ncomp = 3 adds the normal component u_m . n (row a10)."""
    s = c1_press_scene(mu_f=1.0, steps=2, depth=0.2e-3)
    s.params.tol_x = 1e-9
    sim = _sim(s)
    o = O.Oracle(s, params=w.Params(**{**s.params.__dict__, "tol_x": 1e-11}))
    for k in range(2):
        sim.step(_poses(torch, s.poses[k]), s.dt)
        o.step(s.poses[k])
    m3 = sim.markers(ncomp=3).cpu().numpy()[0]
    m2 = sim.markers(ncomp=2).cpu().numpy()[0]
    r3 = o.markers(0, ncomp=3)
    assert np.array_equal(m3[:, :2], m2)
    assert np.abs(r3[:, 2]).max() > 0
    assert np.abs(m3 - r3).max() <= 1e-3 * np.abs(r3).max()


def test_status_flags_and_stats(torch):
    """max_iters reached -> flag 2 without flag 1; converged -> flag 1; env_stats reports
    the step's iterations, peak candidates and anchors consistently."""
    s = c1_press_scene(mu_f=1.0, steps=2, depth=0.2e-3)
    s.params.max_iters = 3
    s.params.tol_x = 1e-14
    sim = _sim(s)
    sim.step(_poses(torch, s.poses[0]), s.dt)
    it, pg, fl = sim.env_status()
    assert int(it[0]) == 3 and int(fl[0]) & 2 and not int(fl[0]) & 1
    s2 = c1_press_scene(mu_f=1.0, steps=2, depth=0.2e-3)
    sim2 = _sim(s2)
    for k in range(2):
        sim2.step(_poses(torch, s2.poses[k]), s2.dt)
    it, pg, fl = sim2.env_status()
    assert int(fl[0]) & 1
    st = sim2.env_stats().cpu().numpy()[0]
    assert st[0] == int(it[0])  # iterations of the last step
    assert st[1] >= 0 and st[2] >= 0 and st[3] >= 0


def test_several_simulators_in_one_process(torch):
    """Kernel attributes are per kernel, not per simulator: a simulator created after a
    smaller one keeps working, and both step correctly (calibration with several shapes)."""
    big = w.scene_small_peg(n_envs=2, n_steps=2)
    small = c1_press_scene(mu_f=1.0, steps=2, depth=0.2e-3)
    for s in (big, small):
        s.params.fixed_iters = 10
    a = _sim(big)
    b = _sim(small)
    for k in range(2):
        a.step(_poses(torch, big.poses[k]), big.dt)
        b.step(_poses(torch, small.poses[k]), small.dt)
    assert torch.isfinite(a.markers()).all() and torch.isfinite(b.markers()).all()


def test_native_marker_gather_world_of_one(torch):
    """tac_gather_markers on a one-rank NCCL communicator created through the C ABI: the
    gathered buffer equals tac_markers' field (the N > 1 exchange is
    the same ncclAllGather over more ranks)."""
    import paper_2603_28475_b200 as P
    from paper_2603_28475_b200.dist import NativeMarkerGather
    s = w.scene_small_peg(n_envs=5, n_steps=2)
    s.params.fixed_iters = 20
    sim = _sim(s)
    sim.step(_poses(torch, s.poses[0]), s.dt)
    g = NativeMarkerGather(sim, 5, sim.nm, 2, 0, 1, "cuda:0")
    buf = g.gather()
    ref = sim.markers()
    torch.cuda.synchronize()
    assert torch.equal(buf, ref)
    g3 = NativeMarkerGather(sim, 5, sim.nm, 3, 0, 1, "cuda:0")
    assert torch.equal(g3.gather(), sim.markers(ncomp=3))
    with pytest.raises(P.TacError):
        sim.gather_markers(g.comm, torch.empty((5, sim.nm, 4), device="cuda"), ncomp=4)
    g.close()
    g3.close()


def test_graph_replay_matches_direct_launches(torch):
    """The iteration loop replayed from CUDA graphs (default; chunks of check_every iterations
    in the tolerance mode) and launched kernel by kernel (TAC_NO_GRAPH=1, read at create) run
    the same kernels: converged steps agree far inside the oracle gates, and the per-step launch
    counts are equal.  (Unconverged fixed-iteration trajectories are not compared: fp32
    atomics' ordering noise changes Armijo / rebuild decisions along an NCG path.)"""
    import os
    s = w.scene_small_peg(n_envs=5, n_steps=3)
    s.params.tol_x = 1e-9
    s.params.stagnation = 3000
    a = _sim(s)
    os.environ["TAC_NO_GRAPH"] = "1"
    try:
        b = _sim(s)
    finally:
        del os.environ["TAC_NO_GRAPH"]
    for k in range(3):
        a.step(_poses(torch, s.poses[k]), s.dt)
        b.step(_poses(torch, s.poses[k]), s.dt)
    ia, _, fa = a.env_status()
    ib, _, fb = b.env_status()
    assert all(int(f) & 1 for f in fa) and all(int(f) & 1 for f in fb)
    ma, mb = a.markers().cpu().numpy(), b.markers().cpu().numpy()
    scale = np.abs(ma).max()
    assert scale > 0 and np.abs(ma - mb).max() <= 1e-4 * scale
    for e in range(5):
        ua, ub = a.get_state(e)[0], b.get_state(e)[0]
        assert np.abs(ua - ub).max() <= 1e-5 * 16e-3
    # launch counts of a fixed-iteration step: graph replay counts its captured launches
    s.params.fixed_iters = 20
    a2 = _sim(s)
    os.environ["TAC_NO_GRAPH"] = "1"
    try:
        b2 = _sim(s)
    finally:
        del os.environ["TAC_NO_GRAPH"]
    a2.step(_poses(torch, s.poses[0]), s.dt)
    b2.step(_poses(torch, s.poses[0]), s.dt)
    assert a2.last_launch_count() == b2.last_launch_count() > 20


def test_reset_clears_pose_multipliers(torch):
    """R29: tac_reset zeroes an env's AL multipliers, so a reset env steps like a fresh one."""
    s = c1_press_scene(mu_f=1.0, steps=3, depth=0.2e-3)
    s.params.pose_al = 1
    s.params.fixed_iters = 60
    sim = _sim(s)
    for k in range(3):
        sim.step(_poses(torch, s.poses[k]), s.dt)
    sim.reset(torch.ones(1, dtype=torch.uint8, device="cuda"), _poses(torch, s.init_poses))
    sim.step(_poses(torch, s.poses[0]), s.dt)
    fresh = _sim(s)
    fresh.step(_poses(torch, s.poses[0]), s.dt)
    u1, u2 = sim.get_state(0)[0], fresh.get_state(0)[0]
    assert np.abs(u1 - u2).max() <= 1e-6 * 16e-3


def test_checkpoint_resume_reproduces_the_steps(torch):
    """tac_checkpoint_save / tac_checkpoint_load (SURVEY §5 checkpoint / resume): the marker
    field right after a load equals the saved one bit for bit; stepping on from the loaded
    state with the same targets reproduces the converged steps taken after the save (pose
    noise included: the step counter keying the Philox streams, R27, is part of the
    checkpoint); a checkpoint of a simulator of another size is refused."""
    import paper_2603_28475_b200 as P
    s = w.scene_small_peg(n_envs=5, n_steps=4)
    s.params.tol_x = 1e-9
    s.params.stagnation = 3000
    sim = _sim(s)
    sim.set_pose_noise(2e-5, 1e-3, 7)
    sim.step(_poses(torch, s.poses[0]), s.dt)
    ck = sim.checkpoint_save()
    m_saved = sim.markers().clone()
    for k in (1, 2):
        sim.step(_poses(torch, s.poses[k]), s.dt)
    a = [sim.get_state(e) for e in range(5)]
    fa = sim.env_status()[2].cpu().numpy()
    sim.checkpoint_load(ck)
    assert torch.equal(sim.markers(), m_saved)
    for k in (1, 2):
        sim.step(_poses(torch, s.poses[k]), s.dt)
    fb = sim.env_status()[2].cpu().numpy()
    assert np.all(fa & 1) and np.all(fb & 1)
    for e in range(5):
        ub, _, cb, Rb = sim.get_state(e)
        ua, _, ca, Ra = a[e]
        assert np.abs(ua - ub).max() <= 1e-5 * 16e-3
        assert np.abs(ca - cb).max() <= 1e-8 and np.abs(Ra - Rb).max() <= 1e-6
    small = _sim(w.scene_small_peg(n_envs=3, n_steps=2))
    with pytest.raises(P.TacError, match="size"):
        small.checkpoint_load(ck)


def test_tolerance_mode_device_loop_matches_host_polled(torch):
    """Tolerance mode runs its iteration loop under device-side control (a CUDA-graph WHILE
    node over one PNCG iteration + a loop-control kernel: no host round trip inside a step).
    It converges every env to the same states as the host-polled chunked loop
    (TAC_NO_WHILE=1, read at create), stops as soon as no env iterates, and the launch count
    it reports covers the loop's device-side trips."""
    import os
    s = w.scene_small_peg(n_envs=5, n_steps=3)
    s.params.tol_x = 1e-9
    s.params.stagnation = 3000
    a = _sim(s)
    os.environ["TAC_NO_WHILE"] = "1"
    try:
        b = _sim(s)
    finally:
        del os.environ["TAC_NO_WHILE"]
    for k in range(3):
        a.step(_poses(torch, s.poses[k]), s.dt)
        la = a.last_launch_count()
        b.step(_poses(torch, s.poses[k]), s.dt)
        lb = b.last_launch_count()
        ia, _, fa = a.env_status()
        ib, _, fb = b.env_status()
        assert all(int(f) & 1 for f in fa) and all(int(f) & 1 for f in fb)
        # the device loop runs max(iterations) - 1 trips (16 launches each: the iteration's
        # kernels, k_alpha's last block running the loop control) + the final evaluation and
        # the step's setup / finalize
        assert 15 * (int(ia.max()) - 2) < la <= 17 * int(ia.max()) + 40, (la, lb, int(ia.max()))
    for e in range(5):
        ua, ub = a.get_state(e)[0], b.get_state(e)[0]
        assert np.abs(ua - ub).max() <= 1e-5 * 16e-3


def test_tolerance_mode_c3_never_fails_or_overflows(torch):
    """The bench's tolerance-mode configuration (C3, 1,024 envs, tol_x 1e-7 m, 2,000 iterations)
    over 20 steps of press / shear / twist: no env step fails (NaN, infeasible, candidate
    overflow) and no state goes non-finite.  (Round 1 saw NaN envs here: near-touching pairs
    made the fp32 block-Jacobi inverse singular; the contact blocks now live apart from the
    elastic ones and the inverse is formed in fp64 -- DESIGN.md R24.)"""
    s = w.scene_c3(n_envs=1024, n_steps=20)
    s.params.fixed_iters = 0
    s.params.tol_x = 1e-7
    s.params.max_iters = 2000
    sim = _sim(s)
    poses = _poses(torch, s.poses)
    for k in range(20):
        sim.step(poses[k], s.dt)
        it, pg, fl = sim.env_status()
        assert int(((fl & (4 | 8 | 32)) != 0).sum()) == 0, (k, np.nonzero((fl & 44).cpu().numpy())[0])
        assert torch.isfinite(pg).all()
    m = sim.markers()
    assert torch.isfinite(m).all()
    st = sim.env_stats().cpu().numpy()
    assert st[:, 1].max() < 32768 and st[:, 2].mean() > 100


def test_sharded_simulators_reproduce_one_simulator(torch):
    """SURVEY §8e / P:179-182: environments are independent, so ranks own contiguous env ranges
    (dist.env_range) and simulators holding those ranges -- with env_offset so their pose-noise
    streams are the global envs' (R27) -- reproduce one simulator of all envs; the marker
    fields in rank order are the all-gather's layout."""
    from paper_2603_28475_b200.dist import env_range
    s = w.scene_small_peg(n_envs=7, n_steps=3)
    s.params.tol_x = 1e-9
    s.params.stagnation = 3000
    noise = (2e-5, 1e-3, 77)
    full = _sim(s)
    full.set_pose_noise(*noise)
    shards = []
    for r in range(2):
        a, b = env_range(r, 2, 7)
        sub = w.scene_small_peg(n_envs=7, n_steps=3)
        sub.params = s.params
        sub.init_poses = s.init_poses[a:b]
        sub.poses = s.poses[:, a:b]
        sim = _sim(sub)
        sim.set_pose_noise(*noise, env_offset=a)
        shards.append((a, b, sim))
    for k in range(3):
        full.step(_poses(torch, s.poses[k]), s.dt)
        for a, b, sim in shards:
            sim.step(_poses(torch, s.poses[k][a:b]), s.dt)
    gathered = torch.cat([sim.markers() for _, _, sim in shards])
    ref = full.markers()
    scale = ref.abs().max().item()
    assert scale > 0 and (gathered - ref).abs().max().item() <= 1e-3 * scale
    for a, b, sim in shards:
        for j in range(b - a):
            assert np.abs(sim.get_state(j)[0] - full.get_state(a + j)[0]).max() <= 1e-5 * 16e-3
            assert np.abs(sim.get_state(j)[2] - full.get_state(a + j)[2]).max() <= 1e-9


def test_tolerance_tail_block_remap_matches_identity(torch):
    """Tolerance-mode tail: once few envs still iterate, the per-env contact passes deal their
    CTAs over k_alpha's list of active envs and the vertex / element passes deal the idle env
    groups' blocks to the active groups (tools/diag_tail.py).  A 1,024-env
    simulator with four envs in contact (the rest at rest, done after one iteration) converges
    them under the remapped tail and under the identity mapping (TAC_REMAP_BLOCKS=0, read at
    create) to states the fp64 oracle certifies as stationary (|P g|_disp <= 2 tol_x), with equal
    energies up to the spread of distinct minima (R25: summation-order noise can steer a
    sliding contact into a neighbouring minimum -- tools/diag_remap.py found one of four envs
    there in one of two remapped runs, 1.9 % apart in E, while identical runs agree to 3e-8 m)."""
    import os
    from helpers import pg_disp
    s = w.scene_c3(n_envs=1024, n_steps=12)
    pf = w.Params(**s.params.__dict__)
    pf.fixed_iters = 50
    fixed = _sim(s, params=pf)
    poses = _poses(torch, s.poses)
    k = 10
    for j in range(k):
        fixed.step(poses[j], s.dt)
    acts = [5, 300, 301, 777]  # groups 0, 9, 24: the group remap applies (<= 16 of 32 groups)
    sts = {e: fixed.get_state(e) for e in acts}
    fixed.close()
    pt = w.Params(**s.params.__dict__)
    pt.fixed_iters = 0
    pt.tol_x = 1e-9
    pt.max_iters = 6000
    pt.stagnation = 3000
    tgt = _poses(torch, s.init_poses)
    for e in acts:
        tgt[e] = poses[k][e]
    rho = float(np.linalg.norm(s.Y, axis=1).max())
    energies = {}
    for remap in ("512", "0"):
        os.environ["TAC_REMAP_BLOCKS"] = remap
        try:
            sim = _sim(s, params=pt)
        finally:
            del os.environ["TAC_REMAP_BLOCKS"]
        sim.reset(torch.ones(1024, dtype=torch.uint8, device="cuda"), _poses(torch, s.init_poses))
        for e in acts:
            sim.set_state(e, *sts[e])
        sim.step(tgt, s.dt)
        it, pg, fl = sim.env_status()
        fl = fl.cpu().numpy()
        assert all(fl[e] & 1 for e in acts), fl[acts]
        assert int(it.cpu().numpy()[acts].min()) > 20  # a real tail
        rest = np.setdiff1d(np.arange(1024), acts)
        assert int(it.cpu().numpy()[rest].max()) <= 2
        for e in acts:
            o = O.Oracle(s, init_poses=s.init_poses[[e]])
            u, _, c, R = sim.get_state(e)
            ev = o.eval(*sts[e], u, c, R, s.poses[k][e].astype(np.float64))
            assert pg_disp(o, s, ev, rho) <= 2 * pt.tol_x, (remap, e)
            energies[(remap, e)] = ev["E"]
        sim.close()
    for e in acts:
        ea, eb = energies[("512", e)], energies[("0", e)]
        assert abs(ea - eb) <= 0.05 * abs(eb), (e, ea, eb)
