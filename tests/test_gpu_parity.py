"""CUDA path vs the fp64 oracle, through the C ABI (SURVEY §8c gates).

Bars (BASELINE north_star):
  * broad-phase candidate sets: bit-exact on identical fp32 inputs;
  * marker -> tet indices: bit-exact;
  * kernel level on identical inputs: gradient and diagonal blocks <= 1e-5 relative;
  * converged steps: marker displacement within 1e-3 of the max marker displacement
    (relative L-inf), gel positions within 1e-4 of the pad size.
"""
import numpy as np
import pytest

import oracle as O
import workloads as w
from helpers import c1_press_scene, rot_exp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _sim(scene, **kw):
    import paper_2603_28475_b200 as P
    return P.TacSim.from_scene(scene, **kw)


def _canon(pairs, surf, tris):
    """Map (kind, a, b) to vertex-id keys so both sides' numbering can differ."""
    sv, se, st, ie = surf
    out = set()
    for k, a, b in pairs:
        if k == 0:
            out.add((0, int(sv[a]), tuple(sorted(tris[b]))))
        elif k == 1:
            out.add((1, int(a), tuple(sorted(st[b]))))
        else:
            out.add((2, tuple(sorted(se[a])), tuple(sorted(ie[b]))))
    return out


def _pressed_state():
    s = c1_press_scene(mu_f=1.0, steps=4, depth=0.25e-3)
    s.params.tol_x = 1e-10
    o = O.Oracle(s)
    for k in range(3):
        o.step(s.poses[k])
    st = o.get_state(0)
    o.step(s.poses[3])
    u, _, c, R = o.get_state(0)
    rng = np.random.default_rng(5)
    # away from equilibrium (|g| not a small difference of large terms), still feasible
    u = u + 1e-6 * rng.standard_normal(u.shape)
    u[s.fixed] = 0
    u = u.astype(np.float32).astype(np.float64)  # identical fp32 inputs on both sides
    c = c + 1e-7 * rng.standard_normal(3)
    R = rot_exp(1e-5 * rng.standard_normal(3)) @ R
    tgt = s.poses[3][0].copy()
    tgt[2] -= 2e-5
    return s, o, st, (u, c, R), tgt


def test_marker_map_bitexact(torch_cuda):
    for scene in (w.scene_c1(), w.scene_c2(steps=1)):
        sim = _sim(scene)
        o = O.Oracle(scene)
        t1, i1, w1 = sim.debug_marker_map()
        t2, i2, w2 = o.marker_map()
        assert np.array_equal(t1, t2)
        assert np.array_equal(i1, i2)
        assert np.abs(w1 - w2).max() < 1e-12


def test_kuhn_cell_decomposition(torch_cuda):
    """The register-blocked gradient covers every tet of the (pseudo-structured and jittered,
    renumbered) Kuhn pads; a mesh without cells falls back to the generic kernel."""
    for s in (w.scene_c1(), w.scene_c2(steps=1), _small_unstructured()):
        sim = _sim(s)
        assert sim.n_cells * 6 == sim.nt and sim.n_other_tets == 0
    s = w.scene_c1()
    s.tets = s.tets[1:]  # break one cell: its 5 remaining tets go to the generic kernel
    s.markers = s.markers[:1] * 0 + np.array([[0.0, 0.0, -1.0e-3]])
    s.markers = np.repeat(s.markers, 63, axis=0)
    sim = _sim(s)
    assert sim.n_other_tets == 5 and sim.n_cells * 6 + 5 == sim.nt


def test_surface_matches(torch_cuda):
    s = w.scene_c1()
    sim = _sim(s)
    o = O.Oracle(s)
    for a, b in zip(sim.debug_surface(), o.surface()):
        assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("case", ["c1_pressed", "peg_c2_mesh"])
def test_broadphase_bitexact(torch_cuda, case):
    if case == "c1_pressed":
        s, o, _, (u, c, R), _ = _pressed_state()
        states = [(u, c, R)]
    else:
        s = w.scene_c3(n_envs=3, n_steps=8)
        o = O.Oracle(s)
        rng = np.random.default_rng(1)
        states = []
        for e in range(3):
            p = s.poses[6, e]
            R = O.quat_to_R(p)
            c = p[:3].astype(np.float64) + np.array([0, 0, 0.35e-3])
            u = np.zeros_like(s.X)
            u[:, 2] = -2e-4 * np.exp(-((s.X[:, 0] - c[0]) ** 2 + (s.X[:, 1] - c[1]) ** 2) / (3e-3) ** 2)
            u *= (1 + s.X[:, 2] / 5e-3)[:, None]
            u += 1e-6 * rng.standard_normal(u.shape)
            u[s.fixed] = 0
            states.append((u.astype(np.float32).astype(np.float64), c, R))
    sim = _sim(s)
    gsurf = sim.debug_surface()
    osurf = o.surface()
    for env, (u, c, R) in enumerate(states):
        for r in (3e-4, 1e-4):
            gpu = sim.debug_broadphase(min(env, s.n_envs - 1), u, c, R, r)
            ref = o.broadphase_state(u, c, R, r)
            assert len(ref) > 0
            assert len(gpu) == len(ref)
            assert _canon(gpu, gsurf, s.tris) == _canon(ref, osurf, s.tris)


EPS32 = 2.0 ** -24


def _assert_eval_parity(s, o, ref, gpu, u_t, v_t, u):
    """Kernel-level bars of SURVEY §8c (gradient and diagonal blocks <= 1e-5 relative, fp32),
    applied element-wise: the gradient in norm, every free vertex's 3x3 block against its own
    magnitude, the rigid gradient, and each energy part against its own value.  The inertia
    part is a sum of m |u - u^|^2 with u^ = u^t + h v^t formed in fp32 on the device, so its bar
    adds the propagated fp32 rounding of u^ and of u - u^ (a derived bound; at a state near
    the prediction the part is a small difference of fp32 numbers)."""
    free = np.setdiff1d(np.arange(len(u)), s.fixed)
    g_ref, g_gpu = ref["g"][free], gpu["g"][free]
    assert np.linalg.norm(g_gpu - g_ref) <= 1e-5 * np.linalg.norm(g_ref)
    D_ref, D_gpu = ref["D"][free], gpu["D"][free]
    blk = np.abs(D_gpu - D_ref).reshape(len(free), 9).max(axis=1)
    scale = np.abs(D_ref).reshape(len(free), 9).max(axis=1)
    assert np.all(blk <= 1e-5 * scale), (blk / scale).max()
    assert np.linalg.norm(gpu["grig"] - ref["grig"]) <= 1e-5 * np.linalg.norm(ref["grig"])
    m, _ = o.mass_vol()
    uh = u_t + s.dt * v_t
    du = (u - uh)[free]
    in_bar = (m[free, None] * np.abs(du) * 4 * EPS32 * (np.abs(u_t) + s.dt * np.abs(v_t) + np.abs(u))[free]).sum()
    assert abs(gpu["parts"][0] - ref["parts"][0]) <= 1e-5 * abs(ref["parts"][0]) + in_bar, (gpu["parts"][0], ref["parts"][0], in_bar)
    for k in range(1, 5):
        assert abs(gpu["parts"][k] - ref["parts"][k]) <= 1e-5 * abs(ref["parts"][k]) + 1e-30, \
            (k, gpu["parts"][k], ref["parts"][k])


def test_kernel_parity_gradient_diag(torch_cuda):
    s, o, (u_t, v_t, c_t, R_t), (u, c, R), tgt = _pressed_state()
    sim = _sim(s)
    ut32 = u_t.astype(np.float32).astype(np.float64)
    vt32 = v_t.astype(np.float32).astype(np.float64)
    ref = o.eval(ut32, vt32, c_t, R_t, u, c, R, tgt)
    gpu = sim.debug_eval(0, ut32, vt32, c_t, R_t, u, c, R, tgt, s.dt)
    assert ref["parts"][2] > 0 and ref["parts"][3] > 0  # barrier and friction present
    _assert_eval_parity(s, o, ref, gpu, ut32, vt32, u)


def _iteration_inputs(s, o, st, x1, tgt):
    """A realistic PNCG iteration for rows a6-a8: x_{k-1} = x1, the oracle's restart step from it
    gives p_{k-1} and x_k = x_{k-1} + alpha p_{k-1} (O4g); everything the GPU stores in fp32 is
    rounded to fp32 on both sides."""
    u1, c1, R1 = x1
    nv = len(u1)
    r32 = lambda a: a.astype(np.float32).astype(np.float64)
    zero = np.zeros(3 * nv + 6)
    p1, it1 = o.iteration(*st, u1, c1, R1, tgt, zero, zero, 1.0, restart=True)
    ev1 = o.eval(*st, u1, c1, R1, tgt)
    g_prev = np.concatenate([r32(ev1["g"]).ravel(), ev1["grig"]])
    p_prev = np.concatenate([r32(p1[:3 * nv]), p1[3 * nv:]])
    a = it1["alpha"]
    assert a > 0
    u = r32(u1 + a * p_prev[:3 * nv].reshape(nv, 3))
    u[s.fixed] = 0
    c = c1 + a * p_prev[3 * nv:3 * nv + 3]
    R = rot_exp(a * p_prev[3 * nv + 3:]) @ R1
    return (u, c, R), g_prev, p_prev, it1["gPg"]


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("beta_rule,precond", [(0, 0), (1, 0), (2, 0), (3, 0), (0, 1)])
def test_kernel_parity_direction_curvature_step_bounds(torch_cuda, beta_rule, precond):
    """Rows a6-a8 at kernel level on identical inputs (SURVEY §4 tier 2): the GPU's Dai-Kou beta
    (and the PR+ / FR / DK+ variants, scalar Jacobi P:457), direction p, g^T p, |P g|_disp,
    p^T H p, alpha_upper, alpha_bar, alpha_ccd (R15) and alpha vs the
    oracle's at a C1 contact state with friction, for a restart (p = -P g) and a conjugate step.
    Bars (derived from the kernel-level gradient bar): the gradient matches to 1e-5 of the force
    level of the non-equilibrium state x_{k-1}; at x_k the error relative to g grows by
    amp = sqrt(g_{k-1}^T P g_{k-1} / g_k^T P g_k), so e1 = 1e-5 amp on quantities linear in g
    (p, |P g|, M, alpha_upper, L_rel), 2 e1 on quadratic ones (g^T P g, g^T p, p^T H p,
    alpha_ccd), 3 e1 on beta and 4 e1 on alpha_bar = -g^T p / p^T H p and alpha."""
    s, o, (u_t, v_t, c_t, R_t), x1, tgt = _pressed_state()
    s.params.beta_rule = beta_rule
    s.params.precond = precond
    o = O.Oracle(s, params=s.params)
    r32 = lambda a: a.astype(np.float32).astype(np.float64)
    st = (r32(u_t), r32(v_t), c_t, R_t)
    (u, c, R), g_prev, p_prev, gPg_prev = _iteration_inputs(s, o, st, x1, tgt)
    sim = _sim(s)
    nv = len(u)
    free = np.setdiff1d(np.arange(nv), s.fixed)
    for restart in (True, False):
        p_o, r_o = o.iteration(*st, u, c, R, tgt, g_prev, p_prev, gPg_prev, restart=restart)
        p_g, r_g = sim.debug_iteration(0, *st, u, c, R, tgt, s.dt, g_prev, p_prev, gPg_prev, restart=restart)
        assert r_o["restarted"] == (1.0 if restart else 0.0) == r_g["restarted"], (restart, r_o, r_g)
        # derived bar: the gradient at x_{k-1} matches to 1e-5 of its size (test above); at x_k,
        # closer to equilibrium, the same absolute rounding is a larger share of the smaller g
        amp = max(1.0, np.sqrt(gPg_prev / r_o["gPg"]))
        e1 = 1e-5 * amp
        if not restart:
            assert r_o["beta"] != 0 and _rel(r_g["beta"], r_o["beta"]) <= 3 * e1, (r_g["beta"], r_o["beta"])
        pv_o, pv_g = p_o[:3 * nv].reshape(nv, 3)[free], p_g[:3 * nv].reshape(nv, 3)[free]
        assert np.abs(pv_g - pv_o).max() <= e1 * np.abs(pv_o).max()
        # the rigid gradient is a sum of contact forces and the pose spring that nearly cancel
        # near equilibrium: its rounding scales with the force level, i.e. with the previous
        # (restart) direction's rigid part, not with the small remainder
        rig_scale = max(np.abs(p_o[3 * nv:]).max(), np.abs(p_prev[3 * nv:]).max())
        assert np.abs(p_g[3 * nv:] - p_o[3 * nv:]).max() <= e1 * rig_scale, (p_g[3 * nv:], p_o[3 * nv:], rig_scale)
        for k, bar in (("pg_disp", e1), ("M", e1), ("alpha_upper", e1), ("L_rel", e1), ("gPg", 2 * e1),
                       ("gp", 2 * e1), ("pHp", 2 * e1), ("alpha_ccd", 2 * e1), ("alpha_bar", 4 * e1),
                       ("alpha", 4 * e1)):
            assert np.isfinite(r_o[k]) and r_o[k] != 0 and _rel(r_g[k], r_o[k]) <= bar, (restart, k, r_g[k], r_o[k], bar)
        assert r_o["pHp"] > 0 and r_o["alpha"] > 0


def _run_both(scene, steps, tol_gpu=1e-9, tol_or=1e-11):
    import torch
    scene.params.tol_x = tol_gpu
    scene.params.max_iters = 8000
    scene.params.stagnation = 3000
    sim = _sim(scene)
    p_or = w.Params(**{**scene.params.__dict__})
    p_or.tol_x = tol_or
    p_or.stagnation = 3000
    o = O.Oracle(scene, params=p_or)
    E = scene.n_envs
    mk = torch.empty((E, 63, 2), device="cuda", dtype=torch.float32)
    for k in range(steps):
        tgt = torch.tensor(scene.poses[k], dtype=torch.float32, device="cuda").contiguous()
        sim.step(tgt, scene.dt)
        o.step(scene.poses[k], threads=min(E, 8))
    sim.markers(mk)
    torch.cuda.synchronize()
    return sim, o, mk.cpu().numpy()


def _assert_parity(scene, sim, o, mk, env):
    u_g, _, c_g, _ = sim.get_state(env)
    u_o, _, c_o, _ = o.get_state(env)
    pad = max(scene.extent)
    assert np.abs(u_g - u_o).max() <= 1e-4 * pad
    m_o = o.markers(env)
    scale = np.abs(m_o).max()
    if scale > 1e-7:
        assert np.abs(mk[env] - m_o).max() <= 1e-3 * scale
    assert np.all(u_g[scene.fixed] == 0)


def test_converged_step_parity_c1(torch_cuda):
    s = c1_press_scene(mu_f=1.0, steps=3, depth=0.2e-3)
    sim, o, mk = _run_both(s, 3)
    it, pg, fl = sim.env_status()
    assert int(fl[0]) & 1, int(fl[0])  # converged
    _assert_parity(s, sim, o, mk, 0)


@pytest.mark.parametrize("beta_rule,precond", [(1, 0), (0, 1), (3, 0)])
def test_solver_variants_converged_parity(torch_cuda, beta_rule, precond):
    """SURVEY 8f-3 switches (beta rule PR+ of P:454's family, DK+ truncation (R28), scalar
    Jacobi of P:457):
    GPU and oracle converge to the same states, with comparable iteration counts."""
    s = w.scene_small_peg(n_envs=2, n_steps=3)
    s.params.beta_rule = beta_rule
    s.params.precond = precond
    sim, o, mk = _run_both(s, 3)
    it, pg, fl = sim.env_status()
    for e in range(2):
        assert int(fl[e]) & 1, (e, int(fl[e]))
        assert o.status_of(e)["flags"] & 1
        _assert_parity(s, sim, o, mk, e)
        it_o = o.status_of(e)["iters"]
        assert int(it[e]) <= 3 * it_o + 50 and it_o <= 3 * int(it[e]) + 50, (int(it[e]), it_o)


def test_augmented_lagrangian_pose_parity(torch_cuda):
    """R29 (SURVEY 8f-3 augmented-Lagrangian pose enforcement): a C1 press held for three
    steps with pose_al = 1 converges to the oracle's states, and the indenter reaches its
    target to the solver tolerance where the penalty alone leaves F / k_t."""
    res = {}
    for al in (0, 1):
        s = c1_press_scene(mu_f=1.0, steps=3, depth=0.3e-3)
        s.poses = np.concatenate([s.poses, np.repeat(s.poses[-1:], 3, axis=0)])
        s.params.pose_al = al
        sim, o, mk = _run_both(s, len(s.poses))
        it, pg, fl = sim.env_status()
        assert int(fl[0]) & 1, int(fl[0])
        _assert_parity(s, sim, o, mk, 0)
        c_g = sim.get_state(0)[2]
        res[al] = np.linalg.norm(c_g - s.poses[-1][0][:3])
        assert np.linalg.norm(c_g - o.get_state(0)[2]) <= 1e-4 * max(s.extent)
    assert res[0] > 1e-9 and res[1] < 0.1 * res[0], res


def test_ee_mollifier_kernel_and_converged_parity(torch_cuda):
    """R30 (SURVEY 8f-3 edge-edge mollifier): a peg lying along the pad's x edges (nearly
    parallel edge-edge contacts).  Kernel level: the GPU's gradient, blocks and energy parts at a
    perturbed contact state match the oracle's with the mollifier on (<= 1e-5); converged
    steps match the oracle's states."""
    from helpers import parallel_peg_scene
    s = parallel_peg_scene(steps=2, depth=0.05e-3)
    s.params.ee_mollifier = 1
    s.params.tol_x = 1e-10
    o = O.Oracle(s)
    o.step(s.poses[0])
    u_t, v_t, c_t, R_t = o.get_state(0)
    o.step(s.poses[1])
    u, _, c, R = o.get_state(0)
    rng = np.random.default_rng(11)
    u = u + 2e-7 * rng.standard_normal(u.shape)
    u[s.fixed] = 0
    tgt = s.poses[1][0]
    sim = _sim(s)
    ut32 = u_t.astype(np.float32).astype(np.float64)
    vt32 = v_t.astype(np.float32).astype(np.float64)
    u32 = u.astype(np.float32).astype(np.float64)
    ref = o.eval(ut32, vt32, c_t, R_t, u32, c, R, tgt)
    gpu = sim.debug_eval(0, ut32, vt32, c_t, R_t, u32, c, R, tgt, s.dt)
    _assert_eval_parity(s, o, ref, gpu, ut32, vt32, u32)
    s2 = parallel_peg_scene(steps=3, depth=0.1e-3, offset_y=0.37e-3)
    s2.params.ee_mollifier = 1
    sim2, o2, mk = _run_both(s2, 3)
    it, pg, fl = sim2.env_status()
    assert int(fl[0]) & 1, int(fl[0])
    _assert_parity(s2, sim2, o2, mk, 0)


def test_fletcher_reeves_matches_oracle_behaviour(torch_cuda):
    """FR (beta rule 2) without restarts jams on the second C1 press step in the fp64
    oracle (stagnation); the GPU reproduces the converged first step and the jam."""
    s = c1_press_scene(mu_f=1.0, steps=2, depth=0.2e-3)
    s.params.beta_rule = 2
    sim, o, mk = _run_both(s, 1)
    it, pg, fl = sim.env_status()
    assert int(fl[0]) & 1 and o.status_of(0)["flags"] & 1
    _assert_parity(s, sim, o, mk, 0)
    import torch
    sim.step(torch.tensor(s.poses[1], dtype=torch.float32, device="cuda").contiguous(), s.dt)
    o.step(s.poses[1])
    it, pg, fl = sim.env_status()
    assert not (int(fl[0]) & 1) and int(fl[0]) & (2 | 64), int(fl[0])
    assert not (o.status_of(0)["flags"] & 1)


def test_per_env_material_converged_parity(torch_cuda):
    """per-env theta = [E, nu, rho, mu_f] in one batch (the calibration of
    Eqs. 6-7, evaluates a CMA-ES population as envs): every env matches an
    oracle built with that env's material; an invalid theta is refused."""
    import copy
    import torch
    s = w.scene_small_peg(n_envs=3, n_steps=3)
    s.params.tol_x = 1e-9
    s.params.max_iters = 8000
    s.params.stagnation = 3000
    th = dict(E=[0.6e5, 1.0e5, 1.8e5], nu=[0.40, 0.45, 0.48], rho=[900.0, 1100.0, 1500.0], mu_f=[0.4, 1.0, 1.5])
    sim = _sim(s)
    sim.set_env_material(**th)
    with pytest.raises(Exception):
        sim.set_env_material(nu=[0.3, 0.5, 0.4])
    for k in range(3):
        sim.step(torch.tensor(s.poses[k], dtype=torch.float32, device="cuda").contiguous(), s.dt)
    mk = sim.markers().cpu().numpy()
    it, pg, fl = sim.env_status()
    for e in range(3):
        assert int(fl[e]) & 1, (e, int(fl[e]))
        se = copy.deepcopy(s)
        se.material = w.Material(E=th["E"][e], nu=th["nu"][e], rho=th["rho"][e], mu_f=th["mu_f"][e])
        se.init_poses = s.init_poses[e:e + 1]
        se.poses = s.poses[:, e:e + 1]
        p_or = w.Params(**{**s.params.__dict__})
        p_or.tol_x = 1e-11
        o = O.Oracle(se, params=p_or)
        for k in range(3):
            o.step(se.poses[k])
        u_g, _, c_g, _ = sim.get_state(e)
        u_o, _, c_o, _ = o.get_state(0)
        assert np.abs(u_g - u_o).max() <= 1e-4 * max(s.extent)
        m_o = o.markers(0)
        assert np.abs(mk[e] - m_o).max() <= 1e-3 * np.abs(m_o).max()
    # the materials differ enough to matter: env responses are not interchangeable
    assert np.abs(mk[0] - mk[2]).max() > 1e-2 * np.abs(mk[2]).max()


def test_converged_parity_multi_env_ragged(torch_cuda):
    s = w.scene_small_peg(n_envs=5, n_steps=4)
    sim, o, mk = _run_both(s, 4)
    for e in range(s.n_envs):
        _assert_parity(s, sim, o, mk, e)


def test_fixed_iteration_mode_runs_and_is_finite(torch_cuda):
    import torch
    s = w.scene_small_peg(n_envs=33, n_steps=3)
    s.params.fixed_iters = 50
    sim = _sim(s)
    for k in range(3):
        sim.step(torch.tensor(s.poses[k], dtype=torch.float32, device="cuda"), s.dt)
    it, pg, fl = sim.env_status()
    assert torch.all(it == 50)
    m = sim.markers()
    assert torch.isfinite(m).all()
    for e in (0, 17, 32):
        u, _, c, R = sim.get_state(e)
        assert np.all(np.isfinite(u)) and np.all(u[s.fixed] == 0)
        assert O.Oracle(s).dmin(u, c, R) > 0


# ---------------------------------------------------------------- full size (BASELINE configs[2])
SAMPLED = (0, 511, 1023)


def test_full_size_c3_bench_config_sampled(torch_cuda):
    """C3 at full size in the launch configuration bench.py times (1,024 envs, fixed 50
    iterations): no env flagged, every sampled env intersection-free by brute force with
    fixed vertices at 0, and kernel-level parity of E, g, D, rigid g at the GPU's state."""
    import torch
    s = w.scene_c3(n_envs=1024, n_steps=6)
    s.params.fixed_iters = 50
    sim = _sim(s)
    for k in range(5):
        sim.step(torch.tensor(s.poses[k], dtype=torch.float32, device="cuda"), s.dt)
    it, pg, fl = sim.env_status()
    assert torch.all(it == 50) and int(((fl & (4 | 8 | 32)) != 0).sum()) == 0
    stats = sim.env_stats().cpu().numpy()
    assert stats[:, 1].max() < 16384 and stats[:, 2].mean() > 100  # capacity, contact present
    o = O.Oracle(s, init_poses=s.init_poses[list(SAMPLED)])
    for e in SAMPLED:
        u, v, c, R = sim.get_state(e)
        assert np.all(u[s.fixed] == 0)
        assert o.dmin(u, c, R) > 0
        tgt = s.poses[5][e].astype(np.float64)
        ref = o.eval(u, v, c, R, u, c, R, tgt)
        gpu = sim.debug_eval(e, u, v, c, R, u, c, R, tgt, s.dt)
        assert ref["n_cand"] > 0
        _assert_eval_parity(s, o, ref, gpu, u, v, u)


# (round 1's test_full_size_c3_converged_sampled -- 3 envs, independent history, no certification of
# other local minimisers, R25 -- is superseded by tests/test_gpu_converged.py's full-size tests)


def test_c2_sphere_press_converged_parity(torch_cuda):
    """BASELINE configs[1] (C2: GelSight-Mini-like 19,800-tet pad, R = 5 mm icosphere): the first
    four steps of its press (to 0.3 mm) converge to the oracle's states on the north_star gates."""
    s = w.scene_c2(steps=4)
    sim, o, mk = _run_both(s, 4)
    it, pg, fl = sim.env_status()
    assert int(fl[0]) & 1, int(fl[0])
    assert o.status_of(0)["flags"] & 1
    _assert_parity(s, sim, o, mk, 0)
    assert np.abs(o.markers(0)).max() > 1e-6  # the press reaches the markers


# ---------------------------------------------------------------- §8f-1 unstructured mesh, C5 stress
def _small_unstructured(n_envs=3, n_steps=3):
    s = w.scene_small_peg(n_envs=n_envs, n_steps=n_steps)
    s.X, s.tets, s.fixed = w.make_pad_unstructured(s.extent, s.cells)
    return s


def test_unstructured_maps_and_broadphase_bitexact(torch_cuda):
    s = _small_unstructured()
    sim = _sim(s)
    o = O.Oracle(s)
    t1, i1, w1 = sim.debug_marker_map()
    t2, i2, w2 = o.marker_map()
    assert np.array_equal(t1, t2) and np.array_equal(i1, i2) and np.abs(w1 - w2).max() < 1e-12
    rng = np.random.default_rng(3)
    for e in range(s.n_envs):
        p = s.poses[1, e]
        R = O.quat_to_R(p)
        c = p[:3].astype(np.float64)
        u = 1e-6 * rng.standard_normal(s.X.shape)
        u[s.fixed] = 0
        u = u.astype(np.float32).astype(np.float64)
        gpu = sim.debug_broadphase(e, u, c, R, 3e-4)
        ref = o.broadphase_state(u, c, R, 3e-4)
        assert len(ref) > 0 and len(gpu) == len(ref)
        assert _canon(gpu, sim.debug_surface(), s.tris) == _canon(ref, o.surface(), s.tris)


def test_unstructured_converged_parity(torch_cuda):
    s = _small_unstructured(n_envs=3, n_steps=3)
    sim, o, mk = _run_both(s, 3)
    for e in range(s.n_envs):
        _assert_parity(s, sim, o, mk, e)


def test_c5_stress_bench_config_sampled(torch_cuda):
    """C5 (103,680 tets, sharp square peg, 256 envs) in the bench configuration: no env
    flagged, sampled envs intersection-free with fixed vertices 0, kernel-level parity."""
    import torch
    s = w.scene_c5(n_envs=256, n_steps=14)
    s.params.fixed_iters = 50
    sim = _sim(s)
    for k in range(13):
        sim.step(torch.tensor(s.poses[k], dtype=torch.float32, device="cuda"), s.dt)
    it, pg, fl = sim.env_status()
    assert int(((fl & (4 | 8 | 32)) != 0).sum()) == 0
    st = sim.env_stats().cpu().numpy()
    assert st[:, 2].mean() > 100
    idx = [0, 255]
    o = O.Oracle(s, init_poses=s.init_poses[idx])
    for e in idx:
        u, v, c, R = sim.get_state(e)
        assert np.all(u[s.fixed] == 0)
        tgt = s.poses[13][e].astype(np.float64)
        ref = o.eval(u, v, c, R, u, c, R, tgt)
        gpu = sim.debug_eval(e, u, v, c, R, u, c, R, tgt, s.dt)
        _assert_eval_parity(s, o, ref, gpu, u, v, u)


# ---------------------------------------------------------------- pose noise (R27)
def test_pose_noise_streams_match_oracle(torch_cuda):
    """Free indenter: each step ends at the perturbed target, so the GPU's converged pose
    equals the oracle's to far below the noise amplitude -- both implementations of
    Philox4x32-10 and of the perturbation draw the same stream."""
    import torch
    s = w.scene_c1(n_envs=40, steps=3)
    s.init_poses[:, 2] = 3e-3 + 5e-3
    s.poses[:, :, 2] = 3e-3 + 5e-3
    s.params.tol_x = 1e-12
    st, sr, seed = 2e-5, 1e-3, 1234
    sim = _sim(s)
    sim.set_pose_noise(st, sr, seed)
    o = O.Oracle(s)
    o.set_pose_noise(st, sr, seed)
    for k in range(3):
        sim.step(torch.tensor(s.poses[k], dtype=torch.float32, device="cuda").contiguous(), s.dt)
        o.step(s.poses[k], threads=8)
        for e in (0, 17, 39):
            _, _, c_g, R_g = sim.get_state(e)
            _, _, c_o, R_o = o.get_state(e)
            assert np.abs(c_g - c_o).max() < 1e-3 * st, (k, e)
            assert np.abs(R_g - R_o).max() < 1e-3 * sr, (k, e)
            assert np.abs(c_g - s.poses[k][e][:3]).max() > 1e-3 * st  # the noise is applied


def test_pose_noise_contact_parity_and_env_offset(torch_cuda):
    """Contact steps with noise converge to the oracle's states; a simulator holding envs
    [1, 3) with env_offset = 1 draws the same streams as the full batch."""
    import copy
    import torch
    s = w.scene_small_peg(n_envs=3, n_steps=3)
    st, sr, seed = 3e-5, 2e-3, 99
    s.params.tol_x = 1e-9
    s.params.max_iters = 8000
    s.params.stagnation = 3000
    sim = _sim(s)
    sim.set_pose_noise(st, sr, seed)
    p_or = w.Params(**{**s.params.__dict__})
    p_or.tol_x = 1e-11
    o = O.Oracle(s, params=p_or)
    o.set_pose_noise(st, sr, seed)
    sub = copy.deepcopy(s)
    sub.init_poses = s.init_poses[1:]
    sub.poses = s.poses[:, 1:]
    sim2 = _sim(sub)
    sim2.set_pose_noise(st, sr, seed, env_offset=1)
    for k in range(3):
        tgt = torch.tensor(s.poses[k], dtype=torch.float32, device="cuda").contiguous()
        sim.step(tgt, s.dt)
        sim2.step(tgt[1:].contiguous(), s.dt)
        o.step(s.poses[k], threads=3)
    mk = sim.markers().cpu().numpy()
    mk2 = sim2.markers().cpu().numpy()
    for e in range(3):
        _assert_parity(s, sim, o, mk, e)
    scale = np.abs(mk[1:]).max()
    assert np.abs(mk2 - mk[1:]).max() <= 1e-3 * scale


# ---------------------------------------------------------------- R33 constraint deduplication
def test_dedup_kernel_parity_and_closed_form(torch_cuda):
    """IPC-toolkit constraint deduplication on the GPU (dedup = 1): at a pressed C1 contact state
    the energy parts, gradient, blocks (element-wise bars) and the a6-a8 quantities match the
    oracle's deduplicated ones, and differ from the literal sum's.  (The closed form under an
    inverted pyramid's tip is pinned on the oracle only: there the tip projects exactly onto a
    mesh vertex, on a boundary between closest-feature regions, where the classification -- and
    R33's energy -- depends on the last bit of the barycentric solve, which two implementations
    with different operation orders need not share; the literal sum does not depend on it.)"""
    from test_oracle_dedup import _pyramid_scene
    h = 0.5e-4
    s = _pyramid_scene(h)
    sim = _sim(s)
    o = O.Oracle(s)
    z = np.zeros_like(s.X)
    c = s.init_poses[0, :3].astype(np.float64)
    gpu = sim.debug_eval(0, z, z, c, np.eye(3), z, c, np.eye(3), s.init_poses[0], s.dt)
    ref = o.eval(z, z, c, np.eye(3), z, c, np.eye(3), s.init_poses[0])
    assert abs(gpu["parts"][2] - ref["parts"][2]) <= 1e-9 * ref["parts"][2]  # literal: m kappa b(h)
    s, o0, (u_t, v_t, c_t, R_t), (u, c, R), tgt = _pressed_state()
    s.params.dedup = 1
    o = O.Oracle(s, params=s.params)
    sim = _sim(s)
    ut32 = u_t.astype(np.float32).astype(np.float64)
    vt32 = v_t.astype(np.float32).astype(np.float64)
    ref = o.eval(ut32, vt32, c_t, R_t, u, c, R, tgt)
    gpu = sim.debug_eval(0, ut32, vt32, c_t, R_t, u, c, R, tgt, s.dt)
    lit = o0.eval(ut32, vt32, c_t, R_t, u, c, R, tgt)
    assert lit["parts"][2] > ref["parts"][2] * (1 + 1e-3)  # duplicates exist here
    _assert_eval_parity(s, o, ref, gpu, ut32, vt32, u)
    st = (ut32, vt32, c_t, R_t)
    (u2, c2, R2), g_prev, p_prev, gPg_prev = _iteration_inputs(s, o, st, (u, c, R), tgt)
    p_o, r_o = o.iteration(*st, u2, c2, R2, tgt, g_prev, p_prev, gPg_prev, restart=True)
    p_g, r_g = sim.debug_iteration(0, *st, u2, c2, R2, tgt, s.dt, g_prev, p_prev, gPg_prev, restart=True)
    amp = max(1.0, np.sqrt(gPg_prev / r_o["gPg"]))
    for k in ("pHp", "alpha_bar", "alpha_ccd", "alpha"):
        assert _rel(r_g[k], r_o[k]) <= 4e-5 * amp, (k, r_g[k], r_o[k])


def test_dedup_converged_parity(torch_cuda):
    """Converged steps with deduplicated constraints (small peg, 3 ragged envs x 3 steps) match
    the oracle's on the north_star gates."""
    s = w.scene_small_peg(n_envs=3, n_steps=3)
    s.params.dedup = 1
    sim, o, mk = _run_both(s, 3)
    it, pg, fl = sim.env_status()
    for e in range(3):
        assert int(fl[e]) & 1 and o.status_of(e)["flags"] & 1, (e, int(fl[e]), o.status_of(e))
        _assert_parity(s, sim, o, mk, e)
