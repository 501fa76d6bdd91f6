"""Converged-step parity of the CUDA path with the fp64 oracle beyond the press: BASELINE
configs as stated, the sliding / rotating regime (P:305-307 press, slide and rotate
increments; friction P:436-446 is the physics of sliding), many sampled envs at full size,
and both contact-grid settings (the order of the fp32 atomic sums changes with it).

Gates (north_star): gel vertex positions within 1e-4 of the pad size, markers within 1e-3 of
the maximum marker displacement (relative L-inf).  Both sides converge every step: GPU
tol_x = 3e-10 m, oracle 1e-11 m.

Two kinds of comparison:
  * independent history -- both sides run the same targets from the same initial state;
  * same start -- the oracle runs step k from the GPU's own step-start state (read through the
    C ABI), so one step of the method is compared on identical inputs whatever the earlier
    steps did (that is how the sliding / twisting / releasing windows deep into a C3
    trajectory are compared without running the oracle through all the earlier steps).
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest

import oracle as O
import workloads as w

pytestmark = pytest.mark.gpu
MM = 1e-3
# GPU tolerance of these runs: 3e-10 m on |P g|_disp (the fp32 floor is ~1e-10 m); at 1e-9 m a
# step's error (~2e-8 m) exceeds 1e-3 of a first-contact marker field (~1.6e-5 m)
GPU_TOL = 3e-10


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _sim(scene, bps=None, **kw):
    import paper_2603_28475_b200 as P
    old = os.environ.get("TAC_CONTACT_BPS")
    if bps is not None:
        os.environ["TAC_CONTACT_BPS"] = str(bps)
    try:
        return P.TacSim.from_scene(scene, **kw)
    finally:
        if bps is not None:
            if old is None:
                del os.environ["TAC_CONTACT_BPS"]
            else:
                os.environ["TAC_CONTACT_BPS"] = old


def _tol_params(p, tol):
    q = w.Params(**p.__dict__)
    q.fixed_iters = 0
    q.tol_x = tol
    q.max_iters = 20000
    q.stagnation = 5000
    return q


def _oracle_converged(st):
    """The oracle reached tol_x (1e-11 m), or stopped on stagnation within 1e-10 m (its fp64
    floor on a few hard steps) -- inside the GPU's 3e-10 m."""
    return bool(st["flags"] & 1) or (bool(st["flags"] & 64) and st["pg"] <= 1e-10)


def _gates(scene, u_g, u_o, m_g, m_o, what, check=True):
    """north_star gates; returns |u_g - u_o|_inf (with check=False: whether both gates hold)."""
    pad = max(scene.extent)
    du = np.abs(u_g - u_o).max()
    scale = np.abs(m_o).max()
    dm = np.abs(m_g - m_o).max() if scale > 1e-7 else 0.0
    if not check:
        return du <= 1e-4 * pad and dm <= 1e-3 * scale
    assert du <= 1e-4 * pad, (what, du, 1e-4 * pad)
    assert dm <= 1e-3 * scale, (what, dm, scale)
    assert np.all(u_g[scene.fixed] == 0)
    return du


def _compare(scene, p_or, e, start, target, u_g, c_g, R_g, m_g, u_o, m_o, what, alt, oracle_ok=True):
    """Gates against the oracle's minimiser; where they fail, the GPU has reached ANOTHER local
    minimiser of the same step's incremental potential (the IPC potential is not convex: a gel
    vertex against a faceted indenter, R25) -- certified by the oracle itself: its
    PNCG started at the GPU's result (same anchors, same target) converges without leaving it
    (north_star gates between the GPU's state and the polished one).  `alt` collects these, and
    the steps whose own oracle solve stagnated (oracle_ok False) are certified the same way."""
    if oracle_ok and _gates(scene, u_g, u_o, m_g, m_o, what, check=False):
        return _gates(scene, u_g, u_o, m_g, m_o, what)
    o1 = O.Oracle(scene, params=p_or, init_poses=scene.init_poses[[0]])
    o1.set_state(0, *start)
    o1.step_from(0, target, u_g, c_g, R_g)
    st = o1.status_of(0)
    assert _oracle_converged(st), (what, "polish", st)
    du = _gates(scene, u_g, o1.get_state(0)[0], m_g, o1.markers(0), what + " (polished GPU minimiser)")
    alt.append((what, float(np.abs(u_g - u_o).max()), du))
    return du


@pytest.mark.parametrize("mu_f", [0.0, 1.0])
def test_c1_as_stated(torch_cuda, mu_f):
    """BASELINE configs[0] as stated: the 288-tet C1 pad, the R 3 mm sphere starting 0.2 mm
    above the pad pressed 0.5 mm below its top in ONE step, mu_f in {0, 1}.  (The step starts
    out of contact, so no friction anchor exists -- anchors are lagged at x^t, R7 -- and both
    mu_f give the same state; the test checks that too.)"""
    torch = torch_cuda
    s = w.scene_c1(mu_f=mu_f)
    sim = _sim(s, params=_tol_params(s.params, GPU_TOL))
    o = O.Oracle(s, params=_tol_params(s.params, 1e-11))
    sim.step(torch.tensor(s.poses[0], dtype=torch.float32, device="cuda").contiguous(), s.dt)
    o.step(s.poses[0])
    it, _, fl = sim.env_status()
    assert int(fl[0]) & 1 and _oracle_converged(o.status_of(0)), (int(fl[0]), o.status_of(0))
    u_g = sim.get_state(0)[0]
    u_o = o.get_state(0)[0]
    m_o = o.markers(0)
    assert np.abs(m_o).max() > 5e-5  # the press reaches the markers
    _gates(s, u_g, u_o, sim.markers().cpu().numpy()[0], m_o, f"C1 mu_f={mu_f}")
    s0 = w.scene_c1(mu_f=0.0 if mu_f else 1.0)
    o0 = O.Oracle(s0, params=_tol_params(s0.params, 1e-11))
    o0.step(s0.poses[0])
    assert np.abs(o0.get_state(0)[0] - u_o).max() == 0.0


def test_c2_press_and_slide(torch_cuda):
    """BASELINE configs[1] through its slide: C2's 19,800-tet pad and R 5 mm sphere, pressed
    11 x 0.1 mm then slid 10 x 0.05 mm along x with friction (mu_f = 1); independent histories,
    compared after every step of the slide (steps 11-20) and at the end of the press."""
    torch = torch_cuda
    s = w.scene_c2(steps=21)
    sim = _sim(s, params=_tol_params(s.params, GPU_TOL))
    o = O.Oracle(s, params=_tol_params(s.params, 1e-11))
    ex = cf.ThreadPoolExecutor(1)
    oracle_states = []

    def run_oracle():  # the oracle's ctypes calls release the GIL: it runs beside the GPU
        for k in range(21):
            o.step(s.poses[k])
            oracle_states.append((o.get_state(0)[0], o.markers(0), o.status_of(0)))
    fut = ex.submit(run_oracle)
    gpu_states = []
    for k in range(21):
        sim.step(torch.tensor(s.poses[k], dtype=torch.float32, device="cuda").contiguous(), s.dt)
        it, _, fl = sim.env_status()
        gpu_states.append((sim.get_state(0)[0], sim.markers().cpu().numpy()[0], int(fl[0])))
    fut.result()
    anchors_seen = 0
    for k in [10] + list(range(11, 21)):
        u_g, m_g, fg = gpu_states[k]
        u_o, m_o, so = oracle_states[k]
        assert fg & 1 and _oracle_converged(so), (k, fg, so)
        _gates(s, u_g, u_o, m_g, m_o, f"C2 step {k}")
    # sliding really happened: tangential marker motion grows along the slide
    assert np.abs(oracle_states[20][1][:, 0]).max() > 2 * np.abs(oracle_states[11][1][:, 0]).max()


def _phase_of(seed, k):
    """Phase of step k of a C3 trajectory from its noise-free path (the same draws as the
    noisy one): press / release (normal motion), shear (lateral), twist (yaw), hold."""
    _, p = w.peg_trajectory(seed, 64, noise=False)
    d = p[k] - p[k - 1]
    if abs(d[2]) > 1e-7:
        return "press" if d[2] < 0 else "release"
    if np.linalg.norm(d[:2]) > 1e-7:
        return "shear"
    if np.abs(p[k, 3:] - p[k - 1, 3:]).max() > 1e-9:
        return "twist"
    return "hold"


@pytest.mark.parametrize("bps", [8, 16])
def test_c3_full_size_windows_shear_twist_release(torch_cuda, bps):
    """C3 at full size (1,024 envs) in tolerance mode through step 30 of its trajectories; at
    steps 10, 20 and 30, 32 sampled envs per window (covering shear, twist and release steps)
    are compared with the oracle's step from the GPU's own step-start state.  Both
    contact-grid settings."""
    torch = torch_cuda
    s = w.scene_c3(n_envs=1024, n_steps=64)
    sim = _sim(s, bps=bps, params=_tol_params(s.params, GPU_TOL))
    p_or = _tol_params(s.params, 1e-11)
    nproc = os.cpu_count() or 1
    poses = torch.tensor(s.poses, dtype=torch.float32, device="cuda").contiguous()
    seen = {"press": 0, "release": 0, "shear": 0, "twist": 0, "hold": 0}
    worst = 0.0
    ex = cf.ThreadPoolExecutor(1)
    pending = []
    for k in range(31):
        if k in (10, 20, 30):
            phases = {e: _phase_of(20260000 + e, k) for e in range(1024)}
            pick = []
            for ph in ("shear", "twist", "release", "press", "hold"):
                pick += [e for e in range(1024) if phases[e] == ph][:10 if ph in ("shear", "twist", "release") else 3]
            pick = sorted(set(pick))[:32]
            starts = {e: sim.get_state(e) for e in pick}
        sim.step(poses[k], s.dt)
        it, _, fl = sim.env_status()
        fl = fl.cpu().numpy()
        # at 3e-10 m a few envs per step stop on stagnation instead (|P g| ~ 1e-7 m)
        assert (fl & 1).sum() >= 0.98 * 1024, (k, int((fl & 1).sum()))
        if k not in (10, 20, 30):
            continue
        mk = sim.markers().cpu().numpy()
        finals = {e: (sim.get_state(e), mk[e], int(fl[e])) for e in pick}

        def run_oracle(k=k, pick=pick, starts=starts):  # beside the GPU's next steps
            o = O.Oracle(s, params=p_or, init_poses=s.init_poses[pick])
            for j, e in enumerate(pick):
                o.set_state(j, *starts[e])
            o.step(s.poses[k][pick], threads=min(len(pick), nproc))
            return [(o.get_state(j)[0], o.markers(j), o.status_of(j)) for j in range(len(pick))]
        pending.append((k, pick, phases, starts, finals, ex.submit(run_oracle)))
    alt = []
    for k, pick, phases, starts, finals, fut in pending:
        res = fut.result()
        for j, e in enumerate(pick):
            seen[phases[e]] += 1
            u_o, m_o, st = res[j]
            (u_g, _, c_g, R_g), m_g, fg = finals[e]
            assert fg & (1 | 64), (k, e, fg)  # converged (or stagnated at |Pg| ~ 1e-7)
            # an oracle solve that stagnates from this start (seen once in ~600 env-steps, |Pg|
            # 2e-5 m after 5,600 iterations) is replaced by certifying the GPU's result
            worst = max(worst, _compare(s, p_or, e, starts[e], s.poses[k][e], u_g, c_g, R_g, m_g, u_o, m_o,
                                        f"C3 step {k} env {e} ({phases[e]})" + ("" if _oracle_converged(st)
                                                                                 else " [oracle stagnated]"),
                                        alt, oracle_ok=_oracle_converged(st)))
    n = sum(seen.values())
    print(f"bps {bps}: worst |u_gpu - u_oracle| = {worst:.3e} m over {n} env-steps {seen}; "
          f"other local minimisers: {alt}")
    assert seen["shear"] >= 8 and seen["twist"] >= 8 and seen["release"] >= 4, seen
    # measured 2-5 % of the deep shear / twist / release steps land on another certified minimiser
    assert len(alt) <= 0.1 * n, alt


@pytest.mark.parametrize("bps", [8, 16])
def test_c3_full_size_independent_history_32_envs(torch_cuda, bps):
    """C3 at full size in tolerance mode for its first 4 steps (press), 32 envs sampled across
    the batch, independent histories: every sampled env converges at every step and matches
    the oracle after every step.  Both contact-grid settings."""
    torch = torch_cuda
    s = w.scene_c3(n_envs=1024, n_steps=4)
    sim = _sim(s, bps=bps, params=_tol_params(s.params, GPU_TOL))
    idx = list(range(5, 1024, 32))
    o = O.Oracle(s, params=_tol_params(s.params, 1e-11), init_poses=s.init_poses[idx])
    nproc = os.cpu_count() or 1
    ex = cf.ThreadPoolExecutor(1)
    worst = 0.0
    alt = []
    p_or = _tol_params(s.params, 1e-11)
    for k in range(4):
        starts = {e: sim.get_state(e) for e in idx}
        fut = ex.submit(o.step, s.poses[k][idx], None, min(len(idx), nproc))
        sim.step(torch.tensor(s.poses[k], dtype=torch.float32, device="cuda"), s.dt)
        it, _, fl = sim.env_status()
        fl = fl.cpu().numpy()
        mk = sim.markers().cpu().numpy()
        fut.result()
        assert (fl & 1).sum() >= 0.98 * 1024
        for j, e in enumerate(idx):
            assert _oracle_converged(o.status_of(j)), (k, e, o.status_of(j))
            assert fl[e] & (1 | 64), (k, e, int(fl[e]))
            u_g, _, c_g, R_g = sim.get_state(e)
            n_alt = len(alt)
            worst = max(worst, _compare(s, p_or, e, starts[e], s.poses[k][e], u_g, c_g, R_g, mk[e],
                                        o.get_state(j)[0], o.markers(j), f"C3 step {k} env {e}", alt))
            if len(alt) > n_alt:  # the histories part here: the oracle continues from the GPU's state
                o.set_state(j, *sim.get_state(e))
    print(f"bps {bps}: worst |u_gpu - u_oracle| = {worst:.3e} m; other local minimisers: {alt}")
    assert len(alt) <= 0.1 * len(idx) * 4, alt


def test_c5_converged_same_start(torch_cuda):
    """C5 (103,680 tets, sharp square peg, 256 envs) in tolerance mode through step 6 of its face
    press; two sampled envs' step 6 matches the oracle's step from the same start."""
    torch = torch_cuda
    s = w.scene_c5(n_envs=256, n_steps=8)
    tol = _sim(s, params=_tol_params(s.params, GPU_TOL))
    poses = torch.tensor(s.poses, dtype=torch.float32, device="cuda").contiguous()
    for k in range(6):
        tol.step(poses[k], s.dt)
    pick = [0, 255]
    starts = {e: tol.get_state(e) for e in pick}
    tol.step(poses[6], s.dt)
    it, _, fl = tol.env_status()
    mk = tol.markers().cpu().numpy()
    assert tol.env_stats().cpu().numpy()[pick, 2].min() > 0  # friction anchors: in contact
    o = O.Oracle(s, params=_tol_params(s.params, 1e-11), init_poses=s.init_poses[pick])
    for j, e in enumerate(pick):
        o.set_state(j, *starts[e])
    o.step(s.poses[6][pick], threads=2)
    alt = []
    for j, e in enumerate(pick):
        assert _oracle_converged(o.status_of(j)) and int(fl[e]) & (1 | 64), (e, o.status_of(j), int(fl[e]))
        u_g, _, c_g, R_g = tol.get_state(e)
        _compare(s, _tol_params(s.params, 1e-11), e, starts[e], s.poses[6][e], u_g, c_g, R_g, mk[e],
                 o.get_state(j)[0], o.markers(j), f"C5 env {e}", alt)
    print(f"other local minimisers: {alt}")
