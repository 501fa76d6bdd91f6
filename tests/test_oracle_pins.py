"""Pins of the fp64 oracle against what the paper and the mathematics fix
(SURVEY §8c.4).  None of these re-call the oracle routine under test to produce
the expected value: expected values come from closed forms, the paper's printed
formulas, finite differences, brute force, or independent numpy code.
"""
import math

import numpy as np
import pytest

import oracle as O
import workloads as w
from helpers import c1_press_scene, quat_R, rot_exp

DHAT = 1e-4


# ---------------------------------------------------------------- barrier
def test_barrier_closed_forms():
    # b(dhat/2) with dhat = 1 -> 0.25 ln 2
    assert O.barrier(0.5, 1.0) == pytest.approx(0.25 * math.log(2), rel=1e-15)
    # C^2 at dhat: b = b' = b'' = 0 (activation threshold)
    for k in range(3):
        assert O.barrier(1.0, 1.0, k) == 0.0
        assert abs(O.barrier(1.0 - 1e-9, 1.0, k)) < 1e-7
    # monotone decreasing on (0, dhat) and unbounded at 0
    ds = np.linspace(1e-6, 1 - 1e-6, 200)
    b = [O.barrier(d, 1.0) for d in ds]
    assert np.all(np.diff(b) < 0)
    assert O.barrier(1e-8, 1.0) > O.barrier(1e-4, 1.0)


@pytest.mark.parametrize("d", [0.3, 0.05, 0.7])
def test_barrier_derivatives_fd(d):
    h = 1e-6
    for k in range(2):
        fd = (O.barrier(d + h, 1.0, k) - O.barrier(d - h, 1.0, k)) / (2 * h)
        assert O.barrier(d, 1.0, k + 1) == pytest.approx(fd, rel=1e-6)


def test_friction_force_magnitude_closed_form():
    # App. B: -b'(0.5 dhat) = dhat (ln 2 + 0.5)
    assert -O.barrier(0.5 * DHAT, DHAT, 1) == pytest.approx(DHAT * (math.log(2) + 0.5), rel=1e-12)


# ---------------------------------------------------------------- mollifier
def test_mollifier_values():
    eps = 1e-5
    assert O.mollifier(0, eps) == eps / 3  # f(0) = eps/3
    assert O.mollifier(0, eps, 1) == 0.0
    assert O.mollifier(eps, eps) == pytest.approx(eps, rel=1e-15)  # f(eps) = eps
    assert O.mollifier(2 * eps, eps) == 2 * eps  # linear branch
    # C^1 at the knot from both sides
    lo = eps * (1 - 1e-10)
    assert abs(O.mollifier(lo, eps) - eps) < 1e-10 * eps * 10
    assert abs(O.mollifier(lo, eps, 1) - 1.0) < 1e-9
    assert O.mollifier(eps, eps, 1) == 1.0
    # the printed polynomial at s = eps/2
    s = eps / 2
    assert O.mollifier(s, eps) == pytest.approx(-s ** 3 / (3 * eps ** 2) + s * s / eps + eps / 3, rel=1e-15)


# ---------------------------------------------------------------- SNH (DESIGN R1)
def test_psi_rest_rotation_and_small_strain():
    E, nu = 1e5, 0.45
    mu = E / (2 * (1 + nu))
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    assert abs(O.psi(E, nu, np.eye(3))) < 1e-9
    Q = rot_exp([0.3, -0.2, 0.5])
    assert abs(O.psi(E, nu, Q)) < 1e-8 * mu
    rng = np.random.default_rng(1)
    for eps in (1e-3, 1e-4):
        G = eps * rng.standard_normal((3, 3))
        lin = mu * np.sum(((G + G.T) / 2) ** 2) + lam / 2 * np.trace(G) ** 2  # Lame linear elasticity
        val = O.psi(E, nu, np.eye(3) + G)
        assert abs(val - lin) < 20 * eps * abs(lin)  # O(G^3) difference


# ---------------------------------------------------------------- distances
def _bf_pt(p, t0, t1, t2, n=400):
    a, b = np.meshgrid(np.linspace(0, 1, n + 1), np.linspace(0, 1, n + 1))
    m = a + b <= 1
    a, b = a[m], b[m]
    pts = t0 + a[:, None] * (t1 - t0) + b[:, None] * (t2 - t0)
    return np.min(np.linalg.norm(pts - p, axis=1))


def _bf_ee(a0, a1, b0, b1, n=600):
    s = np.linspace(0, 1, n + 1)
    A = a0 + s[:, None] * (a1 - a0)
    B = b0 + s[:, None] * (b1 - b0)
    return np.min(np.linalg.norm(A[:, None, :] - B[None, :, :], axis=2))


def test_distance_closed_forms():
    # point above the interior of a large triangle at height dhat/2
    d, wgt = O.dist_pt([0.2, 0.2, 0.5 * DHAT], [0, 0, 0], [1, 0, 0], [0, 1, 0])
    assert d == pytest.approx(0.5 * DHAT, rel=1e-12)
    assert wgt[0] == 1 and wgt[1:].sum() == pytest.approx(-1)
    # perpendicular skew edges with gap g
    g = 3e-5
    d, wgt = O.dist_ee([-1, 0, 0], [1, 0, 0], [0, -1, g], [0, 1, g])
    assert d == pytest.approx(g, rel=1e-12)
    assert np.allclose(wgt, [0.5, 0.5, -0.5, -0.5])
    # parallel edges: fall back to endpoint distances
    d, _ = O.dist_ee([0, 0, 0], [1, 0, 0], [0.5, 0, g], [2, 0, g])
    assert d == pytest.approx(g, rel=1e-12)


def test_distance_random_vs_bruteforce():
    rng = np.random.default_rng(7)
    for _ in range(25):
        p, t0, t1, t2 = rng.standard_normal((4, 3))
        d, wgt = O.dist_pt(p, t0, t1, t2)
        bf = _bf_pt(p, t0, t1, t2)
        scale = max(np.linalg.norm(t1 - t0), np.linalg.norm(t2 - t0))
        assert d <= bf + 1e-12
        assert bf - d <= 2.5 * scale / 400
        r = wgt[0] * p + wgt[1] * t0 + wgt[2] * t1 + wgt[3] * t2
        assert np.linalg.norm(r) == pytest.approx(d, rel=1e-10)
        assert wgt[1:].sum() == pytest.approx(-1, abs=1e-12) and np.all(wgt[1:] <= 1e-15)
        a0, a1, b0, b1 = rng.standard_normal((4, 3))
        d, wgt = O.dist_ee(a0, a1, b0, b1)
        bf = _bf_ee(a0, a1, b0, b1)
        assert d <= bf + 1e-12
        assert bf - d <= 2.5 * max(np.linalg.norm(a1 - a0), np.linalg.norm(b1 - b0)) / 600
        r = wgt[0] * a0 + wgt[1] * a1 + wgt[2] * b0 + wgt[3] * b1
        assert np.linalg.norm(r) == pytest.approx(d, rel=1e-10)


def test_certificate_closed_forms():
    """R15 far-pair certificates: the largest axis gap between the corner boxes (normal =
    that axis, oriented from side B to side A); failing that, the primitive-plane gap,
    which equals the exact distance when the closest points are interior."""
    t0, t1, t2 = np.array([0, 0, 0.0]), np.array([1e-3, 0, 0]), np.array([0, 1e-3, 0])
    ok, g, n = O.certificate(np.stack([[2e-4, 3e-4, 2 * DHAT], t0, t1, t2]), 1, DHAT)
    assert ok and g == pytest.approx(2 * DHAT, rel=1e-12) and np.array_equal(n, [0, 0, 1])
    ok, g, n = O.certificate(np.stack([[2e-4, 3e-4, -0.5 * DHAT], t0, t1, t2]), 1, DHAT)
    assert not ok and g == pytest.approx(0.5 * DHAT, rel=1e-12)
    # triangle tilted about x, point 2 dhat above its interior along the normal: the boxes
    # overlap on every axis, the triangle's plane certifies the exact distance
    c, s = math.cos(0.6), math.sin(0.6)
    t0, t1, t2 = np.array([-1e-3, -1e-3 * c, -1e-3 * s]), np.array([1e-3, -1e-3 * c, -1e-3 * s]), \
        np.array([0, 1e-3 * c, 1e-3 * s])
    nrm = np.cross(t1 - t0, t2 - t0)
    nrm /= np.linalg.norm(nrm)
    p = 2 * DHAT * nrm
    z = np.stack([p, t0, t1, t2])
    assert np.all((p > z[1:].min(0)) & (p < z[1:].max(0)))
    ok, g, n = O.certificate(z, 1, DHAT)
    assert ok and g == pytest.approx(2 * DHAT, rel=1e-9) and n @ nrm == pytest.approx(1, abs=1e-12)
    assert g <= O.dist_pt(p, t0, t1, t2)[0] * (1 + 1e-12)
    ok, g, _ = O.certificate(np.stack([0.5 * DHAT * nrm, t0, t1, t2]), 1, DHAT)
    assert not ok and g == pytest.approx(0.5 * DHAT, rel=1e-9)
    # crossing skew segments 1.5 dhat apart along a tilted common normal
    e = np.array([0, c, s])
    m = np.cross([1, 0, 0], e)
    z = np.stack([[-1e-3, 0, 0], [1e-3, 0, 0], -1e-3 * e + 1.5 * DHAT * m, 1e-3 * e + 1.5 * DHAT * m])
    ok, g, _ = O.certificate(z, 2, DHAT)
    assert ok and g == pytest.approx(1.5 * DHAT, rel=1e-9)
    # parallel segments: no plane certificate from the degenerate cross product
    z = np.stack([[0, 0, 0], [1e-3, 0, 0], [2e-4, 0, 0.5 * DHAT], [1.2e-3, 1e-9, 0.5 * DHAT]])
    ok, g, _ = O.certificate(z, 2, DHAT)
    assert not ok and g < DHAT


def test_certificate_never_exceeds_distance():
    """Any certified separation is a lower bound of the exact distance (brute force)."""
    rng = np.random.default_rng(11)
    n_ok = 0
    for _ in range(200):
        z = rng.standard_normal((4, 3)) * 1e-3
        for na in (1, 2):
            ok, g, _ = O.certificate(z, na, DHAT)
            bf = _bf_pt(*z) if na == 1 else _bf_ee(*z)
            assert g <= bf * (1 + 1e-9) + 1e-15
            n_ok += ok
    assert 50 < n_ok < 400


# ---------------------------------------------------------------- DK-NCG
def _pcg(A, b, x0, iters, Pdiag):
    """Textbook preconditioned CG (Hestenes-Stiefel / Saad Alg. 9.1)."""
    x = x0.copy()
    r = b - A @ x
    z = Pdiag * r
    p = z.copy()
    xs = [x.copy()]
    for _ in range(iters):
        Ap = A @ p
        a = (r @ z) / (p @ Ap)
        x = x + a * p
        r2 = r - a * Ap
        z2 = Pdiag * r2
        beta = (r2 @ z2) / (r @ z)
        p = z2 + beta * p
        r, z = r2, z2
        xs.append(x.copy())
    return np.array(xs)


@pytest.mark.parametrize("rule", [0, 3])
@pytest.mark.parametrize("identity", [True, False])
def test_dk_equals_pcg_on_spd_quadratics(identity, rule):
    """On SPD quadratics with exact line search the paper's DK beta and
    alpha_bar reproduce textbook (P)CG iterates.  DK+ (rule 3,
    R28) truncates beta below at 0.5 g_{k+1}^T p_k / |p_k|^2, which is 0 under exact line
    search while the PCG beta is positive: the same iterates."""
    rng = np.random.default_rng(3)
    for n in (5, 20, 40):
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        A = Q @ np.diag(rng.uniform(0.5, 20, n)) @ Q.T
        A += np.diag(rng.uniform(0, 30, n))  # make Jacobi non-trivial
        b = rng.standard_normal(n)
        x0 = rng.standard_normal(n)
        it = min(n, 15)
        xs = O.ncg_quadratic(A, b, x0, it, precond_identity=identity, rule=rule)
        ref = _pcg(A, b, x0, it, np.ones(n) if identity else 1 / np.diag(A))
        assert np.max(np.abs(xs - ref)) < 1e-9 * np.max(np.abs(ref))
        if n <= 20:  # converges within n (+5) iterations
            xs = O.ncg_quadratic(A, b, x0, n + 5, precond_identity=identity, rule=rule)
            assert np.linalg.norm(A @ xs[-1] - b) < 1e-8 * np.linalg.norm(b)


def test_alpha_bar_identity_hessian():
    # H = I, p = -g  =>  alpha_bar = 1: one step lands on the minimiser
    b = np.array([1.0, -2.0, 3.0])
    xs = O.ncg_quadratic(np.eye(3), b, np.zeros(3), 1, precond_identity=True)
    assert np.allclose(xs[1], b, atol=1e-15)


# ---------------------------------------------------------------- SO(3)
def test_so3_and_quaternion():
    rng = np.random.default_rng(2)
    for _ in range(10):
        wv = rng.standard_normal(3)
        wv *= rng.uniform(1e-9, 3.0) / np.linalg.norm(wv)  # angle below pi: log is the principal branch
        R, l = O.so3_exp_log(wv)
        assert np.allclose(R, rot_exp(wv), atol=1e-14)
        assert np.allclose(l, wv, rtol=1e-9, atol=1e-15)
        q = rng.standard_normal(4)
        assert np.allclose(O.quat_to_R(np.concatenate([[0, 0, 0], q])), quat_R(q), atol=1e-15)


# ---------------------------------------------------------------- pose noise (R27)
def _kat():
    import os
    rows = []
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")):
        if line.strip() and not line.startswith("#"):
            v = [int(x, 16) for x in line.split()]
            rows.append((v[:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers():
    rows = _kat()
    assert len(rows) == 3
    for ctr, key, out in rows:
        assert [int(x) for x in O.philox4x32_10(ctr, key)] == out


def test_pose_noise_statistics_and_determinism():
    """Free indenter (no contact): one step ends at the perturbed target, so c - c_target
    samples s_t * U(-1, 1)^3 and the rotation vector of R R_target^T samples s_r *
    U(-1, 1)^3 (scipy's rotation-vector map, independent of the oracle); per-env streams
    are reproducible and distinct."""
    from scipy.spatial.transform import Rotation
    s = w.scene_c1(n_envs=96)
    R0 = 3e-3
    s.init_poses[:, 2] = R0 + 5e-3
    s.poses[:, :, 2] = R0 + 5e-3
    s.params.tol_x = 1e-12
    st, sr = 2e-5, 1e-3
    outs = []
    for seed in (7, 7, 8):
        o = O.Oracle(s)
        o.set_pose_noise(st, sr, seed)
        o.step(s.poses[0], threads=8)
        dc, rv = [], []
        for e in range(s.n_envs):
            _, _, c, R = o.get_state(e)
            dc.append(c - s.poses[0][e][:3])
            rv.append(Rotation.from_matrix(R @ O.quat_to_R(s.poses[0][e]).T).as_rotvec())
        outs.append((np.array(dc), np.array(rv)))
    (dc, rv), (dc2, rv2), (dc3, _) = outs
    assert np.array_equal(dc, dc2) and np.array_equal(rv, rv2) and not np.allclose(dc, dc3)
    assert len({tuple(np.round(d / st, 9)) for d in dc}) == s.n_envs
    for x, sig in ((dc, st), (rv, sr)):
        assert np.abs(x).max() <= sig * (1 + 1e-5)
        assert abs(x.mean()) < 0.15 * sig
        assert abs((x ** 2).mean() / (sig ** 2 / 3) - 1) < 0.2
