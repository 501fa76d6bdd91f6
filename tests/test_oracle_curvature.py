"""Pins of the oracle's curvature p^T H p ("p^T H p ... in parallel with
minimal FLOPs") and of the step-length quantities built on it.

Expected values never come from `curvature()` itself:
  * the inertia, elastic (exact SNH second derivative) and pose-spring terms are the
    second derivative d^2/dt^2 E(x + t p) of the pinned energy, by Richardson-extrapolated
    central differences, at a contact-free state whose pose spring sits in its quadratic
    branch with R = R* (there the spring's Gauss-Newton form is its exact Hessian);
  * the contact terms are the Gauss-Newton forms of DESIGN.md R8 written from their
    definitions: kappa b''(d_k) (d d_k/dt)^2 per barrier pair, with d_k(t) evaluated by the
    pinned point-triangle / edge-edge distance functions along the path and differentiated
    numerically, plus the friction term, which at the step start (every slip Delta_k = 0)
    equals the exact second derivative of the friction energy (f''(0) = f'(s)/s -> 2/eps).
A dropped term, a wrong factor on the 2(lambda'(J-1) - mu) F:cof(dF) term, a missing kappa
or b'' sign, or a friction weight off by a factor fails one of these."""
import numpy as np
import pytest

import oracle as O
import workloads as w
from helpers import c1_press_scene, rot_exp

H = 5e-3


def _E(o, st, u, c, R, tgt, parts=None):
    r = o.eval(*st, u, c, R, tgt)
    return r["E"] if parts is None else sum(r["parts"][k] for k in parts)


def _second_derivative(f, t):
    """d^2 f / dt^2 at 0: central differences at t and t/2, Richardson-extrapolated (O(t^4))."""
    d1 = (f(t) - 2 * f(0.0) + f(-t)) / t ** 2
    d2 = (f(t / 2) - 2 * f(0.0) + f(-t / 2)) / (t / 2) ** 2
    return (4 * d2 - d1) / 3, abs(d2 - d1)


def _path(u, c, R, p, pc, pth, t):
    """The oracle's update x + t p (O4g): u + t p, c + t p_c, R <- exp([t p_theta]) R."""
    return u + t * p, c + t * pc, rot_exp(t * pth) @ R


def test_curvature_elastic_inertia_spring_exact():
    """Contact-free C1 state: p^T H p = d^2/dt^2 E(x + t p) (inertia, exact SNH quadratic form,
    quadratic-branch pose spring with R = R*)."""
    s = w.scene_c1()
    s.init_poses[0, 2] = 8e-3  # sphere 5 mm above the pad: no candidate pair
    o = O.Oracle(s)
    rng = np.random.default_rng(3)
    X = s.X
    free = np.setdiff1d(np.arange(len(X)), s.fixed)
    # a smooth, finite deformation (strains ~1e-2: the nonlinear SNH terms matter)
    u_t = np.zeros_like(X)
    u_t[:, 0] = 1.5e-4 * np.sin(X[:, 1] / 4e-3) * (X[:, 2] + 4e-3) / 4e-3
    u_t[:, 2] = -2e-4 * np.cos(X[:, 0] / 5e-3) * (X[:, 2] + 4e-3) / 4e-3
    u_t[s.fixed] = 0
    v_t = 1e-3 * rng.standard_normal(X.shape)
    v_t[s.fixed] = 0
    u = u_t + 3e-5 * rng.standard_normal(X.shape)
    u[s.fixed] = 0
    c_t = s.init_poses[0, :3].astype(np.float64)
    R_t = O.quat_to_R(s.init_poses[0])
    c = c_t + np.array([2e-8, -1e-8, 3e-8])  # |c - c*| << F_max / k_t = 1e-7 m: quadratic branch
    R = R_t.copy()
    tgt = s.init_poses[0].astype(np.float64)  # R* = R
    st = (u_t, v_t, c_t, R_t)
    assert o.eval(*st, u, c, R, tgt)["n_cand"] == 0
    for trial in range(3):
        p = rng.standard_normal(X.shape) * 1e-5
        p[s.fixed] = 0
        pc = rng.standard_normal(3) * 1e-9
        pth = rng.standard_normal(3) * 1e-7
        q = o.curvature(u_t, c_t, R_t, u, c, R, p, np.concatenate([pc, pth]), tgt)
        # |t p_theta| <= T_max / k_r = 5e-8 rad: the torque spring stays in its quadratic branch
        f = lambda t: _E(o, st, *_path(u, c, R, p, pc, pth, t), tgt)
        ref, err = _second_derivative(f, 0.2)
        assert q > 0
        assert abs(q - ref) <= 1e-6 * abs(ref) + 10 * err, (trial, q, ref, err)
    # the pin bites: dropping the det term (2 (lambda'(J-1) - mu) F:cof dF) changes q by far more
    # than the tolerance at this strain level -- checked via a direction along the deformation
    p = u_t.copy()
    q = o.curvature(u_t, c_t, R_t, u, c, R, p, np.zeros(6), tgt)
    ref, err = _second_derivative(lambda t: _E(o, st, *_path(u, c, R, p, np.zeros(3), np.zeros(3), t), tgt), 0.05)
    assert abs(q - ref) <= 1e-6 * abs(ref) + 10 * err


def _pair_corners(o, s, surf, kind, a, b, u, c, R):
    sv, se, st_, ie = surf
    x = s.X + u
    y = (R @ s.Y.T).T + c
    if kind == 0:
        return x[sv[a]], y[s.tris[b, 0]], y[s.tris[b, 1]], y[s.tris[b, 2]]
    if kind == 1:
        return y[a], x[st_[b, 0]], x[st_[b, 1]], x[st_[b, 2]]
    return x[se[a, 0]], x[se[a, 1]], y[ie[b, 0]], y[ie[b, 1]]


def _quat_of(R):
    """(w, x, y, z) of a rotation matrix near the identity."""
    wq = 0.5 * np.sqrt(1.0 + np.trace(R))
    return np.array([wq, (R[2, 1] - R[1, 2]) / (4 * wq), (R[0, 2] - R[2, 0]) / (4 * wq), (R[1, 0] - R[0, 1]) / (4 * wq)])


def _dist(kind, z):
    return (O.dist_ee(*z) if kind == 2 else O.dist_pt(*z))[0]


@pytest.mark.parametrize("mu_f", [0.0, 1.0])
def test_curvature_contact_gauss_newton(mu_f):
    """Pressed C1 state at its step start (every friction slip 0): p^T H p = exact second
    derivative of the smooth parts (inertia, elastic, pose with R = R*) + sum over pairs with
    d < dhat of kappa b''(d) (d'(0))^2 (R8) + the friction term (exact at zero slip)."""
    sc = c1_press_scene(mu_f=mu_f, steps=4, depth=0.25e-3)
    sc.params.tol_x = 1e-10
    o = O.Oracle(sc)
    for k in range(3):
        o.step(sc.poses[k])
    u_t, v_t, c_t, R_t = o.get_state(0)
    u, c, R = u_t.copy(), c_t.copy(), R_t.copy()
    tgt = np.concatenate([c_t, _quat_of(R_t)])  # target = the current pose: R* = R, c* = c
    assert np.abs(O.quat_to_R(tgt) - R_t).max() < 1e-14
    st = (u_t, v_t, c_t, R_t)
    r0 = o.eval(*st, u, c, R, tgt)
    assert r0["parts"][2] > 0 and (mu_f == 0 or r0["n_anchor"] > 3)
    surf = o.surface()
    pairs = o.broadphase_state(u, c, R, o.params.dhat + o.params.bp_margin)
    kappa = H * H * o.kappa_phys
    dhat = o.params.dhat
    rng = np.random.default_rng(17)
    for trial in range(3):
        # every term present and significant: gel motion (elastic ~80 %, friction ~10 %, barrier
        # ~1-2 %, inertia ~3e-4 of the total) plus a small rigid motion (pose spring ~10 %)
        p = rng.standard_normal(u.shape) * 1e-6
        p[np.linalg.norm(sc.X + u - c, axis=1) < 3.6e-3] *= 10  # emphasise the gel under the sphere
        p[sc.fixed] = 0
        pc = rng.standard_normal(3) * 1e-8
        pth = rng.standard_normal(3) * 1e-8
        q = o.curvature(u_t, c_t, R_t, u, c, R, p, np.concatenate([pc, pth]), tgt)
        smooth = lambda t: _E(o, st, *_path(u, c, R, p, pc, pth, t), tgt, parts=(0, 1, 4))
        ref_s, err_s = _second_derivative(smooth, 2e-3)
        # the friction energy is C^2 but not C^3 at zero slip (f has an |s|^3 term): its central
        # differences converge at O(t) only -- a short step (slip 1e-10 m << eps = 1e-5 m) on the
        # friction part alone (small, so little cancellation)
        fric, err_f = _second_derivative(lambda t: _E(o, st, *_path(u, c, R, p, pc, pth, t), tgt, parts=(3,)), 2e-5)
        ref_b = 0.0
        for kind, a, b in pairs:
            z0 = _pair_corners(o, sc, surf, kind, a, b, u, c, R)
            d0 = _dist(kind, z0)
            if d0 >= dhat:
                continue
            tt = 1e-4
            dp = _dist(kind, _pair_corners(o, sc, surf, kind, a, b, *_path(u, c, R, p, pc, pth, tt)))
            dm = _dist(kind, _pair_corners(o, sc, surf, kind, a, b, *_path(u, c, R, p, pc, pth, -tt)))
            ref_b += kappa * O.barrier(d0, dhat, 2) * ((dp - dm) / (2 * tt)) ** 2
        ref = ref_s + fric + ref_b
        tol = 1e-6 * abs(ref) + 10 * (err_s + err_f)
        # the pin bites: a 10 % error in the barrier or friction term exceeds the tolerance
        assert tol < 0.1 * ref_b and (mu_f == 0 or tol < 0.1 * fric), (tol, ref_b, fric)
        assert abs(q - ref) <= tol, (trial, q, ref_s, ref_b, err_s)
