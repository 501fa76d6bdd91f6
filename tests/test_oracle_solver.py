"""Pins of the oracle's energy, gradient, diagonal blocks, broad phase, step
bound, whole-step minimiser and invariants (BASELINE north_star
oracle checks).  Expected values come from finite differences, closed forms,
independent numpy code (linear elasticity, point location, box predicate,
Newton's method) or invariants — never from the routine under test."""
import numpy as np
import pytest

import oracle as O
import workloads as w
from helpers import c1_press_scene, rot_exp

H = 5e-3


@pytest.fixture(scope="module")
def pressed():
    """Oracle-generated feasible contact state of C1 (sphere pressed 0.15 mm), with
    friction anchors from the previous step."""
    s = c1_press_scene(mu_f=1.0, steps=4, depth=0.25e-3)
    s.params.tol_x = 1e-10
    o = O.Oracle(s)
    assert o.status == 0
    for k in range(3):
        o.step(s.poses[k])
    u_t, v_t, c_t, R_t = o.get_state(0)
    o.step(s.poses[3])
    u, _, c, R = o.get_state(0)
    rng = np.random.default_rng(5)
    u = u + 2e-7 * rng.standard_normal(u.shape)
    u[s.fixed] = 0
    c = c + 1e-7 * rng.standard_normal(3)
    R = rot_exp(1e-5 * rng.standard_normal(3)) @ R
    tgt = s.poses[3][0].copy()
    tgt[2] -= 2e-5  # target not at the current pose: spring active in its linear (capped) branch
    return s, o, (u_t, v_t, c_t, R_t), (u, c, R), tgt


def test_state_has_contact_and_friction(pressed):
    s, o, st, (u, c, R), tgt = pressed
    r = o.eval(*st, u, c, R, tgt)
    assert r["n_anchor"] > 3 and r["parts"][2] > 0 and r["parts"][3] > 0
    assert o.dmin(u, c, R) < 1e-4


def test_gradient_matches_central_fd(pressed):
    """north_star: gradients match central finite differences to 1e-6 relative."""
    s, o, st, (u, c, R), tgt = pressed
    r = o.eval(*st, u, c, R, tgt)
    free = np.setdiff1d(np.arange(len(u)), s.fixed)
    eps = 1e-9
    fd = np.zeros_like(u)
    for v in free:
        for a in range(3):
            up = u.copy(); up[v, a] += eps
            um = u.copy(); um[v, a] -= eps
            fd[v, a] = (o.eval(*st, up, c, R, tgt)["E"] - o.eval(*st, um, c, R, tgt)["E"]) / (2 * eps)
    g = r["g"][free]
    assert np.linalg.norm(fd[free] - g) <= 1e-6 * np.linalg.norm(g)
    # rigid DOFs: c and the left-trivialised rotation R <- exp([d]) R (DESIGN R18)
    fr = np.zeros(6)
    for a in range(3):
        e = np.zeros(3); e[a] = eps
        fr[a] = (o.eval(*st, u, c + e, R, tgt)["E"] - o.eval(*st, u, c - e, R, tgt)["E"]) / (2 * eps)
        e = np.zeros(3); e[a] = 1e-8
        fr[3 + a] = (o.eval(*st, u, c, rot_exp(e) @ R, tgt)["E"] - o.eval(*st, u, c, rot_exp(-e) @ R, tgt)["E"]) / 2e-8
    assert np.linalg.norm(fr - r["grig"]) <= 1e-6 * np.linalg.norm(r["grig"])


def test_inertia_closed_form():
    """single node of mass 2 displaced (1,0,0) -> value 1, gradient (2,0,0)."""
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]) * 1e-3
    tets = np.array([[0, 1, 2, 3]], np.int32)
    vol = 1e-9 / 6
    Y, tris = w.make_icosphere(1e-3, 0)
    sc = w.Scene("one", X, tets, np.array([1, 2, 3], np.int32), Y, tris, np.array([[0.2e-3, 0.2e-3, 0.0]]),
                 np.eye(3), np.array([w.pose((0, 0, 1.0), [1, 0, 0, 0])]), np.zeros((1, 1, 7)))
    sc.material = w.Material(E=0.0, nu=0.3, rho=2.0 * 4 / vol, mu_f=0.0)
    sc.params.kappa_phys = 1.0
    o = O.Oracle(sc)
    z = np.zeros((4, 3))
    u = z.copy(); u[0] = (1, 0, 0)
    r = o.eval(z, z, [0, 0, 1.0], np.eye(3), u, [0, 0, 1.0], np.eye(3), [0, 0, 1.0, 1, 0, 0, 0])
    assert r["parts"][0] == pytest.approx(1.0, rel=1e-12)
    assert np.allclose(r["g"][0], [2, 0, 0], rtol=1e-12)
    assert np.allclose(np.diag(r["D"][0]), [2, 2, 2], rtol=1e-12)
    m, v = o.mass_vol()
    assert m[0] == pytest.approx(2.0) and v[0] == pytest.approx(vol, rel=1e-12)


def _no_contact_scene():
    s = w.scene_c1(mu_f=0.0)
    s.init_poses = np.stack([w.pose((0, 0, 0.05), [1, 0, 0, 0])])  # indenter 5 cm away
    s.poses = np.stack([s.init_poses])
    return s


def test_rest_rotation_patch_and_diag_blocks():
    s = _no_contact_scene()
    o = O.Oracle(s)
    z = np.zeros_like(s.X)
    far = np.array([0, 0, 0.05])
    tgt = s.init_poses[0]
    r = o.eval(z, z, far, np.eye(3), z, far, np.eye(3), tgt)
    assert abs(r["parts"][1]) < 1e-18 and np.abs(r["g"]).max() < 1e-16  # typical values: 1e-7, 1e-8
    # rigid rotation of the whole pad: zero elastic energy (frame invariance)
    Q = rot_exp([0.2, 0.1, -0.3])
    uq = s.X @ Q.T - s.X
    r = o.eval(z, uq / H, far, np.eye(3), uq, far, np.eye(3), tgt)  # x^ = x: no inertia
    assert abs(r["parts"][1]) < 1e-12 * 1e5 * 1e-7 * H * H
    # patch test: an affine displacement of all nodes gives zero force on interior free vertices
    G = 1e-3 * np.array([[1.0, 0.3, -0.2], [0.1, -0.5, 0.2], [0.4, 0.2, 0.7]])
    ua = s.X @ G.T
    r = o.eval(z, ua / H, far, np.eye(3), ua, far, np.eye(3), tgt)
    ext = np.array(s.extent)
    interior = np.all(np.abs(s.X[:, :2]) < ext[:2] / 2 - 1e-9, axis=1) & (s.X[:, 2] < -1e-9) & (s.X[:, 2] > -ext[2] + 1e-9)
    assert interior.sum() > 3
    gscale = np.abs(r["g"]).max()
    assert gscale > 0 and np.abs(r["g"][interior]).max() < 1e-9 * gscale
    # 3x3 diagonal blocks = FD Hessian diagonal blocks (elastic + inertia, no contact)
    rng = np.random.default_rng(0)
    u = 1e-4 * rng.standard_normal(s.X.shape)
    u[s.fixed] = 0
    r = o.eval(z, z, far, np.eye(3), u, far, np.eye(3), tgt)
    free = np.setdiff1d(np.arange(len(u)), s.fixed)
    eps = 1e-9
    for v in free[::7]:
        Hb = np.zeros((3, 3))
        for a in range(3):
            up = u.copy(); up[v, a] += eps
            um = u.copy(); um[v, a] -= eps
            Hb[:, a] = (o.eval(z, z, far, np.eye(3), up, far, np.eye(3), tgt)["g"][v] -
                        o.eval(z, z, far, np.eye(3), um, far, np.eye(3), tgt)["g"][v]) / (2 * eps)
        assert np.abs(Hb - r["D"][v]).max() <= 1e-6 * np.abs(r["D"][v]).max()


def _body(X, u, c, R):
    """Gel vertices in the indenter body frame, b_a = (R_0a d_0 + R_1a d_1) + R_2a d_2 (no FMA)."""
    d = (X + u) - c
    return np.stack([(R[0, a] * d[:, 0] + R[1, a] * d[:, 1]) + R[2, a] * d[:, 2] for a in range(3)], axis=1)


def _box_pairs(o, gx, iy, r):
    """Independent numpy evaluation of the inflated-box predicate."""
    sv, se, st, ie = o.surface()
    it = o.scene.tris

    def boxes(P, idx):
        pts = P[idx]
        return pts.min(axis=1), pts.max(axis=1)

    out = []
    for kind, (A, B) in enumerate([(boxes(gx, sv[:, None]), boxes(iy, it)), (boxes(iy, np.arange(len(iy))[:, None]),
                                                                            boxes(gx, st)),
                                   (boxes(gx, se), boxes(iy, ie))]):
        lo_a, hi_a = A
        lo_b, hi_b = B
        ok = np.all((lo_a[:, None, :] <= hi_b[None, :, :] + r) & (lo_b[None, :, :] <= hi_a[:, None, :] + r), axis=2)
        a, b = np.nonzero(ok)
        out += [(kind, x, y) for x, y in zip(a, b)]
    return sorted(out)


def test_broadphase_matches_box_predicate_and_is_complete(pressed):
    s, o, st, (u, c, R), tgt = pressed
    r = 3e-4
    gx = _body(s.X, u, c, R)
    iy = s.Y
    got = sorted(map(tuple, o.broadphase_body(gx, r).tolist()))
    assert got == _box_pairs(o, gx, iy, r)
    assert sorted(map(tuple, o.broadphase_state(u, c, R, r).tolist())) == got
    # completeness: every primitive pair closer than r is a candidate (brute-force distances)
    allp = o.broadphase_body(gx, 1.0)
    sv, se, stri, ie = o.surface()
    cand = set(got)
    for kind, a, b in allp.tolist():
        if kind == 0:
            d, _ = O.dist_pt(gx[sv[a]], *iy[s.tris[b]])
        elif kind == 1:
            d, _ = O.dist_pt(iy[a], *gx[stri[b]])
        else:
            d, _ = O.dist_ee(gx[se[a][0]], gx[se[a][1]], iy[ie[b][0]], iy[ie[b][1]])
        if d < r:
            assert (kind, a, b) in cand


def test_ccd_bound_is_safe(pressed):
    """alpha_ccd (R15) vs brute force over ALL primitive pairs along the path."""
    s, o, st, (u, c, R), tgt = pressed
    rng = np.random.default_rng(11)
    d0 = o.dmin(u, c, R)
    for trial in range(4):
        p = 1e-4 * rng.standard_normal(u.shape)
        p[:, 2] += 3e-4 * (trial % 2)  # push the gel up into the sphere on half the trials
        p[s.fixed] = 0
        pr = np.concatenate([[0, 0, -3e-4], 0.02 * rng.standard_normal(3)])
        M = max(np.linalg.norm(p, axis=1).max(), np.linalg.norm(pr[:3]) + np.linalg.norm(s.Y, axis=1).max() * np.linalg.norm(pr[3:]))
        a = min(o.alpha_ccd(u, c, R, p, pr), 1e-4 / (2 * M))
        assert np.isfinite(a) and a > 0
        for t in np.linspace(0, a, 41)[1:]:
            d = o.dmin(u + t * p, c + t * pr[:3], rot_exp(t * pr[3:]) @ R)
            assert d >= 0.1 * d0 * (1 - 1e-9)


def test_marker_map_properties():
    s = w.scene_c1()
    o = O.Oracle(s)
    tet, idx, wgt = o.marker_map()
    assert np.all(wgt >= 0) and np.allclose(wgt.sum(1), 1, atol=1e-14)
    # independent point location: barycentric coordinates by numpy solve, lowest tet index wins
    for m, p in enumerate(s.markers):
        for e, t in enumerate(s.tets):
            Dm = np.stack([s.X[t[k]] - s.X[t[0]] for k in (1, 2, 3)], axis=1)
            l = np.linalg.solve(Dm, p - s.X[t[0]])
            b = np.concatenate([[1 - l.sum()], l])
            if np.all(b >= -1e-12):
                assert tet[m] == e
                assert np.allclose(wgt[m], np.clip(b, 0, None) / np.clip(b, 0, None).sum(), atol=1e-14)
                break
    # affine displacement reproduced exactly; rest -> 0
    G = np.array([[1e-4, 2e-5, 0], [-3e-5, 5e-5, 1e-5], [0, 1e-5, 2e-5]])
    t = np.array([1e-5, -2e-5, 3e-6])
    ua = s.X @ G.T + t
    o.set_state(0, ua, 0 * ua, s.init_poses[0][:3], np.eye(3))
    mk = o.markers(0, 3)
    assert np.allclose(mk, s.markers @ G.T + t, rtol=0, atol=1e-18)
    o.set_state(0, 0 * ua, 0 * ua, s.init_poses[0][:3], np.eye(3))
    assert np.all(o.markers(0) == 0)


def test_knn_marker_mode():
    s = w.scene_c1()
    o = O.Oracle(s, marker_mode=1, knn_k=4)
    tet, idx, wgt = o.marker_map()
    assert np.allclose(wgt.sum(1), 1) and np.all(wgt > 0)
    sv = o.surface()[0]
    for m in range(len(s.markers)):
        d = np.linalg.norm(s.X[sv] - s.markers[m], axis=1)
        order = sv[np.lexsort((sv, d))][:4]
        assert list(idx[m]) == list(order)
        dd = np.linalg.norm(s.X[order] - s.markers[m], axis=1)
        assert np.allclose(wgt[m], (1 / dd) / (1 / dd).sum())


def test_contact_free_small_velocity_limit():
    """No contact, tiny initial velocity: the step solves (M + h^2 K) dx = h M v (linear
    elasticity with Lame mu, lambda; App. B linearisation) up to O(|v|^2)."""
    s = _no_contact_scene()
    s.params.tol_x = 1e-17  # |dx| ~ 5e-11 m: residual tolerance 2e-7 relative
    s.params.stagnation = 0
    o = O.Oracle(s)
    mass, vol = o.mass_vol()
    E, nu = s.material.E, s.material.nu
    mu = E / (2 * (1 + nu))
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    nv = len(s.X)
    K = np.zeros((3 * nv, 3 * nv))
    for e, t in enumerate(s.tets):  # linear FEM stiffness written out independently
        Dm = np.stack([s.X[t[k]] - s.X[t[0]] for k in (1, 2, 3)], axis=1)
        Bi = np.linalg.inv(Dm)
        grads = np.vstack([-Bi.sum(0), Bi])  # shape-function gradients
        for a in range(4):
            for b in range(4):
                ga, gb = grads[a], grads[b]
                Kab = vol[e] * (mu * (ga @ gb) * np.eye(3) + mu * np.outer(gb, ga) + lam * np.outer(ga, gb))
                K[3 * t[a]:3 * t[a] + 3, 3 * t[b]:3 * t[b] + 3] += Kab
    rng = np.random.default_rng(4)
    v0 = 1e-6 * np.stack([np.sin(300 * s.X[:, 0]), np.cos(200 * s.X[:, 1]), np.sin(500 * s.X[:, 0] + 100 * s.X[:, 1])], 1)
    v0[s.fixed] = 0
    o.set_state(0, np.zeros_like(v0), v0, s.init_poses[0][:3], np.eye(3))
    o.step(s.init_poses)
    u, _, _, _ = o.get_state(0)
    free = np.setdiff1d(np.arange(nv), s.fixed)
    dofs = (3 * free[:, None] + np.arange(3)).ravel()
    Mv = np.repeat(mass, 3)
    A = np.diag(Mv) + H * H * K
    dx = np.linalg.solve(A[np.ix_(dofs, dofs)], (H * Mv * v0.ravel())[dofs])
    assert np.abs(u.ravel()[dofs] - dx).max() <= 1e-4 * np.abs(dx).max()


def _run_steps(scene, nsteps=None, trace=False, debug=False, tol=1e-11):
    scene.params.tol_x = tol
    scene.params.stagnation = 3000
    o = O.Oracle(scene, debug=debug)
    tr = []
    for k in range(len(scene.poses) if nsteps is None else nsteps):
        if trace:
            o.set_trace(0)
        o.step(scene.poses[k])
        if trace:
            tr.append(o.trace(0))
    return o, tr


def test_invariants_monotone_feasible_fixed_and_cap():
    """Per accepted iterate: E non-increasing, brute-force d_min > 0, |alpha p|_disp <= dhat/2;
    fixed vertices exactly 0 (north_star oracle checks)."""
    s = c1_press_scene(mu_f=1.0, steps=3, depth=0.15e-3)
    o, trs = _run_steps(s, trace=True, debug=True)
    for tr in trs:
        acc = tr[tr[:, 2] == 1]
        assert np.all(np.diff(acc[:, 1]) <= 0)
        assert np.all(acc[:, 12] > 0)
        assert np.all(acc[:, 3] * acc[:, 7] <= 0.5e-4 * (1 + 1e-12))
    st = o.status_of(0)
    assert st["flags"] & 1 and st["dmin"] > 0
    u, _, _, _ = o.get_state(0)
    assert np.all(u[s.fixed] == 0)


def test_translation_invariance():
    s1 = c1_press_scene(mu_f=1.0, steps=2, depth=0.1e-3)
    s2 = c1_press_scene(mu_f=1.0, steps=2, depth=0.1e-3)
    sh = np.array([2.0 ** -10, -2.0 ** -11, 2.0 ** -12])
    s2.X = s2.X + sh
    s2.markers = s2.markers + sh
    s2.init_poses[:, :, ] = s2.init_poses
    s2.init_poses[:, :3] += sh
    s2.poses[:, :, :3] += sh
    o1, _ = _run_steps(s1, tol=1e-12)
    o2, _ = _run_steps(s2, tol=1e-12)
    u1, _, c1, _ = o1.get_state(0)
    u2, _, c2, _ = o2.get_state(0)
    assert np.abs(u1 - u2).max() <= 1e-6 * np.abs(u1).max()
    assert np.abs(o1.markers(0) - o2.markers(0)).max() <= 1e-6 * np.abs(o1.markers(0)).max()


def test_recovery_after_retraction():
    """P:269 / S:301: after retraction and 50 settling steps the gel returns to rest (< 1 %)."""
    s = c1_press_scene(mu_f=1.0, steps=3, depth=0.2e-3)
    q = [1.0, 0, 0, 0]
    up = [w.pose((0, 0, 3e-3 + z), q)[None] for z in (0.0, 1e-4, 3e-4, 6e-4)]
    s.poses = np.concatenate([s.poses, np.stack(up), np.stack([up[-1]] * 50)])
    o, _ = _run_steps(s, nsteps=3, tol=1e-10)
    peak = np.abs(o.get_state(0)[0]).max()
    peak_mk = np.abs(o.markers(0)).max()
    for k in range(3, len(s.poses)):
        o.step(s.poses[k])
    u, _, _, _ = o.get_state(0)
    assert np.abs(u).max() < 0.01 * peak
    assert np.abs(o.markers(0)).max() < 0.01 * peak_mk


def test_reflection_equivariance():
    """Mirror symmetry, as equivariance: reflecting the whole problem about x = 0
    (gel, indenter, poses, markers) reflects the solution.  An off-centre press keeps the
    minimiser unique (a centred frictionless press of the faceted sphere's tip vertex onto a
    gel vertex is a saddle the solver legitimately leaves)."""
    S = np.diag([-1.0, 1.0, 1.0])
    s1 = c1_press_scene(mu_f=1.0, steps=2, depth=0.1e-3)
    off = np.array([0.7e-3, 0.4e-3, 0.0])
    s1.init_poses[:, :3] += off
    s1.poses[:, :, :3] += off
    s2 = c1_press_scene(mu_f=1.0, steps=2, depth=0.1e-3)
    s2.X = s1.X @ S
    s2.tets = s1.tets[:, [0, 2, 1, 3]].copy()
    s2.Y = s1.Y @ S
    s2.tris = s1.tris[:, [0, 2, 1]].copy()
    s2.markers = s1.markers @ S
    s2.frame = s1.frame @ S
    s2.init_poses = s1.init_poses.copy()
    s2.init_poses[:, 0] *= -1
    s2.poses = s1.poses.copy()
    s2.poses[:, :, 0] *= -1
    o1, _ = _run_steps(s1, tol=1e-12)
    o2, _ = _run_steps(s2, tol=1e-12)
    u1 = o1.get_state(0)[0]
    u2 = o2.get_state(0)[0]
    assert np.abs(u1).max() > 1e-5
    assert np.abs(u2 - u1 @ S).max() <= 1e-6 * np.abs(u1).max()
    # markers: frame t1 reflected too, so the (t1, t2) components are equal
    assert np.abs(o2.markers(0) - o1.markers(0)).max() <= 1e-6 * np.abs(o1.markers(0)).max()


def test_newton_pins_whole_step_minimiser():
    """Dense fp64 Newton (FD Hessian of the oracle's pinned gradient, PSD projection,
    backtracking with a feasibility filter and the dhat/2 displacement cap) reaches
    the same minimiser as the PNCG oracle (SURVEY §8c.4 whole-step pin)."""
    s = c1_press_scene(mu_f=0.0, steps=2, depth=0.1e-3)
    s.params.tol_x = 1e-12
    s.params.stagnation = 3000
    o = O.Oracle(s)
    o.step(s.poses[0])
    st = o.get_state(0)
    u_t, v_t, c_t, R_t = st
    tgt = s.poses[1][0]
    o.step(s.poses[1])
    u_ref, _, c_ref, R_ref = o.get_state(0)
    free = np.setdiff1d(np.arange(len(u_t)), s.fixed)
    n = 3 * len(free) + 6

    def unpack(x0, dx):
        u, c, R = x0
        u2 = u.copy(); u2[free] += dx[:-6].reshape(-1, 3)
        return u2, c + dx[-6:-3], rot_exp(dx[-3:]) @ R

    def grad(x):
        r = o.eval(u_t, v_t, c_t, R_t, *x, tgt)
        return r["E"], np.concatenate([r["g"][free].ravel(), r["grig"]])

    x = (u_t.copy(), c_t.copy(), R_t.copy())
    for it in range(60):
        E0, g = grad(x)
        if np.linalg.norm(g) < 1e-13:
            break
        Hm = np.zeros((n, n))
        for j in range(n):
            e = np.zeros(n); e[j] = 1e-10
            Hm[:, j] = (grad(unpack(x, e))[1] - grad(unpack(x, -e))[1]) / 2e-10
        Hm = (Hm + Hm.T) / 2
        lam_, V = np.linalg.eigh(Hm)
        dx = -V @ ((V.T @ g) / np.maximum(lam_, 1e-8 * lam_.max()))
        m = max(np.linalg.norm(dx[:-6].reshape(-1, 3), axis=1).max(), np.linalg.norm(dx[-6:-3]) +
                np.linalg.norm(s.Y, axis=1).max() * np.linalg.norm(dx[-3:]))
        a = min(1.0, 0.5e-4 / m)
        while True:
            xn = unpack(x, a * dx)
            En = grad(xn)[0]
            if np.isfinite(En) and En <= E0 + 1e-4 * a * (g @ dx) and o.dmin(*xn) > 0:
                break
            a *= 0.5
            assert a > 1e-12
        x = xn
    u_n, c_n, R_n = x
    assert np.abs(u_n - u_ref).max() <= 1e-9 * 16e-3
    assert np.linalg.norm(c_n - c_ref) <= 1e-9 * 16e-3


def test_unstructured_mesh_invariants():
    """§8f-1: the oracle on a jittered, renumbered pad keeps its invariants (monotone E,
    brute-force d_min > 0, fixed vertices 0) and converges."""
    s = c1_press_scene(mu_f=1.0, steps=2, depth=0.1e-3)
    s.X, s.tets, s.fixed = w.make_pad_unstructured(s.extent, s.cells)
    o, trs = _run_steps(s, trace=True, debug=True, tol=1e-10)
    for tr in trs:
        acc = tr[tr[:, 2] == 1]
        assert np.all(np.diff(acc[:, 1]) <= 0) and np.all(acc[:, 12] > 0)
    assert o.status_of(0)["flags"] & 1
    u = o.get_state(0)[0]
    assert np.all(u[s.fixed] == 0) and np.abs(u).max() > 1e-6


# ---------------------------------------------------------------- augmented Lagrangian (R29)
def test_pose_multiplier_gradient_matches_central_fd(pressed):
    """The multiplier term h^2 (lam_t . dc + lam_r . phi) of R29: its left-trivialised
    rotation gradient J_l(phi)^-T lam_r (and h^2 lam_t) against central differences, with a
    target rotated 0.2 rad away so that the J_l correction is ~10 % of the term."""
    s, o, st, (u, c, R), tgt = pressed
    tgt = tgt.copy()
    ax = np.array([0.3, -0.5, 0.8]) / np.linalg.norm([0.3, -0.5, 0.8])
    Rt = rot_exp(0.2 * ax) @ O.quat_to_R(tgt).reshape(3, 3)
    tgt[3:] = rig_quat(Rt)
    lam = np.array([0.3, -0.2, 0.5, 0.01, -0.02, 0.015])
    g0 = o.eval(*st, u, c, R, tgt)["grig"]
    o.set_eval_lambda(lam)
    try:
        r = o.eval(*st, u, c, R, tgt)
        fr = np.zeros(6)
        eps = 1e-9
        for a in range(3):
            e = np.zeros(3); e[a] = eps
            fr[a] = (o.eval(*st, u, c + e, R, tgt)["E"] - o.eval(*st, u, c - e, R, tgt)["E"]) / (2 * eps)
            e = np.zeros(3); e[a] = 1e-8
            fr[3 + a] = (o.eval(*st, u, c, rot_exp(e) @ R, tgt)["E"]
                         - o.eval(*st, u, c, rot_exp(-e) @ R, tgt)["E"]) / 2e-8
        assert np.linalg.norm(fr - r["grig"]) <= 1e-6 * np.linalg.norm(r["grig"])
        h2 = s.dt ** 2
        assert np.allclose(r["grig"][:3] - g0[:3], h2 * lam[:3], rtol=1e-9, atol=0)
        # the rotation part is not h^2 lam_r: the J_l(phi)^-T correction is there
        assert np.linalg.norm(r["grig"][3:] - g0[3:] - h2 * lam[3:]) > 0.02 * h2 * np.linalg.norm(lam[3:])
    finally:
        o.set_eval_lambda(np.zeros(6))


def rig_quat(R):
    from paper_2603_28475_b200.rig import R_to_quat
    return R_to_quat(R)


def test_augmented_lagrangian_removes_the_pose_residual():
    """R29: holding a press, the penalty spring leaves the indenter short of its target by
    F / k_t; the AL multiplier absorbs the contact force after a step, so the residual drops
    to the solver tolerance and lam_t equals the spring force the penalty run carries."""
    res = {}
    lam = None
    for al in (0, 1):
        s = c1_press_scene(mu_f=1.0, steps=3, depth=0.3e-3)
        s.poses = np.concatenate([s.poses, np.repeat(s.poses[-1:], 4, axis=0)])  # hold the press
        s.params.tol_x = 1e-11
        s.params.pose_al = al
        o = O.Oracle(s)
        for k in range(len(s.poses)):
            o.step(s.poses[k])
            assert o.status_of(0)["flags"] & 1
        c = o.get_state(0)[2]
        res[al] = np.linalg.norm(c - s.poses[-1][0][:3])
        if al:
            lam = o.lambda_of(0)
    k_t = s.params.k_t
    assert res[0] > 1e-9                       # penalty residual F / k_t at ~0.1-1 N
    assert res[1] < 0.05 * res[0]              # AL: gone to the solver's tolerance
    assert np.linalg.norm(lam[:3]) == pytest.approx(k_t * res[0], rel=0.05)


# ---------------------------------------------------------------- EE mollifier (R30)
def test_ee_mollifier_gradient_matches_central_fd():
    """R30: with the edge-edge mollifier on, the energy m(c) kappa b(d) of nearly parallel edge
    pairs (a peg's axial edge over the pad's x edges) has the gradient m kappa b' w n +
    kappa b m'(c) dc/dz: central differences agree, and the m' term is really present."""
    from helpers import parallel_peg_scene
    s = parallel_peg_scene(steps=2, depth=0.05e-3)
    s.params.tol_x = 1e-10
    s.params.ee_mollifier = 1
    o = O.Oracle(s)
    o.step(s.poses[0])
    st = o.get_state(0)
    o.step(s.poses[1])
    u, _, c, R = o.get_state(0)
    rng = np.random.default_rng(11)
    u = u + 2e-7 * rng.standard_normal(u.shape)
    u[s.fixed] = 0
    tgt = s.poses[1][0]
    r = o.eval(*st, u, c, R, tgt)
    s0 = parallel_peg_scene(steps=2, depth=0.05e-3)
    o0 = O.Oracle(s0)
    r0 = o0.eval(*st, u, c, R, tgt)
    assert r["parts"][2] > 0 and r["parts"][2] < r0["parts"][2]  # mollified EE barrier energy
    free = np.setdiff1d(np.arange(len(u)), s.fixed)
    eps = 1e-9
    fd = np.zeros_like(u)
    for v in free:
        for a in range(3):
            up = u.copy(); up[v, a] += eps
            um = u.copy(); um[v, a] -= eps
            fd[v, a] = (o.eval(*st, up, c, R, tgt)["E"] - o.eval(*st, um, c, R, tgt)["E"]) / (2 * eps)
    g = r["g"][free]
    assert np.linalg.norm(fd[free] - g) <= 1e-6 * np.linalg.norm(g)
    fr = np.zeros(6)
    for a in range(3):
        e = np.zeros(3); e[a] = eps
        fr[a] = (o.eval(*st, u, c + e, R, tgt)["E"] - o.eval(*st, u, c - e, R, tgt)["E"]) / (2 * eps)
        e = np.zeros(3); e[a] = 1e-8
        fr[3 + a] = (o.eval(*st, u, c, rot_exp(e) @ R, tgt)["E"] - o.eval(*st, u, c, rot_exp(-e) @ R, tgt)["E"]) / 2e-8
    assert np.linalg.norm(fr - r["grig"]) <= 1e-6 * np.linalg.norm(r["grig"])
    # gradient differs from the unmollified one beyond the FD tolerance
    assert np.linalg.norm(r["g"][free] - r0["g"][free]) > 1e-4 * np.linalg.norm(g)


def test_ee_mollifier_converges_and_stays_feasible():
    """The mollified problem still converges with brute-force d_min > 0 (debug checks)."""
    from helpers import parallel_peg_scene
    s = parallel_peg_scene(steps=3, depth=0.1e-3)
    s.params.tol_x = 1e-10
    s.params.ee_mollifier = 1
    o = O.Oracle(s, debug=True)
    for k in range(3):
        o.step(s.poses[k])
        st = o.status_of(0)
        assert st["flags"] & 1 and st["dmin"] > 0, st
