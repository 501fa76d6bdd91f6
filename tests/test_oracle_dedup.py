"""Pins of the oracle's IPC-toolkit constraint deduplication (R33):
each contact constraint -- identified by its closest features, the corners with a non-zero
closest-point weight on each side -- carries its barrier (and friction anchor) once, where the
literal sum of P:432 counts it once per primitive pair that realises it.

Expected values come from a closed form (a single point-point constraint under an inverted
pyramid's tip: kappa b(h) once, or m times literally, m counted by brute force with the pinned
distance routines), from a brute-force enumeration of the unique features, and from central
finite differences of the energy -- never from the routine under test."""
import numpy as np
import pytest

import oracle as O
import workloads as w
from helpers import c1_press_scene, rot_exp

H = 5e-3
MM = 1e-3


def _pyramid_scene(h):
    """C1 pad and an inverted square pyramid whose tip is h above the pad's top-centre vertex."""
    s = w.scene_c1()
    wd, hh = 2 * MM, 1 * MM
    s.Y = np.array([[0, 0, 0], [-wd, -wd, hh], [wd, -wd, hh], [wd, wd, hh], [-wd, wd, hh]], float)
    s.tris = np.array([[0, 2, 1], [0, 3, 2], [0, 4, 3], [0, 1, 4], [1, 2, 3], [1, 3, 4]], np.int32)
    s.init_poses = np.array([[0, 0, h, 1, 0, 0, 0]], float)
    s.poses = s.init_poses[None].copy()
    return s


def _corners(s, surf, kind, a, b, u, c, R):
    sv, se, st_, ie = surf
    x = s.X + u
    y = (R @ s.Y.T).T + c
    if kind == 0:
        return [x[sv[a]], y[s.tris[b, 0]], y[s.tris[b, 1]], y[s.tris[b, 2]]], [sv[a]], list(s.tris[b])
    if kind == 1:
        return [y[a], x[st_[b, 0]], x[st_[b, 1]], x[st_[b, 2]]], list(st_[b]), [a]
    return [x[se[a, 0]], x[se[a, 1]], y[ie[b, 0]], y[ie[b, 1]]], list(se[a]), list(ie[b])


def _pairs_with_features(o, s, u, c, R, dhat):
    """(d, gel feature, indenter feature) of every candidate pair with d < dhat, from the pinned
    distance routines (weights: point-triangle (1, -b0, -b1, -b2), edge-edge (1-s, s, -(1-t), -t))."""
    surf = o.surface()
    out = []
    for kind, a, b in o.broadphase_state(u, c, R, dhat + o.params.bp_margin):
        z, gid, yid = _corners(s, surf, kind, a, b, u, c, R)
        dd, wt = (O.dist_ee(*z) if kind == 2 else O.dist_pt(*z))
        if dd >= dhat:
            continue
        ids = ([gid[0]] + yid) if kind == 0 else (([yid[0]] + gid) if kind == 1 else gid + yid)
        gel = ids[:1] if kind == 0 else (ids[1:] if kind == 1 else ids[:2])
        ind = ids[1:] if kind == 0 else (ids[:1] if kind == 1 else ids[2:])
        wg = wt[:1] if kind == 0 else (wt[1:] if kind == 1 else wt[:2])
        wy = wt[1:] if kind == 0 else (wt[:1] if kind == 1 else wt[2:])
        fg = tuple(sorted(int(i) for i, x in zip(gel, wg) if x != 0))
        fy = tuple(sorted(int(i) for i, x in zip(ind, wy) if x != 0))
        out.append((dd, fg, fy))
    return out


def _unique_sum(pairs, kappa, dhat):
    seen, tot = set(), 0.0
    for dd, fg, fy in pairs:
        shared = not (len(fg) == 3 or len(fy) == 3 or (len(fg) == 2 and len(fy) == 2))
        if shared:
            if (fg, fy) in seen:
                continue
            seen.add((fg, fy))
        tot += kappa * O.barrier(dd, dhat)
    return tot


def test_point_point_constraint_counted_once():
    h = 0.5e-4
    s = _pyramid_scene(h)
    kappa = None
    res = {}
    for dedup in (0, 1):
        s.params.dedup = dedup
        o = O.Oracle(s)
        assert o.status == 0
        kappa = H * H * o.kappa_phys
        u = np.zeros_like(s.X)
        c = s.init_poses[0, :3].copy()
        R = np.eye(3)
        r = o.eval(u, u, c, R, u, c, R, s.init_poses[0])
        res[dedup] = r["parts"][2]
    pairs = _pairs_with_features(o, s, np.zeros_like(s.X), s.init_poses[0, :3], np.eye(3), o.params.dhat)
    m = len(pairs)
    assert m >= 8 and all(abs(dd - h) < 1e-15 for dd, _, _ in pairs)
    assert len({(fg, fy) for _, fg, fy in pairs}) == 1  # one constraint: (gel vertex, pyramid tip)
    bh = kappa * O.barrier(h, o.params.dhat)
    assert abs(res[1] - bh) <= 1e-12 * bh
    assert abs(res[0] - m * bh) <= 1e-12 * m * bh


@pytest.fixture(scope="module")
def pressed_dedup():
    s = c1_press_scene(mu_f=1.0, steps=4, depth=0.25e-3)
    s.params.tol_x = 1e-10
    s.params.dedup = 1
    o = O.Oracle(s)
    for k in range(3):
        o.step(s.poses[k])
    u_t, v_t, c_t, R_t = o.get_state(0)
    o.step(s.poses[3])
    u, _, c, R = o.get_state(0)
    rng = np.random.default_rng(8)
    u = u + 2e-7 * rng.standard_normal(u.shape)
    u[s.fixed] = 0
    c = c + 1e-7 * rng.standard_normal(3)
    R = rot_exp(1e-5 * rng.standard_normal(3)) @ R
    return s, o, (u_t, v_t, c_t, R_t), (u, c, R), s.poses[3][0].copy()


def test_dedup_barrier_matches_unique_feature_enumeration(pressed_dedup):
    """At a pressed contact state the deduplicated barrier equals the brute-force sum over unique
    closest-feature constraints, the literal barrier the sum over all pairs, and they differ."""
    s, o, st, (u, c, R), tgt = pressed_dedup
    kappa = H * H * o.kappa_phys
    pairs = _pairs_with_features(o, s, u, c, R, o.params.dhat)
    ref_u = _unique_sum(pairs, kappa, o.params.dhat)
    ref_l = sum(kappa * O.barrier(dd, o.params.dhat) for dd, _, _ in pairs)
    e1 = o.eval(*st, u, c, R, tgt)["parts"][2]
    s0 = c1_press_scene(mu_f=1.0, steps=4, depth=0.25e-3)
    o0 = O.Oracle(s0)
    e0 = o0.eval(*st, u, c, R, tgt)["parts"][2]
    assert abs(e1 - ref_u) <= 1e-10 * ref_u and abs(e0 - ref_l) <= 1e-10 * ref_l
    assert ref_l > ref_u * (1 + 1e-3)  # duplicates exist at this state


def test_dedup_gradient_matches_central_fd(pressed_dedup):
    """The deduplicated potential's gradient (gel and rigid DOFs) matches central differences to
    1e-6 (away from region boundaries, where the constraint set -- and R33's energy -- changes)."""
    s, o, st, (u, c, R), tgt = pressed_dedup
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
    gr = np.zeros(6)
    for a in range(3):
        dc = np.zeros(3); dc[a] = 1e-10
        gr[a] = (o.eval(*st, u, c + dc, R, tgt)["E"] - o.eval(*st, u, c - dc, R, tgt)["E"]) / 2e-10
        dt = np.zeros(3); dt[a] = 1e-9
        gr[3 + a] = (o.eval(*st, u, c, rot_exp(dt) @ R, tgt)["E"] - o.eval(*st, u, c, rot_exp(-dt) @ R, tgt)["E"]) / 2e-9
    assert np.linalg.norm(gr - r["grig"]) <= 1e-6 * np.linalg.norm(r["grig"])


def test_dedup_step_converges_feasible():
    """Deduplicated solves: the small peg's steps converge (tolerance mode) and stay
    intersection-free.  On the faceted C1 sphere a gel vertex's minimiser can sit on a region
    boundary of the constraint set, where R33's potential jumps (the IPC-toolkit formulation is
    not continuous there), and the solve stops on stagnation instead -- still feasible."""
    s = w.scene_small_peg(n_envs=3, n_steps=3)
    s.params.dedup = 1
    s.params.tol_x = 1e-10
    o = O.Oracle(s, debug=True)
    for k in range(3):
        o.step(s.poses[k], threads=3)
        for e in range(3):
            st = o.status_of(e)
            assert st["flags"] & 1 and st["dmin"] > 0, (k, e, st)
    s = c1_press_scene(mu_f=1.0, steps=2, depth=0.1e-3)
    s.params.dedup = 1
    s.params.tol_x = 1e-10
    o = O.Oracle(s, debug=True)
    o.step(s.poses[0])
    st = o.status_of(0)
    assert st["flags"] & (1 | 64) and st["dmin"] > 0, st
