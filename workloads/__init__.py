"""Seeded synthetic input generators shared by the oracle tests, the CUDA parity
tests, ``bench.py`` and ``__graft_entry__.smoke()``.

This module holds NO arithmetic of the method (no energies, distances, surface
extraction, broad phase, marker location or solver logic).  It only produces
raw inputs with the shapes of the paper's workloads:

* a Freudenthal 6-tet gel pad (the paper's "pseudo-structured" mesh, PAPER.md
  P:272 "pseudo-structured mesh"), bottom face fixed (the bonded sensor base,
  P:594-595 / SPEC S:39),
* rigid indenters as closed triangle shells in their body frame: icosphere,
  cylinder peg of diameter 8 mm, sharp-edged square peg,
* the 7 x 9 marker lattice on the contact face,
* indenter pose trajectories (press / slide / twist / release with the
  "IPC Rand. Move. Noise" of Table `random`),

following the recipe in DESIGN.md §"Input recipe".  Every
coordinate is rounded to an fp32-representable double so both the fp64 oracle
and the fp32 device path see bit-identical inputs.

Gel frame: x in [-Lx/2, Lx/2], y in [-Ly/2, Ly/2], z in [-Lz, 0]; the contact
face is z = 0 with outward normal +z; the base z = -Lz is fixed.
Poses: (t_x, t_y, t_z, q_w, q_x, q_y, q_z), body frame -> gel frame, metres.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

MM = 1e-3


def f32(a):
    """Round to the nearest fp32 value, returned as float64."""
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


# ----------------------------------------------------------------------------
# gel pad
# ----------------------------------------------------------------------------
def make_pad(extent, cells, mirror=False):
    """Box [-Lx/2,Lx/2]x[-Ly/2,Ly/2]x[-Lz,0] split into nx*ny*nz cells, each cell
    into 6 tets around one cube diagonal (Kuhn/Freudenthal split).

    mirror=True flips the cell diagonal in the lower halves of x and y, giving a
    mesh that is mirror-symmetric about x=0 and y=0 (conforming for even nx, ny).
    Returns (X [V,3] f64 fp32-representable, tets [T,4] int32 positively
    oriented, fixed [F] int32 = base-face vertices).
    """
    Lx, Ly, Lz = extent
    nx, ny, nz = cells
    if min(cells) < 1 or min(extent) <= 0:
        raise ValueError("extent and cells must be positive")
    xs = f32(-Lx / 2 + Lx * np.arange(nx + 1) / nx)
    ys = f32(-Ly / 2 + Ly * np.arange(ny + 1) / ny)
    zs = f32(-Lz + Lz * np.arange(nz + 1) / nz)
    zs[-1] = 0.0
    X = np.zeros(((nx + 1) * (ny + 1) * (nz + 1), 3))
    vid = lambda i, j, k: i + (nx + 1) * (j + (ny + 1) * k)
    for k in range(nz + 1):
        for j in range(ny + 1):
            for i in range(nx + 1):
                X[vid(i, j, k)] = (xs[i], ys[j], zs[k])
    tets = []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                fx = 1 if (mirror and 2 * i < nx) else 0
                fy = 1 if (mirror and 2 * j < ny) else 0
                corner = lambda a, b, c: vid(i + (a ^ fx), j + (b ^ fy), k + c)
                for perm in itertools.permutations(range(3)):
                    loc = [0, 0, 0]
                    path = [tuple(loc)]
                    for ax in perm:
                        loc[ax] = 1
                        path.append(tuple(loc))
                    t = [corner(*p) for p in path]
                    d = np.linalg.det(np.stack([X[t[1]] - X[t[0]], X[t[2]] - X[t[0]], X[t[3]] - X[t[0]]]))
                    if d < 0:
                        t[1], t[2] = t[2], t[1]
                    tets.append(t)
    fixed = np.array([vid(i, j, 0) for j in range(ny + 1) for i in range(nx + 1)], dtype=np.int32)
    return X, np.asarray(tets, dtype=np.int32), fixed


# ----------------------------------------------------------------------------
# indenters (closed, outward-oriented triangle shells in the body frame)
# ----------------------------------------------------------------------------
def make_icosphere(radius, subdiv):
    t = (1.0 + 5 ** 0.5) / 2.0
    V = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
         (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    V = [np.array(v, float) / np.linalg.norm(v) for v in V]
    F = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6),
         (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10),
         (8, 6, 7), (9, 8, 1)]
    for _ in range(subdiv):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = V[a] + V[b]
                V.append(m / np.linalg.norm(m))
                cache[key] = len(V) - 1
            return cache[key]

        F2 = []
        for a, b, c in F:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            F2 += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        F = F2
    Y = f32(np.array(V) * radius)
    return Y, np.asarray(F, dtype=np.int32)


def make_cylinder(radius, length, n_around, n_along):
    """Cylinder with axis along body x, centred at the origin, capped ends."""
    Y = []
    for s in range(n_along + 1):
        x = -length / 2 + length * s / n_along
        for k in range(n_around):
            a = 2 * np.pi * k / n_around
            Y.append((x, radius * np.cos(a), radius * np.sin(a)))
    c0 = len(Y)
    Y.append((-length / 2, 0.0, 0.0))
    c1 = len(Y)
    Y.append((length / 2, 0.0, 0.0))
    F = []
    ring = lambda s, k: s * n_around + (k % n_around)
    for s in range(n_along):
        for k in range(n_around):
            a, b, c, d = ring(s, k), ring(s, k + 1), ring(s + 1, k + 1), ring(s + 1, k)
            F += [(a, b, c), (a, c, d)]
    for k in range(n_around):
        F.append((c0, ring(0, k + 1), ring(0, k)))
        F.append((c1, ring(n_along, k), ring(n_along, k + 1)))
    Y = f32(np.array(Y))
    F = np.asarray(F, dtype=np.int32)
    return _orient_outward(Y, F)


def make_square_peg(side, length, split):
    """Sharp-edged square peg (axis along body x), each face split into squares
    of edge ~`split`, two triangles per square."""
    n_s = max(1, int(round(side / split)))
    n_l = max(1, int(round(length / split)))
    verts = {}
    Y, F = [], []

    def vi(p):
        key = tuple(np.round(np.asarray(p) / (split * 1e-3)).astype(np.int64))
        if key not in verts:
            verts[key] = len(Y)
            Y.append(tuple(p))
        return verts[key]

    h, L = side / 2, length / 2

    def face(origin, du, dv, nu, nv):
        for a in range(nu):
            for b in range(nv):
                p = [np.asarray(origin) + du * (a + da) / nu + dv * (b + db) / nv for da, db in ((0, 0), (1, 0), (1, 1), (0, 1))]
                q = [vi(x) for x in p]
                F.append((q[0], q[1], q[2]))
                F.append((q[0], q[2], q[3]))

    ex, ey, ez = np.eye(3)
    face((-L, -h, -h), 2 * L * ex, 2 * h * ey, n_l, n_s)
    face((-L, -h, h), 2 * L * ex, 2 * h * ey, n_l, n_s)
    face((-L, -h, -h), 2 * L * ex, 2 * h * ez, n_l, n_s)
    face((-L, h, -h), 2 * L * ex, 2 * h * ez, n_l, n_s)
    face((-L, -h, -h), 2 * h * ey, 2 * h * ez, n_s, n_s)
    face((L, -h, -h), 2 * h * ey, 2 * h * ez, n_s, n_s)
    Y = f32(np.array(Y))
    return _orient_outward(Y, np.asarray(F, dtype=np.int32))


def _orient_outward(Y, F):
    """Orient every triangle so its normal points away from the shell centroid
    (valid for the convex shells generated here)."""
    F = F.copy()
    cen = Y.mean(axis=0)
    for i, (a, b, c) in enumerate(F):
        n = np.cross(Y[b] - Y[a], Y[c] - Y[a])
        if np.dot(n, (Y[a] + Y[b] + Y[c]) / 3 - cen) < 0:
            F[i] = (a, c, b)
    return Y, F


# ----------------------------------------------------------------------------
# markers: 7 rows x 9 cols on the contact face z = 0
# ----------------------------------------------------------------------------
def make_markers(extent, cells, rows=7, cols=9):
    """Centred lattice, pitch (Lx/10, Ly/8), shifted by (0.173 cx, 0.291 cy) so no
    marker sits on a cell line or a face diagonal.  Row-major,
    row i along y, column j along x."""
    Lx, Ly, Lz = extent
    cx, cy = Lx / cells[0], Ly / cells[1]
    xs = (np.arange(cols) - (cols - 1) / 2) * Lx / (cols + 1) + 0.173 * cx
    ys = (np.arange(rows) - (rows - 1) / 2) * Ly / (rows + 1) + 0.291 * cy
    M = np.array([(x, y, 0.0) for y in ys for x in xs])
    M = f32(M)
    # margin from cell lines and both cell diagonals, in cell units
    fx = (M[:, 0] + Lx / 2) / cx
    fy = (M[:, 1] + Ly / 2) / cy
    rx, ry = fx - np.floor(fx), fy - np.floor(fy)
    margin = np.minimum.reduce([rx, 1 - rx, ry, 1 - ry, np.abs(rx - ry) / 2 ** 0.5, np.abs(rx + ry - 1) / 2 ** 0.5])
    assert margin.min() >= 1e-3, margin.min()
    assert np.all(np.abs(M[:, 0]) < Lx / 2) and np.all(np.abs(M[:, 1]) < Ly / 2)
    frame = np.array([[1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0]])  # t1, t2, n
    return M, frame


# ----------------------------------------------------------------------------
# poses
# ----------------------------------------------------------------------------
def quat_axis_angle(axis, ang):
    axis = np.asarray(axis, float)
    axis = axis / np.linalg.norm(axis)
    return np.concatenate([[np.cos(ang / 2)], np.sin(ang / 2) * axis])


def quat_mul(a, b):
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def pose(t, q):
    q = np.asarray(q, float)
    q = q / np.linalg.norm(q)
    if q[0] < 0:
        q = -q
    return f32(np.concatenate([np.asarray(t, float), q]))


# ----------------------------------------------------------------------------
# BASELINE configs as concrete synthetic inputs
# ----------------------------------------------------------------------------
@dataclass
class Material:
    E: float = 1e5          # Pa (P:494-501 range 1e4..2e5)
    nu: float = 0.45        # (range 0.4..0.497)
    rho: float = 1100.0     # kg/m^3 (range 1e-3..5e-3 g/mm^3 -> 1e3..5e3 kg/m^3)
    mu_f: float = 1.0       # (range 0.25..2.5)


@dataclass
class Params:
    dhat: float = 1e-4      # m
    kappa_phys: float = 0.0  # N/m; 0 -> default rule of DESIGN.md reading R4
    eps_v: float = 2e-3     # m/s (eps = eps_v * h = 1e-5 m)
    tol_x: float = 1e-9     # m, on ||P g||_disp
    k_t: float = 1e8        # N/m pose spring (force-capped, R18)
    k_r: float = 1e6        # N m/rad
    f_max: float = 10.0     # N   force cap of the pose spring (peg at 1 mm press needs ~5 N)
    t_max: float = 0.05     # N m torque cap
    ccd_s: float = 0.1
    bp_margin: float = 2e-4  # m_r = 2 dhat
    c1: float = 1e-4
    eps_E: float = 1e-6
    max_iters: int = 5000
    fixed_iters: int = 0
    beta_rule: int = 0      # 0 DK, 1 PR+, 2 FR, 3 DK+
    precond: int = 0        # 0 3x3 block Jacobi, 1 scalar Jacobi
    max_halvings: int = 10
    stagnation: int = 3000
    max_candidates: int = 0   # 0 -> library default (32768 per env)
    max_anchors: int = 0      # 0 -> library default (4096 per env)
    pose_al: int = 0          # 1: augmented-Lagrangian pose enforcement (R29)
    ee_mollifier: int = 0     # 1: IPC edge-edge parallel mollifier (R30)
    dedup: int = 0            # 1: IPC-toolkit constraint deduplication (R33)


@dataclass
class Scene:
    name: str
    X: np.ndarray
    tets: np.ndarray
    fixed: np.ndarray
    Y: np.ndarray
    tris: np.ndarray
    markers: np.ndarray
    frame: np.ndarray
    init_poses: np.ndarray          # [E,7]
    poses: np.ndarray               # [S,E,7] target pose for step s
    dt: float = 5e-3
    material: Material = field(default_factory=Material)
    params: Params = field(default_factory=Params)
    extent: tuple = (0, 0, 0)
    cells: tuple = (0, 0, 0)

    @property
    def n_envs(self):
        return self.init_poses.shape[0]


def scene_c1(mu_f=1.0, n_envs=1, mirror=False, depth=0.5 * MM, steps=1):
    """C1: 16x12x4 mm pad, 6x4x2 cells (288 tets / 105 verts); icosphere R=3 mm
    subdiv 2 starting 0.2 mm above the top centre, pressed to 0.5 mm below the
    undeformed top in `steps` steps."""
    ext, cells = (16 * MM, 12 * MM, 4 * MM), (6, 4, 2)
    X, T, Fx = make_pad(ext, cells, mirror=mirror)
    R = 3 * MM
    Y, tris = make_icosphere(R, 2)
    M, frame = make_markers(ext, cells)
    q = [1.0, 0, 0, 0]
    init = np.stack([pose((0, 0, R + 0.2 * MM), q)] * n_envs)
    z = np.linspace(R + 0.2 * MM, R - depth, steps + 1)[1:]
    poses = np.stack([np.stack([pose((0, 0, zz), q)] * n_envs) for zz in z])
    return Scene("C1", X, T, Fx, Y, tris, M, frame, init, poses, material=Material(mu_f=mu_f),
                 extent=ext, cells=cells)


def scene_c2(steps=50, subdiv=4):
    """C2: GelSight-Mini-like 32x24x5 mm pad, 30x22x5 cells (19,800 tets / 4,278
    verts); icosphere R=5 mm; press 10 x 0.1 mm from a 0.1 mm gap, slide +x
    20 x 0.05 mm, retract 10 x 0.1 mm, settle."""
    ext, cells = (32 * MM, 24 * MM, 5 * MM), (30, 22, 5)
    X, T, Fx = make_pad(ext, cells)
    R = 5 * MM
    Y, tris = make_icosphere(R, subdiv)
    M, frame = make_markers(ext, cells)
    q = [1.0, 0, 0, 0]
    c = np.array([0.0, 0.0, R + 0.1 * MM])
    traj = []
    for _ in range(11):
        c = c + (0, 0, -0.1 * MM)
        traj.append(c.copy())
    for _ in range(20):
        c = c + (0.05 * MM, 0, 0)
        traj.append(c.copy())
    for _ in range(10):
        c = c + (0, 0, 0.11 * MM)
        traj.append(c.copy())
    while len(traj) < steps:
        traj.append(c.copy())
    traj = traj[:steps]
    init = pose((0, 0, R + 0.1 * MM), q)[None]
    poses = np.stack([pose(cc, q)[None] for cc in traj])
    return Scene("C2", X, T, Fx, Y, tris, M, frame, init, poses, extent=ext, cells=cells)


def peg_trajectory(seed, n_steps=64, noise=True):
    """One env of the peg-insertion-shaped workload (C3): yaw ~ U[-35,35] deg
    (P:332), lateral offset ~ U[-3,3] mm, press depth ~ U[0.3,1.0] mm
    at <= 0.1 mm/step, then random-order shear / twist / partial-release phases,
    repeated in cycles (a fresh press depth and phase order per cycle) until the last
    n_steps // 10 steps, which lift the peg off (~10 % of the env-steps
    out of contact, the rest in contact); per-step noise N(0,(0.01 mm)^2) and
    N(0,(0.05 deg)^2) (Table `random`, scaled as stated in DESIGN.md)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    rad = 4 * MM
    yaw = np.deg2rad(rng.uniform(-35, 35))
    off = rng.uniform(-3, 3) * MM
    depth = rng.uniform(0.3, 1.0) * MM
    q0 = quat_axis_angle((0, 0, 1), yaw)
    lateral = np.array([-np.sin(yaw), np.cos(yaw), 0.0])
    c = lateral * off + np.array([0, 0, rad + 0.1 * MM])
    c_start = c.copy()
    init = pose(c, q0)
    traj_c, traj_ang = [], []
    ang = 0.0
    n_tail = n_steps // 10
    cycle = 0
    while len(traj_c) < n_steps - n_tail:
        if cycle > 0:
            depth = rng.uniform(0.3, 1.0) * MM
        zt = rad - depth
        while abs(c[2] - zt) > 1e-12:  # press (or rise) to this cycle's depth at <= 0.1 mm/step
            c = c.copy()
            c[2] = max(zt, c[2] - 0.1 * MM) if c[2] > zt else min(zt, c[2] + 0.1 * MM)
            traj_c.append(c)
            traj_ang.append(ang)
        phases = ["shear", "twist", "release"]
        rng.shuffle(phases)
        for ph in phases:
            if ph == "shear":
                th = rng.uniform(0, 2 * np.pi)
                dxy = (c - c_start)[:2]
                if cycle > 0 and np.linalg.norm(dxy) > 1.5 * MM:  # later cycles drift back toward the start
                    th = np.arctan2(-dxy[1], -dxy[0]) + rng.uniform(-1.0, 1.0)
                d = np.array([np.cos(th), np.sin(th), 0.0])
                step = rng.uniform(0.03, 0.1) * MM
                for _ in range(rng.integers(5, 16)):
                    c = c + d * step
                    traj_c.append(c)
                    traj_ang.append(ang)
            elif ph == "twist":
                dang = np.deg2rad(rng.uniform(-0.5, 0.5))
                for _ in range(rng.integers(4, 9)):
                    ang += dang
                    traj_c.append(c)
                    traj_ang.append(ang)
            else:  # partial release: 20-80 % of the current depth, the peg stays in contact
                up = rng.uniform(0.2, 0.8) * (rad - c[2])
                n = max(1, int(np.ceil(up / (0.1 * MM))))
                for _ in range(n):
                    c = c + (0, 0, up / n)
                    traj_c.append(c)
                    traj_ang.append(ang)
        cycle += 1
    del traj_c[n_steps - n_tail:], traj_ang[n_steps - n_tail:]
    # lift-off tail: out of contact for the last n_tail steps once clear of the gel
    while len(traj_c) < n_steps:
        c = c.copy()
        c[2] = min(c[2] + 0.1 * MM, rad + 0.3 * MM)
        traj_c.append(c)
        traj_ang.append(ang)
    poses = []
    for s in range(n_steps):
        cc = np.array(traj_c[s], float)
        a = traj_ang[s]
        q = quat_mul(quat_axis_angle((0, 0, 1), a), q0)
        if noise:
            cc = cc + rng.normal(0, 0.01 * MM, 3) * np.array([1, 1, 0.2])
            q = quat_mul(quat_axis_angle(rng.normal(size=3), np.deg2rad(rng.normal(0, 0.05))), q)
        poses.append(pose(cc, q))
    return init, np.stack(poses)


def scene_c3(n_envs=1024, n_steps=64, seed0=20260000, cells=(30, 22, 5), noise=True):
    """C3: C2 pad, cylinder peg of diameter 8 mm, length 24 mm, 64 x 24
    facets + caps, axis in the pad plane; per-env random trajectories."""
    ext = (32 * MM, 24 * MM, 5 * MM)
    X, T, Fx = make_pad(ext, cells)
    Y, tris = make_cylinder(4 * MM, 24 * MM, 64, 24)
    M, frame = make_markers(ext, cells)
    inits, poses = [], []
    for e in range(n_envs):
        i0, p = peg_trajectory(seed0 + e, n_steps, noise=noise)
        inits.append(i0)
        poses.append(p)
    return Scene("C3", X, T, Fx, Y, tris, M, frame, np.stack(inits), np.stack(poses, axis=1),
                 extent=ext, cells=cells)


def scene_small_peg(n_envs=5, n_steps=4, seed0=20260000):
    """Small multi-env peg scene for parity tests: C1-sized pad (so the oracle
    finishes in seconds), a scaled-down peg, ragged env count."""
    ext, cells = (16 * MM, 12 * MM, 4 * MM), (6, 4, 2)
    X, T, Fx = make_pad(ext, cells)
    Y, tris = make_cylinder(4 * MM, 14 * MM, 24, 8)
    M, frame = make_markers(ext, cells)
    inits, poses = [], []
    for e in range(n_envs):
        i0, p = peg_trajectory(seed0 + e, n_steps, noise=True)
        inits.append(i0)
        poses.append(p)
    return Scene("small_peg", X, T, Fx, Y, tris, M, frame, np.stack(inits), np.stack(poses, axis=1),
                 extent=ext, cells=cells)


# ----------------------------------------------------------------------------
# §8f-1: unstructured-mesh workload ("unstructured mesh", 1,665 vs 4,465 FPS)
# ----------------------------------------------------------------------------
def make_pad_unstructured(extent, cells, jitter=0.2, seed=7, shuffle=True):
    """Kuhn pad with every strictly interior vertex jittered by up to `jitter` cells per
    axis (irregular element shapes) and, with `shuffle`, random vertex and tet numbering
    (irregular memory access).  Boundary vertices keep their grid positions so the faces
    stay planar and the fixed base / contact face are unchanged.  Positive volumes are
    asserted."""
    rng = np.random.Generator(np.random.PCG64(seed))
    X, T, F = make_pad(extent, cells)
    Lx, Ly, Lz = extent
    c = np.array([Lx / cells[0], Ly / cells[1], Lz / cells[2]])
    lo = np.array([-Lx / 2, -Ly / 2, -Lz])
    hi = np.array([Lx / 2, Ly / 2, 0.0])
    interior = np.all((X > lo + 1e-9) & (X < hi - 1e-9), axis=1)
    X = X.copy()
    X[interior] += rng.uniform(-jitter, jitter, (interior.sum(), 3)) * c
    X = f32(X)
    if shuffle:
        perm = rng.permutation(len(X))          # new id -> old id
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(X))
        X = X[perm]
        T = inv[T]
        F = np.sort(inv[F]).astype(np.int32)
        T = T[rng.permutation(len(T))]
    T = np.asarray(T, dtype=np.int32)
    vol = np.einsum("ij,ij->i", np.cross(X[T[:, 1]] - X[T[:, 0]], X[T[:, 2]] - X[T[:, 0]]), X[T[:, 3]] - X[T[:, 0]])
    assert vol.min() > 0, vol.min()
    return X, T, np.asarray(F, dtype=np.int32)


def scene_c3_unstructured(n_envs=1024, n_steps=64, seed0=20260000, cells=(30, 22, 5)):
    s = scene_c3(n_envs=n_envs, n_steps=n_steps, seed0=seed0, cells=cells)
    s.X, s.tets, s.fixed = make_pad_unstructured(s.extent, cells)
    s.name = "C3u"
    return s


def scene_c5(n_envs=256, n_steps=64, seed0=20270000):
    """C5 stress: 32x24x5 mm pad, 48x36x10 cells (103,680 tets / 19,943 verts); sharp-edged
    8x8x24 mm square peg, faces split at 0.5 mm; press onto a face, then onto an edge
    (rolled 45 deg), slide 2 mm, twist at 0.5 deg/step."""
    ext, cells = (32 * MM, 24 * MM, 5 * MM), (48, 36, 10)
    X, T, Fx = make_pad(ext, cells)
    Y, tris = make_square_peg(8 * MM, 24 * MM, 0.5 * MM)
    M, frame = make_markers(ext, cells)
    inits, poses = [], []
    for e in range(n_envs):
        rng = np.random.Generator(np.random.PCG64(seed0 + e))
        edge = e % 2 == 1  # half the envs press onto an edge
        roll = quat_axis_angle((1, 0, 0), np.pi / 4) if edge else np.array([1.0, 0, 0, 0])
        yaw = np.deg2rad(rng.uniform(-35, 35))
        q0 = quat_mul(quat_axis_angle((0, 0, 1), yaw), roll)
        h = 4 * MM * (2 ** 0.5 if edge else 1.0)
        c = np.array([rng.uniform(-2, 2) * MM, rng.uniform(-2, 2) * MM, h + 0.1 * MM])
        init = pose(c, q0)
        traj = []
        ang = 0.0
        d = np.array([np.cos(yaw), np.sin(yaw), 0.0])
        for s_ in range(n_steps):
            if s_ < 11:
                c = c + (0, 0, -0.1 * MM)
            elif s_ < 31:
                c = c + d * 0.1 * MM
            elif s_ < 51:
                ang += np.deg2rad(0.5) * (1 if s_ < 41 else -1)
            traj.append(pose(c, quat_mul(quat_axis_angle((0, 0, 1), ang), q0)))
        inits.append(init)
        poses.append(np.stack(traj))
    sc = Scene("C5", X, T, Fx, Y, tris, M, frame, np.stack(inits), np.stack(poses, axis=1), extent=ext, cells=cells)
    sc.params.max_candidates = 65536  # edge presses of the split square peg reach ~46k pairs per env
    sc.params.max_anchors = 16384
    return sc

# ----------------------------------------------------------------------------
# §8f-2: batched material calibration (Eqs. 6-7)
# ----------------------------------------------------------------------------
def scene_calib(frames=6, cells=(16, 12, 4), f_max=0.2, shape="sphere"):
    """Calibration workload: N = 4 indentation trajectories of a 3 mm sphere on a
    16x12x4 mm pad ("different deformation modes": press + shear x, off-centre
    press + shear y, deep press, press + twist), `frames` frames each.  The pose spring's
    force cap f_max (R18) is lowered so the deep frames are force-limited: with a purely
    displacement-driven indenter the quasi-static marker field carries almost no
    information about E.  Poses [frames][4][7]; the reference fields come from the
    simulator at a hidden theta_true (synthetic)."""
    ext = (16 * MM, 12 * MM, 4 * MM)
    X, T, Fx = make_pad(ext, cells)
    if shape == "sphere":
        R = 3 * MM  # centre height above the contact point
        Y, tris = make_icosphere(R, 2)
    elif shape == "cylinder":  # lying cylinder (axis along body x): line contact
        R = 2.5 * MM
        Y, tris = make_cylinder(R, 8 * MM, 24, 6)
    elif shape == "cube":  # 5 mm cube pressed flat-face down
        R = 2.5 * MM
        Y, tris = make_square_peg(5 * MM, 5 * MM, 1.25 * MM)
    else:
        raise ValueError(shape)
    M, frame = make_markers(ext, cells)
    q0 = [1.0, 0, 0, 0]
    gap = 0.05 * MM
    half = frames // 2
    trajs = []
    specs = [((0.0, 0.0), 0.4 * MM, (0.3 * MM, 0.0), 0.0),
             ((2.0 * MM, -1.0 * MM), 0.3 * MM, (0.0, 0.3 * MM), 0.0),
             ((-1.5 * MM, 1.0 * MM), 0.9 * MM, (0.0, 0.0), 0.0),
             ((0.0, 1.0 * MM), 0.35 * MM, (0.0, 0.0), 5.0)]
    inits = []
    for (x0, y0), depth, (sx, sy), twist_deg in specs:
        inits.append(pose((x0, y0, R + gap), q0))
        fr = []
        for k in range(frames):
            if k < half:
                t = (k + 1) / half
                fr.append(pose((x0, y0, R + gap - t * (gap + depth)), q0))
            else:
                t = (k + 1 - half) / (frames - half)
                a = np.deg2rad(twist_deg) * t
                q = [np.cos(a / 2), 0.0, 0.0, np.sin(a / 2)]
                fr.append(pose((x0 + t * sx, y0 + t * sy, R - depth), q))
        trajs.append(fr)
    poses = np.stack([np.stack([trajs[i][k] for i in range(len(specs))]) for k in range(frames)])
    sc = Scene("calib_" + shape, X, T, Fx, Y, tris, M, frame, np.stack(inits), poses, extent=ext, cells=cells)
    sc.params.f_max = f_max
    # a generation waits for its slowest candidate: near-incompressible candidates (nu -> 0.497)
    # are capped at 1,000 iterations per step (their loss is then noisier, which CMA-ES tolerates)
    sc.params.max_iters = 1000
    return sc


def scene_calib_shapes(frames=6, f_max=0.2):
    """Several indenter shapes for one calibration (P:305 uses four: cube, cylinder, moon,
    triangle): sphere, lying cylinder and cube, one scene (= one simulator) each."""
    return [scene_calib(frames=frames, f_max=f_max, shape=sh) for sh in ("sphere", "cylinder", "cube")]
