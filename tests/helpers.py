"""Shared test helpers."""
import numpy as np

import workloads as w


def rot_exp(wv):
    """Rodrigues formula, written out here independently of the oracle."""
    wv = np.asarray(wv, float)
    th = np.linalg.norm(wv)
    K = np.array([[0, -wv[2], wv[1]], [wv[2], 0, -wv[0]], [-wv[1], wv[0], 0]])
    if th < 1e-12:
        return np.eye(3) + K
    return np.eye(3) + np.sin(th) / th * K + (1 - np.cos(th)) / th ** 2 * K @ K


def quat_R(q):
    wq, x, y, z = np.asarray(q, float) / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - wq * z), 2 * (x * z + wq * y)],
                     [2 * (x * y + wq * z), 1 - 2 * (x * x + z * z), 2 * (y * z - wq * x)],
                     [2 * (x * z - wq * y), 2 * (y * z + wq * x), 1 - 2 * (x * x + y * y)]])


def c1_press_scene(mu_f=1.0, steps=4, depth=0.2e-3, start_gap=0.05e-3, mirror=False):
    """C1 mesh + sphere, starting `start_gap` above the top, pressed to `depth`
    below it in `steps` equal steps (the paper's 0.1 mm press increments)."""
    s = w.scene_c1(mu_f=mu_f, mirror=mirror)
    R = 3e-3
    q = [1.0, 0, 0, 0]
    s.init_poses = np.stack([w.pose((0, 0, R + start_gap), q)])
    z = np.linspace(R + start_gap, R - depth, steps + 1)[1:]
    s.poses = np.stack([np.stack([w.pose((0, 0, zz), q)]) for zz in z])
    return s


def parallel_peg_scene(steps=2, depth=0.05e-3, start_gap=0.05e-3, offset_y=0.0):
    """C1 pad and the small peg lying along the pad's x axis (yaw 0), its bottom axial edge
    parallel to the pad's x edges: pressed to `depth` in `steps` steps.  Edge-edge pairs of
    nearly parallel edges carry contact (the EE mollifier's case, R30)."""
    s = w.scene_small_peg(n_envs=1, n_steps=steps)
    r = 4e-3  # make_cylinder(4 mm, 14 mm, 24, 8): a vertex line at the bottom
    q = [1.0, 0, 0, 0]
    s.init_poses = np.stack([w.pose((0, offset_y, r + start_gap), q)])
    z = np.linspace(r + start_gap, r - depth, steps + 1)[1:]
    s.poses = np.stack([np.stack([w.pose((0, offset_y, zz), q)]) for zz in z])
    return s


def pg_disp(o, scene, ev, rho_max):
    """fp64 |P g|_disp of an oracle evaluation (block-Jacobi P: the 3x3 D^-1 per free vertex and
    the rigid blocks; the convergence measure of P:465 / R12): the stationarity certificate of a
    state, independent of the solver that produced it."""
    free = np.setdiff1d(np.arange(len(scene.X)), scene.fixed)
    g, D = ev["g"], ev["D"]
    m = 0.0
    for v in free:
        m = max(m, np.linalg.norm(np.linalg.solve(D[v], g[v])))
    pc = np.linalg.solve(ev["Drig"][0], ev["grig"][:3])
    pt = np.linalg.solve(ev["Drig"][1], ev["grig"][3:])
    return max(m, np.linalg.norm(pc) + rho_max * np.linalg.norm(pt))
