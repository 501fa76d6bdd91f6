"""Two-finger gripper rig: both gel pads of a parallel gripper in one simulator.

PAPER.md P:384 mounts two GelSight Mini sensors on the Franka gripper "to maintain force
equilibrium" and feeds only the right finger's marker field to the policy.
The pads do not touch each other; each one is pressed by the held object (the indenter),
seen through its own sensor frame.  So a rig is two envs of ONE simulator -- env 2i is the
left pad of rig i, env 2i + 1 the right pad -- and one launch per phase still serves every
pad of every rig (no kernel change).  This module only maps the object's pose in the
gripper frame to each pad's relative pose (host-side pose bookkeeping, like the poses a
policy sends), then calls tac_step / tac_markers through the binding.

Gripper frame (g): fingers close along y_g, the left pad's contact face at y_g = +w/2
facing -y_g, the right pad's at y_g = -w/2 facing +y_g, w = opening.  Sensor frames
(gel frame of include/tac.h: contact face z = 0, outward normal +z, x along x_g):

    left:  R_gl = [x_g, z_g, -y_g],  t_gl = (0, +w/2, 0)
    right: R_gr = [x_g, -z_g, y_g],  t_gr = (0, -w/2, 0)

and the object in sensor s: R_so = R_gs^T R_go, t_so = R_gs^T (t_go - t_gs).
"""
from __future__ import annotations

import numpy as np

R_LEFT = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, -1.0], [0.0, 1.0, 0.0]])   # columns x_g, z_g, -y_g
R_RIGHT = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 1.0], [0.0, -1.0, 0.0]])  # columns x_g, -z_g, y_g


def quat_to_R(q):
    """Unit quaternion (w, x, y, z) -> rotation matrix."""
    w, x, y, z = np.asarray(q, dtype=np.float64) / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def R_to_quat(R):
    """Rotation matrix -> unit quaternion (w, x, y, z), w >= 0 (Shepperd's branches)."""
    R = np.asarray(R, dtype=np.float64)
    t = np.trace(R)
    if t > 0:
        s = 2.0 * np.sqrt(1.0 + t)
        q = np.array([0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s])
    else:
        i = int(np.argmax(np.diag(R)))
        j, k = (i + 1) % 3, (i + 2) % 3
        s = 2.0 * np.sqrt(1.0 + R[i, i] - R[j, j] - R[k, k])
        q = np.empty(4)
        q[0] = (R[k, j] - R[j, k]) / s
        q[1 + i] = 0.25 * s
        q[1 + j] = (R[j, i] + R[i, j]) / s
        q[1 + k] = (R[k, i] + R[i, k]) / s
    q /= np.linalg.norm(q)
    return q if q[0] >= 0 else -q


def finger_frames(opening):
    """((R_gl, t_gl), (R_gr, t_gr)) for a gripper opening w [m] (contact faces w apart)."""
    h = 0.5 * float(opening)
    return (R_LEFT, np.array([0.0, h, 0.0])), (R_RIGHT, np.array([0.0, -h, 0.0]))


def pad_poses(object_poses, openings):
    """Object poses in the gripper frame [N, 7] (t, q_wxyz) and openings [N] -> the relative
    poses the simulator takes, [2N, 7]: row 2i for the left pad, 2i + 1 for the right."""
    P = np.asarray(object_poses, dtype=np.float64).reshape(-1, 7)
    w = np.broadcast_to(np.asarray(openings, dtype=np.float64), (len(P),))
    out = np.empty((2 * len(P), 7))
    for i, (p, wi) in enumerate(zip(P, w)):
        R_go = quat_to_R(p[3:])
        for s, (R_gs, t_gs) in enumerate(finger_frames(wi)):
            out[2 * i + s, :3] = R_gs.T @ (p[:3] - t_gs)
            out[2 * i + s, 3:] = R_to_quat(R_gs.T @ R_go)
    return out


class TwoFingerRig:
    """n_rigs two-pad rigs in one TacSim (2 n_rigs envs).  `sim` must have been created with
    n_envs = 2 n_rigs and initial poses from pad_poses(...)."""

    def __init__(self, sim):
        assert sim.n_envs % 2 == 0, "a rig holds two envs per gripper"
        self.sim = sim
        self.n_rigs = sim.n_envs // 2

    def step(self, object_poses, openings, dt, stream=None):
        import torch
        poses = torch.tensor(pad_poses(object_poses, openings), dtype=torch.float32,
                             device=f"cuda:{self.sim.device}")
        self.sim.step(poses, dt, stream=stream)
        return poses

    def markers(self, finger="right", ncomp=2, stream=None):
        """Marker fields [n_rigs, n_markers, ncomp] of one finger ("left" / "right"; the paper's
        policy reads the right one), or [n_rigs, 2, n_markers, ncomp] for "both"."""
        m = self.sim.markers(ncomp=ncomp, stream=stream).view(self.n_rigs, 2, self.sim.nm, ncomp)
        if finger == "both":
            return m
        return m[:, 0 if finger == "left" else 1]
