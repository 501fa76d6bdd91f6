"""Two-finger rig: the host pose bookkeeping on CPU, and on
the GPU both pads of a rig stepped as two envs of one simulator."""
import numpy as np
import pytest

from paper_2603_28475_b200 import rig


def _rand_R(rng):
    q = rng.standard_normal(4)
    return rig.quat_to_R(q / np.linalg.norm(q))


def test_quaternion_round_trip_and_frames():
    rng = np.random.default_rng(5)
    for _ in range(50):
        R = _rand_R(rng)
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-12) and np.isclose(np.linalg.det(R), 1.0)
        assert np.allclose(rig.quat_to_R(rig.R_to_quat(R)), R, atol=1e-12)
    for Rs in (rig.R_LEFT, rig.R_RIGHT):  # proper rotations, x along the gripper's x
        assert np.allclose(Rs @ Rs.T, np.eye(3)) and np.isclose(np.linalg.det(Rs), 1.0)
        assert np.allclose(Rs[:, 0], [1, 0, 0])


def test_pad_normals_face_each_other():
    (Rl, tl), (Rr, tr) = rig.finger_frames(10e-3)
    # each pad's outward normal (sensor +z) points from its face towards the other finger
    assert np.allclose(Rl[:, 2], (tr - tl) / np.linalg.norm(tr - tl))
    assert np.allclose(Rr[:, 2], (tl - tr) / np.linalg.norm(tl - tr))


def test_centred_object_is_seen_alike_by_both_pads():
    # object at the gripper origin: both pads see it w/2 above their contact face
    p = np.array([[0, 0, 0, 1, 0, 0, 0]], dtype=float)
    out = rig.pad_poses(p, 8e-3)
    assert np.allclose(out[0, :3], [0, 0, 4e-3]) and np.allclose(out[1, :3], [0, 0, 4e-3])
    # shifted towards the left finger by d: the left pad sees it d closer, the right d farther
    p[0, 1] = 1e-3
    out = rig.pad_poses(p, 8e-3)
    assert np.isclose(out[0, 2], 3e-3) and np.isclose(out[1, 2], 5e-3)
    # a shift along the gripper's x is the same in-plane shift for both pads
    p[0, :3] = [2e-3, 0, 0]
    out = rig.pad_poses(p, 8e-3)
    assert np.allclose(out[:, :3], [[2e-3, 0, 4e-3], [2e-3, 0, 4e-3]])


def test_relative_pose_composes_back():
    rng = np.random.default_rng(9)
    P = np.zeros((6, 7))
    P[:, :3] = rng.uniform(-2e-3, 2e-3, (6, 3))
    for i in range(6):
        P[i, 3:] = rig.R_to_quat(_rand_R(rng))
    w = rng.uniform(6e-3, 12e-3, 6)
    out = rig.pad_poses(P, w)
    for i in range(6):
        for s, (Rgs, tgs) in enumerate(rig.finger_frames(w[i])):
            Rso, tso = rig.quat_to_R(out[2 * i + s, 3:]), out[2 * i + s, :3]
            assert np.allclose(Rgs @ Rso, rig.quat_to_R(P[i, 3:]), atol=1e-12)
            assert np.allclose(Rgs @ tso + tgs, P[i, :3], atol=1e-15)


@pytest.mark.gpu
def test_rig_pads_step_in_one_simulator():
    """A peg squeezed symmetrically between the two pads: both pads' marker fields agree (the
    faceted cylinder is symmetric under the half turn relating the two sensor views), and the
    right pad's field equals a one-pad simulator driven by the right pad's relative poses."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_28475_b200 as P
    import workloads as w
    s = w.scene_small_peg(n_envs=2, n_steps=2)
    s.params.fixed_iters = 0
    s.params.tol_x = 1e-9
    s.params.stagnation = 300
    # peg axis along the gripper's x, turned half a facet (7.5 deg) about it so that flat faces,
    # not facet edges, rest on the pads: an edge over the pad's mid vertex line is a symmetric
    # saddle of the frictional minimiser (R25) and the two pads could break it apart
    a = np.deg2rad(7.5)
    R_peg = np.array([[1, 0, 0], [0, np.cos(a), -np.sin(a)], [0, np.sin(a), np.cos(a)]])
    radius = 4e-3 * np.cos(np.pi / 24)  # face distance of make_cylinder(4 mm, 14 mm, 24 facets)
    openings = [2 * radius + 0.1e-3, 2 * radius - 0.1e-3]  # first touching-free, then 50 um into each pad
    obj = np.array([[0, 0, 0, *rig.R_to_quat(R_peg)]])
    init = rig.pad_poses(obj, openings[0])
    s.init_poses = init
    sim = P.TacSim.from_scene(s, n_envs=2, init_poses=init)
    tw = rig.TwoFingerRig(sim)
    solo = P.TacSim.from_scene(s, n_envs=1, init_poses=init[1:2])
    for wk in openings:
        poses = tw.step(obj, wk, s.dt)
        solo.step(poses[1:2].contiguous(), s.dt)
    m = tw.markers("both").cpu().numpy()[0]
    scale = np.abs(m).max()
    assert scale > 0
    assert np.abs(m[0] - m[1]).max() <= 1e-3 * scale
    ms = solo.markers().cpu().numpy()[0]
    assert np.abs(tw.markers("right").cpu().numpy()[0] - ms).max() <= 1e-3 * scale
