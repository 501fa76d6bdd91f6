"""Thin ctypes binding of libtac (include/tac.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of csrc/; PyTorch is used for
device memory (tensors' data_ptr) and streams.  There is no CPU fallback: if the
library or a CUDA device is missing, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtac.so")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)

FLAG_CONVERGED, FLAG_MAXITER, FLAG_NAN, FLAG_INFEASIBLE = 1, 2, 4, 8
FLAG_LARGE_MOTION, FLAG_OVERFLOW, FLAG_STAGNATION = 16, 32, 64


class TetMesh(C.Structure):
    _fields_ = [("n_verts", C.c_int32), ("rest_xyz", _dp), ("n_tets", C.c_int32), ("tets", _ip),
                ("n_fixed", C.c_int32), ("fixed", _ip)]


class TriMesh(C.Structure):
    _fields_ = [("n_verts", C.c_int32), ("rest_xyz", _dp), ("n_tris", C.c_int32), ("tris", _ip)]


class Material(C.Structure):
    _fields_ = [("E", C.c_double), ("nu", C.c_double), ("rho", C.c_double), ("mu_f", C.c_double)]


class MarkerSet(C.Structure):
    _fields_ = [("rows", C.c_int32), ("cols", C.c_int32), ("rest_xyz", _dp), ("t1", C.c_double * 3),
                ("t2", C.c_double * 3), ("n", C.c_double * 3), ("mode", C.c_int32), ("k", C.c_int32)]


class SolverParams(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("dhat", "kappa_phys", "eps_v", "tol_x", "k_t", "k_r", "f_max", "t_max",
                                           "ccd_s", "bp_margin", "c1", "eps_E")] + \
               [(n, C.c_int32) for n in ("max_iters", "fixed_iters", "beta_rule", "precond", "max_halvings",
                                          "stagnation", "max_candidates", "max_anchors", "check_every", "pose_al",
                                          "ee_mollifier", "dedup")]


class CreateInfo(C.Structure):
    _fields_ = [("gel", C.POINTER(TetMesh)), ("mat", C.POINTER(Material)), ("markers", C.POINTER(MarkerSet)),
                ("indenter", C.POINTER(TriMesh)), ("params", C.POINTER(SolverParams)), ("n_envs", C.c_int32),
                ("device", C.c_int32), ("init_poses", _fp)]


_lib = None


def lib():
    """Load libtac.so (build it in-tree first if the sources are newer)."""
    global _lib
    if _lib is None:
        from . import build as _build
        alt = os.environ.get("TAC_LIB")  # A/B measurements: another in-tree build of libtac
        if not alt:
            try:
                _build.build()
            except Exception as exc:  # no nvcc on this host: use the prebuilt library if present
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(f"libtac.so missing and cannot be built: {exc}") from exc
        L = C.CDLL(alt or LIB_PATH)
        vp = C.c_void_p
        L.tac_create.argtypes = [C.POINTER(CreateInfo), C.POINTER(vp)]
        L.tac_step.argtypes = [vp, vp, C.c_float, vp]
        L.tac_markers.argtypes = [vp, vp, C.c_int32, vp]
        L.tac_reset.argtypes = [vp, vp, vp, vp]
        L.tac_env_status.argtypes = [vp, vp, vp, vp, vp]
        L.tac_set_env_material.argtypes = [vp, _dp, _dp, _dp, _dp, vp]
        L.tac_marker_sqerr.argtypes = [vp, vp, vp, C.c_int32, vp]
        L.tac_set_pose_noise.argtypes = [vp, C.c_double, C.c_double, C.c_uint64, C.c_int64]
        L.tac_info.argtypes = [vp, _ip]
        L.tac_checkpoint_size.argtypes = [vp, C.POINTER(C.c_uint64)]
        L.tac_checkpoint_save.argtypes = [vp, vp, vp]
        L.tac_checkpoint_load.argtypes = [vp, vp, vp]
        L.tac_nccl_unique_id.argtypes = [vp]
        L.tac_nccl_comm_create.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.POINTER(vp)]
        L.tac_nccl_comm_destroy.argtypes = [vp]
        L.tac_gather_markers.argtypes = [vp, vp, vp, C.c_int32, vp]
        L.tac_last_launch_count.argtypes = [vp]
        L.tac_last_launch_count.restype = C.c_int64
        L.tac_destroy.argtypes = [vp]
        L.tac_last_error.argtypes = [vp]
        L.tac_last_error.restype = C.c_char_p
        L.tac_get_state.argtypes = [vp, C.c_int32, _dp, _dp, _dp, _dp]
        L.tac_set_state.argtypes = [vp, C.c_int32, _dp, _dp, _dp, _dp]
        L.tac_debug_broadphase.argtypes = [vp, C.c_int32, _fp, _dp, _dp, C.c_double, _ip, C.c_int32, _ip]
        L.tac_debug_surface.argtypes = [vp, _ip, _ip, _ip, _ip, _ip]
        L.tac_debug_marker_map.argtypes = [vp, _ip, _ip, _dp]
        L.tac_profile_enable.argtypes = [vp, C.c_int32]
        L.tac_env_stats.argtypes = [vp, vp, vp]
        L.tac_profile_read.argtypes = [vp, _dp, C.POINTER(C.c_int64), C.c_int32]
        L.tac_profile_kernel_name.argtypes = [C.c_int32]
        L.tac_profile_kernel_name.restype = C.c_char_p
        L.tac_debug_eval.argtypes = [vp, C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_double, _dp, _dp,
                                     _dp, _dp, _dp]
        L.tac_debug_iteration.argtypes = [vp, C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_double, _dp, _dp,
                                          C.c_double, C.c_int32, _dp, _dp]
        _lib = L
    return _lib


EXPORTED = ["tac_create", "tac_step", "tac_markers", "tac_reset", "tac_env_status", "tac_info",
            "tac_last_launch_count", "tac_destroy", "tac_last_error", "tac_get_state", "tac_set_state",
            "tac_debug_broadphase", "tac_debug_surface", "tac_debug_marker_map", "tac_debug_eval",
            "tac_profile_enable", "tac_profile_read", "tac_profile_kernel_name", "tac_env_stats",
            "tac_set_env_material", "tac_marker_sqerr", "tac_set_pose_noise", "tac_nccl_unique_id",
            "tac_nccl_comm_create", "tac_nccl_comm_destroy", "tac_gather_markers", "tac_checkpoint_size",
            "tac_checkpoint_save", "tac_checkpoint_load", "tac_debug_iteration"]
N_KERNEL_IDS = 25


class TacError(RuntimeError):
    pass


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(_ip)


def _check_tensor(t, dtype, numel, device, name, at_least=False):
    """Arguments of the C ABI are raw device pointers: refuse anything the kernels would read
    as garbage (wrong dtype, host memory, another device, non-contiguous, wrong size)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TacError(f"{name}: expected a torch.Tensor")
    if t.dtype != dtype:
        raise TacError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if not t.is_cuda or t.device.index != device:
        raise TacError(f"{name}: must live on cuda:{device} (got {t.device})")
    if not t.is_contiguous():
        raise TacError(f"{name}: must be contiguous")
    if (t.numel() < numel) if at_least else (t.numel() != numel):
        raise TacError(f"{name}: {t.numel()} elements, expected {'>= ' if at_least else ''}{numel}")


def _stream_ptr(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


class TacSim:
    """One handle per GPU owning n_envs environments."""

    def __init__(self, X, tets, fixed, Y, tris, markers, frame, material, params, n_envs, init_poses, device=0,
                 marker_mode=0, knn_k=4, rows=7, cols=9):
        import torch
        if not torch.cuda.is_available():
            raise TacError("CUDA device required: libtac has no CPU fallback")
        L = lib()
        self._keep = []
        Xa, Xp = _d(X)
        Ta, Tp = _i(tets)
        Fa, Fp = _i(fixed)
        Ya, Yp = _d(Y)
        Ra, Rp = _i(tris)
        Ma, Mp = _d(markers)
        self._keep += [Xa, Ta, Fa, Ya, Ra, Ma]
        gel = TetMesh(len(Xa), Xp, len(Ta), Tp, len(Fa), Fp)
        ind = TriMesh(len(Ya), Yp, len(Ra), Rp)
        mat = Material(material.E, material.nu, material.rho, material.mu_f)
        fr = np.asarray(frame, float)
        ms = MarkerSet(rows, cols, Mp, (C.c_double * 3)(*fr[0]), (C.c_double * 3)(*fr[1]), (C.c_double * 3)(*fr[2]),
                       marker_mode, knn_k)
        sp = SolverParams(params.dhat, params.kappa_phys, params.eps_v, params.tol_x, params.k_t, params.k_r,
                          params.f_max, params.t_max, params.ccd_s, params.bp_margin, params.c1, params.eps_E,
                          params.max_iters, params.fixed_iters, params.beta_rule, params.precond,
                          params.max_halvings, params.stagnation, getattr(params, "max_candidates", 0),
                          getattr(params, "max_anchors", 0), getattr(params, "check_every", 0),
                          getattr(params, "pose_al", 0), getattr(params, "ee_mollifier", 0),
                          getattr(params, "dedup", 0))
        ip = np.ascontiguousarray(init_poses, dtype=np.float32).reshape(n_envs, 7)
        self._keep.append(ip)
        info = CreateInfo(C.pointer(gel), C.pointer(mat), C.pointer(ms), C.pointer(ind), C.pointer(sp), n_envs,
                          device, ip.ctypes.data_as(_fp))
        h = C.c_void_p()
        torch.cuda.set_device(device)
        st = L.tac_create(C.byref(info), C.byref(h))
        if st != 0:
            raise TacError(f"tac_create failed ({st}): {L.tac_last_error(None).decode()}")
        self.h = h
        self.device = device
        self.n_envs = n_envs
        info = np.zeros(10, np.int32)
        L.tac_info(self.h, info.ctypes.data_as(_ip))
        (self.nv, self.nt, _, self.env_stride, self.nm, self.nsv, self.nse, self.nst, self.n_cells,
         self.n_other_tets) = map(int, info)

    @classmethod
    def from_scene(cls, scene, params=None, material=None, n_envs=None, init_poses=None, **kw):
        p = params or scene.params
        m = material or scene.material
        ip = scene.init_poses if init_poses is None else init_poses
        return cls(scene.X, scene.tets, scene.fixed, scene.Y, scene.tris, scene.markers, scene.frame, m, p,
                   ip.shape[0] if n_envs is None else n_envs, ip, **kw)

    def _check(self, st, what):
        if st != 0:
            raise TacError(f"{what} failed ({st}): {lib().tac_last_error(self.h).decode()}")

    def close(self):
        if getattr(self, "h", None):
            lib().tac_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- hot path ----
    def step(self, target_poses, dt, stream=None):
        """target_poses: CUDA float32 tensor [n_envs, 7] (pose at t + dt)."""
        import torch
        _check_tensor(target_poses, torch.float32, 7 * self.n_envs, self.device, "target_poses")
        self._check(lib().tac_step(self.h, C.c_void_p(target_poses.data_ptr()), float(dt), _stream_ptr(stream)),
                    "tac_step")

    def markers(self, out=None, ncomp=2, stream=None):
        import torch
        if out is None:
            out = torch.empty((self.n_envs, self.nm, ncomp), device=f"cuda:{self.device}", dtype=torch.float32)
        _check_tensor(out, torch.float32, self.n_envs * self.nm * ncomp, self.device, "markers out", at_least=True)
        self._check(lib().tac_markers(self.h, C.c_void_p(out.data_ptr()), ncomp, _stream_ptr(stream)), "tac_markers")
        return out

    def gather_markers(self, comm, recvbuf, ncomp=2, stream=None):
        """tac_gather_markers: this rank's marker field into its slot of recvbuf (CUDA fp32
        [nranks * n_envs, n_markers, ncomp]) and an in-place NCCL all-gather of the slots."""
        import torch
        _check_tensor(recvbuf, torch.float32, comm.nranks * self.n_envs * self.nm * ncomp, self.device, "recvbuf")
        self._check(lib().tac_gather_markers(self.h, comm.handle, C.c_void_p(recvbuf.data_ptr()), ncomp,
                                             _stream_ptr(stream)), "tac_gather_markers")
        return recvbuf

    def set_pose_noise(self, sigma_t, sigma_r, seed, env_offset=0):
        """Per-step target pose noise (R27): translation amplitude [m], rotation [rad]."""
        self._check(lib().tac_set_pose_noise(self.h, float(sigma_t), float(sigma_r), int(seed), int(env_offset)),
                    "tac_set_pose_noise")

    def marker_sqerr(self, ref, acc, stream=None):
        """acc[e] += |markers(e) - ref[e]|^2 (calibration loss term, Eq. 6); ref [E, nm, ncomp] fp32,
        acc [E] fp64, both on this device."""
        import torch
        ncomp = int(ref.shape[-1])
        if ncomp not in (2, 3):
            raise TacError("marker_sqerr: ref must be [n_envs, n_markers, 2 | 3]")
        _check_tensor(ref, torch.float32, self.n_envs * self.nm * ncomp, self.device, "ref")
        _check_tensor(acc, torch.float64, self.n_envs, self.device, "acc")
        self._check(lib().tac_marker_sqerr(self.h, C.c_void_p(ref.data_ptr()), C.c_void_p(acc.data_ptr()), ncomp,
                                           _stream_ptr(stream)), "tac_marker_sqerr")
        return acc

    def reset(self, mask, poses, stream=None):
        """mask: CUDA uint8 [n_envs] (1 = reset), poses: CUDA float32 [n_envs, 7]."""
        import torch
        _check_tensor(mask, torch.uint8, self.n_envs, self.device, "mask")
        _check_tensor(poses, torch.float32, 7 * self.n_envs, self.device, "poses")
        self._check(lib().tac_reset(self.h, C.c_void_p(mask.data_ptr()), C.c_void_p(poses.data_ptr()),
                                    _stream_ptr(stream)), "tac_reset")

    def set_env_material(self, E=None, nu=None, rho=None, mu_f=None, stream=None):
        """Per-env material theta_e: each argument None or n_envs values."""
        arrs = []
        for a in (E, nu, rho, mu_f):
            if a is None:
                arrs.append((None, None))
            else:
                a = np.ascontiguousarray(np.broadcast_to(np.asarray(a, dtype=np.float64), (self.n_envs,)))
                arrs.append((a, a.ctypes.data_as(_dp)))
        self._check(lib().tac_set_env_material(self.h, *[p for _, p in arrs], _stream_ptr(stream)),
                    "tac_set_env_material")

    # ---- checkpoint / resume ----
    def checkpoint_size(self):
        n = C.c_uint64(0)
        self._check(lib().tac_checkpoint_size(self.h, C.byref(n)), "tac_checkpoint_size")
        return int(n.value)

    def checkpoint_save(self, buf=None, stream=None):
        """The carried state (u^t, v^t, per-env records, step counter) into a device uint8 buffer."""
        import torch
        n = self.checkpoint_size()
        if buf is None:
            buf = torch.empty(n, dtype=torch.uint8, device=f"cuda:{self.device}")
        _check_tensor(buf, torch.uint8, n, self.device, "checkpoint buffer", at_least=True)
        self._check(lib().tac_checkpoint_save(self.h, C.c_void_p(buf.data_ptr()), _stream_ptr(stream)),
                    "tac_checkpoint_save")
        return buf

    def checkpoint_load(self, buf, stream=None):
        import torch
        _check_tensor(buf, torch.uint8, self.checkpoint_size(), self.device, "checkpoint buffer", at_least=True)
        self._check(lib().tac_checkpoint_load(self.h, C.c_void_p(buf.data_ptr()), _stream_ptr(stream)),
                    "tac_checkpoint_load")

    def env_status(self, stream=None):
        import torch
        dev = f"cuda:{self.device}"
        it = torch.empty(self.n_envs, dtype=torch.int32, device=dev)
        pg = torch.empty(self.n_envs, dtype=torch.float32, device=dev)
        fl = torch.empty(self.n_envs, dtype=torch.int32, device=dev)
        self._check(lib().tac_env_status(self.h, C.c_void_p(it.data_ptr()), C.c_void_p(pg.data_ptr()),
                                         C.c_void_p(fl.data_ptr()), _stream_ptr(stream)), "tac_env_status")
        return it, pg, fl

    def env_stats(self, stream=None):
        """int32 tensor [n_envs, 4]: iterations, peak candidates, anchors, rebuilds (last step)."""
        import torch
        out = torch.empty((self.n_envs, 4), dtype=torch.int32, device=f"cuda:{self.device}")
        self._check(lib().tac_env_stats(self.h, C.c_void_p(out.data_ptr()), _stream_ptr(stream)), "tac_env_stats")
        return out

    def profile_enable(self, on=True):
        self._check(lib().tac_profile_enable(self.h, int(on)), "tac_profile_enable")

    def profile_read(self):
        """{kernel name: (total ms, launches)} since the last read (synchronises)."""
        ms = np.zeros(N_KERNEL_IDS)
        cnt = np.zeros(N_KERNEL_IDS, np.int64)
        self._check(lib().tac_profile_read(self.h, ms.ctypes.data_as(_dp), cnt.ctypes.data_as(C.POINTER(C.c_int64)),
                                           N_KERNEL_IDS), "tac_profile_read")
        return {lib().tac_profile_kernel_name(k).decode(): (float(ms[k]), int(cnt[k])) for k in range(N_KERNEL_IDS)}

    def last_launch_count(self):
        return int(lib().tac_last_launch_count(self.h))

    # ---- state / debug hooks (synchronous, host arrays) ----
    def get_state(self, env):
        u = np.zeros((self.nv, 3)); v = np.zeros((self.nv, 3)); c = np.zeros(3); R = np.zeros(9)
        self._check(lib().tac_get_state(self.h, env, *(a.ctypes.data_as(_dp) for a in (u, v, c, R))), "tac_get_state")
        return u, v, c, R.reshape(3, 3)

    def set_state(self, env, u, v, c, R):
        arrs = [_d(a) for a in (u, v, c, np.asarray(R).reshape(9))]
        self._check(lib().tac_set_state(self.h, env, *(a[1] for a in arrs)), "tac_set_state")

    def debug_surface(self):
        sv = np.zeros(self.nsv, np.int32); se = np.zeros((self.nse, 2), np.int32); st = np.zeros((self.nst, 3), np.int32)
        cnt = np.zeros(1, np.int32)
        lib().tac_debug_surface(self.h, None, None, None, None, cnt.ctypes.data_as(_ip))
        ie = np.zeros((int(cnt[0]), 2), np.int32)
        self._check(lib().tac_debug_surface(self.h, *(a.ctypes.data_as(_ip) for a in (sv, se, st, ie, cnt))),
                    "tac_debug_surface")
        return sv, se, st, ie

    def debug_marker_map(self):
        t = np.zeros(self.nm, np.int32); idx = np.zeros((self.nm, 4), np.int32); w = np.zeros((self.nm, 4))
        self._check(lib().tac_debug_marker_map(self.h, t.ctypes.data_as(_ip), idx.ctypes.data_as(_ip),
                                               w.ctypes.data_as(_dp)), "tac_debug_marker_map")
        return t, idx, w

    def debug_broadphase(self, env, u, c, R, r, cap=1 << 20):
        uf = np.ascontiguousarray(u, dtype=np.float32)
        ca, cp = _d(c)
        Ra, Rp = _d(np.asarray(R).reshape(9))
        out = np.zeros((cap, 3), np.int32)
        n = C.c_int32(0)
        self._check(lib().tac_debug_broadphase(self.h, env, uf.ctypes.data_as(_fp), cp, Rp, float(r),
                                               out.ctypes.data_as(_ip), cap, C.byref(n)), "tac_debug_broadphase")
        return out[:min(n.value, cap)]

    def debug_eval(self, env, u_t, v_t, c_t, R_t, u, c, R, target7, dt):
        ins = [_d(a) for a in (u_t, v_t, c_t, np.asarray(R_t).reshape(9), u, c, np.asarray(R).reshape(9), target7)]
        parts = np.zeros(5); g = np.zeros((self.nv, 3)); D = np.zeros((self.nv, 3, 3)); gr = np.zeros(6)
        Dr = np.zeros((2, 3, 3))
        self._check(lib().tac_debug_eval(self.h, env, *(a[1] for a in ins), float(dt),
                                         *(a.ctypes.data_as(_dp) for a in (parts, g, D, gr, Dr))), "tac_debug_eval")
        return dict(E=parts.sum(), parts=parts, g=g, D=D, grig=gr, Drig=Dr)

    ITERATION_FIELDS = ["beta", "gp", "gPg", "restarted", "M", "alpha_upper", "pHp", "alpha_bar", "alpha_ccd",
                        "alpha", "L_rel", "pg_disp"]

    def debug_iteration(self, env, u_t, v_t, c_t, R_t, u, c, R, target7, dt, g_prev, p_prev, gPg_prev,
                        restart=False):
        """tac_debug_iteration: (p [nv*3 + 6], dict of ITERATION_FIELDS) of one PNCG iteration."""
        ins = [_d(a) for a in (u_t, v_t, c_t, np.asarray(R_t).reshape(9), u, c, np.asarray(R).reshape(9), target7,
                                g_prev, p_prev)]
        p = np.zeros(3 * self.nv + 6)
        out = np.zeros(12)
        self._check(lib().tac_debug_iteration(self.h, env, *(a[1] for a in ins[:8]), float(dt), ins[8][1], ins[9][1],
                                              float(gPg_prev), int(restart), p.ctypes.data_as(_dp),
                                              out.ctypes.data_as(_dp)), "tac_debug_iteration")
        return p, dict(zip(self.ITERATION_FIELDS, out))


def nccl_unique_id() -> bytes:
    """tac_nccl_unique_id: a fresh 128-byte NCCL unique id (share it with the other ranks)."""
    import torch  # noqa: F401  (load torch's libnccl.so.2 first: the C ABI then resolves that one)
    buf = (C.c_uint8 * 128)()
    st = lib().tac_nccl_unique_id(C.cast(buf, C.c_void_p))
    if st != 0:
        raise TacError(f"tac_nccl_unique_id failed ({st}): NCCL not loadable")
    return bytes(buf)


class NcclComm:
    """An NCCL communicator created through the C ABI (tac_nccl_comm_create); collective."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        assert len(uid) == 128
        import torch  # noqa: F401  (torch's libnccl.so.2, as in nccl_unique_id)
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        st = lib().tac_nccl_comm_create(C.cast(buf, C.c_void_p), nranks, rank, device, C.byref(h))
        if st != 0:
            raise TacError(f"tac_nccl_comm_create failed ({st})")
        self.handle, self.nranks, self.rank = h, nranks, rank

    def close(self):
        if self.handle:
            lib().tac_nccl_comm_destroy(self.handle)
            self.handle = None
