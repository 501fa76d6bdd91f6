"""ctypes wrapper of the fp64 CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product path
(paper_2603_28475_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.cpp")
LIB = os.path.join(HERE, "liboracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def build(force=False):
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC", SRC,
                               "-o", LIB, "-lpthread"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.or_create.restype = C.c_void_p
        L.or_create.argtypes = [C.c_int, _dp, C.c_int, _ip, C.c_int, _ip, C.c_int, _dp, C.c_int, _ip, C.c_int, _dp,
                                _dp, _dp, _dp, _ip, C.c_int, _dp, _ip]
        L.or_destroy.argtypes = [C.c_void_p]
        L.or_kappa_phys.restype = C.c_double
        L.or_kappa_phys.argtypes = [C.c_void_p]
        L.or_counts.argtypes = [C.c_void_p, _ip]
        L.or_surface.argtypes = [C.c_void_p, _ip, _ip, _ip, _ip]
        L.or_mass_vol.argtypes = [C.c_void_p, _dp, _dp]
        L.or_marker_map.argtypes = [C.c_void_p, _ip, _ip, _dp]
        L.or_step.argtypes = [C.c_void_p, _dp, C.c_double, C.c_int, C.c_int, C.c_int]
        L.or_env_status.argtypes = [C.c_void_p, C.c_int, _dp]
        L.or_get_state.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp]
        L.or_set_state.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp]
        L.or_set_trace.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.or_trace.restype = C.c_int
        L.or_trace.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int]
        L.or_markers.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.or_set_eval_lambda.argtypes = [C.c_void_p, _dp]
        L.or_get_lambda.argtypes = [C.c_void_p, C.c_int, _dp]
        L.or_eval.restype = C.c_double
        L.or_eval.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_double, _dp, _dp, _dp, _dp, _dp,
                              _ip, _ip]
        L.or_curvature.restype = C.c_double
        L.or_curvature.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_double]
        L.or_iteration.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_double, _dp, _dp,
                                   C.c_double, C.c_int, _dp, _dp]
        L.or_alpha_ccd.restype = C.c_double
        L.or_alpha_ccd.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp]
        L.or_broadphase_body.restype = C.c_int
        L.or_broadphase_body.argtypes = [C.c_void_p, _dp, C.c_double, _ip, C.c_int]
        L.or_broadphase_state.restype = C.c_int
        L.or_broadphase_state.argtypes = [C.c_void_p, _dp, _dp, _dp, C.c_double, _ip, C.c_int]
        L.or_dmin.restype = C.c_double
        L.or_dmin.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.or_barrier.restype = C.c_double
        L.or_barrier.argtypes = [C.c_double, C.c_double, C.c_int]
        L.or_mollifier.restype = C.c_double
        L.or_mollifier.argtypes = [C.c_double, C.c_double, C.c_int]
        L.or_dist_pt.restype = C.c_double
        L.or_dist_pt.argtypes = [_dp, _dp, _dp, _dp, _dp]
        L.or_dist_ee.restype = C.c_double
        L.or_dist_ee.argtypes = [_dp, _dp, _dp, _dp, _dp]
        L.or_step_from.argtypes = [C.c_void_p, C.c_int, _dp, C.c_double, _dp, _dp, _dp]
        L.or_set_pose_noise.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_uint64, C.c_int64]
        L.or_philox.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.or_certificate.restype = C.c_int
        L.or_certificate.argtypes = [_dp, C.c_int, C.c_double, _dp, _dp]
        L.or_psi.restype = C.c_double
        L.or_psi.argtypes = [C.c_double, C.c_double, _dp]
        L.or_so3.argtypes = [_dp, _dp, _dp]
        L.or_quat_to_R.argtypes = [_dp, _dp]
        L.or_ncg_quadratic.argtypes = [C.c_int, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int, _dp]
    return _lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(_ip)


# --- scalar pins --------------------------------------------------------------
def barrier(d, dhat, deriv=0):
    return lib().or_barrier(float(d), float(dhat), deriv)


def mollifier(s, eps, deriv=0):
    return lib().or_mollifier(float(s), float(eps), deriv)


def dist_pt(p, t0, t1, t2):
    w = np.zeros(4)
    args = [_d(x) for x in (p, t0, t1, t2)]
    d = lib().or_dist_pt(*[a[1] for a in args], w.ctypes.data_as(_dp))
    return d, w


def dist_ee(a0, a1, b0, b1):
    w = np.zeros(4)
    args = [_d(x) for x in (a0, a1, b0, b1)]
    d = lib().or_dist_ee(*[a[1] for a in args], w.ctypes.data_as(_dp))
    return d, w


def philox4x32_10(ctr, key):
    """Philox4x32-10 block (the pose-noise generator, R27): 4 uint32 counter, 2 uint32 key."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    P32 = C.POINTER(C.c_uint32)
    lib().or_philox(c.ctypes.data_as(P32), k.ctypes.data_as(P32), o.ctypes.data_as(P32))
    return o


def certificate(z, na, dhat):
    """R15 far-pair certificate on corners z[4][3] (side A = first na): (ok, g, n)."""
    z, zp = _d(np.asarray(z).reshape(12))
    g = np.zeros(1)
    n = np.zeros(3)
    ok = lib().or_certificate(zp, int(na), float(dhat), g.ctypes.data_as(_dp), n.ctypes.data_as(_dp))
    return bool(ok), float(g[0]), n


def psi(E, nu, F):
    F, Fp = _d(np.asarray(F).reshape(9))
    return lib().or_psi(E, nu, Fp)


def so3_exp_log(w):
    w, wp = _d(w)
    R = np.zeros(9)
    l = np.zeros(3)
    lib().or_so3(wp, R.ctypes.data_as(_dp), l.ctypes.data_as(_dp))
    return R.reshape(3, 3), l


def quat_to_R(pose7):
    p, pp = _d(pose7)
    R = np.zeros(9)
    lib().or_quat_to_R(pp, R.ctypes.data_as(_dp))
    return R.reshape(3, 3)


def ncg_quadratic(A, b, x0, iters, precond_identity=False, rule=0):
    n = len(b)
    A, Ap = _d(A)
    b, bp = _d(b)
    x0, xp = _d(x0)
    xs = np.zeros((iters + 1, n))
    lib().or_ncg_quadratic(n, Ap, bp, xp, iters, int(precond_identity), rule, xs.ctypes.data_as(_dp))
    return xs


# --- the oracle solver ----------------------------------------------------------
TRACE_FIELDS = ["it", "E", "accepted", "alpha", "alpha_upper", "alpha_bar", "alpha_ccd", "M", "pg", "gp", "pHp",
                "rebuilt", "dmin", "n_cand", "n_anchor", "beta"]


class Oracle:
    """fp64 oracle over a workloads.Scene (all envs)."""

    def __init__(self, scene, params=None, material=None, marker_mode=0, knn_k=4, debug=False, init_poses=None):
        L = lib()
        p = params or scene.params
        m = material or scene.material
        self.scene = scene
        self.params = p
        self.nv = scene.X.shape[0]
        self._keep = []
        X, Xp = _d(scene.X)
        T, Tp = _i(scene.tets)
        F, Fp = _i(scene.fixed)
        Y, Yp = _d(scene.Y)
        tr, trp = _i(scene.tris)
        M, Mp = _d(scene.markers)
        fr, frp = _d(scene.frame)
        mat, matp = _d([m.E, m.nu, m.rho, m.mu_f])
        dp, dpp = _d([p.dhat, p.kappa_phys, p.eps_v, p.tol_x, p.k_t, p.k_r, p.ccd_s, p.bp_margin, p.c1, p.f_max,
                      p.t_max])
        ip, ipp = _i([p.max_iters, p.fixed_iters, p.beta_rule, p.precond, p.max_halvings, p.stagnation, marker_mode,
                      knn_k, int(debug), int(getattr(p, "pose_al", 0)), int(getattr(p, "ee_mollifier", 0)),
                      int(getattr(p, "dedup", 0))])
        init = scene.init_poses if init_poses is None else init_poses
        self.n_envs = init.shape[0]
        ini, inip = _d(init)
        st = C.c_int(0)
        self.h = L.or_create(self.nv, Xp, len(scene.tets), Tp, len(scene.fixed), Fp, len(scene.Y), Yp, len(scene.tris),
                             trp, len(scene.markers), Mp, frp, matp, dpp, ipp, self.n_envs, inip, C.byref(st))
        self.status = st.value
        self.nm = len(scene.markers)

    def __del__(self):
        try:
            lib().or_destroy(self.h)
        except Exception:
            pass

    @property
    def kappa_phys(self):
        return lib().or_kappa_phys(self.h)

    def surface(self):
        c = np.zeros(4, np.int32)
        lib().or_counts(self.h, c.ctypes.data_as(_ip))
        sv = np.zeros(c[0], np.int32)
        se = np.zeros((c[1], 2), np.int32)
        st = np.zeros((c[2], 3), np.int32)
        ie = np.zeros((c[3], 2), np.int32)
        lib().or_surface(self.h, *(a.ctypes.data_as(_ip) for a in (sv, se, st, ie)))
        return sv, se, st, ie

    def mass_vol(self):
        m = np.zeros(self.nv)
        v = np.zeros(len(self.scene.tets))
        lib().or_mass_vol(self.h, m.ctypes.data_as(_dp), v.ctypes.data_as(_dp))
        return m, v

    def marker_map(self):
        t = np.zeros(self.nm, np.int32)
        idx = np.zeros((self.nm, 4), np.int32)
        w = np.zeros((self.nm, 4))
        lib().or_marker_map(self.h, t.ctypes.data_as(_ip), idx.ctypes.data_as(_ip), w.ctypes.data_as(_dp))
        return t, idx, w

    def step(self, targets, dt=None, threads=1, env0=0, n=0):
        targets, tp = _d(targets)
        lib().or_step(self.h, tp, float(self.scene.dt if dt is None else dt), threads, env0, n)

    def step_from(self, env, target7, u0, c0, R0, dt=None):
        """Env `env`'s step to target7 from its stored x^t, started at the feasible iterate
        (u0, c0, R0) instead of x^t (anchors from x^t).  Test hook: polish another solver's
        result -- a local minimiser of the step's potential stays where it is."""
        ins = [_d(a) for a in (target7, u0, c0, np.asarray(R0).reshape(9))]
        lib().or_step_from(self.h, int(env), ins[0][1], float(self.scene.dt if dt is None else dt), ins[1][1],
                           ins[2][1], ins[3][1])

    def set_pose_noise(self, sigma_t, sigma_r, seed, env_offset=0):
        """Per-step target-pose noise (R27); one step() call = one step of the envs it covers."""
        lib().or_set_pose_noise(self.h, float(sigma_t), float(sigma_r), int(seed), int(env_offset))

    def status_of(self, env):
        o = np.zeros(5)
        lib().or_env_status(self.h, env, o.ctypes.data_as(_dp))
        return dict(iters=int(o[0]), flags=int(o[1]), pg=o[2], dmin=o[3], pose_res=o[4])

    def get_state(self, env):
        u = np.zeros((self.nv, 3))
        v = np.zeros((self.nv, 3))
        c = np.zeros(3)
        R = np.zeros(9)
        lib().or_get_state(self.h, env, *(a.ctypes.data_as(_dp) for a in (u, v, c, R)))
        return u, v, c, R.reshape(3, 3)

    def set_state(self, env, u, v, c, R):
        arrs = [_d(a) for a in (u, v, c, np.asarray(R).reshape(9))]
        lib().or_set_state(self.h, env, *(a[1] for a in arrs))

    def set_trace(self, env, on=True):
        lib().or_set_trace(self.h, env, int(on))

    def trace(self, env):
        n = lib().or_trace(self.h, env, None, 0)
        out = np.zeros((n, 16))
        lib().or_trace(self.h, env, out.ctypes.data_as(_dp), n)
        return out

    def markers(self, env, ncomp=2):
        out = np.zeros((self.nm, ncomp))
        lib().or_markers(self.h, env, ncomp, out.ctypes.data_as(_dp))
        return out

    def set_eval_lambda(self, lam6):
        """Pose multipliers (lam_t, lam_r) that eval() uses (augmented Lagrangian, R29)."""
        a = np.ascontiguousarray(lam6, dtype=np.float64)
        lib().or_set_eval_lambda(self.h, a.ctypes.data_as(_dp))

    def lambda_of(self, env):
        """Env's current pose multipliers [lam_t (N), lam_r (N m)] after its last step."""
        out = np.zeros(6)
        lib().or_get_lambda(self.h, env, out.ctypes.data_as(_dp))
        return out

    def eval(self, u_t, v_t, c_t, R_t, u, c, R, target7, dt=None):
        dt = self.scene.dt if dt is None else dt
        ins = [_d(a) for a in (u_t, v_t, c_t, np.asarray(R_t).reshape(9), u, c, np.asarray(R).reshape(9), target7)]
        parts = np.zeros(5)
        g = np.zeros((self.nv, 3))
        D = np.zeros((self.nv, 3, 3))
        gr = np.zeros(6)
        Dr = np.zeros((2, 3, 3))
        nc = C.c_int(0)
        na = C.c_int(0)
        E = lib().or_eval(self.h, *(a[1] for a in ins), dt, *(a.ctypes.data_as(_dp) for a in (parts, g, D, gr, Dr)),
                          C.byref(nc), C.byref(na))
        return dict(E=E, parts=parts, g=g, D=D, grig=gr, Drig=Dr, n_cand=nc.value, n_anchor=na.value)

    def curvature(self, u_t, c_t, R_t, u, c, R, p, prig, target7, dt=None):
        dt = self.scene.dt if dt is None else dt
        ins = [_d(a) for a in (u_t, c_t, np.asarray(R_t).reshape(9), u, c, np.asarray(R).reshape(9), p, prig, target7)]
        return lib().or_curvature(self.h, *(a[1] for a in ins), dt)

    ITERATION_FIELDS = ["beta", "gp", "gPg", "restarted", "M", "alpha_upper", "pHp", "alpha_bar", "alpha_ccd",
                        "alpha", "L_rel", "pg_disp"]

    def iteration(self, u_t, v_t, c_t, R_t, u, c, R, target7, g_prev, p_prev, gPg_prev, restart=False, dt=None):
        """One PNCG iteration's a6-a8 quantities at x_k (O4b, O4d-O4f): the direction from the
        previous gradient / direction ([nv*3 + 6] each, gel then c, theta) and the step length.
        Returns (p [nv*3 + 6], dict of ITERATION_FIELDS)."""
        dt = self.scene.dt if dt is None else dt
        ins = [_d(a) for a in (u_t, v_t, c_t, np.asarray(R_t).reshape(9), u, c, np.asarray(R).reshape(9), target7,
                                g_prev, p_prev)]
        p = np.zeros(3 * self.nv + 6)
        out = np.zeros(12)
        lib().or_iteration(self.h, *(a[1] for a in ins[:8]), dt, ins[8][1], ins[9][1], float(gPg_prev), int(restart),
                           p.ctypes.data_as(_dp), out.ctypes.data_as(_dp))
        return p, dict(zip(self.ITERATION_FIELDS, out))

    def alpha_ccd(self, u, c, R, p, prig):
        ins = [_d(a) for a in (u, c, np.asarray(R).reshape(9), p, prig)]
        return lib().or_alpha_ccd(self.h, *(a[1] for a in ins))

    def broadphase_body(self, gb, r):
        """Candidates for gel vertices given in the indenter body frame gb [nv, 3]."""
        gb, gp = _d(gb)
        n = lib().or_broadphase_body(self.h, gp, r, None, 0)
        out = np.zeros((n, 3), np.int32)
        lib().or_broadphase_body(self.h, gp, r, out.ctypes.data_as(_ip), n)
        return out

    def broadphase_state(self, u, c, R, r):
        ins = [_d(a) for a in (u, c, np.asarray(R).reshape(9))]
        n = lib().or_broadphase_state(self.h, *(a[1] for a in ins), r, None, 0)
        out = np.zeros((n, 3), np.int32)
        lib().or_broadphase_state(self.h, *(a[1] for a in ins), r, out.ctypes.data_as(_ip), n)
        return out

    def dmin(self, u, c, R):
        ins = [_d(a) for a in (u, c, np.asarray(R).reshape(9))]
        return lib().or_dmin(self.h, *(a[1] for a in ins))
