"""Batched material calibration.

PAPER.md Sec. "Baseline IPC Calibration": theta = [E, nu, rho, mu], loss
Eq. 6 L(theta) = 1/(K N) sum_k sum_i |u_sim_{k,i}(theta) - u_real_{k,i}|^2 over K frames
and N indenter trajectories, theta* = argmin L (Eq. 7) by CMA-ES (Hansen 2006).  Sec.
"Results for Parameters Calibration": the four parameters are normalised to
[0, 1] over Table params_range, popsize 12, 80 iterations.

Host logic only: the CMA-ES update and the bookkeeping of which env evaluates which
candidate.  One generation = one batch of popsize x N envs in ONE TacSim per indenter
shape (the paper calibrates with several shapes): every simulation step, every
marker field and every loss term runs in libtac's kernels (tac_set_env_material,
tac_reset, tac_step, tac_marker_sqerr).
"""
from __future__ import annotations

import copy

import numpy as np

# Table params_range; rho's 1e-3..5e-3 is in g/mm^3 = 1e3..5e3 kg/m^3
THETA_LO = np.array([1e4, 0.4, 1e3, 0.25])
THETA_HI = np.array([2e5, 0.497, 5e3, 2.5])
THETA_NAMES = ("E", "nu", "rho", "mu_f")


def to_unit(theta):
    """theta -> [0, 1]^4 (P:485 normalisation)."""
    return (np.asarray(theta, dtype=np.float64) - THETA_LO) / (THETA_HI - THETA_LO)


def from_unit(x):
    return THETA_LO + np.clip(np.asarray(x, dtype=np.float64), 0.0, 1.0) * (THETA_HI - THETA_LO)


class CMAES:
    """(mu/mu_w, lambda)-CMA-ES with rank-one and rank-mu updates and cumulative step-size
    adaptation, default constants of Hansen's tutorial ("The CMA Evolution Strategy: A
    Tutorial", 2016, Table 1).  Box constraints by repair: candidates are clipped to
    [lo, hi] and the clipped points enter the update."""

    def __init__(self, x0, sigma0, popsize=12, seed=0, lo=0.0, hi=1.0):
        self.n = n = len(x0)
        self.lam = popsize
        self.mu = mu = popsize // 2
        w = np.log(mu + 0.5) - np.log(np.arange(1, mu + 1))
        self.w = w / w.sum()
        self.mueff = 1.0 / np.sum(self.w ** 2)
        self.cc = (4 + self.mueff / n) / (n + 4 + 2 * self.mueff / n)
        self.cs = (self.mueff + 2) / (n + self.mueff + 5)
        self.c1 = 2 / ((n + 1.3) ** 2 + self.mueff)
        self.cmu = min(1 - self.c1, 2 * (self.mueff - 2 + 1 / self.mueff) / ((n + 2) ** 2 + self.mueff))
        self.damps = 1 + 2 * max(0.0, np.sqrt((self.mueff - 1) / (n + 1)) - 1) + self.cs
        self.chiN = np.sqrt(n) * (1 - 1 / (4 * n) + 1 / (21 * n * n))
        self.m = np.array(x0, dtype=np.float64)
        self.sigma = float(sigma0)
        self.pc = np.zeros(n)
        self.ps = np.zeros(n)
        self.C = np.eye(n)
        self.B = np.eye(n)
        self.D = np.ones(n)
        self.invsqrtC = np.eye(n)
        self.lo, self.hi = lo, hi
        self.rng = np.random.default_rng(seed)
        self.gen = 0

    def ask(self):
        z = self.rng.standard_normal((self.lam, self.n))
        y = z @ (self.B * self.D).T
        return np.clip(self.m + self.sigma * y, self.lo, self.hi)

    def tell(self, X, f):
        X = np.asarray(X, dtype=np.float64)
        idx = np.argsort(np.asarray(f))
        Y = (X[idx[:self.mu]] - self.m) / self.sigma
        ymean = self.w @ Y
        self.m = self.m + self.sigma * ymean
        self.ps = (1 - self.cs) * self.ps + np.sqrt(self.cs * (2 - self.cs) * self.mueff) * (self.invsqrtC @ ymean)
        self.gen += 1
        hsig = (np.linalg.norm(self.ps) / np.sqrt(1 - (1 - self.cs) ** (2 * self.gen)) / self.chiN
                < 1.4 + 2 / (self.n + 1))
        self.pc = (1 - self.cc) * self.pc + hsig * np.sqrt(self.cc * (2 - self.cc) * self.mueff) * ymean
        rank_mu = (Y.T * self.w) @ Y
        self.C = ((1 - self.c1 - self.cmu) * self.C
                  + self.c1 * (np.outer(self.pc, self.pc) + (1 - hsig) * self.cc * (2 - self.cc) * self.C)
                  + self.cmu * rank_mu)
        self.sigma *= np.exp((self.cs / self.damps) * (np.linalg.norm(self.ps) / self.chiN - 1))
        self.C = np.triu(self.C) + np.triu(self.C, 1).T
        d2, self.B = np.linalg.eigh(self.C)
        self.D = np.sqrt(np.maximum(d2, 1e-30))
        self.invsqrtC = (self.B / self.D) @ self.B.T


class _Part:
    """One simulator of the calibration: one indenter shape, N trajectories x popsize."""

    def __init__(self, scene, popsize, device, ncomp):
        import torch
        from .tac import TacSim
        self.N = scene.n_envs
        self.K = len(scene.poses)
        self.P = popsize
        self.dt = scene.dt
        big = copy.copy(scene)
        big.init_poses = np.tile(scene.init_poses, (popsize, 1))
        big.poses = np.tile(scene.poses, (1, popsize, 1))
        self.sim = TacSim.from_scene(big, device=device)
        dev = f"cuda:{device}"
        self.poses = torch.tensor(big.poses, dtype=torch.float32, device=dev).contiguous()
        self.init = torch.tensor(big.init_poses, dtype=torch.float32, device=dev).contiguous()
        self.mask = torch.ones(popsize * self.N, dtype=torch.uint8, device=dev)
        self.acc = torch.zeros(popsize * self.N, dtype=torch.float64, device=dev)
        self.ref = None
        self.ncomp = ncomp

    def set_thetas(self, thetas):
        th = np.repeat(np.asarray(thetas, dtype=np.float64).reshape(-1, 4), self.N, axis=0)
        self.sim.set_env_material(E=th[:, 0], nu=th[:, 1], rho=th[:, 2], mu_f=th[:, 3])


class Calibrator:
    """Evaluates Eq. 6 for a whole CMA-ES population in one batch per indenter shape.

    `scenes`: one scene or a list (one per indenter shape); each holds N
    trajectories (scene.n_envs = N, poses [K][N][7]) and gets its own simulator with
    popsize x N envs, env j*N + i = candidate j on trajectory i.  L(theta) is the mean of
    |u_sim - u_ref|^2 over all frames of all trajectories of all shapes (Eq. 6)."""

    def __init__(self, scenes, popsize=12, device=0, ncomp=2):
        import torch
        self.torch = torch
        self.dev = f"cuda:{device}"
        self.P = popsize
        scenes = scenes if isinstance(scenes, (list, tuple)) else [scenes]
        self.parts = [_Part(sc, popsize, device, ncomp) for sc in scenes]
        self.evals = 0
        # single-shape conveniences (tests, examples)
        self.N, self.K, self.sim = self.parts[0].N, self.parts[0].K, self.parts[0].sim

    @property
    def ref(self):
        return self.parts[0].ref

    def fields(self, theta):
        """Marker fields of every shape at one theta: [K][N][nm][ncomp] per shape (a list
        for several shapes) -- e.g. the synthetic 'real' reference at a hidden theta_true."""
        out = []
        for pt in self.parts:
            pt.set_thetas(np.tile(np.asarray(theta, dtype=np.float64), (self.P, 1)))
            pt.sim.reset(pt.mask, pt.init)
            fr = []
            for k in range(pt.K):
                pt.sim.step(pt.poses[k], pt.dt)
                fr.append(pt.sim.markers(ncomp=pt.ncomp)[:pt.N].clone())
            out.append(self.torch.stack(fr))
        return out if len(out) > 1 else out[0]

    def set_reference(self, ref):
        """ref: [K][N][nm][ncomp] per shape (a list for several shapes), tiled over the population."""
        refs = ref if isinstance(ref, (list, tuple)) else [ref]
        assert len(refs) == len(self.parts)
        for pt, r in zip(self.parts, refs):
            r = self.torch.as_tensor(r, dtype=self.torch.float32, device=self.dev)
            pt.ref = r.repeat(1, self.P, 1, 1).contiguous()

    def losses(self, thetas):
        """Eq. 6 for each of the popsize candidate thetas ([P][4], physical units)."""
        total = None
        count = 0
        for pt in self.parts:
            assert pt.ref is not None, "set_reference first"
            pt.set_thetas(thetas)
            pt.sim.reset(pt.mask, pt.init)
            pt.acc.zero_()
            for k in range(pt.K):
                pt.sim.step(pt.poses[k], pt.dt)
                pt.sim.marker_sqerr(pt.ref[k], pt.acc)
            part = pt.acc.view(self.P, pt.N).sum(dim=1)
            total = part if total is None else total + part
            count += pt.K * pt.N
        self.evals += self.P
        return (total / count).cpu().numpy()

    def run(self, iters=80, x0=None, sigma0=0.25, seed=0, callback=None):
        """CMA-ES over the normalised theta: popsize = self.P, `iters` generations."""
        es = CMAES(np.full(4, 0.5) if x0 is None else to_unit(x0), sigma0, popsize=self.P, seed=seed)
        best_x, best_f, hist = None, np.inf, []
        for g in range(iters):
            X = es.ask()
            f = self.losses(from_unit(X))
            es.tell(X, f)
            j = int(np.argmin(f))
            if f[j] < best_f:
                best_f, best_x = float(f[j]), X[j].copy()
            hist.append(float(np.min(f)))
            if callback:
                callback(g, es, f)
        return dict(theta=from_unit(best_x), loss=best_f, history=np.array(hist), mean=from_unit(es.m),
                    sigma=es.sigma, evals=self.evals)
