"""Host logic of the batched material calibration (Eqs. 6-7,
P:485): parameter normalisation and the CMA-ES update, pinned on functions with known
minimisers.  The GPU calibration itself is in test_gpu_calib.py."""
import numpy as np
import pytest

from paper_2603_28475_b200.calib import CMAES, THETA_HI, THETA_LO, from_unit, to_unit


def test_unit_roundtrip_and_table_bounds():
    # Table params_range: E 1e4..2e5, nu 0.4..0.497, rho 1e-3..5e-3 g/mm^3, mu 0.25..2.5
    assert np.allclose(THETA_LO, [1e4, 0.4, 1e3, 0.25]) and np.allclose(THETA_HI, [2e5, 0.497, 5e3, 2.5])
    th = np.array([6e4, 0.46, 2.0e3, 0.8])
    assert np.allclose(from_unit(to_unit(th)), th, rtol=1e-14)
    assert np.allclose(from_unit([0, 0, 0, 0]), THETA_LO) and np.allclose(from_unit([1, 1, 1, 1]), THETA_HI)
    assert np.allclose(from_unit([-1, 2, 0.5, 0.5])[:2], [THETA_LO[0], THETA_HI[1]])  # clipped to the box


def _run(f, x0, sigma0, gens, seed=0, popsize=12):
    es = CMAES(x0, sigma0, popsize=popsize, seed=seed)
    best = (np.inf, None)
    for _ in range(gens):
        X = es.ask()
        assert X.shape == (popsize, len(x0)) and np.all((X >= 0) & (X <= 1))
        fx = np.array([f(x) for x in X])
        es.tell(X, fx)
        j = int(np.argmin(fx))
        if fx[j] < best[0]:
            best = (fx[j], X[j].copy())
    return best, es


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_cmaes_sphere_in_the_unit_box(seed):
    """popsize 12, 80 generations on a 4-d sphere: the minimiser to 1e-4."""
    xs = np.random.default_rng(100 + seed).uniform(0.15, 0.85, 4)
    (fb, xb), es = _run(lambda x: float(np.sum((x - xs) ** 2)), np.full(4, 0.5), 0.25, 80, seed)
    assert np.abs(xb - xs).max() < 1e-4
    assert fb < 1e-8


def test_cmaes_learns_an_ill_conditioned_metric():
    """Ellipsoid with axis scales 1..1e3 (condition 1e6): covariance adaptation must
    align C with the metric; the minimiser to 1e-3 within 150 generations."""
    xs = np.array([0.3, 0.6, 0.45, 0.7])
    sc = 10.0 ** np.linspace(0, 3, 4)
    (fb, xb), es = _run(lambda x: float(np.sum((sc * (x - xs)) ** 2)), np.full(4, 0.5), 0.3, 150)
    assert np.abs(xb - xs).max() < 1e-3
    ev = np.linalg.eigvalsh(es.C)
    assert ev.max() / ev.min() > 1e3  # learned anisotropy


def test_cmaes_minimiser_on_the_box_boundary():
    """Minimiser outside [0, 1]^4: the repaired (clipped) search ends on the face."""
    xs = np.array([1.4, 0.5, -0.3, 0.2])
    (fb, xb), _ = _run(lambda x: float(np.sum((x - xs) ** 2)), np.full(4, 0.5), 0.25, 80)
    assert np.allclose(xb, np.clip(xs, 0, 1), atol=1e-3)
