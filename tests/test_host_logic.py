"""Host-side logic of the drop-in (no GPU): config validation, update
coefficients, the public stopping-rule utility (solvers.py:34-99, 174-192)."""

import math

import numpy as np
import pytest

from paper_2311_04362_b200 import SolverConfig, damping_params, momentum_params, should_stop
from paper_2311_04362_b200.solvers import update_coeffs


def test_validate_messages_match_reference():
    with pytest.raises(ValueError, match="must be >= n"):
        SolverConfig(d=5).validate(10)
    with pytest.raises(ValueError, match="unknown variant"):
        SolverConfig(d=50, variant="bogus").validate(10)
    with pytest.raises(ValueError, match="unknown init"):
        SolverConfig(d=50, init="x").validate(10)
    with pytest.raises(ValueError):
        SolverConfig(d=50, zeta=0).validate(10)
    with pytest.raises(ValueError):
        SolverConfig(d=50, max_iters=-1).validate(10)
    with pytest.raises(ValueError):
        SolverConfig(d=50, unit_roundoff=1.0).validate(10)


def test_defaults_identical_to_reference():
    c = SolverConfig(d=10)
    assert (c.zeta, c.variant, c.init, c.max_iters, c.unit_roundoff, c.stop_gamma, c.stop_rho,
            c.epsilon_for_params, c.rng_seed, c.extra_iters, c.track_be) == (
        8, "basic", "sketch_and_solve", 50, 2.0**-53, 1.0, 0.04, None, 0, 0, False)


def test_update_coeffs_values():
    assert update_coeffs(SolverConfig(d=4000), 200) == (1.0, 0.0)
    a, b = update_coeffs(SolverConfig(d=4000, variant="damped"), 200)
    assert a == pytest.approx(0.859524, abs=1e-6) and b == 0.0
    a, b = update_coeffs(SolverConfig(d=4000, variant="momentum"), 200)
    assert a == pytest.approx(0.9025) and b == pytest.approx(0.05)
    a, b = update_coeffs(SolverConfig(d=24000, variant="momentum"), 2000)
    assert a == pytest.approx(0.840278, abs=1e-6) and b == pytest.approx(1 / 12)
    with pytest.raises(ValueError):
        update_coeffs(SolverConfig(d=10, variant="damped", epsilon_for_params=1.0), 5)


def test_param_formulas():
    assert damping_params(0.0) == (1.0, 0.0)
    assert damping_params(0.5)[0] == pytest.approx(0.45)
    assert momentum_params(0.5) == (pytest.approx(0.5625), pytest.approx(0.25))
    grid = np.linspace(0.0, 0.9, 91)
    assert np.all(np.diff([damping_params(e)[0] for e in grid]) < 0)
    # test_solvers.py:59-71: momentum at 0, beta < 1 on [0, 1), the domain errors
    assert momentum_params(0.0) == (1.0, 0.0) and damping_params(0.5)[1] == 0.0
    assert all(momentum_params(e)[1] < 1.0 for e in np.linspace(0.0, 0.999, 50))
    for fn in (damping_params, momentum_params):
        with pytest.raises(ValueError):
            fn(1.0)
        with pytest.raises(ValueError):
            fn(-0.1)


def test_should_stop_inclusive_boundary():
    r_next, r_curr, x = np.array([1.0, 0.0]), np.array([0.0, 0.0]), np.array([1.0, 0.0])
    assert should_stop(r_next, r_curr, x, 1.0, 25.0, 0.5, gamma=1.0, rho=0.04)
    assert not should_stop(np.array([1.0, 0.0]), np.zeros(2), np.ones(2), 1.0, 1.0, 1e-16)
    r = np.array([1.0, 2.0])
    assert should_stop(r, r, np.ones(2), 1.0, 1.0, 1e-16)


def test_gen_randsvd_matches_oracle_bitwise():
    from oracle import itsketch_oracle as orc
    from paper_2311_04362_b200 import gen_randsvd

    p = gen_randsvd(300, 7, 1e6, 1e-4, 5)
    a, b, t = orc.gen_randsvd(300, 7, 1e6, 1e-4, 5)
    assert np.array_equal(p.a, a) and np.array_equal(p.b, b) and np.array_equal(p.truth.x, t.x)
    assert math.isclose(np.linalg.norm(p.truth.r), 1e-4, rel_tol=1e-12)


def test_qrfactors_q_without_vectors_raises_clearly():
    """A QrFactors built by hand (no Householder vectors behind it) cannot
    form Q: reading .q says so instead of returning None;
    householder_qr_econ's result forms Q on request (tests/test_gpu_parity.py)."""
    import pytest

    from paper_2311_04362_b200.linalg import QrFactors

    f = QrFactors(r=np.eye(2), z=np.zeros(2))
    with pytest.raises(AttributeError, match="without the Householder vectors"):
        f.q
    assert not hasattr(f, "q")
