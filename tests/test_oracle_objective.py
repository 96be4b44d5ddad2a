"""Objective / optimiser / stepper checks of the CPU oracle.

The reference leaves these unpinned by tests (test_objective.cpp etc. are
empty stubs); this file reuses the reference's runtime audit instead
(check_derivatives, benchmark.cpp:54-159: FD gradient of the step objective)
plus the stepper invariants stated in stepper.hpp:47-64.
"""
import numpy as np
import pytest

import oracle
from paper_1709_04145_b200.scenes import (make_chain_scene, make_humanoid_scene, make_single_hinge_chain_scene,
                                          make_spider_scene, make_swimmer_scene, mt19937_uniform)
from paper_1709_04145_b200.types import ObjectiveKind, OptimizerConfig, OptimizerKind, SimConfig

from _ref_helpers import fd_gradient, fd_jacobian, rel_err


def _eval(m, f, order, dt, obj, h0, h1, x, want_gn=False):
    return oracle.step_eval(m, f, order, dt, obj, h0, h1, x, True, want_gn)


@pytest.mark.parametrize("scene", ["chain", "humanoid", "spider", "swimmer"])
def test_energy_objective_gradient_matches_fd(scene):
    rng = np.random.default_rng(1)
    sc = {"chain": lambda: make_chain_scene(4), "humanoid": make_humanoid_scene,
          "spider": lambda: make_spider_scene(oracle.rotation_vector_matrix), "swimmer": make_swimmer_scene}[scene]()
    m = oracle.Model(sc.links)
    n = m.n_dofs
    h0 = sc.q0 + rng.uniform(-0.05, 0.05, n)
    h1 = sc.q0 + rng.uniform(-0.05, 0.05, n)
    x = h1 + rng.uniform(-0.05, 0.05, n)
    f = sc.forces()
    v, g, gn = _eval(m, f, 2, 0.01, 0, h0, h1, x, want_gn=True)
    fd = fd_gradient(lambda y: oracle.step_eval(m, f, 2, 0.01, 0, h0, h1, y, False)[0], x, h=1e-6)
    assert rel_err(g, fd) < 1e-4 * max(1.0, np.max(np.abs(g))) / max(1.0, np.max(np.abs(g))) + 1e-4
    assert np.array_equal(gn, gn.T)
    # the GN matrix is the Hessian up to the dropped second-order potential terms
    assert np.linalg.eigvalsh(gn).min() > -1e-8 * np.linalg.norm(gn)


def test_value_equals_evaluate_value():
    sc = make_single_hinge_chain_scene(7)
    m = oracle.Model(sc.links)
    rng = np.random.default_rng(2)
    h0, h1, x = (rng.uniform(-0.3, 0.3, 7) for _ in range(3))
    v0 = oracle.step_eval(m, sc.forces(), 2, 0.02, 0, h0, h1, x, False)[0]
    v1 = oracle.step_eval(m, sc.forces(), 2, 0.02, 0, h0, h1, x, True)[0]
    assert v0 == v1


@pytest.mark.parametrize("order", [3, 4])
def test_residual_objective_gradient_and_gn(order):
    sc = make_single_hinge_chain_scene(4)
    m = oracle.Model(sc.links)
    rng = np.random.default_rng(order)
    n, u = 4, order - 1
    h0, h1 = rng.uniform(-0.2, 0.2, n), rng.uniform(-0.2, 0.2, n)
    x = np.tile(h1, u) + rng.uniform(-0.02, 0.02, n * u)
    f = sc.forces()
    v, g, gn = oracle.step_eval(m, f, order, 0.01, 1, h0, h1, x, True, True)
    fd = fd_gradient(lambda y: oracle.step_eval(m, f, order, 0.01, 1, h0, h1, y, False)[0], x, h=1e-7)
    assert rel_err(g, fd) < 1e-4
    assert np.array_equal(gn, gn.T)


def test_spd_solve_and_failure_rule():
    rng = np.random.default_rng(4)
    A = rng.normal(size=(6, 6))
    A = A @ A.T + 6 * np.eye(6)
    b = rng.normal(size=6)
    x = oracle.spd_solve(A, b)
    assert np.allclose(A @ x, b, atol=1e-12)
    assert oracle.spd_solve(-np.eye(3), np.ones(3)) is None


def _sims(sc, n, B, seed, dt, steps, kind, lo=-0.3, hi=0.3, **kw):
    out = []
    for b in range(B):
        s = SimConfig(dt=dt, duration=dt * steps, **kw)
        s.optimizer.kind = kind
        s.q0 = mt19937_uniform(seed + b, n, lo, hi) if hi > lo else sc.q0.copy()
        s.qdot0 = np.zeros(n)
        out.append(s)
    return out


def test_batch_equals_serial_simulate():
    """stepper.hpp:57-60: per-trajectory results identical to simulate()."""
    sc = make_single_hinge_chain_scene(8)
    m = oracle.Model(sc.links)
    sims = _sims(sc, 8, 4, 3, 0.02, 5, OptimizerKind.lbfgs)
    par = oracle.batch_simulate(m, sc.forces(), sims, workers=4)
    for s, p in zip(sims, par):
        ser = oracle.simulate(m, sc.forces(), s)
        assert np.array_equal(ser.q, p.q) and np.array_equal(ser.iterations, p.iterations)


def test_energy_log_and_samples_shape():
    sc = make_single_hinge_chain_scene(5)
    m = oracle.Model(sc.links)
    s = SimConfig(dt=0.01, duration=0.05, q0=np.zeros(5), qdot0=np.zeros(5))
    tr = oracle.simulate(m, sc.forces(), s)
    assert tr.n_samples == 6 and tr.error is None
    assert tr.times[5] == pytest.approx(0.05)
    assert tr.energy[0, 0] == 0.0  # at rest
    # released from rest: kinetic energy grows while the chain falls
    assert np.all(tr.energy[1:6, 0] > 0.0)
    assert np.all(np.diff(tr.energy[:6, 1]) < 0.0)


def test_fail_limit_error_text():
    sc = make_chain_scene(20)
    m = oracle.Model(sc.links)
    s = _sims(sc, 40, 1, 1, 0.1, 6, OptimizerKind.lbfgs, consecutive_fail_limit=1)[0]
    s.optimizer.max_iters = 3
    tr = oracle.simulate(m, sc.forces(), s)
    assert tr.error is not None and tr.error.startswith("optimizer failed 2 consecutive steps around t=")


def test_nonfinite_initial_state_is_reported():
    sc = make_single_hinge_chain_scene(3)
    m = oracle.Model(sc.links)
    s = SimConfig(dt=0.01, duration=0.02, q0=np.array([0.0, np.nan, 0.0]), qdot0=np.zeros(3))
    tr = oracle.batch_simulate(m, sc.forces(), [s])[0]
    assert tr.error == "configuration contains a non-finite entry"


def test_lm_converges_on_small_chain():
    sc = make_single_hinge_chain_scene(6)
    m = oracle.Model(sc.links)
    s = _sims(sc, 6, 1, 9, 0.01, 3, OptimizerKind.lm)[0]
    tr = oracle.simulate(m, sc.forces(), s)
    assert tr.error is None and tr.iterations[:3].max() < 60
