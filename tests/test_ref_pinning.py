"""Pins the C oracle to the reference itself: /root/reference/proj/src compiled
unmodified against oracle/eigen_lite (oracle/_ref/libpbad_ref.so).  Every
comparison is bit-exact (the oracle restates the reference under the same
numeric contract), which carries over to the CUDA path through
test_gpu_parity.py.  Skipped where oracle/_ref has not been built."""
import subprocess

import numpy as np
import pytest

import oracle
from paper_1709_04145_b200.scenes import (make_chain_scene, make_humanoid_scene, make_single_hinge_chain_scene,
                                          make_spider_scene, make_swimmer_scene, mt19937_uniform)
from paper_1709_04145_b200.types import ObjectiveKind, OptimizerKind, SimConfig

from _ref_helpers import random_tree

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def scenes():
    rng = np.random.default_rng(12)
    return {
        "single_hinge": make_single_hinge_chain_scene(7),
        "chain": make_chain_scene(5),
        "humanoid": make_humanoid_scene(),
        "spider": make_spider_scene(oracle.rotation_vector_matrix),
        "swimmer": make_swimmer_scene(),
        "random_tree": type("S", (), {"links": random_tree(rng, 8), "forces": lambda self: None})(),
    }


def test_reference_unit_tests_pass_on_the_shim():
    import os
    exe = os.path.join(os.path.dirname(oracle.REF_LIB_PATH), "pbad_ref_tests")
    if not os.path.exists(exe):
        pytest.skip("reference test binary not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout


@pytest.mark.parametrize("name", list(scenes().keys()))
def test_model_and_kinematics_bit_exact(name):
    sc = scenes()[name]
    R = oracle.RefModel(sc.links)
    O = oracle.Model(sc.links)
    ri, oi = R.info(), O.info()
    for k in ("S", "mass", "dof_offset", "axis", "sample_count"):
        assert np.array_equal(ri[k], oi[k]), k
    rng = np.random.default_rng(1)
    for _ in range(5):
        qa, qb = rng.uniform(-1, 1, O.n_dofs), rng.uniform(-1, 1, O.n_dofs)
        assert np.array_equal(oracle.ref_forward_pass(R, qa), oracle.forward_pass(O, qa))
        for a, b in zip(oracle.ref_correlation(R, qa, qb), oracle.correlation(O, qa, qb)):
            assert np.array_equal(np.asarray(a), np.asarray(b))


def test_collocation_bit_exact():
    for k in range(2, 8):
        a = oracle.ref_build_scheme(k, 0.01)
        b = oracle.build_scheme(k, 0.01)
        assert np.array_equal(a["times"], b["times"]) and np.array_equal(a["H2"], b["H2"])


@pytest.mark.parametrize("name", ["single_hinge", "chain", "humanoid", "spider", "swimmer"])
@pytest.mark.parametrize("order,objective", [(2, 0), (3, 1), (4, 1)])
def test_step_objective_bit_exact(name, order, objective):
    sc = scenes()[name]
    R, O = oracle.RefModel(sc.links), oracle.Model(sc.links)
    n = O.n_dofs
    u = order - 1
    rng = np.random.default_rng(order * 7 + objective)
    f = sc.forces()
    if name == "spider":
        f.drag_d = 0.7
    for _ in range(3):
        h0 = sc.q0 + rng.uniform(-0.1, 0.1, n)
        h1 = sc.q0 + rng.uniform(-0.1, 0.1, n)
        x = np.tile(h1, u) + rng.uniform(-0.05, 0.05, n * u)
        tau = rng.uniform(-1, 1, (u, n))
        for want_grad, want_gn in ((False, False), (True, False), (True, True)):
            a = oracle.ref_step_eval(R, f, order, 0.01, objective, h0, h1, x, want_grad, want_gn, tau)
            b = oracle.step_eval(O, f, order, 0.01, objective, h0, h1, x, want_grad, want_gn, tau)
            assert a[0] == b[0]
            if want_grad:
                assert np.array_equal(a[1], b[1])
            if want_gn:
                assert np.array_equal(a[2], b[2])


def _sims(n, B, seed, dt, steps, kind, q0=None, **kw):
    out = []
    for b in range(B):
        s = SimConfig(dt=dt, duration=dt * steps, **kw)
        s.optimizer.kind = kind
        s.q0 = mt19937_uniform(seed + b, n, -0.3, 0.3) if q0 is None else q0.copy()
        s.qdot0 = np.zeros(n)
        out.append(s)
    return out


@pytest.mark.parametrize("case", ["c1_lbfgs", "c1_lm", "c3_lbfgs", "humanoid_lm", "spider_lm", "swimmer_lm",
                                  "residual_k3", "fail_limit"])
def test_rollouts_bit_exact(case):
    if case == "c1_lbfgs":
        sc, sims = make_single_hinge_chain_scene(10), None
        sims = _sims(10, 2, 0, 0.01, 12, OptimizerKind.lbfgs)
    elif case == "c1_lm":
        sc = make_single_hinge_chain_scene(10)
        sims = _sims(10, 2, 0, 0.01, 12, OptimizerKind.lm)
    elif case == "c3_lbfgs":
        sc = make_chain_scene(100)
        sims = _sims(200, 1, 1, 0.1, 2, OptimizerKind.lbfgs)
    elif case == "humanoid_lm":
        sc = make_humanoid_scene()
        sims = _sims(41, 1, 2, 0.01, 5, OptimizerKind.lm, q0=sc.q0)
    elif case == "spider_lm":
        sc = make_spider_scene(oracle.rotation_vector_matrix)
        sims = _sims(22, 1, 0, 0.01, 5, OptimizerKind.lm, q0=sc.q0)
    elif case == "swimmer_lm":
        sc = make_swimmer_scene()
        sims = _sims(9, 1, 0, 0.05, 5, OptimizerKind.lm, q0=sc.q0)
    elif case == "residual_k3":
        sc = make_single_hinge_chain_scene(5)
        sims = _sims(5, 1, 4, 0.01, 3, OptimizerKind.lm, order=3, objective=ObjectiveKind.residual_form)
    else:
        sc = make_chain_scene(20)
        sims = _sims(40, 1, 1, 0.1, 6, OptimizerKind.lbfgs, consecutive_fail_limit=1)
        sims[0].optimizer.max_iters = 3
    R, O = oracle.RefModel(sc.links), oracle.Model(sc.links)
    ref = oracle.ref_batch_simulate(R, sc.forces(), sims, workers=2)
    ora = oracle.batch_simulate(O, sc.forces(), sims, workers=2)
    for r, o in zip(ref, ora):
        k = r.n_samples
        assert o.n_samples == k
        assert np.array_equal(r.q[:k], o.q[:k])
        assert np.array_equal(r.energy[:k], o.energy[:k])
        nrep = max(0, k - 1)
        assert np.array_equal(r.iterations[:nrep], o.iterations[:nrep])
        assert np.array_equal(r.converged[:nrep], o.converged[:nrep])
        assert np.array_equal(r.final_value[:nrep], o.final_value[:nrep])
        assert r.error == o.error
