"""Parity at BASELINE.json's full batch sizes.

The bench configurations (bench.py CONFIGS: C3 4096 x 200-DOF chains, C4 /
C4b 4096 humanoids, C5 256 x U=300 collocation windows) run on the GPU at
their full batch; a deterministic sample of environments is replayed on the
CPU oracle (bit-exact), and size-independent properties are checked on the
whole batch: run-to-run determinism, batch-composition invariance (an
environment's trajectory does not depend on its neighbours), and finiteness.
"""
import numpy as np
import pytest

import bench
import oracle
from paper_1709_04145_b200 import api

from _parity_util import assert_traj_equal

pytestmark = pytest.mark.gpu


def _setup(name, steps, max_iters=None):
    cfg = bench.CONFIGS[name]
    scene = bench.build_scene(cfg)
    model = api.build_model(scene.links)
    n = model.total_dofs
    sim = bench.sim_config(cfg, steps, 1 << 30)
    if max_iters is not None:
        sim.optimizer.max_iters = max_iters
    q0 = bench.initial_states(cfg, scene, n, 0, cfg["batch"])
    return cfg, scene, model, n, sim, q0


def _rollout(model, scene, sim, q0):
    B, n = q0.shape
    ctx = api.GpuContext(model, scene.forces(), sim, max_batch=B)
    return ctx.rollout(q0, np.zeros((B, n)), want_q=True, want_energy=True), ctx.path


def _oracle_env(scene, sim, q0_row):
    s = type(sim)(**{**sim.__dict__})
    s.q0 = q0_row.copy()
    s.qdot0 = np.zeros_like(q0_row)
    return oracle.batch_simulate(oracle.Model(scene.links), scene.forces(), [s], workers=1)[0]


def _check_sample(out, scene, sim, q0, envs):
    for b in envs:
        ref = _oracle_env(scene, sim, q0[b])
        k = ref.n_samples
        np.testing.assert_array_equal(out["q"][b, :k], ref.q[:k])
        np.testing.assert_array_equal(out["energy"][b, :k], ref.energy[:k])
        nrep = len(ref.iterations)
        np.testing.assert_array_equal(out["iterations"][b, :nrep], ref.iterations[:nrep])


@pytest.mark.parametrize("name,steps,max_iters,expect_path", [
    ("C3", 1, None, 6),
    ("C4", 2, None, 3),
    ("C4b", 2, None, 3),
    ("C5", 1, 6, 4),
])
def test_full_batch_sample_matches_oracle_and_is_deterministic(name, steps, max_iters, expect_path):
    cfg, scene, model, n, sim, q0 = _setup(name, steps, max_iters)
    out1, path = _rollout(model, scene, sim, q0)
    assert path == expect_path
    B = q0.shape[0]
    assert np.all(np.isfinite(out1["q"]))
    # run-to-run determinism over the whole batch
    out2, _ = _rollout(model, scene, sim, q0)
    np.testing.assert_array_equal(out1["q"], out2["q"])
    np.testing.assert_array_equal(out1["iterations"], out2["iterations"])
    # first, last and a spread of environments replayed on the CPU oracle
    envs = sorted(set([0, 1, B // 3, B // 2, B - 2, B - 1]))
    _check_sample(out1, scene, sim, q0, envs)


@pytest.mark.parametrize("name,steps,max_iters", [("C3", 1, None), ("C4", 2, None), ("C5", 1, 6)])
def test_batch_composition_invariance(name, steps, max_iters):
    """An environment's trajectory is independent of the rest of the batch:
    the full batch reversed gives the reversed results bit for bit."""
    cfg, scene, model, n, sim, q0 = _setup(name, steps, max_iters)
    out, _ = _rollout(model, scene, sim, q0)
    rev, _ = _rollout(model, scene, sim, np.ascontiguousarray(q0[::-1]))
    np.testing.assert_array_equal(out["q"], rev["q"][::-1])
    np.testing.assert_array_equal(out["iterations"], rev["iterations"][::-1])
