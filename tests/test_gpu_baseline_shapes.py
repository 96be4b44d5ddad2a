"""Parity at the shapes BASELINE.json quotes its configurations on.

Each case runs the bench configuration (bench.py CONFIGS) on the GPU at its
full per-GPU batch and for the step count BASELINE.json names, then replays
environments of that batch on the CPU checker and requires every sample,
energy-log entry, per-step iteration count, accepted count, convergence flag
and final objective value to be bit-identical:

* C1  10-link chain, L-BFGS, dt 0.01, 1000 steps (1024 replicas); both with
  the reference's default fail limit (the trajectory aborts with the
  reference's error text) and unbounded (all 1000 steps, divergence curve);
* C2  1024 x 50-link chains, 100 steps;
* C3  4096 x 200-DOF chains, dt 0.1, 50 steps (512 L-BFGS iterations every step);
* C4 / C4b  4096 humanoids, LM, 100 steps;
* C5  256 x U = 300 collocation windows at the reference's max_iters = 512
  (every step runs all 512 LM iterations).

The checker is the reference itself (oracle/_ref: /root/reference/proj/src
compiled unmodified) where it replays in seconds, else the C restatement
pinned to it bit for bit (tests/test_ref_pinning.py).  Set
PBAD_DIVERGENCE_OUT=<file> to write the per-step divergence curves as JSON.
"""
import json
import os

import numpy as np
import pytest

import bench
import oracle
from paper_1709_04145_b200 import api

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

_CURVES = {}


def _sim(cfg, steps, fail_limit, max_iters=None):
    sim = bench.sim_config(cfg, steps, fail_limit)
    if max_iters is not None:
        sim.optimizer.max_iters = max_iters
    return sim


def _gpu(name, steps, fail_limit, max_iters=None):
    cfg = bench.CONFIGS[name]
    scene = bench.build_scene(cfg)
    model = api.build_model(scene.links)
    n = model.total_dofs
    q0 = bench.initial_states(cfg, scene, n, 0, cfg["batch"])
    sim = _sim(cfg, steps, fail_limit, max_iters)
    ctx = api.GpuContext(model, scene.forces(), sim, max_batch=q0.shape[0])
    out = ctx.rollout(q0, np.zeros_like(q0), want_q=True, want_energy=True)
    out["_ctx"] = ctx
    return cfg, scene, sim, q0, out


def _replay(cfg, scene, sim, q0, envs, use_ref):
    sims = []
    for b in envs:
        s = type(sim)(**{**sim.__dict__})
        s.q0 = q0[b].copy()
        s.qdot0 = np.zeros_like(q0[b])
        sims.append(s)
    if use_ref and oracle.ref_available():
        return oracle.ref_batch_simulate(oracle.RefModel(scene.links), scene.forces(), sims,
                                         workers=min(len(sims), os.cpu_count() or 1)), "reference"
    return oracle.batch_simulate(oracle.Model(scene.links), scene.forces(), sims,
                                 workers=min(len(sims), os.cpu_count() or 1)), "port"


def _compare(tag, out, b, ref):
    k = ref.n_samples
    nrep = ref.n_reports
    assert out["n_samples"][b] == k, (tag, b, out["n_samples"][b], k)
    dq = np.max(np.abs(out["q"][b, :k] - ref.q[:k]), axis=1)
    _CURVES.setdefault(tag, {})[int(b)] = dq.tolist()
    np.testing.assert_array_equal(out["q"][b, :k], ref.q[:k])
    np.testing.assert_array_equal(out["energy"][b, :k], ref.energy[:k])
    np.testing.assert_array_equal(out["iterations"][b, :nrep], ref.iterations[:nrep])
    if np.all(ref.accepted[:nrep] >= 0):  # the reference's SolveReport has no accepted count (-1); the port's does
        np.testing.assert_array_equal(out["accepted"][b, :nrep], ref.accepted[:nrep])
    np.testing.assert_array_equal(out["converged"][b, :nrep], ref.converged[:nrep])
    np.testing.assert_array_equal(out["final_value"][b, :nrep], ref.final_value[:nrep])
    # the Trajectory the GPU step API builds for this env: same error text
    tr = _traj(out, b)
    assert (tr.error or None) == ref.error, (tag, b, tr.error, ref.error)
    assert len(tr.solve_reports) == nrep
    return k, nrep


def _traj(out, b):
    ctx = out["_ctx"]
    one = {key: v[b:b + 1] for key, v in out.items() if isinstance(v, np.ndarray)}
    return api._trajectories(ctx, [ctx.sim], one)[0]


def _dump():
    path = os.environ.get("PBAD_DIVERGENCE_OUT")
    if path:
        cur = json.load(open(path)) if os.path.exists(path) else {}
        cur.update({k: {"max_abs_dq_per_sample": v} for k, v in _CURVES.items()})
        json.dump(cur, open(path, "w"))


def test_c1_1000_steps_default_fail_limit():
    """The reference's own SimConfig default (consecutive_fail_limit = 25):
    the C1 chain's L-BFGS stops converging and the trajectory aborts with the
    reference's error text; the GPU aborts at the same step with the same text."""
    cfg, scene, sim, q0, out = _gpu("C1", 1000, 25)
    refs, _ = _replay(cfg, scene, sim, q0, [0], use_ref=True)
    ref = refs[0]
    assert ref.error is not None and ref.error.startswith("optimizer failed 26 consecutive steps")
    _compare("C1_default_fail_limit", out, 0, ref)
    # the 1024 replicas are identical environments
    for key in ("q", "iterations", "n_samples", "status"):
        assert np.all(out[key] == out[key][:1]), key


def test_c1_1000_steps_full():
    cfg, scene, sim, q0, out = _gpu("C1", 1000, 1 << 30)
    refs, _ = _replay(cfg, scene, sim, q0, [0], use_ref=True)
    k, _ = _compare("C1_1000_steps", out, 0, refs[0])
    assert k == 1001
    for key in ("q", "energy", "iterations"):
        assert np.all(out[key] == out[key][:1]), key
    _dump()


def test_c2_100_steps():
    cfg, scene, sim, q0, out = _gpu("C2", 100, 1 << 30)
    B = q0.shape[0]
    envs = [0, B // 2, B - 1]
    refs, _ = _replay(cfg, scene, sim, q0, envs, use_ref=True)
    for b, r in zip(envs, refs):
        k, _ = _compare("C2_100_steps", out, b, r)
        assert k == 101
    _dump()


def test_c2_default_fail_limit_error_text():
    cfg, scene, sim, q0, out = _gpu("C2", 100, 25)
    refs, _ = _replay(cfg, scene, sim, q0, [0, 1023], use_ref=True)
    for b, r in zip([0, 1023], refs):
        _compare("C2_default_fail_limit", out, b, r)
    got = api.batch_simulate(api.build_model(scene.links), scene.forces(), [_with_q0(sim, q0[0])])[0]
    assert got.error == refs[0].error


def _with_q0(sim, q0):
    s = type(sim)(**{**sim.__dict__})
    s.q0 = q0.copy()
    s.qdot0 = np.zeros_like(q0)
    return s


def test_c3_50_steps():
    cfg, scene, sim, q0, out = _gpu("C3", 50, 1 << 30)
    B = q0.shape[0]
    envs = [0, B - 1]
    refs, _ = _replay(cfg, scene, sim, q0, envs, use_ref=False)
    for b, r in zip(envs, refs):
        k, nrep = _compare("C3_50_steps", out, b, r)
        assert k == 51 and nrep == 50
    assert np.all(out["iterations"] == 512)  # the bench's step is the full 512-iteration solve
    _dump()


@pytest.mark.parametrize("name", ["C4", "C4b"])
def test_c4_100_steps(name):
    cfg, scene, sim, q0, out = _gpu(name, 100, 25)
    B = q0.shape[0]
    envs = [0, 1, B // 2, B - 1]
    refs, _ = _replay(cfg, scene, sim, q0, envs, use_ref=True)
    for b, r in zip(envs, refs):
        _compare(f"{name}_100_steps", out, b, r)
    _dump()


def test_c5_max_iters_512():
    """The bench's C5 step: 512 LM iterations of the U = 300 residual form."""
    cfg, scene, sim, q0, out = _gpu("C5", 1, 1 << 30)
    assert sim.optimizer.max_iters == 512
    B = q0.shape[0]
    envs = [0, B - 1]
    refs, _ = _replay(cfg, scene, sim, q0, envs, use_ref=False)
    for b, r in zip(envs, refs):
        _compare("C5_max_iters_512", out, b, r)
        assert r.iterations[0] == 512
    # accepted LM steps per env (DESIGN.md quotes 249 for env 0)
    assert int(out["accepted"][0, 0]) == int(refs[0].accepted[0])
    _dump()
