"""Stepper features beyond the default path, bit-exact against the
reference itself (oracle/_ref, /root/reference/proj/src compiled unmodified):
refined_bootstrap (stepper.cpp:46-59, the RK4 Newton-Euler history),
lbfgs_memory <= 0 (optim.cpp:183-186: every pair is pushed and popped, i.e.
steepest descent), and SolveReport::per_iteration_values (optim.cpp:30-37)
recorded by every kernel family."""
import numpy as np
import pytest

import oracle
from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import make_chain_scene, make_humanoid_scene, make_single_hinge_chain_scene
from paper_1709_04145_b200.types import ObjectiveKind, OptimizerKind, SimConfig

from _parity_util import assert_traj_equal

pytestmark = pytest.mark.gpu


def _sims(n, B, seed, **kw):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(B):
        s = SimConfig(**{k: v for k, v in kw.items() if k != "opt"})
        for k, v in kw.get("opt", {}).items():
            setattr(s.optimizer, k, v)
        s.q0 = rng.uniform(-0.3, 0.3, n)
        s.qdot0 = rng.uniform(-1.0, 1.0, n)
        out.append(s)
    return out


def _ref(scene, sims):
    return oracle.ref_batch_simulate(oracle.RefModel(scene.links), scene.forces(), sims, workers=4)


@pytest.mark.parametrize("kind,order,objective,path", [
    (OptimizerKind.lbfgs, 2, ObjectiveKind.energy_form, 5),
    (OptimizerKind.lm, 2, ObjectiveKind.energy_form, 3),
    (OptimizerKind.lm, 4, ObjectiveKind.residual_form, 4),
])
def test_refined_bootstrap(kind, order, objective, path):
    sc = make_single_hinge_chain_scene(8)
    sims = _sims(8, 3, 5, dt=0.02, duration=0.08, order=order, objective=objective, refined_bootstrap=True,
                 opt=dict(kind=kind))
    m = api.build_model(sc.links)
    assert api.GpuContext(m, sc.forces(), sims[0], max_batch=1).path == path
    gpu = api.batch_simulate(m, sc.forces(), sims)
    for g, r in zip(gpu, _ref(sc, sims)):
        assert_traj_equal(g, r)


def test_refined_bootstrap_tree():
    sc = make_humanoid_scene()
    rng = np.random.default_rng(3)
    sims = []
    for _ in range(2):
        s = SimConfig(dt=0.01, duration=0.04, refined_bootstrap=True)
        s.q0 = sc.q0.copy()
        s.q0[6:] += rng.uniform(-0.1, 0.1, len(s.q0) - 6)
        s.qdot0 = rng.uniform(-0.5, 0.5, len(s.q0))
        sims.append(s)
    gpu = api.batch_simulate(api.build_model(sc.links), sc.forces(), sims)
    for g, r in zip(gpu, _ref(sc, sims)):
        assert_traj_equal(g, r)


@pytest.mark.parametrize("mem", [0, -3])
@pytest.mark.parametrize("scene,path", [("chain", 5), ("humanoid", 3)])
def test_lbfgs_memory_nonpositive(mem, scene, path):
    sc = make_chain_scene(6) if scene == "chain" else make_humanoid_scene()
    m = api.build_model(sc.links)
    n = m.total_dofs
    sims = _sims(n, 3, 9, dt=0.02, duration=0.06, opt=dict(kind=OptimizerKind.lbfgs, lbfgs_memory=mem))
    if scene == "humanoid":
        for s in sims:
            s.q0 = sc.q0 + np.concatenate([np.zeros(6), 0.3 * s.q0[6:]])
            s.qdot0 = np.zeros(n)
    assert api.GpuContext(m, sc.forces(), sims[0], max_batch=1).path == path
    gpu = api.batch_simulate(m, sc.forces(), sims)
    for g, r in zip(gpu, _ref(sc, sims)):
        assert_traj_equal(g, r)


@pytest.mark.parametrize("case", ["chain4", "tree_lm", "tree_lbfgs", "resid", "general"])
def test_per_iteration_values(case, monkeypatch):
    """The value after every iteration (optim.cpp:64-67): its count equals
    the iteration count, its last entry the final value, and it equals the
    general kernel's record (which follows the reference's finish_iteration
    line for line); the reference's own values are compared in
    tests/dropin/dropin_check.cpp."""
    if case in ("chain4", "general"):
        sc = make_single_hinge_chain_scene(10)
        kw = dict(dt=0.02, duration=0.06, opt=dict(kind=OptimizerKind.lbfgs))
    elif case == "tree_lm":
        sc = make_humanoid_scene()
        kw = dict(dt=0.01, duration=0.05)
    elif case == "tree_lbfgs":
        sc = make_humanoid_scene()
        kw = dict(dt=0.01, duration=0.05, opt=dict(kind=OptimizerKind.lbfgs))
    else:
        sc = make_single_hinge_chain_scene(6)
        kw = dict(dt=0.01, duration=0.03, order=4, objective=ObjectiveKind.residual_form)
    m = api.build_model(sc.links)
    n = m.total_dofs
    sims = _sims(n, 3, 11, **kw)
    if "tree" in case:
        for s in sims:
            s.q0 = sc.q0 + np.concatenate([np.zeros(6), 0.3 * s.q0[6:]])
            s.qdot0 = np.zeros(n)
    if case == "general":
        monkeypatch.setenv("PBAD_GPU_FORCE_GENERAL", "1")
    gpu = api.batch_simulate(m, sc.forces(), sims, record_iteration_values=True)
    monkeypatch.setenv("PBAD_GPU_FORCE_GENERAL", "1")
    gen = api.batch_simulate(m, sc.forces(), sims, record_iteration_values=True)
    for g, h in zip(gpu, gen):
        assert len(g.solve_reports) > 0
        for rg, rh in zip(g.solve_reports, h.solve_reports):
            assert len(rg.per_iteration_values) == rg.iterations
            if rg.iterations:
                assert rg.per_iteration_values[-1] == rg.final_value
            assert rg.per_iteration_values == rh.per_iteration_values
