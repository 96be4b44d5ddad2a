"""Golden vectors produced by the reference itself (scripts/make_golden.py
runs oracle/_ref: /root/reference/proj compiled unmodified against
eigen_lite).  The CPU oracle must reproduce them bit for bit (runs
anywhere); the CUDA path too (gpu marker)."""
import glob
import os

import numpy as np
import pytest

import oracle
from paper_1709_04145_b200.types import ObjectiveKind, OptimizerKind, SimConfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROLLOUTS = sorted(glob.glob(os.path.join(HERE, "golden", "rollout_*.npz")))
EVALS = sorted(glob.glob(os.path.join(HERE, "golden", "eval_*.npz")))


def _scene(name):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "scripts"))
    from make_golden import scene
    return scene(name)


def _sim(g):
    s = SimConfig(dt=float(g["dt"]), duration=float(g["dt"]) * int(g["steps"]), order=int(g["order"]),
                  objective=ObjectiveKind.energy_form if int(g["order"]) == 2 else ObjectiveKind.residual_form)
    s.optimizer.kind = OptimizerKind.lbfgs if str(g["optimizer"]) == "lbfgs" else OptimizerKind.lm
    s.q0 = g["q0"]
    s.qdot0 = np.zeros(len(g["q0"]))
    return s


def _check(q, energy, its, conv, fv, g):
    k = len(g["q"])
    assert np.array_equal(np.asarray(q)[:k], g["q"])
    assert np.array_equal(np.asarray(energy)[:k], g["energy"])
    assert np.array_equal(np.asarray(its)[:k - 1], g["iterations"])
    assert np.array_equal(np.asarray(conv)[:k - 1], g["converged"])
    assert np.array_equal(np.asarray(fv)[:k - 1], g["final_value"])


def test_golden_fixtures_present():
    assert len(ROLLOUTS) >= 6 and len(EVALS) >= 4


@pytest.mark.parametrize("path", ROLLOUTS, ids=[os.path.basename(p) for p in ROLLOUTS])
def test_oracle_matches_reference_golden_rollout(path):
    g = np.load(path)
    sc = _scene(str(g["scene"]))
    tr = oracle.batch_simulate(oracle.Model(sc.links), sc.forces(), [_sim(g)])[0]
    _check(tr.q, tr.energy, tr.iterations, tr.converged, tr.final_value, g)


@pytest.mark.parametrize("path", EVALS, ids=[os.path.basename(p) for p in EVALS])
def test_oracle_matches_reference_golden_eval(path):
    g = np.load(path)
    sc = _scene(str(g["scene"]))
    v, gr, gn = oracle.step_eval(oracle.Model(sc.links), sc.forces(), int(g["order"]), float(g["dt"]),
                                 int(g["objective"]), g["h0"], g["h1"], g["x"], True, True)
    assert v == float(g["value"])
    assert np.array_equal(gr, g["grad"]) and np.array_equal(gn, g["gn"])


@pytest.mark.gpu
@pytest.mark.parametrize("path", ROLLOUTS, ids=[os.path.basename(p) for p in ROLLOUTS])
def test_gpu_matches_reference_golden_rollout(path):
    from paper_1709_04145_b200 import api
    g = np.load(path)
    sc = _scene(str(g["scene"]))
    tr = api.batch_simulate(api.build_model(sc.links), sc.forces(), [_sim(g)])[0]
    q = np.array([s[1] for s in tr.samples])
    e = np.array([[x.kinetic, x.potential] for x in tr.energy_log])
    _check(q, e, [r.iterations for r in tr.solve_reports], [int(r.converged) for r in tr.solve_reports],
           [r.final_value for r in tr.solve_reports], g)


@pytest.mark.gpu
@pytest.mark.parametrize("path", EVALS, ids=[os.path.basename(p) for p in EVALS])
def test_gpu_matches_reference_golden_eval(path):
    from paper_1709_04145_b200 import api
    g = np.load(path)
    sc = _scene(str(g["scene"]))
    sim = SimConfig(dt=float(g["dt"]), duration=float(g["dt"]), order=int(g["order"]),
                    objective=ObjectiveKind(int(g["objective"])))
    sim.optimizer.kind = OptimizerKind.lm
    ctx = api.GpuContext(api.build_model(sc.links), sc.forces(), sim, max_batch=1)
    v, gr, gn = ctx.eval(np.concatenate([g["h0"], g["h1"]])[None], g["x"][None], True, True)
    assert v[0] == float(g["value"])
    assert np.array_equal(gr[0], g["grad"]) and np.array_equal(gn[0], g["gn"])
