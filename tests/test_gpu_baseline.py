"""Newton-Euler baselines on the GPU (pbad_gpu_simulate_baseline,
SURVEY.md §8(f) item 4) against the reference's own simulate_baseline
(stepper.cpp:168-202, baseline.cpp:56-206, compiled into oracle/_ref):
samples, KE / PE log and error texts bit for bit, every scheme."""
import numpy as np
import pytest

import oracle
from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import (make_humanoid_scene, make_single_hinge_chain_scene,
                                          make_spider_scene, make_swimmer_scene)
from paper_1709_04145_b200.types import (BaselineScheme, ContactModel, ForceModel, JointKind, JointSpec, LinkSpec,
                                         PointMassGeometry, SimConfig)

from _parity_util import random_tree

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")]

SCHEMES = list(BaselineScheme)


def _compare(links, forces, sims, scheme):
    m = api.build_model(links)
    gpu = api.batch_simulate_baseline(m, forces, scheme, sims)
    rm = oracle.RefModel(links)
    for g, sim in zip(gpu, sims):
        r = oracle.ref_simulate_baseline(rm, forces, scheme, sim)
        k = r.n_samples
        assert len(g.samples) == k
        np.testing.assert_array_equal(np.array([s[1] for s in g.samples]), r.q[:k])
        np.testing.assert_array_equal(np.array([[e.kinetic, e.potential] for e in g.energy_log]), r.energy[:k])
        assert g.error == r.error
    return gpu


def _sims(sim, B, q0_fn, qd_fn):
    out = []
    for b in range(B):
        s = SimConfig(**{**sim.__dict__})
        s.q0 = q0_fn(b)
        s.qdot0 = qd_fn(b)
        out.append(s)
    return out


@pytest.mark.parametrize("scheme", SCHEMES)
def test_baseline_hinge_chain(scheme):
    sc = make_single_hinge_chain_scene(8)
    rng = np.random.default_rng(int(scheme))
    sim = SimConfig(dt=0.002, duration=0.02)
    _compare(sc.links, sc.forces(), _sims(sim, 4, lambda b: rng.uniform(-0.5, 0.5, 8),
                                           lambda b: rng.uniform(-1, 1, 8)), scheme)


@pytest.mark.parametrize("scheme", [BaselineScheme.semi_implicit, BaselineScheme.rk4])
def test_baseline_humanoid_free_and_ball_joints(scheme):
    sc = make_humanoid_scene()
    rng = np.random.default_rng(5)
    n = 41
    sim = SimConfig(dt=0.002, duration=0.01)

    def q0(b):
        q = sc.q0.copy()
        q[6:] = rng.uniform(-0.2, 0.2, n - 6)
        return q
    _compare(sc.links, sc.forces(), _sims(sim, 3, q0, lambda b: rng.uniform(-0.5, 0.5, n)), scheme)


@pytest.mark.parametrize("scheme", [BaselineScheme.forward_euler, BaselineScheme.rk3])
def test_baseline_spider_contact_and_swimmer_drag(scheme):
    sp = make_spider_scene(api.rotation_vector_matrix)
    sim = SimConfig(dt=0.002, duration=0.02)
    q = sp.q0.copy()
    q[2] = 0.05  # feet below the plane: contact with velocity damping
    _compare(sp.links, sp.forces(), _sims(sim, 2, lambda b: q + 0.01 * b, lambda b: np.full(22, 0.1 * (b + 1))),
             scheme)
    sw = make_swimmer_scene()
    f = sw.forces()
    f.actuation = None
    f.tau = np.linspace(-1.0, 1.0, 9)  # generalized_force adds a constant tau (baseline.cpp:131)
    _compare(sw.links, f, _sims(SimConfig(dt=0.01, duration=0.05), 2, lambda b: np.full(9, 0.1 * b),
                                lambda b: np.full(9, -0.2)), scheme)


@pytest.mark.parametrize("seed", [71, 72])
def test_baseline_random_trees_drag_contact(seed):
    rng = np.random.default_rng(seed)
    links = random_tree(rng, 6)
    forces = ForceModel(gravity=(0.3, -0.2, -9.81), drag_d=0.4,
                        contact=ContactModel((0.0, 0.0, 1.0), 0.2, 3e3, 30.0))
    n = api.build_model(links).total_dofs
    sim = SimConfig(dt=0.004, duration=0.02)
    _compare(links, forces, _sims(sim, 3, lambda b: rng.uniform(-0.5, 0.5, n), lambda b: rng.uniform(-1, 1, n)),
             BaselineScheme.rk2)


def test_baseline_divergence_and_singular_mass_errors():
    sc = make_single_hinge_chain_scene(4)
    sim = SimConfig(dt=5.0, duration=200.0)  # explicit Euler blows up
    gpu = _compare(sc.links, sc.forces(), _sims(sim, 1, lambda b: np.full(4, 0.5), lambda b: np.full(4, 3.0)),
                   BaselineScheme.forward_euler)
    assert gpu[0].error is not None
    massless = [LinkSpec(parent=None, joint=JointSpec(JointKind.hinge, (0.0, 1.0, 0.0)),
                         geometry=PointMassGeometry([]))]
    gpu = _compare(massless, ForceModel(gravity=(0.0, 0.0, -9.81)),
                   _sims(SimConfig(dt=0.01, duration=0.03), 1, lambda b: np.zeros(1), lambda b: np.zeros(1)),
                   BaselineScheme.semi_implicit)
    assert gpu[0].error == "step failed: singular generalized mass matrix"
