"""GPU parity of the residual-form (high-order collocation) Newton kernel,
pbad_resid.cu, against the CPU oracle: bit-exact trajectories, iteration
counts, convergence flags, final objective values and energy logs."""
import numpy as np
import pytest

import oracle
from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import Scene, make_single_hinge_chain_scene, mt19937_uniform
from paper_1709_04145_b200.types import (ActuationKind, ActuationSpec, ContactModel, JointKind, JointSpec, LinkSpec,
                                         ObjectiveKind, SimConfig)

from _parity_util import assert_traj_equal, random_tree

pytestmark = pytest.mark.gpu

PATH_RESID = 4


def _sims(sim, n, B, q0_fn):
    out = []
    for b in range(B):
        s = SimConfig(**{**sim.__dict__})
        s.q0 = q0_fn(b)
        s.qdot0 = np.zeros(n)
        out.append(s)
    return out


def _check(scene, sim, sims, path=PATH_RESID):
    m = api.build_model(scene.links)
    ctx = api.GpuContext(m, scene.forces(), sim, max_batch=1)
    assert ctx.path == path, ctx.path
    gpu = api.batch_simulate(m, scene.forces(), sims)
    ref = oracle.batch_simulate(oracle.Model(scene.links), scene.forces(), sims, workers=4)
    for g, r in zip(gpu, ref):
        assert_traj_equal(g, r)
    return gpu, ref


@pytest.mark.parametrize("order", [3, 4, 5])
def test_resid_chain(order):
    sc = make_single_hinge_chain_scene(6)
    sim = SimConfig(dt=0.01, duration=0.05, order=order, objective=ObjectiveKind.residual_form)
    _check(sc, sim, _sims(sim, 6, 3, lambda b: mt19937_uniform(b + 3, 6, -0.3, 0.3)))


def test_resid_order2():
    sc = make_single_hinge_chain_scene(5)
    sim = SimConfig(dt=0.02, duration=0.06, order=2, objective=ObjectiveKind.residual_form)
    _check(sc, sim, _sims(sim, 5, 2, lambda b: mt19937_uniform(b + 8, 5, -0.3, 0.3)))


@pytest.mark.parametrize("seed", [41, 42])
def test_resid_hinge_tree(seed):
    """Branched hinge tree, tilted axes, rotated offsets, point masses: the
    non-chain J (zero blocks between unrelated links)."""
    rng = np.random.default_rng(seed)
    base = random_tree(rng, 7)
    links = []
    for l in base:
        ax = rng.uniform(-1, 1, 3)
        links.append(LinkSpec(l.parent, JointSpec(JointKind.hinge, tuple(ax / np.linalg.norm(ax)), l.joint.offset),
                              l.geometry))
    sc = Scene(links=links, gravity=(0.3, -1.0, -9.81))
    sim = SimConfig(dt=0.02, duration=0.06, order=3, objective=ObjectiveKind.residual_form)
    _check(sc, sim, _sims(sim, 7, 2, lambda b: rng.uniform(-0.4, 0.4, 7)))


def test_resid_actuated():
    sc = make_single_hinge_chain_scene(5)
    sc.actuation = ActuationSpec(ActuationKind.sinusoidal, np.linspace(-2, 2, 5), 3.0, np.linspace(0, 1, 5))
    sim = SimConfig(dt=0.02, duration=0.06, order=4, objective=ObjectiveKind.residual_form)
    _check(sc, sim, _sims(sim, 5, 2, lambda b: mt19937_uniform(b, 5, -0.3, 0.3)))


def test_resid_c5_shape_bounded_iterations():
    """The C5 shape (100-link chain, K = 4, U = 300: ragged GEMM and Cholesky
    blocks) with a small iteration cap so the oracle finishes quickly."""
    sc = make_single_hinge_chain_scene(100)
    sim = SimConfig(dt=0.01, duration=0.02, order=4, objective=ObjectiveKind.residual_form,
                    consecutive_fail_limit=10)
    sim.optimizer.max_iters = 12
    _check(sc, sim, _sims(sim, 100, 2, lambda b: mt19937_uniform(3, 200, -0.3, 0.3)[100 * b:100 * (b + 1)]))


def test_resid_equals_general_kernel(monkeypatch):
    sc = make_single_hinge_chain_scene(6)
    sim = SimConfig(dt=0.01, duration=0.04, order=4, objective=ObjectiveKind.residual_form)
    m = api.build_model(sc.links)
    sims = _sims(sim, 6, 5, lambda b: mt19937_uniform(b + 20, 6, -0.3, 0.3))
    a = api.batch_simulate(m, sc.forces(), sims)
    monkeypatch.setenv("PBAD_GPU_FORCE_GENERAL", "1")
    assert api.GpuContext(m, sc.forces(), sim, max_batch=1).path == 0
    b = api.batch_simulate(m, sc.forces(), sims)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(np.array([s[1] for s in x.samples]), np.array([s[1] for s in y.samples]))
        assert [r.iterations for r in x.solve_reports] == [r.iterations for r in y.solve_reports]


# --- drag in the residual form (serial chains): per-instant cotangents and the
# pot.hess term 2 D / (t_m dt)^2 hess_ab in the fused diagonal-block walks
# (objective.cpp:60-71,131-134, 296-313)

@pytest.mark.parametrize("order", [2, 3, 4])
def test_resid_drag_chain(order):
    sc = make_single_hinge_chain_scene(6)
    sc.drag_d = 1.5
    sim = SimConfig(dt=0.01, duration=0.05, order=order, objective=ObjectiveKind.residual_form)
    _check(sc, sim, _sims(sim, 6, 3, lambda b: mt19937_uniform(b + 50, 6, -0.4, 0.4)))


def test_resid_drag_no_gravity_actuated():
    """Drag alone (no gravity cotangent) plus sinusoidal actuation, tilted
    hinge axes and rotated offsets on a serial chain."""
    rng = np.random.default_rng(12)
    base = random_tree(rng, 7, chain=True)
    links = []
    for l in base:
        ax = rng.uniform(-1, 1, 3)
        links.append(LinkSpec(l.parent, JointSpec(JointKind.hinge, tuple(ax / np.linalg.norm(ax)), l.joint.offset),
                              l.geometry))
    sc = Scene(links=links, gravity=(0.0, 0.0, 0.0))
    sc.drag_d = 3.0
    sc.actuation = ActuationSpec(ActuationKind.sinusoidal, np.linspace(-2, 2, 7), 2.0, np.linspace(0, 1, 7))
    sim = SimConfig(dt=0.02, duration=0.06, order=3, objective=ObjectiveKind.residual_form)
    _check(sc, sim, _sims(sim, 7, 2, lambda b: rng.uniform(-0.4, 0.4, 7)))


def test_resid_drag_c5_shape_bounded_iterations():
    """The C5 shape with drag (U = 300), a small iteration cap."""
    sc = make_single_hinge_chain_scene(100)
    sc.drag_d = 0.8
    sim = SimConfig(dt=0.01, duration=0.02, order=4, objective=ObjectiveKind.residual_form,
                    consecutive_fail_limit=10)
    sim.optimizer.max_iters = 10
    _check(sc, sim, _sims(sim, 100, 2, lambda b: mt19937_uniform(7, 200, -0.3, 0.3)[100 * b:100 * (b + 1)]))


@pytest.mark.parametrize("seed", [5, 6])
def test_resid_drag_tree(seed):
    """Drag on a branched hinge tree in the residual form: the diagonal pair's
    ab goes through PH into pot.hess (zero blocks between unrelated links)."""
    rng = np.random.default_rng(seed)
    base = random_tree(rng, 7)
    links = []
    for l in base:
        ax = rng.uniform(-1, 1, 3)
        links.append(LinkSpec(l.parent, JointSpec(JointKind.hinge, tuple(ax / np.linalg.norm(ax)), l.joint.offset),
                              l.geometry))
    assert not all(l.parent == (None if i == 0 else i - 1) for i, l in enumerate(links))
    sc = Scene(links=links, gravity=(0.3, -1.0, -9.81))
    sc.drag_d = 1.2
    sim = SimConfig(dt=0.02, duration=0.06, order=3, objective=ObjectiveKind.residual_form)
    _check(sc, sim, _sims(sim, 7, 2, lambda b: rng.uniform(-0.4, 0.4, 7)))


# --- contact in the residual form: per-sample cotangents dqdx ph^T and the
# pot.hess term jx^T hxx jx of every active sample, added after the drag term
# and before functional_hess(cot) (objective.cpp:74-135); the contact scenes
# run the tree walks (chains included)

def _contact_links(rng, n, chain, per_link=2, spread=0.15):
    base = random_tree(rng, n, chain=chain)
    links = []
    for l in base:
        ax = rng.uniform(-1, 1, 3)
        samples = [tuple(rng.uniform(-spread, spread, 3)) for _ in range(per_link)]
        links.append(LinkSpec(l.parent, JointSpec(JointKind.hinge, tuple(ax / np.linalg.norm(ax)), l.joint.offset),
                              l.geometry, contact_samples=samples))
    return links


@pytest.mark.parametrize("chain,order,d2", [(True, 3, 40.0), (False, 3, 40.0), (True, 4, 0.0), (False, 2, 25.0)])
def test_resid_contact(chain, order, d2):
    """Contact samples on every link against a tilted plane through the
    structure: samples enter and leave contact along the trajectory."""
    rng = np.random.default_rng(100 + order + (0 if chain else 7))
    n = 7
    sc = Scene(links=_contact_links(rng, n, chain), gravity=(0.2, -0.5, -9.81))
    nrm = np.array([0.3, -0.2, 1.0])
    sc.contact = ContactModel(tuple(nrm / np.linalg.norm(nrm)), 0.05, 3.0e3, d2)
    sim = SimConfig(dt=0.01, duration=0.06, order=order, objective=ObjectiveKind.residual_form)
    gpu, ref = _check(sc, sim, _sims(sim, n, 3, lambda b: rng.uniform(-0.6, 0.6, n)))


def test_resid_contact_with_drag_no_gravity():
    """Contact with drag and no gravity: the contact pot.hess terms land on
    (0 + 2 scale ab) before functional_hess (objective.cpp:69-71, 118-123)."""
    rng = np.random.default_rng(77)
    n = 6
    sc = Scene(links=_contact_links(rng, n, False, per_link=3), gravity=(0.0, 0.0, 0.0))
    sc.drag_d = 1.1
    sc.contact = ContactModel((0.0, 0.0, 1.0), 0.02, 5.0e3, 60.0)
    sim = SimConfig(dt=0.02, duration=0.08, order=3, objective=ObjectiveKind.residual_form)
    _check(sc, sim, _sims(sim, n, 2, lambda b: rng.uniform(-0.8, 0.8, n)))


def test_resid_contact_larger_chain():
    """A 40-link chain, samples on alternate links, K = 3."""
    rng = np.random.default_rng(5)
    n = 40
    links = _contact_links(rng, n, True, per_link=1)
    for i in range(1, n, 2):
        links[i].contact_samples = []
    sc = Scene(links=links, gravity=(0.0, 0.0, -9.81))
    sc.contact = ContactModel((0.0, 0.0, 1.0), -0.05, 2.0e3, 10.0)
    sim = SimConfig(dt=0.01, duration=0.03, order=3, objective=ObjectiveKind.residual_form)
    _check(sc, sim, _sims(sim, n, 2, lambda b: rng.uniform(-0.4, 0.4, n)))


def test_resid_u2_beyond_320():
    """Residual form K = 3 (u = 2) on a 180-link chain: U = 360 unknowns."""
    sc = make_single_hinge_chain_scene(180)
    sim = SimConfig(dt=0.01, duration=0.02, order=3, objective=ObjectiveKind.residual_form,
                    consecutive_fail_limit=10)
    sim.optimizer.max_iters = 12
    _check(sc, sim, _sims(sim, 180, 2, lambda b: mt19937_uniform(b + 60, 180, -0.3, 0.3)))


def test_resid_persistent_multistep(tmp_path):
    """The CTA kernel runs a window of steps in one persistent launch
    (k_resid_steps, pbad_resid.cu), one CTA per SM claiming env-steps in
    order.  300 environments on 148 SMs: environments change SM between
    steps and wait on their previous step.  The whole batch is bit-identical
    to one launch per step (PBAD_RESID_PERSIST=0), and a sample matches the
    oracle."""
    import _persist_run as pr
    B, steps = 300, 4
    one, per = pr.run_pair("resid", tmp_path, B, steps, "PBAD_RESID_PERSIST")
    assert int(one["path"]) == PATH_RESID
    assert int(one["launches"]) == 1 and int(per["launches"]) == steps
    for k in ("q", "energy", "iterations"):
        np.testing.assert_array_equal(one[k], per[k])
    sc = pr.scene("resid")
    n = 12
    q0 = pr.inputs("resid", B, n, sc.q0)
    sim = pr.sim("resid", steps)
    envs = [0, 149, B - 1]
    ref = oracle.batch_simulate(oracle.Model(sc.links), sc.forces(), _sims(sim, n, len(envs), lambda i: q0[envs[i]]),
                                workers=3)
    for i, b in enumerate(envs):
        k = ref[i].n_samples
        np.testing.assert_array_equal(one["q"][b, :k], ref[i].q[:k])
        np.testing.assert_array_equal(one["iterations"][b, :len(ref[i].iterations)], ref[i].iterations)
