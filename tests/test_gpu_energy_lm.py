"""GPU parity of the energy-form Newton (LM) path for large hinge trees on the
CTA-per-environment kernel (pbad_resid.cu "energy form"): the shapes the
warp-per-environment tree kernel cannot hold (n > 96), among them the
BASELINE C3 chain with LM ("K=2, LBFGS (LM as variant)").
Bit-exact against the CPU oracle: samples, energy log, per-step iteration
counts, convergence flags, final values (objective.cpp:215-256,
optim.cpp:80-139)."""
import numpy as np
import pytest

import oracle
from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import Scene, make_chain_scene, make_single_hinge_chain_scene, mt19937_uniform
from paper_1709_04145_b200.types import (ActuationKind, ActuationSpec, JointKind, JointSpec, LinkSpec,
                                         OptimizerKind, SimConfig)

from _parity_util import assert_traj_equal, random_tree

pytestmark = pytest.mark.gpu

PATH_RESID, PATH_TREE = 4, 3


def _sims(sim, n, B, q0_fn):
    out = []
    for b in range(B):
        s = SimConfig(**{**sim.__dict__})
        s.optimizer = sim.optimizer
        s.q0 = q0_fn(b)
        s.qdot0 = np.zeros(n)
        out.append(s)
    return out


def _lm(dt, duration, **kw):
    sim = SimConfig(dt=dt, duration=duration, **kw)
    sim.optimizer.kind = OptimizerKind.lm
    return sim


def _check(scene, sim, sims, path=PATH_RESID):
    m = api.build_model(scene.links)
    ctx = api.GpuContext(m, scene.forces(), sim, max_batch=1)
    assert ctx.path == path, ctx.path
    gpu = api.batch_simulate(m, scene.forces(), sims)
    ref = oracle.batch_simulate(oracle.Model(scene.links), scene.forces(), sims, workers=4)
    for g, r in zip(gpu, ref):
        assert_traj_equal(g, r)
    return gpu, ref


def test_c3_lm_shape():
    """C3's 200-link chain (100 massless Z-hinge connectors + 100 Y-hinge
    boxes, n = 200) with LM at dt = 0.1: the survey's C3-LM variant."""
    sc = make_chain_scene(100)
    sim = _lm(0.1, 0.2)
    q0 = mt19937_uniform(1, 2 * 200, -0.3, 0.3)
    gpu, ref = _check(sc, sim, _sims(sim, 200, 2, lambda b: q0[200 * b:200 * (b + 1)]))
    assert all(len(g.solve_reports) == 2 for g in gpu)


def test_single_hinge_chain_actuated():
    """120-link single-hinge chain, sinusoidal actuation, warm start."""
    sc = make_single_hinge_chain_scene(120)
    sc.actuation = ActuationSpec(ActuationKind.sinusoidal, np.linspace(-2, 2, 120), 2.0, np.linspace(0, 1, 120))
    sim = _lm(0.01, 0.03)
    _check(sc, sim, _sims(sim, 120, 2, lambda b: mt19937_uniform(b + 5, 120, -0.3, 0.3)))


def test_branched_hinge_tree_over_96_dofs():
    """A 104-link branched hinge tree (tilted axes, rotated offsets, boxes and
    point masses, tilted gravity): zero GN blocks between unrelated links."""
    rng = np.random.default_rng(7)
    base = random_tree(rng, 104)
    links = []
    for l in base:
        ax = rng.uniform(-1, 1, 3)
        links.append(LinkSpec(l.parent, JointSpec(JointKind.hinge, tuple(ax / np.linalg.norm(ax)), l.joint.offset),
                              l.geometry))
    sc = Scene(links=links, gravity=(0.4, -1.0, -9.81))
    sim = _lm(0.02, 0.04)
    _check(sc, sim, _sims(sim, 104, 2, lambda b: rng.uniform(-0.3, 0.3, 104)))


def test_zero_gravity_and_fail_limit():
    """No gravity (no potential terms) and an iteration cap with fail limit 1:
    the reference's error text after the second failing step."""
    sc = make_single_hinge_chain_scene(100)
    sc.gravity = (0.0, 0.0, 0.0)
    sim = _lm(0.05, 0.1, consecutive_fail_limit=1)
    sim.optimizer.max_iters = 3
    gpu, ref = _check(sc, sim, _sims(sim, 100, 2, lambda b: mt19937_uniform(b + 30, 100, -1.0, 1.0)))


@pytest.mark.parametrize("name", ["chain", "tree"])
def test_small_shapes_match_tree_kernel(name, monkeypatch):
    """Where the warp-per-environment tree kernel fits, PBAD_GPU_RESID_ENERGY
    routes the same energy-form LM through the CTA kernel: both are
    bit-identical to the oracle (and therefore to each other)."""
    if name == "chain":
        sc = make_single_hinge_chain_scene(8)
    else:
        rng = np.random.default_rng(3)
        base = random_tree(rng, 9)
        links = [LinkSpec(l.parent, JointSpec(JointKind.hinge, (0.0, 1.0, 0.0), l.joint.offset), l.geometry)
                 for l in base]
        sc = Scene(links=links, gravity=(0.0, -2.0, -9.81))
    m = api.build_model(sc.links)
    n = m.total_dofs
    sim = _lm(0.01, 0.05)
    sims = _sims(sim, n, 5, lambda b: mt19937_uniform(b + 11, n, -0.5, 0.5))
    tree_gpu, _ = _check(sc, sim, sims, path=PATH_TREE)
    monkeypatch.setenv("PBAD_GPU_RESID_ENERGY", "1")
    resid_gpu, _ = _check(sc, sim, sims, path=PATH_RESID)
    for a, b in zip(tree_gpu, resid_gpu):
        np.testing.assert_array_equal(np.array([s[1] for s in a.samples]), np.array([s[1] for s in b.samples]))


def test_chain_beyond_320_dofs():
    """A 360-link single-hinge chain (U = 360 > the round-1 bound of 320):
    the larger accumulator tiles of the Cholesky block-column update."""
    sc = make_single_hinge_chain_scene(360)
    sim = _lm(0.01, 0.02)
    sim.optimizer.max_iters = 40
    _check(sc, sim, _sims(sim, 360, 2, lambda b: mt19937_uniform(b + 90, 360, -0.2, 0.2)))
