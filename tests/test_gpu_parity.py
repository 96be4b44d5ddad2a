"""GPU parity: the CUDA path through the C ABI against the CPU oracle.

The bar is bit-exact equality (the numeric contract in DESIGN.md fixes every
rounding order), which implies the north-star gates: per-eval energy /
gradient / GN within 1e-10 relative, equal optimizer iteration counts and
joint positions within 1e-8 after a short rollout.
"""
import numpy as np
import pytest

import oracle
from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import (make_chain_scene, make_humanoid_scene, make_single_hinge_chain_scene,
                                          make_spider_scene, make_swimmer_scene, mt19937_uniform)
from paper_1709_04145_b200.types import ObjectiveKind, OptimizerKind, SimConfig

from _parity_util import assert_traj_equal, random_tree

pytestmark = pytest.mark.gpu


def _eval_case(links, forces, order, dt, objective, seed, lm=False, tau=False, scale=0.5):
    rng = np.random.default_rng(seed)
    m = api.build_model(links)
    mo = oracle.Model(links)
    n = m.total_dofs
    u = order - 1
    sim = SimConfig(dt=dt, duration=dt, order=order, objective=objective)
    sim.optimizer.kind = OptimizerKind.lm if lm else OptimizerKind.lbfgs
    ctx = api.GpuContext(m, forces, sim, max_batch=4)
    B = 3
    hist = rng.uniform(-scale, scale, (B, 2 * n))
    x = rng.uniform(-scale, scale, (B, u * n))
    taus = rng.uniform(-1, 1, (B, u * n)) if tau else None
    v, g, gn = ctx.eval(hist, x, want_grad=True, want_gn=lm, tau=taus)
    v0, _, _ = ctx.eval(hist, x, want_grad=False, tau=taus)
    for b in range(B):
        ov, og, ogn = oracle.step_eval(mo, forces, order, dt, int(objective), hist[b, :n], hist[b, n:], x[b],
                                       True, lm, None if taus is None else taus[b].reshape(u, n))
        assert v[b] == ov, (b, v[b], ov)
        assert v0[b] == ov
        np.testing.assert_array_equal(g[b], og)
        if lm:
            np.testing.assert_array_equal(gn[b], ogn)


def test_eval_energy_chain():
    sc = make_single_hinge_chain_scene(10)
    _eval_case(sc.links, sc.forces(), 2, 0.01, ObjectiveKind.energy_form, 1)
    _eval_case(sc.links, sc.forces(), 2, 0.033, ObjectiveKind.energy_form, 2, lm=True)


def test_eval_energy_two_hinge_chain():
    sc = make_chain_scene(8)
    _eval_case(sc.links, sc.forces(), 2, 0.1, ObjectiveKind.energy_form, 3, lm=True)


def test_eval_energy_humanoid_tree():
    sc = make_humanoid_scene()
    _eval_case(sc.links, sc.forces(), 2, 0.01, ObjectiveKind.energy_form, 4, lm=True, scale=0.2)


@pytest.mark.parametrize("seed", [5, 6, 7])
def test_eval_random_trees(seed):
    rng = np.random.default_rng(seed)
    links = random_tree(rng, 7)
    from paper_1709_04145_b200.types import ForceModel
    f = ForceModel(gravity=(0.3, -1.0, -9.81))
    _eval_case(links, f, 2, 0.02, ObjectiveKind.energy_form, seed, lm=True, tau=True)


def test_eval_contact_and_drag():
    sc = make_spider_scene(api.rotation_vector_matrix)
    f = sc.forces()
    f.drag_d = 1.5
    _eval_case(sc.links, f, 2, 0.01, ObjectiveKind.energy_form, 8, lm=True, scale=0.3)


@pytest.mark.parametrize("order", [3, 4])
def test_eval_residual_form(order):
    sc = make_single_hinge_chain_scene(5)
    _eval_case(sc.links, sc.forces(), order, 0.01, ObjectiveKind.residual_form, 9, lm=True)


def test_eval_residual_form_contact():
    sc = make_spider_scene(api.rotation_vector_matrix)
    _eval_case(sc.links, sc.forces(), 3, 0.01, ObjectiveKind.residual_form, 10, lm=True, scale=0.2)


def _rollout_case(scene, sim, B=1, seed=None, lo=-0.3, hi=0.3):
    m = api.build_model(scene.links)
    mo = oracle.Model(scene.links)
    n = m.total_dofs
    sims = []
    for b in range(B):
        s = SimConfig(**{**sim.__dict__})
        q0 = scene.q0.copy()
        if seed is not None:
            q0 = mt19937_uniform(seed + b, n, lo, hi)
        s.q0 = q0
        s.qdot0 = np.zeros(n)
        sims.append(s)
    gpu = api.batch_simulate(m, scene.forces(), sims)
    ref = oracle.batch_simulate(mo, scene.forces(), sims, workers=4)
    for b in range(B):
        assert_traj_equal(gpu[b], ref[b])
    return gpu, ref


def test_rollout_c1_lbfgs():
    sc = make_single_hinge_chain_scene(10)
    sim = SimConfig(dt=0.01, duration=0.2)
    sim.optimizer.kind = OptimizerKind.lbfgs
    _rollout_case(sc, sim)


def test_rollout_c1_lm():
    sc = make_single_hinge_chain_scene(10)
    sim = SimConfig(dt=0.01, duration=0.2)
    _rollout_case(sc, sim)


def test_rollout_c2_small_batch():
    sc = make_single_hinge_chain_scene(50)
    sim = SimConfig(dt=0.033, duration=0.033 * 4)
    sim.optimizer.kind = OptimizerKind.lbfgs
    _rollout_case(sc, sim, B=3, seed=0)


def test_rollout_c3_two_steps():
    sc = make_chain_scene(100)
    sim = SimConfig(dt=0.1, duration=0.2)
    sim.optimizer.kind = OptimizerKind.lbfgs
    _rollout_case(sc, sim, B=2, seed=1)


def test_rollout_c4_humanoid_lm():
    sc = make_humanoid_scene()
    sim = SimConfig(dt=0.01, duration=0.05)
    gpu, _ = _rollout_case(sc, sim, B=1)


def test_rollout_spider_contact():
    sc = make_spider_scene(api.rotation_vector_matrix)
    sim = SimConfig(dt=0.01, duration=0.04)
    _rollout_case(sc, sim)


def test_rollout_swimmer_drag_actuation():
    sc = make_swimmer_scene()
    sim = SimConfig(dt=0.05, duration=0.2)
    _rollout_case(sc, sim)


def test_rollout_residual_k3():
    sc = make_single_hinge_chain_scene(6)
    sim = SimConfig(dt=0.01, duration=0.03, order=3, objective=ObjectiveKind.residual_form)
    _rollout_case(sc, sim)


def test_fail_limit_reported_like_reference():
    sc = make_chain_scene(100)
    sim = SimConfig(dt=0.1, duration=0.5, consecutive_fail_limit=2)
    sim.optimizer.kind = OptimizerKind.lbfgs
    sim.optimizer.max_iters = 20
    gpu, ref = _rollout_case(sc, sim, B=1, seed=1)
    assert gpu[0].error is not None and gpu[0].error == ref[0].error


def test_nonfinite_q0_isolated_in_batch():
    sc = make_single_hinge_chain_scene(4)
    m = api.build_model(sc.links)
    good = SimConfig(dt=0.01, duration=0.03, q0=np.zeros(4), qdot0=np.zeros(4))
    bad = SimConfig(dt=0.01, duration=0.03, q0=np.array([0.0, np.nan, 0.0, 0.0]), qdot0=np.zeros(4))
    out = api.batch_simulate(m, sc.forces(), [good, bad, good])
    assert out[1].error == "configuration contains a non-finite entry"
    assert out[0].error is None and out[2].error is None
    np.testing.assert_array_equal(out[0].samples[-1][1], out[2].samples[-1][1])


def test_minimize_matches_oracle():
    sc = make_single_hinge_chain_scene(12)
    m = api.build_model(sc.links)
    mo = oracle.Model(sc.links)
    sim = SimConfig(dt=0.02, duration=0.02)
    sim.optimizer.kind = OptimizerKind.lbfgs
    ctx = api.GpuContext(m, sc.forces(), sim, max_batch=2)
    rng = np.random.default_rng(3)
    hist = rng.uniform(-0.3, 0.3, (2, 24))
    x0 = hist[:, 12:].copy()
    xo, it, cv, fv, gnm = ctx.minimize(hist, x0)
    import ctypes as C
    for b in range(2):
        ox = np.zeros(12)
        oit = C.c_int32()
        ocv = C.c_int32()
        ofv = C.c_double()
        ogn = C.c_double()
        cfg = oracle.optimizer_c(sim.optimizer)
        h = np.ascontiguousarray(hist[b])
        xx = np.ascontiguousarray(x0[b])
        f = oracle.forces_c(sc.forces(), 12, [])
        oracle.lib().pbo_step_minimize(mo.h, C.byref(f), 2, 0.02, 0, oracle._ptr(h), None, oracle._ptr(xx),
                                       C.byref(cfg), oracle._ptr(ox), C.byref(oit), C.byref(ocv), C.byref(ofv),
                                       C.byref(ogn), None)
        np.testing.assert_array_equal(xo[b], ox)
        assert it[b] == oit.value and cv[b] == ocv.value and fv[b] == ofv.value


def _random_hinge_chain(seed, links):
    """Hinge chain with tilted axes, rotated offsets and mixed geometry: the
    chain kernel's general (non-specialised) link class."""
    from paper_1709_04145_b200.types import JointKind, JointSpec, LinkSpec
    from _parity_util import random_offset
    rng = np.random.default_rng(seed)
    base = random_tree(rng, links, chain=True)
    out = []
    for i, l in enumerate(base):
        ax = rng.uniform(-1, 1, 3)
        j = JointSpec(JointKind.hinge, tuple(ax / np.linalg.norm(ax)),
                      random_offset(rng) if i % 3 else np.eye(4))
        out.append(LinkSpec(l.parent, j, l.geometry))
    return out


def test_rollout_chain_kernel_general_links():
    from paper_1709_04145_b200.scenes import Scene
    sc = Scene(links=_random_hinge_chain(11, 9), gravity=(0.5, -2.0, -9.81))
    sc.q0 = np.zeros(9)
    sc.qdot0 = np.zeros(9)
    sim = SimConfig(dt=0.02, duration=0.1)
    sim.optimizer.kind = OptimizerKind.lbfgs
    _rollout_case(sc, sim, B=3, seed=5)


def test_rollout_chain_kernel_actuated():
    sc = make_single_hinge_chain_scene(6)
    from paper_1709_04145_b200.types import ActuationKind, ActuationSpec
    sc.actuation = ActuationSpec(ActuationKind.sinusoidal, np.linspace(-3, 3, 6), 1.5, np.linspace(0, 1, 6))
    sim = SimConfig(dt=0.02, duration=0.1)
    sim.optimizer.kind = OptimizerKind.lbfgs
    _rollout_case(sc, sim, B=2, seed=7)


# --- chain kernel v4 (pbad_chain4.cu): warp-synchronous lockstep rounds -----

def _axis_chain(seed, links):
    """Serial chain of axis-aligned hinges (X / Y / Z), pure-translation
    offsets and mixed box / point-mass / massless links: the v4 kernel's
    per-link dispatch path (no compiled link pattern matches)."""
    from paper_1709_04145_b200.types import BoxGeometry, JointKind, JointSpec, LinkSpec, PointMass, PointMassGeometry
    rng = np.random.default_rng(seed)
    out = []
    for i in range(links):
        ax = [(1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0)][int(rng.integers(0, 3))]
        off = np.eye(4)
        if i:
            off[:3, 3] = rng.uniform(-0.6, 0.6, 3)
        u = rng.uniform()
        if u < 0.3:
            g = PointMassGeometry([])
        elif u < 0.5:
            g = PointMassGeometry([PointMass(0.2 + rng.uniform(), tuple(rng.uniform(-0.3, 0.3, 3)))])
        else:
            g = BoxGeometry(tuple(0.1 + rng.uniform(0, 0.5, 3)), 300.0 + 900.0 * rng.uniform(),
                            tuple(rng.uniform(-0.3, 0.3, 3)))
        out.append(LinkSpec(None if i == 0 else i - 1, JointSpec(JointKind.hinge, ax, off), g))
    return out


def _path(scene, sim):
    m = api.build_model(scene.links)
    return api.GpuContext(m, scene.forces(), sim, max_batch=1).path


CHAIN_KERNELS = [("v5", 5), ("v7", 7), ("v6", 6), ("v4", 2)]


def _chain_kernel(monkeypatch, version):
    if version == "v4":
        monkeypatch.setenv("PBAD_GPU_CHAIN_V4", "1")
    if version == "v6":
        monkeypatch.setenv("PBAD_GPU_CHAIN_V6", "1")
    if version == "v7":
        monkeypatch.setenv("PBAD_GPU_CHAIN_V7", "1")


@pytest.mark.parametrize("version,path", CHAIN_KERNELS)
def test_chain4_dispatch_path_ragged_batch(version, path, monkeypatch):
    """13 links (a partial last chunk), 11 environments (a padded warp), the
    generic per-link dispatch: bit-exact against the oracle."""
    _chain_kernel(monkeypatch, version)
    from paper_1709_04145_b200.scenes import Scene
    sc = Scene(links=_axis_chain(21, 13), gravity=(1.0, -2.0, -9.81))
    sc.q0 = np.zeros(13)
    sc.qdot0 = np.zeros(13)
    sim = SimConfig(dt=0.02, duration=0.1)
    sim.optimizer.kind = OptimizerKind.lbfgs
    assert _path(sc, sim) == path
    _rollout_case(sc, sim, B=11, seed=9, lo=-0.5, hi=0.5)


@pytest.mark.parametrize("version,path", CHAIN_KERNELS)
def test_chain4_lockstep_divergent_envs(version, path, monkeypatch):
    """Environments of one warp converge, fail and abort at different
    iterations / steps (max_iters small, fail limit 1)."""
    _chain_kernel(monkeypatch, version)
    sc = make_single_hinge_chain_scene(10)
    sim = SimConfig(dt=0.01, duration=0.08, consecutive_fail_limit=1)
    sim.optimizer.kind = OptimizerKind.lbfgs
    sim.optimizer.max_iters = 60
    assert _path(sc, sim) == path
    gpu, ref = _rollout_case(sc, sim, B=11, seed=3, lo=-1.0, hi=1.0)
    errs = {g.error for g in gpu}
    assert len(errs) >= 1


def test_chain4_matches_chain_v3(monkeypatch):
    """The v3 quad kernel (PBAD_GPU_CHAIN_V3), v4 (PBAD_GPU_CHAIN_V4), v6, v7 and
    v5 produce identical trajectories (all are pinned to the oracle)."""
    sc = make_chain_scene(12)
    sim = SimConfig(dt=0.1, duration=0.3)
    sim.optimizer.kind = OptimizerKind.lbfgs
    m = api.build_model(sc.links)
    n = m.total_dofs
    sims = []
    for b in range(5):
        s = SimConfig(**{**sim.__dict__})
        s.q0 = mt19937_uniform(40 + b, n, -0.3, 0.3)
        s.qdot0 = np.zeros(n)
        sims.append(s)
    assert _path(sc, sim) == 5
    v5 = api.batch_simulate(m, sc.forces(), sims)
    monkeypatch.setenv("PBAD_GPU_CHAIN_V7", "1")
    assert _path(sc, sim) == 7
    v7 = api.batch_simulate(m, sc.forces(), sims)
    monkeypatch.delenv("PBAD_GPU_CHAIN_V7")
    monkeypatch.setenv("PBAD_GPU_CHAIN_V6", "1")
    assert _path(sc, sim) == 6
    v6 = api.batch_simulate(m, sc.forces(), sims)
    monkeypatch.delenv("PBAD_GPU_CHAIN_V6")
    monkeypatch.setenv("PBAD_GPU_CHAIN_V4", "1")
    assert _path(sc, sim) == 2
    v4 = api.batch_simulate(m, sc.forces(), sims)
    monkeypatch.setenv("PBAD_GPU_CHAIN_V3", "1")
    assert _path(sc, sim) == 1
    v3 = api.batch_simulate(m, sc.forces(), sims)
    for a, b, c, d, e in zip(v5, v4, v3, v6, v7):
        for o in (b, c, d, e):
            np.testing.assert_array_equal(np.array([s[1] for s in a.samples]), np.array([s[1] for s in o.samples]))
            assert [r.iterations for r in a.solve_reports] == [r.iterations for r in o.solve_reports]
