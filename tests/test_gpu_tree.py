"""GPU parity of the tree (warp-per-environment Newton / LM) kernel,
pbad_tree.cu, against the CPU oracle: bit-exact trajectories, iteration
counts, convergence flags, final objective values and energy logs
(the north-star Newton-path gates: Hessian/GN within 1e-10, iteration counts
equal, positions within 1e-8, all implied by bit equality)."""
import numpy as np
import pytest

import oracle
from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import Scene, make_humanoid_scene, make_single_hinge_chain_scene, mt19937_uniform
from paper_1709_04145_b200.types import ActuationKind, ActuationSpec, OptimizerKind, SimConfig

from _parity_util import assert_traj_equal, random_tree

pytestmark = pytest.mark.gpu

PATH_TREE = 3


def _sims(sim, n, B, q0_fn):
    out = []
    for b in range(B):
        s = SimConfig(**{**sim.__dict__})
        s.q0 = q0_fn(b)
        s.qdot0 = np.zeros(n)
        out.append(s)
    return out


def _humanoid_q0(scene, n, seed):
    def f(b):
        q = scene.q0.copy()
        q[6:] = mt19937_uniform(seed + b, n - 6, -0.1, 0.1)
        return q
    return f


def _check(scene, sim, sims, path=PATH_TREE):
    m = api.build_model(scene.links)
    ctx = api.GpuContext(m, scene.forces(), sim, max_batch=1)
    assert ctx.path == path, ctx.path
    gpu = api.batch_simulate(m, scene.forces(), sims)
    ref = oracle.batch_simulate(oracle.Model(scene.links), scene.forces(), sims, workers=4)
    for g, r in zip(gpu, ref):
        assert_traj_equal(g, r)
    return gpu, ref


def test_tree_path_humanoid_lm():
    sc = make_humanoid_scene()
    sim = SimConfig(dt=0.01, duration=0.05)
    n = 41
    _check(sc, sim, _sims(sim, n, 5, _humanoid_q0(sc, n, 2)))


def test_tree_path_single_hinge_chain_lm():
    sc = make_single_hinge_chain_scene(10)
    sim = SimConfig(dt=0.01, duration=0.1)
    _check(sc, sim, _sims(sim, 10, 3, lambda b: mt19937_uniform(b, 10, -0.5, 0.5)))


@pytest.mark.parametrize("seed", [31, 32, 33, 34])
def test_tree_path_random_trees(seed):
    """Mixed hinge / ball / free joints, rotated offsets, box and point-mass
    links, tilted gravity, random branching."""
    rng = np.random.default_rng(seed)
    links = random_tree(rng, 6 + seed % 5)
    sc = Scene(links=links, gravity=(0.4, -1.0, -9.81))
    m = api.build_model(links)
    n = m.total_dofs
    sc.q0 = np.zeros(n)
    sc.qdot0 = np.zeros(n)
    sim = SimConfig(dt=0.02, duration=0.1)
    _check(sc, sim, _sims(sim, n, 3, lambda b: rng.uniform(-0.4, 0.4, n)))


@pytest.mark.parametrize("kind", [ActuationKind.constant, ActuationKind.sinusoidal])
def test_tree_path_actuated(kind):
    sc = make_humanoid_scene()
    n = 41
    sc.actuation = ActuationSpec(kind, np.linspace(-2.0, 2.0, n), 2.0, np.linspace(0.0, 1.0, n))
    sim = SimConfig(dt=0.01, duration=0.04)
    _check(sc, sim, _sims(sim, n, 2, _humanoid_q0(sc, n, 9)))


def test_tree_path_zero_gravity():
    rng = np.random.default_rng(5)
    links = random_tree(rng, 7)
    sc = Scene(links=links, gravity=(0.0, 0.0, 0.0))
    m = api.build_model(links)
    n = m.total_dofs
    sc.q0 = np.zeros(n)
    sc.qdot0 = np.zeros(n)
    sim = SimConfig(dt=0.02, duration=0.06)
    _check(sc, sim, _sims(sim, n, 2, lambda b: rng.uniform(-0.4, 0.4, n)))


def test_tree_path_fail_limit_and_divergent_envs():
    """max_iters small and fail limit 1: environments abort at different
    steps; the per-trajectory errors match the reference's text."""
    sc = make_humanoid_scene()
    sim = SimConfig(dt=0.05, duration=0.3, consecutive_fail_limit=1)
    sim.optimizer.max_iters = 3
    n = 41
    gpu, ref = _check(sc, sim, _sims(sim, n, 6, _humanoid_q0(sc, n, 17)))
    assert any(g.error for g in gpu)


def test_tree_path_nonfinite_q0_isolated():
    sc = make_humanoid_scene()
    m = api.build_model(sc.links)
    sim = SimConfig(dt=0.01, duration=0.03)
    good = SimConfig(**{**sim.__dict__})
    good.q0 = sc.q0.copy()
    good.qdot0 = np.zeros(41)
    bad = SimConfig(**{**sim.__dict__})
    bad.q0 = sc.q0.copy()
    bad.q0[7] = np.inf
    bad.qdot0 = np.zeros(41)
    out = api.batch_simulate(m, sc.forces(), [good, bad, good])
    assert out[1].error == "configuration contains a non-finite entry"
    assert out[0].error is None and out[2].error is None
    np.testing.assert_array_equal(out[0].samples[-1][1], out[2].samples[-1][1])


def test_tree_path_equals_general_kernel(monkeypatch):
    """Tree kernel and the general thread-per-environment kernel agree bit for
    bit on a ragged batch (33 environments)."""
    sc = make_humanoid_scene()
    sim = SimConfig(dt=0.01, duration=0.03)
    n = 41
    m = api.build_model(sc.links)
    sims = _sims(sim, n, 33, _humanoid_q0(sc, n, 100))
    a = api.batch_simulate(m, sc.forces(), sims)
    monkeypatch.setenv("PBAD_GPU_FORCE_GENERAL", "1")
    assert api.GpuContext(m, sc.forces(), sim, max_batch=1).path == 0
    b = api.batch_simulate(m, sc.forces(), sims)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(np.array([s[1] for s in x.samples]), np.array([s[1] for s in y.samples]))
        assert [r.iterations for r in x.solve_reports] == [r.iterations for r in y.solve_reports]
        assert [r.final_value for r in x.solve_reports] == [r.final_value for r in y.solve_reports]


# --- potentials on the tree path: drag and ground contact (objective.cpp:60-131) ---

def _humanoid_contact():
    from paper_1709_04145_b200.types import ContactModel
    sc = make_humanoid_scene()
    sc.contact = ContactModel(plane_normal=(0.0, 0.0, 1.0), plane_offset=0.0, d1=2e4, d2=2e2)
    return sc


def test_tree_path_humanoid_contact_c4b():
    """C4b: the humanoid dropped onto the ground plane (pelvis lowered so the
    feet are in contact from the first step)."""
    sc = _humanoid_contact()
    sim = SimConfig(dt=0.01, duration=0.06)
    n = 41

    def q0(b):
        q = sc.q0.copy()
        q[2] = 0.9
        q[6:] = mt19937_uniform(60 + b, n - 6, -0.1, 0.1)
        return q
    _check(sc, sim, _sims(sim, n, 4, q0))


@pytest.mark.parametrize("seed", [51, 52])
def test_tree_path_drag_contact_random_trees(seed):
    from paper_1709_04145_b200.types import ContactModel
    rng = np.random.default_rng(seed)
    links = random_tree(rng, 6)
    sc = Scene(links=links, gravity=(0.2, -0.5, -9.81), drag_d=0.8,
               contact=ContactModel(plane_normal=(0.0, 0.3, 0.95), plane_offset=0.4, d1=5e3, d2=50.0))
    m = api.build_model(links)
    n = m.total_dofs
    sc.q0 = np.zeros(n)
    sc.qdot0 = np.zeros(n)
    sim = SimConfig(dt=0.02, duration=0.08)
    _check(sc, sim, _sims(sim, n, 3, lambda b: rng.uniform(-0.5, 0.5, n)))


def test_tree_path_drag_only_zero_gravity():
    rng = np.random.default_rng(7)
    links = random_tree(rng, 5)
    sc = Scene(links=links, gravity=(0.0, 0.0, 0.0), drag_d=2.0)
    m = api.build_model(links)
    n = m.total_dofs
    sc.q0 = np.zeros(n)
    sc.qdot0 = np.zeros(n)
    sim = SimConfig(dt=0.02, duration=0.06)
    _check(sc, sim, _sims(sim, n, 2, lambda b: rng.uniform(-0.4, 0.4, n)))


def test_tree_path_contact_equals_general_kernel(monkeypatch):
    sc = _humanoid_contact()
    sim = SimConfig(dt=0.01, duration=0.03)
    n = 41
    m = api.build_model(sc.links)

    def q0(b):
        q = sc.q0.copy()
        q[2] = 0.85
        q[6:] = mt19937_uniform(80 + b, n - 6, -0.1, 0.1)
        return q
    sims = _sims(sim, n, 9, q0)
    a = api.batch_simulate(m, sc.forces(), sims)
    monkeypatch.setenv("PBAD_GPU_FORCE_GENERAL", "1")
    b = api.batch_simulate(m, sc.forces(), sims)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(np.array([s[1] for s in x.samples]), np.array([s[1] for s in y.samples]))
        assert [r.iterations for r in x.solve_reports] == [r.iterations for r in y.solve_reports]


# --- L-BFGS on trees (LbfgsSolver, optim.cpp:141-232) ---

def test_tree_path_humanoid_lbfgs():
    sc = make_humanoid_scene()
    sim = SimConfig(dt=0.01, duration=0.04)
    sim.optimizer.kind = OptimizerKind.lbfgs
    n = 41
    _check(sc, sim, _sims(sim, n, 4, _humanoid_q0(sc, n, 7)))


@pytest.mark.parametrize("seed,mem", [(61, 8), (62, 3)])
def test_tree_path_lbfgs_random_trees_contact(seed, mem):
    from paper_1709_04145_b200.types import ContactModel
    rng = np.random.default_rng(seed)
    links = random_tree(rng, 6)
    sc = Scene(links=links, gravity=(0.2, -0.5, -9.81), drag_d=0.5,
               contact=ContactModel(plane_normal=(0.0, 0.0, 1.0), plane_offset=0.3, d1=5e3, d2=20.0))
    m = api.build_model(links)
    n = m.total_dofs
    sc.q0 = np.zeros(n)
    sc.qdot0 = np.zeros(n)
    sim = SimConfig(dt=0.02, duration=0.08)
    sim.optimizer.kind = OptimizerKind.lbfgs
    sim.optimizer.lbfgs_memory = mem
    _check(sc, sim, _sims(sim, n, 3, lambda b: rng.uniform(-0.5, 0.5, n)))


def test_tree_path_lbfgs_equals_general_kernel(monkeypatch):
    sc = make_humanoid_scene()
    sim = SimConfig(dt=0.01, duration=0.03)
    sim.optimizer.kind = OptimizerKind.lbfgs
    sim.optimizer.max_iters = 40
    n = 41
    m = api.build_model(sc.links)
    sims = _sims(sim, n, 17, _humanoid_q0(sc, n, 300))
    a = api.batch_simulate(m, sc.forces(), sims)
    monkeypatch.setenv("PBAD_GPU_FORCE_GENERAL", "1")
    b = api.batch_simulate(m, sc.forces(), sims)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(np.array([s[1] for s in x.samples]), np.array([s[1] for s in y.samples]))
        assert [r.iterations for r in x.solve_reports] == [r.iterations for r in y.solve_reports]


def test_tree_persistent_multistep_contact(tmp_path):
    """Contact scenes run a window of steps in one persistent launch
    (k_tree_steps, pbad_tree.cu): warps claim tasks (PBAD_TREE_CHUNK
    consecutive steps of one environment) in order and wait for the
    environment's previous task, which ran on another SM.  With a batch
    larger than the resident warps and 1- or 2-step tasks, environments change
    SM between steps.  The whole batch is bit-identical to one launch per
    step (PBAD_TREE_PERSIST=0) for task lengths 1, 2 and the default, and a
    sample matches the oracle."""
    import _persist_run as pr
    B, steps = 2500, 5
    per = pr.run_env("tree_contact", tmp_path, B, steps, "per_step", PBAD_TREE_PERSIST=0)
    assert int(per["launches"]) == steps
    for chunk in (1, 2, None):
        env = {"PBAD_TREE_PERSIST": 1}
        if chunk:
            env["PBAD_TREE_CHUNK"] = chunk
        one = pr.run_env("tree_contact", tmp_path, B, steps, f"chunk{chunk}", **env)
        assert int(one["path"]) == PATH_TREE
        assert int(one["launches"]) == 1
        for k in ("q", "energy", "iterations"):
            np.testing.assert_array_equal(one[k], per[k])
    assert one["iterations"].max() > one["iterations"].min()  # the iteration counts do vary
    sc = pr.scene("tree_contact")
    n = 41
    q0 = pr.inputs("tree_contact", B, n, sc.q0)
    sim = pr.sim("tree_contact", steps)
    envs = [0, 1777, B - 1]
    ref = oracle.batch_simulate(oracle.Model(sc.links), sc.forces(), _sims(sim, n, len(envs), lambda i: q0[envs[i]]),
                                workers=3)
    for i, b in enumerate(envs):
        k = ref[i].n_samples
        np.testing.assert_array_equal(one["q"][b, :k], ref[i].q[:k])
        np.testing.assert_array_equal(one["iterations"][b, :len(ref[i].iterations)], ref[i].iterations)
