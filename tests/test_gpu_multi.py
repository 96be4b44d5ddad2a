"""Multi-context execution on the GPU: a batch sharded over
several contexts (pbad_gpu_rollout_sharded) equals one context's rollout bit
for bit; windowed trajectory output (PBAD_TRAJ_WINDOW_MB) equals the
whole-trajectory output; the device-side final-state copy that feeds the NCCL
gather equals the last recorded samples; and `bench.py --gpus 2` runs two
ranks (on one device here: the oversubscribed dry run) and reports n_gpus 2."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import bench
from paper_1709_04145_b200 import api

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("q", "energy", "iterations", "converged", "accepted", "final_value", "final_grad_norm", "n_samples",
        "status", "fail_streak", "n_reports")


def _case(name, steps, batch, max_iters=None):
    cfg = dict(bench.CONFIGS[name])
    scene = bench.build_scene(cfg)
    model = api.build_model(scene.links)
    n = model.total_dofs
    sim = bench.sim_config(cfg, steps, 25)
    if max_iters is not None:
        sim.optimizer.max_iters = max_iters
    q0 = bench.initial_states(cfg, scene, n, 0, batch)
    return scene, model, sim, q0


def _equal(a, b):
    for k in KEYS:
        if a[k] is None:
            continue
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


@pytest.mark.parametrize("name,steps,batch,max_iters,shards", [
    ("C2", 3, 40, None, 2),    # chain path, ragged blocks
    ("C4b", 4, 70, None, 3),   # tree Newton path with contact
    ("C5", 1, 5, 4, 2),        # residual path
])
def test_sharded_equals_single(name, steps, batch, max_iters, shards):
    scene, model, sim, q0 = _case(name, steps, batch, max_iters)
    qd = np.zeros_like(q0)
    one = api.GpuContext(model, scene.forces(), sim, max_batch=batch).rollout(q0, qd)
    per = -(-batch // shards)
    ctxs = [api.GpuContext(model, scene.forces(), sim, device=0, max_batch=per) for _ in range(shards)]
    got = api.rollout_sharded(ctxs, q0, qd)
    _equal(got, one)


def test_sharded_rejects_bad_shards():
    scene, model, sim, q0 = _case("C2", 1, 10)
    c = api.GpuContext(model, scene.forces(), sim, max_batch=3)
    with pytest.raises(ValueError):
        api.rollout_sharded([c, c], q0, np.zeros_like(q0))  # the same context twice
    c2 = api.GpuContext(model, scene.forces(), sim, max_batch=3)
    with pytest.raises(ValueError):
        api.rollout_sharded([c, c2], q0, np.zeros_like(q0))  # 5 envs per shard > max_batch 3


def test_batch_simulate_devices_list():
    scene, model, sim, q0 = _case("C4", 3, 9)
    sims = []
    for b in range(9):
        s = type(sim)(**{**sim.__dict__})
        s.q0 = q0[b]
        s.qdot0 = np.zeros(model.total_dofs)
        sims.append(s)
    a = api.batch_simulate(model, scene.forces(), sims)
    b = api.batch_simulate(model, scene.forces(), sims, devices=[0, 0, 0])
    for x, y in zip(a, b):
        np.testing.assert_array_equal(np.array([s[1] for s in x.samples]), np.array([s[1] for s in y.samples]))
        assert [r.iterations for r in x.solve_reports] == [r.iterations for r in y.solve_reports]
        assert x.error == y.error


@pytest.mark.parametrize("name,steps,batch", [("C1", 40, 16), ("C4", 12, 33)])
def test_windowed_output_equals_whole(name, steps, batch, monkeypatch):
    scene, model, sim, q0 = _case(name, steps, batch)
    qd = np.zeros_like(q0)
    whole = api.GpuContext(model, scene.forces(), sim, max_batch=batch).rollout(q0, qd)
    n = model.total_dofs
    # a budget of about 5 steps of this batch: 8+ windows, the last one ragged
    mb = 5 * batch * (8.0 * (n + 2) + 28.0) / 1048576.0
    monkeypatch.setenv("PBAD_TRAJ_WINDOW_MB", repr(mb))
    win = api.GpuContext(model, scene.forces(), sim, max_batch=batch).rollout(q0, qd)
    _equal(win, whole)


def test_final_state_device_copy():
    import torch
    scene, model, sim, q0 = _case("C2", 4, 24)
    ctx = api.GpuContext(model, scene.forces(), sim, max_batch=24)
    dq = torch.from_numpy(q0).cuda()
    dqd = torch.zeros_like(dq)
    torch.cuda.synchronize()
    ctx.begin(24, dq.data_ptr(), dqd.data_ptr())
    ctx.advance(4)
    fin = torch.empty_like(dq)
    ctx.final_state(fin.data_ptr())
    out = ctx.sync_outputs()
    torch.cuda.synchronize()
    last = np.stack([out["q"][b, out["n_samples"][b] - 1] for b in range(24)])
    np.testing.assert_array_equal(fin.cpu().numpy(), last)


def test_bench_two_ranks_dry_run():
    """bench.py --gpus 2 re-launches itself as two ranks (torchrun), each
    rank steps its own shard and the line reports the whole job."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                        "--config", "C4", "--no-cpu-baseline"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    assert d["config"]["global_batch"] == 2 * bench.CONFIGS["C4"]["batch"]
    assert d["gathered_envs"] == 2 * bench.CONFIGS["C4"]["batch"]
    assert d["value"] > 0 and d["e2e"]["value"] > 0
