"""N>1 host logic on CPU: two gloo ranks each own a contiguous shard of the
global env batch (bench.py's weak-scaling partition), step
it independently (the CPU oracle stands in for the device on this box), and
gather the final states to rank 0.  The gathered result must be bit-identical
to a single-process run over the whole batch: environments are independent,
so sharding introduces no exchange and no numerical difference."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_states(rank, world, per_rank, out_dict):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import bench
    import oracle
    cfg = dict(bench.CONFIGS["C2"])
    cfg["links"] = 6
    scene = bench.build_scene(cfg)
    n = 6
    q0 = bench.initial_states(cfg, scene, n, rank * per_rank, per_rank)
    sims = []
    for b in range(per_rank):
        s = bench.sim_config(cfg, 2, 1 << 30)
        s.q0 = q0[b]
        s.qdot0 = np.zeros(n)
        sims.append(s)
    trs = oracle.batch_simulate(oracle.Model(scene.links), scene.forces(), sims, workers=1)
    fin = torch.from_numpy(np.stack([t.q[t.n_samples - 1] for t in trs]))
    allq = [torch.empty_like(fin) for _ in range(world)]
    dist.all_gather(allq, fin)
    if rank == 0:
        out_dict["gathered"] = torch.cat(allq).numpy()


def _worker(rank, world, port, per_rank, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = {}
    _shard_states(rank, world, per_rank, d)
    if rank == 0:
        ret.put(d["gathered"])
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_and_gather_matches_single_process():
    sys.path.insert(0, ROOT)
    import bench
    import oracle
    world, per_rank = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = dict(bench.CONFIGS["C2"])
    cfg["links"] = 6
    scene = bench.build_scene(cfg)
    q0 = bench.initial_states(cfg, scene, 6, 0, world * per_rank)
    sims = []
    for b in range(world * per_rank):
        s = bench.sim_config(cfg, 2, 1 << 30)
        s.q0 = q0[b]
        s.qdot0 = np.zeros(6)
        sims.append(s)
    trs = oracle.batch_simulate(oracle.Model(scene.links), scene.forces(), sims, workers=2)
    ref = np.stack([t.q[t.n_samples - 1] for t in trs])
    assert np.array_equal(gathered, ref)


def test_shard_partition_is_contiguous_slice_of_global_draws():
    sys.path.insert(0, ROOT)
    import bench
    cfg = bench.CONFIGS["C3"]
    scene = bench.build_scene(cfg)
    full = bench.initial_states(cfg, scene, 200, 0, 16)
    parts = [bench.initial_states(cfg, scene, 200, r * 4, 4) for r in range(4)]
    assert np.array_equal(np.concatenate(parts), full)
