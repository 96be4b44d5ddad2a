#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref: the
unmodified /root/reference/proj sources compiled against eigen_lite).

    make -C oracle/ref && python scripts/make_golden.py

Each fixture stores the inputs (scene name, schedule, q0) and the reference's
outputs (samples, energy log, per-step iterations / converged / final value,
or per-evaluation value / grad / GN).  Committed so parity stays pinned on
machines without /root/reference (the GPU box)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1709_04145_b200.scenes import (make_chain_scene, make_humanoid_scene,  # noqa: E402
                                          make_single_hinge_chain_scene, make_spider_scene, mt19937_uniform)
from paper_1709_04145_b200.types import ObjectiveKind, OptimizerKind, SimConfig  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

ROLLOUTS = {
    # name: (scene, dt, steps, optimizer, order, seed or None, lo/hi)
    "c1_lbfgs": ("single_hinge10", 0.01, 20, "lbfgs", 2, None),
    "c2_lbfgs": ("single_hinge50", 0.033, 3, "lbfgs", 2, 0),
    "c3_lbfgs": ("chain100", 0.1, 2, "lbfgs", 2, 1),
    "c4_lm": ("humanoid", 0.01, 5, "lm", 2, 2),
    "spider_lm": ("spider", 0.01, 5, "lm", 2, None),
    "residual_k4": ("single_hinge6", 0.01, 3, "lm", 4, 3),
}


def scene(name):
    if name.startswith("single_hinge"):
        return make_single_hinge_chain_scene(int(name[len("single_hinge"):]))
    if name == "chain100":
        return make_chain_scene(100)
    if name == "humanoid":
        return make_humanoid_scene()
    if name == "spider":
        return make_spider_scene(oracle.rotation_vector_matrix)
    raise KeyError(name)


def initial(name, sc, n, seed):
    if seed is None:
        return sc.q0.copy()
    if name == "humanoid":
        q = sc.q0.copy()
        q[6:] = mt19937_uniform(seed, n - 6, -0.1, 0.1)
        return q
    return mt19937_uniform(seed, n, -0.3, 0.3)


def main():
    assert oracle.ref_available(), "build oracle/_ref first (make -C oracle/ref)"
    os.makedirs(OUT, exist_ok=True)
    for key, (sname, dt, steps, opt, order, seed) in ROLLOUTS.items():
        sc = scene(sname)
        R = oracle.RefModel(sc.links)
        n = R.n_dofs
        s = SimConfig(dt=dt, duration=dt * steps, order=order,
                      objective=ObjectiveKind.energy_form if order == 2 else ObjectiveKind.residual_form)
        s.optimizer.kind = OptimizerKind.lbfgs if opt == "lbfgs" else OptimizerKind.lm
        s.q0 = initial(sname, sc, n, seed)
        s.qdot0 = np.zeros(n)
        tr = oracle.ref_batch_simulate(R, sc.forces(), [s])[0]
        k = tr.n_samples
        np.savez_compressed(os.path.join(OUT, f"rollout_{key}.npz"), scene=sname, dt=dt, steps=steps, optimizer=opt,
                            order=order, q0=s.q0, q=tr.q[:k], energy=tr.energy[:k], iterations=tr.iterations[:k - 1],
                            converged=tr.converged[:k - 1], final_value=tr.final_value[:k - 1])
        print(key, "samples", k, "iterations", tr.iterations[:k - 1].tolist())
    rng = np.random.default_rng(2024)
    for sname, order, obj in (("humanoid", 2, 0), ("chain100", 2, 0), ("spider", 2, 0), ("single_hinge6", 4, 1)):
        sc = scene(sname)
        R = oracle.RefModel(sc.links)
        n = R.n_dofs
        u = order - 1
        h0 = sc.q0 + rng.uniform(-0.1, 0.1, n)
        h1 = sc.q0 + rng.uniform(-0.1, 0.1, n)
        x = np.tile(h1, u) + rng.uniform(-0.05, 0.05, n * u)
        v, g, gn = oracle.ref_step_eval(R, sc.forces(), order, 0.01, obj, h0, h1, x, True, True)
        np.savez_compressed(os.path.join(OUT, f"eval_{sname}_k{order}.npz"), scene=sname, order=order, objective=obj,
                            dt=0.01, h0=h0, h1=h1, x=x, value=v, grad=g, gn=gn)
        print("eval", sname, order, v)


if __name__ == "__main__":
    main()
