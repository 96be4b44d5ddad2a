"""Per-step LM/L-BFGS iteration distribution of a bench config (for load
balance / scheduling decisions): python scripts/iter_dist.py C4b 4096 20"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1709_04145_b200 import api  # noqa: E402

name, B, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = bench.CONFIGS[name]
scene = bench.build_scene(cfg)
m = api.build_model(scene.links)
n = m.total_dofs
sim = bench.sim_config(cfg, steps, 1 << 30)
ctx = api.GpuContext(m, scene.forces(), sim, max_batch=B)
q0 = bench.initial_states(cfg, scene, n, 0, B)
t = time.time()
out = ctx.rollout(q0, np.zeros((B, n)), want_q=False)
it = out["iterations"]
print(name, "B", B, "steps", steps, "path", ctx.path, "device_ms", round(out["device_ms"][0], 1))
for s in range(steps):
    x = it[:, s]
    print(f"step {s:3d} mean {x.mean():7.1f} p50 {np.percentile(x, 50):5.0f} p90 {np.percentile(x, 90):5.0f} "
          f"p99 {np.percentile(x, 99):5.0f} max {x.max():4d}  sum/max*slots {x.sum() / max(1, x.max()):8.1f}")
