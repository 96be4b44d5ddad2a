"""Run one configuration's rollout with the bench's inputs (for ncu):
    python scripts/prof_run.py C3 4096 1 [max_iters]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1709_04145_b200 import api  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = bench.CONFIGS[cfg_name]
scene = bench.build_scene(cfg)
m = api.build_model(scene.links)
n = m.total_dofs
sim = bench.sim_config(cfg, steps, 1000)
if len(sys.argv) > 4:
    sim.optimizer.max_iters = int(sys.argv[4])
ctx = api.GpuContext(m, scene.forces(), sim, max_batch=B)
q0 = bench.initial_states(cfg, scene, n, 0, B)
out = ctx.rollout(q0, np.zeros((B, n)), want_q=False)
print(cfg_name, "B", B, "steps", steps, "path", ctx.path, "device_ms", out["device_ms"][0], "iters",
      out["iterations"].mean())
