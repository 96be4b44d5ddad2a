"""Run one configuration's rollout (for ncu): python scripts/prof_run.py C3 4096 1"""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import *
from paper_1709_04145_b200.types import *

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
table = {"C1": (make_single_hinge_chain_scene(10), 0.01, OptimizerKind.lbfgs),
         "C2": (make_single_hinge_chain_scene(50), 0.033, OptimizerKind.lbfgs),
         "C3": (make_chain_scene(100), 0.1, OptimizerKind.lbfgs),
         "C4": (make_humanoid_scene(), 0.01, OptimizerKind.lm),
         "C5": (make_single_hinge_chain_scene(100), 0.01, OptimizerKind.lm)}
sc, dt, kind = table[cfg]
m = api.build_model(sc.links); n = m.total_dofs
sim = SimConfig(dt=dt, duration=dt * steps, consecutive_fail_limit=1000)
if cfg == "C5":
    sim.order, sim.objective = 4, ObjectiveKind.residual_form
sim.optimizer.kind = kind
if len(sys.argv) > 4:
    sim.optimizer.max_iters = int(sys.argv[4])
ctx = api.GpuContext(m, sc.forces(), sim, max_batch=B)
q0 = mt19937_uniform(1, B * n, -0.3, 0.3).reshape(B, n) if cfg != "C4" else np.tile(sc.q0, (B, 1))
out = ctx.rollout(q0, np.zeros((B, n)), want_q=False)
print(cfg, "B", B, "steps", steps, "device_ms", out["device_ms"][0], "iters", out["iterations"].mean())
