import time, numpy as np, sys
sys.path.insert(0, '.')
from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import *
from paper_1709_04145_b200.types import *
import torch
for (name, sc, dt, B, steps, kind) in [("C1", make_single_hinge_chain_scene(10), 0.01, 1024, 5, OptimizerKind.lbfgs),
                                        ("C2", make_single_hinge_chain_scene(50), 0.033, 1024, 3, OptimizerKind.lbfgs),
                                        ("C3", make_chain_scene(100), 0.1, 4096, 1, OptimizerKind.lbfgs),
                                        ("C4", make_humanoid_scene(), 0.01, 4096, 3, OptimizerKind.lm)]:
    m = api.build_model(sc.links); n = m.total_dofs
    sim = SimConfig(dt=dt, duration=dt*steps, consecutive_fail_limit=1000); sim.optimizer.kind = kind
    ctx = api.GpuContext(m, sc.forces(), sim, max_batch=B)
    q0 = mt19937_uniform(1, B*n, -0.3, 0.3).reshape(B, n) if name != "C4" else np.tile(sc.q0, (B,1))
    t = time.time(); out = ctx.rollout(q0, np.zeros((B, n)), want_q=False); el = time.time()-t
    it = out['iterations'].sum()
    print(name, "B", B, "steps", steps, "device_ms", out['device_ms'][0], "wall", el, "mean iters/step", it / (B*steps), "env-steps/s", B*steps/(out['device_ms'][0]/1e3), flush=True)
