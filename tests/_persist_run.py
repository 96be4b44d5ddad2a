"""Helper of the persistent multi-step launch tests (test_gpu_tree.py,
test_gpu_resid.py): one rollout of a scene on the tree or the residual
kernel, results to an .npz.  Run in a subprocess so the PBAD_*_PERSIST
switch, read once per process, can differ between runs."""
import sys

import numpy as np

from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import make_humanoid_scene, make_single_hinge_chain_scene, mt19937_uniform
from paper_1709_04145_b200.types import ContactModel, ObjectiveKind, SimConfig


def scene(kind):
    if kind == "tree_contact":  # C4b's humanoid on the ground plane
        sc = make_humanoid_scene()
        sc.contact = ContactModel(plane_normal=(0.0, 0.0, 1.0), plane_offset=0.0, d1=2e4, d2=2e2)
        return sc
    return make_single_hinge_chain_scene(12)  # "resid": K = 3 collocation on a 12-link chain


def sim(kind, steps):
    if kind == "tree_contact":
        return SimConfig(dt=0.01, duration=0.01 * steps)
    return SimConfig(dt=0.01, duration=0.01 * steps, order=3, objective=ObjectiveKind.residual_form)


def inputs(kind, B, n, q_base):
    q0 = np.empty((B, n))
    for b in range(B):
        if kind == "tree_contact":
            q = q_base.copy()
            q[2] = 0.9
            q[6:] = mt19937_uniform(700 + b, n - 6, -0.1, 0.1)
        else:
            q = mt19937_uniform(900 + b, n, -0.3, 0.3)
        q0[b] = q
    return q0


def main(kind, out_path, B, steps):
    sc = scene(kind)
    m = api.build_model(sc.links)
    n = m.total_dofs
    ctx = api.GpuContext(m, sc.forces(), sim(kind, steps), max_batch=B)
    r = ctx.rollout(inputs(kind, B, n, sc.q0), np.zeros((B, n)), want_q=True, want_energy=True)
    np.savez(out_path, q=r["q"], energy=r["energy"], iterations=r["iterations"], path=ctx.path,
             launches=ctx.kernel_launches())


def run_env(kind, tmp_path, B, steps, tag, **env_vars):
    """The rollout in its own process with the given environment variables."""
    import os
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    p = tmp_path / f"{kind}_{tag}.npz"
    env = dict(os.environ, PYTHONPATH=os.path.dirname(here))
    env.update({k: str(v) for k, v in env_vars.items()})
    subprocess.run([sys.executable, os.path.abspath(__file__), kind, str(p), str(B), str(steps)], check=True, env=env,
                   timeout=900)
    return np.load(p)


def run_pair(kind, tmp_path, B, steps, switch):
    """The rollout with the persistent launch (switch=1) and with one launch
    per step (switch=0), each in its own process."""
    return (run_env(kind, tmp_path, B, steps, "p1", **{switch: 1}),
            run_env(kind, tmp_path, B, steps, "p0", **{switch: 0}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
