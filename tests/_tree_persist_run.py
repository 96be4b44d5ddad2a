"""Helper of test_gpu_tree.py::test_tree_persistent_multistep_contact: one
contact-humanoid rollout on the tree kernel, results to an .npz (run in a
subprocess so PBAD_TREE_PERSIST, read once per process, can differ)."""
import sys

import numpy as np

from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import make_humanoid_scene, mt19937_uniform
from paper_1709_04145_b200.types import ContactModel, SimConfig


def scene():
    sc = make_humanoid_scene()
    sc.contact = ContactModel(plane_normal=(0.0, 0.0, 1.0), plane_offset=0.0, d1=2e4, d2=2e2)
    return sc


def inputs(B, n, q_base):
    q0 = np.empty((B, n))
    for b in range(B):
        q = q_base.copy()
        q[2] = 0.9
        q[6:] = mt19937_uniform(700 + b, n - 6, -0.1, 0.1)
        q0[b] = q
    return q0


def main(out_path, B, steps):
    sc = scene()
    m = api.build_model(sc.links)
    n = m.total_dofs
    sim = SimConfig(dt=0.01, duration=0.01 * steps)
    ctx = api.GpuContext(m, sc.forces(), sim, max_batch=B)
    r = ctx.rollout(inputs(B, n, sc.q0), np.zeros((B, n)), want_q=True, want_energy=True)
    np.savez(out_path, q=r["q"], energy=r["energy"], iterations=r["iterations"], path=ctx.path,
             launches=ctx.kernel_launches())


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
