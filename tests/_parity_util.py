"""Shared helpers for parity tests (trajectory comparison, random trees)."""
import numpy as np

from paper_1709_04145_b200.types import (BoxGeometry, JointKind, JointSpec, LinkSpec, PointMass,
                                         PointMassGeometry)


def assert_traj_equal(gpu, ref, exact=True):
    """Bit-exact comparison of a GPU Trajectory with an oracle trajectory."""
    k = ref.n_samples
    assert len(gpu.samples) == k, (len(gpu.samples), k)
    q = np.array([s[1] for s in gpu.samples])
    e = np.array([[x.kinetic, x.potential] for x in gpu.energy_log])
    its = np.array([r.iterations for r in gpu.solve_reports], dtype=np.int32)
    conv = np.array([r.converged for r in gpu.solve_reports], dtype=np.int32)
    nrep = len(gpu.solve_reports)
    np.testing.assert_array_equal(its, ref.iterations[:nrep])
    np.testing.assert_array_equal(conv, ref.converged[:nrep])
    if exact:
        np.testing.assert_array_equal(q, ref.q[:k])
        np.testing.assert_array_equal(e, ref.energy[:k])
        fv = np.array([r.final_value for r in gpu.solve_reports])
        np.testing.assert_array_equal(fv, ref.final_value[:nrep])
    else:
        np.testing.assert_allclose(q, ref.q[:k], rtol=0, atol=1e-8)
    assert (gpu.error or None) == ref.error, (gpu.error, ref.error)


def random_offset(rng):
    from paper_1709_04145_b200 import api
    m = np.eye(4)
    m[:3, :3] = api.rotation_vector_matrix(rng.uniform(-0.5, 0.5, 3))
    m[:3, 3] = rng.uniform(-1.0, 1.0, 3)
    return m


def random_tree(rng, links, chain=False):
    """test_helpers.hpp:75-116 analogue: mixed hinge/ball/free, box/point masses."""
    specs = []
    for i in range(links):
        parent = None if i == 0 else (i - 1 if chain else int(rng.integers(0, i)))
        kind = rng.uniform()
        if i == 0 and kind < 0.3:
            j = JointSpec(JointKind.free_joint)
        elif kind < 0.55:
            j = JointSpec(JointKind.ball)
        else:
            ax = rng.uniform(-0.5, 0.5, 3)
            if np.linalg.norm(ax) < 1e-3:
                ax = np.array([0.0, 0.0, 1.0])
            j = JointSpec(JointKind.hinge, tuple(ax / np.linalg.norm(ax)))
        j.offset = random_offset(rng)
        if rng.uniform() < 0.25:
            cnt = 1 + int(rng.uniform() * 3)
            g = PointMassGeometry([PointMass(0.1 + rng.uniform(), tuple(rng.uniform(-0.5, 0.5, 3)))
                                   for _ in range(cnt)])
        else:
            g = BoxGeometry(tuple(0.2 + rng.uniform(0, 1, 3)), 200.0 + 1800.0 * rng.uniform(),
                            tuple(rng.uniform(-0.5, 0.5, 3)))
        specs.append(LinkSpec(parent, j, g))
    return specs
