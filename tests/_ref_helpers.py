"""Test fixtures mirroring /root/reference/proj/tests/test_helpers.hpp."""
import numpy as np

import oracle
from paper_1709_04145_b200.types import (BoxGeometry, JointKind, JointSpec, LinkSpec, PointMass,
                                         PointMassGeometry)

FD_STEP = 1e-5  # kFdStep, test_helpers.hpp:12


def rel_err(a, b):
    """max|a-b| / max(1, max|b|) (test_helpers.hpp:14-26)."""
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b))) if b.size else 1.0))


def fd_gradient(f, x, h=FD_STEP):
    g = np.zeros(len(x))
    for i in range(len(x)):
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        g[i] = (f(xp) - f(xm)) / (2 * h)
    return g


def fd_jacobian(f, x, h=FD_STEP):
    cols = []
    for j in range(len(x)):
        xp, xm = x.copy(), x.copy()
        xp[j] += h
        xm[j] -= h
        cols.append((np.asarray(f(xp)) - np.asarray(f(xm))) / (2 * h))
    return np.array(cols).T


def random_offset(rng):
    m = np.eye(4)
    m[:3, :3] = oracle.rotation_vector_matrix(rng.uniform(-0.5, 0.5, 3))
    m[:3, 3] = 2 * rng.uniform(-0.5, 0.5, 3)
    return m


def random_tree(rng, links, chain=False):
    """test_helpers.hpp:75-116: hinge/ball/free joints, boxes and point masses."""
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


def planar_chain(links, axis=(0.0, 0.0, 1.0)):
    """test_helpers.hpp:119-136."""
    specs = []
    for i in range(links):
        off = np.eye(4)
        off[0, 3] = 1.0
        specs.append(LinkSpec(None if i == 0 else i - 1, JointSpec(JointKind.hinge, axis, off),
                              BoxGeometry((1.0, 0.1, 0.1), 1000.0, (0.5, 0.0, 0.0))))
    return specs


def naive_correlation(model, S, mass, qa, qb):
    """test_helpers.hpp:140-150: direct sum over world transforms."""
    ta = oracle.forward_pass(model, qa)
    tb = oracle.forward_pass(model, qb)
    v = 0.0
    for i in range(model.n_links):
        v += np.trace(ta[i].T @ tb[i] @ S[i]) - mass[i]
    return v
