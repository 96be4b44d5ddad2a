"""The reference's own unit tests, ported onto the CPU oracle (pins it).

Mirrors /root/reference/proj/tests/test_model.cpp, test_kinematics.cpp,
test_adjoint.cpp (minus the out-of-scope parallel suite) and
test_collocation.cpp: the known-answer values, the grid-quadrature, naive-sum,
forward-mode and finite-difference oracles.
"""
import math

import numpy as np
import pytest

import oracle
from paper_1709_04145_b200.types import (BoxGeometry, JointKind, JointSpec, LinkSpec, PointMass,
                                         PointMassGeometry)

from _ref_helpers import FD_STEP, fd_gradient, fd_jacobian, naive_correlation, planar_chain, random_offset, \
    random_tree, rel_err


def body(geom):
    link = LinkSpec(None, JointSpec(JointKind.hinge, (0, 0, 1)), geom)
    m = oracle.Model([link])
    info = m.info()
    return info["S"][0], info["mass"][0]


# --- test_model.cpp -----------------------------------------------------------
def grid_quadrature(box, cells):
    h = np.array(box.size) / cells
    dv = float(np.prod(h))
    ax = [np.array(box.center)[d] - 0.5 * box.size[d] + (np.arange(cells) + 0.5) * h[d] for d in range(3)]
    X, Y, Z = np.meshgrid(*ax, indexing="ij")
    P = np.stack([X.ravel(), Y.ravel(), Z.ravel(), np.ones(X.size)], axis=1)
    return box.density * dv * P.T @ P


def test_unit_cube_body_integral():
    S, m = body(BoxGeometry((1, 1, 1), 1.0, (0, 0, 0)))
    assert np.max(np.abs(S - np.diag([1 / 12, 1 / 12, 1 / 12, 1.0]))) < 1e-15
    assert m == pytest.approx(1.0)


def test_point_mass_body_integral():
    S, m = body(PointMassGeometry([PointMass(2.0, (1, 0, 0))]))
    exp = np.zeros((4, 4))
    exp[0, 0] = exp[0, 3] = exp[3, 0] = exp[3, 3] = 2.0
    assert np.array_equal(S, exp)
    assert m == pytest.approx(2.0)


def test_offset_box_matches_grid_quadrature():
    box = BoxGeometry((2, 1, 1), 3.0, (0, 0, 0.5))
    S, m = body(box)
    q = grid_quadrature(box, 48)
    assert rel_err(S, q) < 1e-3
    assert S[3, 3] == pytest.approx(m)
    assert rel_err(np.trace(S) - m, np.trace(q) - q[3, 3]) < 1e-3


def test_body_integral_invariants():
    rng = np.random.default_rng(7)
    for _ in range(20):
        box = BoxGeometry(tuple(rng.uniform(0.1, 2.0, 3)), 100.0 * rng.uniform(0.1, 2.0),
                          tuple(rng.uniform(0.1, 2.0, 3) - 1))
        S, _ = body(box)
        assert np.max(np.abs(S - S.T)) < 1e-12 * np.max(np.abs(S))
        assert np.linalg.eigvalsh(S).min() > -1e-10 * np.max(np.abs(S))
    a = [PointMass(1.0, (1, 2, 3)), PointMass(2.0, (-1, 0, 1)), PointMass(0.5, (0, 4, -2))]
    Sa, _ = body(PointMassGeometry(a))
    Sb, _ = body(PointMassGeometry([a[2], a[0], a[1]]))
    assert np.array_equal(Sa, Sb)
    base = BoxGeometry((0.7, 0.3, 1.1), 800.0, (0.2, -0.1, 0.4))
    shift = np.array([0.5, 0.25, -0.3])
    moved = BoxGeometry(base.size, base.density, tuple(np.array(base.center) + shift))
    S0, m0 = body(base)
    S1, _ = body(moved)
    c0 = np.array(base.center)
    d = np.zeros((4, 4))
    d[:3, :3] = m0 * (np.outer(shift, shift) + np.outer(shift, c0) + np.outer(c0, shift))
    d[:3, 3] = m0 * shift
    d[3, :3] = m0 * shift
    assert np.max(np.abs(S1 - S0 - d)) < 1e-9


@pytest.mark.parametrize("case", ["order", "density", "pointmass", "axis"])
def test_build_model_validation(case):
    box = BoxGeometry()
    a = LinkSpec(None, JointSpec(JointKind.hinge, (0, 0, 1)), box)
    if case == "order":
        links = [LinkSpec(1, a.joint, box), LinkSpec(None, a.joint, box)]
    elif case == "density":
        links = [LinkSpec(None, a.joint, BoxGeometry(density=0.0))]
    elif case == "pointmass":
        links = [LinkSpec(None, a.joint, PointMassGeometry([PointMass(-1.0, (0, 0, 0))]))]
    else:
        links = [LinkSpec(None, JointSpec(JointKind.hinge, (0, 0, 0)), box)]
    with pytest.raises(oracle.OracleError):
        oracle.Model(links)


def test_contact_samples_default_to_box_corners():
    m = oracle.Model([LinkSpec(None, JointSpec(JointKind.hinge, (0, 0, 1)), BoxGeometry())])
    c = m.samples(0)
    assert c.shape == (8, 3)
    for p in c:
        assert np.max(np.abs(p)) == pytest.approx(0.5)


# --- test_kinematics.cpp --------------------------------------------------------
HZ = (JointKind.hinge, (0.0, 0.0, 1.0))


def check_jet_fd(kind, axis, offset, q):
    v, d1, d2 = oracle.joint_jet(kind, axis, offset, q)
    dof = len(q)
    tri = lambda j, l: (max(j, l) * (max(j, l) + 1)) // 2 + min(j, l)
    for j in range(dof):
        qp, qm = q.copy(), q.copy()
        qp[j] += FD_STEP
        qm[j] -= FD_STEP
        fd1 = (oracle.joint_transform(kind, axis, offset, qp) - oracle.joint_transform(kind, axis, offset, qm)) / (
            2 * FD_STEP)
        assert rel_err(d1[j], fd1) < 1e-6
        _, d1p, _ = oracle.joint_jet(kind, axis, offset, qp)
        _, d1m, _ = oracle.joint_jet(kind, axis, offset, qm)
        for l in range(dof):
            assert rel_err(d2[tri(j, l)], (d1p[l] - d1m[l]) / (2 * FD_STEP)) < 1e-6


def test_hinge_jet_at_zero_is_generator():
    v, d1, d2 = oracle.joint_jet(*HZ, np.eye(4), np.zeros(1))
    assert np.max(np.abs(v - np.eye(4))) == 0.0
    gen = np.zeros((4, 4))
    gen[0, 1], gen[1, 0] = -1.0, 1.0
    assert np.max(np.abs(d1[0] - gen)) < 1e-15
    gen2 = np.zeros((4, 4))
    gen2[0, 0] = gen2[1, 1] = -1.0
    assert np.max(np.abs(d2[0] - gen2)) < 1e-15


def test_hinge_jet_at_half_pi():
    q = np.array([math.pi / 2])
    v, _, _ = oracle.joint_jet(*HZ, np.eye(4), q)
    assert abs(v[0, 0]) < 1e-12
    assert v[0, 1] == pytest.approx(-1.0)
    assert v[1, 0] == pytest.approx(1.0)
    check_jet_fd(*HZ, np.eye(4), q)


def test_ball_jet_matches_rotation_vector_and_fd():
    q = np.array([0.3, -0.2, 0.1])
    v, _, _ = oracle.joint_jet(JointKind.ball, (0, 0, 1), np.eye(4), q)
    assert np.max(np.abs(v[:3, :3] - oracle.rotation_vector_matrix(q))) == 0.0
    check_jet_fd(JointKind.ball, (0, 0, 1), np.eye(4), q)


def test_random_jets_fd_every_joint_kind():
    rng = np.random.default_rng(11)
    for _ in range(25):
        ax = rng.uniform(-1, 1, 3)
        if np.linalg.norm(ax) < 1e-3:
            ax = np.array([1.0, 0, 0])
        check_jet_fd(JointKind.hinge, tuple(ax / np.linalg.norm(ax)), random_offset(rng), rng.uniform(-2.5, 2.5, 1))
        check_jet_fd(JointKind.ball, (0, 0, 1), random_offset(rng), rng.uniform(-1.2, 1.2, 3))
        check_jet_fd(JointKind.free_joint, (0, 0, 1), random_offset(rng), rng.uniform(-1.2, 1.2, 6))


def test_small_angle_switch_continuity():
    d = np.array([1.0, 2.0, -0.5])
    d /= np.linalg.norm(d)
    a = oracle.joint_jet(JointKind.ball, (0, 0, 1), np.eye(4), (1e-4 - 1e-9) * d)
    b = oracle.joint_jet(JointKind.ball, (0, 0, 1), np.eye(4), (1e-4 + 1e-9) * d)
    for x, y in zip(a, b):
        assert np.max(np.abs(np.asarray(x) - np.asarray(y))) < 1e-8


def test_forward_pass():
    rng = np.random.default_rng(3)
    links = random_tree(rng, 8)
    m = oracle.Model(links)
    w = oracle.forward_pass(m, np.zeros(m.n_dofs))
    for i, l in enumerate(links):
        exp = l.joint.offset if l.parent is None else w[l.parent] @ l.joint.offset
        assert np.max(np.abs(w[i] - exp)) < 1e-14
    pc = oracle.Model(planar_chain(2))
    w = oracle.forward_pass(pc, np.array([math.pi / 2, -math.pi / 2]))
    assert w[1][:3, 3] == pytest.approx([1.0, 1.0, 0.0])
    assert np.max(np.abs(w[1][:3, :3] - np.eye(3))) < 1e-14
    rng = np.random.default_rng(5)
    m = oracle.Model(random_tree(rng, 30, chain=True))
    for t in oracle.forward_pass(m, rng.uniform(-10, 10, m.n_dofs)):
        assert np.max(np.abs(t[:3, :3].T @ t[:3, :3] - np.eye(3))) < 1e-9
        assert t[3, 0] == 0.0 and t[3, 3] == 1.0


# --- test_adjoint.cpp -------------------------------------------------------------
class ForwardMode:
    """Forward-mode differentiation oracle (test_adjoint.cpp:13-73)."""

    def __init__(self, links, model, q):
        self.links = links
        self.m = model
        info = model.info()
        self.off = info["dof_offset"]
        self.dof = [l.joint.dof_count() for l in links]
        self.par = [-1 if l.parent is None else l.parent for l in links]
        self.jets = []
        for i, l in enumerate(links):
            qi = q[self.off[i]:self.off[i] + self.dof[i]]
            self.jets.append(oracle.joint_jet(int(l.joint.kind), info["axis"][i], l.joint.offset, qi))
        self.world = []
        for i in range(len(links)):
            p = self.par[i]
            self.world.append(self.world[p] @ self.jets[i][0] if p >= 0 else self.jets[i][0])

    def owner(self, dof):
        for i in range(len(self.links)):
            if self.off[i] <= dof < self.off[i] + self.dof[i]:
                return i

    def dT(self, dof):
        l = self.owner(dof)
        loc = dof - self.off[l]
        d = []
        for mm in range(len(self.links)):
            p = self.par[mm]
            pw = self.world[p] if p >= 0 else np.eye(4)
            pd = d[p] if p >= 0 else np.zeros((4, 4))
            x = pd @ self.jets[mm][0]
            if mm == l:
                x = x + pw @ self.jets[mm][1][loc]
            d.append(x)
        return d

    def d2T(self, a, b):
        la, lb = self.owner(a), self.owner(b)
        ja, jb = a - self.off[la], b - self.off[lb]
        da, db = self.dT(a), self.dT(b)
        tri = lambda j, l: (max(j, l) * (max(j, l) + 1)) // 2 + min(j, l)
        d2 = []
        for mm in range(len(self.links)):
            p = self.par[mm]
            pw = self.world[p] if p >= 0 else np.eye(4)
            z = np.zeros((4, 4))
            x = (d2[p] if p >= 0 else z) @ self.jets[mm][0]
            if mm == la:
                x = x + (db[p] if p >= 0 else z) @ self.jets[mm][1][ja]
            if mm == lb:
                x = x + (da[p] if p >= 0 else z) @ self.jets[mm][1][jb]
            if mm == la and mm == lb:
                x = x + pw @ self.jets[mm][2][tri(ja, jb)]
            d2.append(x)
        return d2


def test_unit_cube_correlation_is_quarter():
    m = oracle.Model([LinkSpec(None, JointSpec(JointKind.hinge, (0, 0, 1)), BoxGeometry((1, 1, 1), 1.0, (0, 0, 0)))])
    v, g, bb, ab = oracle.correlation(m, [0.0], [0.0])
    assert v == pytest.approx(0.25, rel=1e-14)
    assert np.max(np.abs(g)) < 1e-14
    assert bb[0, 0] == pytest.approx(-1 / 6, rel=1e-12)
    assert ab[0, 0] == pytest.approx(1 / 6, rel=1e-12)


def test_correlation_matches_naive_sum_and_symmetry():
    rng = np.random.default_rng(21)
    links = random_tree(rng, 10, chain=True)
    m = oracle.Model(links)
    info = m.info()
    qa, qb = rng.uniform(-1, 1, m.n_dofs), rng.uniform(-1, 1, m.n_dofs)
    v = oracle.correlation(m, qa, qb)[0]
    nv = naive_correlation(m, info["S"], info["mass"], qa, qb)
    assert abs(v - nv) < 1e-12 * max(1.0, abs(nv))
    for t in range(10):
        links = random_tree(rng, 8)
        m = oracle.Model(links)
        qa, qb = rng.uniform(-1, 1, m.n_dofs), rng.uniform(-1, 1, m.n_dofs)
        a = oracle.correlation(m, qa, qb)[0]
        b = oracle.correlation(m, qb, qa)[0]
        assert abs(a - b) <= 1e-12 * max(1.0, abs(a))


def test_gradient_matches_fd_on_hinge_chain():
    links = planar_chain(6)
    m = oracle.Model(links)
    info = m.info()
    rng = np.random.default_rng(23)
    q = rng.uniform(-1, 1, 6)
    g = oracle.correlation(m, q, q)[1]
    fd = fd_gradient(lambda qb: naive_correlation(m, info["S"], info["mass"], q, qb), q)
    assert rel_err(g, fd) < 1e-6


def test_adjoint_equals_forward_mode_oracle():
    rng = np.random.default_rng(24)
    for _ in range(6):
        links = random_tree(rng, 5)
        m = oracle.Model(links)
        info = m.info()
        n = m.n_dofs
        qa, qb = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        v, g, bb, ab = oracle.correlation(m, qa, qb)
        A, Bf = ForwardMode(links, m, qa), ForwardMode(links, m, qb)
        og = np.array([sum(np.sum((A.world[k] @ info["S"][k]) * d[k]) for k in range(len(links)))
                       for d in (Bf.dT(j) for j in range(n))])
        assert rel_err(g, og) < 1e-10
        obb = np.zeros((n, n))
        oab = np.zeros((n, n))
        for j in range(n):
            da = A.dT(j)
            for k in range(n):
                d2 = Bf.d2T(j, k)
                db = Bf.dT(k)
                obb[j, k] = sum(np.sum((A.world[i] @ info["S"][i]) * d2[i]) for i in range(len(links)))
                oab[j, k] = sum(np.sum((da[i] @ info["S"][i]) * db[i]) for i in range(len(links)))
        assert rel_err(bb, obb) < 1e-10
        assert rel_err(bb, bb.T) < 1e-10
        assert rel_err(ab, oab) < 1e-10


def test_hessians_match_fd_of_gradient():
    rng = np.random.default_rng(25)
    m = oracle.Model(random_tree(rng, 5, chain=True))
    n = m.n_dofs
    qa, qb = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    _, _, bb, ab = oracle.correlation(m, qa, qb)
    assert rel_err(bb, fd_jacobian(lambda q: oracle.correlation(m, qa, q)[1], qb)) < 1e-5
    assert rel_err(ab, fd_jacobian(lambda q: oracle.correlation(m, q, qb)[1], qa).T) < 1e-5


def test_block_sparsity_two_branch_tree():
    def mk(parent, axis):
        off = np.eye(4)
        off[0, 3] = 0.7
        return LinkSpec(parent, JointSpec(JointKind.hinge, axis, off), BoxGeometry((0.4, 0.2, 0.2), 500.0, (0.2, 0, 0)))
    links = [mk(None, (0, 0, 1)), mk(0, (0, 1, 0)), mk(1, (0, 0, 1)), mk(0, (1, 0, 0)), mk(3, (0, 1, 0))]
    m = oracle.Model(links)
    rng = np.random.default_rng(26)
    _, _, bb, ab = oracle.correlation(m, rng.uniform(-1, 1, 5), rng.uniform(-1, 1, 5))
    for j in (1, 2):
        for k in (3, 4):
            assert bb[j, k] == 0.0 and bb[k, j] == 0.0 and ab[j, k] == 0.0 and ab[k, j] == 0.0


def test_hess_ab_psd_and_weights():
    rng = np.random.default_rng(27)
    for _ in range(6):
        m = oracle.Model(random_tree(rng, 7))
        q = rng.uniform(-1, 1, m.n_dofs)
        ab = oracle.correlation(m, q, q)[3]
        assert rel_err(ab, ab.T) < 1e-10
        assert np.linalg.eigvalsh(0.5 * (ab + ab.T)).min() >= -1e-8 * np.linalg.norm(ab)
    links = random_tree(rng, 6, chain=True)
    m = oracle.Model(links)
    info = m.info()
    qa, qb = rng.uniform(-1, 1, m.n_dofs), rng.uniform(-1, 1, m.n_dofs)
    w = rng.uniform(0.2, 2.0, m.n_links)
    v = oracle.correlation(m, qa, qb, weights=w)[0]
    ta, tb = oracle.forward_pass(m, qa), oracle.forward_pass(m, qb)
    exp = sum(w[i] * (np.trace(ta[i].T @ tb[i] @ info["S"][i]) - info["mass"][i]) for i in range(m.n_links))
    assert abs(v - exp) < 1e-11 * max(1.0, abs(exp))


# --- test_collocation.cpp -----------------------------------------------------
def test_legendre_points():
    assert list(oracle.legendre_points(2)) == [1.0]
    a = oracle.legendre_points(3)
    assert a[0] == pytest.approx(0.5, rel=1e-14) and a[1] == 1.0
    a = oracle.legendre_points(4)
    assert a[0] == pytest.approx(0.2113248654051871, rel=1e-12)
    assert a[1] == pytest.approx(0.7886751345948129, rel=1e-12)
    assert a[2] == 1.0
    for k in range(3, 7):
        a = oracle.legendre_points(k)
        for i in range(len(a) - 1):
            assert abs(a[i] + a[len(a) - 2 - i] - 1.0) < 1e-12
    with pytest.raises(oracle.OracleError):
        oracle.legendre_points(1)


def test_scheme_identities():
    for k in (2, 3, 4):
        s = oracle.build_scheme(k, 0.01)
        V = np.array([[t ** p for t in s["times"]] for p in range(k + 1)])
        assert np.max(np.abs(s["H"] @ V - np.eye(k + 1))) < 1e-10
    w = oracle.build_scheme(2, 0.25)["H2"][:, 2]
    assert w == pytest.approx([1.0, -2.0, 1.0], rel=1e-12)
    s = oracle.build_scheme(3, 0.1)
    for f, d2 in ((lambda t: t * t, lambda t: 2.0), (lambda t: t ** 3, lambda t: 6.0 * t)):
        smp = np.array([f(t) for t in s["times"]])
        for mm in range(2):
            assert abs(s["H2"][:, 2 + mm] @ smp - d2(s["times"][2 + mm])) < 1e-10
    for k in (2, 3, 4, 5, 6):
        s = oracle.build_scheme(k, 0.01)
        f = lambda t: 0.3 + sum((0.7 - 0.13 * p) * t ** p for p in range(1, k + 1))
        d2 = lambda t: sum((0.7 - 0.13 * p) * p * (p - 1) * t ** (p - 2) for p in range(2, k + 1))
        smp = np.array([f(t) for t in s["times"]])
        for mm in range(k - 1):
            e = d2(s["times"][2 + mm])
            assert abs(s["H2"][:, 2 + mm] @ smp - e) < 1e-9 * max(1.0, abs(e))
    with pytest.raises(oracle.OracleError):
        oracle.build_scheme(1, 0.1)
    with pytest.raises(oracle.OracleError):
        oracle.build_scheme(3, 0.0)
    s = oracle.build_scheme(4, 0.1)
    assert s["times"][-1] == 1.0 and all(np.diff(s["times"]) > 0)
