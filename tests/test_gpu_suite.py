"""The large-N correlation suite and the standalone linear functional on the
GPU (pbad_corr.cu: one CTA per request) against the reference itself
(oracle/_ref: parallel_correlation_suite, functional_value / _grad / _hess
from /root/reference/proj/src/adjoint.cpp compiled unmodified): bit-exact
values, gradients and Hessians on random trees with hinge, ball and free
joints, weighted bodies, a 600-link chain (the large-N case), and against
the thread-per-pair correlation path."""
import numpy as np
import pytest

import oracle
from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import make_chain_scene

from _parity_util import random_tree

pytestmark = pytest.mark.gpu


def _q(rng, model, scale=0.6):
    return rng.uniform(-scale, scale, model.total_dofs)


def _same(a, b):
    np.testing.assert_array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("seed,links", [(1, 9), (2, 17), (3, 31)])
@pytest.mark.parametrize("weighted", [False, True])
def test_suite_matches_reference(seed, links, weighted):
    rng = np.random.default_rng(seed)
    specs = random_tree(rng, links)
    m = api.build_model(specs)
    ref = oracle.RefModel(specs)
    w = rng.uniform(0.5, 2.0, links) if weighted else None
    qa, qb = _q(rng, m), _q(rng, m)
    got = api.parallel_correlation_suite(api.CorrelationRequest(m, qa, qb, w), workers=3)
    v, g, bb, ab = oracle.ref_correlation_suite(ref, qa, qb, w, workers=3)
    assert got.value == v
    _same(got.grad_b, g)
    _same(got.hess_bb, bb)
    _same(got.hess_ab, ab)


def test_suite_batch_equals_pairwise_path():
    """Batched suite (one CTA per pair) == the thread-per-pair correlation
    kernel on every pair (the serial functions), up to the sign of zero
    gradient entries (the suite assigns, correlation_grad_b accumulates)."""
    rng = np.random.default_rng(7)
    specs = random_tree(rng, 12)
    m = api.build_model(specs)
    ctx = api._corr_ctx(m)
    qa = rng.uniform(-0.5, 0.5, (5, m.total_dofs))
    qb = rng.uniform(-0.5, 0.5, (5, m.total_dofs))
    s = ctx.correlation_suite(qa, qb)
    p = ctx.correlation(qa, qb)
    _same(s[0], p[0])
    np.testing.assert_array_equal(s[1] + 0.0, p[1] + 0.0)
    _same(s[2], p[2])
    _same(s[3], p[3])


def test_suite_large_chain():
    """The large-N case: a 600-link (300-segment) chain in one CTA."""
    sc = make_chain_scene(300)
    m = api.build_model(sc.links)
    ref = oracle.RefModel(sc.links)
    rng = np.random.default_rng(11)
    qa, qb = _q(rng, m, 0.3), _q(rng, m, 0.3)
    got = api.parallel_correlation_suite(api.CorrelationRequest(m, qa, qb), workers=2)
    v, g, bb, ab = oracle.ref_correlation_suite(ref, qa, qb, None, workers=2)
    assert got.value == v
    _same(got.grad_b, g)
    _same(got.hess_bb, bb)
    _same(got.hess_ab, ab)


@pytest.mark.parametrize("seed,links", [(4, 8), (5, 23)])
def test_functional_matches_reference(seed, links):
    rng = np.random.default_rng(seed)
    specs = random_tree(rng, links)
    m = api.build_model(specs)
    ref = oracle.RefModel(specs)
    q = _q(rng, m)
    seeds = rng.normal(size=(links, 4, 4))
    v, g, h = oracle.ref_functional(ref, q, seeds)
    assert api.functional_value(m, seeds, q) == v
    _same(api.functional_grad(m, seeds, q), g)
    _same(api.functional_hess(m, seeds, q), h)
    # batched: B requests with different seeds in one launch
    qs = rng.uniform(-0.6, 0.6, (3, m.total_dofs))
    ss = rng.normal(size=(3, links, 4, 4))
    bv, bg, bh = api._corr_ctx(m).functional(qs, ss)
    for b in range(3):
        rv, rg, rh = oracle.ref_functional(ref, qs[b], ss[b])
        assert bv[b] == rv
        _same(bg[b], rg)
        _same(bh[b], rh)


def test_suite_rejects_bad_inputs():
    rng = np.random.default_rng(0)
    m = api.build_model(random_tree(rng, 5))
    with pytest.raises(api.ModelError):
        api.parallel_correlation_suite(api.CorrelationRequest(m, np.zeros(m.total_dofs), np.zeros(m.total_dofs)),
                                       workers=0)
    with pytest.raises(api.ModelError):
        api.parallel_correlation_suite(api.CorrelationRequest(m, np.zeros(m.total_dofs), np.zeros(m.total_dofs),
                                                              np.ones(3)))
