"""Batched correlation derivatives on the GPU (pbad_gpu_correlation:
correlation_and_grad / hessian_bb / hessian_ab, adjoint.cpp:113-192) against
the CPU oracle, bit for bit, with and without per-body weights; unit weights
also against the reference's own adjoint.cpp (oracle/_ref)."""
import numpy as np
import pytest

import oracle
from paper_1709_04145_b200 import api
from paper_1709_04145_b200.scenes import make_chain_scene, make_humanoid_scene, make_spider_scene
from paper_1709_04145_b200.types import ModelError

from _parity_util import random_tree

pytestmark = pytest.mark.gpu


def _models():
    rng = np.random.default_rng(11)
    yield "humanoid", make_humanoid_scene().links
    yield "chain6", make_chain_scene(6).links
    yield "spider", make_spider_scene(api.rotation_vector_matrix).links
    for k in range(3):
        yield f"tree{k}", random_tree(rng, 5 + 2 * k)


@pytest.mark.parametrize("name,links", list(_models()), ids=[m[0] for m in _models()])
@pytest.mark.parametrize("weighted", [False, True])
def test_correlation_matches_oracle(name, links, weighted):
    rng = np.random.default_rng(sum(map(ord, name)) + int(weighted))
    m = api.build_model(links)
    om = oracle.Model(links)
    n = m.total_dofs
    B = 5
    qa = rng.uniform(-0.8, 0.8, (B, n))
    qb = qa + rng.uniform(-0.2, 0.2, (B, n))
    w = rng.uniform(0.2, 2.0, len(links)) if weighted else None
    ctx = api.GpuContext(m, None, api.SimConfig(dt=0.01, duration=0.01))
    v, g, bb, ab = ctx.correlation(qa, qb, w)
    for b in range(B):
        ov, og, obb, oab = oracle.correlation(om, qa[b], qb[b], w)
        assert v[b] == ov
        np.testing.assert_array_equal(g[b], og)
        np.testing.assert_array_equal(bb[b], obb)
        np.testing.assert_array_equal(ab[b], oab)
        if not weighted and oracle.ref_available():
            rm = oracle.RefModel(links)
            rv, rg, rbb, rab = oracle.ref_correlation(rm, qa[b], qb[b])
            assert v[b] == rv
            np.testing.assert_array_equal(g[b], rg)
            np.testing.assert_array_equal(bb[b], rbb)
            np.testing.assert_array_equal(ab[b], rab)


def test_reference_shaped_entry_points():
    """CorrelationRequest -> correlation_and_grad / hessian_bb / hessian_ab;
    hess_ab(q, q) is the mass matrix J^T M J (symmetric PSD,
    test_adjoint.cpp:287-298)."""
    links = make_humanoid_scene().links
    m = api.build_model(links)
    rng = np.random.default_rng(3)
    q = rng.uniform(-0.5, 0.5, m.total_dofs)
    req = api.CorrelationRequest(m, q, q)
    v, g = api.correlation_and_grad(req)
    ab = api.hessian_ab(req)
    np.testing.assert_allclose(ab, ab.T, rtol=0, atol=1e-12 * np.abs(ab).max())
    assert np.linalg.eigvalsh(0.5 * (ab + ab.T)).min() > -1e-9
    bb = api.hessian_bb(req)
    ov, og, obb, oab = oracle.correlation(oracle.Model(links), q, q)
    assert v == ov
    np.testing.assert_array_equal(g, og)
    np.testing.assert_array_equal(bb, obb)
    np.testing.assert_array_equal(ab, oab)
    with pytest.raises(ModelError, match="weight_per_body length"):
        api.hessian_bb(api.CorrelationRequest(m, q, q, np.ones(3)))


def test_nonfinite_propagates_like_reference():
    links = make_chain_scene(3).links
    m = api.build_model(links)
    q = np.zeros(m.total_dofs)
    qb = q.copy()
    qb[1] = np.nan
    v, g, bb, ab = api.GpuContext(m, None, api.SimConfig(dt=0.01, duration=0.01)).correlation(q[None], qb[None])
    assert np.isnan(v[0])
