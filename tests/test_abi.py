"""C ABI: the library loads, exports every symbol include/pbad_gpu.h declares,
and its host-side parts (build_model, body_integral, build_scheme,
rotation_vector_matrix, validation) are bit-identical to the oracle.  No
GPU needed (compute entry points are exercised by the gpu-marked tests)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from paper_1709_04145_b200 import _lib, api
from paper_1709_04145_b200.scenes import (make_chain_scene, make_humanoid_scene, make_spider_scene,
                                          make_swimmer_scene)
from paper_1709_04145_b200.types import (BoxGeometry, JointKind, JointSpec, LinkSpec, ModelError, PointMass,
                                         PointMassGeometry, SimConfig)

from _ref_helpers import random_tree

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pbad_gpu.h")).read()
    return sorted(set(re.findall(r"\b(pbad_gpu_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(_lib.HEADER_SYMBOLS)
    assert lib.pbad_gpu_abi_version() == 1


@pytest.mark.parametrize("scene", ["chain", "humanoid", "spider", "swimmer", "random"])
def test_host_model_bit_identical_to_oracle(scene):
    rng = np.random.default_rng(3)
    sc = {"chain": lambda: make_chain_scene(5).links, "humanoid": lambda: make_humanoid_scene().links,
          "spider": lambda: make_spider_scene(api.rotation_vector_matrix).links,
          "swimmer": lambda: make_swimmer_scene().links, "random": lambda: random_tree(rng, 9)}[scene]()
    m = api.build_model(sc)
    o = oracle.Model(sc).info()
    assert np.array_equal(m.body_S, o["S"])
    assert np.array_equal(m.body_mass, o["mass"])
    assert np.array_equal(m.axes, o["axis"])
    assert list(m.dof_offsets) == list(o["dof_offset"])
    assert np.array_equal(m.sample_counts, o["sample_count"])


def test_host_scheme_and_rotation_bit_identical():
    for k in range(2, 8):
        a = api.build_scheme(k, 0.013)
        b = oracle.build_scheme(k, 0.013)
        assert np.array_equal(a.H, b["H"]) and np.array_equal(a.H2, b["H2"]) and np.array_equal(a.times, b["times"])
    rng = np.random.default_rng(5)
    for _ in range(200):
        th = rng.uniform(-4, 4, 3) * (10.0 ** rng.integers(-6, 2))
        assert np.array_equal(api.rotation_vector_matrix(th), oracle.rotation_vector_matrix(th))


def test_portable_sincos_accuracy():
    # the shared sin/cos is within 2 ulp of libm on the angle range the path sees
    rng = np.random.default_rng(6)
    for x in np.concatenate([rng.uniform(-50, 50, 2000), [0.0, 1e-300, np.pi / 4, 1e4]]):
        s, c = oracle.sincos(x)
        assert abs(s - np.sin(x)) <= 2 * np.spacing(max(abs(np.sin(x)), 1e-300)) + 1e-300 or abs(s - np.sin(x)) < 4e-16
        assert abs(c - np.cos(x)) <= 2 * np.spacing(max(abs(np.cos(x)), 1e-300)) or abs(c - np.cos(x)) < 4e-16


@pytest.mark.parametrize("case,msg", [
    ("order", "link 0: parent index must be smaller than own index"),
    ("density", "link 0: non-positive density"),
    ("pointmass", "link 0: non-positive point mass"),
    ("axis", "link 0: zero-norm hinge axis"),
])
def test_model_errors_match_reference_text(case, msg):
    j = JointSpec(JointKind.hinge, (0, 0, 1))
    if case == "order":
        links = [LinkSpec(1, j, BoxGeometry()), LinkSpec(None, j, BoxGeometry())]
    elif case == "density":
        links = [LinkSpec(None, j, BoxGeometry(density=0.0))]
    elif case == "pointmass":
        links = [LinkSpec(None, j, PointMassGeometry([PointMass(-1.0, (0, 0, 0))]))]
    else:
        links = [LinkSpec(None, JointSpec(JointKind.hinge, (0, 0, 0)), BoxGeometry())]
    with pytest.raises(ModelError, match=re.escape(msg)):
        api.build_model(links)
    with pytest.raises(oracle.OracleError, match=re.escape(msg)):
        oracle.Model(links)


def test_validate_configuration():
    m = api.build_model(make_chain_scene(3).links)
    api.validate_configuration(m, np.zeros(6))
    with pytest.raises(ModelError, match="does not match model DOF count"):
        api.validate_configuration(m, np.zeros(5))
    with pytest.raises(ModelError, match="non-finite"):
        api.validate_configuration(m, np.array([0, 0, np.nan, 0, 0, 0]))


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    m = api.build_model(make_chain_scene(2).links)
    sim = SimConfig(dt=0.01, duration=0.02)
    with pytest.raises(_lib.PbadGpuError, match="CUDA"):
        api.GpuContext(m, None, sim)
