"""ctypes binding of libpbad_gpu.so (include/pbad_gpu.h).

The shared library is built in-tree (paper_1709_04145_b200/build.py).  There
is no Python or CPU fallback for the hot path: if the library is missing the
import of the GPU entry points fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PBAD_GPU_LIB: an alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("PBAD_GPU_LIB") or os.path.join(_HERE, "libpbad_gpu.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_fp = C.POINTER(C.c_float)

HEADER_SYMBOLS = [
    "pbad_gpu_abi_version", "pbad_gpu_last_error", "pbad_gpu_error_string", "pbad_gpu_default_optimizer",
    "pbad_gpu_default_sim", "pbad_gpu_model_create", "pbad_gpu_model_destroy", "pbad_gpu_model_dofs",
    "pbad_gpu_model_links", "pbad_gpu_model_info", "pbad_gpu_body_integral", "pbad_gpu_rotation_vector_matrix",
    "pbad_gpu_rotation_vector_from_matrix",
    "pbad_gpu_build_scheme", "pbad_gpu_validate_configuration", "pbad_gpu_create", "pbad_gpu_destroy",
    "pbad_gpu_total_steps", "pbad_gpu_path", "pbad_gpu_kernel_launches", "pbad_gpu_rollout", "pbad_gpu_begin", "pbad_gpu_advance", "pbad_gpu_sync_outputs",
    "pbad_gpu_state_device", "pbad_gpu_eval", "pbad_gpu_minimize", "pbad_gpu_correlation",
    "pbad_gpu_simulate_baseline", "pbad_gpu_rollout_sharded", "pbad_gpu_final_state",
    "pbad_gpu_device_count", "pbad_gpu_correlation_suite", "pbad_gpu_functional",
]


class LinkSpec(C.Structure):
    _fields_ = [
        ("parent", C.c_int32), ("joint_kind", C.c_int32), ("axis", C.c_double * 3),
        ("offset", C.c_double * 16), ("geom_kind", C.c_int32), ("box_size", C.c_double * 3),
        ("box_density", C.c_double), ("box_center", C.c_double * 3), ("n_points", C.c_int32),
        ("point_mass", _dp), ("point_pos", _dp), ("n_samples", C.c_int32), ("samples", _dp),
    ]


class Forces(C.Structure):
    _fields_ = [
        ("gravity", C.c_double * 3), ("drag_d", C.c_double), ("has_contact", C.c_int32),
        ("plane_normal", C.c_double * 3), ("plane_offset", C.c_double), ("contact_d1", C.c_double),
        ("contact_d2", C.c_double), ("tau_len", C.c_int32), ("tau", _dp), ("has_actuation", C.c_int32),
        ("act_kind", C.c_int32), ("act_len", C.c_int32), ("act_amplitude", _dp),
        ("act_frequency_hz", C.c_double), ("act_phase_len", C.c_int32), ("act_phase", _dp),
    ]


class OptimizerConfig(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("max_iters", C.c_int32), ("grad_tol", C.c_double), ("grad_rtol", C.c_double),
        ("ftol", C.c_double), ("lbfgs_memory", C.c_int32), ("lm_lambda0", C.c_double),
        ("lm_lambda_factor", C.c_double), ("lm_lambda_max", C.c_double), ("armijo_c1", C.c_double),
        ("backtrack_factor", C.c_double), ("max_line_search", C.c_int32),
    ]


class SimDesc(C.Structure):
    _fields_ = [
        ("dt", C.c_double), ("duration", C.c_double), ("order", C.c_int32), ("objective", C.c_int32),
        ("opt", OptimizerConfig), ("consecutive_fail_limit", C.c_int32), ("refined_bootstrap", C.c_int32),
        ("warm_start", C.c_int32),
    ]


class RolloutOut(C.Structure):
    _fields_ = [
        ("q", _dp), ("energy", _dp), ("iterations", _ip), ("converged", _ip), ("accepted", _ip),
        ("final_value", _dp), ("final_grad_norm", _dp), ("n_samples", _ip), ("status", _ip),
        ("fail_streak", _ip), ("n_reports", _ip), ("device_ms", _fp), ("iteration_values", _dp),
    ]


_lib = None


class PbadGpuError(RuntimeError):
    pass


def load():
    """Load libpbad_gpu.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise PbadGpuError(f"{LIB_PATH} is missing: run `python -m paper_1709_04145_b200.build` "
                           "(the PBAD hot path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    sig = {
        "pbad_gpu_abi_version": ([], C.c_int32),
        "pbad_gpu_last_error": ([], C.c_char_p),
        "pbad_gpu_error_string": ([C.c_int32], C.c_char_p),
        "pbad_gpu_default_optimizer": ([C.POINTER(OptimizerConfig)], None),
        "pbad_gpu_default_sim": ([C.POINTER(SimDesc)], None),
        "pbad_gpu_model_create": ([C.POINTER(LinkSpec), C.c_int32, C.POINTER(vp)], C.c_int32),
        "pbad_gpu_model_destroy": ([vp], None),
        "pbad_gpu_model_dofs": ([vp], C.c_int32),
        "pbad_gpu_model_links": ([vp], C.c_int32),
        "pbad_gpu_model_info": ([vp, _dp, _dp, _ip, _dp, _ip], C.c_int32),
        "pbad_gpu_body_integral": ([C.POINTER(LinkSpec), _dp, _dp], C.c_int32),
        "pbad_gpu_correlation": ([vp, C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp, _dp], C.c_int32),
        "pbad_gpu_simulate_baseline": ([vp, C.c_int32, C.c_int32, _dp, _dp, _dp, _dp, _ip, _ip], C.c_int32),
        "pbad_gpu_rotation_vector_matrix": ([_dp, _dp], C.c_int32),
        "pbad_gpu_rotation_vector_from_matrix": ([_dp, _dp], C.c_int32),
        "pbad_gpu_build_scheme": ([C.c_int32, C.c_double, _dp, _dp, _dp, _dp], C.c_int32),
        "pbad_gpu_validate_configuration": ([vp, _dp, C.c_int32], C.c_int32),
        "pbad_gpu_create": ([vp, C.POINTER(Forces), C.POINTER(SimDesc), C.c_int32, C.c_int32, C.POINTER(vp)],
                            C.c_int32),
        "pbad_gpu_destroy": ([vp], None),
        "pbad_gpu_total_steps": ([vp], C.c_int32),
        "pbad_gpu_path": ([vp], C.c_int32),
        "pbad_gpu_kernel_launches": ([vp], C.c_int64),
        "pbad_gpu_rollout": ([vp, C.c_int32, _dp, _dp, C.POINTER(RolloutOut)], C.c_int32),
        "pbad_gpu_begin": ([vp, C.c_int32, vp, vp, vp], C.c_int32),
        "pbad_gpu_advance": ([vp, C.c_int32, vp], C.c_int32),
        "pbad_gpu_sync_outputs": ([vp, C.POINTER(RolloutOut)], C.c_int32),
        "pbad_gpu_state_device": ([vp], vp),
        "pbad_gpu_rollout_sharded": ([C.POINTER(vp), C.c_int32, C.c_int32, _dp, _dp, C.POINTER(RolloutOut)],
                                     C.c_int32),
        "pbad_gpu_final_state": ([vp, vp, vp], C.c_int32),
        "pbad_gpu_device_count": ([], C.c_int32),
        "pbad_gpu_correlation_suite": ([vp, C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp, _dp], C.c_int32),
        "pbad_gpu_functional": ([vp, C.c_int32, _dp, _dp, _dp, _dp, _dp], C.c_int32),
        "pbad_gpu_eval": ([vp, C.c_int32, _dp, _dp, _dp, C.c_int32, C.c_int32, _dp, _dp, _dp], C.c_int32),
        "pbad_gpu_minimize": ([vp, C.c_int32, _dp, _dp, _dp, _dp, _ip, _ip, _dp, _dp], C.c_int32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.pbad_gpu_abi_version() != 1:
        raise PbadGpuError("libpbad_gpu.so ABI version mismatch")
    _lib = L
    return L


def check(rc: int):
    if rc != 0:
        msg = load().pbad_gpu_last_error().decode(errors="replace")
        kind = load().pbad_gpu_error_string(rc).decode()
        from .types import ModelError
        if rc == -1:
            raise ModelError(msg)
        if rc == -2:
            raise ValueError(msg)
        raise PbadGpuError(f"{kind}: {msg}")
