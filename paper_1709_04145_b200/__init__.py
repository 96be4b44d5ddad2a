"""B200-native PBAD hot path (arXiv 1709.04145): reference-shaped API.

The numeric work runs in libpbad_gpu.so (sm_100a kernels + host C++ behind
include/pbad_gpu.h).  Importing this package does not need a GPU or even the
built library; creating a model or a GpuContext loads the library, and
contexts fail loudly without an sm_100 device (there is no CPU fallback).
"""
from .types import (ActuationKind, ActuationSpec, BaselineScheme, BoxGeometry, ContactModel, EnergySample, ForceModel, JointKind,
                    JointSpec, LinkSpec, ModelError, ObjectiveKind, OptimizerConfig, OptimizerKind, PointMass,
                    PointMassGeometry, SimConfig, SolveReport, Trajectory)
from . import scenes
from .api import (CollocationScheme, CorrelationDerivatives, CorrelationRequest, GpuContext, KinematicModel,
                  StepObjective, StepProblem, batch_correlation, batch_simulate, batch_simulate_baseline, body_integral, build_model,
                  build_scheme, correlation_and_grad, hessian_ab, hessian_bb, legendre_points,
                  rotation_vector_from_matrix, rotation_vector_matrix, simulate, simulate_baseline, total_steps,
                  validate_configuration)
