"""Python mirror of the reference's model / force / solver / stepper value types.

Field names, defaults and meaning follow the C++ headers one to one:
  JointSpec, BoxGeometry, PointMass(Geometry), LinkSpec   model.hpp:19-62
  ContactModel, ActuationSpec, ForceModel, ObjectiveKind  objective.hpp:20-61
  OptimizerKind, OptimizerConfig, SolveReport             optim.hpp:13-36
  EnergySample, Trajectory, SimConfig                     stepper.hpp:15-44
Matrices are row-major numpy arrays here (the C ABI converts to the
reference's column-major Eigen layout).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import List, Optional, Tuple, Union

import numpy as np


class ModelError(ValueError):
    """Invalid model definition or configuration (model.hpp:14-17)."""


class JointKind(enum.IntEnum):
    hinge = 0
    ball = 1
    free_joint = 2


def _identity4():
    return np.eye(4)


@dataclass
class JointSpec:
    kind: JointKind = JointKind.hinge
    axis: Tuple[float, float, float] = (0.0, 0.0, 1.0)
    offset: np.ndarray = field(default_factory=_identity4)

    def dof_count(self) -> int:
        return {JointKind.hinge: 1, JointKind.ball: 3, JointKind.free_joint: 6}[JointKind(self.kind)]


@dataclass
class BoxGeometry:
    size: Tuple[float, float, float] = (1.0, 1.0, 1.0)
    density: float = 1000.0
    center: Tuple[float, float, float] = (0.0, 0.0, 0.0)


@dataclass
class PointMass:
    mass: float = 0.0
    position: Tuple[float, float, float] = (0.0, 0.0, 0.0)


@dataclass
class PointMassGeometry:
    masses: List[PointMass] = field(default_factory=list)


Geometry = Union[BoxGeometry, PointMassGeometry]


@dataclass
class LinkSpec:
    parent: Optional[int] = None
    joint: JointSpec = field(default_factory=JointSpec)
    geometry: Geometry = field(default_factory=BoxGeometry)
    contact_samples: List[Tuple[float, float, float]] = field(default_factory=list)


@dataclass
class ContactModel:
    plane_normal: Tuple[float, float, float] = (0.0, 0.0, 1.0)
    plane_offset: float = 0.0
    d1: float = 0.0
    d2: float = 0.0


class ActuationKind(enum.IntEnum):
    constant = 0
    sinusoidal = 1


@dataclass
class ActuationSpec:
    kind: ActuationKind = ActuationKind.constant
    amplitude: Optional[np.ndarray] = None
    frequency_hz: float = 0.0
    phase: Optional[np.ndarray] = None


@dataclass
class ForceModel:
    gravity: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    drag_d: float = 0.0
    contact: Optional[ContactModel] = None
    tau: Optional[np.ndarray] = None
    actuation: Optional[ActuationSpec] = None


class BaselineScheme(enum.IntEnum):
    """baseline.hpp:17"""
    forward_euler = 0
    semi_implicit = 1
    rk2 = 2
    rk3 = 3
    rk4 = 4


class ObjectiveKind(enum.IntEnum):
    energy_form = 0
    residual_form = 1


class OptimizerKind(enum.IntEnum):
    lbfgs = 0
    lm = 1


@dataclass
class OptimizerConfig:
    kind: OptimizerKind = OptimizerKind.lm
    max_iters: int = 512
    grad_tol: float = 1e-8
    grad_rtol: float = 0.0
    ftol: float = 1e-14
    lbfgs_memory: int = 8
    lm_lambda0: float = 1e-3
    lm_lambda_factor: float = 10.0
    lm_lambda_max: float = 1e12
    armijo_c1: float = 1e-4
    backtrack_factor: float = 0.5
    max_line_search: int = 40


@dataclass
class SolveReport:
    iterations: int = 0
    final_value: float = 0.0
    final_grad_norm: float = 0.0
    converged: bool = False
    accepted: int = 0  # accepted iterations (derivable from per_iteration_values)
    per_iteration_values: List[float] = field(default_factory=list)  # optim.cpp:30-37 (on request)


@dataclass
class EnergySample:
    time: float = 0.0
    kinetic: float = 0.0
    potential: float = 0.0

    def total(self) -> float:
        return self.kinetic + self.potential


@dataclass
class Trajectory:
    samples: List[Tuple[float, np.ndarray]] = field(default_factory=list)
    energy_log: List[EnergySample] = field(default_factory=list)
    solve_reports: List[SolveReport] = field(default_factory=list)
    error: Optional[str] = None


@dataclass
class SimConfig:
    dt: float = 0.01
    duration: float = 1.0
    order: int = 2
    objective: ObjectiveKind = ObjectiveKind.energy_form
    optimizer: OptimizerConfig = field(default_factory=OptimizerConfig)
    q0: Optional[np.ndarray] = None
    qdot0: Optional[np.ndarray] = None
    consecutive_fail_limit: int = 25
    refined_bootstrap: bool = False
    warm_start: bool = True

    def same_schedule(self, other: "SimConfig") -> bool:
        """True when two configs differ at most in their initial state."""
        return (self.dt == other.dt and self.duration == other.duration and self.order == other.order
                and self.objective == other.objective and self.optimizer == other.optimizer
                and self.consecutive_fail_limit == other.consecutive_fail_limit
                and self.refined_bootstrap == other.refined_bootstrap
                and self.warm_start == other.warm_start)
