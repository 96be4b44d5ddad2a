"""Benchmark scene builders (the scene JSON layer is scene_io.py).

make_chain_scene / make_single_hinge_chain_scene / make_swimmer_scene /
make_spider_scene follow /root/reference/proj/src/scene.cpp:430-618;
make_humanoid_scene is SURVEY.md Appendix B (the C4 tree).  Synthetic initial
states mirror benchmark.cpp:278-288: std::mt19937(seed) +
uniform_real_distribution, env-major then DOF (see mt19937_uniform).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .types import (ActuationKind, ActuationSpec, BoxGeometry, ContactModel, ForceModel, JointKind,
                    JointSpec, LinkSpec, ObjectiveKind, OptimizerConfig, OptimizerKind,
                    PointMassGeometry, SimConfig)


def translation(x: float, y: float, z: float) -> np.ndarray:
    m = np.eye(4)
    m[0, 3], m[1, 3], m[2, 3] = x, y, z
    return m


@dataclass
class Scene:
    links: List[LinkSpec] = field(default_factory=list)
    gravity: tuple = (0.0, 0.0, 0.0)
    drag_d: float = 0.0
    contact: Optional[ContactModel] = None
    actuation: Optional[ActuationSpec] = None
    order: int = 2
    objective: ObjectiveKind = ObjectiveKind.energy_form
    optimizer: OptimizerKind = OptimizerKind.lm
    dt: float = 0.0
    duration: float = 0.0
    q0: Optional[np.ndarray] = None
    qdot0: Optional[np.ndarray] = None
    # scene-file fields (scene.hpp:20-44): which links listed contact_samples
    # explicitly, and the integrator kind ("pbad" or a baseline scheme)
    link_has_samples: Optional[List[bool]] = None
    integrator_kind: str = "pbad"

    def forces(self) -> ForceModel:
        return ForceModel(gravity=self.gravity, drag_d=self.drag_d, contact=self.contact,
                          actuation=self.actuation)

    def sim_config(self) -> SimConfig:
        return SimConfig(dt=self.dt, duration=self.duration, order=self.order,
                         objective=self.objective,
                         optimizer=OptimizerConfig(kind=self.optimizer),
                         q0=None if self.q0 is None else self.q0.copy(),
                         qdot0=None if self.qdot0 is None else self.qdot0.copy())


def _chain_link_box() -> BoxGeometry:
    return BoxGeometry(size=(0.5, 0.1, 0.1), density=1000.0, center=(0.25, 0.0, 0.0))


def make_chain_scene(segment_count: int) -> Scene:
    """scene.cpp:455-486: massless Z-hinge connector + Y-hinge box per segment."""
    s = Scene()
    for i in range(segment_count):
        s.links.append(LinkSpec(parent=None if i == 0 else 2 * i - 1,
                                joint=JointSpec(JointKind.hinge, (0.0, 0.0, 1.0),
                                                np.eye(4) if i == 0 else translation(0.5, 0.0, 0.0)),
                                geometry=PointMassGeometry([])))
        s.links.append(LinkSpec(parent=2 * i, joint=JointSpec(JointKind.hinge, (0.0, 1.0, 0.0), np.eye(4)),
                                geometry=_chain_link_box()))
    s.gravity = (0.0, 0.0, -9.81)
    s.dt, s.duration = 0.0025, 10.0
    s.q0 = np.zeros(2 * segment_count)
    s.qdot0 = np.zeros(2 * segment_count)
    return s


def make_single_hinge_chain_scene(link_count: int) -> Scene:
    """scene.cpp:488-510: one Y-hinge box per link, 0.5 m pitch."""
    s = Scene()
    for i in range(link_count):
        s.links.append(LinkSpec(parent=None if i == 0 else i - 1,
                                joint=JointSpec(JointKind.hinge, (0.0, 1.0, 0.0),
                                                np.eye(4) if i == 0 else translation(0.5, 0.0, 0.0)),
                                geometry=_chain_link_box()))
    s.gravity = (0.0, 0.0, -9.81)
    s.dt, s.duration = 0.0025, 10.0
    s.q0 = np.zeros(link_count)
    s.qdot0 = np.zeros(link_count)
    return s


def make_swimmer_scene() -> Scene:
    """scene.cpp:512-552: free head + 3 Z-hinge segments, drag, sinusoidal actuation."""
    s = Scene()
    hb = BoxGeometry(size=(0.5, 0.1, 0.05), density=1000.0, center=(0.25, 0.0, 0.0))
    s.links.append(LinkSpec(parent=None, joint=JointSpec(JointKind.free_joint), geometry=hb))
    for i in range(3):
        s.links.append(LinkSpec(parent=i, joint=JointSpec(JointKind.hinge, (0.0, 0.0, 1.0),
                                                          translation(0.5, 0.0, 0.0)), geometry=hb))
    s.drag_d = 2.0
    amp = np.zeros(9)
    ph = np.zeros(9)
    for i in range(3):
        amp[6 + i] = 6.0
        ph[6 + i] = i * (math.pi / 2.0)
    s.actuation = ActuationSpec(ActuationKind.sinusoidal, amp, 0.5, ph)
    s.dt, s.duration = 0.05, 10.0
    s.q0 = np.zeros(9)
    s.qdot0 = np.zeros(9)
    return s


def _rotation_z(angle: float, rotation_vector_matrix) -> np.ndarray:
    m = np.eye(4)
    m[:3, :3] = rotation_vector_matrix((0.0, 0.0, angle))
    return m


def make_spider_scene(rotation_vector_matrix) -> Scene:
    """scene.cpp:554-618: free torso + 4 legs (ball hip, Y-hinge knee), contact.

    rotation_vector_matrix must be the canonical (bit-reproducible) map, e.g.
    paper_1709_04145_b200.rotation_vector_matrix, because the hip offsets use it.
    """
    s = Scene()
    s.links.append(LinkSpec(parent=None, joint=JointSpec(JointKind.free_joint),
                            geometry=BoxGeometry((0.4, 0.4, 0.1), 1000.0, (0.0, 0.0, 0.0))))
    leg = BoxGeometry((0.25, 0.06, 0.06), 1000.0, (0.125, 0.0, 0.0))
    c = 0.18
    angles = [math.pi / 4.0, 3.0 * math.pi / 4.0, -3.0 * math.pi / 4.0, -math.pi / 4.0]
    cx = [c, -c, -c, c]
    cy = [c, c, -c, -c]
    for l in range(4):
        off = translation(cx[l], cy[l], 0.0) @ _rotation_z(angles[l], rotation_vector_matrix)
        s.links.append(LinkSpec(parent=0, joint=JointSpec(JointKind.ball, (0.0, 0.0, 1.0), off),
                                geometry=leg))
        s.links.append(LinkSpec(parent=1 + 2 * l,
                                joint=JointSpec(JointKind.hinge, (0.0, 1.0, 0.0), translation(0.25, 0.0, 0.0)),
                                geometry=leg))
    s.gravity = (0.0, 0.0, -9.81)
    s.contact = ContactModel((0.0, 0.0, 1.0), 0.0, 2.0e4, 2.0e2)
    s.dt, s.duration = 0.01, 3.0
    s.q0 = np.zeros(22)
    s.qdot0 = np.zeros(22)
    s.q0[2] = 0.4
    for l in range(4):
        s.q0[6 + 4 * l + 1] = 0.5
        s.q0[6 + 4 * l + 3] = 0.4
    return s


def make_humanoid_scene() -> Scene:
    """18-link, 41-DOF humanoid tree (C4)."""
    X, Y = (1.0, 0.0, 0.0), (0.0, 1.0, 0.0)
    rows = [
        # parent, kind, axis, offset translation, size, center
        (None, JointKind.free_joint, None, (0, 0, 0), (0.30, 0.20, 0.15), (0, 0, 0)),
        (0, JointKind.ball, None, (0, 0, 0.075), (0.25, 0.18, 0.20), (0, 0, 0.10)),
        (1, JointKind.ball, None, (0, 0, 0.20), (0.30, 0.20, 0.25), (0, 0, 0.125)),
        (2, JointKind.ball, None, (0, 0, 0.25), (0.15, 0.15, 0.20), (0, 0, 0.10)),
        (2, JointKind.ball, None, (0, 0.18, 0.22), (0.08, 0.08, 0.28), (0, 0, -0.14)),
        (4, JointKind.hinge, Y, (0, 0, -0.28), (0.07, 0.07, 0.25), (0, 0, -0.125)),
        (5, JointKind.hinge, X, (0, 0, -0.25), (0.05, 0.08, 0.10), (0, 0, -0.05)),
        (2, JointKind.ball, None, (0, -0.18, 0.22), (0.08, 0.08, 0.28), (0, 0, -0.14)),
        (7, JointKind.hinge, Y, (0, 0, -0.28), (0.07, 0.07, 0.25), (0, 0, -0.125)),
        (8, JointKind.hinge, X, (0, 0, -0.25), (0.05, 0.08, 0.10), (0, 0, -0.05)),
        (0, JointKind.ball, None, (0, 0.10, -0.075), (0.10, 0.10, 0.40), (0, 0, -0.20)),
        (10, JointKind.hinge, Y, (0, 0, -0.40), (0.09, 0.09, 0.38), (0, 0, -0.19)),
        (11, JointKind.ball, None, (0, 0, -0.38), (0.18, 0.08, 0.05), (0.05, 0, -0.025)),
        (12, JointKind.hinge, Y, (0.14, 0, -0.05), (0.06, 0.08, 0.03), (0.03, 0, 0)),
        (0, JointKind.ball, None, (0, -0.10, -0.075), (0.10, 0.10, 0.40), (0, 0, -0.20)),
        (14, JointKind.hinge, Y, (0, 0, -0.40), (0.09, 0.09, 0.38), (0, 0, -0.19)),
        (15, JointKind.ball, None, (0, 0, -0.38), (0.18, 0.08, 0.05), (0.05, 0, -0.025)),
        (16, JointKind.hinge, Y, (0.14, 0, -0.05), (0.06, 0.08, 0.03), (0.03, 0, 0)),
    ]
    s = Scene()
    for parent, kind, axis, t, size, center in rows:
        s.links.append(LinkSpec(parent=parent,
                                joint=JointSpec(kind, axis if axis is not None else (0.0, 0.0, 1.0),
                                                translation(*[float(v) for v in t])),
                                geometry=BoxGeometry(tuple(float(v) for v in size), 1000.0,
                                                     tuple(float(v) for v in center))))
    s.gravity = (0.0, 0.0, -9.81)
    s.dt, s.duration = 0.01, 1.0
    s.q0 = np.zeros(41)
    s.q0[2] = 1.0
    s.qdot0 = np.zeros(41)
    return s


class MT19937:
    """std::mt19937 (32-bit Mersenne Twister), bit-exact with libstdc++."""

    def __init__(self, seed: int = 5489):
        self.mt = [0] * 624
        self.mt[0] = seed & 0xFFFFFFFF
        for i in range(1, 624):
            self.mt[i] = (1812433253 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 30)) + i) & 0xFFFFFFFF
        self.idx = 624

    def _twist(self):
        mt = self.mt
        for i in range(624):
            y = (mt[i] & 0x80000000) | (mt[(i + 1) % 624] & 0x7FFFFFFF)
            v = mt[(i + 397) % 624] ^ (y >> 1)
            if y & 1:
                v ^= 0x9908B0DF
            mt[i] = v
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 624:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= y >> 11
        y ^= (y << 7) & 0x9D2C5680
        y ^= (y << 15) & 0xEFC60000
        y ^= y >> 18
        return y & 0xFFFFFFFF


def _mt_words(seed: int, count: int) -> np.ndarray:
    """count 32-bit outputs of std::mt19937(seed), twist and tempering vectorised."""
    mt = np.zeros(624, dtype=np.uint64)
    mt[0] = seed & 0xFFFFFFFF
    for i in range(1, 624):
        prev = int(mt[i - 1])
        mt[i] = (1812433253 * (prev ^ (prev >> 30)) + i) & 0xFFFFFFFF
    mt = mt.astype(np.uint32)
    out = np.empty(count, dtype=np.uint32)
    upper, lower, matrix = np.uint32(0x80000000), np.uint32(0x7FFFFFFF), np.uint32(0x9908B0DF)

    def twist(mt):
        mt = mt.copy()
        for a, b in ((0, 227), (227, 454), (454, 623)):
            y = (mt[a:b] & upper) | (mt[a + 1:b + 1] & lower)
            sh = 397 if a < 227 else 397 - 624
            v = mt[a + sh:b + sh] ^ (y >> np.uint32(1))
            v ^= np.where((y & np.uint32(1)) != 0, matrix, np.uint32(0))
            mt[a:b] = v
        y = (mt[623] & upper) | (mt[0] & lower)
        v = mt[396] ^ (y >> np.uint32(1))
        if y & 1:
            v ^= matrix
        mt[623] = v
        return mt

    pos = 0
    while pos < count:
        mt = twist(mt)
        y = mt.copy()
        y ^= y >> np.uint32(11)
        y ^= (y << np.uint32(7)) & np.uint32(0x9D2C5680)
        y ^= (y << np.uint32(15)) & np.uint32(0xEFC60000)
        y ^= y >> np.uint32(18)
        take = min(624, count - pos)
        out[pos:pos + take] = y[:take]
        pos += take
    return out


def mt19937_uniform(seed: int, count: int, lo: float, hi: float) -> np.ndarray:
    """count draws of std::uniform_real_distribution<double>(lo, hi)(std::mt19937(seed)).

    libstdc++ generate_canonical<double, 53> consumes two 32-bit words:
    (w0 + w1 * 2^32) / 2^64, clamped below 1, then (hi - lo) * u + lo.
    """
    w = _mt_words(seed, 2 * count).astype(np.float64)
    s = w[0::2] + w[1::2] * 4294967296.0
    u = s / 18446744073709551616.0
    u = np.where(u >= 1.0, 1.0 - 2.0 ** -53, u)
    return (u * (hi - lo)) + lo
