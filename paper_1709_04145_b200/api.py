"""Reference-shaped Python API over the C ABI (drop-in for the step path).

Mirrors /root/reference/proj/include/pbad:
  build_model / body_integral / validate_configuration   model.hpp:91-100
  rotation_vector_matrix                                  kinematics.hpp:39
  build_scheme / CollocationScheme                        collocation.hpp:14-39
  StepProblem / StepObjective (value, evaluate)           objective.hpp:64-132
  minimize                                                optim.hpp:58-60
  simulate / batch_simulate                               stepper.hpp:49-64
Every numeric routine runs in libpbad_gpu.so (host parts of build_model /
build_scheme in C++, everything per-step in sm_100a kernels).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import check
from .types import (EnergySample, ForceModel, JointKind, LinkSpec, ModelError, ObjectiveKind, OptimizerConfig,
                    OptimizerKind, SimConfig, SolveReport, Trajectory)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


def _f64(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a.reshape(shape) if shape is not None else a


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _pi(a):
    return None if a is None else a.ctypes.data_as(_ip)


def _link_struct(link: LinkSpec, keep: list) -> _lib.LinkSpec:
    s = _lib.LinkSpec()
    s.parent = -1 if link.parent is None else int(link.parent)
    j = link.joint
    s.joint_kind = int(j.kind)
    s.axis[:] = [float(v) for v in j.axis]
    s.offset[:] = [float(v) for v in _f64(j.offset).reshape(4, 4).T.reshape(-1)]
    g = link.geometry
    if hasattr(g, "masses"):
        s.geom_kind = 1
        pm = _f64([m.mass for m in g.masses])
        pp = _f64([list(m.position) for m in g.masses]) if g.masses else np.zeros((0, 3))
        keep += [pm, pp]
        s.n_points = len(g.masses)
        s.point_mass = _p(pm)
        s.point_pos = _p(pp)
    else:
        s.geom_kind = 0
        s.box_size[:] = [float(v) for v in g.size]
        s.box_density = float(g.density)
        s.box_center[:] = [float(v) for v in g.center]
    if link.contact_samples:
        smp = _f64([list(p) for p in link.contact_samples])
        keep.append(smp)
        s.n_samples = len(link.contact_samples)
        s.samples = _p(smp)
    return s


class KinematicModel:
    """Immutable articulated tree built by build_model (model.hpp:71-88)."""

    def __init__(self, links: Sequence[LinkSpec]):
        L = _lib.load()
        keep: list = []
        arr = (_lib.LinkSpec * max(1, len(links)))()
        for i, l in enumerate(links):
            arr[i] = _link_struct(l, keep)
        h = C.c_void_p()
        check(L.pbad_gpu_model_create(arr, len(links), C.byref(h)))
        self._h = h
        self.links = list(links)
        self.total_dofs = L.pbad_gpu_model_dofs(h)
        N = L.pbad_gpu_model_links(h)
        S = np.zeros((N, 16))
        mass = np.zeros(N)
        off = np.zeros(N, dtype=np.int32)
        axis = np.zeros((N, 3))
        sc = np.zeros(N, dtype=np.int32)
        L.pbad_gpu_model_info(h, _p(S), _p(mass), _pi(off), _p(axis), _pi(sc))
        self.body_S = S.reshape(N, 4, 4).transpose(0, 2, 1).copy()  # row-major
        self.body_mass = mass
        self.dof_offsets = off.tolist()
        self.axes = axis
        self.sample_counts = sc

    @property
    def handle(self):
        return self._h

    def link_count(self) -> int:
        return len(self.links)

    def dof_offset(self, link: int) -> int:
        return self.dof_offsets[link]

    def dof_count(self, link: int) -> int:
        return self.links[link].joint.dof_count()

    def parent(self, link: int) -> int:
        p = self.links[link].parent
        return -1 if p is None else p

    def total_mass(self) -> float:
        m = 0.0
        for v in self.body_mass:
            m += float(v)
        return m

    def __del__(self):
        try:
            _lib.load().pbad_gpu_model_destroy(self._h)
        except Exception:
            pass


def build_model(links: Sequence[LinkSpec]) -> KinematicModel:
    return KinematicModel(links)


def body_integral(geometry) -> Tuple[np.ndarray, float]:
    keep: list = []
    s = _link_struct(LinkSpec(geometry=geometry), keep)
    S = np.zeros(16)
    m = C.c_double()
    check(_lib.load().pbad_gpu_body_integral(C.byref(s), _p(S), C.byref(m)))
    return S.reshape(4, 4).T.copy(), m.value


def validate_configuration(model: KinematicModel, q) -> None:
    q = _f64(q)
    check(_lib.load().pbad_gpu_validate_configuration(model.handle, _p(q), len(q)))


def rotation_vector_matrix(theta) -> np.ndarray:
    R = np.zeros(9)
    check(_lib.load().pbad_gpu_rotation_vector_matrix(_p(_f64(theta)), _p(R)))
    return R.reshape(3, 3).T.copy()


def rotation_vector_from_matrix(R) -> np.ndarray:
    """Principal-branch rotation vector of a 3x3 rotation (scene.cpp:66-86)."""
    th = np.zeros(3)
    check(_lib.load().pbad_gpu_rotation_vector_from_matrix(_p(_f64(np.asarray(R, dtype=np.float64).T.reshape(9))),
                                                           _p(th)))
    return th


@dataclass
class CollocationScheme:
    order: int
    alphas: np.ndarray
    times: np.ndarray
    H: np.ndarray
    H2: np.ndarray

    def point_count(self) -> int:
        return self.order + 1

    def unknown_count(self) -> int:
        return self.order - 1

    def unknown_index(self, m: int) -> int:
        return 2 + m

    def stencil(self, m: int) -> np.ndarray:
        return self.H2[:, self.unknown_index(m)].copy()


def build_scheme(order: int, dt: float) -> CollocationScheme:
    k = order + 1
    if order < 2:
        raise ValueError("collocation order must be >= 2")
    al = np.zeros(max(1, order - 1))
    t = np.zeros(k)
    H = np.zeros(k * k)
    H2 = np.zeros(k * k)
    check(_lib.load().pbad_gpu_build_scheme(order, float(dt), _p(al), _p(t), _p(H), _p(H2)))
    return CollocationScheme(order, al[: order - 1], t, H.reshape(k, k).T.copy(), H2.reshape(k, k).T.copy())


def legendre_points(order: int) -> np.ndarray:
    return build_scheme(order, 1.0).alphas


def _forces_struct(forces: Optional[ForceModel], keep: list) -> _lib.Forces:
    f = _lib.Forces()
    if forces is None:
        return f
    f.gravity[:] = [float(v) for v in forces.gravity]
    f.drag_d = float(forces.drag_d)
    if forces.contact is not None:
        c = forces.contact
        f.has_contact = 1
        f.plane_normal[:] = [float(v) for v in c.plane_normal]
        f.plane_offset = float(c.plane_offset)
        f.contact_d1 = float(c.d1)
        f.contact_d2 = float(c.d2)
    if forces.tau is not None and len(forces.tau):
        t = _f64(forces.tau)
        keep.append(t)
        f.tau_len = len(t)
        f.tau = _p(t)
    if forces.actuation is not None:
        a = forces.actuation
        f.has_actuation = 1
        f.act_kind = int(a.kind)
        amp = _f64(a.amplitude if a.amplitude is not None else [])
        ph = _f64(a.phase if a.phase is not None else [])
        keep += [amp, ph]
        f.act_len = len(amp)
        f.act_amplitude = _p(amp)
        f.act_frequency_hz = float(a.frequency_hz)
        f.act_phase_len = len(ph)
        f.act_phase = _p(ph)
    return f


def _sim_struct(sim: SimConfig) -> _lib.SimDesc:
    s = _lib.SimDesc()
    s.dt = float(sim.dt)
    s.duration = float(sim.duration)
    s.order = int(sim.order)
    s.objective = int(sim.objective)
    o = sim.optimizer
    s.opt.kind = int(o.kind)
    s.opt.max_iters = int(o.max_iters)
    s.opt.grad_tol = float(o.grad_tol)
    s.opt.grad_rtol = float(o.grad_rtol)
    s.opt.ftol = float(o.ftol)
    s.opt.lbfgs_memory = int(o.lbfgs_memory)
    s.opt.lm_lambda0 = float(o.lm_lambda0)
    s.opt.lm_lambda_factor = float(o.lm_lambda_factor)
    s.opt.lm_lambda_max = float(o.lm_lambda_max)
    s.opt.armijo_c1 = float(o.armijo_c1)
    s.opt.backtrack_factor = float(o.backtrack_factor)
    s.opt.max_line_search = int(o.max_line_search)
    s.consecutive_fail_limit = int(sim.consecutive_fail_limit)
    s.refined_bootstrap = int(bool(sim.refined_bootstrap))
    s.warm_start = int(bool(sim.warm_start))
    return s


def total_steps(sim: SimConfig) -> int:
    return int(math.ceil(sim.duration / sim.dt - 1e-9))


TRAJ_OK, TRAJ_FAIL_LIMIT, TRAJ_NONFINITE_INIT, TRAJ_NONFINITE_CFG, TRAJ_RUNNING = 0, 1, 2, 3, 4
TRAJ_BOOTSTRAP_SINGULAR = 8


class GpuContext:
    """pbad_gpu_ctx: one model + forces + schedule bound to one device."""

    def __init__(self, model: KinematicModel, forces: Optional[ForceModel], sim: SimConfig, device: int = 0,
                 max_batch: int = 1):
        self.model = model
        self.sim = sim
        self._keep: list = []
        f = _forces_struct(forces, self._keep)
        s = _sim_struct(sim)
        h = C.c_void_p()
        check(_lib.load().pbad_gpu_create(model.handle, C.byref(f), C.byref(s), int(device), int(max_batch),
                                          C.byref(h)))
        self._h = h
        self.max_batch = max_batch
        self.total_steps = _lib.load().pbad_gpu_total_steps(h)
        # kernel family: 0 general, 1 chain (quad), 2 chain v4 (warp-synchronous)
        self.path = _lib.load().pbad_gpu_path(h)
        self.n = model.total_dofs
        self.dim = self.n * (sim.order - 1)

    def __del__(self):
        try:
            _lib.load().pbad_gpu_destroy(self._h)
        except Exception:
            pass

    def _out_struct(self, B: int, want_q=True, want_energy=True, pinned=False, want_itv=False):
        S, n = self.total_steps, self.n
        if pinned:
            import torch

            def z(shape, dt=np.float64):
                tdt = {np.float64: torch.float64, np.int32: torch.int32, np.float32: torch.float32}[dt]
                return torch.zeros(shape, dtype=tdt).pin_memory().numpy()
        else:
            def z(shape, dt=np.float64):
                return np.zeros(shape, dt)
        bufs = dict(
            q=z((B, S + 1, n)) if want_q else None,
            energy=z((B, S + 1, 2)) if want_energy else None,
            iterations=z((B, S), np.int32), converged=z((B, S), np.int32),
            accepted=z((B, S), np.int32), final_value=z((B, S)),
            final_grad_norm=z((B, S)), n_samples=z(B, np.int32), status=z(B, np.int32),
            fail_streak=z(B, np.int32), n_reports=z(B, np.int32),
            device_ms=z(1, np.float32),
            iteration_values=z((B, S, max(1, self.sim.optimizer.max_iters))) if want_itv else None)
        o = _lib.RolloutOut()
        for k, v in bufs.items():
            if v is None:
                continue
            if v.dtype == np.float64:
                setattr(o, k, _p(v))
            elif v.dtype == np.int32:
                setattr(o, k, _pi(v))
            else:
                setattr(o, k, v.ctypes.data_as(C.POINTER(C.c_float)))
        return o, bufs

    def make_outputs(self, B: int, want_q=True, want_energy=True, pinned=False, want_itv=False):
        """Caller-owned host output buffers for rollout(out=...) (the C ABI
        writes into buffers the caller allocated, stepper.hpp's Trajectory)."""
        return self._out_struct(B, want_q, want_energy, pinned, want_itv)

    def rollout(self, q0, qdot0, want_q=True, want_energy=True, pinned=False, out=None,
                want_itv=False) -> Dict[str, np.ndarray]:
        q0 = _f64(q0)
        B = q0.shape[0]
        q0 = _f64(q0, (B, self.n))
        qdot0 = _f64(qdot0, (B, self.n))
        if out is not None:
            o, bufs = out
            S = self.total_steps
            if bufs["status"].shape[0] != B or bufs["iterations"].shape != (B, S):
                raise ValueError("rollout: out buffers were allocated for a different batch or step count")
            for k, tail in (("q", (S + 1, self.n)), ("energy", (S + 1, 2))):
                if bufs[k] is not None and bufs[k].shape != (B,) + tail:
                    raise ValueError(f"rollout: out[{k!r}] has shape {bufs[k].shape}, expected {(B,) + tail}")
        else:
            o, bufs = self._out_struct(B, want_q, want_energy, pinned, want_itv)
        check(_lib.load().pbad_gpu_rollout(self._h, B, _p(q0), _p(qdot0), C.byref(o)))
        return bufs

    # device-resident stepping (bench `value` leg); pointers are device addresses
    def begin(self, B: int, d_q0: int, d_qdot0: int, stream: int = 0):
        check(_lib.load().pbad_gpu_begin(self._h, int(B), C.c_void_p(d_q0), C.c_void_p(d_qdot0),
                                         C.c_void_p(stream) if stream else None))
        self._B = B

    def advance(self, n_steps: int, stream: int = 0):
        check(_lib.load().pbad_gpu_advance(self._h, int(n_steps), C.c_void_p(stream) if stream else None))

    def kernel_launches(self) -> int:
        """Step kernels this context has launched so far (pbad_gpu_kernel_launches)."""
        return int(_lib.load().pbad_gpu_kernel_launches(self._h))

    def sync_outputs(self, want_q=True, want_energy=True) -> Dict[str, np.ndarray]:
        o, bufs = self._out_struct(self._B, want_q, want_energy)
        check(_lib.load().pbad_gpu_sync_outputs(self._h, C.byref(o)))
        return bufs

    def state_device_ptr(self) -> int:
        return _lib.load().pbad_gpu_state_device(self._h)

    def final_state(self, d_dst: int, stream: int = 0):
        """Latest configuration of every environment of the current batch into
        the device buffer d_dst [B][n] (no host round trip)."""
        check(_lib.load().pbad_gpu_final_state(self._h, C.c_void_p(d_dst), C.c_void_p(stream) if stream else None))

    def eval(self, history, x, want_grad=True, want_gn=False, tau=None):
        history = _f64(history)
        B = history.shape[0]
        x = _f64(x, (B, self.dim))
        tau = None if tau is None else _f64(tau, (B, self.dim))
        value = np.zeros(B)
        grad = np.zeros((B, self.dim))
        gn = np.zeros((B, self.dim, self.dim)) if want_gn else None
        check(_lib.load().pbad_gpu_eval(self._h, B, _p(history), _p(tau), _p(x), int(want_grad), int(want_gn),
                                        _p(value), _p(grad), _p(gn)))
        if gn is not None:
            gn = gn.transpose(0, 2, 1).copy()  # column-major -> row-major
        return value, grad, gn

    def simulate_baseline(self, scheme, q0, qdot0, want_q=True, want_energy=True) -> Dict[str, np.ndarray]:
        """Explicit Newton-Euler rollouts (simulate_baseline, stepper.cpp:168-202)
        with this context's model, forces, dt and duration."""
        q0 = _f64(q0)
        B = q0.shape[0]
        n, S = self.n, self.total_steps
        q0 = _f64(q0, (B, n))
        qdot0 = _f64(qdot0, (B, n))
        q = np.zeros((B, S + 1, n)) if want_q else None
        en = np.zeros((B, S + 1, 2)) if want_energy else None
        ns = np.zeros(B, np.int32)
        st = np.zeros(B, np.int32)
        check(_lib.load().pbad_gpu_simulate_baseline(self._h, int(scheme), B, _p(q0), _p(qdot0), _p(q), _p(en),
                                                     _pi(ns), _pi(st)))
        return dict(q=q, energy=en, n_samples=ns, status=st)

    def correlation(self, qa, qb, weight_per_body=None, want=("value", "grad", "bb", "ab")):
        """Batched correlation derivatives of (qa[b], qb[b]) (adjoint.cpp:178-192):
        value [B], grad_b [B, n], hess_bb / hess_ab [B, n, n] (None where not
        wanted)."""
        qa = _f64(qa)
        B = qa.shape[0]
        n = self.n
        qa = _f64(qa, (B, n))
        qb = _f64(qb, (B, n))
        w = None
        if weight_per_body is not None and len(weight_per_body) != 0:
            w = _f64(weight_per_body)
            if len(w) != self.model.link_count():
                raise ModelError("weight_per_body length does not match link count")
        v = np.zeros(B) if "value" in want else None
        g = np.zeros((B, n)) if "grad" in want else None
        bb = np.zeros((B, n, n)) if "bb" in want else None
        ab = np.zeros((B, n, n)) if "ab" in want else None
        check(_lib.load().pbad_gpu_correlation(self._h, B, _p(qa), _p(qb), _p(w), _p(v), _p(g), _p(bb), _p(ab)))
        if bb is not None:
            bb = bb.transpose(0, 2, 1).copy()  # column-major -> row-major
        if ab is not None:
            ab = ab.transpose(0, 2, 1).copy()
        return v, g, bb, ab

    def correlation_suite(self, qa, qb, weight_per_body=None, want=("value", "grad", "bb", "ab")):
        """parallel_correlation_suite (adjoint.cpp:241-336) for a batch of pairs:
        one CTA per pair, the per-link work items over its threads; outputs as
        correlation()."""
        qa = _f64(qa)
        B = qa.shape[0]
        n = self.n
        qa = _f64(qa, (B, n))
        qb = _f64(qb, (B, n))
        w = None
        if weight_per_body is not None and len(weight_per_body) != 0:
            w = _f64(weight_per_body)
            if len(w) != self.model.link_count():
                raise ModelError("weight_per_body length does not match link count")
        v = np.zeros(B) if "value" in want else None
        g = np.zeros((B, n)) if "grad" in want else None
        bb = np.zeros((B, n, n)) if "bb" in want else None
        ab = np.zeros((B, n, n)) if "ab" in want else None
        check(_lib.load().pbad_gpu_correlation_suite(self._h, B, _p(qa), _p(qb), _p(w), _p(v), _p(g), _p(bb), _p(ab)))
        t = (lambda a: None if a is None else a.transpose(0, 2, 1).copy())
        return v, g, t(bb), t(ab)

    def functional(self, q, seeds, want=("value", "grad", "hess")):
        """functional_value / functional_grad / functional_hess (adjoint.cpp:43-101)
        of f(q) = sum_i ddot(C_i, T^i(q)): q [B, n], seeds [B, N, 4, 4]."""
        q = _f64(q)
        B = q.shape[0]
        n, N = self.n, self.model.link_count()
        q = _f64(q, (B, n))
        sd = np.asarray(seeds, dtype=np.float64)
        if sd.shape != (B, N, 4, 4):
            raise ValueError(f"seeds must have shape {(B, N, 4, 4)}")
        sd = np.ascontiguousarray(sd.transpose(0, 1, 3, 2))  # column-major 4x4 blocks
        v = np.zeros(B) if "value" in want else None
        g = np.zeros((B, n)) if "grad" in want else None
        h = np.zeros((B, n, n)) if "hess" in want else None
        check(_lib.load().pbad_gpu_functional(self._h, B, _p(q), _p(sd), _p(v), _p(g), _p(h)))
        return v, g, (None if h is None else h.transpose(0, 2, 1).copy())

    def minimize(self, history, x0, tau=None):
        history = _f64(history)
        B = history.shape[0]
        x0 = _f64(x0, (B, self.dim))
        tau = None if tau is None else _f64(tau, (B, self.dim))
        xo = np.zeros((B, self.dim))
        it = np.zeros(B, np.int32)
        cv = np.zeros(B, np.int32)
        fv = np.zeros(B)
        gnm = np.zeros(B)
        check(_lib.load().pbad_gpu_minimize(self._h, B, _p(history), _p(tau), _p(x0), _p(xo), _pi(it), _pi(cv),
                                            _p(fv), _p(gnm)))
        return xo, it, cv, fv, gnm


def _trajectories(ctx: GpuContext, sims: Sequence[SimConfig], bufs) -> List[Trajectory]:
    out = []
    for b, sim in enumerate(sims):
        tr = Trajectory()
        k = int(bufs["n_samples"][b])
        for s in range(k):
            tr.samples.append((s * sim.dt, bufs["q"][b, s].copy()))
            tr.energy_log.append(EnergySample(s * sim.dt, float(bufs["energy"][b, s, 0]),
                                              float(bufs["energy"][b, s, 1])))
        for s in range(int(bufs["n_reports"][b])):
            its = int(bufs["iterations"][b, s])
            itv = bufs.get("iteration_values")
            tr.solve_reports.append(SolveReport(its, float(bufs["final_value"][b, s]),
                                                float(bufs["final_grad_norm"][b, s]),
                                                bool(bufs["converged"][b, s]), int(bufs["accepted"][b, s]),
                                                [] if itv is None else itv[b, s, :its].tolist()))
        st = int(bufs["status"][b])
        if st == TRAJ_FAIL_LIMIT:
            steps = max(0, k - 1)
            tr.error = (f"optimizer failed {int(bufs['fail_streak'][b])} consecutive steps around "
                        f"t={steps * sim.dt:f}")
        elif st == TRAJ_NONFINITE_INIT:
            tr.error = "objective is non-finite at the initial point"
        elif st == TRAJ_NONFINITE_CFG:
            tr.error = "configuration contains a non-finite entry"
        elif st == TRAJ_BOOTSTRAP_SINGULAR:
            tr.error = "singular generalized mass matrix"
        out.append(tr)
    return out


def rollout_sharded(ctxs: Sequence[GpuContext], q0, qdot0, want_q=True, want_energy=True, pinned=False,
                    out=None, want_itv=False) -> Dict[str, np.ndarray]:
    """One batch over several contexts (one per device, or several on one):
    context i steps the contiguous shard [B*i/k, B*(i+1)/k) of the batch,
    all concurrently (pbad_gpu_rollout_sharded); equal to one context's
    rollout bit for bit."""
    if not ctxs:
        raise ValueError("rollout_sharded needs at least one context")
    c0 = ctxs[0]
    q0 = _f64(q0)
    B = q0.shape[0]
    q0 = _f64(q0, (B, c0.n))
    qdot0 = _f64(qdot0, (B, c0.n))
    o, bufs = out if out is not None else c0._out_struct(B, want_q, want_energy, pinned, want_itv)
    arr = (C.c_void_p * len(ctxs))(*[c._h for c in ctxs])
    check(_lib.load().pbad_gpu_rollout_sharded(arr, len(ctxs), B, _p(q0), _p(qdot0), C.byref(o)))
    return bufs


def _check_sim(model: KinematicModel, sim: SimConfig):
    validate_configuration(model, sim.q0)
    if sim.qdot0 is None or len(sim.qdot0) != model.total_dofs:
        raise ModelError("initial velocity length does not match model DOF count")
    if sim.dt <= 0.0 or sim.duration <= 0.0:
        raise ModelError("dt and duration must be positive")


def batch_simulate(model: KinematicModel, forces: ForceModel, sims: Sequence[SimConfig], workers: int = 1,
                   device: int = 0, devices: Optional[Sequence[int]] = None,
                   record_iteration_values: bool = False) -> List[Trajectory]:
    """stepper.cpp:204-270: per-trajectory results equal simulate(); errors are
    recorded per trajectory.  `workers` is accepted for signature parity (the
    GPU grid replaces the WorkerPool).  `devices` shards every group of
    trajectories over those devices (one context each, contiguous shards)."""
    if workers < 1:
        raise ModelError("worker count must be >= 1")
    results: List[Optional[Trajectory]] = [None] * len(sims)
    groups: List[Tuple[SimConfig, List[int]]] = []
    for i, sim in enumerate(sims):
        try:
            _check_sim(model, sim)
        except (ModelError, ValueError) as e:
            results[i] = Trajectory(error=str(e))
            continue
        for rep, idx in groups:
            if rep.same_schedule(sim):
                idx.append(i)
                break
        else:
            groups.append((sim, [i]))
    for rep, idx in groups:
        q0 = np.stack([_f64(sims[i].q0) for i in idx])
        qd = np.stack([_f64(sims[i].qdot0) for i in idx])
        devs = list(devices) if devices else [device]
        devs = devs[:len(idx)]
        if len(devs) > 1:
            shard = -(-len(idx) // len(devs))
            ctxs = [GpuContext(model, forces, rep, device=d, max_batch=shard) for d in devs]
            ctx = ctxs[0]
            bufs = rollout_sharded(ctxs, q0, qd, want_itv=record_iteration_values)
        else:
            ctx = GpuContext(model, forces, rep, device=devs[0], max_batch=len(idx))
            bufs = ctx.rollout(q0, qd, want_itv=record_iteration_values)
        for i, tr in zip(idx, _trajectories(ctx, [sims[i] for i in idx], bufs)):
            results[i] = tr
    return results  # type: ignore[return-value]


def simulate(model: KinematicModel, forces: ForceModel, sim: SimConfig, device: int = 0) -> Trajectory:
    """stepper.cpp:151-166: raises RuntimeError when the fail limit is hit."""
    _check_sim(model, sim)
    ctx = GpuContext(model, forces, sim, device=device, max_batch=1)
    bufs = ctx.rollout(_f64(sim.q0)[None], _f64(sim.qdot0)[None])
    tr = _trajectories(ctx, [sim], bufs)[0]
    st = int(bufs["status"][0])
    if st in (TRAJ_FAIL_LIMIT, TRAJ_BOOTSTRAP_SINGULAR):
        raise RuntimeError(tr.error)
    if st == TRAJ_NONFINITE_INIT:
        raise ValueError(tr.error)
    if st == TRAJ_NONFINITE_CFG:
        raise ModelError(tr.error)
    return tr


@dataclass
class StepProblem:
    """objective.hpp:64-74 (scheme given by order)."""
    model: KinematicModel
    order: int
    history: Tuple[np.ndarray, np.ndarray]
    dt: float
    forces: ForceModel = field(default_factory=ForceModel)
    kind: ObjectiveKind = ObjectiveKind.energy_form
    tau_at_instants: Optional[List[np.ndarray]] = None


class StepObjective:
    """objective.hpp:115-132 on the GPU (batch of one; see GpuContext.eval)."""

    def __init__(self, problem: StepProblem, device: int = 0):
        self.problem = problem
        sim = SimConfig(dt=problem.dt, duration=problem.dt, order=problem.order, objective=problem.kind,
                        optimizer=OptimizerConfig(kind=OptimizerKind.lm))
        self._ctx = GpuContext(problem.model, problem.forces, sim, device=device, max_batch=1)
        self._hist = np.concatenate([_f64(problem.history[0]), _f64(problem.history[1])])[None]
        self._tau = None
        if problem.tau_at_instants:
            self._tau = np.concatenate([_f64(t) for t in problem.tau_at_instants])[None]

    def dim(self) -> int:
        return self._ctx.dim

    def value(self, x) -> float:
        v, _, _ = self._ctx.eval(self._hist, _f64(x)[None], want_grad=False, tau=self._tau)
        return float(v[0])

    def evaluate(self, x, want_gn: bool = False):
        v, g, gn = self._ctx.eval(self._hist, _f64(x)[None], want_grad=True, want_gn=want_gn, tau=self._tau)
        return float(v[0]), g[0], (gn[0] if gn is not None else None)


# --- correlation functional (adjoint.hpp:15-82) --------------------------------

@dataclass
class CorrelationRequest:
    model: KinematicModel
    qa: np.ndarray
    qb: np.ndarray
    weight_per_body: Optional[np.ndarray] = None  # empty / None = all ones


@dataclass
class CorrelationDerivatives:
    value: float
    grad_b: np.ndarray
    hess_bb: np.ndarray
    hess_ab: np.ndarray


def _corr_ctx(model: KinematicModel, device: int = 0) -> GpuContext:
    # one cached context per (model, device)
    per_dev = model.__dict__.setdefault("_corr_ctx", {})
    ctx = per_dev.get(device)
    if ctx is None:
        ctx = GpuContext(model, ForceModel(), SimConfig(dt=0.01, duration=0.01), device=device)
        per_dev[device] = ctx
    return ctx


def correlation_and_grad(req: CorrelationRequest) -> Tuple[float, np.ndarray]:
    v, g, _, _ = _corr_ctx(req.model).correlation(_f64(req.qa)[None], _f64(req.qb)[None], req.weight_per_body,
                                                    want=("value", "grad"))
    return float(v[0]), g[0]


def hessian_bb(req: CorrelationRequest) -> np.ndarray:
    return _corr_ctx(req.model).correlation(_f64(req.qa)[None], _f64(req.qb)[None], req.weight_per_body,
                                            want=("bb",))[2][0]


def hessian_ab(req: CorrelationRequest) -> np.ndarray:
    return _corr_ctx(req.model).correlation(_f64(req.qa)[None], _f64(req.qb)[None], req.weight_per_body,
                                            want=("ab",))[3][0]


def batch_correlation(model: KinematicModel, qa, qb, weight_per_body=None, device: int = 0):
    """All four derivatives for a batch of pairs in one launch."""
    v, g, bb, ab = _corr_ctx(model, device).correlation(qa, qb, weight_per_body)
    return [CorrelationDerivatives(float(v[b]), g[b], bb[b], ab[b]) for b in range(len(v))]


def parallel_correlation_suite(req: CorrelationRequest, workers: int = 1, device: int = 0) -> CorrelationDerivatives:
    """adjoint.hpp:103-108: value, grad_b, hess_bb, hess_ab in one launch, the
    per-link work items spread over one CTA (the large-N mode).  `workers` is
    validated like the reference (>= 1); the CTA's threads replace the pool."""
    if workers < 1:
        raise ModelError("worker count must be >= 1")
    v, g, bb, ab = _corr_ctx(req.model, device).correlation_suite(_f64(req.qa)[None], _f64(req.qb)[None],
                                                                  req.weight_per_body)
    return CorrelationDerivatives(float(v[0]), g[0], bb[0], ab[0])


def functional_value(model: KinematicModel, seeds, q, device: int = 0) -> float:
    """adjoint.hpp:55 on the GPU: sum_i ddot(C_i, T^i(q)), seeds [N, 4, 4]."""
    return float(_corr_ctx(model, device).functional(_f64(q)[None], np.asarray(seeds)[None], want=("value",))[0][0])


def functional_grad(model: KinematicModel, seeds, q, device: int = 0) -> np.ndarray:
    """adjoint.hpp:56-57 on the GPU."""
    return _corr_ctx(model, device).functional(_f64(q)[None], np.asarray(seeds)[None], want=("grad",))[1][0]


def functional_hess(model: KinematicModel, seeds, q, device: int = 0) -> np.ndarray:
    """adjoint.hpp:58-59 on the GPU: the exact Hessian of the linear functional."""
    return _corr_ctx(model, device).functional(_f64(q)[None], np.asarray(seeds)[None], want=("hess",))[2][0]


# --- Newton-Euler baselines (stepper.hpp:54-55) -------------------------------

_BL_ERRORS = {6: "step failed: singular generalized mass matrix",
              7: "step failed: configuration contains a non-finite entry"}


def simulate_baseline(model: KinematicModel, forces: ForceModel, scheme, sim: SimConfig,
                      device: int = 0) -> Trajectory:
    """stepper.cpp:168-202 on the GPU: samples, analytic KE / PE log, the
    reference's error texts (no solve reports)."""
    return batch_simulate_baseline(model, forces, scheme, [sim], device)[0]


def batch_simulate_baseline(model: KinematicModel, forces: ForceModel, scheme, sims: Sequence[SimConfig],
                            device: int = 0) -> List[Trajectory]:
    """simulate_baseline for trajectories that share dt / duration (one launch)."""
    sims = list(sims)
    for sim in sims:
        validate_configuration(model, sim.q0)
        if sim.qdot0 is None or len(sim.qdot0) != model.total_dofs:
            raise ModelError("initial velocity length does not match model DOF count")
        if not sims[0].same_schedule(sim):
            raise ValueError("batch_simulate_baseline: trajectories must share dt and duration")
    ctx = GpuContext(model, forces, sims[0], device=device, max_batch=1)
    out = ctx.simulate_baseline(scheme, np.stack([_f64(s.q0) for s in sims]),
                                np.stack([_f64(s.qdot0) for s in sims]))
    trs = []
    for b, sim in enumerate(sims):
        tr = Trajectory()
        k = int(out["n_samples"][b])
        for s in range(k):
            tr.samples.append((s * sim.dt, out["q"][b, s].copy()))
            tr.energy_log.append(EnergySample(s * sim.dt, float(out["energy"][b, s, 0]),
                                              float(out["energy"][b, s, 1])))
        st = int(out["status"][b])
        if st == 5:
            tr.error = f"diverged to a non-finite state at t={(k - 1) * sim.dt:f}"
        elif st in _BL_ERRORS:
            tr.error = _BL_ERRORS[st]
        trs.append(tr)
    return trs
