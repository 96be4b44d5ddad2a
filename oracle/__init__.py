"""TEST INFRASTRUCTURE ONLY: ctypes binding of the CPU oracle (pbad_oracle.c).

The oracle restates the reference PBAD hot path in plain C and is the parity
checker for the CUDA path.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libpbad_oracle.so")
_lib = None

HINGE, BALL, FREE = 0, 1, 2
BOX, POINTS = 0, 1
LBFGS, LM = 0, 1
ENERGY, RESIDUAL = 0, 1

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class LinkSpecC(C.Structure):
    _fields_ = [
        ("parent", C.c_int32), ("joint_kind", C.c_int32), ("axis", C.c_double * 3),
        ("offset", C.c_double * 16), ("geom_kind", C.c_int32),
        ("box_size", C.c_double * 3), ("box_density", C.c_double),
        ("box_center", C.c_double * 3), ("n_points", C.c_int32),
        ("point_mass", _dp), ("point_pos", _dp), ("n_samples", C.c_int32),
        ("samples", _dp),
    ]


class ForcesC(C.Structure):
    _fields_ = [
        ("gravity", C.c_double * 3), ("drag_d", C.c_double), ("has_contact", C.c_int32),
        ("plane_normal", C.c_double * 3), ("plane_offset", C.c_double),
        ("contact_d1", C.c_double), ("contact_d2", C.c_double), ("tau_len", C.c_int32),
        ("tau", _dp), ("has_actuation", C.c_int32), ("act_kind", C.c_int32),
        ("act_len", C.c_int32), ("act_amplitude", _dp), ("act_frequency_hz", C.c_double),
        ("act_phase_len", C.c_int32), ("act_phase", _dp),
    ]


class OptimizerC(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("max_iters", C.c_int32), ("grad_tol", C.c_double),
        ("grad_rtol", C.c_double), ("ftol", C.c_double), ("lbfgs_memory", C.c_int32),
        ("lm_lambda0", C.c_double), ("lm_lambda_factor", C.c_double),
        ("lm_lambda_max", C.c_double), ("armijo_c1", C.c_double),
        ("backtrack_factor", C.c_double), ("max_line_search", C.c_int32),
    ]


class SimC(C.Structure):
    _fields_ = [
        ("dt", C.c_double), ("duration", C.c_double), ("order", C.c_int32),
        ("objective", C.c_int32), ("opt", OptimizerC), ("q0", _dp), ("qdot0", _dp),
        ("consecutive_fail_limit", C.c_int32), ("refined_bootstrap", C.c_int32),
        ("warm_start", C.c_int32),
    ]


class TrajectoryC(C.Structure):
    _fields_ = [
        ("capacity_steps", C.c_int32), ("n_samples", C.c_int32), ("times", _dp),
        ("q", _dp), ("energy", _dp), ("iterations", _ip), ("converged", _ip),
        ("accepted", _ip), ("final_value", _dp), ("final_grad_norm", _dp),
        ("has_error", C.c_int32), ("error", C.c_char * 256),
    ]


def build():
    """Compile the oracle with its own Makefile (test infrastructure)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.pbo_model_create.argtypes = [C.POINTER(LinkSpecC), C.c_int32, C.POINTER(C.c_void_p), C.c_char_p, C.c_int32]
        L.pbo_model_free.argtypes = [C.c_void_p]
        L.pbo_model_dofs.argtypes = [C.c_void_p]
        L.pbo_model_links.argtypes = [C.c_void_p]
        L.pbo_model_info.argtypes = [C.c_void_p, _dp, _dp, _ip, _dp, _ip]
        L.pbo_model_samples.argtypes = [C.c_void_p, C.c_int32, _dp]
        L.pbo_body_integral.argtypes = [C.POINTER(LinkSpecC), _dp, _dp]
        L.pbo_rotation_vector_matrix.argtypes = [_dp, _dp]
        L.pbo_joint_jet.argtypes = [C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp]
        L.pbo_joint_transform.argtypes = [C.c_int32, _dp, _dp, _dp, _dp]
        L.pbo_forward_pass.argtypes = [C.c_void_p, _dp, _dp]
        L.pbo_correlation.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.pbo_functional.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp]
        L.pbo_legendre_points.argtypes = [C.c_int32, _dp]
        L.pbo_build_scheme.argtypes = [C.c_int32, C.c_double, _dp, _dp, _dp, _dp]
        L.pbo_eval_potentials.argtypes = [C.c_void_p, C.POINTER(ForcesC), _dp, _dp, C.c_double, C.c_int32, C.c_int32, _dp, _dp, _dp, _dp]
        L.pbo_step_eval.argtypes = [C.c_void_p, C.POINTER(ForcesC), C.c_int32, C.c_double, C.c_int32, _dp, _dp, _dp, C.c_int32, C.c_int32, _dp, _dp, _dp]
        L.pbo_step_minimize.argtypes = [C.c_void_p, C.POINTER(ForcesC), C.c_int32, C.c_double, C.c_int32, _dp, _dp, _dp, C.POINTER(OptimizerC), _dp, _ip, _ip, _dp, _dp, _dp]
        L.pbo_spd_solve.argtypes = [_dp, _dp, C.c_int32, _dp]
        L.pbo_simulate.argtypes = [C.c_void_p, C.POINTER(ForcesC), C.POINTER(SimC), C.POINTER(TrajectoryC)]
        L.pbo_batch_simulate.argtypes = [C.c_void_p, C.POINTER(ForcesC), C.POINTER(SimC), C.c_int32, C.c_int32, C.POINTER(TrajectoryC)]
        L.pbo_kinetic_energy.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.pbo_gravity_potential.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.pbo_sincos.argtypes = [C.c_double, _dp, _dp]
        L.pbo_default_optimizer.argtypes = [C.POINTER(OptimizerC)]
        for name in ("pbo_model_create", "pbo_joint_jet", "pbo_joint_transform", "pbo_forward_pass",
                     "pbo_correlation", "pbo_functional", "pbo_legendre_points", "pbo_build_scheme",
                     "pbo_eval_potentials", "pbo_step_eval", "pbo_step_minimize", "pbo_spd_solve",
                     "pbo_simulate", "pbo_batch_simulate", "pbo_kinetic_energy",
                     "pbo_gravity_potential", "pbo_model_dofs", "pbo_model_links", "pbo_model_samples"):
            getattr(L, name).restype = C.c_int32
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _iptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_ip)


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


class OracleError(RuntimeError):
    pass


def link_spec_c(link, keep):
    """Convert a product-side LinkSpec (duck-typed) into the oracle struct."""
    s = LinkSpecC()
    s.parent = -1 if link.parent is None else int(link.parent)
    j = link.joint
    s.joint_kind = int(j.kind)
    s.axis[:] = [float(v) for v in j.axis]
    s.offset[:] = [float(v) for v in np.asarray(j.offset, dtype=np.float64).reshape(4, 4).T.reshape(-1)]
    g = link.geometry
    if hasattr(g, "masses"):
        s.geom_kind = POINTS
        pm = _f64([m.mass for m in g.masses])
        pp = _f64([list(m.position) for m in g.masses] or np.zeros((0, 3)))
        keep += [pm, pp]
        s.n_points = len(g.masses)
        s.point_mass = _ptr(pm)
        s.point_pos = _ptr(pp)
    else:
        s.geom_kind = BOX
        s.box_size[:] = [float(v) for v in g.size]
        s.box_density = float(g.density)
        s.box_center[:] = [float(v) for v in g.center]
    if link.contact_samples:
        smp = _f64([list(p) for p in link.contact_samples])
        keep.append(smp)
        s.n_samples = len(link.contact_samples)
        s.samples = _ptr(smp)
    return s


class Model:
    """Built oracle model (build_model, model.cpp:62-112)."""

    def __init__(self, links):
        keep = []
        arr = (LinkSpecC * max(1, len(links)))()
        for i, l in enumerate(links):
            arr[i] = link_spec_c(l, keep)
        h = C.c_void_p()
        err = C.create_string_buffer(256)
        rc = lib().pbo_model_create(arr, len(links), C.byref(h), err, 256)
        if rc != 0:
            raise OracleError(err.value.decode())
        self.h = h
        self.n_links = lib().pbo_model_links(h)
        self.n_dofs = lib().pbo_model_dofs(h)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().pbo_model_free(self.h)
        except Exception:
            pass

    def info(self):
        N = self.n_links
        S = np.zeros((N, 16))
        mass = np.zeros(N)
        off = np.zeros(N, dtype=np.int32)
        axis = np.zeros((N, 3))
        sc = np.zeros(N, dtype=np.int32)
        lib().pbo_model_info(self.h, _ptr(S), _ptr(mass), _iptr(off), _ptr(axis), _iptr(sc))
        return dict(S=S.reshape(N, 4, 4).transpose(0, 2, 1).copy(), mass=mass, dof_offset=off,
                    axis=axis, sample_count=sc)

    def samples(self, link):
        k = lib().pbo_model_samples(self.h, link, None)
        out = np.zeros((k, 3))
        lib().pbo_model_samples(self.h, link, _ptr(out))
        return out


def forces_c(forces, n, keep):
    f = ForcesC()
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
        f.tau = _ptr(t)
    if forces.actuation is not None:
        a = forces.actuation
        f.has_actuation = 1
        f.act_kind = int(a.kind)
        amp = _f64(a.amplitude)
        ph = _f64(a.phase if a.phase is not None else [])
        keep += [amp, ph]
        f.act_len = len(amp)
        f.act_amplitude = _ptr(amp)
        f.act_frequency_hz = float(a.frequency_hz)
        f.act_phase_len = len(ph)
        f.act_phase = _ptr(ph)
    return f


def optimizer_c(cfg):
    o = OptimizerC()
    lib().pbo_default_optimizer(C.byref(o))
    if cfg is None:
        return o
    o.kind = int(cfg.kind)
    for k in ("max_iters", "lbfgs_memory", "max_line_search"):
        setattr(o, k, int(getattr(cfg, k)))
    for k in ("grad_tol", "grad_rtol", "ftol", "lm_lambda0", "lm_lambda_factor", "lm_lambda_max",
              "armijo_c1", "backtrack_factor"):
        setattr(o, k, float(getattr(cfg, k)))
    return o


def sim_c(sim, n, keep):
    s = SimC()
    s.dt = float(sim.dt)
    s.duration = float(sim.duration)
    s.order = int(sim.order)
    s.objective = int(sim.objective)
    s.opt = optimizer_c(sim.optimizer)
    q0 = _f64(sim.q0)
    qd = _f64(sim.qdot0)
    keep += [q0, qd]
    if len(q0) != n:
        raise OracleError(f"configuration length {len(q0)} does not match model DOF count {n}")
    if len(qd) != n:
        raise OracleError("initial velocity length does not match model DOF count")
    s.q0 = _ptr(q0)
    s.qdot0 = _ptr(qd)
    s.consecutive_fail_limit = int(sim.consecutive_fail_limit)
    s.refined_bootstrap = int(bool(sim.refined_bootstrap))
    s.warm_start = int(bool(sim.warm_start))
    return s


def total_steps(sim):
    import math
    return int(math.ceil(sim.duration / sim.dt - 1e-9))


class OracleTrajectory:
    def __init__(self, n, cap):
        self.cap = cap
        self.times = np.zeros(cap + 1)
        self.q = np.zeros((cap + 1, n))
        self.energy = np.zeros((cap + 1, 2))
        self.iterations = np.zeros(cap, dtype=np.int32)
        self.converged = np.zeros(cap, dtype=np.int32)
        self.accepted = np.zeros(cap, dtype=np.int32)
        self.final_value = np.zeros(cap)
        self.final_grad_norm = np.zeros(cap)
        self.c = TrajectoryC()
        c = self.c
        c.capacity_steps = cap
        c.times = _ptr(self.times)
        c.q = _ptr(self.q)
        c.energy = _ptr(self.energy)
        c.iterations = _iptr(self.iterations)
        c.converged = _iptr(self.converged)
        c.accepted = _iptr(self.accepted)
        c.final_value = _ptr(self.final_value)
        c.final_grad_norm = _ptr(self.final_grad_norm)

    def finalize(self):
        k = self.c.n_samples
        self.n_samples = k
        steps = max(0, k - 1)
        # the solve report of a failing final step is recorded too
        nrep = steps + (1 if self.c.has_error and steps < self.cap and self.iterations[steps] > 0 else 0)
        self.n_reports = nrep
        self.error = self.c.error.decode() if self.c.has_error else None
        return self


def simulate(model, forces, sim):
    keep = []
    n = model.n_dofs
    f = forces_c(forces, n, keep)
    s = sim_c(sim, n, keep)
    tr = OracleTrajectory(n, total_steps(sim))
    lib().pbo_simulate(model.h, C.byref(f), C.byref(s), C.byref(tr.c))
    return tr.finalize()


def batch_simulate(model, forces, sims, workers=1):
    keep = []
    n = model.n_dofs
    f = forces_c(forces, n, keep)
    arr = (SimC * len(sims))()
    trs = []
    tarr = (TrajectoryC * len(sims))()
    for i, sim in enumerate(sims):
        arr[i] = sim_c(sim, n, keep)
        tr = OracleTrajectory(n, total_steps(sim))
        trs.append(tr)
        tarr[i] = tr.c
    lib().pbo_batch_simulate(model.h, C.byref(f), arr, len(sims), int(workers), tarr)
    for i, tr in enumerate(trs):
        tr.c = tarr[i]
        tr.finalize()
    return trs


def step_eval(model, forces, order, dt, objective, hist0, hist1, x, want_grad=True, want_gn=False,
              tau_instants=None):
    keep = []
    n = model.n_dofs
    f = forces_c(forces, n, keep)
    hist = _f64(np.concatenate([np.asarray(hist0, float), np.asarray(hist1, float)]))
    x = _f64(x)
    dim = len(x)
    tau = None if tau_instants is None else _f64(tau_instants)
    value = C.c_double()
    grad = np.zeros(dim)
    gn = np.zeros((dim, dim)) if want_gn else None
    rc = lib().pbo_step_eval(model.h, C.byref(f), order, dt, objective, _ptr(hist), _ptr(tau), _ptr(x),
                             int(want_grad), int(want_gn), C.byref(value), _ptr(grad),
                             _ptr(gn) if gn is not None else None)
    if rc != 0:
        raise OracleError("step_eval failed")
    if gn is not None:
        gn = gn.T.copy()  # column-major -> row-major
    return value.value, grad, gn


def correlation(model, qa, qb, weights=None, want=("value", "grad", "bb", "ab")):
    n = model.n_dofs
    qa = _f64(qa)
    qb = _f64(qb)
    w = None if weights is None else _f64(weights)
    v = C.c_double()
    g = np.zeros(n)
    bb = np.zeros((n, n))
    ab = np.zeros((n, n))
    rc = lib().pbo_correlation(model.h, _ptr(qa), _ptr(qb), _ptr(w), C.byref(v), _ptr(g), _ptr(bb), _ptr(ab))
    if rc != 0:
        raise OracleError("correlation failed")
    return v.value, g, bb.T.copy(), ab.T.copy()


def forward_pass(model, q):
    N = model.n_links
    w = np.zeros((N, 16))
    rc = lib().pbo_forward_pass(model.h, _ptr(_f64(q)), _ptr(w))
    if rc != 0:
        raise OracleError("configuration contains a non-finite entry")
    return w.reshape(N, 4, 4).transpose(0, 2, 1).copy()


def joint_jet(kind, axis, offset, q):
    dof = {HINGE: 1, BALL: 3, FREE: 6}[kind]
    v = np.zeros(16)
    d1 = np.zeros((dof, 16))
    d2 = np.zeros((dof * (dof + 1) // 2, 16))
    off = _f64(np.asarray(offset, float).reshape(4, 4).T.reshape(-1))
    lib().pbo_joint_jet(kind, _ptr(_f64(axis)), _ptr(off), _ptr(_f64(q)), _ptr(v), _ptr(d1), _ptr(d2))
    t = lambda a: a.reshape(-1, 4, 4).transpose(0, 2, 1).copy()
    return t(v)[0], t(d1), t(d2)


def joint_transform(kind, axis, offset, q):
    v = np.zeros(16)
    off = _f64(np.asarray(offset, float).reshape(4, 4).T.reshape(-1))
    lib().pbo_joint_transform(kind, _ptr(_f64(axis)), _ptr(off), _ptr(_f64(q)), _ptr(v))
    return v.reshape(4, 4).T.copy()


def rotation_vector_matrix(theta):
    R = np.zeros(9)
    lib().pbo_rotation_vector_matrix(_ptr(_f64(theta)), _ptr(R))
    return R.reshape(3, 3).T.copy()


def build_scheme(order, dt):
    k = order + 1
    alphas = np.zeros(max(1, order - 1))
    times = np.zeros(k)
    H = np.zeros(k * k)
    H2 = np.zeros(k * k)
    rc = lib().pbo_build_scheme(order, dt, _ptr(alphas), _ptr(times), _ptr(H), _ptr(H2))
    if rc != 0:
        raise OracleError("invalid collocation scheme")
    return dict(alphas=alphas[: order - 1], times=times, H=H.reshape(k, k).T.copy(),
                H2=H2.reshape(k, k).T.copy())


def legendre_points(order):
    out = np.zeros(max(1, order - 1))
    if lib().pbo_legendre_points(order, _ptr(out)) != 0:
        raise OracleError("collocation order must be >= 2")
    return out[: order - 1]


def spd_solve(A, b):
    A = _f64(np.asarray(A, float).T)  # to column-major
    b = _f64(b)
    x = np.zeros(len(b))
    rc = lib().pbo_spd_solve(_ptr(A), _ptr(b), len(b), _ptr(x))
    return None if rc else x


def sincos(x):
    s = C.c_double()
    c = C.c_double()
    lib().pbo_sincos(float(x), C.byref(s), C.byref(c))
    return s.value, c.value


def eval_potentials(model, forces, q_next, q_prev, dt, want_gn=True, want_hess=False):
    keep = []
    n = model.n_dofs
    f = forces_c(forces, n, keep)
    v = C.c_double()
    g = np.zeros(n)
    gn = np.zeros((n, n))
    h = np.zeros((n, n))
    rc = lib().pbo_eval_potentials(model.h, C.byref(f), _ptr(_f64(q_next)), _ptr(_f64(q_prev)), dt,
                                   int(want_gn), int(want_hess), C.byref(v), _ptr(g), _ptr(gn), _ptr(h))
    if rc != 0:
        raise OracleError("eval_potentials failed")
    return v.value, g, gn.T.copy(), h.T.copy()


# ---------------------------------------------------------------------------
# oracle/_ref: the reference's own sources compiled against eigen_lite
# (oracle/ref/Makefile).  Only buildable where /root/reference exists; the
# built .so travels to the GPU box like the other in-tree libraries.
REF_LIB_PATH = os.path.join(_HERE, "_ref", "libpbad_ref.so")
_ref = None


def ref_available():
    return os.path.exists(REF_LIB_PATH)


def ref_lib():
    global _ref
    if _ref is None:
        R = C.CDLL(REF_LIB_PATH)
        vp = C.c_void_p
        R.pbr_last_error.restype = C.c_char_p
        R.pbr_model_create.argtypes = [C.POINTER(LinkSpecC), C.c_int, C.POINTER(vp)]
        R.pbr_model_free.argtypes = [vp]
        R.pbr_model_dofs.argtypes = [vp]
        R.pbr_model_info.argtypes = [vp, _dp, _dp, _ip, _dp, _ip]
        R.pbr_forward_pass.argtypes = [vp, _dp, _dp]
        R.pbr_correlation.argtypes = [vp, _dp, _dp, _dp, _dp, _dp, _dp]
        R.pbr_build_scheme.argtypes = [C.c_int, C.c_double, _dp, _dp]
        R.pbr_correlation_suite.argtypes = [vp, _dp, _dp, _dp, C.c_int, _dp, _dp, _dp, _dp]
        R.pbr_functional.argtypes = [vp, _dp, _dp, _dp, _dp, _dp]
        R.pbr_step_eval.argtypes = [vp, C.POINTER(ForcesC), C.c_int, C.c_double, C.c_int, _dp, _dp, _dp, C.c_int,
                                    C.c_int, _dp, _dp, _dp]
        R.pbr_simulate.argtypes = [vp, C.POINTER(ForcesC), C.POINTER(SimC), C.POINTER(TrajectoryC)]
        R.pbr_batch_simulate.argtypes = [vp, C.POINTER(ForcesC), C.POINTER(SimC), C.c_int, C.c_int,
                                         C.POINTER(TrajectoryC)]
        R.pbr_scene_roundtrip.restype = C.c_char_p
        R.pbr_scene_roundtrip.argtypes = [C.c_char_p]
        R.pbr_bundled_scene.restype = C.c_char_p
        R.pbr_bundled_scene.argtypes = [C.c_char_p]
        R.pbr_scene_simulate_csv.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p]
        R.pbr_simulate_baseline.argtypes = [vp, C.POINTER(ForcesC), C.c_int, C.POINTER(SimC), C.POINTER(TrajectoryC)]
        _ref = R
    return _ref


def ref_scene_roundtrip(text):
    """The reference's parse_scene + serialize_scene; raises OracleError with
    the reference's exception text."""
    out = ref_lib().pbr_scene_roundtrip(text.encode())
    if out is None:
        raise OracleError(ref_lib().pbr_last_error().decode())
    return out.decode()


def ref_bundled_scene(name):
    """serialize_scene of a reference scene builder: chain<N>, single<N>, swimmer, spider."""
    out = ref_lib().pbr_bundled_scene(name.encode())
    if out is None:
        raise OracleError(ref_lib().pbr_last_error().decode())
    return out.decode()


def ref_scene_simulate_csv(text, traj_csv, energy_csv):
    """The reference CLI's simulate path: scene text -> trajectory.csv, energy.csv."""
    if ref_lib().pbr_scene_simulate_csv(text.encode(), traj_csv.encode(), energy_csv.encode()) != 0:
        raise OracleError(ref_lib().pbr_last_error().decode())


class RefModel:
    """KinematicModel built by the reference's own build_model."""

    def __init__(self, links):
        keep = []
        arr = (LinkSpecC * max(1, len(links)))()
        for i, l in enumerate(links):
            arr[i] = link_spec_c(l, keep)
        h = C.c_void_p()
        if ref_lib().pbr_model_create(arr, len(links), C.byref(h)) != 0:
            raise OracleError(ref_lib().pbr_last_error().decode())
        self.h = h
        self.n_links = len(links)
        self.n_dofs = ref_lib().pbr_model_dofs(h)

    def __del__(self):
        try:
            ref_lib().pbr_model_free(self.h)
        except Exception:
            pass

    def info(self):
        N = self.n_links
        S = np.zeros((N, 16))
        mass = np.zeros(N)
        off = np.zeros(N, dtype=np.int32)
        axis = np.zeros((N, 3))
        sc = np.zeros(N, dtype=np.int32)
        ref_lib().pbr_model_info(self.h, _ptr(S), _ptr(mass), _iptr(off), _ptr(axis), _iptr(sc))
        return dict(S=S.reshape(N, 4, 4).transpose(0, 2, 1).copy(), mass=mass, dof_offset=off, axis=axis,
                    sample_count=sc)


def ref_forward_pass(model, q):
    N = model.n_links
    w = np.zeros((N, 16))
    if ref_lib().pbr_forward_pass(model.h, _ptr(_f64(q)), _ptr(w)) != 0:
        raise OracleError(ref_lib().pbr_last_error().decode())
    return w.reshape(N, 4, 4).transpose(0, 2, 1).copy()


def ref_correlation(model, qa, qb):
    n = model.n_dofs
    v = C.c_double()
    g = np.zeros(n)
    bb = np.zeros((n, n))
    ab = np.zeros((n, n))
    if ref_lib().pbr_correlation(model.h, _ptr(_f64(qa)), _ptr(_f64(qb)), C.byref(v), _ptr(g), _ptr(bb),
                                 _ptr(ab)) != 0:
        raise OracleError(ref_lib().pbr_last_error().decode())
    return v.value, g, bb.T.copy(), ab.T.copy()


def ref_correlation_suite(model, qa, qb, weights=None, workers=4):
    """The reference's parallel_correlation_suite (adjoint.cpp:241-336):
    (value, grad_b, hess_bb, hess_ab), Hessians row-major numpy."""
    n = model.n_dofs
    v = C.c_double()
    g = np.zeros(n)
    bb = np.zeros((n, n))
    ab = np.zeros((n, n))
    w = None if weights is None else _f64(weights)
    if ref_lib().pbr_correlation_suite(model.h, _ptr(_f64(qa)), _ptr(_f64(qb)), _ptr(w) if w is not None else None,
                                       int(workers), C.byref(v), _ptr(g), _ptr(bb), _ptr(ab)) != 0:
        raise OracleError(ref_lib().pbr_last_error().decode())
    return v.value, g, bb.T.copy(), ab.T.copy()


def ref_functional(model, q, seeds):
    """The reference's functional_value / _grad / _hess (adjoint.cpp:43-101)
    of seeds [N][4][4] (row-major numpy matrices) at q."""
    n = model.n_dofs
    s = np.ascontiguousarray(np.transpose(np.asarray(seeds, float), (0, 2, 1)).reshape(-1))  # column-major
    v = C.c_double()
    g = np.zeros(n)
    h = np.zeros((n, n))
    if ref_lib().pbr_functional(model.h, _ptr(_f64(q)), _ptr(s), C.byref(v), _ptr(g), _ptr(h)) != 0:
        raise OracleError(ref_lib().pbr_last_error().decode())
    return v.value, g, h.T.copy()


def ref_build_scheme(order, dt):
    k = order + 1
    t = np.zeros(k)
    H2 = np.zeros(k * k)
    if ref_lib().pbr_build_scheme(order, dt, _ptr(t), _ptr(H2)) != 0:
        raise OracleError(ref_lib().pbr_last_error().decode())
    return dict(times=t, H2=H2.reshape(k, k).T.copy())


def ref_step_eval(model, forces, order, dt, objective, hist0, hist1, x, want_grad=True, want_gn=False,
                  tau_instants=None):
    keep = []
    f = forces_c(forces, model.n_dofs, keep)
    hist = _f64(np.concatenate([np.asarray(hist0, float), np.asarray(hist1, float)]))
    x = _f64(x)
    dim = len(x)
    tau = None if tau_instants is None else _f64(tau_instants)
    v = C.c_double()
    g = np.zeros(dim)
    gn = np.zeros((dim, dim)) if want_gn else None
    if ref_lib().pbr_step_eval(model.h, C.byref(f), order, dt, objective, _ptr(hist), _ptr(tau), _ptr(x),
                               int(want_grad), int(want_gn), C.byref(v), _ptr(g),
                               _ptr(gn) if gn is not None else None) != 0:
        raise OracleError(ref_lib().pbr_last_error().decode())
    return v.value, g, (gn.T.copy() if gn is not None else None)


def ref_batch_simulate(model, forces, sims, workers=1):
    keep = []
    n = model.n_dofs
    f = forces_c(forces, n, keep)
    arr = (SimC * len(sims))()
    trs = []
    tarr = (TrajectoryC * len(sims))()
    for i, sim in enumerate(sims):
        arr[i] = sim_c(sim, n, keep)
        tr = OracleTrajectory(n, total_steps(sim))
        trs.append(tr)
        tarr[i] = tr.c
    if ref_lib().pbr_batch_simulate(model.h, C.byref(f), arr, len(sims), int(workers), tarr) != 0:
        raise OracleError(ref_lib().pbr_last_error().decode())
    for i, tr in enumerate(trs):
        tr.c = tarr[i]
        tr.finalize()
    return trs


def ref_simulate_baseline(model, forces, scheme, sim):
    """The reference's simulate_baseline (stepper.cpp:168-202) on a RefModel."""
    keep = []
    n = model.n_dofs
    f = forces_c(forces, n, keep)
    sc = sim_c(sim, n, keep)
    tr = OracleTrajectory(n, total_steps(sim))
    if ref_lib().pbr_simulate_baseline(model.h, C.byref(f), int(scheme), C.byref(sc), C.byref(tr.c)) != 0:
        raise OracleError(ref_lib().pbr_last_error().decode())
    return tr.finalize()
