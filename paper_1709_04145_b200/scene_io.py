"""Scene files and CSV output: the reference's scene JSON layer and CSV writers
on top of the GPU step API.

  parse_scene / load_scene / serialize_scene      scene.cpp:179-378
  scene_model / scene_forces / scene_sim_config   scene.cpp:380-418
  write_trajectory_csv / write_energy_csv         benchmark.cpp:12-36, csv.hpp
  simulate_scene                                  pbad_cli.cpp:25-63 (`simulate`)

Parsing is strict like the reference: unknown fields and malformed values
raise SceneError("scene: <field>: <what>") naming the offending field, with
the reference's texts.  serialize_scene reproduces nlohmann::json's
dump(2) (sorted keys, two-space indent, Grisu2 doubles in its
fixed/exponent layout), so a scene file written by either side is
byte-identical.  The CSV writers print every double with "%.17g" like
CsvWriter, so trajectory.csv / energy.csv from the GPU path diff clean
against the reference CLI's on the same scene (tests/test_scene_io.py).
"""
from __future__ import annotations

import json
import math
import os
from fractions import Fraction
from typing import List, Optional, Sequence

import numpy as np

from . import api
from .scenes import Scene
from .types import (ActuationKind, ActuationSpec, BaselineScheme, BoxGeometry, ContactModel, ForceModel, JointKind, JointSpec,
                    LinkSpec, ModelError, ObjectiveKind, OptimizerKind, PointMass, PointMassGeometry, SimConfig,
                    Trajectory)


class SceneError(RuntimeError):
    """scene.hpp:13-16 (a std::runtime_error)."""


class SceneTypeError(TypeError):
    """A JSON value of the wrong type where the reference calls
    json::get<std::string>() (nlohmann type_error.302, not a SceneError)."""


_BASELINE_KINDS = ("semi_implicit", "forward_euler", "rk2", "rk3", "rk4")


# ---------------------------------------------------------------- helpers ---

def _fail(where: str, what: str):
    raise SceneError(f"scene: {where}: {what}")


def _is_int(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def _is_number(v) -> bool:
    return (isinstance(v, (int, float))) and not isinstance(v, bool)


def _json_type_name(v) -> str:
    if v is None:
        return "null"
    if isinstance(v, bool):
        return "boolean"
    if isinstance(v, (int, float)):
        return "number"
    if isinstance(v, str):
        return "string"
    if isinstance(v, list):
        return "array"
    return "object"


def _string(v) -> str:
    if not isinstance(v, str):
        raise SceneTypeError(f"[json.exception.type_error.302] type must be string, but is {_json_type_name(v)}")
    return v


def _require(j: dict, where: str, key: str):
    if key not in j:
        _fail(where, f"missing field '{key}'")
    return j[key]


def _check_keys(j, where: str, allowed: Sequence[str]):
    if not isinstance(j, dict):
        _fail(where, "expected an object")
    for key in sorted(j):  # nlohmann objects iterate in key order
        if key not in allowed:
            _fail(where, f"unknown field '{key}'")


def _number(v, where: str) -> float:
    if not _is_number(v):
        _fail(where, "expected a number")
    return float(v)


def _vec3(v, where: str):
    if not isinstance(v, list) or len(v) != 3:
        _fail(where, "expected an array of 3 numbers")
    return (_number(v[0], where), _number(v[1], where), _number(v[2], where))


def _vecx(v, where: str) -> np.ndarray:
    if not isinstance(v, list):
        _fail(where, "expected an array of numbers")
    return np.array([_number(x, where) for x in v], dtype=np.float64)


def _fma(a: float, b: float, c: float) -> float:
    """Correctly rounded a*b+c (std::fma) via exact rationals."""
    if not (math.isfinite(a) and math.isfinite(b) and math.isfinite(c)):
        return a * b + c
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _norm3(v) -> float:
    # Vec3::norm(): first product, then fma in index order
    acc = v[0] * v[0]
    acc = _fma(v[1], v[1], acc)
    acc = _fma(v[2], v[2], acc)
    return math.sqrt(acc)


# ------------------------------------------------------------------- parse ---

def _parse_offset(j, where: str) -> np.ndarray:
    _check_keys(j, where, ("translation", "rotation_vector"))
    m = np.eye(4)
    if "translation" in j:
        m[:3, 3] = _vec3(j["translation"], where + ".translation")
    if "rotation_vector" in j:
        m[:3, :3] = api.rotation_vector_matrix(_vec3(j["rotation_vector"], where + ".rotation_vector"))
    return m


def _parse_link(j, where: str):
    _check_keys(j, where, ("parent", "joint", "geometry", "contact_samples"))
    link = LinkSpec()
    jp = _require(j, where, "parent")
    if jp is None:
        link.parent = None
    elif _is_int(jp):
        link.parent = int(jp)
    else:
        _fail(where + ".parent", "expected an integer or null")

    jj = _require(j, where, "joint")
    _check_keys(jj, where + ".joint", ("kind", "axis", "offset"))
    kind = _string(_require(jj, where + ".joint", "kind"))
    joint = JointSpec()
    if kind == "hinge":
        joint.kind = JointKind.hinge
        joint.axis = _vec3(_require(jj, where + ".joint", "axis"), where + ".joint.axis")
    elif kind == "ball":
        joint.kind = JointKind.ball
    elif kind == "free":
        joint.kind = JointKind.free_joint
    else:
        _fail(where + ".joint.kind", "expected hinge, ball or free")
    if "offset" in jj:
        joint.offset = _parse_offset(jj["offset"], where + ".joint.offset")
    link.joint = joint

    jg = _require(j, where, "geometry")
    _check_keys(jg, where + ".geometry", ("box", "point_masses"))
    if ("box" in jg) == ("point_masses" in jg):
        _fail(where + ".geometry", "expected exactly one of box or point_masses")
    if "box" in jg:
        jb = jg["box"]
        w = where + ".geometry.box"
        _check_keys(jb, w, ("size", "density", "center"))
        box = BoxGeometry()
        box.size = _vec3(_require(jb, w, "size"), w + ".size")
        box.density = _number(_require(jb, w, "density"), w + ".density")
        if "center" in jb:
            box.center = _vec3(jb["center"], w + ".center")
        link.geometry = box
    else:
        ja = jg["point_masses"]
        if not isinstance(ja, list):
            _fail(where + ".geometry.point_masses", "expected an array")
        pm = PointMassGeometry([])
        for i, e in enumerate(ja):
            pw = f"{where}.geometry.point_masses[{i}]"
            _check_keys(e, pw, ("mass", "position"))
            pm.masses.append(PointMass(_number(_require(e, pw, "mass"), pw + ".mass"),
                                       _vec3(_require(e, pw, "position"), pw + ".position")))
        link.geometry = pm

    has_samples = "contact_samples" in j
    if has_samples:
        js = j["contact_samples"]
        if not isinstance(js, list):
            _fail(where + ".contact_samples", "expected an array")
        link.contact_samples = [_vec3(v, f"{where}.contact_samples[{i}]") for i, v in enumerate(js)]
    return link, has_samples


def _reject_constant(tok):
    raise ValueError(f"invalid literal '{tok}'")


def parse_scene(json_text: str) -> Scene:
    """scene.cpp:179-283."""
    try:
        j = json.loads(json_text, parse_constant=_reject_constant)
    except (ValueError, RecursionError) as e:
        raise SceneError(f"scene: JSON parse error: {e}") from None
    _check_keys(j, "top level", ("links", "gravity", "drag_D", "contact", "actuation", "integrator", "dt",
                                 "duration", "initial"))
    s = Scene()
    s.link_has_samples = []
    jl = _require(j, "top level", "links")
    if not isinstance(jl, list) or not jl:
        _fail("links", "expected a non-empty array")
    for i, e in enumerate(jl):
        link, has = _parse_link(e, f"links[{i}]")
        s.links.append(link)
        s.link_has_samples.append(has)

    s.gravity = _vec3(_require(j, "top level", "gravity"), "gravity")
    if "drag_D" in j:
        s.drag_d = _number(j["drag_D"], "drag_D")
        if s.drag_d < 0.0:
            _fail("drag_D", "must be non-negative")
    if "contact" in j:
        jc = j["contact"]
        _check_keys(jc, "contact", ("normal", "offset", "D1", "D2"))
        normal = _vec3(_require(jc, "contact", "normal"), "contact.normal")
        if abs(_norm3(normal) - 1.0) > 1e-9:
            _fail("contact.normal", "must have unit norm")
        cm = ContactModel(normal, _number(_require(jc, "contact", "offset"), "contact.offset"),
                          _number(_require(jc, "contact", "D1"), "contact.D1"),
                          _number(_require(jc, "contact", "D2"), "contact.D2"))
        if cm.d1 < 0.0 or cm.d2 < 0.0:
            _fail("contact", "penalties must be non-negative")
        s.contact = cm
    if "actuation" in j:
        ja = j["actuation"]
        _check_keys(ja, "actuation", ("kind", "amplitude", "frequency_hz", "phase"))
        kind = _string(_require(ja, "actuation", "kind"))
        if kind == "constant":
            act = ActuationSpec(ActuationKind.constant)
        elif kind == "sinusoidal":
            act = ActuationSpec(ActuationKind.sinusoidal)
        else:
            _fail("actuation.kind", "expected constant or sinusoidal")
        act.amplitude = _vecx(_require(ja, "actuation", "amplitude"), "actuation.amplitude")
        act.phase = np.zeros(0)
        if kind == "sinusoidal":
            act.frequency_hz = _number(_require(ja, "actuation", "frequency_hz"), "actuation.frequency_hz")
            if "phase" in ja:
                act.phase = _vecx(ja["phase"], "actuation.phase")
            if act.phase.size and act.phase.size != act.amplitude.size:
                _fail("actuation.phase", "length must match amplitude")
        s.actuation = act

    ji = _require(j, "top level", "integrator")
    _check_keys(ji, "integrator", ("kind", "order", "objective", "optimizer"))
    s.integrator_kind = _string(_require(ji, "integrator", "kind"))
    if s.integrator_kind != "pbad" and s.integrator_kind not in _BASELINE_KINDS:
        _fail("integrator.kind", f"unknown integrator '{s.integrator_kind}'")
    s.order = 2
    if "order" in ji:
        if not _is_int(ji["order"]):
            _fail("integrator.order", "expected an integer")
        s.order = int(ji["order"])
        if s.order < 2 or s.order > 6:
            _fail("integrator.order", "order must be in [2, 6]")
    if "objective" in ji:
        obj = _string(ji["objective"])
        if obj not in ("energy", "residual"):
            _fail("integrator.objective", "expected energy or residual")
    else:
        obj = "energy" if s.order == 2 else "residual"
    if obj == "energy" and s.order != 2:
        _fail("integrator.objective", "the energy objective requires order 2")
    s.objective = ObjectiveKind.energy_form if obj == "energy" else ObjectiveKind.residual_form
    s.optimizer = OptimizerKind.lm
    if "optimizer" in ji:
        opt = _string(ji["optimizer"])
        if opt not in ("lm", "lbfgs"):
            _fail("integrator.optimizer", "expected lm or lbfgs")
        s.optimizer = OptimizerKind.lm if opt == "lm" else OptimizerKind.lbfgs

    s.dt = _number(_require(j, "top level", "dt"), "dt")
    if s.dt <= 0.0:
        _fail("dt", "must be positive")
    s.duration = _number(_require(j, "top level", "duration"), "duration")
    if s.duration <= 0.0:
        _fail("duration", "must be positive")
    j0 = _require(j, "top level", "initial")
    _check_keys(j0, "initial", ("q", "qdot"))
    s.q0 = _vecx(_require(j0, "initial", "q"), "initial.q")
    s.qdot0 = _vecx(_require(j0, "initial", "qdot"), "initial.qdot")
    if s.q0.size != s.qdot0.size:
        _fail("initial", "q and qdot must have the same length")
    return s


def load_scene(path: str) -> Scene:
    """scene.cpp:285-292."""
    try:
        with open(path, "r") as f:
            text = f.read()
    except OSError:
        raise SceneError(f"scene: cannot open '{path}'") from None
    return parse_scene(text)


# --------------------------------------------------------------- serialize ---

# nlohmann::json prints doubles with Grisu2 (Loitsch 2010, nlohmann's
# detail::dtoa_impl), which is not always the shortest round-trip form (about
# 1 value in 200 gets a 17th digit where repr() stops at 16), so the digit
# generation is restated here exactly, in integer arithmetic.
_M64 = (1 << 64) - 1


def _diy_mul(xf: int, xe: int, yf: int, ye: int):
    u_lo, u_hi = xf & 0xFFFFFFFF, xf >> 32
    v_lo, v_hi = yf & 0xFFFFFFFF, yf >> 32
    p0, p1, p2, p3 = u_lo * v_lo, u_lo * v_hi, u_hi * v_lo, u_hi * v_hi
    q = (p0 >> 32) + (p1 & 0xFFFFFFFF) + (p2 & 0xFFFFFFFF) + (1 << 31)
    h = p3 + (p2 >> 32) + (p1 >> 32) + (q >> 32)
    return h & _M64, xe + ye + 64


def _diy_normalize(f: int, e: int):
    while not (f >> 63):
        f <<= 1
        e -= 1
    return f, e


def _cached_power(k: int):
    """Normalised 64-bit significand of 10^k, rounded to nearest."""
    x = Fraction(10) ** k
    e = x.numerator.bit_length() - x.denominator.bit_length() - 64
    while x / Fraction(2) ** e >= (1 << 64):
        e += 1
    while x / Fraction(2) ** e < (1 << 63):
        e -= 1
    return round(x / Fraction(2) ** e), e


_CACHED = {}


def _grisu2(value: float):
    """(digits, decimal_exponent) of nlohmann's dtoa_impl::grisu2 for value > 0."""
    bits = int.from_bytes(np.float64(value).tobytes(), "little")
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    vf, ve = (F, 1 - 1075) if E == 0 else (F + (1 << 52), E - 1075)
    closer = F == 0 and E > 1
    mpf, mpe = _diy_normalize(2 * vf + 1, ve - 1)
    mmf, mme = (4 * vf - 1, ve - 2) if closer else (2 * vf - 1, ve - 1)
    mmf, mme = mmf << (mme - mpe), mpe
    vf, ve = _diy_normalize(vf, ve)
    # cached power c = 10^-k with alpha <= e_c + e + 64 <= gamma
    f = -60 - mpe - 1
    kk = int((f * 78913) / (1 << 18)) if f * 78913 >= 0 else -((-f * 78913) // (1 << 18))
    kk += 1 if f > 0 else 0
    index = (300 + kk + 7) // 8
    ck = -300 + 8 * index
    if ck not in _CACHED:
        _CACHED[ck] = _cached_power(ck)
    cf, ce = _CACHED[ck]
    wf, we = _diy_mul(vf, ve, cf, ce)
    wmf, wme = _diy_mul(mmf, mme, cf, ce)
    wpf, wpe = _diy_mul(mpf, mpe, cf, ce)
    Mm, Mp = wmf + 1, wpf - 1
    dec_exp = -ck
    # digit generation (grisu2_digit_gen)
    delta = Mp - Mm
    dist = Mp - wf
    shift = -wpe
    one = 1 << shift
    p1 = Mp >> shift
    p2 = Mp & (one - 1)
    digits = []
    n = len(str(p1))
    pow10 = 10 ** (n - 1)
    while n > 0:
        d, r = divmod(p1, pow10)
        digits.append(d)
        p1 = r
        n -= 1
        rest = (p1 << shift) + p2
        if rest <= delta:
            dec_exp += n
            _grisu2_round(digits, dist, delta, rest, pow10 << shift)
            return digits, dec_exp
        pow10 //= 10
    m = 0
    while True:
        p2 = (p2 * 10) & _M64
        digits.append(p2 >> shift)
        p2 &= one - 1
        m += 1
        delta = (delta * 10) & _M64
        dist = (dist * 10) & _M64
        if p2 <= delta:
            break
    dec_exp -= m
    _grisu2_round(digits, dist, delta, p2, one)
    return digits, dec_exp


def _grisu2_round(digits, dist, delta, rest, ten_k):
    while rest < dist and delta - rest >= ten_k and (rest + ten_k < dist or dist - rest > rest + ten_k - dist):
        digits[-1] -= 1
        rest += ten_k


def _fmt_double(x: float) -> str:
    """nlohmann::json's number_float output: Grisu2 digits laid out by
    dtoa_impl::format_buffer (fixed for decimal exponents in (-4, 15], else
    d.ddde+XX)."""
    if not math.isfinite(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    sign = "-" if x < 0 else ""
    dg, dec_exp = _grisu2(abs(x))
    digits = "".join(str(d) for d in dg)
    k = len(digits)
    n = k + dec_exp  # value = 0.d1d2..dk * 10^n
    if k <= n <= 15:
        return sign + digits + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + digits[:n] + "." + digits[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + digits
    e = n - 1
    mant = digits if k == 1 else digits[0] + "." + digits[1:]
    es = "-" if e < 0 else "+"
    ae = abs(e)
    return sign + mant + "e" + es + (f"{ae:02d}" if ae < 100 else str(ae))


def _dump(v, ind: int) -> str:
    if isinstance(v, dict):
        if not v:
            return "{}"
        pad = " " * (ind + 2)
        items = [f"{pad}{json.dumps(k)}: {_dump(v[k], ind + 2)}" for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + " " * ind + "}"
    if isinstance(v, (list, tuple)):
        if len(v) == 0:
            return "[]"
        pad = " " * (ind + 2)
        return "[\n" + ",\n".join(pad + _dump(x, ind + 2) for x in v) + "\n" + " " * ind + "]"
    if v is None:
        return "null"
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return _fmt_double(float(v))
    if isinstance(v, str):
        return json.dumps(v)
    raise TypeError(f"cannot serialise {type(v)}")


def _floats(v):
    return [float(x) for x in v]


def serialize_scene(scene: Scene) -> str:
    """scene.cpp:294-378: lossless, byte-identical to the reference's output."""
    links = []
    has = getattr(scene, "link_has_samples", None) or []
    for i, link in enumerate(scene.links):
        kind = JointKind(link.joint.kind)
        jj = {"kind": {JointKind.hinge: "hinge", JointKind.ball: "ball", JointKind.free_joint: "free"}[kind]}
        if kind == JointKind.hinge:
            jj["axis"] = _floats(link.joint.axis)
        off = np.asarray(link.joint.offset, dtype=np.float64)
        jj["offset"] = {"translation": _floats(off[:3, 3]),
                        "rotation_vector": _floats(api.rotation_vector_from_matrix(off[:3, :3]))}
        g = link.geometry
        if isinstance(g, BoxGeometry):
            jg = {"box": {"size": _floats(g.size), "density": float(g.density), "center": _floats(g.center)}}
        else:
            jg = {"point_masses": [{"mass": float(p.mass), "position": _floats(p.position)} for p in g.masses]}
        jl = {"parent": None if link.parent is None else int(link.parent), "joint": jj, "geometry": jg}
        if i < len(has) and has[i]:
            jl["contact_samples"] = [_floats(c) for c in link.contact_samples]
        links.append(jl)
    j = {"links": links, "gravity": _floats(scene.gravity)}
    if scene.drag_d > 0.0:
        j["drag_D"] = float(scene.drag_d)
    if scene.contact is not None:
        c = scene.contact
        j["contact"] = {"normal": _floats(c.plane_normal), "offset": float(c.plane_offset), "D1": float(c.d1),
                        "D2": float(c.d2)}
    if scene.actuation is not None:
        a = scene.actuation
        ja = {"kind": "constant" if a.kind == ActuationKind.constant else "sinusoidal",
              "amplitude": _floats(a.amplitude)}
        if a.kind == ActuationKind.sinusoidal:
            ja["frequency_hz"] = float(a.frequency_hz)
            if a.phase is not None and len(a.phase):
                ja["phase"] = _floats(a.phase)
        j["actuation"] = ja
    j["integrator"] = {"kind": getattr(scene, "integrator_kind", "pbad"), "order": int(scene.order),
                       "objective": "energy" if scene.objective == ObjectiveKind.energy_form else "residual",
                       "optimizer": "lm" if scene.optimizer == OptimizerKind.lm else "lbfgs"}
    j["dt"] = float(scene.dt)
    j["duration"] = float(scene.duration)
    j["initial"] = {"q": _floats(scene.q0), "qdot": _floats(scene.qdot0)}
    return _dump(j, 0) + "\n"


# ------------------------------------------------------- model / config ---

def scene_model(scene: Scene) -> api.KinematicModel:
    """scene.cpp:380-392."""
    model = api.build_model(scene.links)
    if len(scene.q0) != model.total_dofs:
        raise SceneError(f"scene: initial.q length {len(scene.q0)} does not match model DOF count "
                         f"{model.total_dofs}")
    if scene.actuation is not None and len(scene.actuation.amplitude) != model.total_dofs:
        raise SceneError("scene: actuation.amplitude length does not match DOF count")
    return model


def scene_forces(scene: Scene) -> ForceModel:
    """scene.cpp:394-401."""
    return scene.forces()


def scene_sim_config(scene: Scene) -> SimConfig:
    """scene.cpp:403-416."""
    return scene.sim_config()


def scene_is_pbad(scene: Scene) -> bool:
    return getattr(scene, "integrator_kind", "pbad") == "pbad"


def scene_baseline_scheme(scene: Scene) -> BaselineScheme:
    """scene.cpp:420-428."""
    k = getattr(scene, "integrator_kind", "pbad")
    try:
        return BaselineScheme[k]
    except KeyError:
        raise SceneError(f"scene: integrator '{k}' is not a baseline scheme") from None


# ---------------------------------------------------------------- CSV out ---

def _csv_row(values) -> str:
    return ",".join("%.17g" % float(v) for v in values) + "\n"


def write_trajectory_csv(path: str, trajectory: Trajectory) -> None:
    """benchmark.cpp:12-24: time,q_0..q_{n-1}; "%.17g"; LF."""
    n = len(trajectory.samples[0][1]) if trajectory.samples else 0
    try:
        f = open(path, "w", newline="\n")
    except OSError:
        raise RuntimeError(f"cannot open output file '{path}'") from None
    with f:
        f.write(",".join(["time"] + [f"q_{i}" for i in range(n)]) + "\n")
        for t, q in trajectory.samples:
            f.write(_csv_row([t, *[q[i] for i in range(n)]]))


def write_energy_csv(path: str, trajectory: Trajectory) -> None:
    """benchmark.cpp:26-36: time,kinetic,potential,total,iterations."""
    try:
        f = open(path, "w", newline="\n")
    except OSError:
        raise RuntimeError(f"cannot open output file '{path}'") from None
    with f:
        f.write("time,kinetic,potential,total,iterations\n")
        reps = trajectory.solve_reports
        for i, e in enumerate(trajectory.energy_log):
            iters = float(reps[i - 1].iterations) if (i > 0 and i - 1 < len(reps)) else 0.0
            f.write(_csv_row([e.time, e.kinetic, e.potential, e.total(), iters]))


def simulate_scene(scene_path: str, out_dir: str, dt: float = 0.0, duration: float = 0.0, order: int = 0,
                   optimizer: str = "", objective: str = "", device: int = 0) -> Trajectory:
    """The reference CLI's `simulate` subcommand (pbad_cli.cpp:25-63) on the GPU
    step API: load the scene, apply the overrides, simulate, write
    <out_dir>/trajectory.csv and energy.csv; baseline integrator kinds run
    simulate_baseline on the GPU (pbad_cli.cpp:49-53)."""
    scene = load_scene(scene_path)
    if dt > 0.0:
        scene.dt = dt
    if duration > 0.0:
        scene.duration = duration
    if order > 0:
        scene.order = order
        if not objective and order != 2:
            scene.objective = ObjectiveKind.residual_form
    if optimizer:
        scene.optimizer = OptimizerKind.lm if optimizer == "lm" else OptimizerKind.lbfgs
    if objective:
        scene.objective = ObjectiveKind.energy_form if objective == "energy" else ObjectiveKind.residual_form
    if scene.objective == ObjectiveKind.energy_form and scene.order != 2:
        raise SceneError("scene: the energy objective requires order 2")
    model = scene_model(scene)
    os.makedirs(out_dir, exist_ok=True)
    if scene_is_pbad(scene):
        traj = api.simulate(model, scene_forces(scene), scene_sim_config(scene), device=device)
    else:
        traj = api.simulate_baseline(model, scene_forces(scene), scene_baseline_scheme(scene),
                                     scene_sim_config(scene), device=device)
    write_trajectory_csv(os.path.join(out_dir, "trajectory.csv"), traj)
    write_energy_csv(os.path.join(out_dir, "energy.csv"), traj)
    return traj
