"""Scene JSON + CSV compatibility: the scene layer
(scene_io.py) against the reference's own scene.cpp / benchmark.cpp compiled
into oracle/_ref — byte-identical serialisation, identical error texts,
byte-identical trajectory.csv / energy.csv (CPU oracle trajectory here, the
GPU path in the gpu-marked test)."""
import json
import math

import numpy as np
import pytest

import oracle
from paper_1709_04145_b200 import api, scene_io, scenes
from paper_1709_04145_b200.types import EnergySample, SolveReport, Trajectory

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")

BUNDLED = {
    "chain10": lambda: scenes.make_chain_scene(10),
    "chain100": lambda: scenes.make_chain_scene(100),
    "single7": lambda: scenes.make_single_hinge_chain_scene(7),
    "swimmer": scenes.make_swimmer_scene,
    "spider": lambda: scenes.make_spider_scene(api.rotation_vector_matrix),
}


@pytest.mark.parametrize("name", sorted(BUNDLED))
def test_bundled_scenes_serialise_byte_identical(name):
    ref = oracle.ref_bundled_scene(name)
    assert scene_io.serialize_scene(BUNDLED[name]()) == ref
    assert scene_io.serialize_scene(scene_io.parse_scene(ref)) == ref


def _base_doc():
    return json.loads(oracle.ref_bundled_scene("spider"))


def _assert_roundtrip(doc_or_text):
    text = doc_or_text if isinstance(doc_or_text, str) else json.dumps(doc_or_text)
    ref = oracle.ref_scene_roundtrip(text)
    assert scene_io.serialize_scene(scene_io.parse_scene(text)) == ref


def test_roundtrip_number_formatting():
    """Grisu2 digits (not always the shortest) in nlohmann's fixed / exponent layout."""
    rng = np.random.default_rng(0)
    special = [1e-05, 1e-4, 2e-4, 1.5e-4, 0.1, 1 / 3, 1e15, 1e16, 123456789012345.0, 1234567890123456.0,
               -0.0, 0.0, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 1e100, -1e-100, 1e22, 1e21,
               9007199254740993.0, 0.5, 100.0, -2.5e-7]
    vals = special + list(rng.uniform(-1, 1, 300)) + list(10.0 ** rng.uniform(-30, 30, 300))
    doc = _base_doc()
    doc["initial"]["q"] = [float(v) for v in vals]
    doc["initial"]["qdot"] = [float(v) for v in reversed(vals)]
    _assert_roundtrip(doc)


def test_roundtrip_rotations_and_optional_fields():
    """Rotated joint offsets through every branch of the log map (generic,
    near zero, near pi), explicit contact samples, actuation, drag, residual
    integrator settings, point-mass geometry."""
    doc = _base_doc()
    rots = [[0.3, -0.2, 0.9], [1e-12, 0.0, 0.0], [0.0, 0.0, math.pi - 1e-8], [math.pi - 1e-7, 0.0, 0.0],
            [0.0, -(math.pi - 3e-7), 0.0], [0.5, 0.5, 0.5], [2.0, -1.0, 0.5], [0.0, 0.0, 0.0], [1e-10, 2e-10, 0.0]]
    for i, link in enumerate(doc["links"]):
        link["joint"]["offset"]["rotation_vector"] = rots[i % len(rots)]
    doc["links"][1]["contact_samples"] = [[0.25, 0.0, 0.0], [0.125, 0.01, -0.02]]
    doc["links"][2]["contact_samples"] = []
    doc["links"][3]["geometry"] = {"point_masses": [{"mass": 0.5, "position": [0.1, 0.0, 0.0]},
                                                    {"mass": 1.25, "position": [0.0, 0.2, -0.1]}]}
    doc["drag_D"] = 0.75
    n = len(doc["initial"]["q"])
    doc["actuation"] = {"kind": "sinusoidal", "amplitude": [0.1 * i for i in range(n)], "frequency_hz": 0.5,
                        "phase": [0.01 * i for i in range(n)]}
    doc["integrator"] = {"kind": "pbad", "order": 4, "optimizer": "lbfgs"}
    _assert_roundtrip(doc)
    doc["actuation"] = {"kind": "constant", "amplitude": [1.0] * n, "frequency_hz": 3.0}
    doc["integrator"] = {"kind": "rk4"}
    _assert_roundtrip(doc)
    doc["actuation"] = {"kind": "sinusoidal", "amplitude": [1.0] * n, "frequency_hz": 3.0}
    _assert_roundtrip(doc)


def test_roundtrip_humanoid_and_random_trees():
    from _parity_util import random_tree
    sc = scenes.make_humanoid_scene()
    _assert_roundtrip(scene_io.serialize_scene(sc))
    rng = np.random.default_rng(3)
    for k in range(4):
        sc = scenes.Scene(links=random_tree(rng, 5 + k), gravity=(0.1, -0.2, -9.81))
        n = api.build_model(sc.links).total_dofs
        sc.q0 = rng.uniform(-1, 1, n)
        sc.qdot0 = rng.uniform(-1, 1, n)
        sc.dt, sc.duration = 0.01, 0.5
        text = scene_io.serialize_scene(sc)
        _assert_roundtrip(text)
        # parse(serialize(x)) rebuilds the same model bit for bit
        m0, m1 = api.build_model(sc.links), scene_io.scene_model(scene_io.parse_scene(text))
        np.testing.assert_array_equal(m0.body_S, m1.body_S)


def _mutations():
    def m(f):
        def g():
            d = _base_doc()
            f(d)
            return d
        return g
    L = lambda d: d["links"]  # noqa: E731
    return [
        ("top_list", lambda: [1, 2]),
        ("unknown_top", m(lambda d: d.__setitem__("foo", 1))),
        ("missing_links", m(lambda d: d.pop("links"))),
        ("empty_links", m(lambda d: d.__setitem__("links", []))),
        ("link_not_object", m(lambda d: L(d).__setitem__(0, 3))),
        ("missing_parent", m(lambda d: L(d)[1].pop("parent"))),
        ("parent_string", m(lambda d: L(d)[1].__setitem__("parent", "a"))),
        ("parent_float", m(lambda d: L(d)[1].__setitem__("parent", 1.5))),
        ("joint_kind", m(lambda d: L(d)[2]["joint"].__setitem__("kind", "slider"))),
        ("joint_kind_type", m(lambda d: L(d)[2]["joint"].__setitem__("kind", 5))),
        ("hinge_no_axis", m(lambda d: L(d)[2]["joint"].pop("axis"))),
        ("axis_len", m(lambda d: L(d)[2]["joint"].__setitem__("axis", [0.0, 1.0]))),
        ("axis_type", m(lambda d: L(d)[2]["joint"].__setitem__("axis", ["a", 0, 0]))),
        ("axis_bool", m(lambda d: L(d)[2]["joint"].__setitem__("axis", [True, 0, 0]))),
        ("offset_key", m(lambda d: L(d)[2]["joint"]["offset"].__setitem__("scale", 1))),
        ("joint_key", m(lambda d: L(d)[2]["joint"].__setitem__("limit", 1))),
        ("geom_both", m(lambda d: L(d)[1]["geometry"].__setitem__("point_masses", []))),
        ("geom_none", m(lambda d: L(d)[1].__setitem__("geometry", {}))),
        ("box_no_density", m(lambda d: L(d)[1]["geometry"]["box"].pop("density"))),
        ("box_key", m(lambda d: L(d)[1]["geometry"]["box"].__setitem__("color", "red"))),
        ("pm_not_array", m(lambda d: L(d)[1].__setitem__("geometry", {"point_masses": 1}))),
        ("pm_key", m(lambda d: L(d)[1].__setitem__("geometry", {"point_masses": [{"mass": 1, "pos": [0, 0, 0]}]}))),
        ("pm_no_position", m(lambda d: L(d)[1].__setitem__("geometry", {"point_masses": [{"mass": 1}]}))),
        ("samples_not_array", m(lambda d: L(d)[1].__setitem__("contact_samples", 2))),
        ("sample_bad", m(lambda d: L(d)[1].__setitem__("contact_samples", [[0, 0, 0], [1, 2]]))),
        ("missing_gravity", m(lambda d: d.pop("gravity"))),
        ("drag_negative", m(lambda d: d.__setitem__("drag_D", -1.0))),
        ("drag_type", m(lambda d: d.__setitem__("drag_D", "x"))),
        ("contact_normal", m(lambda d: d["contact"].__setitem__("normal", [0.0, 0.0, 1.1]))),
        ("contact_penalty", m(lambda d: d["contact"].__setitem__("D1", -1.0))),
        ("contact_key", m(lambda d: d["contact"].__setitem__("mu", 1.0))),
        ("contact_missing", m(lambda d: d["contact"].pop("D2"))),
        ("act_kind", m(lambda d: d.__setitem__("actuation", {"kind": "pd", "amplitude": []}))),
        ("act_amp", m(lambda d: d.__setitem__("actuation", {"kind": "constant", "amplitude": 1}))),
        ("act_freq", m(lambda d: d.__setitem__("actuation", {"kind": "sinusoidal", "amplitude": [1.0]}))),
        ("act_phase", m(lambda d: d.__setitem__("actuation", {"kind": "sinusoidal", "amplitude": [1.0, 2.0],
                                                              "frequency_hz": 1.0, "phase": [0.0]}))),
        ("integ_kind", m(lambda d: d["integrator"].__setitem__("kind", "verlet"))),
        ("integ_order", m(lambda d: d["integrator"].__setitem__("order", 7))),
        ("integ_order_float", m(lambda d: d["integrator"].__setitem__("order", 2.0))),
        ("integ_objective", m(lambda d: d["integrator"].__setitem__("objective", "x"))),
        ("integ_energy_order", m(lambda d: d["integrator"].update(order=3, objective="energy"))),
        ("integ_optimizer", m(lambda d: d["integrator"].__setitem__("optimizer", "newton"))),
        ("integ_key", m(lambda d: d["integrator"].__setitem__("tol", 1e-3))),
        ("dt_zero", m(lambda d: d.__setitem__("dt", 0))),
        ("duration_negative", m(lambda d: d.__setitem__("duration", -1.0))),
        ("initial_no_qdot", m(lambda d: d["initial"].pop("qdot"))),
        ("initial_len", m(lambda d: d["initial"]["qdot"].pop())),
        ("initial_key", m(lambda d: d["initial"].__setitem__("t", 0))),
    ]


@pytest.mark.parametrize("name,make", _mutations(), ids=[m[0] for m in _mutations()])
def test_parse_errors_match_reference(name, make):
    text = json.dumps(make())
    with pytest.raises(oracle.OracleError) as ref:
        oracle.ref_scene_roundtrip(text)
    with pytest.raises((scene_io.SceneError, scene_io.SceneTypeError)) as mine:
        scene_io.parse_scene(text)
    assert str(mine.value) == str(ref.value)


@pytest.mark.parametrize("text", ["{", "not json", '{"links": NaN}', ""])
def test_json_syntax_errors(text):
    with pytest.raises(oracle.OracleError) as ref:
        oracle.ref_scene_roundtrip(text)
    with pytest.raises(scene_io.SceneError) as mine:
        scene_io.parse_scene(text)
    prefix = "scene: JSON parse error: "
    assert str(ref.value).startswith(prefix) and str(mine.value).startswith(prefix)


def test_scene_model_dof_mismatch():
    doc = _base_doc()
    doc["initial"]["q"].append(0.0)
    doc["initial"]["qdot"].append(0.0)
    sc = scene_io.parse_scene(json.dumps(doc))
    with pytest.raises(scene_io.SceneError, match="initial.q length 23 does not match model DOF count 22"):
        scene_io.scene_model(sc)


def _short_scene(name, duration, **integ):
    doc = json.loads(oracle.ref_bundled_scene(name))
    doc["duration"] = duration
    doc["integrator"].update(integ)
    return doc


def _oracle_trajectory(sc):
    """Trajectory of the C oracle for a parsed scene (CPU), in the API's types."""
    m = oracle.Model(sc.links)
    sim = scene_io.scene_sim_config(sc)
    r = oracle.simulate(m, scene_io.scene_forces(sc), sim)
    tr = Trajectory()
    for s in range(r.n_samples):
        tr.samples.append((s * sim.dt, r.q[s].copy()))
        tr.energy_log.append(EnergySample(s * sim.dt, float(r.energy[s, 0]), float(r.energy[s, 1])))
    for s in range(r.n_reports):
        tr.solve_reports.append(SolveReport(int(r.iterations[s])))
    return tr


CSV_CASES = [("single5", 0.1, {}), ("spider", 0.05, {}), ("chain3", 0.05, {"optimizer": "lbfgs"}),
             ("single4", 0.04, {"order": 3, "objective": "residual"})]


@pytest.mark.parametrize("name,duration,integ", CSV_CASES)
def test_csv_writers_byte_identical(tmp_path, name, duration, integ):
    doc = _short_scene(name, duration, **integ)
    text = json.dumps(doc)
    oracle.ref_scene_simulate_csv(text, str(tmp_path / "ref_traj.csv"), str(tmp_path / "ref_energy.csv"))
    tr = _oracle_trajectory(scene_io.parse_scene(text))
    scene_io.write_trajectory_csv(str(tmp_path / "traj.csv"), tr)
    scene_io.write_energy_csv(str(tmp_path / "energy.csv"), tr)
    assert (tmp_path / "traj.csv").read_bytes() == (tmp_path / "ref_traj.csv").read_bytes()
    assert (tmp_path / "energy.csv").read_bytes() == (tmp_path / "ref_energy.csv").read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name,duration,integ", CSV_CASES + [("swimmer", 0.5, {}),
                                                              ("single5", 0.05, {"kind": "rk4"}),
                                                              ("spider", 0.03, {"kind": "semi_implicit"})])
def test_simulate_scene_on_gpu_matches_reference_csv(tmp_path, name, duration, integ):
    """The reference CLI's `simulate` on a scene file vs the GPU step API
    driven from the same file: trajectory.csv and energy.csv byte-identical."""
    doc = _short_scene(name, duration, **integ)
    text = json.dumps(doc)
    path = tmp_path / "scene.json"
    path.write_text(text)
    oracle.ref_scene_simulate_csv(text, str(tmp_path / "ref_traj.csv"), str(tmp_path / "ref_energy.csv"))
    scene_io.simulate_scene(str(path), str(tmp_path / "out"))
    assert (tmp_path / "out" / "trajectory.csv").read_bytes() == (tmp_path / "ref_traj.csv").read_bytes()
    assert (tmp_path / "out" / "energy.csv").read_bytes() == (tmp_path / "ref_energy.csv").read_bytes()
