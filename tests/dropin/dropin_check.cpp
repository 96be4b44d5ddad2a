// dropin_check.cpp -- TEST INFRASTRUCTURE: runs the reference's own
// pbad::batch_simulate / pbad::simulate (the /root/reference/proj sources
// compiled unmodified, oracle/ref/Makefile) and the GPU drop-in
// pbad::gpu::batch_simulate / simulate (paper_1709_04145_b200/dropin) on the
// same inputs and compares every Trajectory field bit for bit: samples
// (time, q), energy log (time, KE, PE), solve reports (iterations, final
// value, final gradient norm, converged, per_iteration_values) and the
// error text.  Exit code 0 = every case equal.  Driven by
// tests/test_gpu_dropin.py on the GPU box (built here, where the reference
// sources exist).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "pbad/scene.hpp"
#include "pbad/stepper.hpp"
#include "pbad_gpu_dropin.hpp"

using namespace pbad;

namespace {

int g_fail = 0;

bool same_d(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0 || (std::isnan(a) && std::isnan(b)); }

bool same_vec(const VecX& a, const VecX& b) {
  if (a.size() != b.size()) return false;
  for (int i = 0; i < a.size(); ++i)
    if (!same_d(a[i], b[i])) return false;
  return true;
}

std::string cmp(const Trajectory& r, const Trajectory& g, bool itv = true) {
  if (r.samples.size() != g.samples.size())
    return "samples " + std::to_string(r.samples.size()) + " vs " + std::to_string(g.samples.size());
  for (size_t k = 0; k < r.samples.size(); ++k) {
    if (!same_d(r.samples[k].first, g.samples[k].first)) return "sample time " + std::to_string(k);
    if (!same_vec(r.samples[k].second, g.samples[k].second)) return "sample q " + std::to_string(k);
  }
  if (r.energy_log.size() != g.energy_log.size()) return "energy_log size";
  for (size_t k = 0; k < r.energy_log.size(); ++k) {
    const auto &a = r.energy_log[k], &b = g.energy_log[k];
    if (!same_d(a.time, b.time) || !same_d(a.kinetic, b.kinetic) || !same_d(a.potential, b.potential))
      return "energy " + std::to_string(k);
  }
  if (r.solve_reports.size() != g.solve_reports.size())
    return "solve_reports " + std::to_string(r.solve_reports.size()) + " vs " + std::to_string(g.solve_reports.size());
  for (size_t k = 0; k < r.solve_reports.size(); ++k) {
    const auto &a = r.solve_reports[k], &b = g.solve_reports[k];
    if (a.iterations != b.iterations)
      return "iterations step " + std::to_string(k) + ": " + std::to_string(a.iterations) + " vs " +
             std::to_string(b.iterations);
    if (!same_d(a.final_value, b.final_value)) return "final_value " + std::to_string(k);
    if (!same_d(a.final_grad_norm, b.final_grad_norm)) return "final_grad_norm " + std::to_string(k);
    if (a.converged != b.converged) return "converged " + std::to_string(k);
    if (itv) {  // the reference always records them; the GPU on request
      if (a.per_iteration_values.size() != b.per_iteration_values.size())
        return "per_iteration_values size " + std::to_string(k) + ": " +
               std::to_string(a.per_iteration_values.size()) + " vs " + std::to_string(b.per_iteration_values.size());
      for (size_t j = 0; j < a.per_iteration_values.size(); ++j)
        if (!same_d(a.per_iteration_values[j], b.per_iteration_values[j]))
          return "per_iteration_values " + std::to_string(k) + "[" + std::to_string(j) + "]";
    }
  }
  if (r.error != g.error)
    return "error '" + r.error.value_or("<none>") + "' vs '" + g.error.value_or("<none>") + "'";
  return "";
}

void check_batch(const char* name, const KinematicModel& model, const ForceModel& forces,
                 const std::vector<SimConfig>& sims, bool itv) {
  gpu::set_record_iteration_values(itv);
  const auto ref = batch_simulate(model, forces, sims, 8);
  const auto got = gpu::batch_simulate(model, forces, sims, 8);
  int bad = 0;
  size_t samples = 0, reports = 0, errors = 0;
  for (size_t t = 0; t < sims.size(); ++t) {
    std::string w = cmp(ref[t], got[t], itv);
    if (itv) {  // the reference always records the values: the GPU must too
      for (const auto& r : got[t].solve_reports)
        if ((int)r.per_iteration_values.size() != r.iterations) w = "per_iteration_values not recorded";
    }
    samples += ref[t].samples.size();
    reports += ref[t].solve_reports.size();
    errors += ref[t].error.has_value();
    if (!w.empty()) {
      std::printf("MISMATCH %s traj %zu: %s\n", name, t, w.c_str());
      ++bad;
    }
  }
  std::printf("%s %s: %zu trajectories, %zu samples, %zu solve reports, %zu errors%s\n", bad ? "FAIL" : "ok  ", name,
              sims.size(), samples, reports, errors, itv ? ", per_iteration_values compared" : "");
  g_fail += bad;
}

SimConfig sim_of(const Scene& sc, double dt, double duration, OptimizerKind kind, const VecX& q0) {
  SimConfig s = scene_sim_config(sc);
  s.dt = dt;
  s.duration = duration;
  s.optimizer.kind = kind;
  s.q0 = q0;
  s.qdot0 = VecX::Zero(q0.size());
  return s;
}

VecX uniform(std::mt19937& rng, int n, double lo, double hi) {
  std::uniform_real_distribution<double> u(lo, hi);
  VecX v(n);
  for (int i = 0; i < n; ++i) v[i] = u(rng);
  return v;
}

}  // namespace

int main() {
  std::mt19937 rng(7);
  {
    // heterogeneous schedules in one call: L-BFGS / LM / residual form /
    // cold start / memory 0 / tiny fail limit; invalid runs fail alone
    const Scene sc = make_single_hinge_chain_scene(12);
    const KinematicModel model = scene_model(sc);
    const ForceModel forces = scene_forces(sc);
    const int n = model.total_dofs;
    std::vector<SimConfig> sims;
    for (int b = 0; b < 3; ++b) sims.push_back(sim_of(sc, 0.01, 0.05, OptimizerKind::lbfgs, uniform(rng, n, -0.3, 0.3)));
    for (int b = 0; b < 2; ++b) sims.push_back(sim_of(sc, 0.02, 0.06, OptimizerKind::lm, uniform(rng, n, -0.3, 0.3)));
    for (int b = 0; b < 2; ++b) {
      SimConfig s = sim_of(sc, 0.02, 0.06, OptimizerKind::lm, uniform(rng, n, -0.3, 0.3));
      s.order = 3;
      s.objective = ObjectiveKind::residual_form;
      sims.push_back(s);
    }
    {
      SimConfig s = sim_of(sc, 0.02, 0.06, OptimizerKind::lbfgs, uniform(rng, n, -0.3, 0.3));
      s.warm_start = false;
      sims.push_back(s);
    }
    for (int mem : {0, -2}) {
      SimConfig s = sim_of(sc, 0.01, 0.04, OptimizerKind::lbfgs, uniform(rng, n, -0.3, 0.3));
      s.optimizer.lbfgs_memory = mem;
      sims.push_back(s);
    }
    {
      SimConfig s = sim_of(sc, 0.05, 0.5, OptimizerKind::lbfgs, uniform(rng, n, -0.3, 0.3));
      s.optimizer.max_iters = 4;
      s.consecutive_fail_limit = 2;  // "optimizer failed 3 consecutive steps around t=..."
      sims.push_back(s);
    }
    {
      SimConfig s = sim_of(sc, 0.01, 0.03, OptimizerKind::lbfgs, uniform(rng, n, -0.3, 0.3));
      s.order = 3;  // energy form with order 3: the first begin_step throws
      sims.push_back(s);
    }
    {
      SimConfig s = sim_of(sc, 0.01, 0.03, OptimizerKind::lm, uniform(rng, n, -0.3, 0.3));
      s.order = 1;  // build_scheme throws in init_pbad_run
      sims.push_back(s);
    }
    sims.push_back(sim_of(sc, 0.01, 0.03, OptimizerKind::lbfgs, uniform(rng, n - 1, -0.3, 0.3)));  // q0 length
    {
      SimConfig s = sim_of(sc, 0.01, 0.03, OptimizerKind::lbfgs, uniform(rng, n, -0.3, 0.3));
      s.q0[3] = std::nan("");
      sims.push_back(s);
    }
    {
      SimConfig s = sim_of(sc, 0.01, 0.03, OptimizerKind::lbfgs, uniform(rng, n, -0.3, 0.3));
      s.qdot0 = VecX::Zero(n + 1);
      sims.push_back(s);
    }
    sims.push_back(sim_of(sc, -0.01, 0.03, OptimizerKind::lbfgs, uniform(rng, n, -0.3, 0.3)));
    check_batch("hinge-chain-12 mixed schedules", model, forces, sims, false);
    check_batch("hinge-chain-12 mixed schedules (per_iteration_values)", model, forces, sims, true);
  }
  {
    const Scene sc = make_chain_scene(10);
    const KinematicModel model = scene_model(sc);
    std::vector<SimConfig> sims;
    for (int b = 0; b < 5; ++b)
      sims.push_back(sim_of(sc, 0.1, 0.3, OptimizerKind::lbfgs, uniform(rng, model.total_dofs, -0.3, 0.3)));
    check_batch("chain-scene-10 dt 0.1 L-BFGS", model, scene_forces(sc), sims, true);
  }
  {
    const Scene sc = make_spider_scene();  // contact, ball joints
    const KinematicModel model = scene_model(sc);
    std::vector<SimConfig> sims;
    for (int b = 0; b < 3; ++b) {
      SimConfig s = scene_sim_config(sc);
      s.duration = 5 * s.dt;
      VecX q = s.q0;
      for (int i = 6; i < q.size(); ++i) q[i] += uniform(rng, 1, -0.05, 0.05)[0];
      s.q0 = q;
      sims.push_back(s);
    }
    check_batch("spider (contact)", model, scene_forces(sc), sims, true);
  }
  {
    const Scene sc = make_swimmer_scene();  // drag + actuation
    const KinematicModel model = scene_model(sc);
    std::vector<SimConfig> sims;
    for (int b = 0; b < 2; ++b) {
      SimConfig s = scene_sim_config(sc);
      s.duration = 4 * s.dt;
      sims.push_back(s);
    }
    check_batch("swimmer (drag, actuation)", model, scene_forces(sc), sims, false);
  }
  {
    // refined_bootstrap: the RK4 Newton-Euler history (stepper.cpp:46-59)
    const Scene sc = make_single_hinge_chain_scene(8);
    const KinematicModel model = scene_model(sc);
    std::vector<SimConfig> sims;
    for (int b = 0; b < 3; ++b) {
      SimConfig s = sim_of(sc, 0.02, 0.08, b == 2 ? OptimizerKind::lm : OptimizerKind::lbfgs,
                           uniform(rng, model.total_dofs, -0.3, 0.3));
      s.qdot0 = uniform(rng, model.total_dofs, -1.0, 1.0);
      s.refined_bootstrap = true;
      if (b == 1) {
        s.order = 4;
        s.objective = ObjectiveKind::residual_form;
        s.optimizer.kind = OptimizerKind::lm;
      }
      sims.push_back(s);
    }
    check_batch("hinge-chain-8 refined_bootstrap", model, scene_forces(sc), sims, false);
  }
  {
    // error paths of the calls themselves
    gpu::set_record_iteration_values(true);
    const Scene sc = make_single_hinge_chain_scene(5);
    const KinematicModel model = scene_model(sc);
    const ForceModel forces = scene_forces(sc);
    std::vector<SimConfig> sims{sim_of(sc, 0.01, 0.02, OptimizerKind::lbfgs, VecX::Zero(5))};
    std::string a, b;
    try { batch_simulate(model, forces, sims, 0); } catch (const ModelError& e) { a = e.what(); }
    try { gpu::batch_simulate(model, forces, sims, 0); } catch (const ModelError& e) { b = e.what(); }
    const bool ok1 = !a.empty() && a == b;
    SimConfig s = sim_of(sc, 0.05, 1.0, OptimizerKind::lbfgs, uniform(rng, 5, -0.3, 0.3));
    s.optimizer.max_iters = 2;
    s.consecutive_fail_limit = 1;
    a.clear();
    b.clear();
    try { simulate(model, forces, s); } catch (const std::runtime_error& e) { a = e.what(); }
    try { gpu::simulate(model, forces, s); } catch (const std::runtime_error& e) { b = e.what(); }
    const bool ok2 = !a.empty() && a == b;
    s = sim_of(sc, 0.01, 0.05, OptimizerKind::lm, uniform(rng, 5, -0.3, 0.3));
    const std::string w = cmp(simulate(model, forces, s), gpu::simulate(model, forces, s));
    const bool ok3 = w.empty();
    std::printf("%s exceptions: workers<1 %s, simulate fail limit '%s' %s, simulate result %s\n",
                ok1 && ok2 && ok3 ? "ok  " : "FAIL", ok1 ? "equal" : "DIFFERENT", a.c_str(), ok2 ? "equal" : "DIFFERENT",
                ok3 ? "equal" : w.c_str());
    if (!(ok1 && ok2 && ok3)) ++g_fail;
  }
  std::printf(g_fail ? "DROPIN MISMATCHES: %d\n" : "DROPIN ALL EQUAL\n", g_fail);
  return g_fail ? 1 : 0;
}
