// pbad_gpu_dropin.cpp -- pbad::gpu::batch_simulate / simulate over the C ABI
// (include/pbad_gpu.h).  See pbad_gpu_dropin.hpp.
//
// Reference behaviour mirrored here (stepper.cpp):
//  * batch_simulate (204-270): worker count < 1 -> ModelError; every
//    trajectory independent; an exception of init_pbad_run / begin_step
//    becomes Trajectory::error (validate_configuration's and the
//    qdot0 / dt checks' texts, "objective is non-finite at the initial
//    point", "configuration contains a non-finite entry"); the fail limit
//    sets "optimizer failed N consecutive steps around t=..." and keeps the
//    samples and solve reports recorded so far.
//  * simulate (151-166): the same run, exceptions thrown instead.
#include "pbad_gpu_dropin.hpp"

#include <algorithm>
#include <cmath>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <variant>
#include <vector>

#include "pbad_gpu.h"

namespace pbad::gpu {
namespace {

std::mutex g_mu;
std::vector<int> g_devices;
bool g_iter_values = false;

[[noreturn]] void raise(int32_t rc) {
  const std::string msg = pbad_gpu_last_error();
  if (rc == PBAD_E_MODEL) throw ModelError(msg);
  if (rc == PBAD_E_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(std::string(pbad_gpu_error_string(rc)) + ": " + msg);
}

void check(int32_t rc) {
  if (rc != PBAD_OK) raise(rc);
}

struct ModelHandle {
  pbad_gpu_model* h = nullptr;
  ~ModelHandle() { pbad_gpu_model_destroy(h); }
};

struct CtxHandle {
  pbad_gpu_ctx* h = nullptr;
  CtxHandle() = default;
  CtxHandle(const CtxHandle&) = delete;
  CtxHandle(CtxHandle&& o) noexcept : h(o.h) { o.h = nullptr; }
  ~CtxHandle() { pbad_gpu_destroy(h); }
};

// KinematicModel (model.hpp:71-88, already through build_model) -> link specs
std::unique_ptr<ModelHandle> make_model(const KinematicModel& model, std::vector<std::vector<double>>& keep) {
  const int N = model.link_count();
  std::vector<pbad_link_spec> specs(N);
  for (int i = 0; i < N; ++i) {
    const LinkSpec& L = model.links[i];
    pbad_link_spec& s = specs[i];
    s.parent = L.parent ? *L.parent : -1;
    s.joint_kind = L.joint.kind == JointKind::hinge ? PBAD_HINGE : L.joint.kind == JointKind::ball ? PBAD_BALL : PBAD_FREE;
    for (int k = 0; k < 3; ++k) s.axis[k] = L.joint.axis[k];
    for (int c = 0; c < 4; ++c)
      for (int r = 0; r < 4; ++r) s.offset[r + 4 * c] = L.joint.offset(r, c);
    if (const auto* box = std::get_if<BoxGeometry>(&L.geometry)) {
      s.geom_kind = PBAD_GEOM_BOX;
      for (int k = 0; k < 3; ++k) {
        s.box_size[k] = box->size[k];
        s.box_center[k] = box->center[k];
      }
      s.box_density = box->density;
    } else {
      const auto& pm = std::get<PointMassGeometry>(L.geometry);
      s.geom_kind = PBAD_GEOM_POINTS;
      s.n_points = (int32_t)pm.masses.size();
      keep.emplace_back();
      auto& m = keep.back();
      keep.emplace_back();
      auto& p = keep.back();
      for (const auto& x : pm.masses) {
        m.push_back(x.mass);
        for (int k = 0; k < 3; ++k) p.push_back(x.position[k]);
      }
      s.point_mass = m.data();
      s.point_pos = p.data();
    }
    keep.emplace_back();
    auto& cs = keep.back();
    for (const auto& v : L.contact_samples)
      for (int k = 0; k < 3; ++k) cs.push_back(v[k]);
    s.n_samples = (int32_t)L.contact_samples.size();
    s.samples = cs.data();
  }
  auto h = std::make_unique<ModelHandle>();
  check(pbad_gpu_model_create(specs.data(), N, &h->h));
  return h;
}

pbad_forces make_forces(const ForceModel& f, std::vector<std::vector<double>>& keep) {
  pbad_forces d{};
  for (int k = 0; k < 3; ++k) d.gravity[k] = f.gravity[k];
  d.drag_d = f.drag_d;
  if (f.contact) {
    d.has_contact = 1;
    for (int k = 0; k < 3; ++k) d.plane_normal[k] = f.contact->plane_normal[k];
    d.plane_offset = f.contact->plane_offset;
    d.contact_d1 = f.contact->d1;
    d.contact_d2 = f.contact->d2;
  }
  auto vec = [&](const VecX& v) -> const double* {
    keep.emplace_back(v.data(), v.data() + v.size());
    return keep.back().data();
  };
  d.tau_len = (int32_t)f.tau.size();
  d.tau = d.tau_len ? vec(f.tau) : nullptr;
  if (f.actuation) {
    d.has_actuation = 1;
    d.act_kind = f.actuation->kind == ActuationSpec::Kind::constant ? 0 : 1;
    d.act_len = (int32_t)f.actuation->amplitude.size();
    d.act_amplitude = d.act_len ? vec(f.actuation->amplitude) : nullptr;
    d.act_frequency_hz = f.actuation->frequency_hz;
    d.act_phase_len = (int32_t)f.actuation->phase.size();
    d.act_phase = d.act_phase_len ? vec(f.actuation->phase) : nullptr;
  }
  return d;
}

pbad_sim_desc make_sim(const SimConfig& s) {
  pbad_sim_desc d{};
  pbad_gpu_default_sim(&d);
  d.dt = s.dt;
  d.duration = s.duration;
  d.order = s.order;
  d.objective = s.objective == ObjectiveKind::energy_form ? PBAD_ENERGY_FORM : PBAD_RESIDUAL_FORM;
  const OptimizerConfig& o = s.optimizer;
  d.opt.kind = o.kind == OptimizerKind::lbfgs ? PBAD_LBFGS : PBAD_LM;
  d.opt.max_iters = o.max_iters;
  d.opt.grad_tol = o.grad_tol;
  d.opt.grad_rtol = o.grad_rtol;
  d.opt.ftol = o.ftol;
  d.opt.lbfgs_memory = o.lbfgs_memory;
  d.opt.lm_lambda0 = o.lm_lambda0;
  d.opt.lm_lambda_factor = o.lm_lambda_factor;
  d.opt.lm_lambda_max = o.lm_lambda_max;
  d.opt.armijo_c1 = o.armijo_c1;
  d.opt.backtrack_factor = o.backtrack_factor;
  d.opt.max_line_search = o.max_line_search;
  d.consecutive_fail_limit = s.consecutive_fail_limit;
  d.refined_bootstrap = s.refined_bootstrap ? 1 : 0;
  d.warm_start = s.warm_start ? 1 : 0;
  return d;
}

// everything in SimConfig except q0 / qdot0 (one context per schedule)
bool same_schedule(const SimConfig& a, const SimConfig& b) {
  const OptimizerConfig &x = a.optimizer, &y = b.optimizer;
  return a.dt == b.dt && a.duration == b.duration && a.order == b.order && a.objective == b.objective &&
         a.consecutive_fail_limit == b.consecutive_fail_limit && a.refined_bootstrap == b.refined_bootstrap &&
         a.warm_start == b.warm_start && x.kind == y.kind && x.max_iters == y.max_iters &&
         x.grad_tol == y.grad_tol && x.grad_rtol == y.grad_rtol && x.ftol == y.ftol &&
         x.lbfgs_memory == y.lbfgs_memory && x.lm_lambda0 == y.lm_lambda0 &&
         x.lm_lambda_factor == y.lm_lambda_factor && x.lm_lambda_max == y.lm_lambda_max &&
         x.armijo_c1 == y.armijo_c1 && x.backtrack_factor == y.backtrack_factor &&
         x.max_line_search == y.max_line_search;
}

// init_pbad_run's validation (stepper.cpp:62-70): validate_configuration,
// the qdot0 length, dt / duration; throws the reference's exception types
void validate_run(const pbad_gpu_model* m, int n, const SimConfig& s) {
  check(pbad_gpu_validate_configuration(m, s.q0.data(), (int32_t)s.q0.size()));
  if (s.qdot0.size() != n) throw ModelError("initial velocity length does not match model DOF count");
  if (s.dt <= 0.0 || s.duration <= 0.0) throw ModelError("dt and duration must be positive");
}

std::vector<int> active_devices() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_devices.empty()) return g_devices;
  const int n = pbad_gpu_device_count();
  if (n < 1) throw std::runtime_error("no CUDA device available (the PBAD GPU path has no CPU fallback)");
  std::vector<int> d(n);
  for (int i = 0; i < n; ++i) d[i] = i;
  return d;
}

// Steps one schedule group on the GPUs and writes its trajectories.
void run_group(const pbad_gpu_model* model, const pbad_forces& forces, const SimConfig& rep,
               const std::vector<const SimConfig*>& sims, const std::vector<Trajectory*>& outs) {
  const int n = pbad_gpu_model_dofs(model);
  const long B = (long)sims.size();
  std::vector<int> devs = active_devices();
  if ((long)devs.size() > B) devs.resize(B);
  const int k = (int)devs.size();
  const pbad_sim_desc sd = make_sim(rep);
  std::vector<CtxHandle> ctxs(k);
  std::vector<pbad_gpu_ctx*> raw(k);
  const long shard = (B + k - 1) / k;
  for (int i = 0; i < k; ++i) {
    check(pbad_gpu_create(model, &forces, &sd, devs[i], (int32_t)shard, &ctxs[i].h));
    raw[i] = ctxs[i].h;
  }
  const long S = pbad_gpu_total_steps(raw[0]);
  const int mi = std::max(0, rep.optimizer.max_iters);
  std::vector<double> q0((size_t)B * n), qd0((size_t)B * n);
  for (long b = 0; b < B; ++b)
    for (int j = 0; j < n; ++j) {
      q0[b * n + j] = sims[b]->q0[j];
      qd0[b * n + j] = sims[b]->qdot0[j];
    }
  std::vector<double> q((size_t)B * (S + 1) * n), en((size_t)B * (S + 1) * 2), fv((size_t)B * S), gn((size_t)B * S);
  std::vector<int32_t> it((size_t)B * S), cv((size_t)B * S), ns(B), st(B), fs(B), nr(B);
  std::vector<double> iv;
  std::vector<int32_t> ivn;
  pbad_rollout_out o{};
  o.q = q.data();
  o.energy = en.data();
  o.iterations = it.data();
  o.converged = cv.data();
  o.final_value = fv.data();
  o.final_grad_norm = gn.data();
  o.n_samples = ns.data();
  o.status = st.data();
  o.fail_streak = fs.data();
  o.n_reports = nr.data();
  if (g_iter_values && mi > 0) {
    iv.resize((size_t)B * S * mi);
    o.iteration_values = iv.data();
  }
  check(pbad_gpu_rollout_sharded(raw.data(), k, (int32_t)B, q0.data(), qd0.data(), &o));
  const double dt = rep.dt;
  for (long b = 0; b < B; ++b) {
    Trajectory& tr = *outs[b];
    const int K = ns[b];
    for (int s = 0; s < K; ++s) {
      VecX x(n);
      for (int j = 0; j < n; ++j) x[j] = q[((size_t)b * (S + 1) + s) * n + j];
      const double t = s * dt;
      tr.samples.push_back({t, std::move(x)});
      tr.energy_log.push_back({t, en[((size_t)b * (S + 1) + s) * 2], en[((size_t)b * (S + 1) + s) * 2 + 1]});
    }
    for (int s = 0; s < nr[b]; ++s) {
      SolveReport r;
      const size_t ix = (size_t)b * S + s;
      r.iterations = it[ix];
      r.final_value = fv[ix];
      r.final_grad_norm = gn[ix];
      r.converged = cv[ix] != 0;
      if (!iv.empty()) r.per_iteration_values.assign(iv.begin() + ix * mi, iv.begin() + ix * mi + it[ix]);
      tr.solve_reports.push_back(std::move(r));
    }
    switch (st[b]) {
      case PBAD_TRAJ_FAIL_LIMIT:
        tr.error = "optimizer failed " + std::to_string(fs[b]) + " consecutive steps around t=" +
                   std::to_string(std::max(0, K - 1) * dt);
        break;
      case PBAD_TRAJ_NONFINITE_INIT: tr.error = "objective is non-finite at the initial point"; break;
      case PBAD_TRAJ_NONFINITE_CFG: tr.error = "configuration contains a non-finite entry"; break;
      case PBAD_TRAJ_BOOTSTRAP_SINGULAR: tr.error = "singular generalized mass matrix"; break;
      default: break;
    }
  }
}

// Sample 0 and its energy-log entry (init_pbad_run, stepper.cpp:71-77) for
// runs whose first begin_step throws (the reference has already recorded
// them): KE / PE through the GPU baseline path's kinetic_energy /
// gravity_potential (baseline.cpp:208-229), one step of a throw-away schedule.
void initial_samples(const pbad_gpu_model* model, const pbad_forces& forces, const SimConfig& rep,
                     const std::vector<const SimConfig*>& sims, const std::vector<Trajectory*>& outs) {
  const int n = pbad_gpu_model_dofs(model);
  const long B = (long)sims.size();
  pbad_sim_desc sd{};
  pbad_gpu_default_sim(&sd);
  sd.dt = rep.dt;
  sd.duration = rep.dt;
  CtxHandle c;
  check(pbad_gpu_create(model, &forces, &sd, active_devices()[0], (int32_t)B, &c.h));
  std::vector<double> q0((size_t)B * n), qd0((size_t)B * n), q((size_t)B * 2 * n), en((size_t)B * 2 * 2);
  std::vector<int32_t> ns(B), st(B);
  for (long b = 0; b < B; ++b)
    for (int j = 0; j < n; ++j) {
      q0[b * n + j] = sims[b]->q0[j];
      qd0[b * n + j] = sims[b]->qdot0[j];
    }
  check(pbad_gpu_simulate_baseline(c.h, PBAD_BASELINE_FORWARD_EULER, (int32_t)B, q0.data(), qd0.data(), q.data(),
                                   en.data(), ns.data(), st.data()));
  for (long b = 0; b < B; ++b) {
    VecX x(n);
    for (int j = 0; j < n; ++j) x[j] = q[(size_t)b * 2 * n + j];
    outs[b]->samples.push_back({0.0, std::move(x)});
    outs[b]->energy_log.push_back({0.0, en[(size_t)b * 4], en[(size_t)b * 4 + 1]});
  }
}

}  // namespace

void set_devices(const std::vector<int>& devices) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_devices = devices;
}

std::vector<int> devices() { return active_devices(); }

void set_record_iteration_values(bool on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_iter_values = on;
}

std::vector<Trajectory> batch_simulate(const KinematicModel& model, const ForceModel& forces,
                                       const std::vector<SimConfig>& sims, int workers) {
  if (workers < 1) throw ModelError("worker count must be >= 1");
  std::vector<std::vector<double>> keep;
  const auto m = make_model(model, keep);
  const pbad_forces f = make_forces(forces, keep);
  const int n = pbad_gpu_model_dofs(m->h);
  std::vector<Trajectory> out(sims.size());
  // schedule groups, in first-appearance order; invalid runs fail alone
  std::vector<std::vector<size_t>> groups;
  for (size_t i = 0; i < sims.size(); ++i) {
    try {
      validate_run(m->h, n, sims[i]);
    } catch (const std::exception& e) {
      out[i].error = e.what();
      continue;
    }
    auto g = std::find_if(groups.begin(), groups.end(), [&](const std::vector<size_t>& gr) {
      return same_schedule(sims[gr[0]], sims[i]);
    });
    if (g == groups.end()) groups.push_back({i});
    else g->push_back(i);
  }
  for (const auto& g : groups) {
    std::vector<const SimConfig*> ss;
    std::vector<Trajectory*> oo;
    for (size_t i : g) {
      ss.push_back(&sims[i]);
      oo.push_back(&out[i]);
    }
    try {
      run_group(m->h, f, sims[g[0]], ss, oo);
    } catch (const std::invalid_argument& e) {  // ModelError included
      // a schedule the reference rejects per run, every run of the group
      // carries the error: build_scheme's order check throws in
      // init_pbad_run (no samples yet), StepObjective's energy-form order
      // check in the first begin_step (sample 0 already recorded)
      const std::string msg = e.what();
      if (msg == "the energy objective is only defined for order 2") initial_samples(m->h, f, sims[g[0]], ss, oo);
      for (Trajectory* t : oo) t->error = msg;
    }
  }
  return out;
}

Trajectory simulate(const KinematicModel& model, const ForceModel& forces, const SimConfig& sim) {
  std::vector<std::vector<double>> keep;
  const auto m = make_model(model, keep);
  const pbad_forces f = make_forces(forces, keep);
  validate_run(m->h, pbad_gpu_model_dofs(m->h), sim);
  Trajectory tr;
  run_group(m->h, f, sim, {&sim}, {&tr});
  if (tr.error) {
    if (tr.error->rfind("optimizer failed", 0) == 0 || *tr.error == "singular generalized mass matrix")
      throw std::runtime_error(*tr.error);
    if (*tr.error == "objective is non-finite at the initial point") throw std::invalid_argument(*tr.error);
    throw ModelError(*tr.error);
  }
  return tr;
}

}  // namespace pbad::gpu
