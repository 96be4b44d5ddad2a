/*
 * pbad_gpu.h -- C ABI of the B200-native PBAD hot path.
 *
 * Drop-in for the reference's step API (/root/reference/proj):
 *   pbad_gpu_model_create   replaces build_model            model.hpp:94, model.cpp:62-112
 *   pbad_gpu_create         binds ForceModel + SimConfig    objective.hpp:50-59, stepper.hpp:29-44
 *   pbad_gpu_rollout        replaces batch_simulate/simulate stepper.hpp:49-64, stepper.cpp:151-270
 *   pbad_gpu_eval           replaces StepObjective::evaluate/value objective.hpp:106-132
 *   pbad_gpu_minimize       replaces minimize()             optim.hpp:58-60, optim.cpp:244-250
 *   pbad_gpu_simulate_baseline replaces simulate_baseline     stepper.hpp:54-55, stepper.cpp:168-202
 *   pbad_gpu_correlation    replaces correlation_and_grad / hessian_bb / hessian_ab
 *                                                           adjoint.hpp:80-82, adjoint.cpp:178-192
 *   pbad_gpu_begin/advance/ device-resident stepping for callers that keep
 *   pbad_gpu_sync_outputs   state in HBM (the bench's `value` leg)
 *   pbad_gpu_body_integral  replaces body_integral          model.hpp:100, model.cpp:35-60
 *   pbad_gpu_rotation_vector_matrix                          kinematics.hpp:39
 *   pbad_gpu_rotation_vector_from_matrix                     scene.cpp:66-86 (scene serialisation)
 *   pbad_gpu_build_scheme   replaces build_scheme           collocation.hpp:39
 *
 * Plain pointers and sizes only.  Matrices are column-major (Eigen's
 * default), all arithmetic FP64.  Every call returns 0 on success or a
 * negative pbad_gpu_status; pbad_gpu_last_error() holds the message (the
 * text of the exception the reference would have thrown).  Per-trajectory
 * failures in a rollout are NOT call errors: they are reported in
 * status[]/fail_step[] exactly like Trajectory::error (stepper.cpp:225-256).
 * A ctx is bound to one CUDA device and is not thread-safe.
 * No CPU fallback: without a usable sm_100 device pbad_gpu_create fails.
 */
#ifndef PBAD_GPU_H
#define PBAD_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBAD_GPU_ABI_VERSION 1

typedef enum {
  PBAD_OK = 0,
  PBAD_E_MODEL = -1,       /* ModelError (invalid_argument) */
  PBAD_E_ARGUMENT = -2,    /* std::invalid_argument (scheme, solver init) */
  PBAD_E_CUDA = -3,        /* CUDA runtime failure / no device */
  PBAD_E_UNSUPPORTED = -4, /* outside the GPU path's scope */
  PBAD_E_RUNTIME = -5      /* std::runtime_error (simulate fail limit) */
} pbad_gpu_status;

enum { PBAD_HINGE = 0, PBAD_BALL = 1, PBAD_FREE = 2 };
enum { PBAD_GEOM_BOX = 0, PBAD_GEOM_POINTS = 1 };
enum { PBAD_LBFGS = 0, PBAD_LM = 1 };
enum { PBAD_ENERGY_FORM = 0, PBAD_RESIDUAL_FORM = 1 };

/* per-trajectory status (Trajectory::error) */
enum {
  PBAD_TRAJ_OK = 0,
  PBAD_TRAJ_FAIL_LIMIT = 1,     /* "optimizer failed N consecutive steps around t=..." */
  PBAD_TRAJ_NONFINITE_INIT = 2, /* "objective is non-finite at the initial point" */
  PBAD_TRAJ_NONFINITE_CFG = 3,  /* "configuration contains a non-finite entry" */
  PBAD_TRAJ_RUNNING = 4,
  /* simulate_baseline (pbad_gpu_simulate_baseline) */
  PBAD_TRAJ_DIVERGED = 5,       /* "diverged to a non-finite state at t=..." */
  PBAD_TRAJ_SINGULAR_MASS = 6,  /* "step failed: singular generalized mass matrix" */
  PBAD_TRAJ_STAGE_NONFINITE = 7, /* "step failed: configuration contains a non-finite entry" */
  /* refined_bootstrap (stepper.cpp:46-59): baseline_step threw inside
   * init_pbad_run, before sample 0 was recorded */
  PBAD_TRAJ_BOOTSTRAP_SINGULAR = 8 /* "singular generalized mass matrix" */
};

/* BaselineScheme (baseline.hpp:17) */
enum { PBAD_BASELINE_FORWARD_EULER = 0, PBAD_BASELINE_SEMI_IMPLICIT = 1, PBAD_BASELINE_RK2 = 2,
       PBAD_BASELINE_RK3 = 3, PBAD_BASELINE_RK4 = 4 };

/* LinkSpec (model.hpp:57-62) with JointSpec and Geometry flattened. */
typedef struct {
  int32_t parent;       /* -1 = root (std::nullopt) */
  int32_t joint_kind;   /* PBAD_HINGE / PBAD_BALL / PBAD_FREE */
  double axis[3];       /* hinge axis (normalised by build_model) */
  double offset[16];    /* column-major 4x4 joint offset */
  int32_t geom_kind;    /* PBAD_GEOM_BOX / PBAD_GEOM_POINTS */
  double box_size[3];
  double box_density;
  double box_center[3];
  int32_t n_points;
  const double* point_mass; /* [n_points] */
  const double* point_pos;  /* [n_points][3] */
  int32_t n_samples;        /* 0 = default contact samples */
  const double* samples;    /* [n_samples][3] */
} pbad_link_spec;

/* ForceModel (objective.hpp:50-59) incl. ContactModel and ActuationSpec. */
typedef struct {
  double gravity[3];
  double drag_d;
  int32_t has_contact;
  double plane_normal[3];
  double plane_offset;
  double contact_d1;
  double contact_d2;
  int32_t tau_len; /* 0 = no constant actuation */
  const double* tau;
  int32_t has_actuation;
  int32_t act_kind; /* 0 constant, 1 sinusoidal */
  int32_t act_len;
  const double* act_amplitude;
  double act_frequency_hz;
  int32_t act_phase_len;
  const double* act_phase;
} pbad_forces;

/* OptimizerConfig (optim.hpp:15-28) */
typedef struct {
  int32_t kind;
  int32_t max_iters;
  double grad_tol;
  double grad_rtol;
  double ftol;
  int32_t lbfgs_memory;
  double lm_lambda0;
  double lm_lambda_factor;
  double lm_lambda_max;
  double armijo_c1;
  double backtrack_factor;
  int32_t max_line_search;
} pbad_optimizer_config;

/* SimConfig (stepper.hpp:29-44) minus the per-trajectory q0/qdot0. */
typedef struct {
  double dt;
  double duration;
  int32_t order;
  int32_t objective;
  pbad_optimizer_config opt;
  int32_t consecutive_fail_limit;
  int32_t refined_bootstrap; /* RK4 Newton-Euler history bootstrap (stepper.cpp:46-59) */
  int32_t warm_start;
} pbad_sim_desc;

/* Caller-owned host output buffers of a rollout (any pointer may be NULL).
 * S = total steps = ceil(duration/dt - 1e-9). */
typedef struct {
  double* q;               /* [B][S+1][n] samples (t_k = k*dt) */
  double* energy;          /* [B][S+1][2] kinetic, potential */
  int32_t* iterations;     /* [B][S] SolveReport::iterations */
  int32_t* converged;      /* [B][S] */
  int32_t* accepted;       /* [B][S] accepted iterations */
  double* final_value;     /* [B][S] */
  double* final_grad_norm; /* [B][S] */
  int32_t* n_samples;      /* [B] recorded samples */
  int32_t* status;         /* [B] PBAD_TRAJ_* */
  int32_t* fail_streak;    /* [B] streak at abort (error text) */
  int32_t* n_reports;      /* [B] recorded solve reports */
  float* device_ms;        /* [1] device time of the stepping kernels */
  double* iteration_values; /* [B][S][max_iters] SolveReport::per_iteration_values
                               (optim.cpp:30-37, 64-67): the objective value after
                               each iteration of step s, iterations[b][s] entries;
                               pbad_gpu_rollout / _sharded only, NULL = off */
} pbad_rollout_out;

typedef struct pbad_gpu_model pbad_gpu_model;
typedef struct pbad_gpu_ctx pbad_gpu_ctx;

int32_t pbad_gpu_abi_version(void);
const char* pbad_gpu_last_error(void);
const char* pbad_gpu_error_string(int32_t code);

/* visible CUDA devices (0 when none: the GPU path has no CPU fallback) */
int32_t pbad_gpu_device_count(void);

void pbad_gpu_default_optimizer(pbad_optimizer_config* cfg);
void pbad_gpu_default_sim(pbad_sim_desc* sim);

/* model (host-side validation, body integrals, default contact samples) */
int32_t pbad_gpu_model_create(const pbad_link_spec* links, int32_t n_links,
                              pbad_gpu_model** out);
void pbad_gpu_model_destroy(pbad_gpu_model* model);
int32_t pbad_gpu_model_dofs(const pbad_gpu_model* model);
int32_t pbad_gpu_model_links(const pbad_gpu_model* model);
int32_t pbad_gpu_model_info(const pbad_gpu_model* model, double* S /*[N][16]*/,
                            double* mass /*[N]*/, int32_t* dof_offset /*[N]*/,
                            double* axis /*[N][3]*/, int32_t* sample_count /*[N]*/);
int32_t pbad_gpu_body_integral(const pbad_link_spec* link, double* S /*[16]*/,
                               double* mass);
int32_t pbad_gpu_rotation_vector_matrix(const double theta[3], double R[9]);
int32_t pbad_gpu_rotation_vector_from_matrix(const double R[9], double theta[3]);
int32_t pbad_gpu_build_scheme(int32_t order, double dt, double* alphas, double* times,
                              double* H, double* H2);
int32_t pbad_gpu_validate_configuration(const pbad_gpu_model* model, const double* q,
                                        int32_t len);

/* context: device copy of the model + forces + schedule, sized for max_batch */
int32_t pbad_gpu_create(const pbad_gpu_model* model, const pbad_forces* forces,
                        const pbad_sim_desc* sim, int32_t device, int32_t max_batch,
                        pbad_gpu_ctx** out);
void pbad_gpu_destroy(pbad_gpu_ctx* ctx);
int32_t pbad_gpu_total_steps(const pbad_gpu_ctx* ctx);
/* which kernel family steps this context's rollouts (no reference
 * counterpart; reported by bench.py and asserted by the tests) */
#define PBAD_PATH_GENERAL 0 /* thread per environment, any model (pbad_kernels.cu) */
#define PBAD_PATH_CHAIN 1   /* quad per environment, hinge chains (pbad_chain.cu) */
#define PBAD_PATH_CHAIN4 2  /* warp-synchronous quads, axis-aligned hinge chains (pbad_chain4.cu) */
#define PBAD_PATH_TREE 3    /* warp per environment, trees with LM / Newton (pbad_tree.cu) */
#define PBAD_PATH_RESID 4   /* CTA per environment, residual (collocation) form with LM (pbad_resid.cu) */
#define PBAD_PATH_CHAIN5 5  /* warp per environment, axis-aligned hinge chains, shared-memory L-BFGS (pbad_chain5.cu) */
#define PBAD_PATH_CHAIN6 6  /* 8 lanes per environment (two per row), axis-aligned hinge chains (pbad_chain6.cu) */
#define PBAD_PATH_CHAIN7 7  /* 16 lanes per environment, link-parallel energy terms, axis-aligned hinge chains (pbad_chain7.cu) */
int32_t pbad_gpu_path(const pbad_gpu_ctx* ctx);
/* step kernels this context has launched so far (no reference counterpart;
 * bench.py's gpu_launches): one per PBAD step, except the tree family's
 * persistent multi-step launch for contact scenes (one per window) */
int64_t pbad_gpu_kernel_launches(const pbad_gpu_ctx* ctx);

/* batch_simulate on the GPU: q0/qdot0 host [B][n]; copies in, steps every
 * trajectory to completion, copies the requested outputs back.  The device
 * keeps a window of the trajectory (all of it when B*(S+1)*(n+2) doubles fit
 * PBAD_TRAJ_WINDOW_MB, default 2048) and drains each window to the host
 * buffers between launches, so long rollouts do not need B*S*n of HBM.
 * device_ms: device time from the first step launch to the last (it includes
 * the drains of all windows but the last when the rollout is windowed). */
int32_t pbad_gpu_rollout(pbad_gpu_ctx* ctx, int32_t B, const double* q0,
                         const double* qdot0, pbad_rollout_out* out);

/* batch_simulate sharded over several contexts (stepper.cpp:204-270: the
 * trajectories share only the immutable model), one per device or several
 * per device: context i steps the contiguous environments
 * [B*i/n_ctx, B*(i+1)/n_ctx) of the host arrays, all contexts concurrently
 * (no collective: every trajectory is independent).  The contexts must share
 * the model's DOF count and the step count; results equal pbad_gpu_rollout
 * of the whole batch on one context bit for bit.  device_ms = the slowest
 * context's device time. */
int32_t pbad_gpu_rollout_sharded(pbad_gpu_ctx* const* ctxs, int32_t n_ctx, int32_t B,
                                 const double* q0, const double* qdot0,
                                 pbad_rollout_out* out);

/* device-resident stepping: q0/qdot0 are DEVICE pointers [B][n]; stream is
 * a cudaStream_t (NULL = the ctx stream).  advance() launches n_steps PBAD
 * steps for the whole batch without host synchronisation. */
int32_t pbad_gpu_begin(pbad_gpu_ctx* ctx, int32_t B, const double* d_q0,
                       const double* d_qdot0, void* stream);
int32_t pbad_gpu_advance(pbad_gpu_ctx* ctx, int32_t n_steps, void* stream);
/* copy outputs of the current batch to host buffers (synchronises the ctx
 * stream after the stream of the last begin/advance; no device-wide barrier) */
int32_t pbad_gpu_sync_outputs(pbad_gpu_ctx* ctx, pbad_rollout_out* out);
/* the latest configuration of every environment of the current batch
 * (its last recorded sample) into a DEVICE buffer [B][n], env-major, on
 * `stream` (NULL = ctx stream), without a host round trip: the source of the
 * multi-GPU final-state gather */
int32_t pbad_gpu_final_state(pbad_gpu_ctx* ctx, double* d_dst, void* stream);
/* device pointer of the current configurations hist1 [B][n] */
const double* pbad_gpu_state_device(const pbad_gpu_ctx* ctx);

/* StepObjective on a batch: history [B][2][n] (times[0], times[1]);
 * tau [B][K-1][n] or NULL (forces.tau); x [B][dim], dim=(K-1)n.
 * want_grad=0 gives StepObjective::value.  gn [B][dim][dim] column-major. */
int32_t pbad_gpu_eval(pbad_gpu_ctx* ctx, int32_t B, const double* history,
                      const double* tau, const double* x, int32_t want_grad,
                      int32_t want_gn, double* value, double* grad, double* gn);

/* simulate_baseline (stepper.cpp:168-202, baseline.cpp:56-206): explicit
 * Newton-Euler integration with the context's model, forces (gravity, drag,
 * contact, constant tau) and dt / duration; q_out [B][S+1][n] and energy
 * [B][S+1][2] (KE, PE) optional, n_samples / status (PBAD_TRAJ_*) [B]. */
int32_t pbad_gpu_simulate_baseline(pbad_gpu_ctx* ctx, int32_t scheme, int32_t B, const double* q0,
                                   const double* qdot0, double* q_out, double* energy,
                                   int32_t* n_samples, int32_t* status);

/* Correlation derivatives of a batch of configuration pairs (adjoint.hpp:80-82:
 * correlation_and_grad, hessian_bb, hessian_ab), qa/qb [B][n];
 * weight_per_body [n_links] or NULL (all ones, WeightedBody::make); outputs
 * value [B], grad_b [B][n], hess_bb / hess_ab [B][n][n] column-major, each
 * optional (NULL = not computed).  Non-finite inputs propagate like the
 * reference's ConfigPass::make. */
int32_t pbad_gpu_correlation(pbad_gpu_ctx* ctx, int32_t B, const double* qa, const double* qb,
                             const double* weight_per_body, double* value, double* grad_b,
                             double* hess_bb, double* hess_ab);

/* parallel_correlation_suite (adjoint.hpp:103-108, adjoint.cpp:241-336): the
 * same four derivatives as pbad_gpu_correlation for B configuration pairs,
 * computed the large-N way: one CTA per pair, the reference's per-link work
 * items (value slot + grad_b, hess_bb block, hess_ab block) spread over its
 * threads.  grad_b is assigned, as the suite does (pbad_gpu_correlation
 * accumulates like correlation_grad_b: they differ only in the sign of a
 * zero).  Same output layouts, each optional. */
int32_t pbad_gpu_correlation_suite(pbad_gpu_ctx* ctx, int32_t B, const double* qa, const double* qb,
                                   const double* weight_per_body, double* value, double* grad_b,
                                   double* hess_bb, double* hess_ab);

/* functional_value / functional_grad / functional_hess (adjoint.hpp:52-60,
 * adjoint.cpp:43-101) of f(q) = sum_i ddot(C_i, T^i(q)) for B (q, seeds)
 * pairs: q [B][n], seeds [B][n_links][16] column-major cotangents C_i;
 * value [B], grad [B][n], hess [B][n][n] column-major, each optional.
 * One CTA per pair (pbad_corr.cu). */
int32_t pbad_gpu_functional(pbad_gpu_ctx* ctx, int32_t B, const double* q, const double* seeds,
                            double* value, double* grad, double* hess);

/* minimize() of a batch of step problems (same inputs as eval, x0 [B][dim]). */
int32_t pbad_gpu_minimize(pbad_gpu_ctx* ctx, int32_t B, const double* history,
                          const double* tau, const double* x0, double* x_out,
                          int32_t* iterations, int32_t* converged, double* final_value,
                          double* final_grad_norm);

#ifdef __cplusplus
}
#endif

#endif /* PBAD_GPU_H */
