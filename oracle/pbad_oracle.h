/*
 * pbad_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the PBAD reference hot path (arXiv 1709.04145 reference,
 * /root/reference/proj), used as the parity checker for the CUDA path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  Every function cites the reference file:line it follows.
 * Arithmetic follows the canonical contract in pbo_math.h, so the oracle is
 * bit-identical to the reference compiled against oracle/eigen_lite.
 */
#ifndef PBAD_ORACLE_H
#define PBAD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PBO_HINGE = 0, PBO_BALL = 1, PBO_FREE = 2 };
enum { PBO_BOX = 0, PBO_POINTS = 1 };
enum { PBO_LBFGS = 0, PBO_LM = 1 };
enum { PBO_ENERGY = 0, PBO_RESIDUAL = 1 };

/* LinkSpec / JointSpec / Geometry, model.hpp:24-62 */
typedef struct {
  int32_t parent; /* -1 = root */
  int32_t joint_kind;
  double axis[3];
  double offset[16]; /* column-major 4x4 */
  int32_t geom_kind;
  double box_size[3];
  double box_density;
  double box_center[3];
  int32_t n_points;
  const double* point_mass; /* [n_points] */
  const double* point_pos;  /* [n_points][3] */
  int32_t n_samples;        /* 0 = default (box corners / point positions) */
  const double* samples;    /* [n_samples][3] */
} pbo_link_spec;

/* ForceModel, objective.hpp:20-59 */
typedef struct {
  double gravity[3];
  double drag_d;
  int32_t has_contact;
  double plane_normal[3];
  double plane_offset;
  double contact_d1;
  double contact_d2;
  int32_t tau_len;
  const double* tau;
  int32_t has_actuation;
  int32_t act_kind; /* 0 constant, 1 sinusoidal */
  int32_t act_len;
  const double* act_amplitude;
  double act_frequency_hz;
  int32_t act_phase_len;
  const double* act_phase;
} pbo_forces;

/* OptimizerConfig, optim.hpp:15-28 */
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
} pbo_optimizer_config;

/* SimConfig, stepper.hpp:29-44 */
typedef struct {
  double dt;
  double duration;
  int32_t order;
  int32_t objective;
  pbo_optimizer_config opt;
  const double* q0;
  const double* qdot0;
  int32_t consecutive_fail_limit;
  int32_t refined_bootstrap;
  int32_t warm_start;
} pbo_sim_config;

/* Trajectory (stepper.hpp:22-27), caller-owned buffers */
typedef struct {
  int32_t capacity_steps;   /* in */
  int32_t n_samples;        /* out: recorded samples (steps + 1) */
  double* times;            /* [cap+1] */
  double* q;                /* [cap+1][n] */
  double* energy;           /* [cap+1][2] kinetic, potential */
  int32_t* iterations;      /* [cap] */
  int32_t* converged;       /* [cap] */
  int32_t* accepted;        /* [cap] accepted iterations (derived from values) */
  double* final_value;      /* [cap] */
  double* final_grad_norm;  /* [cap] */
  int32_t has_error;
  char error[256];
} pbo_trajectory;

typedef struct pbo_model pbo_model;

void pbo_default_optimizer(pbo_optimizer_config* cfg);
void pbo_default_sim(pbo_sim_config* sim);

/* build_model, model.cpp:62-112.  Returns 0 or -1 with err filled. */
int pbo_model_create(const pbo_link_spec* links, int32_t n_links, pbo_model** out,
                     char* err, int32_t errlen);
void pbo_model_free(pbo_model* m);
int32_t pbo_model_dofs(const pbo_model* m);
int32_t pbo_model_links(const pbo_model* m);
/* body integrals / dof offsets / normalised axes / samples of the built model */
void pbo_model_info(const pbo_model* m, double* S /*[N][16]*/, double* mass /*[N]*/,
                    int32_t* dof_offset /*[N]*/, double* axis /*[N][3]*/,
                    int32_t* sample_count /*[N]*/);
int32_t pbo_model_samples(const pbo_model* m, int32_t link, double* out /*[k][3]*/);

/* body_integral, model.cpp:35-60 */
void pbo_body_integral(const pbo_link_spec* link, double* S, double* mass);

/* kinematics, kinematics.cpp:89-181 */
void pbo_rotation_vector_matrix(const double theta[3], double R[9]);
int pbo_joint_jet(int32_t kind, const double axis[3], const double offset[16],
                  const double* q_local, double value[16], double* d1 /*[dof][16]*/,
                  double* d2 /*[dof(dof+1)/2][16]*/);
int pbo_joint_transform(int32_t kind, const double axis[3], const double offset[16],
                        const double* q_local, double value[16]);
int pbo_forward_pass(const pbo_model* m, const double* q, double* world /*[N][16]*/);

/* adjoint.cpp:113-200: correlation value, grad_b, hess_bb, hess_ab */
int pbo_correlation(const pbo_model* m, const double* qa, const double* qb,
                    const double* weights /*[N] or NULL*/, double* value,
                    double* grad_b /*[n] or NULL*/, double* hess_bb /*[n][n] or NULL*/,
                    double* hess_ab /*[n][n] or NULL*/);
/* functional_grad / functional_hess, adjoint.cpp:49-101 */
int pbo_functional(const pbo_model* m, const double* seeds /*[N][16]*/, const double* q,
                   double* value, double* grad, double* hess);

/* collocation, collocation.cpp:26-95 */
int pbo_legendre_points(int32_t order, double* out /*[order-1]*/);
int pbo_build_scheme(int32_t order, double dt, double* alphas /*[K-1]*/,
                     double* times /*[K+1]*/, double* H /*[(K+1)^2] col-major*/,
                     double* H2 /*[(K+1)^2] col-major*/);

/* eval_potentials, objective.cpp:140-153 (value, grad[n], gn[n][n], hess[n][n]) */
int pbo_eval_potentials(const pbo_model* m, const pbo_forces* f, const double* q_next,
                        const double* q_prev, double dt, int32_t want_gn,
                        int32_t want_hess, double* value, double* grad, double* gn,
                        double* hess);

/* StepObjective::evaluate / value, objective.cpp:155-343.
 * history: [2][n]; tau_instants: [K-1][n] or NULL; x: [(K-1) n].
 * want_grad=0 reproduces StepObjective::value(). */
int pbo_step_eval(const pbo_model* m, const pbo_forces* f, int32_t order, double dt,
                  int32_t objective, const double* history, const double* tau_instants,
                  const double* x, int32_t want_grad, int32_t want_gn, double* value,
                  double* grad, double* gn);

/* minimize, optim.cpp:236-250 on a StepObjective (iters/values reported). */
int pbo_step_minimize(const pbo_model* m, const pbo_forces* f, int32_t order, double dt,
                      int32_t objective, const double* history,
                      const double* tau_instants, const double* x0,
                      const pbo_optimizer_config* cfg, double* x_out,
                      int32_t* iterations, int32_t* converged, double* final_value,
                      double* final_grad_norm, double* per_iter_values /*[max_iters]*/);

/* spd_solve, optim.cpp:11-15. Returns 0 ok, 1 not SPD. */
int pbo_spd_solve(const double* A /*[n][n] col-major*/, const double* b, int32_t n,
                  double* x);

/* simulate, stepper.cpp:151-166.  Returns 0, or -1 when it would throw (the
 * trajectory error string is filled and the recorded prefix is valid). */
int pbo_simulate(const pbo_model* m, const pbo_forces* f, const pbo_sim_config* sim,
                 pbo_trajectory* out);

/* batch_simulate, stepper.cpp:204-270 (threads over independent envs). */
int pbo_batch_simulate(const pbo_model* m, const pbo_forces* f,
                       const pbo_sim_config* sims, int32_t count, int32_t workers,
                       pbo_trajectory* outs);

/* kinetic_energy / gravity_potential, baseline.cpp:208-229 */
int pbo_kinetic_energy(const pbo_model* m, const double* q, const double* qdot,
                       double* ke);
int pbo_gravity_potential(const pbo_model* m, const double g[3], const double* q,
                          double* pe);

void pbo_sincos(double x, double* s, double* c);

#ifdef __cplusplus
}
#endif

#endif
