// pbad_kernels.cuh -- device-side data layout shared by the host launcher
// and the kernels.  One CUDA thread owns one environment (trajectory);
// per-environment arrays are stored structure-of-arrays (element k of env e
// at base[k * B + e]) so a warp's 32 envs touch 32 consecutive doubles.
#pragma once

#include <cstdint>

namespace pbad_gpu {

struct DModel {
  int N, n, n_d2;
  const int* parent;
  const int* kind;
  const int* dof_off;
  const int* dof_cnt;
  const int* d2_off;
  const double* axis;    // [N][3]
  const double* offset;  // [N][16]
  const double* S;       // [N][16]
  const double* mass;    // [N]
  const int* sample_off; // [N+1]
  const double* samples; // [*][3]
  const int* jkind;      // chain path: 0 general hinge, 1/2/3 axis X/Y/Z with identity-rotation offset
  const int* skind;      // chain path: 0 massless (S == 0), 1 general S
  const double* crec;    // chain path: packed link records [N][20]: S (16), offset translation (3), pad
  const int* ckind;      // chain path: jkind | skind << 2
  const int* croff;      // chain v4: per-link record offsets [N+1] (doubles, per warp)
  double weighted_mass;  // WeightedBody::make with unit weights (adjoint.cpp:29-41)
};

struct DForces {
  double gravity[3];
  int gravity_nonzero;  // !gravity.isZero()
  double drag_d;
  int has_contact;
  double normal[3];
  double plane_offset, d1, d2;
  int tau_len;
  const double* tau;  // device
  int has_act, act_kind, act_len;
  const double* act_amp;  // device
  double act_freq;
  int act_phase_len;
  const double* act_phase;  // device
};

struct DOpt {
  int kind, max_iters, mem, max_line_search;
  double grad_tol, grad_rtol, ftol, lm_lambda0, lm_lambda_factor, lm_lambda_max, armijo_c1,
      backtrack_factor;
};

struct DSchedule {
  double dt;
  int order, objective, u, U, K1;
  int fail_limit, warm_start, total_steps;
  double times[9];
  double H2[81];  // column-major (K+1)^2
  DOpt opt;
};

// Offsets (in per-env doubles) of every array in the double workspace.
struct Layout {
  long hist0, hist1, x, grad, cand, dir, tmp, step, evgrad, hs, hy, hsy, alpha, tau;
  long hw0, hw1;                 // history world transforms [N*16]
  long gn, damped, evgn;         // LM (U*U)
  long pass;                     // u passes back to back
  long pass_stride;              // doubles per pass
  long p_value, p_d1, p_d2, p_world, p_lever;  // offsets inside a pass
  long seeds, cot, adj;          // [N*16]
  long potgrad, potgn, pothess, ab, fh, resid, J, g, jx, dd, jr, tmp3;
  long scal;                     // scalar slots
  long total;
};
enum {
  SC_VALUE = 0,
  SC_GRAD0,
  SC_LAMBDA,
  SC_HISTCONST,
  SC_EVVALUE,
  SC_COUNT
};
// int workspace slots (per env)
enum {
  IS_STATUS = 0,   // solver status
  IS_ITERS,
  IS_STAG,
  IS_ACC,
  IS_HSTART,
  IS_HCOUNT,
  IS_FAIL,         // fail streak
  IS_STEP,         // PBAD step counter
  IS_RUN,          // trajectory status PBAD_TRAJ_*
  IS_NSAMP,
  IS_NREP,
  IS_COUNT
};

// Chain-path workspace (pbad_chain.cu): link arrays [N][B][16] (row r at
// +4r) and quad-interleaved vectors (element k at ((k>>2)*B + e)*4 + k%4).
struct ChainLayout {
  long tk, tk1, seed, lev, lmat;            // link arrays
  long h0, h1, x, g, cand, dir, q, evg, tau; // vectors
  long hs, hy, vstride;                      // L-BFGS ring, vstride per vector
  long hsy, histc;                           // [cap][B], [B]
  long rec, rec_w, hist;                     // chain v4: link records [warp][rec_w], hist rotations [warp][N][8][6]
  long total;
};

// Tree path (pbad_tree.cu): warp-per-environment Newton (LM) for articulated
// trees.  Host-precomputed structure; the per-env global workspace `tws` is
// env-major with stride `gstride` doubles: GN lower-packed [np], history
// world transforms hw0/hw1 [N][16] and their body products T0/T1 [N][16].
struct TreeDesc {
  int N, n, D, np;         // links, dofs, max depth, n(n+1)/2
  int n_tasks;
  const int* lvl_start;    // [D+2] offsets into lvl_links
  const int* lvl_links;    // links ordered by depth (ascending index within a level)
  const int* ch_start;     // [N+1]
  const int* ch_list;      // children of each link in DESCENDING index order (adjoint.cpp:54-62)
  const int* task_start;   // [D+2] GN tasks of walk step s (0 = own block)
  const int* tasks;        // packed i | l<<8 | j<<16 | k<<20
  const int* anc;          // [N][D+1]: s-th ancestor of link i (anc[i][0] = i), -1 beyond the root
  const int* depth;        // [N]
  const int* pk;           // [np] packed lower index -> row | col<<16
  const int* dof_link;     // [n] link owning each dof
  int smem_doubles;        // per environment
  long gstride;            // per-env doubles of tws
  long o_hw0, o_hw1, o_t0, o_t1;  // offsets inside one env's tws block (GN at 0)
  long o_gs;                      // GN composite-inertia scratch [4][N][18] (PBAD_TREE_GN_GLOBAL)
  // drag / contact potentials (objective.cpp:60-131)
  int pot;                        // 1: drag and/or contact present (slow GN path)
  int ns;                         // total contact samples (0 without contact)
  long o_abl, o_abu;              // packed ab(col,row) / ab(row,col) [np] (pot path)
  long o_cs;                      // contact sample scratch [ns][4n]: dd (n), jr (3n)
  // L-BFGS on trees (optim.cpp:141-232): s / y ring [(mem+1)][n], s.y and alpha [mem+1]
  int lb;
  long o_hs, o_hy, o_hsy, o_alpha;
};

// Residual-form path (pbad_resid.cu): CTA-per-environment LM for hinge
// trees.  Per-env global workspace `rws`, env-major, stride gstride doubles.
struct ResidDesc {
  int N, n, u, U, D;
  int chain;               // serial chain: every dof pair is ancestor-related (J dense)
  const int* lvl_start;    // [D+2]
  const int* lvl_links;    // [N]
  const int* ch_start;     // [N+1]
  const int* ch_list;      // children, descending index
  const int* walk_order;   // [N] links by depth, deepest first (walk load balance)
  long pstride;            // doubles per link pass (value, world, d1, d2, lever: 5 x 16N)
  long gstride;
  long oJ, oGN, oDM, oFH, oPH, oPass, oHW0, oHW1, oHA, oFA, oSeeds, oCot, oX, oGrad, oCand, oRes, oPg, oTau, oStep;
  int ns;    // contact samples (0: no contact terms)
  long oCJ;  // contact: [u][ns][3n + 10] (hxx, active, jx column-major 3 x n)
};

struct Outputs {
  double* q;        // [B][qs][n]: sample qbase + j in slot j
  double* energy;   // [B][qs][2]
  int* iterations;  // [B][rs]: report of step rbase + j in slot j
  int* converged;
  int* accepted;
  double* final_value;
  double* final_grad_norm;
  // slot geometry: the whole trajectory (qs = S + 1, rs = S, bases 0), or a
  // window of it that pbad_gpu_rollout drains to the host between launches
  long qs, qbase, rs, rbase;
  // SolveReport::per_iteration_values [B][rs][itv_n] (itv_n = max_iters), or null
  double* itv;
  long itv_n;
  __host__ __device__ long qrow(long e, long sample) const { return e * qs + (sample - qbase); }
  __host__ __device__ long rrow(long e, long step) const { return e * rs + (step - rbase); }
};

}  // namespace pbad_gpu
