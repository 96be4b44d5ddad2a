// pbad_launch.h -- host-callable launchers for the kernels in pbad_kernels.cu
#pragma once

#include <cuda_runtime.h>

#include "pbad_kernels.cuh"

namespace pbad_gpu {

// Dynamic shared memory a kernel has been enabled for, per device:
// cudaFuncSetAttribute acts on the current device only, so one process
// driving several GPUs (pbad_gpu_rollout_sharded) sets it on each.
struct SmemAttr {
  size_t bytes[64] = {};
  size_t& here() {
    int d = 0;
    cudaGetDevice(&d);
    return bytes[d & 63];
  }
};

struct KernelArgs {
  DModel m;
  DForces f;
  DSchedule sc;
  Layout L;
  double* ws;
  int* iws;
  long B;
};

struct ChainArgs {
  DModel m;
  DForces f;
  DSchedule sc;
  ChainLayout L;
  double* cw;
  int* ci;
  long B;
};

cudaError_t launch_chain_init(const ChainArgs& a, const double* q0, const double* qdot0, const double* hist0,
                              const Outputs& out, cudaStream_t s);
cudaError_t launch_chain_step(const ChainArgs& a, const Outputs& out, cudaStream_t s);
int chain_max_memory();
int chain_max_links();
// chain v4 (pbad_chain4.cu): axis-aligned hinge chains, warp-synchronous L-BFGS
int chain4_pattern(const int* kinds, int N);
cudaError_t launch_chain4_step(const ChainArgs& a, int pattern, const Outputs& out, cudaStream_t s);
size_t chain4_smem_bytes(int N);
int chain4_max_memory();
long chain4_record_doubles(bool massive);
long chain4_hist_doubles();
// chain v5 (pbad_chain5.cu): warp per environment, shared-memory-resident L-BFGS
bool chain5_fits(int N, int n, int mem);
int chain5_waves(int N, int n, int mem, long B, int pattern, int device);
// chain v6 (pbad_chain6.cu): v4 with two lanes per row, 4 environments per warp
bool chain6_fits(int N, int mem);
long chain6_vector_doubles(long B, int n);
cudaError_t launch_chain6_steps(const ChainArgs& a, int pattern, const Outputs& out, int nsteps, cudaStream_t s,
                                long* launches);
cudaError_t launch_chain5_step(const ChainArgs& a, int pattern, long recw, const Outputs& out, cudaStream_t s);
// chain v7 (pbad_chain7.cu): 16 lanes per environment, link-parallel energy terms
bool chain7_fits(int N, int mem, int pattern);
long chain7_vector_doubles(long B, int n);
cudaError_t launch_chain7_step(const ChainArgs& a, int pattern, const Outputs& out, cudaStream_t s);

// tree path (pbad_tree.cu): warp-per-environment LM for articulated trees
bool tree_eligible_sizes(int N, int n);
size_t tree_smem_bytes(const TreeDesc& td);
cudaError_t launch_tree_step(const KernelArgs& a, const TreeDesc& td, double* tws, const Outputs& out,
                             cudaStream_t s);
cudaError_t launch_tree_steps(const KernelArgs& a, const TreeDesc& td, double* tws, const Outputs& out, int nsteps,
                              int* sync, cudaStream_t s, long* launches);
// L-BFGS on trees (pbad_tree_lbfgs.cu, same device code compiled as its own
// translation unit so the LM kernel's register allocation is unaffected)
cudaError_t launch_tree_lbfgs(const KernelArgs& a, const TreeDesc& td, double* tws, const Outputs& out,
                              cudaStream_t s);

// residual-form path (pbad_resid.cu): CTA-per-environment LM, hinge trees
bool resid_eligible_sizes(int N, int u);
size_t resid_smem_bytes(int N, int u);
cudaError_t launch_resid_step(const KernelArgs& a, const ResidDesc& rd, double* rws, const Outputs& out,
                              cudaStream_t s);
cudaError_t launch_resid_steps(const KernelArgs& a, const ResidDesc& rd, double* rws, const Outputs& out, int nsteps,
                               int* sync, cudaStream_t s, long* launches);

cudaError_t launch_init(const KernelArgs& a, const double* q0, const double* qdot0, const double* hist0,
                        const Outputs& out, cudaStream_t s);
cudaError_t launch_step(const KernelArgs& a, const Outputs& out, cudaStream_t s);
// refined_bootstrap history (stepper.cpp:46-59): hist0 [B][n], status [B]
cudaError_t launch_refined_bootstrap(const KernelArgs& a, const Layout& L, double* ws, long B, const double* q0,
                                     const double* qd0, double hs, double* hist0, int* status, cudaStream_t s);
cudaError_t launch_baseline(const KernelArgs& a, const Layout& L, double* ws, long B, int scheme, const double* q0,
                            const double* qd0, double* oq, double* oe, int* nsamp, int* status, cudaStream_t s);
// correlation suite / functional derivatives, one CTA per request (pbad_corr.cu)
struct SuiteLayout {
  long va, wa, d1a, la, vb, wb, pwb, d1b, lb, d2b, seeds, adj, acc, vslot, total;
};
SuiteLayout suite_layout(int N, int n, int n_d2);
cudaError_t launch_suite(const DModel& m, const SuiteLayout& L, double* ws, long B, const double* qa, const double* qb,
                         const double* seeds, int mode, double* value, double* grad, double* hbb, double* hab,
                         cudaStream_t s);
cudaError_t launch_correlation(const DModel& m, const Layout& L, double* ws, long B, const double* qa,
                               const double* qb, double* value, double* grad, double* hbb, double* hab,
                               cudaStream_t s);
cudaError_t launch_eval(const KernelArgs& a, const double* hist, const double* tau, const double* x,
                        int want_grad, int want_gn, double* value, double* grad, double* gn, int* err,
                        cudaStream_t s);
cudaError_t launch_minimize(const KernelArgs& a, const double* hist, const double* tau, const double* x0,
                            double* xout, int* iters, int* conv, double* fval, double* gnorm, int* err,
                            cudaStream_t s);

}  // namespace pbad_gpu
