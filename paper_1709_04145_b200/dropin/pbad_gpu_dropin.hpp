// pbad_gpu_dropin.hpp -- C++ drop-in for the reference's step API on the
// B200 path.
//
// A program written against the reference (/root/reference/proj/include/pbad)
// swaps
//     pbad::batch_simulate(model, forces, sims, workers)   stepper.hpp:61-64
//     pbad::simulate(model, forces, sim)                   stepper.hpp:49-50
// for pbad::gpu::batch_simulate / pbad::gpu::simulate with the same argument
// and result types (KinematicModel, ForceModel, SimConfig, Trajectory from the
// reference's own headers) and the same per-trajectory semantics
// (stepper.cpp:151-166, 204-270): heterogeneous SimConfigs in one call,
// per-trajectory error strings instead of exceptions in the batch, the
// runtime_error of simulate() on the fail limit, ModelError for a worker
// count < 1.  Trajectories are grouped by schedule (everything in SimConfig
// except q0 / qdot0); each group is sharded over the visible GPUs (or
// set_devices()) with pbad_gpu_rollout_sharded and no collective.  Results
// are bit-identical to the reference's own batch_simulate (tests:
// tests/test_gpu_dropin.py runs tests/dropin/dropin_check.cpp).
//
// SolveReport::per_iteration_values is filled when
// set_record_iteration_values(true) (off by default: it is
// B x steps x max_iters doubles).
#pragma once

#include <vector>

#include "pbad/stepper.hpp"

namespace pbad::gpu {

/// stepper.hpp:61-64 on the GPU; `workers` is validated like the reference
/// (>= 1) and otherwise unused: the GPU grid replaces the WorkerPool.
std::vector<Trajectory> batch_simulate(const KinematicModel& model, const ForceModel& forces,
                                       const std::vector<SimConfig>& sims, int workers = 1);

/// stepper.hpp:49-50 on the GPU: throws std::runtime_error when the optimizer
/// fails consecutive_fail_limit steps in a row, ModelError / invalid_argument
/// like the reference for invalid input.
Trajectory simulate(const KinematicModel& model, const ForceModel& forces, const SimConfig& sim);

/// Devices the batch is sharded over (empty = every visible device).
void set_devices(const std::vector<int>& devices);
std::vector<int> devices();

/// Record SolveReport::per_iteration_values (optim.cpp:30-37).
void set_record_iteration_values(bool on);

}  // namespace pbad::gpu
