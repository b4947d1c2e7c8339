// Drop-in GPU backend for the reference simulator's hot path.
//
// A maintainer of the reference (arXiv 2506.18796 artifact, proj/) adds this
// header + cacesim_gpu.cpp to src/ and links libcace_gpu.so; call sites swap
// cacesim::run / cacesim::run_grid for cacesim::gpu::run / run_grid.  Same
// types, same results (bit-exact), same SimError behaviour.  See
// INTEGRATION.md.
#pragma once

#include "cacesim/engine.hpp"
#include "cacesim/experiment.hpp"

namespace cacesim::gpu {

// engine.hpp:60-61 — one replay on the GPU, full SimulationReport.
SimulationReport run(const Trace& trace, const ModelCatalog& catalog, const ClusterConfig& cluster,
                     const Policy& policy);

// experiment.hpp:54-55 — every (pattern, variant, seed) run of the grid as
// ONE GPU sweep (the OpenMP cell fan-out of experiment.cpp:105 becomes the
// scenario batch); metrics/averaging stay the reference's own functions.
GridResult run_grid(const ExperimentConfig& cfg, const ModelCatalog& catalog);

// Many independent replays of (trace, policy, cluster) triples — the
// scenario sweep of BASELINE configs 3/4 — returning one report each.
std::vector<SimulationReport> run_many(const std::vector<const Trace*>& traces,
                                       const ModelCatalog& catalog,
                                       const std::vector<std::pair<PolicyConfig, ClusterConfig>>& runs,
                                       const std::vector<int>& trace_of_run);

}  // namespace cacesim::gpu
