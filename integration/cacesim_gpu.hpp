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
// ONE GPU sweep (the OpenMP cell fan-out of experiment.cpp:100-115 becomes
// the scenario batch); metrics/averaging stay the reference's own functions.
// parallel (as in the reference): spread the sweep over every visible GPU,
// one host thread each; false = device 0 only.  Results are identical.
GridResult run_grid(const ExperimentConfig& cfg, const ModelCatalog& catalog, bool parallel = true);

// Many independent replays of (trace, policy, cluster) triples — the
// scenario sweep of BASELINE configs 3/4 — returning one report each.
std::vector<SimulationReport> run_many(const std::vector<const Trace*>& traces,
                                       const ModelCatalog& catalog,
                                       const std::vector<std::pair<PolicyConfig, ClusterConfig>>& runs,
                                       const std::vector<int>& trace_of_run, bool parallel = true);

// metrics.cpp:35-62 — compute_run_metrics of many replays, computed on the
// device (cace_run_metrics_batch): no per-request outcomes leave the GPU.
// Counts, nearest-rank percentiles, max, hit rate, load overhead and
// evictions are bit-identical to compute_run_metrics(run(...)); mean_s
// divides the replay-order sum instead of the sorted-order one (~1e-15
// relative).
std::vector<RunMetrics> run_metrics_many(const std::vector<const Trace*>& traces,
                                         const ModelCatalog& catalog,
                                         const std::vector<std::pair<PolicyConfig, ClusterConfig>>& runs,
                                         const std::vector<int>& trace_of_run, bool parallel = true);

// experiment.hpp:54-55 — run_grid whose per-seed metrics come from the
// device (run_metrics_many) and are averaged with the reference's
// average_metrics; the cells' reports carry counters and meta but no
// outcomes (the whole point: 10^11 outcomes never cross PCIe).
GridResult run_grid_metrics(const ExperimentConfig& cfg, const ModelCatalog& catalog,
                            bool parallel = true);

}  // namespace cacesim::gpu
