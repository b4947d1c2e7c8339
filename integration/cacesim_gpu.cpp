// Reference-side binding of the B200 engine (include/cace_gpu.h) — see
// cacesim_gpu.hpp and INTEGRATION.md.  Converts the reference's types to the
// C ABI's structure-of-arrays form and the dumped outcomes back.
#include "cacesim_gpu.hpp"

#include <algorithm>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>

#include "cace_gpu.h"
#include "cacesim/metrics.hpp"

namespace cacesim::gpu {
namespace {

struct CatalogSoA {
  std::vector<double> lt, pr, dr;
  std::vector<int32_t> tok, lex, cls;
  std::vector<const char*> ids;
  cace_catalog_t abi{};
  explicit CatalogSoA(const ModelCatalog& c) {
    const auto& ms = c.models();
    const int M = static_cast<int>(ms.size());
    std::vector<int> order(M);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(),
              [&](int a, int b) { return ms[a].model_id < ms[b].model_id; });  // policy.cpp:92-98
    lex.assign(M, 0);
    for (int r = 0; r < M; ++r) lex[order[r]] = r;
    for (const auto& m : ms) {
      lt.push_back(m.load_time_s);
      pr.push_back(m.prefill_rate_tps);
      dr.push_back(m.decode_rate_tps);
      tok.push_back(m.expected_output_tokens);
      cls.push_back(static_cast<int32_t>(m.task_class));
      ids.push_back(m.model_id.c_str());
    }
    abi = cace_catalog_t{M, lt.data(), pr.data(), dr.data(), tok.data(), lex.data(), cls.data(),
                         ids.data()};
  }
};

struct TraceSoA {
  std::vector<double> arrival;
  std::vector<int32_t> model, prompt, output;
  TraceSoA(const Trace& t, const ModelCatalog& c) {
    const ModelDescriptor* base = c.models().data();
    for (const auto& r : t.requests) {
      arrival.push_back(r.arrival_time_s);
      model.push_back(static_cast<int32_t>(&c.lookup(r.language, r.task_class) - base));  // throws like run()
      prompt.push_back(r.prompt_tokens);
      output.push_back(r.output_tokens);
    }
  }
  cace_trace_t abi() const {
    return cace_trace_t{static_cast<int64_t>(arrival.size()), arrival.data(), model.data(),
                        prompt.data(), output.data()};
  }
};

cace_scenario_t scenario(int trace, const PolicyConfig& p, const ClusterConfig& c) {
  return cace_scenario_t{trace, static_cast<int32_t>(p.variant), static_cast<int32_t>(p.p1_mode),
                         p.window_length, p.output_token_normalizer, c.num_accelerators,
                         c.models_per_accelerator, 0, p.w1, c.unload_time_s};
}

// run_config_hash (engine.cpp:64-72) restated: fnv1a of the same string.
std::uint64_t config_hash(const ClusterConfig& cluster, const PolicyConfig& cfg) {
  std::ostringstream ss;
  ss << cluster.num_accelerators << '|' << cluster.models_per_accelerator << '|'
     << cluster.unload_time_s << '|' << to_string(cfg.variant) << '|' << cfg.w1 << '|'
     << cfg.window_length << '|' << cfg.output_token_normalizer << '|' << to_string(cfg.p1_mode);
  return fnv1a(ss.str());
}

// Runs [b, e) of the sweep on one device: a full dump (outcomes + eviction
// log) straight into the caller's outcome columns (the runs' outcomes are
// contiguous there, at off[b]).
struct DumpCols {
  std::vector<uint8_t> cold;
  std::vector<double> qw, lw, pf, dc, tt, ee;
  std::vector<int64_t> n_ev;
  std::vector<cace_summary_t> summ;
};

void replay_range(int device, const CatalogSoA& cat, const std::vector<cace_trace_t>& tabi,
                  const std::vector<cace_scenario_t>& sc, const std::vector<int64_t>& off, int64_t b,
                  int64_t e, DumpCols& d, int32_t& rc, std::string& err) {
  const int64_t n = e - b;
  std::vector<int64_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  const int64_t o = off[b];
  cace_dump_t dump{static_cast<int32_t>(n), idx.data(), d.cold.data() + o, d.qw.data() + o, d.lw.data() + o,
                   d.pf.data() + o, d.dc.data() + o, d.tt.data() + o, d.ee.data() + o, 0, nullptr, nullptr,
                   d.n_ev.data() + b};
  cace_opts_t opts{device, CACE_KERNEL_AUTO, -1, 0, nullptr};
  char msg[512] = {0};
  rc = cace_replay_batch(&cat.abi, tabi.data(), static_cast<int32_t>(tabi.size()), sc.data() + b, n,
                         d.summ.data() + b, &dump, &opts, msg, sizeof msg);
  if (rc != CACE_OK) err = msg;
}

}  // namespace

std::vector<SimulationReport> run_many(const std::vector<const Trace*>& traces,
                                       const ModelCatalog& catalog,
                                       const std::vector<std::pair<PolicyConfig, ClusterConfig>>& runs,
                                       const std::vector<int>& trace_of_run, bool parallel) {
  // run() preconditions first, in the reference's order (engine.cpp:79-82),
  // then the per-request catalog lookups (engine.cpp:87-92).
  for (const auto& [pc, cc] : runs) {
    if (pc.window_length < 1) throw SimError("run: window_length must be >= 1");
    if (cc.num_accelerators < 1) throw SimError("run: need at least one accelerator");
  }
  CatalogSoA cat(catalog);
  std::vector<TraceSoA> tsoa;
  std::vector<cace_trace_t> tabi;
  for (const Trace* t : traces) tsoa.emplace_back(*t, catalog);
  for (const auto& t : tsoa) tabi.push_back(t.abi());
  const int64_t S = static_cast<int64_t>(runs.size());
  std::vector<cace_scenario_t> sc;
  for (int64_t i = 0; i < S; ++i) sc.push_back(scenario(trace_of_run[i], runs[i].first, runs[i].second));
  std::vector<int64_t> off(S + 1, 0);
  for (int64_t i = 0; i < S; ++i) off[i + 1] = off[i] + tabi[trace_of_run[i]].n_requests;
  const int64_t total = off[S];
  DumpCols d;
  d.cold.resize(total);
  for (auto* v : {&d.qw, &d.lw, &d.pf, &d.dc, &d.tt, &d.ee}) v->resize(total);
  d.n_ev.resize(S);
  d.summ.resize(S);
  // The device-scale form of run_grid's OpenMP fan-out (experiment.cpp:100-115):
  // with parallel and several GPUs, contiguous run ranges of about equal
  // request count go to one host thread + device each; serial = device 0.
  const int nd = parallel ? std::max(1, std::min<int>(cace_device_count(), static_cast<int>(S))) : 1;
  std::vector<int64_t> cut(nd + 1, S);
  cut[0] = 0;
  for (int k = 1; k < nd; ++k)
    cut[k] = std::lower_bound(off.begin(), off.end() - 1, total * k / nd) - off.begin();
  std::vector<int32_t> rcs(nd, CACE_OK);
  std::vector<std::string> errs(nd);
  if (nd == 1) {
    replay_range(0, cat, tabi, sc, off, 0, S, d, rcs[0], errs[0]);
  } else {
    std::vector<std::thread> th;
    for (int k = 0; k < nd; ++k)
      if (cut[k] < cut[k + 1])
        th.emplace_back(replay_range, k, std::cref(cat), std::cref(tabi), std::cref(sc), std::cref(off),
                        cut[k], cut[k + 1], std::ref(d), std::ref(rcs[k]), std::ref(errs[k]));
    for (auto& t : th) t.join();
  }
  // the first failing run in sweep order wins, as the serial loop would raise it
  for (int k = 0; k < nd; ++k)
    if (rcs[k] != CACE_OK) throw SimError(errs[k]);  // same text as the reference's SimError
  std::vector<SimulationReport> out(S);
  for (int64_t i = 0; i < S; ++i) {
    const Trace& t = *traces[trace_of_run[i]];
    const auto& [pc, cc] = runs[i];
    SimulationReport& rep = out[i];
    rep.meta.variant = pc.variant;
    rep.meta.seed = t.seed;
    rep.meta.pattern = t.pattern;
    rep.meta.config_hash = config_hash(cc, pc);
    rep.counters.hits = d.summ[i].hits;
    rep.counters.misses = d.summ[i].misses;
    rep.counters.evictions = d.summ[i].evictions;
    rep.counters.load_overhead_s = d.summ[i].load_overhead_s;
    rep.loads = d.summ[i].loads;
    rep.max_resident = d.summ[i].max_resident;
    rep.outcomes.resize(t.requests.size());
    for (size_t k = 0; k < t.requests.size(); ++k) {
      const int64_t o = off[i] + static_cast<int64_t>(k);
      const Request& r = t.requests[k];
      RequestOutcome& oc = rep.outcomes[k];
      oc.request_id = r.request_id;
      oc.model_id = catalog.lookup(r.language, r.task_class).model_id;
      oc.task_class = r.task_class;
      oc.cold_start = d.cold[o] != 0;
      oc.queue_wait_s = d.qw[o];
      oc.load_wait_s = d.lw[o];
      oc.prefill_s = d.pf[o];
      oc.decode_s = d.dc[o];
      oc.ttft_s = d.tt[o];
      oc.e2e_s = d.ee[o];
    }
  }
  return out;
}

SimulationReport run(const Trace& trace, const ModelCatalog& catalog, const ClusterConfig& cluster,
                     const Policy& policy) {
  return run_many({&trace}, catalog, {{policy.config(), cluster}}, {0}, false).front();
}

std::vector<RunMetrics> run_metrics_many(const std::vector<const Trace*>& traces,
                                         const ModelCatalog& catalog,
                                         const std::vector<std::pair<PolicyConfig, ClusterConfig>>& runs,
                                         const std::vector<int>& trace_of_run, bool parallel) {
  for (const auto& [pc, cc] : runs) {  // engine.cpp:79-82, in the reference's order
    if (pc.window_length < 1) throw SimError("run: window_length must be >= 1");
    if (cc.num_accelerators < 1) throw SimError("run: need at least one accelerator");
  }
  CatalogSoA cat(catalog);
  std::vector<TraceSoA> tsoa;
  std::vector<cace_trace_t> tabi;
  for (const Trace* t : traces) tsoa.emplace_back(*t, catalog);
  for (const auto& t : tsoa) tabi.push_back(t.abi());
  const int64_t S = static_cast<int64_t>(runs.size());
  std::vector<cace_scenario_t> sc;
  for (int64_t i = 0; i < S; ++i) sc.push_back(scenario(trace_of_run[i], runs[i].first, runs[i].second));
  std::vector<cace_run_metrics_t> m(S);
  // same device fan-out as run_many, cut by request count
  std::vector<int64_t> off(S + 1, 0);
  for (int64_t i = 0; i < S; ++i) off[i + 1] = off[i] + tabi[trace_of_run[i]].n_requests;
  const int nd = parallel ? std::max(1, std::min<int>(cace_device_count(), static_cast<int>(S))) : 1;
  std::vector<int64_t> cut(nd + 1, S);
  cut[0] = 0;
  for (int k = 1; k < nd; ++k)
    cut[k] = std::lower_bound(off.begin(), off.end() - 1, off[S] * k / nd) - off.begin();
  std::vector<int32_t> rcs(nd, CACE_OK);
  std::vector<std::string> errs(nd);
  auto part = [&](int k) {
    const int64_t b = cut[k], n = cut[k + 1] - cut[k];
    if (n == 0) return;
    cace_opts_t opts{k, CACE_KERNEL_AUTO, -1, 0, nullptr};
    char msg[512] = {0};
    rcs[k] = cace_run_metrics_batch(&cat.abi, tabi.data(), static_cast<int32_t>(tabi.size()), sc.data() + b, n,
                                    m.data() + b, nullptr, &opts, msg, sizeof msg);
    if (rcs[k] != CACE_OK) errs[k] = msg;
  };
  if (nd == 1) {
    part(0);
  } else {
    std::vector<std::thread> th;
    for (int k = 0; k < nd; ++k) th.emplace_back(part, k);
    for (auto& t : th) t.join();
  }
  for (int k = 0; k < nd; ++k)
    if (rcs[k] != CACE_OK) throw SimError(errs[k]);
  std::vector<RunMetrics> out(S);
  for (int64_t i = 0; i < S; ++i) {
    RunMetrics& r = out[i];
    r.cache_hit_rate = m[i].cache_hit_rate;
    r.load_overhead_s = m[i].load_overhead_s;
    r.evictions = m[i].evictions;
    const cace_latency_summary_t* src[2] = {&m[i].ttft_completion, &m[i].e2e_reasoning};
    LatencySummary* dst[2] = {&r.ttft_completion, &r.e2e_reasoning};
    for (int c = 0; c < 2; ++c) {
      dst[c]->count = static_cast<std::size_t>(src[c]->count);
      dst[c]->mean_s = src[c]->mean_s;
      dst[c]->p50_s = src[c]->p50_s;
      dst[c]->p95_s = src[c]->p95_s;
      dst[c]->p99_s = src[c]->p99_s;
      dst[c]->max_s = src[c]->max_s;
    }
  }
  return out;
}

GridResult run_grid_metrics(const ExperimentConfig& cfg, const ModelCatalog& catalog, bool parallel) {
  cfg.validate();
  std::vector<Trace> traces;
  std::vector<const Trace*> tp;
  for (PatternName p : cfg.patterns)
    for (std::uint64_t seed : cfg.seeds)
      traces.push_back(build_trace(p, cfg.rate, cfg.duration, seed, catalog, cfg.tokens, cfg.windows));
  for (const auto& t : traces) tp.push_back(&t);
  std::vector<std::pair<PolicyConfig, ClusterConfig>> runs;
  std::vector<int> tof;
  const int ns = static_cast<int>(cfg.seeds.size());
  for (size_t pi = 0; pi < cfg.patterns.size(); ++pi)
    for (Variant v : cfg.variants)
      for (int si = 0; si < ns; ++si) {
        runs.emplace_back(make_policy_config(cfg, v, catalog), cfg.cluster);
        tof.push_back(static_cast<int>(pi) * ns + si);
      }
  std::vector<RunMetrics> ms = run_metrics_many(tp, catalog, runs, tof, parallel);
  GridResult result;
  size_t r = 0;
  for (size_t pi = 0; pi < cfg.patterns.size(); ++pi)
    for (Variant v : cfg.variants) {
      GridCell cell;
      cell.pattern = cfg.patterns[pi];
      cell.variant = v;
      std::vector<RunMetrics> per_seed(ms.begin() + r, ms.begin() + r + ns);
      for (int si = 0; si < ns; ++si) {
        SimulationReport rep;
        const Trace& t = traces[pi * ns + si];
        rep.meta.variant = v;
        rep.meta.seed = t.seed;
        rep.meta.pattern = t.pattern;
        rep.meta.config_hash = config_hash(cfg.cluster, runs[r + si].first);
        cell.reports.push_back(std::move(rep));
      }
      r += ns;
      cell.averaged = average_metrics(per_seed);
      result.cells.push_back(std::move(cell));
    }
  return result;
}

GridResult run_grid(const ExperimentConfig& cfg, const ModelCatalog& catalog, bool parallel) {
  cfg.validate();
  // Traces per (pattern, seed), exactly as run_cell builds them (experiment.cpp:74-80).
  std::vector<Trace> traces;
  std::vector<const Trace*> tp;
  for (PatternName p : cfg.patterns)
    for (std::uint64_t seed : cfg.seeds)
      traces.push_back(build_trace(p, cfg.rate, cfg.duration, seed, catalog, cfg.tokens, cfg.windows));
  for (const auto& t : traces) tp.push_back(&t);
  std::vector<std::pair<PolicyConfig, ClusterConfig>> runs;
  std::vector<int> tof;
  const int ns = static_cast<int>(cfg.seeds.size());
  for (size_t pi = 0; pi < cfg.patterns.size(); ++pi)
    for (Variant v : cfg.variants)
      for (int si = 0; si < ns; ++si) {
        runs.emplace_back(make_policy_config(cfg, v, catalog), cfg.cluster);
        tof.push_back(static_cast<int>(pi) * ns + si);
      }
  std::vector<SimulationReport> reps = run_many(tp, catalog, runs, tof, parallel);
  GridResult result;
  size_t r = 0;
  for (PatternName p : cfg.patterns)
    for (Variant v : cfg.variants) {
      GridCell cell;
      cell.pattern = p;
      cell.variant = v;
      std::vector<RunMetrics> per_seed;
      for (int si = 0; si < ns; ++si) {
        per_seed.push_back(compute_run_metrics(reps[r]));
        cell.reports.push_back(std::move(reps[r]));
        ++r;
      }
      cell.averaged = average_metrics(per_seed);
      result.cells.push_back(std::move(cell));
    }
  return result;
}

}  // namespace cacesim::gpu
