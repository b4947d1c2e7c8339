// Drop-in check of the reference-side binding (cacesim_gpu.cpp): the
// reference's own run()/run_grid() vs cacesim::gpu::run()/run_grid() on the
// reference's own fixtures, compared on the reference's own serialisations
// (serialize_report, emit_metrics_csv, emit(compare(...))) — byte for byte,
// the acceptance criterion 9 standard (acceptance.cpp:452-470).
// Runs on a GPU box; prints one ADAPTER line per check, exits 1 on mismatch.
#include <cmath>
#include <cstdio>
#include <string>

#include "cacesim/experiment.hpp"
#include "cacesim/metrics.hpp"
#include "cacesim_gpu.hpp"

using namespace cacesim;

static int fails = 0;

static void check(bool ok, const std::string& what) {
  std::printf("ADAPTER %s %s\n", ok ? "OK" : "FAIL", what.c_str());
  if (!ok) ++fails;
}

static std::string render(const GridResult& g) {
  std::string blob = emit_metrics_csv(g.rows());
  blob += emit(compare(g.rows(), std::string(to_string(g.cells.front().variant))), EmitFormat::Json);
  for (const auto& c : g.cells)
    for (const auto& r : c.reports) blob += serialize_report(r);
  return blob;
}

int main() {
  const ModelCatalog catalog = ModelCatalog::build_default();
  // acceptance.cpp:33-57 fixtures
  ExperimentConfig cmp;
  cmp.variants = {Variant::Lru, Variant::CaceMinusP4, Variant::CaceFull};
  cmp.rate = 15.0;
  cmp.duration = 30.0;
  cmp.w1 = 0.5;
  cmp.window_length = 10;
  ExperimentConfig abl;
  abl.patterns = {PatternName::PopularitySkewed};
  abl.variants = {Variant::CaceFull, Variant::CaceMinusP1, Variant::CaceMinusP2,
                  Variant::CaceMinusP3, Variant::CaceMinusP4};
  abl.rate = 4.0;
  abl.duration = 30.0;
  abl.w1 = 1.0;
  abl.window_length = 2;
  ExperimentConfig all;  // every variant, 8 seeds (bench_grid.cpp:31-36)
  all.variants = {Variant::Lru, Variant::CaceFull, Variant::CaceMinusP1, Variant::CaceMinusP2,
                  Variant::CaceMinusP3, Variant::CaceMinusP4};
  all.seeds = {1, 2, 3, 4, 5, 6, 7, 8};
  all.cluster.num_accelerators = 3;
  all.cluster.unload_time_s = 0.75;
  all.p1_mode = P1Mode::Verbatim;
  for (auto* cfg : {&cmp, &abl, &all}) {
    const GridResult want = run_grid(*cfg, catalog, false);
    const GridResult got = gpu::run_grid(*cfg, catalog, true);
    const GridResult got_serial = gpu::run_grid(*cfg, catalog, false);
    check(render(got) == render(got_serial), "run_grid parallel == serial (all visible devices vs device 0)");
    const std::string a = render(want), b = render(got);
    check(a == b, "run_grid byte-identical (" + std::to_string(a.size()) + " bytes, " +
                      std::to_string(cfg->patterns.size() * cfg->variants.size() * cfg->seeds.size()) +
                      " runs)");
  }
  // device RunMetrics (run_metrics_many / run_grid_metrics) vs the reference's
  // compute_run_metrics / average_metrics: exact except the mean (sorted-order
  // sum in the reference, replay-order sum on the device)
  for (auto* cfg : {&cmp, &all}) {
    const GridResult want = run_grid(*cfg, catalog, false);
    const GridResult got = gpu::run_grid_metrics(*cfg, catalog);
    bool ok = want.cells.size() == got.cells.size();
    double worst = 0.0;
    for (size_t c = 0; ok && c < want.cells.size(); ++c) {
      const RunMetrics &a = want.cells[c].averaged, &b = got.cells[c].averaged;
      ok = ok && a.cache_hit_rate == b.cache_hit_rate && a.load_overhead_s == b.load_overhead_s &&
           a.evictions == b.evictions;
      for (auto mem : {&RunMetrics::ttft_completion, &RunMetrics::e2e_reasoning}) {
        const LatencySummary &x = a.*mem, &y = b.*mem;
        ok = ok && x.count == y.count && x.p50_s == y.p50_s && x.p95_s == y.p95_s &&
             x.p99_s == y.p99_s && x.max_s == y.max_s;
        worst = std::max(worst, std::abs(x.mean_s - y.mean_s) / std::max(std::abs(x.mean_s), 1e-300));
      }
    }
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.2e", worst);
    check(ok && worst <= 1e-12, std::string("run_grid_metrics: averaged metrics exact (mean rel diff ") + buf +
                                    ", " + std::to_string(want.cells.size()) + " cells)");
  }
  // criterion 2 number through the GPU grid
  {
    const GridResult g = gpu::run_grid(cmp, catalog);
    double best = 1e9;
    for (PatternName p : {PatternName::Uniform, PatternName::IdeHeavy, PatternName::PopularitySkewed})
      best = std::min(best, g.cell(p, Variant::CaceFull).averaged.evictions /
                                g.cell(p, Variant::Lru).averaged.evictions);
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.6g", best);
    check(std::string(buf) == "0.785513", std::string("criterion 2 ratio via GPU = ") + buf);
  }
  // single runs, engine.hpp:60 signature
  for (std::uint64_t seed = 1; seed <= 6; ++seed) {
    Trace t = build_trace(static_cast<PatternName>(seed % 3), 12.0, 20.0, seed, catalog);
    PolicyConfig pc;
    pc.variant = static_cast<Variant>(seed % 6);
    pc.window_length = static_cast<int>(1 + seed * 3);
    pc.w1 = 0.25 * static_cast<double>(seed);
    ClusterConfig cc;
    cc.num_accelerators = static_cast<int>(1 + seed % 5);
    const Policy pol = make_policy(pc);
    const std::string a = serialize_report(run(t, catalog, cc, pol));
    const std::string b = serialize_report(gpu::run(t, catalog, cc, pol));
    check(a == b, "run() report byte-identical, seed " + std::to_string(seed));
  }
  // SimError behaviour (engine.cpp:79-82)
  {
    Trace t = build_trace(PatternName::Uniform, 5.0, 5.0, 1, catalog);
    PolicyConfig pc;
    pc.window_length = 0;
    std::string ea, eb;
    try { run(t, catalog, ClusterConfig{}, make_policy(pc)); } catch (const SimError& e) { ea = e.what(); }
    try { gpu::run(t, catalog, ClusterConfig{}, make_policy(pc)); } catch (const SimError& e) { eb = e.what(); }
    check(!ea.empty() && ea == eb, "SimError text identical: " + eb);
  }
  std::printf("ADAPTER %s\n", fails ? "FAILED" : "ALL_OK");
  return fails ? 1 : 0;
}
