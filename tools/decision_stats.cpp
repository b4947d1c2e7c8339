// TEST/ANALYSIS-ONLY: per-request decision statistics of the lane replay,
// from the host emulation (tests/emul/replay_emul.cpp) with the CACE_STAT
// hook bound to a per-scenario bitmap.  Used by tools/decision_stats.py to
// measure how many lanes of a warp take each branch of the replay loop.
#include <cstdint>
#include <vector>
static uint8_t* g_bits = nullptr;  // [6][n] bytes for the scenario being replayed
static int64_t g_n = 0;
#define CACE_STAT(kind, k) (g_bits ? (void)(g_bits[(int64_t)(kind) * g_n + (k)] = 1) : (void)0)
#include "../tests/emul/replay_emul.cpp"

extern "C" int32_t stats_replay(const cace_catalog_t* catalog, const cace_trace_t* trace,
                                const cace_scenario_t* sc, int64_t n_sc, uint8_t* bits) {
  g_n = trace->n_requests;
  std::vector<cace_summary_t> out(1);
  for (int64_t i = 0; i < n_sc; ++i) {
    g_bits = bits + i * 6 * g_n;
    const int32_t rc = emul_replay_batch(catalog, trace, 1, sc + i, 1, out.data(), 0, nullptr, nullptr, nullptr,
                                         nullptr, nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr, 1, 0);
    if (rc) return rc;
  }
  g_bits = nullptr;
  return 0;
}
