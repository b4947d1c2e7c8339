// Plain data structures shared by the replay kernels, the host-side trace
// layout (layout.hpp) and the test-only host emulation build.
#pragma once
#include <stdint.h>

#include "../../include/cace_gpu.h"

namespace cace {

enum : int { ST_IDLE = 0, ST_BUSY = 1, ST_LOADING = 2 };

// One request in replay (sorted) order, 48 B (three 16-B cp.async chunks).
// The first 32 B are what a replay step reads; `nxa` feeds the lookahead
// window (arrival time of the next request for the same model).
struct alignas(16) ReqRec {
  double arrival;  // Request::arrival_time_s
  double prefill;  // service_times(): prompt / prefill_rate   (engine.cpp:21-22)
  double decode;   // service_times(): max(out,1) / decode_rate (engine.cpp:23-24)
  uint32_t nxt;    // next sorted index with the same model (n if none)
  uint32_t mc;     // model | task_class << 16
  double nxa;      // arrival of request nxt (+inf if none)
  uint32_t ci;     // index among the trace's requests of the same task class (replay order)
  uint32_t prv;    // previous sorted index with the same model (0xffffffff if none)
};
static_assert(sizeof(ReqRec) == 48, "ReqRec layout");

struct DevCatalog {
  int M;
  const double* load_time;  // [M] ModelDescriptor::load_time_s
  const double* p2;         // [M] 1 / (1 + load_time / 100)  (policy.cpp:55)
  const double* tokens;     // [M] (double) expected_output_tokens
  const int* lex;           // [M] rank of model_id under std::string <
};

struct DumpDev {
  const int32_t* slot;  // [n_scenarios] dump slot or -1; NULL = no dump
  const int64_t* dump_off;  // [n_dump] offset of slot's per-request block
  uint8_t* cold;
  double *queue_wait, *load_wait, *prefill, *decode, *ttft, *e2e;
  int64_t evict_cap;
  int32_t* evict_model;
  double* evict_clock;
  int64_t* n_evict;
  // metrics samples: per dumped scenario, TTFT of its completion requests
  // then E2E of its reasoning requests, each in replay order, from dump_off
  double* samples;
};

struct ReplayParams {
  const ReqRec* rec;        // all traces, concatenated, sorted order
  const int64_t* trace_off; // [T+1]
  const uint32_t* first0;   // [T][M] first sorted index of each model
  const uint32_t* perm;     // sorted index -> caller's request index
  const uint32_t* trace_ncomp;  // [T] completion-class requests per trace
  DevCatalog cat;
  const double* log_tab;
  const double* log_tab2;
  int log_variant;
  const cace_scenario_t* scen;
  const int64_t* order;     // plan: scenario indices grouped by capacity
  int64_t seg_begin, seg_end;
  cace_summary_t* out;
  DumpDev dump;
};

}  // namespace cace
