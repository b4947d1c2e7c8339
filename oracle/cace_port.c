/* TEST INFRASTRUCTURE ONLY — see cace_port.h.
 *
 * A direct restatement of the reference's discrete-event replay: the same
 * min-heap of (time, kind, seq) events (engine.cpp:35-55), the same pending
 * FIFO and head-of-line dispatch (engine.cpp:157-210), the same residency
 * state machine (engine.cpp:57-62, 219-230), dedup_window / eviction_score /
 * select_victim (policy.cpp:22-115) with the model_id tie-break replaced by
 * lex_rank (the rank of model_id under std::string operator<).  Deliberately
 * NOT the GPU engine's event algebra (no lazy arrivals, no incremental
 * window) so it is an independent cross-check.  Built -ffp-contract=off: every
 * fp64 operation rounds separately, in the reference's order; P1 calls this
 * host's libm log exactly as policy.cpp:51 does. */
#include "cace_port.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

enum { ABSENT = 0, LOADING = 1, IDLE = 2, BUSY = 3 };
enum { EV_LOAD = 0, EV_SERVICE = 1, EV_ARRIVAL = 2 };

typedef struct {
  double t;
  int kind;
  uint64_t seq;
  int64_t req;
  int32_t model;
} Event;

typedef struct {
  Event* a;
  int64_t n, cap;
} Heap;

static int ev_after(const Event* x, const Event* y) { /* EventAfter, engine.cpp:49-55 */
  if (x->t != y->t) return x->t > y->t;
  if (x->kind != y->kind) return x->kind > y->kind;
  return x->seq > y->seq;
}

static void heap_push(Heap* h, Event e) {
  if (h->n == h->cap) {
    h->cap = h->cap ? h->cap * 2 : 64;
    h->a = (Event*)realloc(h->a, (size_t)h->cap * sizeof(Event));
  }
  int64_t i = h->n++;
  h->a[i] = e;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!ev_after(&h->a[p], &h->a[i])) break;
    Event t = h->a[p];
    h->a[p] = h->a[i];
    h->a[i] = t;
    i = p;
  }
}

static Event heap_pop(Heap* h) {
  Event top = h->a[0];
  h->a[0] = h->a[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && ev_after(&h->a[m], &h->a[l])) m = l;
    if (r < h->n && ev_after(&h->a[m], &h->a[r])) m = r;
    if (m == i) break;
    Event t = h->a[m];
    h->a[m] = h->a[i];
    h->a[i] = t;
    i = m;
  }
  return top;
}

static inline uint64_t mix(uint64_t h, uint64_t x) {
  /* CACE_HASH, include/cace_gpu.h */
  const uint32_t lo = (uint32_t)h * 0x9e3779b1u + (uint32_t)x;
  const uint32_t hi = (uint32_t)(h >> 32) * 0x85ebca77u + (uint32_t)(x >> 32);
  return ((uint64_t)hi << 32) | lo;
}
static inline uint64_t bits(double d) {
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
}

static void put(char* msg, size_t cap, const char* s) {
  if (msg && cap) {
    strncpy(msg, s, cap - 1);
    msg[cap - 1] = 0;
  }
}

int32_t port_run(const port_catalog_t* cat, const double* arrival, const int32_t* model,
                 const int32_t* prompt, const int32_t* output, int64_t n,
                 const port_scenario_t* sc, port_summary_t* S, uint8_t* cold_out,
                 double* queue_wait, double* load_wait_out, double* prefill_out,
                 double* decode_out, double* ttft_out, double* e2e_out, int32_t* evict_model,
                 double* evict_clock, int64_t evict_cap, int64_t* n_evict, char* msg,
                 size_t msg_cap) {
  memset(S, 0, sizeof(*S));
  S->eviction_hash = S->outcome_hash = 0x6a09e667f3bcc909ULL;
  if (n_evict) *n_evict = 0;
  const int w = sc->window_length;
  if (w < 1) { put(msg, msg_cap, "run: window_length must be >= 1"); return S->status = 1; }
  if (sc->num_accelerators < 1) { put(msg, msg_cap, "run: need at least one accelerator"); return S->status = 2; }
  const int capacity = sc->num_accelerators * sc->models_per_accelerator;
  const int M = cat->n_models;
  for (int64_t i = 0; i < n; ++i)
    if (model[i] < 0 || model[i] >= M) { put(msg, msg_cap, "catalog: no model registered"); return S->status = 3; }

  int32_t* state = (int32_t*)calloc((size_t)M, sizeof(int32_t));
  double* last_used = (double*)calloc((size_t)M, sizeof(double));
  int64_t* pending = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  char* classified = (char*)calloc((size_t)(n > 0 ? n : 1), 1);
  double* lw = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  uint8_t* cold = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  double* tt = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double* ee = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  int64_t* served_order = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  int32_t* win = (int32_t*)malloc((size_t)(w < M ? w : M) * sizeof(int32_t) + 4);
  int32_t* win_pos = (int32_t*)malloc((size_t)M * sizeof(int32_t));
  int32_t* idle = (int32_t*)malloc((size_t)M * sizeof(int32_t));
  for (int m = 0; m < M; ++m) win_pos[m] = -1;
  int64_t ph = 0, pt = 0, served = 0;
  int resident = 0;
  uint64_t seq = 0;
  int32_t status = 0;
  Heap H = {0, 0, 0};
  for (int64_t i = 0; i < n; ++i) heap_push(&H, (Event){arrival[i], EV_ARRIVAL, seq++, i, -1});

  while (H.n > 0 && status == 0) {
    Event ev = heap_pop(&H);
    if (ev.kind == EV_ARRIVAL) {
      pending[pt++] = ev.req;
    } else {
      state[ev.model] = IDLE; /* engine.cpp:219-230 */
      last_used[ev.model] = ev.t;
    }
    const double now = ev.t;
    /* dispatch (engine.cpp:157-210) */
    while (ph < pt && status == 0) {
      const int64_t req = pending[ph];
      const int m = model[req];
      if (!classified[req]) {
        classified[req] = 1;
        if (state[m] != ABSENT && state[m] != LOADING) {
          S->hits++;
        } else {
          S->misses++;
          cold[req] = 1;
        }
      }
      if (state[m] != ABSENT) {
        if (state[m] == IDLE) {
          ph++;
          /* start_service (engine.cpp:134-153) + service_times (15-26) */
          if (cat->prefill_rate_tps[m] <= 0 || cat->decode_rate_tps[m] <= 0) {
            put(msg, msg_cap, "service_times: rates must be positive");
            status = 4 | (m << 8);
            break;
          }
          const double prefill = (double)prompt[req] / cat->prefill_rate_tps[m];
          const double decode = (double)(output[req] > 1 ? output[req] : 1) / cat->decode_rate_tps[m];
          state[m] = BUSY;
          const double qw = (now - arrival[req]) - lw[req];
          const double ttft = (now - arrival[req]) + prefill;
          const double e2e = ttft + decode;
          if (queue_wait) queue_wait[req] = qw;
          if (prefill_out) prefill_out[req] = prefill;
          if (decode_out) decode_out[req] = decode;
          tt[req] = ttft;
          ee[req] = e2e;
          served_order[served++] = req;
          heap_push(&H, (Event){now + prefill + decode, EV_SERVICE, seq++, req, m});
          continue;
        }
        break; /* busy or loading */
      }
      double unload = 0.0;
      if (resident < capacity) {
        /* free slot (engine.cpp:184-187) */
      } else {
        /* window (engine.cpp:189-195) + dedup_window (policy.cpp:22-37) */
        const int64_t lim = (pt - ph) < (int64_t)w ? (pt - ph) : (int64_t)w;
        int nwin = 0;
        for (int64_t k = 0; k < lim; ++k) {
          const int mm = model[pending[ph + k]];
          if (win_pos[mm] < 0) {
            win_pos[mm] = nwin;
            win[nwin++] = mm;
          }
        }
        /* idle residents sorted by (last_used, lex) (policy.cpp:85-98) */
        int ni = 0;
        for (int mm = 0; mm < M; ++mm)
          if (state[mm] == IDLE) idle[ni++] = mm;
        for (int a = 1; a < ni; ++a) { /* insertion sort */
          const int x = idle[a];
          int b = a - 1;
          while (b >= 0 && (last_used[x] < last_used[idle[b]] ||
                            (!(last_used[idle[b]] < last_used[x]) &&
                             cat->lex_rank[x] < cat->lex_rank[idle[b]]))) {
            idle[b + 1] = idle[b];
            --b;
          }
          idle[b + 1] = x;
        }
        int victim = -1;
        if (ni > 0) {
          if (sc->variant == 0) {
            victim = idle[0];
          } else {
            double best_total = 0.0;
            for (int k = 0; k < ni; ++k) {
              const int e = idle[k];
              if (now < last_used[e]) { /* policy.cpp:43-46 */
                put(msg, msg_cap, "eviction_score: clock precedes last_used_s");
                status = 5 | (e << 8);
                break;
              }
              const double d = now - last_used[e];
              const double t = d < 1.0 ? 1.0 : d;
              const double p1v = 1.0 / (1.0 + log(t));
              double p1 = sc->p1_mode == 1 ? p1v : 1.0 - p1v;
              double p2 = 1.0 / (1.0 + cat->load_time_s[e] / 100.0);
              double p3 = win_pos[e] < 0 ? 1.0 : (double)win_pos[e] / (double)w;
              double p4 = sc->w1 * ((double)cat->expected_output_tokens[e] /
                                    (double)sc->output_token_normalizer);
              switch (sc->variant) {
                case 2: p1 = 0.0; break;
                case 3: p2 = 0.0; break;
                case 4: p3 = 0.0; break;
                case 5: p4 = 0.0; break;
                default: break;
              }
              const double total = p1 + p2 + p3 + p4;
              if (victim < 0 || total > best_total) {
                victim = e;
                best_total = total;
              }
            }
          }
        }
        for (int k = 0; k < nwin; ++k) win_pos[win[k]] = -1;
        if (status) break;
        if (victim < 0) break; /* all busy (engine.cpp:203) */
        state[victim] = ABSENT;
        resident--;
        if (evict_model && S->evictions < (uint64_t)evict_cap) evict_model[S->evictions] = victim;
        if (evict_clock && S->evictions < (uint64_t)evict_cap) evict_clock[S->evictions] = now;
        S->eviction_hash = mix(S->eviction_hash, bits(now) ^ ((uint64_t)victim << 32));
        S->evictions++;
        unload = sc->unload_time_s;
      }
      /* start_load (engine.cpp:123-132) */
      state[m] = LOADING;
      last_used[m] = now;
      resident++;
      if (resident > S->max_resident) S->max_resident = resident;
      const double ready = now + unload + cat->load_time_s[m];
      lw[req] = ready - now;
      S->load_overhead_s += cat->load_time_s[m];
      S->loads++;
      heap_push(&H, (Event){ready, EV_LOAD, seq++, req, m});
      break;
    }
  }
  if (status == 0 && (ph < pt || served != n)) {
    put(msg, msg_cap, "run: deadlock");
    status = 6;
  }
  if (status == 0) {
    for (int64_t k = 0; k < served; ++k) {
      const int64_t r = served_order[k];
      if (cat->task_class[model[r]] == 0) {
        S->n_completion++;
        S->sum_ttft_completion += tt[r];
        if (tt[r] > S->max_ttft_completion) S->max_ttft_completion = tt[r];
      } else {
        S->n_reasoning++;
        S->sum_e2e_reasoning += ee[r];
        if (ee[r] > S->max_e2e_reasoning) S->max_e2e_reasoning = ee[r];
      }
      S->outcome_hash = mix(S->outcome_hash, bits(tt[r]) ^ (uint64_t)cold[r]);
    }
    for (int64_t i = 0; i < n; ++i) {
      if (cold_out) cold_out[i] = cold[i];
      if (load_wait_out) load_wait_out[i] = lw[i];
      if (ttft_out) ttft_out[i] = tt[i];
      if (e2e_out) e2e_out[i] = ee[i];
    }
    if (n_evict) *n_evict = (int64_t)S->evictions;
  }
  S->status = status;
  free(H.a);
  free(state); free(last_used); free(pending); free(classified); free(lw); free(cold);
  free(tt); free(ee); free(served_order); free(win); free(win_pos); free(idle);
  return status;
}

typedef struct {
  const port_catalog_t* cat;
  const double* arrival;
  const int32_t *model, *prompt, *output;
  const int64_t* offsets;
  const port_scenario_t* sc;
  int64_t n;
  port_summary_t* out;
  int64_t next;
  pthread_mutex_t mu;
} Batch;

static void* worker(void* p) {
  Batch* b = (Batch*)p;
  for (;;) {
    pthread_mutex_lock(&b->mu);
    const int64_t i = b->next++;
    pthread_mutex_unlock(&b->mu);
    if (i >= b->n) break;
    const port_scenario_t* s = &b->sc[i];
    const int64_t o = b->offsets[s->trace], len = b->offsets[s->trace + 1] - o;
    char msg[128];
    port_run(b->cat, b->arrival + o, b->model + o, b->prompt + o, b->output + o, len, s, &b->out[i], 0, 0,
             0, 0, 0, 0, 0, 0, 0, 0, 0, msg, sizeof msg);
  }
  return 0;
}

int32_t port_run_batch(const port_catalog_t* cat, const double* arrival, const int32_t* model,
                       const int32_t* prompt, const int32_t* output, const int64_t* offsets,
                       int32_t n_traces, const port_scenario_t* sc, int64_t n_scenarios,
                       int32_t threads, port_summary_t* out, double* seconds) {
  (void)n_traces;
  Batch b = {cat, arrival, model, prompt, output, offsets, sc, n_scenarios, out, 0};
  pthread_mutex_init(&b.mu, 0);
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int k = 0; k < threads; ++k) pthread_create(&th[k], 0, worker, &b);
  for (int k = 0; k < threads; ++k) pthread_join(th[k], 0);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  if (seconds) *seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  free(th);
  pthread_mutex_destroy(&b.mu);
  for (int64_t i = 0; i < n_scenarios; ++i)
    if (out[i].status) return out[i].status & 0xff;
  return 0;
}
