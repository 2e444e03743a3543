/*
 * lpsim_oracle.h — plain, slow CPU oracle of LPSim's per-timestep vehicle update.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2406_08496_b200/) never links, imports or calls it,
 * and shares no code, header, table or constant generator with it.
 *
 * Paper: Jiang, Sengupta, Demmel, Williams, "Large Scale Multi-GPU Based
 * Parallel Traffic Simulation for Accelerated Traffic Assignment and
 * Propagation", arXiv 2406.08496.  Citations "P:Lnnn" are
 * PAPER.md lines; "Qnn" are the readings listed in DESIGN.md §3 (taken from
 * SURVEY.md §8(c)) where the paper is silent.
 *
 * Arithmetic: IEEE binary32 with a fixed operation order (the kernel's
 * precision — the paper does not fix one, and floating point here decides
 * integer state such as the cell index, so both sides decide in fp32).
 * Build with  -O2 -ffp-contract=off -fno-fast-math  (no FMA contraction).
 *
 * Parity status of each function: see the header comment of each function in
 * lpsim_oracle.c and DESIGN.md §4.  Whole-run outcomes on generated networks
 * are "parity unpinned w.r.t. the paper" (the paper prints no trajectories).
 */
#ifndef LPSIM_ORACLE_H
#define LPSIM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  float dt;            /* Δt [s] (Q1; the paper's "T, Timestep") */
  float a, b, s0, T;   /* IDM a, b, s0, desired headway T */
  int32_t delta;       /* IDM exponent δ, integer (Q6) */
  float x0;            /* mandatory-LC critical distance */
  float g_a, g_b;      /* desired lead / lag gap */
  float alpha_i, alpha_a, alpha_b; /* anticipation times */
  float sigma_a, sigma_b;          /* scale of ε_a, ε_b (Q15) */
  int32_t h_min;       /* probe floor H_min (Q7) */
  int32_t h_max;       /* probe cap; 0 -> ceil(2·Δt·max v0) + 2 */
  int32_t lc_window;   /* LC scan window n (Eq. Gap Acceptance, l_{i±n}); 0 -> h_max */
  float signal_cycle_s; /* Q30: 0 = unsignalised (Q18); > 0 = fixed-cycle two-phase signals */
  int32_t vfree;        /* ablation: literal "v <- v_free" (Alg. 1) when no leader (Q9 otherwise) */
  int32_t reserved;
  uint64_t seed;       /* Philox key (Q27) */
} lo_params;

typedef struct {
  int64_t step;            /* k: the snapshot currently held */
  int64_t waiting, on_road, finished;
  int64_t updates;         /* Σ on-road vehicles advanced (BASELINE.md metric unit) */
  int64_t departures, transitions, lane_changes, arrivals;
  int64_t lost_claims;     /* contenders that lost a same-cell claim (A9) */
  uint64_t digest;         /* order-independent digest of snapshot `step` */
} lo_stats;

enum { LO_WAITING = 0, LO_ON_ROAD = 1, LO_FINISHED = 2 };

typedef struct lo_sim lo_sim;

/* Defaults of SURVEY §8(c) (Q5): Δt .5, a 1.5, b 2, s0 2, T 1.5, δ 4, x0 100,
 * g 2, α .5, σ .5, H_min 2, seed 1. */
void lo_default_params(lo_params *p);

/* Returns NULL on invalid input and writes a message into err. */
lo_sim *lo_create(int32_t num_nodes, int32_t num_edges, const int64_t *row_ptr,
                  const int32_t *dst, const float *length_m, const uint8_t *lanes,
                  const float *speed_limit, const float *node_xy /* [2n] or NULL */, const lo_params *p,
                  char *err, int32_t errlen);
int32_t lo_load_demand(lo_sim *s, int64_t num_trips, const double *depart_s,
                       const int64_t *route_ptr, const int32_t *route_edges,
                       char *err, int32_t errlen);
/* Advance n steps.  Returns 0, or step+1 of the first invariant violation (negated). */
int64_t lo_step(lo_sim *s, int64_t n);
void lo_stats_get(const lo_sim *s, lo_stats *out);
int32_t lo_results(const lo_sim *s, int64_t n, int64_t *arrival_step,
                   double *arrival_time_s, double *distance_m);
/* Per-trip state of the current snapshot (cursor = index into the trip's route). */
/* t_start of every route entry (Alg. 1): out[route_ptr[i] + j] = the step of the
 * snapshot at which trip i is first on its route edge j (departure: j = 0), -1 if not (yet). */
int32_t lo_edge_entry(const lo_sim *s, int64_t r_total, int64_t *out);
int32_t lo_trip_state(const lo_sim *s, int64_t n, int32_t *status, int32_t *edge,
                      int32_t *lane, float *pos, float *v, int64_t *cursor);
/* Byte image of the current snapshot laid out edge by edge, lane by lane (a0). */
int64_t lo_lane_map_size(const lo_sim *s);
int32_t lo_lane_map_dump(const lo_sim *s, uint8_t *out, int64_t size);
int32_t lo_h_max(const lo_sim *s);
/* Test scaffolding: place the simulation at snapshot `step` with the given per-trip state (arrays of
 * num_trips as lo_trip_state / lo_results return them; arrival_step may be NULL).  Returns 0, or
 * 1 + the first offending trip. */
int32_t lo_set_state(lo_sim *s, int64_t step, int64_t n, const int32_t *status, const int32_t *edge,
                     const int32_t *lane, const float *pos, const float *v, const int64_t *cursor,
                     const int64_t *arrival_step);
/* Leader probe (a3) of an on-road trip on the current snapshot.
 * Returns 1 with *gap, *vf, *same_edge if a leader is seen, else 0; -1 if not on road. */
int32_t lo_probe_trip(const lo_sim *s, int64_t id, int32_t *gap, int32_t *vf, int32_t *same_edge);
void lo_destroy(lo_sim *s);

/* Pure helpers, exported for the pin tests. */
void lo_lane_map_layout(int32_t num_edges, const uint8_t *lanes, const float *length_m,
                        uint64_t *base_out, uint64_t *total_out);
float lo_idm_accel(const lo_params *p, float v, float v0, int32_t has_leader, int32_t s, int32_t vf);
void lo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
float lo_u24(uint64_t seed, uint32_t id, uint32_t k, uint32_t stream);
float lo_eps(uint64_t seed, uint32_t id, uint32_t k, uint32_t stream, float sigma);
int64_t lo_depart_step(double depart_s, float dt);

#ifdef __cplusplus
}
#endif
#endif
