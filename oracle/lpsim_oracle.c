/*
 * lpsim_oracle.c — plain, slow, single-threaded CPU oracle of LPSim's
 * per-timestep microscopic vehicle update (arXiv 2406.08496).
 *
 * TEST INFRASTRUCTURE ONLY (see lpsim_oracle.h).  It shares no code with the
 * CUDA path: its data structures are deliberately different (per-edge lane
 * arrays, array-of-structs trips, every trip visited every step, claims
 * resolved by sorting (cell, id)).
 *
 * The simulation is an iteration, so this file follows the paper's algorithm
 * step by step: Eq. (1) P:L239-242 (every state at k+1 is a function of the
 * snapshot at k only), Alg. 1 "Vehicle Propagation Algorithm" P:L298-336,
 * the lane-map encoding P:L256-266 and the Remarks P:L247-251, with the
 * readings Q1-Q29 of DESIGN.md §3 where the paper is silent.  Each function
 * names the passage it follows.
 *
 * Compile: gcc -std=c11 -O2 -ffp-contract=off -fno-fast-math -fPIC -shared
 */
#include "lpsim_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* Random numbers: Philox4x32-10 (Salmon et al., SC'11 / Random123).  Q27.   */
/* Pinned by the published Random123 known-answer vectors (tests).           */
/* ------------------------------------------------------------------------- */
void lo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void philox_words(uint64_t seed, uint32_t id, uint32_t k, uint32_t stream, uint32_t w[4]) {
  /* Q27: key = (seed_lo, seed_hi), counter = (id, k, stream, 0). */
  uint32_t ctr[4] = {id, k, stream, 0u};
  uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
  lo_philox4x32_10(ctr, key, w);
}

/* Q27: u = (x0 >> 8) · 2^-24, uniform on [0,1) with 24 exact bits. */
float lo_u24(uint64_t seed, uint32_t id, uint32_t k, uint32_t stream) {
  uint32_t w[4];
  philox_words(seed, id, k, stream, w);
  return (float)(w[0] >> 8) * 0x1p-24f;
}

/* Q15: ε = σ·√3·(Σ_{j<4} u22_j − 2), Irwin–Hall(4) approximate normal with
 * variance σ² (4 · 1/12 · 3 = 1).  The integer sum is < 2^24, so the float
 * conversion and the shift by 2 are exact; one rounding in the final product. */
float lo_eps(uint64_t seed, uint32_t id, uint32_t k, uint32_t stream, float sigma) {
  uint32_t w[4];
  philox_words(seed, id, k, stream, w);
  uint32_t sum = (w[0] >> 10) + (w[1] >> 10) + (w[2] >> 10) + (w[3] >> 10);
  float scale = sigma * sqrtf(3.0f);
  return ((float)sum * 0x1p-22f - 2.0f) * scale;
}

/* Q22: depart_step = smallest k with k·Δt ≥ depart_s ("Current Time < t_depart
 * → Wait", Alg. 1 line 2), evaluated in double. */
int64_t lo_depart_step(double depart_s, float dt) {
  double h = (double)dt;
  int64_t k = (int64_t)ceil(depart_s / h);
  if (k < 0) k = 0;
  while (k > 0 && (double)(k - 1) * h >= depart_s) --k;
  while ((double)k * h < depart_s) ++k;
  return k;
}

/* ------------------------------------------------------------------------- */
/* a0  Lane map layout (Fig. "Data Movement" P:L275-280):        */
/* "1 Byte in Memory = 1 Meter", lanes of an edge "in order", the whole      */
/* network one 1-D array; a 4-lane 8 m edge is 1 x 32.  Lc = ceil(length)   */
/* (Q29).  base[e] = Σ_{e'<e} lanes[e']·Lc(e').                               */
/* Pinned: paper's 4x8 -> 32 example; SPEC offsets example; bijectivity.     */
/* ------------------------------------------------------------------------- */
static int32_t cells_of(float length_m) { return (int32_t)ceilf(length_m); }

void lo_lane_map_layout(int32_t num_edges, const uint8_t *lanes, const float *length_m,
                        uint64_t *base_out, uint64_t *total_out) {
  uint64_t acc = 0;
  for (int32_t e = 0; e < num_edges; ++e) {
    if (base_out) base_out[e] = acc;
    acc += (uint64_t)lanes[e] * (uint64_t)cells_of(length_m[e]);
  }
  if (total_out) *total_out = acc;
}

/* ------------------------------------------------------------------------- */
/* a4  IDM acceleration, Eq. (Car Following) P:L218-220, parameters         */
/* (a, δ, b, s0, T) P:L195-203 / P:L302.  Standard IDM (Q3):                 */
/*   a [ 1 − (v/v0)^δ − (s_star / s)² ],  s_star = s0 + max(0, vT + vΔv/(2√(ab)))      */
/* Δv = v − v_f (Q4); free road (no leader within d_front): a[1 − (v/v0)^δ]  */
/* (Q9).  Fixed fp32 operation order.                         */
/* Pinned: free-road at v0 -> 0, standing start -> a, equilibrium gap.       */
/* ------------------------------------------------------------------------- */
static float pow_int(float r, int32_t d) {
  /* exponentiation by squaring, LSB first (δ = 4 gives (r·r)·(r·r)) */
  float result = 1.0f, base = r;
  while (d > 0) {
    if (d & 1) result = result * base;
    base = base * base;
    d >>= 1;
  }
  return result;
}

float lo_idm_accel(const lo_params *p, float v, float v0, int32_t has_leader, int32_t s, int32_t vf) {
  float r = v / v0;
  float rd = pow_int(r, p->delta);
  if (!has_leader) return p->a * (1.0f - rd);
  float c_ab = 2.0f * sqrtf(p->a * p->b);
  float dv = v - (float)vf;
  float t = v * p->T + (v * dv) / c_ab;
  t = fmaxf(0.0f, t);
  float ss = p->s0 + t;
  float q = ss / (float)s;
  return p->a * ((1.0f - rd) - q * q);
}

void lo_default_params(lo_params *p) {
  memset(p, 0, sizeof(*p));
  p->dt = 0.5f;
  p->a = 1.5f; p->b = 2.0f; p->s0 = 2.0f; p->T = 1.5f; p->delta = 4;
  p->x0 = 100.0f;
  p->g_a = 2.0f; p->g_b = 2.0f;
  p->alpha_i = 0.5f; p->alpha_a = 0.5f; p->alpha_b = 0.5f;
  p->sigma_a = 0.5f; p->sigma_b = 0.5f;
  p->h_min = 2; p->h_max = 0; p->lc_window = 0;
  p->seed = 1;
}

/* ------------------------------------------------------------------------- */
/* Simulator state                                                            */
/* ------------------------------------------------------------------------- */
typedef struct {
  int32_t status;   /* LO_WAITING / LO_ON_ROAD / LO_FINISHED */
  int32_t edge, lane;
  float pos, v;
  int64_t j;        /* index of the current edge within the trip's route */
} trip_state;

typedef struct {   /* a same-cell claim (Remark "Switch"; A9) */
  int32_t edge, lane, cell;
  int64_t id;
} claim;

struct lo_sim {
  lo_params p;
  int32_t n_nodes, n_edges;
  int64_t *row_ptr;
  int32_t *src, *dst, *ncells, *lanes;
  float *length, *v0;
  int32_t h_max, lc_n;
  /* Q30 signals: cycle in steps (0 = none), per edge: ends at a signalised node, approach phase */
  int32_t sig_cycle;
  uint8_t *sig, *sig_phase;
  /* lane maps: map[b][e] is an array of lanes[e]*ncells[e] bytes */
  uint8_t **map[2];
  int cur;                       /* map[cur] is M_k */
  /* bytes written into each map: list of (edge, index) so the map can be reset */
  int64_t *wr_e[2], *wr_i[2], wr_n[2];
  /* demand */
  int64_t n_trips;
  int64_t *route_ptr;
  int32_t *route;
  int64_t *depart_step, *arrival_step;
  /* t_start of every route edge (Alg. 1 "If Moving on a New Edge ... t_start <- Current Time",
   * P:L305-307): the step of the snapshot at which the trip is first on route edge j, -1 before */
  int64_t *edge_entry;
  trip_state *st, *nx;
  claim *claims;
  trip_state *proposal;
  int64_t step;
  lo_stats stats;
  int loaded;
};

static void set_err(char *err, int32_t errlen, const char *msg, long long idx) {
  if (err && errlen > 0) snprintf(err, (size_t)errlen, "%s (index %lld)", msg, idx);
}

lo_sim *lo_create(int32_t num_nodes, int32_t num_edges, const int64_t *row_ptr,
                  const int32_t *dst, const float *length_m, const uint8_t *lanes,
                  const float *speed_limit, const float *node_xy, const lo_params *p, char *err, int32_t errlen) {
  if (num_nodes <= 0 || num_edges < 0 || !row_ptr || (num_edges > 0 && (!dst || !length_m || !lanes || !speed_limit)) || !p) {
    set_err(err, errlen, "null or negative argument", -1);
    return NULL;
  }
  if (row_ptr[0] != 0 || row_ptr[num_nodes] != num_edges) { set_err(err, errlen, "row_ptr bounds", 0); return NULL; }
  for (int32_t u = 0; u < num_nodes; ++u)
    if (row_ptr[u + 1] < row_ptr[u]) { set_err(err, errlen, "row_ptr not monotone", u); return NULL; }
  for (int32_t e = 0; e < num_edges; ++e) {
    if (dst[e] < 0 || dst[e] >= num_nodes) { set_err(err, errlen, "dst out of range", e); return NULL; }
    if (!(length_m[e] >= 1.0f) || !isfinite(length_m[e])) { set_err(err, errlen, "length_m < 1", e); return NULL; }
    if (lanes[e] < 1) { set_err(err, errlen, "lanes < 1", e); return NULL; }
    if (!(speed_limit[e] > 0.0f && speed_limit[e] <= 254.0f)) { set_err(err, errlen, "speed limit not in (0,254]", e); return NULL; }
  }
  if (p->dt <= 0.0f || p->a <= 0.0f || p->b <= 0.0f || p->delta < 1 || p->h_min < 1 || p->x0 <= 0.0f) {
    set_err(err, errlen, "invalid parameters", -1);
    return NULL;
  }
  lo_sim *s = (lo_sim *)calloc(1, sizeof(lo_sim));
  s->p = *p;
  s->n_nodes = num_nodes;
  s->n_edges = num_edges;
  s->row_ptr = (int64_t *)malloc(sizeof(int64_t) * (size_t)(num_nodes + 1));
  memcpy(s->row_ptr, row_ptr, sizeof(int64_t) * (size_t)(num_nodes + 1));
  size_t E = (size_t)(num_edges > 0 ? num_edges : 1);
  s->src = (int32_t *)malloc(sizeof(int32_t) * E);
  s->dst = (int32_t *)malloc(sizeof(int32_t) * E);
  s->ncells = (int32_t *)malloc(sizeof(int32_t) * E);
  s->lanes = (int32_t *)malloc(sizeof(int32_t) * E);
  s->length = (float *)malloc(sizeof(float) * E);
  s->v0 = (float *)malloc(sizeof(float) * E);
  float vmax = 0.0f;
  for (int32_t u = 0; u < num_nodes; ++u)
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) s->src[e] = u;
  for (int32_t e = 0; e < num_edges; ++e) {
    s->dst[e] = dst[e];
    s->length[e] = length_m[e];
    s->ncells[e] = cells_of(length_m[e]);
    s->lanes[e] = lanes[e];
    s->v0[e] = speed_limit[e];
    if (speed_limit[e] > vmax) vmax = speed_limit[e];
  }
  /* H_max = ceil(2·Δt·max v0) + 2 (Q7) */
  s->h_max = p->h_max > 0 ? p->h_max : (int32_t)ceilf((2.0f * p->dt) * vmax) + 2;
  s->lc_n = p->lc_window > 0 ? p->lc_window : s->h_max;
  /* Q30 (Alg. 1 "Proceed according to I's signal controls"): a node with >= 3 in-edges
   * has a fixed-cycle two-phase signal; an approach is in phase 0 if it runs east-west
   * (|dx| >= |dy| from its source node to its destination node), else phase 1; without
   * coordinates by the parity of its rank among the node's in-edges (edge-id order). */
  s->sig = (uint8_t *)calloc(E, 1);
  s->sig_phase = (uint8_t *)calloc(E, 1);
  s->sig_cycle = 0;
  if (p->signal_cycle_s > 0.0f) {
    s->sig_cycle = (int32_t)floorf(p->signal_cycle_s / p->dt + 0.5f);
    if (s->sig_cycle < 2) { set_err(err, errlen, "signal cycle shorter than two steps", -1); lo_destroy(s); return NULL; }
    int32_t *indeg = (int32_t *)calloc((size_t)num_nodes, sizeof(int32_t));
    int32_t *rank = (int32_t *)calloc(E, sizeof(int32_t));
    for (int32_t e = 0; e < num_edges; ++e) rank[e] = indeg[dst[e]]++;
    for (int32_t e = 0; e < num_edges; ++e) {
      const int32_t u = s->src[e], w = dst[e];
      if (indeg[w] < 3) continue;
      s->sig[e] = 1;
      if (node_xy) {
        float dx = node_xy[2 * w] - node_xy[2 * u], dy = node_xy[2 * w + 1] - node_xy[2 * u + 1];
        s->sig_phase[e] = fabsf(dx) >= fabsf(dy) ? 0 : 1;
      } else {
        s->sig_phase[e] = (uint8_t)(rank[e] & 1);
      }
    }
    free(indeg);
    free(rank);
  }
  for (int b = 0; b < 2; ++b) {
    s->map[b] = (uint8_t **)malloc(sizeof(uint8_t *) * E);
    for (int32_t e = 0; e < num_edges; ++e) {
      size_t n = (size_t)s->lanes[e] * (size_t)s->ncells[e];
      s->map[b][e] = (uint8_t *)malloc(n);
      memset(s->map[b][e], 255, n); /* "Value 255 = Not Occupied" P:L259 */
    }
  }
  s->cur = 0;
  return s;
}

int32_t lo_h_max(const lo_sim *s) { return s->h_max; }

int32_t lo_load_demand(lo_sim *s, int64_t num_trips, const double *depart_s,
                       const int64_t *route_ptr, const int32_t *route_edges,
                       char *err, int32_t errlen) {
  if (s->loaded) { set_err(err, errlen, "demand already loaded", -1); return 4; }
  if (num_trips < 0 || (num_trips > 0 && (!depart_s || !route_ptr || !route_edges))) {
    set_err(err, errlen, "null or negative argument", -1);
    return 1;
  }
  if (num_trips > 0 && route_ptr[0] != 0) { set_err(err, errlen, "route_ptr[0] != 0", 0); return 3; }
  for (int64_t i = 0; i < num_trips; ++i) {
    if (!(depart_s[i] >= 0.0) || !isfinite(depart_s[i])) { set_err(err, errlen, "bad depart_s", i); return 3; }
    if (route_ptr[i + 1] <= route_ptr[i]) { set_err(err, errlen, "empty route", i); return 3; }
    for (int64_t r = route_ptr[i]; r < route_ptr[i + 1]; ++r) {
      int32_t e = route_edges[r];
      if (e < 0 || e >= s->n_edges) { set_err(err, errlen, "route edge out of range", i); return 3; }
      if (r > route_ptr[i] && s->dst[route_edges[r - 1]] != s->src[e]) {
        set_err(err, errlen, "route not connected", i);
        return 3;
      }
    }
  }
  int64_t R = num_trips > 0 ? route_ptr[num_trips] : 0;
  size_t N = (size_t)(num_trips > 0 ? num_trips : 1);
  s->n_trips = num_trips;
  s->route_ptr = (int64_t *)malloc(sizeof(int64_t) * (N + 1));
  s->route_ptr[0] = 0;
  if (num_trips > 0) memcpy(s->route_ptr, route_ptr, sizeof(int64_t) * (size_t)(num_trips + 1));
  s->route = (int32_t *)malloc(sizeof(int32_t) * (size_t)(R > 0 ? R : 1));
  if (R > 0) memcpy(s->route, route_edges, sizeof(int32_t) * (size_t)R);
  s->depart_step = (int64_t *)malloc(sizeof(int64_t) * N);
  s->arrival_step = (int64_t *)malloc(sizeof(int64_t) * N);
  s->edge_entry = (int64_t *)malloc(sizeof(int64_t) * (size_t)(R > 0 ? R : 1));
  for (int64_t r = 0; r < R; ++r) s->edge_entry[r] = -1;
  s->st = (trip_state *)calloc(N, sizeof(trip_state));
  s->nx = (trip_state *)calloc(N, sizeof(trip_state));
  s->proposal = (trip_state *)calloc(N, sizeof(trip_state));
  s->claims = (claim *)calloc(N, sizeof(claim));
  for (int b = 0; b < 2; ++b) {
    s->wr_e[b] = (int64_t *)malloc(sizeof(int64_t) * N);
    s->wr_i[b] = (int64_t *)malloc(sizeof(int64_t) * N);
    s->wr_n[b] = 0;
  }
  for (int64_t i = 0; i < num_trips; ++i) {
    s->depart_step[i] = lo_depart_step(depart_s[i], s->p.dt);
    s->arrival_step[i] = -1;
    s->st[i].status = LO_WAITING;
    s->st[i].edge = route_edges[route_ptr[i]];
    s->st[i].lane = 0;
    s->st[i].pos = 0.0f;
    s->st[i].v = 0.0f;
    s->st[i].j = 0;
  }
  s->step = 0;
  memset(&s->stats, 0, sizeof(s->stats));
  s->stats.waiting = num_trips;
  s->loaded = 1;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Lane-map accessors.  Cell c of lane l of edge e ("organizing lanes */
/* in order").                                                                */
/* ------------------------------------------------------------------------- */
static uint8_t map_get(const lo_sim *s, int b, int32_t e, int32_t l, int32_t c) {
  return s->map[b][e][(size_t)l * (size_t)s->ncells[e] + (size_t)c];
}

/* ------------------------------------------------------------------------- */
/* a3  Leader probe: "Front car within d_front", d_front = 2·Δt·v           */
/* (Alg. 1 lines 11, 14).  H = min(H_max, max(H_min,         */
/* ceil(2Δt·v))) (Q7).  Scans own lane c+1..min(c+H, Lc−1); if nothing and a */
/* next route edge exists, continues into the next edge's entry lane l' =    */
/* min(l, lanes(e')−1) cells 0..c+H−Lc ("check the downstream road segment", */
/* P:L249; Q10, Q21).  The gap is in cells; v_f is the occupant byte.*/
/* Pinned: brute-force all-pairs leader search on tiny networks (tests).      */
/* ------------------------------------------------------------------------- */
typedef struct { int found; int32_t gap; int32_t vf; int same_edge; int32_t cf; } probe_result;

/* d_front = H = min(H_max, max(H_min, ceil(2·Δt·v))) cells (Alg. 1 line 11, Q7) */
static int32_t probe_h(const lo_sim *s, float v) {
  int32_t H = (int32_t)ceilf((2.0f * s->p.dt) * v);
  if (H < s->p.h_min) H = s->p.h_min;
  if (H > s->h_max) H = s->h_max;
  return H;
}

static probe_result probe(const lo_sim *s, int b, int32_t e, int32_t l, int32_t c, float v, int32_t next_e) {
  probe_result r = {0, 0, 0, 0, 0};
  int32_t H = probe_h(s, v);
  int32_t Lc = s->ncells[e];
  int32_t last = c + H < Lc - 1 ? c + H : Lc - 1;
  for (int32_t c2 = c + 1; c2 <= last; ++c2) {
    uint8_t byte = map_get(s, b, e, l, c2);
    if (byte != 255) {
      r.found = 1; r.gap = c2 - c; r.vf = byte; r.same_edge = 1; r.cf = c2;
      return r;
    }
  }
  if (next_e >= 0 && c + H >= Lc) {
    int32_t l2 = l < s->lanes[next_e] - 1 ? l : s->lanes[next_e] - 1;
    int32_t reach = c + H - Lc;
    if (reach > s->ncells[next_e] - 1) reach = s->ncells[next_e] - 1;
    for (int32_t c2 = 0; c2 <= reach; ++c2) {
      uint8_t byte = map_get(s, b, next_e, l2, c2);
      if (byte != 255) {
        r.found = 1; r.gap = (Lc - c) + c2; r.vf = byte; r.same_edge = 0; r.cf = c2;
        return r;
      }
    }
  }
  return r;
}

int32_t lo_probe_trip(const lo_sim *s, int64_t id, int32_t *gap, int32_t *vf, int32_t *same_edge) {
  if (id < 0 || id >= s->n_trips) return -1;
  const trip_state *t = &s->st[id];
  if (t->status != LO_ON_ROAD) return -1;
  int64_t rj = s->route_ptr[id] + t->j;
  int32_t next_e = (rj + 1 < s->route_ptr[id + 1]) ? s->route[rj + 1] : -1;
  probe_result r = probe(s, s->cur, t->edge, t->lane, (int32_t)floorf(t->pos), t->v, next_e);
  if (!r.found) return 0;
  *gap = r.gap; *vf = r.vf; *same_edge = r.same_edge;
  return 1;
}

/* ------------------------------------------------------------------------- */
/* Digest of a snapshot: Σ over on-road trips of a 64-bit mix of            */
/* (id, edge, lane, cell, bits(pos), bits(v), cursor), mod 2^64 (test aid). */
/* ------------------------------------------------------------------------- */
static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t trip_hash(int64_t id, const trip_state *t) {
  uint32_t pb, vb;
  memcpy(&pb, &t->pos, 4);
  memcpy(&vb, &t->v, 4);
  uint64_t h = mix64((uint64_t)id);
  h = mix64(h ^ (uint64_t)(uint32_t)t->edge);
  h = mix64(h ^ (uint64_t)(uint32_t)t->lane);
  h = mix64(h ^ (uint64_t)(uint32_t)(int32_t)floorf(t->pos));
  h = mix64(h ^ (uint64_t)pb);
  h = mix64(h ^ (uint64_t)vb);
  h = mix64(h ^ (uint64_t)t->j);
  return h;
}

/* Next free claim record.  The OpenMP build (liblpsim_oracle_omp.so: the CPU
 * baseline on all host cores) runs the per-trip loop of one_step in parallel; claims are
 * sorted by (cell, id) before they are resolved, so the result does not depend on the order in
 * which they were recorded.  The parity build has no OpenMP: this is ncl++. */
static int64_t next_claim(int64_t *ncl) {
#ifdef _OPENMP
  int64_t i;
#pragma omp atomic capture
  i = (*ncl)++;
  return i;
#else
  return (*ncl)++;
#endif
}

static int claim_cmp(const void *pa, const void *pb) {
  const claim *a = (const claim *)pa, *b = (const claim *)pb;
  if (a->edge != b->edge) return a->edge < b->edge ? -1 : 1;
  if (a->lane != b->lane) return a->lane < b->lane ? -1 : 1;
  if (a->cell != b->cell) return a->cell < b->cell ? -1 : 1;
  if (a->id != b->id) return a->id < b->id ? -1 : 1;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* One step k -> k+1: Eq. (1) P:L239-242 and Alg. 1 P:L298-336.              */
/* All reads come from snapshot k (st, map[cur]); all writes go to k+1.      */
/* Returns 0 or a negative code if an invariant fails.                       */
/* ------------------------------------------------------------------------- */
static int64_t one_step(lo_sim *s) {
  const lo_params *P = &s->p;
  const int b = s->cur;                 /* M_k  */
  const int nb = 1 - s->cur;            /* M_{k+1} */
  const int64_t k = s->step;
  const float dt = P->dt;
  const float dt2 = dt * dt;
  const float half_a_dt2 = (0.5f * P->a) * dt2;
  int64_t ncl = 0;
  int64_t updates = 0;

#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 2048) reduction(+ : updates)
#endif
  for (int64_t id = 0; id < s->n_trips; ++id) {
    const trip_state *t = &s->st[id];
    trip_state *o = &s->nx[id];
    *o = *t;
    if (t->status == LO_FINISHED) continue;

    if (t->status == LO_WAITING) {
      /* A7: depart when Current Time ≥ t_depart and R (the entry cell) is
       * not occupied (Alg. 1 line 2); lane l0 = id mod lanes (Q22). */
      if (s->depart_step[id] > k) continue;
      int32_t e1 = s->route[s->route_ptr[id]];
      int32_t l0 = (int32_t)(id % s->lanes[e1]);
      if (map_get(s, b, e1, l0, 0) == 255) {
        claim *c = &s->claims[next_claim(&ncl)];
        c->edge = e1; c->lane = l0; c->cell = 0; c->id = id;
        trip_state *pr = &s->proposal[id];
        pr->status = LO_ON_ROAD; pr->edge = e1; pr->lane = l0;
        pr->pos = 0.0f; pr->v = 0.0f; pr->j = 0;
      }
      continue;
    }

    /* ON_ROAD */
    ++updates;
    const int32_t e = t->edge, l = t->lane;
    const float p = t->pos, v = t->v;
    const int32_t c = (int32_t)floorf(p);
    const int32_t Lc = s->ncells[e];
    const int64_t rj = s->route_ptr[id] + t->j;
    const int has_next = (rj + 1 < s->route_ptr[id + 1]);
    const int32_t e_next = has_next ? s->route[rj + 1] : -1;

    /* a3 probe */
    probe_result pr = probe(s, b, e, l, c, v, e_next);
    /* Q30: a red signal at the end of e (its approach's phase is not the one green at step k: phase 0
     * is green in the first half of every cycle, all signals in phase) is a stopped leader just
     * past the last cell, seen by a vehicle whose probe reaches the line; it takes the place of a
     * leader on the next edge, and the no-overtake clamp below then keeps the vehicle on e. */
    if (s->sig_cycle > 0 && has_next && s->sig[e] && c + probe_h(s, v) >= Lc) {
      const int green = (k % s->sig_cycle) < (s->sig_cycle / 2) ? 0 : 1;
      if (s->sig_phase[e] != green && !(pr.found && pr.same_edge)) {
        pr.found = 1; pr.gap = Lc - c; pr.vf = 0; pr.same_edge = 1; pr.cf = Lc;
      }
    }
    /* a4 IDM (Eq. Car Following) */
    float acc = lo_idm_accel(P, v, s->v0[e], pr.found, pr.gap, pr.vf);
    /* a4 kinematics (Q11): ballistic update, stop within the step if v would turn negative */
    float vn = v + acc * dt;
    float dx;
    if (!pr.found && P->vfree) {
      /* ablation: Alg. 1 "Else v <- v_free" taken literally: the speed becomes the free-flow
       * speed v0 over the step, the position advances by the mean of the two speeds */
      vn = s->v0[e];
      dx = (0.5f * (v + s->v0[e])) * dt;
    } else if (vn < 0.0f) {
      dx = (acc < 0.0f) ? -((0.5f * v) * v) / acc : 0.0f;
      vn = 0.0f;
    } else {
      dx = v * dt + (0.5f * acc) * dt2;
    }
    float pn = p + dx;
    vn = fminf(vn, 254.0f);  /* byte encoding caps speed at 254 */
    /* no overtaking within the lane: "One byte can only be occupied by one vehicle" */
    if (pr.found && pr.same_edge && (int32_t)floorf(pn) >= pr.cf) {
      pn = fmaxf(p, (float)(pr.cf - 1));
      vn = fminf(vn, (float)pr.vf);
    }

    if (pn >= (float)Lc) {
      /* a5 intersection reached (Alg. 1 lines 15-16; Remark P:L249) */
      if (!has_next) {
        /* Q24: crossing the end of the last route edge finishes the trip */
        o->status = LO_FINISHED;
        s->arrival_step[id] = k + 1;
        continue;
      }
      int32_t l2 = l < s->lanes[e_next] - 1 ? l : s->lanes[e_next] - 1;   /* Q21 */
      /* fallback: wait at the stop line (Q23) */
      o->pos = fmaxf(p, (float)(Lc - 1));
      o->v = 0.0f;
      if (map_get(s, b, e_next, l2, 0) == 255) {
        claim *cl = &s->claims[next_claim(&ncl)];
        cl->edge = e_next; cl->lane = l2; cl->cell = 0; cl->id = id;
        trip_state *q = &s->proposal[id];
        q->status = LO_ON_ROAD; q->edge = e_next; q->lane = l2;
        q->pos = 0.0f; q->v = vn; q->j = t->j + 1;   /* Q20 */
      }
      continue;
    }

    o->pos = pn;
    o->v = vn;

    /* a6 mandatory lane change + gap acceptance (Alg. 1 lines 18-23;
     * Eq. (Lane Change) P:L222-225; Eq. (Gap Acceptance) P:L228-235; Q13-Q17). */
    const int32_t cn = (int32_t)floorf(pn);
    if (has_next && cn >= 1) {
      const int32_t node = s->dst[e];
      const int32_t K = (int32_t)(s->row_ptr[node + 1] - s->row_ptr[node]);
      const int32_t r = (int32_t)(e_next - s->row_ptr[node]);
      const int32_t L = s->lanes[e];
      const int32_t lo = (r * L) / K;
      int32_t hi = ((r + 1) * L + K - 1) / K - 1;
      if (hi < lo) hi = lo;
      int32_t tl = -1;
      if (l < lo) tl = l + 1;
      else if (l > hi) tl = l - 1;
      if (tl >= 0) {
        float x = (float)Lc - p;                      /* x_i(k): distance to the exit */
        float plc = (P->x0 - x) / P->x0;
        plc = fminf(fmaxf(plc, 0.0f), 1.0f);
        float u = lo_u24(P->seed, (uint32_t)id, (uint32_t)k, 0u);
        if (u < plc && map_get(s, b, e, tl, cn) == 255) {
          const int32_t n = s->lc_n;
          int has_ld = 0, has_lg = 0;
          int32_t g_ld = 0, b_ld = 0, g_lg = 0, b_lg = 0;
          int32_t hi_c = cn + n < Lc - 1 ? cn + n : Lc - 1;
          for (int32_t c2 = cn + 1; c2 <= hi_c; ++c2) {
            uint8_t by = map_get(s, b, e, tl, c2);
            if (by != 255) { has_ld = 1; g_ld = c2 - cn; b_ld = by; break; }
          }
          int32_t lo_c = cn - n > 0 ? cn - n : 0;
          for (int32_t c2 = cn - 1; c2 >= lo_c; --c2) {
            uint8_t by = map_get(s, b, e, tl, c2);
            if (by != 255) { has_lg = 1; g_lg = cn - c2; b_lg = by; break; }
          }
          float eps_a = lo_eps(P->seed, (uint32_t)id, (uint32_t)k, 1u, P->sigma_a);
          float eps_b = lo_eps(P->seed, (uint32_t)id, (uint32_t)k, 2u, P->sigma_b);
          float g_lead = fmaxf(0.0f, ((P->g_a + P->alpha_i * v) - P->alpha_a * (float)b_ld) + eps_a);
          float g_lag = fmaxf(0.0f, ((P->g_b + P->alpha_b * (float)b_lg) - P->alpha_i * v) + eps_b);
          int accept = 1;
          if (has_ld && !((float)g_ld >= g_lead)) accept = 0;
          if (has_lg) {
            int32_t safe = (int32_t)ceilf(((float)b_lg + 1.0f) * dt + half_a_dt2) + 1;
            if (!((float)g_lg >= g_lag) || g_lg < safe) accept = 0;
          }
          if (accept) {
            claim *cl = &s->claims[next_claim(&ncl)];
            cl->edge = e; cl->lane = tl; cl->cell = cn; cl->id = id;
            trip_state *q = &s->proposal[id];
            *q = *o;
            q->lane = tl;
          }
        }
      }
    }
  }

  /* Resolve (A9, Q19): for every contended cell the lowest id wins.
   * lost_claims counts the losing parties: each losing on-road
   * vehicle, and a slot's departure queue once (its lowest waiting id). */
  qsort(s->claims, (size_t)ncl, sizeof(claim), claim_cmp);
  int waiting_seen = 0;
  for (int64_t i = 0; i < ncl; ++i) {
    const claim *cl = &s->claims[i];
    int first = (i == 0) || s->claims[i - 1].edge != cl->edge ||
                s->claims[i - 1].lane != cl->lane || s->claims[i - 1].cell != cl->cell;
    if (first) waiting_seen = 0;
    const int is_waiting = s->st[cl->id].status == LO_WAITING;
    if (!first) {
      if (!is_waiting || !waiting_seen) s->stats.lost_claims++;
      if (is_waiting) waiting_seen = 1;
      continue;
    }
    if (is_waiting) waiting_seen = 1;
    const int64_t id = cl->id;
    const trip_state *t = &s->st[id];
    if (t->status == LO_WAITING) s->stats.departures++;
    else if (s->proposal[id].j != t->j) s->stats.transitions++;
    else s->stats.lane_changes++;
    s->nx[id] = s->proposal[id];
    /* a departure or a transition puts the trip on route edge j at snapshot k+1: t_start */
    if (t->status == LO_WAITING || s->proposal[id].j != t->j)
      s->edge_entry[s->route_ptr[id] + s->proposal[id].j] = k + 1;
  }

  /* Write M_{k+1}: reset the bytes written two steps ago, then every on-road
   * vehicle writes (uint8)min(v,254) at its cell.  Check the
   * invariants: one vehicle per byte, non-255 count = on-road count,
   * conservation waiting + on-road + finished = N. */
  for (int64_t w = 0; w < s->wr_n[nb]; ++w) s->map[nb][s->wr_e[nb][w]][s->wr_i[nb][w]] = 255;
  s->wr_n[nb] = 0;
  int64_t waiting = 0, on_road = 0, finished = 0;
  uint64_t digest = 0;
  for (int64_t id = 0; id < s->n_trips; ++id) {
    const trip_state *o = &s->nx[id];
    if (o->status == LO_WAITING) { ++waiting; continue; }
    if (o->status == LO_FINISHED) { ++finished; continue; }
    ++on_road;
    int32_t c = (int32_t)floorf(o->pos);
    if (c < 0 || c >= s->ncells[o->edge] || o->lane < 0 || o->lane >= s->lanes[o->edge]) return -(k + 1);
    size_t idx = (size_t)o->lane * (size_t)s->ncells[o->edge] + (size_t)c;
    if (s->map[nb][o->edge][idx] != 255) return -(k + 1);   /* two vehicles in one byte */
    s->map[nb][o->edge][idx] = (uint8_t)(int32_t)fminf(o->v, 254.0f);
    s->wr_e[nb][s->wr_n[nb]] = o->edge;
    s->wr_i[nb][s->wr_n[nb]] = (int64_t)idx;
    s->wr_n[nb]++;
    digest += trip_hash(id, o);
  }
  if (waiting + on_road + finished != s->n_trips) return -(k + 1);

  /* arrivals of this step */
  int64_t arrivals = 0;
  for (int64_t id = 0; id < s->n_trips; ++id)
    if (s->st[id].status == LO_ON_ROAD && s->nx[id].status == LO_FINISHED) ++arrivals;

  trip_state *tmp = s->st; s->st = s->nx; s->nx = tmp;
  s->cur = nb;
  s->step = k + 1;
  s->stats.step = k + 1;
  s->stats.waiting = waiting;
  s->stats.on_road = on_road;
  s->stats.finished = finished;
  s->stats.updates += updates;
  s->stats.arrivals += arrivals;
  s->stats.digest = digest;
  return 0;
}

int64_t lo_step(lo_sim *s, int64_t n) {
  if (!s->loaded) return -1;
  for (int64_t i = 0; i < n; ++i) {
    int64_t r = one_step(s);
    if (r != 0) return r;
  }
  return 0;
}

void lo_stats_get(const lo_sim *s, lo_stats *out) { *out = s->stats; }

/* Results: arrival step (−1 if not arrived), arrival time =
 * step·Δt, distance = Σ length of completed route edges (+ pos on the current
 * edge for trips still en route), in double. */
int32_t lo_results(const lo_sim *s, int64_t n, int64_t *arrival_step,
                   double *arrival_time_s, double *distance_m) {
  if (n != s->n_trips) return 1;
  for (int64_t id = 0; id < n; ++id) {
    const trip_state *t = &s->st[id];
    int64_t a = s->arrival_step[id];
    if (arrival_step) arrival_step[id] = a;
    if (arrival_time_s) arrival_time_s[id] = a >= 0 ? (double)a * (double)s->p.dt : -1.0;
    if (distance_m) {
      double d = 0.0;
      if (t->status == LO_FINISHED) {
        for (int64_t r = s->route_ptr[id]; r < s->route_ptr[id + 1]; ++r) d += (double)s->length[s->route[r]];
      } else if (t->status == LO_ON_ROAD) {
        for (int64_t r = s->route_ptr[id]; r < s->route_ptr[id] + t->j; ++r) d += (double)s->length[s->route[r]];
        d += (double)t->pos;
      }
      distance_m[id] = d;
    }
  }
  return 0;
}

int32_t lo_edge_entry(const lo_sim *s, int64_t r_total, int64_t *out) {
  if (!s->loaded) return -1;
  const int64_t R = s->n_trips > 0 ? s->route_ptr[s->n_trips] : 0;
  if (r_total != R) return -2;
  for (int64_t r = 0; r < R; ++r) out[r] = s->edge_entry[r];
  return 0;
}

int32_t lo_trip_state(const lo_sim *s, int64_t n, int32_t *status, int32_t *edge,
                      int32_t *lane, float *pos, float *v, int64_t *cursor) {
  if (n != s->n_trips) return 1;
  for (int64_t id = 0; id < n; ++id) {
    const trip_state *t = &s->st[id];
    if (status) status[id] = t->status;
    if (edge) edge[id] = t->edge;
    if (lane) lane[id] = t->lane;
    if (pos) pos[id] = t->pos;
    if (v) v[id] = t->v;
    if (cursor) cursor[id] = t->j;
  }
  return 0;
}

/* Test scaffolding (no arithmetic of the method): put the simulation at
 * snapshot `step` with the given per-trip state, as a checkpoint would hold it
 * (status / edge / lane / pos / v / cursor as lo_trip_state returns them,
 * arrival_step as lo_results).  M_k is rebuilt from the on-road trips with the
 * byte encoding of P:L259-263 ((uint8)min(v, 254), 255 = free); the other map
 * is cleared; event counters restart at zero.  Used by the scripted pins
 * (lead/lag gap acceptance, stop within the step, the SURVEY worked cases).
 * Returns 0, or 1 + the first offending trip (not on its route, cell out of
 * range, two vehicles in one byte). */
int32_t lo_set_state(lo_sim *s, int64_t step, int64_t n, const int32_t *status, const int32_t *edge,
                     const int32_t *lane, const float *pos, const float *v, const int64_t *cursor,
                     const int64_t *arrival_step) {
  if (!s->loaded || n != s->n_trips || step < 0) return -1;
  for (int b = 0; b < 2; ++b) {
    for (int32_t e = 0; e < s->n_edges; ++e) memset(s->map[b][e], 255, (size_t)s->lanes[e] * (size_t)s->ncells[e]);
    s->wr_n[b] = 0;
  }
  int64_t waiting = 0, on_road = 0, finished = 0;
  for (int64_t id = 0; id < n; ++id) {
    trip_state *t = &s->st[id];
    t->status = status[id];
    t->edge = s->route[s->route_ptr[id]];
    t->lane = 0; t->pos = 0.0f; t->v = 0.0f; t->j = 0;
    s->arrival_step[id] = arrival_step ? arrival_step[id] : -1;
    if (t->status == LO_WAITING) { ++waiting; continue; }
    if (t->status == LO_FINISHED) { ++finished; continue; }
    if (t->status != LO_ON_ROAD) return (int32_t)(1 + id);
    const int64_t j = cursor[id];
    if (j < 0 || s->route_ptr[id] + j >= s->route_ptr[id + 1] || s->route[s->route_ptr[id] + j] != edge[id])
      return (int32_t)(1 + id);
    const int32_t e = edge[id], c = (int32_t)floorf(pos[id]);
    if (lane[id] < 0 || lane[id] >= s->lanes[e] || !(pos[id] >= 0.0f) || c >= s->ncells[e] ||
        !(v[id] >= 0.0f && v[id] <= 254.0f))
      return (int32_t)(1 + id);
    const size_t idx = (size_t)lane[id] * (size_t)s->ncells[e] + (size_t)c;
    if (s->map[s->cur][e][idx] != 255) return (int32_t)(1 + id);
    s->map[s->cur][e][idx] = (uint8_t)(int32_t)fminf(v[id], 254.0f);
    s->wr_e[s->cur][s->wr_n[s->cur]] = e;
    s->wr_i[s->cur][s->wr_n[s->cur]] = (int64_t)idx;
    s->wr_n[s->cur]++;
    t->edge = e; t->lane = lane[id]; t->pos = pos[id]; t->v = v[id]; t->j = j;
    ++on_road;
  }
  memset(&s->stats, 0, sizeof(s->stats));
  s->step = step;
  s->stats.step = step;
  s->stats.waiting = waiting;
  s->stats.on_road = on_road;
  s->stats.finished = finished;
  return 0;
}

int64_t lo_lane_map_size(const lo_sim *s) {
  int64_t n = 0;
  for (int32_t e = 0; e < s->n_edges; ++e) n += (int64_t)s->lanes[e] * s->ncells[e];
  return n;
}

int32_t lo_lane_map_dump(const lo_sim *s, uint8_t *out, int64_t size) {
  int64_t off = 0;
  for (int32_t e = 0; e < s->n_edges; ++e) {
    int64_t n = (int64_t)s->lanes[e] * s->ncells[e];
    if (off + n > size) return 1;
    memcpy(out + off, s->map[s->cur][e], (size_t)n);
    off += n;
  }
  return off == size ? 0 : 1;
}

void lo_destroy(lo_sim *s) {
  if (!s) return;
  free(s->sig);
  free(s->sig_phase);
  for (int b = 0; b < 2; ++b) {
    if (s->map[b]) {
      for (int32_t e = 0; e < s->n_edges; ++e) free(s->map[b][e]);
      free(s->map[b]);
    }
    free(s->wr_e[b]);
    free(s->wr_i[b]);
  }
  free(s->row_ptr); free(s->src); free(s->dst); free(s->ncells); free(s->lanes);
  free(s->length); free(s->v0);
  free(s->route_ptr); free(s->route); free(s->depart_step); free(s->arrival_step); free(s->edge_entry);
  free(s->st); free(s->nx); free(s->claims); free(s->proposal);
  free(s);
}
