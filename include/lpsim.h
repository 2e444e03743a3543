/*
 * lpsim.h — C ABI of the B200-native LPSim per-timestep vehicle update.
 *
 * Method: Jiang, Sengupta, Demmel, Williams, "Large Scale Multi-GPU Based
 * Parallel Traffic Simulation for Accelerated Traffic Assignment and
 * Propagation", arXiv 2406.08496 (PAPER.md; "P:Lnnn" = line nnn).  Readings
 * "Qnn" where the paper is silent are listed in DESIGN.md §3.
 *
 * The library owns its device memory (cudaMalloc) and runs every step of the
 * path in its own sm_100a kernels.  All entry points are synchronous with
 * respect to the host unless stated, return an lpsim_status, and never mutate
 * state on error.  A context is not thread-safe.  Call order:
 *   lpsim_create -> lpsim_load_demand (once) -> lpsim_step* ->
 *   lpsim_results / lpsim_stats / lpsim_trip_state (any time after load) ->
 *   lpsim_destroy.  Anything else returns LPSIM_E_STATE.
 * Ownership: the caller owns every input array; the library copies what it
 * needs during the call and keeps no pointer.  Output arrays are
 * caller-allocated with the sizes stated.  On error, lpsim_last_error()
 * returns a message naming the first offending index.
 */
#ifndef LPSIM_H
#define LPSIM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LPSIM_ABI_VERSION 1

typedef struct lpsim_ctx lpsim_ctx;

typedef enum {
  LPSIM_OK = 0,
  LPSIM_E_INVALID_ARG = 1,    /* null pointer, bad size, struct_size mismatch, bad parameter */
  LPSIM_E_INVALID_GRAPH = 2,  /* CSR / attribute validation failed */
  LPSIM_E_INVALID_DEMAND = 3, /* route / departure validation failed */
  LPSIM_E_STATE = 4,          /* call out of order */
  LPSIM_E_NOMEM = 5,          /* host or device allocation failed */
  LPSIM_E_CAPACITY = 6,       /* an index does not fit the packed device layout */
  LPSIM_E_CUDA = 7,           /* CUDA runtime error or no CUDA device */
  LPSIM_E_COMM = 8,           /* inter-partition exchange failed */
  LPSIM_E_INVARIANT = 9       /* a device-side check failed (debug flag) */
} lpsim_status;

/* Road graph in CSR (adjacency list; per edge the number of
 * lanes, its index on the lane map, upstream and downstream node).
 * Edge id == CSR position.  Validation: row_ptr[0] = 0, monotone,
 * row_ptr[num_nodes] = num_edges; 0 <= dst < num_nodes; length_m >= 1 and
 * finite (1 byte = 1 m); 1 <= lanes <= 63;
 * 0 < speed_limit <= 254 (byte encoding); out-degree <= 1023. */
typedef struct {
  uint32_t struct_size;           /* = sizeof(lpsim_graph) */
  int32_t num_nodes, num_edges;
  const int64_t *row_ptr;         /* [num_nodes+1] out-edges of u: [row_ptr[u], row_ptr[u+1]) */
  const int32_t *dst;             /* [num_edges] downstream node */
  const float *length_m;          /* [num_edges] >= 1.0; Lc = ceil(length_m) cells */
  const uint8_t *lanes;           /* [num_edges] 1..63 */
  const float *speed_limit_mps;   /* [num_edges] (0, 254]; the IDM v0 of the edge */
  const float *node_xy;           /* [2*num_nodes] x,y (m) for the partitioner; may be NULL */
} lpsim_graph;

/* Flags */
#define LPSIM_FLAG_DIGESTS 0x1u    /* record a per-step state digest (parity tests) */
#define LPSIM_FLAG_CHECKS  0x2u    /* invariant checks (slower): in every step each byte of M_{k+1} is written
                                      only over a free cell (one vehicle per cell; atomic check), and
                                      after each lpsim_step call (one process) the occupied cells of M_k equal
                                      the on-road vehicles and the other lane map is clean; a
                                      violation returns LPSIM_E_INVARIANT naming the step (and the cell) and
                                      leaves the context unusable */
#define LPSIM_FLAG_NO_SORT 0x4u    /* disable the periodic locality sort (a9); compaction still runs */
#define LPSIM_FLAG_TIMING  0x8u    /* per-phase device timers (globaltimer, barrier to barrier) */
#define LPSIM_FLAG_EDGE_TIMES 0x10u /* record t_start of every route edge (Alg. 1); must be set
                                       at lpsim_create: lpsim_load_demand allocates the table */
/* Ablations (§8(f) item 4), off by default: */
#define LPSIM_FLAG_RACY  0x20u     /* paper-faithful racy claims: the first contender to reach a cell's claim
                                      word wins, instead of the lowest trip id (A9); results then
                                      depend on thread timing */
#define LPSIM_FLAG_VFREE 0x40u     /* literal "v <- v_free" of Alg. 1 when no leader is within
                                      d_front: v' = v0 of the edge, dx = (v + v0)/2 * dt, instead of the
                                      IDM free-road term (Q9) */

typedef struct {
  uint32_t struct_size;  /* = sizeof(lpsim_config) */
  float dt_s;            /* Δt (Q1), default 0.5 */
  float a, b, s0, T_headway;  /* IDM (Q3), defaults 1.5, 2, 2, 1.5 */
  int32_t delta;         /* IDM exponent, integer >= 1 (Q6), default 4 */
  float x0;              /* mandatory-LC distance (Q13), default 100 */
  float g_a, g_b;        /* desired lead / lag gap (Q15), default 2, 2 */
  float alpha_i, alpha_a, alpha_b;  /* anticipation times, default .5 */
  float sigma_a, sigma_b;           /* scale of ε_a, ε_b (Q15), default .5 */
  int32_t h_min;         /* probe floor (Q7), default 2 */
  int32_t h_max;         /* probe cap; 0 = ceil(2·Δt·max v0) + 2 */
  int32_t lc_window;     /* LC scan window n; 0 = h_max */
  int32_t sort_every;    /* locality sort + compaction period in steps (a9); 0 = default 256 */
  uint64_t seed;         /* Philox key (Q27), default 1 */
  int32_t device;        /* CUDA device ordinal, default 0 */
  int32_t num_parts;     /* graph partitions simulated by this process (§8(e)); default 1 */
  const int32_t *node_part;  /* [num_nodes] partition of each node, or NULL = built-in */
  void *stream;          /* cudaStream_t to run on, or NULL = library-owned stream */
  uint32_t flags;        /* LPSIM_FLAG_* */
  int32_t rank, world;   /* multi-process mode (world > 1): this process simulates partition `rank`
                            of a `world`-way partition on its own GPU; every process passes identical
                            graph / demand / config (SPMD) and exchanges peer memory with
                            lpsim_ipc_handle / lpsim_ipc_attach before stepping.  Default 0, 1. */
  float signal_cycle_s;  /* §8(f) signalised intersections (Alg. 1 "Proceed according to I's signal
                            controls"; reading Q30 in DESIGN.md): 0 = unsignalised (Q18, the
                            default); > 0 = fixed-cycle two-phase signal of that cycle at every node
                            with >= 3 in-edges, all in phase */
  int32_t reserved[4];
} lpsim_config;

typedef struct {
  uint32_t struct_size;            /* = sizeof(lpsim_stats) */
  int64_t step;                    /* k of the snapshot currently held */
  int64_t waiting, on_road, finished;
  int64_t updates;                 /* Σ on-road vehicles advanced (one "vehicle-update" each) */
  int64_t departures, transitions, lane_changes, arrivals, lost_claims;
  uint64_t digest;                 /* digest of snapshot `step` (LPSIM_FLAG_DIGESTS), else 0 */
  double step_ms;                  /* device time of the last lpsim_step call (CUDA events) */
  double exchange_ms;              /* LPSIM_FLAG_TIMING, multi-process: device time of the per-step cross-GPU
                                      barrier (migrant-count push + flag release/acquire over NVLink) during
                                      the last lpsim_step; the peer stores of migrants and halo bytes are part
                                      of phases A and C (§8(e)); 0 in one process */
  int64_t num_parts;
  int64_t device_bytes;            /* device memory held by the context */
  int64_t kernel_launches;         /* launches of the library's own kernels by the last lpsim_step */
  int64_t phase_ns[3];             /* LPSIM_FLAG_TIMING: ns in phases A (move), C (resolve) and in the
                                      cross-GPU barrier during the last lpsim_step */
  int64_t sort_ns;                 /* device time of the a9 locality sorts (compaction included) during the
                                      last lpsim_step (CUDA events around each sort launch) */
  int64_t soa_entries;             /* vehicle SoA entries of this process (live + dead: the dead entries
                                      that arrivals and migrations leave until the next a9 compaction) */
} lpsim_stats;

/* Fills *cfg with the defaults above (struct_size must be set by the caller). */
lpsim_status lpsim_config_default(lpsim_config *cfg);

/* Validates the graph, builds the lane-map layout (a0) on the device and
 * allocates the graph-side device state.  *out is NULL on failure. */
lpsim_status lpsim_create(const lpsim_graph *graph, const lpsim_config *cfg, lpsim_ctx **out);

/* Loads OD trips "after the routing": trip i departs at depart_s[i]
 * (>= 0, finite; depart step = smallest k with k·Δt >= depart_s, Q22) along
 * route_edges[route_ptr[i] .. route_ptr[i+1]) (non-empty, consecutive edges
 * connected).  origin/destination (nullable) must equal from(first edge) /
 * to(last edge) and differ.  Trip id i is the only tie-break key (A9). */
lpsim_status lpsim_load_demand(lpsim_ctx *ctx, int64_t num_trips, const double *depart_s,
                               const int64_t *route_ptr, const int32_t *route_edges,
                               const int32_t *origin, const int32_t *destination);

/* Advances n >= 0 steps k -> k+1 (Eq. 1, Alg. 1) and returns when done.  After
 * a device-side error (LPSIM_E_CAPACITY, LPSIM_E_INVARIANT, LPSIM_E_COMM,
 * LPSIM_E_CUDA) the state of the failed step is partial and the context is
 * unusable: every later lpsim_step returns LPSIM_E_STATE. */
lpsim_status lpsim_step(lpsim_ctx *ctx, int64_t n);

/* Per trip (arrays of num_trips, any may be NULL): arrival step (-1 = not
 * arrived), arrival time = step·Δt (-1 if not arrived), distance = Σ length of
 * traversed edges in route order in double (+ position on the current edge
 * for trips still en route; 0 for trips not yet departed). */
lpsim_status lpsim_results(lpsim_ctx *ctx, int64_t num_trips, int64_t *arrival_step,
                           double *arrival_time_s, double *distance_m);

lpsim_status lpsim_stats_get(lpsim_ctx *ctx, lpsim_stats *out);

/* Per-trip state of the current snapshot (arrays of num_trips, any may be
 * NULL): status 0 waiting / 1 on road / 2 finished; for on-road trips the
 * edge, lane, position (m), speed (m/s) and cursor (index of the edge in
 * the trip's route).  Waiting trips report (route[0], 0, 0, 0, 0); the other
 * fields of finished trips are unspecified. */
lpsim_status lpsim_trip_state(lpsim_ctx *ctx, int64_t num_trips, int32_t *status, int32_t *edge,
                              int32_t *lane, float *pos, float *v, int64_t *cursor);

/* Byte image of the current snapshot M_k in the global layout of a0
 * (edges in id order, lanes in order, cells along the lane).
 * size must equal lpsim_lane_map_size(). */
int64_t lpsim_lane_map_size(const lpsim_ctx *ctx);
lpsim_status lpsim_lane_map(lpsim_ctx *ctx, uint8_t *out, int64_t size);
/* base[e] of the global layout, [num_edges]. */
lpsim_status lpsim_lane_map_base(lpsim_ctx *ctx, uint64_t *base, int64_t num_edges);

/* Digests of the snapshots produced by the last lpsim_step call
 * (LPSIM_FLAG_DIGESTS): out[i] = digest of snapshot step_before + 1 + i. */
lpsim_status lpsim_digests(lpsim_ctx *ctx, uint64_t *out, int64_t n);

/* t_start per route edge (Alg. 1 "If Moving on a New Edge ... t_start <- Current Time",
 * P:L305-307; the per-edge entry times a traffic-assignment outer loop consumes):
 * out[route_ptr[i] + j] = k, the step of the first snapshot at which trip i is
 * on its route edge j (j = 0: its departure), -1 if it has not (yet) entered it.
 * Time = k * dt_s.  r_total = route_ptr[num_trips]; out is caller-allocated.
 * Needs LPSIM_FLAG_EDGE_TIMES at lpsim_create (else LPSIM_E_STATE).  In
 * multi-process mode each rank holds the entries its partition wrote (others
 * -1): combine with an element-wise max. */
lpsim_status lpsim_edge_entry_steps(lpsim_ctx *ctx, int64_t r_total, int32_t *out);

/* Checkpoint / restore (§8(f) item 3).  A checkpoint of snapshot `step` is
 * what lpsim_trip_state, lpsim_results (arrival_step) and lpsim_stats_get
 * return at that step, plus lpsim_edge_entry_steps with
 * LPSIM_FLAG_EDGE_TIMES: per-trip state is the whole simulation state at a
 * step boundary (claim words are free, M_{k+1} is clean, M_k and the
 * departure queues follow from the trips).  lpsim_restore rebuilds the device
 * state of snapshot `step` from it, into a context created and loaded with the
 * same graph, demand and config (any partition count), before any lpsim_step;
 * stepping on then produces exactly the results of the uninterrupted run.
 *   status/edge/lane/pos/v/cursor: as lpsim_trip_state ([num_trips]);
 *   arrival_step: as lpsim_results (-1 = not arrived);
 *   counters: {updates, departures, transitions, lane_changes, arrivals,
 *              lost_claims} of lpsim_stats at `step` (nullable: zeros; in
 *              multi-process mode rank 0 carries them);
 *   edge_entry: [route_ptr[num_trips]] as lpsim_edge_entry_steps, or NULL.
 * Errors: LPSIM_E_STATE (not freshly loaded), LPSIM_E_INVALID_ARG naming the
 * first offending trip (status, arrival, cursor outside the route or not on
 * the given edge, lane, position, speed) — all checked on the host before any
 * device write.  A device-side failure (not expected after the host checks)
 * leaves the context unusable (later calls: LPSIM_E_STATE). */
lpsim_status lpsim_restore(lpsim_ctx *ctx, int64_t step, int64_t num_trips, const int32_t *status,
                           const int32_t *edge, const int32_t *lane, const float *pos, const float *v,
                           const int64_t *cursor, const int64_t *arrival_step, const int64_t *counters,
                           const int32_t *edge_entry);

/* Changes the LPSIM_FLAG_* bits of a loaded context between lpsim_step calls
 * (e.g. LPSIM_FLAG_TIMING for a measured window).  Results do not depend on
 * the flags.  LPSIM_E_STATE before lpsim_load_demand. */
lpsim_status lpsim_set_flags(lpsim_ctx *ctx, uint32_t flags);

/* Diagnostics (LPSIM_FLAG_TIMING): per CTA b of the step kernel, 16 words:
 * out[b,0|1] ns from the start of phase A|C to the CTA's last chunk, summed
 * over the last lpsim_step call; out[b,2|3] start of phase A|C and
 * out[b,4|5] arrival at the grid barrier after phase A|C, in the last step
 * (globaltimer ns); out[b,6|7] ns spent in the barrier after phase A|C,
 * summed; out[b,8|9] end of the CTA's work in phase A|C in the last step;
 * out[b,10] chunk rounds of phase A in the last step; thread 0 of the CTA,
 * ns from the phase start summed: out[b,11] to its first vehicle move,
 * out[b,12] to the end of its vehicle chunks, out[b,13] to the end of its
 * admit chunks (phase A), out[b,14] to the end of its claim chunks,
 * out[b,15] to the end of its departure chunks (phase C); out[b,16] to its
 * first vehicle's probe data, out[b,17] to its first vehicle's longitudinal
 * move (phase A); out[b,18] departures | claimed admit positions << 32 and
 * out[b,19] relisted slots in the CTA's admit chunks (phase C, summed);
 * warp 0 of the CTA, its first admit chunk, ns from the phase C start summed:
 * out[b,20] admit position loaded, out[b,21] claim words resolved,
 * out[b,22] successor searches done, out[b,23] appends and relists written.
 * n = 24 x grid size (the stride is 24 words: out[24b + w]). */
lpsim_status lpsim_debug_block_times(lpsim_ctx *ctx, uint64_t *out, int64_t n);

/* Occupied (non-0xFF) cells of the two lane-map buffers over the owned edges of
 * every partition of this context (entry halos excluded), at the current step
 * k: out[0] in M_k, out[1] in the other buffer.  Every on-road vehicle holds
 * exactly one cell of M_k and resolve/commit clears M_k's cells before the
 * buffer is reused, so at a step boundary
 * out[0] == on-road vehicles and out[1] == 0.  Test instrumentation; blocks;
 * LPSIM_E_STATE before lpsim_load_demand. */
lpsim_status lpsim_debug_map_occupancy(lpsim_ctx *ctx, uint64_t out[2]);

/* Test instrumentation: overwrite byte `cell` (global layout) of the current
 * snapshot M_k with `value`, e.g. to corrupt the state for the
 * LPSIM_FLAG_CHECKS tests.  Single-partition contexts only (LPSIM_E_STATE
 * otherwise or before lpsim_load_demand); LPSIM_E_INVALID_ARG for a cell out
 * of range. */
lpsim_status lpsim_debug_poke_map(lpsim_ctx *ctx, int64_t cell, uint8_t value);

/* Weighted recursive coordinate bisection of the nodes into k parts (§8(e)):
 * split points balance `weight` (route visit counts; NULL = unit),
 * nodes with zero weight follow their coordinates into the enclosing part
 * ("nearest subgraph").  node_xy [2*num_nodes] may be NULL (node id
 * order is then the coordinate).  Host-only, deterministic; writes part_out
 * [num_nodes] in 0..k-1.  The built-in partition (lpsim_config.node_part
 * NULL, num_parts > 1) is lpsim_partition_multilevel on the route visits;
 * RCB serves graphs with fewer than 8 nodes per part. */
lpsim_status lpsim_partition_rcb(int32_t num_nodes, const float *node_xy, const double *weight, int32_t k,
                                 int32_t *part_out);

/* Balanced multilevel k-way partition of the nodes (§8(f) item 1, the METIS
 * scheme of P:L413-421): the directed graph is symmetrised (edge weight =
 * edge_weight[e], NULL = lanes[e], so the default objective is the number of
 * cut lanes = migrant slots + entry halos), coarsened by heavy-edge matching,
 * split by recursive greedy graph growing and refined level by level with
 * greedy boundary moves, each part's vertex weight kept below
 * (1 + imbalance) x total / k.  node_weight [num_nodes] = route visit counts
 * over the studied window (NULL = unit; zero-visit nodes get a tiny
 * weight and follow their neighbours).  Host-only, deterministic for
 * a given seed; writes part_out [num_nodes] in 0..k-1.  The built-in
 * partition when lpsim_config.node_part is NULL and num_parts > 1. */
lpsim_status lpsim_partition_multilevel(const lpsim_graph *graph, const double *node_weight,
                                        const double *edge_weight, int32_t k, double imbalance,
                                        uint64_t seed, int32_t *part_out);

/* Unbalanced Leiden + k-means partition (§8(f) item 1): the
 * symmetrised graph (edge weight as for the multilevel partition) is split
 * into modularity communities at the given resolution (local moving, then
 * every community split into its connected components — Leiden's
 * connectivity guarantee — then aggregation, repeated until stable); the
 * communities are grouped into k parts by k-means (k-means++ seeding from
 * `seed`) on their centroids, weighted by node_weight (route visits, P:L457;
 * NULL = unit).  Needs graph->node_xy.  No balance bound (the paper's point:
 * fewer cut edges at small k); parts are numbered densely from 0 and there
 * may be fewer than k if the graph has fewer communities.  Host-only,
 * deterministic per seed. */
lpsim_status lpsim_partition_leiden_kmeans(const lpsim_graph *graph, const double *node_weight,
                                           const double *edge_weight, int32_t k, double resolution,
                                           uint64_t seed, int32_t *part_out);

/* Multi-process mode (§8(e), one partition per GPU over NVLink): after
 * lpsim_load_demand, each process writes its export record (CUDA IPC handles
 * of its migrant receive queues, its two lane-map buffers, its migrant-count
 * array and its barrier flags) into
 * `blob` (LPSIM_IPC_BLOB_BYTES bytes); the caller all-gathers the records in
 * rank order (e.g. torch.distributed) and passes all `world` of them to
 * lpsim_ipc_attach, which maps the peers' memory.  The step kernel then writes
 * migrants and entry-halo bytes straight into the peers' memory from its
 * move and resolve phases and synchronises the GPUs once per step with flags
 * in peer memory; no host round trip per step.
 * lpsim_results / lpsim_trip_state / stats then describe this process's
 * partition: combine arrival_step with an element-wise max and distance_m with
 * a sum over ranks (every trip is held by exactly one partition). */
#define LPSIM_IPC_BLOB_BYTES 512
lpsim_status lpsim_ipc_handle(lpsim_ctx *ctx, void *blob, int64_t size);
lpsim_status lpsim_ipc_attach(lpsim_ctx *ctx, const void *blobs, int64_t size);

/* Host-only plan query (no device): number of cut lanes from upstream
 * partition p to owner partition q (edge owner = partition of its downstream
 * node), out[p*k + q], for the given node partition — the static migrant slot
 * and entry-halo shapes every process derives identically (§8(e)). */
lpsim_status lpsim_plan_cut_lanes(const lpsim_graph *graph, const int32_t *node_part, int32_t k, int64_t *out);

const char *lpsim_last_error(const lpsim_ctx *ctx);
void lpsim_destroy(lpsim_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif
