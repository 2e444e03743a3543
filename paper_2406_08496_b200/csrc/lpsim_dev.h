// lpsim_dev.h — device data layout of the B200 LPSim step (product code).
//
// Shared by lpsim_capi.cu (host runtime) and lpsim_step.cu (kernels) only.
// Independent of oracle/ (no shared code).  DESIGN.md §6 describes the HBM
// layout; each field names the paper passage it represents.
#pragma once
#include <cstddef>
#include <cstdint>

namespace lpsim {

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr uint32_t EDGE_BITS = 25;                 // edge id in the packed vehicle word
constexpr uint32_t EDGE_MASK = (1u << EDGE_BITS) - 1;
constexpr uint32_t LANE_SHIFT = 25, LANE_MASK = 63; // lane in bits 25..30
constexpr uint32_t LAST_BIT = 1u << 31;             // "current edge is the last route edge"
constexpr uint32_t ROUTE_EDGE_MASK = 0x7FFFFFFFu;   // route entry: edge | (last << 31)

// Edge record, 16 B ("number of lanes, its index on lane map, upstream
// intersection, and downstream intersection").  meta packs:
//   lanes (6 b) | rank of this edge among its source's out-edges (10 b) |
//   out-degree of its destination node (10 b) | HALO (1 b) | REMOTE (1 b)
struct __align__(16) EdgeRec {
  uint32_t base;    // local lane-map offset of (lane 0, cell 0)
  uint32_t ncells;  // Lc = ceil(length_m)
  float v0;         // speed limit (IDM v0)
  uint32_t meta;
};
constexpr uint32_t META_LANES_MASK = 63;
constexpr uint32_t META_RANK_SHIFT = 6, META_RANK_MASK = 1023;
constexpr uint32_t META_KOUT_SHIFT = 16, META_KOUT_MASK = 1023;
constexpr uint32_t META_HALO = 1u << 26;    // only the first h_max cells per lane are held (entry halo)
constexpr uint32_t META_REMOTE = 1u << 27;  // not held by this partition at all
constexpr uint32_t META_SIG = 1u << 28;     // the edge ends at a signalised node (Q30)
constexpr uint32_t META_PHASE = 1u << 29;   // its approach belongs to signal phase 1 (else 0)
constexpr uint32_t META_MIRROR = 1u << 30;  // owned cut edge: its first h_max cells are mirrored into the
                                            // upstream part's entry halo (PartDev::mirror)

// Claim record of a vehicle contending for a cell (Remark "Switch").
// Its fallback state is already in SoA_{k+1}[idx]; phase C overwrites it with
// the proposal if the claim is won.
struct __align__(16) ClaimRec {
  uint32_t idx;      // index of the vehicle in SoA_{k+1}
  uint32_t id;       // trip id (the tie-break key, A9)
  uint32_t cell;     // contended local cell
  uint32_t el_new, cur_new;
  float pos_new, v_new;
  uint32_t fb_cell;  // cell of the fallback state
  uint32_t fb_byte;  // fallback lane-map byte | kind << 8 (1 transition, 2 lane change)
  uint32_t pcell;    // cell held at snapshot k
  uint32_t x[6];     // edge context of the proposal (Ctx in lpsim_step.cu), prepared in phase A
  uint32_t pad[4];
};

static_assert(sizeof(ClaimRec) % 16 == 0, "claim records are loaded as uint4");

// Migrant (§8(e)): a vehicle that won the entry cell of a cut edge on the
// upstream partition and continues on the edge owner, at pos 0 of that edge.
// The sender writes it into the owner's receive queue in phase C of step k;
// the owner moves it in phase A of step k+1 as an entry of its SoA.
struct __align__(16) MigSlot {
  uint32_t id;
  uint32_t el;       // edge | lane << 25 | last << 31
  float v;
  uint32_t cur;      // absolute route index of the edge
  uint32_t cell;     // cell 0 of its lane in the owner's local lane map
  uint32_t pad[3];
};

// Control block of one partition (device memory).
struct PartCtl {
  unsigned n_veh[2];       // vehicles in SoA buffer b
  unsigned n_dead[2];      // dead entries (left vehicles) in SoA buffer b
  unsigned n_res[2];       // SoA entries reserved in phase A for the departures of the step (buffer b)
  unsigned error;          // first device-side error code (0 = none)
  unsigned error_info;
  unsigned long long updates, departures, transitions, lane_changes, arrivals, lost_claims;
  unsigned long long digest;   // digest of the snapshot being built
  unsigned long long exch_ns;  // exchange phase device time (globaltimer)
  unsigned pad[4];
};

struct GridCtl {
  unsigned bar_count;
  unsigned bar_gen;
  unsigned error;
  unsigned err_step;             // step of the first error (0xFFFFFFFF = none)
  unsigned long long step;       // k of the current snapshot
  unsigned xgo;                  // multi-process: epoch of the last cross-GPU barrier block 0 completed
  unsigned xgo_pad;
  unsigned long long digest[2];  // digest accumulators by step parity
  unsigned long long t_phase[4]; // LPSIM_FLAG_TIMING: ns spent in phases A, C, X (barrier to barrier)
  unsigned long long* t_block;   // LPSIM_FLAG_TIMING: per CTA [grid][TB_N]: ns from phase start to the
                                 // CTA's last chunk (A, C), phase starts, barrier arrivals, barrier waits
};

constexpr unsigned long long TB_N = 24;  // words of GridCtl::t_block per CTA
constexpr unsigned ERR_TIMEOUT = 1, ERR_CAPACITY = 2, ERR_INVARIANT = 3;
constexpr unsigned NSH = 64;        // shards of the hot work lists
constexpr unsigned SH_STRIDE = 32;  // shard counters 128 B apart

struct PartDev {
  // graph (local view)
  const EdgeRec* edges;       // [E] (remote edges flagged)
  uint8_t* map[2];            // lane maps; map[k & 1] is M_k, map[(k + 1) & 1] M_{k+1} (§8 a0/a7)
  uint32_t* claim;            // [cells] NONE = unclaimed
  uint32_t ncells;            // local cells (owned + halo)
  // vehicles: double-buffered SoA (active on-road vehicles only)
  uint32_t* vid[2];
  uint32_t* vel[2];           // edge | lane << 25 | last << 31
  float* vpos[2];
  float* vv[2];
  uint32_t* vcur[2];          // absolute index of the current edge in route[]
  uint32_t* vcell[2];         // local lane-map cell at the current snapshot
  uint32_t* vpcell[2];        // cell held at the previous snapshot (to clear), NONE for entrants
  // cached edge context of each vehicle (see Ctx in lpsim_step.cu); buffer xb is
  // current — written only when a vehicle enters an edge, swapped by the sort
  uint32_t* xc0[2];
  float* xv0[2];
  uint32_t* xc2[2];
  uint32_t* xc3[2];
  uint32_t* xc4[2];
  uint32_t* xrn[2];
  uint32_t xb;
  uint32_t veh_cap;
  // departures (A7): per (first edge, lane) slot, a multi-level bitmap over
  // the slot's trips in id order; bit set = released (depart step <= k) and
  // not yet departed.  Releases set bits in phase A, departures clear them in
  // phase C; summary bits are exact at every barrier.
  uint32_t n_slot_total;
  const uint4* slot_info;     // per slot: {entry cell (e1, l0, 0), bitmap offset, width n, offset into slot_trip}
  const uint32_t* slot_trip;  // trip ids, ascending within a slot
  uint32_t* bm;
  // admit positions of step k = the pending slots carried over from step k-1 (sharded list)
  // followed by the release list of step k (rs_*: the distinct slots of the trips released at k)
  uint32_t* slot_list[2];     // carried-over slots, sharded: [NSH * slot_shcap]
  uint4* slot_li[2];          // their slot_info
  uint2* slot_lc[2];          // their candidate {rank, trip id} (lowest released, not departed; NONE = empty)
  uint2* slot_cw;             // [S] candidate of a slot not in the carried list (NONE when empty)
  uint32_t* slot_nrel;        // [S] released trips not yet departed
  uint32_t* sh_slot[2];       // shard counters of slot_list[b] ([NSH * SH_STRIDE])
  uint32_t slot_shcap;
  uint32_t* slot_relk;        // [S] = k+1 while the slot is in the release list of step k+1 (phase A of k)
  uint4* slot_cand;           // per admit position: {rank | NONE, trip id, claimed entry cell | NONE, slot}
  uint4* slot_ci;             // per admit position: the slot's slot_info
  // departure state of each trip of this partition, prepared at load (k_trip_ctx):
  // packed edge/lane/last on the first edge, and its edge context
  uint32_t* tel;              // [N] (indexed by trip id; only own trips are set)
  uint32_t* tx[6];            // [N] Ctx words
  const uint4* rel4;          // releases in depart-step order: {slot, rank in slot, bitmap offset, width}
  const uint32_t* rel_ptr;    // [rel_steps + 2]
  uint32_t rel_steps;
  const uint32_t* rs_ptr;     // [rel_steps + 2] release lists by step
  const uint32_t* rs_slot;    // distinct slots released at each step
  const uint4* rs_info;       // their slot_info
  const uint2* rs_cand;       // their lowest trip released at that step {rank, trip id}
  const uint32_t* rs_r2;      // their second lowest rank released at that step (NONE if one release)
  uint4* slot_cs;             // per admit position, from phase A: {the candidate's successor rank if it
                              //   departs, its reserved entry of the next pending list, its reserved SoA
                              //   entry (offset past the step's in-place count), 0}
  ClaimRec* crec[2];          // claim records at the claimant's SoA index: [veh_cap]
  uint32_t* cbits[2];         // claimant bitmap of SoA_k (one ballot word per warp): [veh_cap / 32 + 1]
  // exchange (num_parts > 1), §8(e), written straight into the peer's memory by phases A and C:
  // receive queues of the migrants on this part at snapshot k (inq[k & 1]); sender u writes its
  // migrants of a step into its region [rq_off[u], rq_off[u] + cut lanes u -> this part)
  MigSlot* inq[2];
  uint32_t n_in;              // incoming cut lanes (queue capacity)
  const uint32_t* rq_off;     // [num_parts + 1] region offsets by sender
  const uint32_t* send_off;   // [num_parts] offset of this part's region in each receiver's queue
  const uint2* halo_dst;      // [E] for halo edges: {owner, cell 0 of lane 0 in the owner's map}
  const uint2* mirror;        // [E] for META_MIRROR edges: {upstream part, halo cell 0 of lane 0 there}
  uint32_t halo_lo;           // the entry halos are cells [halo_lo, ncells) of this part's map
  PartCtl* ctl;
};

// phase A's next-round prefetch walks these pointer pairs as tables
static_assert(offsetof(PartDev, vel) == offsetof(PartDev, vid) + 16 && offsetof(PartDev, vpos) == offsetof(PartDev, vid) + 32 &&
              offsetof(PartDev, vv) == offsetof(PartDev, vid) + 48 && offsetof(PartDev, vcur) == offsetof(PartDev, vid) + 64 &&
              offsetof(PartDev, vcell) == offsetof(PartDev, vid) + 80, "SoA pointer pairs are consecutive");
static_assert(offsetof(PartDev, xv0) == offsetof(PartDev, xc0) + 16 && offsetof(PartDev, xc2) == offsetof(PartDev, xc0) + 32 &&
              offsetof(PartDev, xc3) == offsetof(PartDev, xc0) + 48 && offsetof(PartDev, xc4) == offsetof(PartDev, xc0) + 64 &&
              offsetof(PartDev, xrn) == offsetof(PartDev, xc0) + 80, "context pointer pairs are consecutive");

struct Params {
  float dt, a, b, s0, T;
  int delta;
  float x0, g_a, g_b, alpha_i, alpha_a, alpha_b;
  float sigma_a_s3, sigma_b_s3;   // σ·√3 (Q15)
  float c_ab;                     // 2·sqrt(a·b)
  float dt2, half_a_dt2;          // Δt², (0.5·a)·Δt²
  int h_min, h_max, lc_n;
  int sig_cycle;                  // signal cycle in steps (Q30), 0 = unsignalised
  uint32_t seed_lo, seed_hi;
  uint32_t flags;
};

struct Global {
  // partitions simulated by this process: parts[part0 .. part0 + n_local)
  uint32_t part0, n_local;
  // multi-process mode (one partition per GPU, §8(e)): flag barrier over peer memory
  uint32_t world, rank;
  uint32_t* xflag_local;        // [world] written by the peers (epoch reached)
  uint32_t** xflag_peer;        // [world] peer flag arrays (CUDA IPC mappings)
  // migrant counts [2][n_parts][n_parts] (parity of the snapshot the migrants are on, sender,
  // receiver); multi-process: each GPU's copy, the sender's row pushed to the peers at the barrier
  uint32_t* mig_cnt;
  uint32_t** mig_cnt_peer;      // [world] peers' copies (CUDA IPC mappings), multi-process only
  const uint32_t* route;        // edge | last << 31
  const uint32_t* trip_rstart;  // first route entry of each trip
  int32_t* arrival_step;        // [N]
  int32_t* edge_entry;          // [route entries] t_start per route edge (LPSIM_FLAG_EDGE_TIMES), else null
  unsigned long long* digest_log;
  uint32_t digest_cap;
  uint32_t n_parts;
  PartDev* parts;               // [n_parts] (device memory)
  GridCtl* grid;
  unsigned long long* ctr_block;  // [grid][5] per-CTA event counters: transitions, lane changes,
                                  // lost claims, departures, arrivals (summed by the host)
};

}  // namespace lpsim
