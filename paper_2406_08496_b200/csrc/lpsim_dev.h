// lpsim_dev.h — device data layout of the B200 LPSim step (product code).
//
// Shared by lpsim_capi.cu (host runtime) and lpsim_step.cu (kernels) only.
// Independent of oracle/ (no shared code).  DESIGN.md §6 describes the HBM
// layout; each field names the paper passage it represents.
//
// Spatial tiling.  The road graph's nodes are split into parts (one per GPU,
// §8(e)) and each part into tiles, one tile per CTA of the persistent step
// kernel.  Edge e = (u -> v) belongs to tile(v); a waiting trip to
// tile(from(first edge)).  Every claim on a cell (entry cells of a node's
// out-edges, lane-change targets on an edge) is then made by vehicles of ONE
// tile (Remark "Switch", resolved with the lowest id, A9), so claims
// resolve in the CTA's shared memory; tiles synchronise only with their
// neighbour tiles (flags), never grid-wide.
#pragma once
#include <cstddef>
#include <cstdint>

namespace lpsim {

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr uint32_t EDGE_BITS = 25;                 // edge id in packed words
constexpr uint32_t EDGE_MASK = (1u << EDGE_BITS) - 1;
constexpr uint32_t LAST_BIT = 1u << 31;             // "this edge is the last route edge"
constexpr uint32_t ROUTE_EDGE_MASK = 0x7FFFFFFFu;   // route entry: edge | (last << 31)
constexpr uint32_t LC_MASK = (1u << 20) - 1;        // Lc = ceil(length) cells, < 2^20 (validated)
constexpr uint32_t LI_SHIFT = 26, LI_MASK = 63;     // neighbour index (see EdgeRec.lc / Ctx.c2)
constexpr uint32_t LI_SAME = 63;                    // "the same tile"
constexpr uint32_t MAX_NB = 62;                     // neighbour tiles per tile
constexpr uint32_t CELL_MASK = 0x7FFFFFFFu;         // global cell index (< 2^31, validated)

// Edge record, 16 B ("number of lanes, its index on lane map, upstream
// intersection, and downstream intersection").
//   base: global lane-map index of (lane 0, cell 0) (a0)
//   lc:   Lc (20 b) | lanes (6 b) << 20 | li << 26: index of tile(dst) in
//         tile(src)'s neighbour list (LI_SAME if tile(src) == tile(dst))
//   meta: rank among the source's out-edges (10 b) | out-degree of the
//         destination (10 b) << 10 | SIG | PHASE | MIRROR
struct __align__(16) EdgeRec {
  uint32_t base;
  uint32_t lc;
  float v0;  // speed limit (IDM v0)
  uint32_t meta;
};
constexpr uint32_t LANES_SHIFT = 20, LANES_MASK = 63;
constexpr uint32_t META_RANK_MASK = 1023;
constexpr uint32_t META_KOUT_SHIFT = 10, META_KOUT_MASK = 1023;
constexpr uint32_t META_SIG = 1u << 28;     // the edge ends at a signalised node (Q30)
constexpr uint32_t META_PHASE = 1u << 29;   // its approach belongs to signal phase 1 (else 0)
constexpr uint32_t META_MIRROR = 1u << 30;  // tile(src) is on another part: the first h_max cells of
                                            // every lane are mirrored into that part's lane map (§8(e))

// Per-trip edge context, 32 B, rewritten only when the trip enters an edge
// ("previous edge, current edge, next edge"), kept in the context array
// of the part that holds the trip.  Everything the move needs from the current
// and the next route edge, so its only dependent loads are lane-map bytes.
struct __align__(16) Ctx {
  uint32_t edge;  // edge | last << 31
  uint32_t cur;   // absolute index of the edge in route[]
  uint32_t c0;    // Lc | lanes << 20 | sig << 26 | phase << 27 | mirror << 28
  float v0;       // speed limit of the edge
  uint32_t c2;    // Lc' | lanes' << 20 | li' << 26 of the next route edge e' (0 on the last edge)
  uint32_t c3;    // allowed lanes [lo, hi] toward e' (Q14): lo | hi << 8 (0 on the last edge)
  uint32_t rn;    // route[cur + 1] = e' | last(e') << 31 (0 on the last edge)
  uint32_t pad;
};
constexpr uint32_t C0_SIG = 1u << 26, C0_PHASE = 1u << 27, C0_MIRROR = 1u << 28;

// Entrant handed to a neighbour tile (§8(e) migrant; P:L503 replication): its
// state at k+1 on the tile's edge.  Its context is written by the sender.
struct __align__(16) MigRec {
  uint32_t id;
  uint32_t ln;    // lane | last << 6 | Lc << 11 (the record's lane word)
  float v;
  uint32_t cell;  // cell 0 of its lane
  uint32_t c4;    // entry cell of its next route edge (NONE on the last edge)
  uint32_t pad[3];
};

// Static description of one tile (host-built).
struct TileInfo {
  uint32_t seg, cap;     // vehicle records: [seg, seg + cap) of the record arrays
  uint32_t pseg, pcap;   // pending departure slots: [pseg, pseg + pcap)
  uint32_t rel0, rel1;   // releases of the tile's slots, in step order: rel[rel0 .. rel1)
  uint32_t nb0, nnb;     // neighbour entries [nb0, nb0 + nnb) of the flat neighbour tables
};

// Dynamic state of one tile (device; written by its CTA between steps).
struct __align__(128) TileCtl {
  uint32_t n[2];         // records of list buffer b (the current list is buffer k & 1)
  uint32_t np[2];        // pending slots of plist buffer b
  uint32_t rel_cur;      // next release to apply
  uint32_t pad0[3];
  unsigned long long ctr[6];  // updates, departures, transitions, lane changes, arrivals, lost claims
  unsigned long long t[4];    // LPSIM_FLAG_TIMING: ns waiting for neighbours, moving, resolving, steps
};
enum { C_UPD = 0, C_DEP, C_TRANS, C_LC, C_ARR, C_LOST, C_N };

constexpr unsigned ERR_TIMEOUT = 1, ERR_CAPACITY = 2, ERR_INVARIANT = 3;

struct ErrCtl {
  unsigned error;      // first error code (0 = none)
  unsigned info;       // site / cell
  unsigned step;       // step of the first error
  unsigned tile;
};

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
  uint32_t sort_every;            // a9 period (steps), 0 = never
};

// Memory of one part (GPU) as seen by this process: its own allocations, or
// CUDA IPC mappings of a peer process's.
struct PartPtrs {
  uint8_t* map[3];              // lane maps, global layout; map[k % 3] = M_k
  unsigned long long* flag;     // [2][nbt]: (step << 32 | migrant count) written by neighbour tiles
  MigRec* chan;                 // [2][chan_total]: migrant channels into the part's tiles
  Ctx* ctx;                     // [n_trips] edge contexts of the trips the part holds
};

struct Global {
  uint32_t tile0;               // first tile of this launch (blockIdx.x + tile0)
  uint32_t n_parts;
  uint32_t nbt;                 // neighbour entries in total
  uint32_t chan_total;          // channel records per buffer
  uint32_t world;               // processes (> 1: flags and peer writes at system scope)
  const TileInfo* tinfo;        // [tiles]
  TileCtl* tctl;                // [tiles]
  const uint8_t* tile_part;     // [tiles]
  const uint32_t* nb_tile;      // [nbt] the neighbour
  const uint32_t* nb_back;      // [nbt] index of this tile's entry in the neighbour's list
  const uint32_t* ch_off;       // [nbt] channel neighbour -> this tile: offset in the part's chan buffer
  const uint32_t* ch_cap;       // [nbt] its capacity (0: the neighbour is not upstream)
  const PartPtrs* parts;        // [n_parts]
  // vehicle records, per-tile segments, double-buffered (list of step k = buffer k & 1)
  uint32_t* rid[2];             // trip id, NONE = dead (left at k; its pcell is cleared at k+1)
  uint32_t* rln[2];             // lane | last << 6 | (mirror part of pcell + 1) << 7 | Lc << 11
  float* rpos[2];
  float* rv[2];
  uint32_t* rcell[2];           // global cell at the snapshot
  uint32_t* rpcell[2];          // cell at the previous snapshot (cleared in M_{k-1}), NONE for entrants
  uint32_t* rc4[2];             // entry cell of the next route edge in this lane (NONE on the last edge)
  uint4* cl;                    // per-tile claim list scratch [seg, seg + cap)
  // graph
  const EdgeRec* edges;
  const uint8_t* edge_mpart;    // [E] part holding the mirror of a META_MIRROR edge
  const uint32_t* route;        // edge | last << 31
  const uint4* rinfo;           // per route position j (not last): {route[j+1], lc of route[j+1], base of
                                // route[j+1], allowed lanes of route[j] toward route[j+1] (Q14)}
  const uint32_t* trip_rstart;  // first route entry of each trip
  int32_t* arrival_step;        // [N]
  int32_t* edge_entry;          // [route entries] t_start per route edge (LPSIM_FLAG_EDGE_TIMES), else null
  // departures (A7): slot = (first edge, lane), owned by tile(from(first edge))
  const uint4* slot_a;          // {entry cell, bitmap offset, width, offset into slot_trip}
  const uint2* slot_b;          // {first edge | last << 31, lane | li << 8}
  const uint32_t* slot_trip;    // trip ids by rank (ascending ids) within each slot
  uint32_t* bm;                 // multi-level release bitmaps (bit = released, not departed)
  uint32_t* slot_nrel;          // released, not departed
  uint32_t* slot_cand;          // lowest released, not departed rank (NONE: empty)
  uint32_t* slot_cid;           // its trip id (rank order = id order within a slot)
  uint2* plist[2];              // pending slots {slot, entry cell}, per-tile segments
  uint4* adm;                   // admit scratch per pending position {slot, trip id, claimed cell | NONE, flags}
  const uint4* rel;             // {slot, rank, step, trip id} per tile in step order
  const uint2* dep;             // [N] departure record: {lane word, entry cell of the second route edge}
  // instrumentation
  unsigned long long* digest_log;  // [digest_cap] digest of snapshot k0 + 1 + i
  uint32_t digest_cap;
  ErrCtl* err;
};

}  // namespace lpsim
