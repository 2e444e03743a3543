// lpsim_step.cu — sm_100a kernels of the LPSim per-timestep vehicle update.
//
// Method: arXiv 2406.08496, Eq. (1) P:L239-242 (every vehicle at k+1 is a
// function of the snapshot at k), Alg. 1, lane map P:L256-266,
// Remarks P:L247-251.  Readings Qnn: DESIGN.md §3.  Layout: lpsim_dev.h.
//
// One persistent kernel (k_tile) executes whole steps.  CTA = tile: a region
// of the road graph that owns the in-edges of its nodes, their vehicles and
// the departures of its nodes.  Step k of a tile:
//   1  releases of step k into its departure bitmaps (A7)
//   2  wait until every neighbour tile finished step k-1 (flags in memory;
//      no grid-wide barrier), read the migrant counts they left
//   3  for every input (own records, migrants): clear its k-1 cell in M_{k-1}
//      (three lane maps: M_{k-1} is read by nobody in step k), probe M_k (a3),
//      IDM + kinematics (a4), transition (a5), lane change (a6); claims go to a
//      shared-memory hash table (cell -> lowest id, A9); the output record is
//      written at its compacted index (a2)
//   4  admit departures of its pending slots (A7)
//   5  resolve claims: winners commit, losers keep their fallback; entrants of
//      another tile's edge go to that tile's channel (a8), possibly on
//      another GPU over NVLink; every byte of M_{k+1} is written (a7)
//   6  publish "step k done" (+ migrant count) to every neighbour tile.
// Floating point follows the fixed IEEE fp32 operation order of DESIGN.md §3
// (compiled with --fmad=false, no fast math): integer state is bit-exact
// against the oracle.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lpsim.h"  // LPSIM_FLAG_* (the C ABI flags the kernels honour)
#include "lpsim_kernels.h"

namespace lpsim {

constexpr int BS = TILE_BS;
constexpr unsigned long long TIMEOUT_NS = 20000000000ull;  // 20 s without progress of a neighbour
constexpr unsigned HT_BITS = TILE_HT_BITS, HT = 1u << HT_BITS;  // claim hash table entries per CTA
constexpr unsigned LCQ = 512;                                  // lane-change candidates held per CTA
constexpr unsigned long long HT_EMPTY = ~0ull;

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void set_error(const Global& G, unsigned code, unsigned info, uint32_t k, uint32_t tile) {
  if (atomicCAS(&G.err->error, 0u, code) == 0u) {
    G.err->info = info;
    G.err->step = k;
    G.err->tile = tile;
  }
}
__device__ __forceinline__ bool has_error(const Global& G) { return *((volatile unsigned*)&G.err->error) != 0u; }

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11), counter (id, k, stream, 0) (Q27)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                       uint32_t k1, uint32_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// ε = ((Σ_j x_j >> 10)·2^-22 − 2)·σ√3  (Q15); the first two steps are exact
__device__ __forceinline__ float eps_draw(const Params& P, uint32_t id, uint32_t k, uint32_t stream, float sig_s3) {
  uint32_t w[4];
  philox(id, k, stream, 0u, P.seed_lo, P.seed_hi, w);
  const uint32_t s = (w[0] >> 10) + (w[1] >> 10) + (w[2] >> 10) + (w[3] >> 10);
  return __fmul_rn(__fadd_rn(__fmul_rn((float)s, 0x1p-22f), -2.0f), sig_s3);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// state digest term (test instrumentation; same definition as DESIGN.md §7)
__device__ __forceinline__ uint64_t veh_hash(uint32_t id, uint32_t edge, uint32_t lane, float pos, float v,
                                             uint32_t cursor) {
  uint64_t h = mix64((uint64_t)id);
  h = mix64(h ^ (uint64_t)edge);
  h = mix64(h ^ (uint64_t)lane);
  h = mix64(h ^ (uint64_t)(uint32_t)(int)pos);
  h = mix64(h ^ (uint64_t)__float_as_uint(pos));
  h = mix64(h ^ (uint64_t)__float_as_uint(v));
  h = mix64(h ^ (uint64_t)cursor);
  return h;
}

__device__ __forceinline__ EdgeRec load_edge(const EdgeRec* edges, uint32_t e) {
  const uint4 r = __ldg(reinterpret_cast<const uint4*>(edges) + e);
  EdgeRec E;
  E.base = r.x; E.lc = r.y; E.v0 = __uint_as_float(r.z); E.meta = r.w;
  return E;
}

__device__ __forceinline__ uint8_t speed_byte(float v) {  // byte = speed (m/s), cap 254
  return (uint8_t)(int)fminf(v, 254.0f);
}

// ---------------------------------------------------------------------------
// lane-map byte stores.  LPSIM_FLAG_CHECKS: a byte of M_{k+1} may only be
// written over a free cell ("one byte can only be occupied by one
// vehicle"); the store is then an atomicCAS on the enclosing word.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool put_byte_checked(uint8_t* map, uint32_t cell, uint8_t b) {
  unsigned* w = reinterpret_cast<unsigned*>(map + (cell & ~3u));
  const unsigned sh = (cell & 3u) * 8u;
  unsigned old = *((volatile unsigned*)w);
  for (;;) {
    if (((old >> sh) & 255u) != 255u) return false;
    const unsigned nw = (old & ~(255u << sh)) | ((unsigned)b << sh);
    const unsigned got = atomicCAS(w, old, nw);
    if (got == old) return true;
    old = got;
  }
}

// ---------------------------------------------------------------------------
// departure bitmaps (A7): multi-level, 32-ary; level 0 = 1 top word
// ---------------------------------------------------------------------------
__device__ __forceinline__ int bm_depth(uint32_t n) {
  int d = 1;
  uint64_t cap = 32;
  while (cap < n) { cap *= 32; ++d; }
  return d;
}
__device__ __forceinline__ uint32_t bm_words(uint32_t n, int d, int i) {
  uint32_t shift = 5u * (uint32_t)(d - i);
  return (uint32_t)(((uint64_t)n + (1ull << shift) - 1) >> shift);
}
constexpr int BM_MAXD = 4;
// Departure of rank r (the slot's lowest set bit): clear it, return the next lowest set rank or NONE.
// Only the slot's owner tile touches its bitmap, and the releases of the step are applied before
// its admits (barrier), so the words read here are exact.
__device__ uint32_t bm_next(uint32_t* bm, uint32_t n, uint32_t r, bool empty_after) {
  const int d = bm_depth(n);
  uint32_t offs[BM_MAXD];
  uint32_t off = 0, loff = 0;
#pragma unroll
  for (int i = 0; i < BM_MAXD; ++i) {
    offs[i] = off;
    if (i == d - 1) loff = off;
    if (i < d) off += bm_words(n, d, i);
  }
  const uint32_t bl = 1u << (r & 31u);
  const uint32_t leaf = atomicAnd(&bm[loff + (r >> 5)], ~bl) & ~bl;
  if (empty_after || leaf != 0u) {
    if (empty_after) {  // the slot is empty: clear r's ancestors (each bit's child word just emptied)
#pragma unroll
      for (int i = 0; i < BM_MAXD - 1; ++i)
        if (i < d - 1) {
          const uint32_t x = r >> (5 * (d - 1 - i));
          atomicAnd(&bm[offs[i] + (x >> 5)], ~(1u << (x & 31u)));
        }
      return NONE;
    }
    return (r & ~31u) | (uint32_t)(__ffs(leaf) - 1);
  }
  // r's leaf word emptied: climb, clearing each emptied word's bit, to the first non-empty ancestor
  uint32_t x = NONE;
  int lvl = -1;
#pragma unroll
  for (int i = BM_MAXD - 2; i >= 0; --i) {
    if (i < d - 1 && lvl < 0) {
      const uint32_t y = r >> (5 * (d - 1 - i));
      const uint32_t b = 1u << (y & 31u);
      const uint32_t rem = atomicAnd(&bm[offs[i] + (y >> 5)], ~b) & ~b;
      if (rem) {
        x = (y & ~31u) | (uint32_t)(__ffs(rem) - 1);
        lvl = i;
      }
    }
  }
  if (lvl < 0) return NONE;  // not reached: the count says a trip is waiting
#pragma unroll
  for (int l = 1; l < BM_MAXD; ++l)  // descend from level lvl + 1 to the leaf
    if (l > lvl && l < d) x = (x << 5) | (uint32_t)(__ffs(*((volatile uint32_t*)&bm[offs[l] + x])) - 1);
  return x;
}

__device__ __forceinline__ void bm_set(uint32_t* bm, uint32_t n, uint32_t r) {
  const int d = bm_depth(n);
  uint32_t off = 0;
  for (int i = 0; i < d - 1; ++i) off += bm_words(n, d, i);
  uint32_t x = r;
  for (int i = d - 1; i >= 0; --i) {  // leaf first, then the summaries
    atomicOr(&bm[off + (x >> 5)], 1u << (x & 31u));
    x >>= 5;
    if (i > 0) off -= bm_words(n, d, i - 1);
  }
}

// ---------------------------------------------------------------------------
// vectorised lane-map scans: occupancy bit per byte (byte != 255)
// ---------------------------------------------------------------------------
// 8 bytes -> 8 bits: 0x80 in every byte != 0xFF (borrow-free), then the byte MSBs gathered by a multiply
__device__ __forceinline__ uint32_t occ8(uint64_t w) {
  const uint64_t x = ~w;
  const uint64_t t = (((x & 0x7F7F7F7F7F7F7F7Full) + 0x7F7F7F7F7F7F7F7Full) | x) & 0x8080808080808080ull;
  return (uint32_t)(((t >> 7) * 0x0102040810204080ull) >> 56);
}
__device__ __forceinline__ uint64_t occ16(ulonglong2 q) { return (uint64_t)occ8(q.x) | ((uint64_t)occ8(q.y) << 8); }
__device__ __forceinline__ bool all_free(ulonglong2 q) { return (q.x & q.y) == ~0ull; }
// occupancy of the 48 bytes [a, a+48), a multiple of 16; chunks past `hi` are not loaded
__device__ __forceinline__ uint64_t occ48(const uint8_t* M, uint32_t a, uint32_t hi) {
  const ulonglong2* q = reinterpret_cast<const ulonglong2*>(M + a);
  const ulonglong2 ones = make_ulonglong2(~0ull, ~0ull);
  const ulonglong2 q0 = q[0];
  const ulonglong2 q1 = (a + 16u <= hi) ? q[1] : ones;
  const ulonglong2 q2 = (a + 32u <= hi) ? q[2] : ones;
  uint64_t m = 0;
  if (!all_free(q0)) m = occ16(q0);
  if (!all_free(q1)) m |= occ16(q1) << 16;
  if (!all_free(q2)) m |= occ16(q2) << 32;
  return m;
}
// first occupied byte address in [lo, hi] (hi >= lo), or NONE
__device__ __noinline__ uint32_t scan_first(const uint8_t* M, uint32_t lo, uint32_t hi) {
  for (uint32_t a = lo & ~15u;; a += 48u) {
    uint64_t m = occ48(M, a, hi);
    if (lo > a) m &= ~0ull << (lo - a);
    if (hi - a < 47u) m &= (2ull << (hi - a)) - 1ull;
    if (m) return a + (uint32_t)(__ffsll((long long)m) - 1);
    if (hi - a < 48u) return NONE;
  }
}
// last occupied byte address in [lo, hi] (hi >= lo), or NONE
__device__ __noinline__ uint32_t scan_last(const uint8_t* M, uint32_t lo, uint32_t hi) {
  for (uint32_t a = hi & ~15u;;) {
    const uint32_t s = a >= 32u ? a - 32u : 0u;  // span [s, s+48) ends at a+16 > hi
    uint64_t m = occ48(M, s, hi);
    if (lo > s) m &= ~0ull << (lo - s);
    if (hi - s < 47u) m &= (2ull << (hi - s)) - 1ull;
    if (m) return s + 63u - (uint32_t)__clzll((long long)m);
    if (lo >= s || s == 0u) return NONE;
    a = s - 16u;
  }
}

// allowed lanes [lo, hi] on e toward e' (Q14): L = lanes(e), K = out-degree of to(e), r = rank of e'
__device__ __forceinline__ uint32_t lane_range(uint32_t L, uint32_t K, uint32_t r) {
  const uint32_t lo = (r * L) / K;
  uint32_t hi = ((r + 1u) * L + K - 1u) / K;
  hi = (hi >= 1u ? hi - 1u : 0u);
  if (hi < lo) hi = lo;
  return lo | (hi << 8);
}

__device__ __forceinline__ uint32_t ctx_c0(const EdgeRec& E) {
  return (E.lc & (LC_MASK | (LANES_MASK << LANES_SHIFT))) | ((E.meta & META_SIG) ? C0_SIG : 0u) |
         ((E.meta & META_PHASE) ? C0_PHASE : 0u) | ((E.meta & META_MIRROR) ? C0_MIRROR : 0u);
}

// context of a trip on route position `cur` (route[cur] = er = edge | last) in lane l: the current
// edge's record and the route-position table entry of cur (the next edge's data), two independent
// loads; c4 = entry cell of the next route edge in the lane the trip will use there (Q21)
__device__ __forceinline__ Ctx make_ctx(const EdgeRec* __restrict__ edges, const uint4* __restrict__ rinfo,
                                        uint32_t er, uint32_t cur, uint32_t l, uint32_t& c4) {
  const EdgeRec E = load_edge(edges, er & ROUTE_EDGE_MASK);
  const bool last = (er & LAST_BIT) != 0u;
  const uint4 ri = last ? make_uint4(0u, 0u, 0u, 0u) : __ldg(&rinfo[cur]);
  Ctx x;
  x.edge = er;
  x.cur = cur;
  x.c0 = ctx_c0(E);
  x.v0 = E.v0;
  x.pad = 0;
  x.rn = ri.x;
  x.c2 = ri.y;
  x.c3 = ri.w;
  c4 = last ? NONE : ri.z + min(l, ((ri.y >> LANES_SHIFT) & LANES_MASK) - 1u) * (ri.y & LC_MASK);
  return x;
}

// the record's packed lane word: lane | last << 6 | (mirror part of pcell + 1) << 7 | Lc << 11
constexpr uint32_t LN_LANE = 63u, LN_LAST = 1u << 6, LN_PM_SHIFT = 7, LN_PM_MASK = 15u, LN_LC_SHIFT = 11;
__device__ __forceinline__ uint32_t ln_pack(uint32_t lane, bool last, uint32_t pm1, uint32_t Lc) {
  return lane | (last ? LN_LAST : 0u) | (pm1 << LN_PM_SHIFT) | (Lc << LN_LC_SHIFT);
}

// ---------------------------------------------------------------------------
// per-vehicle move: a3 probe, a4 IDM + kinematics, a5, a6 candidate
// ---------------------------------------------------------------------------
struct MoveOut {
  float pos, v;          // state at k+1 (or the fallback of a claimant)
  uint32_t cell_new;
  bool claimant, finished;
  bool lc;               // a lane change is possible: decided by the CTA's lane-change batch
  float plc;             // its probability (Eq. Lane Change, Q13)
  float cv;              // speed proposed by a transition
};

// the probe windows: own lane [cell+1, cell+H], next edge's entry lane [c4, c4 + reach].  Lc and
// `last` come with the record, so both windows are requested before the context arrives (the three
// loads are in flight together).
__device__ __forceinline__ void move_vehicle(const Params& P, const uint8_t* Mk, uint32_t gp, uint32_t l, bool last,
                                             int Lc, float p, float v, uint32_t cell, uint32_t c4, const Ctx& X,
                                             MoveOut& o) {
  const int c = (int)p;  // p >= 0: truncation == floor
  const uint32_t lane0 = cell - (uint32_t)c;
  // H = min(H_max, max(H_min, ceil(2Δt·v))) (Alg. 1 l.11, Q7)
  int H = (int)ceilf(__fmul_rn(__fmul_rn(2.0f, P.dt), v));
  H = max(H, P.h_min);
  H = min(H, P.h_max);
  o.claimant = false;
  o.finished = false;
  o.lc = false;
  // a3: leader probe — own lane cells c+1 .. min(c+H, Lc-1), then the next edge's entry lane (Q10)
  const int lim = min(c + H, Lc - 1);
  const bool near = !last && c + H >= Lc;
  const uint32_t a1 = (cell + 1u) & ~15u, h1 = lane0 + (uint32_t)max(lim, c + 1);
  const uint32_t a2 = c4 & ~15u;
  const bool fit1 = h1 - a1 < 48u;
  uint64_t m1 = 0, m2 = 0;
  if (lim >= c + 1 && fit1) m1 = occ48(Mk, a1, h1);
  if (near) m2 = occ48(Mk, a2, c4 + (uint32_t)(H - 1));  // reach <= H - 1 (masked below)
  bool found = false, same = false;
  int gap = 0, vf = 0, cf = 0;
  // Q30: a red signal at the end of e is a stopped leader just past the last cell for a vehicle whose
  // probe reaches the line; gp = the phase that is green at step k
  const bool red = near && (X.c0 & C0_SIG) != 0u && ((X.c0 & C0_PHASE) ? 1u : 0u) != gp;
  const int reach = near ? min(c + H - Lc, (int)(X.c2 & LC_MASK) - 1) : 0;
  const uint32_t h2 = near ? c4 + (uint32_t)reach : 0u;
  const bool fit2 = h2 - a2 < 48u;
  if (lim >= c + 1) {
    uint32_t hit;
    if (fit1) {
      uint64_t m = m1 & (~0ull << (cell + 1u - a1));
      m &= (2ull << (h1 - a1)) - 1ull;
      hit = m ? a1 + (uint32_t)(__ffsll((long long)m) - 1) : NONE;
    } else {
      hit = scan_first(Mk, cell + 1u, h1);
    }
    if (hit != NONE) {
      found = true; same = true;
      cf = (int)(hit - lane0);
      gap = cf - c;
      vf = Mk[hit];
    }
  }
  bool entry_free = true;  // cell 0 of the next edge's entry lane, M_k
  if (red) {
    entry_free = false;
    if (!found) {  // the stop line: the no-overtake clamp at cell Lc keeps the vehicle on this edge
      found = true; same = true;
      cf = Lc;
      gap = Lc - c;
      vf = 0;
    }
  } else if (near) {
    uint32_t hit;
    if (fit2) {
      uint64_t m = m2 & (~0ull << (c4 - a2));
      m &= (2ull << (h2 - a2)) - 1ull;
      hit = m ? a2 + (uint32_t)(__ffsll((long long)m) - 1) : NONE;
      entry_free = ((m2 >> (c4 - a2)) & 1ull) == 0ull;
    } else {
      hit = scan_first(Mk, c4, h2);
      entry_free = Mk[c4] == 255;
    }
    if (!found && hit != NONE) {
      found = true;
      cf = (int)(hit - c4);
      gap = (Lc - c) + cf;
      vf = Mk[hit];
    }
  }

  // a4: IDM (Eq. Car Following, Q3/Q4/Q9), fixed op order
  const float r = __fdiv_rn(v, X.v0);
  float rd;  // (v/v0)^δ by squaring, LSB first (Q6); δ = 4 is (r·r)·(r·r) of that sequence
  if (P.delta == 4) {
    const float r2 = __fmul_rn(r, r);
    rd = __fmul_rn(r2, r2);
  } else {
    rd = 1.0f;
    float base = r;
    for (int dd = P.delta; dd > 0; dd >>= 1) {
      if (dd & 1) rd = __fmul_rn(rd, base);
      base = __fmul_rn(base, base);
    }
  }
  float acc;
  if (!found) {
    acc = __fmul_rn(P.a, __fsub_rn(1.0f, rd));
  } else {
    const float dv = __fsub_rn(v, (float)vf);
    float t = __fadd_rn(__fmul_rn(v, P.T), __fdiv_rn(__fmul_rn(v, dv), P.c_ab));
    t = fmaxf(0.0f, t);
    const float ss = __fadd_rn(P.s0, t);
    const float q = __fdiv_rn(ss, (float)gap);
    acc = __fmul_rn(P.a, __fsub_rn(__fsub_rn(1.0f, rd), __fmul_rn(q, q)));
  }
  // kinematics (Q11): ballistic, stop within the step
  float vn = __fadd_rn(v, __fmul_rn(acc, P.dt));
  float dx;
  if (!found && (P.flags & LPSIM_FLAG_VFREE)) {
    // ablation: the literal "v <- v_free" of Alg. 1: v' = v0, dx = (v + v0)/2 * dt
    vn = X.v0;
    dx = __fmul_rn(__fmul_rn(0.5f, __fadd_rn(v, X.v0)), P.dt);
  } else if (vn < 0.0f) {
    dx = (acc < 0.0f) ? __fdiv_rn(-__fmul_rn(__fmul_rn(0.5f, v), v), acc) : 0.0f;
    vn = 0.0f;
  } else {
    dx = __fadd_rn(__fmul_rn(v, P.dt), __fmul_rn(__fmul_rn(0.5f, acc), P.dt2));
  }
  float pn = __fadd_rn(p, dx);
  vn = fminf(vn, 254.0f);
  if (found && same && (int)pn >= cf) {  // no overtaking
    pn = fmaxf(p, (float)(cf - 1));
    vn = fminf(vn, (float)vf);
  }

  if (pn >= (float)Lc) {
    // a5: intersection (Alg. 1 l.15-16; Remark P:L249)
    if (last) {  // Q24
      o.finished = true;
      return;
    }
    // fallback: wait at the stop line (Q23); the claim is on the entry cell c4 (Q20, Q21)
    o.pos = fmaxf(p, (float)(Lc - 1));
    o.v = 0.0f;
    o.cell_new = lane0 + (uint32_t)(Lc - 1);
    o.claimant = entry_free;
    o.cv = vn;
    return;
  }
  o.pos = pn;
  o.v = vn;
  const int cn = (int)pn;
  o.cell_new = lane0 + (uint32_t)cn;
  // a6: mandatory lane change candidate (Eq. Lane Change, Q13-Q14); decided by the lane-change batch
  if (!last && cn >= 1) {
    const uint32_t lo = X.c3 & 255u, hi = (X.c3 >> 8) & 255u;
    if (l < lo || l > hi) {
      const float x = __fsub_rn((float)Lc, p);
      float plc = __fdiv_rn(__fsub_rn(P.x0, x), P.x0);
      plc = fminf(fmaxf(plc, 0.0f), 1.0f);
      if (plc > 0.0f) {  // u in [0, 1): no change for plc == 0
        o.lc = true;
        o.plc = plc;
      }
    }
  }
}

// The lane-change decision (Eq. Lane Change P:L222-225, Eq. Gap Acceptance P:L228-235, Q13-Q17): the
// Bernoulli draw, then the target cell, lead and lag in the target lane of M_k (one round of loads:
// the window [cn-n, cn+n]), the critical gaps and the lag's kinematic bound.  v = the step-k speed;
// returns the target cell or NONE.
__device__ __forceinline__ uint32_t lc_decide(const Params& P, const uint8_t* Mk, uint32_t k, uint32_t id, float v,
                                              float plc, uint32_t lane0, uint32_t l, int cn, int Lc, uint32_t lo,
                                              uint32_t& tl_out) {
  const int tl = l < lo ? (int)l + 1 : (int)l - 1;
  tl_out = (uint32_t)tl;
  bool draw = plc >= 1.0f;  // u in [0, 1): the draw decides only for 0 < plc < 1
  if (plc > 0.0f && plc < 1.0f) {
    uint32_t w[4];
    philox(id, k, 0u, 0u, P.seed_lo, P.seed_hi, w);
    draw = __fmul_rn((float)(w[0] >> 8), 0x1p-24f) < plc;
  }
  if (!draw) return NONE;
  const uint32_t tl0 = (uint32_t)((int)lane0 + (tl - (int)l) * Lc);
  const uint32_t tc = tl0 + (uint32_t)cn;
  const int n = P.lc_n;
  const uint32_t wlo = tl0 + (uint32_t)max(cn - n, 0), whi = tl0 + (uint32_t)min(cn + n, Lc - 1);
  const uint32_t aw = wlo & ~15u;
  bool tfree = false;
  uint32_t ld = NONE, lg = NONE;
  if (whi - aw < 96u) {
    const uint64_t w0 = occ48(Mk, aw, whi);
    const uint64_t w1 = (aw + 48u <= whi) ? occ48(Mk, aw + 48u, whi) : 0ull;
    const unsigned bt = tc - aw;  // bit of the target cell
    tfree = ((bt < 48u ? (w0 >> bt) : (w1 >> (bt - 48u))) & 1ull) == 0ull;
    // lead: first occupied in (tc, whi]; lag: last occupied in [wlo, tc)
    const uint64_t lo_mask0 = w0 & ~((bt + 1u >= 48u) ? 0xFFFFFFFFFFFFull : ((1ull << (bt + 1u)) - 1ull));
    const uint64_t lo_mask1 = w1 & ((bt + 1u > 48u) ? ~((1ull << (bt + 1u - 48u)) - 1ull) : ~0ull);
    const unsigned hb = whi - aw;
    const uint64_t hm0 = hb >= 47u ? 0xFFFFFFFFFFFFull : ((2ull << hb) - 1ull);
    const uint64_t hm1 = hb >= 48u ? ((2ull << (hb - 48u)) - 1ull) : 0ull;
    const uint64_t f0 = lo_mask0 & hm0, f1 = lo_mask1 & hm1;
    if (f0) ld = aw + (uint32_t)(__ffsll((long long)f0) - 1);
    else if (f1) ld = aw + 48u + (uint32_t)(__ffsll((long long)f1) - 1);
    const unsigned lb0 = wlo - aw;
    const uint64_t b0 = w0 & ((bt >= 48u) ? 0xFFFFFFFFFFFFull : ((1ull << bt) - 1ull)) & (~0ull << lb0);
    const uint64_t b1 = (bt > 48u) ? (w1 & ((1ull << (bt - 48u)) - 1ull)) : 0ull;
    if (b1) lg = aw + 48u + 63u - (uint32_t)__clzll((long long)b1);
    else if (b0) lg = aw + 63u - (uint32_t)__clzll((long long)b0);
  } else {
    tfree = Mk[tc] == 255;
    if (tfree) {
      ld = (cn + 1 <= Lc - 1) ? scan_first(Mk, tc + 1u, whi) : NONE;
      lg = scan_last(Mk, wlo, tc - 1u);
    }
  }
  if (!tfree) return NONE;
  const bool has_ld = ld != NONE, has_lg = lg != NONE;
  const int g_ld = has_ld ? (int)(ld - tc) : 0, b_ld = has_ld ? Mk[ld] : 0;
  const int g_lg = has_lg ? (int)(tc - lg) : 0, b_lg = has_lg ? Mk[lg] : 0;
  // critical gaps (Q15); a draw is made only where its gap is tested (same values either way)
  if (has_ld) {
    const float eps_a = eps_draw(P, id, k, 1u, P.sigma_a_s3);
    const float g_lead = fmaxf(0.0f, __fadd_rn(__fsub_rn(__fadd_rn(P.g_a, __fmul_rn(P.alpha_i, v)),
                                                        __fmul_rn(P.alpha_a, (float)b_ld)), eps_a));
    if (!((float)g_ld >= g_lead)) return NONE;
  }
  if (has_lg) {
    const int safe = (int)ceilf(__fadd_rn(__fmul_rn(__fadd_rn((float)b_lg, 1.0f), P.dt), P.half_a_dt2)) + 1;
    if (g_lg < safe) return NONE;
    const float eps_b = eps_draw(P, id, k, 2u, P.sigma_b_s3);
    const float g_lag = fmaxf(0.0f, __fadd_rn(__fsub_rn(__fadd_rn(P.g_b, __fmul_rn(P.alpha_b, (float)b_lg)),
                                                       __fmul_rn(P.alpha_i, v)), eps_b));
    if (!((float)g_lg >= g_lag)) return NONE;
  }
  return tc;
}

// ---------------------------------------------------------------------------
// CTA-level helpers
// ---------------------------------------------------------------------------
// exclusive prefix of a 0/1 flag over the CTA; s: 2 x 33 words (ping-pong by `ph`)
__device__ __forceinline__ uint32_t block_flag_scan(bool f, uint32_t* s, unsigned ph, uint32_t& total) {
  uint32_t* sw = s + (ph & 1u) * 33u;
  const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, f);
  if (lane == 0) sw[w] = (uint32_t)__popc(b);
  __syncthreads();
  if (w == 0) {
    uint32_t x = lane < (unsigned)(BS / 32) ? sw[lane] : 0u;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (unsigned)o) incl += y;
    }
    if (lane < (unsigned)(BS / 32)) sw[lane] = incl - x;
    if (lane == 31) sw[32] = incl;
  }
  __syncthreads();
  total = sw[32];
  return sw[w] + (uint32_t)__popc(b & ((1u << lane) - 1u));
}

__device__ __forceinline__ unsigned ht_hash(uint32_t cell) { return (cell * 0x9E3779B1u) >> (32 - HT_BITS); }

// claim `cell` for `id`: the lowest id wins (A9); LPSIM_FLAG_RACY: the first to arrive.
// Entries (cell << 32 | id) of one cell share the high word, so a 64-bit min keeps the lowest id.
__device__ __forceinline__ bool ht_claim(unsigned long long* T, uint32_t cell, uint32_t id, bool racy) {
  const unsigned long long mine = ((unsigned long long)cell << 32) | id;
  unsigned h = ht_hash(cell);
  for (unsigned probe = 0; probe < HT; ++probe, h = (h + 1u) & (HT - 1u)) {
    const unsigned long long old = atomicCAS(&T[h], HT_EMPTY, mine);
    if (old == HT_EMPTY) return true;
    if ((uint32_t)(old >> 32) == cell) {
      if (!racy) atomicMin(&T[h], mine);
      return true;
    }
  }
  return false;  // table full (capacity error)
}
__device__ __forceinline__ uint32_t ht_winner(const unsigned long long* T, uint32_t cell) {
  unsigned h = ht_hash(cell);
  for (unsigned probe = 0; probe < HT; ++probe, h = (h + 1u) & (HT - 1u)) {
    const unsigned long long e = T[h];
    if ((uint32_t)(e >> 32) == cell) return (uint32_t)e;
    if (e == HT_EMPTY) break;
  }
  return NONE;
}

// a byte of M_{k+1} (and of the mirror copy on another part, §8(e))
__device__ __forceinline__ void put(const Global& G, const Params& P, uint8_t* Mn, unsigned mn, uint32_t cell,
                                    uint8_t b, unsigned mirror_part1, uint32_t k, uint32_t tile) {
  if (P.flags & LPSIM_FLAG_CHECKS) {
    if (!put_byte_checked(Mn, cell, b)) set_error(G, ERR_INVARIANT, cell, k, tile);
  } else {
    Mn[cell] = b;
  }
  if (mirror_part1) G.parts[mirror_part1 - 1u].map[mn][cell] = b;
}

// mirror part (+1, 0 = none) of a cell of the current edge (first h_max cells of a META_MIRROR edge)
__device__ __forceinline__ unsigned mirror_of(const Global& G, const Params& P, const Ctx& X, int c) {
  if (!(X.c0 & C0_MIRROR) || c >= P.h_max) return 0u;
  return (unsigned)__ldg(&G.edge_mpart[X.edge & EDGE_MASK]) + 1u;
}

__device__ __forceinline__ Ctx load_ctx(const Ctx* a, uint32_t id) {
  const uint4* q = reinterpret_cast<const uint4*>(a + id);
  const uint4 u = q[0], w = q[1];
  Ctx x;
  x.edge = u.x; x.cur = u.y; x.c0 = u.z; x.v0 = __uint_as_float(u.w);
  x.c2 = w.x; x.c3 = w.y; x.rn = w.z; x.pad = w.w;
  return x;
}
__device__ __forceinline__ void store_ctx(Ctx* a, uint32_t id, const Ctx& x) {
  uint4* q = reinterpret_cast<uint4*>(a + id);
  q[0] = make_uint4(x.edge, x.cur, x.c0, __float_as_uint(x.v0));
  q[1] = make_uint4(x.c2, x.c3, x.rn, x.pad);
}

__device__ __forceinline__ void warp_add(unsigned long long* s, bool pred) {
  const unsigned b = __ballot_sync(0xffffffffu, pred);
  if ((threadIdx.x & 31u) == 0u && b) atomicAdd(s, (unsigned long long)__popc(b));
}
__device__ __forceinline__ void warp_digest(const Global& G, unsigned slot, uint64_t h) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0 && h) atomicAdd(&G.digest_log[slot], (unsigned long long)h);
}

__device__ __forceinline__ unsigned long long ld_flag(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_flag(unsigned long long* p, unsigned long long v, bool sys) {
  if (sys) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// claim list entry (per-tile scratch, written in the move, read in the resolve):
// {output record index | kind << 31 (1: lane change), claimed cell, trip id, proposed speed}
// admit scratch entry per pending position: {slot, trip id, claimed entry cell | NONE, DEP_* flags}
constexpr uint32_t DEP_GONE = 1u, DEP_EMPTY = 2u;

// ---------------------------------------------------------------------------
// the persistent step kernel
// ---------------------------------------------------------------------------
struct __align__(16) LcTask {  // a lane-change candidate of the move phase (everything lc_decide needs)
  uint32_t o;                  // output record index
  uint32_t id;
  float v;                     // step-k speed
  float plc;
  uint32_t cell;               // cell at k+1 in the current lane (the fallback)
  float pn, vn;                // state at k+1 (the fallback)
  uint32_t lm;                 // lane | lo << 8 (allowed range start, Q14) | mirror << 16
  uint32_t Lc;
  uint32_t edge, cursor;       // digest
  uint32_t pad;
};

// successor search of the departures of the previous step (A7): the next lowest released trip of the
// slot becomes its candidate.  Deferred off the step's critical path: a slot whose trip departed at
// k has that vehicle in its entry cell at k+1, so its candidate is first needed at k+2.
__device__ __forceinline__ void departed_successors(const Global& G, uint32_t pseg, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += BS) {
    const uint4 ad = G.adm[pseg + i];
    if (!(ad.w & DEP_GONE)) continue;
    const uint4 sa = __ldg(&G.slot_a[ad.x]);
    const uint32_t r = G.slot_cand[ad.x];
    const uint32_t nx = bm_next(G.bm + sa.y, sa.z, r, (ad.w & DEP_EMPTY) != 0u);
    G.slot_cand[ad.x] = nx;
    G.slot_cid[ad.x] = nx != NONE ? __ldg(&G.slot_trip[sa.w + nx]) : NONE;
  }
}

template <bool FULL>
__device__ __forceinline__ void tile_run(const Global& G, const Params& P, unsigned long long k0, unsigned nsteps) {
  const uint32_t X = G.tile0 + blockIdx.x;
  const unsigned tid = threadIdx.x;
  extern __shared__ __align__(16) unsigned long long s_ht[];  // claim hash table [HT]
  LcTask* s_lcq = reinterpret_cast<LcTask*>(s_ht + HT);
  __shared__ TileInfo sI;
  __shared__ uint32_t s_nb_tile[MAX_NB], s_out_back[MAX_NB], s_out_cap[MAX_NB], s_out_off[MAX_NB];
  __shared__ uint32_t s_nb_part[MAX_NB], s_in_off[MAX_NB], s_in_pre[MAX_NB + 1];
  __shared__ uint32_t s_out_cnt[MAX_NB];
  __shared__ uint32_t s_scan[66];
  __shared__ unsigned long long s_ctr[C_N];
  __shared__ unsigned long long s_t[4];
  __shared__ uint32_t s_n, s_np, s_np2, s_app, s_ncl, s_lcn, s_rc, s_stop, s_part, s_npa;
  const bool dig = FULL && (P.flags & LPSIM_FLAG_DIGESTS) != 0u;
  const bool timing = FULL && (P.flags & LPSIM_FLAG_TIMING) != 0u;
  const bool racy = (P.flags & LPSIM_FLAG_RACY) != 0u;
  const bool sys = G.world > 1u;

  if (tid == 0) {
    sI = G.tinfo[X];
    const TileCtl& C = G.tctl[X];
    s_n = C.n[k0 & 1u];
    s_np = C.np[k0 & 1u];
    s_rc = C.rel_cur;
    s_part = G.tile_part[X];
    s_stop = 0;
    s_npa = 0;
  }
  if (tid < C_N) s_ctr[tid] = 0ull;
  if (tid < 4) s_t[tid] = 0ull;
  for (unsigned h = tid; h < HT; h += BS) s_ht[h] = HT_EMPTY;
  __syncthreads();
  const uint32_t nnb = sI.nnb;
  if (tid < nnb) {
    const uint32_t j = sI.nb0 + tid;
    const uint32_t N = G.nb_tile[j], back = G.nb_back[j];
    s_nb_tile[tid] = N;
    s_nb_part[tid] = G.tile_part[N];
    s_out_back[tid] = back;
    s_out_cap[tid] = G.ch_cap[back];
    s_out_off[tid] = G.ch_off[back];
    s_in_off[tid] = G.ch_off[j];
  }
  __syncthreads();
  const unsigned mypart = s_part;
  const PartPtrs MP = G.parts[mypart];
  const uint32_t seg = sI.seg, cap = sI.cap, pseg = sI.pseg;

  for (unsigned it = 0; it < nsteps; ++it) {
    const uint32_t k = (uint32_t)(k0 + it);
    const unsigned cb = k & 1u, nb = cb ^ 1u;
    const unsigned mk = (unsigned)((k0 + it) % 3ull), mn = (mk + 1u) % 3u, mp = (mk + 2u) % 3u;
    const uint8_t* Mk = MP.map[mk];
    uint8_t* Mn = MP.map[mn];
    uint8_t* Mp = MP.map[mp];
    // Q30: the signal phase green at step k (all signals in phase: phase 0 green in the first half)
    const uint32_t gp = P.sig_cycle > 0 ? ((k % (uint32_t)P.sig_cycle) < (uint32_t)(P.sig_cycle / 2) ? 0u : 1u) : 0u;
    unsigned long long t_a = timing ? globaltimer() : 0ull;

    // ---- 1. successors of the previous step's departures, then the releases of step k: bitmap bit,
    //         count, candidate; a slot that becomes pending joins the pending list of this step
    //         (A7: depart_step <= k) ----
    if (s_npa) {
      departed_successors(G, pseg, s_npa);
      __syncthreads();
    }
    for (;;) {
      const uint32_t rc = s_rc;
      const uint32_t j = rc + tid;
      bool rel = false;
      uint4 r = make_uint4(0, 0, 0, 0);
      if (j < sI.rel1) {
        r = __ldg(&G.rel[j]);  // {slot, rank, step, trip id}
        rel = r.z == k;
      }
      if (rel) {
        const uint4 sa = __ldg(&G.slot_a[r.x]);
        bm_set(G.bm + sa.y, sa.z, r.y);
        atomicMin(&G.slot_cand[r.x], r.y);
        atomicMin(&G.slot_cid[r.x], r.w);  // rank order = id order within a slot
        if (atomicAdd(&G.slot_nrel[r.x], 1u) == 0u) {
          const uint32_t q = atomicAdd(&s_np, 1u);
          G.plist[cb][pseg + q] = make_uint2(r.x, sa.x);
        }
      }
      const int cnt = __syncthreads_count(rel);
      if (tid == 0) s_rc = rc + (uint32_t)cnt;
      __syncthreads();
      if (cnt < BS) break;
    }

    // ---- 2. wait for the neighbours to finish step k-1 (their M_k bytes, channels, clears) ----
    if (tid < 32) {
      const unsigned lane = tid;
      uint32_t cnt[2] = {0u, 0u};
      bool bad = false;
#pragma unroll
      for (unsigned q = 0; q < 2; ++q) {
        const unsigned j = lane + 32u * q;
        if (j >= nnb) continue;
        const unsigned long long* f = MP.flag + (size_t)cb * G.nbt + sI.nb0 + j;
        unsigned long long v = ld_flag(f);
        unsigned long long t0 = 0;
        unsigned spins = 0;
        while ((uint32_t)(v >> 32) != k) {
          if ((++spins & 63u) == 0u) {
            if (has_error(G)) { bad = true; break; }
            const unsigned long long t = globaltimer();
            if (t0 == 0) t0 = t;
            else if (t - t0 > TIMEOUT_NS) {
              set_error(G, ERR_TIMEOUT, s_nb_tile[j], k, X);
              bad = true;
              break;
            }
          }
          v = ld_flag(f);
        }
        cnt[q] = bad ? 0u : (uint32_t)v;
      }
      // acquire: the neighbours' stores before their flags are visible to this CTA after the barrier
      if (lane < nnb) {
        if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
        else asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      // s_in_pre[j] = migrants of the channels before neighbour j (entries lane, then lane + 32)
      uint32_t i0 = cnt[0], i1 = cnt[1];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y0 = __shfl_up_sync(0xffffffffu, i0, o), y1 = __shfl_up_sync(0xffffffffu, i1, o);
        if (lane >= (unsigned)o) { i0 += y0; i1 += y1; }
      }
      const uint32_t sum0 = __shfl_sync(0xffffffffu, i0, 31), sum1 = __shfl_sync(0xffffffffu, i1, 31);
      if (lane < nnb) s_in_pre[lane] = i0 - cnt[0];
      if (lane + 32u < nnb) s_in_pre[lane + 32u] = sum0 + i1 - cnt[1];
      if (lane == 0) s_in_pre[nnb] = sum0 + sum1;
      if (__any_sync(0xffffffffu, bad) && lane == 0) s_stop = 1;
      if (lane < nnb) s_out_cnt[lane] = 0;
      if (lane + 32u < nnb) s_out_cnt[lane + 32u] = 0;
      if (lane == 0) { s_app = 0; s_ncl = 0; s_lcn = 0; s_np2 = 0; }
    }
    __syncthreads();
    if (s_stop) break;
    if (timing && tid == 0) {
      const unsigned long long t = globaltimer();
      s_t[0] += t - t_a;
      t_a = t;
    }

    // ---- 3. admits (A7): the lowest released trip of every pending slot claims its entry cell if it
    //         is free in M_k (two loads: the entry cell's byte and the cached candidate id) ----
    const uint32_t np = s_np;
    for (uint32_t i = tid; i < np; i += BS) {
      const uint2 e = G.plist[cb][pseg + i];  // {slot, entry cell}
      const uint32_t id = G.slot_cid[e.x];
      uint32_t cell = NONE;
      if (Mk[e.y] == 255) {
        if (!ht_claim(s_ht, e.y, id, racy)) set_error(G, ERR_CAPACITY, 2, k, X);
        cell = e.y;
      }
      G.adm[pseg + i] = make_uint4(e.x, id, cell, 0u);
    }

    // ---- 4. move every input: own records [0, n), then the migrants of the channels ----
    const uint32_t n_own = s_n, n_in = n_own + s_in_pre[nnb];
    uint32_t out_base = 0;
    unsigned ph = 0;
    uint64_t hsum = 0;
    for (uint32_t r0 = 0; r0 < n_in; r0 += BS, ++ph) {
      const uint32_t i = r0 + tid;
      uint32_t id = NONE, ln = 0, cell = 0, pcell = NONE, c4 = NONE;
      float p = 0.0f, v = 0.0f;
      if (i < n_own) {
        const uint32_t a = seg + i;
        id = G.rid[cb][a]; ln = G.rln[cb][a]; p = G.rpos[cb][a]; v = G.rv[cb][a];
        cell = G.rcell[cb][a]; pcell = G.rpcell[cb][a]; c4 = G.rc4[cb][a];
      } else if (i < n_in) {
        const uint32_t f = i - n_own;
        unsigned lo = 0, hi = nnb;  // channel j with s_in_pre[j] <= f < s_in_pre[j+1]
        while (hi - lo > 1) {
          const unsigned mid = (lo + hi) >> 1;
          if (s_in_pre[mid] <= f) lo = mid; else hi = mid;
        }
        const uint4* q = reinterpret_cast<const uint4*>(MP.chan + (size_t)cb * G.chan_total + s_in_off[lo] +
                                                        (f - s_in_pre[lo]));
        const uint4 m0 = q[0], m1 = q[1];
        id = m0.x; ln = m0.y; v = __uint_as_float(m0.z); cell = m0.w; c4 = m1.x;
      }
      const bool alive = id != NONE;
      Ctx Xc{};
      if (alive) Xc = load_ctx(MP.ctx, id);
      // clear of M_{k-1}: the cell this entry held at k-1 (its own part's copy and the mirror)
      if (pcell != NONE) {
        Mp[pcell] = 255;
        const unsigned pm = (ln >> LN_PM_SHIFT) & LN_PM_MASK;
        if (pm) G.parts[pm - 1u].map[mp][pcell] = 255;
      }
      uint32_t tot;
      const uint32_t o = out_base + block_flag_scan(alive, s_scan, ph, tot);
      out_base += tot;
      bool keep = false, fin = false, lcq = false;
      uint64_t h = 0;
      MoveOut mo;
      mo.lc = false;
      if (alive) {
        if (o >= cap) {
          set_error(G, ERR_CAPACITY, 1, k, X);
        } else {
          const uint32_t l = ln & LN_LANE, Lc = ln >> LN_LC_SHIFT;
          const bool last = (ln & LN_LAST) != 0u;
          move_vehicle(P, Mk, gp, l, last, (int)Lc, p, v, cell, c4, Xc, mo);
          const uint32_t pm_new = mirror_of(G, P, Xc, (int)p);  // the mirror part of the k cell
          const uint32_t a = seg + o;
          const uint32_t lnk = ln_pack(l, last, pm_new, Lc);
          if (mo.finished) {  // Q24: arrival at k+1; the k cell is cleared at k+1 (dead record)
            G.arrival_step[id] = (int32_t)(k + 1);
            G.rid[nb][a] = NONE;
            G.rln[nb][a] = lnk;
            G.rpcell[nb][a] = cell;
            fin = true;
          } else {
            G.rid[nb][a] = id;
            G.rln[nb][a] = lnk;
            G.rpos[nb][a] = mo.pos;
            G.rv[nb][a] = mo.v;
            G.rcell[nb][a] = mo.cell_new;
            G.rpcell[nb][a] = cell;
            G.rc4[nb][a] = c4;
            if (mo.claimant) {
              // contend for the entry cell (the state above is the fallback); resolved after the barrier.
              // The winner's next context needs the next edge's record and route-position entry: into L1.
              if (!ht_claim(s_ht, c4, id, racy)) set_error(G, ERR_CAPACITY, 2, k, X);
              const uint32_t q = atomicAdd(&s_ncl, 1u);
              if (q < cap) G.cl[seg + q] = make_uint4(o, c4, id, __float_as_uint(mo.cv));
              asm volatile("prefetch.global.L1 [%0];" ::"l"(G.edges + (Xc.rn & ROUTE_EDGE_MASK)));
              asm volatile("prefetch.global.L1 [%0];" ::"l"(G.rinfo + Xc.cur + 1u));
            } else if (mo.lc) {
              lcq = true;
            } else {
              const int cn = (int)mo.pos;
              put(G, P, Mn, mn, mo.cell_new, speed_byte(mo.v), mirror_of(G, P, Xc, cn), k, X);
              keep = true;
              if (dig) h = veh_hash(id, Xc.edge & EDGE_MASK, l, mo.pos, mo.v, Xc.cur - __ldg(&G.trip_rstart[id]));
            }
          }
        }
      }
      warp_add(&s_ctr[C_UPD], alive);
      warp_add(&s_ctr[C_ARR], fin);
      if (dig) hsum += keep ? h : 0ull;
      // lane-change candidates -> the CTA's batch (warp-aggregated); decided on full warps below
      {
        const unsigned bl = __ballot_sync(0xffffffffu, lcq);
        unsigned base = 0;
        if ((tid & 31u) == 0u && bl) base = atomicAdd(&s_lcn, (unsigned)__popc(bl));
        base = __shfl_sync(0xffffffffu, base, 0) + __popc(bl & ((1u << (tid & 31u)) - 1u));
        if (lcq) {
          if (base < LCQ) {
            LcTask t;
            t.o = o; t.id = id; t.v = v; t.plc = mo.plc;
            t.cell = mo.cell_new; t.pn = mo.pos; t.vn = mo.v;
            t.lm = (ln & LN_LANE) | ((Xc.c3 & 255u) << 8) | (mirror_of(G, P, Xc, (int)mo.pos) << 16);
            t.Lc = ln >> LN_LC_SHIFT;
            t.edge = Xc.edge & EDGE_MASK;
            t.cursor = dig ? Xc.cur - __ldg(&G.trip_rstart[id]) : 0u;
            t.pad = 0;
            s_lcq[base] = t;
          } else {
            set_error(G, ERR_CAPACITY, 3, k, X);  // not reached: the queue is flushed below
          }
        }
      }
      __syncthreads();
      const bool flush = s_lcn + BS > LCQ || r0 + BS >= n_in;  // block-uniform
      if (flush && s_lcn) {
        // the lane-change batch (a6): one candidate per thread, on full warps
        const unsigned nq = min(s_lcn, LCQ);
        for (unsigned t = tid; t < nq; t += BS) {
          const LcTask tk = s_lcq[t];
          const uint32_t l = tk.lm & 255u;
          const int cn = (int)tk.pn;
          uint32_t tl;
          const uint32_t tc = lc_decide(P, Mk, k, tk.id, tk.v, tk.plc, tk.cell - (uint32_t)cn, l, cn, (int)tk.Lc,
                                        (tk.lm >> 8) & 255u, tl);
          if (tc != NONE) {
            if (!ht_claim(s_ht, tc, tk.id, racy)) set_error(G, ERR_CAPACITY, 2, k, X);
            const uint32_t q = atomicAdd(&s_ncl, 1u);
            if (q < cap) G.cl[seg + q] = make_uint4(tk.o | 0x80000000u, tc, tk.id, __float_as_uint(tk.vn));
          } else {
            put(G, P, Mn, mn, tk.cell, speed_byte(tk.vn), tk.lm >> 16, k, X);
            if (dig) hsum += veh_hash(tk.id, tk.edge, l, tk.pn, tk.vn, tk.cursor);
          }
        }
        __syncthreads();
        if (tid == 0) s_lcn = 0;
        __syncthreads();
      }
    }
    if (n_in == 0) __syncthreads();  // the admits' claims before the resolve
    if (s_ncl > cap) set_error(G, ERR_CAPACITY, 4, k, X);
    if (timing && tid == 0) {
      const unsigned long long t = globaltimer();
      s_t[1] += t - t_a;
      t_a = t;
    }

    // ---- 5. resolve (A9): vehicle claims, then departures ----
    const uint32_t ncl = min(s_ncl, cap);
    for (uint32_t jb = tid & ~31u; jb < ncl; jb += BS) {  // warp-uniform trip count
      const uint32_t j = jb + (tid & 31u);
      bool won = false, lost = false, is_lc = false, is_tr = false;
      uint64_t h = 0;
      if (j < ncl) {
        const uint4 e = G.cl[seg + j];
        const uint32_t o = e.x & 0x7FFFFFFFu, ccell = e.y, id = e.z;
        const float cv = __uint_as_float(e.w);
        is_lc = (e.x >> 31) != 0u;
        is_tr = !is_lc;
        const uint32_t a = seg + o;
        const uint32_t ln = G.rln[nb][a], l = ln & LN_LANE;
        const Ctx Xv = load_ctx(MP.ctx, id);
        won = ht_winner(s_ht, ccell) == id;
        lost = !won;
        if (!won) {
          // the fallback state is already in the record: its byte of M_{k+1}
          const uint32_t fc = G.rcell[nb][a];
          const float fp = G.rpos[nb][a], fv = G.rv[nb][a];
          put(G, P, Mn, mn, fc, speed_byte(fv), mirror_of(G, P, Xv, (int)fp), k, X);
          if (dig) h = veh_hash(id, Xv.edge & EDGE_MASK, l, fp, fv, Xv.cur - __ldg(&G.trip_rstart[id]));
        } else if (is_lc) {
          // lane change: same edge, cell ccell in lane tl; only the next edge's entry cell moves
          const uint32_t lo = Xv.c3 & 255u, tl = l < lo ? l + 1u : l - 1u;
          const float fp = G.rpos[nb][a];
          G.rln[nb][a] = tl | (ln & ~LN_LANE);
          G.rcell[nb][a] = ccell;
          if (!(Xv.edge & LAST_BIT)) {
            const uint32_t nl = (Xv.c2 >> LANES_SHIFT) & LANES_MASK, st = Xv.c2 & LC_MASK;
            G.rc4[nb][a] = G.rc4[nb][a] - min(l, nl - 1u) * st + min(tl, nl - 1u) * st;
          }
          put(G, P, Mn, mn, ccell, speed_byte(cv), mirror_of(G, P, Xv, (int)fp), k, X);
          if (dig) h = veh_hash(id, Xv.edge & EDGE_MASK, tl, fp, cv, Xv.cur - __ldg(&G.trip_rstart[id]));
        } else {
          // transition onto e' (Q20: pos 0, speed kept, Q21: lane min(l, lanes(e') - 1))
          const uint32_t nl = (Xv.c2 >> LANES_SHIFT) & LANES_MASK, l2 = min(l, nl - 1u);
          const uint32_t li = Xv.c2 >> LI_SHIFT;
          const uint32_t cur2 = Xv.cur + 1u;
          uint32_t c4n;
          const Ctx Y = make_ctx(G.edges, G.rinfo, Xv.rn, cur2, l2, c4n);
          if (G.edge_entry) G.edge_entry[cur2] = (int32_t)(k + 1);  // t_start of the new edge
          const unsigned tpart = li == LI_SAME ? mypart : s_nb_part[li];
          store_ctx(G.parts[tpart].ctx, id, Y);
          put(G, P, Mn, mn, ccell, speed_byte(cv), tpart != mypart ? tpart + 1u : 0u, k, X);
          const uint32_t Lc2 = Y.c0 & LC_MASK;
          const bool last2 = (Xv.rn & LAST_BIT) != 0u;
          if (li == LI_SAME) {
            G.rln[nb][a] = ln_pack(l2, last2, (ln >> LN_PM_SHIFT) & LN_PM_MASK, Lc2);
            G.rpos[nb][a] = 0.0f;
            G.rv[nb][a] = cv;
            G.rcell[nb][a] = ccell;
            G.rc4[nb][a] = c4n;
          } else {
            // entrant of a neighbour tile's edge: into its channel (§8(e) migrant); this record
            // stays as a dead entry that clears the k cell at k+1
            G.rid[nb][a] = NONE;
            const uint32_t q = atomicAdd(&s_out_cnt[li], 1u);
            if (q < s_out_cap[li]) {
              uint4* d = reinterpret_cast<uint4*>(G.parts[tpart].chan + (size_t)nb * G.chan_total + s_out_off[li] + q);
              d[0] = make_uint4(id, ln_pack(l2, last2, 0u, Lc2), __float_as_uint(cv), ccell);
              d[1] = make_uint4(c4n, 0u, 0u, 0u);
            } else {
              set_error(G, ERR_CAPACITY, 5, k, X);
            }
          }
          if (dig) h = veh_hash(id, Xv.rn & EDGE_MASK, l2, 0.0f, cv, cur2 - __ldg(&G.trip_rstart[id]));
        }
      }
      warp_add(&s_ctr[C_TRANS], won && is_tr);
      warp_add(&s_ctr[C_LC], won && is_lc);
      warp_add(&s_ctr[C_LOST], lost);
      if (dig) hsum += h;
    }
    // departures: the slot's candidate departs if it holds the claim (its successor is found at the
    // start of the next step); the slot stays pending while released trips wait
    for (uint32_t ib = tid & ~31u; ib < np; ib += BS) {  // warp-uniform trip count
      const uint32_t i = ib + (tid & 31u);
      bool dep = false, lost = false;
      uint64_t h = 0;
      if (i < np) {
        const uint4 ad = G.adm[pseg + i];
        const uint32_t s = ad.x, id = ad.y;
        bool pend = true;
        if (ad.z != NONE) {
          const uint2 sb = __ldg(&G.slot_b[s]);
          const uint2 dp = __ldg(&G.dep[id]);  // {record lane word, entry cell of the second edge}
          if (ht_winner(s_ht, ad.z) == id) {
            dep = true;
            const uint32_t li = (sb.y >> 8) & 63u, l0 = sb.y & 255u;
            const unsigned tpart = li == LI_SAME ? mypart : s_nb_part[li];
            if (G.edge_entry) G.edge_entry[__ldg(&G.trip_rstart[id])] = (int32_t)(k + 1);  // t_start
            put(G, P, Mn, mn, ad.z, 0, tpart != mypart ? tpart + 1u : 0u, k, X);
            if (li == LI_SAME) {
              const uint32_t q = atomicAdd(&s_app, 1u);
              const uint32_t o = out_base + q;
              if (o < cap) {
                const uint32_t a = seg + o;
                G.rid[nb][a] = id; G.rln[nb][a] = dp.x; G.rpos[nb][a] = 0.0f; G.rv[nb][a] = 0.0f;
                G.rcell[nb][a] = ad.z; G.rpcell[nb][a] = NONE; G.rc4[nb][a] = dp.y;
              } else {
                set_error(G, ERR_CAPACITY, 6, k, X);
              }
            } else {
              const uint32_t q = atomicAdd(&s_out_cnt[li], 1u);
              if (q < s_out_cap[li]) {
                uint4* d = reinterpret_cast<uint4*>(G.parts[tpart].chan + (size_t)nb * G.chan_total + s_out_off[li] + q);
                d[0] = make_uint4(id, dp.x, 0u, ad.z);
                d[1] = make_uint4(dp.y, 0u, 0u, 0u);
              } else {
                set_error(G, ERR_CAPACITY, 5, k, X);
              }
            }
            const uint32_t left = atomicSub(&G.slot_nrel[s], 1u) - 1u;
            G.adm[pseg + i].w = DEP_GONE | (left == 0u ? DEP_EMPTY : 0u);
            pend = left != 0u;
            if (dig) h = veh_hash(id, sb.x & EDGE_MASK, l0, 0.0f, 0.0f, 0u);
          } else {
            lost = true;  // the slot's queue is one losing party
          }
        }
        if (pend) {
          const uint32_t q = atomicAdd(&s_np2, 1u);
          G.plist[nb][pseg + q] = G.plist[cb][pseg + i];
        }
      }
      warp_add(&s_ctr[C_DEP], dep);
      warp_add(&s_ctr[C_LOST], lost);
      if (dig) hsum += h;
    }
    if (dig) warp_digest(G, it, hsum);
    __syncthreads();

    // ---- 6. publish: step k done (+ migrants per channel) to every neighbour ----
    if (tid < 32) {
      if (tid == 0) {
        if (sys) __threadfence_system();
        else __threadfence();
      }
      __syncwarp();
      for (unsigned j = tid; j < nnb; j += 32u) {
        const unsigned long long v = ((unsigned long long)(k + 1u) << 32) | (s_out_cap[j] ? s_out_cnt[j] : 0u);
        unsigned long long* f = G.parts[s_nb_part[j]].flag + (size_t)nb * G.nbt + s_out_back[j];
        st_flag(f, v, sys);
      }
    }
    for (unsigned h = tid; h < HT; h += BS) s_ht[h] = HT_EMPTY;
    if (tid == 0) {
      s_n = out_base + s_app;
      s_npa = np;
      s_np = s_np2;
      if (s_n > cap) set_error(G, ERR_CAPACITY, 7, k, X);
    }
    if (timing && tid == 0) {
      const unsigned long long t = globaltimer();
      s_t[2] += t - t_a;
      s_t[3] += 1ull;
    }
    __syncthreads();
  }
  // the successors of the last step's departures (canonical slot state between launches)
  if (s_npa && !s_stop) departed_successors(G, pseg, s_npa);
  // state of the tile for the next launch / the host queries
  if (tid == 0) {
    TileCtl& C = G.tctl[X];
    const unsigned long long kend = k0 + nsteps;
    C.n[kend & 1ull] = s_n;
    C.np[kend & 1ull] = s_np;
    C.rel_cur = s_rc;
    for (int c = 0; c < C_N; ++c) C.ctr[c] += s_ctr[c];
    for (int c = 0; c < 4; ++c) C.t[c] += s_t[c];
  }
}

__global__ void __launch_bounds__(BS, TILE_MINB) k_tile(Global G, Params P, unsigned long long k0, unsigned nsteps) {
  tile_run<false>(G, P, k0, nsteps);
}
__global__ void __launch_bounds__(BS, TILE_MINB) k_tile_full(Global G, Params P, unsigned long long k0,
                                                             unsigned nsteps) {
  tile_run<true>(G, P, k0, nsteps);
}

// ---------------------------------------------------------------------------
// setup / query kernels
// ---------------------------------------------------------------------------
__global__ void k_fill_u8(uint8_t* p, uint8_t v, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_fill_u32(uint32_t* p, uint32_t v, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

// a0 lane-map builder: cells per edge = lanes·ceil(length) (Q29)
__global__ void k_edge_cells(const float* length, const uint8_t* lanes, uint64_t* cells, uint32_t* ncells, int E) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const uint32_t Lc = (uint32_t)ceilf(length[e]);
    ncells[e] = Lc;
    cells[e] = (uint64_t)Lc * lanes[e];
  }
}

// exclusive scan of u64 (three-pass: block sums, scan of sums, add)
constexpr int SCAN_BS = SCAN_BLOCK;
__global__ void k_scan_blocks(const uint64_t* in, uint64_t* out, uint64_t* sums, int n) {
  __shared__ uint64_t sh[SCAN_BS];
  const int i = blockIdx.x * SCAN_BS + threadIdx.x;
  uint64_t x = i < n ? in[i] : 0ull;
  sh[threadIdx.x] = x;
  __syncthreads();
  for (int o = 1; o < SCAN_BS; o <<= 1) {
    uint64_t y = threadIdx.x >= (unsigned)o ? sh[threadIdx.x - o] : 0ull;
    __syncthreads();
    sh[threadIdx.x] += y;
    __syncthreads();
  }
  if (i < n) out[i] = sh[threadIdx.x] - x;
  if (threadIdx.x == SCAN_BS - 1) sums[blockIdx.x] = sh[threadIdx.x];
}
__global__ void k_scan_sums(uint64_t* sums, int nb, uint64_t* total) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    uint64_t acc = 0;
    for (int b = 0; b < nb; ++b) {
      const uint64_t s = sums[b];
      sums[b] = acc;
      acc += s;
    }
    *total = acc;
  }
}
__global__ void k_scan_add(uint64_t* out, const uint64_t* sums, int n) {
  const int i = blockIdx.x * SCAN_BS + threadIdx.x;
  if (i < n) out[i] += sums[blockIdx.x];
}

// a0: the 16-byte edge records from the scanned bases
__global__ void k_build_edges(int E, const uint64_t* base, const uint32_t* ncells, const uint8_t* lanes, const float* v0,
                              const uint32_t* li, const uint32_t* meta, EdgeRec* out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    EdgeRec R;
    R.base = (uint32_t)base[e];
    R.lc = ncells[e] | ((uint32_t)lanes[e] << LANES_SHIFT) | (li[e] << LI_SHIFT);
    R.v0 = v0[e];
    R.meta = meta[e];
    out[e] = R;
  }
}

__global__ void k_route_info(const uint32_t* route, const EdgeRec* edges, int64_t R, uint4* rinfo) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < R; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = route[j];
    if (r & LAST_BIT) continue;
    const uint32_t rn = route[j + 1];
    const EdgeRec E = edges[r & ROUTE_EDGE_MASK], N = edges[rn & ROUTE_EDGE_MASK];
    rinfo[j] = make_uint4(rn, N.lc, N.base,
                          lane_range((E.lc >> LANES_SHIFT) & LANES_MASK, (E.meta >> META_KOUT_SHIFT) & META_KOUT_MASK,
                                     N.meta & META_RANK_MASK));
  }
}

__global__ void k_trip_ctx(const EdgeRec* edges, const uint32_t* route, const uint4* rinfo,
                           const uint32_t* trip_rstart, const uint8_t* edge_opart, const PartPtrs* parts,
                           unsigned n_parts, int64_t n, uint2* dep) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t rs = trip_rstart[t];
    const uint32_t r0 = route[rs];
    const uint32_t e1 = r0 & ROUTE_EDGE_MASK;
    const uint32_t lc = edges[e1].lc;
    const uint32_t lanes = (lc >> LANES_SHIFT) & LANES_MASK;
    const uint32_t l0 = (uint32_t)(t % lanes);  // Q22: departure lane id mod lanes
    uint32_t c4;
    const Ctx X = make_ctx(edges, rinfo, r0, rs, l0, c4);
    const unsigned p = edge_opart[e1];
    if (p < n_parts && parts[p].ctx) store_ctx(parts[p].ctx, (uint32_t)t, X);
    dep[t] = make_uint2(ln_pack(l0, (r0 & LAST_BIT) != 0u, 0u, lc & LC_MASK), c4);
  }
}

__global__ void k_scatter_trips(Global G, uint32_t t0, uint32_t t1, unsigned long long k, int32_t* status,
                                int32_t* edge, int32_t* lane, float* pos, float* v, int64_t* cursor) {
  const unsigned cb = (unsigned)(k & 1ull);
  for (uint32_t X = t0 + blockIdx.x; X < t1; X += gridDim.x) {
    const TileInfo I = G.tinfo[X];
    const PartPtrs& MP = G.parts[G.tile_part[X]];
    const uint32_t n = G.tctl[X].n[cb];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t a = I.seg + i, id = G.rid[cb][a];
      if (id == NONE) continue;
      const Ctx c = load_ctx(MP.ctx, id);
      status[id] = 1;
      edge[id] = (int32_t)(c.edge & EDGE_MASK);
      lane[id] = (int32_t)(G.rln[cb][a] & LN_LANE);
      pos[id] = G.rpos[cb][a];
      v[id] = G.rv[cb][a];
      cursor[id] = (int64_t)(c.cur - G.trip_rstart[id]);
    }
    // entrants in flight: the channels into X written in step k-1
    for (uint32_t j = 0; j < I.nnb; ++j) {
      const uint32_t jj = I.nb0 + j;
      if (G.ch_cap[jj] == 0u) continue;
      const unsigned long long f = MP.flag[(size_t)cb * G.nbt + jj];
      if ((uint32_t)(f >> 32) != (uint32_t)k) continue;
      const uint32_t m = (uint32_t)f;
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const MigRec r = MP.chan[(size_t)cb * G.chan_total + G.ch_off[jj] + i];
        const Ctx c = load_ctx(MP.ctx, r.id);
        status[r.id] = 1;
        edge[r.id] = (int32_t)(c.edge & EDGE_MASK);
        lane[r.id] = (int32_t)(r.ln & LN_LANE);
        pos[r.id] = 0.0f;
        v[r.id] = r.v;
        cursor[r.id] = (int64_t)(c.cur - G.trip_rstart[r.id]);
      }
    }
  }
}

// distance (double, route order) per trip
__global__ void k_distances(int64_t n, const uint32_t* route, const uint32_t* trip_rstart, const float* length,
                            const int32_t* status, const float* pos, const int64_t* cursor, const int32_t* arrival,
                            double* dist) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t rs = trip_rstart[t];
    double d = 0.0;
    if (arrival[t] >= 0) {
      uint32_t j = rs;
      for (;;) {
        const uint32_t r = route[j++];
        d += (double)length[r & ROUTE_EDGE_MASK];
        if (r & LAST_BIT) break;
      }
    } else if (status[t] == 1) {
      for (int64_t j = 0; j < cursor[t]; ++j) d += (double)length[route[rs + j] & ROUTE_EDGE_MASK];
      d += (double)pos[t];
    }
    dist[t] = d;
  }
}

__global__ void k_gather_map(const uint8_t* map, const EdgeRec* edges, const uint8_t* edge_opart, unsigned p, int E,
                             uint8_t* out) {
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    if (edge_opart[e] != p) continue;
    const EdgeRec R = edges[e];
    const uint32_t n = (R.lc & LC_MASK) * ((R.lc >> LANES_SHIFT) & LANES_MASK);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) out[(size_t)R.base + i] = map[(size_t)R.base + i];
  }
}

// occupied (non-free) cells of the edges owned by part p: the a7 invariant check
__global__ void k_count_occupied(const uint8_t* map, const EdgeRec* edges, const uint8_t* edge_opart, unsigned p,
                                 int E, unsigned long long* out) {
  unsigned long long n_occ = 0;
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    if (edge_opart[e] != p) continue;
    const EdgeRec R = edges[e];
    const uint32_t n = (R.lc & LC_MASK) * ((R.lc >> LANES_SHIFT) & LANES_MASK);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) n_occ += map[(size_t)R.base + i] != 255 ? 1u : 0u;
  }
  atomicAdd(out, n_occ);
}

// restore (§8(f) checkpoint/restore): at a step boundary the state of snapshot k is the per-trip
// state; on-road trips of this part's tiles become records of the list of k with no previous cell,
// their contexts are rebuilt and their bytes written into M_k (also the mirror windows of cut edges
// this part probes); err = first offending trip (atomicMin)
__global__ void k_restore_trips(Global G, unsigned local_part, unsigned mk, unsigned cb, int h_max, int64_t n,
                                const uint32_t* tile_of_edge, const int32_t* status, const int32_t* edge,
                                const int32_t* lane, const float* pos, const float* v, const int64_t* cursor,
                                uint32_t* err) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    if (status[t] != 1) continue;
    const uint32_t id = (uint32_t)t, e = (uint32_t)edge[t], l = (uint32_t)lane[t];
    const uint32_t cur = G.trip_rstart[t] + (uint32_t)cursor[t];
    const uint32_t r = G.route[cur];
    const EdgeRec E = G.edges[e];
    const uint32_t Lc = E.lc & LC_MASK, nl = (E.lc >> LANES_SHIFT) & LANES_MASK;
    const float p = pos[t], sp = v[t];
    const int c = (int)p;
    if ((r & ROUTE_EDGE_MASK) != e || l >= nl || !(p >= 0.0f) || c >= (int)Lc || !(sp >= 0.0f && sp <= 254.0f)) {
      atomicMin(err, id);
      continue;
    }
    const uint32_t cell = E.base + l * Lc + (uint32_t)c;
    const uint8_t byte = speed_byte(sp);
    const uint32_t X = tile_of_edge[e];
    const unsigned part = G.tile_part[X];
    const bool all = local_part == 0xFFFFFFFFu;  // one process simulates every part
    if (all || part == local_part) {
      const TileInfo I = G.tinfo[X];
      const uint32_t i = atomicAdd(&G.tctl[X].n[cb], 1u);
      if (i >= I.cap) { atomicMin(err, id); continue; }
      const uint32_t a = I.seg + i;
      uint32_t c4;
      const Ctx Xc = make_ctx(G.edges, G.rinfo, r, cur, l, c4);
      store_ctx(G.parts[part].ctx, id, Xc);
      G.rid[cb][a] = id; G.rln[cb][a] = ln_pack(l, (r & LAST_BIT) != 0u, 0u, Lc);
      G.rpos[cb][a] = p; G.rv[cb][a] = sp;
      G.rcell[cb][a] = cell; G.rpcell[cb][a] = NONE; G.rc4[cb][a] = c4;
      G.parts[part].map[mk][cell] = byte;
    }
    if ((E.meta & META_MIRROR) && c < h_max) {  // the mirror window the upstream part probes
      const unsigned mpart = G.edge_mpart[e];
      if (all || mpart == local_part) G.parts[mpart].map[mk][cell] = byte;
    }
  }
}

__global__ void k_restore_released(Global G, uint32_t t0, uint32_t t1, uint32_t k, const int32_t* status) {
  const unsigned cb = k & 1u;
  for (uint32_t X = t0 + blockIdx.x; X < t1; X += gridDim.x) {
    const TileInfo I = G.tinfo[X];
    for (uint32_t j = I.rel0 + threadIdx.x; j < I.rel1; j += blockDim.x) {
      const uint4 r = G.rel[j];
      if (r.z >= k) continue;
      const uint4 sa = G.slot_a[r.x];
      const uint32_t id = r.w;
      if (status[id] != 0) continue;
      bm_set(G.bm + sa.y, sa.z, r.y);
      atomicMin(&G.slot_cand[r.x], r.y);
      atomicMin(&G.slot_cid[r.x], id);
      if (atomicAdd(&G.slot_nrel[r.x], 1u) == 0u) {
        const uint32_t q = atomicAdd(&G.tctl[X].np[cb], 1u);
        G.plist[cb][I.pseg + q] = make_uint2(r.x, sa.x);
      }
    }
  }
}

size_t tile_dyn_smem() { return (size_t)HT * sizeof(unsigned long long) + (size_t)LCQ * sizeof(LcTask); }

}  // namespace lpsim
