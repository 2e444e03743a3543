// lpsim_step.cu — sm_100a kernels of the LPSim per-timestep vehicle update.
//
// Method: arXiv 2406.08496, Eq. (1) P:L239-242 (every vehicle at k+1 is a
// function of the snapshot at k), Alg. 1, lane map P:L256-266,
// Remarks P:L247-251.  Readings Qnn: DESIGN.md §3.  Layout: lpsim_dev.h.
//
// One persistent cooperative kernel (k_run) executes whole steps; each step
// is two (one partition) or three (several partitions) grid-wide phases:
//   A  admit departures / move every active vehicle: probe M_k (a3), IDM
//      (a4), transition (a5), lane change (a6); vehicles without a claim
//      write SoA_{k+1} and M_{k+1} at once, claimants atomicMin a per-cell
//      claim word and leave a claim record; releases of step k
//   C  clear M_k, resolve claims (lowest trip id wins, A9), departures,
//      migrants straight into their edge owner's receive queue and lane map
// With several partitions (§8(e)) the exchange is part of A and C: bytes of the
// first h_max cells of a cut edge are mirrored into the upstream part's entry
// halo as they are written, migrants are written into the owner's memory, and
// the owner moves them in phase A of the next step; one barrier per step.
// Floating point follows the fixed IEEE fp32 operation order of DESIGN.md §3
// (compiled with --fmad=false, no fast math): integer state is bit-exact
// against the oracle.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lpsim.h"  // LPSIM_FLAG_* (the C ABI flags the kernels honour)
#include "lpsim_kernels.h"

namespace lpsim {

constexpr int BS = STEP_BS;
#ifndef LPSIM_CLEAR_LATE
#define LPSIM_CLEAR_LATE 1  // phase C clears M_k after its claim rounds (0: before; 1 measured -0.15 us)
#endif
#ifndef LPSIM_MINB
#define LPSIM_MINB 3  // resident CTAs per SM the register budget is sized for (80 regs)
#endif
constexpr unsigned long long TIMEOUT_NS = 60000000000ull;  // 60 s: a peer that makes no progress (gone)
// trip id of a slot candidate not yet looked up (phase C of a departure finds the next rank; the
// admit of the next step, where the slot is blocked by the departed vehicle, looks the id up)
constexpr uint32_t IDUNK = 0xFFFFFFFEu;

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// grid barrier (sense by generation counter); bails out on error / timeout
// ---------------------------------------------------------------------------
#ifndef LPSIM_BARRIER
#define LPSIM_BARRIER 2  // 0: fence + atomic + spin; 1: release/acquire PTX spin; 2: cooperative_groups grid sync
#endif
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ bool grid_sync(GridCtl* g) {
#if LPSIM_BARRIER == 2
  // measured 1.2 us per barrier on B200 at 148-296 CTAs (tools/barrier_bench.cu),
  // vs 2.0 us for the hand-written spin barrier.  Errors do not exit early here:
  // every CTA reaches every barrier, and k_run leaves the step loop on a
  // step-stamped error word that all CTAs read consistently (see k_run).
  cooperative_groups::this_grid().sync();
  (void)g;
  return true;
#else
  __shared__ int s_ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    int ok = 1;
#if LPSIM_BARRIER == 1
    const unsigned gen = ld_acquire(&g->bar_gen);
    const unsigned arrived = atom_add_acq_rel(&g->bar_count, 1u);
    if (arrived == gridDim.x - 1) {
      g->bar_count = 0;  // ordered before the release below
      st_release(&g->bar_gen, gen + 1u);
    } else {
      unsigned long long t0 = 0;
      unsigned spins = 0;
      while (ld_acquire(&g->bar_gen) == gen) {
        if ((++spins & 255u) == 0u) {
          if (ld_acquire(&g->error)) { ok = 0; break; }
          const unsigned long long t = globaltimer();
          if (t0 == 0) t0 = t;
          else if (t - t0 > TIMEOUT_NS) {
            atomicCAS(&g->error, 0u, ERR_TIMEOUT);
            ok = 0;
            break;
          }
        }
      }
    }
    if (ld_acquire(&g->error)) ok = 0;
#else
    volatile unsigned* genp = &g->bar_gen;
    volatile unsigned* errp = &g->error;
    unsigned gen = *genp;
    __threadfence();
    unsigned arrived = atomicAdd(&g->bar_count, 1u);
    if (arrived == gridDim.x - 1) {
      g->bar_count = 0;
      __threadfence();
      atomicAdd(&g->bar_gen, 1u);
    } else {
      unsigned long long t0 = globaltimer();
      while (*genp == gen) {
        if (*errp) { ok = 0; break; }
        if (globaltimer() - t0 > TIMEOUT_NS) {
          atomicCAS(&g->error, 0u, ERR_TIMEOUT);
          ok = 0;
          break;
        }
      }
    }
    __threadfence();
    if (*errp) ok = 0;
#endif
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
#endif
}

// first device-side error; stamped with the step so that every CTA leaves the
// step loop at the same step (k_run checks err_step < k during phase A of step k, before its barrier)
// Barrier across the GPUs of a multi-process run (after the local grid barrier
// that ends a step): one thread per GPU pushes its migrant counts and publishes
// the epoch into every peer's flag array over NVLink (st.release.sys) and
// waits until every peer published it here; a flag then releases the local
// CTAs.  Peer writes of the step (migrants, their bytes, mirrored halo bytes)
// precede the release store (cumulativity).  One such barrier per step.
__device__ __forceinline__ void cross_gpu_sync(const Global& G, uint32_t epoch, uint32_t k);

__device__ __forceinline__ void set_error(GridCtl* g, PartCtl* c, unsigned code, unsigned info, uint32_t k) {
  if (atomicCAS(&c->error, 0u, code) == 0u) c->error_info = info;
  atomicCAS(&g->error, 0u, code);
  atomicMin(&g->err_step, k);
}

// A claim on a cell (A9: the lowest trip id wins; LPSIM_FLAG_RACY: the first contender)
__device__ __forceinline__ void claim_cell(uint32_t* w, uint32_t id, bool racy) {
  if (racy) atomicCAS(w, NONE, id);
  else atomicMin(w, id);
}

// A byte of M_{k+1}.  LPSIM_FLAG_CHECKS: it may only be written over a free cell ("one byte can
// only be occupied by one vehicle"): an atomicCAS on the enclosing word, a violation is an invariant
// error naming the cell and the step.
__device__ __forceinline__ void put_map(const Params& P, const Global& G, PartCtl* ctl, uint8_t* Mn, uint32_t cell,
                                        uint8_t b, uint32_t k) {
  if (!(P.flags & LPSIM_FLAG_CHECKS)) {
    Mn[cell] = b;
    return;
  }
  unsigned* w = reinterpret_cast<unsigned*>(Mn + (cell & ~3u));
  const unsigned sh = (cell & 3u) * 8u;
  unsigned old = *((volatile unsigned*)w);
  for (;;) {
    if (((old >> sh) & 255u) != 255u) {
      set_error(G.grid, ctl, ERR_INVARIANT, cell, k);
      return;
    }
    const unsigned got = atomicCAS(w, old, (old & ~(255u << sh)) | ((unsigned)b << sh));
    if (got == old) return;
    old = got;
  }
}

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
__device__ __forceinline__ uint64_t veh_hash(uint32_t id, uint32_t el, float pos, float v, uint32_t j) {
  uint64_t h = mix64((uint64_t)id);
  h = mix64(h ^ (uint64_t)(el & EDGE_MASK));
  h = mix64(h ^ (uint64_t)((el >> LANE_SHIFT) & LANE_MASK));
  h = mix64(h ^ (uint64_t)(uint32_t)(int)pos);
  h = mix64(h ^ (uint64_t)__float_as_uint(pos));
  h = mix64(h ^ (uint64_t)__float_as_uint(v));
  h = mix64(h ^ (uint64_t)j);
  return h;
}

__device__ __forceinline__ EdgeRec load_edge(const EdgeRec* edges, uint32_t e) {
  const uint4 r = __ldg(reinterpret_cast<const uint4*>(edges) + e);
  EdgeRec E;
  E.base = r.x; E.ncells = r.y; E.v0 = __uint_as_float(r.z); E.meta = r.w;
  return E;
}

__device__ __forceinline__ uint32_t lane_stride(const EdgeRec& E, int h_max) {
  return (E.meta & META_HALO) ? (uint32_t)h_max : E.ncells;
}

__device__ __forceinline__ uint8_t speed_byte(float v) {  // byte = speed (m/s), cap 254
  return (uint8_t)(int)fminf(v, 254.0f);
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
// words of level i (0 = top) for depth d and width n
__device__ __forceinline__ uint32_t bm_words(uint32_t n, int d, int i) {
  uint32_t shift = 5u * (uint32_t)(d - i);
  return (uint32_t)(((uint64_t)n + (1ull << shift) - 1) >> shift);
}

constexpr int BM_MAXD = 4;  // bitmap depth bound (host check: <= 2^20 trips per slot)
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

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

// The successor of a departing candidate of rank r, found in phase A of the step (the departure itself
// is decided in phase C): the first set bit > r, read while the releases of step k may be setting
// bits of the same slot (every bit set before the step is seen: they were set before the last
// barrier, summary bits after their leaf), combined by the caller with the slot's lowest release of
// step k other than r (kmin).  Exact: bits below r are 0 (r is the slot's lowest), a step-k release
// the racy read misses is >= kmin, and the releases of step k are the only bits set during the step.
__device__ uint32_t bm_after(const uint32_t* bm, uint32_t n, uint32_t r) {
  const int d = bm_depth(n);
  uint32_t offs[BM_MAXD];
  uint32_t off = 0;
#pragma unroll
  for (int i = 0; i < BM_MAXD; ++i) {
    offs[i] = off;
    if (i < d) off += bm_words(n, d, i);
  }
  // level i holds one bit per word of level i+1; x = index of r's entry at the level being read
  uint32_t x = r;
  for (int lvl = d - 1; lvl >= 0; --lvl) {
    const unsigned b = x & 31u;
    const uint32_t w = (b == 31u) ? 0u : (*((volatile const uint32_t*)&bm[offs[lvl] + (x >> 5)]) & (~0u << (b + 1u)));
    if (w) {
      x = (x & ~31u) | (uint32_t)(__ffs(w) - 1);
      for (int l = lvl + 1; l < d; ++l)  // descend to the leaf
        x = (x << 5) | (uint32_t)(__ffs(*((volatile const uint32_t*)&bm[offs[l] + x])) - 1);
      return x;
    }
    x >>= 5;
  }
  return NONE;
}

// Departure of rank r with the successor succ found in phase A: clear r's bit and each summary bit
// whose word empties, decided from succ (a word keeps a bit iff succ lies in its range: bits below r
// are 0, none lies between r and succ).  Fire-and-forget atomics: nothing waits for them in the step.
__device__ __forceinline__ void bm_clear(uint32_t* bm, uint32_t n, uint32_t r, uint32_t succ) {
  const int d = bm_depth(n);
  uint32_t offs[BM_MAXD];
  uint32_t off = 0;
#pragma unroll
  for (int i = 0; i < BM_MAXD; ++i) {
    offs[i] = off;
    if (i < d) off += bm_words(n, d, i);
  }
  uint32_t x = r;
  for (int lvl = d - 1; lvl >= 0; --lvl) {
    atomicAnd(&bm[offs[lvl] + (x >> 5)], ~(1u << (x & 31u)));
    const unsigned sh = 5u * (unsigned)(d - lvl);  // this word covers 2^sh ranks
    if (succ != NONE && (succ >> sh) == (r >> sh)) break;  // it keeps succ's bit
    x >>= 5;
  }
}

// ---------------------------------------------------------------------------
// sharded work lists (claim records, pending departure slots): NSH counters
// 128 B apart, warp-aggregated pushes, so thousands of pushes per step do not
// serialise on one L2 address.  Storage index = shard * shcap + position.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned sh_shard(unsigned work_index) { return (work_index >> 5) % NSH; }

// warp-collective: every lane calls; returns the storage index for lanes with pred (NONE on overflow)
__device__ __forceinline__ uint32_t sh_push(uint32_t* cnt, unsigned shard, uint32_t shcap, bool pred) {
  shard = __shfl_sync(0xffffffffu, shard, 0);  // one shard per warp (the counter and the storage must agree)
  const unsigned b = __ballot_sync(0xffffffffu, pred);
  const unsigned lane = threadIdx.x & 31u;
  unsigned base = 0;
  if (lane == 0u && b) base = atomicAdd(&cnt[shard * SH_STRIDE], (unsigned)__popc(b));
  base = __shfl_sync(0xffffffffu, base, 0);
  const unsigned j = base + __popc(b & ((1u << lane) - 1u));
  return (pred && j < shcap) ? shard * shcap + j : NONE;
}

// warp-collective (warp `w` of the block): exclusive prefix of the NSH shard counts into s_pref[0..NSH]
__device__ __forceinline__ void sh_prefix_warp(const uint32_t* cnt, uint32_t shcap, unsigned* s_pref, unsigned w) {
  if ((threadIdx.x >> 5) == w) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned a = min(cnt[(2 * lane) * SH_STRIDE], shcap), b = min(cnt[(2 * lane + 1) * SH_STRIDE], shcap);
    unsigned x = a + b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (unsigned)o) x += y;
    }
    s_pref[2 * lane + 1] = x - b;
    s_pref[2 * lane + 2] = x;
    if (lane == 0) s_pref[0] = 0;
  }
}

// block-collective: exclusive prefix of the NSH shard counts into s_pref[0..NSH]; returns the total
__device__ __forceinline__ unsigned sh_prefix(const uint32_t* cnt, uint32_t shcap, unsigned* s_pref) {
  static_assert(NSH == 64, "sh_prefix assumes 64 shards");
  if (threadIdx.x < 32) {
    const unsigned lane = threadIdx.x;
    const unsigned a = min(cnt[(2 * lane) * SH_STRIDE], shcap), b = min(cnt[(2 * lane + 1) * SH_STRIDE], shcap);
    unsigned x = a + b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (unsigned)o) x += y;
    }
    s_pref[2 * lane + 1] = x - b;
    s_pref[2 * lane + 2] = x;
    if (lane == 0) s_pref[0] = 0;
  }
  __syncthreads();
  return s_pref[NSH];
}

// storage index of flat position f (< total)
__device__ __forceinline__ uint32_t sh_locate(const unsigned* s_pref, unsigned f, uint32_t shcap) {
  unsigned lo = 0, hi = NSH;  // find the shard s with s_pref[s] <= f < s_pref[s+1]
  while (hi - lo > 1) {
    const unsigned mid = (lo + hi) >> 1;
    if (s_pref[mid] <= f) lo = mid;
    else hi = mid;
  }
  return lo * shcap + (f - s_pref[lo]);
}

// ---------------------------------------------------------------------------
// vectorised lane-map scans: occupancy bit per byte (byte != 255)
// ---------------------------------------------------------------------------
// 8 bytes -> 8 bits: 0x80 in every byte != 0xFF (borrow-free: the add cannot carry across bytes),
// then the eight byte MSBs gathered into one byte by a multiply (bit i = byte i occupied)
__device__ __forceinline__ uint32_t occ8(uint64_t w) {
  const uint64_t x = ~w;
  const uint64_t t = (((x & 0x7F7F7F7F7F7F7F7Full) + 0x7F7F7F7F7F7F7F7Full) | x) & 0x8080808080808080ull;
  return (uint32_t)(((t >> 7) * 0x0102040810204080ull) >> 56);
}
__device__ __forceinline__ uint64_t occ16(ulonglong2 q) { return (uint64_t)occ8(q.x) | ((uint64_t)occ8(q.y) << 8); }
__device__ __forceinline__ bool all_free(ulonglong2 q) { return (q.x & q.y) == ~0ull; }
// occupancy of the 48 bytes [a, a+48), a multiple of 16; chunks past `hi` are not loaded.
// Fast path: an all-free window (the common case) costs three ANDs.
__device__ __forceinline__ uint64_t occ48(const uint8_t* M, uint32_t a, uint32_t hi) {
  const ulonglong2* q = reinterpret_cast<const ulonglong2*>(M + a);
  const ulonglong2 ones = make_ulonglong2(~0ull, ~0ull);
  const ulonglong2 q0 = q[0];
  const ulonglong2 q1 = (a + 16u <= hi) ? q[1] : ones;
  const ulonglong2 q2 = (a + 32u <= hi) ? q[2] : ones;
  // per chunk, the occupancy bits are built only if some lane of the (possibly partial) warp has
  // an occupied byte in it: a queued vehicle's short window leaves chunks 1-2 free (not loaded)
  const unsigned am = __activemask();
  const bool o0 = !all_free(q0), o1 = !all_free(q1), o2 = !all_free(q2);
  uint64_t m = 0;
  if (__any_sync(am, o0)) m = o0 ? occ16(q0) : 0ull;
  if (__any_sync(am, o1)) m |= (o1 ? occ16(q1) : 0ull) << 16;
  if (__any_sync(am, o2)) m |= (o2 ? occ16(q2) : 0ull) << 32;
  return m;
}
// first occupied byte address in [lo, hi] (hi >= lo), or NONE
__device__ __forceinline__ uint32_t scan_first(const uint8_t* M, uint32_t lo, uint32_t hi) {
  for (uint32_t a = lo & ~15u;; a += 48u) {
    uint64_t m = occ48(M, a, hi);
    if (lo > a) m &= ~0ull << (lo - a);
    if (hi - a < 47u) m &= (2ull << (hi - a)) - 1ull;
    if (m) return a + (uint32_t)(__ffsll((long long)m) - 1);
    if (hi - a < 48u) return NONE;
  }
}
// last occupied byte address in [lo, hi] (hi >= lo), or NONE
__device__ __forceinline__ uint32_t scan_last(const uint8_t* M, uint32_t lo, uint32_t hi) {
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

// ---------------------------------------------------------------------------
// per-vehicle edge context (cached in the SoA, refreshed only when the vehicle
// changes edge): everything the move needs from the current and the next
// route edge, so the move's only dependent loads are lane-map bytes.
// ---------------------------------------------------------------------------
struct Ctx {
  uint32_t c0;  // Lc | lanes(e) << 24 | signalised(e) << 30 | approach phase(e) << 31 (Q30)
  float v0;     // speed limit of e (IDM v0)
  uint32_t c2;  // Lc' | lanes(e') << 24 | halo(e') << 30     (0 on the last route edge)
  uint32_t c3;  // allowed lanes [lo, hi] toward e' (Q14): lo | hi << 8   (0 on the last edge)
                //   | CTX_MIRROR: e is an owned cut edge whose first h_max cells are mirrored (§8(e))
  uint32_t c4;  // cell 0 of the entry lane min(l, lanes(e')-1) of e'  (NONE on the last edge)
  uint32_t rn;  // route[cur+1] = e' | last(e') << 31              (0 on the last edge)
};

constexpr uint32_t CTX_MIRROR = 1u << 16;
__device__ __forceinline__ uint32_t ctx_mirror(const EdgeRec& E) { return (E.meta & META_MIRROR) ? CTX_MIRROR : 0u; }

__device__ __forceinline__ uint32_t ctx_c0(const EdgeRec& E) {
  return E.ncells | ((E.meta & META_LANES_MASK) << 24) | (((E.meta >> 28) & 3u) << 30);
}

__device__ __forceinline__ uint32_t stride_of(uint32_t c2, int h_max) {
  return (c2 & (1u << 30)) ? (uint32_t)h_max : (c2 & 0xFFFFFFu);
}

// allowed lanes [lo, hi] on e toward e' (Q14): L = lanes(e), K = out-degree of to(e), r = rank of e'
// among the out-edges of to(e).  Fixed per (e, e'), so computed once when the vehicle enters e.
__device__ __forceinline__ uint32_t lane_range(uint32_t L, uint32_t K, uint32_t r) {
  const uint32_t lo = (r * L) / K;
  uint32_t hi = ((r + 1u) * L + K - 1u) / K;
  hi = (hi >= 1u ? hi - 1u : 0u);
  if (hi < lo) hi = lo;
  return lo | (hi << 8);
}

__device__ __forceinline__ Ctx make_ctx(const EdgeRec* __restrict__ edges, const uint32_t* __restrict__ route,
                                        int h_max, uint32_t e, uint32_t l, uint32_t cur, bool last) {
  const EdgeRec E = load_edge(edges, e);
  Ctx x;
  x.c0 = ctx_c0(E);
  x.v0 = E.v0;
  const uint32_t K = (E.meta >> META_KOUT_SHIFT) & META_KOUT_MASK;
  if (last) {
    x.c2 = 0; x.c3 = ctx_mirror(E); x.c4 = NONE; x.rn = 0;
    return x;
  }
  x.rn = __ldg(&route[cur + 1]);
  const EdgeRec N = load_edge(edges, x.rn & ROUTE_EDGE_MASK);
  const uint32_t nl = N.meta & META_LANES_MASK;
  x.c2 = N.ncells | (nl << 24) | ((N.meta & META_HALO) ? (1u << 30) : 0u);
  x.c3 = lane_range(E.meta & META_LANES_MASK, K, (N.meta >> META_RANK_SHIFT) & META_RANK_MASK) | ctx_mirror(E);
  x.c4 = N.base + min(l, nl - 1u) * stride_of(x.c2, h_max);
  return x;
}

// §8(e): a byte of M_{k+1} in the first h_max cells of an owned cut edge is also written into the
// upstream part's entry halo of that lane (peer memory in multi-process mode), where that part's
// probes of step k+1 read it; the halo's holder clears it wholesale in phase C of step k+1.
// mn = index of M_{k+1} in PartDev::map.
__device__ __forceinline__ void put_mirror(const Global& G, const PartDev& D, unsigned mn, uint32_t c3, uint32_t el,
                                           int cn, uint8_t b, int h_max) {
  if (!(c3 & CTX_MIRROR) || cn >= h_max) return;
  const uint2 mr = __ldg(&D.mirror[el & EDGE_MASK]);  // {upstream part, its halo cell 0 of lane 0}
  G.parts[mr.x].map[mn][mr.y + ((el >> LANE_SHIFT) & LANE_MASK) * (uint32_t)h_max + (uint32_t)cn] = b;
}

// ---------------------------------------------------------------------------
// per-vehicle move (phase A): a3 probe, a4 IDM + kinematics, a5, a6
// ---------------------------------------------------------------------------
struct MoveOut {
  uint32_t el, cur, cell_new;  // state at k+1 (or the fallback of a claimant)
  float pos, v;
  bool survive, claimant, finished;
  bool lc;                     // a lane change is possible: decided by the CTA's lane-change batch
  float plc;                   // its probability (Eq. Lane Change, Q13)
  uint32_t ccell, cel, ckind;  // claim: cell, proposed packed edge/lane, kind (1 transition, 2 lane change)
  float cv;                    // proposed speed of a transition
};

__device__ __forceinline__ void move_vehicle(const Params& P, const uint8_t* Mk, uint32_t k, uint32_t gp, uint32_t id,
                                             uint32_t el, float p, float v, uint32_t cur, uint32_t cell, const Ctx& X,
                                             MoveOut& o, unsigned long long* tmark = nullptr, bool noprobe = false) {
  const uint32_t l = (el >> LANE_SHIFT) & LANE_MASK;
  const bool last = (el & LAST_BIT) != 0u;
  const int c = (int)p;  // p >= 0: truncation == floor
  const uint32_t lane0 = cell - (uint32_t)c;
  const int Lc = (int)(X.c0 & 0xFFFFFFu);
  // H = min(H_max, max(H_min, ceil(2Δt·v))) (Alg. 1 l.11, Q7)
  int H = (int)ceilf(__fmul_rn(__fmul_rn(2.0f, P.dt), v));
  H = max(H, P.h_min);
  H = min(H, P.h_max);
  o.claimant = false;
  o.finished = false;
  o.survive = true;
  o.lc = false;

  // a3: leader probe — own lane cells c+1 .. min(c+H, Lc-1), then the next edge's entry lane (Q10).
  // Both windows (and so the entry cell of the next edge) are loaded together when the vehicle is
  // within H of the stop line — the only case in which it can reach the next edge this step.
  bool found = false, same = false;
  int gap = 0, vf = 0, cf = 0;
  const int lim = min(c + H, Lc - 1);
  const bool near = !last && c + H >= Lc;
  // Q30: a red signal at the end of e is a stopped leader just past the last cell (cell Lc of this
  // edge) for a vehicle whose probe reaches the line; gp = the phase that is green at step k
  const bool red = near && (X.c0 & (1u << 30)) != 0u && (X.c0 >> 31) != gp;
  const int reach = near ? min(c + H - Lc, (int)(X.c2 & 0xFFFFFFu) - 1) : 0;
  const uint32_t a1 = (cell + 1u) & ~15u, h1 = lane0 + (uint32_t)max(lim, c + 1);
  const uint32_t a2 = X.c4 & ~15u, h2 = near ? X.c4 + (uint32_t)reach : 0u;
  const bool fit1 = h1 - a1 < 48u, fit2 = h2 - a2 < 48u;
  uint64_t m1 = 0, m2 = 0;
  if (lim >= c + 1 && fit1 && !noprobe) m1 = occ48(Mk, a1, h1);
  if (near && !red && fit2 && !noprobe) m2 = occ48(Mk, a2, h2);
  if (tmark) {  // LPSIM_FLAG_TIMING, thread 0 of the CTA, first chunk: the probe data has arrived
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : "l"(m1 ^ m2));
    tmark[0] = t;
  }
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
    if (!found) {  // the stop line: no-overtake clamp at cell Lc keeps the vehicle on this edge
      found = true; same = true;
      cf = Lc;
      gap = Lc - c;
      vf = 0;
    }
  } else if (near) {
    uint32_t hit;
    if (fit2) {
      uint64_t m = m2 & (~0ull << (X.c4 - a2));
      m &= (2ull << (h2 - a2)) - 1ull;
      hit = m ? a2 + (uint32_t)(__ffsll((long long)m) - 1) : NONE;
      entry_free = ((m2 >> (X.c4 - a2)) & 1ull) == 0ull;
    } else {
      hit = scan_first(Mk, X.c4, h2);
      entry_free = Mk[X.c4] == 255;
    }
    if (!found && hit != NONE) {
      found = true;
      cf = (int)(hit - X.c4);
      gap = (Lc - c) + cf;
      vf = Mk[hit];
    }
  }

  // a4: IDM (Eq. Car Following, Q3/Q4/Q9), fixed op order
  const float r = __fdiv_rn(v, X.v0);
  // (v/v0)^δ by squaring, LSB first (Q6); δ = 4 (the default) is (r·r)·(r·r) of that same sequence
  float rd;
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
      o.survive = false;
      return;
    }
    const uint32_t nl = (X.c2 >> 24) & 63u;
    const uint32_t l2 = min(l, nl - 1u);  // Q21
    // fallback: wait at the stop line (Q23)
    o.el = el;
    o.pos = fmaxf(p, (float)(Lc - 1));
    o.v = 0.0f;
    o.cur = cur;
    o.cell_new = lane0 + (uint32_t)(Lc - 1);
    if (entry_free) {
      o.claimant = true;
      o.ccell = X.c4;
      o.cel = (X.rn & ROUTE_EDGE_MASK) | (l2 << LANE_SHIFT) | (X.rn & LAST_BIT);
      o.ckind = 1u;
      o.cv = vn;
    }
    return;
  }

  o.el = el;
  o.pos = pn;
  o.v = vn;
  o.cur = cur;
  const int cn = (int)pn;
  o.cell_new = lane0 + (uint32_t)cn;

  if (tmark) {  // after IDM, kinematics, the transition test
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : "f"(pn));
    tmark[1] = t;
  }
  // a6: mandatory lane change + gap acceptance (Eq. Lane Change / Gap Acceptance, Q13-Q17).  A vehicle
  // in a wrong lane with p_LC > 0 is a candidate; its draw, target-lane scans and critical gaps are
  // evaluated by the CTA's lane-change batch after the move phase's vehicle chunks (lc_decide), so
  // that divergent, rare work runs on full warps once instead of in every warp that holds one.
  if (!last && cn >= 1) {
    const uint32_t lo = X.c3 & 255u, hi = (X.c3 >> 8) & 255u;
    if (l < lo || l > hi) {
      const float x = __fsub_rn((float)Lc, p);
      float plc = __fdiv_rn(__fsub_rn(P.x0, x), P.x0);
      plc = fminf(fmaxf(plc, 0.0f), 1.0f);
      if (plc > 0.0f) {  // u in [0, 1): no change for plc == 0
        o.lc = true;
        o.plc = plc;
        // the batch's target-lane window (lc_decide, same SM) requested into L1 now, so its one
        // round of loads hits L1 (cold step -0.5 us, tools/ab.sh)
        const uint32_t tl0 = (uint32_t)((int)lane0 + (l < lo ? Lc : -Lc));
        const uint32_t aw = (tl0 + (uint32_t)max(cn - P.lc_n, 0)) & ~15u;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(Mk + aw));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(Mk + aw + 64u));
      }
    }
  }
}

// The lane-change decision of a candidate (Eq. Lane Change P:L222-225, Eq. Gap Acceptance P:L228-235,
// Q13-Q17): the Bernoulli draw, then the target cell, lead and lag in the target lane of M_k (one
// round of loads: the window [cn-n, cn+n] as 96 bytes of occupancy bits), the critical gaps and the
// lag's kinematic bound.  v = the step-k speed; returns the target cell or NONE.
__device__ __forceinline__ uint32_t lc_decide(const Params& P, const uint8_t* Mk, uint32_t k, uint32_t id, float v,
                                              float plc, uint32_t lane0, uint32_t l, int cn, int Lc, uint32_t lo,
                                              uint32_t& tl_out) {
  const int tl = l < lo ? (int)l + 1 : (int)l - 1;
  tl_out = (uint32_t)tl;
  // u in [0, 1): the draw decides only for 0 < plc < 1 (same outcome either way)
  bool draw = plc >= 1.0f;
  if (plc > 0.0f && plc < 1.0f) {
    uint32_t w[4];
    philox(id, k, 0u, 0u, P.seed_lo, P.seed_hi, w);
    draw = __fmul_rn((float)(w[0] >> 8), 0x1p-24f) < plc;
  }
  if (!draw) return NONE;
  {
    {
      const uint32_t tl0 = (uint32_t)((int)lane0 + (tl - (int)l) * Lc);
      const uint32_t tc = tl0 + (uint32_t)cn;
      // target cell, lead and lag scans of the target lane in one round of loads
      // (window [cn-n, cn+n] of the target lane as 96 bytes of occupancy bits)
      const int n = P.lc_n;
      const uint32_t wlo = tl0 + (uint32_t)max(cn - n, 0), whi = tl0 + (uint32_t)min(cn + n, Lc - 1);
      const uint32_t aw = wlo & ~15u;
      const bool fitw = whi - aw < 96u;
      bool tfree = false;
      uint32_t ld = NONE, lg = NONE;
      {
        if (fitw) {
          const uint64_t w0 = occ48(Mk, aw, whi);
          const uint64_t w1 = (aw + 48u <= whi) ? occ48(Mk, aw + 48u, whi) : 0ull;
          const unsigned bt = tc - aw;  // bit of the target cell
          tfree = ((bt < 48u ? (w0 >> bt) : (w1 >> (bt - 48u))) & 1ull) == 0ull;
          // lead: first occupied in (tc, whi]; lag: last occupied in [wlo, tc)
          const uint64_t lo_mask0 = w0 & ~((bt + 1u >= 48u) ? 0xFFFFFFFFFFFFull : ((1ull << (bt + 1u)) - 1ull));
          const uint64_t lo_mask1 = w1 & ((bt + 1u > 48u) ? ~((1ull << (bt + 1u - 48u)) - 1ull) : ~0ull);
          const unsigned hb = whi - aw;  // last valid bit
          const uint64_t hm0 = hb >= 47u ? 0xFFFFFFFFFFFFull : ((2ull << hb) - 1ull);
          const uint64_t hm1 = hb >= 48u ? ((2ull << (hb - 48u)) - 1ull) : 0ull;
          const uint64_t f0 = lo_mask0 & hm0, f1 = lo_mask1 & hm1;
          if (f0) ld = aw + (uint32_t)(__ffsll((long long)f0) - 1);
          else if (f1) ld = aw + 48u + (uint32_t)(__ffsll((long long)f1) - 1);
          const unsigned lb0 = wlo - aw;  // first valid bit
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
      }
      if (tfree) {
        const bool has_ld = ld != NONE, has_lg = lg != NONE;
        const int g_ld = has_ld ? (int)(ld - tc) : 0, b_ld = has_ld ? Mk[ld] : 0;
        const int g_lg = has_lg ? (int)(tc - lg) : 0, b_lg = has_lg ? Mk[lg] : 0;
        // critical gaps (Q15); a draw is made only where its gap is tested (same values either way)
        bool accept = true;
        if (has_ld) {
          const float eps_a = eps_draw(P, id, k, 1u, P.sigma_a_s3);
          const float g_lead = fmaxf(0.0f, __fadd_rn(__fsub_rn(__fadd_rn(P.g_a, __fmul_rn(P.alpha_i, v)),
                                                              __fmul_rn(P.alpha_a, (float)b_ld)), eps_a));
          if (!((float)g_ld >= g_lead)) accept = false;
        }
        if (has_lg && accept) {
          const int safe = (int)ceilf(__fadd_rn(__fmul_rn(__fadd_rn((float)b_lg, 1.0f), P.dt), P.half_a_dt2)) + 1;
          if (g_lg < safe) {
            accept = false;
          } else {
            const float eps_b = eps_draw(P, id, k, 2u, P.sigma_b_s3);
            const float g_lag = fmaxf(0.0f, __fadd_rn(__fsub_rn(__fadd_rn(P.g_b, __fmul_rn(P.alpha_b, (float)b_lg)),
                                                             __fmul_rn(P.alpha_i, v)), eps_b));
            if (!((float)g_lg >= g_lag)) accept = false;
          }
        }
        if (accept) return tc;
      }
    }
  }
  return NONE;
}

// ---------------------------------------------------------------------------
// phases
// ---------------------------------------------------------------------------
__device__ __forceinline__ void warp_digest(GridCtl* g, unsigned slot, uint64_t h, bool active) {
  uint64_t x = active ? h : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0 && x) atomicAdd(&g->digest[slot], (unsigned long long)x);
}

// warp-aggregated counter increment (one atomic per warp, Guideline 12)
// Event counters are accumulated per CTA in shared memory over the whole launch and flushed once
// into the CTA's private slot of Global::ctr_block (the host sums them): thousands of same-address
// global atomics per step (one per warp) serialised at one L2 slice.
enum { C_TRANS = 0, C_LC = 1, C_LOST = 2, C_DEP = 3, C_ARR = 4, C_N = 5 };
__device__ __forceinline__ void warp_count_s(unsigned long long* s_ctr, int which, bool pred) {
  const unsigned b = __ballot_sync(0xffffffffu, pred);
  if ((threadIdx.x & 31u) == 0u && b) atomicAdd(&s_ctr[which], (unsigned long long)__popc(b));
}
__device__ __forceinline__ void warp_count(unsigned long long* ctr, bool pred) {
  const unsigned b = __ballot_sync(0xffffffffu, pred);
  if ((threadIdx.x & 31u) == 0u && b) atomicAdd(ctr, (unsigned long long)__popc(b));
}

// warp-aggregated append slot in the next SoA (departures, migrants)
__device__ __forceinline__ unsigned warp_append(unsigned* ctr, bool pred) {
  const unsigned b = __ballot_sync(0xffffffffu, pred);
  const unsigned lane = threadIdx.x & 31u;
  unsigned base = 0;
  if (lane == 0u && b) base = atomicAdd(ctr, (unsigned)__popc(b));
  base = __shfl_sync(0xffffffffu, base, 0);
  return base + __popc(b & ((1u << lane) - 1u));
}

__device__ __forceinline__ void write_vehicle(const PartDev& D, unsigned nb, unsigned idx, uint32_t id, uint32_t el,
                                              float pos, float v, uint32_t cur, uint32_t cell, uint32_t pcell) {
  D.vid[nb][idx] = id;
  D.vel[nb][idx] = el;
  D.vpos[nb][idx] = pos;
  D.vv[nb][idx] = v;
  D.vcur[nb][idx] = cur;
  D.vcell[nb][idx] = cell;
  D.vpcell[nb][idx] = pcell;
}

__device__ __forceinline__ void write_ctx(const PartDev& D, unsigned idx, const Ctx& X) {
  const unsigned b = D.xb;
  D.xc0[b][idx] = X.c0;
  D.xv0[b][idx] = X.v0;
  D.xc2[b][idx] = X.c2;
  D.xc3[b][idx] = X.c3;
  D.xc4[b][idx] = X.c4;
  D.xrn[b][idx] = X.rn;
}

// On-chip residency of the vehicle state.  Chunk c = lb + j*nbv of a
// partition's SoA is processed by the same CTA (and entry i by the same
// thread) in phases A and C of every step, and nothing else writes entries
// below the step's in-place count (departures and migrants append after it).
// So for the first NSLOT chunk rounds the state of SoA_{k+1} never leaves
// shared memory inside a launch: phase A reads it from there, writes the
// move (or a claimant's fallback) back, phase C overwrites winners.  Entries
// appended during the launch are read from HBM once; the state goes back to
// the HBM SoA at the end of the launch (the sort and the host queries run
// between launches).  Chunk rounds j >= NSLOT use the HBM SoA every step.
#ifndef LPSIM_SLOTS
#define LPSIM_SLOTS 2
#endif
constexpr unsigned NSLOT = LPSIM_SLOTS;
// F_DIRTY: the cached edge context differs from the HBM copy (single-buffered, xb) and is written back
enum { F_ID = 0, F_EL, F_POS, F_V, F_CUR, F_CELL, F_PCELL, F_C0, F_V0, F_C2, F_C3, F_C4, F_RN, F_DIRTY, NF };
enum { G_CELL = 0, G_EL, G_V, G_KIND, NG };  // resident claim: cell (NONE = none), proposed el, speed, kind
// words of shared memory that phase A leaves for phase C of the same step
enum { M_RS0 = 0, M_NRS, M_NVEH, M_N };

struct VState {
  uint32_t id, el, cur, cell, pcell;
  float p, v;
  Ctx X;
};

__device__ __forceinline__ void vs_load(const uint32_t* s, VState& z) {  // s = slot base + threadIdx.x
  z.id = s[F_ID * BS]; z.el = s[F_EL * BS]; z.p = __uint_as_float(s[F_POS * BS]); z.v = __uint_as_float(s[F_V * BS]);
  z.cur = s[F_CUR * BS]; z.cell = s[F_CELL * BS]; z.pcell = s[F_PCELL * BS];
  z.X.c0 = s[F_C0 * BS]; z.X.v0 = __uint_as_float(s[F_V0 * BS]); z.X.c2 = s[F_C2 * BS]; z.X.c3 = s[F_C3 * BS];
  z.X.c4 = s[F_C4 * BS]; z.X.rn = s[F_RN * BS];
}
__device__ __forceinline__ void vs_store_ctx(uint32_t* s, const Ctx& X) {
  s[F_C0 * BS] = X.c0; s[F_V0 * BS] = __float_as_uint(X.v0); s[F_C2 * BS] = X.c2; s[F_C3 * BS] = X.c3;
  s[F_C4 * BS] = X.c4; s[F_RN * BS] = X.rn;
}
__device__ __forceinline__ void vs_store_state(uint32_t* s, uint32_t id, uint32_t el, float p, float v, uint32_t cur,
                                               uint32_t cell, uint32_t pcell) {
  s[F_ID * BS] = id; s[F_EL * BS] = el; s[F_POS * BS] = __float_as_uint(p); s[F_V * BS] = __float_as_uint(v);
  s[F_CUR * BS] = cur; s[F_CELL * BS] = cell; s[F_PCELL * BS] = pcell;
}

// Phase A.  Vehicle i of SoA_k writes its state at k+1 to index i of SoA_{k+1}
// (stable order, no compaction inside the step, so warps never wait for each
// other); a vehicle that leaves (arrival, migration) leaves a dead entry whose
// pcell phase C clears in M_k; the periodic sort / compaction drops it.
// `seen` = entries of the previous step held in shared memory (0 at launch start).
// LPSIM_FLAG_TIMING: t_block[w] += now - t_block[w0] (w0 = the phase start) for this CTA
__device__ __forceinline__ void tb_add(const Global& G, int w, int w0) {
  unsigned long long* tb = G.grid->t_block + TB_N * blockIdx.x;
  tb[w] += globaltimer() - tb[w0];
}

// The CTA's lane-change batch (a6): the candidates its warps flagged in the move phase, one per
// thread: lc_decide, then either the claim (resident: the chunk's shared-memory claim slots; in
// HBM: the claim record and its ballot bit) or the deferred non-claimant byte of M_{k+1}.
constexpr unsigned LCQ_CAP = BS > 512 ? BS : 512;  // tasks held per CTA ({SoA index, round | thread, v_k, p_LC})
template <bool FULL, bool MULTI>
__device__ void lc_batch(const Params& P, const Global& G, const PartDev& D, uint32_t k, const uint8_t* Mk,
                         uint8_t* Mn, unsigned mn, unsigned cb, unsigned nb, uint32_t* s_st, uint32_t* s_cl,
                         unsigned nslot, const uint4* s_lcq, unsigned n) {
  const bool dig = (FULL && (P.flags & 1u) != 0u);
  for (unsigned t = threadIdx.x; t < n; t += BS) {
    const uint4 tk = s_lcq[t];
    const unsigned i = tk.x, j = tk.y >> 16, th = tk.y & 0xFFFFu;
    const bool res = j < nslot;
    uint32_t id, el, cur, cell_new, c0, c3, c2 = 0u, c4 = 0u, pcell = 0u;
    float pn, vn;
    uint32_t* sc = nullptr;
    if (res) {
      const uint32_t* ss = s_st + j * (NF * BS) + th;
      sc = s_cl + j * (NG * BS) + th;
      id = ss[F_ID * BS]; el = ss[F_EL * BS]; pn = __uint_as_float(ss[F_POS * BS]); vn = __uint_as_float(ss[F_V * BS]);
      cur = ss[F_CUR * BS]; cell_new = ss[F_CELL * BS]; c0 = ss[F_C0 * BS]; c3 = ss[F_C3 * BS];
    } else {
      id = D.vid[nb][i]; el = D.vel[nb][i]; pn = D.vpos[nb][i]; vn = D.vv[nb][i]; cur = D.vcur[nb][i];
      cell_new = D.vcell[nb][i]; pcell = D.vpcell[nb][i];
      c0 = D.xc0[D.xb][i]; c3 = D.xc3[D.xb][i]; c2 = D.xc2[D.xb][i]; c4 = D.xc4[D.xb][i];
    }
    const uint32_t l = (el >> LANE_SHIFT) & LANE_MASK;
    const int cn = (int)pn;
    uint32_t tl;
    const uint32_t tc = lc_decide(P, Mk, k, id, __uint_as_float(tk.z), __uint_as_float(tk.w), cell_new - (uint32_t)cn,
                                  l, cn, (int)(c0 & 0xFFFFFFu), c3 & 255u, tl);
    if (tc != NONE) {
      // contend for the target cell (the stored state is the fallback); phase C decides (A9)
      claim_cell(&D.claim[tc], id, (P.flags & LPSIM_FLAG_RACY) != 0u);
      const uint32_t cel = (el & ~(LANE_MASK << LANE_SHIFT)) | (tl << LANE_SHIFT);
      if (res) {
        sc[G_CELL * BS] = tc;
        sc[G_EL * BS] = cel;
        sc[G_V * BS] = __float_as_uint(vn);
        sc[G_KIND * BS] = 2u;
      } else {
        ClaimRec R;
        R.idx = i; R.id = id; R.cell = tc; R.el_new = cel; R.cur_new = cur; R.pos_new = pn; R.v_new = vn;
        R.fb_cell = cell_new;
        R.fb_byte = (uint32_t)speed_byte(vn) | (2u << 8) | (l << 16);
        R.pcell = pcell;
        if (MULTI) {  // the fallback's edge context bits (mirror), its packed edge/lane and cell index
          R.x[0] = c3;
          R.x[1] = el;
          R.x[2] = (uint32_t)cn;
        }
        R.x[4] = c4;  // the lane change moves the cached entry-lane cell of the next edge
        if (!(el & LAST_BIT)) {
          const uint32_t nl = (c2 >> 24) & 63u, st = stride_of(c2, P.h_max);
          R.x[4] = c4 - min(l, nl - 1u) * st + min(tl, nl - 1u) * st;
        }
        D.crec[cb][i] = R;
        atomicOr(&D.cbits[cb][i >> 5], 1u << (i & 31u));  // after the move loop's plain store (CTA sync)
      }
    } else {
      put_map(P, G, D.ctl, Mn, cell_new, speed_byte(vn), k);  // the byte a non-claimant writes in the move loop
      if (MULTI) put_mirror(G, D, mn, c3, el, cn, speed_byte(vn), P.h_max);
      if (dig)
        atomicAdd(&G.grid->digest[k & 1u],
                  (unsigned long long)veh_hash(id, el, pn, vn, cur - __ldg(&G.trip_rstart[id])));
    }
  }
}


// Admit positions go out one warp chunk (32 positions) at a time from the last CTA down.  With
// dedicated admit CTAs (nbv < nbp: CTAs nbv..nbp-1 take no vehicle chunks) they go to those CTAs
// only, so that a departure chain (claim word -> append + successor search -> relist) starts at the
// beginning of phase C instead of after a vehicle chunk round's claims.  Phases A and C agree on the
// map.  Returns NONE for a CTA without admit work.
#ifndef LPSIM_ADM_WARPS
#define LPSIM_ADM_WARPS 8
#endif
constexpr unsigned ADM_WARPS = LPSIM_ADM_WARPS;  // warps whose first admit chunk phase A stashes in shared memory
__device__ __forceinline__ unsigned admit_chunk(unsigned lb, unsigned nbp, unsigned nbv, unsigned r) {
  const unsigned w = (threadIdx.x >> 5) + (BS / 32u) * r;
  if (nbv == nbp) return (nbp - 1u - lb) + nbp * w;
  if (lb < nbv) return NONE;
  return (nbp - 1u - lb) + (nbp - nbv) * w;
}

// block-collective (§8(e)): the migrants on this part at snapshot k, by sender u (counted by the
// senders in phase C of step k-1): exclusive prefix into s_mp[0..np]; returns the total
__device__ __forceinline__ unsigned mig_prefix(const Global& G, const PartDev& D, unsigned part, uint32_t k,
                                               unsigned* s_mp) {
  static_assert(BS >= 256, "one thread per sender (num_parts <= 255)");
  __shared__ unsigned s_w[BS / 32];
  const unsigned np = G.n_parts, u = threadIdx.x, lane = u & 31u, w = u >> 5;
  unsigned x = 0;
  if (u < np && u != part) {
    x = *((volatile const uint32_t*)&G.mig_cnt[(k & 1u) * np * np + u * np + part]);
    x = min(x, __ldg(&D.rq_off[u + 1]) - __ldg(&D.rq_off[u]));  // (at most one per cut lane and step)
  }
  unsigned v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (unsigned)o) v += y;
  }
  if (lane == 31u) s_w[w] = v;
  __syncthreads();
  unsigned before = 0, total = 0;
#pragma unroll
  for (unsigned q = 0; q < BS / 32; ++q) {
    const unsigned t = s_w[q];
    before += q < w ? t : 0u;
    total += t;
  }
  if (u <= np) s_mp[u] = before + v - x;  // u == np: the total
  __syncthreads();
  return total;
}

template <bool FULL, bool MULTI>
__device__ void phase_a(const Params& P, const Global& G, const PartDev& D, unsigned long long k64, unsigned mk, unsigned lb,
                        unsigned nbp, unsigned nbv, unsigned part, unsigned* s_mp, uint4* s_res,
                        unsigned long long* s_ctr, uint32_t* s_st, uint32_t* s_cl, unsigned& seen,
                        unsigned* s_pref, unsigned* s_misc, unsigned nslot, uint4* s_lcq, unsigned* s_lcq_n,
                        uint4* s_adm) {
  const uint32_t k = (uint32_t)k64;
  // Q30: the signal phase that is green at step k (every signal in phase: phase 0 green for the
  // first half of each cycle)
  const uint32_t gp = P.sig_cycle > 0 ? ((k % (uint32_t)P.sig_cycle) < (uint32_t)(P.sig_cycle / 2) ? 0u : 1u) : 0u;
  const unsigned cb = k & 1u, nb = cb ^ 1u;
  const uint8_t* Mk = D.map[mk];
  uint8_t* Mn = D.map[mk ^ 1u];
  PartCtl* ctl = D.ctl;
  const unsigned gtid = lb * BS + threadIdx.x;
  const bool dig = (FULL && (P.flags & 1u) != 0u);
  if ((FULL && (P.flags & 8u)) && threadIdx.x == 0 && G.grid->t_block) G.grid->t_block[TB_N * blockIdx.x + 2] = globaltimer();
  const unsigned nveh = ctl->n_veh[cb];
  // migrants received at snapshot k (§8(e)): entries nveh .. ntot-1 of this step, read from the
  // receive queue; SoA_{k+1} holds them in place like every other entry
  const unsigned nmig = (MULTI && G.n_parts > 1u) ? mig_prefix(G, D, part, k, s_mp) : 0u;
  const unsigned ntot = nveh + nmig;
  if (gtid == 0) {
    const unsigned ndead = ctl->n_dead[cb];
    ctl->n_veh[nb] = ntot;  // in-place indices; phase C appends after them
    ctl->updates += ntot - ndead;  // every live entry is one vehicle-update
    atomicAdd(&ctl->n_dead[nb], ndead);  // dead entries stay dead; new deaths are added as they happen
    if (ntot > D.veh_cap) set_error(G.grid, ctl, ERR_CAPACITY, 8, k);
  }
  // loaded now, used after the vehicle chunks: release-list bounds of steps k and k+1, releases
  // of step k (their bitmap bits are set in this phase; phase C's departure search reads them)
  unsigned rs0 = 0, rs1 = 0, m0 = 0, m1 = 0, r0 = 0, r1 = 0;
  if (k < D.rel_steps) {
    rs0 = __ldg(&D.rs_ptr[k]);
    rs1 = __ldg(&D.rs_ptr[k + 1u]);
    r0 = __ldg(&D.rel_ptr[k]);
    r1 = __ldg(&D.rel_ptr[k + 1u]);
  }
  if (k + 1u < D.rel_steps) {
    m0 = rs1;
    m1 = __ldg(&D.rs_ptr[k + 2u]);
  }
  // the pending-slot counters are loaded now and scanned after the vehicle chunks
  unsigned c_lo = 0, c_hi = 0;
  if (threadIdx.x < 32) {
    c_lo = min(D.sh_slot[cb][(2 * threadIdx.x) * SH_STRIDE], D.slot_shcap);
    c_hi = min(D.sh_slot[cb][(2 * threadIdx.x + 1) * SH_STRIDE], D.slot_shcap);
  }
  // array pointers are read from the shared-memory descriptor where used
  // (hoisting ~25 of them into registers cost ~50 registers per thread)
  const unsigned xb = D.xb;
  if (MULTI && nmig > 0u && lb < nbv) {
    // the migrants received at snapshot k (§8(e)) become entries nveh .. ntot-1 of SoA_k (its free
    // capacity past the count), written by the CTA whose chunks hold them: the chunk loop then reads
    // them like the entries appended in the previous step (no extra path in the loop)
    bool any = false;  // block-uniform
    for (unsigned c = nveh / BS; c * BS < ntot; ++c) {
      if (c % nbv != lb) continue;
      any = true;
      const unsigned i = c * BS + threadIdx.x;
      if (i < nveh || i >= ntot) continue;
      const unsigned jm = i - nveh;
      unsigned lo = 0, hi = G.n_parts;  // its sender u: s_mp[u] <= jm < s_mp[u + 1]
      while (hi - lo > 1u) {
        const unsigned mid = (lo + hi) >> 1;
        if (s_mp[mid] <= jm) lo = mid;
        else hi = mid;
      }
      const MigSlot m = D.inq[k & 1u][__ldg(&D.rq_off[lo]) + (jm - s_mp[lo])];
      write_vehicle(D, cb, i, m.id, m.el, 0.0f, m.v, m.cur, m.cell, NONE);  // at pos 0 of its lane
      write_ctx(D, i, make_ctx(D.edges, G.route, P.h_max, m.el & EDGE_MASK, (m.el >> LANE_SHIFT) & LANE_MASK, m.cur,
                               (m.el & LAST_BIT) != 0u));
    }
    if (any) __syncthreads();
  }
  const unsigned seen_prev = seen;
  unsigned ch0 = lb;
  for (unsigned j = 0;; ++j, ch0 += nbv) {
    if (lb >= nbv) break;  // a dedicated admit CTA (block-uniform)
    if (j * BS + BS > LCQ_CAP && ch0 * BS < ntot) {  // block-uniform: room for one more round of candidates
      __syncthreads();
      if (*s_lcq_n + BS > LCQ_CAP) {
        lc_batch<FULL, MULTI>(P, G, D, k, Mk, Mn, mk ^ 1u, cb, nb, s_st, s_cl, nslot, s_lcq, *s_lcq_n);
        __syncthreads();
        if (threadIdx.x == 0) *s_lcq_n = 0u;
        __syncthreads();
      }
    }
    {
      // the next round's chunk, when it is not held in shared memory: its SoA and edge-context
      // lines are requested into L2 now (12 arrays x 8 lines of 128 B, one per thread), so that
      // round starts from L2 hits instead of HBM (the first step of a launch, > NSLOT rounds)
      const unsigned c1 = ch0 + nbv;
      const bool known1 = j + 1u < nslot && (c1 + 1u) * BS <= seen_prev;  // block-uniform
      if (!known1 && c1 * BS < ntot && threadIdx.x < 96u) {
        const unsigned f = threadIdx.x >> 3, ln = threadIdx.x & 7u;
        const uint32_t* const* tb = f < 6u ? (const uint32_t* const*)&D.vid[0] : (const uint32_t* const*)&D.xc0[0];
        const uint32_t* a = tb[2u * (f < 6u ? f : f - 6u) + (f < 6u ? cb : xb)];
        prefetch_l2(a + c1 * BS + ln * 32u);
      }
    }
    const unsigned i = ch0 * BS + threadIdx.x;
    const bool res = j < nslot;  // block-uniform
    uint32_t* ss = s_st + (res ? j : 0u) * (NF * BS) + threadIdx.x;
    uint32_t* sc = s_cl + (res ? j : 0u) * (NG * BS) + threadIdx.x;
    const bool have = res && i < seen_prev;
    // a chunk held in shared memory is below the previous count, which the current one never
    // undercuts inside a launch (entries are not removed): no wait for the count, no HBM loads
    const bool known = res && (ch0 + 1u) * BS <= seen_prev;  // block-uniform
    VState z;
    // valid: an entry of SoA_k.  Decided inside the branches so that a resident round (known) has no
    // dependency on this step's count (its load is still in flight at the first round)
    bool valid = true;
    if (known) {
      vs_load(ss, z);
    } else {
      // HBM fields loaded at once, before the vehicle count is known (speculative within the
      // buffer's capacity) and with no control dependency on the id
      const bool mem = !have && i < D.veh_cap;
      z.id = mem ? D.vid[cb][i] : NONE;
      z.el = mem ? D.vel[cb][i] : 0u;
      z.p = mem ? D.vpos[cb][i] : 0.0f;
      z.v = mem ? D.vv[cb][i] : 0.0f;
      z.cur = mem ? D.vcur[cb][i] : 0u;
      z.cell = mem ? D.vcell[cb][i] : 0u;
      z.X.c0 = mem ? D.xc0[xb][i] : 0u;
      z.X.v0 = mem ? D.xv0[xb][i] : 1.0f;
      z.X.c2 = mem ? D.xc2[xb][i] : 0u;
      z.X.c3 = mem ? D.xc3[xb][i] : 1u;
      z.X.c4 = mem ? D.xc4[xb][i] : 0u;
      z.X.rn = mem ? D.xrn[xb][i] : 0u;
      if (have) vs_load(ss, z);
      if (ch0 * BS >= ntot) break;  // block-uniform
      valid = have || i < ntot;
    }
    bool keep = false, claim = false, fin = false, lcp = false;
    float lc_plc = 0.0f;
    uint64_t h = 0;
    if (valid) {
      const uint32_t id = z.id, el = z.el, cur = z.cur, cell = z.cell;
      if (res && !have) {
        vs_store_ctx(ss, z.X);
        ss[F_DIRTY * BS] = 0u;
      }
      uint32_t ccell = NONE;
      if (id == NONE) {  // dead entry: stays dead, nothing to clear in phase C
        if (res) {
          ss[F_ID * BS] = NONE;
          ss[F_PCELL * BS] = NONE;
        } else {
          D.vid[nb][i] = NONE;
          D.vpcell[nb][i] = NONE;
        }
      } else {
        MoveOut o;
        unsigned long long tm[2];
        const bool tmk = (FULL && (P.flags & 8u)) && j == 0 && threadIdx.x == 0 && G.grid->t_block;
#ifdef LPSIM_EXP
        move_vehicle(P, Mk, k, gp, id, el, z.p, z.v, cur, cell, z.X, o, tmk ? tm : nullptr,
                     (P.flags & 0x8000u) && j == 1u);  // timing experiments: round 2 without its probe loads
#else
        move_vehicle(P, Mk, k, gp, id, el, z.p, z.v, cur, cell, z.X, o, tmk ? tm : nullptr);
#endif
        if (tmk) {
          unsigned long long* tb = G.grid->t_block + TB_N * blockIdx.x;
          tb[16] += tm[0] - tb[2];  // probe data in
          tb[17] += tm[1] - tb[2];  // longitudinal move done
          tb_add(G, 11, 2);         // move done (lane change included)
        }
        if (o.finished) {  // Q24: arrival at k+1; phase C clears the cell in M_k
          G.arrival_step[id] = (int32_t)(k + 1);
          if (res) {
            ss[F_ID * BS] = NONE;
            ss[F_PCELL * BS] = cell;
          } else {
            D.vid[nb][i] = NONE;
            D.vpcell[nb][i] = cell;
          }
          fin = true;
        } else {
          if (res) {
            vs_store_state(ss, id, o.el, o.pos, o.v, o.cur, o.cell_new, cell);
          } else {
            D.vid[nb][i] = id;
            D.vel[nb][i] = o.el;
            D.vpos[nb][i] = o.pos;
            D.vv[nb][i] = o.v;
            D.vcur[nb][i] = o.cur;
            D.vpcell[nb][i] = cell;
            D.vcell[nb][i] = o.cell_new;
          }
          if (o.claimant) {
            // contend for the cell (the state above is the fallback); phase C decides.
            // A9: the lowest id wins; LPSIM_FLAG_RACY (ablation): the first contender to arrive
            claim_cell(&D.claim[o.ccell], id, (P.flags & LPSIM_FLAG_RACY) != 0u);
            claim = true;
            if (o.ckind == 1u) {  // phase C builds a winner's new edge context from these: into L2 now
              prefetch_l2(D.edges + (z.X.rn & ROUTE_EDGE_MASK));
              if (!(z.X.rn & LAST_BIT)) prefetch_l2(G.route + cur + 2u);
            }
            if (res) {  // resident: the claim stays in shared memory with the fallback state
              ccell = o.ccell;
              sc[G_EL * BS] = o.cel;
              sc[G_V * BS] = __float_as_uint(o.cv);
              sc[G_KIND * BS] = o.ckind;
            } else {
              // the record lives at the vehicle's own index; a ballot word marks the claimants
              ClaimRec R;
              R.idx = i;
              R.id = id;
              R.cell = o.ccell;
              R.el_new = o.cel;
              const bool tr = o.ckind == 1u;
              R.cur_new = tr ? cur + 1u : cur;
              R.pos_new = tr ? 0.0f : o.pos;  // Q20: enter at pos 0
              R.v_new = o.cv;
              R.fb_cell = o.cell_new;
              R.fb_byte = (uint32_t)speed_byte(o.v) | (o.ckind << 8) | (((el >> LANE_SHIFT) & LANE_MASK) << 16);
              R.pcell = cell;
              if (MULTI) {  // the fallback's edge context bits (mirror), its packed edge/lane and cell index
                R.x[0] = z.X.c3;
                R.x[1] = el;
                R.x[2] = (uint32_t)(int)o.pos;
              }
              // a lane change moves the cached entry-lane cell of the next edge (a transition's
              // new context is built in phase C, for winners only)
              R.x[4] = z.X.c4;
              if (!tr && !(el & LAST_BIT)) {
                const uint32_t nl_new = (o.cel >> LANE_SHIFT) & LANE_MASK;
                const uint32_t nl = (z.X.c2 >> 24) & 63u, st = stride_of(z.X.c2, P.h_max);
                const uint32_t ol = (el >> LANE_SHIFT) & LANE_MASK;
                R.x[4] = z.X.c4 - min(ol, nl - 1u) * st + min(nl_new, nl - 1u) * st;
              }
              D.crec[cb][i] = R;
            }
          } else if (o.lc) {
            lcp = true;  // lane-change candidate: decided by the batch (which writes its byte then)
            lc_plc = o.plc;
          } else {
            put_map(P, G, ctl, Mn, o.cell_new, speed_byte(o.v), k);
            if (MULTI) put_mirror(G, D, mk ^ 1u, z.X.c3, o.el, (int)o.pos, speed_byte(o.v), P.h_max);
            keep = true;
            if (dig) h = veh_hash(id, o.el, o.pos, o.v, o.cur - __ldg(&G.trip_rstart[id]));
          }
        }
      }
      if (res) sc[G_CELL * BS] = ccell;
    }
    if (!res) {
      const unsigned bc = __ballot_sync(0xffffffffu, claim);
      if ((threadIdx.x & 31u) == 0u) D.cbits[cb][i >> 5] = bc;  // plain store, no atomic
    }
    if (dig) warp_digest(G.grid, (unsigned)(k & 1u), h, keep);
    {  // lane-change candidates -> the CTA's batch queue (warp-aggregated)
      const unsigned bl = __ballot_sync(0xffffffffu, lcp);
      if (bl) {
        const unsigned lane = threadIdx.x & 31u;
        unsigned base = 0;
        if (lane == 0u) base = atomicAdd(s_lcq_n, (unsigned)__popc(bl));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (lcp)
          s_lcq[base + __popc(bl & ((1u << lane) - 1u))] =
              make_uint4(i, (j << 16) | threadIdx.x, __float_as_uint(z.v), __float_as_uint(lc_plc));
      }
    }
    {  // arrivals (rare): one atomic per warp that has any
      const unsigned bf = __ballot_sync(0xffffffffu, fin);
      if ((threadIdx.x & 31u) == 0u && bf) {
        atomicAdd(&s_ctr[C_ARR], (unsigned long long)__popc(bf));
        atomicAdd(&ctl->n_dead[nb], (unsigned)__popc(bf));
      }
    }
  }
  __syncthreads();
  if (*s_lcq_n) {  // block-uniform
    lc_batch<FULL, MULTI>(P, G, D, k, Mk, Mn, mk ^ 1u, cb, nb, s_st, s_cl, nslot, s_lcq, *s_lcq_n);
    __syncthreads();
    if (threadIdx.x == 0) *s_lcq_n = 0u;
  }
  if ((FULL && (P.flags & 8u)) && threadIdx.x == 0 && G.grid->t_block) tb_add(G, 12, 2);

#ifdef LPSIM_EXP
  if ((P.flags & 0x100000u) && (lb < nbv)) {  // timing experiments: delay this CTA by 2 us (critical-path probe)
    const unsigned long long t0 = globaltimer();
    while (globaltimer() - t0 < 2000ull) {}
  }
#endif
  seen = ntot;
  const unsigned n_vrounds = (ch0 - lb) / nbv;  // vehicle chunk rounds of this CTA
  // admit (A7): lowest released id of each pending slot claims its entry cell if free in M_k.
  // Admit positions = the slots carried over from step k-1 (sharded list) followed by the slots
  // of the release list of step k; admit chunks follow the vehicle chunks in the block's chunk
  // sequence.
  if (threadIdx.x < 32) {
    const unsigned lane = threadIdx.x;
    unsigned x = c_lo + c_hi;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (unsigned)o) x += y;
    }
    s_pref[2 * lane + 1] = x - c_hi;
    s_pref[2 * lane + 2] = x;
    if (lane == 0) {
      s_pref[0] = 0;
      s_misc[M_RS0] = rs0;
      s_misc[M_NRS] = rs1 - rs0;
      s_misc[M_NVEH] = ntot;
    }
  }
  __syncthreads();
  const unsigned nsl = s_pref[NSH];
  const unsigned nfl = nsl + s_misc[M_NRS];
  // admit chunks go to the CTAs from the last one down (vehicle chunks from the first one up), so
  // the admit work does not depend on the vehicle count
  unsigned n_arounds = 0;
  // Admit positions go out one warp (32 positions) at a time, from the last CTA down, so the few
  // hundred positions of a step spread over as many SMs as possible (a 256-position chunk put
  // every departure of the step on one or two CTAs, which then set the resolve phase's length)
  for (unsigned r = 0;; ++r, ++n_arounds) {
    const unsigned ac = admit_chunk(lb, nbp, nbv, r);  // warp chunk
    if (ac == NONE || ac * 32u >= nfl) break;  // warp-uniform
#ifdef LPSIM_EXP
    if (P.flags & 0x200u) break;  // timing experiment builds only: no admits (with 0x100)
#endif
    const unsigned f = ac * 32u + (threadIdx.x & 31u);
    if (f < nfl) {
      // the slot's lowest released, not departed trip {rank, id}: carried in the list entry, or for
      // a slot of the release list of step k the minimum of the slot's word (written by phase C of
      // step k-1, NONE if the slot was empty) and the step's lowest release (rank order = id order)
      uint32_t s;
      uint4 si;  // {entry cell, bitmap offset, width, offset into slot_trip}
      uint2 cw;
      uint32_t kmin = NONE;  // the slot's lowest release of step k other than the candidate (bm_after)
      if (f < nsl) {
        const uint32_t j = sh_locate(s_pref, f, D.slot_shcap);
        s = D.slot_list[cb][j];  // NONE: a reserved entry left unused by phase C of step k-1
        si = D.slot_li[cb][j];
        cw = D.slot_lc[cb][j];
        if (s == NONE) cw = make_uint2(NONE, NONE);
      } else {
        const uint32_t j = s_misc[M_RS0] + (f - nsl);
        s = __ldg(&D.rs_slot[j]);
        si = __ldg(&D.rs_info[j]);
        const uint2 rc = __ldg(&D.rs_cand[j]);
        const uint32_t r2 = __ldg(&D.rs_r2[j]);
        const uint2 old = D.slot_cw[s];
        cw = old.x < rc.x ? old : rc;
        kmin = cw.x == rc.x ? r2 : rc.x;  // (a carried slot has no release at step k)
      }
      // entry cell state and (after a departure) the candidate's id, loaded together
      const bool unk = cw.x != NONE && cw.y == IDUNK;
      const uint32_t lid = unk ? __ldg(&D.slot_trip[si.w + cw.x]) : 0u;
      const bool free_cell = cw.x != NONE && Mk[si.x] == 255;
      if (unk) cw.y = lid;
      uint32_t cell = NONE, succ = NONE;
      if (free_cell) {  // entry cell free in M_k: contend (A7)
        claim_cell(&D.claim[si.x], cw.y, (P.flags & LPSIM_FLAG_RACY) != 0u);
        cell = si.x;
        // the candidate's successor if it departs, found now (off phase C's departure chain)
        succ = min(bm_after(D.bm + si.y, si.z, cw.x), kmin);
        prefetch_l2(G.trip_rstart + cw.y);
        prefetch_l2(D.tel + cw.y);
#pragma unroll
        for (int t = 0; t < 6; ++t) prefetch_l2(D.tx[t] + cw.y);
      }
      // reservations, so that phase C's departure chain is one round trip (claim word -> stores): an
      // entry of the pending list of step k+1 for every position with a candidate (left unused -- slot
      // NONE -- if the slot drops out or goes to the release list of step k+1), a SoA_{k+1} entry for
      // every claim (a dead entry if the claim is lost or the departure migrates)
      const bool rq = cw.x != NONE, ra = cell != NONE;
      const unsigned lane = threadIdx.x & 31u, below = (1u << lane) - 1u;
      const unsigned shard = __shfl_sync(__activemask(), sh_shard(f), 0);
      const unsigned am = __activemask();
      const unsigned bq = __ballot_sync(am, rq), ba = __ballot_sync(am, ra);
      const unsigned leader = __ffs(am) - 1u;
      unsigned base_q = 0, base_a = 0;
      if (lane == leader) {
        if (bq) base_q = atomicAdd(&D.sh_slot[nb][shard * SH_STRIDE], (unsigned)__popc(bq));
        if (ba) base_a = atomicAdd(&ctl->n_res[nb], (unsigned)__popc(ba));
      }
      base_q = __shfl_sync(am, base_q, leader);
      base_a = __shfl_sync(am, base_a, leader);
      const unsigned jq = base_q + __popc(bq & below);
      const uint4 res = make_uint4(succ, (rq && jq < D.slot_shcap) ? shard * D.slot_shcap + jq : NONE,
                                   ra ? base_a + __popc(ba & below) : NONE, 0u);
      if (rq && jq >= D.slot_shcap) set_error(G.grid, ctl, ERR_CAPACITY, 7, k);
      if (s_adm && r == 0u && (threadIdx.x >> 5) < ADM_WARPS) {  // the warp's first chunk: phase C of this CTA reads it here
        const unsigned sa = (threadIdx.x >> 5) * 64u + (threadIdx.x & 31u);
        s_adm[sa] = make_uint4(cw.x, cw.y, cell, s);
        s_adm[sa + 32u] = si;
        s_res[threadIdx.x] = res;
      } else {
        D.slot_cand[f] = make_uint4(cw.x, cw.y, cell, s);
        D.slot_ci[f] = si;
        D.slot_cs[f] = res;
      }
    }
  }
  if ((FULL && (P.flags & 8u)) && threadIdx.x == 0 && G.grid->t_block) tb_add(G, 13, 2);
  // releases of step k (depart step k): bitmap bits only, read by phase C's departure search
#ifdef LPSIM_EXP
  if (P.flags & 0x400u) r1 = r0;  // timing experiment builds only: no releases
#endif
  for (unsigned j = r0 + (nbp - 1u - lb) * BS + threadIdx.x; j < r1; j += nbp * BS) {
    const uint4 rl = __ldg(&D.rel4[j]);  // {slot, rank in slot, bitmap offset, width}
    bm_set(D.bm + rl.z, rl.w, rl.y);
    atomicAdd(&D.slot_nrel[rl.x], 1u);
  }
  // mark the slots of the release list of step k+1 (read by phase C's carry-over); done by the
  // part's last CTAs, which have the least other work
  for (unsigned j = m0 + (nbp - 1u - lb) * BS + threadIdx.x; j < m1; j += nbp * BS) D.slot_relk[__ldg(&D.rs_slot[j])] = k + 1u;
  if ((FULL && (P.flags & 8u)) && G.grid->t_block) {  // slowest warp of the CTA
    __shared__ unsigned long long s_tend;
    if (threadIdx.x == 0) s_tend = 0ull;
    __syncthreads();
    if ((threadIdx.x & 31u) == 0u) atomicMax(&s_tend, globaltimer());
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long* tb = G.grid->t_block + TB_N * blockIdx.x;
      tb[0] += s_tend - tb[2];
      tb[8] = s_tend;
      tb[10] = n_vrounds + n_arounds;  // chunk rounds of this CTA (vehicle + admit)
    }
  }
}

// Hand a vehicle that won the entry cell of a cut edge (cell hcell of this part's entry halo) to the
// edge owner (§8(e)), straight into the owner's memory: the migrant record into its receive queue of
// snapshot k+1 (this part's region, position from this part's own counter), its byte into the
// owner's M_{k+1}, and into this part's entry halo of M_{k+1}.  The owner moves it in phase A of step
// k+1; the counts reach the owner at the step's barrier.  Lc = cells per lane of the edge.
__device__ __forceinline__ void send_migrant(const Global& G, const PartDev& D, unsigned part, unsigned mk, uint32_t k,
                                             uint32_t id, uint32_t el, float v, uint32_t cur, uint32_t Lc,
                                             uint32_t hcell) {
  const uint32_t e = el & EDGE_MASK, l = (el >> LANE_SHIFT) & LANE_MASK;
  const uint2 hd = __ldg(&D.halo_dst[e]);  // {owner, its cell 0 of lane 0}
  const uint32_t q = hd.x, np = G.n_parts, par = (k + 1u) & 1u;
  const uint32_t t = atomicAdd(&G.mig_cnt[par * np * np + part * np + q], 1u);  // <= one per cut lane
  MigSlot m;
  m.id = id;
  m.el = el;
  m.v = v;
  m.cur = cur;
  m.cell = hd.y + l * Lc;
  m.pad[0] = m.pad[1] = m.pad[2] = 0u;
  const uint8_t b = speed_byte(v);
  const PartDev* Q = G.parts + q;
  Q->inq[par][__ldg(&D.send_off[q]) + t] = m;
  Q->map[mk ^ 1u][m.cell] = b;
  D.map[mk ^ 1u][hcell] = b;
}

template <bool FULL, bool MULTI>
__device__ void phase_c(const Params& P, const Global& G, const PartDev& D, unsigned long long k64, unsigned mk, unsigned lb,
                        unsigned nbp, unsigned nbv, unsigned part, const uint4* s_res, unsigned long long* s_ctr,
                        uint32_t* s_st, uint32_t* s_cl,
                        const unsigned* s_pref, const unsigned* s_misc, unsigned nslot, const uint4* s_adm) {
  const uint32_t k = (uint32_t)k64;
  const unsigned cb = k & 1u, nb = cb ^ 1u;
  uint8_t* Mn = D.map[mk ^ 1u];
  // M_k is read only in phase A: here every entry of SoA_{k+1} clears the cell it held at k
  // (pcell; a vehicle that left keeps its dead entry's).  Every occupied cell of M_k belongs to
  // exactly one entry, so M_k is all free afterwards and its buffer serves as M_{k+2} (two maps,
  // no memset)
  uint8_t* Mk = D.map[mk];
  PartCtl* ctl = D.ctl;
  const unsigned gtid = lb * BS + threadIdx.x;
  const bool dig = (FULL && (P.flags & 1u) != 0u);
  if ((FULL && (P.flags & 8u)) && threadIdx.x == 0 && G.grid->t_block) G.grid->t_block[TB_N * blockIdx.x + 3] = globaltimer();
  // Work items: claim chunks (the same chunk -> CTA map as phase A's vehicle chunks), then
  // admit-position chunks (the same map as phase A's admit chunks).  Sizes come from phase A
  // through shared memory (no global loads before the first item).
  const unsigned nveh_k = s_misc[M_NVEH];  // entries of SoA_k (appends of this step go to SoA_{k+1})
  if (MULTI && G.n_parts > 1u) {
    // §8(e): this part's entry halos of M_k were read by phase A only; cleared wholesale (their bytes
    // were written by the edge owners and by this part's migrants), the buffer is M_{k+2}.  The counts
    // of the migrants received at snapshot k were read by the owners in phase A: reset for step k+1.
    for (uint32_t c = D.halo_lo + gtid; c < D.ncells; c += nbp * BS) Mk[c] = 255;
    if (gtid < G.n_parts) G.mig_cnt[(k & 1u) * G.n_parts * G.n_parts + part * G.n_parts + gtid] = 0u;
  }
  const unsigned n_cc = (nveh_k + BS - 1) / BS;
  const unsigned nfl = s_pref[NSH] + s_misc[M_NRS];  // admit positions of this step
  const uint32_t k1 = k + 1u;
  unsigned jr = 0;  // chunk round of this CTA (phase A's j)
  for (unsigned q = lb; lb < nbv && q < n_cc; q += nbv, ++jr) {
    {
      // resolve vehicle claims: lowest id wins (A9); the winner resets the claim word
      uint64_t h = 0;
      bool act = false, won = false, lost = false, mig = false;
      uint32_t kind = 0;
      const unsigned iv = q * BS + threadIdx.x;  // vehicle index in SoA_k
#if !LPSIM_CLEAR_LATE
      if (jr >= nslot) {  // (a resident chunk has the cell in shared memory, below)
        const uint32_t pc = iv < nveh_k ? D.vpcell[nb][iv] : NONE;
        if (pc != NONE) Mk[pc] = 255;  // clear of M_k
      }
#endif
      if (jr < nslot) {
        // resident chunk: claim and fallback state are in shared memory
        uint32_t* ss = s_st + jr * (NF * BS) + threadIdx.x;
        const uint32_t* sc = s_cl + jr * (NG * BS) + threadIdx.x;
        const uint32_t ccell = iv < nveh_k ? sc[G_CELL * BS] : NONE;
#if !LPSIM_CLEAR_LATE
        const uint32_t pc = iv < nveh_k ? ss[F_PCELL * BS] : NONE;
        if (pc != NONE) Mk[pc] = 255;  // clear of M_k
#endif
        if (ccell != NONE) {
          const uint32_t id = ss[F_ID * BS];
          const uint32_t cel = sc[G_EL * BS];
          const float cv = __uint_as_float(sc[G_V * BS]);
          kind = sc[G_KIND * BS];
          const bool tr = kind == 1u;
          const uint32_t cur = ss[F_CUR * BS];
          const uint32_t cur_new = tr ? cur + 1u : cur;
          const uint32_t e_new = cel & EDGE_MASK;
          const bool nlast = (cel & LAST_BIT) != 0u;
          const EdgeRec En = tr ? load_edge(D.edges, e_new) : EdgeRec{};
          const uint32_t rn2 = (tr && !nlast) ? __ldg(&G.route[cur_new + 1u]) : 0u;
          won = (D.claim[ccell] == id);
          lost = !won;
          if (won) {
            D.claim[ccell] = NONE;
            if (tr && G.edge_entry) G.edge_entry[cur_new] = (int32_t)k1;  // t_start of the new edge
            mig = MULTI && tr && (En.meta & META_HALO) != 0u;
            if (mig) {  // continues on another partition: migrant; its old cell is cleared above
              send_migrant(G, D, part, mk, k, id, cel, cv, cur_new, En.ncells, ccell);
              ss[F_ID * BS] = NONE;
              if (dig) { h = veh_hash(id, cel, 0.0f, cv, cur_new - __ldg(&G.trip_rstart[id])); act = true; }
            } else {
              const float pos_new = tr ? 0.0f : __uint_as_float(ss[F_POS * BS]);  // Q20: enter at pos 0
              const uint32_t el_old = ss[F_EL * BS];
              ss[F_EL * BS] = cel;
              ss[F_POS * BS] = __float_as_uint(pos_new);
              ss[F_V * BS] = __float_as_uint(cv);
              ss[F_CUR * BS] = cur_new;
              ss[F_CELL * BS] = ccell;
              put_map(P, G, ctl, Mn, ccell, speed_byte(cv), k);
              if (MULTI && !tr) put_mirror(G, D, mk ^ 1u, ss[F_C3 * BS], cel, (int)pos_new, speed_byte(cv), P.h_max);
              if (tr) {  // new edge: its cached context (make_ctx with the loads issued above)
                Ctx Y;
                Y.c0 = ctx_c0(En);
                Y.v0 = En.v0;
                const uint32_t K = (En.meta >> META_KOUT_SHIFT) & META_KOUT_MASK;
                if (nlast) {
                  Y.c2 = 0; Y.c3 = MULTI ? ctx_mirror(En) : 0u; Y.c4 = NONE; Y.rn = 0;
                } else {
                  const EdgeRec N2 = load_edge(D.edges, rn2 & ROUTE_EDGE_MASK);
                  const uint32_t nl2 = N2.meta & META_LANES_MASK;
                  Y.rn = rn2;
                  Y.c2 = N2.ncells | (nl2 << 24) | ((N2.meta & META_HALO) ? (1u << 30) : 0u);
                  Y.c3 = lane_range(En.meta & META_LANES_MASK, K, (N2.meta >> META_RANK_SHIFT) & META_RANK_MASK) |
                         (MULTI ? ctx_mirror(En) : 0u);
                  const uint32_t nl_new = (cel >> LANE_SHIFT) & LANE_MASK;
                  Y.c4 = N2.base + min(nl_new, nl2 - 1u) * stride_of(Y.c2, P.h_max);
                }
                vs_store_ctx(ss, Y);
                ss[F_DIRTY * BS] = 1u;
              } else if (!(cel & LAST_BIT)) {  // lane change: only the entry-lane cell of the next edge moves
                const uint32_t c2 = ss[F_C2 * BS];
                const uint32_t nl = (c2 >> 24) & 63u, st = stride_of(c2, P.h_max);
                const uint32_t ol = (el_old >> LANE_SHIFT) & LANE_MASK, nl_new = (cel >> LANE_SHIFT) & LANE_MASK;
                ss[F_C4 * BS] = ss[F_C4 * BS] - min(ol, nl - 1u) * st + min(nl_new, nl - 1u) * st;
                ss[F_DIRTY * BS] = 1u;
              }
              if (dig) { h = veh_hash(id, cel, pos_new, cv, cur_new - __ldg(&G.trip_rstart[id])); act = true; }
            }
          } else {
            put_map(P, G, ctl, Mn, ss[F_CELL * BS], speed_byte(__uint_as_float(ss[F_V * BS])), k);
            if (MULTI)
              put_mirror(G, D, mk ^ 1u, ss[F_C3 * BS], ss[F_EL * BS], (int)__uint_as_float(ss[F_POS * BS]),
                       speed_byte(__uint_as_float(ss[F_V * BS])), P.h_max);
            if (dig) {
              h = veh_hash(id, ss[F_EL * BS], __uint_as_float(ss[F_POS * BS]), __uint_as_float(ss[F_V * BS]),
                           cur - __ldg(&G.trip_rstart[id]));
              act = true;
            }
          }
        }
      } else if ((iv < nveh_k ? D.cbits[cb][iv >> 5] : 0u) >> (threadIdx.x & 31u) & 1u) {
        // one vectorised load of the record (a reference would re-load fields after every aliasing store)
        ClaimRec R;
        {
          const uint4* src = reinterpret_cast<const uint4*>(&D.crec[cb][iv]);
          uint4* dst = reinterpret_cast<uint4*>(&R);
#pragma unroll
          for (int qi = 0; qi < (int)(sizeof(ClaimRec) / 16); ++qi) dst[qi] = src[qi];
        }
        kind = (R.fb_byte >> 8) & 255u;
        // speculative loads of a transition's next-edge context, in parallel with the claim word
        const bool tr = kind == 1u;
        const uint32_t e_new = R.el_new & EDGE_MASK;
        const bool nlast = (R.el_new & LAST_BIT) != 0u;
        const EdgeRec En = tr ? load_edge(D.edges, e_new) : EdgeRec{};
        const uint32_t rn2 = (tr && !nlast) ? __ldg(&G.route[R.cur_new + 1u]) : 0u;
        won = (D.claim[R.cell] == R.id);
        lost = !won;
        if (won) {
          D.claim[R.cell] = NONE;
          if (tr && G.edge_entry) G.edge_entry[R.cur_new] = (int32_t)k1;  // t_start of the new edge
          mig = MULTI && tr && (En.meta & META_HALO) != 0u;
          if (mig) {  // continues on another partition: migrant; its old cell is cleared above
            send_migrant(G, D, part, mk, k, R.id, R.el_new, R.v_new, R.cur_new, En.ncells, R.cell);
            D.vid[nb][R.idx] = NONE;
            if (dig) { h = veh_hash(R.id, R.el_new, 0.0f, R.v_new, R.cur_new - __ldg(&G.trip_rstart[R.id])); act = true; }
          } else {
            D.vel[nb][R.idx] = R.el_new;
            D.vpos[nb][R.idx] = R.pos_new;
            D.vv[nb][R.idx] = R.v_new;
            D.vcur[nb][R.idx] = R.cur_new;
            D.vcell[nb][R.idx] = R.cell;
            put_map(P, G, ctl, Mn, R.cell, speed_byte(R.v_new), k);
            if (MULTI && !tr) put_mirror(G, D, mk ^ 1u, R.x[0], R.el_new, (int)R.pos_new, speed_byte(R.v_new), P.h_max);
            if (tr) {  // new edge: its cached context (make_ctx with the loads issued above)
              Ctx Y;
              Y.c0 = ctx_c0(En);
              Y.v0 = En.v0;
              const uint32_t K = (En.meta >> META_KOUT_SHIFT) & META_KOUT_MASK;
              if (nlast) {
                Y.c2 = 0; Y.c3 = MULTI ? ctx_mirror(En) : 0u; Y.c4 = NONE; Y.rn = 0;
              } else {
                const EdgeRec N2 = load_edge(D.edges, rn2 & ROUTE_EDGE_MASK);
                const uint32_t nl2 = N2.meta & META_LANES_MASK;
                Y.rn = rn2;
                Y.c2 = N2.ncells | (nl2 << 24) | ((N2.meta & META_HALO) ? (1u << 30) : 0u);
                Y.c3 = lane_range(En.meta & META_LANES_MASK, K, (N2.meta >> META_RANK_SHIFT) & META_RANK_MASK) |
                       (MULTI ? ctx_mirror(En) : 0u);
                const uint32_t nl_new = (R.el_new >> LANE_SHIFT) & LANE_MASK;
                Y.c4 = N2.base + min(nl_new, nl2 - 1u) * stride_of(Y.c2, P.h_max);
              }
              write_ctx(D, R.idx, Y);
            } else {  // lane change: only the entry-lane cell moves
              D.xc4[D.xb][R.idx] = R.x[4];
            }
            if (dig) { h = veh_hash(R.id, R.el_new, R.pos_new, R.v_new, R.cur_new - __ldg(&G.trip_rstart[R.id])); act = true; }
          }
        } else {
          put_map(P, G, ctl, Mn, R.fb_cell, (uint8_t)(R.fb_byte & 255u), k);
          if (MULTI) put_mirror(G, D, mk ^ 1u, R.x[0], R.x[1], (int)R.x[2], (uint8_t)(R.fb_byte & 255u), P.h_max);
          if (dig) {
            h = veh_hash(R.id, D.vel[nb][R.idx], D.vpos[nb][R.idx], D.vv[nb][R.idx],
                         D.vcur[nb][R.idx] - __ldg(&G.trip_rstart[R.id]));
            act = true;
          }
        }
      }
      warp_count_s(s_ctr, C_TRANS, won && kind == 1u);
      warp_count_s(s_ctr, C_LC, won && kind == 2u);
      warp_count_s(s_ctr, C_LOST, lost);
      {
        const unsigned b = __ballot_sync(0xffffffffu, mig);
        if ((threadIdx.x & 31u) == 0u && b) atomicAdd(&ctl->n_dead[nb], (unsigned)__popc(b));
      }
      if (dig) warp_digest(G.grid, (unsigned)(k & 1u), h, act);
    }
  }
#if LPSIM_CLEAR_LATE
  // clear of M_k after the claim rounds: the claim-word loads (and the admit CTAs'
  // departure chains) do not queue behind these stores at the start of the phase
  jr = 0;
  for (unsigned q = lb; lb < nbv && q < n_cc; q += nbv, ++jr) {
    const unsigned iv = q * BS + threadIdx.x;
    const uint32_t pc = iv >= nveh_k ? NONE : jr < nslot ? s_st[jr * (NF * BS) + F_PCELL * BS + threadIdx.x] : D.vpcell[nb][iv];
    if (pc != NONE) Mk[pc] = 255;
  }
#endif
  if ((FULL && (P.flags & 8u)) && threadIdx.x == 0 && G.grid->t_block) tb_add(G, 14, 3);

#ifdef LPSIM_EXP
  if ((P.flags & 0x40000u) && (lb < nbv)) {  // timing experiments: delay this CTA by 2 us (critical-path probe)
    const unsigned long long t0 = globaltimer();
    while (globaltimer() - t0 < 2000ull) {}
  }
#endif
  for (unsigned r = 0;; ++r) {  // admit positions by warp chunks, as in phase A
    const unsigned ac = admit_chunk(lb, nbp, nbv, r);
    if (ac == NONE || ac * 32u >= nfl) break;  // warp-uniform
#ifdef LPSIM_EXP
    if (P.flags & 0x100u) break;  // timing experiment builds only: no departures (wrong results)
#endif
    {
      // departures: the slot's candidate departs if it holds the claim (then the slot's next lowest
      // released trip comes from its bitmap); the slot carries over to step k+1 with its candidate,
      // unless it is in the release list of step k+1 (marked in phase A): then the candidate goes to
      // the slot's word, where that list's admit merges it with the new releases
      const unsigned f = ac * 32u + (threadIdx.x & 31u);
      uint64_t h = 0;
      bool act = false, dep = false, lost = false, local = false, relist = false;
      uint32_t id = 0, el = 0, rs = 0, cell = 0, s = NONE, succ = NONE;
      uint4 si = make_uint4(0u, 0u, 0u, 0u);
      uint4 res = make_uint4(NONE, NONE, NONE, 0u);  // {successor, reserved list entry, reserved SoA entry, 0}
      uint2 cw = make_uint2(NONE, NONE);
      Ctx X{};
      const bool tmd = (FULL && (P.flags & 8u)) && r == 0u && threadIdx.x < 32u && G.grid->t_block;
      if (f < nfl) {
        const bool sm = s_adm && r == 0u && (threadIdx.x >> 5) < ADM_WARPS;  // stashed by phase A
        const unsigned sa = (threadIdx.x >> 5) * 64u + (threadIdx.x & 31u);
        const uint4 cd = sm ? s_adm[sa] : D.slot_cand[f];  // {rank, id, claimed cell | NONE, slot}
        si = sm ? s_adm[sa + 32u] : D.slot_ci[f];
        res = sm ? s_res[threadIdx.x] : D.slot_cs[f];  // successor and reservations (phase A)
        succ = res.x;
        s = cd.w;
        if (tmd && threadIdx.x == 0u) {  // LPSIM_FLAG_TIMING: admit position loaded
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : "r"(cd.w ^ si.y));
          G.grid->t_block[TB_N * blockIdx.x + 20] += t - G.grid->t_block[TB_N * blockIdx.x + 3];
        }
        cw = make_uint2(cd.x, cd.y);
        const uint32_t rk = s != NONE ? D.slot_relk[s] : k1;
        if (cd.z != NONE) {
          cell = cd.z;
          id = cd.y;
          // everything a departure needs, loaded with the claim word
          const uint32_t cwd = D.claim[cell];
          rs = __ldg(&G.trip_rstart[id]);
          el = __ldg(&D.tel[id]);
          X.c0 = __ldg(&D.tx[0][id]);
          X.v0 = __uint_as_float(__ldg(&D.tx[1][id]));
          X.c2 = __ldg(&D.tx[2][id]);
          X.c3 = __ldg(&D.tx[3][id]);
          X.c4 = __ldg(&D.tx[4][id]);
          X.rn = __ldg(&D.tx[5][id]);
          if (cwd == id) {
            D.claim[cell] = NONE;
            dep = true;
            if (G.edge_entry) G.edge_entry[rs] = (int32_t)k1;  // t_start of the first edge
            const EdgeRec E1 = (MULTI && G.n_parts > 1u) ? load_edge(D.edges, el & EDGE_MASK) : EdgeRec{};
            if (MULTI && G.n_parts > 1u && (E1.meta & META_HALO) != 0u) {
              send_migrant(G, D, part, mk, k, id, el, 0.0f, rs, E1.ncells, cell);
              if (dig) { h = veh_hash(id, el, 0.0f, 0.0f, 0u); act = true; }
            } else {
              local = true;
            }
          } else {
            lost = true;
          }
        }
        // an emptied slot leaves the lists (its word NONE); a departed one is relisted before its
        // next candidate is known (a NONE candidate drops out at the next step)
        relist = rk != k1 && cw.x != NONE;
      }
      if (tmd) {  // claim words resolved
        __syncwarp();
        if (threadIdx.x == 0u) tb_add(G, 21, 3);
      }
      if (dep) {  // the departed rank's bits out of the bitmap; the successor (phase A) is the candidate
        bm_clear(D.bm + si.y, si.z, cw.x, succ);
        atomicSub(D.slot_nrel + s, 1u);
        cw.x = succ;
        cw.y = succ != NONE ? IDUNK : NONE;
      }
      if (tmd) {  // successor searches done
        __syncwarp();
        if (threadIdx.x == 0u) tb_add(G, 22, 3);
      }
      if (f < nfl && s != NONE && !relist) D.slot_cw[s] = cw;
      if (f < nfl && res.y != NONE) {  // the reserved entry of the pending list of step k+1
        D.slot_list[nb][res.y] = relist ? s : NONE;
        if (relist) {
          D.slot_li[nb][res.y] = si;
          D.slot_lc[nb][res.y] = cw;
        }
      }
      const unsigned ntot_k = s_misc[M_NVEH];
      bool dead_res = false;  // a reserved SoA entry this position leaves unused
      if (f < nfl && res.z != NONE && !local) {
        const unsigned idx = ntot_k + res.z;
        if (idx < D.veh_cap) {
          D.vid[nb][idx] = NONE;
          D.vpcell[nb][idx] = NONE;
          dead_res = true;
        }
      }
      {
        const unsigned bd = __ballot_sync(0xffffffffu, dead_res);
        if ((threadIdx.x & 31u) == 0u && bd) atomicAdd(&ctl->n_dead[nb], (unsigned)__popc(bd));
      }
      if (local) {
        const unsigned idx = ntot_k + res.z;
        if (idx < D.veh_cap) {
          write_vehicle(D, nb, idx, id, el, 0.0f, 0.0f, rs, cell, NONE);
          write_ctx(D, idx, X);  // prepared at load time (k_trip_ctx)
          put_map(P, G, ctl, Mn, cell, 0, k);
          if (dig) { h = veh_hash(id, el, 0.0f, 0.0f, 0u); act = true; }
        } else {
          set_error(G.grid, ctl, ERR_CAPACITY, 4, k);
        }
      }
      if (tmd) {  // appends and relists written
        __syncwarp();
        if (threadIdx.x == 0u) tb_add(G, 23, 3);
      }
      warp_count_s(s_ctr, C_DEP, dep);
      if ((FULL && (P.flags & 8u)) && G.grid->t_block) {  // diagnostics: departures / claimed / relisted per CTA
        const unsigned bd = __ballot_sync(0xffffffffu, dep), bc = __ballot_sync(0xffffffffu, f < nfl && cell != 0u);
        const unsigned br = __ballot_sync(0xffffffffu, relist);
        if ((threadIdx.x & 31u) == 0u) {
          unsigned long long* tb = G.grid->t_block + TB_N * blockIdx.x;
          atomicAdd(&tb[18], (unsigned long long)__popc(bd) | ((unsigned long long)__popc(bc) << 32));
          atomicAdd(&tb[19], (unsigned long long)__popc(br));
        }
      }
      warp_count_s(s_ctr, C_LOST, lost);
      if (dig) warp_digest(G.grid, (unsigned)(k & 1u), h, act);
    }
  }
  if ((FULL && (P.flags & 8u)) && threadIdx.x == 0 && G.grid->t_block) tb_add(G, 15, 3);

#ifdef LPSIM_EXP
  if ((P.flags & 0x80000u) && (lb >= nbv)) {  // timing experiments: delay this CTA by 2 us (critical-path probe)
    const unsigned long long t0 = globaltimer();
    while (globaltimer() - t0 < 2000ull) {}
  }
#endif
  if (gtid == 0) {
    ctl->n_dead[cb] = 0;  // the input buffer's dead count is no longer needed
    // SoA_{k+1} = the step's in-place entries + the entries reserved for its departures in phase A
    const unsigned n1 = s_misc[M_NVEH] + *((volatile unsigned*)&ctl->n_res[nb]);
    ctl->n_veh[nb] = n1;
    if (n1 > D.veh_cap) set_error(G.grid, ctl, ERR_CAPACITY, 4, k);
    ctl->n_res[cb] = 0;  // (reserved for SoA_k in step k-1, counted then)
  }
  if (gtid < NSH) D.sh_slot[cb][gtid * SH_STRIDE] = 0;  // the list of step k was read in phase A: empty for step k+2
  if ((FULL && (P.flags & 8u)) && G.grid->t_block) {  // slowest warp of the CTA
    __shared__ unsigned long long s_tend;
    if (threadIdx.x == 0) s_tend = 0ull;
    __syncthreads();
    if ((threadIdx.x & 31u) == 0u) atomicMax(&s_tend, globaltimer());
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long* tb = G.grid->t_block + TB_N * blockIdx.x;
      tb[1] += s_tend - tb[3];
      tb[9] = s_tend;
    }
  }
}

__device__ __forceinline__ void cross_gpu_sync(const Global& G, uint32_t epoch, uint32_t k) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // this part's migrant counts of snapshot k+1 (final after the local grid barrier) into the
    // receivers' copies; the release below orders them, the migrants and the halo bytes
    const uint32_t np = G.n_parts, par = (k + 1u) & 1u;
    const volatile uint32_t* row = G.mig_cnt + par * np * np + G.rank * np;
    for (uint32_t q = 0; q < G.world; ++q)
      if (q != G.rank) G.mig_cnt_peer[q][par * np * np + G.rank * np + q] = row[q];
    __threadfence_system();
    for (uint32_t q = 0; q < G.world; ++q) {
      if (q == G.rank) continue;
      uint32_t* f = G.xflag_peer[q] + G.rank;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
    }
    const unsigned long long t0 = globaltimer();
    for (uint32_t q = 0; q < G.world; ++q) {
      if (q == G.rank) continue;
      const uint32_t* f = G.xflag_local + q;
      for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if ((int32_t)(v - epoch) >= 0) break;
        if (globaltimer() - t0 > TIMEOUT_NS) {  // a peer is gone: fail the step instead of hanging the GPU
          atomicCAS(&G.grid->error, 0u, ERR_TIMEOUT);
          atomicMin(&G.grid->err_step, k);
          break;
        }
      }
    }
    // release the local CTAs with one flag (cheaper than a second grid barrier); the error of a
    // timeout is written before it, so every CTA sees the same verdict at the next phase A
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&G.grid->xgo), "r"(epoch) : "memory");
  } else if (threadIdx.x == 0) {
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&G.grid->xgo) : "memory");
      if ((int32_t)(v - epoch) >= 0) break;
    }
  }
  __syncthreads();
}

// LPSIM_FLAG_TIMING: per CTA, t_block[TB_N*b + 4|5] = barrier arrival after phase A|C (last
// step, absolute), t_block[TB_N*b + 6|7] += time spent in that barrier
template <bool FULL>
__device__ __forceinline__ void bar_mark(const Params& P, const Global& G, int w) {
  if ((FULL && (P.flags & 8u)) && threadIdx.x == 0 && G.grid->t_block) {
    unsigned long long* tb = G.grid->t_block + TB_N * blockIdx.x;
    const unsigned long long t = globaltimer();
    if (w < 6) tb[w] = t;
    else tb[w] += t - tb[w - 2];
  }
}

// ---------------------------------------------------------------------------
// the persistent step kernel
// ---------------------------------------------------------------------------
// FULL: the instrumented instantiation (LPSIM_FLAG_DIGESTS / LPSIM_FLAG_TIMING honoured); the lean one
// compiles the digest and timing code out (26% fewer instructions: less i-cache pressure, no spills)
template <bool FULL, bool MULTI>
__device__ __forceinline__ void run_dev(const Global& G, const Params& P, const PartParam& PP, unsigned long long k0,
                                                          unsigned nsteps) {
  const unsigned nl = G.n_local;  // partitions of this process (all of them, or one per GPU)
  // CTAs split among the local partitions (32-bit: grid <= 2^16 CTAs, nl <= 2^8); one partition
  // (the production case, one per GPU) needs no division
  unsigned lp = 0, b0 = 0, b1 = gridDim.x;
  if (nl > 1u) {
    lp = (blockIdx.x * nl) / gridDim.x;
    b0 = (lp * gridDim.x + nl - 1) / nl;
    b1 = ((lp + 1) * gridDim.x + nl - 1) / nl;
  }
  const unsigned part = G.part0 + lp;
  const unsigned lb = blockIdx.x - b0, nbp = b1 - b0;
  // CTAs nbv..nbp-1 of the partition are dedicated admit CTAs (admit_chunk): one per LPSIM_NAD CTAs
  // when the partition has 2 x LPSIM_NAD CTAs or more, one below that down to LPSIM_NAD_MIN CTAs (round
  // 1 measured one admit CTA in a partition of 55 CTAs slower, with the route-visit partition whose
  // largest part carried 1.5x the mean load), else admits run on the vehicle CTAs
#ifndef LPSIM_NAD
#define LPSIM_NAD 64
#endif
// partitions of LPSIM_NAD_MIN .. 2 x LPSIM_NAD - 1 CTAs (several partitions in one process) get one
// dedicated admit CTA: with partitions balanced for the load (multi.pilot_partition), K = 4 / 8 in
// one process 22.15 -> 21.35 / 24.36 -> 23.36 us per steady step (tools/r4_parts.sh)
#ifndef LPSIM_NAD_MIN
#define LPSIM_NAD_MIN 32
#endif

  const unsigned nbv = (LPSIM_NAD > 0 && nbp >= 2u * LPSIM_NAD) ? nbp - nbp / LPSIM_NAD
                       : (LPSIM_NAD_MIN > 0 && nbp >= LPSIM_NAD_MIN) ? nbp - 1u : nbp;
  // the partition's descriptor lives in shared memory: loaded once per launch,
  // never evicted by the L1 invalidations of the grid barriers
  __shared__ PartDev sD;
  __shared__ unsigned long long s_ctr[C_N];
  // dynamic shared memory (step_dyn_smem() bytes): resident vehicle state (see phase_a), resident
  // claims, lane-change candidates of the move phase (lc_batch)
  extern __shared__ __align__(16) uint32_t s_dyn[];
  uint32_t* const s_st = s_dyn;
  uint32_t* const s_cl = s_st + NSLOT * NF * BS;
  uint4* const s_lcq = reinterpret_cast<uint4*>(s_cl + NSLOT * NG * BS);
  // migrants received, prefix by sender (mig_prefix): used before phase A's vehicle chunks only, so it
  // shares the lane-change queue's memory (empty until the chunks)
  unsigned* const s_mp = reinterpret_cast<unsigned*>(s_lcq);
  static_assert(LCQ_CAP * 16 >= (BS + 1) * 4, "s_mp fits the lane-change queue");
  __shared__ unsigned s_pref[NSH + 1];         // admit list prefix (phase A -> phase C)
  __shared__ unsigned s_lcq_n;
  __shared__ unsigned s_misc[M_N];
  // a dedicated admit CTA (no vehicle chunks) keeps the first admit chunk of each warp {candidate,
  // slot_info} and their successors and reservations (A -> C) in its unused resident-state slots; with
  // admits on the vehicle CTAs (small partitions) they go through HBM.  (As static arrays they cost the
  // vehicle CTAs 12 KB of L1 each.)
  static_assert(ADM_WARPS * 96 * 16 <= NSLOT * NF * BS * 4, "admit stash fits the resident slots");
  uint4* const s_adm = (nbv < nbp && lb >= nbv) ? reinterpret_cast<uint4*>(s_st) : nullptr;
  uint4* const s_res = s_adm ? s_adm + ADM_WARPS * 64 : nullptr;
  {
    static_assert(sizeof(PartDev) % 4 == 0, "descriptor copied as words");
    constexpr unsigned NW = sizeof(PartDev) / 4;
    const uint32_t* src = PP.valid ? reinterpret_cast<const uint32_t*>(&PP.d)
                                   : reinterpret_cast<const uint32_t*>(G.parts + part);
    for (unsigned w = threadIdx.x; w < NW; w += BS) reinterpret_cast<uint32_t*>(&sD)[w] = src[w];
  }
  if (threadIdx.x < C_N) s_ctr[threadIdx.x] = 0ull;
  if (threadIdx.x == 0) s_lcq_n = 0u;
  __syncthreads();
  const PartDev& D = sD;
  const bool timing = (FULL && (P.flags & 8u)) != 0u && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long t0 = timing ? globaltimer() : 0ull;
  unsigned seen = 0;     // entries of the current snapshot held in shared memory
  unsigned wb_buf = 0;   // SoA buffer of the current snapshot
  unsigned mk = PP.mk;
  // (a one-step launch keeping the state in HBM instead measured slower: claim records then go
  // through HBM between phases A and C)
  const unsigned nslot = NSLOT;
  for (unsigned it = 0; it < nsteps; ++it, mk = mk ^ 1u) {
    const unsigned long long k = k0 + it;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      // digest of snapshot k (built during step k-1) -> log; reset its accumulator
      if (FULL && (P.flags & 1u) && it > 0 && it - 1 < G.digest_cap) G.digest_log[it - 1] = G.grid->digest[(k - 1) & 1];
      G.grid->digest[(k - 1) & 1] = 0ull;
    }
    // errors are stamped with their step; every error of a step < k was set before the last
    // barrier, so all CTAs read the same verdict here.  The load overlaps phase A; the CTAs leave
    // together before the barrier that ends it.
    const uint32_t err_prev = *((volatile uint32_t*)&G.grid->err_step);
    phase_a<FULL, MULTI>(P, G, D, k, mk, lb, nbp, nbv, part, s_mp, s_res, s_ctr, s_st, s_cl, seen, s_pref, s_misc, nslot, s_lcq, &s_lcq_n, s_adm);
    if (err_prev < (uint32_t)k) break;
    wb_buf = (unsigned)((k + 1) & 1);
    bar_mark<FULL>(P, G, 4);
    if (!grid_sync(G.grid)) return;
    bar_mark<FULL>(P, G, 6);
    if (timing) { const unsigned long long t = globaltimer(); G.grid->t_phase[0] += t - t0; t0 = t; }
    phase_c<FULL, MULTI>(P, G, D, k, mk, lb, nbp, nbv, part, s_res, s_ctr, s_st, s_cl, s_pref, s_misc, nslot, s_adm);
    bar_mark<FULL>(P, G, 5);
    // the barrier that ends the launch's last step is the kernel's completion (the next launch, the
    // sort and the host read after it), unless this step's digest is read below or a peer GPU must
    // see the step's stores before its own next step
    const bool last = it + 1u == nsteps && !(FULL && (P.flags & 1u)) && !(MULTI && G.world > 1);
    if (!last && !grid_sync(G.grid)) return;
    bar_mark<FULL>(P, G, 7);
    if (timing) { const unsigned long long t = globaltimer(); G.grid->t_phase[1] += t - t0; t0 = t; }
    if (MULTI && G.world > 1) {  // migrants, their counts and the mirrored halo bytes delivered
      cross_gpu_sync(G, (uint32_t)k + 1u, (uint32_t)k);
      if (timing) { const unsigned long long t = globaltimer(); G.grid->t_phase[2] += t - t0; t0 = t; }
    }
  }
  // resident state back to the HBM SoA of the current snapshot (the sort and the host read it)
  for (unsigned j = 0; lb < nbv && j < nslot; ++j) {
    const unsigned i = (lb + j * nbv) * BS + threadIdx.x;
    if (i >= seen) break;
    const uint32_t* ss = s_st + j * (NF * BS) + threadIdx.x;
    // (vpcell, the cell held one snapshot earlier, is not written back: the next step rewrites it
    // before anything reads it)
    D.vid[wb_buf][i] = ss[F_ID * BS];
    D.vel[wb_buf][i] = ss[F_EL * BS];
    D.vpos[wb_buf][i] = __uint_as_float(ss[F_POS * BS]);
    D.vv[wb_buf][i] = __uint_as_float(ss[F_V * BS]);
    D.vcur[wb_buf][i] = ss[F_CUR * BS];
    D.vcell[wb_buf][i] = ss[F_CELL * BS];
    if (ss[F_DIRTY * BS]) {
      VState z;
      vs_load(ss, z);
      write_ctx(D, i, z.X);
    }
  }
  __syncthreads();
  if (threadIdx.x < C_N) G.ctr_block[(unsigned long long)C_N * blockIdx.x + threadIdx.x] += s_ctr[threadIdx.x];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long k = k0 + nsteps;
    if (FULL && (P.flags & 1u) && nsteps > 0 && nsteps - 1 < G.digest_cap) G.digest_log[nsteps - 1] = G.grid->digest[(k - 1) & 1];
    G.grid->step = k;
  }
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

// per-trip view of the on-road vehicles (trip_state / results)
// (with several partitions also the migrants in the receive queues of snapshot k, at pos 0 of their
// edge: the owner moves them in phase A of the next step, §8(e))
__global__ void k_scatter_trips(PartDev* parts, unsigned np, unsigned buf, const uint32_t* mig_cnt,
                                const uint32_t* trip_rstart, int32_t* status, int32_t* edge, int32_t* lane, float* pos,
                                float* v, int64_t* cursor) {
  const unsigned t0 = blockIdx.x * blockDim.x + threadIdx.x, ts = gridDim.x * blockDim.x;
  for (unsigned p = 0; p < np; ++p) {
    const PartDev D = parts[p];
    if (D.ctl == nullptr) continue;  // a partition of another process
    const unsigned n = D.ctl->n_veh[buf];
    for (unsigned i = t0; i < n; i += ts) {
      const uint32_t id = D.vid[buf][i], el = D.vel[buf][i];
      if (id == NONE) continue;
      status[id] = 1;
      edge[id] = (int32_t)(el & EDGE_MASK);
      lane[id] = (int32_t)((el >> LANE_SHIFT) & LANE_MASK);
      pos[id] = D.vpos[buf][i];
      v[id] = D.vv[buf][i];
      cursor[id] = (int64_t)(D.vcur[buf][i] - trip_rstart[id]);
    }
    if (np < 2u || mig_cnt == nullptr) continue;
    for (unsigned u = 0; u < np; ++u) {
      if (u == p) continue;
      const unsigned r0 = D.rq_off[u], cnt = min(mig_cnt[buf * np * np + u * np + p], D.rq_off[u + 1] - r0);
      for (unsigned i = t0; i < cnt; i += ts) {
        const MigSlot m = D.inq[buf][r0 + i];
        status[m.id] = 1;
        edge[m.id] = (int32_t)(m.el & EDGE_MASK);
        lane[m.id] = (int32_t)((m.el >> LANE_SHIFT) & LANE_MASK);
        pos[m.id] = 0.0f;
        v[m.id] = m.v;
        cursor[m.id] = (int64_t)(m.cur - trip_rstart[m.id]);
      }
    }
  }
}

// distance (double, route order) per trip
// route table on the device: the caller's edge ids, the last entry of each trip's route marked
// (edge | last << 31); routes are contiguous in trip order (route_ptr validated on the host)
__global__ void k_mark_last(int64_t n, int64_t R, const uint32_t* trip_rstart, uint32_t* route) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t end = i + 1 < n ? (int64_t)trip_rstart[i + 1] : R;
    route[end - 1] |= LAST_BIT;
  }
}

// per-trip views before k_scatter_trips fills in the on-road trips: waiting (first route edge, lane 0,
// 0, 0, cursor 0) or finished (arrival step set)
__global__ void k_trip_defaults(int64_t n, const int32_t* arrival, const uint32_t* route, const uint32_t* trip_rstart,
                                int32_t* status, int32_t* edge, int32_t* lane, float* pos, float* v, int64_t* cur) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    status[i] = arrival[i] >= 0 ? 2 : 0;
    edge[i] = (int32_t)(route[trip_rstart[i]] & ROUTE_EDGE_MASK);
    lane[i] = 0;
    pos[i] = 0.0f;
    v[i] = 0.0f;
    cur[i] = 0;
  }
}

// Distance per trip (§1): the route edges traversed, in double.  One warp per trip reads the route
// 32 entries at a time (coalesced) and gathers their lengths.  The sum is exact in any order: every
// length is a float >= 1 m (Q29), so each term and partial sum is a multiple of 2^-23 below 2^30,
// which a double holds exactly; the position on the current edge is added last, as in route order.
// R = entries of the route array (reads past a trip's route stay inside it).
__global__ void k_distances(int64_t n, const uint32_t* route, int64_t R, const uint32_t* trip_rstart,
                            const float* length, const int32_t* status, const float* pos, const int64_t* cursor,
                            const int32_t* arrival, double* dist) {
  const unsigned lane = threadIdx.x & 31u;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n; t += nw) {
    const bool arr = arrival[t] >= 0;
    const bool on = !arr && status[t] == 1;
    double d = 0.0;
    if (arr || on) {  // warp-uniform
      const int64_t rs = trip_rstart[t];
      const int64_t lim = arr ? R - rs : min(cursor[t], R - rs);  // entries counted: j < lim (and up to LAST)
      for (int64_t b0 = 0; b0 < lim; b0 += 32) {
        const int64_t j = b0 + lane;
        const uint32_t r = j < lim ? route[rs + j] : 0u;
        const unsigned lm = __ballot_sync(0xffffffffu, (r & LAST_BIT) != 0u);
        const unsigned first = lm ? (unsigned)__ffs(lm) - 1u : 32u;
        if (j < lim && lane <= first) d += (double)length[r & ROUTE_EDGE_MASK];
        if (lm) break;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      if (on) d += (double)pos[t];
    }
    if (lane == 0u) dist[t] = d;
  }
}

// gather of the lane map (local layout -> global layout), one partition
__global__ void k_gather_map(const uint8_t* local, const uint64_t* gbase, const EdgeRec* edges, int E, uint8_t* out,
                             const uint8_t* lanes) {
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    const EdgeRec R = edges[e];
    if (R.meta & (META_HALO | META_REMOTE)) continue;
    const uint64_t n = (uint64_t)R.ncells * lanes[e];
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) out[gbase[e] + i] = local[R.base + i];
  }
}

// occupied (non-free) cells of a lane map over the partition's owned edges (entry halos hold
// copies of another partition's cells and are skipped): the a7 invariant check of the tests
__global__ void k_count_occupied(const uint8_t* map, const EdgeRec* edges, int E, const uint8_t* lanes,
                                 unsigned long long* out) {
  unsigned long long n_occ = 0;
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    const EdgeRec R = edges[e];
    if (R.meta & (META_HALO | META_REMOTE)) continue;
    const uint64_t n = (uint64_t)R.ncells * lanes[e];
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) n_occ += map[R.base + i] != 255 ? 1u : 0u;
  }
  atomicAdd(out, n_occ);
}

// ---------------------------------------------------------------------------
// a9: periodic locality sort of the active SoA, one cooperative kernel, no host round trip
// ---------------------------------------------------------------------------
// Counting sort of the live entries into buckets of 2^SORT_SHIFT consecutive lane-map cells (about
// one lane of one edge; the cell index encodes (edge, lane, cell)), dead entries dropped.
// The order inside a bucket is whatever the scatter atomics produce: results do not depend on the
// SoA order (each vehicle is a pure function of the snapshot, conflicts go to the lowest id), which
// the parity tests check with sort periods 1, 3, 16, 128 and none.  mode 1 (LPSIM_FLAG_NO_SORT):
// buckets of 2^SORT_SHIFT consecutive SoA indices, i.e. compaction only.
// block-wide sum of x (all threads get it); s: >= 32 words of shared scratch
__device__ __forceinline__ unsigned block_sum(unsigned x, unsigned* s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  if ((threadIdx.x & 31u) == 0u) s[threadIdx.x >> 5] = x;
  __syncthreads();
  unsigned t = 0;
  for (unsigned w = 0; w < (blockDim.x >> 5); ++w) t += s[w];
  return t;
}
// block-wide exclusive scan of x; s: >= 32 words of shared scratch
__device__ __forceinline__ unsigned block_excl_scan(unsigned x, unsigned* s) {
  const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  unsigned v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (unsigned)o) v += y;
  }
  __syncthreads();
  if (lane == 31u) s[w] = v;
  __syncthreads();
  unsigned before = 0;
  for (unsigned q = 0; q < w; ++q) before += s[q];
  return before + v - x;
}

__global__ void __launch_bounds__(256) k_bucket_sort(const PartDev* parts, const SortBufs* sbs, unsigned p0,
                                                     unsigned nl, unsigned buf, unsigned mode) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned s_scr[32];
  // CTAs split among the partitions (one launch for all of a process's partitions); every grid.sync
  // below is reached by all CTAs, each working on its own partition
  unsigned lp = 0, b0 = 0, b1 = gridDim.x;
  if (nl > 1u) {
    lp = (blockIdx.x * nl) / gridDim.x;
    b0 = (lp * gridDim.x + nl - 1) / nl;
    b1 = ((lp + 1) * gridDim.x + nl - 1) / nl;
  }
  const unsigned lb = blockIdx.x - b0, nbp = b1 - b0;
  __shared__ PartDev sD;
  for (unsigned w = threadIdx.x; w < sizeof(PartDev) / 4; w += blockDim.x)
    reinterpret_cast<uint32_t*>(&sD)[w] = reinterpret_cast<const uint32_t*>(parts + p0 + lp)[w];
  __syncthreads();
  const PartDev& D = sD;
  const SortBufs B = sbs[p0 + lp];
  uint32_t* const bcount = B.bcount;
  uint32_t* const bcur = B.bcur;
  uint32_t* const bsum = B.bsum;
  uint32_t* const perm = B.perm;
  const uint32_t nb = B.nb;
  const unsigned n = D.ctl->n_veh[buf];
  const unsigned gt = lb * blockDim.x + threadIdx.x, gs = nbp * blockDim.x;
  // 1. bucket counts of the live entries (bcount is all zero on entry)
  for (unsigned i = gt; i < n; i += gs) {
    if (D.vid[buf][i] == NONE) continue;  // dead entry: dropped (its cell was cleared in phase C)
    atomicAdd(&bcount[mode == 0u ? (D.vcell[buf][i] >> SORT_SHIFT) : (i >> SORT_SHIFT)], 1u);
  }
  grid.sync();
  // 2. exclusive scan of the counts: one segment per CTA, then the segment offsets
  const unsigned seg = (nb + nbp - 1) / nbp, per = (seg + blockDim.x - 1) / blockDim.x;
  const unsigned s0 = min(nb, lb * seg), s1 = min(nb, s0 + seg);
  const unsigned t0 = min(s1, s0 + threadIdx.x * per), t1 = min(s1, t0 + per);
  unsigned mine = 0;
  for (unsigned b = t0; b < t1; ++b) mine += bcount[b];
  const unsigned segsum = block_sum(mine, s_scr);
  if (threadIdx.x == 0) bsum[lb] = segsum;
  grid.sync();
  unsigned before = 0, total = 0;
  for (unsigned q = threadIdx.x; q < nbp; q += blockDim.x) {
    const unsigned x = bsum[q];
    total += x;
    if (q < lb) before += x;
  }
  before = block_sum(before, s_scr);
  total = block_sum(total, s_scr);  // live entries
  unsigned run = before + block_excl_scan(mine, s_scr);
  for (unsigned b = t0; b < t1; ++b) {
    const unsigned cnt = bcount[b];
    bcur[b] = run;
    run += cnt;
    bcount[b] = 0u;  // zero for the next sort
  }
  grid.sync();
  // 3. scatter the live indices
  for (unsigned i = gt; i < n; i += gs) {
    if (D.vid[buf][i] == NONE) continue;
    const uint32_t b = mode == 0u ? (D.vcell[buf][i] >> SORT_SHIFT) : (i >> SORT_SHIFT);
    perm[atomicAdd(&bcur[b], 1u)] = i;
  }
  grid.sync();
  // 4. gather into buffer buf^1 (the context into xb^1); the host swaps the buffer roles
  const unsigned ob = buf ^ 1u, xb = D.xb, xo = xb ^ 1u;
  for (unsigned j = gt; j < total; j += gs) {
    const uint32_t q = perm[j];
    D.vid[ob][j] = D.vid[buf][q];
    D.vel[ob][j] = D.vel[buf][q];
    D.vpos[ob][j] = D.vpos[buf][q];
    D.vv[ob][j] = D.vv[buf][q];
    D.vcur[ob][j] = D.vcur[buf][q];
    D.vpcell[ob][j] = D.vpcell[buf][q];
    D.vcell[ob][j] = D.vcell[buf][q];
    D.xc0[xo][j] = D.xc0[xb][q];
    D.xv0[xo][j] = D.xv0[xb][q];
    D.xc2[xo][j] = D.xc2[xb][q];
    D.xc3[xo][j] = D.xc3[xb][q];
    D.xc4[xo][j] = D.xc4[xb][q];
    D.xrn[xo][j] = D.xrn[xb][q];
  }
  if (gt == 0) {  // counters of the compacted buffer (it becomes buffer `buf` after the swap)
    D.ctl->n_veh[buf] = total;
    D.ctl->n_dead[buf] = 0;
  }
}

// ---------------------------------------------------------------------------
// restore (§8(f) checkpoint/restore): the device state of snapshot k rebuilt from per-trip state.
// At a step boundary the claim words are all free and every map but M_k is clean, so a fresh context plus M_k, the SoA, the departure bitmaps / counts / candidates and the
// carried admit list is the whole state.
// ---------------------------------------------------------------------------
// on-road trips -> SoA_k of their edge's owner, their byte in M_k (and in an upstream part's entry
// halo); err = first offending trip (atomicMin)
__global__ void k_restore_trips(PartDev* parts, unsigned np, uint32_t buf, uint32_t mk, int h_max, int64_t n,
                                const uint32_t* route, const uint32_t* trip_rstart, const int32_t* edge_owner,
                                const int32_t* edge_up, const int32_t* status, const int32_t* edge,
                                const int32_t* lane, const float* pos, const float* v, const int64_t* cursor,
                                uint32_t* err) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    if (status[t] != 1) continue;
    const uint32_t id = (uint32_t)t, e = (uint32_t)edge[t], l = (uint32_t)lane[t];
    const uint32_t cur = trip_rstart[t] + (uint32_t)cursor[t];
    const uint32_t r = route[cur];
    const int q = edge_owner[e], u = edge_up[e];
    const float p = pos[t], sp = v[t];
    if ((r & ROUTE_EDGE_MASK) != e || !(p >= 0.0f) || !(sp >= 0.0f && sp <= 254.0f)) { atomicMin(err, id); continue; }
    const int c = (int)p;
    const uint8_t byte = (uint8_t)(int)fminf(sp, 254.0f);
    if (q < (int)np && parts[q].ctl != nullptr) {
      const PartDev& D = parts[q];
      const EdgeRec E = D.edges[e];
      if (l >= (E.meta & META_LANES_MASK) || c >= (int)E.ncells) { atomicMin(err, id); continue; }
      const uint32_t cell = E.base + l * E.ncells + (uint32_t)c;
      const unsigned i = atomicAdd(&D.ctl->n_veh[buf], 1u);
      if (i >= D.veh_cap) { atomicMin(err, id); continue; }
      D.vid[buf][i] = id;
      D.vel[buf][i] = e | (l << LANE_SHIFT) | (r & LAST_BIT);
      D.vpos[buf][i] = p;
      D.vv[buf][i] = sp;
      D.vcur[buf][i] = cur;
      D.vcell[buf][i] = cell;
      D.vpcell[buf][i] = NONE;
      const Ctx X = make_ctx(D.edges, route, h_max, e, l, cur, (r & LAST_BIT) != 0u);
      D.xc0[D.xb][i] = X.c0;
      D.xv0[D.xb][i] = X.v0;
      D.xc2[D.xb][i] = X.c2;
      D.xc3[D.xb][i] = X.c3;
      D.xc4[D.xb][i] = X.c4;
      D.xrn[D.xb][i] = X.rn;
      D.map[mk][cell] = byte;
    }
    if (u != q && u < (int)np && parts[u].ctl != nullptr && c < h_max) {  // entry halo on the upstream part
      const PartDev& U = parts[u];
      const EdgeRec E = U.edges[e];
      U.map[mk][E.base + l * (uint32_t)h_max + (uint32_t)c] = byte;
    }
  }
}

// waiting trips released before step k: their bits and counts (the releases of step k itself are
// applied by phase A of step k)
__global__ void k_restore_released(PartDev* parts, unsigned p, uint32_t k, const int32_t* status) {
  const PartDev D = parts[p];
  if (k >= D.rel_steps + 1u) return;
  const uint32_t j1 = D.rel_ptr[min(k, D.rel_steps)];
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < j1; j += gridDim.x * blockDim.x) {
    const uint4 rl = D.rel4[j];  // {slot, rank, bitmap offset, width}
    const uint32_t id = D.slot_trip[D.slot_info[rl.x].w + rl.y];
    if (status[id] != 0) continue;
    bm_set(D.bm + rl.z, rl.w, rl.y);
    atomicAdd(&D.slot_nrel[rl.x], 1u);
  }
}

// per slot: its candidate (lowest released rank: exact summaries, top-down), then the slot's word
// (slots in the release list of step k, marked slot_relk == k) or the carried list of step k
__global__ void k_restore_slots(PartDev* parts, unsigned p, uint32_t k, uint32_t* err) {
  const PartDev D = parts[p];
  const unsigned cb = k & 1u;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < D.n_slot_total; s += gridDim.x * blockDim.x) {
    if (D.slot_nrel[s] == 0u) continue;
    const uint4 si = D.slot_info[s];
    const int d = bm_depth(si.z);
    uint32_t off = 0, x = 0;
    for (int lvl = 0; lvl < d; ++lvl) {
      x = (x << 5) | (uint32_t)(__ffs(D.bm[si.y + off + x]) - 1);
      off += bm_words(si.z, d, lvl);
    }
    const uint2 cw = make_uint2(x, D.slot_trip[si.w + x]);
    if (D.slot_relk[s] == k) {
      D.slot_cw[s] = cw;
    } else {
      const unsigned shard = s % NSH;
      const unsigned j = atomicAdd(&D.sh_slot[cb][shard * SH_STRIDE], 1u);
      if (j >= D.slot_shcap) { atomicMin(err, 0xFFFFFFFEu); continue; }
      D.slot_list[cb][shard * D.slot_shcap + j] = s;
      D.slot_li[cb][shard * D.slot_shcap + j] = si;
      D.slot_lc[cb][shard * D.slot_shcap + j] = cw;
    }
  }
}
__global__ void k_mark_release_list(PartDev* parts, unsigned p, uint32_t k) {
  const PartDev D = parts[p];
  if (k >= D.rel_steps) return;
  for (uint32_t j = D.rs_ptr[k] + blockIdx.x * blockDim.x + threadIdx.x; j < D.rs_ptr[k + 1]; j += gridDim.x * blockDim.x)
    D.slot_relk[D.rs_slot[j]] = k;
}

// departure state of every trip owned by partition p (first edge, lane id mod
// lanes, its edge context), computed once at load time
__global__ void k_trip_ctx(PartDev* parts, unsigned p, const uint32_t* route, const uint32_t* trip_rstart,
                           const uint32_t* trips, uint32_t n, int h_max) {
  const PartDev D = parts[p];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const uint32_t id = trips[t];
    const uint32_t rs = trip_rstart[id];
    const uint32_t r0 = route[rs];
    const uint32_t e1 = r0 & ROUTE_EDGE_MASK;
    const uint32_t lanes = D.edges[e1].meta & META_LANES_MASK;
    const uint32_t l0 = id % lanes;
    D.tel[id] = e1 | (l0 << LANE_SHIFT) | (r0 & LAST_BIT);
    const Ctx X = make_ctx(D.edges, route, h_max, e1, l0, rs, (r0 & LAST_BIT) != 0u);
    D.tx[0][id] = X.c0;
    D.tx[1][id] = __float_as_uint(X.v0);
    D.tx[2][id] = X.c2;
    D.tx[3][id] = X.c3;
    D.tx[4][id] = X.c4;
    D.tx[5][id] = X.rn;
  }
}

// a0: assemble the 16-byte edge records from the scanned bases
__global__ void k_build_edges(int E, const uint64_t* base, const uint32_t* ncells, const float* v0,
                              const uint32_t* meta, EdgeRec* out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    EdgeRec R;
    R.base = (uint32_t)base[e];
    R.ncells = ncells[e];
    R.v0 = v0[e];
    R.meta = meta[e];
    out[e] = R;
  }
}

// dynamic shared memory of k_run / k_run_full (the per-CTA arrays scale with BS)
size_t step_dyn_smem() {
  static_assert((NSLOT * (NF + NG) * BS * 4) % 16 == 0, "lane-change queue 16-byte aligned");
  return (size_t)NSLOT * (NF + NG) * BS * 4 + (size_t)LCQ_CAP * 16;
}

// k_run: lean, one partition (the exchange code compiled out); k_run_multi: lean, several partitions
// (in one process or one per GPU); k_run_full: instrumented, any partition count
__global__ void __launch_bounds__(BS, LPSIM_MINB) k_run(Global G, Params P, PartParam PP, unsigned long long k0,
                                                          unsigned nsteps) {
  run_dev<false, false>(G, P, PP, k0, nsteps);
}
__global__ void __launch_bounds__(BS, LPSIM_MINB) k_run_multi(Global G, Params P, PartParam PP,
                                                                unsigned long long k0, unsigned nsteps) {
  run_dev<false, true>(G, P, PP, k0, nsteps);
}
__global__ void __launch_bounds__(BS, LPSIM_MINB) k_run_full(Global G, Params P, PartParam PP, unsigned long long k0,
                                                               unsigned nsteps) {
  run_dev<true, true>(G, P, PP, k0, nsteps);
}

}  // namespace lpsim
