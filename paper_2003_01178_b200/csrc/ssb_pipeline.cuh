// ssb_pipeline.cuh -- the sm_100a fused join pipeline for SSB flights 2-4.
//
// Replaces the hot loop of run_joins (ssb_queries.cpp:233-263): per lineorder
// tile, probe every dimension join in plan order and fold the survivors into
// the dense group-by table, in ONE pass with no materialisation.
//
// Shape (one persistent CTA per SM):
//   * warp W (producer): one elected lane streams the plan's fact columns
//     through a STAGES-deep shared-memory ring with TMA bulk copies
//     (cp.async.bulk ... mbarrier::complete_tx, L2 evict_first), one 1-D copy
//     per column per tile.  `full[s]` completes when the bytes land; the
//     consumer warps release the slot through `empty[s]`.
//   * warps 0..W-1 (consumers): each owns TILE/W consecutive rows of a stage.
//       phase A (dense)  probe join 0 for every row (vector LDS of the keys,
//                        table usually shared-memory resident), then compact
//                        the survivors (warp ballot/scan) into a warp list;
//       phase B (sparse) one survivor per lane: fetch the remaining keys and
//                        the aggregate columns from the stage, issue every
//                        remaining probe before consuming any (the loads
//                        overlap), chain the join masks in plan order for
//                        QueryStats, and add into the group-by table.
//     No CTA barrier inside the loop; warps only meet at the mbarriers.
//
// Dimension probe tables (built per query by dim_filter_kernel, SSB keys are
// dense integer ranges so the build is a perfect hash over [kmin, kmin+n)):
//   kTabBitmap  1 bit per key: joins that only filter (no payload)
//   kTabU8/U16  one code per key: 0xFF(FF) = not a member, 0xFE(FE) = member
//               whose payload falls outside its group domain (ContractError
//               if such a row reaches the aggregate, ssb_queries.cpp:32-33),
//               else payload - lo, i.e. the group-part digit itself
//   kTabHash    the reference's linear-probing table (hash_table.hpp:41-51)
//               for key columns without a usable range
// Tables that fit the shared-memory budget are copied into every CTA.
#pragma once

#include "async.cuh"
#include "crystal.cuh"

namespace crys {
namespace pipe {

enum TabKind : int32_t { kTabBitmap = 0, kTabU8 = 1, kTabU16 = 2, kTabHash = 3 };
constexpr uint32_t kU8Absent = 0xFFu, kU8Bad = 0xFEu, kU16Absent = 0xFFFFu, kU16Bad = 0xFFFEu;
constexpr int kMaxJ = 4, kMaxC = 6;

struct ProbeTab {
  const void* g;    // device table: bitmap words / u8 codes / u16 codes / int2 slots
  uint32_t kmin;    // key domain [kmin, kmin + n) of the direct tables
  uint32_t n;
  int32_t kind;     // TabKind
  int32_t smem;     // byte offset of the CTA's shared copy; -1: probed through L2
  uint32_t bytes;   // table bytes (multiple of 16)
  int32_t gstride;  // mixed-radix stride of the group part fed by this join (0: none)
  int32_t meta;     // HtMeta index (kTabHash)
  // direct tables, uniform decode: entry = ((word[o >> sh5] >> ((o & emask) << lb)) & mask) ^ flip
  // absent <=> entry == mask, bad digit <=> entry == badc, else entry is the digit
  uint32_t lb, sh5, emask, mask, flip, badc;
};

struct PipeArgs {
  int64_t n;                   // lineorder rows of the shard
  const int32_t* col[kMaxC];   // fk_0 .. fk_{NJ-1}, revenue [, supplycost]
  ProbeTab tab[kMaxJ];
  const HtMeta* meta;
  int32_t cells;
  int32_t smem_agg;            // byte offset of the shared aggregate (-1: global atomics)
  unsigned long long* g_sum;   // [cells]
  unsigned long long* g_cnt;   // [cells]
  unsigned long long* surv;    // [4]
  int32_t* err;
  int32_t l2_ahead;            // > 0: bulk-prefetch tile it + l2_ahead into L2 when issuing tile it
  // split plans (ssb_scan.cuh): every row alive after the dense joins goes
  // to its CTA's region of the survivor list as {row, partial group index |
  // bad << 31}; ssb_gather_kernel runs the rest of the plan over the list
  uint2* list;                 // [gridDim.x][list_cap]
  int64_t list_cap;
  unsigned* list_count;        // [gridDim.x] entries per region
};

// Host: fill the uniform-decode fields of a direct table.
inline void set_decode(ProbeTab& t) {
  t.lb = t.kind == kTabBitmap ? 0u : (t.kind == kTabU8 ? 3u : 4u);
  t.sh5 = 5u - t.lb;
  t.emask = (32u >> t.lb) - 1u;
  t.mask = t.kind == kTabBitmap ? 1u : (t.kind == kTabU8 ? kU8Absent : kU16Absent);
  t.flip = t.kind == kTabBitmap ? 1u : 0u;  // bitmap: bit 1 = member -> entry 0 (digit 0)
  t.badc = t.kind == kTabBitmap ? 2u : t.mask - 1u;
}

// PTX helpers (mbarrier, 1-D TMA bulk copy): async.cuh

// 64-bit add into shared memory as 32-bit halves: sm_100a has no native
// 64-bit shared atomic add (atomicAdd(u64*) on shared compiles to an
// ATOMS.CAST.SPIN.64 compare-and-swap loop, which serialises under the
// contention of a few hot groups, e.g. q3.1's 150 live cells).  One native
// ATOMS.ADD on the low word; the high word only takes the carry out of it
// plus the sign extension of a negative value (q4: revenue - supplycost).
__device__ __forceinline__ void smem_add_i64(unsigned long long* cell, long long v) {
  unsigned* w = reinterpret_cast<unsigned*>(cell);  // little-endian: w[0] low, w[1] high
  const unsigned lo = (unsigned)v;
  const unsigned hi = (unsigned)((unsigned long long)v >> 32);
  const unsigned old = atomicAdd(w, lo);
  const unsigned carry = (old + lo) < old ? 1u : 0u;
  if (hi + carry) atomicAdd(w + 1, hi + carry);
}

// ------------------------------------------------------------- probes
// Split into fetch (one load) and decode so a caller issues the loads of
// several probes before consuming any.

// linear-probing table (hash_table.hpp:41-51).  Returns -2 for a miss, else
// the stored digit (payload - lo, or -1 for a payload outside the group
// domain).  Scalar arguments and a scalar result: a reference into the
// kernel's parameter block, or an out-pointer, would force local memory.
__device__ __noinline__ int32_t hash_probe_slots(const int2* slots, uint32_t mask, int shift,
                                                 int32_t key) {
  if (key == kEmptyKey) return -2;  // unstorable, aliases empty slots
  uint32_t s = ht_slot_of(key, shift);
  int2 e = __ldg(slots + s);
  while (e.x != key && e.x != kEmptyKey) {
    s = (s + 1) & mask;
    e = __ldg(slots + s);
  }
  return e.x == key ? e.y : -2;
}

__device__ __forceinline__ int32_t hash_probe(const ProbeTab& t, const HtMeta* meta, int32_t key) {
  const HtMeta* m = meta + t.meta;
  return hash_probe_slots(reinterpret_cast<const int2*>(t.g), m->mask, m->shift, key);
}

// Later joins, hoisted into registers once per CTA: the uniform decode of a
// direct table through a generic pointer (shared copy or global), or the
// linear-probing walk (hash != 0).
struct RegTab {
  const uint32_t* p;
  uint32_t kmin, n, sh5, emask, lb, mask, flip, badc, gstride, hash;
};
__device__ __forceinline__ RegTab reg_tab(const ProbeTab& t, const char* sbase) {
  RegTab r;
  r.p = t.smem >= 0 ? reinterpret_cast<const uint32_t*>(sbase + t.smem)
                    : reinterpret_cast<const uint32_t*>(t.g);
  r.kmin = t.kmin;
  r.n = t.n;
  r.sh5 = t.sh5;
  r.emask = t.emask;
  r.lb = t.lb;
  r.mask = t.mask;
  r.flip = t.flip;
  r.badc = t.badc;
  r.gstride = (uint32_t)t.gstride;
  r.hash = t.kind == kTabHash;
  return r;
}

// Phase-A specialisation of join 0: K0 = table kind, S0 = table in shared memory.
template <int K0, bool S0>
__device__ __forceinline__ uint32_t first_fetch(const ProbeTab& t, const char* sbase, uint32_t off) {
  const uint32_t o = off < t.n ? off : 0u;
  constexpr int sh5 = K0 == kTabBitmap ? 5 : (K0 == kTabU8 ? 2 : 1);
  const uint32_t* w = S0 ? reinterpret_cast<const uint32_t*>(sbase + t.smem)
                         : reinterpret_cast<const uint32_t*>(t.g);
  return S0 ? w[o >> sh5] : __ldg(w + (o >> sh5));
}
// member? digit in *code (0xFFFF: member whose digit is outside its domain)
template <int K0>
__device__ __forceinline__ bool first_decode(const ProbeTab& t, uint32_t off, uint32_t w, uint32_t* code) {
  if constexpr (K0 == kTabBitmap) {
    *code = 0;
    return off < t.n && ((w >> (off & 31u)) & 1u);
  } else if constexpr (K0 == kTabU8) {
    const uint32_t e = (w >> ((off & 3u) << 3)) & 0xFFu;
    *code = e == kU8Bad ? 0xFFFFu : e;
    return off < t.n && e != kU8Absent;
  } else {
    const uint32_t e = (w >> ((off & 1u) << 4)) & 0xFFFFu;
    *code = e;  // kU16Bad == 0xFFFE: mapped below
    if (e == kU16Bad) *code = 0xFFFFu;
    return off < t.n && e != kU16Absent;
  }
}

// ------------------------------------------------------------- the kernel
// NJ joins, NC staged columns (NC - NJ = 1: revenue; 2: revenue - supplycost),
// W consumer warps, TILE rows per stage, STAGES-deep ring; K0/S0 specialise
// the dense probe of join 0 (K0 = kTabHash: generic).
template <int NJ, int NC, int W, int TILE, int STAGES, int K0, bool S0>
__global__ void __launch_bounds__((W + 1) * 32, 1) ssb_pipeline_kernel(const PipeArgs a) {
  constexpr int R = TILE / W;   // rows per consumer warp per stage
  constexpr int V = R / 128;    // int4 key vectors per lane (phase A)
  static_assert(R % 128 == 0 && V >= 1 && V <= 4, "phase A: 4..16 rows per lane");
  constexpr int NA = NC - NJ;   // aggregate columns: revenue [, supplycost]
  static_assert(NA == 1 || NA == 2, "aggregate columns");
  extern __shared__ __align__(128) unsigned char smem[];
  int32_t* ring = reinterpret_cast<int32_t*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * NC * TILE * 4);
  uint64_t* empty = full + STAGES;
  uint32_t* lists = reinterpret_cast<uint32_t*>(empty + STAGES);
  const char* sbase = reinterpret_cast<const char*>(smem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (a.n + TILE - 1) / TILE;
  const int my_tiles = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, W);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  uint64_t policy = 0;
  auto issue = [&](int it) {  // producer lane: stage `it` of this CTA
    const int s = it % STAGES;
    const int64_t base = (blockIdx.x + (int64_t)it * gridDim.x) * (int64_t)TILE;
    const int64_t rows = min((int64_t)TILE, a.n - base);
    const uint32_t bytes = (uint32_t)((rows * 4 + 15) & ~15ll);  // column buffers carry >= 256 B slack
    mbar_expect_tx(full + s, bytes * NC);
#pragma unroll
    for (int c = 0; c < NC; ++c)
      tma_load_1d(ring + ((size_t)s * NC + c) * TILE, a.col[c] + base, bytes, full + s, policy);
    if (a.l2_ahead > 0) {  // the tile l2_ahead loads later: into L2 now (more bytes in flight than the ring holds)
      const int64_t pb = (blockIdx.x + (int64_t)(it + a.l2_ahead) * gridDim.x) * (int64_t)TILE;
      if (pb < a.n) {
        const uint32_t pbytes = (uint32_t)((min((int64_t)TILE, a.n - pb) * 4 + 15) & ~15ll);
#pragma unroll
        for (int c = 0; c < NC; ++c) l2_prefetch_bulk(a.col[c] + pb, pbytes);
      }
    }
  };
  if (warp == W && lane == 0) {
    policy = policy_evict_first();
    for (int it = 0; it < my_tiles && it < STAGES; ++it) issue(it);
  }

  pdl_wait();  // the dimension builds (and the prologue) are complete from here on
  // shared copies of the dimension tables + the CTA-private aggregate
  // (overlaps the first loads)
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const ProbeTab& t = a.tab[j];
    if (t.smem < 0) continue;
    const int4* src = reinterpret_cast<const int4*>(t.g);
    int4* d = reinterpret_cast<int4*>(smem + t.smem);
    for (uint32_t i = threadIdx.x; i < t.bytes / 16; i += blockDim.x) d[i] = __ldg(src + i);
  }
  if (a.smem_agg >= 0) {
    unsigned long long* s_sum = reinterpret_cast<unsigned long long*>(smem + a.smem_agg);
    unsigned* s_cnt = reinterpret_cast<unsigned*>(s_sum + a.cells);
    for (int c = threadIdx.x; c < a.cells; c += blockDim.x) {
      s_sum[c] = 0;
      s_cnt[c] = 0;
    }
  }
  __syncthreads();

  if (warp == W) {  // ---------------------------------------------- producer
    if (lane == 0) {
      for (int it = STAGES; it < my_tiles; ++it) {
        const int s = it % STAGES;
        mbar_wait(empty + s, (uint32_t)(((it / STAGES) - 1) & 1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(it);
      }
    }
  } else {  // ------------------------------------------------------ consumers
    const ProbeTab t0 = a.tab[0];
    const HtMeta* meta = a.meta;
    uint32_t* list = lists + warp * R;
    unsigned long long* s_sum = reinterpret_cast<unsigned long long*>(smem + (a.smem_agg >= 0 ? a.smem_agg : 0));
    unsigned* s_cnt = reinterpret_cast<unsigned*>(s_sum + a.cells);
    const bool g0 = t0.gstride != 0;
    RegTab rt[NJ];
#pragma unroll
    for (int j = 1; j < NJ; ++j) rt[j] = reg_tab(a.tab[j], sbase);
    const unsigned lt = (1u << lane) - 1u;
    uint32_t surv[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) surv[j] = 0;
    bool bad_any = false;
    // one round of phase B: up to 32 survivors, one per lane
    struct Pending {
      int32_t key[NJ];
      uint32_t raw[NJ];
      int32_t va, vb;
      uint32_t ent;
      bool act;
    };
    auto gather = [&](const int32_t* st, int b, int total) {
      Pending q;
      q.act = b + lane < total;
      q.ent = q.act ? list[b + lane] : 0u;
      const int row = (int)(q.ent >> 16);
#pragma unroll
      for (int j = 1; j < NJ; ++j) q.key[j] = st[j * TILE + row];
      q.va = st[NJ * TILE + row];
      q.vb = NA == 2 ? st[(NJ + 1) * TILE + row] : 0;
#pragma unroll
      for (int j = 1; j < NJ; ++j) {  // every probe load in flight before any is used
        const uint32_t off = (uint32_t)q.key[j] - rt[j].kmin;
        q.raw[j] = rt[j].p[(off < rt[j].n ? off : 0u) >> rt[j].sh5];
      }
      return q;
    };
    auto finish = [&](const Pending& q) {
      bool alive = q.act;
      const uint32_t c0 = q.ent & 0xFFFFu;
      bool bad = g0 && c0 == 0xFFFFu;
      uint32_t idx = c0 * (uint32_t)t0.gstride;
#pragma unroll
      for (int j = 1; j < NJ; ++j) {
        const RegTab& t = rt[j];
        uint32_t c;
        bool hit, bj;
        if (!t.hash) {
          const uint32_t off = (uint32_t)q.key[j] - t.kmin;
          c = ((q.raw[j] >> ((off & t.emask) << t.lb)) & t.mask) ^ t.flip;
          hit = off < t.n && c != t.mask;
          bj = c == t.badc;
        } else {
          const int32_t r = alive ? hash_probe(a.tab[j], meta, q.key[j]) : -2;
          hit = r != -2;
          bj = r == -1;
          c = r < 0 ? 0u : (uint32_t)r;
        }
        alive = alive && hit;
        surv[j] += __popc(__ballot_sync(0xffffffffu, alive));
        idx += c * t.gstride;  // gstride 0: the join feeds no group part
        bad = bad || (t.gstride != 0 && bj);
      }
      if (alive) {
        if (bad || idx >= (uint32_t)a.cells) {
          bad_any = true;
        } else {
          long long v = q.va;
          if (NA == 2) v -= (long long)q.vb;
          if (a.smem_agg >= 0) {
            smem_add_i64(&s_sum[idx], v);
            atomicAdd(&s_cnt[idx], 1u);
          } else {
            atomicAdd(&a.g_sum[idx], (unsigned long long)v);
            atomicAdd(&a.g_cnt[idx], 1ull);
          }
        }
      }
    };
    Pending pb;
    bool pend = false;
    int64_t row0 = (int64_t)blockIdx.x * TILE + warp * R;  // first row of this warp's slice
    const int64_t row_step = (int64_t)gridDim.x * TILE;

    for (int it = 0; it < my_tiles; ++it, row0 += row_step) {
      const int s = it % STAGES;
      const int64_t left = a.n - row0;
      const int valid = left >= R ? R : (left > 0 ? (int)left : 0);
      mbar_wait(full + s, (uint32_t)((it / STAGES) & 1));
      const int32_t* st = ring + (size_t)s * NC * TILE + warp * R;

      // ---- phase A: join 0 over every row of the warp's slice, compacted
      int total = 0;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int4 k4 = reinterpret_cast<const int4*>(st)[v * 32 + lane];
        const int32_t kk[4] = {k4.x, k4.y, k4.z, k4.w};
        uint32_t off[4], w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          off[e] = (uint32_t)kk[e] - t0.kmin;
          if constexpr (K0 != kTabHash) w[e] = first_fetch<K0, S0>(t0, sbase, off[e]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = v * 128 + lane * 4 + e;
          uint32_t c = 0;
          bool hit;
          if constexpr (K0 != kTabHash) {
            hit = first_decode<K0>(t0, off[e], w[e], &c);
          } else {
            const int32_t r = hash_probe(t0, meta, kk[e]);
            hit = r != -2;
            c = r < 0 ? 0xFFFFu : (uint32_t)r;
          }
          hit = hit && row < valid;
          const unsigned b = __ballot_sync(0xffffffffu, hit);
          if (hit) list[total + __popc(b & lt)] = ((uint32_t)row << 16) | c;
          total += __popc(b);
        }
      }
      __syncwarp();
      surv[0] += total;

      // ---- phase B, software-pipelined by one tile: the probes of this
      // tile's first round were issued at the end of the previous iteration
      // and are consumed here, after the wait + phase A above hid their
      // latency.  (Earlier rounds read only registers.)
      if (pend) finish(pb);
      for (int b = 32; b < total; b += 32) {  // further rounds (rare), synchronous
        Pending q = gather(st, b, total);
        finish(q);
      }
      pb = gather(st, 0, total);  // keys/values into registers, probe loads in flight
      pend = total > 0;
      release_slot(empty + s, lane == 0);  // the stage is no longer read
    }
    if (pend) finish(pb);
    // all counters are warp-uniform (ballot-derived)
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        if (surv[j]) atomicAdd(&a.surv[j], (unsigned long long)surv[j]);
    }
    if (__any_sync(0xffffffffu, bad_any) && lane == 0) atomicExch(a.err, 2);
  }

  if (a.smem_agg >= 0) {
    __syncthreads();
    const unsigned long long* s_sum = reinterpret_cast<const unsigned long long*>(smem + a.smem_agg);
    const unsigned* s_cnt = reinterpret_cast<const unsigned*>(s_sum + a.cells);
    for (int c = threadIdx.x; c < a.cells; c += blockDim.x) {
      const unsigned k = s_cnt[c];
      if (k) {
        atomicAdd(&a.g_sum[c], s_sum[c]);
        atomicAdd(&a.g_cnt[c], (unsigned long long)k);
      }
    }
  }
}

// Shared-memory bytes of the ring + barriers + survivor lists (tables and the
// aggregate go after `fixed_smem`).
template <int NC, int TILE, int STAGES>
constexpr size_t fixed_smem() {
  return ((size_t)STAGES * NC * TILE * 4 + 2 * STAGES * 8 + (size_t)TILE * 4 + 127) & ~(size_t)127;
}

}  // namespace pipe
}  // namespace crys
