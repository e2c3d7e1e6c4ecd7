// ssb_scan.cuh -- the dense head of a SPLIT SSB plan on sm_100a: joins 0..D-1
// over every lineorder row, survivors written to a list (ssb_gather.cuh runs
// the rest of the plan over it).
//
// Same TMA ring as ssb_pipeline.cuh (producer warp W streams the D key
// columns with cp.async.bulk + mbarrier complete_tx, L2 evict_first, plus an
// L2 bulk prefetch `l2_ahead` tiles ahead), but the consumers are cut to the
// minimum per row, because a one-column ring delivers rows 4x faster than the
// four-column one and the all-purpose consumer was issue-bound here (ncu:
// 75 % issue active, 45 warp instructions per 32 rows at 2.3 TB/s):
//   * each lane owns 4*V rows (V 128-bit LDS of keys per column per tile);
//   * join 0 is probed for all of them with ONE byte / halfword / word load
//     per row (table kind / placement specialised: K0, S0; a key outside the
//     table's range is clamped onto its extra absent entry instead of being
//     tested); group digits are only formed for live rows, and later dense
//     joins are only probed for them;
//   * live rows are then taken one per lane per round: join 0's digit is
//     re-read from the stage, the later dense joins probed, and each round's
//     survivors stored with one shared atomic (the list region is per CTA).
#pragma once

#include "ssb_pipeline.cuh"

namespace crys {
namespace pipe {

// Join 0's probe of one key: the table entry (a bitmap bit as 0/1, or the
// u8 / u16 code) at min(key - kmin, n); entry n is the table's absent pad.
template <int K0, bool S0>
__device__ __forceinline__ uint32_t probe_entry(const ProbeTab& t, const char* sbase, int32_t key) {
  const uint32_t o = min((uint32_t)key - t.kmin, t.n);
  const char* base = S0 ? sbase + t.smem : reinterpret_cast<const char*>(t.g);
  if constexpr (K0 == kTabBitmap) {
    const uint32_t w = S0 ? reinterpret_cast<const uint32_t*>(base)[o >> 5]
                          : __ldg(reinterpret_cast<const uint32_t*>(base) + (o >> 5));
    return (w >> (o & 31u)) & 1u;
  } else if constexpr (K0 == kTabU8) {
    return S0 ? (uint32_t)reinterpret_cast<const uint8_t*>(base)[o]
              : (uint32_t)__ldg(reinterpret_cast<const uint8_t*>(base) + o);
  } else {
    return S0 ? (uint32_t)reinterpret_cast<const uint16_t*>(base)[o]
              : (uint32_t)__ldg(reinterpret_cast<const uint16_t*>(base) + o);
  }
}
template <int K0>
__device__ __forceinline__ bool entry_hit(uint32_t e) {
  return K0 == kTabBitmap ? e != 0u : (K0 == kTabU8 ? e != kU8Absent : e != kU16Absent);
}
// group digit of a hit entry; 0xFFFF: a payload outside its group domain
template <int K0>
__device__ __forceinline__ uint32_t entry_digit(uint32_t e) {
  if constexpr (K0 == kTabBitmap) return 0u;
  else if constexpr (K0 == kTabU8) return e == kU8Bad ? 0xFFFFu : e;
  else return e == kU16Bad ? 0xFFFFu : e;
}

// A later join's probe (uniform decode of a direct table, or the
// linear-probing walk): member?  *c = its digit, *bad = digit outside the
// group domain.
__device__ __forceinline__ bool probe_reg(const RegTab& t, const ProbeTab& pt, const HtMeta* meta, int32_t key,
                                          uint32_t* c, bool* bad) {
  if (!t.hash) {
    const uint32_t off = (uint32_t)key - t.kmin;
    const uint32_t word = t.p[(off < t.n ? off : 0u) >> t.sh5];
    *c = ((word >> ((off & t.emask) << t.lb)) & t.mask) ^ t.flip;
    *bad = *c == t.badc;
    return off < t.n && *c != t.mask;
  }
  const int32_t r = hash_probe(pt, meta, key);
  *bad = r == -1;
  *c = r < 0 ? 0u : (uint32_t)r;
  return r != -2;
}

template <int D, int W, int TILE, int V, int STAGES, int K0, bool S0>
__global__ void __launch_bounds__((W + 1) * 32, 1) ssb_scan_emit_kernel(const PipeArgs a) {
  constexpr int R = TILE / W;  // rows per consumer warp per stage
  static_assert(R == 128 * V && V >= 1 && V <= 4, "4*V rows per lane");
  static_assert(D >= 1 && D <= 3, "dense joins");
  constexpr int NB = 4 * V;    // rows per lane
  extern __shared__ __align__(128) unsigned char smem[];
  int32_t* ring = reinterpret_cast<int32_t*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * D * TILE * 4);
  uint64_t* empty = full + STAGES;
  const char* sbase = reinterpret_cast<const char*>(smem);
  __shared__ unsigned s_list_n;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (a.n + TILE - 1) / TILE;
  const int my_tiles = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, W);
    }
    s_list_n = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  uint64_t policy = 0;
  auto issue = [&](int it) {  // producer lane: stage `it` of this CTA
    const int s = it % STAGES;
    const int64_t base = (blockIdx.x + (int64_t)it * gridDim.x) * (int64_t)TILE;
    const int64_t rows = min((int64_t)TILE, a.n - base);
    const uint32_t bytes = (uint32_t)((rows * 4 + 15) & ~15ll);  // columns carry >= 256 B slack
    mbar_expect_tx(full + s, bytes * D);
#pragma unroll
    for (int c = 0; c < D; ++c)
      tma_load_1d(ring + ((size_t)s * D + c) * TILE, a.col[c] + base, bytes, full + s, policy);
    if (a.l2_ahead > 0) {
      const int64_t pb = (blockIdx.x + (int64_t)(it + a.l2_ahead) * gridDim.x) * (int64_t)TILE;
      if (pb < a.n) {
        const uint32_t pbytes = (uint32_t)((min((int64_t)TILE, a.n - pb) * 4 + 15) & ~15ll);
#pragma unroll
        for (int c = 0; c < D; ++c) l2_prefetch_bulk(a.col[c] + pb, pbytes);
      }
    }
  };
  if (warp == W && lane == 0) {
    policy = policy_evict_first();
    for (int it = 0; it < my_tiles && it < STAGES; ++it) issue(it);
  }
  pdl_wait();  // the dimension builds (and the prologue) are complete from here on
  // shared copies of the dense joins' tables (overlaps the first loads)
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const ProbeTab& t = a.tab[j];
    if (t.smem < 0) continue;
    const int4* src = reinterpret_cast<const int4*>(t.g);
    int4* d = reinterpret_cast<int4*>(smem + t.smem);
    for (uint32_t i = threadIdx.x; i < t.bytes / 16; i += blockDim.x) d[i] = __ldg(src + i);
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
    return;
  }
  // ------------------------------------------------------------------ consumers
  const ProbeTab t0 = a.tab[0];
  const HtMeta* meta = a.meta;
  RegTab rt[D];
#pragma unroll
  for (int j = 1; j < D; ++j) rt[j] = reg_tab(a.tab[j], sbase);
  uint2* my_list = a.list + (int64_t)blockIdx.x * a.list_cap;
  uint32_t surv[D];
#pragma unroll
  for (int j = 0; j < D; ++j) surv[j] = 0;
  int64_t row0 = (int64_t)blockIdx.x * TILE + warp * R;  // first row of this warp's slice
  const int64_t row_step = (int64_t)gridDim.x * TILE;

  const unsigned lt = (1u << lane) - 1u;
  // Everything after join 0 for one tile (`stp` = its stage, still held):
  // join 1's probe words `raw` were issued one tile earlier (software
  // pipelining: the L2 probes of a large join-1 table overlap the next
  // stage's wait and join-0 pass), later joins are probed here; the rows alive
  // after every dense join go to the list one per lane per round (rounds are
  // warp-uniform), their group digits re-read from the stage; then the stage
  // is released.
  auto finish = [&](const int32_t* stp, int sp, unsigned h, const uint32_t (&raw)[NB], int64_t r0) {
    if constexpr (D >= 2) {
      const RegTab& t = rt[1];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (!((h >> b) & 1u)) continue;
        const int32_t key = stp[TILE + (b >> 2) * 128 + 4 * lane + (b & 3)];
        bool hit1;
        if (!t.hash) {
          const uint32_t off = (uint32_t)key - t.kmin;
          const uint32_t c = ((raw[b] >> ((off & t.emask) << t.lb)) & t.mask) ^ t.flip;
          hit1 = off < t.n && c != t.mask;
        } else {
          uint32_t c;
          bool bj;
          hit1 = probe_reg(t, a.tab[1], meta, key, &c, &bj);
        }
        if (!hit1) h &= ~(1u << b);
      }
      surv[1] += __popc(h);
#pragma unroll
      for (int jj = 2; jj < D; ++jj) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          uint32_t c;
          bool bj;
          if (((h >> b) & 1u) &&
              !probe_reg(rt[jj], a.tab[jj], meta, stp[jj * TILE + (b >> 2) * 128 + 4 * lane + (b & 3)], &c, &bj))
            h &= ~(1u << b);
        }
        surv[jj] += __popc(h);
      }
    }
    const uint32_t lrow = (uint32_t)r0 + (uint32_t)lane * 4u;
    while (__any_sync(0xffffffffu, h != 0)) {
      const bool act = h != 0;
      const int b = act ? __ffs(h) - 1 : 0;
      h &= h - 1u;
      const int r = (b >> 2) * 128 + 4 * lane + (b & 3);  // row in the warp slice
      const uint32_t c0 = entry_digit<K0>(probe_entry<K0, S0>(t0, sbase, stp[r]));
      uint32_t idx = (t0.gstride != 0 && c0 == 0xFFFFu) ? 0x80000000u : c0 * (uint32_t)t0.gstride;
#pragma unroll
      for (int jj = 1; jj < D; ++jj) {
        uint32_t c;
        bool bj;
        probe_reg(rt[jj], a.tab[jj], meta, stp[jj * TILE + r], &c, &bj);
        if (rt[jj].gstride != 0 && bj) idx = 0x80000000u;
        else if (!(idx >> 31)) idx += c * rt[jj].gstride;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, act);
      const int leader = __ffs(bal) - 1;
      unsigned base = 0;
      if (lane == leader) base = atomicAdd(&s_list_n, (unsigned)__popc(bal));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (act) my_list[base + __popc(bal & lt)] = make_uint2(lrow + (uint32_t)((b >> 2) * 128 + (b & 3)), idx);
    }
    release_slot(empty + sp, lane == 0);  // the stage is no longer read
  };

  // the previous tile, waiting for its join-1 probe words (D >= 2)
  unsigned p_hit = 0;
  uint32_t p_raw[NB];
  int p_s = -1;
  int64_t p_row0 = 0;
#pragma unroll
  for (int b = 0; b < NB; ++b) p_raw[b] = 0;

  for (int it = 0; it < my_tiles; ++it, row0 += row_step) {
    const int s = it % STAGES;
    const int64_t left = a.n - row0;
    const int valid = left >= R ? R : (left > 0 ? (int)left : 0);
    mbar_wait(full + s, (uint32_t)((it / STAGES) & 1));
    const int32_t* st = ring + (size_t)s * D * TILE + warp * R;

    // join 0 over every row: row b of the lane is slice row (b >> 2) * 128 + 4 * lane + (b & 3)
    uint32_t ent[NB];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int4 k4 = reinterpret_cast<const int4*>(st)[v * 32 + lane];
      ent[4 * v + 0] = probe_entry<K0, S0>(t0, sbase, k4.x);
      ent[4 * v + 1] = probe_entry<K0, S0>(t0, sbase, k4.y);
      ent[4 * v + 2] = probe_entry<K0, S0>(t0, sbase, k4.z);
      ent[4 * v + 3] = probe_entry<K0, S0>(t0, sbase, k4.w);
    }
    unsigned hit = 0;
#pragma unroll
    for (int b = 0; b < NB; ++b) hit |= (entry_hit<K0>(ent[b]) ? 1u : 0u) << b;
    if (valid < R) {  // the shard's last tile
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if ((b >> 2) * 128 + 4 * lane + (b & 3) >= valid) hit &= ~(1u << b);
    }
    surv[0] += __popc(hit);
    if constexpr (D == 1) {
      finish(st, s, hit, p_raw, row0);
    } else {
      // join 1's probe words for this tile's live rows, consumed next iteration
      uint32_t raw[NB];
      const RegTab& t = rt[1];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const bool any = ((hit >> (v * 4)) & 0xFu) != 0;
        int4 k4 = make_int4(0, 0, 0, 0);
        if (any && !t.hash) k4 = reinterpret_cast<const int4*>(st + TILE)[v * 32 + lane];
        const int32_t kk[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t off = (uint32_t)kk[e] - t.kmin;
          raw[4 * v + e] = (((hit >> (4 * v + e)) & 1u) && !t.hash) ? t.p[(off < t.n ? off : 0u) >> t.sh5] : 0u;
        }
      }
      if (p_s >= 0) finish(ring + (size_t)p_s * D * TILE + warp * R, p_s, p_hit, p_raw, p_row0);
      p_s = s;
      p_hit = hit;
      p_row0 = row0;
#pragma unroll
      for (int b = 0; b < NB; ++b) p_raw[b] = raw[b];
    }
  }
  if (D >= 2 && p_s >= 0) finish(ring + (size_t)p_s * D * TILE + warp * R, p_s, p_hit, p_raw, p_row0);
  // survivors of the dense joins (per-lane counts): one atomic per warp and join
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const uint32_t wsum = warp_sum(surv[j]);
    if (lane == 0 && wsum) atomicAdd(&a.surv[j], (unsigned long long)wsum);
  }
  asm volatile("bar.sync 1, %0;" ::"n"(W * 32));  // consumers only
  pdl_trigger();  // the main loop is done: the next kernel may start launching
  if (threadIdx.x == 0) a.list_count[blockIdx.x] = s_list_n;
}

}  // namespace pipe
}  // namespace crys
