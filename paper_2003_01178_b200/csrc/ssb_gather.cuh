// ssb_gather.cuh -- the sparse tail of a SPLIT SSB plan on sm_100a.
//
// A plan's joins run in plan order (QueryStats.survivors[j] counts the rows
// alive after joins 0..j, ssb_queries.cpp:268-271), so once the first joins
// are selective most fact rows are dead and the later fact columns are only
// needed at the few 128-byte lines that still hold a live row
// (profiles/r02_min_bytes.json: 11.3 GB instead of 21.1 GB over q2-q4 at
// SF=20).  A split plan therefore runs in two kernels:
//
//   ssb_scan_emit_kernel<D, ...> (ssb_scan.cuh)  streams the first D join keys
//       densely through the TMA ring and writes every row alive after them to
//       its CTA's region of a survivor list: {row, partial group index | bad}
//   ssb_gather_kernel<NJ - D, NA, ...>     runs joins D..NJ-1 and the aggregate
//       over the list: per thread K entries, every gather (4-byte loads of the
//       later fact columns at the listed rows) and every probe of a stage in
//       flight before any is used, so DRAM latency is covered by memory-level
//       parallelism instead of a shared-memory ring.
//
// The DRAM lines a gather touches are exactly the lines the plan needs.
#pragma once

#include "ssb_pipeline.cuh"

namespace crys {
namespace pipe {

constexpr int kMaxRegions = 1024;

struct GatherArgs {
  const uint2* list;          // [regions][list_cap] {row, idx | bad << 31}
  int64_t list_cap;
  const unsigned* list_count; // entries per region
  int32_t nregions;           // <= kMaxRegions
  const int32_t* col[kMaxJ + 2];  // fact keys of joins D..NJ-1, then revenue [, supplycost]
  ProbeTab tab[kMaxJ];        // joins D..NJ-1 (smem offsets of THIS kernel)
  const HtMeta* meta;
  int32_t cells;
  int32_t smem_agg;           // byte offset of the shared aggregate (-1: global atomics)
  unsigned long long* g_sum;
  unsigned long long* g_cnt;
  unsigned long long* surv;   // survivors[D..NJ-1]
  int32_t* err;
  // late-materialising plans (ssb_scanbm.cuh): entries {row, key, key, key};
  // the first NPRE keys are those of the dense joins that feed a group part,
  // whose digits are decoded here from their code tables (membership was
  // already decided by the bitmaps)
  const uint4* list4;
  ProbeTab pre[3];
};

template <int NJB, int NA, int BT, int K, int NPRE = 0>
__global__ void __launch_bounds__(BT) ssb_gather_kernel(const GatherArgs a) {
  pdl_wait();  // the dense head's survivor list
  static_assert(NJB >= 1 && NJB <= kMaxJ && (NA == 1 || NA == 2), "gather shape");
  static_assert(NPRE >= 0 && NPRE <= 3, "digit joins of the dense head");
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ long long s_pre[kMaxRegions + 1];  // entries before each region
  __shared__ long long s_scan[BT / 32 + 1];
  const int lane = threadIdx.x & 31;
  // the list regions as one index space: exclusive prefix of the counts
  long long run = 0;
  for (int r0 = 0; r0 < a.nregions; r0 += BT) {
    const int r = r0 + (int)threadIdx.x;
    const long long c = r < a.nregions ? (long long)a.list_count[r] : 0;
    long long tot;
    const long long ex = BlockScan<BT>(c, s_scan, tot);
    if (r < a.nregions) s_pre[r] = run + ex;
    run += tot;
  }
  if (threadIdx.x == 0) s_pre[a.nregions] = run;
  // the CTA-private aggregate (small group domains: hot cells stay on chip)
  unsigned long long* s_sum = reinterpret_cast<unsigned long long*>(smem);
  unsigned* s_cnt = reinterpret_cast<unsigned*>(s_sum + a.cells);
  if (a.smem_agg >= 0)
    for (int c = threadIdx.x; c < a.cells; c += BT) {
      s_sum[c] = 0;
      s_cnt[c] = 0;
    }
  __syncthreads();
  const long long total = s_pre[a.nregions];

  // dimension tables are probed in L2 (they are small and hot; a per-CTA
  // shared copy costs more than the probes it would serve)
  RegTab rt[NJB];
#pragma unroll
  for (int j = 0; j < NJB; ++j) rt[j] = reg_tab(a.tab[j], nullptr);
  RegTab rp[NPRE > 0 ? NPRE : 1];
#pragma unroll
  for (int p = 0; p < NPRE; ++p) rp[p] = reg_tab(a.pre[p], nullptr);
  uint32_t surv[NJB];
#pragma unroll
  for (int j = 0; j < NJB; ++j) surv[j] = 0;
  bool bad_any = false;

  // the loop bound is uniform over the CTA (ballots below)
  for (long long base = (long long)blockIdx.x * BT * K; base < total; base += (long long)gridDim.x * BT * K) {
    uint32_t row[K], idx[K];
    bool alive[K], bad[K];
    uint32_t pkey[NPRE > 0 ? NPRE : 1][K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const long long i = base + k * BT + threadIdx.x;
      alive[k] = i < total;
      long long at = 0;
      if (alive[k]) {
        int lo = 0, hi = a.nregions;  // region: the last r with s_pre[r] <= i
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (s_pre[mid] <= i) lo = mid;
          else hi = mid;
        }
        at = (long long)lo * a.list_cap + (i - s_pre[lo]);
      }
      if (a.list4 == nullptr) {
        const uint2 e = alive[k] ? a.list[at] : make_uint2(0u, 0u);
        row[k] = e.x;
        bad[k] = (e.y >> 31) != 0;
        idx[k] = e.y & 0x7fffffffu;
      } else {
        const uint4 e = alive[k] ? a.list4[at] : make_uint4(0u, 0u, 0u, 0u);
        row[k] = e.x;
        bad[k] = false;
        idx[k] = 0;
        pkey[0][k] = e.y;
        if (NPRE > 1) pkey[NPRE > 1 ? 1 : 0][k] = e.z;
        if (NPRE > 2) pkey[NPRE > 2 ? 2 : 0][k] = e.w;
      }
    }
    // digits of the dense joins' group parts (K code probes in flight per join)
#pragma unroll
    for (int p = 0; p < NPRE; ++p) {
      const RegTab& t = rp[p];
      uint32_t raw[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t off = pkey[p][k] - t.kmin;
        raw[k] = alive[k] ? __ldg(t.p + ((off < t.n ? off : 0u) >> t.sh5)) : 0u;
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t off = pkey[p][k] - t.kmin;
        const uint32_t c = ((raw[k] >> ((off & t.emask) << t.lb)) & t.mask) ^ t.flip;
        alive[k] = alive[k] && off < t.n && c != t.mask;
        idx[k] += c * t.gstride;
        bad[k] = bad[k] || c == t.badc;
      }
    }
#pragma unroll
    for (int j = 0; j < NJB; ++j) {
      const RegTab& t = rt[j];
      int32_t key[K];
#pragma unroll
      for (int k = 0; k < K; ++k) key[k] = alive[k] ? ld_stream1(a.col[j] + row[k]) : 0;  // K gathers in flight
      uint32_t raw[K];
      if (!t.hash) {
#pragma unroll
        for (int k = 0; k < K; ++k) {  // K probes in flight
          const uint32_t off = (uint32_t)key[k] - t.kmin;
          raw[k] = alive[k] ? __ldg(t.p + ((off < t.n ? off : 0u) >> t.sh5)) : 0u;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        uint32_t c;
        bool hit, bj;
        if (!t.hash) {
          const uint32_t off = (uint32_t)key[k] - t.kmin;
          c = ((raw[k] >> ((off & t.emask) << t.lb)) & t.mask) ^ t.flip;
          hit = off < t.n && c != t.mask;
          bj = c == t.badc;
        } else {
          const int32_t r = alive[k] ? hash_probe(a.tab[j], a.meta, key[k]) : -2;
          hit = r != -2;
          bj = r == -1;
          c = r < 0 ? 0u : (uint32_t)r;
        }
        alive[k] = alive[k] && hit;
        idx[k] += c * t.gstride;
        bad[k] = bad[k] || (t.gstride != 0 && bj);
        surv[j] += __popc(__ballot_sync(0xffffffffu, alive[k]));
      }
    }
    int32_t va[K], vb[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      va[k] = alive[k] ? ld_stream1(a.col[NJB] + row[k]) : 0;
      vb[k] = (NA == 2 && alive[k]) ? ld_stream1(a.col[NJB + 1] + row[k]) : 0;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!alive[k]) continue;
      if (bad[k] || idx[k] >= (uint32_t)a.cells) {
        bad_any = true;
        continue;
      }
      long long v = va[k];
      if (NA == 2) v -= (long long)vb[k];
      if (a.smem_agg >= 0) {
        smem_add_i64(&s_sum[idx[k]], v);
        atomicAdd(&s_cnt[idx[k]], 1u);
      } else {
        atomicAdd(&a.g_sum[idx[k]], (unsigned long long)v);
        atomicAdd(&a.g_cnt[idx[k]], 1ull);
      }
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NJB; ++j)
      if (surv[j]) atomicAdd(&a.surv[j], (unsigned long long)surv[j]);
  }
  if (__any_sync(0xffffffffu, bad_any) && lane == 0) atomicExch(a.err, 2);
  pdl_trigger();  // the main loop is done: the compaction may start launching
  if (a.smem_agg >= 0) {
    __syncthreads();
    for (int c = threadIdx.x; c < a.cells; c += BT) {
      const unsigned k = s_cnt[c];
      if (k) {
        atomicAdd(&a.g_sum[c], s_sum[c]);
        atomicAdd(&a.g_cnt[c], (unsigned long long)k);
      }
    }
  }
}

}  // namespace pipe
}  // namespace crys
