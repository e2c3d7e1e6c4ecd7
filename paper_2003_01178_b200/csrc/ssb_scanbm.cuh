// ssb_scanbm.cuh -- the dense head of a LATE-MATERIALISING SSB plan on sm_100a:
// joins 0..D-1 tested against MEMBERSHIP BITMAPS over every lineorder row,
// the rows alive after them written to a survivor list with the keys whose
// group digits are still needed; ssb_gather_kernel<NPRE > 0> resolves those
// digits, runs joins D..NJ-1 and the aggregate over the list.
//
// Why: in q2.x / q3.1 / q3.2 / q4.x the first two joins decide almost every
// row (q2.1: 0.8 % survive supplier and part), so streaming the date key and
// the aggregate columns densely (the fused pipeline, 1.92 GB / 2.88 GB) moves
// 2-4x the bytes the plan needs.  Streaming only the first D keys and
// gathering the rest at the survivors' rows cuts that to the lines that still
// hold a live row (profiles/r02_min_bytes.json).  The earlier split head
// (ssb_scan.cuh) probed join 1's u8/u16 CODE table through L2 for every row
// alive after join 0 (20 % of the rows); here a join's membership is one bit
// in a shared-memory bitmap (part: 1.06 M keys = 133 KB at SF=20, customer
// 75 KB, supplier 5 KB), so the dense pass never leaves the SM, and the group
// digits are fetched from the code tables only for the final survivors (in
// the gather kernel, where occupancy hides the L2 latency).
//
//   producer warp W: TMA ring of the D key columns (cp.async.bulk + mbarrier
//     complete_tx, L2 evict_first, L2 bulk prefetch l2_ahead tiles ahead)
//   consumer warps: each lane owns 4*V rows of its warp's slice (128-bit LDS);
//     join 0's bit for every row, joins 1..D-1 only for rows still alive;
//     survivors one per lane per round to the CTA's list region:
//     {row, key of digit join 0, 1, 2} (unused words 0).
#pragma once

#include "ssb_pipeline.cuh"

namespace crys {
namespace pipe {

struct BmArgs {
  int64_t n;                 // lineorder rows of the shard
  const int32_t* col[3];     // dense join keys, plan order
  const uint32_t* bm[3];     // membership bitmaps (bit nk: absent pad)
  uint32_t kmin[3], nk[3];   // key domain [kmin, kmin + nk)
  int32_t smem[3];           // byte offset of the shared copy (-1: probed through L2)
  uint32_t words[3];         // bitmap words (multiple of 4)
  int32_t key_of[3];         // entry word 1..3 <- the key of dense join key_of[w-1] (-1: 0)
  uint4* list;               // [gridDim.x][list_cap]
  int64_t list_cap;
  unsigned* list_count;      // [gridDim.x]
  unsigned long long* surv;  // survivors[0..D-1]
  int32_t l2_ahead;
};

// sbm: the shared copy (used when `shared`), gbm: the global bitmap
__device__ __forceinline__ uint32_t bm_test(const uint32_t* sbm, const uint32_t* gbm, uint32_t kmin, uint32_t nk,
                                            int32_t key, bool shared) {
  const uint32_t off = min((uint32_t)key - kmin, nk);  // out of range -> the absent pad bit
  if (shared) {  // byte-granular shared load: address = base + (off >> 3) is one LEA.HI
    uint32_t b;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(b) : "r"(s_addr(sbm) + (off >> 3)));
    return (b >> (off & 7u)) & 1u;
  }
  const uint32_t w = __ldg(gbm + (off >> 5));
  return (w >> (off & 31u)) & 1u;
}

// ALLSH: every bitmap is in shared memory (plain LDS probes); otherwise each
// join's placement is tested at run time.
template <int D, int W, int V, int STAGES, bool ALLSH = false>
__global__ void __launch_bounds__((W + 1) * 32, 1) ssb_scan_bm_kernel(const BmArgs a) {
  constexpr int R = 128 * V;   // rows per consumer warp per stage
  constexpr int TILE = W * R;  // rows per stage
  constexpr int NB = 4 * V;    // rows per lane
  static_assert(D >= 1 && D <= 3 && V >= 1 && V <= 8, "scan shape");
  extern __shared__ __align__(128) unsigned char smem[];
  int32_t* ring = reinterpret_cast<int32_t*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * D * TILE * 4);
  uint64_t* empty = full + STAGES;
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

  auto issue = [&](int it, uint64_t policy) {
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
    const uint64_t policy = policy_evict_first();
    for (int it = 0; it < my_tiles && it < STAGES; ++it) issue(it, policy);
  }
  pdl_wait();  // the dimension builds (and the prologue) are complete from here on
  // shared copies of the bitmaps (overlap the first loads)
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (a.smem[j] < 0) continue;
    const uint4* src = reinterpret_cast<const uint4*>(a.bm[j]);
    uint4* dst = reinterpret_cast<uint4*>(smem + a.smem[j]);
    for (uint32_t i = threadIdx.x; i < a.words[j] / 4; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  __syncthreads();

  if (warp == W) {  // ---------------------------------------------- producer
    if (lane == 0) {
      const uint64_t policy = policy_evict_first();
      for (int it = STAGES; it < my_tiles; ++it) {
        const int s = it % STAGES;
        mbar_wait(empty + s, (uint32_t)(((it / STAGES) - 1) & 1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(it, policy);
      }
    }
    return;
  }
  // ------------------------------------------------------------------ consumers
  const uint32_t *sbm[3], *gbm[3];
  bool sh[3];
  uint32_t kmin[3], nk[3];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    sh[j] = ALLSH || a.smem[j] >= 0;
    sbm[j] = reinterpret_cast<const uint32_t*>(smem + (sh[j] ? a.smem[j] : 0));
    gbm[j] = a.bm[j];
    kmin[j] = a.kmin[j];
    nk[j] = a.nk[j];
  }
  const int k1 = a.key_of[0], k2 = a.key_of[1], k3 = a.key_of[2];
  uint4* my_list = a.list + (int64_t)blockIdx.x * a.list_cap;
  uint32_t surv[D];
#pragma unroll
  for (int j = 0; j < D; ++j) surv[j] = 0;
  const unsigned lt = (1u << lane) - 1u;
  int64_t row0 = (int64_t)blockIdx.x * TILE + warp * R;
  const int64_t row_step = (int64_t)gridDim.x * TILE;

  for (int it = 0; it < my_tiles; ++it, row0 += row_step) {
    const int s = it % STAGES;
    const int64_t left = a.n - row0;
    const int valid = left >= R ? R : (left > 0 ? (int)left : 0);
    mbar_wait(full + s, (uint32_t)((it / STAGES) & 1));
    const int32_t* st = ring + (size_t)s * D * TILE + warp * R;
    // join 0 for every row: row b of the lane = slice row (b >> 2) * 128 + 4 * lane + (b & 3)
    unsigned h = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int4 k4 = reinterpret_cast<const int4*>(st)[v * 32 + lane];
      h |= (bm_test(sbm[0], gbm[0], kmin[0], nk[0], k4.x, sh[0]) << (4 * v + 0)) |
           (bm_test(sbm[0], gbm[0], kmin[0], nk[0], k4.y, sh[0]) << (4 * v + 1)) |
           (bm_test(sbm[0], gbm[0], kmin[0], nk[0], k4.z, sh[0]) << (4 * v + 2)) |
           (bm_test(sbm[0], gbm[0], kmin[0], nk[0], k4.w, sh[0]) << (4 * v + 3));
    }
    if (valid < R) {
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if ((b >> 2) * 128 + 4 * lane + (b & 3) >= valid) h &= ~(1u << b);
    }
    surv[0] += __popc(h);
    // later dense joins, only where a row is still alive (whole vectors skipped)
#pragma unroll
    for (int j = 1; j < D; ++j) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const unsigned hv = (h >> (4 * v)) & 0xFu;
        if (!hv) continue;
        const int4 k4 = reinterpret_cast<const int4*>(st + j * TILE)[v * 32 + lane];
        unsigned m;
        if (ALLSH || sh[j]) {
          m = bm_test(sbm[j], gbm[j], kmin[j], nk[j], k4.x, true) |
              (bm_test(sbm[j], gbm[j], kmin[j], nk[j], k4.y, true) << 1) |
              (bm_test(sbm[j], gbm[j], kmin[j], nk[j], k4.z, true) << 2) |
              (bm_test(sbm[j], gbm[j], kmin[j], nk[j], k4.w, true) << 3);
        } else {
          // a bitmap probed through L2 costs one L1tex wavefront per loading
          // lane: load only for the rows still alive, not the whole vector
          const int32_t kk[4] = {k4.x, k4.y, k4.z, k4.w};
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t off = min((uint32_t)kk[e] - kmin[j], nk[j]);
            w[e] = ((hv >> e) & 1u) ? __ldg(gbm[j] + (off >> 5)) : 0u;
          }
          m = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t off = min((uint32_t)kk[e] - kmin[j], nk[j]);
            m |= ((w[e] >> (off & 31u)) & 1u) << e;
          }
        }
        h &= ~((hv & ~m) << (4 * v));
      }
      surv[j] += __popc(h);
    }
    // survivors, one per lane per round (rounds are warp-uniform)
    while (__any_sync(0xffffffffu, h != 0)) {
      const bool act = h != 0;
      const int b = act ? __ffs(h) - 1 : 0;
      h &= h - 1u;
      const int r = (b >> 2) * 128 + 4 * lane + (b & 3);
      const unsigned bal = __ballot_sync(0xffffffffu, act);
      const int leader = __ffs(bal) - 1;
      unsigned base = 0;
      if (lane == leader) base = atomicAdd(&s_list_n, (unsigned)__popc(bal));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (act) {
        uint4 e;
        e.x = (uint32_t)row0 + (uint32_t)r;  // shard row (< 2^31)
        e.y = k1 >= 0 ? (uint32_t)st[k1 * TILE + r] : 0u;
        e.z = k2 >= 0 ? (uint32_t)st[k2 * TILE + r] : 0u;
        e.w = k3 >= 0 ? (uint32_t)st[k3 * TILE + r] : 0u;
        my_list[base + __popc(bal & lt)] = e;
      }
    }
    release_slot(empty + s, lane == 0);  // the stage is no longer read
  }
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const uint32_t ws = warp_sum(surv[j]);
    if (lane == 0 && ws) atomicAdd(&a.surv[j], (unsigned long long)ws);
  }
  asm volatile("bar.sync 1, %0;" ::"n"(W * 32));  // consumers only
  pdl_trigger();  // the main loop is done: the next kernel may start launching
  if (threadIdx.x == 0) a.list_count[blockIdx.x] = s_list_n;
}

}  // namespace pipe
}  // namespace crys
