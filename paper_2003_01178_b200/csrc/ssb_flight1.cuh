// ssb_flight1.cuh -- flight 1 (q1.1-q1.3) as a TMA ring over the date column
// for selective date filters (q1.2: 1/84 of the rows, q1.3: 1/365).
//
// The register-tile kernel (ssb_flight1_kernel) keeps at most one tile of the
// first column in flight per thread: 4 CTAs x 256 threads x 32 B = 32 KB per
// SM, which at a loaded HBM latency of ~1.5 us caps the date stream near
// 3 TB/s (measured: q1.3 0.172 ms for 0.54 GB of DRAM).  Here a producer warp
// streams lo_orderdate alone through a STAGES-deep shared-memory ring with
// cp.async.bulk (plus an L2 bulk prefetch `l2_ahead` tiles further), so
// ~190 KB per SM are in flight, and the consumer warps only:
//   * evaluate the date range over their 4*V rows per lane (128-bit LDS);
//   * release the stage at once (the date column is not read again);
//   * take the surviving rows one per lane per round (ballot rounds), and
//     issue the discount / quantity / extended-price loads of those rows;
//   * resolve the PREVIOUS tile's loads (software pipelining: the gather
//     latency overlaps this tile's wait and date pass).  The first PR rounds
//     of a tile are pipelined; further rounds (dense tiles, q1.1) resolve at
//     once.
// The result is the conjunction of the three predicates and the sum of
// extendedprice * discount over it, exactly run_flight1
// (P:src/ssb_queries.cpp:157-210); only the load order differs.
#pragma once
// Included by ssb_query.cu inside namespace crys (Flight1Args, warp_sum).

// ST: striped ownership (row b of a lane = b * 32 + lane, scalar LDS) instead
// of 4-row vectors.  An order's lines are consecutive rows with one date, so
// the date survivors come in runs of ~4; striped, a run spreads over 4 lanes
// and is gathered in ONE round instead of four.
// D: dense columns in the ring.  1: the date only; 2: date and discount (the
// discount's lines are mostly live anyway when the date filter keeps 1/7 of
// the rows, q1.1), so only quantity and price are gathered, for rows passing
// both.
// CHN (D == 1): chained gathers, as the reference orders them.  A tile's date
// survivors first load their discount only; one tile later the rows whose
// discount passes load quantity and price; one more tile later those resolve.
// Two pipeline levels instead of one, but the quantity / price lines of rows
// failing the discount are never fetched (ncu, q1.2: 0.95 GB of DRAM reads
// with all three gathered per date survivor).
template <int W, int V, int STAGES, int PR, bool ST = false, int D = 1, bool CHN = false>
__global__ void __launch_bounds__((W + 1) * 32, 1) ssb_flight1_ring_kernel(const Flight1Args a) {
  static_assert(D == 1 || D == 2, "dense ring columns");
  // chained level 1: the discount (D == 1) or the quantity (D == 2)
  constexpr int R = 128 * V;   // rows per consumer warp per stage
  constexpr int TILE = W * R;  // rows per stage
  constexpr int NB = 4 * V;    // rows per lane
  static_assert(NB <= 32, "a lane's hits are a 32-bit mask");
  extern __shared__ __align__(128) unsigned char smem[];
  int32_t* ring = reinterpret_cast<int32_t*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * D * TILE * 4);
  uint64_t* empty = full + STAGES;
  __shared__ long long red[2][W];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (a.n + TILE - 1) / TILE;
  const int my_tiles = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      pipe::mbar_init(full + s, 1);
      pipe::mbar_init(empty + s, W);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == W) {  // ------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t policy = pipe::policy_evict_first();
      for (int it = 0; it < my_tiles; ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) {
          pipe::mbar_wait(empty + s, (uint32_t)(((it / STAGES) - 1) & 1));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        const int64_t base = (blockIdx.x + (int64_t)it * gridDim.x) * (int64_t)TILE;
        const int64_t rows = min((int64_t)TILE, a.n - base);
        const uint32_t bytes = (uint32_t)((rows * 4 + 15) & ~15ll);  // columns carry >= 256 B slack
        pipe::mbar_expect_tx(full + s, bytes * D);
#pragma unroll
        for (int c = 0; c < D; ++c)
          pipe::tma_load_1d(ring + ((size_t)s * D + c) * TILE, a.fcol[c] + base, bytes, full + s, policy);
        if (a.l2_ahead > 0) {
          const int64_t pb = (blockIdx.x + (int64_t)(it + a.l2_ahead) * gridDim.x) * (int64_t)TILE;
          if (pb < a.n) {
#pragma unroll
            for (int c = 0; c < D; ++c)
              pipe::l2_prefetch_bulk(a.fcol[c] + pb, (uint32_t)((min((int64_t)TILE, a.n - pb) * 4 + 15) & ~15ll));
          }
        }
      }
    }
    return;
  }
  // ----------------------------------------------------------------- consumers
  const int32_t lo0 = a.flo[0], hi0 = a.fhi[0];
  const int32_t lo1 = a.flo[1], hi1 = a.fhi[1], lo2 = a.flo[2], hi2 = a.fhi[2];
  const int32_t* __restrict__ c1 = a.fcol[1];
  const int32_t* __restrict__ c2 = a.fcol[2];
  const int32_t* __restrict__ pa = a.agg_a;
  const int32_t* __restrict__ pb = a.agg_b;
  const bool b_is_f1 = a.agg_b_is_f1 != 0;
  long long sum = 0;
  unsigned cnt = 0;
  // pending gathers of the previous tile: PR rounds, one row per lane each
  bool pv[PR];
  int32_t pd[PR], pq[PR], pp[PR], pm[PR];
#pragma unroll
  for (int r = 0; r < PR; ++r) pv[r] = false;
  // CHN: discount loads in flight (level 1): valid, row, discount
  bool cv[PR];
  int64_t crow[PR];
  int32_t cd[PR], cx[PR];  // level-1 value; D == 2: the row's discount (from the stage)
#pragma unroll
  for (int r = 0; r < PR; ++r) {
    cv[r] = false;
    crow[r] = 0;
    cd[r] = cx[r] = 0;
  }
  const int32_t* __restrict__ l1col = D == 1 ? c1 : c2;
  const int32_t l1lo = D == 1 ? lo1 : lo2, l1hi = D == 1 ? hi1 : hi2;

  auto resolve = [&](bool v, int32_t d, int32_t q, int32_t p, int32_t m) {
    if (v && (D == 2 || (d >= lo1 && d <= hi1)) && q >= lo2 && q <= hi2) {
      sum += (long long)p * (long long)(b_is_f1 ? d : m);
      ++cnt;
    }
  };

  int64_t row0 = (int64_t)blockIdx.x * TILE + warp * R;
  const int64_t row_step = (int64_t)gridDim.x * TILE;
  for (int it = 0; it < my_tiles; ++it, row0 += row_step) {
    const int s = it % STAGES;
    const int64_t left = a.n - row0;
    const int valid = left >= R ? R : (left > 0 ? (int)left : 0);
    pipe::mbar_wait(full + s, (uint32_t)((it / STAGES) & 1));
    const int32_t* st = ring + (size_t)s * D * TILE + warp * R;
    // slice row of this lane's item b
    auto srow = [&](int b) { return ST ? b * 32 + lane : (b >> 2) * 128 + 4 * lane + (b & 3); };
    unsigned h = 0;
    if constexpr (ST) {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int32_t k = st[b * 32 + lane];
        bool hit = k >= lo0 && k <= hi0;
        if constexpr (D == 2) {
          const int32_t k1 = st[TILE + b * 32 + lane];
          hit = hit && k1 >= lo1 && k1 <= hi1;
        }
        h |= (unsigned)hit << b;
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int4 k4 = reinterpret_cast<const int4*>(st)[v * 32 + lane];
        h |= ((unsigned)(k4.x >= lo0 && k4.x <= hi0) << (4 * v + 0)) |
             ((unsigned)(k4.y >= lo0 && k4.y <= hi0) << (4 * v + 1)) |
             ((unsigned)(k4.z >= lo0 && k4.z <= hi0) << (4 * v + 2)) |
             ((unsigned)(k4.w >= lo0 && k4.w <= hi0) << (4 * v + 3));
      }
      if constexpr (D == 2) {
        unsigned h1 = 0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int4 k4 = reinterpret_cast<const int4*>(st + TILE)[v * 32 + lane];
          h1 |= ((unsigned)(k4.x >= lo1 && k4.x <= hi1) << (4 * v + 0)) |
                ((unsigned)(k4.y >= lo1 && k4.y <= hi1) << (4 * v + 1)) |
                ((unsigned)(k4.z >= lo1 && k4.z <= hi1) << (4 * v + 2)) |
                ((unsigned)(k4.w >= lo1 && k4.w <= hi1) << (4 * v + 3));
        }
        h &= h1;
      }
    }
    if (D == 1) pipe::release_slot(empty + s, lane == 0);  // the date stage is not read again
    if (valid < R) {
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (srow(b) >= valid) h &= ~(1u << b);
    }
    // this tile's first PR rounds: issue the gathers (consumed next tile)
    bool nv[PR];
    int32_t nd[PR], nq[PR], np[PR], nm[PR];
#pragma unroll
    for (int r = 0; r < PR; ++r) {
      const bool h1v = h != 0;
      nv[r] = h1v;
      const int b = h1v ? __ffs(h) - 1 : 0;
      h &= h - 1u;
      const int64_t row = row0 + srow(b);
      nd[r] = nq[r] = np[r] = nm[r] = 0;
      if constexpr (CHN) {
        // level 2 from the previous tile's level-1 values; level 1 for this tile
        const bool go = cv[r] && cd[r] >= l1lo && cd[r] <= l1hi;
        nv[r] = go;
        nd[r] = D == 1 ? cd[r] : cx[r];
        nq[r] = D == 1 ? 0 : cd[r];
        if (go) {
          if (D == 1) nq[r] = __ldg(c2 + crow[r]);
          np[r] = __ldg(pa + crow[r]);
          if (!b_is_f1) nm[r] = __ldg(pb + crow[r]);
        }
        cv[r] = h1v;
        crow[r] = row;
        if (h1v) {
          cd[r] = __ldg(l1col + row);
          if (D == 2) cx[r] = st[TILE + srow(b)];
        }
      } else if (nv[r]) {
        nd[r] = D == 2 ? st[TILE + srow(b)] : __ldg(c1 + row);
        nq[r] = __ldg(c2 + row);
        np[r] = __ldg(pa + row);
        if (!b_is_f1) nm[r] = __ldg(pb + row);
      }
    }
    // the previous tile's gathers
#pragma unroll
    for (int r = 0; r < PR; ++r) resolve(pv[r], pd[r], pq[r], pp[r], pm[r]);
    // rounds beyond PR (dense tiles): resolved at once
    while (__any_sync(0xffffffffu, h != 0)) {
      const bool act = h != 0;
      const int b = act ? __ffs(h) - 1 : 0;
      h &= h - 1u;
      if (act) {
        const int64_t row = row0 + srow(b);
        const int32_t d = D == 2 ? st[TILE + srow(b)] : __ldg(c1 + row);
        if (!CHN || D == 2 || (d >= lo1 && d <= hi1)) {
          const int32_t q = __ldg(c2 + row);
          if (!CHN || (q >= lo2 && q <= hi2)) {
            const int32_t p = __ldg(pa + row);
            resolve(true, d, q, p, b_is_f1 ? 0 : __ldg(pb + row));
          }
        }
      }
    }
    if (D == 2) pipe::release_slot(empty + s, lane == 0);  // discounts of the gathered rows read
#pragma unroll
    for (int r = 0; r < PR; ++r) {
      pv[r] = nv[r];
      pd[r] = nd[r];
      pq[r] = nq[r];
      pp[r] = np[r];
      pm[r] = nm[r];
    }
  }
#pragma unroll
  for (int r = 0; r < PR; ++r) resolve(pv[r], pd[r], pq[r], pp[r], pm[r]);
  if constexpr (CHN) {  // the last tile's level-1 values
#pragma unroll
    for (int r = 0; r < PR; ++r)
      if (cv[r] && cd[r] >= l1lo && cd[r] <= l1hi)
        resolve(true, D == 1 ? cd[r] : cx[r], D == 1 ? __ldg(c2 + crow[r]) : cd[r], __ldg(pa + crow[r]),
                b_is_f1 ? 0 : __ldg(pb + crow[r]));
  }
  const long long ws = warp_sum(sum);
  const long long wc = warp_sum((long long)cnt);
  if (lane == 0) {
    red[0][warp] = ws;
    red[1][warp] = wc;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(W * 32));  // consumers only
  pdl_trigger();  // the main loop is done: the next kernel may start launching
  pdl_wait();  // the prologue zeroed the aggregate (the scan above overlapped it)
  if (threadIdx.x == 0) {
    long long s = 0, c = 0;
    for (int w = 0; w < W; ++w) {
      s += red[0][w];
      c += red[1][w];
    }
    atomicAdd(a.g_sum, (unsigned long long)s);
    atomicAdd(a.g_cnt, (unsigned long long)c);
    atomicAdd(a.surv, (unsigned long long)c);
  }
}
