// ssb_query.cu -- fused Star Schema Benchmark pipelines on sm_100a.
//
// Replaces run_query / run_flight1 / run_joins / build_dim_table /
// AggregateTable / grouped_result of the reference (ssb_queries.cpp:15-286).
// Per query:
//   1. dimension builds (3 launches covering every join of the plan):
//        dim_filter_kernel  filter + compact each dimension (build_dim_table,
//                           ssb_queries.cpp:99-118), count on device
//        dim_init_kernel    capacity = max(2, bit_ceil(2n)) decided on device
//                           (ssb_queries.cpp:119), slots <- {EMPTY,0}
//        dim_insert_kernel  BlockBuildHashTable, 64-bit CAS claims
//   2. ONE fused pass over the lineorder shard (the hot loop, ssb_queries.cpp:
//      181-201 / 233-263): vectorised column loads, chained predicates or up to
//      four pipelined hash probes with selective loads of later columns, and the
//      group-by folded into a shared-memory-privatised dense table (or global
//      atomics when the domain is too large), no materialisation.
//   3. finalize_kernel compacts occupied cells (occupancy, not sum != 0:
//      ssb_queries.cpp:32-35) and one D2H copy returns them; the host orders
//      rows by cell index = lexicographic group order (ssb_queries.cpp:153).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "crystal.cuh"
#include "internal.hpp"

namespace crys {

namespace {

constexpr int kMaxJoins = 4;

struct DimBuildDesc {
  const int32_t* key;
  const int32_t* payload;  // null: payload 0 (ssb_queries.cpp:116)
  const int32_t* fcol[2];
  int32_t nranges[2];
  int32_t r[2][2][2];
  int32_t nf;
  int64_t rows;
  int64_t maxcap;
  int2* compact;
  int2* slots;
  uint32_t* bitmap;  // exact key-range membership bitmap (null: linear-probing HT)
  int32_t* payarr;   // payload indexed by key - kmin (null: join carries no payload)
  int32_t kmin;
  uint32_t nbits;
};

struct DimBuildArgs {
  DimBuildDesc d[kMaxJoins];
  HtMeta* meta;
};

struct JoinDesc {
  const int32_t* fk;  // lineorder foreign-key column (shard)
  const int2* slots;
  int32_t glo, gcard, gstride;  // group part fed by this join's payload (gcard 0: none)
  const uint32_t* bitmap;       // membership bitmap over [kmin, kmin+nbits) (null: probe the HT)
  const int32_t* payarr;        // payload of member key k at payarr[k - kmin]
  int32_t kmin;
  uint32_t nbits;
  int32_t need_payload;
};

struct FusedArgs {
  int64_t n;  // rows in the shard
  JoinDesc j[kMaxJoins];
  const HtMeta* meta;
  const int32_t* fcol[3];  // flight 1 filter columns
  int32_t flo[3], fhi[3];
  const int32_t* agg_a;
  const int32_t* agg_b;
  int32_t agg_b_is_f1;
  int32_t cells;
  unsigned long long* g_sum;  // [cells]
  unsigned long long* g_cnt;  // [cells]
  unsigned long long* surv;   // [4]
  int32_t* err;
  int32_t smem_bm_words;      // shared-memory room for the first join's bitmap
};

struct ResultHeader {
  unsigned long long nrows;
  unsigned long long surv[4];
  int32_t err;
  int32_t ht_err;
  int32_t pad[4];
};
static_assert(sizeof(ResultHeader) == 64, "header is one 64 B line");

struct RowOut {
  long long cell;
  long long sum;
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------- dimension builds

__global__ void dim_filter_kernel(const DimBuildArgs a) {
  const DimBuildDesc& d = a.d[blockIdx.y];
  HtMeta* m = a.meta + blockIdx.y;
  const unsigned lane = lane_id();
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < d.rows;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = base + threadIdx.x;
    bool pass = row < d.rows;
    if (pass) {
      for (int f = 0; f < d.nf; ++f) {
        const int32_t v = d.fcol[f][row];
        bool hit = false;
        for (int r = 0; r < d.nranges[f]; ++r) hit |= v >= d.r[f][r][0] && v <= d.r[f][r][1];
        pass = pass && hit;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, pass);
    if (bal == 0) continue;
    const int leader = __ffs(bal) - 1;
    int pos0 = 0;
    if ((int)lane == leader) pos0 = atomicAdd(&m->count, __popc(bal));  // build size (both layouts)
    pos0 = __shfl_sync(0xffffffffu, pos0, leader);
    if (pass) {
      const int32_t key = d.key[row];
      const int32_t pay = d.payload ? d.payload[row] : 0;
      if (d.bitmap) {
        // perfect hash over the key range: set the member bit, store the payload
        const uint32_t off = (uint32_t)key - (uint32_t)d.kmin;  // < nbits by the column statistics
        if (off < d.nbits) {
          const uint32_t old = atomicOr(d.bitmap + (off >> 5), 1u << (off & 31));
          if ((old >> (off & 31)) & 1u) atomicCAS(&m->err, 0, 2);  // duplicate key (BuildError)
          if (d.payarr) d.payarr[off] = pay;
        }
      } else {
        const int pos = pos0 + __popc(bal & lanemask_lt());
        d.compact[pos] = make_int2(key, pay);
      }
    }
  }
}

__global__ void dim_init_kernel(const DimBuildArgs a) {
  const DimBuildDesc& d = a.d[blockIdx.y];
  HtMeta* m = a.meta + blockIdx.y;
  if (d.bitmap) return;  // perfect-hash layout needs no slot table
  const int64_t n = m->count;
  int64_t cap = 2;
  while (cap < 2 * n) cap <<= 1;  // max(2, bit_ceil(2n))
  if (cap > d.maxcap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) m->err = 3;
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    m->mask = (uint32_t)(cap - 1);
    m->shift = 32 - (63 - __clzll((unsigned long long)cap));
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap;
       i += (int64_t)gridDim.x * blockDim.x)
    d.slots[i] = make_int2(kEmptyKey, 0);
}

__global__ void dim_insert_kernel(const DimBuildArgs a) {
  const DimBuildDesc& d = a.d[blockIdx.y];
  HtMeta* m = a.meta + blockIdx.y;
  if (d.bitmap) return;
  const int64_t n = m->count;
  if (m->err) return;
  const uint32_t mask = m->mask;
  const int shift = m->shift;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int2 e = d.compact[i];
    ht_insert(d.slots, mask, shift, e.x, e.y, &m->err);
  }
}

// ---------------------------------------------------------- fused pipelines

template <int BT, class T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  v = warp_sum(v);
  const unsigned warp = threadIdx.x >> 5;
  if (lane_id() == 0) red[warp] = v;
  __syncthreads();
  T s = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < BT / 32; ++w) s += red[w];
  __syncthreads();
  return s;  // valid in thread 0
}

// One join of the pipeline (BlockProbeHashTable).  When the dimension key
// column has a compact value range the build uses the perfect-hash layout of
// the Crystal paper's SSB kernels: an exact membership bitmap over
// [kmin, kmin+nbits) plus a payload array indexed by key - kmin, so a probe is
// one bit test (+ one payload load for members).  Otherwise the build is the
// reference's linear-probing table and every probe walks it
// (hash_table.hpp:41-51).  `bm` is the bitmap (a shared-memory copy for the
// first join when staged).
template <int IPT>
__device__ __forceinline__ void probe_join(const JoinDesc& jd, const uint32_t* bm, bool bm_smem,
                                           uint32_t mask, int shift, const int32_t (&key)[IPT],
                                           unsigned& f, int32_t (&pay)[IPT]) {
  if (bm) {
    const uint32_t kmin = (uint32_t)jd.kmin, nbits = jd.nbits;
    // Branch-free: every item issues its bitmap-word load (word 0 when out of
    // range or already dead) before any word is examined, so a thread keeps
    // IPT independent loads in flight.
    uint32_t off[IPT], w[IPT];
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      off[k] = (uint32_t)key[k] - kmin;  // bijective, so only [kmin, kmin+nbits) lands < nbits
      const bool in = ((f >> k) & 1u) && off[k] < nbits;
      f &= ~((unsigned)!in << k);
      const uint32_t wi = in ? (off[k] >> 5) : 0u;
      w[k] = bm_smem ? bm[wi] : __ldg(bm + wi);
    }
#pragma unroll
    for (int k = 0; k < IPT; ++k) f &= ~((((w[k] >> (off[k] & 31)) & 1u) ^ 1u) << k);
    if (jd.need_payload) {
#pragma unroll
      for (int k = 0; k < IPT; ++k)
        if ((f >> k) & 1u) pay[k] = __ldg(jd.payarr + off[k]);
    }
    return;
  }
  BlockProbeHashTable<IPT>(key, f, pay, jd.slots, mask, shift);
}

// Flight 1 (run_flight1, ssb_queries.cpp:157-210): three chained range
// predicates (INIT, AND, AND), SUM(extendedprice * discount) in 8 bytes.
template <int BT, int IPT>
__global__ void __launch_bounds__(BT) ssb_flight1_kernel(const FusedArgs a) {
  using L = VecLayout<BT, IPT>;
  __shared__ long long red[BT / 32];
  long long sum = 0;
  unsigned cnt = 0;
  const int64_t ntiles = (a.n + L::TILE - 1) / L::TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * L::TILE;
    const int valid = (int)min((int64_t)L::TILE, a.n - base);
    int32_t x[IPT], d[IPT], e[IPT];
    BlockLoad<BT, IPT>(a.fcol[0] + base, valid, x);
    unsigned f = BlockPred<IPT>(x, a.flo[0], a.fhi[0], BlockValidMask<BT, IPT>(valid));
    BlockLoadSel<BT, IPT>(a.fcol[1] + base, valid, f, d);
    f = BlockPredAnd<IPT>(d, a.flo[1], a.fhi[1], f);
    BlockLoadSel<BT, IPT>(a.fcol[2] + base, valid, f, x);
    f = BlockPredAnd<IPT>(x, a.flo[2], a.fhi[2], f);
    BlockLoadSel<BT, IPT>(a.agg_a + base, valid, f, e);
    if (!a.agg_b_is_f1) BlockLoadSel<BT, IPT>(a.agg_b + base, valid, f, d);
#pragma unroll
    for (int k = 0; k < IPT; ++k)
      if ((f >> k) & 1u) sum += (long long)e[k] * (long long)d[k];
    cnt += __popc(f);
  }
  const long long s = block_sum<BT>(sum, red);
  const long long c = block_sum<BT>((long long)cnt, red);
  if (threadIdx.x == 0) {
    atomicAdd(a.g_sum, (unsigned long long)s);
    atomicAdd(a.g_cnt, (unsigned long long)c);
    atomicAdd(a.surv, (unsigned long long)c);
  }
}

// Flights 2-4 (run_joins, ssb_queries.cpp:212-273).  NJ joins probed in plan
// order; AGG = revenue or revenue - supplycost; SMEM selects a CTA-private
// dense aggregate in shared memory (flushed once per CTA) vs global atomics.
template <int NJ, int AGG, bool SMEM, int BT, int IPT>
__global__ void __launch_bounds__(BT) ssb_join_kernel(const FusedArgs a) {
  using L = VecLayout<BT, IPT>;
  extern __shared__ unsigned long long s_dyn[];
  __shared__ unsigned long long red[BT / 32];
  unsigned long long* s_sum = s_dyn;
  unsigned* s_cnt = reinterpret_cast<unsigned*>(s_dyn + a.cells);

  uint32_t mask[NJ];
  int shift[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    mask[j] = a.meta[j].mask;
    shift[j] = a.meta[j].shift;
  }
  if constexpr (SMEM) {
    for (int c = threadIdx.x; c < a.cells; c += BT) {
      s_sum[c] = 0;
      s_cnt[c] = 0;
    }
    __syncthreads();
  }
  unsigned surv[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) surv[j] = 0;
  int bad = 0;

  const int64_t ntiles = (a.n + L::TILE - 1) / L::TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * L::TILE;
    const int valid = (int)min((int64_t)L::TILE, a.n - base);
    unsigned f = BlockValidMask<BT, IPT>(valid);
    int32_t key[IPT], pay[IPT], idx[IPT];
#pragma unroll
    for (int k = 0; k < IPT; ++k) idx[k] = 0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      if (j == 0)
        BlockLoad<BT, IPT>(a.j[0].fk + base, valid, key);
      else
        BlockLoadSel<BT, IPT>(a.j[j].fk + base, valid, f, key);
      probe_join<IPT>(a.j[j], a.j[j].bitmap, false, mask[j], shift[j], key, f, pay);
      if (a.j[j].gcard) {
        const int32_t glo = a.j[j].glo, gcard = a.j[j].gcard, gst = a.j[j].gstride;
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
          if ((f >> k) & 1u) {
            const int32_t u = pay[k] - glo;
            if ((uint32_t)u >= (uint32_t)gcard) bad = 1;  // ssb_queries.cpp:32-33
            idx[k] += u * gst;
          }
        }
      }
      surv[j] += __popc(f);
    }
    int32_t va[IPT], vb[IPT];
    BlockLoadSel<BT, IPT>(a.agg_a + base, valid, f, va);
    if constexpr (AGG == kAggRevenueMinusSupplyCost) BlockLoadSel<BT, IPT>(a.agg_b + base, valid, f, vb);
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      if ((f >> k) & 1u) {
        long long v = va[k];
        if constexpr (AGG == kAggRevenueMinusSupplyCost) v -= (long long)vb[k];
        const uint32_t c = (uint32_t)idx[k];
        if (c < (uint32_t)a.cells) {
          if constexpr (SMEM) {
            atomicAdd(&s_sum[c], (unsigned long long)v);
            atomicAdd(&s_cnt[c], 1u);
          } else {
            atomicAdd(&a.g_sum[c], (unsigned long long)v);
            atomicAdd(&a.g_cnt[c], 1ull);
          }
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const unsigned long long s = block_sum<BT>((unsigned long long)surv[j], red);
    if (threadIdx.x == 0 && s) atomicAdd(&a.surv[j], s);
  }
  if (bad) atomicExch(a.err, 2);
  if constexpr (SMEM) {
    __syncthreads();
    for (int c = threadIdx.x; c < a.cells; c += BT) {
      const unsigned n = s_cnt[c];
      if (n) {
        atomicAdd(&a.g_sum[c], s_sum[c]);
        atomicAdd(&a.g_cnt[c], (unsigned long long)n);
      }
    }
  }
}

// Occupied cells -> (cell, sum) rows (grouped_result, ssb_queries.cpp:145-155).
// Flight 1 always yields its single row (ssb_queries.cpp:207-209).
__global__ void finalize_kernel(const unsigned long long* sums, const unsigned long long* cnts,
                                int64_t cells, int flight1, ResultHeader* hdr, RowOut* rows,
                                const unsigned long long* surv, const int32_t* err,
                                const HtMeta* meta, int nj) {
  const unsigned lane = lane_id();
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // QueryStats + error words ride in the header
    for (int j = 0; j < 4; ++j) hdr->surv[j] = surv ? surv[j] : 0;
    hdr->err = err ? *err : 0;
    int e = 0;
    for (int j = 0; j < nj; ++j)
      if (meta[j].err) e = meta[j].err;
    hdr->ht_err = e;
  }
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < cells;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = base + threadIdx.x;
    const bool take = c < cells && (cnts[c] != 0 || (flight1 && c == 0));
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (!bal) continue;
    const int leader = __ffs(bal) - 1;
    unsigned long long p0 = 0;
    if ((int)lane == leader) p0 = atomicAdd(&hdr->nrows, (unsigned long long)__popc(bal));
    p0 = __shfl_sync(0xffffffffu, p0, leader);
    if (take) {
      RowOut r;
      r.cell = c;
      r.sum = (long long)sums[c];
      rows[p0 + __popc(bal & lanemask_lt())] = r;
    }
  }
}



// ---------------------------------------------------------- async-staged pipeline
// Native sm_100a form of the fused join flights.  Every warp runs its own
// software pipeline over "warp-tiles" of 32 x IPT rows: while it probes tile
// t, the referenced lineorder columns of its next D tiles are already in
// flight into a warp-private shared-memory ring through cp.async (LDGSTS,
// 16 B per lane per column, zero-filled past the shard end, L1 bypassed).
// Each lane reads back only the chunks it copied, so no warp/CTA barrier is
// needed per tile; warps drift freely and the SM always has D tiles per warp
// of HBM traffic outstanding.  The dependent chain left per tile is the
// dimension probes (shared-memory bitmap for the first join, L1/L2 for the
// rest), which the 16-32 resident warps per SM overlap.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int NJ, int AGG>
struct StagedCols {
  static constexpr int NC = NJ + (AGG == kAggRevenueMinusSupplyCost ? 2 : 1);
};

template <int NJ, int AGG, bool SMEM, int WARPS, int IPT, int D>
__global__ void __launch_bounds__(WARPS * 32) ssb_join_async_kernel(const FusedArgs a) {
  constexpr int NC = StagedCols<NJ, AGG>::NC;
  constexpr int WT = 32 * IPT;  // rows per warp-tile
  constexpr int NV = IPT / 4;   // 16 B chunks per lane per column
  static_assert(IPT % 4 == 0, "16-byte chunks");
  constexpr int SLOT = NC * WT;  // int32 per ring slot
  extern __shared__ unsigned long long s_dyn[];
  int32_t* s_ints = reinterpret_cast<int32_t*>(s_dyn);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  int32_t* ring = s_ints + (size_t)warp * (D + 1) * SLOT;
  unsigned long long* s_sum = reinterpret_cast<unsigned long long*>(s_ints + (size_t)WARPS * (D + 1) * SLOT);
  unsigned* s_cnt = reinterpret_cast<unsigned*>(s_sum + (SMEM ? a.cells : 0));
  uint32_t* s_bm = s_cnt + (SMEM ? a.cells : 0);

  const int bm_words = a.smem_bm_words;
  for (int i = threadIdx.x; i < bm_words; i += blockDim.x) s_bm[i] = __ldg(a.j[0].bitmap + i);
  if constexpr (SMEM) {
    for (int c = threadIdx.x; c < a.cells; c += blockDim.x) {
      s_sum[c] = 0;
      s_cnt[c] = 0;
    }
  }
  __syncthreads();

  const int32_t* cols[NC];
#pragma unroll
  for (int j = 0; j < NJ; ++j) cols[j] = a.j[j].fk;
  cols[NJ] = a.agg_a;
  if constexpr (NC > NJ + 1) cols[NJ + 1] = a.agg_b;
  uint32_t mask[NJ];
  int shift[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    mask[j] = a.meta[j].mask;
    shift[j] = a.meta[j].shift;
  }

  const int64_t nwt = (a.n + WT - 1) / WT;
  const int64_t tw = (int64_t)gridDim.x * WARPS;
  const int64_t t0 = (int64_t)blockIdx.x * WARPS + warp;

  auto issue = [&](int64_t t, int slot) {
    int32_t* dst = ring + slot * SLOT;
    const int64_t base = t * WT;
    if (base + WT <= a.n) {  // interior tile (warp-uniform): no bounds arithmetic
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int off = (v * 32 + lane) * 4;
          cp_async16(dst + c * WT + off, cols[c] + base + off, 16);
        }
      return;
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int off = (v * 32 + lane) * 4;
        const int64_t row = base + off;
        const int64_t rem = a.n - row;
        const int bytes = rem >= 4 ? 16 : (rem > 0 ? (int)rem * 4 : 0);
        cp_async16(dst + c * WT + off, cols[c] + (bytes ? row : 0), bytes);
      }
    }
  };

#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (t0 + d * tw < nwt) issue(t0 + d * tw, d);
    cp_async_commit();
  }

  unsigned surv[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) surv[j] = 0;
  int bad = 0;
  int it = 0;
  for (int64_t t = t0; t < nwt; t += tw, ++it) {
    const int64_t tn = t + (int64_t)D * tw;
    if (tn < nwt) issue(tn, (it + D) % (D + 1));
    cp_async_commit();
    cp_async_wait<D>();
    const int32_t* st = ring + (it % (D + 1)) * SLOT;
    const int64_t base = t * WT;
    const int valid = (int)min((int64_t)WT, a.n - base);
    unsigned f = (1u << IPT) - 1u;
    if (valid < WT) {
      f = 0;
#pragma unroll
      for (int k = 0; k < IPT; ++k) f |= (unsigned)(((k >> 2) * 32 + lane) * 4 + (k & 3) < valid) << k;
    }
    int32_t key[IPT], pay[IPT], idx[IPT];
#pragma unroll
    for (int k = 0; k < IPT; ++k) idx[k] = 0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      if (f == 0) break;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int4 x = *reinterpret_cast<const int4*>(st + j * WT + (v * 32 + lane) * 4);
        key[v * 4 + 0] = x.x; key[v * 4 + 1] = x.y; key[v * 4 + 2] = x.z; key[v * 4 + 3] = x.w;
      }
      if (j == 0 && bm_words)
        probe_join<IPT>(a.j[0], s_bm, true, mask[0], shift[0], key, f, pay);
      else
        probe_join<IPT>(a.j[j], a.j[j].bitmap, false, mask[j], shift[j], key, f, pay);
      if (a.j[j].gcard) {
        const int32_t glo = a.j[j].glo, gcard = a.j[j].gcard, gst = a.j[j].gstride;
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
          if ((f >> k) & 1u) {
            const int32_t u = pay[k] - glo;
            if ((uint32_t)u >= (uint32_t)gcard) bad = 1;
            idx[k] += u * gst;
          }
        }
      }
      surv[j] += __popc(f);
    }
    if (f) {
#pragma unroll
      for (int k = 0; k < IPT; ++k) {
        if ((f >> k) & 1u) {
          const int o = ((k >> 2) * 32 + lane) * 4 + (k & 3);
          long long v = st[NJ * WT + o];
          if constexpr (AGG == kAggRevenueMinusSupplyCost) v -= (long long)st[(NJ + 1) * WT + o];
          const uint32_t c = (uint32_t)idx[k];
          if (c < (uint32_t)a.cells) {
            if constexpr (SMEM) {
              atomicAdd(&s_sum[c], (unsigned long long)v);
              atomicAdd(&s_cnt[c], 1u);
            } else {
              atomicAdd(&a.g_sum[c], (unsigned long long)v);
              atomicAdd(&a.g_cnt[c], 1ull);
            }
          }
        }
      }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const unsigned long long w = warp_sum((unsigned long long)surv[j]);
    if (lane == 0 && w) atomicAdd(&a.surv[j], w);
  }
  if (bad) atomicExch(a.err, 2);
  if constexpr (SMEM) {
    __syncthreads();
    for (int c = threadIdx.x; c < a.cells; c += blockDim.x) {
      const unsigned n = s_cnt[c];
      if (n) {
        atomicAdd(&a.g_sum[c], s_sum[c]);
        atomicAdd(&a.g_cnt[c], (unsigned long long)n);
      }
    }
  }
}

template <int NJ, int AGG, int WARPS, int IPT, int D>
size_t staged_smem(bool smem_agg, int64_t cells, int bm_words) {
  return sizeof(int32_t) * (size_t)WARPS * (D + 1) * StagedCols<NJ, AGG>::NC * 32 * IPT +
         (smem_agg ? (size_t)cells * 12 : 0) + sizeof(uint32_t) * (size_t)bm_words;
}

// ---------------------------------------------------------- dispatch tables

#define CRYS_SSB_SHAPES(X) X(128, 4) X(256, 16) X(128, 16) X(512, 8)
constexpr int kNativeBT = 256, kNativeIPT = 16;  // flight 1 fallback shape

using KernelFn = void (*)(const FusedArgs);

template <int BT, int IPT>
KernelFn pick_kernel(int njoins, int agg, bool smem) {
  if (njoins == 0) return ssb_flight1_kernel<BT, IPT>;
  if (njoins == 3 && agg == kAggRevenue)
    return smem ? ssb_join_kernel<3, kAggRevenue, true, BT, IPT>
                : ssb_join_kernel<3, kAggRevenue, false, BT, IPT>;
  if (njoins == 4 && agg == kAggRevenueMinusSupplyCost)
    return smem ? ssb_join_kernel<4, kAggRevenueMinusSupplyCost, true, BT, IPT>
                : ssb_join_kernel<4, kAggRevenueMinusSupplyCost, false, BT, IPT>;
  fail(CRYS_ENOTBUILT, "no fused kernel for this plan shape");
}

struct Launch {
  KernelFn fn;
  int bt, ipt;
};

Launch select_kernel(int bt, int ipt, int njoins, int agg, bool smem) {
#define X(B, I) \
  if (bt == B && ipt == I) return {pick_kernel<B, I>(njoins, agg, smem), B, I};
  CRYS_SSB_SHAPES(X)
#undef X
  // Results are tile-invariant (test_ssb.cpp:251-261), so an uncompiled but
  // valid TileConfig runs the native sm_100a shape.
  return {pick_kernel<kNativeBT, kNativeIPT>(njoins, agg, smem), kNativeBT, kNativeIPT};
}

int blocks_per_sm(crys_ctx* ctx, KernelFn fn, int bt, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, size_t>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair((const void*)fn, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  ensure_dyn_smem((const void*)fn, smem);
  int nb = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, bt, smem));
  if (nb < 1) nb = 1;
  cache[key] = nb;
  (void)ctx;
  return nb;
}

template <int NJ, int AGG, int WARPS, int IPT, int D>
void launch_staged(crys_ctx* ctx, FusedArgs fa, bool smem_agg, int64_t cells, int64_t n,
                   const std::string& name) {
  if (smem_agg && staged_smem<NJ, AGG, WARPS, IPT, D>(true, cells, fa.smem_bm_words) > 227 * 1024)
    smem_agg = false;  // the CTA-private table does not fit: global atomics
  KernelFn fn = smem_agg ? ssb_join_async_kernel<NJ, AGG, true, WARPS, IPT, D>
                         : ssb_join_async_kernel<NJ, AGG, false, WARPS, IPT, D>;
  const int threads = WARPS * 32;
  size_t dyn = staged_smem<NJ, AGG, WARPS, IPT, D>(smem_agg, cells, fa.smem_bm_words);
  if (dyn > 200 * 1024 && fa.smem_bm_words) {  // no room to stage the first bitmap
    fa.smem_bm_words = 0;
    dyn = staged_smem<NJ, AGG, WARPS, IPT, D>(smem_agg, cells, 0);
  }
  CRYS_CHECK(dyn <= 227 * 1024, CRYS_ENOTBUILT, "staged pipeline exceeds shared memory");
  ensure_dyn_smem((const void*)fn, dyn);
  const int nb = blocks_per_sm(ctx, fn, threads, dyn);
  const int64_t wt = 32 * IPT;
  const int64_t nwt = (n + wt - 1) / wt;
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((nwt + WARPS - 1) / WARPS, (int64_t)nb * ctx->num_sms));
  fn<<<grid, threads, dyn, ctx->stream>>>(fa);
  CRYS_LAUNCHED(std::string("fused-staged ") + name + " grid=" + std::to_string(grid) + " smem=" +
                std::to_string(dyn));
}

template <int NJ, int AGG>
void launch_staged_cfg(crys_ctx* ctx, const FusedArgs& fa, bool smem_agg, int64_t cells, int64_t n,
                       const std::string& name) {
  static const int cfg = [] {
    const char* e = getenv("CRYS_STAGED_CFG");  // tuning knob
    return e ? atoi(e) : 5;
  }();
  switch (cfg) {
    case 1: launch_staged<NJ, AGG, 8, 4, 1>(ctx, fa, smem_agg, cells, n, name); break;
    case 2: launch_staged<NJ, AGG, 8, 8, 1>(ctx, fa, smem_agg, cells, n, name); break;
    case 3: launch_staged<NJ, AGG, 16, 4, 2>(ctx, fa, smem_agg, cells, n, name); break;
    case 4: launch_staged<NJ, AGG, 4, 4, 3>(ctx, fa, smem_agg, cells, n, name); break;
    case 5: launch_staged<NJ, AGG, 32, 4, 1>(ctx, fa, smem_agg, cells, n, name); break;
    case 6: launch_staged<NJ, AGG, 16, 4, 1>(ctx, fa, smem_agg, cells, n, name); break;
    default: launch_staged<NJ, AGG, 8, 4, 2>(ctx, fa, smem_agg, cells, n, name); break;
  }
}

}  // namespace

// ---------------------------------------------------------- workspace

struct QueryWorkspace {
  DevBuf agg;      // u64 [2*cells]
  DevBuf counters; // u64 surv[4] + i32 err
  DevBuf meta;     // HtMeta[4]
  DevBuf slots[kMaxJoins];
  DevBuf compact[kMaxJoins];
  DevBuf bitmap;   // membership bitmaps of all joins, contiguous (one memset)
  DevBuf payarr[kMaxJoins];  // perfect-hash payload arrays
  DevBuf result;   // ResultHeader + RowOut[cells]
  PinnedBuf host;
};

void WsDeleter::operator()(QueryWorkspace* p) const { delete p; }

static QueryWorkspace& ws_of(crys_ctx* ctx) {
  if (!ctx->qws) ctx->qws.reset(new QueryWorkspace());
  return *ctx->qws;
}

static int64_t bit_ceil64(int64_t v) {
  int64_t c = 1;
  while (c < v) c <<= 1;
  return c;
}

void ssb_query_partial(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt,
                       unsigned long long* d_agg, unsigned long long* d_surv, int32_t* d_err) {
  const QueryPlan& plan = plan_for(qid);
  CRYS_CHECK(bt > 0 && ipt > 0, CRYS_ECONFIG, "TileConfig: block_threads/items_per_thread must be positive");
  QueryWorkspace& ws = ws_of(ctx);
  cudaStream_t st = ctx->stream;
  const int nj = (int)plan.joins.size();
  const int64_t cells = plan.cells();

  int64_t n = 0;
  const std::string& first_col = nj ? plan.joins[0].fact_key : plan.fact_filters[0].column;
  db->col("lineorder", first_col, &n);

  FusedArgs fa;
  std::memset(&fa, 0, sizeof(fa));
  fa.n = n;
  fa.cells = (int32_t)cells;
  fa.g_sum = d_agg;
  fa.g_cnt = d_agg + cells;
  fa.surv = d_surv;
  fa.err = d_err;

  ws.meta.reserve(sizeof(HtMeta) * kMaxJoins);
  fa.meta = ws.meta.as<HtMeta>();

  if (nj) {
    // ---- dimension builds (build_dim_table, ssb_queries.cpp:99-121)
    DimBuildArgs da;
    std::memset(&da, 0, sizeof(da));
    da.meta = ws.meta.as<HtMeta>();
    int64_t max_rows = 0, max_cap = 0;
    for (int j = 0; j < nj; ++j) {
      const DimJoin& dj = plan.joins[j];
      DimBuildDesc& d = da.d[j];
      int64_t rows = 0;
      d.key = db->col(dj.dim_table, dj.dim_key, &rows);
      d.rows = rows;
      d.payload = dj.payload.empty() ? nullptr : db->col(dj.dim_table, dj.payload, &rows);
      CRYS_CHECK((int)dj.filters.size() <= 2, CRYS_ENOTBUILT, "at most two filters per join");
      d.nf = (int)dj.filters.size();
      for (int f = 0; f < d.nf; ++f) {
        d.fcol[f] = db->col(dj.dim_table, dj.filters[f].column, &rows);
        CRYS_CHECK(dj.filters[f].ranges.size() <= 2, CRYS_ENOTBUILT, "at most two ranges per filter");
        d.nranges[f] = (int)dj.filters[f].ranges.size();
        for (int r = 0; r < d.nranges[f]; ++r) {
          d.r[f][r][0] = dj.filters[f].ranges[r].first;
          d.r[f][r][1] = dj.filters[f].ranges[r].second;
        }
      }
      d.maxcap = std::max<int64_t>(2, bit_ceil64(2 * d.rows));
      ws.slots[j].reserve(sizeof(int2) * d.maxcap);
      ws.compact[j].reserve(sizeof(int2) * std::max<int64_t>(1, d.rows));
      d.slots = ws.slots[j].as<int2>();
      d.compact = ws.compact[j].as<int2>();
      max_rows = std::max(max_rows, d.rows);
      max_cap = std::max(max_cap, d.maxcap);

      JoinDesc& jd = fa.j[j];
      jd.fk = db->col("lineorder", dj.fact_key, &rows);
      CRYS_CHECK(rows == n, CRYS_ECONTRACT, "lineorder columns of different length");
      jd.slots = d.slots;
    }
    // exact key-range membership bitmaps (dimension key statistics permitting)
    constexpr int64_t kMaxBitmapBits = int64_t(1) << 25;  // 4 MB bitmap / 128 MB payloads per join
    int64_t words_total = 0, word_off[kMaxJoins] = {0, 0, 0, 0};
    for (int j = 0; j < nj; ++j) {
      const DimJoin& dj = plan.joins[j];
      int32_t lo = 0, hi = -1;
      word_off[j] = -1;
      if (db->col_range(dj.dim_table, dj.dim_key, &lo, &hi) && (int64_t)hi - lo + 1 <= kMaxBitmapBits) {
        da.d[j].kmin = lo;
        da.d[j].nbits = (uint32_t)((int64_t)hi - lo + 1);
        word_off[j] = words_total;
        words_total += (da.d[j].nbits + 31) / 32 + 4;  // keep each bitmap 16 B aligned
      }
    }
    if (words_total) {
      ws.bitmap.reserve(sizeof(uint32_t) * (size_t)words_total);
      CUDA_TRY(cudaMemsetAsync(ws.bitmap.p, 0, sizeof(uint32_t) * (size_t)words_total, st));
    }
    bool any_ht = false;
    for (int j = 0; j < nj; ++j) {
      if (word_off[j] < 0) {
        any_ht = true;
        continue;
      }
      da.d[j].bitmap = ws.bitmap.as<uint32_t>() + word_off[j];
      fa.j[j].bitmap = da.d[j].bitmap;
      fa.j[j].kmin = da.d[j].kmin;
      fa.j[j].nbits = da.d[j].nbits;
      if (!plan.joins[j].payload.empty()) {
        ws.payarr[j].reserve(sizeof(int32_t) * da.d[j].nbits);
        da.d[j].payarr = ws.payarr[j].as<int32_t>();
        fa.j[j].payarr = da.d[j].payarr;
      }
    }
    for (int j = 0; j < nj; ++j) fa.j[j].need_payload = !plan.joins[j].payload.empty();
    if (fa.j[0].bitmap) {
      const int64_t w0 = (fa.j[0].nbits + 31) / 32;
      fa.smem_bm_words = w0 <= 12288 ? (int32_t)w0 : 0;  // <= 48 KB of shared memory
    }
    // group parts -> (join, lo, card, stride): mixed radix, last part fastest
    int64_t stride = 1;
    for (int g = (int)plan.group.size() - 1; g >= 0; --g) {
      const GroupPart& gp = plan.group[g];
      JoinDesc& jd = fa.j[gp.join_index];
      CRYS_CHECK(jd.gcard == 0, CRYS_ENOTBUILT, "one group part per join payload");
      jd.glo = gp.lo;
      jd.gcard = gp.hi - gp.lo + 1;
      jd.gstride = (int32_t)stride;
      stride *= (int64_t)(gp.hi - gp.lo + 1);
    }
    CUDA_TRY(cudaMemsetAsync(ws.meta.p, 0, sizeof(HtMeta) * kMaxJoins, st));
    const int tpb = 256;
    const int gx_rows = (int)std::min<int64_t>((max_rows + tpb - 1) / tpb, (int64_t)ctx->num_sms * 8);
    const int gx_cap = (int)std::min<int64_t>((max_cap + tpb - 1) / tpb, (int64_t)ctx->num_sms * 8);
    dim_filter_kernel<<<dim3(std::max(gx_rows, 1), nj), tpb, 0, st>>>(da);
    CRYS_LAUNCHED("dim_filter_kernel");
    count_launch(ctx);
    if (any_ht) {  // linear-probing builds (hash_table.cpp:20-94) for sparse key domains
      dim_init_kernel<<<dim3(std::max(gx_cap, 1), nj), tpb, 0, st>>>(da);
      CRYS_LAUNCHED("dim_init_kernel");
      dim_insert_kernel<<<dim3(std::max(gx_rows, 1), nj), tpb, 0, st>>>(da);
      CRYS_LAUNCHED("dim_insert_kernel");
      count_launch(ctx, 2);
    }
  } else {
    int64_t rows = 0;
    for (int f = 0; f < 3; ++f) {
      fa.fcol[f] = db->col("lineorder", plan.fact_filters[f].column, &rows);
      CRYS_CHECK(rows == n, CRYS_ECONTRACT, "lineorder columns of different length");
      fa.flo[f] = plan.fact_filters[f].lo;
      fa.fhi[f] = plan.fact_filters[f].hi;
    }
  }
  // aggregate columns (agg_fact_columns, ssb_plans.cpp:287-299)
  int64_t rows = 0;
  if (plan.agg == kAggExtPriceTimesDiscount) {
    fa.agg_a = db->col("lineorder", "lo_extendedprice", &rows);
    fa.agg_b = db->col("lineorder", "lo_discount", &rows);
    fa.agg_b_is_f1 = plan.fact_filters.size() > 1 && plan.fact_filters[1].column == "lo_discount";
  } else {
    fa.agg_a = db->col("lineorder", "lo_revenue", &rows);
    if (plan.agg == kAggRevenueMinusSupplyCost) fa.agg_b = db->col("lineorder", "lo_supplycost", &rows);
  }

  const size_t smem_bytes = (size_t)cells * 12;
  static const size_t smem_max = [] {
    const char* e = getenv("CRYS_SMEM_AGG_MAX");  // tuning knob (bytes)
    return e ? (size_t)atoll(e) : (size_t)64 * 1024;
  }();
  const bool smem = nj > 0 && smem_bytes <= smem_max;
  // The join flights run the async-staged pipeline (its warp-tile shape is
  // fixed; results are tile-invariant, test_ssb.cpp:251-261).  The register-
  // tile Crystal kernels remain reachable for ablation with
  // CRYS_SSB_JOIN_KERNEL=register (TileConfig then picks the instantiation).
  static const bool register_tiles = [] {
    const char* e = getenv("CRYS_SSB_JOIN_KERNEL");
    return e && std::string(e) == "register";
  }();
  if (nj > 0 && !register_tiles) {
    timing_kernel_begin(ctx);
    if (nj == 3 && plan.agg == kAggRevenue)
      launch_staged_cfg<3, kAggRevenue>(ctx, fa, smem, cells, n, plan.name);
    else if (nj == 4 && plan.agg == kAggRevenueMinusSupplyCost)
      launch_staged_cfg<4, kAggRevenueMinusSupplyCost>(ctx, fa, smem, cells, n, plan.name);
    else
      fail(CRYS_ENOTBUILT, "no staged pipeline for this plan shape");
    timing_kernel_end(ctx);
    count_launch(ctx);
    return;
  }
  Launch L = select_kernel(bt, ipt, nj, plan.agg, smem);
  const size_t dyn = smem ? smem_bytes : 0;
  const int nb = blocks_per_sm(ctx, L.fn, L.bt, dyn);
  const int64_t ntiles = (n + (int64_t)L.bt * L.ipt - 1) / ((int64_t)L.bt * L.ipt);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)nb * ctx->num_sms));
  timing_kernel_begin(ctx);
  L.fn<<<grid, L.bt, dyn, st>>>(fa);
  CRYS_LAUNCHED(std::string("fused ") + plan.name + " bt=" + std::to_string(L.bt) + " ipt=" +
                std::to_string(L.ipt) + " grid=" + std::to_string(grid) + " smem=" + std::to_string(dyn));
  timing_kernel_end(ctx);
  count_launch(ctx);
}

static void finalize_impl(crys_ctx* ctx, int qid, const unsigned long long* d_agg,
                          const unsigned long long* d_surv, const int32_t* d_err, ResultRows* out) {
  const QueryPlan& plan = plan_for(qid);
  QueryWorkspace& ws = ws_of(ctx);
  cudaStream_t st = ctx->stream;
  const int64_t cells = plan.cells();
  ws.result.reserve(sizeof(ResultHeader) + sizeof(RowOut) * (size_t)cells);
  ResultHeader* hdr = ws.result.as<ResultHeader>();
  RowOut* rows = reinterpret_cast<RowOut*>(hdr + 1);
  CUDA_TRY(cudaMemsetAsync(hdr, 0, sizeof(ResultHeader), st));
  const int tpb = 256;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((cells + tpb - 1) / tpb, (int64_t)ctx->num_sms * 8));
  finalize_kernel<<<grid, tpb, 0, st>>>(d_agg, d_agg + cells, cells, plan.joins.empty() ? 1 : 0, hdr,
                                        rows, d_surv, d_err, ws.meta.as<HtMeta>(),
                                        d_surv ? (int)plan.joins.size() : 0);
  CRYS_LAUNCHED("finalize_kernel");
  count_launch(ctx);
  const int64_t first = std::min<int64_t>(cells, 2048);
  const size_t first_bytes = sizeof(ResultHeader) + sizeof(RowOut) * (size_t)first;
  ws.host.reserve(sizeof(ResultHeader) + sizeof(RowOut) * (size_t)cells);
  CUDA_TRY(cudaMemcpyAsync(ws.host.p, hdr, first_bytes, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const ResultHeader* h = ws.host.as<ResultHeader>();
  const int64_t nrows = (int64_t)h->nrows;
  if (nrows > first) {
    CUDA_TRY(cudaMemcpyAsync(ws.host.as<char>() + first_bytes, rows + first,
                             sizeof(RowOut) * (size_t)(nrows - first), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  for (int j = 0; j < 4; ++j) out->survivors[j] = (int64_t)h->surv[j];
  out->err = h->err;
  const int32_t ht_err = h->ht_err;
  const RowOut* hr = reinterpret_cast<const RowOut*>(h + 1);
  std::vector<std::pair<int64_t, int64_t>> v((size_t)nrows);
  for (int64_t i = 0; i < nrows; ++i) v[(size_t)i] = {hr[i].cell, hr[i].sum};
  std::sort(v.begin(), v.end());  // ascending mixed-radix index = lexicographic
  out->cell.resize((size_t)nrows);
  out->sum.resize((size_t)nrows);
  for (int64_t i = 0; i < nrows; ++i) {
    out->cell[(size_t)i] = v[(size_t)i].first;
    out->sum[(size_t)i] = v[(size_t)i].second;
  }
  if (ht_err == 1) fail(CRYS_EBUILD, "HashTable: key equals empty sentinel");
  if (ht_err == 2) fail(CRYS_EBUILD, "HashTable: duplicate key");
  if (ht_err == 3) fail(CRYS_EBUILD, "HashTable: capacity overflow");
  if (out->err) fail(CRYS_ECONTRACT, "group value outside its declared domain");
}

void ssb_finalize_device(crys_ctx* ctx, int qid, const unsigned long long* d_agg,
                         ResultRows* out) {
  ws_of(ctx).meta.reserve(sizeof(HtMeta) * kMaxJoins);
  finalize_impl(ctx, qid, d_agg, nullptr, nullptr, out);
}

void ssb_run_query(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt, ResultRows* out) {
  const QueryPlan& plan = plan_for(qid);
  QueryWorkspace& ws = ws_of(ctx);
  cudaStream_t st = ctx->stream;
  const int64_t cells = plan.cells();
  ws.agg.reserve(sizeof(unsigned long long) * 2 * (size_t)cells);
  ws.counters.reserve(64);
  timing_begin(ctx);
  CUDA_TRY(cudaMemsetAsync(ws.agg.p, 0, sizeof(unsigned long long) * 2 * (size_t)cells, st));
  CUDA_TRY(cudaMemsetAsync(ws.counters.p, 0, 64, st));
  auto* agg = ws.agg.as<unsigned long long>();
  auto* surv = ws.counters.as<unsigned long long>();
  auto* err = reinterpret_cast<int32_t*>(surv + 4);
  ssb_query_partial(ctx, db, qid, bt, ipt, agg, surv, err);
  finalize_impl(ctx, qid, agg, surv, err, out);
  timing_end(ctx);
}

}  // namespace crys
