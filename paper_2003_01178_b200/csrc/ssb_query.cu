// ssb_query.cu -- fused Star Schema Benchmark pipelines on sm_100a.
//
// Replaces run_query / run_flight1 / run_joins / build_dim_table /
// AggregateTable / grouped_result of the reference (ssb_queries.cpp:15-286).
// Per query, all on the context's stream with ONE host synchronisation:
//   1. query_prologue_kernel  zeroes the dense aggregate, the counters, the
//                             result header and every dimension table
//   2. dim_filter_kernel      build_dim_table (ssb_queries.cpp:99-121) for all
//                             joins at once (grid.y = join): filter the
//                             dimension and insert the survivors into its
//                             probe table (perfect hash over the dense key
//                             range; linear-probing table otherwise, then
//                             dim_init_kernel + dim_insert_kernel)
//   3. the fused lineorder pass (the hot loop, ssb_queries.cpp:181-201 /
//      233-263):  flight 1 -> ssb_flight1_kernel (register tiles, chained
//      predicates, selective loads);  flights 2-4 -> ssb_pipeline_kernel
//      (TMA/mbarrier ring, dense first probe, compacted sparse tail,
//      ssb_pipeline.cuh)
//   4. finalize_kernel        compacts occupied cells (occupancy, not
//                             sum != 0: ssb_queries.cpp:32-35) + QueryStats +
//                             error words into one buffer; one D2H copy
//                             returns it and the host orders rows by cell
//                             index = lexicographic group order (:153).
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "crystal.cuh"
#include "internal.hpp"
#include "ssb_gather.cuh"
#include "ssb_pipeline.cuh"
#include "ssb_scan.cuh"
#include "ssb_scanbm.cuh"

namespace crys {

namespace {

using pipe::ProbeTab;
using pipe::kTabBitmap;
using pipe::kTabU8;
using pipe::kTabU16;
using pipe::kTabHash;

constexpr int kMaxJoins = 4;

struct DimBuildDesc {
  const int32_t* key;
  const int32_t* payload;  // null: payload 0 (ssb_queries.cpp:116)
  const int32_t* fcol[2];
  int32_t nranges[2];
  int32_t r[2][2][2];
  int32_t nf;
  int32_t kind;            // pipe::TabKind of the probe table
  int64_t rows;
  void* tbl;               // bitmap words / u8 codes / u16 codes
  uint32_t kmin, nkeys;    // key domain of the direct tables
  int32_t glo, gcard;      // group part fed by the payload (gcard 0: none)
  int64_t maxcap;          // kTabHash: slot capacity bound
  int2* compact;           // kTabHash: filtered {key, digit}
  int2* slots;             // kTabHash: linear-probing slots
  uint32_t clear_words;    // 32-bit words of the table to clear
  uint32_t clear_value;    // 0 (bitmap) or 0xFFFFFFFF (codes: all absent)
  uint32_t* bits;          // code tables: the membership bitmap beside them (late-materialising plans)
};

struct DimBuildArgs {
  DimBuildDesc d[kMaxJoins];
  HtMeta* meta;
  int32_t cta0[kMaxJoins + 1];  // dim_filter_kernel: CTAs [cta0[j], cta0[j+1]) build dimension j
};

struct PrologueArgs {
  DimBuildArgs* unused;
  uint32_t* tbl[2 * kMaxJoins];  // probe tables, then the membership bitmaps of code tables
  uint32_t words[2 * kMaxJoins];
  uint32_t value[2 * kMaxJoins];
  unsigned long long* zero64;  // aggregate [2*cells] + counters (may be null)
  int64_t zero64_n;
  unsigned long long* zero64b; // result header (may be null)
  int64_t zero64b_n;
  HtMeta* meta;
};

struct Flight1Args {
  int64_t n;
  const int32_t* fcol[3];
  int32_t flo[3], fhi[3];
  const int32_t* agg_a;
  const int32_t* agg_b;
  int32_t agg_b_is_f1;
  int32_t l2_ahead;  // ring kernel: L2 bulk-prefetch distance (tiles)
  unsigned long long* g_sum;
  unsigned long long* g_cnt;
  unsigned long long* surv;
};

struct ResultHeader {
  unsigned long long nrows;
  unsigned long long surv[4];
  int32_t err;     // rows that reached the aggregate with a group value outside its domain
  int32_t ht_err;  // first join (plan order) whose build failed: (join << 8) | code
  int32_t pad[4];
};
static_assert(sizeof(ResultHeader) == 64, "header is one 64 B line");

// The group-by sub-box a query can occupy (host-built plan part + the device
// digit extents in HtMeta): part g is fed by join `join[g]`, its full domain
// has fcard[g] values and mixed-radix stride fstride[g] (last part fastest).
enum BoxMode : int32_t { kBoxFull = 0, kBoxMeta = 1, kBoxExplicit = 2 };
struct BoxPlan {
  int32_t nparts;
  int32_t join[3];
  int32_t fcard[3];
  int32_t mode;            // BoxMode: whole domain / digit extents in HtMeta / xmin+xcard
  int32_t xmin[3], xcard[3];
  int64_t fstride[3];
};
struct BoxD {
  int32_t dmin[3], card[3];
  int64_t cells;
};

__device__ __forceinline__ BoxD box_of(const BoxPlan& p, const HtMeta* meta) {
  BoxD b;
  b.cells = 1;
  for (int g = 0; g < 3; ++g) {
    b.dmin[g] = 0;
    b.card[g] = 1;
    if (g >= p.nparts) continue;
    int32_t lo = 0, hi = p.fcard[g] - 1;
    if (p.mode == kBoxMeta) {
      const HtMeta& m = meta[p.join[g]];
      lo = max(lo, m.dmin);
      hi = min(hi, m.dmax);
    } else if (p.mode == kBoxExplicit) {
      lo = max(lo, p.xmin[g]);
      hi = min(hi, p.xmin[g] + p.xcard[g] - 1);
    }
    b.dmin[g] = lo;
    b.card[g] = hi >= lo ? hi - lo + 1 : 0;
    b.cells *= b.card[g];
  }
  return b;
}

// box cell -> full mixed-radix cell index
__device__ __forceinline__ int64_t box_to_full(const BoxPlan& p, const BoxD& b, int64_t i) {
  int64_t full = 0;
  for (int g = p.nparts - 1; g >= 0; --g) {
    const int64_t d = i % b.card[g];
    i /= b.card[g];
    full += (b.dmin[g] + d) * p.fstride[g];
  }
  return full;
}

struct RowOut {
  long long cell;
  long long sum;
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------- prologue

__global__ void query_prologue_kernel(const PrologueArgs a) {
  pdl_trigger();
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int j = 0; j < 2 * kMaxJoins; ++j) {
    uint32_t* t = a.tbl[j];
    if (!t) continue;
    const uint32_t v = a.value[j];
    for (int64_t i = tid; i < a.words[j]; i += stride) t[i] = v;
  }
  for (int64_t i = tid; i < a.zero64_n; i += stride) a.zero64[i] = 0;
  for (int64_t i = tid; i < a.zero64b_n; i += stride) a.zero64b[i] = 0;
  if (tid < kMaxJoins) a.meta[tid] = HtMeta{0, 0u, 0, 0, INT_MAX, INT_MIN, {0, 0}};
}

// ---------------------------------------------------------- dimension builds

// group digit of a dimension row's payload: payload - lo, or "bad" when it
// falls outside the declared domain (the reference throws only if such a
// row reaches the aggregate, ssb_queries.cpp:32-33)
__device__ __forceinline__ int32_t digit_of(const DimBuildDesc& d, int32_t pay) {
  if (d.gcard == 0) return 0;
  const int32_t u = pay - d.glo;
  return (uint32_t)u < (uint32_t)d.gcard ? u : -1;
}

// claim byte/half `off` of a code table: absent (all ones) -> code with ONE
// atomicAnd (clearing the bits that are 0 in the code); anything but all ones
// before is a duplicate key (BuildError, hash_table.cpp:51-93) -- the table
// content no longer matters once the build has failed.
template <int BITS>
__device__ __forceinline__ bool claim_code(void* tbl, uint32_t off, uint32_t code) {
  constexpr uint32_t kMask = (1u << BITS) - 1u;
  constexpr uint32_t kPer = 32 / BITS;
  uint32_t* w = reinterpret_cast<uint32_t*>(tbl) + off / kPer;
  const unsigned sh = (off % kPer) * BITS;
  const uint32_t old = atomicAnd(w, ~((~code & kMask) << sh));
  return ((old >> sh) & kMask) == kMask;
}

// Warp-aggregated forms for a warp whose lanes hold the consecutive offsets
// off0 .. off0 + 31 (lane l: off0 + l).  warp_bitmap_or sets the bits of the
// lanes in `bal` with at most two atomics and returns, per lane, whether its
// bit was already set.
__device__ __forceinline__ bool warp_bitmap_or(uint32_t* bm, uint32_t off0, unsigned bal, unsigned lane) {
  const uint32_t w0 = off0 >> 5, s = off0 & 31u;
  const uint32_t lo = bal << s, hi = s ? bal >> (32u - s) : 0u;
  uint32_t o0 = 0, o1 = 0;
  if (lane == 0) {
    if (lo) o0 = atomicOr(bm + w0, lo);
    if (hi) o1 = atomicOr(bm + w0 + 1, hi);
  }
  o0 = __shfl_sync(0xffffffffu, o0, 0);
  o1 = __shfl_sync(0xffffffffu, o1, 0);
  const uint32_t p = s + lane;
  return (((p < 32u ? o0 : o1) >> (p & 31u)) & 1u) != 0u;
}

// claim_code for the lanes with `pass`, off0 aligned to the codes per word:
// the lanes sharing a word AND their masks together, one atomic per word.
template <int BITS>
__device__ __forceinline__ bool warp_claim_code(void* tbl, uint32_t off0, bool pass, uint32_t code, unsigned lane) {
  constexpr uint32_t kMask = (1u << BITS) - 1u;
  constexpr uint32_t kPer = 32 / BITS;
  const unsigned sh = (lane % kPer) * BITS;
  uint32_t m = pass ? ~((~code & kMask) << sh) : 0xffffffffu;
#pragma unroll
  for (uint32_t o = 1; o < kPer; o <<= 1) m &= __shfl_xor_sync(0xffffffffu, m, o);
  uint32_t old = 0xffffffffu;
  if (lane % kPer == 0 && m != 0xffffffffu)
    old = atomicAnd(reinterpret_cast<uint32_t*>(tbl) + off0 / kPer + lane / kPer, m);
  old = __shfl_sync(0xffffffffu, old, lane & ~(kPer - 1));
  return ((old >> sh) & kMask) == kMask;
}

// build_dim_table for every join at once (grid.y = join).  Each thread owns
// kDimU rows per pass and issues all of their column loads before any
// predicate is evaluated (one memory latency per pass, not one per column).
constexpr int kDimU = 2;
__global__ void __launch_bounds__(256) dim_filter_kernel(const DimBuildArgs a) {
  pdl_wait();  // the prologue cleared the tables
  pdl_trigger();
  // one 1-D grid over all dimensions, each sized by its own row count (a
  // uniform grid.y = join launched max-rows CTAs for the 2556-row date table too)
  int dj = 0;
#pragma unroll
  for (int j = 1; j < kMaxJoins; ++j)
    if ((int)blockIdx.x >= a.cta0[j]) dj = j;
  const int cta = (int)blockIdx.x - a.cta0[dj], nctas = a.cta0[dj + 1] - a.cta0[dj];
  const DimBuildDesc& d = a.d[dj];
  HtMeta* m = a.meta + dj;
  const unsigned lane = lane_id();
  // build size: per-warp atomics only where the compaction needs positions
  // (kTabHash); a direct table's count is never read, so none is kept (the
  // per-CTA adds to one address serialised in L2)
  __shared__ int s_dmin, s_dmax;
  if (threadIdx.x == 0) {
    s_dmin = INT_MAX;
    s_dmax = INT_MIN;
  }
  __syncthreads();
  int32_t dmin = INT_MAX, dmax = INT_MIN;  // digits of this thread's passing rows
  const bool hashed = d.kind == kTabHash;
  const int64_t span = (int64_t)blockDim.x * kDimU;
  // the filters as a fixed 2 x 2 table of inclusive ranges in registers
  // (an absent filter: one all-pass range; an absent range: an empty one),
  // so the per-row test is branch-free (the runtime-bounded loops over the
  // descriptor made the build instruction-bound: 70 % issue, ~200 per row)
  int32_t flo[2][2], fhi[2][2];
#pragma unroll
  for (int f = 0; f < 2; ++f)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const bool used = f < d.nf && r < d.nranges[f];
      const bool all = f >= d.nf && r == 0;
      flo[f][r] = used ? d.r[f][r][0] : (all ? INT_MIN : INT_MAX);
      fhi[f][r] = used ? d.r[f][r][1] : (all ? INT_MAX : INT_MIN);
    }
  const int64_t drows = d.rows;
  for (int64_t base = (int64_t)cta * span; base < drows; base += (int64_t)nctas * span) {
    int32_t fv[2][kDimU], key[kDimU], pay[kDimU];
#pragma unroll
    for (int u = 0; u < kDimU; ++u) {
      const int64_t row = base + u * blockDim.x + threadIdx.x;
      const bool in = row < d.rows;
#pragma unroll
      for (int f = 0; f < 2; ++f) fv[f][u] = (in && f < d.nf) ? __ldg(d.fcol[f] + row) : 0;
      key[u] = in ? __ldg(d.key + row) : 0;
      pay[u] = (in && d.payload) ? __ldg(d.payload + row) : 0;
    }
#pragma unroll
    for (int u = 0; u < kDimU; ++u) {
      const int64_t row = base + u * blockDim.x + threadIdx.x;
      bool pass = row < drows;
#pragma unroll
      for (int f = 0; f < 2; ++f)
        pass = pass && ((fv[f][u] >= flo[f][0] && fv[f][u] <= fhi[f][0]) ||
                        (fv[f][u] >= flo[f][1] && fv[f][u] <= fhi[f][1]));
      const unsigned bal = __ballot_sync(0xffffffffu, pass);
      if (bal == 0) continue;
      const int leader = __ffs(bal) - 1;
      int pos0 = 0;
      if (hashed) {  // (a direct table never reads its build count: no count kept for it)
        if ((int)lane == leader) pos0 = atomicAdd(&m->count, __popc(bal));
        pos0 = __shfl_sync(0xffffffffu, pos0, leader);
      }
      if (!hashed) {
        // a warp whose 32 rows carry 32 consecutive keys (every generated
        // dimension: key = row + 1) updates the direct table with one atomic
        // per bitmap word / per code word instead of one per row (the
        // per-row atomics serialised 32-way on the same word)
        const uint32_t off = (uint32_t)key[u] - d.kmin;
        const uint32_t off0 = __shfl_sync(0xffffffffu, off, 0);
        const bool dense = __all_sync(0xffffffffu, row < d.rows && off == off0 + lane) && off0 + 31u < d.nkeys;
        if (dense) {  // warp-uniform
          const int32_t dig = pass ? digit_of(d, pay[u]) : 0;
          if (pass && dig >= 0) {
            dmin = min(dmin, dig);
            dmax = max(dmax, dig);
          }
          bool dup;
          if (d.kind == kTabBitmap) dup = warp_bitmap_or(reinterpret_cast<uint32_t*>(d.tbl), off0, bal, lane);
          else if (d.kind == kTabU8 && (off0 & 3u) == 0)
            dup = !warp_claim_code<8>(d.tbl, off0, pass, dig < 0 ? pipe::kU8Bad : (uint32_t)dig, lane);
          else if (d.kind == kTabU16 && (off0 & 1u) == 0)
            dup = !warp_claim_code<16>(d.tbl, off0, pass, dig < 0 ? pipe::kU16Bad : (uint32_t)dig, lane);
          else
            dup = pass && !(d.kind == kTabU8 ? claim_code<8>(d.tbl, off, dig < 0 ? pipe::kU8Bad : (uint32_t)dig)
                                             : claim_code<16>(d.tbl, off, dig < 0 ? pipe::kU16Bad : (uint32_t)dig));
          if (d.bits) warp_bitmap_or(d.bits, off0, bal, lane);
          if (pass && dup) atomicCAS(&m->err, 0, 2);  // duplicate key (BuildError)
          continue;
        }
      }
      if (!pass) continue;
      const int32_t dig = digit_of(d, pay[u]);
      if (dig >= 0) {
        dmin = min(dmin, dig);
        dmax = max(dmax, dig);
      }
      if (hashed) {
        d.compact[pos0 + __popc(bal & lanemask_lt())] = make_int2(key[u], dig);
        continue;
      }
      const uint32_t off = (uint32_t)key[u] - d.kmin;  // < nkeys by the column statistics
      if (off >= d.nkeys) {
        atomicCAS(&m->err, 0, 4);  // statistics do not cover the key: cannot happen for valid stats
        continue;
      }
      bool ok;
      if (d.kind == kTabBitmap) {
        const uint32_t bit = 1u << (off & 31);
        ok = !(atomicOr(reinterpret_cast<uint32_t*>(d.tbl) + (off >> 5), bit) & bit);
      } else if (d.kind == kTabU8) {
        ok = claim_code<8>(d.tbl, off, dig < 0 ? pipe::kU8Bad : (uint32_t)dig);
      } else {
        ok = claim_code<16>(d.tbl, off, dig < 0 ? pipe::kU16Bad : (uint32_t)dig);
      }
      if (d.bits) atomicOr(d.bits + (off >> 5), 1u << (off & 31));
      if (!ok) atomicCAS(&m->err, 0, 2);  // duplicate key (BuildError)
    }
  }
  if (d.gcard) {  // warp, then CTA, then one global min/max per CTA
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dmin = min(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
      dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    if (lane == 0 && dmin <= dmax) {
      atomicMin(&s_dmin, dmin);
      atomicMax(&s_dmax, dmax);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_dmin <= s_dmax) {
      atomicMin(&m->dmin, s_dmin);
      atomicMax(&m->dmax, s_dmax);
    }
  }
}

__global__ void dim_init_kernel(const DimBuildArgs a) {
  pdl_wait();
  pdl_trigger();
  const DimBuildDesc& d = a.d[blockIdx.y];
  HtMeta* m = a.meta + blockIdx.y;
  if (d.kind != kTabHash) return;
  const int64_t n = m->count;
  int64_t cap = 2;
  while (cap < 2 * n) cap <<= 1;  // max(2, bit_ceil(2n)), ssb_queries.cpp:119
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
  pdl_wait();
  pdl_trigger();
  const DimBuildDesc& d = a.d[blockIdx.y];
  HtMeta* m = a.meta + blockIdx.y;
  if (d.kind != kTabHash) return;
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

// ---------------------------------------------------------- flight 1

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

// run_flight1 (ssb_queries.cpp:157-210): three chained range predicates
// (INIT, AND, AND), SUM(extendedprice * discount) in 8 bytes.  A later
// column is read only in vectors that still hold a live row (BlockLoadSel),
// so dead 32 B sectors are never fetched.
// PF: the NEXT tile's first column is loaded before this tile's dependent
// (selective) loads, so the chain of selective latencies overlaps a
// streaming read.
// CH: depth of the dependent chain of selective loads.  The result is the
//   conjunction of the three predicates whatever the order the columns are
//   fetched in; only the bytes and the latencies differ:
//   0  discount by f0, quantity by f01, price by f012 (3 round trips; the
//      reference's order, fewest bytes)
//   1  discount by f0, then quantity and price together by f01 (2)
//   2  discount, quantity and price together by f0 (1; most bytes: pays when
//      the date filter is selective, q1.2 / q1.3)
template <int BT, int IPT, bool PF = false, int CH = 0>
__global__ void __launch_bounds__(BT) ssb_flight1_kernel(const Flight1Args a) {
  using L = VecLayout<BT, IPT>;
  __shared__ long long red[BT / 32];
  long long sum = 0;
  unsigned cnt = 0;
  const int64_t ntiles = (a.n + L::TILE - 1) / L::TILE;
  int32_t nx[IPT];
  if (PF && blockIdx.x < ntiles)
    BlockLoad<BT, IPT>(a.fcol[0] + (int64_t)blockIdx.x * L::TILE,
                       (int)min((int64_t)L::TILE, a.n - (int64_t)blockIdx.x * L::TILE), nx);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * L::TILE;
    const int valid = (int)min((int64_t)L::TILE, a.n - base);
    int32_t x[IPT], d[IPT], e[IPT];
    if constexpr (PF) {
#pragma unroll
      for (int k = 0; k < IPT; ++k) x[k] = nx[k];
      const int64_t nt = tile + gridDim.x;
      if (nt < ntiles)
        BlockLoad<BT, IPT>(a.fcol[0] + nt * L::TILE, (int)min((int64_t)L::TILE, a.n - nt * L::TILE), nx);
    } else {
      BlockLoad<BT, IPT>(a.fcol[0] + base, valid, x);
    }
    unsigned f = BlockPred<IPT>(x, a.flo[0], a.fhi[0], BlockValidMask<BT, IPT>(valid));
    if constexpr (CH == 0) {
      BlockLoadSel<BT, IPT>(a.fcol[1] + base, valid, f, d);
      f = BlockPredAnd<IPT>(d, a.flo[1], a.fhi[1], f);
      BlockLoadSel<BT, IPT>(a.fcol[2] + base, valid, f, x);
      f = BlockPredAnd<IPT>(x, a.flo[2], a.fhi[2], f);
      BlockLoadSel<BT, IPT>(a.agg_a + base, valid, f, e);
      if (!a.agg_b_is_f1) BlockLoadSel<BT, IPT>(a.agg_b + base, valid, f, d);
    } else if constexpr (CH == 1) {
      BlockLoadSel<BT, IPT>(a.fcol[1] + base, valid, f, d);
      f = BlockPredAnd<IPT>(d, a.flo[1], a.fhi[1], f);
      BlockLoadSel<BT, IPT>(a.fcol[2] + base, valid, f, x);
      BlockLoadSel<BT, IPT>(a.agg_a + base, valid, f, e);
      f = BlockPredAnd<IPT>(x, a.flo[2], a.fhi[2], f);
      if (!a.agg_b_is_f1) BlockLoadSel<BT, IPT>(a.agg_b + base, valid, f, d);
    } else {
      BlockLoadSel<BT, IPT>(a.fcol[1] + base, valid, f, d);
      BlockLoadSel<BT, IPT>(a.fcol[2] + base, valid, f, x);
      BlockLoadSel<BT, IPT>(a.agg_a + base, valid, f, e);
      f = BlockPredAnd<IPT>(d, a.flo[1], a.fhi[1], f);
      f = BlockPredAnd<IPT>(x, a.flo[2], a.fhi[2], f);
      if (!a.agg_b_is_f1) BlockLoadSel<BT, IPT>(a.agg_b + base, valid, f, d);
    }
#pragma unroll
    for (int k = 0; k < IPT; ++k)
      if ((f >> k) & 1u) sum += (long long)e[k] * (long long)d[k];
    cnt += __popc(f);
  }
  const long long s = block_sum<BT>(sum, red);
  const long long c = block_sum<BT>((long long)cnt, red);
  pdl_wait();  // the prologue zeroed the aggregate
  if (threadIdx.x == 0) {
    atomicAdd(a.g_sum, (unsigned long long)s);
    atomicAdd(a.g_cnt, (unsigned long long)c);
    atomicAdd(a.surv, (unsigned long long)c);
  }
}

// (included inside crys::{anonymous}: it uses Flight1Args)
#include "ssb_flight1.cuh"

// Occupied cells -> (cell, sum) rows (grouped_result, ssb_queries.cpp:145-155).
// Flight 1 always yields its single row (ssb_queries.cpp:207-209).  Only the
// group-by sub-box the dimension builds allow is scanned (q4.3: 800 of 1.75 M
// cells); `packed` sources hold exactly the box cells (a reduced partial),
// otherwise they are the full dense aggregate.
__global__ void finalize_kernel(const unsigned long long* sums, const unsigned long long* cnts,
                                BoxPlan bp, int packed, int flight1, ResultHeader* hdr, RowOut* rows,
                                const unsigned long long* surv, const int32_t* err,
                                const HtMeta* meta, int nj) {
  pdl_wait();
  pdl_trigger();
  const unsigned lane = lane_id();
  const BoxD box = box_of(bp, meta);
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // QueryStats + error words ride in the header
    for (int j = 0; j < 4; ++j) hdr->surv[j] = surv ? surv[j] : 0;
    hdr->err = err ? *err : 0;
    int e = 0;
    for (int j = nj - 1; j >= 0; --j)  // the first failing build in plan order wins
      if (meta[j].err) e = (j << 8) | meta[j].err;
    hdr->ht_err = e;
  }
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < box.cells;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = base + threadIdx.x;
    int64_t c = 0, src = 0;
    if (b < box.cells) {
      c = box_to_full(bp, box, b);
      src = packed ? b : c;
    }
    const bool take = b < box.cells && (cnts[src] != 0 || (flight1 && c == 0));
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (!bal) continue;
    const int leader = __ffs(bal) - 1;
    unsigned long long p0 = 0;
    if ((int)lane == leader) p0 = atomicAdd(&hdr->nrows, (unsigned long long)__popc(bal));
    p0 = __shfl_sync(0xffffffffu, p0, leader);
    if (take) {
      RowOut r;
      r.cell = c;
      r.sum = (long long)sums[src];
      rows[p0 + __popc(bal & lanemask_lt())] = r;
    }
  }
}

// The dimension builds' digit extents -> host-mapped memory (the host sizes
// the collective from them while the fused pass runs), then a ready flag.
struct HostBox {
  int32_t dmin[kMaxJoins], dmax[kMaxJoins];
  volatile int32_t ready;
  int32_t pad[7];
};
__global__ void box_publish_kernel(const HtMeta* meta, int nj, HostBox* hb) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int j = 0; j < nj; ++j) {
      hb->dmin[j] = meta[j].dmin;
      hb->dmax[j] = meta[j].dmax;
    }
    __threadfence_system();
    hb->ready = 1;
  }
}

// Packs this device's dense aggregate into the partial layout of
// crystal_b200.h (CRYS_PARTIAL_HEADER int64 header, then the box's sums and
// counts) -- the payload of the one NCCL reduce.  Header words ADD into
// `out` (several shards of one device accumulate before the pack).
__global__ void pack_partial_kernel(const unsigned long long* sums, const unsigned long long* cnts,
                                    BoxPlan bp, const HtMeta* meta, int nj,
                                    const unsigned long long* surv, const int32_t* err,
                                    long long* out, int64_t cap) {
  const BoxD box = box_of(bp, meta);
  if (CRYS_PARTIAL_HEADER + 2 * box.cells > cap) return;  // the host raises ContractError
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int j = 0; j < 4; ++j) out[j] = surv ? (long long)surv[j] : 0;
    out[4] = (err && *err) ? 1 : 0;
    for (int i = 5; i < CRYS_PARTIAL_HEADER; ++i) out[i] = 0;
    for (int j = 0; j < nj; ++j) {
      const int e = meta[j].err;
      if (e >= 1 && e <= 4) out[8 + 4 * j + (e - 1)] = 1;
    }
  }
  long long* ps = out + CRYS_PARTIAL_HEADER;
  long long* pc = ps + box.cells;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < box.cells;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = box_to_full(bp, box, b);
    ps[b] = (long long)sums[c];
    pc[b] = (long long)cnts[c];
  }
}

// The header words of a packed partial -> the ResultHeader error fields
// (finalize of a reduced buffer; survivors are copied by finalize_kernel).
__global__ void unpack_errors_kernel(const long long* hdr_in, ResultHeader* hdr) {
  if (threadIdx.x == 0) {
    // every finalize_kernel thread reads err / meta errors through here
    int e = 0;
    for (int j = 3; j >= 0; --j)
      for (int c = 4; c >= 1; --c)
        if (hdr_in[8 + 4 * j + (c - 1)]) e = (j << 8) | c;
    hdr->err = hdr_in[4] ? 1 : 0;
    hdr->ht_err = e;
  }
}

// ---------------------------------------------------------- dispatch

#define CRYS_F1_SHAPES(X) X(128, 4) X(256, 16) X(128, 16) X(512, 8) X(256, 8)

using F1Fn = void (*)(const Flight1Args);

struct F1Launch {
  F1Fn fn;
  int bt, ipt;
  int tile = 0;      // rows per CTA per iteration (0: bt * ipt)
  size_t smem = 0;   // dynamic shared memory (ring kernels)
  int l2 = 0;        // ring kernels: L2 bulk-prefetch distance
};
template <int W, int V, int S, int PR, int L2, bool ST = false, int D = 1, bool CHN = false>
constexpr F1Launch f1_ring() {
  return F1Launch{ssb_flight1_ring_kernel<W, V, S, PR, ST, D, CHN>, (W + 1) * 32, 0, W * 128 * V,
                  ((size_t)S * D * W * 128 * V * 4 + 2 * S * 8 + 127) & ~(size_t)127, L2};
}

// Results are tile-invariant (test_ssb.cpp:251-261), so the TileConfig of a
// query is validated but the GPU runs its own tuned shape; CRYS_F1_TILE=BTxIPT
// forces a compiled (non-prefetching) shape (ablation / tuning).
F1Launch select_flight1() {
  static const std::pair<int, int> forced = [] {
    const char* e = getenv("CRYS_F1_TILE");
    int b = 0, i = 0;
    if (e && sscanf(e, "%dx%d", &b, &i) == 2) return std::make_pair(b, i);
    return std::make_pair(0, 0);  // no override: the prefetching default below
  }();
#define X(B, I) \
  if (forced.first == B && forced.second == I) return {ssb_flight1_kernel<B, I>, B, I};
  CRYS_F1_SHAPES(X)
#undef X
  // default: 256 x 8 with the next tile's first column prefetched (measured on
  // B200, tools/tune_f1pf.sh: q1.2 0.204 -> 0.193 ms, q1.3 0.184 -> 0.177 ms)
  return {ssb_flight1_kernel<256, 8, true>, 256, 8};
}

// Autotuner candidates of flight 1: register tiles (chain depth CH) and the
// date-column TMA ring (ssb_flight1.cuh; warps x rows/lane x stages x
// pipelined rounds, L2 look-ahead).
// Measured on B200 at SF=20 (tools/f1_probe.py, profiles/r02_flight1.txt):
// q1.1 wins with the two-column ring and chained gathers (0.262 -> 0.221 ms),
// q1.2 / q1.3 with the date-only ring and chained gathers (0.192 -> 0.111,
// 0.177 -> 0.078 ms).
constexpr int kTuneF1 = 8;
const F1Launch kF1Cands[kTuneF1] = {
    {ssb_flight1_kernel<256, 8, true, 0>, 256, 8}, f1_ring<24, 4, 4, 2, 2>(),
    f1_ring<16, 4, 3, 2, 0, true, 2>(),            f1_ring<16, 8, 3, 2, 0, true, 1, true>(),
    f1_ring<24, 4, 4, 2, 2, true, 1, true>(),      f1_ring<16, 8, 3, 3, 0, false, 1, true>(),
    f1_ring<16, 4, 3, 2, 0, true, 2, true>(),      f1_ring<16, 4, 3, 3, 2, false, 2, true>()};
// CRYS_F1_CAND=k forces candidate k (A/B runs); -1: autotuned
int flight1_cand() {
  static const int k = [] {
    const char* e = getenv("CRYS_F1_CAND");
    const int v = e ? atoi(e) : -1;
    return v >= 0 && v < kTuneF1 ? v : -1;
  }();
  return k;
}
bool flight1_forced() {
  static const bool f = getenv("CRYS_F1_TILE") != nullptr || flight1_cand() >= 0;
  return f;
}

int blocks_per_sm(const void* fn, int bt, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, size_t>, int> cache;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(dev, fn, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  ensure_dyn_smem(fn, smem);
  int nb = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, bt, smem));
  if (nb < 1) nb = 1;
  cache[key] = nb;
  return nb;
}

// 227 KB of shared memory per CTA on sm_100a, less a margin for the kernels'
// few static __shared__ words
constexpr size_t kSmemOptin = 232448 - 256;

// Shared-memory placement of the probe tables (plan order: join 0 is probed
// for every row, later joins only for survivors) and then of the CTA-private
// aggregate, inside what the ring leaves of 227 KB.
size_t place_smem(pipe::PipeArgs& pa, int nj, size_t fixed, int64_t cells) {
  size_t off = fixed;
  for (int j = 0; j < nj; ++j) {
    ProbeTab& t = pa.tab[j];
    t.smem = -1;
    if (t.kind == kTabHash || t.bytes == 0) continue;
    if (off + t.bytes <= kSmemOptin) {
      t.smem = (int32_t)off;
      off += t.bytes;
    }
  }
  pa.smem_agg = -1;
  const size_t agg = ((size_t)cells * 12 + 15) & ~(size_t)15;
  if (off + agg <= kSmemOptin) {
    pa.smem_agg = (int32_t)off;
    off += agg;
  }
  return off;
}

template <int NJ, int NC, int W, int TILE, int STAGES, int K0, bool S0>
int launch_pipeline(crys_ctx* ctx, pipe::PipeArgs pa, size_t dyn, const std::string& name) {
  auto fn = pipe::ssb_pipeline_kernel<NJ, NC, W, TILE, STAGES, K0, S0>;
  const int threads = (W + 1) * 32;
  const int nb = blocks_per_sm((const void*)fn, threads, dyn);
  const int64_t ntiles = (pa.n + TILE - 1) / TILE;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)nb * ctx->num_sms));
  launch_k(fn, grid, threads, dyn, ctx->stream, pa);
  CRYS_LAUNCHED(std::string("ssb_pipeline ") + name + " grid=" + std::to_string(grid) +
                " smem=" + std::to_string(dyn));
  return grid;
}

template <int NJ, int NC, int W, int TILE, int STAGES>
int launch_pipeline_k0(crys_ctx* ctx, pipe::PipeArgs pa, int64_t cells, const std::string& name) {
  const size_t fixed = pipe::fixed_smem<NC, TILE, STAGES>();
  CRYS_CHECK(fixed <= kSmemOptin, CRYS_ENOTBUILT, "pipeline ring exceeds shared memory");
  const size_t dyn = place_smem(pa, NJ, fixed, cells);
  const bool s0 = pa.tab[0].smem >= 0;
  switch (pa.tab[0].kind) {
    case kTabBitmap:
      if (s0) return launch_pipeline<NJ, NC, W, TILE, STAGES, kTabBitmap, true>(ctx, pa, dyn, name);
      return launch_pipeline<NJ, NC, W, TILE, STAGES, kTabBitmap, false>(ctx, pa, dyn, name);
    case kTabU8:
      if (s0) return launch_pipeline<NJ, NC, W, TILE, STAGES, kTabU8, true>(ctx, pa, dyn, name);
      return launch_pipeline<NJ, NC, W, TILE, STAGES, kTabU8, false>(ctx, pa, dyn, name);
    case kTabU16:
      if (s0) return launch_pipeline<NJ, NC, W, TILE, STAGES, kTabU16, true>(ctx, pa, dyn, name);
      return launch_pipeline<NJ, NC, W, TILE, STAGES, kTabU16, false>(ctx, pa, dyn, name);
    default:
      return launch_pipeline<NJ, NC, W, TILE, STAGES, kTabHash, false>(ctx, pa, dyn, name);
  }
}

// Dense half of a split plan (ssb_scan.cuh): the first D joins streamed
// through a ring of the D key columns only (deeper for the same shared
// memory), survivors to the per-CTA list regions.  Returns the grid.
template <int D, int W, int TILE, int STAGES, int K0, bool S0>
int launch_scan(crys_ctx* ctx, pipe::PipeArgs pa, size_t dyn, const std::string& name) {
  auto fn = pipe::ssb_scan_emit_kernel<D, W, TILE, TILE / W / 128, STAGES, K0, S0>;
  const int threads = (W + 1) * 32;
  const int nb = blocks_per_sm((const void*)fn, threads, dyn);
  const int64_t ntiles = (pa.n + TILE - 1) / TILE;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)nb * ctx->num_sms));
  const int64_t cap = ((ntiles + grid - 1) / grid) * TILE;  // every row of the CTA's tiles
  CRYS_CHECK(cap * grid <= pa.list_cap, CRYS_ECONTRACT, "survivor list workspace too small");
  pa.list_cap = cap;
  launch_k(fn, grid, threads, dyn, ctx->stream, pa);
  CRYS_LAUNCHED(std::string("ssb_scan_emit ") + name + " grid=" + std::to_string(grid) + " smem=" +
                std::to_string(dyn));
  return grid;
}

// Ring shapes (consumer warps W, rows per tile, stages): scan_shape() picks
// one of these per launch (the autotuner's candidates).
template <int D, int W, int TILE, int S>
int launch_emit_shape(crys_ctx* ctx, pipe::PipeArgs pa, const std::string& name, int64_t* list_cap);

int scan_cfg_env() {
  static const int v = [] {
    const char* e = getenv("CRYS_SCAN_CFG");
    return e ? atoi(e) : -1;
  }();
  return v;
}

template <int D>
int launch_emit(crys_ctx* ctx, pipe::PipeArgs pa, const std::string& name, int64_t* list_cap, int shape) {
  if (scan_cfg_env() >= 0) shape = scan_cfg_env();
  switch (shape) {
    case 1: return launch_emit_shape<D, 16, D == 1 ? 4096 : 2048, D == 1 ? 6 : 4>(ctx, pa, name, list_cap);
    case 2: return launch_emit_shape<D, 8, D == 1 ? 4096 : 2048, 4>(ctx, pa, name, list_cap);
    case 3: return launch_emit_shape<D, 16, D == 1 ? 8192 : 4096, 3>(ctx, pa, name, list_cap);
    default: return launch_emit_shape<D, 16, D == 1 ? 8192 : (D == 2 ? 4096 : 2048), 4>(ctx, pa, name, list_cap);
  }
}

template <int D, int W, int TILE, int S>
int launch_emit_shape(crys_ctx* ctx, pipe::PipeArgs pa, const std::string& name, int64_t* list_cap) {
  const size_t fixed = ((size_t)S * D * TILE * 4 + 2 * S * 8 + 127) & ~(size_t)127;
  const size_t dyn = place_smem(pa, D, fixed, 0);
  const bool s0 = pa.tab[0].smem >= 0;
  const int64_t ntiles = (pa.n + TILE - 1) / TILE;
  int grid;
  switch (pa.tab[0].kind) {
    case kTabBitmap:
      grid = s0 ? launch_scan<D, W, TILE, S, kTabBitmap, true>(ctx, pa, dyn, name)
                : launch_scan<D, W, TILE, S, kTabBitmap, false>(ctx, pa, dyn, name);
      break;
    case kTabU8:
      grid = s0 ? launch_scan<D, W, TILE, S, kTabU8, true>(ctx, pa, dyn, name)
                : launch_scan<D, W, TILE, S, kTabU8, false>(ctx, pa, dyn, name);
      break;
    case kTabU16:
      grid = s0 ? launch_scan<D, W, TILE, S, kTabU16, true>(ctx, pa, dyn, name)
                : launch_scan<D, W, TILE, S, kTabU16, false>(ctx, pa, dyn, name);
      break;
    default:
      grid = launch_scan<D, W, TILE, S, kTabHash, false>(ctx, pa, dyn, name);
  }
  *list_cap = ((ntiles + grid - 1) / grid) * TILE;
  return grid;
}

// Gather half: joins D..NJ-1 and the aggregate over the survivor list.  A
// persistent grid (4 CTAs of 256 threads per SM, 4 list entries per thread
// per round); the aggregate is CTA-private in shared memory for small group
// domains (q2.x, q3.1, q4.1, q4.2: hot cells), global atomics otherwise.
constexpr int kGatherBT = 256, kGatherK = 4;
template <int NJB, int NA, int NPRE = 0>
void launch_gather(crys_ctx* ctx, pipe::GatherArgs ga, int regions, int64_t cells, const std::string& name) {
  CRYS_CHECK(regions <= pipe::kMaxRegions, CRYS_ENOTBUILT, "too many survivor-list regions");
  ga.nregions = regions;
  for (int j = 0; j < NJB; ++j) ga.tab[j].smem = -1;
  for (int p = 0; p < 3; ++p) ga.pre[p].smem = -1;  // probed through L2 here
  const size_t agg = ((size_t)cells * 12 + 15) & ~(size_t)15;
  ga.smem_agg = cells <= 8192 ? 0 : -1;
  const size_t dyn = ga.smem_agg >= 0 ? agg : 0;
  auto fn = pipe::ssb_gather_kernel<NJB, NA, kGatherBT, kGatherK, NPRE>;
  const int nb = blocks_per_sm((const void*)fn, kGatherBT, dyn);
  const int grid = std::min(nb, 4) * ctx->num_sms;
  launch_k(fn, grid, kGatherBT, dyn, ctx->stream, ga);
  CRYS_LAUNCHED(std::string("ssb_gather ") + name + " smem=" + std::to_string(dyn));
}

template <int NJB, int NA>
void gather_pre(crys_ctx* ctx, pipe::GatherArgs ga, int regions, int64_t cells, const std::string& name, int npre) {
  switch (npre) {
    case 0: return launch_gather<NJB, NA, 0>(ctx, ga, regions, cells, name);
    case 1: return launch_gather<NJB, NA, 1>(ctx, ga, regions, cells, name);
    case 2: return launch_gather<NJB, NA, 2>(ctx, ga, regions, cells, name);
    default: return launch_gather<NJB, NA, 3>(ctx, ga, regions, cells, name);
  }
}

// Late-materialising plan (ssb_scanbm.cuh): the dense membership head over
// joins 0..D-1.  Ring shapes (consumer warps, rows per lane / 4, stages) in
// order of preference; the bitmaps go into what the ring leaves of 227 KB
// (join 0 first: it is tested for every row), the rest are tested in L2.
struct BmShape {
  int w, v, s;
};
// ring shapes {consumer warps, 128-row vectors per lane, stages}; families by
// the autotuner's preference: 0 = 16 warps, 1 = 31 warps (a full 1024-thread
// CTA), 2 = 24 warps.  The dense head is latency-bound (issue ~60 % with 17
// warps per SM; fewer warps with more rows each measured slower: 8 x 16 rows
// +15 %, 4 x 32 rows +60 %), so the wider families trade rows per lane for
// warps.
constexpr int kBmShapeN = 11;
constexpr BmShape kBmShapes[kBmShapeN] = {{16, 2, 4}, {16, 2, 3}, {16, 2, 2}, {16, 1, 4}, {31, 1, 4}, {31, 1, 3},
                                          {31, 1, 2}, {24, 2, 3}, {24, 2, 2}, {24, 1, 4}, {24, 1, 3}};
constexpr int kBmFamily[4] = {0, 4, 7, kBmShapeN};  // first shape of each preference family

template <int D, int W, int V, int S>
int launch_scanbm_shape(crys_ctx* ctx, pipe::BmArgs ba, size_t dyn, const std::string& name, int64_t* cap) {
  constexpr int TILE = W * 128 * V;
  bool allsh = true;
  for (int j = 0; j < D; ++j) allsh = allsh && ba.smem[j] >= 0;
  auto fn = allsh ? pipe::ssb_scan_bm_kernel<D, W, V, S, true> : pipe::ssb_scan_bm_kernel<D, W, V, S, false>;
  const int threads = (W + 1) * 32;
  const int nb = blocks_per_sm((const void*)fn, threads, dyn);
  const int64_t ntiles = (ba.n + TILE - 1) / TILE;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)nb * ctx->num_sms));
  *cap = ((ntiles + grid - 1) / grid) * TILE;  // every row of the CTA's tiles
  CRYS_CHECK(*cap * grid <= ba.list_cap, CRYS_ECONTRACT, "survivor list workspace too small");
  ba.list_cap = *cap;
  launch_k(fn, grid, threads, dyn, ctx->stream, ba);
  CRYS_LAUNCHED(std::string("ssb_scan_bm ") + name + " D=" + std::to_string(D) + " grid=" + std::to_string(grid) +
                " smem=" + std::to_string(dyn));
  return grid;
}

template <int D>
int launch_scanbm(crys_ctx* ctx, pipe::BmArgs ba, int pref, const std::string& name, int64_t* cap) {
  size_t bytes[3] = {0, 0, 0};
  for (int j = 0; j < D; ++j) bytes[j] = (size_t)ba.words[j] * 4;
  // placement for shape k: bitmaps in join order while they fit
  auto place = [&](int k, int32_t* off) {
    const BmShape& sh = kBmShapes[k];
    size_t at = ((size_t)sh.s * D * sh.w * 128 * sh.v * 4 + 2 * sh.s * 8 + 127) & ~(size_t)127;
    bool all = true;
    for (int j = 0; j < D; ++j) {
      if (at + bytes[j] <= kSmemOptin) {
        off[j] = (int32_t)at;
        at += bytes[j];
      } else {
        off[j] = -1;
        all = false;
      }
    }
    return std::make_pair(all, at);
  };
  int32_t off[3] = {-1, -1, -1};
  // the deepest ring of the preferred family that keeps every bitmap on chip,
  // else that family's deepest ring
  const int f = pref >= 0 && pref < 3 ? pref : 0;
  int k = kBmFamily[f];
  for (; k < kBmFamily[f + 1] && !place(k, off).first; ++k) {
  }
  if (k == kBmFamily[f + 1]) k = kBmFamily[f];
  const size_t dyn = place(k, off).second;
  for (int j = 0; j < 3; ++j) ba.smem[j] = j < D ? off[j] : -1;
  switch (k) {
    case 0: return launch_scanbm_shape<D, 16, 2, 4>(ctx, ba, dyn, name, cap);
    case 1: return launch_scanbm_shape<D, 16, 2, 3>(ctx, ba, dyn, name, cap);
    case 2: return launch_scanbm_shape<D, 16, 2, 2>(ctx, ba, dyn, name, cap);
    case 3: return launch_scanbm_shape<D, 16, 1, 4>(ctx, ba, dyn, name, cap);
    case 4: return launch_scanbm_shape<D, 31, 1, 4>(ctx, ba, dyn, name, cap);
    case 5: return launch_scanbm_shape<D, 31, 1, 3>(ctx, ba, dyn, name, cap);
    case 6: return launch_scanbm_shape<D, 31, 1, 2>(ctx, ba, dyn, name, cap);
    case 7: return launch_scanbm_shape<D, 24, 2, 3>(ctx, ba, dyn, name, cap);
    case 8: return launch_scanbm_shape<D, 24, 2, 2>(ctx, ba, dyn, name, cap);
    case 9: return launch_scanbm_shape<D, 24, 1, 4>(ctx, ba, dyn, name, cap);
    default: return launch_scanbm_shape<D, 24, 1, 3>(ctx, ba, dyn, name, cap);
  }
}

// Tuning knob CRYS_PIPE_CFG selects the (consumer warps, tile rows, stages)
// instantiation; 0 is the default.
int pipe_cfg() {
  static const int cfg = [] {
    const char* e = getenv("CRYS_PIPE_CFG");
    return e ? atoi(e) : 0;
  }();
  return cfg;
}

// CRYS_L2_AHEAD=k: the producer also bulk-prefetches into L2 the tile it will
// load k iterations later (0 = off).
int l2_ahead() {
  static const int v = [] {
    const char* e = getenv("CRYS_L2_AHEAD");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// CRYS_SPLIT=D forces split plans at join D (0 = the all-dense pipeline);
// read with CRYS_PIPE_CFG / CRYS_L2_AHEAD, which disable the autotuner.
int split_env() {
  static const int v = [] {
    const char* e = getenv("CRYS_SPLIT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// CRYS_BM=1: split plans (CRYS_SPLIT=D) run late-materialising (membership
// bitmaps, ssb_scanbm.cuh) with ring preference CRYS_PIPE_CFG.
int bm_env() {
  static const int v = [] {
    const char* e = getenv("CRYS_BM");
    return e ? atoi(e) : 0;
  }();
  return v;
}

}  // namespace

// Programmatic dependent launch along each query's chain (launch_k; CRYS_PDL=0
// turns it off).  Only the prologue and the dimension builds trigger their
// dependents early: the fused head's TMA ring starts streaming lineorder while
// the builds drain and waits (griddepcontrol.wait) only before it copies the
// tables.  Early triggers in the heads and gathers as well made the suite
// slower (3.26 -> 3.58 ms: the dependents' CTAs launched into the heads' SMs);
// with the triggers where they are: 3.14 -> 3.10 ms per step.
bool pdl_enabled() {
  static const bool v = [] {
    const char* e = getenv("CRYS_PDL");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

namespace {

int dim_grid_per_sm() {
  static const int v = [] {
    const char* e = getenv("CRYS_DIM_GRID");
    return e ? std::max(1, atoi(e)) : 8;
  }();
  return v;
}

// CRYS_TUNE=0 disables the per-query pipeline autotuner (default instantiation).
bool tune_enabled() {
  static const bool on = [] {
    const char* e = getenv("CRYS_TUNE");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

template <int NJ, int NC>
void launch_pipeline_cfg(crys_ctx* ctx, const pipe::PipeArgs& pa, int64_t cells,
                         const std::string& name, int cfg) {
  // Ring depth: 4 x 32 KB (q2/q3) or 3 x 48 KB (q4) stages.  Measured on
  // B200 (profiles/r01_pipeline_tuning.txt): the bytes in flight matter far
  // more than keeping a later join's table in shared memory -- dropping a
  // stage to fit q3.1's date table costs 2.3x.  cfg 3/4/6 trade shared memory
  // for more consumer warps (24 x 3072-row tiles / 20 x 2560): faster when
  // the plan's tables and aggregate do not need that memory (picked per
  // query by the autotuner below).
  constexpr int S = NC <= 4 ? 4 : 3;
  switch (cfg) {
    case 1: launch_pipeline_k0<NJ, NC, 16, 4096, 2>(ctx, pa, cells, name); break;
    case 3: launch_pipeline_k0<NJ, NC, 24, 3072, NC <= 4 ? 3 : 2>(ctx, pa, cells, name); break;
    case 4: launch_pipeline_k0<NJ, NC, 20, 2560, NC <= 4 ? 4 : 3>(ctx, pa, cells, name); break;
    case 6: launch_pipeline_k0<NJ, NC, 20, 2560, NC <= 4 ? 3 : 2>(ctx, pa, cells, name); break;
    default: launch_pipeline_k0<NJ, NC, 16, 2048, S>(ctx, pa, cells, name); break;
  }
}

}  // namespace

// ---------------------------------------------------------- workspace

// A replayable query: every launch + the result copy of one (db, qid) as a
// CUDA graph.  `sig` is every device/host address and column the captured work
// depends on; any change (a workspace buffer grew, a column was re-uploaded,
// another stream) re-captures.
struct QueryGraph {
  cudaGraphExec_t exec = nullptr;
  std::vector<uintptr_t> sig;
  int64_t kernels = 0;  // kernel nodes in the graph (launch accounting)
};

// Autotuning of the join-pipeline instantiation for 4-column plans (q2.x,
// q3.x): on a database's first execution of such a query every candidate runs
// twice back to back (aggregate re-zeroed before each run; the second run of
// each is timed with CUDA events), the fastest is kept for every later call.
// Results are identical for every candidate (the plans are tile-invariant);
// only the shared-memory split between ring, tables and aggregate differs.
// Candidates: (instantiation, L2 look-ahead distance).  4-column plans
// (q2.x, q3.x) try four instantiations with and without the L2 bulk prefetch;
// 6-column plans (q4.x, whose 48 KB stages leave no room for wider rings)
// only the look-ahead distances of the default instantiation.
// split > 0: the plan runs split at join `split` (EMIT kernel over joins
// 0..split-1, then the gather kernel; ssb_gather.cuh).
struct TuneCand {
  int cfg, l2, split;
  int bm = 0;  // 1: late-materialising split (membership bitmaps, ssb_scanbm.cuh); cfg = ring preference
};
// Split candidates run the dense head with one join (the measured winner
// whenever join 0 is selective: q3.2-q3.4, q4.3); cfg then names the scan
// ring shape (launch_emit).  Splitting after two joins was measured slower
// everywhere (the second join's L2 probes stall the scan's consumers).
// bm candidates: the late-materialising split after two joins (ssb_scanbm.cuh)
// with L2 look-ahead 0 / 2 / 4 (B200, SF=20: q2.1 0.323 -> 0.237 ms, q2.3
// 0.289 -> 0.171, q4.2 0.477 -> 0.376).
// bm candidates with cfg 1 / 2 use the 31-warp / 24-warp ring shapes (kBmShapes).
constexpr int kTuneN = 18;
constexpr TuneCand kTune4[kTuneN] = {{0, 0, 0},    {4, 0, 0},    {3, 0, 0},    {6, 0, 0},    {0, 2, 0},
                                     {4, 2, 0},    {3, 2, 0},    {6, 2, 0},    {3, 2, 1},    {3, 4, 1},
                                     {2, 2, 1},    {0, 0, 2, 1}, {0, 2, 2, 1}, {0, 4, 2, 1}, {1, 0, 2, 1},
                                     {1, 2, 2, 1}, {2, 0, 2, 1}, {2, 2, 2, 1}};
constexpr int kTuneN6 = 13;
constexpr TuneCand kTune6[kTuneN6] = {{0, 0, 0},    {0, 2, 0},    {0, 4, 0},    {3, 2, 1},    {3, 4, 1},
                                      {2, 2, 1},    {0, 0, 2, 1}, {0, 2, 2, 1}, {0, 4, 2, 1}, {1, 0, 2, 1},
                                      {1, 2, 2, 1}, {2, 0, 2, 1}, {2, 2, 2, 1}};
struct PipeTune {
  int chosen = -1;  // index into the plan shape's candidate list once decided
  int ncand = 0;
  cudaEvent_t e0[kTuneN] = {}, e1[kTuneN] = {};  // round 1 (candidates back to back)
  cudaEvent_t e2[kTuneN] = {}, e3[kTuneN] = {};  // round 2 (the same order again)
  bool in_flight = false;  // the query in flight carries the measurements
};

// Graph / tuning caches are keyed by the database's unique id (never reused,
// unlike its address), the query and the kind of sequence.
enum SeqKind { kSeqQuery = 0, kSeqPartial = 1 };
using SeqKey = std::tuple<uint64_t, int, int>;

struct QueryWorkspace {
  DevBuf agg;      // u64 [2*cells] + counters: surv[4] + err
  DevBuf meta;     // HtMeta[4]
  DevBuf slots[kMaxJoins];
  DevBuf compact[kMaxJoins];
  DevBuf tables;   // every join's direct probe table, contiguous, 16 B aligned
  DevBuf result;   // ResultHeader + RowOut[cells]
  DevBuf packed;   // the packed partial of a device group member (NCCL payload)
  DevBuf list;     // split plans: survivor list (uint2 per entry), regions of list_cap
  DevBuf list4;    // late-materialising plans: {row, key, key, key} per entry
  DevBuf list_count;
  PinnedBuf host;
  HostBox* hbox = nullptr;  // host-mapped digit extents (box_publish_kernel)
  std::map<SeqKey, QueryGraph> graphs;
  std::map<std::pair<uint64_t, int>, PipeTune> tune;
  PipeTune* measuring = nullptr;  // set by enqueue_query, completed after the sync
  ~QueryWorkspace() {
    for (auto& kv : graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    for (auto& kv : tune) destroy_events(kv.second);
    if (hbox) cudaFreeHost(hbox);
  }
  static void destroy_events(PipeTune& t) {
    for (int k = 0; k < kTuneN; ++k) {
      if (t.e0[k]) cudaEventDestroy(t.e0[k]);
      if (t.e1[k]) cudaEventDestroy(t.e1[k]);
      if (t.e2[k]) cudaEventDestroy(t.e2[k]);
      if (t.e3[k]) cudaEventDestroy(t.e3[k]);
    }
  }
};

void WsDeleter::operator()(QueryWorkspace* p) const { delete p; }

static QueryWorkspace& ws_of(crys_ctx* ctx) {
  if (!ctx->qws) ctx->qws.reset(new QueryWorkspace());
  return *ctx->qws;
}

// crys_db_free: drop every graph / tuning entry of that database.
void forget_db(crys_ctx* ctx, uint64_t uid) {
  if (!ctx || !ctx->qws) return;
  QueryWorkspace& ws = *ctx->qws;
  for (auto it = ws.graphs.begin(); it != ws.graphs.end();) {
    if (std::get<0>(it->first) == uid) {
      if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
      it = ws.graphs.erase(it);
    } else {
      ++it;
    }
  }
  for (auto it = ws.tune.begin(); it != ws.tune.end();) {
    if (it->first.first == uid) {
      if (ws.measuring == &it->second) ws.measuring = nullptr;
      QueryWorkspace::destroy_events(it->second);
      it = ws.tune.erase(it);
    } else {
      ++it;
    }
  }
}

static int64_t bit_ceil64(int64_t v) {
  int64_t c = 1;
  while (c < v) c <<= 1;
  return c;
}

// The plan's group parts as a box plan (mixed radix, last part fastest).
static BoxPlan box_plan(const QueryPlan& plan, BoxMode mode) {
  BoxPlan bp;
  std::memset(&bp, 0, sizeof(bp));
  bp.nparts = (int32_t)plan.group.size();
  CRYS_CHECK(bp.nparts <= 3, CRYS_ENOTBUILT, "at most three group parts");
  bp.mode = plan.joins.empty() ? kBoxFull : mode;
  int64_t stride = 1;
  for (int g = bp.nparts - 1; g >= 0; --g) {
    bp.join[g] = plan.group[g].join_index;
    bp.fcard[g] = plan.group[g].hi - plan.group[g].lo + 1;
    bp.fstride[g] = stride;
    stride *= bp.fcard[g];
  }
  return bp;
}

// Per-(database, query) autotuning: once decided, *chosen = the candidate and
// false is returned.  Otherwise every candidate is enqueued three times (the
// first run warms it up, the other two are timed together with events;
// [sums | counts | survivors | err] re-zeroed between runs, the last run's
// result is kept), the measurement is left in flight for tune_done() and true
// is returned.
template <class F>
static bool tune_or_measure(QueryWorkspace& ws, uint64_t uid, int qid, int ncand, cudaStream_t st,
                            unsigned long long* d_agg, int64_t cells, int* chosen, F&& launch_k) {
  PipeTune& tn = ws.tune[{uid, qid}];
  if (tn.chosen >= 0) {
    *chosen = tn.chosen;
    return false;
  }
  CRYS_CHECK(ncand <= kTuneN, CRYS_ENOTBUILT, "too many autotuner candidates");
  tn.ncand = ncand;
  // two interleaved rounds over the candidates, the best of both per
  // candidate: one timed run each could crown a candidate by HBM / clock drift
  for (int k = 0; k < ncand; ++k) {
    if (!tn.e0[k]) {
      CUDA_TRY(cudaEventCreate(&tn.e0[k]));
      CUDA_TRY(cudaEventCreate(&tn.e1[k]));
      CUDA_TRY(cudaEventCreate(&tn.e2[k]));
      CUDA_TRY(cudaEventCreate(&tn.e3[k]));
    }
  }
  for (int round = 0; round < 2; ++round) {
    for (int k = 0; k < ncand; ++k) {
      for (int rep = 0; rep < 2; ++rep) {
        if (round + k + rep > 0)  // the prologue zeroed it once
          CUDA_TRY(cudaMemsetAsync(d_agg, 0, sizeof(unsigned long long) * (size_t)(2 * cells + 5), st));
        if (rep == 1) CUDA_TRY(cudaEventRecord(round ? tn.e2[k] : tn.e0[k], st));
        launch_k(k);
        if (rep == 1) CUDA_TRY(cudaEventRecord(round ? tn.e3[k] : tn.e1[k], st));
      }
    }
  }
  tn.in_flight = true;
  ws.measuring = &tn;
  return true;
}

// Enqueues dimension builds (from `dimdb`) + the fused lineorder pass of `qid`
// over every fact shard in `facts` (lineorder columns; several shards of one
// device accumulate into the same aggregate), into d_agg = [sums | counts]
// (cells each), d_surv[4] and d_err.  `prologue_zero` additionally zeroes
// those buffers and the result header in the same prologue launch; the
// accumulating partial API hands in caller-zeroed buffers.  `hbox`: publish
// the builds' digit extents to host-mapped memory right after the builds.
static void enqueue_query(crys_ctx* ctx, const crys_db* dimdb, const std::vector<const crys_db*>& facts,
                          int qid, int bt, int ipt, unsigned long long* d_agg,
                          unsigned long long* d_surv, int32_t* d_err, unsigned long long* zero_extra,
                          int64_t zero_extra_n, bool prologue_zero, bool tune_ok, HostBox* hbox) {
  const QueryPlan& plan = plan_for(qid);
  CRYS_CHECK(bt > 0 && ipt > 0, CRYS_ECONFIG, "TileConfig: block_threads/items_per_thread must be positive");
  CRYS_CHECK(!facts.empty(), CRYS_ECONFIG, "no lineorder shard");
  QueryWorkspace& ws = ws_of(ctx);
  cudaStream_t st = ctx->stream;
  const int nj = (int)plan.joins.size();
  const int64_t cells = plan.cells();

  // rows of every fact shard
  const std::string& first_col = nj ? plan.joins[0].fact_key : plan.fact_filters[0].column;
  std::vector<int64_t> nrows(facts.size());
  for (size_t f = 0; f < facts.size(); ++f) facts[f]->col("lineorder", first_col, &nrows[f]);

  ws.meta.reserve(sizeof(HtMeta) * kMaxJoins);
  PrologueArgs pro;
  std::memset(&pro, 0, sizeof(pro));
  pro.meta = ws.meta.as<HtMeta>();
  if (prologue_zero) {
    // d_agg [2*cells] and the counters are contiguous in ws.agg
    pro.zero64 = d_agg;
    pro.zero64_n = 2 * cells + 5;
    pro.zero64b = zero_extra;
    pro.zero64b_n = zero_extra_n;
  }

  DimBuildArgs da;
  std::memset(&da, 0, sizeof(da));
  da.meta = ws.meta.as<HtMeta>();
  pipe::PipeArgs pa;
  std::memset(&pa, 0, sizeof(pa));
  int64_t max_rows = 0, max_cap = 0;
  bool any_ht = false;
  // membership bitmaps of the direct joins (late-materialising plans)
  const uint32_t* mem[kMaxJoins] = {nullptr, nullptr, nullptr, nullptr};
  size_t mem_bytes[kMaxJoins] = {0, 0, 0, 0}, mem_off[kMaxJoins];
  if (nj) {
    CRYS_CHECK(nj <= kMaxJoins, CRYS_ENOTBUILT, "at most four joins");
    // group parts -> (join, lo, card, stride): mixed radix, last part fastest
    int64_t stride = 1;
    int32_t glo[kMaxJoins] = {0, 0, 0, 0}, gcard[kMaxJoins] = {0, 0, 0, 0};
    for (int g = (int)plan.group.size() - 1; g >= 0; --g) {
      const GroupPart& gp = plan.group[g];
      CRYS_CHECK(gcard[gp.join_index] == 0, CRYS_ENOTBUILT, "one group part per join payload");
      glo[gp.join_index] = gp.lo;
      gcard[gp.join_index] = gp.hi - gp.lo + 1;
      pa.tab[gp.join_index].gstride = (int32_t)stride;
      stride *= (int64_t)(gp.hi - gp.lo + 1);
    }
    size_t tbl_bytes[kMaxJoins] = {0, 0, 0, 0}, tbl_off[kMaxJoins] = {0, 0, 0, 0}, tbl_total = 0;
    mem_off[0] = mem_off[1] = mem_off[2] = mem_off[3] = SIZE_MAX;
    constexpr int64_t kMaxDirect = int64_t(1) << 26;  // key-range bound of the direct tables
    for (int j = 0; j < nj; ++j) {
      const DimJoin& dj = plan.joins[j];
      DimBuildDesc& d = da.d[j];
      int64_t rows = 0;
      d.key = dimdb->col(dj.dim_table, dj.dim_key, &rows);
      d.rows = rows;
      d.payload = dj.payload.empty() ? nullptr : dimdb->col(dj.dim_table, dj.payload, &rows);
      CRYS_CHECK((int)dj.filters.size() <= 2, CRYS_ENOTBUILT, "at most two filters per join");
      d.nf = (int)dj.filters.size();
      for (int f = 0; f < d.nf; ++f) {
        d.fcol[f] = dimdb->col(dj.dim_table, dj.filters[f].column, &rows);
        CRYS_CHECK(dj.filters[f].ranges.size() <= 2, CRYS_ENOTBUILT, "at most two ranges per filter");
        d.nranges[f] = (int)dj.filters[f].ranges.size();
        for (int r = 0; r < d.nranges[f]; ++r) {
          d.r[f][r][0] = dj.filters[f].ranges[r].first;
          d.r[f][r][1] = dj.filters[f].ranges[r].second;
        }
      }
      d.glo = glo[j];
      d.gcard = gcard[j];
      CRYS_CHECK(d.gcard <= 65534, CRYS_ENOTBUILT, "group domain too large for a 16-bit digit");
      max_rows = std::max(max_rows, d.rows);
      // table layout: a perfect hash over the dense key range when the key
      // column's statistics allow it, else the linear-probing table
      int32_t lo = 0, hi = -1;
      const bool direct = dimdb->col_range(dj.dim_table, dj.dim_key, &lo, &hi) &&
                          (int64_t)hi - lo + 1 <= kMaxDirect;
      if (direct) {
        d.kmin = (uint32_t)lo;
        d.nkeys = (uint32_t)((int64_t)hi - lo + 1);
        if (dj.payload.empty() || d.gcard == 0) {
          d.kind = kTabBitmap;
          // one extra (absent) entry past the key range: probes may clamp an
          // out-of-range key to index nkeys instead of testing it (ssb_scan.cuh)
          tbl_bytes[j] = ((size_t)(d.nkeys + 1 + 31) / 32) * 4;
          d.clear_value = 0u;
        } else {
          d.kind = d.gcard <= 254 ? kTabU8 : kTabU16;
          tbl_bytes[j] = (size_t)(d.nkeys + 1) * (d.kind == kTabU8 ? 1 : 2);
          d.clear_value = 0xFFFFFFFFu;
        }
        tbl_bytes[j] = (tbl_bytes[j] + 15) & ~(size_t)15;
        d.clear_words = (uint32_t)(tbl_bytes[j] / 4);
        tbl_off[j] = tbl_total;
        tbl_total += tbl_bytes[j];
        // membership bitmap over the same domain (bit nkeys: the absent pad)
        mem_bytes[j] = ((size_t)(d.nkeys + 1 + 127) / 128) * 16;
        if (d.kind != kTabBitmap) {
          mem_off[j] = tbl_total;
          tbl_total += mem_bytes[j];
        }
      } else {
        d.kind = kTabHash;
        any_ht = true;
        d.maxcap = std::max<int64_t>(2, bit_ceil64(2 * d.rows));
        ws.slots[j].reserve(sizeof(int2) * d.maxcap);
        ws.compact[j].reserve(sizeof(int2) * std::max<int64_t>(1, d.rows));
        d.slots = ws.slots[j].as<int2>();
        d.compact = ws.compact[j].as<int2>();
        max_cap = std::max(max_cap, d.maxcap);
      }
      ProbeTab& t = pa.tab[j];
      t.kind = d.kind;
      t.kmin = d.kmin;
      t.n = d.nkeys;
      t.bytes = (uint32_t)tbl_bytes[j];
      t.meta = j;
      t.g = d.kind == kTabHash ? (const void*)d.slots : nullptr;
      if (d.kind != kTabHash) pipe::set_decode(t);
    }
    if (tbl_total) ws.tables.reserve(tbl_total);
    for (int j = 0; j < nj; ++j) {
      if (da.d[j].kind == kTabHash) continue;
      da.d[j].tbl = ws.tables.as<char>() + tbl_off[j];
      pa.tab[j].g = da.d[j].tbl;
      pro.tbl[j] = reinterpret_cast<uint32_t*>(da.d[j].tbl);
      pro.words[j] = da.d[j].clear_words;
      pro.value[j] = da.d[j].clear_value;
      // the join's membership bitmap: the table itself, or the one beside the codes
      mem[j] = reinterpret_cast<const uint32_t*>(da.d[j].tbl);
      if (mem_off[j] != SIZE_MAX) {
        da.d[j].bits = reinterpret_cast<uint32_t*>(ws.tables.as<char>() + mem_off[j]);
        mem[j] = da.d[j].bits;
        pro.tbl[kMaxJoins + j] = da.d[j].bits;
        pro.words[kMaxJoins + j] = (uint32_t)(mem_bytes[j] / 4);
        pro.value[kMaxJoins + j] = 0u;
      }
    }
  }
  // ---- launches: prologue, dimension builds
  {
    int64_t work = std::max<int64_t>(pro.zero64_n, pro.zero64b_n);
    for (int j = 0; j < 2 * kMaxJoins; ++j) work = std::max<int64_t>(work, pro.words[j]);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)ctx->num_sms * 4));
    query_prologue_kernel<<<grid, 256, 0, st>>>(pro);
    CRYS_LAUNCHED("query_prologue_kernel");
    count_launch(ctx);
  }
  if (nj) {
    const int tpb = 256;
    const int gx_rows = (int)std::min<int64_t>((max_rows + tpb - 1) / tpb, (int64_t)ctx->num_sms * 8);
    // CTAs per dimension: CRYS_DIM_GRID per SM (default 8; measured on the
    // SF=20 suite: 1 -> 18-41 us per build, 2 -> 12-24, 4 and 8 -> 9-20)
    const int gx_filter = (int)std::min<int64_t>((max_rows + tpb * kDimU - 1) / (tpb * kDimU),
                                                 (int64_t)ctx->num_sms * dim_grid_per_sm());
    // per dimension: ~2 passes of tpb x kDimU rows per CTA, at most gx_filter CTAs
    int total = 0;
    for (int j = 0; j <= kMaxJoins; ++j) {
      da.cta0[j] = total;
      if (j < nj) {
        const int64_t want = (da.d[j].rows + 2 * tpb * kDimU - 1) / (2 * tpb * kDimU);
        total += (int)std::max<int64_t>(1, std::min<int64_t>(want, std::max(gx_filter, 1)));
      }
    }
    launch_k(dim_filter_kernel, dim3(total), tpb, 0, st, da);
    CRYS_LAUNCHED("dim_filter_kernel");
    count_launch(ctx);
    if (any_ht) {  // linear-probing builds (hash_table.cpp:20-94) for sparse key domains
      const int gx_cap = (int)std::min<int64_t>((max_cap + tpb - 1) / tpb, (int64_t)ctx->num_sms * 8);
      launch_k(dim_init_kernel, dim3(std::max(gx_cap, 1), nj), tpb, 0, st, da);
      CRYS_LAUNCHED("dim_init_kernel");
      launch_k(dim_insert_kernel, dim3(std::max(gx_rows, 1), nj), tpb, 0, st, da);
      CRYS_LAUNCHED("dim_insert_kernel");
      count_launch(ctx, 2);
    }
    if (hbox) {
      launch_k(box_publish_kernel, 1, 32, 0, st, ws.meta.as<HtMeta>(), nj, hbox);
      CRYS_LAUNCHED("box_publish_kernel");
      count_launch(ctx);
    }
  }

  // ---- the fused lineorder pass, once per fact shard
  int64_t rows = 0;
  if (nj) {
    pa.meta = ws.meta.as<HtMeta>();
    pa.l2_ahead = l2_ahead();
    pa.cells = (int32_t)cells;
    pa.g_sum = d_agg;
    pa.g_cnt = d_agg + cells;
    pa.surv = d_surv;
    pa.err = d_err;
    CRYS_CHECK(plan.agg != kAggExtPriceTimesDiscount, CRYS_ENOTBUILT, "join flights aggregate revenue");
    // late materialisation needs direct tables (membership bitmaps) for joins 0..D-1
    auto bm_eligible = [&](int D) {
      for (int j = 0; j < D; ++j)
        if (!mem[j]) return false;
      return true;
    };
    auto launch = [&](TuneCand c) {
      pa.l2_ahead = c.l2;
      for (size_t f = 0; f < facts.size(); ++f) {
        pa.n = nrows[f];
        for (int j = 0; j < nj; ++j) {
          pa.col[j] = facts[f]->col("lineorder", plan.joins[j].fact_key, &rows);
          CRYS_CHECK(rows == pa.n, CRYS_ECONTRACT, "lineorder columns of different length");
        }
        pa.col[nj] = facts[f]->col("lineorder", "lo_revenue", &rows);
        CRYS_CHECK(rows == pa.n, CRYS_ECONTRACT, "lineorder columns of different length");
        if (plan.agg == kAggRevenueMinusSupplyCost) {
          pa.col[nj + 1] = facts[f]->col("lineorder", "lo_supplycost", &rows);
          CRYS_CHECK(rows == pa.n, CRYS_ECONTRACT, "lineorder columns of different length");
        }
        const bool shape3 = nj == 3 && plan.agg == kAggRevenue;
        const bool shape4 = nj == 4 && plan.agg == kAggRevenueMinusSupplyCost;
        CRYS_CHECK(shape3 || shape4, CRYS_ENOTBUILT, "no fused pipeline for this plan shape");
        if (c.bm && c.split > 0 && c.split < nj && bm_eligible(c.split)) {  // late materialisation
          const int D = c.split;
          pipe::BmArgs ba;
          std::memset(&ba, 0, sizeof(ba));
          ba.n = pa.n;
          int npre = 0, pre_j[3] = {-1, -1, -1};
          for (int j = 0; j < D; ++j) {
            ba.col[j] = pa.col[j];
            ba.bm[j] = mem[j];
            ba.kmin[j] = pa.tab[j].kmin;
            ba.nk[j] = pa.tab[j].n;
            ba.words[j] = (uint32_t)(mem_bytes[j] / 4);
            if (pa.tab[j].gstride != 0) pre_j[npre++] = j;
          }
          for (int w = 0; w < 3; ++w) ba.key_of[w] = pre_j[w];
          ba.list = ws.list4.as<uint4>();
          ba.list_cap = (int64_t)(ws.list4.bytes / sizeof(uint4));
          ba.list_count = ws.list_count.as<unsigned>();
          ba.surv = pa.surv;
          ba.l2_ahead = c.l2;
          int64_t cap = 0;
          const int grid = D == 1   ? launch_scanbm<1>(ctx, ba, c.cfg, plan.name, &cap)
                           : D == 2 ? launch_scanbm<2>(ctx, ba, c.cfg, plan.name, &cap)
                                    : launch_scanbm<3>(ctx, ba, c.cfg, plan.name, &cap);
          pipe::GatherArgs ga;
          std::memset(&ga, 0, sizeof(ga));
          ga.list4 = ba.list;
          ga.list_cap = cap;
          ga.list_count = ba.list_count;
          const int nb = nj - D;
          for (int j = 0; j < nb; ++j) {
            ga.col[j] = pa.col[D + j];
            ga.tab[j] = pa.tab[D + j];
          }
          ga.col[nb] = pa.col[nj];
          ga.col[nb + 1] = pa.col[nj + 1];
          for (int p = 0; p < npre; ++p) ga.pre[p] = pa.tab[pre_j[p]];
          ga.meta = pa.meta;
          ga.cells = (int32_t)cells;
          ga.g_sum = pa.g_sum;
          ga.g_cnt = pa.g_cnt;
          ga.surv = pa.surv + D;
          ga.err = pa.err;
          if (shape3 && nb == 1) gather_pre<1, 1>(ctx, ga, grid, cells, plan.name, npre);
          else if (shape3 && nb == 2) gather_pre<2, 1>(ctx, ga, grid, cells, plan.name, npre);
          else if (shape4 && nb == 1) gather_pre<1, 2>(ctx, ga, grid, cells, plan.name, npre);
          else if (shape4 && nb == 2) gather_pre<2, 2>(ctx, ga, grid, cells, plan.name, npre);
          else gather_pre<3, 2>(ctx, ga, grid, cells, plan.name, npre);
          count_launch(ctx, 2);
          continue;
        }
        if (c.split > 0 && c.split < nj && !c.bm) {  // dense joins 0..D-1, survivor list, gather tail
          const int D = c.split, nb = nj - D;
          pipe::PipeArgs pe = pa;
          pe.cells = 0;
          pe.list = ws.list.as<uint2>();
          pe.list_cap = (int64_t)(ws.list.bytes / sizeof(uint2));
          pe.list_count = ws.list_count.as<unsigned>();
          int64_t cap = 0;
          const int grid = D == 1   ? launch_emit<1>(ctx, pe, plan.name, &cap, c.cfg)
                           : D == 2 ? launch_emit<2>(ctx, pe, plan.name, &cap, c.cfg)
                                    : launch_emit<3>(ctx, pe, plan.name, &cap, c.cfg);
          pipe::GatherArgs ga;
          std::memset(&ga, 0, sizeof(ga));
          ga.list = pe.list;
          ga.list_cap = cap;
          ga.list_count = pe.list_count;
          for (int j = 0; j < nb; ++j) {
            ga.col[j] = pa.col[D + j];
            ga.tab[j] = pa.tab[D + j];
          }
          ga.col[nb] = pa.col[nj];
          ga.col[nb + 1] = pa.col[nj + 1];
          ga.meta = pa.meta;
          ga.cells = (int32_t)cells;
          ga.g_sum = pa.g_sum;
          ga.g_cnt = pa.g_cnt;
          ga.surv = pa.surv + D;
          ga.err = pa.err;
          if (shape3 && nb == 1) launch_gather<1, 1>(ctx, ga, grid, cells, plan.name);
          else if (shape3 && nb == 2) launch_gather<2, 1>(ctx, ga, grid, cells, plan.name);
          else if (shape4 && nb == 1) launch_gather<1, 2>(ctx, ga, grid, cells, plan.name);
          else if (shape4 && nb == 2) launch_gather<2, 2>(ctx, ga, grid, cells, plan.name);
          else launch_gather<3, 2>(ctx, ga, grid, cells, plan.name);
          count_launch(ctx, 2);
          continue;
        }
        if (shape3)
          launch_pipeline_cfg<3, 4>(ctx, pa, cells, plan.name, c.cfg);
        else
          launch_pipeline_cfg<4, 6>(ctx, pa, cells, plan.name, c.cfg);
        count_launch(ctx);
      }
    };
    {  // survivor-list workspace of split plans (regions of whole CTA tile sets)
      int64_t nmax = 0;
      for (int64_t r : nrows) nmax = std::max(nmax, r);
      ws.list.reserve(sizeof(uint2) * (size_t)(nmax + ((int64_t)ctx->num_sms * 4 + 1) * 4096));
      // (slack: every CTA rounds its share up to whole ring tiles of <= 8192 rows)
      ws.list4.reserve(sizeof(uint4) * (size_t)(nmax + ((int64_t)ctx->num_sms + 1) * 8192));
      ws.list_count.reserve(sizeof(unsigned) * (size_t)ctx->num_sms * 8);
    }
    const int cfg = pipe_cfg();  // CRYS_PIPE_CFG > 0 forces an instantiation
    TuneCand run{cfg, l2_ahead(), split_env(), bm_env()};
    const TuneCand* cands = nj == 3 ? kTune4 : kTune6;
    const int ncand = nj == 3 ? kTuneN : kTuneN6;
    if (cfg == 0 && l2_ahead() == 0 && split_env() == 0 && (nj == 3 || nj == 4) && tune_enabled() && tune_ok) {
      int chosen = -1;
      if (tune_or_measure(ws, dimdb->uid, qid, ncand, st, d_agg, cells, &chosen,
                          [&](int k) { launch(cands[k]); }))
        return;
      run = cands[chosen];
    }
    timing_kernel_begin(ctx);
    launch(run);
    timing_kernel_end(ctx);
    return;
  }
  Flight1Args fa;
  std::memset(&fa, 0, sizeof(fa));
  fa.g_sum = d_agg;
  fa.g_cnt = d_agg + cells;
  fa.surv = d_surv;
  auto launch_f1 = [&](F1Launch L) {
  const int nb = blocks_per_sm((const void*)L.fn, L.bt, L.smem);
  const int64_t tile = L.tile ? L.tile : (int64_t)L.bt * L.ipt;
  fa.l2_ahead = L.l2;
  for (size_t f = 0; f < facts.size(); ++f) {
    const int64_t n = nrows[f];
    fa.n = n;
    for (int k = 0; k < 3; ++k) {
      fa.fcol[k] = facts[f]->col("lineorder", plan.fact_filters[k].column, &rows);
      CRYS_CHECK(rows == n, CRYS_ECONTRACT, "lineorder columns of different length");
      fa.flo[k] = plan.fact_filters[k].lo;
      fa.fhi[k] = plan.fact_filters[k].hi;
    }
    // aggregate columns (agg_fact_columns, ssb_plans.cpp:287-299)
    fa.agg_a = facts[f]->col("lineorder", "lo_extendedprice", &rows);
    fa.agg_b = facts[f]->col("lineorder", "lo_discount", &rows);
    fa.agg_b_is_f1 = plan.fact_filters.size() > 1 && plan.fact_filters[1].column == "lo_discount";
    const int64_t ntiles = (n + tile - 1) / tile;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)nb * ctx->num_sms));
    launch_k(L.fn, grid, L.bt, L.smem, st, fa);
    CRYS_LAUNCHED(std::string("fused ") + plan.name + " bt=" + std::to_string(L.bt) + " ipt=" +
                  std::to_string(L.ipt) + " grid=" + std::to_string(grid));
    count_launch(ctx);
  }
  };
  F1Launch L = flight1_cand() >= 0 ? kF1Cands[flight1_cand()] : select_flight1();
  if (!flight1_forced() && tune_enabled() && tune_ok) {
    int chosen = -1;
    if (tune_or_measure(ws, dimdb->uid, qid, kTuneF1, st, d_agg, cells, &chosen,
                        [&](int k) { launch_f1(kF1Cands[k]); }))
      return;
    L = kF1Cands[chosen];
  }
  timing_kernel_begin(ctx);
  launch_f1(L);
  timing_kernel_end(ctx);
}

// Adds this call's error words into a partial header (accumulating API).
__global__ void partial_errors_kernel(const HtMeta* meta, int nj, const int32_t* err, long long* hdr) {
  if (threadIdx.x == 0) {
    if (*err) atomicAdd(reinterpret_cast<unsigned long long*>(hdr + 4), 1ull);
    for (int j = 0; j < nj; ++j) {
      const int e = meta[j].err;
      if (e >= 1 && e <= 4) atomicAdd(reinterpret_cast<unsigned long long*>(hdr + 8 + 4 * j + (e - 1)), 1ull);
    }
  }
}

void ssb_query_partial(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt,
                       unsigned long long* d_agg, long long* d_hdr) {
  const QueryPlan& plan = plan_for(qid);
  ctx->scratch2.reserve(64);
  int32_t* err = ctx->scratch2.as<int32_t>();
  CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int32_t), ctx->stream));
  enqueue_query(ctx, db, {db}, qid, bt, ipt, d_agg, reinterpret_cast<unsigned long long*>(d_hdr), err,
                nullptr, 0, false, false, nullptr);
  partial_errors_kernel<<<1, 32, 0, ctx->stream>>>(ws_of(ctx).meta.as<HtMeta>(), (int)plan.joins.size(),
                                                   err, d_hdr);
  CRYS_LAUNCHED("partial_errors_kernel");
  count_launch(ctx);
}

// Compaction kernel + the copy of the header and the first 2048 rows (stream
// work only, so it can be captured into a query graph).  `src` is the dense
// aggregate (packed = false) or a packed partial's box cells; with
// `hdr_in` (a packed partial's header) the survivors and errors come from it.
static void finalize_enqueue(crys_ctx* ctx, int qid, const unsigned long long* d_sums,
                             const unsigned long long* d_cnts, const BoxPlan& bp, bool packed,
                             const unsigned long long* d_surv, const int32_t* d_err,
                             const long long* hdr_in, bool hdr_zeroed) {
  const QueryPlan& plan = plan_for(qid);
  QueryWorkspace& ws = ws_of(ctx);
  cudaStream_t st = ctx->stream;
  const int64_t cells = plan.cells();
  ResultHeader* hdr = ws.result.as<ResultHeader>();
  RowOut* rows = reinterpret_cast<RowOut*>(hdr + 1);
  if (!hdr_zeroed) CUDA_TRY(cudaMemsetAsync(hdr, 0, sizeof(ResultHeader), st));
  const int tpb = 256;
  // grid-stride over the BOX (known on the device only): the box is a few
  // hundred to a few thousand cells, so one CTA per SM at most (~1200 mostly
  // idle CTAs for q3.2-q4.3's large full domains cost launch time)
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((cells + tpb - 1) / tpb, (int64_t)ctx->num_sms));
  const int nj = d_err ? (int)plan.joins.size() : 0;  // build errors of this ctx's own dimension builds
  launch_k(finalize_kernel, grid, tpb, 0, st, d_sums, d_cnts, bp, packed ? 1 : 0, plan.joins.empty() ? 1 : 0, hdr,
           rows, hdr_in ? reinterpret_cast<const unsigned long long*>(hdr_in) : d_surv, d_err,
           (const HtMeta*)ws.meta.as<HtMeta>(), nj);
  CRYS_LAUNCHED("finalize_kernel");
  count_launch(ctx);
  if (hdr_in) {
    unpack_errors_kernel<<<1, 32, 0, st>>>(hdr_in, hdr);
    CRYS_LAUNCHED("unpack_errors_kernel");
    count_launch(ctx);
  }
  const int64_t first = std::min<int64_t>(cells, 2048);
  const size_t first_bytes = sizeof(ResultHeader) + sizeof(RowOut) * (size_t)first;
  CUDA_TRY(cudaMemcpyAsync(ws.host.p, hdr, first_bytes, cudaMemcpyDeviceToHost, st));
}

static void finalize_reserve(crys_ctx* ctx, int64_t cells) {
  QueryWorkspace& ws = ws_of(ctx);
  ws.result.reserve(sizeof(ResultHeader) + sizeof(RowOut) * (size_t)cells);
  ws.host.reserve(sizeof(ResultHeader) + sizeof(RowOut) * (size_t)cells);
  ws.meta.reserve(sizeof(HtMeta) * kMaxJoins);
}

static const char* ht_error_message(int code) {
  switch (code) {
    case 1: return "HashTable: key equals empty sentinel";
    case 2: return "HashTable: duplicate key";
    case 3: return "HashTable: capacity overflow";
    default: return "dimension key outside its column statistics";
  }
}

// Host side after the stream work: wait, fetch any rows past the first 2048,
// order them and map the error words.
static void finalize_host_part(crys_ctx* ctx, int qid, ResultRows* out) {
  const QueryPlan& plan = plan_for(qid);
  QueryWorkspace& ws = ws_of(ctx);
  cudaStream_t st = ctx->stream;
  const int64_t cells = plan.cells();
  RowOut* rows = reinterpret_cast<RowOut*>(ws.result.as<ResultHeader>() + 1);
  const int64_t first = std::min<int64_t>(cells, 2048);
  const size_t first_bytes = sizeof(ResultHeader) + sizeof(RowOut) * (size_t)first;
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
  // the build errors of the first failing join in plan order (the reference
  // builds the dimension tables in plan order and throws at the first)
  if (ht_err) {
    const int code = ht_err & 0xFF;
    fail(code == 4 ? CRYS_ECONTRACT : CRYS_EBUILD,
         std::string(ht_error_message(code)) + " (join " + std::to_string(ht_err >> 8) + " of " + plan.name + ")");
  }
  if (out->err) fail(CRYS_ECONTRACT, "group value outside its declared domain");
}

// Finalize of a caller's dense [sums | counts] (+ optional partial header).
void ssb_finalize_device(crys_ctx* ctx, int qid, const unsigned long long* d_agg, const long long* d_hdr,
                         ResultRows* out) {
  const int64_t cells = plan_for(qid).cells();
  finalize_reserve(ctx, cells);
  const BoxPlan bp = box_plan(plan_for(qid), kBoxFull);
  finalize_enqueue(ctx, qid, d_agg, d_agg + cells, bp, false, nullptr, nullptr, d_hdr, false);
  finalize_host_part(ctx, qid, out);
}

// Finalize of a (reduced) packed partial whose box the caller knows.
void ssb_finalize_packed(crys_ctx* ctx, int qid, const crys_group_box& box, const long long* d_buf,
                         ResultRows* out) {
  const QueryPlan& plan = plan_for(qid);
  finalize_reserve(ctx, plan.cells());
  BoxPlan bp = box_plan(plan, kBoxExplicit);
  CRYS_CHECK(box.nparts == bp.nparts, CRYS_ECONTRACT, "group box does not match the query's group parts");
  int64_t cells = 1;
  for (int g = 0; g < bp.nparts; ++g) {
    bp.xmin[g] = box.lo[g] - plan.group[g].lo;
    bp.xcard[g] = box.card[g];
    CRYS_CHECK(box.card[g] >= 0 && bp.xmin[g] >= 0 && bp.xmin[g] + box.card[g] <= bp.fcard[g],
               CRYS_ECONTRACT, "group box outside the query's group domain");
    cells *= box.card[g];
  }
  CRYS_CHECK(cells == box.cells, CRYS_ECONTRACT, "group box cell count mismatch");
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(d_buf + CRYS_PARTIAL_HEADER);
  finalize_enqueue(ctx, qid, s, s + cells, bp, true, nullptr, nullptr, d_buf, false);
  finalize_host_part(ctx, qid, out);
}

// CRYS_GRAPHS=0 disables the per-query graph replay (A/B).
static bool graphs_enabled() {
  static const bool on = [] {
    const char* e = getenv("CRYS_GRAPHS");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

static void db_signature(const crys_db* db, std::vector<uintptr_t>& sig) {
  sig.push_back((uintptr_t)db->uid);
  for (const auto& kv : db->cols) {
    sig.push_back((uintptr_t)kv.second.buf->p);
    sig.push_back((uintptr_t)kv.second.rows);
    sig.push_back(((uintptr_t)(uint32_t)kv.second.vmin << 32) | (uint32_t)kv.second.vmax);
    sig.push_back((uintptr_t)kv.second.stats);
  }
  sig.push_back((uintptr_t)db->lo_begin);
  sig.push_back((uintptr_t)db->lo_end);
}

static std::vector<uintptr_t> query_signature(crys_ctx* ctx, const std::vector<const crys_db*>& dbs) {
  QueryWorkspace& ws = ws_of(ctx);
  std::vector<uintptr_t> sig = {(uintptr_t)ctx->stream, (uintptr_t)ws.agg.p, ws.agg.bytes,
                                (uintptr_t)ws.meta.p, (uintptr_t)ws.tables.p, ws.tables.bytes,
                                (uintptr_t)ws.result.p, ws.result.bytes, (uintptr_t)ws.host.p, ws.host.bytes,
                                (uintptr_t)ws.packed.p, ws.packed.bytes, (uintptr_t)ws.hbox,
                                (uintptr_t)ws.list.p, ws.list.bytes, (uintptr_t)ws.list_count.p};
  for (int j = 0; j < kMaxJoins; ++j) {
    sig.push_back((uintptr_t)ws.slots[j].p);
    sig.push_back((uintptr_t)ws.compact[j].p);
  }
  for (const crys_db* db : dbs) db_signature(db, sig);
  return sig;
}

static bool any_pending(const std::vector<const crys_db*>& dbs) {
  bool pending = false;
  for (const crys_db* db : dbs)
    for (const auto& kv : db->cols) pending = pending || kv.second.pending;
  return pending;
}

// after the host part (stream synchronised): pick the fastest candidate
static void tune_done(crys_ctx* ctx) {
  QueryWorkspace& ws = ws_of(ctx);
  PipeTune* tn = ws.measuring;
  ws.measuring = nullptr;
  if (!tn || !tn->in_flight) return;
  tn->in_flight = false;
  float best = 1e30f;
  for (int k = 0; k < tn->ncand; ++k) {
    float ms = 0, ms2 = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, tn->e0[k], tn->e1[k]));
    CUDA_TRY(cudaEventElapsedTime(&ms2, tn->e2[k], tn->e3[k]));
    ms = std::min(ms, ms2);
    if (ms < best) {
      best = ms;
      tn->chosen = k;
    }
  }
}

static bool still_tuning(crys_ctx* ctx, const crys_db* dimdb, int qid) {
  const QueryPlan& plan = plan_for(qid);
  QueryWorkspace& ws = ws_of(ctx);
  const bool tunable = plan.joins.empty()
                           ? tune_enabled() && !flight1_forced()
                           : (plan.joins.size() == 3 || plan.joins.size() == 4) && tune_enabled() &&
                                 pipe_cfg() == 0 && l2_ahead() == 0 && split_env() == 0;
  if (!tunable) return false;
  auto it = ws.tune.find({dimdb->uid, qid});
  return it == ws.tune.end() || it->second.chosen < 0;
}

// Runs `enqueue` (stream work only) either directly or through a CUDA graph
// keyed by `key`: the launch sequence of a query is fixed for a given database
// and workspace, so after one direct run (which sizes every buffer) it is
// captured once and then replayed with ONE launch.  Not with per-query timing
// (events), columns still in flight from an async upload, or while the
// pipeline is being autotuned.  Graphs run on the context's own graph stream,
// fenced after the caller's earlier work; the caller's stream is fenced after
// them again when the scope ends.  `after` (host work that waits on the
// stream, e.g. the result copy) runs inside the scope.
template <class Enq, class After>
static void run_sequence(crys_ctx* ctx, SeqKey key, const std::vector<const crys_db*>& dbs, bool direct,
                         Enq&& enqueue, After&& after) {
  QueryWorkspace& ws = ws_of(ctx);
  if (!graphs_enabled() || ctx->timing || direct || any_pending(dbs)) {
    timing_begin(ctx);
    enqueue();
    after();
    timing_end(ctx);
    return;
  }
  QueryGraph& g = ws.graphs[key];
  if (!ctx->graph_stream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->graph_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->graph_fence, cudaEventDisableTiming));
  }
  struct StreamSwap {
    crys_ctx* c;
    cudaStream_t saved;
    ~StreamSwap() {
      // the caller's later work orders after everything this scope enqueued
      cudaEventRecord(c->graph_fence, c->stream);
      c->stream = saved;
      cudaStreamWaitEvent(saved, c->graph_fence, 0);
    }
  };
  CUDA_TRY(cudaEventRecord(ctx->graph_fence, ctx->stream));
  CUDA_TRY(cudaStreamWaitEvent(ctx->graph_stream, ctx->graph_fence, 0));
  StreamSwap swap{ctx, ctx->stream};
  ctx->stream = ctx->graph_stream;
  const std::vector<uintptr_t> sig = query_signature(ctx, dbs);
  if (g.sig != sig) {  // first run (or a changed layout): direct, then remember the layout
    if (g.exec) {
      cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
    }
    enqueue();
    after();
    g.sig = query_signature(ctx, dbs);
    return;
  }
  if (!g.exec) {
    const int64_t launches0 = ctx->launches;
    cudaGraph_t graph;
    CUDA_TRY(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
    try {
      enqueue();
    } catch (...) {
      cudaStreamEndCapture(ctx->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    CUDA_TRY(cudaStreamEndCapture(ctx->stream, &graph));
    CUDA_TRY(cudaGraphInstantiate(&g.exec, graph, 0));
    CUDA_TRY(cudaGraphDestroy(graph));
    g.kernels = ctx->launches - launches0;
    ctx->launches = launches0;
  }
  CUDA_TRY(cudaGraphLaunch(g.exec, ctx->stream));
  ctx->launches += g.kernels;
  after();
}

void ssb_run_query(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt, ResultRows* out) {
  const QueryPlan& plan = plan_for(qid);
  QueryWorkspace& ws = ws_of(ctx);
  const int64_t cells = plan.cells();
  CRYS_CHECK(bt > 0 && ipt > 0, CRYS_ECONFIG, "TileConfig: block_threads/items_per_thread must be positive");
  ws.agg.reserve(sizeof(unsigned long long) * (2 * (size_t)cells + 5));
  finalize_reserve(ctx, cells);
  auto* agg = ws.agg.as<unsigned long long>();
  auto* surv = agg + 2 * cells;
  auto* err = reinterpret_cast<int32_t*>(surv + 4);
  const std::vector<const crys_db*> dbs = {db};
  const BoxPlan bp = box_plan(plan, kBoxMeta);
  auto enqueue = [&] {
    ws.measuring = nullptr;
    enqueue_query(ctx, db, dbs, qid, bt, ipt, agg, surv, err, ws.result.as<unsigned long long>(),
                  sizeof(ResultHeader) / 8, true, true, nullptr);
    finalize_enqueue(ctx, qid, agg, agg + cells, bp, false, surv, err, nullptr, true);
  };
  auto after = [&] {
    finalize_host_part(ctx, qid, out);
    tune_done(ctx);
  };
  run_sequence(ctx, SeqKey{db->uid, qid, kSeqQuery}, dbs, still_tuning(ctx, db, qid), enqueue, after);
}

// ---------------------------------------------------------- packed partials

// Host view of the box published by box_publish_kernel.
static crys_group_box host_box(const QueryPlan& plan, const HostBox* hb) {
  crys_group_box b;
  std::memset(&b, 0, sizeof(b));
  b.nparts = (int32_t)plan.group.size();
  b.cells = 1;
  for (int g = 0; g < b.nparts; ++g) {
    const GroupPart& gp = plan.group[g];
    const int32_t full = gp.hi - gp.lo + 1;
    const int32_t lo = std::max(0, hb->dmin[gp.join_index]);
    const int32_t hi = std::min(full - 1, hb->dmax[gp.join_index]);
    b.lo[g] = gp.lo + (hi >= lo ? lo : 0);  // an empty part keeps its domain's low value
    b.card[g] = hi >= lo ? hi - lo + 1 : 0;
    b.cells *= b.card[g];
  }
  return b;
}

static HostBox* host_box_buffer(QueryWorkspace& ws) {
  if (!ws.hbox) {
    void* p = nullptr;
    CUDA_TRY(cudaHostAlloc(&p, sizeof(HostBox), cudaHostAllocMapped | cudaHostAllocPortable));
    ws.hbox = static_cast<HostBox*>(p);
    std::memset(p, 0, sizeof(HostBox));
  }
  return ws.hbox;
}

// Waits for box_publish_kernel (spin on host-mapped memory; the stream keeps
// running the fused pass meanwhile).
static void wait_box(crys_ctx* ctx, HostBox* hb) {
  for (uint64_t spins = 0; hb->ready == 0; ++spins) {
    if ((spins & 1023) == 1023) {
      const cudaError_t e = cudaStreamQuery(ctx->stream);
      if (e != cudaSuccess && e != cudaErrorNotReady)
        fail(CRYS_ECUDA, std::string("waiting for the dimension builds: ") + cudaGetErrorString(e));
      if (e == cudaSuccess && hb->ready == 0) fail(CRYS_ECUDA, "dimension builds finished without a box");
    }
  }
}

// One shard group's partial on this device (dimensions from facts[0]):
// prologue + builds + box publish + fused passes over every fact shard +
// pack into d_out (capacity `cap` int64).  Returns with *box / *len set while
// the fused pass may still run.  Graph-replayed like a query.
void ssb_partial_box(crys_ctx* ctx, const std::vector<const crys_db*>& facts, int qid, int bt, int ipt,
                     long long* d_out, int64_t cap, crys_group_box* box, int64_t* len, bool defer_tune) {
  const QueryPlan& plan = plan_for(qid);
  QueryWorkspace& ws = ws_of(ctx);
  const int64_t cells = plan.cells();
  const int nj = (int)plan.joins.size();
  CRYS_CHECK(bt > 0 && ipt > 0, CRYS_ECONFIG, "TileConfig: block_threads/items_per_thread must be positive");
  CRYS_CHECK(d_out != nullptr, CRYS_ECONFIG, "null partial buffer");
  ws.agg.reserve(sizeof(unsigned long long) * (2 * (size_t)cells + 5));
  ws.meta.reserve(sizeof(HtMeta) * kMaxJoins);
  HostBox* hb = nj ? host_box_buffer(ws) : nullptr;
  auto* agg = ws.agg.as<unsigned long long>();
  auto* surv = agg + 2 * cells;
  auto* err = reinterpret_cast<int32_t*>(surv + 4);
  const BoxPlan bp = box_plan(plan, kBoxMeta);
  if (hb) hb->ready = 0;
  auto enqueue = [&] {
    ws.measuring = nullptr;
    enqueue_query(ctx, facts[0], facts, qid, bt, ipt, agg, surv, err, nullptr, 0, true, true, hb);
    const int tpb = 256;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((cells + tpb - 1) / tpb, (int64_t)ctx->num_sms * 8));
    pack_partial_kernel<<<grid, tpb, 0, ctx->stream>>>(agg, agg + cells, bp, ws.meta.as<HtMeta>(), nj, surv,
                                                       err, d_out, cap);
    CRYS_LAUNCHED("pack_partial_kernel");
    count_launch(ctx);
  };
  auto after = [&] {
    if (hb) {
      wait_box(ctx, hb);
      *box = host_box(plan, hb);
    } else {
      std::memset(box, 0, sizeof(*box));
      box->cells = 1;
    }
    *len = CRYS_PARTIAL_HEADER + 2 * box->cells;
    CRYS_CHECK(*len <= cap, CRYS_ECONTRACT,
               "partial buffer too small: need " + std::to_string(*len) + " int64");
    if (!defer_tune) {
      if (ws.measuring) CUDA_TRY(cudaStreamSynchronize(ctx->stream));
      tune_done(ctx);
    }
  };
  std::vector<const crys_db*> dbs(facts.begin(), facts.end());
  run_sequence(ctx, SeqKey{facts[0]->uid, qid, kSeqPartial}, dbs, still_tuning(ctx, facts[0], qid), enqueue,
               after);
}

void ssb_tune_done(crys_ctx* ctx) {
  if (ctx->qws && ctx->qws->measuring) {
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    tune_done(ctx);
  }
}

long long* ssb_group_buffer(crys_ctx* ctx, int64_t n) {
  QueryWorkspace& ws = ws_of(ctx);
  ws.packed.reserve(sizeof(long long) * (size_t)n);
  return ws.packed.as<long long>();
}

}  // namespace crys
