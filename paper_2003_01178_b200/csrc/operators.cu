// operators.cu -- selection, projection and hash-join microbenchmark kernels.
//
//   select_rr_ws_kernel    select_{branching,predicated}_into(workers=1)
//                          (select.hpp:56-91): input-order output, persistent
//                          round-robin over L2-sized segments (count warps read
//                          HBM, write warps re-read L2 two rounds later, both
//                          roles in every CTA; select_rr_kernel alternates the
//                          two phases in all warps, CRYS_SEL_RR=12); select_seg_kernel
//                          (segmented launches) and select_input_kernel
//                          (decoupled look-back) are the A/B forms
//   select_rr_crystal_ws_kernel / select_rr_crystal_kernel /
//   select_crystal_reg_kernel / select_crystal_kernel
//                          select_tile_into(config, kDeterministic)
//                          (select.hpp:107-135): the exact Crystal order for any
//                          TileConfig (round-robin units of 32 logical threads
//                          when bt % 32 == 0 and ipt is a power of two <= 16)
//   project_kernel         project_{linear,sigmoid}_into (project.hpp:21-64)
//   ht_init/insert_kernel  HashTable::build (hash_table.cpp:20-94)
//   join_probe_kernel      join_probe_* (join.cpp:11-96): Q4 checksum, the
//                          table staged in shared memory when it fits, else
//                          probed L2/HBM-resident
#include <algorithm>
#include <map>
#include <tuple>
#include <mutex>

#include "async.cuh"
#include "crystal.cuh"
#include "internal.hpp"

namespace crys {
namespace {

// Each write-pass tile bulk-prefetches tile + k into L2 when that tile has
// matches (CRYS_SEL_L2=k, 0 = off; default 592 = four CTAs per SM ahead:
// sigma 0.5 1.007 -> 0.965 ms on B200).
int sel_l2_ahead() {
  static const int v = [] {
    const char* e = getenv("CRYS_SEL_L2");
    return e ? atoi(e) : 592;
  }();
  return v;
}

// A/B knob for the input-order select: 0 = segmented (default), 1 = single
// pass with a decoupled look-back, 3 = count / scan / write (all produce the
// same result).
int sel_cfg() {
  static const int cfg = [] {
    const char* e = getenv("CRYS_SEL_CFG");
    return e ? atoi(e) : 0;
  }();
  return cfg;
}

// CRYS_SEL_PDL=0: launch the segments without programmatic dependent launch.
bool sel_pdl() {
  static const bool v = [] {
    const char* e = getenv("CRYS_SEL_PDL");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

// CRYS_SEL_SEG: tiles per segment of the segmented select (multiple of 64).
long long sel_seg() {
  static const long long v = [] {
    const char* e = getenv("CRYS_SEL_SEG");
    const long long x = e ? atoll(e) : 32768;
    return std::max(64ll, x / 64 * 64);
  }();
  return v;
}

// Input-order selection (select_branching/predicated_into, workers=1: output
// in input order).  Tile layout is WARP-CONTIGUOUS: warp w owns slots [w*32*IPT, (w+1)*32*IPT),
// lane l's vector v is the 4 slots at w*32*IPT + v*128 + 4*l, so a warp's
// order is (v, lane, element) and every load is a 128-bit coalesced read.
// Positions come from per-vector warp scans (popc + shuffles) and one barrier
// for the warp totals; the compacted tile is staged in shared memory and
// stored with coalesced writes.
template <int BT, int IPT>
struct SelTile {
  static constexpr int TILE = BT * IPT;
  static constexpr int W = BT / 32;
  static_assert(IPT % 4 == 0, "128-bit vectors");
};

__device__ __forceinline__ int4 ld_hint4(const int32_t* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// POL: 0 = default L2 policy, 1 = evict_last, 2 = evict_first
template <int BT, int IPT, int POL = 0>
__device__ __forceinline__ void sel_load(const int32_t* __restrict__ in, int64_t base, int valid,
                                         int4 (&v)[IPT / 4]) {
  uint64_t pol = 0;
  if constexpr (POL == 1) pol = pipe::policy_evict_last();
  if constexpr (POL == 2) pol = pipe::policy_evict_first();
  const int wb = (threadIdx.x >> 5) * 32 * IPT + 4 * (int)lane_id();
  // tiles are 16 KB apart, so one check of the span's base decides the path
  const bool vec_ok = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
#pragma unroll
  for (int j = 0; j < IPT / 4; ++j) {
    const int s = wb + j * 128;
    if (vec_ok && s + 4 <= valid) {
      if constexpr (POL == 0) v[j] = ld_stream4(in + base + s);
      else v[j] = ld_hint4(in + base + s, pol);
    } else {
      v[j] = make_int4(0, 0, 0, 0);
      if (s + 0 < valid) v[j].x = ld_stream1(in + base + s + 0);
      if (s + 1 < valid) v[j].y = ld_stream1(in + base + s + 1);
      if (s + 2 < valid) v[j].z = ld_stream1(in + base + s + 2);
      if (s + 3 < valid) v[j].w = ld_stream1(in + base + s + 3);
    }
  }
}

// Per-vector predicate bits and warp-local positions of one tile; the block
// total via one barrier.  Returns the tile's match count; woff = this warp's
// offset inside the tile.
template <int BT, int IPT>
__device__ __forceinline__ int sel_count(const int4 (&v)[IPT / 4], int valid, int32_t lo, int32_t hi,
                                         int* s_warp, unsigned (&bits)[IPT / 4], int (&pos)[IPT / 4],
                                         int& woff) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const int wb = warp * 32 * IPT + 4 * (int)lane;
  int run = 0;
#pragma unroll
  for (int j = 0; j < IPT / 4; ++j) {
    const int s = wb + j * 128;
    unsigned b = 0;
    b |= (unsigned)(s + 0 < valid && v[j].x >= lo && v[j].x <= hi) << 0;
    b |= (unsigned)(s + 1 < valid && v[j].y >= lo && v[j].y <= hi) << 1;
    b |= (unsigned)(s + 2 < valid && v[j].z >= lo && v[j].z <= hi) << 2;
    b |= (unsigned)(s + 3 < valid && v[j].w >= lo && v[j].w <= hi) << 3;
    bits[j] = b;
    const int c = __popc(b);
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if ((int)lane >= o) x += y;
    }
    pos[j] = run + x - c;
    run += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 31) s_warp[warp] = run;
  __syncthreads();
  int total = 0;
  woff = 0;
#pragma unroll
  for (int w = 0; w < BT / 32; ++w) {
    const int t = s_warp[w];
    woff += (w < (int)warp) ? t : 0;
    total += t;
  }
  return total;
}

template <int IPT>
__device__ __forceinline__ void sel_scatter(const int4 (&v)[IPT / 4], const unsigned (&bits)[IPT / 4],
                                            const int (&pos)[IPT / 4], int woff, int32_t* s_items) {
#pragma unroll
  for (int j = 0; j < IPT / 4; ++j) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(s_items + woff + pos[j]);
    const uint32_t b = bits[j];
    sts_if(a, v[j].x, b & 1u);
    a += 4u * (b & 1u);
    sts_if(a, v[j].y, b & 2u);
    a += 2u * (b & 2u);
    sts_if(a, v[j].z, b & 4u);
    a += b & 4u;
    sts_if(a, v[j].w, b & 8u);
  }
}

// Compacts one tile into s_items; returns the tile's match count.
template <int BT, int IPT>
__device__ __forceinline__ int sel_compact(const int4 (&v)[IPT / 4], int valid, int32_t lo, int32_t hi,
                                           int32_t* s_items, int* s_warp) {
  unsigned bits[IPT / 4];
  int pos[IPT / 4];
  int woff;
  const int total = sel_count<BT, IPT>(v, valid, lo, hi, s_warp, bits, pos, woff);
  sel_scatter<IPT>(v, bits, pos, woff, s_items);
  return total;
}

// Single-pass form (A/B only, CRYS_SEL_CFG=1): one tile per CTA (tile =
// blockIdx.x, dispatch order), block-wide decoupled look-back.  Correct, but
// the look-back latency under load makes it slower than reduce-then-scan
// (profiles/r01_select_tuning.txt).
template <int BT, int IPT>
__global__ void __launch_bounds__(BT) select_input_kernel(const int32_t* __restrict__ in, int64_t n,
                                                          int32_t lo, int32_t hi,
                                                          int32_t* __restrict__ out,
                                                          unsigned long long* status,
                                                          long long ntiles, long long* total_out) {
  using T = SelTile<BT, IPT>;
  __shared__ __align__(16) int32_t s_items[T::TILE];
  __shared__ int s_warp[T::W];
  __shared__ long long s_red[T::W + T::W / 2 + 1];
  const long long tile = blockIdx.x;
  const int64_t base = tile * T::TILE;
  const int valid = (int)min((int64_t)T::TILE, (int64_t)(n - base));
  int4 v[IPT / 4];
  sel_load<BT, IPT>(in, base, valid, v);
  const int total = sel_compact<BT, IPT>(v, valid, lo, hi, s_items, s_warp);
  const long long off = block_lookback<BT>(status, tile, total, s_red);
  for (int i = threadIdx.x; i < total; i += BT) out[off + i] = s_items[i];
  if (threadIdx.x == 0 && tile == ntiles - 1) *total_out = off + total;
}

// Reduce-then-scan form (no look-back latency on the critical path): pass 1
// streams the input and writes one count per tile, a single CTA scans the
// counts, pass 2 re-streams the input and writes every tile at its known
// offset.  8N + 4*matched bytes instead of 4N + 4*matched, but both passes
// are pure streaming (measured on B200: a tile's chained look-back costs ~7 us
// under full HBM load, 4x its load).
template <int BT, int IPT>
__global__ void __launch_bounds__(BT) select_count_kernel(const int32_t* __restrict__ in, int64_t n,
                                                          int32_t lo, int32_t hi, long long ntiles,
                                                          unsigned* counts) {
  using T = SelTile<BT, IPT>;
  __shared__ int s_warp[T::W];
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * T::TILE;
    const int valid = (int)min((int64_t)T::TILE, (int64_t)(n - base));
    int4 v[IPT / 4];
    sel_load<BT, IPT>(in, base, valid, v);
    const unsigned lane = lane_id();
    const int wb = (threadIdx.x >> 5) * 32 * IPT + 4 * (int)lane;
    int c = 0;
#pragma unroll
    for (int j = 0; j < IPT / 4; ++j) {
      const int s0 = wb + j * 128;
      c += (s0 + 0 < valid && v[j].x >= lo && v[j].x <= hi) + (s0 + 1 < valid && v[j].y >= lo && v[j].y <= hi) +
           (s0 + 2 < valid && v[j].z >= lo && v[j].z <= hi) + (s0 + 3 < valid && v[j].w >= lo && v[j].w <= hi);
    }
    c = warp_sum(c);
    if (lane == 0) s_warp[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
#pragma unroll
      for (int w = 0; w < T::W; ++w) t += s_warp[w];
      counts[tile] = (unsigned)t;
    }
    __syncthreads();
  }
}

// Exclusive scan of the per-tile counts, two tiny kernels with coalesced
// 128-bit reads (a single CTA walking 131 K counts serially took 119 us):
// select_scan_local_kernel scans each 4096-count block into local offsets and
// a block total; select_scan_blocks_kernel scans the block totals into bases
// (bases[nblk] = the grand total).  Offset of tile c = local[c] + bases[c>>12].
constexpr int kScanBlk = 4096;
__global__ void __launch_bounds__(1024) select_scan_local_kernel(const unsigned* counts, long long ntiles,
                                                                 long long* local, long long* btot) {
  __shared__ long long sm[33];
  const long long b0 = (long long)blockIdx.x * kScanBlk + 4 * threadIdx.x;
  unsigned v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = b0 + k < ntiles ? counts[b0 + k] : 0u;
  const long long mine = (long long)v[0] + v[1] + v[2] + v[3];
  long long tot;
  long long run = BlockScan<1024>(mine, sm, tot);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (b0 + k < ntiles) local[b0 + k] = run;
    run += v[k];
  }
  if (threadIdx.x == 0) btot[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) select_scan_blocks_kernel(const long long* btot, int nblk,
                                                                  long long* bases) {
  __shared__ long long sm[33];
  long long run = 0;
  for (int b0 = 0; b0 < nblk; b0 += 1024) {  // nblk <= 1024 for < 2^32 rows
    const long long v = b0 + (int)threadIdx.x < nblk ? btot[b0 + threadIdx.x] : 0;
    long long tot;
    const long long ex = BlockScan<1024>(v, sm, tot);
    if (b0 + (int)threadIdx.x < nblk) bases[b0 + threadIdx.x] = run + ex;
    run += tot;
  }
  if (threadIdx.x == 0) bases[nblk] = run;
}

__device__ __forceinline__ long long sel_offset(const long long* local, const long long* bases, long long c,
                                                long long ntiles) {
  return c < ntiles ? local[c] + bases[c / kScanBlk] : bases[(ntiles + kScanBlk - 1) / kScanBlk];
}

template <int BT, int IPT>
__global__ void __launch_bounds__(BT) select_write_kernel(const int32_t* __restrict__ in, int64_t n,
                                                          int32_t lo, int32_t hi, long long ntiles,
                                                          const long long* local, const long long* bases,
                                                          int32_t* __restrict__ out, int l2_ahead) {
  using T = SelTile<BT, IPT>;
  __shared__ __align__(16) int32_t s_items[T::TILE];
  __shared__ int s_warp[T::W];
  const long long tile = blockIdx.x;
  const int64_t base = tile * T::TILE;
  const int valid = (int)min((int64_t)T::TILE, (int64_t)(n - base));
  const long long off = sel_offset(local, bases, tile, ntiles);
  const int total = (int)(sel_offset(local, bases, tile + 1, ntiles) - off);
  if (total == 0) return;  // whole CTA: uniform
  if (l2_ahead > 0 && threadIdx.x == 0) {  // the tile ~one resident wave later, if it has matches: into L2
    const long long pt = tile + l2_ahead;
    const int64_t pb = pt * T::TILE;
    if (pb + T::TILE <= n && (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
        sel_offset(local, bases, pt + 1, ntiles) != sel_offset(local, bases, pt, ntiles))
      pipe::l2_prefetch_bulk(in + pb, 4u * T::TILE);
  }
  int4 v[IPT / 4];
  sel_load<BT, IPT>(in, base, valid, v);
  sel_compact<BT, IPT>(v, valid, lo, hi, s_items, s_warp);
  __syncthreads();
  for (int i = threadIdx.x; i < total; i += BT) out[off + i] = s_items[i];
}

// Segmented select (the default input-order path).  The input is cut into
// segments of `seg` tiles and launch s runs two roles side by side: COUNT
// CTAs stream segment s and publish per-tile counts (plus 64-tile group sums
// and the segment total, by atomics); WRITE CTAs re-read segment s - 1,
// counted by the previous launch, and write each tile at its offset = the
// segment totals before it + the group sums before it in its segment + the
// tile counts before it in its group (one round of loads per CTA: no scan
// kernel, no look-back).  Launches are chained with programmatic dependent
// launch: the next launch's count CTAs start while this one drains, and only
// its write CTAs wait (griddepcontrol.wait) for this grid.
//
// Measured on B200 (2^29 rows, profiles/r01_select_segmented.txt): with
// seg = 32768 (512 MB) the mixed roles and the missing scan kernels beat
// count / scan / write by 8-20 %.  Segments of <= 32 MB with evict_last on
// the count read DO make the re-read an L2 hit (DRAM reads 2.15 GB instead of
// 4.2 GB; the default policy keeps < 16 MB of a stream), but the extra
// launches cost more than the HBM bytes saved, so they are off by default
// (CRYS_SEL_SEG).
constexpr int kSegGroup = 64;

template <int BT, int IPT, bool HINT>
__global__ void __launch_bounds__(BT) select_seg_kernel(const int32_t* __restrict__ in, int64_t n, int32_t lo,
                                                        int32_t hi, int32_t* __restrict__ out, long long ntiles,
                                                        long long seg, long long s, unsigned* counts,
                                                        unsigned* gsum, unsigned long long* stot,
                                                        long long* total_out) {
  using T = SelTile<BT, IPT>;
  __shared__ __align__(16) int32_t s_items[T::TILE];
  __shared__ int s_warp[T::W];
  __shared__ long long s_red[T::W];
  const unsigned lane = lane_id();
  // roles interleaved by CTA index so HBM (count) and L2 (write) traffic mix
  const long long c0 = s * seg, c1 = min(ntiles, c0 + seg);  // count range
  const long long w0 = c0 - seg, w1 = c0;                    // write range (segment s-1)
  const long long nc = max(0ll, c1 - c0), nw = s > 0 ? w1 - w0 : 0;
  const long long b = blockIdx.x, both = min(nc, nw);
  bool is_count;
  long long tile;
  if (b < 2 * both) {
    is_count = (b & 1) == 0;
    tile = (is_count ? c0 : w0) + (b >> 1);
  } else {
    is_count = nc > nw;
    tile = (is_count ? c0 : w0) + both + (b - 2 * both);
  }
  const int64_t base = tile * T::TILE;
  const int valid = (int)min((int64_t)T::TILE, (int64_t)(n - base));
  // programmatic dependent launch: the next launch's CTAs may start as this
  // one drains; only its WRITE role waits for this grid to complete
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  int4 v[IPT / 4];
  if (is_count) {
    sel_load<BT, IPT, HINT ? 1 : 0>(in, base, valid, v);
    const int wb = (threadIdx.x >> 5) * 32 * IPT + 4 * (int)lane;
    int c = 0;
#pragma unroll
    for (int j = 0; j < IPT / 4; ++j) {
      const int s0 = wb + j * 128;
      c += (s0 + 0 < valid && v[j].x >= lo && v[j].x <= hi) + (s0 + 1 < valid && v[j].y >= lo && v[j].y <= hi) +
           (s0 + 2 < valid && v[j].z >= lo && v[j].z <= hi) + (s0 + 3 < valid && v[j].w >= lo && v[j].w <= hi);
    }
    c = warp_sum(c);
    if (lane == 0) s_warp[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned t = 0;
#pragma unroll
      for (int w = 0; w < T::W; ++w) t += (unsigned)s_warp[w];
      counts[tile] = t;
      if (t) {
        atomicAdd(gsum + tile / kSegGroup, t);
        atomicAdd(stot + s, (unsigned long long)t);
      }
    }
    return;
  }
  // write role: offset = segments before + groups before (in segment) + tiles before (in group)
  asm volatile("griddepcontrol.wait;" ::: "memory");  // segment s-1 counted (and everything before)
  const unsigned mine = counts[tile];
  if (mine == 0) return;  // uniform; nothing to write
  sel_load<BT, IPT, HINT ? 2 : 0>(in, base, valid, v);  // in flight while the offset is summed
  const long long sw = s - 1, g = tile / kSegGroup, g0 = (sw * seg) / kSegGroup, j0 = g * kSegGroup;
  long long part = 0;
  for (long long i = threadIdx.x; i < sw; i += BT) part += (long long)stot[i];
  for (long long i = g0 + threadIdx.x; i < g; i += BT) part += gsum[i];
  for (long long i = j0 + threadIdx.x; i < tile; i += BT) part += counts[i];
  part = warp_sum(part);
  if (lane == 0) s_red[threadIdx.x >> 5] = part;
  sel_compact<BT, IPT>(v, valid, lo, hi, s_items, s_warp);  // its barrier also publishes s_red
  __syncthreads();  // s_items complete
  long long off = 0;
#pragma unroll
  for (int w = 0; w < T::W; ++w) off += s_red[w];
  for (int i = threadIdx.x; i < (int)mine; i += BT) __stcs(out + off + i, s_items[i]);
}

// Round-robin persistent select (the default input-order path): every input
// row is read from HBM ONCE, then once more from L2, with no chained
// look-back.  Grid = two co-resident CTAs per SM (cooperative launch).  Round k
// is the segment [k SEG, (k+1) SEG) (SEG = G CTAs x W warps x WU rows, ~16 MB:
// L2-sized); warp w of CTA c owns the contiguous WU rows at (c W + w) WU.
//   iteration k:  COUNT round k (128-bit loads, L2 evict_last) -> the warp's
//                 count in smem, the CTA's in counts[k][c] (+1: 0 = not yet);
//                 WRITE round k - LAG (re-read from L2, evict_first): offset =
//                 rows before the round + the round's counts of CTAs < c + the
//                 counts of warps < w; per 32-row group one ballot, stores
//                 straight to global memory in input order.
// A CTA keeps its own running base (it reads all G counts of every round),
// so the only cross-CTA dependence is "round k - LAG has been counted", which
// was published a whole count phase earlier: the exchange latency (~2 us
// under full HBM load) is hidden behind that phase instead of chaining tile
// after tile like a decoupled look-back (profiles/r01_select_tuning.txt).
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned lanemask_lt_u32() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ int32_t ld_hint1(const int32_t* p, uint64_t pol) {
  int32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}

constexpr int kRrMaxG = 32 * 10;  // counts per round read by one warp (<= 10 per lane; 2 CTAs x 148 SMs = 296)

template <int BT, int WU, int LAG, int UW>
__global__ void __launch_bounds__(BT, 2) select_rr_kernel(const int32_t* __restrict__ in, int64_t n, int32_t lo,
                                                          int32_t hi, int32_t* __restrict__ out, int rounds,
                                                          uint32_t* counts, long long* total_out) {
  constexpr int W = BT / 32;
  constexpr int PER = (kRrMaxG + 31) / 32;
  constexpr int U = WU >= 1024 ? 8 : WU / 128;  // count phase: 128-bit loads in flight per lane
  constexpr int NS = LAG + 1;                   // rounds in flight per CTA
  static_assert(WU % (128 * U) == 0 && WU % (32 * UW) == 0, "warp unit");
  __shared__ int s_wc[NS][W];
  __shared__ long long s_off;
  const int G = gridDim.x, c = blockIdx.x;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt_u32();
  const uint32_t span = (uint32_t)hi - (uint32_t)lo;  // lo <= x <= hi  <=>  x - lo <= hi - lo (unsigned)
  const int64_t seg = (int64_t)G * W * WU;
  const uint64_t keep = pipe::policy_evict_last(), drop = pipe::policy_evict_first();
  const bool vec_ok = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  long long base = 0;   // warp 0: rows selected in rounds [0, resolved)
  int resolved = 0;     // warp 0: rounds whose totals are in base
  long long mine = 0;   // thread 0: this CTA's selected rows (the grand total is their sum)
  for (int k = 0; k < rounds + LAG; ++k) {
    const int j = k - LAG;
    uint32_t cv[PER];  // warp 0: the counts of round j, in flight during the count phase
    if (warp == 0 && j >= 0) {
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int cc = i * 32 + (int)lane;
        cv[i] = cc < G ? ld_relaxed_u32(counts + (size_t)j * G + cc) : 1u;
      }
    }
    if (k < rounds) {  // ---- COUNT round k
      const int64_t r0 = k * seg + ((int64_t)c * W + warp) * WU;
      int cnt = 0;
      if (vec_ok && r0 + WU <= n) {
        for (int u = 0; u < WU; u += 128 * U) {
          int4 v[U];
#pragma unroll
          for (int q = 0; q < U; ++q) v[q] = ld_hint4(in + r0 + u + q * 128 + 4 * lane, keep);
#pragma unroll
          for (int q = 0; q < U; ++q)
            cnt += ((uint32_t)v[q].x - (uint32_t)lo <= span) + ((uint32_t)v[q].y - (uint32_t)lo <= span) +
                   ((uint32_t)v[q].z - (uint32_t)lo <= span) + ((uint32_t)v[q].w - (uint32_t)lo <= span);
        }
      } else {
        for (int64_t i = r0 + lane; i < min(r0 + WU, n); i += 32)
          cnt += (uint32_t)ld_hint1(in + i, keep) - (uint32_t)lo <= span;
      }
      cnt = warp_sum(cnt);
      if (lane == 0) s_wc[k % NS][warp] = cnt;
      __syncthreads();
      if (threadIdx.x == 0) {
        int tot = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) tot += s_wc[k % NS][w];
        st_relaxed_u32(counts + (size_t)k * G + c, (uint32_t)tot + 1u);
        mine += tot;
      }
    }
    if (j < 0) continue;  // uniform
    {  // a round this CTA selected nothing from needs no offset: no exchange wait
      int any = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) any |= s_wc[j % NS][w];
      if (!any) continue;  // uniform
    }
    if (warp == 0) {  // ---- offset of this CTA's share of round j
      for (; resolved < j; ++resolved) {  // totals of skipped rounds (rare: only near-empty selections)
        long long t = 0;
        for (int cc = (int)lane; cc < G; cc += 32) {
          uint32_t x;
          while ((x = ld_relaxed_u32(counts + (size_t)resolved * G + cc)) == 0u) __nanosleep(32);
          t += (long long)x - 1;
        }
        base += warp_sum(t);
      }
      long long before = 0, all = 0;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int cc = i * 32 + (int)lane;
        while (cv[i] == 0u) {
          __nanosleep(32);
          cv[i] = ld_relaxed_u32(counts + (size_t)j * G + cc);
        }
        const long long x = cc < G ? (long long)cv[i] - 1 : 0;
        all += x;
        before += cc < c ? x : 0;
      }
      before = warp_sum(before);
      all = warp_sum(all);
      if (lane == 0) s_off = base + before;
      base += all;
      resolved = j + 1;
    }
    __syncthreads();  // s_off published (the next write of s_off follows the next count barrier)
    // ---- WRITE round j: this warp's rows, re-read from L2, in input order
    if (s_wc[j % NS][warp] == 0) continue;  // nothing selected in this warp's rows: no re-read
    long long off = s_off;
#pragma unroll
    for (int w = 0; w < W; ++w) off += w < (int)warp ? s_wc[j % NS][w] : 0;
    int32_t* o = out + off;
    const int64_t r0 = j * seg + ((int64_t)c * W + warp) * WU;
    if (r0 + WU <= n) {
      for (int u = 0; u < WU; u += 32 * UW) {
        int32_t x[UW];
#pragma unroll
        for (int q = 0; q < UW; ++q) x[q] = ld_hint1(in + r0 + u + q * 32 + lane, drop);
#pragma unroll
        for (int q = 0; q < UW; ++q) {
          const bool p = (uint32_t)x[q] - (uint32_t)lo <= span;
          const unsigned m = __ballot_sync(0xffffffffu, p);
          if (p) __stcs(o + __popc(m & lt), x[q]);
          o += __popc(m);
        }
      }
    } else {
      for (int64_t i0 = r0; i0 < min(r0 + WU, n); i0 += 32) {
        const int64_t i = i0 + lane;
        const int32_t x = i < n ? ld_hint1(in + i, drop) : 0;
        const bool p = i < n && (uint32_t)x - (uint32_t)lo <= span;
        const unsigned m = __ballot_sync(0xffffffffu, p);
        if (p) __stcs(o + __popc(m & lt), x);
        o += __popc(m);
      }
    }
  }
  if (threadIdx.x == 0 && mine) atomicAdd(reinterpret_cast<unsigned long long*>(total_out), (unsigned long long)mine);
}

// Warp-specialised form of select_rr_kernel (same rounds, counts and output):
// warps [0, W/2) only COUNT (HBM, evict_last) and warps [W/2, W) only WRITE
// (L2 re-read, evict_first), each role synchronised on its own named barrier,
// both joined once per iteration.  In the phase-alternating kernel every CTA
// (and, through the count exchange, the whole grid) alternates between an
// HBM read burst and an L2-read / HBM-write burst, so an iteration costs
// t_count + t_write; here the two overlap inside every SM.  Write warp ww
// re-reads the rows count warp ww counted LAG iterations earlier; write warp 0
// loads the next round's CTA counts at the end of an iteration so the
// exchange read is in flight across the iteration barrier.
// PF 1: each count warp bulk-prefetches its NEXT round's rows into L2 as it
// starts counting this round's (more HBM bytes in flight than its registers hold; half the
// warps count, so a count-only round -- sigma = 0 -- is otherwise short of
// memory-level parallelism: sigma 0 0.39 -> 0.37 ms), but the extra L2
// footprint pushes counted rows out before the write warps re-read them
// (sigma 0.5 0.65 -> 0.73 ms), so it is off by default; prefetching only after
// rounds the CTA selected nothing from measured 0.41 ms at sigma 0 and was dropped.
// VW: the write warps re-read their rows with 128-bit loads (UW int4 per lane
// in flight), place each lane's matches in a per-warp shared staging buffer
// with predicated stores at positions from four ballots, and copy the batch
// out coalesced (the scalar form issues one 4-byte load, ballot and store per
// 32 rows).
template <int BT, int WU, int LAG, int UW, int U, int PF = 0, bool VW = false>
__global__ void __launch_bounds__(BT, 2) select_rr_ws_kernel(const int32_t* __restrict__ in, int64_t n, int32_t lo,
                                                             int32_t hi, int32_t* __restrict__ out, int rounds,
                                                             uint32_t* counts, long long* total_out) {
  constexpr int W = BT / 32, CW = W / 2;
  constexpr int PER = (kRrMaxG + 31) / 32;
  constexpr int NS = LAG + 1;
  static_assert(W % 2 == 0 && WU % (128 * U) == 0 && WU % (32 * UW) == 0, "warp unit");
  static_assert(!VW || WU % (128 * UW) == 0, "vector write batch");
  __shared__ int s_wc[NS][CW];
  __shared__ long long s_off;
  __shared__ int32_t s_wst[VW ? CW * 128 * UW : 1];  // VW: per write warp, one batch of compacted rows
  const int G = gridDim.x, c = blockIdx.x;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt_u32();
  const uint32_t span = (uint32_t)hi - (uint32_t)lo;
  const int64_t seg = (int64_t)G * CW * WU;
  const bool vec_ok = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  long long base = 0;  // write warp 0: rows selected in rounds [0, resolved)
  int resolved = 0;
  long long mine = 0;  // thread 0: this CTA's selected rows
  uint32_t cv[PER];    // write warp 0: the counts of the next round to write
#pragma unroll
  for (int i = 0; i < PER; ++i) cv[i] = 0u;
  for (int k = 0; k < rounds + LAG; ++k) {
    const int j = k - LAG;
    if (warp < CW) {
      if (k < rounds) {  // ---- COUNT round k
        const uint64_t keep = pipe::policy_evict_last();
        const int64_t r0 = k * seg + ((int64_t)c * CW + warp) * WU;
        if constexpr (PF == 1) {  // in flight alongside this round's loads
          const int64_t rn = r0 + seg;
          if (lane == 0 && vec_ok && rn + WU <= n) pipe::l2_prefetch_bulk(in + rn, 4u * WU);
        }
        int cnt = 0;
        if (vec_ok && r0 + WU <= n) {
          for (int u = 0; u < WU; u += 128 * U) {
            int4 v[U];
#pragma unroll
            for (int q = 0; q < U; ++q) v[q] = ld_hint4(in + r0 + u + q * 128 + 4 * lane, keep);
#pragma unroll
            for (int q = 0; q < U; ++q)
              cnt += ((uint32_t)v[q].x - (uint32_t)lo <= span) + ((uint32_t)v[q].y - (uint32_t)lo <= span) +
                     ((uint32_t)v[q].z - (uint32_t)lo <= span) + ((uint32_t)v[q].w - (uint32_t)lo <= span);
          }
        } else {
          for (int64_t i = r0 + lane; i < min(r0 + WU, n); i += 32)
            cnt += (uint32_t)ld_hint1(in + i, keep) - (uint32_t)lo <= span;
        }
        cnt = warp_sum(cnt);
        if (lane == 0) s_wc[k % NS][warp] = cnt;
        asm volatile("bar.sync 1, %0;" ::"n"(BT / 2) : "memory");  // count warps only
        if (threadIdx.x == 0) {
          int tot = 0;
#pragma unroll
          for (int w = 0; w < CW; ++w) tot += s_wc[k % NS][w];
          st_relaxed_u32(counts + (size_t)k * G + c, (uint32_t)tot + 1u);
          mine += tot;
        }
      }
    } else if (j >= 0) {
      const int ww = (int)warp - CW;
      int any = 0;
#pragma unroll
      for (int w = 0; w < CW; ++w) any |= s_wc[j % NS][w];
      if (any) {  // uniform over the write warps
        if (ww == 0) {  // ---- offset of this CTA's share of round j
          for (; resolved < j; ++resolved) {  // totals of skipped rounds
            long long t = 0;
            for (int cc = (int)lane; cc < G; cc += 32) {
              uint32_t x;
              while ((x = ld_relaxed_u32(counts + (size_t)resolved * G + cc)) == 0u) __nanosleep(32);
              t += (long long)x - 1;
            }
            base += warp_sum(t);
          }
          long long before = 0, all = 0;
#pragma unroll
          for (int i = 0; i < PER; ++i) {
            const int cc = i * 32 + (int)lane;
            if (cc < G)
              while (cv[i] == 0u) {  // not prefetched / not yet published
                cv[i] = ld_relaxed_u32(counts + (size_t)j * G + cc);
                if (cv[i] == 0u) __nanosleep(32);
              }
            const long long x = cc < G ? (long long)cv[i] - 1 : 0;
            all += x;
            before += cc < c ? x : 0;
          }
          before = warp_sum(before);
          all = warp_sum(all);
          if (lane == 0) s_off = base + before;
          base += all;
          resolved = j + 1;
        }
        asm volatile("bar.sync 2, %0;" ::"n"(BT / 2) : "memory");  // write warps only: s_off published
        if (s_wc[j % NS][ww] != 0) {  // ---- WRITE this warp's rows of round j, re-read from L2
          const uint64_t drop = pipe::policy_evict_first();
          long long off = s_off;
#pragma unroll
          for (int w = 0; w < CW; ++w) off += w < ww ? s_wc[j % NS][w] : 0;
          int32_t* o = out + off;
          const int64_t r0 = j * seg + ((int64_t)c * CW + ww) * WU;
          if (VW && vec_ok && r0 + WU <= n) {
            int32_t* wb = s_wst + ww * (128 * UW);
            const uint32_t wb_s = (uint32_t)__cvta_generic_to_shared(wb);
            for (int u = 0; u < WU; u += 128 * UW) {
              int4 v[UW];
#pragma unroll
              for (int q = 0; q < UW; ++q) v[q] = ld_hint4(in + r0 + u + q * 128 + 4 * lane, drop);
              int pos = 0;
#pragma unroll
              for (int q = 0; q < UW; ++q) {
                const bool p0 = (uint32_t)v[q].x - (uint32_t)lo <= span, p1 = (uint32_t)v[q].y - (uint32_t)lo <= span;
                const bool p2 = (uint32_t)v[q].z - (uint32_t)lo <= span, p3 = (uint32_t)v[q].w - (uint32_t)lo <= span;
                const unsigned b0 = __ballot_sync(0xffffffffu, p0), b1 = __ballot_sync(0xffffffffu, p1);
                const unsigned b2 = __ballot_sync(0xffffffffu, p2), b3 = __ballot_sync(0xffffffffu, p3);
                // rows before this lane's 4: all matches of lanes < lane (input order = lane, element)
                const int ex = __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
                uint32_t a = wb_s + 4u * (uint32_t)(pos + ex);
                sts_if(a, v[q].x, p0);
                a += 4u * p0;
                sts_if(a, v[q].y, p1);
                a += 4u * p1;
                sts_if(a, v[q].z, p2);
                a += 4u * p2;
                sts_if(a, v[q].w, p3);
                pos += __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
              }
              __syncwarp();
              for (int i = (int)lane; i < pos; i += 32) __stcs(o + i, wb[i]);
              o += pos;
              __syncwarp();
            }
          } else if (r0 + WU <= n) {
            for (int u = 0; u < WU; u += 32 * UW) {
              int32_t x[UW];
#pragma unroll
              for (int q = 0; q < UW; ++q) x[q] = ld_hint1(in + r0 + u + q * 32 + lane, drop);
#pragma unroll
              for (int q = 0; q < UW; ++q) {
                const bool p = (uint32_t)x[q] - (uint32_t)lo <= span;
                const unsigned m = __ballot_sync(0xffffffffu, p);
                if (p) __stcs(o + __popc(m & lt), x[q]);
                o += __popc(m);
              }
            }
          } else {
            for (int64_t i0 = r0; i0 < min(r0 + WU, n); i0 += 32) {
              const int64_t i = i0 + lane;
              const int32_t x = i < n ? ld_hint1(in + i, drop) : 0;
              const bool p = i < n && (uint32_t)x - (uint32_t)lo <= span;
              const unsigned m = __ballot_sync(0xffffffffu, p);
              if (p) __stcs(o + __popc(m & lt), x);
              o += __popc(m);
            }
          }
        }
      }
      if (ww == 0) {  // the next round's counts: in flight across the barrier
        const int jn = j + 1;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int cc = i * 32 + (int)lane;
          cv[i] = (jn < rounds && cc < G) ? ld_relaxed_u32(counts + (size_t)jn * G + cc) : 0u;
        }
      }
    }
    __syncthreads();  // s_wc of round k visible to the write warps; slot (k+1) % NS free
  }
  if (threadIdx.x == 0 && mine) atomicAdd(reinterpret_cast<unsigned long long*>(total_out), (unsigned long long)mine);
}

// Walks units (logical tile, 32-thread group) in order from unit u0 with one
// division: next() = this lane's first slot of the next unit.
struct UnitCursor {
  int64_t tile_base, lane_off;
  int m, gpt;
  int64_t S;
  __device__ UnitCursor(int64_t u0, int gpt_, int64_t S_, unsigned lane) : gpt(gpt_), S(S_) {
    tile_base = (u0 / gpt_) * S_;
    m = (int)(u0 % gpt_);
    lane_off = lane;
  }
  __device__ __forceinline__ int64_t next() {
    const int64_t s = tile_base + (int64_t)m * 32 + lane_off;
    if (++m == gpt) {
      m = 0;
      tile_base += S;
    }
    return s;
  }
};

// Crystal order (select_tile_into, select.hpp:107-135) on the same
// round-robin scheme, for tiles whose bt is a multiple of 32 and ipt a power
// of two <= 16 (IPTM == ipt: compile-time slot loops).
// The output of logical tile j is thread-major: logical thread t's matches
// (slots j S + t + k bt, k < ipt, in k order), t = 0 .. bt-1.  A UNIT is 32
// consecutive logical threads (j, m): t = 32 m + lane, so a unit's output is
// contiguous and units in (j, m) order are output order.  Lane loads its ipt
// slots (for fixed k the 32 lanes read 128 consecutive bytes), one warp scan
// of the per-lane counts places the unit.  Warp w of CTA c owns UPW
// consecutive units per round; counts and offsets as in select_rr_kernel.
template <int BT, int IPTM, int LAG>
__global__ void __launch_bounds__(BT, 2) select_rr_crystal_kernel(const int32_t* __restrict__ in, int64_t n,
                                                                  int32_t lo, int32_t hi, int bt, int ipt,
                                                                  int32_t* __restrict__ out, int rounds,
                                                                  uint32_t* counts, long long* total_out) {
  constexpr int W = BT / 32;
  constexpr int UPW = 1024 / (32 * IPTM) > 0 ? 1024 / (32 * IPTM) : 1;  // units per warp per round
  constexpr int NB = IPTM >= 16 ? 1 : 16 / IPTM;                        // units per batch of loads
  static_assert(UPW % NB == 0, "batches");
  constexpr int PER = (kRrMaxG + 31) / 32;
  constexpr int NS = LAG + 1;
  __shared__ int s_wc[NS][W];
  __shared__ long long s_off;
  __shared__ int32_t s_stage[W * NB * 32 * IPTM];  // per warp: one batch of compacted output
  const int G = gridDim.x, c = blockIdx.x;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t span = (uint32_t)hi - (uint32_t)lo;
  const int gpt = bt >> 5;                   // units (32-thread groups) per logical tile
  const int64_t S = (int64_t)bt * IPTM;      // slots per logical tile (ipt == IPTM)
  const int64_t upr = (int64_t)G * W * UPW;  // units per round
  const uint64_t keep = pipe::policy_evict_last(), drop = pipe::policy_evict_first();
  // a warp's UPW units are whole logical tiles: count over a contiguous range
  const bool whole = UPW % gpt == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  long long base = 0;
  int resolved = 0;
  long long mine = 0;
  for (int k = 0; k < rounds + LAG; ++k) {
    const int j = k - LAG;
    uint32_t cv[PER];
    if (warp == 0 && j >= 0) {
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int cc = i * 32 + (int)lane;
        cv[i] = cc < G ? ld_relaxed_u32(counts + (size_t)j * G + cc) : 1u;
      }
    }
    if (k < rounds) {  // ---- COUNT round k: this warp's UPW units (order does not matter here)
      const int64_t u0 = k * upr + ((int64_t)c * W + warp) * UPW;
      int cnt = 0;
      if (whole) {  // the units are whole logical tiles: one contiguous range, 128-bit loads
        const int64_t r0 = (u0 / gpt) * S, r1 = min(r0 + (int64_t)(UPW / gpt) * S, n);
        int64_t wb = r0;  // warp-uniform position
        for (; wb + 1024 <= r1; wb += 1024) {
          int4 v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = ld_hint4(in + wb + q * 128 + 4 * lane, keep);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            cnt += ((uint32_t)v[q].x - (uint32_t)lo <= span) + ((uint32_t)v[q].y - (uint32_t)lo <= span) +
                   ((uint32_t)v[q].z - (uint32_t)lo <= span) + ((uint32_t)v[q].w - (uint32_t)lo <= span);
        }
        for (int64_t e = wb + lane; e < r1; e += 32) cnt += (uint32_t)ld_hint1(in + e, keep) - (uint32_t)lo <= span;
      } else {
        UnitCursor uc(u0, gpt, S, lane);
        for (int ub = 0; ub < UPW; ub += NB) {
          int64_t s0[NB];
#pragma unroll
          for (int b2 = 0; b2 < NB; ++b2) s0[b2] = uc.next();
          const bool inb = s0[NB - 1] - (int64_t)lane + 31 + (int64_t)(IPTM - 1) * bt < n;
#pragma unroll
          for (int b2 = 0; b2 < NB; ++b2) {
            const int32_t* p = in + s0[b2];
#pragma unroll
            for (int q = 0; q < IPTM; ++q) {
              if ((inb || s0[b2] + (int64_t)q * bt < n))
                cnt += (uint32_t)ld_hint1(p + q * bt, keep) - (uint32_t)lo <= span;
            }
          }
        }
      }
      cnt = warp_sum(cnt);
      if (lane == 0) s_wc[k % NS][warp] = cnt;
      __syncthreads();
      if (threadIdx.x == 0) {
        int tot = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) tot += s_wc[k % NS][w];
        st_relaxed_u32(counts + (size_t)k * G + c, (uint32_t)tot + 1u);
        mine += tot;
      }
    }
    if (j < 0) continue;
    {
      int any = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) any |= s_wc[j % NS][w];
      if (!any) continue;  // uniform
    }
    if (warp == 0) {
      for (; resolved < j; ++resolved) {
        long long t = 0;
        for (int cc = (int)lane; cc < G; cc += 32) {
          uint32_t x;
          while ((x = ld_relaxed_u32(counts + (size_t)resolved * G + cc)) == 0u) __nanosleep(32);
          t += (long long)x - 1;
        }
        base += warp_sum(t);
      }
      long long before = 0, all = 0;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int cc = i * 32 + (int)lane;
        while (cv[i] == 0u) {
          __nanosleep(32);
          cv[i] = ld_relaxed_u32(counts + (size_t)j * G + cc);
        }
        const long long x = cc < G ? (long long)cv[i] - 1 : 0;
        all += x;
        before += cc < c ? x : 0;
      }
      before = warp_sum(before);
      all = warp_sum(all);
      if (lane == 0) s_off = base + before;
      base += all;
      resolved = j + 1;
    }
    __syncthreads();
    if (s_wc[j % NS][warp] == 0) continue;
    long long off = s_off;
#pragma unroll
    for (int w = 0; w < W; ++w) off += w < (int)warp ? s_wc[j % NS][w] : 0;
    const int64_t u0 = j * upr + ((int64_t)c * W + warp) * UPW;
    UnitCursor uc(u0, gpt, S, lane);
    for (int ub = 0; ub < UPW; ub += NB) {  // ---- WRITE round j: NB units' loads in flight, then unit by unit
      int64_t s0[NB];
#pragma unroll
      for (int b2 = 0; b2 < NB; ++b2) s0[b2] = uc.next();
      if (s0[0] - lane >= n) break;  // warp-uniform
      int32_t x[NB][IPTM];
      // the whole batch inside the input (all but the last tile): no per-slot bounds
      const bool inb = s0[NB - 1] - (int64_t)lane + 31 + (int64_t)(IPTM - 1) * bt < n;
      if (inb) {
#pragma unroll
        for (int b2 = 0; b2 < NB; ++b2) {
          const int32_t* p = in + s0[b2];
#pragma unroll
          for (int q = 0; q < IPTM; ++q) x[b2][q] = ld_hint1(p + q * bt, drop);
        }
      } else {
#pragma unroll
        for (int b2 = 0; b2 < NB; ++b2)
#pragma unroll
          for (int q = 0; q < IPTM; ++q) {
            const int64_t e = s0[b2] + (int64_t)q * bt;
            x[b2][q] = e < n ? ld_hint1(in + e, drop) : 0;
          }
      }
      // the batch's compacted output in this warp's staging buffer, then one
      // coalesced copy (per-lane runs straight to global scatter each store)
      int32_t* wb = s_stage + warp * (NB * 32 * IPTM);
      const uint32_t wb_s = (uint32_t)__cvta_generic_to_shared(wb);
      // one warp scan for PK units at a time: their lane counts packed into
      // FB-bit fields of one word (a unit's prefix is at most 32 * IPTM)
      constexpr int FB = 32 * IPTM < 256 ? 8 : 16;
      // (IPTM < 4 keeps one scan per unit: its 8-16 units per batch already
      // fill the registers)
      constexpr int PK = IPTM < 4 ? 1 : (32 / FB < NB ? 32 / FB : NB);
      int pos = 0;
#pragma unroll
      for (int g = 0; g < NB; g += PK) {
        uint32_t bits[PK];
#pragma unroll
        for (int b = 0; b < PK; ++b) {
          bits[b] = 0;
          if (inb) {
#pragma unroll
            for (int q = 0; q < IPTM; ++q) bits[b] |= (uint32_t)((uint32_t)x[g + b][q] - (uint32_t)lo <= span) << q;
          } else {
#pragma unroll
            for (int q = 0; q < IPTM; ++q) {
              const int64_t e = s0[g + b] + (int64_t)q * bt;
              bits[b] |= (uint32_t)(e < n && (uint32_t)x[g + b][q] - (uint32_t)lo <= span) << q;
            }
          }
        }
        uint32_t word = 0;
#pragma unroll
        for (int b = 0; b < PK; ++b) word |= (uint32_t)__popc(bits[b]) << (FB * b);
        uint32_t pre = word;  // inclusive warp scan of the packed counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
          if ((int)lane >= o) pre += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, pre, 31);
        const uint32_t exc = pre - word;
#pragma unroll
        for (int b = 0; b < PK; ++b) {
          constexpr uint32_t M = (1u << FB) - 1u;
          uint32_t a = wb_s + 4u * (uint32_t)(pos + (int)((exc >> (FB * b)) & M));
#pragma unroll
          for (int q = 0; q < IPTM; ++q) {
            const uint32_t m = (bits[b] >> q) & 1u;
            sts_if(a, x[g + b][q], m);
            a += 4u * m;
          }
          pos += (int)((tot >> (FB * b)) & M);
        }
      }
      __syncwarp();
      for (int i = (int)lane; i < pos; i += 32) __stcs(out + off + i, wb[i]);
      off += pos;
      __syncwarp();
    }
  }
  if (threadIdx.x == 0 && mine) atomicAdd(reinterpret_cast<unsigned long long*>(total_out), (unsigned long long)mine);
}

// Warp-specialised form of select_rr_crystal_kernel (same rounds, counts and
// output; see select_rr_ws_kernel): warps [0, W/2) count 2 UPW units each per
// round from HBM, warps [W/2, W) re-read and write them LAG rounds later, so
// the HBM count stream and the issue-heavy compaction overlap inside an SM.
template <int BT, int IPTM, int LAG>
__global__ void __launch_bounds__(BT, 2) select_rr_crystal_ws_kernel(const int32_t* __restrict__ in, int64_t n,
                                                                     int32_t lo, int32_t hi, int bt, int ipt,
                                                                     int32_t* __restrict__ out, int rounds,
                                                                     uint32_t* counts, long long* total_out) {
  constexpr int W = BT / 32, CW = W / 2;
  constexpr int UPW = 2 * (1024 / (32 * IPTM) > 0 ? 1024 / (32 * IPTM) : 1);  // units per count warp per round
  constexpr int NB = IPTM >= 16 ? 1 : 16 / IPTM;
  static_assert(UPW % NB == 0 && W % 2 == 0, "batches");
  constexpr int PER = (kRrMaxG + 31) / 32;
  constexpr int NS = LAG + 1;
  __shared__ int s_wc[NS][CW];
  __shared__ long long s_off;
  __shared__ int32_t s_stage[CW * NB * 32 * IPTM];  // per write warp: one batch of compacted output
  const int G = gridDim.x, c = blockIdx.x;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t span = (uint32_t)hi - (uint32_t)lo;
  const int gpt = bt >> 5;
  const int64_t S = (int64_t)bt * IPTM;
  const int64_t upr = (int64_t)G * CW * UPW;
  const bool whole = UPW % gpt == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  long long base = 0;
  int resolved = 0;
  long long mine = 0;
  uint32_t cv[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) cv[i] = 0u;
  for (int k = 0; k < rounds + LAG; ++k) {
    const int j = k - LAG;
    if (warp < CW) {
      if (k < rounds) {  // ---- COUNT round k (order does not matter here)
        const uint64_t keep = pipe::policy_evict_last();
        const int64_t u0 = k * upr + ((int64_t)c * CW + warp) * UPW;
        int cnt = 0;
        if (whole) {
          const int64_t r0 = (u0 / gpt) * S, r1 = min(r0 + (int64_t)(UPW / gpt) * S, n);
          int64_t wb = r0;
          for (; wb + 1024 <= r1; wb += 1024) {
            int4 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = ld_hint4(in + wb + q * 128 + 4 * lane, keep);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              cnt += ((uint32_t)v[q].x - (uint32_t)lo <= span) + ((uint32_t)v[q].y - (uint32_t)lo <= span) +
                     ((uint32_t)v[q].z - (uint32_t)lo <= span) + ((uint32_t)v[q].w - (uint32_t)lo <= span);
          }
          for (int64_t e = wb + lane; e < r1; e += 32) cnt += (uint32_t)ld_hint1(in + e, keep) - (uint32_t)lo <= span;
        } else {
          UnitCursor uc(u0, gpt, S, lane);
          for (int ub = 0; ub < UPW; ub += NB) {
            int64_t s0[NB];
#pragma unroll
            for (int b2 = 0; b2 < NB; ++b2) s0[b2] = uc.next();
            const bool inb = s0[NB - 1] - (int64_t)lane + 31 + (int64_t)(IPTM - 1) * bt < n;
#pragma unroll
            for (int b2 = 0; b2 < NB; ++b2) {
              const int32_t* p = in + s0[b2];
#pragma unroll
              for (int q = 0; q < IPTM; ++q)
                if ((inb || s0[b2] + (int64_t)q * bt < n)) cnt += (uint32_t)ld_hint1(p + q * bt, keep) - (uint32_t)lo <= span;
            }
          }
        }
        cnt = warp_sum(cnt);
        if (lane == 0) s_wc[k % NS][warp] = cnt;
        asm volatile("bar.sync 1, %0;" ::"n"(BT / 2) : "memory");  // count warps only
        if (threadIdx.x == 0) {
          int tot = 0;
#pragma unroll
          for (int w = 0; w < CW; ++w) tot += s_wc[k % NS][w];
          st_relaxed_u32(counts + (size_t)k * G + c, (uint32_t)tot + 1u);
          mine += tot;
        }
      }
    } else if (j >= 0) {
      const int ww = (int)warp - CW;
      int any = 0;
#pragma unroll
      for (int w = 0; w < CW; ++w) any |= s_wc[j % NS][w];
      if (any) {  // uniform over the write warps
        if (ww == 0) {
          for (; resolved < j; ++resolved) {
            long long t = 0;
            for (int cc = (int)lane; cc < G; cc += 32) {
              uint32_t x;
              while ((x = ld_relaxed_u32(counts + (size_t)resolved * G + cc)) == 0u) __nanosleep(32);
              t += (long long)x - 1;
            }
            base += warp_sum(t);
          }
          long long before = 0, all = 0;
#pragma unroll
          for (int i = 0; i < PER; ++i) {
            const int cc = i * 32 + (int)lane;
            if (cc < G)
              while (cv[i] == 0u) {
                cv[i] = ld_relaxed_u32(counts + (size_t)j * G + cc);
                if (cv[i] == 0u) __nanosleep(32);
              }
            const long long x = cc < G ? (long long)cv[i] - 1 : 0;
            all += x;
            before += cc < c ? x : 0;
          }
          before = warp_sum(before);
          all = warp_sum(all);
          if (lane == 0) s_off = base + before;
          base += all;
          resolved = j + 1;
        }
        asm volatile("bar.sync 2, %0;" ::"n"(BT / 2) : "memory");  // write warps only: s_off published
        if (s_wc[j % NS][ww] != 0) {
          const uint64_t drop = pipe::policy_evict_first();
          long long off = s_off;
#pragma unroll
          for (int w = 0; w < CW; ++w) off += w < ww ? s_wc[j % NS][w] : 0;
          const int64_t u0 = j * upr + ((int64_t)c * CW + ww) * UPW;
          UnitCursor uc(u0, gpt, S, lane);
          int32_t* wb = s_stage + ww * (NB * 32 * IPTM);
          const uint32_t wb_s = (uint32_t)__cvta_generic_to_shared(wb);
          for (int ub = 0; ub < UPW; ub += NB) {  // ---- WRITE round j
            int64_t s0[NB];
#pragma unroll
            for (int b2 = 0; b2 < NB; ++b2) s0[b2] = uc.next();
            if (s0[0] - lane >= n) break;  // warp-uniform
            int32_t x[NB][IPTM];
            const bool inb = s0[NB - 1] - (int64_t)lane + 31 + (int64_t)(IPTM - 1) * bt < n;
            if (inb) {
#pragma unroll
              for (int b2 = 0; b2 < NB; ++b2) {
                const int32_t* p = in + s0[b2];
#pragma unroll
                for (int q = 0; q < IPTM; ++q) x[b2][q] = ld_hint1(p + q * bt, drop);
              }
            } else {
#pragma unroll
              for (int b2 = 0; b2 < NB; ++b2)
#pragma unroll
                for (int q = 0; q < IPTM; ++q) {
                  const int64_t e = s0[b2] + (int64_t)q * bt;
                  x[b2][q] = e < n ? ld_hint1(in + e, drop) : 0;
                }
            }
            constexpr int FB = 32 * IPTM < 256 ? 8 : 16;
            constexpr int PK = IPTM < 4 ? 1 : (32 / FB < NB ? 32 / FB : NB);
            int pos = 0;
#pragma unroll
            for (int g = 0; g < NB; g += PK) {
              uint32_t bits[PK];
#pragma unroll
              for (int b = 0; b < PK; ++b) {
                bits[b] = 0;
                if (inb) {
#pragma unroll
                  for (int q = 0; q < IPTM; ++q) bits[b] |= (uint32_t)((uint32_t)x[g + b][q] - (uint32_t)lo <= span) << q;
                } else {
#pragma unroll
                  for (int q = 0; q < IPTM; ++q) {
                    const int64_t e = s0[g + b] + (int64_t)q * bt;
                    bits[b] |= (uint32_t)(e < n && (uint32_t)x[g + b][q] - (uint32_t)lo <= span) << q;
                  }
                }
              }
              uint32_t word = 0;
#pragma unroll
              for (int b = 0; b < PK; ++b) word |= (uint32_t)__popc(bits[b]) << (FB * b);
              uint32_t pre = word;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
                if ((int)lane >= o) pre += y;
              }
              const uint32_t tot = __shfl_sync(0xffffffffu, pre, 31);
              const uint32_t exc = pre - word;
#pragma unroll
              for (int b = 0; b < PK; ++b) {
                constexpr uint32_t M = (1u << FB) - 1u;
                uint32_t a = wb_s + 4u * (uint32_t)(pos + (int)((exc >> (FB * b)) & M));
#pragma unroll
                for (int q = 0; q < IPTM; ++q) {
                  const uint32_t m = (bits[b] >> q) & 1u;
                  sts_if(a, x[g + b][q], m);
                  a += 4u * m;
                }
                pos += (int)((tot >> (FB * b)) & M);
              }
            }
            __syncwarp();
            for (int i = (int)lane; i < pos; i += 32) __stcs(out + off + i, wb[i]);
            off += pos;
            __syncwarp();
          }
        }
      }
      if (ww == 0) {  // the next round's counts: in flight across the barrier
        const int jn = j + 1;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int cc = i * 32 + (int)lane;
          cv[i] = (jn < rounds && cc < G) ? ld_relaxed_u32(counts + (size_t)jn * G + cc) : 0u;
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && mine) atomicAdd(reinterpret_cast<unsigned long long*>(total_out), (unsigned long long)mine);
}

__global__ void select_seg_total_kernel(const unsigned long long* stot, long long nseg, long long* total_out) {
  unsigned long long t = 0;
  for (long long i = threadIdx.x; i < nseg; i += 32) t += stot[i];
  t = warp_sum(t);
  if (threadIdx.x == 0) *total_out = (long long)t;
}

// Crystal order for an arbitrary logical (bt, ipt) (select_tile_into,
// select.hpp:107-135 with block_thread_counts + block_scan + block_shuffle,
// block_ops.hpp:73-122): logical thread t of logical tile j owns slots
// j*S + t + k*bt (S = bt*ipt); the tile's matches are laid out thread-major,
// each thread's in k order, and tiles follow each other.  A CTA stages a
// CHUNK of whole logical tiles (~kCrysChunk elements) in shared memory, so
// small logical tiles do not mean small CTAs; one look-back per chunk.
constexpr int kCrysPB = 256;
constexpr int kCrysChunk = 8192;

__global__ void __launch_bounds__(kCrysPB) select_crystal_kernel(
    const int32_t* __restrict__ in, int64_t n, int32_t lo, int32_t hi, int bt, int ipt, int chunk,
    int32_t* __restrict__ out, unsigned long long* status, long long* total_out) {
  extern __shared__ int32_t s_dyn[];
  int32_t* s_in = s_dyn;                 // [chunk]
  int32_t* s_out = s_dyn + chunk;        // [chunk]
  int32_t* s_cnt = s_out + chunk;        // [pairs] counts, then exclusive prefixes
  __shared__ int s_scan[kCrysPB / 32 + 1];
  __shared__ long long s_off;
  const long long c = blockIdx.x;
  const int64_t base = c * (int64_t)chunk;
  const int valid = (int)min((int64_t)chunk, n - base);
  // 1. stage the chunk (128-bit loads where aligned)
  const int32_t* src = in + base;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int nv = valid >> 2;
    for (int i = threadIdx.x; i < nv; i += kCrysPB)
      reinterpret_cast<int4*>(s_in)[i] = ld_stream4(src + 4 * i);
    for (int i = 4 * nv + threadIdx.x; i < valid; i += kCrysPB) s_in[i] = ld_stream1(src + i);
  } else {
    for (int i = threadIdx.x; i < valid; i += kCrysPB) s_in[i] = ld_stream1(src + i);
  }
  __syncthreads();
  const int S = bt * ipt;
  const int tiles = (valid + S - 1) / S;
  const int pairs = tiles * bt;  // (logical tile, logical thread), in output order
  // 2. per-pair match counts; consecutive threads take consecutive logical
  //    threads, so the strided smem reads are bank-conflict free
  for (int p = threadIdx.x; p < pairs; p += kCrysPB) {
    const int j = p / bt, t = p - j * bt;
    const int b = j * S + t;
    int cnt = 0;
    for (int k = 0; k < ipt; ++k) {
      const int i = b + k * bt;
      if (i < valid) {
        const int32_t x = s_in[i];
        cnt += (x >= lo && x <= hi);
      }
    }
    s_cnt[p] = cnt;
  }
  __syncthreads();
  // 3. exclusive scan of the counts in pair order: thread u owns a contiguous run
  const int per = (pairs + kCrysPB - 1) / kCrysPB;
  const int p0 = min(pairs, (int)threadIdx.x * per), p1 = min(pairs, p0 + per);
  int mine = 0;
  for (int p = p0; p < p1; ++p) mine += s_cnt[p];
  int total;
  int run = BlockScan<kCrysPB>(mine, s_scan, total);
  for (int p = p0; p < p1; ++p) {
    const int cc = s_cnt[p];
    s_cnt[p] = run;
    run += cc;
  }
  __syncthreads();
  // 4. block_shuffle: each logical thread's matches, in k order, at its prefix
  for (int p = threadIdx.x; p < pairs; p += kCrysPB) {
    const int j = p / bt, t = p - j * bt;
    const int b = j * S + t;
    int pos = s_cnt[p];
    for (int k = 0; k < ipt; ++k) {
      const int i = b + k * bt;
      if (i < valid) {
        const int32_t x = s_in[i];
        if (x >= lo && x <= hi) s_out[pos++] = x;
      }
    }
  }
  if (threadIdx.x < 32) {
    const long long off = tile_lookback(status, c, total);
    if (threadIdx.x == 0) s_off = off;
  }
  __syncthreads();
  const long long off = s_off;
  BlockStore<kCrysPB, int32_t>(s_out, total, out + off);
  if (threadIdx.x == 0 && base + chunk >= n) *total_out = off + total;
}

// Crystal order, register form: physical thread u of a round owns logical
// pairs p = p0 + g*256 + u (g < G); pair p = (logical tile j, logical thread
// t) reads its IPT slots j*S + t + k*bt straight from HBM (consecutive u ->
// consecutive t: coalesced, the reference's striped ownership), counts are
// packed 16 bits per g into one 64-bit block scan, and matches land in the
// chunk's shared-memory output at their Crystal positions.  One look-back per
// chunk.  IPTM >= ipt is the unrolled item bound (items stay in registers).
// KNOWN: the chunk offsets come from a count pass + scan (offsets[c]) instead
// of the look-back (the reduce-then-scan form, as for the input-order select).
// One chunk of whole logical tiles compacted into s_out in Crystal order
// (thread-major per logical tile, tiles in order); returns the match count.
template <int IPTM, int G>
__device__ __forceinline__ int crystal_compact(const int32_t* __restrict__ in, int64_t base, int valid, int32_t lo,
                                               int32_t hi, int bt, int ipt, unsigned bt_magic, int32_t* s_out,
                                               unsigned long long* s_scan) {
  const int S = bt * ipt;
  const int pairs = ((valid + S - 1) / S) * bt;
  const int32_t* src = in + base;
  int run = 0;
  for (int p0 = 0; p0 < pairs; p0 += kCrysPB * G) {
    int32_t x[G][IPTM];
    unsigned f[G];
    unsigned long long packed = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      f[g] = 0;
      const int p = p0 + g * kCrysPB + (int)threadIdx.x;
      if (p < pairs) {
        // j = p / bt by a multiply-high (exact: p * bt < 2^32 here)
        const int j = bt == 1 ? p : (int)__umulhi((unsigned)p, bt_magic), t = p - j * bt;
        const int b = j * S + t;
#pragma unroll
        for (int k = 0; k < IPTM; ++k) {
          const int i = b + k * bt;
          if (k < ipt && i < valid) {
            x[g][k] = ld_stream1(src + i);
            f[g] |= (unsigned)(x[g][k] >= lo && x[g][k] <= hi) << k;
          }
        }
      }
      packed |= (unsigned long long)__popc(f[g]) << (16 * g);
    }
    unsigned long long tot;
    const unsigned long long ex = BlockScan<kCrysPB>(packed, s_scan, tot);
    int before = run;
#pragma unroll
    for (int g = 0; g < G; ++g) {  // BlockShuffle of pair group g at its Crystal position
      BlockShuffle<IPTM, int32_t>(x[g], f[g], before + (int)((ex >> (16 * g)) & 0xffff), s_out);
      before += (int)((tot >> (16 * g)) & 0xffff);
    }
    run = before;
  }
  return run;
}

template <int IPTM, int G, bool KNOWN = false>
__global__ void __launch_bounds__(kCrysPB) select_crystal_reg_kernel(
    const int32_t* __restrict__ in, int64_t n, int32_t lo, int32_t hi, int bt, int ipt, int chunk,
    int32_t* __restrict__ out, unsigned long long* status, long long* total_out,
    const long long* local = nullptr, const long long* bases = nullptr) {
  // ceil(2^32 / bt) (bt = 1 would need 2^32: handled without the multiply)
  const unsigned bt_magic = bt > 1 ? (unsigned)((0x100000000ull + (unsigned)bt - 1) / (unsigned)bt) : 0u;
  static_assert(G >= 1 && G <= 4, "four 16-bit count fields per scan word");
  extern __shared__ int32_t s_dyn[];
  int32_t* s_out = s_dyn;  // [chunk]
  __shared__ unsigned long long s_scan[kCrysPB / 32 + 1];
  __shared__ long long s_red[kCrysPB / 32 + kCrysPB / 64 + 1];
  const long long c = blockIdx.x;
  const int64_t base = c * (int64_t)chunk;
  const int valid = (int)min((int64_t)chunk, n - base);
  const long long nchunks = (n + chunk - 1) / chunk;
  if constexpr (KNOWN) {
    const long long o = sel_offset(local, bases, c, nchunks);
    if (sel_offset(local, bases, c + 1, nchunks) == o) {  // no match in this chunk (uniform exit)
      if (threadIdx.x == 0 && base + chunk >= n) *total_out = o;
      return;
    }
  }
  const int run = crystal_compact<IPTM, G>(in, base, valid, lo, hi, bt, ipt, bt_magic, s_out, s_scan);
  __syncthreads();  // s_out complete (the look-back's barriers would also order it)
  long long off;
  if constexpr (KNOWN) {
    off = sel_offset(local, bases, c, nchunks);
  } else {
    off = block_lookback<kCrysPB>(status, c, run, s_red);
  }
  BlockStore<kCrysPB, int32_t>(s_out, run, out + off);
  if (threadIdx.x == 0 && base + chunk >= n) *total_out = off + run;
}

// Per-chunk match counts for the Crystal-order reduce-then-scan (chunks of any
// length; scalar coalesced loads, four in flight per thread).
__global__ void __launch_bounds__(256) select_chunk_count_kernel(const int32_t* __restrict__ in, int64_t n,
                                                                 int32_t lo, int32_t hi, int chunk,
                                                                 long long nchunks, unsigned* counts) {
  __shared__ int s_warp[8];
  for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t base = c * (int64_t)chunk;
    const int valid = (int)min((int64_t)chunk, n - base);
    int cnt = 0;
    int i = threadIdx.x;
    const int32_t* cb = in + base;
    const int lead = min(valid, (int)(((16 - (reinterpret_cast<uintptr_t>(cb) & 15)) & 15) / 4));
    if ((reinterpret_cast<uintptr_t>(cb) & 3) == 0) {
      // 128-bit body from the first 16 B boundary (the count is order-free)
      if ((int)threadIdx.x < lead) {
        const int32_t a = ld_stream1(cb + threadIdx.x);
        cnt += (a >= lo && a <= hi);
      }
      const int nv = (valid - lead) / 4;
      const int32_t* vb = cb + lead;
      for (int v = threadIdx.x; v < nv; v += 256) {
        const int4 q = ld_stream4(vb + 4 * v);
        cnt += (q.x >= lo && q.x <= hi) + (q.y >= lo && q.y <= hi) + (q.z >= lo && q.z <= hi) + (q.w >= lo && q.w <= hi);
      }
      for (int r = lead + 4 * nv + threadIdx.x; r < valid; r += 256) {
        const int32_t a = ld_stream1(cb + r);
        cnt += (a >= lo && a <= hi);
      }
      i = valid;  // done
    }
    for (; i + 3 * 256 < valid; i += 4 * 256) {
      const int32_t a = ld_stream1(in + base + i), b = ld_stream1(in + base + i + 256);
      const int32_t e = ld_stream1(in + base + i + 512), f = ld_stream1(in + base + i + 768);
      cnt += (a >= lo && a <= hi) + (b >= lo && b <= hi) + (e >= lo && e <= hi) + (f >= lo && f <= hi);
    }
    for (; i < valid; i += 256) {
      const int32_t a = ld_stream1(in + base + i);
      cnt += (a >= lo && a <= hi);
    }
    cnt = warp_sum(cnt);
    if (lane_id() == 0) s_warp[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += s_warp[w];
      counts[c] = (unsigned)t;
    }
    __syncthreads();
  }
}

// project.hpp:49-64.  Linear: float mul, float mul, float add with no FMA
// contraction (explicit _rn intrinsics).  Sigmoid: double z (the two products
// are exact in double), 1/(1+exp(-z)) in double, rounded once to float.
// 2^(j/64) as an unevaluated double-double (hi + lo), j = 0..63.
__device__ const double2 kExp2Tab[64] = {
    {1.0, 0.0},
    {1.0108892860517005, -1.5234778603368577e-17},
    {1.0218971486541166, 5.109225028973444e-17},
    {1.0330248790212284, 7.600838874027088e-18},
    {1.0442737824274138, 8.551889705537965e-17},
    {1.0556451783605572, 1.759325738772092e-18},
    {1.0671404006768237, -7.899853966841582e-17},
    {1.0787607977571199, -6.656660436056593e-17},
    {1.0905077326652577, -3.046782079812471e-17},
    {1.102382583307841, 5.2660368715706944e-17},
    {1.1143867425958924, 1.0410278456845571e-16},
    {1.1265216186082418, 5.165856758795457e-17},
    {1.1387886347566916, 8.912812676025408e-17},
    {1.1511892299529827, 3.250710218863827e-17},
    {1.1637248587775775, 3.8292048369240935e-17},
    {1.1763969916502812, 5.554203254218079e-17},
    {1.189207115002721, 3.982015231465646e-17},
    {1.202156731452703, 6.644981499252301e-17},
    {1.215247359980469, -7.712630692681488e-17},
    {1.22848053610687, -1.89878163130253e-17},
    {1.241857812073484, 4.658027591836937e-17},
    {1.255380757024691, -6.7113898212968784e-18},
    {1.2690509571917332, 2.667932131342186e-18},
    {1.2828700160787783, 1.713594918243561e-17},
    {1.2968395546510096, 2.5382502794888315e-17},
    {1.3109612115247644, -7.181536135519454e-17},
    {1.3252366431597413, -2.8587312100388614e-17},
    {1.339667524053303, 8.927282594831732e-17},
    {1.3542555469368927, 7.70094837980299e-17},
    {1.3690024229745905, 9.593797919118849e-17},
    {1.383909881963832, -6.770511658794786e-17},
    {1.3989796725383112, -9.614213209051323e-17},
    {1.4142135623730951, -9.667293313452913e-17},
    {1.42961333839197, -1.2031642489053655e-17},
    {1.4451808069770467, -3.0237581349939873e-17},
    {1.460917794180647, -5.600377186075216e-17},
    {1.4768261459394993, -3.483994556892796e-17},
    {1.4929077282912648, 1.4192920154284036e-17},
    {1.5091644275934228, -1.016455327754295e-16},
    {1.5255981507445384, -1.1024941712342561e-16},
    {1.5422108254079407, 7.949834809697621e-17},
    {1.559004400237837, 3.7812070533575275e-17},
    {1.5759808451078865, -1.0136916471278304e-17},
    {1.593142151342267, -1.0094406542311964e-16},
    {1.6104903319492543, 2.4707192569797888e-17},
    {1.6280274218573478, -6.712955084707084e-17},
    {1.645755478153965, -1.0125679913674773e-16},
    {1.6636765803267364, 5.8909926967131e-17},
    {1.681792830507429, 8.199010020581497e-17},
    {1.7001063537185235, -8.0237193703977e-18},
    {1.718619298122478, -1.851380418263111e-17},
    {1.7373338352737062, 3.164389299292957e-17},
    {1.7562521603732995, 2.960140695448873e-17},
    {1.7753764925265212, 6.429731796556572e-17},
    {1.7947090750031072, 1.8227458427912087e-17},
    {1.8142521755003989, -9.969531538920349e-17},
    {1.8340080864093424, 3.283107224245627e-17},
    {1.8539791250833855, 9.761887490727594e-17},
    {1.8741676341103, -6.122763413004143e-17},
    {1.8945759815869656, 3.4034035352165297e-17},
    {1.9152065613971474, -1.0619946056195963e-16},
    {1.9360617934922943, 1.0332385960676326e-16},
    {1.9571441241754002, 8.960767791036668e-17},
    {1.978456026387951, 4.0388753109278167e-17},
};

// exp(x) for |x| <= 700 with a 64-entry table + degree-6 polynomial
// (x = (64 m + j) ln2/64 + r, |r| <= ln2/128): ~11 FP64 operations against
// ~25 for the generic exp(), within one ulp (the table's low part keeps the
// reconstruction near correctly rounded).  The sigmoid projection is bound by
// FP64 issue on B200, so this is what takes it to the HBM roofline.
__device__ __forceinline__ double exp_table(double x) {
  const double nd = rint(x * 92.33248261689366);  // 64 / ln2
  const int n = (int)nd;
  double r = fma(-nd, 0.010830424667801708, x);    // ln2/64, high part (exact product)
  r = fma(-nd, 2.8447437476627285e-11, r);          // ln2/64, low part
  double p = fma(r, 1.0 / 720, 1.0 / 120);
  p = fma(p, r, 1.0 / 24);
  p = fma(p, r, 1.0 / 6);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = p * r;                                         // exp(r) - 1
  const double2 t = __ldg(&kExp2Tab[n & 63]);
  const double e = t.x + fma(t.x, p, t.y);           // 2^(j/64) * exp(r)
  // scale by 2^(n >> 6) in the exponent field (|n >> 6| <= 1010 for |x| <= 700)
  const long long bits = __double_as_longlong(e) + ((long long)(n >> 6) << 52);
  return __longlong_as_double(bits);
}

// Fast sigmoid candidate for |z| <= 80 (a normal float result):
// y ~ 1/(1+exp(-z)) with relative error < 2^-43 (degree-4 polynomial on the
// 2^(j/64) table, |r|^5/120 < 2^-44.6; one Newton step on the hardware
// reciprocal seed).  Returns RN_float(y) and `sure` = y lies more than
// 2^-13 half-ulps from the nearest float rounding midpoint, so the
// reference's double result (within ~2^-50 of the true value) rounds to the
// same float; otherwise the caller takes the near-correctly-rounded path.
// Rounding to an integer is the 1.5*2^52 trick (no FRND / F2I on the XU
// pipe, which bounded the previous version).
// The fast path's double constants from constant memory: DFMA/DADD take a
// c[bank][offset] operand directly, where an inline literal is rebuilt into
// uniform registers (UMOV pairs) in every unrolled copy.
__constant__ double kSigK[9] = {92.33248261689366, 0x1.8p52, 0.010830424667801708, 2.8447437476627285e-11,
                                1.0 / 24, 1.0 / 6, 0.5, 1.0, -0x1p-13};

__device__ __forceinline__ float sigmoid_fast(double z, bool& sure) {
  const double x = -z;
  const double sh = fma(x, kSigK[0], kSigK[1]);  // 64/ln2, rounded to an integer in the low bits
  const int n = __double2loint(sh);
  const double nd = sh - kSigK[1];
  double r = fma(-nd, kSigK[2], x);
  r = fma(-nd, kSigK[3], r);
  double p = fma(r, kSigK[4], kSigK[5]);
  p = fma(p, r, kSigK[6]);
  p = fma(p, r, kSigK[7]);
  p = p * r;
  const double t = __ldg(&kExp2Tab[n & 63].x);
  const double e = __longlong_as_double(__double_as_longlong(fma(t, p, t)) + ((long long)(n >> 6) << 52));
  const double den = kSigK[7] + e;
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(den));
  y = fma(y, fma(-den, y, kSigK[7]), y);
  const float f = __double2float_rn(y);
  const double d = y - (double)f;  // exact (Sterbenz)
  const int fb = __float_as_int(f);
  // half an ulp of f towards d: 2^(ef - 151), one binade lower below a power of two
  const int ef = (fb >> 23) & 0xff;
  const int k = ef - 151 - ((d < 0.0 && (fb & 0x7fffff) == 0) ? 1 : 0);
  const double hu = __hiloint2double((k + 1023) << 20, 0);
  sure = fabs(d) < fma(hu, kSigK[8], hu);
  return f;
}

template <bool SIGMOID>
__device__ __forceinline__ float project_one(float u, float v, float a, float b, double da, double db) {
  if constexpr (!SIGMOID) {
    return __fadd_rn(__fmul_rn(a, u), __fmul_rn(b, v));
  } else {
    // float(1 / (1 + exp(-z))) with z in double (project.hpp:56-64); the
    // products of two floats are exact in double, so one fma rounds z once
    // (da, db: a and b in double, converted once per thread)
    const double z = fma(da, (double)u, __dmul_rn(db, (double)v));
    if (fabs(z) <= 80.0) {  // the float result is a normal number
      bool sure;
      const float f = sigmoid_fast(z, sure);
      if (sure) return f;
    }
    const double e = fabs(z) <= 700.0 ? exp_table(-z) : exp(-z);
    return __double2float_rn(__drcp_rn(__dadd_rn(1.0, e)));
  }
}

template <bool SIGMOID>
__global__ void __launch_bounds__(256) project_kernel(const float* __restrict__ x1,
                                                      const float* __restrict__ x2, int64_t n,
                                                      float a, float b, float* __restrict__ out) {
  // float4 body only when all three spans are 16 B aligned (else scalar)
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(x1) | reinterpret_cast<uintptr_t>(x2) |
                        reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const int64_t n4 = vec_ok ? n / 4 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double da = (double)a, db = (double)b;
  // the next vector pair is loaded before this one is computed: the sigmoid
  // is long enough per element that one pair in flight per thread leaves
  // HBM latency exposed
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float4 un = make_float4(0.f, 0.f, 0.f, 0.f), vn = un;
  if (i < n4) {
    un = ld_stream4f(x1 + 4 * i);
    vn = ld_stream4f(x2 + 4 * i);
  }
  for (; i < n4; i += stride) {
    const float4 u = un, v = vn;
    if (i + stride < n4) {
      un = ld_stream4f(x1 + 4 * (i + stride));
      vn = ld_stream4f(x2 + 4 * (i + stride));
    }
    float4 r;
    r.x = project_one<SIGMOID>(u.x, v.x, a, b, da, db);
    r.y = project_one<SIGMOID>(u.y, v.y, a, b, da, db);
    r.z = project_one<SIGMOID>(u.z, v.z, a, b, da, db);
    r.w = project_one<SIGMOID>(u.w, v.w, a, b, da, db);
    st_stream4f(out + 4 * i, r);
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = project_one<SIGMOID>(x1[i], x2[i], a, b, da, db);
}

__global__ void ht_init_kernel(int2* slots, int64_t cap) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap;
       i += (int64_t)gridDim.x * blockDim.x)
    slots[i] = make_int2(kEmptyKey, 0);
}

__global__ void ht_insert_kernel(int2* slots, uint32_t mask, int shift, const int32_t* __restrict__ keys,
                                 const int32_t* __restrict__ pays, int64_t n, int32_t* err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    ht_insert(slots, mask, shift, keys[i], pays[i], err);
}

// join.cpp:69-96 (tile variant): BlockLoad keys + payloads, BlockProbeHashTable,
// BlockAggregate(SUM) of build payload + probe payload over hits.
template <int BT, int IPT, bool SMEM>
__global__ void __launch_bounds__(BT) join_probe_kernel(const int32_t* __restrict__ keys,
                                                        const int32_t* __restrict__ pays, int64_t n,
                                                        const int2* __restrict__ slots,
                                                        uint32_t mask, int shift,
                                                        unsigned long long* out) {
  using L = VecLayout<BT, IPT>;
  extern __shared__ int2 s_slots[];
  __shared__ long long red[BT / 32];
  const bool aligned = ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(pays)) & 15) == 0;
  if constexpr (SMEM) {
    const int cap = (int)mask + 1;
    for (int i = threadIdx.x; i < cap; i += BT) s_slots[i] = __ldg(slots + i);
    __syncthreads();
  }
  long long sum = 0;
  const int64_t ntiles = (n + L::TILE - 1) / L::TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * L::TILE;
    const int valid = (int)min((int64_t)L::TILE, n - base);
    int32_t k[IPT], p[IPT], hit[IPT];
    if (aligned) {
      BlockLoad<BT, IPT>(keys + base, valid, k);
      BlockLoad<BT, IPT>(pays + base, valid, p);
    } else {
      BlockLoadUnaligned<BT, IPT>(keys + base, valid, k);
      BlockLoadUnaligned<BT, IPT>(pays + base, valid, p);
    }
    unsigned f = BlockValidMask<BT, IPT>(valid);
    if constexpr (SMEM)
      BlockProbeHashTableSmem<IPT>(k, f, hit, s_slots, mask, shift);
    else
      BlockProbeHashTable<IPT>(k, f, hit, slots, mask, shift);
#pragma unroll
    for (int i = 0; i < IPT; ++i)
      if ((f >> i) & 1u) sum += (long long)hit[i] + (long long)p[i];
  }
  sum = warp_sum(sum);
  if (lane_id() == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int w = 0; w < BT / 32; ++w) s += red[w];
    if (s) atomicAdd(out, (unsigned long long)s);
  }
}

// join_probe_tile as a streaming pipeline (the SSB join ring specialised to
// one join and a checksum): one persistent CTA per SM; warp W (producer)
// streams the probe keys and payloads through a STAGES-deep shared-memory
// ring with 1-D TMA bulk copies; consumer warps own R rows of a stage, issue
// all of a lane's first-slot probes (shared-memory copy of the table when it
// fits, else L2/HBM) before resolving any, walk collisions with every
// pending item's next slot in flight, and accumulate hits in 64 bits.
constexpr int kJW = 16;          // consumer warps
constexpr int kJTile = 4096;     // rows per stage (R = 256 per warp, 8 per lane)
constexpr int kJR = kJTile / kJW;

template <int STAGES, bool SMEM>
__global__ void __launch_bounds__((kJW + 1) * 32, 1) join_ring_kernel(
    const int32_t* __restrict__ keys, const int32_t* __restrict__ pays, int64_t n,
    const int2* __restrict__ gslots, uint32_t mask, int shift, unsigned long long* out, int l2_ahead,
    uint32_t slo, uint32_t shi) {
  constexpr int IT = kJR / 32;  // rows per lane per stage
  extern __shared__ __align__(128) unsigned char smem[];
  int32_t* ring = reinterpret_cast<int32_t*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * 2 * kJTile * 4);
  uint64_t* empty = full + STAGES;
  int2* s_slots = reinterpret_cast<int2*>(empty + STAGES);
  __shared__ long long red[kJW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + kJTile - 1) / kJTile;
  const int my_tiles = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      pipe::mbar_init(full + s, 1);
      pipe::mbar_init(empty + s, kJW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t policy = 0;
  auto issue = [&](int it) {
    const int s = it % STAGES;
    const int64_t base = (blockIdx.x + (int64_t)it * gridDim.x) * (int64_t)kJTile;
    const int64_t rows = min((int64_t)kJTile, n - base);
    const uint32_t bytes = (uint32_t)(rows * 4);  // host guarantees 16 B multiples
    pipe::mbar_expect_tx(full + s, 2 * bytes);
    pipe::tma_load_1d(ring + (size_t)s * 2 * kJTile, keys + base, bytes, full + s, policy);
    pipe::tma_load_1d(ring + (size_t)s * 2 * kJTile + kJTile, pays + base, bytes, full + s, policy);
    if (l2_ahead > 0) {  // the tile l2_ahead loads later: into L2 now
      const int64_t pb = (blockIdx.x + (int64_t)(it + l2_ahead) * gridDim.x) * (int64_t)kJTile;
      if (pb < n) {
        const uint32_t pbytes = (uint32_t)(min((int64_t)kJTile, n - pb) * 4);
        pipe::l2_prefetch_bulk(keys + pb, pbytes);
        pipe::l2_prefetch_bulk(pays + pb, pbytes);
      }
    }
  };
  if (warp == kJW && lane == 0) {
    policy = pipe::policy_evict_first();
    for (int it = 0; it < my_tiles && it < STAGES; ++it) issue(it);
  }
  if constexpr (SMEM) {
    const int cap = (int)mask + 1;
    for (int i = threadIdx.x; i < cap; i += blockDim.x) s_slots[i] = __ldg(gslots + i);
  }
  __syncthreads();
  const int2* slots = SMEM ? s_slots : gslots;
  long long sum = 0;
  if (warp == kJW) {
    if (lane == 0) {
      for (int it = STAGES; it < my_tiles; ++it) {
        const int s = it % STAGES;
        pipe::mbar_wait(empty + s, (uint32_t)(((it / STAGES) - 1) & 1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(it);
      }
    }
  } else {
    int64_t row0 = (int64_t)blockIdx.x * kJTile + warp * kJR;
    const int64_t step = (int64_t)gridDim.x * kJTile;
    for (int it = 0; it < my_tiles; ++it, row0 += step) {
      const int s = it % STAGES;
      const int64_t left = n - row0;
      const int valid = left >= kJR ? kJR : (left > 0 ? (int)left : 0);
      pipe::mbar_wait(full + s, (uint32_t)((it / STAGES) & 1));
      const int32_t* sk = ring + (size_t)s * 2 * kJTile + warp * kJR;
      const int32_t* sp = sk + kJTile;
      int32_t k[IT], p[IT];
#pragma unroll
      for (int v = 0; v < IT / 4; ++v) {
        const int4 a = reinterpret_cast<const int4*>(sk)[v * 32 + lane];
        const int4 b = reinterpret_cast<const int4*>(sp)[v * 32 + lane];
        k[v * 4 + 0] = a.x; k[v * 4 + 1] = a.y; k[v * 4 + 2] = a.z; k[v * 4 + 3] = a.w;
        p[v * 4 + 0] = b.x; p[v * 4 + 1] = b.y; p[v * 4 + 2] = b.z; p[v * 4 + 3] = b.w;
      }
      pipe::release_slot(empty + s, lane == 0);  // keys/payloads are in registers now
      uint32_t sl[IT];
      int2 e[IT];
      unsigned pending = 0;
#pragma unroll
      for (int i = 0; i < IT; ++i) {
        const int row = (i / 4) * 128 + lane * 4 + (i & 3);
        // INT32_MIN is unstorable: always a miss.  A multi-pass probe takes
        // only the keys whose home slot is in this pass's slice [slo, shi).
        sl[i] = ht_slot_of(k[i], shift);
        if (row < valid && k[i] != kEmptyKey && sl[i] - slo < shi - slo) {
          pending |= 1u << i;
          e[i] = SMEM ? slots[sl[i]] : __ldg(slots + sl[i]);
        }
      }
      while (pending) {  // hash_table.hpp:41-51, every pending item's next slot in flight
        unsigned next = 0;
#pragma unroll
        for (int i = 0; i < IT; ++i) {
          if ((pending >> i) & 1u) {
            if (e[i].x == k[i]) sum += (long long)e[i].y + (long long)p[i];
            else if (e[i].x != kEmptyKey) next |= 1u << i;
          }
        }
        pending = next;
#pragma unroll
        for (int i = 0; i < IT; ++i) {
          if ((pending >> i) & 1u) {
            sl[i] = (sl[i] + 1) & mask;
            e[i] = SMEM ? slots[sl[i]] : __ldg(slots + sl[i]);
          }
        }
      }
    }
    sum = warp_sum(sum);
    if (lane == 0) red[warp] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < kJW; ++w) t += red[w];
    if (t) atomicAdd(out, (unsigned long long)t);
  }
}

// The probe ring's producer can also bulk-prefetch tile it + k into L2
// (CRYS_JOIN_L2=k).  r01 measured k = 2 faster with the table on chip
// (0.361 -> 0.347 ms at 8 KB); r02 measures k = 0 faster everywhere (32 KB:
// 0.380 -> 0.369 ms; through L2 the prefetched lines compete with the
// table), so the default is 0.
// ---- radix-partitioned probe for tables far beyond L2 (PAPER's radix join;
// the checksum is order-free).  Bucket = the top k bits of the Fibonacci
// hash = the top k bits of the home slot, so bucket p's probes start inside
// slots [p cap/2^k, (p+1) cap/2^k): one ~8 MB slice of the table.  A
// histogram pass and a scatter pass (per-tile bucket ranks by shared-memory
// atomics, one global claim per bucket per tile) group the probe pairs by
// bucket; the TMA-ring probe then streams them in bucket order, so the CTAs
// in flight share one L2-resident slice instead of missing to HBM.
constexpr int kHpBT = 256, kHpIPT = 16, kHpTile = kHpBT * kHpIPT;

__device__ __forceinline__ uint32_t hp_bucket(int32_t key, int bshift) {
  return (uint32_t)((uint32_t)key * kFibonacci) >> bshift;
}

// CTA c of `grid` owns the contiguous tiles [c T / grid, (c+1) T / grid) in
// both passes, so the scatter needs no global atomics: its per-bucket
// offsets come from the histogram pass (hp_offsets_kernel).
__device__ __forceinline__ void hp_chunk(int64_t ntiles, int& t0, int& t1) {
  t0 = (int)(((int64_t)blockIdx.x * ntiles) / gridDim.x);
  t1 = (int)(((int64_t)(blockIdx.x + 1) * ntiles) / gridDim.x);
}

__global__ void __launch_bounds__(kHpBT) hp_hist_kernel(const int32_t* __restrict__ keys, int64_t n, int bshift,
                                                        int nb, unsigned* hist, unsigned* totals) {
  __shared__ unsigned h[kHpBT / 32][256];  // per-warp sub-histograms: less atomic contention
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (kHpBT / 32) * 256; i += kHpBT) (&h[0][0])[i] = 0;
  __syncthreads();
  int t0, t1;
  hp_chunk((n + kHpTile - 1) / kHpTile, t0, t1);
  const int64_t v0 = (int64_t)t0 * (kHpTile / 4), v1 = min((int64_t)t1 * (kHpTile / 4), n / 4);
  for (int64_t i = v0 + threadIdx.x; i < v1; i += kHpBT) {  // n % 4 == 0, 16 B aligned (host)
    const int4 k = ld_stream4(keys + 4 * i);
    atomicAdd(&h[warp][hp_bucket(k.x, bshift)], 1u);
    atomicAdd(&h[warp][hp_bucket(k.y, bshift)], 1u);
    atomicAdd(&h[warp][hp_bucket(k.z, bshift)], 1u);
    atomicAdd(&h[warp][hp_bucket(k.w, bshift)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += kHpBT) {
    unsigned t = 0;
#pragma unroll
    for (int w = 0; w < kHpBT / 32; ++w) t += h[w][b];
    hist[(size_t)blockIdx.x * nb + b] = t;
    if (t) atomicAdd(&totals[b], t);
  }
}

// One CTA per bucket b: off[c][b] = (sum of the totals before b) + (the
// counts of bucket b in the CTAs before c).
__global__ void __launch_bounds__(kHpBT) hp_offsets_kernel(const unsigned* hist, const unsigned* totals, int nb,
                                                           int grid, unsigned* off) {
  __shared__ unsigned s_scan[kHpBT / 32 + 1];
  __shared__ unsigned s_base;
  const int b = blockIdx.x;
  {
    unsigned v = 0;
    for (int i = threadIdx.x; i < b; i += kHpBT) v += totals[i];
    v = warp_sum(v);
    if (lane_id() == 0) s_scan[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned t = 0;
      for (int w = 0; w < kHpBT / 32; ++w) t += s_scan[w];
      s_base = t;
    }
    __syncthreads();
  }
  unsigned run = s_base;
  for (int c0 = 0; c0 < grid; c0 += kHpBT) {
    const int c = c0 + (int)threadIdx.x;
    const unsigned v = c < grid ? hist[(size_t)c * nb + b] : 0u;
    unsigned all;
    const unsigned ex = BlockScan<kHpBT>(v, s_scan, all);
    if (c < grid) off[(size_t)c * nb + b] = run + ex;
    run += all;
    __syncthreads();  // s_scan reuse
  }
}

__global__ void __launch_bounds__(kHpBT, 4) hp_scatter_kernel(const int32_t* __restrict__ keys,
                                                           const int32_t* __restrict__ pays, int64_t n, int bshift,
                                                           int nb, const unsigned* off,
                                                           int32_t* __restrict__ ok, int32_t* __restrict__ op) {
  constexpr int W = kHpBT / 32;
  __shared__ unsigned s_cur[256];
  __shared__ long long s_dst[256];   // global position of the tile's bucket run minus its tile offset
  __shared__ unsigned s_wc[W][256];  // per-warp bucket counters, then per-warp slots in the tile
  __shared__ unsigned s_scan[kHpBT / 32 + 1];
  __shared__ int32_t s_k[kHpTile], s_p[kHpTile];
  const int warp = threadIdx.x >> 5;
  for (int b = threadIdx.x; b < nb; b += kHpBT) s_cur[b] = off[(size_t)blockIdx.x * nb + b];
  int t0, t1;
  hp_chunk((n + kHpTile - 1) / kHpTile, t0, t1);
  for (int t = t0; t < t1; ++t) {
    for (int i = threadIdx.x; i < W * 256; i += kHpBT) (&s_wc[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)t * kHpTile;
    const int valid = (int)min((int64_t)kHpTile, n - base);
    int4 kv[kHpIPT / 4], pv[kHpIPT / 4];
    uint32_t rk[kHpIPT];
#pragma unroll
    for (int v = 0; v < kHpIPT / 4; ++v) {
      const int64_t i = base + 4 * ((int64_t)v * kHpBT + threadIdx.x);
      if (i < n) {  // n % 4 == 0: whole vectors
        kv[v] = ld_stream4(keys + i);
        pv[v] = ld_stream4(pays + i);
      }
    }
    // rank inside (tile, warp, bucket) with warp-private counters (the order
    // inside a bucket is free: the checksum does not depend on it)
#pragma unroll
    for (int v = 0; v < kHpIPT / 4; ++v) {
      const int64_t i = base + 4 * ((int64_t)v * kHpBT + threadIdx.x);
      const int32_t kk[4] = {kv[v].x, kv[v].y, kv[v].z, kv[v].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t b = hp_bucket(kk[e], bshift);
        rk[4 * v + e] = i < n ? (b << 16) | atomicAdd(&s_wc[warp][b], 1u) : 0xFFFFFFFFu;
      }
    }
    __syncthreads();
    {  // tile offsets of the buckets (block scan), per-warp slots, global runs
      const int b = threadIdx.x;  // kHpBT == 256 >= nb
      unsigned c = 0;
      if (b < nb)
#pragma unroll
        for (int w = 0; w < W; ++w) c += s_wc[w][b];
      unsigned all;
      const unsigned ts = BlockScan<kHpBT>(c, s_scan, all);
      if (b < nb) {
        unsigned run = ts;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const unsigned x = s_wc[w][b];
          s_wc[w][b] = run;
          run += x;
        }
        s_dst[b] = (long long)s_cur[b] - (long long)ts;
        s_cur[b] += c;
      }
    }
    __syncthreads();
#pragma unroll
    for (int v = 0; v < kHpIPT / 4; ++v) {  // into bucket order in shared memory
      const int32_t kk[4] = {kv[v].x, kv[v].y, kv[v].z, kv[v].w};
      const int32_t pp[4] = {pv[v].x, pv[v].y, pv[v].z, pv[v].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t r = rk[4 * v + e];
        if (r != 0xFFFFFFFFu) {
          const unsigned slot = s_wc[warp][r >> 16] + (r & 0xFFFFu);
          s_k[slot] = kk[e];
          s_p[slot] = pp[e];
        }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < valid; i += kHpBT) {  // bucket runs: coalesced stores
      const int32_t k = s_k[i];
      const long long dst = s_dst[hp_bucket(k, bshift)] + i;
      ok[dst] = k;
      op[dst] = s_p[i];
    }
    __syncthreads();  // s_wc / s_k / s_p reuse
  }
}

// CRYS_JOIN_PART_SLICE_KB: table bytes per partition of the partitioned probe.
// Default 16 MB, 32 MB from 512 MB tables (r02 sweep, kernel ms 16 / 32 MB
// slices: 256 MB 2.05 / 2.07, 512 MB 2.14 / 2.12, 1 GB 2.34 / 2.17).
size_t join_part_slice(size_t tbytes) {
  static const int64_t v = [] {
    const char* e = getenv("CRYS_JOIN_PART_SLICE_KB");
    return e ? (int64_t)atoll(e) << 10 : (int64_t)-1;
  }();
  if (v >= 0) return (size_t)v;
  return tbytes >= (size_t(512) << 20) ? size_t(32) << 20 : size_t(16) << 20;
}

// CRYS_JOIN_PART_MB: tables of at least this many MB take the partitioned
// probe (0 = never).  Default 256: a 128 MB table probed in one pass took
// 3.03 ms against 3.24 partitioned (r02 sweep).
int64_t join_part_min_bytes() {
  static const int64_t v = [] {
    const char* e = getenv("CRYS_JOIN_PART_MB");
    return (int64_t)(e ? atoll(e) : 256) << 20;
  }();
  return v;
}

// CRYS_JOIN_PART_MINK: at least 2^k buckets in the partitioned probe (few
// buckets serialise the scatter's shared-memory rank atomics).
int join_part_min_k() {
  static const int v = [] {
    const char* e = getenv("CRYS_JOIN_PART_MINK");
    return e ? std::max(0, std::min(8, atoi(e))) : 0;
  }();
  return v;
}

// CRYS_JOIN_PASS_MB: tables larger than this (and below the partitioned
// sizes) are probed in ceil(table / this) slot-slice passes (0 = one pass).
int64_t join_pass_bytes() {
  static const int64_t v = [] {
    const char* e = getenv("CRYS_JOIN_PASS_MB");
    return (int64_t)(e ? atoll(e) : 0) << 20;
  }();
  return v;
}

// Ring depth of the probe through L2 (2, 4 or 6 stages of 32 KB).  A random
// probe costs one L1tex wavefront per lane (~1 line per SM-cycle: 2^28 probes
// >= 0.92 ms on 148 SMs), so what is left to win is L1 hits: a shallower ring
// leaves more of the SM's 256 KB to cache table lines.  Measured on B200
// (2^28 probes, profiles/r02_join_stages.txt): 2 stages are fastest up to
// 8 MB and from 64 MB on (64 MB 3.45 -> 2.42 ms, 1 GB partitioned 2.63 ->
// 2.32), 4 stages at 16-32 MB.  CRYS_JOIN_L2_STAGES forces one.
int join_l2_stages(size_t tbytes, bool partitioned) {
  static const int v = [] {
    const char* e = getenv("CRYS_JOIN_L2_STAGES");
    const int x = e ? atoi(e) : 0;
    return x == 2 || x == 4 || x == 6 ? x : 0;
  }();
  if (v) return v;
  if (partitioned) return 2;
  return tbytes > (8u << 20) && tbytes < (48u << 20) ? 4 : 2;
}

int join_l2_ahead(bool table_on_chip) {
  static const int v = [] {
    const char* e = getenv("CRYS_JOIN_L2");
    return e ? atoi(e) : -1;
  }();
  return v >= 0 ? v : 0;  // r02: the bulk L2 prefetch no longer pays on chip either (0.380 -> 0.369 ms at 32 KB)
}

int occupancy(const void* fn, int bt, size_t smem) {
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
  cache[key] = std::max(nb, 1);
  return cache[key];
}

struct ScanBufs {
  unsigned* counts = nullptr;
  long long* local = nullptr;
  long long* btot = nullptr;
  long long* bases = nullptr;
  int nblk = 0;
};

// counts[ntiles] | local[ntiles] | btot[nblk] | bases[nblk + 1] in ctx->scratch2
ScanBufs scan_bufs(crys_ctx* ctx, int64_t ntiles) {
  ScanBufs b;
  b.nblk = (int)((ntiles + kScanBlk - 1) / kScanBlk);
  CRYS_CHECK(b.nblk <= 1024 * 64, CRYS_ENOTBUILT, "select: too many tiles");
  const size_t nc = ((size_t)ntiles + 1) & ~(size_t)1;
  ctx->scratch2.reserve(4 * nc + 8 * ((size_t)ntiles + 2 * (size_t)b.nblk + 1) + 64);
  b.counts = ctx->scratch2.as<unsigned>();
  b.local = reinterpret_cast<long long*>(b.counts + nc);
  b.btot = b.local + ntiles;
  b.bases = b.btot + b.nblk;
  return b;
}

void launch_scan(const ScanBufs& b, int64_t ntiles, cudaStream_t st) {
  select_scan_local_kernel<<<b.nblk, 1024, 0, st>>>(b.counts, ntiles, b.local, b.btot);
  select_scan_blocks_kernel<<<1, 1024, 0, st>>>(b.btot, b.nblk, b.bases);
}

// CRYS_SEL_RR: round-robin select instantiation <threads, rows per warp per
// round, lag, write loads per lane> (the table in rr_plan).
int sel_rr_variant() {
  static const int v = [] {
    const char* e = getenv("CRYS_SEL_RR");
    return e ? atoi(e) : 0;
  }();
  return v;
}

struct RrLaunch {
  const void* fn = nullptr;
  int bt = 0, grid = 0, rounds = 0;
  uint32_t* counts = nullptr;
};

RrLaunch rr_plan(crys_ctx* ctx, int64_t n) {
  RrLaunch r;
  int wu = 0, cwarps = 0;
  auto pick = [&](auto fn, int bt, int rows_per_warp, int count_warps = 0) {
    r.fn = (const void*)fn;
    r.bt = bt;
    wu = rows_per_warp;
    cwarps = count_warps ? count_warps : bt / 32;
  };
  switch (sel_rr_variant()) {  // segment = 296 CTAs x warps x rows per warp (x 4 B)
    case 1: pick(select_rr_kernel<512, 1024, 2, 16>, 512, 1024); break;  // 19.4 MB, lag 2, 16 loads
    case 2: pick(select_rr_kernel<512, 768, 2, 8>, 512, 768); break;     // 14.5 MB, lag 2
    case 3: pick(select_rr_kernel<512, 768, 3, 8>, 512, 768); break;     // 14.5 MB, lag 3
    case 4: pick(select_rr_kernel<512, 1024, 2, 4>, 512, 1024); break;   // 19.4 MB, lag 2, 4 loads
    // warp-specialised (half the warps count, half write): rows per COUNT warp
    case 5: pick(select_rr_ws_kernel<512, 2048, 2, 16, 8>, 512, 2048, 8); break;  // 19.4 MB, lag 2
    case 6: pick(select_rr_ws_kernel<512, 2048, 2, 8, 8>, 512, 2048, 8); break;   // 19.4 MB, lag 2, 8 loads
    case 7: pick(select_rr_ws_kernel<512, 1024, 2, 16, 8>, 512, 1024, 8); break;  // 9.7 MB, lag 2
    case 8: pick(select_rr_ws_kernel<512, 2048, 3, 16, 8>, 512, 2048, 8); break;  // 19.4 MB, lag 3
    case 9: pick(select_rr_ws_kernel<512, 4096, 2, 16, 8>, 512, 4096, 8); break;  // 38.8 MB, lag 2
    case 10: pick(select_rr_ws_kernel<512, 2048, 2, 16, 8, 1>, 512, 2048, 8); break;  // 5 + next-round L2 prefetch
    case 11: pick(select_rr_ws_kernel<512, 1024, 2, 16, 8, 1>, 512, 1024, 8); break;  // 7 + next-round L2 prefetch
    case 12: pick(select_rr_kernel<512, 1024, 2, 8>, 512, 1024); break;  // phase-alternating (r02 default before the split roles)
    case 13: pick(select_rr_ws_kernel<512, 2048, 2, 4, 8, 0, true>, 512, 2048, 8); break;  // default with 4 loads in flight
    default: pick(select_rr_ws_kernel<512, 2048, 2, 8, 8, 0, true>, 512, 2048, 8); break;  // 5 + 128-bit staged writes (r02 final)
  }
  const int per_sm = occupancy(r.fn, r.bt, 0);
  const int64_t per_cta = (int64_t)cwarps * wu;
  r.grid = (int)std::min<int64_t>({(int64_t)per_sm * ctx->num_sms, (int64_t)kRrMaxG, (n + per_cta - 1) / per_cta});
  const int64_t seg = (int64_t)r.grid * per_cta;
  r.rounds = (int)((n + seg - 1) / seg);
  return r;
}

// CRYS_SEL_RRC=0: Crystal-order selects take the count/scan/write kernels.
bool sel_rr_crystal() {
  static const bool v = [] {
    const char* e = getenv("CRYS_SEL_RRC");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

// CRYS_SEL_RRC_WS=0: Crystal-order selects on the phase-alternating kernel
// (default: the warp-specialised one; 128x4 sigma 0.5 0.95 -> 0.85 ms, sigma 0
// 0.37 -> 0.41).
bool sel_rrc_ws() {
  static const bool v = [] {
    const char* e = getenv("CRYS_SEL_RRC_WS");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

RrLaunch rr_plan_crystal(crys_ctx* ctx, int64_t n, int bt, int ipt) {
  RrLaunch r;
  constexpr int kBT = 512, kLag = 2;
  // units of 32 logical threads x ipt slots, ~1024 slots per warp per round
  // (a ~19 MB segment, as the input-order kernel); IPTM = ipt rounded up
  int iptm = 1;
  while (iptm < ipt) iptm <<= 1;
  if (sel_rrc_ws()) {  // warp-specialised: half the warps count 2x the units (same segment)
    switch (iptm) {
      case 1: r.fn = (const void*)select_rr_crystal_ws_kernel<kBT, 1, kLag>; break;
      case 2: r.fn = (const void*)select_rr_crystal_ws_kernel<kBT, 2, kLag>; break;
      case 4: r.fn = (const void*)select_rr_crystal_ws_kernel<kBT, 4, kLag>; break;
      case 8: r.fn = (const void*)select_rr_crystal_ws_kernel<kBT, 8, kLag>; break;
      default: r.fn = (const void*)select_rr_crystal_ws_kernel<kBT, 16, kLag>; break;
    }
  } else {
    switch (iptm) {
      case 1: r.fn = (const void*)select_rr_crystal_kernel<kBT, 1, kLag>; break;
      case 2: r.fn = (const void*)select_rr_crystal_kernel<kBT, 2, kLag>; break;
      case 4: r.fn = (const void*)select_rr_crystal_kernel<kBT, 4, kLag>; break;
      case 8: r.fn = (const void*)select_rr_crystal_kernel<kBT, 8, kLag>; break;
      default: r.fn = (const void*)select_rr_crystal_kernel<kBT, 16, kLag>; break;
    }
  }
  const int upw = std::max(1, 1024 / (32 * iptm));
  r.bt = kBT;
  const int per_sm = occupancy(r.fn, r.bt, 0);
  const int64_t gpt = bt / 32;
  const int64_t units = ((n + (int64_t)bt * ipt - 1) / ((int64_t)bt * ipt)) * gpt;
  const int64_t per_cta = (int64_t)(kBT / 32) * upw;
  r.grid = (int)std::min<int64_t>({(int64_t)per_sm * ctx->num_sms, (int64_t)kRrMaxG, (units + per_cta - 1) / per_cta});
  const int64_t upr = (int64_t)r.grid * per_cta;
  r.rounds = (int)((units + upr - 1) / upr);
  return r;
}

}  // namespace

int64_t select_i32(crys_ctx* ctx, const int32_t* d_in, int64_t n, int32_t lo, int32_t hi,
                   int32_t* d_out, int order, int bt, int ipt) {
  CRYS_CHECK(bt > 0 && ipt > 0, CRYS_ECONFIG, "TileConfig: block_threads/items_per_thread must be positive");
  CRYS_CHECK(n >= 0, CRYS_ECONFIG, "negative input length");
  if (n == 0) return 0;
  cudaStream_t st = ctx->stream;
  int64_t tile;
  size_t dyn = 0;
  int chunk = 0;
  const int cfg = sel_cfg();
  if (order == CRYS_ORDER_INPUT) {
    tile = 4096;  // 128 threads x 32 items
  } else {
    CRYS_CHECK(order == CRYS_ORDER_CRYSTAL, CRYS_ECONFIG, "unknown select order");
    const int64_t S = (int64_t)bt * ipt;
    CRYS_CHECK(S <= 16384, CRYS_ENOTBUILT, "Crystal-order tile too large for shared memory");
    chunk = (int)(S >= kCrysChunk ? S : S * (kCrysChunk / S));
    tile = chunk;
    const int64_t pairs = (chunk / S) * bt;
    dyn = sizeof(int32_t) * (size_t)(2 * chunk + pairs);
  }
  const int64_t ntiles = (n + tile - 1) / tile;
  // the round-robin path (default for 16 B-aligned input): its per-round
  // counts share the zeroed status buffer
  RrLaunch rr{};
  // (lo > hi is the empty predicate: the segmented path handles it; the
  // round-robin kernel tests x - lo <= hi - lo unsigned)
  if (order == CRYS_ORDER_INPUT && cfg == 0 && lo <= hi)
    rr = rr_plan(ctx, n);
  // Crystal order on the round-robin scheme: bt a multiple of 32, ipt in {1, 2, 4, 8, 16}
  RrLaunch rrc{};
  if (order == CRYS_ORDER_CRYSTAL && cfg == 0 && lo <= hi && bt % 32 == 0 && ipt <= 16 && (ipt & (ipt - 1)) == 0 &&
      sel_rr_crystal())
    rrc = rr_plan_crystal(ctx, n, bt, ipt);
  const size_t words = (size_t)(ntiles + 3) + (rr.fn ? (size_t)(rr.rounds * (int64_t)rr.grid + 1) / 2 : 0) +
                       (rrc.fn ? (size_t)(rrc.rounds * (int64_t)rrc.grid + 1) / 2 : 0);
  ctx->status.reserve(sizeof(unsigned long long) * words);
  auto* status = ctx->status.as<unsigned long long>();
  auto* total = reinterpret_cast<long long*>(status + ntiles + 1);
  if (rr.fn) rr.counts = reinterpret_cast<uint32_t*>(status + ntiles + 3);
  if (rrc.fn) rrc.counts = reinterpret_cast<uint32_t*>(status + ntiles + 3);
  CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * words, st));
  timing_kernel_begin(ctx);
  if (order == CRYS_ORDER_INPUT) {
    constexpr int BT = 128, IPT = 32;
    if (rr.fn) {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3((unsigned)rr.grid);
      lc.blockDim = dim3((unsigned)rr.bt);
      lc.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident (they wait on each other's counts)
      attr[0].val.cooperative = 1;
      lc.attrs = attr;
      lc.numAttrs = 1;
      void* args[] = {(void*)&d_in, (void*)&n, (void*)&lo, (void*)&hi, (void*)&d_out, (void*)&rr.rounds,
                      (void*)&rr.counts, (void*)&total};
      CUDA_TRY(cudaLaunchKernelExC(&lc, rr.fn, args));
    } else if (cfg == 1) {
      select_input_kernel<BT, IPT><<<(unsigned)ntiles, BT, 0, st>>>(d_in, n, lo, hi, d_out, status, ntiles, total);
    } else if (cfg != 3) {
      const long long seg = sel_seg();
      const long long nseg = (ntiles + seg - 1) / seg;
      const size_t ng = (size_t)((ntiles + kSegGroup - 1) / kSegGroup);
      ctx->scratch2.reserve(sizeof(unsigned) * (size_t)(ntiles + ng) + sizeof(unsigned long long) * (size_t)nseg + 16);
      auto* counts = ctx->scratch2.as<unsigned>();
      auto* gsum = counts + ntiles;
      auto* stot = reinterpret_cast<unsigned long long*>(
          (reinterpret_cast<uintptr_t>(gsum + ng) + 15) & ~(uintptr_t)15);
      CUDA_TRY(cudaMemsetAsync(gsum, 0, reinterpret_cast<char*>(stot + nseg) - reinterpret_cast<char*>(gsum), st));
      for (long long sg = 0; sg <= nseg; ++sg) {
        const long long nc = sg < nseg ? std::min(seg, ntiles - sg * seg) : 0;
        const long long nw = sg > 0 ? std::min(seg, ntiles - (sg - 1) * seg) : 0;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)(nc + nw));
        lc.blockDim = dim3(BT);
        lc.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = attr;
        lc.numAttrs = sg > 0 && sel_pdl() ? 1 : 0;  // launch 0 follows the memset normally
        // segments small enough to stay in L2 between the two roles
        // (<= 32 MB) keep the counted tiles with evict_last
        CUDA_TRY(cudaLaunchKernelEx(&lc, seg <= 2048 ? select_seg_kernel<BT, IPT, true> : select_seg_kernel<BT, IPT, false>,
                                    d_in, n, lo, hi, d_out, (long long)ntiles, seg, sg, counts, gsum, stot, total));
      }
      select_seg_total_kernel<<<1, 32, 0, st>>>(stot, nseg, total);
      count_launch(ctx, (int)nseg + 1);
    } else {
      ScanBufs sb = scan_bufs(ctx, ntiles);
      const int gc = (int)std::min<int64_t>(
          ntiles, (int64_t)occupancy((const void*)select_count_kernel<BT, IPT>, BT, 0) * ctx->num_sms);
      select_count_kernel<BT, IPT><<<gc, BT, 0, st>>>(d_in, n, lo, hi, ntiles, sb.counts);
      launch_scan(sb, ntiles, st);
      select_write_kernel<BT, IPT><<<(unsigned)ntiles, BT, 0, st>>>(d_in, n, lo, hi, ntiles, sb.local, sb.bases,
                                                                    d_out, sel_l2_ahead());
      CUDA_TRY(cudaMemcpyAsync(total, sb.bases + sb.nblk, sizeof(long long), cudaMemcpyDeviceToDevice, st));
      count_launch(ctx, 4);
    }
  } else if (rrc.fn) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)rrc.grid);
    lc.blockDim = dim3((unsigned)rrc.bt);
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident (they wait on each other's counts)
    attr[0].val.cooperative = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    void* args[] = {(void*)&d_in, (void*)&n, (void*)&lo, (void*)&hi, (void*)&bt, (void*)&ipt, (void*)&d_out,
                    (void*)&rrc.rounds, (void*)&rrc.counts, (void*)&total};
    CUDA_TRY(cudaLaunchKernelExC(&lc, rrc.fn, args));
  } else if (ipt <= 32) {
    // reduce-then-scan (CRYS_SEL_CFG=1: single pass with the look-back)
    const size_t dyn2 = sizeof(int32_t) * (size_t)chunk;
    const bool known = cfg != 1;
    ScanBufs sb{};
    if (known) {
      sb = scan_bufs(ctx, ntiles);
      const int gc = (int)std::min<int64_t>(ntiles, (int64_t)ctx->num_sms * 8);
      select_chunk_count_kernel<<<gc, 256, 0, st>>>(d_in, n, lo, hi, chunk, ntiles, sb.counts);
      launch_scan(sb, ntiles, st);
      count_launch(ctx, 3);
    }
    auto launch = [&](auto fn, size_t dyn_bytes) {
      occupancy((const void*)fn, kCrysPB, dyn_bytes);
      fn<<<(unsigned)ntiles, kCrysPB, dyn_bytes, st>>>(d_in, n, lo, hi, bt, ipt, chunk, d_out, status, total,
                                                       sb.local, sb.bases);
    };
    // (a TMA-staged chunk variant measured slower: 3 instead of 5 CTAs per
    // SM, profiles/r01_select_segmented.txt)
    if (known) {
      if (ipt <= 1) launch(select_crystal_reg_kernel<1, 4, true>, dyn2);
      else if (ipt <= 2) launch(select_crystal_reg_kernel<2, 4, true>, dyn2);
      else if (ipt <= 4) launch(select_crystal_reg_kernel<4, 4, true>, dyn2);
      else if (ipt <= 8) launch(select_crystal_reg_kernel<8, 2, true>, dyn2);
      else if (ipt <= 16) launch(select_crystal_reg_kernel<16, 1, true>, dyn2);
      else launch(select_crystal_reg_kernel<32, 1, true>, dyn2);
    } else {
      if (ipt <= 1) launch(select_crystal_reg_kernel<1, 4>, dyn2);
      else if (ipt <= 2) launch(select_crystal_reg_kernel<2, 4>, dyn2);
      else if (ipt <= 4) launch(select_crystal_reg_kernel<4, 4>, dyn2);
      else if (ipt <= 8) launch(select_crystal_reg_kernel<8, 2>, dyn2);
      else if (ipt <= 16) launch(select_crystal_reg_kernel<16, 1>, dyn2);
      else launch(select_crystal_reg_kernel<32, 1>, dyn2);
    }
  } else {
    occupancy((const void*)select_crystal_kernel, kCrysPB, dyn);
    select_crystal_kernel<<<(unsigned)ntiles, kCrysPB, dyn, st>>>(d_in, n, lo, hi, bt, ipt, chunk, d_out,
                                                                 status, total);
  }
  timing_kernel_end(ctx);
  count_launch(ctx);
  CUDA_TRY(cudaGetLastError());
  long long h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, total, sizeof(h), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return h;
}

void project_f32(crys_ctx* ctx, const float* x1, const float* x2, int64_t n, float a, float b,
                 float* out, int sigmoid) {
  CRYS_CHECK(n >= 0, CRYS_ECONFIG, "negative input length");
  if (n == 0) return;
  cudaStream_t st = ctx->stream;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n / 4 + 255) / 256, (int64_t)ctx->num_sms * 8));
  timing_kernel_begin(ctx);
  if (sigmoid)
    project_kernel<true><<<grid, 256, 0, st>>>(x1, x2, n, a, b, out);
  else
    project_kernel<false><<<grid, 256, 0, st>>>(x1, x2, n, a, b, out);
  timing_kernel_end(ctx);
  count_launch(ctx);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
}

void ht_build(crys_ctx* ctx, crys_ht* ht, const int32_t* d_keys, const int32_t* d_payloads,
              int64_t n) {
  cudaStream_t st = ctx->stream;
  int2* slots = ht->slots.as<int2>();
  const int64_t cap = ht->capacity;
  const int g1 = (int)std::max<int64_t>(1, std::min<int64_t>((cap + 255) / 256, (int64_t)ctx->num_sms * 16));
  ht_init_kernel<<<g1, 256, 0, st>>>(slots, cap);
  ctx->scratch.reserve(64);
  int32_t* err = ctx->scratch.as<int32_t>();
  CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
  if (n > 0) {
    const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 16));
    ht_insert_kernel<<<g2, 256, 0, st>>>(slots, (uint32_t)(cap - 1), ht->shift, d_keys, d_payloads, n, err);
  }
  count_launch(ctx, n > 0 ? 2 : 1);
  CUDA_TRY(cudaGetLastError());
  int32_t h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, err, sizeof(h), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (h == 1) fail(CRYS_EBUILD, "HashTable: key equals empty sentinel");
  if (h == 2) fail(CRYS_EBUILD, "HashTable: duplicate key");
  ht->size = n;
}

int64_t join_probe_sum(crys_ctx* ctx, const int32_t* d_keys, const int32_t* d_payloads, int64_t n,
                       const crys_ht* ht) {
  cudaStream_t st = ctx->stream;
  ctx->scratch.reserve(64);
  auto* out = ctx->scratch.as<unsigned long long>() + 1;
  CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(unsigned long long), st));
  const bool aligned = ((reinterpret_cast<uintptr_t>(d_keys) | reinterpret_cast<uintptr_t>(d_payloads)) & 15) == 0 &&
                       (n & 3) == 0;
  if (n > 0 && aligned) {
    // TMA ring: 4 stages x 32 KB; the table joins it in shared memory when it fits
    const size_t tbytes = sizeof(int2) * (size_t)ht->capacity;
    constexpr size_t ring4 = 4 * 2 * kJTile * 4 + 2 * 4 * 8;
    constexpr size_t ring6 = 6 * 2 * kJTile * 4 + 2 * 6 * 8;
    constexpr size_t ring2 = 2 * 2 * kJTile * 4 + 2 * 2 * 8;
    const bool smem = ring4 + tbytes <= 227 * 1024;
    const bool smem2 = !smem && ring2 + tbytes <= 227 * 1024;  // a shallower ring keeps 128 KB tables on chip
    const int64_t ntiles = (n + kJTile - 1) / kJTile;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, ctx->num_sms));
    const uint32_t mask = (uint32_t)(ht->capacity - 1);
    timing_kernel_begin(ctx);
    if (smem2) {
      auto fn = join_ring_kernel<2, true>;
      ensure_dyn_smem((const void*)fn, ring2 + tbytes);
      fn<<<grid, (kJW + 1) * 32, ring2 + tbytes, st>>>(d_keys, d_payloads, n, ht->slots.as<int2>(), mask,
                                                       ht->shift, out, join_l2_ahead(true), 0u, ~0u);
    } else if (smem) {
      auto fn = join_ring_kernel<4, true>;
      ensure_dyn_smem((const void*)fn, ring4 + tbytes);
      fn<<<grid, (kJW + 1) * 32, ring4 + tbytes, st>>>(d_keys, d_payloads, n, ht->slots.as<int2>(), mask,
                                                       ht->shift, out, join_l2_ahead(true), 0u, ~0u);
    } else {
      const int64_t pmin = join_part_min_bytes();
      const int logcap = 32 - ht->shift;
      int k = std::min(join_part_min_k(), logcap);  // buckets of <= join_part_slice() table slices
      while (k < 8 && k < logcap && (tbytes >> k) > join_part_slice(tbytes)) ++k;
      const int32_t* pk = d_keys;
      const int32_t* pp = d_payloads;
      if (pmin > 0 && (int64_t)tbytes >= pmin && k > 0 && n >= kHpTile && n < (int64_t(1) << 31)) {
        const int nb = 1 << k, bshift = 32 - k;
        const int64_t hp_tiles = (n + kHpTile - 1) / kHpTile;
        const int g = (int)std::min<int64_t>(hp_tiles, (int64_t)ctx->num_sms *
                                                         occupancy((const void*)hp_scatter_kernel, kHpBT, 0));
        ctx->part.reserve(2 * sizeof(int32_t) * (size_t)n + (2 * (size_t)g * nb + 256) * sizeof(unsigned) + 64);
        int32_t* ok = ctx->part.as<int32_t>();
        int32_t* op = ok + n;
        unsigned* totals = reinterpret_cast<unsigned*>(op + n);
        unsigned* hist = totals + 256;
        unsigned* offs = hist + (size_t)g * nb;
        CUDA_TRY(cudaMemsetAsync(totals, 0, 256 * sizeof(unsigned), st));
        hp_hist_kernel<<<g, kHpBT, 0, st>>>(d_keys, n, bshift, nb, hist, totals);
        hp_offsets_kernel<<<nb, kHpBT, 0, st>>>(hist, totals, nb, g, offs);
        hp_scatter_kernel<<<g, kHpBT, 0, st>>>(d_keys, d_payloads, n, bshift, nb, offs, ok, op);
        count_launch(ctx, 3);
        pk = ok;
        pp = op;
      }
      // Tables between the on-chip sizes and the partitioned ones: K passes
      // over the probe stream, pass p probing only the keys whose home slot
      // lies in slice p (cap / K slots), so each pass's slice stays
      // L2-resident (the streamed keys/payloads are evict_first).
      int passes = 1;
      if (pk == d_keys) {
        const int64_t slice = join_pass_bytes();
        if (slice > 0 && (int64_t)tbytes > slice)
          passes = (int)std::min<int64_t>(16, ((int64_t)tbytes + slice - 1) / slice);
      }
      const int stages = join_l2_stages(tbytes, pk != d_keys);
      const void* fnp = stages == 2 ? (const void*)join_ring_kernel<2, false>
                      : stages == 4 ? (const void*)join_ring_kernel<4, false>
                                    : (const void*)join_ring_kernel<6, false>;
      const size_t ring = stages == 2 ? ring2 : stages == 4 ? ring4 : ring6;
      ensure_dyn_smem(fnp, ring);
      const uint64_t cap = (uint64_t)ht->capacity;
      for (int p = 0; p < passes; ++p) {
        const uint32_t slo = passes == 1 ? 0u : (uint32_t)(cap * p / passes);
        const uint32_t shi = passes == 1 ? ~0u : (uint32_t)(cap * (p + 1) / passes);
        const int2* slots = ht->slots.as<int2>();
        int l2a = join_l2_ahead(false);
        void* args[] = {(void*)&pk, (void*)&pp, (void*)&n, (void*)&slots, (void*)&mask, (void*)&ht->shift,
                        (void*)&out, (void*)&l2a, (void*)&slo, (void*)&shi};
        CUDA_TRY(cudaLaunchKernel(fnp, dim3(grid), dim3((kJW + 1) * 32), args, ring, st));
      }
      count_launch(ctx, passes - 1);
    }
    timing_kernel_end(ctx);
    count_launch(ctx);
    CUDA_TRY(cudaGetLastError());
  } else if (n > 0) {
    constexpr int BT = 256, IPT = 16;
    const size_t tbytes = sizeof(int2) * (size_t)ht->capacity;
    const bool smem = tbytes <= 96 * 1024;
    const void* fn = smem ? (const void*)join_probe_kernel<BT, IPT, true>
                          : (const void*)join_probe_kernel<BT, IPT, false>;
    const int nb = occupancy(fn, BT, smem ? tbytes : 0);
    const int64_t ntiles = (n + BT * IPT - 1) / (BT * IPT);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)nb * ctx->num_sms));
    timing_kernel_begin(ctx);
    if (smem)
      join_probe_kernel<BT, IPT, true><<<grid, BT, tbytes, st>>>(
          d_keys, d_payloads, n, ht->slots.as<int2>(), (uint32_t)(ht->capacity - 1), ht->shift, out);
    else
      join_probe_kernel<BT, IPT, false><<<grid, BT, 0, st>>>(
          d_keys, d_payloads, n, ht->slots.as<int2>(), (uint32_t)(ht->capacity - 1), ht->shift, out);
    timing_kernel_end(ctx);
    count_launch(ctx);
    CUDA_TRY(cudaGetLastError());
  }
  unsigned long long h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, out, sizeof(h), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return (int64_t)h;
}

// Read-only HBM stream (the roofline's read-side reference): every 16 B of
// [d, d + bytes) loaded once with L1-bypassing 128-bit loads, XOR-folded
// into one word so nothing is optimised away.  4 loads in flight per thread.
__global__ void __launch_bounds__(512) stream_read_kernel(const int4* __restrict__ d, int64_t n16,
                                                          unsigned long long* sink) {
  unsigned acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    const int4 a = ld_stream4(reinterpret_cast<const int32_t*>(d + i));
    const int4 b = ld_stream4(reinterpret_cast<const int32_t*>(d + i + stride));
    const int4 c = ld_stream4(reinterpret_cast<const int32_t*>(d + i + 2 * stride));
    const int4 e = ld_stream4(reinterpret_cast<const int32_t*>(d + i + 3 * stride));
    acc ^= (unsigned)(a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ e.x ^ e.y ^ e.z ^ e.w);
  }
  for (; i < n16; i += stride) {
    const int4 a = ld_stream4(reinterpret_cast<const int32_t*>(d + i));
    acc ^= (unsigned)(a.x ^ a.y ^ a.z ^ a.w);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc == 0x9e3779b9u) atomicAdd(sink, 1ull);  // practically never
}

double stream_read(crys_ctx* ctx, const void* d, size_t bytes, int reps) {
  CRYS_CHECK(d && bytes >= 16 && reps >= 1, CRYS_ECONFIG, "stream read: bad argument");
  ctx->scratch2.reserve(64);
  auto* sink = ctx->scratch2.as<unsigned long long>();
  const int64_t n16 = (int64_t)(bytes / 16);
  const int grid = ctx->num_sms * 4;
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  stream_read_kernel<<<grid, 512, 0, ctx->stream>>>(static_cast<const int4*>(d), n16, sink);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CUDA_TRY(cudaEventRecord(e0, ctx->stream));
    stream_read_kernel<<<grid, 512, 0, ctx->stream>>>(static_cast<const int4*>(d), n16, sink);
    CUDA_TRY(cudaEventRecord(e1, ctx->stream));
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  count_launch(ctx, reps + 1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CRYS_LAUNCHED("stream_read_kernel");
  return (double)(n16 * 16) / (best * 1e-3) / 1e9;
}

}  // namespace crys
