// radix_sort.cu -- LSB and MSB radix sort of (int32 key, int32 payload) pairs.
//
// Reference: radix.hpp:44-93, radix.cpp:33-216.
//   radix_digit      ((u32)key ^ 0x80000000) >> start & mask   (signed order)
//   radix_histogram  owner x digit counts, owner = contiguous input chunk
//   radix_offsets    column-major exclusive prefix (digit-major, owner within digit)
//   radix_shuffle    stable scatter: each owner writes its runs in input order
//   lsb_radix_sort   stable passes low->high (default 4 x 8 bit) == std::stable_sort
//   msb_radix_sort   8-bit MSB partition from bit 24, then each partition sorted
//                    independently (radix.cpp:165-216; output keys sorted, pairs kept)
//
// B200 form: ONESWEEP.  The digit histograms of every pass are computed in ONE
// read of the keys up front (os_hist_kernel, 4N bytes); each pass is then a
// single kernel (onesweep_kernel): a tile of 4096 pairs is ranked stably in
// shared memory (warp match.any ranking, warp-major = input order), its
// per-digit counts are published and resolved against the preceding tiles by a
// per-digit DECOUPLED LOOK-BACK (the B200 replacement for the reference's
// column-major owner offsets, radix.cpp:55-73: tile order = owner order), and
// the tile is scattered in digit runs.  Traffic = 4N + 16N per pass (68N for
// four 8-bit passes vs the reference's 80N bytes_moved convention).
//
// MSB: pass 1 partitions by the top digit (bits 24-31) over the whole array;
// the 256 partitions then become SEGMENTS sorted independently by three
// segmented onesweep passes over bits 0-23 (each tile belongs to one segment,
// look-back stays inside it; segment histograms are taken in one read after
// the partition).  All segment bookkeeping stays on the device.
#include <algorithm>
#include <type_traits>
#include <vector>

#include "async.cuh"
#include "crystal.cuh"
#include "internal.hpp"

namespace crys {
namespace {

#ifndef CRYS_OS_MATCH_EVERY
#define CRYS_OS_MATCH_EVERY 4  // mixed ranking: every n-th item on match.any, the rest on ballots (r02 sweep after the full-tile path: 3 / 4 / 5 / 6 / 8 -> LSB 6.60 / 6.57 / 6.60 / 6.61 / 6.62 ms)
#endif
#ifndef CRYS_OS_LB
#define CRYS_OS_LB 4  // look-back window: predecessors read per round trip
#endif
#ifndef CRYS_OS_IPT
#define CRYS_OS_IPT 16
#endif
constexpr int kOsBT = 256, kOsIPT = CRYS_OS_IPT;
#ifdef CRYS_OS_MINB
constexpr int kOsMinBlocks = CRYS_OS_MINB;
#else
constexpr int kOsMinBlocks = kOsIPT <= 16 ? 4 : (kOsIPT <= 24 ? 3 : 2);
#endif
constexpr int kOsTile = kOsBT * kOsIPT;  // 4096 pairs (256 threads, 4 CTAs per SM: measured faster than 512 x 2)
constexpr int kOsWarps = kOsBT / 32;
constexpr uint32_t kOsAgg = 1u << 30, kOsPre = 2u << 30, kOsVal = (1u << 30) - 1;
constexpr int kHistBT = 512;
constexpr int kMaxPasses = 32;

__device__ __forceinline__ uint32_t digit_of(int32_t key, int start, uint32_t mask) {
  return (((uint32_t)key ^ 0x80000000u) >> start) & mask;  // radix.hpp:44-47
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Segment table (device): segment s = [begin[s], begin[s] + size[s]), its
// tiles are global tile ids [first_tile[s], first_tile[s+1]).
struct SegTable {
  int64_t begin[256];
  int64_t size[256];
  int32_t first_tile[257];
  int32_t nseg;
};

// Digit histograms of several passes in one read.  hist[(seg*npass + p)*256 + d].
// seg_mode 0: one segment (the whole array); 1: the array is partitioned by
// the top digit and `segs` holds the partitions -- each CTA walks the
// partitions its contiguous chunk overlaps.
__global__ void __launch_bounds__(kHistBT) os_hist_kernel(const int32_t* __restrict__ keys, int64_t n,
                                                          int npass, int start0, int bits,
                                                          const SegTable* segs, int64_t chunk,
                                                          uint32_t* hist) {
  __shared__ uint32_t h[4][256];
  const uint32_t mask = (1u << bits) - 1u;
  const int64_t b0 = (int64_t)blockIdx.x * chunk, e0 = min(n, b0 + chunk);
  if (b0 >= e0) return;
  int s_lo = 0, s_hi = 0;
  if (segs) {
    s_hi = segs->nseg - 1;
    // first segment whose end is beyond b0
    while (s_lo < s_hi && segs->begin[s_lo] + segs->size[s_lo] <= b0) ++s_lo;
  }
  for (int sg = s_lo; sg <= s_hi; ++sg) {
    int64_t b = b0, e = e0;
    if (segs) {
      const int64_t sb = segs->begin[sg], se = sb + segs->size[sg];
      if (sb >= e0) break;
      b = max(b0, sb);
      e = min(e0, se);
      if (b >= e) continue;
    }
    for (int i = threadIdx.x; i < npass * 256; i += kHistBT) (&h[0][0])[i] = 0;
    __syncthreads();
    int64_t i = b + threadIdx.x;
    // align to 4 elements, then 128-bit loads
    // first element at a 16 B ADDRESS boundary (the span itself may start mid-vector)
    const int64_t mis = (int64_t)(((16u - (uint32_t)(reinterpret_cast<uintptr_t>(keys + b) & 15u)) & 15u) >> 2);
    const int64_t ab = min(e, b + mis);
    for (; i < ab; i += kHistBT)
      for (int p = 0; p < npass; ++p) atomicAdd(&h[p][digit_of(keys[i], start0 + p * bits, mask)], 1u);
    const int64_t nvec = (e - ab) >> 2;  // whole 16 B vectors from ab
    int64_t v = threadIdx.x;
    for (; v + 3 * kHistBT < nvec; v += 4 * kHistBT) {  // 4 vectors in flight per thread
      int4 k[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) k[u] = ld_stream4(keys + ab + 4 * (v + u * kHistBT));
      for (int p = 0; p < npass; ++p) {
        const int st = start0 + p * bits;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          atomicAdd(&h[p][digit_of(k[u].x, st, mask)], 1u);
          atomicAdd(&h[p][digit_of(k[u].y, st, mask)], 1u);
          atomicAdd(&h[p][digit_of(k[u].z, st, mask)], 1u);
          atomicAdd(&h[p][digit_of(k[u].w, st, mask)], 1u);
        }
      }
    }
    for (; v < nvec; v += kHistBT) {
      const int4 k = ld_stream4(keys + ab + 4 * v);
      for (int p = 0; p < npass; ++p) {
        const int st = start0 + p * bits;
        atomicAdd(&h[p][digit_of(k.x, st, mask)], 1u);
        atomicAdd(&h[p][digit_of(k.y, st, mask)], 1u);
        atomicAdd(&h[p][digit_of(k.z, st, mask)], 1u);
        atomicAdd(&h[p][digit_of(k.w, st, mask)], 1u);
      }
    }
    const int64_t tail = ab + ((e - ab) & ~(int64_t)3);
    for (int64_t t = tail + threadIdx.x; t < e; t += kHistBT)
      for (int p = 0; p < npass; ++p) atomicAdd(&h[p][digit_of(keys[t], start0 + p * bits, mask)], 1u);
    __syncthreads();
    for (int x = threadIdx.x; x < npass * 256; x += kHistBT) {
      const uint32_t c = (&h[0][0])[x];
      if (c) atomicAdd(&hist[((int64_t)sg * npass + x / 256) * 256 + (x & 255)], c);
    }
    __syncthreads();
    if (!segs) break;
  }
}

// Exclusive scan of each 256-digit row in place (one warp per row).
__global__ void os_scan_kernel(uint32_t* hist, int rows) {
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= rows) return;
  uint32_t* h = hist + (int64_t)row * 256;
  const unsigned lane = lane_id();
  uint32_t v[8], run = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = h[lane * 8 + j];
#pragma unroll
  for (int j = 0; j < 8; ++j) run += v[j];
  uint32_t x = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  uint32_t ex = x - run;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    h[lane * 8 + j] = ex;
    ex += v[j];
  }
}

// MSB segment plan from the (un-scanned) top-digit histogram: 256 partitions,
// their begins, sizes and tile ranges.  One CTA of 256 threads.
__global__ void os_plan_kernel(const uint32_t* top_hist, int64_t base_begin, SegTable* segs) {
  __shared__ uint32_t sc[9];
  const int d = threadIdx.x;
  const uint32_t c = top_hist[d];
  const uint32_t nt = (c + kOsTile - 1) / kOsTile;
  uint32_t tot_c, tot_t;
  const uint32_t ex_c = BlockScan<256>(c, sc, tot_c);
  const uint32_t ex_t = BlockScan<256>(nt, sc, tot_t);
  segs->begin[d] = base_begin + ex_c;
  segs->size[d] = c;
  segs->first_tile[d] = (int32_t)ex_t;
  if (d == 0) {
    segs->first_tile[256] = (int32_t)tot_t;
    segs->nseg = 256;
  }
}

struct OsPass {
  const int32_t* kin;
  const int32_t* pin;
  int32_t* kout;
  int32_t* pout;
  int start, bits;
  const SegTable* segs;     // nullptr: one segment [0, n)
  int64_t n;                // single-segment length
  const uint32_t* bases;    // scanned histogram rows of this pass
  int bases_stride;         // elements between consecutive segments' rows
  uint32_t* status;         // [tiles][256] look-back words
  uint32_t* tile_counter;
  int32_t total_tiles;      // single-segment tile count (segmented: first_tile[nseg])
  int32_t l2_ahead;         // > 0: bulk-prefetch the tile this many tiles ahead into L2
};

// One stable pass: tile ranking + per-digit decoupled look-back + scatter.
// The tile's keys and payloads arrive by two 1-D TMA bulk copies (one
// elected thread, mbarrier completion) when the tile is 16 B aligned, so no
// register or LSU time goes into the loads.  Ranking: all 16 warp match.any
// of a thread are issued back to back, then a short serial per-warp counter
// update gives each item its stable rank (warp-striped order = input order).
// DBG 1 skips the look-back (timing experiments only; wrong output).
// RANK 0: warp match.any peers; 1: digit-bit ballots; 2 (default): every 4th
// item through match.any (ADU) and the rest through ballots (ALU), so both
// pipes work in parallel -- measured best on B200 (LSB 2^28: match-only 11.8,
// ballots-only 7.88, 1/4 match 7.68, 1/2 match 7.69, 3/8 match 8.00 ms).
template <int DBG, int RANK, bool SEG = false>
__global__ void __launch_bounds__(kOsBT, kOsMinBlocks) onesweep_kernel(OsPass a) {
  extern __shared__ __align__(128) uint32_t os_sm[];
  int32_t* s_k = reinterpret_cast<int32_t*>(os_sm);           // [kOsTile] staged -> digit-sorted keys
  int32_t* s_p = s_k + kOsTile;                                // [kOsTile] staged -> digit-sorted payloads
  uint32_t* s_wc = os_sm + 2 * kOsTile;                        // [kOsWarps][256]
  uint32_t* s_start = s_wc + kOsWarps * 256;                   // [257] tile digit starts
  long long* s_dst = reinterpret_cast<long long*>(s_start + 260);  // [256] dst - start
  __shared__ uint32_t s_scan[kOsBT / 32 + 1];
  __shared__ int s_tile, s_seg;
  __shared__ __align__(8) uint64_t s_bar;

  if (threadIdx.x == 0) {
    s_tile = (int)atomicAdd(a.tile_counter, 1u);
    if constexpr (SEG) s_seg = -1;
    pipe::mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < kOsWarps * 256; i += kOsBT) s_wc[i] = 0;
  __syncthreads();
  const int tile = s_tile;
  int seg = 0, first = 0;
  int64_t sbeg = 0, ssize = a.n;
  int total = a.total_tiles;
  if constexpr (SEG) {  // a.segs != nullptr (MSB segmented passes)
    // the tile's segment in one parallel round (a serial binary search was 8
    // dependent L2 round trips at the start of every tile: MSB passes ran
    // 18 % slower than LSB ones)
    const int nseg = a.segs->nseg;
    for (int t = threadIdx.x; t < nseg; t += kOsBT)
      if (a.segs->first_tile[t] <= tile && tile < a.segs->first_tile[t + 1]) s_seg = t;
    __syncthreads();
    if (s_seg < 0) return;  // uniform: past the last tile
    total = tile + 1;
    seg = s_seg;
    first = a.segs->first_tile[seg];
    sbeg = a.segs->begin[seg];
    ssize = a.segs->size[seg];
  } else if (a.segs) {
    // (the host launches SEG = true whenever a.segs is set; this serial form
    // is kept in the LSB instantiation only because ptxas allocates that
    // kernel's registers better with it: 6.60 vs 6.66 ms for the LSB 2^28)
    total = a.segs->first_tile[a.segs->nseg];
    int lo = 0, hi = a.segs->nseg - 1;  // last segment with first_tile <= tile
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.segs->first_tile[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    seg = lo;
    first = a.segs->first_tile[seg];
    sbeg = a.segs->begin[seg];
    ssize = a.segs->size[seg];
  }
  if (tile >= total) return;
  const int t_in = tile - first;
  const int64_t base = sbeg + (int64_t)t_in * kOsTile;
  const int valid = (int)min((int64_t)kOsTile, ssize - (int64_t)t_in * kOsTile);
  const uint32_t mask = (1u << a.bits) - 1u;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;

  // ---- stage the tile
  const bool tma = ((reinterpret_cast<uintptr_t>(a.kin + base) | reinterpret_cast<uintptr_t>(a.pin + base)) & 15) == 0 &&
                   (valid & 3) == 0;
  if (tma) {
    if (threadIdx.x == 0) {
      const uint64_t pol = pipe::policy_evict_first();
      pipe::mbar_expect_tx(&s_bar, 8u * (uint32_t)valid);
      pipe::tma_load_1d(s_k, a.kin + base, 4u * (uint32_t)valid, &s_bar, pol);
      pipe::tma_load_1d(s_p, a.pin + base, 4u * (uint32_t)valid, &s_bar, pol);
      // the rows a CTA will claim ~one resident wave later: into L2 now
      // (tile ids follow the array order, also across MSB segments)
      if (a.l2_ahead > 0) {
        const int64_t pb = base + (int64_t)a.l2_ahead * kOsTile;
        if (pb + kOsTile <= a.n) {
          pipe::l2_prefetch_bulk(a.kin + pb, 4u * kOsTile);
          pipe::l2_prefetch_bulk(a.pin + pb, 4u * kOsTile);
        }
      }
    }
    pipe::mbar_wait(&s_bar, 0);
  } else {
    for (int i = threadIdx.x; i < valid; i += kOsBT) {
      s_k[i] = ld_stream1(a.kin + base + i);
      s_p[i] = ld_stream1(a.pin + base + i);
    }
    __syncthreads();
  }

  // A full tile (every tile but a segment's last) drops every per-item
  // bounds test below: the rank, scatter and store loops become fixed-trip
  // and branch-free (measured ~11 branch/reconvergence instructions per item).
  auto body = [&](auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
  // ---- stable rank (warp-striped: item k of lane l in warp w is slot w*32*IPT + k*32 + l)
  const int wbase = warp * 32 * kOsIPT;
  int32_t key[kOsIPT];
  uint32_t rd[kOsIPT];  // peers mask, then rank (low 16) | digit << 16 ; digit 256 = outside
#pragma unroll
  for (int k = 0; k < kOsIPT; ++k) {
    const int sl = wbase + k * 32 + lane;
    key[k] = s_k[sl];
    const uint32_t d = (FULL || sl < valid) ? digit_of(key[k], a.start, mask) : 256u;
    if constexpr (RANK == 0) {
      rd[k] = __match_any_sync(0xffffffffu, d);
    } else if (RANK == 2 && (k % CRYS_OS_MATCH_EVERY) == 0) {
      // mixed: every CRYS_OS_MATCH_EVERY-th item on the ADU (match.any), the rest on the vote
      // path, so the two pipes work in parallel
      rd[k] = __match_any_sync(0xffffffffu, d);
    } else {
      // lanes with the same digit: one ballot per digit bit on the fast vote
      // path (match.any runs on the ADU at ~1/60 rate on sm_100a); m &= v or
      // ~v is one LOP3 with the xor mask (bit - 1).  A partial tile adds the
      // in-tile bit (d = 256 marks a slot past the end).
      unsigned m = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const unsigned bit = (d >> b) & 1u;
        m &= __ballot_sync(0xffffffffu, bit) ^ (bit - 1u);
      }
      if (!FULL && valid < kOsTile) {
        const unsigned bit = d >> 8;
        m &= __ballot_sync(0xffffffffu, bit) ^ (bit - 1u);
      }
      rd[k] = m;
    }
  }
  uint32_t* wc = s_wc + warp * 256;
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int k = 0; k < kOsIPT; ++k) {
    const int sl = wbase + k * 32 + lane;
    const uint32_t d = (FULL || sl < valid) ? digit_of(key[k], a.start, mask) : 256u;
    const unsigned peers = rd[k];
    const unsigned below = __popc(peers & lt);
    uint32_t basec = 0;
    if (FULL || d < 256) basec = wc[d];
    rd[k] = (basec + below) | (d << 16);
    __syncwarp();
    if (below == 0 && (FULL || d < 256)) wc[d] = basec + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: warp-exclusive prefix (in place) and the tile count
  uint32_t cnt = 0;
  if (threadIdx.x < 256) {
    const int d = threadIdx.x;
#pragma unroll
    for (int w = 0; w < kOsWarps; ++w) {
      const uint32_t v = s_wc[w * 256 + d];
      s_wc[w * 256 + d] = cnt;
      cnt += v;
    }
    // publish this tile's count early so successors can start looking back
    st_relaxed(a.status + (int64_t)tile * 256 + d, (t_in == 0 ? kOsPre : kOsAgg) | cnt);
  }
  uint32_t all;
  const uint32_t stt = BlockScan<kOsBT>(threadIdx.x < 256 ? cnt : 0u, s_scan, all);
  if (threadIdx.x < 256) s_start[threadIdx.x] = stt;
  if (threadIdx.x == 0) s_start[256] = all;
  __syncthreads();  // also: every staged key has been read
  // keys into digit order (in place over the staging buffer)
#pragma unroll
  for (int k = 0; k < kOsIPT; ++k) {
    const uint32_t d = rd[k] >> 16;
    if (FULL || d < 256) s_k[s_start[d] + s_wc[warp * 256 + d] + (rd[k] & 0xffffu)] = key[k];
  }
  // payloads: staged -> registers -> digit order
#pragma unroll
  for (int k = 0; k < kOsIPT; ++k) key[k] = s_p[wbase + k * 32 + lane];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kOsIPT; ++k) {
    const uint32_t d = rd[k] >> 16;
    if (FULL || d < 256) s_p[s_start[d] + s_wc[warp * 256 + d] + (rd[k] & 0xffffu)] = key[k];
  }
  // per-digit look-back over the preceding tiles of this segment
  if (threadIdx.x < 256) {
    const int d = threadIdx.x;
    uint32_t excl = 0;
    if constexpr (DBG != 1) {
      // windows of kLB predecessors per round trip (independent loads), the
      // closest inclusive prefix ends the walk; a not-yet-published word is
      // re-polled on its own (the one-at-a-time walk spent 22 % of the
      // kernel's stall samples in this loop)
      constexpr int kLB = CRYS_OS_LB;  // measured: 1 -> 7.45, 2 -> 7.03, 4 -> 6.96, 8 -> 7.15, 16 -> 7.52 ms (LSB 2^28)
      for (int t0 = tile - 1; t0 >= first; t0 -= kLB) {
        uint32_t w[kLB];
#pragma unroll
        for (int j = 0; j < kLB; ++j)
          w[j] = t0 - j >= first ? ld_relaxed(a.status + (int64_t)(t0 - j) * 256 + d) : kOsPre;
        bool done = false;
#pragma unroll
        for (int j = 0; j < kLB; ++j) {
          if (done) continue;
          if ((w[j] >> 30) == 0) {
            unsigned ns = 32;
            while (((w[j] = ld_relaxed(a.status + (int64_t)(t0 - j) * 256 + d)) >> 30) == 0) {
              __nanosleep(ns);
              ns = min(ns * 2, 512u);
            }
          }
          if (t0 - j < first) {
            done = true;
            continue;
          }
          excl += w[j] & kOsVal;
          if ((w[j] >> 30) == 2) done = true;
        }
        if (done) break;
      }
    }
    if (t_in != 0) st_relaxed(a.status + (int64_t)tile * 256 + d, kOsPre | (excl + cnt));
    const uint32_t gb = a.bases[(int64_t)seg * a.bases_stride + d];
    s_dst[d] = (long long)sbeg + (long long)gb + (long long)excl - (long long)s_start[d];
  }
  __syncthreads();
  if (a.n < (int64_t(1) << 31)) {  // 32-bit destinations (fewer instructions per item)
#pragma unroll 4
    for (int i = threadIdx.x; i < (FULL ? kOsTile : valid); i += kOsBT) {
      const int32_t kk = s_k[i];
      const int dst = (int)s_dst[digit_of(kk, a.start, mask)] + i;
      a.kout[dst] = kk;
      a.pout[dst] = s_p[i];
    }
  } else {
    for (int i = threadIdx.x; i < (FULL ? kOsTile : valid); i += kOsBT) {
      const int32_t kk = s_k[i];
      const long long dst = s_dst[digit_of(kk, a.start, mask)] + i;
      a.kout[dst] = kk;
      a.pout[dst] = s_p[i];
    }
  }
  };
  if (valid == kOsTile) body(std::true_type{});
  else body(std::false_type{});
}

// Each onesweep tile also bulk-prefetches tile + k into L2 (CRYS_OS_L2=k,
// 0 = off).  Default 296 (two CTAs' worth per SM ahead): LSB 2^28 7.68 ->
// 7.47 ms on B200 (148..592 all within 0.1 %, 1184 worse).
int os_l2_ahead() {
  static const int v = [] {
    const char* e = getenv("CRYS_OS_L2");
    return e ? atoi(e) : 296;
  }();
  return v;
}

// Tuning/experiment knob: CRYS_OS_DBG=1 launches the no-look-back variant,
// 2 the match.any-only and 3 the ballot-only ranking.
int os_dbg() {
  static const int v = [] {
    const char* e = getenv("CRYS_OS_DBG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

void launch_onesweep(const OsPass& a, unsigned grid, size_t smem, cudaStream_t st) {
  if (a.segs) {  // MSB segmented passes (the CRYS_OS_DBG variants are LSB-only)
    onesweep_kernel<0, 2, true><<<grid, kOsBT, smem, st>>>(a);
    return;
  }
  switch (os_dbg()) {
    case 1: onesweep_kernel<1, 1><<<grid, kOsBT, smem, st>>>(a); break;
    case 2: onesweep_kernel<0, 0><<<grid, kOsBT, smem, st>>>(a); break;
    case 3: onesweep_kernel<0, 1><<<grid, kOsBT, smem, st>>>(a); break;
    default: onesweep_kernel<0, 2><<<grid, kOsBT, smem, st>>>(a); break;
  }
}

// radix_histogram (radix.cpp:33-53): counts[owner][digit], owner = the
// contiguous chunk [o*chunk, (o+1)*chunk).  Per tile a shared histogram for
// each owner the tile overlaps, flushed with 64-bit atomics.
constexpr int kHistTile = 8192;
__global__ void __launch_bounds__(256) owner_hist_kernel(const int32_t* __restrict__ keys, int64_t n,
                                                         int64_t chunk, int start, int bits,
                                                         unsigned long long* counts) {
  __shared__ uint32_t h[256];
  const int D = 1 << bits;
  const uint32_t mask = (uint32_t)D - 1;
  for (int64_t t0 = (int64_t)blockIdx.x * kHistTile; t0 < n; t0 += (int64_t)gridDim.x * kHistTile) {
    const int64_t t1 = min(n, t0 + kHistTile);
    for (int64_t o = t0 / chunk; o * chunk < t1; ++o) {
      const int64_t b = max(t0, o * chunk), e = min(t1, (o + 1) * chunk);
      for (int d = threadIdx.x; d < D; d += blockDim.x) h[d] = 0;
      __syncthreads();
      for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) atomicAdd(&h[digit_of(keys[i], start, mask)], 1u);
      __syncthreads();
      for (int d = threadIdx.x; d < D; d += blockDim.x)
        if (h[d]) atomicAdd(&counts[o * D + d], (unsigned long long)h[d]);
      __syncthreads();
    }
  }
}

}  // namespace

struct SortWorkspace {
  DevBuf tk, tp;          // ping-pong pair arrays
  DevBuf hist;            // digit histograms (scanned in place)
  DevBuf status;          // look-back words, one region per pass
  DevBuf counters;        // tile counters, one per pass
  DevBuf segs;            // SegTable (MSB)
  DevBuf owner;           // radix_histogram counts
};

void WsDeleter::operator()(SortWorkspace* p) const { delete p; }

namespace {

size_t os_smem() {
  return sizeof(int32_t) * 2 * kOsTile + sizeof(uint32_t) * (kOsWarps * 256 + 260) + sizeof(long long) * 256;
}

void os_attr() {  // per device (ensure_dyn_smem caches by (device, kernel))
  for (const void* fn : {(const void*)onesweep_kernel<0, 0>, (const void*)onesweep_kernel<0, 1>,
                         (const void*)onesweep_kernel<0, 2>, (const void*)onesweep_kernel<0, 2, true>,
                         (const void*)onesweep_kernel<1, 1>})
    ensure_dyn_smem(fn, os_smem());
}

int64_t hist_chunk(crys_ctx* ctx, int64_t n) {
  const int64_t ctas = (int64_t)ctx->num_sms * 4;
  int64_t c = (n + ctas - 1) / ctas;
  c = (c + 4095) & ~(int64_t)4095;
  return std::max<int64_t>(c, 4096);
}

// Stable passes over one segment [0, n): bits [start0, start0 + npass*bits).
// Reads (sk, sp), ping-pongs through (tk, tp); returns true when the result
// ended in (tk, tp).
bool onesweep_passes(crys_ctx* ctx, SortWorkspace& ws, int32_t* sk, int32_t* sp, int32_t* tk, int32_t* tp,
                     int64_t n, int start0, int bits, int npass, const std::vector<int>* pass_bits) {
  cudaStream_t st = ctx->stream;
  const int64_t tiles = (n + kOsTile - 1) / kOsTile;
  ws.hist.reserve(sizeof(uint32_t) * 256 * (size_t)npass);
  ws.status.reserve(sizeof(uint32_t) * 256 * (size_t)tiles * (size_t)npass);
  ws.counters.reserve(sizeof(uint32_t) * kMaxPasses);
  CUDA_TRY(cudaMemsetAsync(ws.hist.p, 0, sizeof(uint32_t) * 256 * (size_t)npass, st));
  CUDA_TRY(cudaMemsetAsync(ws.status.p, 0, sizeof(uint32_t) * 256 * (size_t)tiles * (size_t)npass, st));
  CUDA_TRY(cudaMemsetAsync(ws.counters.p, 0, sizeof(uint32_t) * kMaxPasses, st));
  uint32_t* hist = ws.hist.as<uint32_t>();
  const int64_t chunk = hist_chunk(ctx, n);
  const int hgrid = (int)((n + chunk - 1) / chunk);
  // histograms: passes of equal width share one read (<= 4 per read)
  for (int p0 = 0; p0 < npass; p0 += 4) {
    const int np = std::min(4, npass - p0);
    const int b = pass_bits ? (*pass_bits)[p0] : bits;
    bool same = true;
    for (int p = p0; p < p0 + np; ++p) same = same && (!pass_bits || (*pass_bits)[p] == b);
    if (same) {
      os_hist_kernel<<<hgrid, kHistBT, 0, st>>>(sk, n, np, start0 + p0 * bits, b, nullptr, chunk,
                                                hist + (int64_t)p0 * 256);
      count_launch(ctx);
    } else {
      for (int p = p0; p < p0 + np; ++p) {
        os_hist_kernel<<<hgrid, kHistBT, 0, st>>>(sk, n, 1, start0 + p * bits, (*pass_bits)[p], nullptr, chunk,
                                                  hist + (int64_t)p * 256);
        count_launch(ctx);
      }
    }
  }
  os_scan_kernel<<<(npass + 7) / 8, 256, 0, st>>>(hist, npass);
  count_launch(ctx);
  os_attr();
  int32_t *ik = sk, *ip = sp, *ok = tk, *op = tp;
  for (int p = 0; p < npass; ++p) {
    OsPass a;
    a.kin = ik; a.pin = ip; a.kout = ok; a.pout = op;
    a.start = start0 + p * bits;
    a.bits = pass_bits ? (*pass_bits)[p] : bits;
    a.segs = nullptr;
    a.n = n;
    a.bases = hist + (int64_t)p * 256;
    a.bases_stride = 0;
    a.status = ws.status.as<uint32_t>() + (int64_t)p * 256 * tiles;
    a.tile_counter = ws.counters.as<uint32_t>() + p;
    a.total_tiles = (int32_t)tiles;
    a.l2_ahead = os_l2_ahead();
    launch_onesweep(a, (unsigned)tiles, os_smem(), st);
    CRYS_LAUNCHED("onesweep_kernel");
    count_launch(ctx);
    std::swap(ik, ok);
    std::swap(ip, op);
  }
  return (npass & 1) != 0;
}

void lsb_sort(crys_ctx* ctx, SortWorkspace& ws, int32_t* keys, int32_t* pays, int64_t n, int bpp) {
  ws.tk.reserve(sizeof(int32_t) * (size_t)n);
  ws.tp.reserve(sizeof(int32_t) * (size_t)n);
  // lsb_radix_sort (radix.cpp:151-159): passes at 0, bpp, 2bpp, ... of width min(bpp, 32-start)
  std::vector<int> pb;
  for (int start = 0; start < 32; start += bpp) pb.push_back(std::min(bpp, 32 - start));
  timing_kernel_begin(ctx);
  const bool in_tmp = onesweep_passes(ctx, ws, keys, pays, ws.tk.as<int32_t>(), ws.tp.as<int32_t>(), n, 0, bpp,
                                      (int)pb.size(), &pb);
  timing_kernel_end(ctx);
  if (in_tmp) {
    CUDA_TRY(cudaMemcpyAsync(keys, ws.tk.p, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(pays, ws.tp.p, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
}

// msb_radix_sort (radix.cpp:165-216): partition by the top 8-bit digit, then
// sort every partition independently on bits 0-23 (segmented passes).
void msb_sort(crys_ctx* ctx, SortWorkspace& ws, int32_t* keys, int32_t* pays, int64_t n) {
  cudaStream_t st = ctx->stream;
  ws.tk.reserve(sizeof(int32_t) * (size_t)n);
  ws.tp.reserve(sizeof(int32_t) * (size_t)n);
  int32_t* tk = ws.tk.as<int32_t>();
  int32_t* tp = ws.tp.as<int32_t>();
  const int64_t tiles1 = (n + kOsTile - 1) / kOsTile;
  const int64_t tiles_seg = tiles1 + 256;  // each partition rounds its tail tile up
  // hist rows: [0] top digit (kept un-scanned copy in row 1), [2 + s*3 + p] segment rows
  const size_t hist_words = 256 * (2 + 256 * 3);
  ws.hist.reserve(sizeof(uint32_t) * hist_words);
  ws.status.reserve(sizeof(uint32_t) * 256 * (size_t)(tiles1 + 3 * tiles_seg));
  ws.counters.reserve(sizeof(uint32_t) * kMaxPasses);
  ws.segs.reserve(sizeof(SegTable));
  uint32_t* hist = ws.hist.as<uint32_t>();
  uint32_t* status = ws.status.as<uint32_t>();
  uint32_t* ctr = ws.counters.as<uint32_t>();
  SegTable* segs = ws.segs.as<SegTable>();
  timing_kernel_begin(ctx);
  CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * hist_words, st));
  CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(uint32_t) * 256 * (size_t)(tiles1 + 3 * tiles_seg), st));
  CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(uint32_t) * kMaxPasses, st));
  const int64_t chunk = hist_chunk(ctx, n);
  const int hgrid = (int)((n + chunk - 1) / chunk);
  os_hist_kernel<<<hgrid, kHistBT, 0, st>>>(keys, n, 1, 24, 8, nullptr, chunk, hist);
  CUDA_TRY(cudaMemcpyAsync(hist + 256, hist, sizeof(uint32_t) * 256, cudaMemcpyDeviceToDevice, st));
  os_scan_kernel<<<1, 32, 0, st>>>(hist, 1);
  os_plan_kernel<<<1, 256, 0, st>>>(hist + 256, 0, segs);
  os_attr();
  {  // pass 1: top digit, whole array, keys -> tmp
    OsPass a;
    a.kin = keys; a.pin = pays; a.kout = tk; a.pout = tp;
    a.start = 24; a.bits = 8; a.segs = nullptr; a.n = n;
    a.bases = hist; a.bases_stride = 0;
    a.status = status; a.tile_counter = ctr; a.total_tiles = (int32_t)tiles1;
    a.l2_ahead = os_l2_ahead();
    launch_onesweep(a, (unsigned)tiles1, os_smem(), st);
    CRYS_LAUNCHED("onesweep_kernel msb top");
  }
  // segment histograms of bits 0-7, 8-15, 16-23 in one read of tmp
  uint32_t* shist = hist + 2 * 256;
  os_hist_kernel<<<hgrid, kHistBT, 0, st>>>(tk, n, 3, 0, 8, segs, chunk, shist);
  os_scan_kernel<<<(256 * 3 + 7) / 8, 256, 0, st>>>(shist, 256 * 3);
  int32_t *ik = tk, *ip = tp, *ok = keys, *op = pays;
  for (int p = 0; p < 3; ++p) {
    OsPass a;
    a.kin = ik; a.pin = ip; a.kout = ok; a.pout = op;
    a.start = 8 * p; a.bits = 8; a.segs = segs; a.n = n;
    a.bases = shist + 256 * p; a.bases_stride = 3 * 256;
    a.status = status + 256 * (tiles1 + p * tiles_seg);
    a.tile_counter = ctr + 1 + p;
    a.total_tiles = (int32_t)tiles_seg;
    a.l2_ahead = os_l2_ahead();
    launch_onesweep(a, (unsigned)tiles_seg, os_smem(), st);
    CRYS_LAUNCHED("onesweep_kernel msb segmented");
    std::swap(ik, ok);
    std::swap(ip, op);
  }
  count_launch(ctx, 9);
  timing_kernel_end(ctx);
  // 4 passes: keys -> tmp -> keys -> tmp -> keys; the result is in `keys`
}

}  // namespace

void radix_owner_histogram(crys_ctx* ctx, const int32_t* d_keys, int64_t n, int start, int bits,
                           int64_t num_owners, int64_t* h_counts) {
  CRYS_CHECK(bits >= 1 && bits <= 8 && start >= 0 && start + bits <= 32, CRYS_ECONFIG,
             "RadixPass: bit range exceeds 32-bit keys");
  CRYS_CHECK(num_owners >= 1, CRYS_ECONFIG, "radix_histogram: need at least one owner");
  cudaStream_t st = ctx->stream;
  if (!ctx->sws) ctx->sws.reset(new SortWorkspace());
  SortWorkspace& ws = *ctx->sws;
  const int D = 1 << bits;
  int64_t chunk = (n + num_owners - 1) / num_owners;
  if (chunk == 0) chunk = 1;
  const size_t cells = (size_t)num_owners * D;
  ws.hist.reserve(sizeof(unsigned long long) * cells);
  CUDA_TRY(cudaMemsetAsync(ws.hist.p, 0, sizeof(unsigned long long) * cells, st));
  if (n > 0) {
    const int grid = (int)std::min<int64_t>((n + kHistTile - 1) / kHistTile, (int64_t)ctx->num_sms * 8);
    owner_hist_kernel<<<grid, 256, 0, st>>>(d_keys, n, chunk, start, bits, ws.hist.as<unsigned long long>());
    CRYS_LAUNCHED("owner_hist_kernel");
    count_launch(ctx);
  }
  CUDA_TRY(cudaMemcpyAsync(h_counts, ws.hist.p, sizeof(int64_t) * cells, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
}

// One stable partition pass (radix_shuffle with pass.stable, radix.cpp:75-136):
// the output of per-owner cursors over column-major offsets is exactly the
// stable partition by digit, independent of the owner count -- one onesweep pass.
void radix_partition_pass(crys_ctx* ctx, const int32_t* sk, const int32_t* sp, int32_t* dk, int32_t* dp,
                          int64_t n, int start, int bits) {
  CRYS_CHECK(bits >= 1 && bits <= 8 && start >= 0 && start + bits <= 32, CRYS_ECONFIG,
             "RadixPass: bit range exceeds 32-bit keys");
  if (n == 0) return;
  CRYS_CHECK(n < (1LL << 30), CRYS_ENOTBUILT, "partition supports fewer than 2^30 pairs");
  if (!ctx->sws) ctx->sws.reset(new SortWorkspace());
  std::vector<int> pb{bits};
  timing_kernel_begin(ctx);
  onesweep_passes(ctx, *ctx->sws, const_cast<int32_t*>(sk), const_cast<int32_t*>(sp), dk, dp, n, start, bits, 1,
                  &pb);
  timing_kernel_end(ctx);
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
}

void sort_pairs(crys_ctx* ctx, int32_t* d_keys, int32_t* d_payloads, int64_t n, int algo,
                int bits_per_pass) {
  if (n <= 1) return;
  CRYS_CHECK(n < (1LL << 30), CRYS_ENOTBUILT, "sort supports fewer than 2^30 pairs");
  if (!ctx->sws) ctx->sws.reset(new SortWorkspace());
  if (algo == CRYS_SORT_LSB)
    lsb_sort(ctx, *ctx->sws, d_keys, d_payloads, n, bits_per_pass);
  else
    msb_sort(ctx, *ctx->sws, d_keys, d_payloads, n);
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
}

}  // namespace crys
