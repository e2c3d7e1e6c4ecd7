// radix_sort.cu -- LSB and MSB radix sort of (int32 key, int32 payload) pairs.
//
// Reference: radix.hpp:44-93, radix.cpp:33-216.
//   radix_digit      ((u32)key ^ 0x80000000) >> start & mask   (signed order)
//   radix_histogram  owner x digit counts, owner = contiguous input chunk
//   radix_offsets    column-major exclusive prefix (digit-major, owner within digit)
//   radix_shuffle    stable scatter: each owner writes its runs in input order
//   lsb_radix_sort   stable passes low->high (default 4 x 8 bit) == std::stable_sort
//   msb_radix_sort   8-bit MSB recursion from bit 24; small partitions sorted directly
//
// B200 form: an "owner" is a CTA with a contiguous chunk.  One pass =
//   radix_upsweep_kernel    per-CTA digit histogram (smem, vectorised loads)
//   radix_scan_kernel       column-major exclusive scan per segment
//   radix_downsweep_kernel  per tile: warp-level stable ranking (match.any),
//                           shared-memory reorder, coalesced-run scatter
// Traffic per pass = 4N (upsweep) + 8N read + 8N write = 20N, exactly the
// reference's bytes_moved convention (tools/tq_main.cpp:482-483).
// The same kernels run SEGMENTED for MSB: every segment is an independent
// sub-array with its own CTAs and scan; segments that fit shared memory are
// finished by one CTA with a bitonic sort (msb_recurse base case, radix.cpp:184-187).
#include <algorithm>
#include <vector>

#include "crystal.cuh"
#include "internal.hpp"

namespace crys {
namespace {

constexpr int kUpBT = 512;
constexpr int kDnBT = 512, kDnIPT = 16;            // 8192-pair tiles
constexpr int kDnTile = kDnBT * kDnIPT;
constexpr int kDnWarps = kDnBT / 32;
constexpr int kLocalMax = 8192;                     // bitonic base case (64 KB smem)
constexpr int kLocalBT = 1024;

struct SegCta {  // one owner: [begin, end) of segment `seg`
  int64_t begin, end;
  int32_t seg, cta_in_seg;
};
struct SegInfo {
  int64_t begin, size;
  int32_t first_cta, ncta;
};
struct SegLocal {
  int64_t begin, size;
};

__device__ __forceinline__ uint32_t digit_of(int32_t key, int start, uint32_t mask) {
  return (((uint32_t)key ^ 0x80000000u) >> start) & mask;  // radix.hpp:44-47
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// hist layout: segment s occupies [first_cta*D, (first_cta+ncta)*D), digit-major
// inside: index first_cta*D + d*ncta + cta_in_seg (column-major, radix.cpp:55-73).
__global__ void __launch_bounds__(kUpBT) radix_upsweep_kernel(const int32_t* __restrict__ keys,
                                                              const SegCta* ctas,
                                                              const SegInfo* segs, int start,
                                                              int bits, uint32_t* hist) {
  __shared__ uint32_t h[kUpBT / 32][256];
  const int D = 1 << bits;
  const uint32_t mask = (uint32_t)D - 1;
  const unsigned warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (kUpBT / 32) * 256; i += kUpBT) (&h[0][0])[i] = 0;
  __syncthreads();
  const SegCta c = ctas[blockIdx.x];
  int64_t i = c.begin + threadIdx.x * 4;
  // vectorised body when the chunk start is 16 B aligned
  if ((c.begin & 3) == 0 && (reinterpret_cast<uintptr_t>(keys) & 15) == 0) {
    for (; i + 3 < c.end; i += kUpBT * 4) {
      const int4 k = ld_stream4(keys + i);
      atomicAdd(&h[warp][digit_of(k.x, start, mask)], 1u);
      atomicAdd(&h[warp][digit_of(k.y, start, mask)], 1u);
      atomicAdd(&h[warp][digit_of(k.z, start, mask)], 1u);
      atomicAdd(&h[warp][digit_of(k.w, start, mask)], 1u);
    }
    for (int64_t j = i; j < c.end && j < i + 4; ++j) atomicAdd(&h[warp][digit_of(keys[j], start, mask)], 1u);
  } else {
    for (int64_t j = c.begin + threadIdx.x; j < c.end; j += kUpBT)
      atomicAdd(&h[warp][digit_of(keys[j], start, mask)], 1u);
  }
  __syncthreads();
  const SegInfo s = segs[c.seg];
  for (int d = threadIdx.x; d < D; d += kUpBT) {
    uint32_t t = 0;
    for (int w = 0; w < kUpBT / 32; ++w) t += h[w][d];
    hist[(int64_t)s.first_cta * D + (int64_t)d * s.ncta + c.cta_in_seg] = t;
  }
}

// One CTA per segment: in-place exclusive scan of its D*ncta counters; also
// records each digit's base (first owner's offset) for MSB planning.
__global__ void __launch_bounds__(1024) radix_scan_kernel(uint32_t* hist, const SegInfo* segs,
                                                          int bits, uint32_t* digit_base) {
  __shared__ uint32_t sm[33];
  const SegInfo s = segs[blockIdx.x];
  const int D = 1 << bits;
  const int64_t len = (int64_t)D * s.ncta;
  uint32_t* h = hist + (int64_t)s.first_cta * D;
  const int64_t per = (len + 1023) / 1024;
  const int64_t b = threadIdx.x * per, e = min(len, b + per);
  uint32_t local = 0;
  for (int64_t i = b; i < e; ++i) local += h[i];
  uint32_t tot;
  uint32_t run = BlockScan<1024>(local, sm, tot);
  for (int64_t i = b; i < e; ++i) {
    const uint32_t v = h[i];
    h[i] = run;
    run += v;
  }
  __syncthreads();
  if (digit_base)
    for (int d = threadIdx.x; d < D; d += 1024)
      digit_base[(int64_t)blockIdx.x * 256 + d] = h[(int64_t)d * s.ncta];
}

__global__ void __launch_bounds__(kDnBT) radix_downsweep_kernel(
    const int32_t* __restrict__ kin, const int32_t* __restrict__ pin, int32_t* __restrict__ kout,
    int32_t* __restrict__ pout, const SegCta* ctas, const SegInfo* segs, const uint32_t* hist,
    int start, int bits) {
  extern __shared__ int32_t smem[];
  int32_t* s_k = smem;                                       // [kDnTile]
  int32_t* s_p = smem + kDnTile;                             // [kDnTile]
  uint32_t* s_wc = reinterpret_cast<uint32_t*>(smem + 2 * kDnTile);  // [kDnWarps][256]
  uint32_t* s_off = s_wc + kDnWarps * 256;                   // [256] running global offsets
  uint32_t* s_start = s_off + 256;                           // [257] tile digit starts
  __shared__ uint32_t s_scan[kDnBT / 32 + 1];

  const int D = 1 << bits;
  const uint32_t mask = (uint32_t)D - 1;
  const SegCta c = ctas[blockIdx.x];
  const SegInfo sg = segs[c.seg];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < 256; d += kDnBT)
    s_off[d] = d < D ? hist[(int64_t)sg.first_cta * D + (int64_t)d * sg.ncta + c.cta_in_seg] : 0;

  for (int64_t base = c.begin; base < c.end; base += kDnTile) {
    const int valid = (int)min((int64_t)kDnTile, c.end - base);
    for (int i = threadIdx.x; i < kDnWarps * 256; i += kDnBT) s_wc[i] = 0;
    __syncthreads();
    // warp-striped ownership: item k of lane l in warp w is tile slot
    // w*32*IPT + k*32 + l, so (k, lane) order is input order within the warp.
    int32_t key[kDnIPT], pay[kDnIPT];
    uint32_t rank[kDnIPT], dg[kDnIPT];
    const int wbase = warp * 32 * kDnIPT;
#pragma unroll
    for (int k = 0; k < kDnIPT; ++k) {
      const int s = wbase + k * 32 + lane;
      if (s < valid) {
        key[k] = ld_stream1(kin + base + s);
        pay[k] = ld_stream1(pin + base + s);
        dg[k] = digit_of(key[k], start, mask);
      } else {
        dg[k] = 256;  // out-of-tile sentinel, never counted
      }
    }
    uint32_t* wc = s_wc + warp * 256;
#pragma unroll
    for (int k = 0; k < kDnIPT; ++k) {
      const unsigned peers = __match_any_sync(0xffffffffu, dg[k]);
      const unsigned below = __popc(peers & lanemask_lt());
      const bool leader = below == 0;
      uint32_t basec = 0;
      if (dg[k] < 256) basec = wc[dg[k]];
      rank[k] = basec + below;
      __syncwarp();
      if (leader && dg[k] < 256) wc[dg[k]] = basec + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // per digit: warp-exclusive prefix (in place) and the tile total
    uint32_t tot = 0;
    if (threadIdx.x < 256) {
      const int d = threadIdx.x;
      for (int w = 0; w < kDnWarps; ++w) {
        const uint32_t v = s_wc[w * 256 + d];
        s_wc[w * 256 + d] = tot;
        tot += v;
      }
    }
    uint32_t all;
    const uint32_t st = BlockScan<kDnBT>(threadIdx.x < 256 ? tot : 0u, s_scan, all);
    if (threadIdx.x < 256) s_start[threadIdx.x] = st;
    if (threadIdx.x == 0) s_start[256] = all;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kDnIPT; ++k) {
      if (dg[k] < 256) {
        const uint32_t pos = s_start[dg[k]] + s_wc[warp * 256 + dg[k]] + rank[k];
        s_k[pos] = key[k];
        s_p[pos] = pay[k];
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < valid; i += kDnBT) {
      const int32_t kk = s_k[i];
      const uint32_t d = digit_of(kk, start, mask);
      const int64_t dst = sg.begin + (int64_t)s_off[d] + (i - (int64_t)s_start[d]);
      kout[dst] = kk;
      pout[dst] = s_p[i];
    }
    __syncthreads();
    if (threadIdx.x < 256) s_off[threadIdx.x] += s_start[threadIdx.x + 1] - s_start[threadIdx.x];
    __syncthreads();
  }
}

// Base case: one CTA sorts a segment of <= kLocalMax pairs in shared memory
// (bitonic network over a power-of-two padded array; keys ascending).
__global__ void __launch_bounds__(kLocalBT) local_sort_kernel(int32_t* keys, int32_t* pays,
                                                             const SegLocal* segs) {
  extern __shared__ int32_t s_local[];
  int32_t* sk = s_local;
  int32_t* sp = s_local + kLocalMax;
  const SegLocal s = segs[blockIdx.x];
  int n2 = 1;
  while (n2 < s.size) n2 <<= 1;
  for (int i = threadIdx.x; i < n2; i += kLocalBT) {
    if (i < s.size) {
      sk[i] = keys[s.begin + i];
      sp[i] = pays[s.begin + i];
    } else {
      sk[i] = INT32_MAX;
      sp[i] = 0;
    }
  }
  __syncthreads();
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < n2 / 2; t += kLocalBT) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const bool up = (i & size) == 0;
        const int32_t a = sk[i], b = sk[j];
        if ((a > b) == up) {
          sk[i] = b;
          sk[j] = a;
          const int32_t x = sp[i];
          sp[i] = sp[j];
          sp[j] = x;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < s.size; i += kLocalBT) {
    keys[s.begin + i] = sk[i];
    pays[s.begin + i] = sp[i];
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

__global__ void copy_pairs_kernel(const int32_t* ks, const int32_t* ps, int32_t* kd, int32_t* pd,
                                  const SegLocal* segs) {
  const SegLocal s = segs[blockIdx.y];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s.size;
       i += (int64_t)gridDim.x * blockDim.x) {
    kd[s.begin + i] = ks[s.begin + i];
    pd[s.begin + i] = ps[s.begin + i];
  }
}

}  // namespace

struct SortWorkspace {
  DevBuf tk, tp;          // ping-pong pair arrays
  DevBuf ctas, segs, hist, digit_base, locals;
};

void WsDeleter::operator()(SortWorkspace* p) const { delete p; }

namespace {

size_t down_smem() {
  return sizeof(int32_t) * (2 * kDnTile) + sizeof(uint32_t) * (kDnWarps * 256 + 256 + 257);
}

void set_down_smem() {
  static bool done = false;
  if (!done) {
    CUDA_TRY(cudaFuncSetAttribute((const void*)radix_downsweep_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)down_smem()));
    done = true;
  }
}

// Plans owners (CTAs) for a set of segments: ~target pairs per CTA, chunk
// boundaries tile-aligned inside each segment.
void plan_ctas(const std::vector<SegLocal>& in, int64_t target, std::vector<SegCta>& ctas,
               std::vector<SegInfo>& segs) {
  ctas.clear();
  segs.clear();
  for (size_t s = 0; s < in.size(); ++s) {
    const int64_t n = in[s].size;
    int64_t nc = std::max<int64_t>(1, (n + target - 1) / target);
    int64_t chunk = (n + nc - 1) / nc;
    chunk = (chunk + kDnTile - 1) / kDnTile * kDnTile;
    nc = std::max<int64_t>(1, (n + chunk - 1) / chunk);
    SegInfo si{in[s].begin, n, (int32_t)ctas.size(), (int32_t)nc};
    for (int64_t c = 0; c < nc; ++c) {
      const int64_t b = in[s].begin + c * chunk;
      const int64_t e = std::min(in[s].begin + n, b + chunk);
      ctas.push_back({b, e, (int32_t)s, (int32_t)c});
    }
    segs.push_back(si);
  }
}

// One (segmented) radix pass src -> dst over `segments`; returns per-segment
// digit bases (host) when `want_bases`.
void radix_pass(crys_ctx* ctx, SortWorkspace& ws, const int32_t* sk, const int32_t* sp, int32_t* dk,
                int32_t* dp, const std::vector<SegLocal>& segments, int start, int bits,
                std::vector<uint32_t>* bases) {
  cudaStream_t st = ctx->stream;
  std::vector<SegCta> ctas;
  std::vector<SegInfo> segs;
  int64_t total = 0;
  for (auto& s : segments) total += s.size;
  // ~4 owners per SM worth of work when one segment; proportional otherwise
  const int64_t target = std::max<int64_t>(kDnTile, total / ((int64_t)ctx->num_sms * 4) + 1);
  plan_ctas(segments, target, ctas, segs);
  const int D = 1 << bits;
  ws.ctas.reserve(sizeof(SegCta) * ctas.size());
  ws.segs.reserve(sizeof(SegInfo) * segs.size());
  ws.hist.reserve(sizeof(uint32_t) * ctas.size() * (size_t)D);
  ws.digit_base.reserve(sizeof(uint32_t) * segs.size() * 256);
  CUDA_TRY(cudaMemcpyAsync(ws.ctas.p, ctas.data(), sizeof(SegCta) * ctas.size(), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(ws.segs.p, segs.data(), sizeof(SegInfo) * segs.size(), cudaMemcpyHostToDevice, st));
  radix_upsweep_kernel<<<(unsigned)ctas.size(), kUpBT, 0, st>>>(sk, ws.ctas.as<SegCta>(), ws.segs.as<SegInfo>(),
                                                                start, bits, ws.hist.as<uint32_t>());
  radix_scan_kernel<<<(unsigned)segs.size(), 1024, 0, st>>>(ws.hist.as<uint32_t>(), ws.segs.as<SegInfo>(), bits,
                                                            bases ? ws.digit_base.as<uint32_t>() : nullptr);
  set_down_smem();
  radix_downsweep_kernel<<<(unsigned)ctas.size(), kDnBT, down_smem(), st>>>(
      sk, sp, dk, dp, ws.ctas.as<SegCta>(), ws.segs.as<SegInfo>(), ws.hist.as<uint32_t>(), start, bits);
  count_launch(ctx, 3);
  CUDA_TRY(cudaGetLastError());
  if (bases) {
    bases->resize(segs.size() * 256);
    CUDA_TRY(cudaMemcpyAsync(bases->data(), ws.digit_base.p, sizeof(uint32_t) * bases->size(),
                             cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  // host vectors must outlive the async H2D copies
  CUDA_TRY(cudaStreamSynchronize(st));
}

void lsb_sort(crys_ctx* ctx, SortWorkspace& ws, int32_t* keys, int32_t* pays, int64_t n, int bpp) {
  ws.tk.reserve(sizeof(int32_t) * (size_t)n);
  ws.tp.reserve(sizeof(int32_t) * (size_t)n);
  int32_t *sk = keys, *sp = pays, *dk = ws.tk.as<int32_t>(), *dp = ws.tp.as<int32_t>();
  std::vector<SegLocal> one{{0, n}};
  timing_kernel_begin(ctx);
  for (int start = 0; start < 32; start += bpp) {  // lsb_radix_sort, radix.cpp:151-159
    const int bits = std::min(bpp, 32 - start);
    radix_pass(ctx, ws, sk, sp, dk, dp, one, start, bits, nullptr);
    std::swap(sk, dk);
    std::swap(sp, dp);
  }
  timing_kernel_end(ctx);
  if (sk != keys) {
    CUDA_TRY(cudaMemcpyAsync(keys, sk, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(pays, sp, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
}

// msb_recurse (radix.cpp:181-206), level-synchronous: every segment still
// larger than the shared-memory base case takes one more 8-bit pass.
void msb_sort(crys_ctx* ctx, SortWorkspace& ws, int32_t* keys, int32_t* pays, int64_t n) {
  cudaStream_t st = ctx->stream;
  ws.tk.reserve(sizeof(int32_t) * (size_t)n);
  ws.tp.reserve(sizeof(int32_t) * (size_t)n);
  int32_t* bufk[2] = {keys, ws.tk.as<int32_t>()};
  int32_t* bufp[2] = {pays, ws.tp.as<int32_t>()};
  int cur = 0;  // buffer holding the live data of the pending segments
  std::vector<SegLocal> pending{{0, n}};
  std::vector<SegLocal> local_in[2];  // finished-by-local-sort segments per buffer
  std::vector<SegLocal> done_in[2];   // already final (size <= 1 or all bits used)
  timing_kernel_begin(ctx);
  for (int start = 24; start >= 0 && !pending.empty(); start -= 8) {
    std::vector<SegLocal> big, small;
    for (auto& s : pending) {
      if (s.size <= 1) done_in[cur].push_back(s);
      else if (s.size <= kLocalMax) small.push_back(s);
      else big.push_back(s);
    }
    local_in[cur].insert(local_in[cur].end(), small.begin(), small.end());
    pending.clear();
    if (big.empty()) break;
    std::vector<uint32_t> bases;
    radix_pass(ctx, ws, bufk[cur], bufp[cur], bufk[cur ^ 1], bufp[cur ^ 1], big, start, 8, &bases);
    cur ^= 1;
    for (size_t s = 0; s < big.size(); ++s) {
      for (int d = 0; d < 256; ++d) {
        const int64_t lo = bases[s * 256 + d];
        const int64_t hi = d + 1 < 256 ? (int64_t)bases[s * 256 + d + 1] : big[s].size;
        if (hi - lo > 0) pending.push_back({big[s].begin + lo, hi - lo});
      }
    }
    if (start == 0) {  // all 32 bits consumed: segments hold equal keys
      for (auto& s : pending) done_in[cur].push_back(s);
      pending.clear();
    }
  }
  for (auto& s : pending) local_in[cur].push_back(s);
  // Gather every final segment into `keys`: sort locally in place when the
  // segment lives in `keys`, otherwise copy it over first.
  std::vector<SegLocal> to_copy = local_in[1];
  to_copy.insert(to_copy.end(), done_in[1].begin(), done_in[1].end());
  if (!to_copy.empty()) {
    ws.locals.reserve(sizeof(SegLocal) * to_copy.size());
    CUDA_TRY(cudaMemcpyAsync(ws.locals.p, to_copy.data(), sizeof(SegLocal) * to_copy.size(),
                             cudaMemcpyHostToDevice, st));
    for (size_t b = 0; b < to_copy.size(); b += 65535) {
      const unsigned cnt = (unsigned)std::min<size_t>(65535, to_copy.size() - b);
      copy_pairs_kernel<<<dim3(8, cnt), 256, 0, st>>>(bufk[1], bufp[1], keys, pays,
                                                      ws.locals.as<SegLocal>() + b);
      count_launch(ctx);
    }
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  std::vector<SegLocal> locals = local_in[0];
  locals.insert(locals.end(), local_in[1].begin(), local_in[1].end());
  if (!locals.empty()) {
    ws.locals.reserve(sizeof(SegLocal) * locals.size());
    CUDA_TRY(cudaMemcpyAsync(ws.locals.p, locals.data(), sizeof(SegLocal) * locals.size(),
                             cudaMemcpyHostToDevice, st));
    static bool attr = false;
    if (!attr) {
      CUDA_TRY(cudaFuncSetAttribute((const void*)local_sort_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(2 * kLocalMax * sizeof(int32_t))));
      attr = true;
    }
    local_sort_kernel<<<(unsigned)locals.size(), kLocalBT, 2 * kLocalMax * sizeof(int32_t), st>>>(keys, pays, ws.locals.as<SegLocal>());
    count_launch(ctx);
    CUDA_TRY(cudaGetLastError());
  }
  timing_kernel_end(ctx);
  CUDA_TRY(cudaStreamSynchronize(st));
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
// stable partition by digit, independent of the owner count.
void radix_partition_pass(crys_ctx* ctx, const int32_t* sk, const int32_t* sp, int32_t* dk, int32_t* dp,
                          int64_t n, int start, int bits) {
  CRYS_CHECK(bits >= 1 && bits <= 8 && start >= 0 && start + bits <= 32, CRYS_ECONFIG,
             "RadixPass: bit range exceeds 32-bit keys");
  if (n == 0) return;
  CRYS_CHECK(n < (1LL << 32), CRYS_ENOTBUILT, "partition supports fewer than 2^32 pairs");
  if (!ctx->sws) ctx->sws.reset(new SortWorkspace());
  std::vector<SegLocal> one{{0, n}};
  timing_kernel_begin(ctx);
  radix_pass(ctx, *ctx->sws, sk, sp, dk, dp, one, start, bits, nullptr);
  timing_kernel_end(ctx);
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
}

void sort_pairs(crys_ctx* ctx, int32_t* d_keys, int32_t* d_payloads, int64_t n, int algo,
                int bits_per_pass) {
  if (n <= 1) return;
  CRYS_CHECK(n < (1LL << 32), CRYS_ENOTBUILT, "sort supports fewer than 2^32 pairs");
  if (!ctx->sws) ctx->sws.reset(new SortWorkspace());
  if (algo == CRYS_SORT_LSB)
    lsb_sort(ctx, *ctx->sws, d_keys, d_payloads, n, bits_per_pass);
  else
    msb_sort(ctx, *ctx->sws, d_keys, d_payloads, n);
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
}

}  // namespace crys
