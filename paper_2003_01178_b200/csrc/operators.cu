// operators.cu -- selection, projection and hash-join microbenchmark kernels.
//
//   select_input_kernel    select_{branching,predicated}_into(workers=1)
//                          (select.hpp:56-91): input-order output, single pass
//                          with decoupled look-back (no 3-kernel count/scan/write)
//   select_crystal_kernel  select_tile_into(config, kDeterministic)
//                          (select.hpp:107-135): the exact Crystal order for any
//                          TileConfig -- logical threads over a smem-staged tile
//   project_kernel         project_{linear,sigmoid}_into (project.hpp:21-64)
//   ht_init/insert_kernel  HashTable::build (hash_table.cpp:20-94)
//   join_probe_kernel      join_probe_* (join.cpp:11-96): Q4 checksum, the
//                          table staged in shared memory when it fits, else
//                          probed L2/HBM-resident
#include <algorithm>
#include <map>
#include <mutex>

#include "crystal.cuh"
#include "internal.hpp"

namespace crys {
namespace {

constexpr int kSelBT = 256, kSelIPT = 16;  // native select tile (4096 rows, 16 KB)

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Input-order selection: persistent CTAs walk tiles blockIdx.x, +gridDim.x,
// ...; the NEXT tile's 128-bit loads are issued before the current tile's
// scan + decoupled look-back, so HBM reads overlap the serial part.  Every
// CTA is resident and walks its tiles in increasing order, so each tile's
// predecessors are always in progress or done (no look-back deadlock).
template <int BT, int IPT>
__global__ void __launch_bounds__(BT) select_input_kernel(const int32_t* __restrict__ in, int64_t n,
                                                          int32_t lo, int32_t hi,
                                                          int32_t* __restrict__ out,
                                                          unsigned long long* status,
                                                          long long ntiles, long long* total_out) {
  using L = VecLayout<BT, IPT>;
  static_assert(L::NV <= 4 && BT * L::VEC < 65536, "packed 16-bit per-vector counts");
  __shared__ int32_t s_items[L::TILE];
  __shared__ unsigned long long s_scan[BT / 32 + 1];
  __shared__ long long s_off;
  long long tile = blockIdx.x;
  if (tile >= ntiles) return;
  int32_t cur[IPT], nxt[IPT];
  BlockLoad<BT, IPT>(in + tile * L::TILE, (int)min((int64_t)L::TILE, (int64_t)(n - tile * L::TILE)), cur);
  for (; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * L::TILE;
    const int valid = (int)min((int64_t)L::TILE, n - base);
    const long long nt = tile + gridDim.x;
    if (nt < ntiles)  // prefetch: in flight during this tile's scan/look-back/store
      BlockLoad<BT, IPT>(in + nt * L::TILE, (int)min((int64_t)L::TILE, (int64_t)(n - nt * L::TILE)), nxt);
    const unsigned f = BlockPred<IPT>(cur, lo, hi, BlockValidMask<BT, IPT>(valid));
    // Input order inside the tile is (vector v, thread, element): scan the
    // per-vector counts of all threads at once, packed 16 bits per vector.
    unsigned long long packed = 0;
#pragma unroll
    for (int v = 0; v < L::NV; ++v) packed |= (unsigned long long)__popc(L::vec_bits(f, v)) << (16 * v);
    unsigned long long tot;
    const unsigned long long ex = BlockScan<BT>(packed, s_scan, tot);
    int run = 0;
#pragma unroll
    for (int v = 0; v < L::NV; ++v) {
      int pos = run + (int)((ex >> (16 * v)) & 0xffff);
#pragma unroll
      for (int e = 0; e < L::VEC; ++e)
        if ((f >> (v * L::VEC + e)) & 1u) s_items[pos++] = cur[v * L::VEC + e];
      run += (int)((tot >> (16 * v)) & 0xffff);
    }
    const int tile_total = run;
    if (threadIdx.x < 32) {
      const long long off = tile_lookback(status, tile, tile_total);
      if (threadIdx.x == 0) s_off = off;
    }
    __syncthreads();
    const long long off = s_off;
    for (int i = threadIdx.x; i < tile_total; i += BT) out[off + i] = s_items[i];
    if (threadIdx.x == 0 && tile == ntiles - 1) *total_out = off + tile_total;
    __syncthreads();  // s_items / s_off reuse
#pragma unroll
    for (int k = 0; k < IPT; ++k) cur[k] = nxt[k];
  }
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
  for (int i = threadIdx.x; i < total; i += kCrysPB) out[off + i] = s_out[i];
  if (threadIdx.x == 0 && base + chunk >= n) *total_out = off + total;
}

// project.hpp:49-64.  Linear: float mul, float mul, float add with no FMA
// contraction (explicit _rn intrinsics).  Sigmoid: double z (the two products
// are exact in double), 1/(1+exp(-z)) in double, rounded once to float.
template <bool SIGMOID>
__device__ __forceinline__ float project_one(float u, float v, float a, float b) {
  if constexpr (!SIGMOID) {
    return __fadd_rn(__fmul_rn(a, u), __fmul_rn(b, v));
  } else {
    const double z = __dadd_rn(__dmul_rn((double)a, (double)u), __dmul_rn((double)b, (double)v));
    return __double2float_rn(__ddiv_rn(1.0, __dadd_rn(1.0, exp(-z))));
  }
}

template <bool SIGMOID>
__global__ void __launch_bounds__(256) project_kernel(const float* __restrict__ x1,
                                                      const float* __restrict__ x2, int64_t n,
                                                      float a, float b, float* __restrict__ out) {
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 u = ld_stream4f(x1 + 4 * i);
    const float4 v = ld_stream4f(x2 + 4 * i);
    float4 r;
    r.x = project_one<SIGMOID>(u.x, v.x, a, b);
    r.y = project_one<SIGMOID>(u.y, v.y, a, b);
    r.z = project_one<SIGMOID>(u.z, v.z, a, b);
    r.w = project_one<SIGMOID>(u.w, v.w, a, b);
    st_stream4f(out + 4 * i, r);
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = project_one<SIGMOID>(x1[i], x2[i], a, b);
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
    BlockLoad<BT, IPT>(keys + base, valid, k);
    BlockLoad<BT, IPT>(pays + base, valid, p);
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

int occupancy(const void* fn, int bt, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, size_t>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(fn, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  ensure_dyn_smem(fn, smem);
  int nb = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, bt, smem));
  cache[key] = std::max(nb, 1);
  return cache[key];
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
  if (order == CRYS_ORDER_INPUT) {
    tile = (int64_t)kSelBT * kSelIPT;
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
  ctx->status.reserve(sizeof(unsigned long long) * (size_t)(ntiles + 2));
  auto* status = ctx->status.as<unsigned long long>();
  auto* total = reinterpret_cast<long long*>(status + ntiles + 1);
  CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(unsigned long long) * (size_t)(ntiles + 2), st));
  timing_kernel_begin(ctx);
  if (order == CRYS_ORDER_INPUT) {
    auto fn = select_input_kernel<kSelBT, kSelIPT>;
    const int nb = occupancy((const void*)fn, kSelBT, 0);
    const int grid = (int)std::min<int64_t>(ntiles, (int64_t)nb * ctx->num_sms);
    fn<<<grid, kSelBT, 0, st>>>(d_in, n, lo, hi, d_out, status, ntiles, total);
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
  if (n > 0) {
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

}  // namespace crys
