// Diagnostic (not product code): where does a single-pass select tile spend
// its life on B200?  Same structure as select_input_kernel (128 x 32 tile,
// 128-bit loads, warp scans, block look-back); globaltimer stamps at phase
// boundaries for every 64th tile.
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../paper_2003_01178_b200/csrc/crystal.cuh"
using namespace crys;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int MODE>  // 0 block look-back, 1 warp look-back, 2 none
__global__ void __launch_bounds__(128) probe(const int* in, long long n, int lo, int* out,
                                             unsigned long long* status, unsigned long long* stamps) {
  constexpr int BT = 128, IPT = 32, TILE = BT * IPT;
  __shared__ __align__(16) int s_items[TILE];
  __shared__ int s_warp[4];
  __shared__ long long s_red[8], s_off;
  const long long tile = blockIdx.x;
  unsigned long long t0 = gtime();
  const long long base = tile * TILE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int4 v[IPT / 4];
  const int wb = warp * 32 * IPT + 4 * lane;
#pragma unroll
  for (int j = 0; j < IPT / 4; ++j) v[j] = ld_stream4(in + base + wb + j * 128);
  int run = 0, pos[IPT / 4];
  unsigned bits[IPT / 4];
#pragma unroll
  for (int j = 0; j < IPT / 4; ++j) {
    unsigned b = (v[j].x < lo) | ((v[j].y < lo) << 1) | ((v[j].z < lo) << 2) | ((v[j].w < lo) << 3);
    bits[j] = b;
    int c = __popc(b), x = c;
    for (int o = 1; o < 32; o <<= 1) { int y = __shfl_up_sync(~0u, x, o); if (lane >= o) x += y; }
    pos[j] = run + x - c;
    run += __shfl_sync(~0u, x, 31);
  }
  unsigned long long t1 = gtime();
  if (lane == 31) s_warp[warp] = run;
  __syncthreads();
  int woff = 0, total = 0;
  for (int w = 0; w < 4; ++w) { woff += w < warp ? s_warp[w] : 0; total += s_warp[w]; }
#pragma unroll
  for (int j = 0; j < IPT / 4; ++j) {
    int p = woff + pos[j];
    if (bits[j] & 1) s_items[p++] = v[j].x;
    if (bits[j] & 2) s_items[p++] = v[j].y;
    if (bits[j] & 4) s_items[p++] = v[j].z;
    if (bits[j] & 8) s_items[p++] = v[j].w;
  }
  unsigned long long t2 = gtime();
  long long off;
  if (MODE == 0) {
    off = block_lookback<BT>(status, tile, total, s_red);
  } else if (MODE == 1) {
    if (threadIdx.x < 32) { long long o = tile_lookback(status, tile, total); if (threadIdx.x == 0) s_off = o; }
    __syncthreads();
    off = s_off;
  } else {
    __syncthreads();
    off = base;
  }
  unsigned long long t3 = gtime();
  for (int i = threadIdx.x; i < total; i += BT) out[off + i] = s_items[i];
  unsigned long long t4 = gtime();
  if (threadIdx.x == 0 && (tile & 63) == 0) {
    unsigned long long* s = stamps + (tile / 64) * 6;
    s[0] = t0; s[1] = t1; s[2] = t2; s[3] = t3; s[4] = t4;
    unsigned smid; asm("mov.u32 %0, %%smid;" : "=r"(smid)); s[5] = smid;
  }
}

__global__ void fill(int* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)i * 2654435761u; x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = x & ((1 << 20) - 1);
  }
}

template <int MODE>
void run(const int* in, int* out, long long n, unsigned long long* status, unsigned long long* stamps) {
  const long long tiles = n / 4096;
  std::vector<unsigned long long> h(tiles / 64 * 6);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int r = 0; r < 3; ++r) {
    cudaMemset(status, 0, tiles * 8);
    cudaEventRecord(a);
    probe<MODE><<<tiles, 128>>>(in, n, 1 << 19, out, status, stamps);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  cudaMemcpy(h.data(), stamps, h.size() * 8, cudaMemcpyDeviceToHost);
  double ph[4] = {0, 0, 0, 0};
  unsigned long long t_begin = ~0ull;
  for (size_t i = 0; i < h.size() / 6; ++i) t_begin = std::min(t_begin, h[i * 6]);
  for (size_t i = 0; i < h.size() / 6; ++i)
    for (int p = 0; p < 4; ++p) ph[p] += (h[i * 6 + p + 1] - h[i * 6 + p]) / 1000.0;
  const double m = h.size() / 6;
  printf("{\"mode\": %d, \"ms\": %.4f, \"load_us\": %.2f, \"compact_us\": %.2f, \"lookback_us\": %.2f, \"store_us\": %.2f",
         MODE, ms, ph[0] / m, ph[1] / m, ph[2] / m, ph[3] / m);
  // start-time spread of consecutive sampled tiles: dispatch rate
  printf(", \"tile_start_ms_last\": %.4f}\n", (h[(h.size() / 6 - 1) * 6] - t_begin) / 1e6);
}

int main() {
  const long long n = 1ll << 29;
  int *in, *out; unsigned long long *status, *stamps;
  cudaMalloc(&in, n * 4); cudaMalloc(&out, n * 4);
  cudaMalloc(&status, (n / 4096) * 8); cudaMalloc(&stamps, (n / 4096 / 64) * 6 * 8);
  fill<<<4096, 256>>>(in, n);
  run<0>(in, out, n, status, stamps);
  run<1>(in, out, n, status, stamps);
  run<2>(in, out, n, status, stamps);
  return 0;
}
