// Calibration only (not product code): what CUB's stock single-pass select
// and onesweep radix sort reach on this B200 at the microbenchmark sizes, so
// our own kernels' roofline fractions have an empirical yardstick.
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>

struct Lt {
  int v;
  __host__ __device__ bool operator()(const int& x) const { return x < v; }
};

__global__ void fill(int* p, size_t n, unsigned seed, int mod) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = mod ? (int)(x % (unsigned)mod) : (int)x;
  }
}

int main() {
  const size_t n = 1u << 29;
  int *in, *out, *nsel;
  cudaMalloc(&in, n * 4); cudaMalloc(&out, n * 4); cudaMalloc(&nsel, 8);
  fill<<<4096, 256>>>(in, n, 1234, 1 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (double sigma : {0.0, 0.5, 1.0}) {
    Lt op{(int)(sigma * (1 << 20))};
    size_t tmp = 0; void* d_tmp = nullptr;
    cub::DeviceSelect::If(d_tmp, tmp, in, out, nsel, (int)n, op);
    cudaMalloc(&d_tmp, tmp);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      cub::DeviceSelect::If(d_tmp, tmp, in, out, nsel, (int)n, op);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("{\"cub\": \"select_if\", \"n\": %zu, \"sigma\": %.1f, \"ms\": %.4f, \"gbs\": %.1f}\n", n, sigma, best,
           (4.0 * n + 4.0 * sigma * n) / best / 1e6);
    cudaFree(d_tmp);
  }
  const size_t m = 1u << 28;
  int *k0, *k1, *v0, *v1;
  cudaMalloc(&k0, m * 4); cudaMalloc(&k1, m * 4); cudaMalloc(&v0, m * 4); cudaMalloc(&v1, m * 4);
  int* kin; cudaMalloc(&kin, m * 4);
  fill<<<4096, 256>>>(kin, m, 77, 0);
  size_t tmp = 0; void* d_tmp = nullptr;
  cub::DeviceRadixSort::SortPairs(d_tmp, tmp, k0, k1, v0, v1, (int)m);
  cudaMalloc(&d_tmp, tmp);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaMemcpy(k0, kin, m * 4, cudaMemcpyDeviceToDevice);
    cudaEventRecord(a);
    cub::DeviceRadixSort::SortPairs(d_tmp, tmp, k0, k1, v0, v1, (int)m);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  printf("{\"cub\": \"sort_pairs\", \"n\": %zu, \"ms\": %.4f, \"gbs_80N\": %.1f}\n", m, best, 80.0 * m / best / 1e6);
  return 0;
}
