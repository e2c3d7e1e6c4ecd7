// common.cuh -- shared host/device definitions of the B200 Crystal library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "crystal_b200.h"

namespace crys {

// ------------------------------------------------------------------ errors
// Internal C++ error; converted to crys_status at the C ABI (capi.cpp).  The
// reference's exception taxonomy is include/tq/common.hpp:16-34.
struct Error : std::runtime_error {
  crys_status code;
  Error(crys_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(crys_status c, const std::string& m) { throw Error(c, m); }

#define CRYS_CHECK(cond, code, msg)              \
  do {                                           \
    if (!(cond)) ::crys::fail((code), (msg));    \
  } while (0)

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      ::crys::fail(CRYS_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// Checks the launch that was just enqueued, naming it in the error.
#define CRYS_LAUNCHED(name)                                                          \
  do {                                                                               \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess)                                                           \
      ::crys::fail(CRYS_ECUDA, std::string("launch ") + (name) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// ------------------------------------------------------------ constants
// HashTable::kEmptyKey / kFibonacci (hash_table.hpp:23-24).
constexpr int32_t kEmptyKey = INT32_MIN;
constexpr uint32_t kFibonacci = 2654435769u;

// Per-hash-table device metadata; capacity is decided ON THE DEVICE from the
// filtered build count (ssb_queries.cpp:119: cap = max(2, bit_ceil(2n))), so
// the probe kernels read mask/shift from here and no host sync is needed.
struct HtMeta {
  int32_t count;  // filtered build rows
  uint32_t mask;  // capacity - 1
  int32_t shift;  // 32 - log2(capacity)   (hash_table.cpp:12-16)
  int32_t err;    // 1 sentinel key, 2 duplicate key, 3 capacity (BuildError), 4 key outside stats
  // group digits (payload - lo) of the rows that passed the filters: the
  // extent of the group-by sub-box a query can occupy (identical on every
  // shard, since dimensions are replicated).  dmin > dmax: no digit.
  int32_t dmin, dmax;
  int32_t pad[2];
};

// Packs a {key, payload} slot into the 64-bit word atomicCAS operates on
// (int2 little-endian: x = key in the low half).
__host__ __device__ inline unsigned long long pack_slot(int32_t key, int32_t payload) {
  return (unsigned long long)(uint32_t)key | ((unsigned long long)(uint32_t)payload << 32);
}

__host__ __device__ inline uint32_t ht_slot_of(int32_t key, int shift) {
  return (uint32_t)((uint32_t)key * kFibonacci) >> shift;  // hash_table.hpp:35-37
}

// ------------------------------------------------------------ device loads
#ifdef __CUDACC__
// Streaming column loads: read-only path, do not allocate in L1 (each fact
// sector is used once) so L1 stays for hash-table slots.
__device__ __forceinline__ int4 ld_stream4(const int32_t* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int2 ld_stream2(const int32_t* p) {
  int2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int32_t ld_stream1(const int32_t* p) {
  int32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_stream4f(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream4f(float* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w));
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Programmatic dependent launch: a kernel launched with the programmatic
// stream-serialization attribute (launch_k) may become resident while its
// predecessor in the stream still runs.  pdl_wait() blocks until that
// predecessor grid has completed and its writes are visible (a no-op for a
// normally launched kernel); pdl_trigger() lets the successor start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
#endif

}  // namespace crys
