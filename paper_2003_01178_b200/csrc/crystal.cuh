// crystal.cuh -- the Crystal block-wide primitives (PAPER Table 1) for sm_100a.
//
// The reference restates them for a CPU "block" in include/tq/block_ops.hpp
// (block_load :23-32, block_load_sel :36-50, block_pred :54-69, block_scan
// :73-82, block_thread_counts :85-96, block_shuffle :101-122, block_store
// :125-131, block_aggregate :141-173) and include/tq/hash_table.hpp (probe
// :41-51, block_lookup :68-87, build hash_table.cpp:20-94).  Here a tile lives
// in REGISTERS: each of the BT threads of a CTA owns IPT items, and flags are a
// per-thread bitmask (bit k = item k) instead of a 1-byte-per-slot bitmap.
//
// Two ownership layouts:
//   Striped   item k of thread t is tile slot t + k*BT (the reference's
//             logical-thread ownership, tile.hpp:3-8; coalesced scalar loads).
//   VecLayout item k of thread t is slot (k/VEC)*BT*VEC + t*VEC + k%VEC: every
//             load instruction is one VEC-wide vector per lane and a warp
//             covers 32*VEC*4 contiguous bytes -> 128-bit coalesced HBM reads.
//             A selective load (BlockLoadSel) skips a whole vector when none of
//             its VEC flags is set, so dead 32 B sectors are never requested.
#pragma once

#include "common.cuh"

namespace crys {

template <int BT, int IPT>
struct VecLayout {
  static constexpr int VEC = (IPT % 4 == 0) ? 4 : ((IPT % 2 == 0) ? 2 : 1);
  static constexpr int NV = IPT / VEC;
  static constexpr int TILE = BT * IPT;
  static_assert(IPT >= 1 && IPT <= 32, "flags are a 32-bit mask");
  __device__ __forceinline__ static int slot(int t, int k) {
    return (k / VEC) * BT * VEC + t * VEC + (k % VEC);
  }
  __device__ __forceinline__ static unsigned vec_bits(unsigned flags, int v) {
    return (flags >> (v * VEC)) & ((1u << VEC) - 1u);
  }
};

// Items of this thread that fall inside a partial tile of `valid` slots.
template <int BT, int IPT>
__device__ __forceinline__ unsigned BlockValidMask(int valid) {
  using L = VecLayout<BT, IPT>;
  if (valid >= L::TILE) return IPT == 32 ? 0xffffffffu : ((1u << IPT) - 1u);
  unsigned m = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k)
    if (L::slot(threadIdx.x, k) < valid) m |= 1u << k;
  return m;
}

// BlockLoad (block_ops.hpp:23-32): the thread's items of a tile, VecLayout.
// Slots at/after `valid` are not read (their items stay undefined, like the
// reference's poisoned slots).
template <int BT, int IPT>
__device__ __forceinline__ void BlockLoad(const int32_t* __restrict__ tile, int valid,
                                          int32_t (&items)[IPT]) {
  using L = VecLayout<BT, IPT>;
#pragma unroll
  for (int v = 0; v < L::NV; ++v) {
    const int s = v * BT * L::VEC + threadIdx.x * L::VEC;
    const int32_t* p = tile + s;
    if (s + L::VEC <= valid) {
      if constexpr (L::VEC == 4) {
        int4 x = ld_stream4(p);
        items[v * 4 + 0] = x.x; items[v * 4 + 1] = x.y; items[v * 4 + 2] = x.z; items[v * 4 + 3] = x.w;
      } else if constexpr (L::VEC == 2) {
        int2 x = ld_stream2(p);
        items[v * 2 + 0] = x.x; items[v * 2 + 1] = x.y;
      } else {
        items[v] = ld_stream1(p);
      }
    } else {
#pragma unroll
      for (int e = 0; e < L::VEC; ++e)
        if (s + e < valid) items[v * L::VEC + e] = ld_stream1(p + e);
    }
  }
}

// BlockLoad for a tile base that may not be 16 B aligned (a caller's span
// starting mid-vector): same VecLayout, scalar loads.
template <int BT, int IPT>
__device__ __forceinline__ void BlockLoadUnaligned(const int32_t* __restrict__ tile, int valid,
                                                   int32_t (&items)[IPT]) {
  using L = VecLayout<BT, IPT>;
#pragma unroll
  for (int v = 0; v < L::NV; ++v) {
    const int s = v * BT * L::VEC + threadIdx.x * L::VEC;
#pragma unroll
    for (int e = 0; e < L::VEC; ++e)
      if (s + e < valid) items[v * L::VEC + e] = ld_stream1(tile + s + e);
  }
}

// BlockLoadSel (block_ops.hpp:36-50): load only vectors holding a set flag.
// A fully false bitmap touches no source memory, as in the reference.
template <int BT, int IPT>
__device__ __forceinline__ void BlockLoadSel(const int32_t* __restrict__ tile, int valid,
                                             unsigned flags, int32_t (&items)[IPT]) {
  using L = VecLayout<BT, IPT>;
#pragma unroll
  for (int v = 0; v < L::NV; ++v) {
    if (L::vec_bits(flags, v) == 0) continue;
    const int s = v * BT * L::VEC + threadIdx.x * L::VEC;
    const int32_t* p = tile + s;
    if (s + L::VEC <= valid) {
      if constexpr (L::VEC == 4) {
        int4 x = ld_stream4(p);
        items[v * 4 + 0] = x.x; items[v * 4 + 1] = x.y; items[v * 4 + 2] = x.z; items[v * 4 + 3] = x.w;
      } else if constexpr (L::VEC == 2) {
        int2 x = ld_stream2(p);
        items[v * 2 + 0] = x.x; items[v * 2 + 1] = x.y;
      } else {
        items[v] = ld_stream1(p);
      }
    } else {
#pragma unroll
      for (int e = 0; e < L::VEC; ++e)
        if (s + e < valid) items[v * L::VEC + e] = ld_stream1(p + e);
    }
  }
}

// ---------------------------------------------------------------- Striped
// The reference's logical ownership (tile.hpp:3-8, block_ops.hpp:1-8): item k
// of logical thread t is tile slot t + k*bt.  `bt` is a runtime value (any
// positive TileConfig); CTA threads t >= bt own no slot.

// Items of this thread inside a (partial) tile of `valid` slots, ipt <= IPT.
template <int IPT>
__device__ __forceinline__ unsigned BlockValidMaskStriped(int bt, int ipt, int valid) {
  unsigned m = 0;
  if ((int)threadIdx.x >= bt) return 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k)
    if (k < ipt && (int)threadIdx.x + k * bt < valid) m |= 1u << k;
  return m;
}

// Striped BlockLoad: item k of thread t = tile[t + k*bt] for the slots `mask`
// selects (BlockValidMaskStriped; a BlockLoadSel when it is a flag mask).
template <int IPT, class T>
__device__ __forceinline__ void BlockLoadStriped(const T* __restrict__ tile, int bt, unsigned mask,
                                                 T (&items)[IPT]) {
#pragma unroll
  for (int k = 0; k < IPT; ++k)
    if ((mask >> k) & 1u) items[k] = tile[threadIdx.x + k * bt];
}
template <int IPT>
__device__ __forceinline__ void BlockLoadStriped(const int32_t* __restrict__ tile, int bt,
                                                 int valid, int32_t (&items)[IPT]) {
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int s = threadIdx.x + k * bt;
    if (s < valid) items[k] = ld_stream1(tile + s);
  }
}

// Predicated shared store at a 32-bit shared address: one @p STS (the C++
// form `if (bit) wb[p++] = x` compiled to a branch, a reconvergence pair and a
// re-materialised shared base per item -- ~10 instructions per slot).
__device__ __forceinline__ void sts_if(uint32_t addr, int32_t v, uint32_t p) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.b32 [%0], %1;\n\t}" ::"r"(addr), "r"(v),
      "r"(p)
      : "memory");
}

// BlockShuffle (block_ops.hpp:101-122), the per-thread step: this thread's
// flagged items, in item (stride) order, written from s_out[prefix] on --
// with `prefix` from BlockScan of the per-thread counts the tile comes out
// thread-major (the Figure-5 order, e.g. {9,6,8,7,6,9,8,6,7,8}).  Returns the
// thread's count.  The caller barriers before the compacted tile is read.
template <int IPT, class T>
__device__ __forceinline__ int BlockShuffle(const T (&items)[IPT], unsigned flags, int prefix, T* s_out) {
  if constexpr (sizeof(T) == 4) {  // predicated STS, no branch per item
    uint32_t a = (uint32_t)__cvta_generic_to_shared(s_out + prefix);
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const uint32_t m = (flags >> k) & 1u;
      sts_if(a, reinterpret_cast<const int32_t&>(items[k]), m);
      a += 4u * m;
    }
    return __popc(flags & (IPT >= 32 ? 0xffffffffu : ((1u << IPT) - 1u)));
  } else {
    int pos = prefix;
#pragma unroll
    for (int k = 0; k < IPT; ++k)
      if ((flags >> k) & 1u) s_out[pos++] = items[k];
    return pos - prefix;
  }
}

// BlockStore (block_ops.hpp:125-131): the compacted tile s_tile[0, n) to
// dest[0, n), coalesced over the CTA's BT threads.  Bounds are the caller's
// contract (the reference's ContractError is a host-side check).
template <int BT, class T>
__device__ __forceinline__ void BlockStore(const T* s_tile, int n, T* __restrict__ dest) {
  for (int i = threadIdx.x; i < n; i += BT) dest[i] = s_tile[i];
}

// BlockPred / BlockPredAnd (block_ops.hpp:54-69).  Every PredicateSpec op
// (tile.hpp:122-132) is lowered on the host to an inclusive range [lo, hi]
// (lo > hi encodes "never"), so the device evaluates one form.
template <int IPT>
__device__ __forceinline__ unsigned BlockPred(const int32_t (&items)[IPT], int32_t lo, int32_t hi,
                                              unsigned valid_mask) {
  unsigned f = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) f |= (unsigned)(items[k] >= lo && items[k] <= hi) << k;
  return f & valid_mask;
}

template <int IPT>
__device__ __forceinline__ unsigned BlockPredAnd(const int32_t (&items)[IPT], int32_t lo,
                                                 int32_t hi, unsigned flags) {
  unsigned f = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k)
    if ((flags >> k) & 1u) f |= (unsigned)(items[k] >= lo && items[k] <= hi) << k;
  return f;
}

// BlockScan (block_ops.hpp:73-82): exclusive prefix over the CTA's threads in
// thread order, plus the block total.  T is an integer type; `smem` holds
// BT/32 values.  Ends with a barrier so smem can be reused.
template <int BT, class T>
__device__ __forceinline__ T BlockScan(T v, T* smem, T& total) {
  constexpr int W = BT / 32;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  if constexpr (W == 1) {
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
  } else {
    if (lane == 31) smem[warp] = x;
    __syncthreads();
    T w = lane < W ? smem[lane] : T(0);
    if (warp == 0) {
      T s = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= (unsigned)o) s += y;
      }
      if (lane < W) smem[lane] = s - w;  // exclusive warp offsets
      if (lane == W - 1) smem[W] = s;
    }
    __syncthreads();
    T off = smem[warp];
    total = smem[W];
    __syncthreads();
    return off + x - v;
  }
}

// BlockAggregate SUM (block_ops.hpp:141-173): flagged items summed in 8 bytes.
template <int IPT>
__device__ __forceinline__ long long BlockAggregateSum(const int32_t (&items)[IPT], unsigned flags) {
  long long s = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k)
    if ((flags >> k) & 1u) s += items[k];
  return s;
}

// BlockAggregate (block_ops.hpp:133-173): SUM / COUNT / MIN / MAX over the
// items `mask` selects (the valid slots, or the flagged ones), reduced over
// the whole CTA.  Integers accumulate in 8 bytes (AggValue<i32> = i64; 8 x
// INT32_MAX does not wrap); floats in double.  Empty input -> the identity:
// 0 / 0 / numeric_limits<T>::max() / lowest() (+-inf for float).  Every
// thread of the CTA calls it; the result is returned to all of them.
enum BlockAggKind { kBlockSum = 0, kBlockCount = 1, kBlockMin = 2, kBlockMax = 3 };

template <class T>
struct AggTraits;
template <>
struct AggTraits<int32_t> {
  using Acc = long long;
  __device__ static Acc min_identity() { return (Acc)INT32_MAX; }
  __device__ static Acc max_identity() { return (Acc)INT32_MIN; }
};
template <>
struct AggTraits<float> {
  using Acc = double;
  __device__ static Acc min_identity() { return __longlong_as_double(0x7ff0000000000000ll); }
  __device__ static Acc max_identity() { return __longlong_as_double((long long)0xfff0000000000000ull); }
};

template <class Acc>
__device__ __forceinline__ Acc agg_combine(int kind, Acc a, Acc b) {
  return kind == kBlockMin ? (b < a ? b : a) : kind == kBlockMax ? (b > a ? b : a) : a + b;
}

template <int BT, int IPT, class T>
__device__ __forceinline__ typename AggTraits<T>::Acc BlockAggregate(int kind, const T (&items)[IPT], unsigned mask,
                                                                     typename AggTraits<T>::Acc* s_red) {
  using Acc = typename AggTraits<T>::Acc;
  const Acc id = kind == kBlockMin ? AggTraits<T>::min_identity()
                 : kind == kBlockMax ? AggTraits<T>::max_identity() : Acc(0);
  Acc v = id;
#pragma unroll
  for (int k = 0; k < IPT; ++k)
    if ((mask >> k) & 1u) v = agg_combine<Acc>(kind, v, kind == kBlockCount ? Acc(1) : (Acc)items[k]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = agg_combine<Acc>(kind, v, __shfl_xor_sync(0xffffffffu, v, o));
  constexpr int W = BT / 32;
  if constexpr (W > 1) {
    if (lane_id() == 0) s_red[threadIdx.x >> 5] = v;
    __syncthreads();
    v = id;
#pragma unroll
    for (int w = 0; w < W; ++w) v = agg_combine<Acc>(kind, v, s_red[w]);
    __syncthreads();  // s_red reuse
  }
  return v;
}

// BlockProbeHashTable = block_lookup (hash_table.hpp:68-87) over interleaved
// {key,payload} slots.  `flags` is both the probe mask (in) and the found
// bitmap (out); payloads[k] is set for hits.  All first-slot loads are issued
// before any is consumed (IPT independent requests in flight per thread);
// collisions then walk linearly per item (hash_table.hpp:41-51).
template <int IPT>
__device__ __forceinline__ void BlockProbeHashTable(const int32_t (&keys)[IPT], unsigned& flags,
                                                    int32_t (&payloads)[IPT],
                                                    const int2* __restrict__ slots, uint32_t mask,
                                                    int shift) {
  int2 e[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k)
    if ((flags >> k) & 1u) e[k] = __ldg(slots + ht_slot_of(keys[k], shift));
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    if ((flags >> k) & 1u) {
      const int32_t key = keys[k];
      int2 x = e[k];
      uint32_t sl = ht_slot_of(key, shift);
      while (x.x != key && x.x != kEmptyKey) {
        sl = (sl + 1) & mask;
        x = __ldg(slots + sl);
      }
      // INT32_MIN is unstorable and aliases empty slots: always a miss.
      if (x.x == key && key != kEmptyKey)
        payloads[k] = x.y;
      else
        flags &= ~(1u << k);
    }
  }
}

// Same probe against a table staged in shared memory.
template <int IPT>
__device__ __forceinline__ void BlockProbeHashTableSmem(const int32_t (&keys)[IPT],
                                                        unsigned& flags, int32_t (&payloads)[IPT],
                                                        const int2* slots, uint32_t mask,
                                                        int shift) {
  uint32_t s[IPT];
  int2 e[IPT];
  unsigned pending = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    if (((flags >> k) & 1u) && keys[k] != kEmptyKey) {
      pending |= 1u << k;
      s[k] = ht_slot_of(keys[k], shift);
      e[k] = slots[s[k]];
    }
  }
  flags = 0;
  while (pending) {
    unsigned next = 0;
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      if ((pending >> k) & 1u) {
        if (e[k].x == keys[k]) {
          payloads[k] = e[k].y;
          flags |= 1u << k;
        } else if (e[k].x != kEmptyKey) {
          next |= 1u << k;
        }
      }
    }
    pending = next;
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      if ((pending >> k) & 1u) {
        s[k] = (s[k] + 1) & mask;
        e[k] = slots[s[k]];
      }
    }
  }
}

// BlockBuildHashTable (hash_table.cpp:51-93, the CAS-parallel build): claim a
// slot with ONE 64-bit compare-and-swap of {EMPTY,0} -> {key,payload}, so key
// and payload publish together.  err: 1 = sentinel key, 2 = duplicate key.
__device__ __forceinline__ void ht_insert(int2* slots, uint32_t mask, int shift, int32_t key,
                                          int32_t payload, int32_t* err) {
  if (key == kEmptyKey) {
    atomicCAS(err, 0, 1);
    return;
  }
  const unsigned long long empty = pack_slot(kEmptyKey, 0);
  const unsigned long long want = pack_slot(key, payload);
  uint32_t s = ht_slot_of(key, shift);
  for (uint32_t step = 0; step <= mask; ++step, s = (s + 1) & mask) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(slots + s);
    unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(p);
    if ((int32_t)(uint32_t)old == key) {
      atomicCAS(err, 0, 2);
      return;
    }
    if ((int32_t)(uint32_t)old != kEmptyKey) continue;
    old = atomicCAS(p, empty, want);
    if (old == empty) return;
    if ((int32_t)(uint32_t)old == key) {
      atomicCAS(err, 0, 2);
      return;
    }
  }
}

template <int IPT>
__device__ __forceinline__ void BlockBuildHashTable(const int32_t (&keys)[IPT],
                                                    const int32_t (&payloads)[IPT], unsigned flags,
                                                    int2* slots, uint32_t mask, int shift,
                                                    int32_t* err) {
#pragma unroll
  for (int k = 0; k < IPT; ++k)
    if ((flags >> k) & 1u) ht_insert(slots, mask, shift, keys[k], payloads[k], err);
}

// ----------------------------------------------------------------------
// Decoupled look-back (single-pass chained scan) -- the B200 replacement for
// GlobalCursor in deterministic mode (kernel.cpp:22-40): block-ordered output
// offsets without a host-side sequencer.  One 64-bit status word per tile:
// bits 63:62 = 0 invalid / 1 aggregate / 2 inclusive prefix, bits 61:0 value.
// Called by warp 0 of the CTA; returns the tile's exclusive offset.
__device__ __forceinline__ long long tile_lookback(unsigned long long* status, long long tile,
                                                   long long aggregate) {
  const unsigned lane = lane_id();
  constexpr unsigned long long kAgg = 1ull << 62, kPre = 2ull << 62, kVal = (1ull << 62) - 1;
  volatile unsigned long long* st = status;
  if (tile == 0) {
    if (lane == 0) st[0] = kPre | (unsigned long long)aggregate;
    return 0;
  }
  if (lane == 0) st[tile] = kAgg | (unsigned long long)aggregate;
  long long excl = 0;
  long long look = tile - 1;
  while (true) {
    const long long idx = look - (long long)lane;
    unsigned long long w = kPre;  // lanes before tile 0 act as an empty prefix
    if (idx >= 0) {
      unsigned ns = 32;
      while (((w = st[idx]) >> 62) == 0) {
        __nanosleep(ns);
        ns = min(ns * 2, 512u);
      }
    } else {
      w = kPre;
    }
    const unsigned pre = __ballot_sync(0xffffffffu, (w >> 62) == 2);
    const long long val = (long long)(w & kVal);
    if (pre) {
      const int first = __ffs(pre) - 1;  // closest predecessor with a prefix
      long long v = (int)lane <= first ? val : 0;
      excl += warp_sum(v);
      break;
    }
    excl += warp_sum(val);
    look -= 32;
  }
  if (lane == 0) st[tile] = kPre | (unsigned long long)(excl + aggregate);
  return excl;
}

// Publish a tile's aggregate (tile 0: its inclusive prefix) ahead of its
// look-back; pair with block_lookback(..., published = true).
__device__ __forceinline__ void lookback_publish(unsigned long long* status, long long tile,
                                                 long long aggregate) {
  volatile unsigned long long* st = status;
  st[tile] = (tile == 0 ? (2ull << 62) : (1ull << 62)) | (unsigned long long)aggregate;
}

// Block-wide decoupled look-back: the whole CTA reads a window of BT
// predecessors per round trip (instead of a warp's 32), so a tile whose
// nearest inclusive predecessor is a few hundred tiles back -- the normal
// case with ~1000 tiles in flight on 148 SMs -- resolves in one or two L2
// round trips.  Same status-word format as tile_lookback.  Every thread of
// the CTA must call it; returns the tile's exclusive offset to all threads.
template <int BT>
__device__ __forceinline__ long long block_lookback(unsigned long long* status, long long tile,
                                                    long long aggregate, long long* s_red,
                                                    bool published = false) {
  constexpr int W = BT / 32;
  constexpr unsigned long long kAgg = 1ull << 62, kPre = 2ull << 62, kVal = (1ull << 62) - 1;
  volatile unsigned long long* st = status;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  int* s_first = reinterpret_cast<int*>(s_red + W);  // [W]
  if (tile == 0) {
    if (threadIdx.x == 0) st[0] = kPre | (unsigned long long)aggregate;
    return 0;
  }
  if (!published && threadIdx.x == 0) st[tile] = kAgg | (unsigned long long)aggregate;
  long long excl = 0;
  long long look = tile - 1;
  while (true) {
    const long long idx = look - (long long)threadIdx.x;
    unsigned long long w = kPre;  // before tile 0: an empty inclusive prefix
    if (idx >= 0) {
      // exponential back-off: ~1000 CTAs polling the same few status lines
      // otherwise saturate the L2 slice that must also absorb the publishes
      unsigned ns = 32;
      while (((w = st[idx]) >> 62) == 0) {
        __nanosleep(ns);
        ns = min(ns * 2, 512u);
      }
    }
    const unsigned pre = __ballot_sync(0xffffffffu, (w >> 62) == 2);
    if (lane == 0) s_first[warp] = pre ? (int)(warp * 32 + __ffs(pre) - 1) : BT;
    __syncthreads();
    int first = BT;
#pragma unroll
    for (int i = 0; i < W; ++i) first = min(first, s_first[i]);
    long long v = (int)threadIdx.x <= first ? (long long)(w & kVal) : 0;
    v = warp_sum(v);
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    long long sum = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) sum += s_red[i];
    excl += sum;
    __syncthreads();  // s_first / s_red reuse
    if (first < BT) break;
    look -= BT;
  }
  if (threadIdx.x == 0) st[tile] = kPre | (unsigned long long)(excl + aggregate);
  return excl;
}

}  // namespace crys
