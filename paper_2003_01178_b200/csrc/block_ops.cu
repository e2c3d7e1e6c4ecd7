// block_ops.cu -- the Crystal device primitives run one logical tile per CTA
// (the paper's Table-1 pipeline, restated by the reference's
// block_ops.hpp:23-173 for a CPU "block"):
//
//   BlockLoadStriped -> BlockPred -> thread counts -> BlockScan
//     -> BlockShuffle -> BlockStore,  + BlockAggregate SUM/COUNT/MIN/MAX
//
// crys_block_ops_run exposes every intermediate (per-logical-thread counts and
// exclusive prefixes, the compacted tile, the tile totals and aggregates) so
// tests can hold each primitive to block_ops semantics on the Figure-5 tile
// (test_tile_engine.cpp:18-22, :57-79) and on random partial tiles.  The
// production kernels (select, SSB) use the same primitives.
#include <algorithm>

#include "crystal.cuh"
#include "internal.hpp"

namespace crys {
namespace {

constexpr int kBlockOpsMaxIpt = 16;

template <int PB>
__global__ void __launch_bounds__(PB) block_ops_kernel(const int32_t* __restrict__ in, int64_t n, int bt,
                                                       int ipt, int32_t lo, int32_t hi, int32_t* out,
                                                       long long* counts, long long* prefix,
                                                       long long* totals, long long* aggs) {
  extern __shared__ int32_t s_tile[];  // the compacted tile, bt * ipt slots
  __shared__ long long s_scan[PB / 32 + 1];
  __shared__ long long s_red[PB / 32];
  const int S = bt * ipt;
  const int64_t base = (int64_t)blockIdx.x * S;
  const int valid = (int)min((int64_t)S, n - base);
  const int t = threadIdx.x;

  // BlockLoad (block_ops.hpp:23-32): striped ownership t + k*bt
  int32_t items[kBlockOpsMaxIpt];
  const unsigned vmask = BlockValidMaskStriped<kBlockOpsMaxIpt>(bt, ipt, valid);
  BlockLoadStriped<kBlockOpsMaxIpt, int32_t>(in + base, bt, vmask, items);
  // BlockPred (block_ops.hpp:54-69): flags past valid_count stay false
  const unsigned flags = BlockPred<kBlockOpsMaxIpt>(items, lo, hi, vmask);
  // block_thread_counts + block_scan (block_ops.hpp:73-96)
  const long long cnt = __popc(flags);
  long long total;
  const long long pre = BlockScan<PB>(cnt, s_scan, total);
  // BlockShuffle (block_ops.hpp:101-122) into shared memory, BlockStore (:125-131)
  BlockShuffle<kBlockOpsMaxIpt, int32_t>(items, flags, (int)pre, s_tile);
  __syncthreads();
  BlockStore<PB, int32_t>(s_tile, (int)total, out + base);
  // BlockAggregate (block_ops.hpp:141-173): over the flagged slots, then over
  // every valid slot
  long long a[8];
#pragma unroll
  for (int kind = 0; kind < 4; ++kind) {
    a[kind] = BlockAggregate<PB, kBlockOpsMaxIpt, int32_t>(kind, items, flags, s_red);
    a[4 + kind] = BlockAggregate<PB, kBlockOpsMaxIpt, int32_t>(kind, items, vmask, s_red);
  }
  if (t < bt) {
    counts[(int64_t)blockIdx.x * bt + t] = cnt;
    prefix[(int64_t)blockIdx.x * bt + t] = pre;
  }
  if (t == 0) {
    totals[blockIdx.x] = total;
    for (int k = 0; k < 8; ++k) aggs[(int64_t)blockIdx.x * 8 + k] = a[k];
  }
}

template <int PB>
void launch_block_ops(crys_ctx* ctx, int64_t tiles, const int32_t* in, int64_t n, int bt, int ipt, int32_t lo,
                      int32_t hi, int32_t* out, long long* counts, long long* prefix, long long* totals,
                      long long* aggs) {
  const size_t smem = sizeof(int32_t) * (size_t)bt * (size_t)ipt;
  ensure_dyn_smem((const void*)block_ops_kernel<PB>, smem);
  block_ops_kernel<PB><<<(unsigned)tiles, PB, smem, ctx->stream>>>(in, n, bt, ipt, lo, hi, out, counts, prefix,
                                                                   totals, aggs);
  CRYS_LAUNCHED("block_ops_kernel");
  count_launch(ctx);
}

}  // namespace

void block_ops_run(crys_ctx* ctx, const int32_t* in, int64_t n, int bt, int ipt, int32_t lo, int32_t hi,
                   int32_t* out, int64_t* counts, int64_t* prefix, int64_t* totals, int64_t* aggs) {
  CRYS_CHECK(bt >= 1 && bt <= 1024 && ipt >= 1 && ipt <= kBlockOpsMaxIpt, CRYS_ENOTBUILT,
             "block primitives: 1 <= block_threads <= 1024 and 1 <= items_per_thread <= 16");
  CRYS_CHECK(n >= 1, CRYS_ECONFIG, "block primitives: empty input");
  const int64_t S = (int64_t)bt * ipt;
  const int64_t tiles = (n + S - 1) / S;
  auto* c = reinterpret_cast<long long*>(counts);
  auto* p = reinterpret_cast<long long*>(prefix);
  auto* t = reinterpret_cast<long long*>(totals);
  auto* a = reinterpret_cast<long long*>(aggs);
  if (bt <= 32) launch_block_ops<32>(ctx, tiles, in, n, bt, ipt, lo, hi, out, c, p, t, a);
  else if (bt <= 64) launch_block_ops<64>(ctx, tiles, in, n, bt, ipt, lo, hi, out, c, p, t, a);
  else if (bt <= 128) launch_block_ops<128>(ctx, tiles, in, n, bt, ipt, lo, hi, out, c, p, t, a);
  else if (bt <= 256) launch_block_ops<256>(ctx, tiles, in, n, bt, ipt, lo, hi, out, c, p, t, a);
  else if (bt <= 512) launch_block_ops<512>(ctx, tiles, in, n, bt, ipt, lo, hi, out, c, p, t, a);
  else launch_block_ops<1024>(ctx, tiles, in, n, bt, ipt, lo, hi, out, c, p, t, a);
}

}  // namespace crys
