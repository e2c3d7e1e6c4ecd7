#pragma once

/**
 * B200 drop-in for the reference's select.hpp (P:include/tq/select.hpp): the
 * same names, signatures, argument checks and output orders, executed by the
 * sm_100a kernels of libcrystal_b200.so.  Put dropin/include BEFORE the
 * reference's include directory and this header shadows the CPU version.
 *
 *   select_{branching,predicated,per_element}[_into]  input order (the
 *       reference's workers=1 order, select.hpp:56-105; any worker count is a
 *       permutation of it, so input order is always a valid answer)
 *   select_tile[_into]  Crystal order for the given TileConfig: blocks in
 *       order, each block thread-major over strided items (select.hpp:107-135,
 *       block_ops.hpp:98-122).  kArrivalOrder only promises a permutation, so
 *       it is served by the same deterministic kernel.
 *
 * Spans are host memory (staged to HBM inside the call).  The kernels are
 * int32; other element types are rejected at compile time.
 */

#include <span>
#include <type_traits>
#include <vector>

#include "tq/b200_runtime.hpp"
#include "tq/block_ops.hpp"
#include "tq/kernel.hpp"

namespace tq {

inline constexpr i64 kSelectVectorSize = 1024;

namespace b200 {

template <typename T>
crys_pred lower_pred(const PredicateSpec<T>& p) {
  crys_pred c;
  c.op = static_cast<int32_t>(p.op);  // PredOp order == crys_pred_op order (tile.hpp:92)
  c.lo = p.lo;
  c.hi = p.hi;
  return c;
}

template <typename T>
i64 select_run(std::span<const T> in, const PredicateSpec<T>& pred, std::span<T> out, int order,
               const TileConfig& config) {
  static_assert(std::is_same_v<T, i32>, "the B200 select kernels are int32");
  const i64 n = static_cast<i64>(in.size());
  if (n == 0) return 0;
  DeviceArray<i32> d_in(in);
  DeviceArray<i32> d_out(in.size());
  int64_t count = 0;
  check(crys_select_i32(context(), d_in.data(), n, lower_pred(pred), d_out.data(), &count, order,
                        config.block_threads, config.items_per_thread));
  d_out.download(out, static_cast<size_t>(count));
  return count;
}

}  // namespace b200

template <typename T>
i64 select_branching_into(std::span<const T> in, const PredicateSpec<T>& pred,
                          std::span<T> out, int workers = 1) {
  TQ_CONFIG_CHECK(workers >= 1, "select: workers must be >= 1");
  TQ_CHECK(out.size() >= in.size(), "select: output capacity too small");
  return b200::select_run<T>(in, pred, out, CRYS_ORDER_INPUT, TileConfig{});
}

template <typename T>
i64 select_predicated_into(std::span<const T> in, const PredicateSpec<T>& pred,
                           std::span<T> out, int workers = 1) {
  return select_branching_into<T>(in, pred, out, workers);
}

template <typename T>
i64 select_per_element_into(std::span<const T> in, const PredicateSpec<T>& pred,
                            std::span<T> out, int workers = 1) {
  return select_branching_into<T>(in, pred, out, workers);
}

template <typename T>
i64 select_tile_into(std::span<const T> in, const PredicateSpec<T>& pred,
                     std::span<T> out, const TileConfig& config,
                     ScheduleMode mode = ScheduleMode::kDeterministic, int workers = 1) {
  config.validate();
  TQ_CHECK(out.size() >= in.size(), "select_tile: output capacity too small");
  TQ_CONFIG_CHECK(workers >= 1, "run_kernel: workers must be >= 1");
  (void)mode;
  return b200::select_run<T>(in, pred, out, CRYS_ORDER_CRYSTAL, config);
}

template <typename T>
std::vector<T> select_branching(std::span<const T> in, const PredicateSpec<T>& pred,
                                int workers = 1) {
  std::vector<T> out(in.size());
  out.resize(static_cast<size_t>(select_branching_into(in, pred, std::span<T>(out), workers)));
  return out;
}

template <typename T>
std::vector<T> select_predicated(std::span<const T> in, const PredicateSpec<T>& pred,
                                 int workers = 1) {
  std::vector<T> out(in.size());
  out.resize(static_cast<size_t>(select_predicated_into(in, pred, std::span<T>(out), workers)));
  return out;
}

template <typename T>
std::vector<T> select_per_element(std::span<const T> in, const PredicateSpec<T>& pred,
                                  int workers = 1) {
  std::vector<T> out(in.size());
  out.resize(static_cast<size_t>(select_per_element_into(in, pred, std::span<T>(out), workers)));
  return out;
}

template <typename T>
std::vector<T> select_tile(std::span<const T> in, const PredicateSpec<T>& pred,
                           const TileConfig& config,
                           ScheduleMode mode = ScheduleMode::kDeterministic, int workers = 1) {
  std::vector<T> out(in.size());
  out.resize(static_cast<size_t>(select_tile_into(in, pred, std::span<T>(out), config, mode, workers)));
  return out;
}

}  // namespace tq
