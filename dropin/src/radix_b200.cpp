// radix_b200.cpp -- B200 drop-in for P:src/radix.cpp.
//
//   radix_histogram  owner x digit counts on the GPU (owner = contiguous chunk)
//   radix_offsets    the column-major exclusive prefix (host: owners x 2^bits)
//   radix_shuffle    a stable partition pass on the GPU; for a stable pass it
//                    is exactly what per-owner cursors produce, for an
//                    unstable one it is one valid arrival order
//   lsb/msb_radix_sort  the device sorts (LSB == std::stable_sort by key; MSB
//                    keys ascending with pairs preserved)
#include <algorithm>
#include <vector>

#include "tq/b200_runtime.hpp"
#include "tq/radix.hpp"

namespace tq {

RadixHistogram radix_histogram(std::span<const i32> keys, const RadixPass& pass, i64 num_owners,
                               int workers) {
  pass.validate();
  TQ_CONFIG_CHECK(num_owners >= 1, "radix_histogram: need at least one owner");
  (void)workers;
  RadixHistogram hist;
  hist.num_owners = num_owners;
  hist.num_digits = pass.num_digits();
  const i64 n = static_cast<i64>(keys.size());
  hist.chunk = std::max<i64>(1, (n + num_owners - 1) / num_owners);
  hist.counts.assign(static_cast<size_t>(num_owners) * hist.num_digits, 0);
  b200::DeviceArray<i32> dk(keys.size() ? keys : std::span<const i32>());
  b200::check(crys_radix_histogram(b200::context(), dk.data(), n, pass.start_bit, pass.num_bits,
                                   num_owners, hist.counts.data()));
  return hist;
}

RadixOffsets radix_offsets(const RadixHistogram& hist) {
  RadixOffsets off;
  off.num_owners = hist.num_owners;
  off.num_digits = hist.num_digits;
  off.chunk = hist.chunk;
  off.digit_base.assign(static_cast<size_t>(hist.num_digits), 0);
  off.owner_start.assign(hist.counts.size(), 0);
  i64 run = 0;
  for (int d = 0; d < hist.num_digits; ++d) {  // digit-major, owner within digit
    off.digit_base[static_cast<size_t>(d)] = run;
    for (i64 o = 0; o < hist.num_owners; ++o) {
      off.owner_start[static_cast<size_t>(o) * hist.num_digits + d] = run;
      run += hist.at(o, d);
    }
  }
  off.total = run;
  return off;
}

void radix_shuffle(std::span<const i32> keys, std::span<const i32> payloads, const RadixPass& pass,
                   const RadixOffsets& offsets, std::span<i32> out_keys, std::span<i32> out_payloads,
                   int workers) {
  pass.validate();
  (void)workers;
  const i64 n = static_cast<i64>(keys.size());
  TQ_CHECK(keys.size() == payloads.size(), "radix_shuffle: key/payload length mismatch");
  TQ_CHECK(offsets.total == n, "radix_shuffle: offsets built from different input");
  TQ_CHECK(offsets.num_digits == pass.num_digits(), "radix_shuffle: offsets/pass digit mismatch");
  TQ_CHECK(static_cast<i64>(out_keys.size()) == n && static_cast<i64>(out_payloads.size()) == n,
           "radix_shuffle: output size mismatch");
  if (n == 0) return;
  b200::DeviceArray<i32> dk(keys), dp(payloads), ok(keys.size()), op(keys.size());
  b200::check(crys_radix_partition(b200::context(), dk.data(), dp.data(), n, pass.start_bit, pass.num_bits,
                                   ok.data(), op.data()));
  ok.download(out_keys, keys.size());
  op.download(out_payloads, keys.size());
}

namespace {
void sort_on_gpu(std::span<i32> keys, std::span<i32> payloads, int algo, int bits) {
  b200::DeviceArray<i32> dk(std::span<const i32>(keys.data(), keys.size()));
  b200::DeviceArray<i32> dp(std::span<const i32>(payloads.data(), payloads.size()));
  b200::check(crys_sort_pairs(b200::context(), dk.data(), dp.data(), static_cast<int64_t>(keys.size()),
                              algo, bits));
  dk.download(keys, keys.size());
  dp.download(payloads, payloads.size());
}
}  // namespace

void lsb_radix_sort(std::span<i32> keys, std::span<i32> payloads, int workers, int bits_per_pass) {
  TQ_CONFIG_CHECK(bits_per_pass >= 1 && bits_per_pass <= 8,
                  "lsb_radix_sort: bits_per_pass must be in [1,8]");
  TQ_CHECK(keys.size() == payloads.size(), "lsb_radix_sort: key/payload length mismatch");
  (void)workers;
  if (keys.size() <= 1) return;
  sort_on_gpu(keys, payloads, CRYS_SORT_LSB, bits_per_pass);
}

void msb_radix_sort(std::span<i32> keys, std::span<i32> payloads, int workers) {
  TQ_CHECK(keys.size() == payloads.size(), "msb_radix_sort: key/payload length mismatch");
  (void)workers;
  if (keys.size() <= 1) return;
  sort_on_gpu(keys, payloads, CRYS_SORT_MSB, 8);
}

}  // namespace tq
