// join_b200.cpp -- B200 drop-in for P:src/join.cpp.
//
// All three probe variants return the reference's checksum (sum over hits of
// build payload + probe payload, join.hpp:3-10) from join_probe_kernel: probe
// keys/payloads are staged to HBM, the (host) HashTable's slot arrays are
// uploaded as an interleaved {key,payload} table, and the probe runs with the
// table in shared memory when it fits, else L2/HBM resident.
#include "tq/b200_runtime.hpp"
#include "tq/join.hpp"

namespace tq {

namespace {

i64 probe_on_gpu(std::span<const i32> keys, std::span<const i32> payloads, const HashTable& table,
                 const TileConfig& config) {
  if (keys.empty()) return 0;
  crys_ht* ht = nullptr;
  b200::check(crys_ht_upload(b200::context(), table.slot_keys(), table.slot_payloads(),
                             table.capacity(), &ht));
  int64_t sum = 0;
  crys_status s;
  {
    b200::DeviceArray<i32> dk(keys), dp(payloads);
    s = crys_join_probe_sum(b200::context(), dk.data(), dp.data(), static_cast<int64_t>(keys.size()), ht,
                            config.block_threads, config.items_per_thread, &sum);
  }
  crys_ht_free(ht);
  b200::check(s);
  return sum;
}

}  // namespace

i64 join_probe_scalar(std::span<const i32> probe_keys, std::span<const i32> probe_payloads,
                      const HashTable& table, int workers) {
  TQ_CONFIG_CHECK(probe_keys.size() == probe_payloads.size(), "join probe: key/payload length mismatch");
  TQ_CONFIG_CHECK(workers >= 1, "join probe: workers must be >= 1");
  return probe_on_gpu(probe_keys, probe_payloads, table, TileConfig{});
}

i64 join_probe_prefetch(std::span<const i32> probe_keys, std::span<const i32> probe_payloads,
                        const HashTable& table, int workers, int distance) {
  TQ_CONFIG_CHECK(distance >= 1, "join probe: prefetch distance must be >= 1");
  return join_probe_scalar(probe_keys, probe_payloads, table, workers);
}

i64 join_probe_tile(std::span<const i32> probe_keys, std::span<const i32> probe_payloads,
                    const HashTable& table, const TileConfig& config, int workers) {
  TQ_CONFIG_CHECK(probe_keys.size() == probe_payloads.size(), "join probe: key/payload length mismatch");
  config.validate();
  TQ_CONFIG_CHECK(workers >= 1, "run_kernel: workers must be >= 1");
  return probe_on_gpu(probe_keys, probe_payloads, table, config);
}

}  // namespace tq
