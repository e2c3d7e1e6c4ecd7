// hash_table_b200.cpp -- B200 drop-in for P:src/hash_table.cpp.
//
// HashTable::build runs the CAS-parallel build kernel (BlockBuildHashTable,
// 64-bit compare-and-swap of {key,payload}) on the GPU and returns the
// reference's host-resident value type, its slot arrays downloaded from HBM.
// Argument checks and errors are the reference's (hash_table.cpp:20-30).
#include <vector>

#include "tq/b200_runtime.hpp"
#include "tq/hash_table.hpp"

namespace tq {

HashTable HashTable::build(std::span<const i32> keys, std::span<const i32> payloads, i64 capacity,
                           int workers) {
  TQ_CONFIG_CHECK(keys.size() == payloads.size(), "HashTable: key/payload length mismatch");
  TQ_CONFIG_CHECK(capacity >= 2 && (capacity & (capacity - 1)) == 0,
                  "HashTable: capacity must be a power of two >= 2");
  if (static_cast<i64>(keys.size()) * 2 > capacity)
    throw BuildError("HashTable: capacity overflow (fill would exceed 50%)");
  (void)workers;  // the GPU build is always the parallel one (probe-equivalent)
  int lg = 0;
  while ((i64{1} << lg) < capacity) ++lg;
  HashTable table(capacity, 32 - lg);
  crys_ht* ht = nullptr;
  {
    b200::DeviceArray<i32> dk(keys.size() ? keys : std::span<const i32>());
    b200::DeviceArray<i32> dp(payloads.size() ? payloads : std::span<const i32>());
    b200::check(crys_ht_build(b200::context(), dk.data(), dp.data(), static_cast<int64_t>(keys.size()),
                              capacity, &ht));
  }
  const crys_status s = crys_ht_download(ht, table.keys_.data(), table.payloads_.data());
  crys_ht_free(ht);
  b200::check(s);
  table.size_ = static_cast<i64>(keys.size());
  return table;
}

}  // namespace tq
