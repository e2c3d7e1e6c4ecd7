// b200_runtime.hpp -- the C++ side of the drop-in: how reference-API calls
// reach libcrystal_b200.so through the C ABI (include/crystal_b200.h).
//
// * one crys_ctx per host thread (device from CRYS_DEVICE, default 0), and
//   one device group per (thread, shard count) for run_query's `workers`;
// * crys_status -> the reference's exception taxonomy
//   (P:include/tq/common.hpp:16-34): ECONFIG -> ConfigError, ECONTRACT ->
//   ContractError, EBUILD -> BuildError, EIO -> IoError, CUDA/not-built ->
//   std::runtime_error;
// * DeviceArray<T>: RAII device staging for the reference's host spans.
//
// There is no CPU fallback: a missing library or device throws.
#pragma once

#include <cstddef>
#include <span>
#include <string>
#include <vector>

#include "crystal_b200.h"
#include "tq/common.hpp"

namespace tq::b200 {

crys_ctx* context();                 // this thread's context (created on first use)

// The device group `workers` maps to (ssb_queries.hpp:76-78: run_query's
// `workers`): min(workers, visible GPUs) lineorder shards, one per GPU
// (CRYS_DEVICES="0,1,..." picks the GPUs).  CRYS_GROUP_EMULATE=1 keeps
// `workers` shards even on fewer GPUs, placing them round-robin (several
// shards per GPU are summed on that GPU) -- how the sharded path is tested on
// a one-GPU box.  One group per (host thread, shard count), created on first use.
crys_ctx* group_context(int workers);

// HBM copies of host-resident SsbDatabases, cached by identity: the
// database's address, every column's data pointer and length, and a content
// fingerprint (all bytes up to 64 MB in total, else 4096 sampled 64-byte
// blocks per column).  A cache hit does no H2D copy at all; a changed
// signature re-uploads.  Mutating a LARGE database in place without
// reallocating its columns may escape the sampled fingerprint: call
// invalidate(db) (or invalidate_all()) after such a change.
struct SsbDatabaseCache;
void invalidate(const void* db);
void invalidate_all();
// Uploads performed so far by this thread (telemetry for tests).
long long upload_count();
// The HBM database of `cols` on group `g`, uploaded on a cache miss.
crys_db* cached_database(crys_ctx* g, const void* key, const std::vector<crys_host_column>& cols);
[[noreturn]] void raise(crys_status s);
inline void check(crys_status s) {
  if (s != CRYS_OK) raise(s);
}

template <typename T>
class DeviceArray {
 public:
  explicit DeviceArray(size_t n) : n_(n) {
    void* p = nullptr;
    check(crys_device_alloc(context(), n * sizeof(T), &p));
    p_ = static_cast<T*>(p);
  }
  explicit DeviceArray(std::span<const T> host) : DeviceArray(host.size()) { upload(host); }
  DeviceArray(const DeviceArray&) = delete;
  DeviceArray& operator=(const DeviceArray&) = delete;
  ~DeviceArray() { crys_device_free(context(), p_); }

  void upload(std::span<const T> host) {
    check(crys_copy_to_device(context(), p_, host.data(), host.size() * sizeof(T)));
  }
  void download(std::span<T> host, size_t count) const {
    check(crys_copy_to_host(context(), host.data(), p_, count * sizeof(T)));
  }
  T* data() { return p_; }
  const T* data() const { return p_; }
  size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

}  // namespace tq::b200
