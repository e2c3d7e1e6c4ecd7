// b200_runtime.hpp -- the C++ side of the drop-in: how reference-API calls
// reach libcrystal_b200.so through the C ABI (include/crystal_b200.h).
//
// * one crys_ctx per host thread (device from CRYS_DEVICE, default 0);
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

#include "crystal_b200.h"
#include "tq/common.hpp"

namespace tq::b200 {

crys_ctx* context();                 // this thread's context (created on first use)
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
