// Error convention of the C ABI: every entry point returns an sw_status and records a
// thread-local message retrievable with sw_last_error(). Status codes mirror the reference's
// exception classes (tensor.hpp:37-45, errors.hpp:10-35, autodiff.hpp:15-18).
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../include/shardweave_b200.h"

namespace sw {

struct Error : std::runtime_error {
  sw_status code;
  Error(sw_status c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

[[noreturn]] inline void fail(sw_status c, const std::string& msg) { throw Error(c, msg); }

void set_last_error(const std::string& msg);

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    fail(SW_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

// Runs `fn`, translating exceptions to sw_status + message.
template <typename Fn>
sw_status guarded(Fn&& fn) noexcept {
  try {
    fn();
    return SW_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SW_ERR_INTERNAL;
  } catch (...) {
    set_last_error("unknown exception");
    return SW_ERR_INTERNAL;
  }
}

}  // namespace sw
