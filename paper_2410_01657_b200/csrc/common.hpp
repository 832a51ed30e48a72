// Shared host-side plumbing for the hgnn_b200 C-ABI: typed errors that map
// onto the reference's exception hierarchy (error.hpp:8-72) and the
// thread-local last-error string behind hgnn_last_error().
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/hgnn_b200.h"

namespace hgnn_b200 {

constexpr int kEwThreads = 256;  // block size of the element-wise kernels

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

void set_last_error(const std::string& msg);

// Runs f, converting exceptions into status codes.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return HGNN_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return HGNN_ERR_SIZE;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return HGNN_ERR_INTERNAL;
  }
}

}  // namespace hgnn_b200
