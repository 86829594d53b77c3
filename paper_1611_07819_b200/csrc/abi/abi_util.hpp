// SPDX-License-Identifier: Apache-2.0
// Exception -> status-code bridge for the C ABI: C++ code throws
// gridmath::Error (like the reference, common.hpp:11-14); the ABI returns 1
// and keeps the message in a thread-local slot read by gm_last_error().
#pragma once

#include <exception>
#include <string>

namespace gridmath::abi {

void setLastError(const std::string& msg);
const char* lastErrorCStr();

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    setLastError(e.what());
  } catch (...) {
    setLastError("unknown error");
  }
  return 1;
}

}  // namespace gridmath::abi
