// Shared host-side helpers: status/error plumbing for the C ABI.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/flashoverlap.h"

namespace fo {

// Exception carrying an fo_status; converted to a return code at the ABI.
struct Error : std::runtime_error {
  fo_status status;
  Error(fo_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(fo_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  throw Error(s, buf);
}

void set_last_error(const std::string& msg);

// Run `f` and map exceptions to fo_status (the ABI never throws).
template <class F>
fo_status guard(F&& f) {
  try {
    f();
    return FO_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return FO_ERR_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return FO_ERR_INVALID_ARG;
  }
}

}  // namespace fo
