// Shared host-side helpers: status plumbing and the thread-local error message.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/dflow.h"

namespace dflow {

void set_error(const char* fmt, ...);
void clear_error();

// Status-carrying error for internal C++ code; converted at the ABI boundary.
struct Error {
  dflow_status code;
  std::string msg;
};

inline dflow_status fail(dflow_status code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  set_error("%s", buf);
  return code;
}

}  // namespace dflow
