// C-ABI plumbing: version and thread-local error message.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "common.cuh"
#include "../../include/pfgpu.h"

static thread_local char g_err[1024] = {0};

void pf_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" int pf_version(void) { return 1; }

extern "C" int pf_last_error(char* buf, size_t len) {
  if (!buf || len == 0) return -1;
  strncpy(buf, g_err, len - 1);
  buf[len - 1] = 0;
  return 0;
}
