// C-ABI plumbing: version and thread-local error message.
#include <atomic>
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

static std::atomic<long long> g_launches{0};

void pf_note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" int pf_version(void) { return 1; }

// kernels this library has launched in this process (graph captures count once)
extern "C" int64_t pf_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" int pf_last_error(char* buf, size_t len) {
  if (!buf || len == 0) return -1;
  strncpy(buf, g_err, len - 1);
  buf[len - 1] = 0;
  return 0;
}
