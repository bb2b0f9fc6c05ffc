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

// CUDA IPC for the peer-memory collectives (distributed.PeerSlices / PeerVolume): the
// handle of a device allocation (64 bytes, sent to the other ranks over torch.distributed)
// and its mapping in another process, on the same device or a peer over NVLink/NVSwitch.
// A handle names the whole allocation the pointer lies in (a caching allocator hands out
// pieces of larger allocations), so the pointer's offset from the allocation base travels
// with it (driver cuMemGetAddressRange, reached through the runtime's entry-point query).
typedef int (*pf_cu_range_fn)(unsigned long long*, size_t*, unsigned long long);

extern "C" int pf_ipc_handle(const void* ptr, void* handle_out /* 64 bytes */,
                             int64_t* offset_out) {
  PF_ARG_CHECK(ptr && handle_out && offset_out, "pf_ipc_handle: null pointer");
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  PF_CUDA_CHECK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q),
                "pf_ipc_handle: driver entry point");
  PF_ARG_CHECK(fn && q == cudaDriverEntryPointSuccess, "pf_ipc_handle: no cuMemGetAddressRange");
  unsigned long long base = 0;
  size_t size = 0;
  PF_ARG_CHECK(((pf_cu_range_fn)fn)(&base, &size, (unsigned long long)(uintptr_t)ptr) == 0,
               "pf_ipc_handle: cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  PF_CUDA_CHECK(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base), "pf_ipc_handle");
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)((uintptr_t)ptr - (uintptr_t)base);
  return 0;
}

extern "C" int pf_ipc_open(const void* handle, int64_t offset, void** ptr_out) {
  PF_ARG_CHECK(handle && ptr_out && offset >= 0, "pf_ipc_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  PF_CUDA_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "pf_ipc_open");
  *ptr_out = (char*)base + offset;
  return 0;
}

extern "C" int pf_ipc_close(void* base) {
  PF_CUDA_CHECK(cudaIpcCloseMemHandle(base), "pf_ipc_close");
  return 0;
}

extern "C" int pf_last_error(char* buf, size_t len) {
  if (!buf || len == 0) return -1;
  strncpy(buf, g_err, len - 1);
  buf[len - 1] = 0;
  return 0;
}
