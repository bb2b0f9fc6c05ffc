// Shared device helpers for libpfgpu (complex arithmetic, phase reduction,
// error plumbing).  sm_100a only; no host fallback exists anywhere.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PF_TWO_PI 6.283185307179586476925286766559
#define PF_INV_TWO_PI 0.15915494309189533576888376337251

// ---------------------------------------------------------------- complex
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ void cacc(float2& acc, float2 a, float2 b) {  // acc += a*b
  acc.x = fmaf(a.x, b.x, fmaf(-a.y, b.y, acc.x));
  acc.y = fmaf(a.x, b.y, fmaf(a.y, b.x, acc.y));
}

// exp(+1j * phase) with the argument reduced in float64 first (SURVEY F5:
// k*r reaches ~10^3 rad, so the reduction must not happen in float32).
__device__ __forceinline__ float2 expi_reduced(double phase) {
  const double q = rint(phase * PF_INV_TWO_PI);
  const float red = (float)fma(-q, PF_TWO_PI, phase);
  float s, c;
  __sincosf(red, &s, &c);
  return make_float2(c, s);
}

// centred index of natural slot j on a length-n axis: [-n/2, n - n/2)
__device__ __forceinline__ int centred(int j, int n) { return j < n - n / 2 ? j : j - n; }
// natural slot of centred index c (any integer) on a length-n axis
__device__ __forceinline__ int natural(long long c, int n) {
  if (c >= -(long long)n && c < 2LL * n) {   // every hot call site: no 64-bit division
    int m = (int)c;
    m += m < 0 ? n : 0;
    m -= m >= n ? n : 0;
    return m;
  }
  long long m = c % n;
  return (int)(m < 0 ? m + n : m);
}

// ---------------------------------------------------------------- errors
// Thread-local last-error message; every extern "C" entry point returns 0 on
// success, <0 for an argument error, >0 for a CUDA error.
void pf_set_error(const char* fmt, ...);

// One-time-per-device guard for cudaFuncSetAttribute (the attribute is per device, so a
// process driving several GPUs must set it on each): `if (attr.first()) {...}`.
struct PfDevOnce {
  unsigned long long done = 0;   // bit d: device d already configured
  bool first() {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long b = 1ull << (d & 63);
    return (__atomic_fetch_or(&done, b, __ATOMIC_ACQ_REL) & b) == 0;
  }
};
// process-wide count of kernel launches (one per PF_LAUNCH_CHECK; pf_launch_count)
void pf_note_launch();

#define PF_LAUNCH_CHECK(what)                                              \
  do {                                                                     \
    pf_note_launch();                                                      \
    cudaError_t e__ = cudaGetLastError();                                  \
    if (e__ != cudaSuccess) {                                              \
      pf_set_error("%s: %s", what, cudaGetErrorString(e__));               \
      return (int)e__;                                                     \
    }                                                                      \
  } while (0)

#define PF_CUDA_CHECK(call, what)                                          \
  do {                                                                     \
    cudaError_t e__ = (call);                                              \
    if (e__ != cudaSuccess) {                                              \
      pf_set_error("%s: %s", what, cudaGetErrorString(e__));               \
      return (int)e__;                                                     \
    }                                                                      \
  } while (0)

#define PF_ARG_CHECK(cond, msg)                                            \
  do {                                                                     \
    if (!(cond)) {                                                         \
      pf_set_error("%s", msg);                                             \
      return -1;                                                           \
    }                                                                      \
  } while (0)

static inline int pf_cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// SM count of the current device (grid sizing), queried once per process
static inline int pf_sm_count() {
  static int n = 0;
  if (n == 0) {
    int d = 0;
    cudaGetDevice(&d);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

// ---------------------------------------------------------------- async copy
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem_src));
}
// 16-byte copy through L2 only (.cg): both addresses 16-byte aligned
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::); }
