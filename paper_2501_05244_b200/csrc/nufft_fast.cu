// Type-1 NUFFT finish on the register-FFT path: fine-grid FFT + deconvolution for
// 2D plans whose fine grid is exactly twice the modes, mr = 2m, m in {128..1024}
// (on-lattice NURSD1 with a power-of-two pad; config 5: m = 1024, mr = 2048).
//
// Reference spectral.py:356-358 (nufft1): fftn(fine) then the centred modes
// k in [-m/2, m/2) are gathered and divided by ker_y[k_y] * ker_x[k_x].
// Only a quarter of the fine spectrum is kept, so each mr-point transform is
// split once (radix 2, decimation in frequency):
//   X[2j]   = FFT_{mr/2}( x[n] + x[n + mr/2] )[j]
//   X[2j+1] = FFT_{mr/2}( (x[n] - x[n + mr/2]) W_mr^n )[j]
// and both halves run as warp_fft.cuh register transforms (n = mr/2 = 32 L),
// keeping j < mr/8 and j >= 3 mr/8 -- for lane t holding j = t + L q that is
// q < 8 or q >= 24, fixed at compile time.  Pass 1 transforms every fine row
// and writes only the m kept columns, transposed (RT[c_x][y], contiguous y);
// pass 2 transforms only those m columns, deconvolves and writes the modes
// transposed, out[c_x][c_y] (what the register propagation consumes).
#include "warp_fft.cuh"

namespace {

constexpr int NFT = 256;   // 8 warps

__host__ __device__ constexpr bool kept_q(int q) { return q < 8 || q >= 24; }

// natural slot on the m-grid (m = 32 L) of fine-spectrum index k = 2j + odd,
// j = t + L q with q kept: k < m/2 -> k;  k >= 3m/2 -> k - m
template <int L>
__device__ __forceinline__ int mode_slot(int t, int q, int odd) {
  const int k = 2 * (t + L * q) + odd;
  return q < 8 ? k : k - 32 * L;
}

// pass 1: lines = fine rows y (length mr = 64 L), output RT[v][c_x][y]
template <int L>
__global__ void __launch_bounds__(NFT, 2)
k_t1_rows(const float2* __restrict__ fine, long long fine_stride, const float2* __restrict__ w_mr,
          const float2* __restrict__ tw_h, float2* __restrict__ rt) {
  constexpr int H = 32 * L, MR = 2 * H, LPW = 32 / L, RPC = 8 * LPW, SLD = RPC + 1;
  extern __shared__ float2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int r = warp * LPW + line;
  const int y0 = blockIdx.x * RPC;
  const int v = blockIdx.y;
  const float2* row = fine + v * fine_stride + (long long)(y0 + r) * MR + t;
  float2* xch = sm + warp * WFFT_XCH;
  float2 a[32], ke[16];
#pragma unroll
  for (int q = 0; q < 32; q++) a[q] = cadd(__ldg(row + L * q), __ldg(row + L * q + H));
  wfft<L, -1>(a, xch, tw_h);
#pragma unroll
  for (int q = 0, e = 0; q < 32; q++)
    if (kept_q(q)) ke[e++] = a[q];
#pragma unroll
  for (int q = 0; q < 32; q++) {
    const float2 d = csub(__ldg(row + L * q), __ldg(row + L * q + H));
    a[q] = cmul(d, __ldg(w_mr + t + L * q));
  }
  wfft<L, -1>(a, xch, tw_h);
  __syncthreads();   // the tile aliases the exchange buffers
#pragma unroll
  for (int q = 0, e = 0; q < 32; q++) {
    if (kept_q(q)) {
      sm[mode_slot<L>(t, q, 0) * SLD + r] = ke[e++];
      sm[mode_slot<L>(t, q, 1) * SLD + r] = a[q];
    }
  }
  __syncthreads();
  constexpr int KSTEP = NFT / RPC;
  const int rr = threadIdx.x % RPC, c0 = threadIdx.x / RPC;
  float2* d = rt + (long long)v * H * MR + (long long)c0 * MR + y0 + rr;
  const float2* s = sm + c0 * SLD + rr;
#pragma unroll 4
  for (int c = c0; c < H; c += KSTEP) {
    *d = *s;
    d += (long long)KSTEP * MR;
    s += KSTEP * SLD;
  }
}

// pass 2: lines = kept columns c_x (length mr), deconvolve, out[v][c_x][c_y]
template <int L>
__global__ void __launch_bounds__(NFT, 2)
k_t1_cols(const float2* __restrict__ rt, const float2* __restrict__ w_mr,
          const float2* __restrict__ tw_h, const float* __restrict__ ker_y,
          const float* __restrict__ ker_x, float2* __restrict__ out, long long out_stride) {
  constexpr int H = 32 * L, MR = 2 * H, LPW = 32 / L;
  extern __shared__ float2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int cx = (blockIdx.x * 8 + warp) * LPW + line;
  const int v = blockIdx.y;
  const float2* col = rt + (long long)v * H * MR + (long long)cx * MR + t;
  float2* dst = out + v * out_stride + (long long)cx * H;
  float2* xch = sm + warp * WFFT_XCH;
  const float kx = ker_x[centred(cx, H) + H / 2];
  float2 a[32];
#pragma unroll
  for (int q = 0; q < 32; q++) a[q] = cadd(__ldg(col + L * q), __ldg(col + L * q + H));
  wfft<L, -1>(a, xch, tw_h);
#pragma unroll
  for (int q = 0; q < 32; q++) {
    if (kept_q(q)) {
      const int cy = mode_slot<L>(t, q, 0);
      const float den = ker_y[centred(cy, H) + H / 2] * kx;
      dst[cy] = make_float2(a[q].x / den, a[q].y / den);
    }
  }
#pragma unroll
  for (int q = 0; q < 32; q++) {
    const float2 d = csub(__ldg(col + L * q), __ldg(col + L * q + H));
    a[q] = cmul(d, __ldg(w_mr + t + L * q));
  }
  wfft<L, -1>(a, xch, tw_h);
#pragma unroll
  for (int q = 0; q < 32; q++) {
    if (kept_q(q)) {
      const int cy = mode_slot<L>(t, q, 1);
      const float den = ker_y[centred(cy, H) + H / 2] * kx;
      dst[cy] = make_float2(a[q].x / den, a[q].y / den);
    }
  }
}

template <int L>
int run_t1(const float2* fine, long long fine_stride, int nv, float2* rt, const float2* w_mr,
           const float2* tw_h, const float* ky, const float* kx, float2* out, long long out_stride,
           cudaStream_t st) {
  constexpr int H = 32 * L, MR = 2 * H, LPW = 32 / L, RPC = 8 * LPW;
  const size_t sm_r = (size_t)(8 * WFFT_XCH > H * (RPC + 1) ? 8 * WFFT_XCH : H * (RPC + 1)) *
                      sizeof(float2);
  const size_t sm_c = 8 * WFFT_XCH * sizeof(float2);
  static PfDevOnce attr;  
  if (attr.first()) {
    cudaFuncSetAttribute(k_t1_rows<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_t1_cols<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  for (int v0 = 0; v0 < nv; v0 += 65535) {
    const int n = nv - v0 < 65535 ? nv - v0 : 65535;
    k_t1_rows<L><<<dim3(MR / RPC, n), NFT, sm_r, st>>>(fine + v0 * fine_stride, fine_stride, w_mr,
                                                      tw_h, rt + (long long)v0 * H * MR);
    PF_LAUNCH_CHECK("k_t1_rows");
    k_t1_cols<L><<<dim3(H / (8 * LPW), n), NFT, sm_c, st>>>(rt + (long long)v0 * H * MR, w_mr, tw_h,
                                                           ky, kx, out + v0 * out_stride,
                                                           out_stride);
    PF_LAUNCH_CHECK("k_t1_cols");
  }
  return 0;
}

}  // namespace

extern "C" int pf_nufft_type1_finish_pow2(const pf_nufft_geom* g, const void* fine,
                                          int64_t fine_stride, int nv, void* rt,
                                          const pf_fft_plan* plan_mr, const pf_fft_plan* plan_h,
                                          const float* ky, const float* kx, void* out,
                                          int64_t out_stride, void* stream) {
  PF_ARG_CHECK(g && g->dim == 2 && nv >= 1, "pf_nufft_type1_finish_pow2: 2D plans only");
  const int m = g->m[2];
  PF_ARG_CHECK(g->m[1] == m && g->mr[1] == 2 * m && g->mr[2] == 2 * m,
               "pf_nufft_type1_finish_pow2: needs square modes with mr = 2 m");
  PF_ARG_CHECK(plan_mr && plan_h && plan_mr->n == 2 * m && plan_h->n == m,
               "pf_nufft_type1_finish_pow2: plan lengths must be 2m and m");
  const float2* w_mr = (const float2*)plan_mr->tw;   // unit roots W_mr^n first
  const float2* tw_h = (const float2*)plan_h->tw;
  cudaStream_t st = (cudaStream_t)stream;
#define PF_T1_CASE(MM, LL)                                                                    \
  case MM:                                                                                   \
    return run_t1<LL>((const float2*)fine, fine_stride, nv, (float2*)rt, w_mr, tw_h, ky, kx, \
                      (float2*)out, out_stride, st);
  switch (m) {
    PF_T1_CASE(128, 4)
    PF_T1_CASE(256, 8)
    PF_T1_CASE(512, 16)
    PF_T1_CASE(1024, 32)
    default: break;
  }
#undef PF_T1_CASE
  pf_set_error("pf_nufft_type1_finish_pow2: modes must be 128, 256, 512 or 1024");
  return -1;
}
