// Scaled DFT (chirp-z / Bluestein) lines for SRSD.
//
// Reference: SfftPlan.apply (spectral.py:160-168) called through
// sfft_2d_centered (spectral.py:209-218) once per (frequency, illumination,
// plane) in srsd (reconstruct.py:320):
//     U[k] = chirp[k] * IFFT_Q( FFT_Q(pad_Q(u * chirp)) * Khat )[k],  k < M
// with chirp[n] = exp(-1j pi alpha (n-o)^2 / M) and Khat the Q-point FFT of the
// embedded kernel exp(+1j pi alpha l^2 / M) -- both built in float64 on the
// host per (M, alpha, o) (phases reach ~400 rad).  One CTA stages
// `cnt` lines of one plane in shared memory: chirp-multiply on load, Q-point
// Stockham FFT, spectrum product, inverse FFT, chirp-multiply and 1/Q on store.
//
// Line addressing (per plane b = blockIdx.y, line l):
//   input element i (i < n_in) at src + b*src_ps + l*src_ls + i*src_es sits at
//   line slot o_in + i (all other slots are zero: the zero-padded relay);
//   output slot k (k < M) goes to dst + b*dst_ps + l*dst_ls + pos(k)*dst_es with
//   pos(k) = k (slot order) or natural(k - M/2) (centred -> natural FFT order).
#include "fft.cuh"

namespace {

constexpr int BT = 256;

__global__ void __launch_bounds__(BT)
k_bluestein(const float2* __restrict__ src, long long src_ps, long long src_ls, long long src_es,
            int n_in, int o_in, float2* __restrict__ dst, long long dst_ps, long long dst_ls,
            long long dst_es, int natural_out, int M, int nlines, pf_fft_plan plan_q,
            const float2* __restrict__ chirp, const float2* __restrict__ khat, int cnt) {
  extern __shared__ float2 sm[];
  const int Q = plan_q.n;
  const int ld = pf_ld(Q);
  float2* a = sm;
  float2* b = sm + (size_t)cnt * ld;
  const int pb = blockIdx.y;
  const float2* ch = chirp + (long long)pb * M;
  const float2* kh = khat + (long long)pb * Q;
  const long long l0 = (long long)blockIdx.x * cnt;
  const int nl = (int)min((long long)cnt, nlines - l0);
  const bool rows = src_es == 1;
  for (int e = threadIdx.x; e < nl * Q; e += BT) {
    int c, q;
    if (rows) { c = e / Q; q = e - c * Q; } else { q = e / nl; c = e - q * nl; }
    float2 v = make_float2(0.f, 0.f);
    const int i = q - o_in;
    if (q < M && i >= 0 && i < n_in)
      v = cmul(src[pb * src_ps + (l0 + c) * src_ls + (long long)i * src_es], ch[q]);
    a[c * ld + q] = v;
  }
  __syncthreads();
  float2* f = fft_smem<-1>(a, b, ld, nl, plan_q);
  float2* g = (f == a) ? b : a;
  for (int e = threadIdx.x; e < nl * Q; e += BT) {
    const int c = e / Q, q = e - c * Q;
    f[c * ld + q] = cmul(f[c * ld + q], kh[q]);
  }
  __syncthreads();
  const float2* r = fft_smem<1>(f, g, ld, nl, plan_q);
  const float inv_q = 1.0f / (float)Q;
  const bool rows_out = dst_es == 1;
  for (int e = threadIdx.x; e < nl * M; e += BT) {
    int c, k;
    if (rows_out) { c = e / M; k = e - c * M; } else { k = e / nl; c = e - k * nl; }
    const int pos = natural_out ? natural((long long)k - M / 2, M) : k;
    dst[pb * dst_ps + (l0 + c) * dst_ls + (long long)pos * dst_es] =
        cscale(cmul(r[c * ld + k], ch[k]), inv_q);
  }
}

}  // namespace

extern "C" int pf_bluestein_lines(const void* src, int64_t src_ps, int64_t src_ls, int64_t src_es,
                                  int n_in, int o_in, void* dst, int64_t dst_ps, int64_t dst_ls,
                                  int64_t dst_es, int natural_out, int M, int nlines, int nplanes,
                                  const pf_fft_plan* plan_q, const void* chirp, const void* khat,
                                  void* stream) {
  PF_ARG_CHECK(plan_q && plan_q->n >= 2 * M - 1 && M >= 1 && nlines >= 0 && nplanes >= 1,
               "pf_bluestein_lines: bad args");
  if (nlines == 0) return 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_bluestein, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const size_t per = 2 * (size_t)pf_ld(plan_q->n) * sizeof(float2);
  int cnt = (int)((200 * 1024) / per);
  if (cnt < 1) { pf_set_error("pf_bluestein_lines: Q too large"); return -1; }
  if (cnt > 8) cnt = 8;
  if (cnt > nlines) cnt = nlines;
  dim3 grid(pf_cdiv(nlines, cnt), nplanes);
  k_bluestein<<<grid, BT, cnt * per, (cudaStream_t)stream>>>(
      (const float2*)src, src_ps, src_ls, src_es, n_in, o_in, (float2*)dst, dst_ps, dst_ls, dst_es,
      natural_out, M, nlines, *plan_q, (const float2*)chirp, (const float2*)khat, cnt);
  PF_LAUNCH_CHECK("k_bluestein");
  return 0;
}
