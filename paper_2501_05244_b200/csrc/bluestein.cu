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
  static PfDevOnce attr;  
  if (attr.first()) {
    cudaFuncSetAttribute(k_bluestein, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
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

// ---------------------------------------------------------------------------
// Register-FFT Bluestein for power-of-two Q = 32 L (the SRSD configs: M = 512,
// Q = 1024).  One line per L lanes; the Q-point transforms stay in registers
// (warp_fft.cuh).  Two passes of sfft_2d_centered (spectral.py:205-206):
//   X pass: line = relay row iy (contiguous input); output staged through
//           shared memory and stored TRANSPOSED, xT[b][col_nat][iy], so that
//   Y pass: line = column col (contiguous input xT row); output stored as the
//           transposed spectrum Uhat^T[b][col][row_nat] the register
//           propagation path consumes.
#include "warp_fft.cuh"

namespace {

// CW: the SRSD window at compile time (M = Q/2 outputs, n_in = Q/4 inputs at o_in = Q/8:
// the centred N-of-2N relay in a Q = 4N transform), so the zero inputs and the unused
// outputs are constants the compiler folds out of the first and last radix-32 stages.
template <int L, bool XPASS, bool CW = false>
__global__ void __launch_bounds__(256, 2)
k_bluestein_w(const float2* __restrict__ src, long long src_ps, long long src_ls, int n_in_rt,
              int o_in_rt, float2* __restrict__ dst, long long dst_ps, long long dst_ls, int M_rt,
              int nlines, int n_out_lines, const float2* __restrict__ tw,
              const float2* __restrict__ chirp, const float2* __restrict__ khat) {
  constexpr int Q = 32 * L, LPW = 32 / L, LPC = 8 * LPW;
  const int M = CW ? Q / 2 : M_rt, n_in = CW ? Q / 4 : n_in_rt, o_in = CW ? Q / 8 : o_in_rt;
  extern __shared__ float2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int r = warp * LPW + line;
  const int b = blockIdx.y;
  const int l0 = blockIdx.x * LPC;
  const int l = l0 + r;
  const bool active = l < nlines;
  const float2* ch = chirp + (long long)b * M;
  const float2* kh = khat + (long long)b * Q;
  const float2* s = src + b * src_ps + (long long)(active ? l : 0) * src_ls;
  float2 v[32];
  // input window and output length on lane-multiple boundaries (the SRSD pads):
  // element m is inside or outside for the whole warp
  const bool aligned = ((o_in | n_in | M) & (L - 1)) == 0;
  if (aligned) {
    const float2* st = s + t - o_in;
    const float2* ct = ch + t;
#pragma unroll
    for (int m = 0; m < 32; m++) {
      const int base = L * m;
      v[m] = (base < M && base >= o_in && base < o_in + n_in)
                 ? cmul(__ldg(st + base), __ldg(ct + base)) : make_float2(0.f, 0.f);
    }
  } else {
#pragma unroll
    for (int m = 0; m < 32; m++) {
      const int q = t + L * m;
      const int i = q - o_in;
      float2 x = make_float2(0.f, 0.f);
      if (q < M && i >= 0 && i < n_in) x = cmul(__ldg(s + i), __ldg(ch + q));
      v[m] = x;
    }
  }
  float2* xch = sm + warp * WFFT_XCH;
  // CW: inputs only at q in [o_in, o_in + n_in) = [4L, 12L): m in [4, 12) for every lane
  wfft<L, -1, false, CW>(v, xch, tw);
#pragma unroll
  for (int m = 0; m < 32; m++) v[m] = cmul(v[m], __ldg(kh + t + L * m));
  wfft<L, 1>(v, xch, tw);
  const float inv_q = 1.0f / (float)Q;
  if (XPASS) {
    // stage [M][LPC] then write xT[b][col_nat][l0 .. l0+LPC)
    constexpr int SLD = LPC + 1;
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 32; m++) {
      const int k = t + L * m;
      if (k < M) sm[k * SLD + r] = cscale(cmul(v[m], __ldg(ch + k)), inv_q);
    }
    __syncthreads();
    const int nl = min(LPC, nlines - l0);
    float2* d = dst + b * dst_ps + l0;
    const bool pow2 = (M & (M - 1)) == 0;   // natural(k - M/2) = k ^ M/2
    for (int e = threadIdx.x; e < M * LPC; e += 256) {
      const int k = e / LPC, rr = e % LPC;
      const int kn = pow2 ? (k ^ (M >> 1)) : natural((long long)k - M / 2, M);
      if (rr < nl) d[(long long)kn * dst_ls + rr] = sm[k * SLD + rr];
    }
  } else if (active) {
    float2* d = dst + b * dst_ps + (long long)l * dst_ls;
    if (aligned && (M & (M - 1)) == 0) {
      // k = t + L m < M: natural(k - M/2) = k ^ M/2 = t + (L m ^ M/2)
      float2* dt = d + t;
      const float2* ct = ch + t;
#pragma unroll
      for (int m = 0; m < 32; m++) {
        const int base = L * m;
        if (base < M) dt[base ^ (M >> 1)] = cscale(cmul(v[m], __ldg(ct + base)), inv_q);
      }
    } else {
#pragma unroll
      for (int m = 0; m < 32; m++) {
        const int k = t + L * m;
        if (k < M) d[natural((long long)k - M / 2, M)] = cscale(cmul(v[m], __ldg(ch + k)), inv_q);
      }
    }
  }
}

template <int L>
int launch_bw(int xpass, const float2* src, long long src_ps, long long src_ls, int n_in, int o_in,
              float2* dst, long long dst_ps, long long dst_ls, int M, int nlines, int nplanes,
              const float2* tw, const float2* chirp, const float2* khat, cudaStream_t st) {
  constexpr int LPC = 8 * (32 / L), Q = 32 * L;
  static PfDevOnce attr;  
  if (attr.first()) {
    cudaFuncSetAttribute(k_bluestein_w<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_bluestein_w<L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_bluestein_w<L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_bluestein_w<L, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  size_t sm = 8 * WFFT_XCH;
  if (xpass && (size_t)M * (LPC + 1) > sm) sm = (size_t)M * (LPC + 1);
  sm *= sizeof(float2);
  dim3 grid(pf_cdiv(nlines, LPC), nplanes);
  const bool cw = 2 * M == Q && 4 * n_in == Q && 8 * o_in == Q;
  if (xpass && cw)
    k_bluestein_w<L, true, true><<<grid, 256, sm, st>>>(src, src_ps, src_ls, n_in, o_in, dst,
                                                        dst_ps, dst_ls, M, nlines, 0, tw, chirp,
                                                        khat);
  else if (xpass)
    k_bluestein_w<L, true><<<grid, 256, sm, st>>>(src, src_ps, src_ls, n_in, o_in, dst, dst_ps,
                                                  dst_ls, M, nlines, 0, tw, chirp, khat);
  else if (cw)
    k_bluestein_w<L, false, true><<<grid, 256, sm, st>>>(src, src_ps, src_ls, n_in, o_in, dst,
                                                         dst_ps, dst_ls, M, nlines, 0, tw, chirp,
                                                         khat);
  else
    k_bluestein_w<L, false><<<grid, 256, sm, st>>>(src, src_ps, src_ls, n_in, o_in, dst, dst_ps,
                                                   dst_ls, M, nlines, 0, tw, chirp, khat);
  PF_LAUNCH_CHECK("k_bluestein_w");
  return 0;
}

}  // namespace

// Register-path Bluestein pass (Q = plan_q->n in {128, 256, 512, 1024}).
// xpass=1: lines are contiguous rows (src + b*src_ps + l*src_ls + i), output
//          transposed: dst[b*dst_ps + col_nat*dst_ls + l].
// xpass=0: lines are contiguous rows, output dst[b*dst_ps + l*dst_ls + row_nat].
extern "C" int pf_bluestein_warp(int xpass, const void* src, int64_t src_ps, int64_t src_ls,
                                 int n_in, int o_in, void* dst, int64_t dst_ps, int64_t dst_ls,
                                 int M, int nlines, int nplanes, const pf_fft_plan* plan_q,
                                 const void* chirp, const void* khat, void* stream) {
  PF_ARG_CHECK(plan_q && plan_q->n >= 2 * M - 1 && nplanes >= 1 && nlines >= 0,
               "pf_bluestein_warp: bad args");
  if (nlines == 0) return 0;
  const float2* tw = (const float2*)plan_q->tw;
  cudaStream_t st = (cudaStream_t)stream;
#define BW(LL)                                                                                \
  return launch_bw<LL>(xpass, (const float2*)src, src_ps, src_ls, n_in, o_in, (float2*)dst,   \
                       dst_ps, dst_ls, M, nlines, nplanes, tw, (const float2*)chirp,          \
                       (const float2*)khat, st);
  switch (plan_q->n) {
    case 128: BW(4)
    case 256: BW(8)
    case 512: BW(16)
    case 1024: BW(32)
    default: break;
  }
#undef BW
  pf_set_error("pf_bluestein_warp: Q must be 128, 256, 512 or 1024");
  return -1;
}
