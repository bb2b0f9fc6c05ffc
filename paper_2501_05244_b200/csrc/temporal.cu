// K1 - temporal phasor transform.
//
// Replaces reference phasor.to_frequency (phasor.py:107-127):
//     coeff[trace, f] = FFT(h[trace, :])[b_f] * w_f * exp(-1j w_f t0)
// The reference runs a full float64 FFT of every histogram and keeps F ~ 16-32
// of T/2 bins.  Here only the retained bins are formed, with a two-level
// factorisation of the DFT (T = 64 M):
//     X[b] = sum_r W_T^{b r} * Z_r[b mod 64],   Z_r[k] = sum_q h[q M + r] W_64^{k q}
// Thread r of a trace loads the stride-M column h[q M + r] (coalesced across
// r), runs a 64-point real DFT in registers (as a 32-point complex FFT plus
// the split step), parks the 33 non-redundant bins in shared memory, and the
// block then forms every retained bin as an M-term twiddled sum (fp64-built
// twiddles).  The kernel reads each histogram byte exactly once and writes
// F complex64 per trace: it is HBM-bound.
#include "fft.cuh"

namespace {

constexpr int K1_THREADS = 256;
constexpr int K1_L = 64;     // inner DFT length
constexpr int K1_KB = 33;    // non-redundant bins of a real 64-point DFT

// 64-point real DFT of x[0..63] -> X[0..32]
__device__ __forceinline__ void real_dft64(const float* x, float2* X) {
  float2 z[32];
#pragma unroll
  for (int q = 0; q < 32; q++) z[q] = make_float2(x[2 * q], x[2 * q + 1]);
  Dft<32, -1>::run(z);
#pragma unroll
  for (int k = 0; k <= 32; k++) {
    const float2 a = z[k & 31];
    const float2 b = cconj(z[(32 - k) & 31]);
    const float2 e = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y + b.y));
    // o = (a - b) / (2i)
    const float2 o = make_float2(0.5f * (a.y - b.y), -0.5f * (a.x - b.x));
    // W_64^k = exp(-2 pi i k / 64)
    const float c = Unit<64>::c(k & 63), s = -Unit<64>::s(k & 63);
    X[k] = make_float2(e.x + o.x * c - o.y * s, e.y + o.x * s + o.y * c);
  }
}

template <int M>
__global__ void __launch_bounds__(K1_THREADS)
k_temporal_dft(const float* __restrict__ hist, long long n_traces, const int* __restrict__ bins,
               const float2* __restrict__ twt /*[M][twt_ld]*/, int twt_ld,
               const float2* __restrict__ wphase, int F, float2* __restrict__ out,
               long long out_stride) {
  constexpr int G = K1_THREADS / M;          // traces per block pass
  constexpr int TS = M * K1_KB + 1;          // padded per-trace stride (float2)
  constexpr int T = M * K1_L;
  extern __shared__ float2 smem[];
  float2* xs = smem;                 // [G][M][33] (+1 pad per trace)
  float2* tws = smem + G * TS;       // [M][F]
  int* kb = reinterpret_cast<int*>(tws + M * F);  // [F] bin mod 64
  for (int e = threadIdx.x; e < M * F; e += K1_THREADS) tws[e] = twt[(e / F) * twt_ld + e % F];
  for (int e = threadIdx.x; e < F; e += K1_THREADS) kb[e] = bins[e] & 63;
  __syncthreads();

  const int g = threadIdx.x / M;
  const int r = threadIdx.x - g * M;
  const long long n_groups = (n_traces + G - 1) / G;
  for (long long grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const long long trace = grp * G + g;
    if (trace < n_traces) {
      const float* h = hist + trace * (long long)T + r;
      float x[64];
#pragma unroll
      for (int q = 0; q < 64; q++) x[q] = __ldg(h + q * M);
      float2 X[K1_KB];
      real_dft64(x, X);
      float2* dst = xs + g * TS + r * K1_KB;
#pragma unroll
      for (int k = 0; k < K1_KB; k++) dst[k] = X[k];
    }
    __syncthreads();
    for (int p = threadIdx.x; p < G * F; p += K1_THREADS) {
      const int gg = p % G, f = p / G;
      const long long tr = grp * G + gg;
      if (tr >= n_traces) continue;
      const int k = kb[f];
      const bool cj = k > 32;
      const int kk = cj ? 64 - k : k;
      const float2* src = xs + gg * TS + kk;
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll 8
      for (int rr = 0; rr < M; rr++) {
        float2 z = src[rr * K1_KB];
        if (cj) z.y = -z.y;
        cacc(acc, z, tws[rr * F + f]);
      }
      out[(long long)f * out_stride + tr] = cmul(acc, wphase[f]);
    }
    __syncthreads();
  }
}

// Any T: one thread per (trace, bin), trace staged in shared memory.
__global__ void __launch_bounds__(K1_THREADS)
k_temporal_dft_direct(const float* __restrict__ hist, long long n_traces, int T,
                      const int* __restrict__ bins, const float2* __restrict__ wt /*[T] W_T^m*/,
                      const float2* __restrict__ wphase, int F, float2* __restrict__ out,
                      long long out_stride) {
  extern __shared__ float hs[];
  for (long long tr = blockIdx.x; tr < n_traces; tr += gridDim.x) {
    for (int t = threadIdx.x; t < T; t += K1_THREADS) hs[t] = hist[tr * T + t];
    __syncthreads();
    for (int f = threadIdx.x; f < F; f += K1_THREADS) {
      const int b = bins[f] % T;
      float2 acc = make_float2(0.f, 0.f);
      int m = 0;
      for (int t = 0; t < T; t++) {
        const float2 w = __ldg(wt + m);
        acc.x = fmaf(hs[t], w.x, acc.x);
        acc.y = fmaf(hs[t], w.y, acc.y);
        m += b;
        if (m >= T) m -= T;
      }
      out[(long long)f * out_stride + tr] = cmul(acc, wphase[f]);
    }
    __syncthreads();
  }
}

constexpr int K1_FCHUNK = 64;  // retained bins per pass (shared-memory bound)

template <int M>
int launch_k1(const float* hist, long long n_traces, const int* bins, const float2* twt,
              const float2* wphase, int F_total, float2* out, long long out_stride,
              cudaStream_t st) {
  constexpr int G = K1_THREADS / M;
  const int FC = F_total < K1_FCHUNK ? F_total : K1_FCHUNK;
  const size_t smem = (size_t)(G * (M * K1_KB + 1) + M * FC) * sizeof(float2) + FC * sizeof(int);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_temporal_dft<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long groups = (n_traces + G - 1) / G;
  const int grid = (int)(groups < (long long)nsm * 8 ? groups : (long long)nsm * 8);
  for (int f0 = 0; f0 < F_total; f0 += FC) {
    const int F = F_total - f0 < FC ? F_total - f0 : FC;
    k_temporal_dft<M><<<grid, K1_THREADS, smem, st>>>(hist, n_traces, bins + f0, twt + f0,
                                                       F_total, wphase + f0, F,
                                                       out + (long long)f0 * out_stride,
                                                       out_stride);
    PF_LAUNCH_CHECK("k_temporal_dft");
  }
  return 0;
}

}  // namespace

extern "C" int pf_temporal_dft(const float* hist, int64_t n_traces, int n_bins,
                               const int32_t* bins, const void* twiddle, const void* wphase,
                               int n_freq, void* out, int64_t out_stride, void* stream) {
  PF_ARG_CHECK(n_traces >= 0 && n_freq >= 1 && n_bins >= 1, "pf_temporal_dft: bad sizes");
  if (n_traces == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const float2* tw = (const float2*)twiddle;
  const float2* wp = (const float2*)wphase;
  float2* o = (float2*)out;
  const int M = (n_bins % K1_L == 0) ? n_bins / K1_L : 0;
  switch (M) {
    case 1: return launch_k1<1>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, st);
    case 2: return launch_k1<2>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, st);
    case 4: return launch_k1<4>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, st);
    case 8: return launch_k1<8>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, st);
    case 16: return launch_k1<16>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, st);
    case 32: return launch_k1<32>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, st);
    case 64: return launch_k1<64>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, st);
    case 128: return launch_k1<128>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, st);
    case 256: return launch_k1<256>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, st);
    default: break;
  }
  pf_set_error("pf_temporal_dft: n_bins must be 64*M with M a power of two <= 256 "
               "(use pf_temporal_dft_direct)");
  return -1;
}

extern "C" int pf_temporal_dft_direct(const float* hist, int64_t n_traces, int n_bins,
                                      const int32_t* bins, const void* unit_roots,
                                      const void* wphase, int n_freq, void* out,
                                      int64_t out_stride, void* stream) {
  PF_ARG_CHECK(n_traces >= 0 && n_freq >= 1 && n_bins >= 1, "pf_temporal_dft_direct: bad sizes");
  PF_ARG_CHECK(n_bins <= 50 * 1024, "pf_temporal_dft_direct: n_bins too large");
  if (n_traces == 0) return 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_temporal_dft_direct, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  const int grid = (int)(n_traces < 4096 ? n_traces : 4096);
  k_temporal_dft_direct<<<grid, K1_THREADS, n_bins * sizeof(float), (cudaStream_t)stream>>>(
      hist, n_traces, n_bins, bins, (const float2*)unit_roots, (const float2*)wphase, n_freq,
      (float2*)out, out_stride);
  PF_LAUNCH_CHECK("k_temporal_dft_direct");
  return 0;
}
