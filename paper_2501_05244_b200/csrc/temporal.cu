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
#include <stdint.h>
#include <stdlib.h>

#include "fft.cuh"

namespace {

constexpr int K1_THREADS = 256;
constexpr int K1_L = 64;     // inner DFT length
constexpr int K1_KB = 33;    // non-redundant bins of a real 64-point DFT

// 64-point real DFT of x[0..63]: the non-redundant bins k in [0, 32] selected by
// `mask` (bit k; warp-uniform) are stored to dst[0], dst[1], ... in ascending k.
// TWICE: the bins are stored doubled (the split step's two halvings are left to the
// caller, who folds one exact 0.5 into the final scale: 8 instead of 12 instructions a bin).
template <bool TWICE = false>
__device__ __forceinline__ void real_dft64_sel(const float* x, unsigned long long mask,
                                               float2* dst, int stride = 1) {
  float2 z[32];
#pragma unroll
  for (int q = 0; q < 32; q++) z[q] = make_float2(x[2 * q], x[2 * q + 1]);
  Dft<32, -1>::run(z);
#pragma unroll
  for (int k = 0; k <= 32; k++) {
    if ((mask >> k) & 1ull) {
      const float2 a = z[k & 31];
      const float2 b = cconj(z[(32 - k) & 31]);
      const float hf = TWICE ? 1.0f : 0.5f;
      const float2 e = make_float2(hf * (a.x + b.x), hf * (a.y + b.y));
      // o = (a - b) / (2i)
      const float2 o = make_float2(hf * (a.y - b.y), -hf * (a.x - b.x));
      // W_64^k = exp(-2 pi i k / 64)
      const float c = Unit<64>::c(k & 63), sn = -Unit<64>::s(k & 63);
      *dst = make_float2(e.x + o.x * c - o.y * sn, e.y + o.x * sn + o.y * c);
      dst += stride;
    }
  }
}

// all 33 bins (the TMA-fed variant)
__device__ __forceinline__ void real_dft64(const float* x, float2* X) {
  real_dft64_sel<false>(x, (1ull << 33) - 1ull, X);
}

// Only the inner bins k = b mod 64 the retained bins need are formed and
// parked (config 4: 20 of the 33 non-redundant bins), slot-major with the
// column index r fastest: xs[g][slot][r] (row stride MP).  Phase B gives each
// retained bin two threads (even / odd r, combined by one shuffle); the bins
// that fold to 64 - k read conjugated twiddles and conjugate the sum instead
// of every term.  Strides MP = M + 2 and TS = 4 (mod 16) keep the parking
// stores and the phase-B loads free of shared-memory bank conflicts.
template <int M>
__global__ void __launch_bounds__(K1_THREADS)
k_temporal_dft(const float* __restrict__ hist, long long n_traces, const int* __restrict__ bins,
               const float2* __restrict__ twt /*[M][twt_ld]*/, int twt_ld,
               const float2* __restrict__ wphase, int F, float2* __restrict__ out,
               long long out_stride, int ts_cap, unsigned long long inner_mask) {
  constexpr int G = K1_THREADS / M;          // traces per block pass
  constexpr int T = M * K1_L;
  constexpr int MP = M + 2 - (M & 1);
  extern __shared__ float2 smem[];
  float2* tws = smem;                                   // [F][MP]
  int* ks = reinterpret_cast<int*>(tws + F * MP);       // [F] slot | conj << 8
  float2* xs = reinterpret_cast<float2*>(ks + ((F + 1) & ~1));   // [G][TS]
  // the caller's inner-bin set (a kernel argument: warp-uniform branches in the
  // parking loop) or, if not given, the set of this chunk's bins
  unsigned long long mask = inner_mask;
  if (mask == 0) {
    for (int f = 0; f < F; f++) {
      const int k = __ldg(bins + f) & 63;
      mask |= 1ull << (k > 32 ? 64 - k : k);
    }
  }
  const int nk = __popcll(mask);
  const int ts = nk * MP + (((4 - nk * MP) % 16) + 16) % 16;
  if (ts > ts_cap) return;   // unreachable: the launcher checks the bin set on the host
  for (int f = threadIdx.x; f < F; f += K1_THREADS) {
    const int k = bins[f] & 63;
    const int kk = k > 32 ? 64 - k : k;
    ks[f] = __popcll(mask & ((1ull << kk) - 1ull)) | ((k > 32) << 8);
  }
  for (int e = threadIdx.x; e < M * F; e += K1_THREADS) {
    const int rr = e / F, f = e - rr * F;
    float2 w = twt[rr * twt_ld + f];
    if ((bins[f] & 63) > 32) w.y = -w.y;
    tws[f * MP + rr] = w;
  }
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
      real_dft64_sel<false>(x, mask, xs + g * ts + r, MP);
    }
    __syncthreads();
    for (int p0 = 0; p0 < 2 * G * F; p0 += K1_THREADS) {
      const int p = p0 + threadIdx.x;
      const bool valid = p < 2 * G * F;
      const int hh = p & 1, o = p >> 1;
      const int gg = o % G, f = valid ? o / G : 0;
      const int kv = ks[f];
      float2 acc = make_float2(0.f, 0.f);
      if (valid) {
        const float2* src = xs + gg * ts + (kv & 255) * MP + hh;
        const float2* tw = tws + f * MP + hh;
        if (M == 1) {
          if (hh == 0) cacc(acc, src[0], tw[0]);
        } else {
#pragma unroll 16
          for (int j = 0; j < M / 2; j++) cacc(acc, src[2 * j], tw[2 * j]);
        }
      }
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
      const long long tr = grp * G + gg;
      if (valid && hh == 0 && tr < n_traces) {
        if (kv >> 8) acc.y = -acc.y;
        out[(long long)f * out_stride + tr] = cmul(acc, wphase[f]);
      }
    }
    __syncthreads();
  }
}

// Same transform with the traces of a CTA decoupled: the M threads of a trace (M >= 32)
// synchronise among themselves only (a named barrier per trace, or the warp for M = 32)
// and form their own trace's bins in phase B, so one trace's loads overlap another's
// arithmetic instead of every trace of the CTA moving in lock step through
// load -> transform -> park -> sum.
__device__ __forceinline__ void trace_sync(int id, int nthreads) {
  if (nthreads == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
  }
}

template <int M>
__global__ void __launch_bounds__(K1_THREADS)
k_temporal_dft_pair(const float* __restrict__ hist, long long n_traces,
                    const int* __restrict__ bins, const float2* __restrict__ twt, int twt_ld,
                    const float2* __restrict__ wphase, int F, float2* __restrict__ out,
                    long long out_stride, int ts_cap, unsigned long long inner_mask,
                    const unsigned long long* __restrict__ peers = nullptr, int n_peers = 0,
                    long long peer_stride = 0, long long peer_col = 0) {
  static_assert(M >= 32, "one or more whole warps per trace");
  constexpr int G = K1_THREADS / M;
  constexpr int T = M * K1_L;
  // rows of M + 4 float2 (= 4 mod 16): the four bins x two halves of a quarter warp read
  // eight different 16-byte bank groups in phase B's 16-byte loads
  constexpr int MP = M + 4;
  extern __shared__ __align__(16) float2 smem[];
  float2* tws = smem;
  int* ks = reinterpret_cast<int*>(tws + F * MP);
  float2* xs = reinterpret_cast<float2*>(ks + ((F + 3) & ~3));
  unsigned long long mask = inner_mask;
  if (mask == 0) {
    for (int f = 0; f < F; f++) {
      const int k = __ldg(bins + f) & 63;
      mask |= 1ull << (k > 32 ? 64 - k : k);
    }
  }
  const int nk = __popcll(mask);
  const int ts = nk * MP;   // even: every row of every trace stays 16-byte aligned
  if (ts > ts_cap) return;
  for (int f = threadIdx.x; f < F; f += K1_THREADS) {
    const int k = bins[f] & 63;
    const int kk = k > 32 ? 64 - k : k;
    ks[f] = __popcll(mask & ((1ull << kk) - 1ull)) | ((k > 32) << 8);
  }
  for (int e = threadIdx.x; e < M * F; e += K1_THREADS) {
    const int rr = e / F, f = e - rr * F;
    float2 w = twt[rr * twt_ld + f];
    if ((bins[f] & 63) > 32) w.y = -w.y;
    tws[f * MP + rr] = w;
  }
  __syncthreads();
  const int g = threadIdx.x / M;
  const int r = threadIdx.x - g * M;
  float2* xg = xs + g * ts;
  // trace g of CTA b takes traces g*nb + b, g*nb + b + stride, ... (independent streams)
  for (long long trace = (long long)blockIdx.x * G + g; trace < n_traces;
       trace += (long long)gridDim.x * G) {
    const float* h = hist + trace * (long long)T + r;
    float x[64];
#pragma unroll
    for (int q = 0; q < 64; q++) x[q] = __ldg(h + q * M);
    real_dft64_sel<true>(x, mask, xg + r, MP);
    trace_sync(1 + g, M);
    for (int q0 = 0; q0 < 2 * F; q0 += M) {
      const int q = q0 + r;
      const bool valid = q < 2 * F;
      const int hh = q & 1, f = valid ? q >> 1 : 0;
      const int kv = ks[f];
      float2 acc = make_float2(0.f, 0.f);
      if (valid) {
        // the two threads of a bin take the column pairs (4 j + 2 hh, + 1): one 16-byte
        // load each of the parked bins and the twiddles per two terms
        const float4* src = reinterpret_cast<const float4*>(xg + (kv & 255) * MP + 2 * hh);
        const float4* tw = reinterpret_cast<const float4*>(tws + f * MP + 2 * hh);
        float2 acc1 = make_float2(0.f, 0.f);
#pragma unroll 8
        for (int j = 0; j < M / 4; j++) {
          const float4 sv = src[2 * j], tv = tw[2 * j];
          cacc(acc, make_float2(sv.x, sv.y), make_float2(tv.x, tv.y));
          cacc(acc1, make_float2(sv.z, sv.w), make_float2(tv.z, tv.w));
        }
        acc.x += acc1.x;
        acc.y += acc1.y;
      }
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
      if (valid && hh == 0) {
        if (kv >> 8) acc.y = -acc.y;
        // 0.5: the split step's halving (exact), left out of the parked bins
        const float2 val = cscale(cmul(acc, wphase[f]), 0.5f);
        if (n_peers == 0) {
          out[(long long)f * out_stride + trace] = val;
        } else {
          // fused all-gather: this rank's detector shard straight into every rank's full
          // [F][I][D] slice buffer (peer memory over NVLink / NVSwitch)
          const long long o = (long long)f * peer_stride + peer_col + trace;
          for (int j = 0; j < n_peers; j++) reinterpret_cast<float2*>(peers[j])[o] = val;
        }
      }
    }
    trace_sync(1 + g, M);
  }
  if (n_peers) __threadfence_system();   // peer stores visible before the kernel retires
}

static int k1_pair_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PF_K1_PAIR");
    v = e ? atoi(e) : 1;
  }
  return v;
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

// ---- TMA-fed variant (M = 64, i.e. T = 4096, the config 2-4 window) ----------
// The histograms of G consecutive traces are one contiguous run of G*T*4 bytes:
// one elected thread moves it into a shared-memory ring with a 1D bulk copy
// (cp.async.bulk, TMA engine) that completes on the stage's mbarrier, S-1
// groups ahead of the compute.  The threads never issue global loads for the
// payload; they wait on the mbarrier, read their stride-M column from shared
// memory (conflict-free), and phase B uses every thread (two per output).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int G, int S>
__global__ void __launch_bounds__(G * 64, 1)
k_temporal_tma(const float* __restrict__ hist, long long n_traces, const int* __restrict__ bins,
               const float2* __restrict__ twt, int twt_ld, const float2* __restrict__ wphase,
               int F, float2* __restrict__ out, long long out_stride) {
  constexpr int M = 64, T = 64 * M, NT = G * M;
  constexpr int TS = M * K1_KB + 1;
  extern __shared__ __align__(128) unsigned char smraw[];
  float* ring = reinterpret_cast<float*>(smraw);                  // [S][G*T]
  float2* xs = reinterpret_cast<float2*>(ring + (size_t)S * G * T);  // [G][TS]
  float2* tws = xs + G * TS;                                      // [M][F]
  int* kb = reinterpret_cast<int*>(tws + M * F);                  // [F]
  __shared__ __align__(8) unsigned long long full[S];
  const int tid = threadIdx.x;
  for (int e = tid; e < M * F; e += NT) tws[e] = twt[(e / F) * twt_ld + e % F];
  for (int e = tid; e < F; e += NT) kb[e] = bins[e] & 63;
  if (tid == 0) {
    for (int st = 0; st < S; st++) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long n_groups = (n_traces + G - 1) / G;
  const long long first = blockIdx.x, step = gridDim.x;
  auto issue = [&](long long grp, int st) {
    const long long t0 = grp * G;
    const long long cnt = n_traces - t0 < G ? n_traces - t0 : G;
    const unsigned bytes = (unsigned)(cnt * T * sizeof(float));
    mbar_expect_tx(&full[st], bytes);
    bulk_g2s(ring + (size_t)st * G * T, hist + t0 * T, bytes, &full[st]);
  };
  if (tid == 0) {
    for (int k = 0; k < S - 1; k++) {
      const long long grp = first + k * step;
      if (grp < n_groups) issue(grp, k);
    }
  }
  const int g = tid / M, r = tid - (tid / M) * M;
  int it = 0;
  for (long long grp = first; grp < n_groups; grp += step, it++) {
    const int st = it % S;
    if (tid == 0) {   // refill the stage consumed in the previous iteration
      const long long nxt = grp + (long long)(S - 1) * step;
      if (nxt < n_groups) issue(nxt, (it + S - 1) % S);
    }
    mbar_wait(&full[st], (unsigned)((it / S) & 1));
    const long long trace = grp * G + g;
    if (trace < n_traces) {
      const float* h = ring + (size_t)st * G * T + g * T + r;
      float x[64];
#pragma unroll
      for (int q = 0; q < 64; q++) x[q] = h[q * M];
      float2 X[K1_KB];
      real_dft64(x, X);
      float2* dst = xs + g * TS + r * K1_KB;
#pragma unroll
      for (int k = 0; k < K1_KB; k++) dst[k] = X[k];
    }
    __syncthreads();
    // phase B: item = (trace, f, half); the two halves of an item are adjacent lanes
    for (int p = tid; p < G * F * 2; p += NT) {
      const int half = p & 1, q = p >> 1;
      const int gg = q % G, f = q / G;
      const long long tr = grp * G + gg;
      const int k = kb[f];
      const bool cj = k > 32;
      const int kk = cj ? 64 - k : k;
      const float2* src = xs + gg * TS + kk;
      float2 acc = make_float2(0.f, 0.f);
      const int r0 = half * (M / 2);
#pragma unroll 8
      for (int rr = r0; rr < r0 + M / 2; rr++) {
        float2 z = src[rr * K1_KB];
        if (cj) z.y = -z.y;
        cacc(acc, z, tws[rr * F + f]);
      }
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
      if (half == 0 && tr < n_traces) out[(long long)f * out_stride + tr] = cmul(acc, wphase[f]);
    }
    __syncthreads();
  }
}

constexpr int K1_FCHUNK = 64;  // retained bins per pass (shared-memory bound)

template <int M>
int launch_k1(const float* hist, long long n_traces, const int* bins, const float2* twt,
              const float2* wphase, int F_total, float2* out, long long out_stride,
              unsigned long long inner_mask, cudaStream_t st,
              const unsigned long long* peers = nullptr, int n_peers = 0,
              long long peer_stride = 0, long long peer_col = 0) {
  constexpr int G = K1_THREADS / M;
  const int FC = F_total < K1_FCHUNK ? F_total : K1_FCHUNK;
  // parked bins per column: the caller's set of inner bins (bins mod 64 folded to
  // [0, 32]) when given, else the worst case
  inner_mask &= (1ull << 33) - 1ull;
  const int n_inner = __builtin_popcountll(inner_mask);
  // (the kernel parks exactly inner_mask's bins when it is given, else at most min(33, FC)
  // per chunk, so ts <= ts_cap by construction)
  int nk = n_inner >= 1 ? n_inner : (K1_KB < FC ? K1_KB : FC);
  constexpr int MP = M + 4;          // the decoupled kernel's row pitch (>= the lock-step M + 2)
  const int ts_cap = nk * MP + 15;   // per-trace stride incl. the bank-alignment pad
  const size_t smem = ((size_t)G * ts_cap + (size_t)FC * MP) * sizeof(float2) +
                      ((FC + 3) & ~3) * sizeof(int);
  static PfDevOnce attr;  
  if (attr.first()) {
    cudaFuncSetAttribute(k_temporal_dft<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long groups = (n_traces + G - 1) / G;
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_temporal_dft<M>, K1_THREADS, smem);
  if (per < 1) per = 1;
  const long long cap = (long long)nsm * per;
  const int grid_k1 = (int)(groups < cap ? groups : cap);
  constexpr int MPAIR = M >= 32 ? M : 32;
  const bool pair = M >= 32 && (k1_pair_mode() != 0 || n_peers > 0);
  if (n_peers > 0 && !pair) {
    pf_set_error("pf_temporal_dft_peers: needs n_bins = 64 M with M >= 32");
    return -1;
  }
  if (pair) {
    static PfDevOnce attr2;
    if (attr2.first())
      cudaFuncSetAttribute(k_temporal_dft_pair<MPAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           227 * 1024);
  }
  for (int f0 = 0; f0 < F_total; f0 += FC) {
    const int F = F_total - f0 < FC ? F_total - f0 : FC;
    if (pair) {
      k_temporal_dft_pair<MPAIR><<<grid_k1, K1_THREADS, smem, st>>>(
          hist, n_traces, bins + f0, twt + f0, F_total, wphase + f0, F,
          out + (long long)f0 * out_stride, out_stride, ts_cap, inner_mask, peers, n_peers,
          peer_stride, peer_col + (long long)f0 * peer_stride);
      PF_LAUNCH_CHECK("k_temporal_dft_pair");
    } else {
      k_temporal_dft<M><<<grid_k1, K1_THREADS, smem, st>>>(hist, n_traces, bins + f0, twt + f0,
                                                         F_total, wphase + f0, F,
                                                         out + (long long)f0 * out_stride,
                                                         out_stride, ts_cap, inner_mask);
      PF_LAUNCH_CHECK("k_temporal_dft");
    }
  }
  return 0;
}

static int k1_tma_env(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

int launch_k1_tma(const float* hist, long long n_traces, const int* bins, const float2* twt,
                  const float2* wphase, int F, float2* out, long long out_stride,
                  cudaStream_t st) {
  // G traces per stage, S stages (PF_K1_G / PF_K1_S select the measured variants)
  const int G = k1_tma_env("PF_K1_G", 4), S = k1_tma_env("PF_K1_S", 2);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long groups = (n_traces + G - 1) / G;
  const size_t smem = (size_t)S * G * 4096 * sizeof(float) +
                      (size_t)(G * (64 * K1_KB + 1) + 64 * F) * sizeof(float2) + F * sizeof(int);
  if (smem > 220 * 1024) {
    pf_set_error("pf_temporal_dft: TMA ring G=%d S=%d needs %zu bytes of shared memory", G, S, smem);
    return -1;
  }
#define K1_TMA(GG, SS)                                                                        \
  if (G == GG && S == SS) {                                                                   \
    static PfDevOnce attr;                                                                   \
    if (attr.first()) {                                                                              \
      cudaFuncSetAttribute(k_temporal_tma<GG, SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           220 * 1024);                                                       \
    }                                                                                         \
    int per = 0;                                                                              \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_temporal_tma<GG, SS>, GG * 64, smem); \
    if (per < 1) per = 1;                                                                     \
    const int grid = (int)(groups < (long long)nsm * per ? groups : (long long)nsm * per);   \
    k_temporal_tma<GG, SS><<<grid, GG * 64, smem, st>>>(hist, n_traces, bins, twt, F, wphase, \
                                                        F, out, out_stride);                  \
    PF_LAUNCH_CHECK("k_temporal_tma");                                                        \
    return 0;                                                                                 \
  }
  K1_TMA(4, 2)
  K1_TMA(2, 2)
  K1_TMA(2, 3)
  K1_TMA(1, 4)
#undef K1_TMA
  pf_set_error("pf_temporal_dft: unsupported PF_K1_G/PF_K1_S combination");
  return -1;
}

}  // namespace

extern "C" int pf_temporal_dft(const float* hist, int64_t n_traces, int n_bins,
                               const int32_t* bins, const void* twiddle, const void* wphase,
                               int n_freq, void* out, int64_t out_stride,
                               uint64_t inner_mask, void* stream) {
  PF_ARG_CHECK(n_traces >= 0 && n_freq >= 1 && n_bins >= 1, "pf_temporal_dft: bad sizes");
  if (n_traces == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const float2* tw = (const float2*)twiddle;
  const float2* wp = (const float2*)wphase;
  float2* o = (float2*)out;
  const int M = (n_bins % K1_L == 0) ? n_bins / K1_L : 0;
  // TMA-fed variant: opt-in (PF_K1_TMA=1); measured 1.44 ms vs 1.35 ms for the load path at
  // config 4 (K1 is issue-bound, not latency-bound: profiles/r1_k1_variants.json)
  if (M == 64 && ((uintptr_t)hist & 15) == 0 && n_freq <= K1_FCHUNK && getenv("PF_K1_TMA"))
    return launch_k1_tma(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, st);
  switch (M) {
    case 1: return launch_k1<1>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, inner_mask, st);
    case 2: return launch_k1<2>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, inner_mask, st);
    case 4: return launch_k1<4>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, inner_mask, st);
    case 8: return launch_k1<8>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, inner_mask, st);
    case 16: return launch_k1<16>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, inner_mask, st);
    case 32: return launch_k1<32>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, inner_mask, st);
    case 64: return launch_k1<64>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, inner_mask, st);
    case 128: return launch_k1<128>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, inner_mask, st);
    case 256: return launch_k1<256>(hist, n_traces, bins, tw, wp, n_freq, o, out_stride, inner_mask, st);
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
  static PfDevOnce attr;  
  if (attr.first()) {
    cudaFuncSetAttribute(k_temporal_dft_direct, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
  }
  const int grid = (int)(n_traces < 4096 ? n_traces : 4096);
  k_temporal_dft_direct<<<grid, K1_THREADS, n_bins * sizeof(float), (cudaStream_t)stream>>>(
      hist, n_traces, n_bins, bins, (const float2*)unit_roots, (const float2*)wphase, n_freq,
      (float2*)out, out_stride);
  PF_LAUNCH_CHECK("k_temporal_dft_direct");
  return 0;
}

// K1 with the slice all-gather fused into its store (multi-GPU, distributed.PeerSlices):
// every retained bin of this rank's traces goes to peers[j][f * peer_stride + peer_col +
// trace] for each of the n_peers ranks' full slice buffers (this rank's own included).
extern "C" int pf_temporal_dft_peers(const float* hist, int64_t n_traces, int n_bins,
                                     const int32_t* bins, const void* twiddle,
                                     const void* wphase, int n_freq, uint64_t inner_mask,
                                     const uint64_t* peers, int n_peers, int64_t peer_stride,
                                     int64_t peer_col, void* stream) {
  PF_ARG_CHECK(n_traces >= 0 && n_freq >= 1 && peers && n_peers >= 1,
               "pf_temporal_dft_peers: bad arguments");
  if (n_traces == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const float2* tw = (const float2*)twiddle;
  const float2* wp = (const float2*)wphase;
  const unsigned long long* pp = (const unsigned long long*)peers;
  const int M = (n_bins % K1_L == 0) ? n_bins / K1_L : 0;
  switch (M) {
    case 32: return launch_k1<32>(hist, n_traces, bins, tw, wp, n_freq, nullptr, 0, inner_mask, st, pp, n_peers, peer_stride, peer_col);
    case 64: return launch_k1<64>(hist, n_traces, bins, tw, wp, n_freq, nullptr, 0, inner_mask, st, pp, n_peers, peer_stride, peer_col);
    case 128: return launch_k1<128>(hist, n_traces, bins, tw, wp, n_freq, nullptr, 0, inner_mask, st, pp, n_peers, peer_stride, peer_col);
    case 256: return launch_k1<256>(hist, n_traces, bins, tw, wp, n_freq, nullptr, 0, inner_mask, st, pp, n_peers, peer_stride, peer_col);
    default: break;
  }
  pf_set_error("pf_temporal_dft_peers: n_bins must be 64 M with M in {32, 64, 128, 256}");
  return -1;
}
