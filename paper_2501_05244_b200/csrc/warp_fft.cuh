// Register-resident FFT of length n = 32*L (L in {4, 8, 16, 32}) on L lanes.
//
// A warp holds 32/L lines.  Lane (line, t) keeps the 32 elements
// x[t + L*m], m = 0..31, in registers.  Step 1 is a 32-point DFT over m in
// registers, then the W_n^{t k1} twiddles, one shared-memory exchange
// (a 32 x L transpose per line, padded to 33 columns: conflict-free), and a
// L-point DFT over t for each k1 in {t + L q}.  On return lane (line, t) again
// holds X[t + L*m] in v[m] (natural order within the same index set), so a
// forward transform can be followed by a pointwise product and an inverse
// transform without touching shared memory in between.
//
//   X[k1 + 32 k2] = sum_t W_L^{t k2} W_n^{t k1} sum_m x[t + L m] W_32^{m k1}
//
// This replaces the shared-memory Stockham passes of fft.cuh on the
// propagation hot path: ~2 smem round trips per element instead of 2*stages.
#pragma once
#include "fft.cuh"

constexpr int WFFT_XCH = 32 * 33;  // float2 per warp exchange buffer

// `tw` is the plan table: n unit roots followed by the k1-major twiddles
// tw2[k1 * L + t] = W_n^{t k1} (one contiguous run per k1 across the lanes).
// EARLY: issue the 31 twiddle loads before the first 32-point DFT so their
// latency hides behind it (costs 62 registers; for kernels with headroom).
// 32-point DFT of a line whose only nonzero inputs are v[4..11] (the SRSD Bluestein
// window: N relay samples centred in a 4N transform).  Same 4 x 8 factorisation as
// Dft<32>: each radix-4 sub-DFT has a single nonzero input, so it is a broadcast with
// quarter-turn rotations and costs nothing; the twiddles and the radix-8 level remain.
template <int DIR>
__device__ __forceinline__ void dft32_in4_12(float2 (&v)[32]) {
  float2 out[32];
#pragma unroll
  for (int k1 = 0; k1 < 4; k1++) {
    float2 z[8];
#pragma unroll
    for (int n2 = 0; n2 < 8; n2++) {
      const float2 y = n2 >= 4 ? v[n2] : twc<4, DIR>(v[8 + n2], k1);
      z[n2] = twc<32, DIR>(y, n2 * k1);
    }
    Dft<8, DIR>::run(z);
#pragma unroll
    for (int k2 = 0; k2 < 8; k2++) out[k1 + 4 * k2] = z[k2];
  }
#pragma unroll
  for (int m = 0; m < 32; m++) v[m] = out[m];
}

// PRUNE_IN: v[m] is zero for m outside [4, 12) (dft32_in4_12 for the first stage)
template <int L, int DIR, bool EARLY = false, bool PRUNE_IN = false>
__device__ __forceinline__ void wfft(float2 (&v)[32], float2* __restrict__ xch,
                                     const float2* __restrict__ tw_plan) {
  static_assert(L == 4 || L == 8 || L == 16 || L == 32, "L must be 4, 8, 16 or 32");
  const int lane = threadIdx.x & 31;
  const int t = lane % L;
  const float2* __restrict__ tw = tw_plan + 32 * L + t;
  if (EARLY) {
    float2 w[32];
#pragma unroll
    for (int k1 = 1; k1 < 32; k1++) w[k1] = __ldg(tw + k1 * L);
    Dft<32, DIR>::run(v);
#pragma unroll
    for (int k1 = 1; k1 < 32; k1++) v[k1] = DIR < 0 ? cmul(v[k1], w[k1]) : cmulc(v[k1], w[k1]);
  } else {
    if (PRUNE_IN) dft32_in4_12<DIR>(v); else Dft<32, DIR>::run(v);
    if (t != 0) {
#pragma unroll
      for (int k1 = 1; k1 < 32; k1++) {
        const float2 w = __ldg(tw + k1 * L);
        v[k1] = DIR < 0 ? cmul(v[k1], w) : cmulc(v[k1], w);
      }
    }
  }
  float2* row = xch + lane * 33;  // (line, t) row: line*L*33 + t*33
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 32; k1++) row[k1] = v[k1];
  __syncwarp();
  const float2* base = xch + (lane - t) * 33;  // start of this line's block
  constexpr int Q = 32 / L;
#pragma unroll
  for (int q = 0; q < Q; q++) {
    float2 w[L];
#pragma unroll
    for (int tp = 0; tp < L; tp++) w[tp] = base[tp * 33 + t + L * q];
    Dft<L, DIR>::run(w);
    // X[t + L q + 32 k2] = X[t + L (q + Q k2)]
#pragma unroll
    for (int k2 = 0; k2 < L; k2++) v[q + Q * k2] = w[k2];
  }
  __syncwarp();
}
