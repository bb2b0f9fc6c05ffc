// Mixed-radix register FFT for the 7-smooth pads of the reference's pad rule
// (reference spectral.py:48 next_fast_len; reconstruct.py:102-110): n = R * L with
// R = 35 points per lane held in registers and L lanes per line (L in {4, 5, 8, 10, 15,
// 20, 30}: n = 140, 175, 280, 350, 525, 700, 1050).
//
//   X[k1 + R k2] = sum_t W_L^{t k2} W_n^{t k1} sum_m x[t + L m] W_R^{m k1}
//
// Lane t of a line holds x[t + L m] (m < R) on entry.  Stage 1 is an R-point DFT over m
// in registers (5 x 7), then the twiddles W_n^{t k1} (fp64-built table, k1-major), one
// exchange through the line's own row of shared memory (L rows of R elements; R odd, so
// the 8-byte accesses of a line's lanes are conflict-free), and stage 2: L-point DFTs
// over t, k1 = t, t + L, ... assigned round robin (lanes with k1 >= R idle).  On return
// w[j][k2] = X[(t + L j) + R k2] for t + L j < R ("k1-major" layout).  The same code with
// DIR = +1 is the unnormalised inverse.  Lengths that are not a multiple of 32 lanes
// leave the last lanes of a warp idle (they take part in the syncs only).
#pragma once
#include "fft.cuh"

constexpr int XFFT_R = 35;

__host__ __device__ constexpr int xfft_J(int L) { return (XFFT_R + L - 1) / L; }

// supported lane counts; 0 when n is not 35 L with such an L
__host__ __device__ inline int xfft_L(int n) {
  if (n % XFFT_R) return 0;
  const int L = n / XFFT_R;
  return (L == 4 || L == 5 || L == 8 || L == 10 || L == 15 || L == 20 || L == 30) ? L : 0;
}

// v: the lane's R inputs; row: the line's exchange row base in shared memory (>= L R
// elements, the line's own, written and read by this line's lanes only); tw2: the plan's
// k1-major twiddle table [R][L] (W_n^{k1 t}); t: lane within the line.
template <int L, int DIR>
__device__ __forceinline__ void xfft(float2 (&v)[XFFT_R], float2 (&w)[xfft_J(L)][L],
                                     float2* __restrict__ row, const float2* __restrict__ tw2,
                                     int t, bool active) {
  constexpr int R = XFFT_R, J = xfft_J(L);
  Dft<R, DIR>::run(v);
  if (t != 0) {
#pragma unroll
    for (int k1 = 1; k1 < R; k1++) {
      const float2 c = __ldg(tw2 + k1 * L + t);
      v[k1] = DIR < 0 ? cmul(v[k1], c) : cmulc(v[k1], c);
    }
  }
  __syncwarp();
  if (active) {
#pragma unroll
    for (int k1 = 0; k1 < R; k1++) row[t * R + k1] = v[k1];
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < J; j++) {
    const int k1 = t + L * j;
    if (J * L == R || k1 < R) {
#pragma unroll
      for (int tp = 0; tp < L; tp++) w[j][tp] = row[tp * R + k1];
      Dft<L, DIR>::run(w[j]);
    }
  }
  __syncwarp();
}
