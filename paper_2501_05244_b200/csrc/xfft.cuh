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
#include "fft.cuh"   // the register FFT itself lives in fft.cuh (used by fft_smem)
