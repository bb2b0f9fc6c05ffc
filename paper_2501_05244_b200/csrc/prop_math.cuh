// Kernel-synthesis and phase helpers shared by the propagation kernels
// (G = exp(i k r) / r of reference reconstruct.py:128-130 and the
// illumination phase of :133-144).
#pragma once
#include "common.cuh"

// exp(1j * 2 pi * kturns * r) / r with r = sqrt(r2): float rsqrt + one float64
// Newton correction (r = rf + (r2 - rf^2) / (2 rf), error ~ (eps_f)^2 r), phase
// reduced in turns with the large part in float64 and the tiny correction in
// float32 -- no float64 square root or division.
__device__ __forceinline__ float2 turns_to_unit(double t_hi, float t_lo) {
  const float fr = (float)(t_hi - rint(t_hi)) + t_lo;
  float s, c;
  __sincosf(6.28318530717958647692f * fr, &s, &c);
  return make_float2(c, s);
}

__device__ __forceinline__ float2 g_kernel(double r2, double kturns, float kturns_f) {
  const float r2f = (float)r2;
  const float ir = rsqrtf(r2f);
  const float rf = r2f * ir;
  const float e = (float)fma(-(double)rf, (double)rf, r2);
  const float d = 0.5f * e * ir;
  const float2 u = turns_to_unit(kturns * (double)rf, kturns_f * d);
  const float inv = ir * (1.0f - d * ir);   // 1/(rf + d) to first order
  return make_float2(u.x * inv, u.y * inv);
}

__device__ __forceinline__ float2 phase_turns(double r2, double kturns, float kturns_f) {
  const float r2f = (float)r2;
  const float ir = rsqrtf(r2f);
  const float rf = r2f * ir;
  const float e = (float)fma(-(double)rf, (double)rf, r2);
  return turns_to_unit(kturns * (double)rf, kturns_f * (0.5f * e * ir));
}
