// Host-side helpers shared by the whole-algorithm C entry points (algo_rsd.cu,
// algo_srsd.cu): pad rules, FFT plan radices and fp64-built twiddle tables.
#pragma once
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "xfft.cuh"

namespace pfalgo {

constexpr double C_LIGHT = 299792458.0;
constexpr int LANES = 3;
constexpr int HORNER_BLOCK = 32;
constexpr int64_t BATCH_BYTES = 64LL << 20;

inline bool close_rel(double a, double b) {
  return fabs(a - b) <= fmax(1e-9 * fmax(fabs(a), fabs(b)), 1e-12);
}

inline bool smooth11(long n) {
  if (n < 1) return false;
  const int ps[5] = {2, 3, 5, 7, 11};
  for (int p : ps)
    while (n % p == 0) n /= p;
  return n == 1;
}

inline long next_fast_len(long n) {
  if (n < 1) n = 1;
  while (!smooth11(n)) n++;
  return n;
}

inline long exact_pad(double lag_max, double nu_max, long n_min) {
  long need = 2 * (long)ceil(fmax(lag_max, nu_max)) + 2;
  if (need < n_min) need = n_min;
  long p2 = 1;
  while (p2 < need) p2 *= 2;
  if (64 < need && p2 <= 1024 && p2 * 5 <= need * 8) return p2;
  return next_fast_len(need);
}

// stage radices: powers of two merged into as few even stages as possible, then odd primes
// in descending order (_device.radices_for)
inline int radices(long n, int* out) {
  std::vector<int> f;
  long m = n;
  for (int p : {2, 3, 5, 7, 11})
    while (m % p == 0) {
      f.push_back(p);
      m /= p;
    }
  if (m != 1) return -1;
  int k = 0;
  std::vector<int> odd;
  for (int p : f) (p == 2 ? k++ : (odd.push_back(p), 0));
  int ns = 0;
  if (k) {
    const int s = (k + 3) / 4;
    for (int i = 0; i < s; i++) out[ns++] = 1 << (k / s + (i < k % s ? 1 : 0));
  }
  for (int i = (int)odd.size() - 1; i >= 0; i--) out[ns++] = odd[i];   // descending
  return ns;
}

// unit roots exp(-2 pi i m / n) in fp64, rounded to c64; the register-FFT lengths append
// the k1-major twiddles [k1][t] = exp(-2 pi i ((k1 t) mod n) / n), n = 32 L
inline std::vector<float2> twiddles(long n) {
  std::vector<float2> w;
  for (long m = 0; m < n; m++) {
    const double a = -2.0 * M_PI * (double)m / (double)n;
    w.push_back(make_float2((float)cos(a), (float)sin(a)));
  }
  // register FFT tables as the Python plans (_device.xfft_plan_L): L >= 20 by default
  const char* ev = getenv("PF_XFFT");
  long xl = xfft_L((int)n);
  if (ev && strcmp(ev, "0") == 0) xl = 0;
  if (!(ev && strcmp(ev, "all") == 0) && xl < 20) xl = 0;
  if (xl) {   // mixed-radix register FFT: k1-major [35][L]
    for (long k1 = 0; k1 < 35; k1++)
      for (long t = 0; t < xl; t++) {
        const double a = -2.0 * M_PI * (double)((k1 * t) % n) / (double)n;
        w.push_back(make_float2((float)cos(a), (float)sin(a)));
      }
  }
  if (n == 128 || n == 256 || n == 512 || n == 1024) {
    const long L = n / 32;
    for (long k1 = 0; k1 < 32; k1++)
      for (long t = 0; t < L; t++) {
        const double a = -2.0 * M_PI * (double)((k1 * t) % n) / (double)n;
        w.push_back(make_float2((float)cos(a), (float)sin(a)));
      }
  }
  return w;
}


inline int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }

// a pf_fft_plan over a table already in device memory (tw), tagged for the register
// FFT when its table carries the 35 L extension
inline pf_fft_plan make_plan(long n, const void* tw_dev, size_t n_tw) {
  pf_fft_plan p{};
  p.n = (int)n;
  p.nst = radices(n, p.radix);
  p.tw = tw_dev;
  if ((long)n_tw > n && !(n == 128 || n == 256 || n == 512 || n == 1024))
    p.radix[PF_MAX_STAGES - 1] = PF_XFFT_TAG;
  return p;
}

}  // namespace pfalgo
