// Mixed-radix (2,3,4,5,7,8,11,16) self-sorting Stockham FFT on shared memory.
//
// Replaces numpy's pocketfft inside the reference's centred transforms
// (reference spectral.py:107-124, phasor.py:119) with a block-cooperative
// transform: every stage reads R operands at stride n/R, applies the stage
// twiddles W_{Ns R}^{r k} (fp64-built table, float2), runs a compile-time
// radix-R butterfly in registers and writes them at stride Ns, ping-ponging
// between two shared-memory buffers.  Lengths are the reference's 11-smooth
// pads (next_fast_len), so radices 2..11 cover every size the path needs.
#pragma once
#include "common.cuh"
#include "../../include/pfgpu.h"

template <int R>
struct Unit;
#include "unit_roots.inc"

// v * exp(DIR * 1j * theta) given (cos theta, sin theta); DIR=-1 forward.
template <int DIR>
__device__ __forceinline__ float2 rot(float2 v, float c, float s) {
  return DIR < 0 ? make_float2(fmaf(v.x, c, v.y * s), fmaf(v.y, c, -v.x * s))
                 : make_float2(fmaf(v.x, c, -v.y * s), fmaf(v.y, c, v.x * s));
}

template <int R, int DIR>
struct Dft;

template <int DIR>
struct Dft<1, DIR> {
  static __device__ __forceinline__ void run(float2*) {}
};

template <int DIR>
struct Dft<2, DIR> {
  static __device__ __forceinline__ void run(float2* v) {
    float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <int DIR>
struct Dft<4, DIR> {
  static __device__ __forceinline__ void run(float2* v) {
    float2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
    float2 s13 = cadd(v[1], v[3]), d13 = csub(v[1], v[3]);
    // forward: X1 = d02 - i d13, X3 = d02 + i d13
    float2 jd = DIR < 0 ? make_float2(d13.y, -d13.x) : make_float2(-d13.y, d13.x);
    v[0] = cadd(s02, s13);
    v[2] = csub(s02, s13);
    v[1] = cadd(d02, jd);
    v[3] = csub(d02, jd);
  }
};

// radix-2 split of a power-of-two length (8, 16)
template <int R, int DIR>
__device__ __forceinline__ void dft_split(float2* v) {
  float2 e[R / 2], o[R / 2];
#pragma unroll
  for (int i = 0; i < R / 2; i++) {
    e[i] = v[2 * i];
    o[i] = v[2 * i + 1];
  }
  Dft<R / 2, DIR>::run(e);
  Dft<R / 2, DIR>::run(o);
#pragma unroll
  for (int k = 0; k < R / 2; k++) {
    float2 t = (k == 0) ? o[k] : rot<DIR>(o[k], Unit<R>::c(k), Unit<R>::s(k));
    v[k] = cadd(e[k], t);
    v[k + R / 2] = csub(e[k], t);
  }
}

// v * W_N^e (forward, DIR = -1) or v * conj(W_N^e); e is a constant after unrolling,
// so the quarter-turn cases fold to swaps / negations and cost no instructions
template <int N, int DIR>
__device__ __forceinline__ float2 twc(float2 v, int e) {
  e %= N;
  if (e == 0) return v;
  if (2 * e == N) return make_float2(-v.x, -v.y);
  if (4 * e == N) return DIR < 0 ? make_float2(v.y, -v.x) : make_float2(-v.y, v.x);
  if (4 * e == 3 * N) return DIR < 0 ? make_float2(-v.y, v.x) : make_float2(v.y, -v.x);
  return rot<DIR>(v, Unit<N>::c(e), Unit<N>::s(e));
}

// Cooley-Tukey N = A * B in registers: A-point DFTs over n1 of x[B n1 + n2],
// twiddles W_N^{n2 k1}, B-point DFTs over n2; X[k1 + A k2] lands in v[k1 + A k2].
// 4 x 8 for N = 32 takes 432 FP instructions against 470 for the radix-2 split.
template <int A, int B, int DIR>
__device__ __forceinline__ void dft_ct(float2* v) {
  float2 y[B][A];
#pragma unroll
  for (int n2 = 0; n2 < B; n2++) {
#pragma unroll
    for (int n1 = 0; n1 < A; n1++) y[n2][n1] = v[B * n1 + n2];
    Dft<A, DIR>::run(y[n2]);
  }
#pragma unroll
  for (int k1 = 0; k1 < A; k1++) {
    float2 z[B];
#pragma unroll
    for (int n2 = 0; n2 < B; n2++) z[n2] = twc<A * B, DIR>(y[n2][k1], n2 * k1);
    Dft<B, DIR>::run(z);
#pragma unroll
    for (int k2 = 0; k2 < B; k2++) v[k1 + A * k2] = z[k2];
  }
}

// 8 = 4 x 2 with the W_8^1 / W_8^3 rotations folded into the last butterflies:
// t = h (x +- y, ...) feeds z0 +- t as two FFMAs (52 FP instructions instead of 56)
template <int DIR>
struct Dft<8, DIR> {
  static __device__ __forceinline__ void run(float2* v) {
    float2 a[4] = {v[0], v[2], v[4], v[6]}, b[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, DIR>::run(a);
    Dft<4, DIR>::run(b);
    constexpr float h = 0.70710678118654752440f;
    // k1 = 0: X0, X4
    v[0] = cadd(a[0], b[0]);
    v[4] = csub(a[0], b[0]);
    // k1 = 2: W_8^2 = -i (forward): X2, X6
    const float2 q = DIR < 0 ? make_float2(b[2].y, -b[2].x) : make_float2(-b[2].y, b[2].x);
    v[2] = cadd(a[2], q);
    v[6] = csub(a[2], q);
    // k1 = 1: W_8^1 b = h (b.x + b.y, b.y - b.x) forward, h (b.x - b.y, b.y + b.x) inverse
    const float2 s1 = DIR < 0 ? make_float2(b[1].x + b[1].y, b[1].y - b[1].x)
                              : make_float2(b[1].x - b[1].y, b[1].y + b[1].x);
    v[1] = make_float2(fmaf(h, s1.x, a[1].x), fmaf(h, s1.y, a[1].y));
    v[5] = make_float2(fmaf(-h, s1.x, a[1].x), fmaf(-h, s1.y, a[1].y));
    // k1 = 3: W_8^3 b = h (b.y - b.x, -b.x - b.y) forward, h (-b.x - b.y, b.x - b.y) inverse
    const float2 s3 = DIR < 0 ? make_float2(b[3].y - b[3].x, -b[3].x - b[3].y)
                              : make_float2(-b[3].x - b[3].y, b[3].x - b[3].y);
    v[3] = make_float2(fmaf(h, s3.x, a[3].x), fmaf(h, s3.y, a[3].y));
    v[7] = make_float2(fmaf(-h, s3.x, a[3].x), fmaf(-h, s3.y, a[3].y));
  }
};
template <int DIR>
struct Dft<16, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_ct<4, 4, DIR>(v); }
};
template <int DIR>
struct Dft<32, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_ct<4, 8, DIR>(v); }
};

// odd prime radix: pair j with R-j (real cosine / sine halves)
template <int R, int DIR>
__device__ __forceinline__ void dft_odd(float2* v) {
  constexpr int H = (R - 1) / 2;
  float2 sp[H], sm[H];
  float2 x0 = v[0], sum = v[0];
#pragma unroll
  for (int j = 1; j <= H; j++) {
    sp[j - 1] = cadd(v[j], v[R - j]);
    sm[j - 1] = csub(v[j], v[R - j]);
    sum = cadd(sum, sp[j - 1]);
  }
  float2 out[R];
  out[0] = sum;
#pragma unroll
  for (int k = 1; k <= H; k++) {
    float2 a = x0, b = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 1; j <= H; j++) {
      const int m = (j * k) % R;
      const float c = Unit<R>::c(m), s = Unit<R>::s(m);
      a.x = fmaf(sp[j - 1].x, c, a.x);
      a.y = fmaf(sp[j - 1].y, c, a.y);
      b.x = fmaf(sm[j - 1].x, s, b.x);
      b.y = fmaf(sm[j - 1].y, s, b.y);
    }
    // forward: X[k] = a - i b, X[R-k] = a + i b
    out[k] = make_float2(a.x - DIR * b.y, a.y + DIR * b.x);
    out[R - k] = make_float2(a.x + DIR * b.y, a.y - DIR * b.x);
  }
#pragma unroll
  for (int k = 0; k < R; k++) v[k] = out[k];
}

template <int DIR>
struct Dft<3, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_odd<3, DIR>(v); }
};
template <int DIR>
struct Dft<5, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_odd<5, DIR>(v); }
};
template <int DIR>
struct Dft<7, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_odd<7, DIR>(v); }
};
template <int DIR>
struct Dft<11, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_odd<11, DIR>(v); }
};

// Prime-factor (Good-Thomas) N = A * B for coprime A, B: no twiddles between the two
// passes.  Input x[n] with n = n1 (mod A), n = n2 (mod B) (CRT map) -> A-point DFTs over n1,
// B-point DFTs over n2 -> X[(B k1 + A k2) mod N], since W_N^{n B k1} = W_A^{n1 k1} and
// W_N^{n A k2} = W_B^{n2 k2}.  Both index maps are compile-time register renamings.
__host__ __device__ constexpr int pf_inv_mod(int a, int m) {
  int r = 1;
  while ((a * r) % m != 1) r++;
  return r;
}
template <int A, int B, int DIR>
__device__ __forceinline__ void dft_pfa(float2* v) {
  constexpr int N = A * B;
  constexpr int CA = B * pf_inv_mod(B % A, A), CB = A * pf_inv_mod(A % B, B);
  float2 y[B][A];
#pragma unroll
  for (int n2 = 0; n2 < B; n2++) {
#pragma unroll
    for (int n1 = 0; n1 < A; n1++) y[n2][n1] = v[(n1 * CA + n2 * CB) % N];
    Dft<A, DIR>::run(y[n2]);
  }
#pragma unroll
  for (int k1 = 0; k1 < A; k1++) {
    float2 z[B];
#pragma unroll
    for (int n2 = 0; n2 < B; n2++) z[n2] = y[n2][k1];
    Dft<B, DIR>::run(z);
#pragma unroll
    for (int k2 = 0; k2 < B; k2++) v[(B * k1 + A * k2) % N] = z[k2];
  }
}

// composite odd / mixed lengths of the mixed-radix register FFT (xfft.cuh)
template <int DIR>
struct Dft<6, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_pfa<2, 3, DIR>(v); }
};
template <int DIR>
struct Dft<10, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_pfa<2, 5, DIR>(v); }
};
template <int DIR>
struct Dft<15, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_pfa<3, 5, DIR>(v); }
};
template <int DIR>
struct Dft<20, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_pfa<4, 5, DIR>(v); }
};
template <int DIR>
struct Dft<30, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_pfa<5, 6, DIR>(v); }
};
template <int DIR>
struct Dft<35, DIR> {
  static __device__ __forceinline__ void run(float2* v) { dft_pfa<5, 7, DIR>(v); }
};

// One Stockham stage over `cnt` transforms (transform b at buf + b*ld).
// Division by a block-invariant divisor d >= 1 for 0 <= x < 2^22:
// float reciprocal estimate plus one integer correction (exact in that range),
// instead of the ~20-instruction integer division sequence.
struct FastDiv {
  int d;
  float inv;
  __device__ __forceinline__ explicit FastDiv(int dd) : d(dd), inv(1.0f / (float)dd) {}
  __device__ __forceinline__ int div(int x) const {
    int q = __float2int_rz((float)x * inv);
    const int r = x - q * d;
    q += (r >= d) - (r < 0);
    return q;
  }
};

template <int R, int DIR>
__device__ __forceinline__ void stockham_stage(const float2* __restrict__ src,
                                               float2* __restrict__ dst, int n, int Ns,
                                               int cnt, int ld, const float2* __restrict__ tw) {
  const int nb = n / R;
  const int total = nb * cnt;
  const int twstride = n / (Ns * R);
  const FastDiv by_nb(nb), by_ns(Ns);
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int b = by_nb.div(t);
    const int j = t - b * nb;
    const float2* s = src + b * ld;
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; r++) v[r] = s[j + r * nb];
    const int k = j - by_ns.div(j) * Ns;
    if (k != 0) {
#pragma unroll
      for (int r = 1; r < R; r++) {
        const float2 w = __ldg(tw + r * k * twstride);
        v[r] = DIR < 0 ? cmul(v[r], w) : cmulc(v[r], w);
      }
    }
    Dft<R, DIR>::run(v);
    float2* d = dst + b * ld + (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; r++) d[r * Ns] = v[r];
  }
}

// Any radix (large prime factors, e.g. padding="none" on a prime-sized relay):
// direct R-point DFT per butterfly straight from shared memory, O(R^2).
template <int DIR>
__device__ __noinline__ void stockham_stage_any(const float2* __restrict__ src,
                                                float2* __restrict__ dst, int n, int Ns, int R,
                                                int cnt, int ld, const float2* __restrict__ tw) {
  const int nb = n / R;
  const int total = nb * cnt * R;
  const int twstride = n / (Ns * R);
  const int wr = n / R;   // W_R^m = W_n^{m n/R}
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int ro = t % R;
    const int bt = t / R;
    const int b = bt / nb;
    const int j = bt - b * nb;
    const int k = j % Ns;
    const float2* s = src + b * ld;
    float2 acc = make_float2(0.f, 0.f);
    for (int ri = 0; ri < R; ri++) {
      float2 x = s[j + ri * nb];
      if (k != 0 && ri != 0) {
        const float2 w = __ldg(tw + ri * k * twstride);
        x = DIR < 0 ? cmul(x, w) : cmulc(x, w);
      }
      const float2 w2 = __ldg(tw + ((ri * ro) % R) * wr);
      acc = cadd(acc, DIR < 0 ? cmul(x, w2) : cmulc(x, w2));
    }
    dst[b * ld + (j - k) * R + k + ro * Ns] = acc;
  }
}

// ---- mixed-radix register FFT for n = 35 L (see xfft.cuh for the algorithm notes) ----
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
// TWS: the table lives in shared memory (plain loads) instead of global memory (__ldg).
template <int L, int DIR, bool TWS = false>
__device__ __forceinline__ void xfft(float2 (&v)[XFFT_R], float2 (&w)[xfft_J(L)][L],
                                     float2* __restrict__ row, const float2* __restrict__ tw2,
                                     int t, bool active) {
  constexpr int R = XFFT_R, J = xfft_J(L);
  Dft<R, DIR>::run(v);
  if (t != 0) {
#pragma unroll
    for (int k1 = 1; k1 < R; k1++) {
      const float2 c = TWS ? tw2[k1 * L + t] : __ldg(tw2 + k1 * L + t);
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

// All `cnt` lines of a shared-memory tile (row stride ld >= n) by the register FFT, in
// place, natural order in and out; each warp owns 32 / L lines at a time and uses their
// own rows as the exchange buffer.  Block-wide: every thread calls it; synchronised on
// return.
template <int L, int DIR, bool TWS = false>
__device__ __forceinline__ void xfft_tile(float2* __restrict__ a, int ld, int cnt,
                                       const float2* __restrict__ tw2) {
  constexpr int LPW = 32 / L, J = xfft_J(L);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int t = lane % L, line = lane / L;
  for (int c0 = warp * LPW; c0 < cnt; c0 += nw * LPW) {
    const int c = c0 + (line < LPW ? line : 0);
    const bool active = line < LPW && c < cnt;
    float2* row = a + (size_t)(c < cnt ? c : c0) * ld;
    float2 v[XFFT_R];
#pragma unroll
    for (int m = 0; m < XFFT_R; m++) v[m] = row[t + L * m];
    float2 w[J][L];
    xfft<L, DIR, TWS>(v, w, row, tw2, t, active);
    if (active) {
#pragma unroll
      for (int j = 0; j < J; j++) {
        const int k1 = t + L * j;
        if (J * L == XFFT_R || k1 < XFFT_R) {
#pragma unroll
          for (int k2 = 0; k2 < L; k2++) row[k1 + XFFT_R * k2] = w[j][k2];
        }
      }
    }
    __syncwarp();
  }
  __syncthreads();
}

// Run the full transform on `cnt` length-n lines held in `a` (scratch `b`).
// Caller must __syncthreads() after filling `a`.  Returns the buffer holding
// the natural-order result; all threads are synchronised on return.
template <int DIR>
__device__ float2* fft_smem(float2* a, float2* b, int ld, int cnt, const pf_fft_plan& p) {
  int Ns = 1;
  float2* src = a;
  float2* dst = b;
  const float2* tw = reinterpret_cast<const float2*>(p.tw);
  for (int s = 0; s < p.nst; s++) {
    const int R = p.radix[s];
    switch (R) {
      case 2: stockham_stage<2, DIR>(src, dst, p.n, Ns, cnt, ld, tw); break;
      case 3: stockham_stage<3, DIR>(src, dst, p.n, Ns, cnt, ld, tw); break;
      case 4: stockham_stage<4, DIR>(src, dst, p.n, Ns, cnt, ld, tw); break;
      case 5: stockham_stage<5, DIR>(src, dst, p.n, Ns, cnt, ld, tw); break;
      case 7: stockham_stage<7, DIR>(src, dst, p.n, Ns, cnt, ld, tw); break;
      case 8: stockham_stage<8, DIR>(src, dst, p.n, Ns, cnt, ld, tw); break;
      case 11: stockham_stage<11, DIR>(src, dst, p.n, Ns, cnt, ld, tw); break;
      case 16: stockham_stage<16, DIR>(src, dst, p.n, Ns, cnt, ld, tw); break;
      default: stockham_stage_any<DIR>(src, dst, p.n, Ns, R, cnt, ld, tw); break;
    }
    __syncthreads();
    Ns *= R;
    float2* t = src;
    src = dst;
    dst = t;
  }
  return src;
}

// XL = 0: the Stockham stages (scratch b); XL = L: the 35 L register FFT in place (the
// plan carries its twiddle table, PF_XFFT_TAG).  Returns the buffer holding the result.
template <int XL, int DIR>
__device__ __forceinline__ float2* fft_any(float2* a, float2* b, int ld, int cnt,
                                           const pf_fft_plan& p) {
  if constexpr (XL > 0) {
    xfft_tile<XL, DIR>(a, ld, cnt, reinterpret_cast<const float2*>(p.tw) + p.n);
    return a;
  } else {
    return fft_smem<DIR>(a, b, ld, cnt, p);
  }
}

// XL for a plan: the register FFT's lane count when the plan is tagged, else 0
__host__ __device__ inline int plan_xl(const pf_fft_plan& p) {
  return p.radix[PF_MAX_STAGES - 1] == PF_XFFT_TAG ? xfft_L(p.n) : 0;
}

// instantiate CALL with constexpr XL = the plan's register-FFT lane count (0: Stockham)
#define PF_XL_DISPATCH(xl, CALL)                                                            \
  switch (xl) {                                                                             \
    case 4: { constexpr int XL = 4; CALL; } break;                                          \
    case 5: { constexpr int XL = 5; CALL; } break;                                          \
    case 8: { constexpr int XL = 8; CALL; } break;                                          \
    case 10: { constexpr int XL = 10; CALL; } break;                                        \
    case 15: { constexpr int XL = 15; CALL; } break;                                        \
    case 20: { constexpr int XL = 20; CALL; } break;                                        \
    case 30: { constexpr int XL = 30; CALL; } break;                                        \
    default: { constexpr int XL = 0; CALL; } break;                                         \
  }

// padded leading dimension for `cnt` lines of length n in shared memory
__host__ __device__ __forceinline__ int pf_ld(int n) { return n + ((n % 16) == 0 ? 1 : 0); }
