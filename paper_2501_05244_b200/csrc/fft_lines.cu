// Batched strided 1D FFTs over c64 arrays + centred embedding.
//
// pf_fft_lines is the engine's replacement for numpy.fft.fftn/ifftn on the
// hot path (reference spectral.py:107-124, 156, 167, 356, 375): any axis of
// a 2D/3D array is a set of lines (base offset, element stride).  A CTA stages
// `cnt` lines in shared memory with coalesced loads (element-major when the
// lines are columns, line-major when they are rows), runs the Stockham
// transform (fft.cuh), and writes them back in place.
#include <stdlib.h>

#include "xfft.cuh"

namespace {

constexpr int FL_THREADS = 256;
constexpr size_t FL_SMEM_BUDGET = 200 * 1024;

// line l of a three-level set: inner index l % inner (stride istr), middle index
// (l / inner) % mid (stride mstr), outer index l / (inner mid) (stride ostr).  The two-level
// sets of pf_fft_lines pass mid = LLONG_MAX (no outer level).
struct LineSet {
  long long inner, istr, mid, mstr, ostr;
};
__device__ __forceinline__ long long line_base(long long l, const LineSet& s) {
  const long long q = l / s.inner;
  const long long o = q / s.mid;
  return o * s.ostr + (q - o * s.mid) * s.mstr + (l - q * s.inner) * s.istr;
}

template <int DIR>
__global__ void __launch_bounds__(FL_THREADS)
k_fft_lines(float2* __restrict__ data, pf_fft_plan plan, long long nlines, LineSet ls,
            long long estr, int cnt, float scale) {
  extern __shared__ float2 sm[];
  __shared__ long long lbase[64];
  const int n = plan.n;
  const int ld = pf_ld(n);
  float2* a = sm;
  float2* b = sm + (size_t)cnt * ld;
  const long long l0 = (long long)blockIdx.x * cnt;
  const int nl = (int)(nlines - l0 < cnt ? nlines - l0 : cnt);
  const int tot = nl * n;
  const bool rows = (estr == 1);
  // per-line base offsets once (64-bit div/mod), element index split by a fast divide
  for (int c = threadIdx.x; c < nl; c += FL_THREADS) lbase[c] = line_base(l0 + c, ls);
  __syncthreads();
  const FastDiv split(rows ? n : nl);
  for (int e = threadIdx.x; e < tot; e += FL_THREADS) {
    const int q = split.div(e);
    int c, i;
    if (rows) { c = q; i = e - q * n; } else { i = q; c = e - q * nl; }
    a[c * ld + i] = data[lbase[c] + (long long)i * estr];
  }
  __syncthreads();
  const float2* r = fft_smem<DIR>(a, b, ld, nl, plan);
  for (int e = threadIdx.x; e < tot; e += FL_THREADS) {
    const int q = split.div(e);
    int c, i;
    if (rows) { c = q; i = e - q * n; } else { i = q; c = e - q * nl; }
    data[lbase[c] + (long long)i * estr] = cscale(r[c * ld + i], scale);
  }
}

// Lengths n = 35 L (xfft.cuh): the same staging (coalesced tile of lines in shared
// memory), then each warp transforms 32 / L lines in registers, using each line's own
// tile row as its exchange buffer, and writes the result back into the row in natural
// order before the coalesced store.
template <int L, int DIR>
__global__ void __launch_bounds__(FL_THREADS, 2)
k_xfft_lines(float2* __restrict__ data, const float2* __restrict__ tw2, long long nlines,
             LineSet ls, long long estr, float scale) {
  constexpr int N = XFFT_R * L, LD = N + ((N % 16) == 0 ? 1 : 0), LPW = 32 / L;
  constexpr int CNT = 8 * LPW, J = xfft_J(L);
  extern __shared__ float2 sm[];
  __shared__ long long lbase[CNT];
  const long long l0 = (long long)blockIdx.x * CNT;
  const int nl = (int)(nlines - l0 < CNT ? nlines - l0 : CNT);
  const int tot = nl * N;
  const bool rows = (estr == 1);
  for (int c = threadIdx.x; c < nl; c += FL_THREADS) lbase[c] = line_base(l0 + c, ls);
  __syncthreads();
  const FastDiv split(rows ? N : nl);
  for (int e = threadIdx.x; e < tot; e += FL_THREADS) {
    const int q = split.div(e);
    int c, i;
    if (rows) { c = q; i = e - q * N; } else { i = q; c = e - q * nl; }
    sm[c * LD + i] = data[lbase[c] + (long long)i * estr];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const bool active = line < LPW && warp * LPW + line < nl;
  float2* row = sm + (warp * LPW + (line < LPW ? line : 0)) * LD;
  float2 v[XFFT_R];
#pragma unroll
  for (int m = 0; m < XFFT_R; m++) v[m] = row[t + L * m];
  float2 w[J][L];
  xfft<L, DIR>(v, w, row, tw2, t, active);
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
  __syncthreads();
  for (int e = threadIdx.x; e < tot; e += FL_THREADS) {
    const int q = split.div(e);
    int c, i;
    if (rows) { c = q; i = e - q * N; } else { i = q; c = e - q * nl; }
    data[lbase[c] + (long long)i * estr] = cscale(sm[c * LD + i], scale);
  }
}

template <int L, int DIR>
int launch_xlines(float2* data, const pf_fft_plan& p, long long nlines, const LineSet& ls,
                  long long estr, float scale, cudaStream_t st) {
  constexpr int N = XFFT_R * L, LD = N + ((N % 16) == 0 ? 1 : 0), CNT = 8 * (32 / L);
  const size_t smem = (size_t)CNT * LD * sizeof(float2);
  static PfDevOnce attr;
  if (attr.first())
    cudaFuncSetAttribute(k_xfft_lines<L, DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  const long long grid = (nlines + CNT - 1) / CNT;
  const float2* tw2 = reinterpret_cast<const float2*>(p.tw) + N;   // after the n unit roots
  k_xfft_lines<L, DIR><<<(unsigned)grid, FL_THREADS, smem, st>>>(data, tw2, nlines, ls, estr,
                                                                  scale);
  PF_LAUNCH_CHECK("k_xfft_lines");
  return 0;
}

template <int DIR>
int launch_xfft(float2* data, const pf_fft_plan& p, long long nlines, const LineSet& ls,
                long long estr, float scale, cudaStream_t st) {
  switch (xfft_L(p.n)) {
    case 4: return launch_xlines<4, DIR>(data, p, nlines, ls, estr, scale, st);
    case 5: return launch_xlines<5, DIR>(data, p, nlines, ls, estr, scale, st);
    case 8: return launch_xlines<8, DIR>(data, p, nlines, ls, estr, scale, st);
    case 10: return launch_xlines<10, DIR>(data, p, nlines, ls, estr, scale, st);
    case 15: return launch_xlines<15, DIR>(data, p, nlines, ls, estr, scale, st);
    case 20: return launch_xlines<20, DIR>(data, p, nlines, ls, estr, scale, st);
    case 30: return launch_xlines<30, DIR>(data, p, nlines, ls, estr, scale, st);
    default: return 1;
  }
}

// transpose=1 writes dst[bb][jx][jy] (the transposed grid, px rows of py)
__global__ void k_embed_centered(const float2* __restrict__ src, long long nb, int ny, int nx,
                                 long long sbs, float2* __restrict__ dst, int py, int px,
                                 int transpose) {
  const long long total = nb * (long long)py * px;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long bb = e / ((long long)py * px);
    const int rem = (int)(e - bb * (long long)py * px);
    int jy, jx;
    if (transpose) { jx = rem / py; jy = rem - jx * py; } else { jy = rem / px; jx = rem - jy * px; }
    const int iy = centred(jy, py) + ny / 2;
    const int ix = centred(jx, px) + nx / 2;
    float2 v = make_float2(0.f, 0.f);
    if (iy >= 0 && iy < ny && ix >= 0 && ix < nx) v = src[bb * sbs + (long long)iy * nx + ix];
    dst[e] = v;
  }
}

template <int DIR>
int launch_lines(float2* data, const pf_fft_plan& p, long long nlines, const LineSet& ls,
                 long long estr, float scale, cudaStream_t st) {
  static PfDevOnce attr;  
  if (attr.first()) {
    cudaFuncSetAttribute(k_fft_lines<DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)FL_SMEM_BUDGET);
  }
  const int ld = pf_ld(p.n);
  const size_t per_line = 2 * (size_t)ld * sizeof(float2);
  int cnt = (int)(FL_SMEM_BUDGET / per_line);
  if (cnt < 1) {
    pf_set_error("pf_fft_lines: length %d does not fit shared memory", p.n);
    return -1;
  }
  // enough lines per CTA to keep 256 threads busy (4 elements per thread), more (up to
  // 16) while the grid still gives every SM 4 CTAs: fewer barriers per line
  static int nsm = 0;
  if (nsm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm < 1) nsm = 148;
  }
  const long long w_small = (4 * FL_THREADS + p.n - 1) / p.n;
  const long long w_big = (16 * FL_THREADS + p.n - 1) / p.n;
  long long wl = nlines / (4LL * nsm);
  if (wl < w_small) wl = w_small;
  if (wl > w_big) wl = w_big;
  const int want = (int)wl;
  if (cnt > want) cnt = want < 1 ? 1 : want;
  if (estr != 1 && cnt < 8 && (size_t)8 * per_line <= FL_SMEM_BUDGET) cnt = 8;  // coalescing
  if (cnt > 64) cnt = 64;
  if (cnt > nlines) cnt = (int)nlines;
  const int grid = (int)((nlines + cnt - 1) / cnt);
  k_fft_lines<DIR><<<grid, FL_THREADS, cnt * per_line, st>>>(data, p, nlines, ls, estr, cnt,
                                                             scale);
  PF_LAUNCH_CHECK("k_fft_lines");
  return 0;
}

}  // namespace

static int fft_lines_run(void* data, const pf_fft_plan* plan, int64_t nlines, const LineSet& ls,
                         int64_t elem_stride, int dir, float scale, void* stream) {
  PF_ARG_CHECK(plan != nullptr && plan->n >= 1 && plan->nst <= PF_MAX_STAGES,
               "pf_fft_lines: bad plan");
  PF_ARG_CHECK(ls.inner >= 1 && ls.mid >= 1 && nlines >= 0, "pf_fft_lines: bad line layout");
  if (nlines == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  // 35 L lengths: the register mixed-radix kernel (the plan carries its twiddle table)
  // (the plan builder decides: it tags a plan only where the register FFT is wanted)
  if (plan_xl(*plan)) {
    return dir < 0 ? launch_xfft<-1>((float2*)data, *plan, nlines, ls, elem_stride, scale, st)
                   : launch_xfft<1>((float2*)data, *plan, nlines, ls, elem_stride, scale, st);
  }
  if (dir < 0) return launch_lines<-1>((float2*)data, *plan, nlines, ls, elem_stride, scale, st);
  return launch_lines<1>((float2*)data, *plan, nlines, ls, elem_stride, scale, st);
}

extern "C" int pf_fft_lines(void* data, const pf_fft_plan* plan, int64_t nlines, int64_t inner,
                            int64_t inner_stride, int64_t outer_stride, int64_t elem_stride,
                            int dir, float scale, void* stream) {
  const LineSet ls{inner, inner_stride, LLONG_MAX, outer_stride, 0};
  return fft_lines_run(data, plan, nlines, ls, elem_stride, dir, scale, stream);
}

extern "C" int pf_fft_lines3(void* data, const pf_fft_plan* plan, int64_t nlines, int64_t inner,
                             int64_t inner_stride, int64_t mid, int64_t mid_stride,
                             int64_t outer_stride, int64_t elem_stride, int dir, float scale,
                             void* stream) {
  const LineSet ls{inner, inner_stride, mid, mid_stride, outer_stride};
  return fft_lines_run(data, plan, nlines, ls, elem_stride, dir, scale, stream);
}

extern "C" int pf_embed_centered(const void* src, int64_t nb, int ny, int nx,
                                 int64_t src_batch_stride, void* dst, int py, int px,
                                 int transpose, void* stream) {
  PF_ARG_CHECK(nb >= 0 && ny >= 1 && nx >= 1 && py >= ny && px >= nx,
               "pf_embed_centered: bad sizes");
  if (nb == 0) return 0;
  const long long total = nb * (long long)py * px;
  const int grid = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  k_embed_centered<<<grid, 256, 0, (cudaStream_t)stream>>>(
      (const float2*)src, nb, ny, nx, src_batch_stride, (float2*)dst, py, px, transpose);
  PF_LAUNCH_CHECK("k_embed_centered");
  return 0;
}
