// Plane-to-plane RSD propagation (the per-frequency, per-plane hot loop).
//
// Reference: rsd reconstruct.py:254-266, srsd :312-325, nursd1 :372-383,
// nursd3d stage 2 :641-659.  For every (frequency f, plane k):
//     plane = cifft2(Uhat_f * cfft2(G_fk))[rows, cols] * mask_fk,  vol[k] += plane
// G_fk[l] = exp(1j khat r)/r, r = |(lag_x, lag_y, dz_k)|, is synthesised on the
// fly (float64 radius and phase reduction) instead of being built
// and stored per plane (the reference holds Nz kernels per frequency: 4.5 GB
// at config 4).
//
// Symmetry: on the length-p torus the lag of natural slot p-j is minus the lag
// of slot j (slot p/2 is its own mirror), and G depends on lag^2, so G is even
// and Ghat(-k) = Ghat(k) exactly.  Kernel A therefore synthesises only rows
// 0..py/2 and keeps columns 0..px/2 of the x-transform; kernel B rebuilds each
// full column by mirroring, transforms it once and uses it for both column kx
// and px-kx.  That removes ~3/8 of the kernel-spectrum work.
//
// Layouts (c64, natural FFT order):
//   ws_a  [nplanes][py/2+1][px/2+1]     kernel spectrum, x-transformed quadrant
//   uhat  [.. per plane offset ..][n_illum][py][px]
//   ws_b  [nplanes][n_illum][ny][px]    column pass output (rows already cropped)
//   vol   [n_frames][.. plane k at k*ny*nx ..]
#include <stdlib.h>

#include "fft.cuh"

namespace {

constexpr int PT = 256;
constexpr size_t PSMEM = 200 * 1024;

__device__ __forceinline__ float2 rsd_kernel(double khat, double lx, double ly, double dz) {
  const double r = sqrt(fma(lx, lx, fma(ly, ly, dz * dz)));
  const float2 e = expi_reduced(khat * r);
  const float ir = (float)(1.0 / r);
  return make_float2(e.x * ir, e.y * ir);
}

// (A) kernel rows jy in [0, py/2] -> x-FFT -> keep kx in [0, px/2]
// Frequency batch (khat_f != nullptr): blockIdx.z is the frequency, ws_a per-f stride ws_a_fs.
template <int XL>
__global__ void __launch_bounds__(PT)
k_prop_kernel_rows(const pf_plane* __restrict__ planes, double khat, pf_prop_geom g,
                   pf_fft_plan plan_x, float2* __restrict__ ws_a, int rows_per_cta,
                   const double* __restrict__ khat_f = nullptr, long long ws_a_fs = 0) {
  extern __shared__ float2 sm[];
  const pf_plane pl = planes[blockIdx.y];
  if (khat_f) {
    khat = khat_f[blockIdx.z];
    ws_a += blockIdx.z * ws_a_fs;
  }
  const int px = g.px, py = g.py;
  const int rows_a = py / 2 + 1, cols_a = px / 2 + 1;
  const int ld = pf_ld(px);
  const int r0 = blockIdx.x * rows_per_cta;
  const int nr = min(rows_per_cta, rows_a - r0);
  float2* a = sm;
  float2* b = sm + (size_t)rows_per_cta * ld;
  const FastDiv dpx(px), dca(cols_a);
  for (int e = threadIdx.x; e < nr * px; e += PT) {
    const int c = dpx.div(e), jx = e - c * px;
    const double lx = (double)centred(jx, px) * pl.lag_dx;
    const double ly = (double)(r0 + c) * pl.lag_dy;
    a[c * ld + jx] = rsd_kernel(khat, lx, ly, pl.dz);
  }
  __syncthreads();
  const float2* res = fft_any<XL, -1>(a, b, ld, nr, plan_x);
  float2* dst = ws_a + ((long long)blockIdx.y * rows_a + r0) * cols_a;
  for (int e = threadIdx.x; e < nr * cols_a; e += PT) {
    const int c = dca.div(e), kx = e - c * cols_a;
    dst[(long long)c * cols_a + kx] = res[c * ld + kx];
  }
}

// (B) per column kx in [0, px/2]: mirror -> y-FFT (Ghat column) -> for each
// illumination and for columns kx and px-kx: * Uhat column -> y-IFFT -> crop rows
template <int XL>
__global__ void __launch_bounds__(PT)
k_prop_columns(const pf_plane* __restrict__ planes, pf_prop_geom g, pf_fft_plan plan_y,
               const float2* __restrict__ ws_a, const float2* __restrict__ uhat,
               float2* __restrict__ ws_b, int cols_per_cta, int product_only,
               long long ws_a_fs = 0, long long uhat_fs = 0, long long ws_b_fs = 0) {
  extern __shared__ float2 sm[];
  ws_a += blockIdx.z * ws_a_fs;   // frequency batch: blockIdx.z is the frequency
  uhat += blockIdx.z * uhat_fs;
  ws_b += blockIdx.z * ws_b_fs;
  const pf_plane pl = planes[blockIdx.y];
  const int px = g.px, py = g.py, ny = g.ny;
  const int rows_a = py / 2 + 1, cols_a = px / 2 + 1;
  const int ld = pf_ld(py);
  const int C = cols_per_cta;
  const int k0 = blockIdx.x * C;
  const int nc = min(C, cols_a - k0);
  float2* buf0 = sm;
  float2* buf1 = sm + (size_t)C * ld;
  float2* buf2 = sm + (size_t)2 * C * ld;
  const float2* src = ws_a + (long long)blockIdx.y * rows_a * cols_a + k0;
  const FastDiv dnc(nc);
  for (int e = threadIdx.x; e < nc * py; e += PT) {
    const int jy = dnc.div(e), c = e - jy * nc;
    const int sy = jy < rows_a ? jy : py - jy;
    buf0[c * ld + jy] = src[(long long)sy * cols_a + c];
  }
  __syncthreads();
  float2* gh = fft_any<XL, -1>(buf0, buf1, ld, nc, plan_y);
  float2* w0 = (gh == buf0) ? buf1 : buf0;
  float2* w1 = buf2;
  const float2* up = uhat + pl.uhat_off;
  for (int p = 0; p < g.n_illum; p++) {
    const float2* u = up + (long long)p * g.uhat_illum_stride;
    float2* outp = ws_b + ((long long)blockIdx.y * g.n_illum + p) * (long long)ny * px;
    for (int side = 0; side < 2; side++) {
      // column handled by slot c on this side; mirrors that coincide are skipped
      for (int e = threadIdx.x; e < nc * py; e += PT) {
        const int jy = dnc.div(e), c = e - jy * nc;
        const int kx = k0 + c;
        const int col = (side == 0 || kx == 0) ? kx : px - kx;
        w0[c * ld + jy] = cmul(gh[c * ld + jy], u[(long long)jy * px + col]);
      }
      __syncthreads();
      if (product_only) {   // full spectrum column for a type-2 readout: [plane][p][py][px]
        float2* sp = ws_b + ((long long)blockIdx.y * g.n_illum + p) * (long long)py * px;
        for (int e = threadIdx.x; e < nc * py; e += PT) {
          const int jy = dnc.div(e), c = e - jy * nc;
          const int kx = k0 + c;
          const int col = (side == 0 || kx == 0) ? kx : px - kx;
          if (side == 1 && col == kx) continue;
          sp[(long long)jy * px + col] = w0[c * ld + jy];
        }
        __syncthreads();
        continue;
      }
      const float2* res = fft_any<XL, 1>(w0, w1, ld, nc, plan_y);
      for (int e = threadIdx.x; e < nc * ny; e += PT) {
        const int i = dnc.div(e), c = e - i * nc;
        const int kx = k0 + c;
        const int col = (side == 0 || kx == 0) ? kx : px - kx;
        if (side == 1 && col == kx) continue;
        const int jy = natural((long long)g.nu0y + i, py);
        outp[(long long)i * px + col] = res[c * ld + jy];
      }
      __syncthreads();
    }
  }
}

// (C) per output row: x-IFFT -> crop columns -> scale -> illumination phase -> accumulate
template <int XL>
__global__ void __launch_bounds__(PT)
k_prop_rows_out(const pf_plane* __restrict__ planes, double khat, pf_prop_geom g,
                pf_fft_plan plan_x, const float2* __restrict__ ws_b,
                const double* __restrict__ ill, const float2* __restrict__ frame_w, int n_frames,
                float2* __restrict__ vol, long long vol_frame_stride, int rows_per_cta) {
  extern __shared__ float2 sm[];
  const pf_plane pl = planes[blockIdx.y];
  const int px = g.px, nx = g.nx, ny = g.ny;
  const int ld = pf_ld(px);
  const int i0 = blockIdx.x * rows_per_cta;
  const int nr = min(rows_per_cta, ny - i0);
  float2* a = sm;
  float2* b = sm + (size_t)rows_per_cta * ld;
  const float scale = 1.0f / ((float)g.px * (float)g.py);
  const FastDiv dpx(px), dnx(nx);
  for (int p = 0; p < g.n_illum; p++) {
    const float2* src = ws_b + (((long long)blockIdx.y * g.n_illum + p) * ny + i0) * (long long)px;
    for (int e = threadIdx.x; e < nr * px; e += PT) {
      const int c = dpx.div(e), jx = e - c * px;
      a[c * ld + jx] = src[(long long)c * px + jx];
    }
    __syncthreads();
    const float2* res = fft_any<XL, 1>(a, b, ld, nr, plan_x);
    const double sx = ill[3 * p], sy = ill[3 * p + 1], sz = ill[3 * p + 2];
    for (int e = threadIdx.x; e < nr * nx; e += PT) {
      const int c = dnx.div(e), m = e - c * nx;
      float2 v = cscale(res[c * ld + natural((long long)g.nu0x + m, px)], scale);
      if (g.include_illum) {
        const double dx = pl.x0 + pl.dx * m - sx;
        const double dy = pl.y0 + pl.dy * (i0 + c) - sy;
        const double dz = pl.z - sz;
        v = cmul(v, expi_reduced(khat * sqrt(fma(dx, dx, fma(dy, dy, dz * dz)))));
      }
      const long long off = (pl.vol_plane * ny + i0 + c) * (long long)nx + m;
      for (int t = 0; t < n_frames; t++) {
        float2* d = vol + t * vol_frame_stride + off;
        *d = cadd(*d, cmul(v, frame_w[t]));
      }
    }
    __syncthreads();
  }
}

// (C) over all nf frequencies of a batch: per (row tile, plane) the ascending-
// frequency sum is formed in shared memory (acc, fp32, same operation order as
// the per-frequency launches) and added to the volume once.  Single frame.
template <int XL>
__global__ void __launch_bounds__(PT)
k_prop_rows_out_fb(const pf_plane* __restrict__ planes, const double* __restrict__ khat_f, int nf,
                   pf_prop_geom g, pf_fft_plan plan_x, const float2* __restrict__ ws_b,
                   long long ws_b_fs, const double* __restrict__ ill,
                   const float2* __restrict__ frame_w, float2* __restrict__ vol,
                   int rows_per_cta) {
  extern __shared__ float2 sm[];
  const pf_plane pl = planes[blockIdx.y];
  const int px = g.px, nx = g.nx, ny = g.ny;
  const int ld = pf_ld(px);
  const int i0 = blockIdx.x * rows_per_cta;
  const int nr = min(rows_per_cta, ny - i0);
  float2* a = sm;
  float2* b = sm + (size_t)rows_per_cta * ld;
  float2* acc = sm + (size_t)2 * rows_per_cta * ld;   // [nr][nx]
  for (int e = threadIdx.x; e < nr * nx; e += PT) acc[e] = make_float2(0.f, 0.f);
  const float scale = 1.0f / ((float)g.px * (float)g.py);
  const FastDiv dpx(px), dnx(nx);
  for (int f = 0; f < nf; f++) {
    const double khat = khat_f[f];
    const float2 fw = frame_w[f];
    for (int p = 0; p < g.n_illum; p++) {
      const float2* src = ws_b + f * ws_b_fs +
                          (((long long)blockIdx.y * g.n_illum + p) * ny + i0) * (long long)px;
      for (int e = threadIdx.x; e < nr * px; e += PT) {
        const int c = dpx.div(e), jx = e - c * px;
        a[c * ld + jx] = src[(long long)c * px + jx];
      }
      __syncthreads();
      const float2* res = fft_any<XL, 1>(a, b, ld, nr, plan_x);
      const double sx = ill[3 * p], sy = ill[3 * p + 1], sz = ill[3 * p + 2];
      for (int e = threadIdx.x; e < nr * nx; e += PT) {
        const int c = dnx.div(e), m = e - c * nx;
        float2 v = cscale(res[c * ld + natural((long long)g.nu0x + m, px)], scale);
        if (g.include_illum) {
          const double dx = pl.x0 + pl.dx * m - sx;
          const double dy = pl.y0 + pl.dy * (i0 + c) - sy;
          const double dz = pl.z - sz;
          v = cmul(v, expi_reduced(khat * sqrt(fma(dx, dx, fma(dy, dy, dz * dz)))));
        }
        acc[e] = cadd(acc[e], cmul(v, fw));
      }
      __syncthreads();
    }
  }
  for (int e = threadIdx.x; e < nr * nx; e += PT) {
    const int c = dnx.div(e), m = e - c * nx;
    float2* d = vol + (pl.vol_plane * ny + i0 + c) * (long long)nx + m;
    *d = cadd(*d, acc[e]);
  }
}

template <typename K>
void allow_smem(K kern) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PSMEM);
}

int rows_fit(int n, int bufs, int want) {
  const size_t per = (size_t)bufs * pf_ld(n) * sizeof(float2);
  int r = (int)(PSMEM / per);
  return r < want ? r : want;
}

// lines per CTA for a stage: the Stockham path wants enough lines to keep every thread of
// every stage busy; the register FFT (xl > 0) wants 32 / xl lines per warp of the CTA (the
// kernels keep their buffer layout, so the shared-memory budget is the same)
int lines_for(int n, int bufs, int want_stockham, int xl) {
  if (xl > 0) return rows_fit(n, bufs, (PT / 32) * (32 / xl));
  return rows_fit(n, bufs, want_stockham);
}

// instantiate kernel K<XL> for the plan's register-FFT lane count

template <int XL>
void allow_generic() {
  allow_smem(k_prop_kernel_rows<XL>);
  allow_smem(k_prop_columns<XL>);
  allow_smem(k_prop_rows_out_fb<XL>);
  allow_smem(k_prop_rows_out<XL>);
}

void allow_all_generic() {
  allow_generic<0>(); allow_generic<4>(); allow_generic<5>(); allow_generic<8>();
  allow_generic<10>(); allow_generic<15>(); allow_generic<20>(); allow_generic<30>();
}

}  // namespace

int pf_prop_fast_L(const pf_prop_geom* g);
int pf_prop_fast_stage(int stage, const pf_plane* planes, int nplanes, double khat,
                       const pf_prop_geom* g, const pf_fft_plan* plan, const void* ws_a_in,
                       void* ws_a_out, const void* uhat, const void* ws_b_in, void* ws_b_out,
                       const double* ill, const void* frame_w, int n_frames, void* vol,
                       long long vfs, cudaStream_t st);

extern "C" int pf_prop_fast(const pf_prop_geom* g) { return g ? 32 * pf_prop_fast_L(g) : 0; }

int pf_prop_fbatch_stage(int stage, const pf_plane* planes, int nplanes, const double* kturns,
                         int nf, const pf_prop_geom* g, const pf_fft_plan* plan, void* ws_a,
                         long long ws_a_fs, const void* uhat, long long uhat_fs, void* ws_b,
                         long long ws_b_fs, const double* ill, const void* frame_w, void* vol,
                         cudaStream_t st);

// Generic (Stockham) path over all nf frequencies: one launch per stage, blockIdx.z
// the frequency in A and B; C loops the frequencies (khat_f in rad/m, [nf]).
static int prop_fbatch_generic(const pf_plane* planes, int nplanes, const double* khat_f, int nf,
                               const pf_prop_geom* g, const pf_fft_plan* plan_x,
                               const pf_fft_plan* plan_y, void* ws_a, int64_t ws_a_fs,
                               const void* uhat, int64_t uhat_fs, void* ws_b, int64_t ws_b_fs,
                               const double* ill, const void* frame_w, void* vol,
                               cudaStream_t st) {
  static PfDevOnce attr;
  if (attr.first()) allow_all_generic();
  const int rows_a = g->py / 2 + 1, cols_a = g->px / 2 + 1;
  const int xlx = plan_xl(*plan_x), xly = plan_xl(*plan_y);
  // many lines per CTA: every Stockham stage (or every warp of the register FFT) has work
  const int rpc = lines_for(g->px, 2, (8 * PT + g->px - 1) / g->px, xlx);
  const int cpc = lines_for(g->py, 3, 16, xly);
  const int rpo = xlx ? rows_fit(g->px, 3, (PT / 32) * (32 / xlx)) : rows_fit(g->px, 3, 8);
  if (rpc < 1 || cpc < 1 || rpo < 1) { pf_set_error("pf_prop_fbatch: pad too large"); return -1; }
  PF_XL_DISPATCH(xlx, (k_prop_kernel_rows<XL><<<dim3(pf_cdiv(rows_a, rpc), nplanes, nf), PT,
                       (size_t)2 * rpc * pf_ld(g->px) * sizeof(float2), st>>>(
      planes, 0.0, *g, *plan_x, (float2*)ws_a, rpc, khat_f, ws_a_fs)))
  PF_LAUNCH_CHECK("k_prop_kernel_rows");
  PF_XL_DISPATCH(xly, (k_prop_columns<XL><<<dim3(pf_cdiv(cols_a, cpc), nplanes, nf), PT,
                   (size_t)3 * cpc * pf_ld(g->py) * sizeof(float2), st>>>(
      planes, *g, *plan_y, (const float2*)ws_a, (const float2*)uhat, (float2*)ws_b, cpc, 0,
      ws_a_fs, uhat_fs, ws_b_fs)))
  PF_LAUNCH_CHECK("k_prop_columns");
  const size_t smo = ((size_t)2 * rpo * pf_ld(g->px) + (size_t)rpo * g->nx) * sizeof(float2);
  PF_XL_DISPATCH(xlx, (k_prop_rows_out_fb<XL><<<dim3(pf_cdiv(g->ny, rpo), nplanes), PT, smo, st>>>(
      planes, khat_f, nf, *g, *plan_x, (const float2*)ws_b, ws_b_fs, ill, (const float2*)frame_w,
      (float2*)vol, rpo)))
  PF_LAUNCH_CHECK("k_prop_rows_out_fb");
  return 0;
}

extern "C" int pf_prop_fbatch_generic(const pf_plane* planes, int nplanes, const double* khat_f,
                                      int nf, const pf_prop_geom* g, const pf_fft_plan* plan_x,
                                      const pf_fft_plan* plan_y, void* ws_a, int64_t ws_a_fs,
                                      const void* uhat, int64_t uhat_fs, void* ws_b,
                                      int64_t ws_b_fs, const double* ill_xyz,
                                      const void* frame_w, void* vol, void* stream) {
  PF_ARG_CHECK(g && plan_x && plan_y && nf >= 1 && nplanes >= 1 && plan_x->n == g->px &&
                   plan_y->n == g->py,
               "pf_prop_fbatch_generic: bad args");
  return prop_fbatch_generic(planes, nplanes, khat_f, nf, g, plan_x, plan_y, ws_a, ws_a_fs, uhat,
                             uhat_fs, ws_b, ws_b_fs, ill_xyz, frame_w, vol, (cudaStream_t)stream);
}

extern "C" int pf_prop_fbatch(const pf_plane* planes, int nplanes, const double* kturns, int nf,
                              const pf_prop_geom* g, const pf_fft_plan* plan, void* ws_a,
                              int64_t ws_a_fs, const void* uhat, int64_t uhat_fs, void* ws_b,
                              int64_t ws_b_fs, const double* ill_xyz, const void* frame_w,
                              void* vol, void* stream) {
  PF_ARG_CHECK(g && plan && nf >= 1 && nplanes >= 1 && pf_prop_fast_L(g) && plan->n == g->px,
               "pf_prop_fbatch: needs the register path (square power-of-two pad)");
  cudaStream_t st = (cudaStream_t)stream;
  for (int stage = 0; stage < 3; stage++) {
    const int rc = pf_prop_fbatch_stage(stage, planes, nplanes, kturns, nf, g, plan, ws_a, ws_a_fs,
                                        uhat, uhat_fs, ws_b, ws_b_fs, ill_xyz, frame_w, vol, st);
    if (rc) return rc;
  }
  return 0;
}

extern "C" int64_t pf_prop_ws_a(const pf_prop_geom* g, int nplanes) {
  return (int64_t)nplanes * (g->py / 2 + 1) * (g->px / 2 + 1);
}

extern "C" int64_t pf_prop_ws_b(const pf_prop_geom* g, int nplanes) {
  return (int64_t)nplanes * g->n_illum * g->ny * (int64_t)g->px;
}

extern "C" int64_t pf_prop_ws_spectrum(const pf_prop_geom* g, int nplanes) {
  return (int64_t)nplanes * g->n_illum * g->py * (int64_t)g->px;
}

extern "C" int pf_prop_kernel_rows(const pf_plane* planes, int nplanes, double khat,
                                   const pf_prop_geom* g, const pf_fft_plan* plan_x, void* ws_a,
                                   void* stream) {
  PF_ARG_CHECK(g && plan_x && plan_x->n == g->px && nplanes >= 1, "pf_prop_kernel_rows: bad args");
  if (pf_prop_fast_L(g))
    return pf_prop_fast_stage(0, planes, nplanes, khat, g, plan_x, nullptr, ws_a, nullptr, nullptr,
                              nullptr, nullptr, nullptr, 0, nullptr, 0, (cudaStream_t)stream);
  static PfDevOnce attr;
  if (attr.first()) allow_all_generic();
  const int rows_a = g->py / 2 + 1;
  const int xl = plan_xl(*plan_x);
  int rpc = lines_for(g->px, 2, (2 * PT + g->px - 1) / g->px, xl);
  if (rpc < 1) { pf_set_error("pf_prop_kernel_rows: px too large"); return -1; }
  dim3 grid(pf_cdiv(rows_a, rpc), nplanes);
  const size_t smem = (size_t)2 * rpc * pf_ld(g->px) * sizeof(float2);
  PF_XL_DISPATCH(xl, (k_prop_kernel_rows<XL><<<grid, PT, smem, (cudaStream_t)stream>>>(
      planes, khat, *g, *plan_x, (float2*)ws_a, rpc)))
  PF_LAUNCH_CHECK("k_prop_kernel_rows");
  return 0;
}

extern "C" int pf_prop_columns(const pf_plane* planes, int nplanes, const pf_prop_geom* g,
                               const pf_fft_plan* plan_y, const void* ws_a, const void* uhat,
                               void* ws_b, int product_only, void* stream) {
  PF_ARG_CHECK(g && plan_y && plan_y->n == g->py && nplanes >= 1, "pf_prop_columns: bad args");
  PF_ARG_CHECK(!(product_only && pf_prop_fast_L(g)),
               "pf_prop_columns: product_only needs a non-register-path geometry");
  if (pf_prop_fast_L(g))
    return pf_prop_fast_stage(1, planes, nplanes, 0.0, g, plan_y, ws_a, nullptr, uhat, nullptr,
                              ws_b, nullptr, nullptr, 0, nullptr, 0, (cudaStream_t)stream);
  static PfDevOnce attr;
  if (attr.first()) allow_all_generic();
  const int cols_a = g->px / 2 + 1;
  int xl = plan_xl(*plan_y);
  // product-only columns (one forward transform and two products per column) measured
  // faster on the Stockham stages than on the 10-lane register FFT (P = 350: 58.9 vs 73.4 us
  // per launch at config 7); PF_PROP_COLS_XL=1 keeps the register FFT there
  static int cols_xl = -1;
  if (cols_xl < 0) {
    const char* e = getenv("PF_PROP_COLS_XL");
    cols_xl = (e && atoi(e) != 0) ? 1 : 0;
  }
  if (product_only && xl > 0 && xl <= 10 && !cols_xl) xl = 0;
  int cpc = lines_for(g->py, 3, 8, xl);
  if (cpc < 1) { pf_set_error("pf_prop_columns: py too large"); return -1; }
  dim3 grid(pf_cdiv(cols_a, cpc), nplanes);
  const size_t smem = (size_t)3 * cpc * pf_ld(g->py) * sizeof(float2);
  PF_XL_DISPATCH(xl, (k_prop_columns<XL><<<grid, PT, smem, (cudaStream_t)stream>>>(
      planes, *g, *plan_y, (const float2*)ws_a, (const float2*)uhat, (float2*)ws_b, cpc,
      product_only)))
  PF_LAUNCH_CHECK("k_prop_columns");
  return 0;
}

extern "C" int pf_prop_rows_out(const pf_plane* planes, int nplanes, double khat,
                                const pf_prop_geom* g, const pf_fft_plan* plan_x,
                                const void* ws_b, const double* ill_xyz, const void* frame_w,
                                int n_frames, void* vol, int64_t vol_frame_stride, void* stream) {
  PF_ARG_CHECK(g && plan_x && plan_x->n == g->px && nplanes >= 1 && n_frames >= 1,
               "pf_prop_rows_out: bad args");
  if (pf_prop_fast_L(g))
    return pf_prop_fast_stage(2, planes, nplanes, khat, g, plan_x, nullptr, nullptr, nullptr, ws_b,
                              nullptr, ill_xyz, frame_w, n_frames, vol, vol_frame_stride,
                              (cudaStream_t)stream);
  static PfDevOnce attr;
  if (attr.first()) allow_all_generic();
  const int xl = plan_xl(*plan_x);
  int rpc = lines_for(g->px, 2, (2 * PT + g->px - 1) / g->px, xl);
  if (rpc < 1) { pf_set_error("pf_prop_rows_out: px too large"); return -1; }
  dim3 grid(pf_cdiv(g->ny, rpc), nplanes);
  const size_t smem = (size_t)2 * rpc * pf_ld(g->px) * sizeof(float2);
  PF_XL_DISPATCH(xl, (k_prop_rows_out<XL><<<grid, PT, smem, (cudaStream_t)stream>>>(
      planes, khat, *g, *plan_x, (const float2*)ws_b, ill_xyz, (const float2*)frame_w, n_frames,
      (float2*)vol, vol_frame_stride, rpc)))
  PF_LAUNCH_CHECK("k_prop_rows_out");
  return 0;
}
