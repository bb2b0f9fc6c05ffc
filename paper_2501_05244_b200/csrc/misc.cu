// Small elementwise kernels of the non-planar (nursd3d) stage 1 and the
// type-2 readout plumbing.  Reference: _kernel_3d (reconstruct.py:624-638),
// the uhat3 * g3 product and slab extraction (:758-760).
#include "fft.cuh"

namespace {

int grid_for(long long total) {
  long long g = (total + 255) / 256;
  return (int)(g < 148 * 32 ? (g < 1 ? 1 : g) : 148 * 32);
}

// G3 on the natural 3D grid: exp(1j khat r)/r at centred lags, 0 at zero lag
__global__ void k_kernel3d(float2* __restrict__ out, int pz, int py, int px, double dx, double dy,
                           double dz, double khat) {
  const long long total = (long long)pz * py * px;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int jx = (int)(e % px), jy = (int)((e / px) % py), jz = (int)(e / ((long long)px * py));
    const double lx = centred(jx, px) * dx, ly = centred(jy, py) * dy, lz = centred(jz, pz) * dz;
    const double r = sqrt(lx * lx + ly * ly + lz * lz);
    float2 v = make_float2(0.f, 0.f);
    if (r > 0.0) {
      const float2 e2 = expi_reduced(khat * r);
      const float ir = (float)(1.0 / r);
      v = make_float2(e2.x * ir, e2.y * ir);
    }
    out[e] = v;
  }
}

__global__ void k_cmul(float2* __restrict__ a, const float2* __restrict__ b, long long n,
                       long long b_period, float scale) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    a[e] = cscale(cmul(a[e], b[e % b_period]), scale);
}

__global__ void k_slab(const float2* __restrict__ src, int nb, long long src_stride,
                       long long plane_off, long long plane_elems, float2* __restrict__ dst) {
  const long long total = (long long)nb * plane_elems;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / plane_elems, r = e - b * plane_elems;
    dst[e] = src[b * src_stride + plane_off + r];
  }
}

}  // namespace

extern "C" int pf_kernel3d(void* out, int pz, int py, int px, double dx, double dy, double dz,
                           double khat, void* stream) {
  PF_ARG_CHECK(pz >= 1 && py >= 1 && px >= 1, "pf_kernel3d: bad sizes");
  k_kernel3d<<<grid_for((long long)pz * py * px), 256, 0, (cudaStream_t)stream>>>(
      (float2*)out, pz, py, px, dx, dy, dz, khat);
  PF_LAUNCH_CHECK("k_kernel3d");
  return 0;
}

extern "C" int pf_cmul(void* a, const void* b, int64_t n, int64_t b_period, float scale,
                       void* stream) {
  PF_ARG_CHECK(n >= 0 && b_period >= 1, "pf_cmul: bad sizes");
  if (n == 0) return 0;
  k_cmul<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((float2*)a, (const float2*)b, n, b_period,
                                                        scale);
  PF_LAUNCH_CHECK("k_cmul");
  return 0;
}

// ---- even 3D kernels (G3 of the lattice stages is even in every lag) ---------------------
// The transform of an array that is even along an axis is even along it, so the 3D transform
// of G3 needs only the lines of the non-negative half of the other two axes; the mirrored
// halves an axis' own pass reads are filled by copy.
namespace {
// axis 1: buf[b][z][y][x] = buf[b][z][py - y][x] for y in (py/2, py), z <= zmax, x <= xmax
// axis 0: buf[b][z][y][x] = buf[b][pz - z][y][x] for z in (pz/2, pz), y <= ymax, x <= xmax
__global__ void k_mirror_fill(float2* __restrict__ buf, int nb, int pz, int py, int px, int axis,
                              int lim_a, int xmax) {
  const int n_ax = axis == 1 ? py : pz;
  const int h = n_ax / 2;
  const int n_m = n_ax - h - 1;                     // mirrored slots h + 1 .. n_ax - 1
  const long long per = (long long)(lim_a + 1) * n_m * (xmax + 1);
  const long long total = (long long)nb * per;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / per;
    long long r = e - b * per;
    const int x = (int)(r % (xmax + 1));
    r /= (xmax + 1);
    const int m = (int)(r % n_m) + h + 1;
    const int o = (int)(r / n_m);                   // the other (non-mirrored) axis index
    float2* a = buf + b * (long long)pz * py * px;
    if (axis == 1)
      a[((long long)o * py + m) * px + x] = a[((long long)o * py + (py - m)) * px + x];
    else
      a[((long long)m * py + o) * px + x] = a[((long long)(pz - m) * py + o) * px + x];
  }
}

// a[f][i][z][y][x] *= g[f][z][min(y, py - y)][min(x, px - x)] * scale (g valid on that octant)
__global__ void k_cmul_even(float2* __restrict__ a, const float2* __restrict__ g, int nf, int ni,
                            int pz, int py, int px, float scale) {
  const long long n3 = (long long)pz * py * px;
  const long long total = (long long)nf * ni * n3;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long fi = e / n3;
    const long long r = e - fi * n3;
    const int x = (int)(r % px);
    const long long q = r / px;
    const int y = (int)(q % py), z = (int)(q / py);
    const int ym = 2 * y > py ? py - y : y, xm = 2 * x > px ? px - x : x;
    const float2 gv = g[(fi / ni) * n3 + ((long long)z * py + ym) * px + xm];
    a[e] = cscale(cmul(a[e], gv), scale);
  }
}
}  // namespace

extern "C" int pf_mirror_fill(void* buf, int nb, int pz, int py, int px, int axis, int lim,
                              int xmax, void* stream) {
  PF_ARG_CHECK(buf && nb >= 1 && pz >= 1 && py >= 1 && px >= 1 && (axis == 0 || axis == 1) &&
                   lim >= 0 && lim < (axis == 1 ? pz : py) && xmax >= 0 && xmax < px,
               "pf_mirror_fill: bad args");
  const int n_ax = axis == 1 ? py : pz;
  const long long total = (long long)nb * (lim + 1) * (n_ax - n_ax / 2 - 1) * (xmax + 1);
  if (total <= 0) return 0;
  k_mirror_fill<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>((float2*)buf, nb, pz, py, px,
                                                                   axis, lim, xmax);
  PF_LAUNCH_CHECK("k_mirror_fill");
  return 0;
}

extern "C" int pf_cmul_even(void* a, const void* g, int nf, int ni, int pz, int py, int px,
                            float scale, void* stream) {
  PF_ARG_CHECK(a && g && nf >= 1 && ni >= 1 && pz >= 1 && py >= 1 && px >= 1,
               "pf_cmul_even: bad args");
  k_cmul_even<<<grid_for((long long)nf * ni * pz * py * px), 256, 0, (cudaStream_t)stream>>>(
      (float2*)a, (const float2*)g, nf, ni, pz, py, px, scale);
  PF_LAUNCH_CHECK("k_cmul_even");
  return 0;
}

extern "C" int pf_copy_planes(const void* src, int nb, int64_t src_stride, int64_t plane_off,
                              int64_t plane_elems, void* dst, void* stream) {
  PF_ARG_CHECK(nb >= 0 && plane_elems >= 0, "pf_copy_planes: bad sizes");
  if (nb == 0 || plane_elems == 0) return 0;
  k_slab<<<grid_for((long long)nb * plane_elems), 256, 0, (cudaStream_t)stream>>>(
      (const float2*)src, nb, src_stride, plane_off, plane_elems, (float2*)dst);
  PF_LAUNCH_CHECK("k_slab");
  return 0;
}

// Centred window of natural-order planes (the inverse of the centred embed):
// dst[b][i][j] = src[b][(i - ny/2) mod py][(j - nx/2) mod px] -- the virtual plane of the
// 3D stages sampled on an nx x ny lattice window (the crop of reconstruct.py:650-651).
namespace {
__global__ void k_crop_centered(const float2* __restrict__ src, long long nb, int py, int px,
                                float2* __restrict__ dst, int ny, int nx) {
  const long long total = nb * (long long)ny * nx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / ((long long)ny * nx);
    const int rem = (int)(e - b * (long long)ny * nx);
    const int i = rem / nx, j = rem - i * nx;
    const int sy = natural(i - ny / 2, py), sx = natural(j - nx / 2, px);
    dst[e] = src[(b * py + sy) * (long long)px + sx];
  }
}
}  // namespace

extern "C" int pf_crop_centered(const void* src, int64_t nb, int py, int px, void* dst, int ny,
                                int nx, void* stream) {
  PF_ARG_CHECK(nb >= 0 && ny >= 1 && nx >= 1 && ny <= py && nx <= px,
               "pf_crop_centered: bad sizes");
  if (nb == 0) return 0;
  k_crop_centered<<<grid_for(nb * (long long)ny * nx), 256, 0, (cudaStream_t)stream>>>(
      (const float2*)src, nb, py, px, (float2*)dst, ny, nx);
  PF_LAUNCH_CHECK("k_crop_centered");
  return 0;
}

// One output plane of an inverse DFT along the leading axis (nursd3d stage 1,
// reference reconstruct.py:758-759: cifft_n over (z, y, x), then the slab plane):
// dst[b][j] = scale * sum_z src[b][z][j] * w[z], w[z] = exp(+2 pi i z slab / nz) built
// in float64 on the host.  The y/x inverse transforms of that one plane follow, so the
// full 3D inverse transform is never formed.
namespace {
__global__ void k_zslab(const float2* __restrict__ src, int nb, int nz, long long nyx,
                        const float2* __restrict__ w, float scale, float2* __restrict__ dst) {
  const long long total = (long long)nb * nyx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / nyx, j = e - b * nyx;
    const float2* s = src + b * nz * nyx + j;
    float2 acc = make_float2(0.f, 0.f);
    for (int z = 0; z < nz; z++) acc = cadd(acc, cmul(s[(long long)z * nyx], __ldg(w + z)));
    dst[e] = make_float2(acc.x * scale, acc.y * scale);
  }
}
}  // namespace

extern "C" int pf_zslab(const void* src, int nb, int nz, int64_t nyx, const void* w, float scale,
                        void* dst, void* stream) {
  PF_ARG_CHECK(nb >= 0 && nz >= 1 && nyx >= 0, "pf_zslab: bad sizes");
  if (nb == 0 || nyx == 0) return 0;
  k_zslab<<<grid_for((long long)nb * nyx), 256, 0, (cudaStream_t)stream>>>(
      (const float2*)src, nb, nz, nyx, (const float2*)w, scale, (float2*)dst);
  PF_LAUNCH_CHECK("k_zslab");
  return 0;
}

// circular shift of the trailing (up to 3) axes: dst[b][j] = src[b][(j + s) mod n]
// per axis -- ifftshift uses s = n/2, fftshift s = n - n/2 (spectral.py:107-114)
namespace {
__global__ void k_roll3(const float2* __restrict__ src, float2* __restrict__ dst, long long nb,
                        int n0, int n1, int n2, int s0, int s1, int s2) {
  const long long per = (long long)n0 * n1 * n2, total = per * nb;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / per, r = e - b * per;
    const int j2 = (int)(r % n2), j1 = (int)((r / n2) % n1), j0 = (int)(r / ((long long)n1 * n2));
    const int a0 = (j0 + s0) % n0, a1 = (j1 + s1) % n1, a2 = (j2 + s2) % n2;
    dst[e] = src[b * per + ((long long)a0 * n1 + a1) * n2 + a2];
  }
}
}  // namespace

extern "C" int pf_roll(const void* src, void* dst, int64_t nb, int n0, int n1, int n2, int s0,
                       int s1, int s2, void* stream) {
  PF_ARG_CHECK(nb >= 0 && n0 >= 1 && n1 >= 1 && n2 >= 1 && s0 >= 0 && s1 >= 0 && s2 >= 0,
               "pf_roll: bad sizes");
  if (nb == 0) return 0;
  const long long total = nb * (long long)n0 * n1 * n2;
  k_roll3<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>((const float2*)src, (float2*)dst, nb,
                                                             n0, n1, n2, s0, s1, s2);
  PF_LAUNCH_CHECK("k_roll3");
  return 0;
}

// ---- payload check for containers read straight into device memory:
// out[0] = non-finite count (reference read_dataset core.py:727-728 rejects
// NaN/inf), out[1] = negative count (TransientMeasurement requires photon
// counts >= 0).  HBM-bound single pass, 16-byte loads, one atomic per CTA.
__device__ __forceinline__ int neg(float v) { return v < 0.f; }
__global__ void k_count_nonfinite(const float* __restrict__ x, long long n, int* out) {
  int bad = 0, ng = 0;
  const long long n4 = n >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(x4 + i);
    bad += !isfinite(v.x) + !isfinite(v.y) + !isfinite(v.z) + !isfinite(v.w);
    ng += neg(v.x) + neg(v.y) + neg(v.z) + neg(v.w);
  }
  if (blockIdx.x == 0)
    for (long long i = (n4 << 2) + threadIdx.x; i < n; i += blockDim.x) {
      bad += !isfinite(x[i]);
      ng += neg(x[i]);
    }
  bad = __reduce_add_sync(0xffffffffu, bad);
  ng = __reduce_add_sync(0xffffffffu, ng);
  __shared__ int wsum[2][32];
  if ((threadIdx.x & 31) == 0) {
    wsum[0][threadIdx.x >> 5] = bad;
    wsum[1][threadIdx.x >> 5] = ng;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const bool in = threadIdx.x < (blockDim.x >> 5);
    const int b = __reduce_add_sync(0xffffffffu, in ? wsum[0][threadIdx.x] : 0);
    const int g = __reduce_add_sync(0xffffffffu, in ? wsum[1][threadIdx.x] : 0);
    if (threadIdx.x == 0 && b) atomicAdd(out, b);
    if (threadIdx.x == 0 && g) atomicAdd(out + 1, g);
  }
}

extern "C" int pf_count_nonfinite(const float* x, int64_t n, int32_t* out, void* stream) {
  PF_ARG_CHECK(n >= 0 && out && (n == 0 || x), "pf_count_nonfinite: bad arguments");
  PF_ARG_CHECK(((uintptr_t)x & 15) == 0, "pf_count_nonfinite: x must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(out, 0, 2 * sizeof(int32_t), st);
  if (n == 0) return 0;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  long long want = ((n >> 2) + 255) / 256;
  const int grid = (int)(want < 8LL * nsm ? (want > 0 ? want : 1) : 8LL * nsm);
  k_count_nonfinite<<<grid, 256, 0, st>>>(x, n, out);
  PF_LAUNCH_CHECK("k_count_nonfinite");
  return 0;
}

// ---- rsd3d stage-1 gridding (reference reconstruct.py:680-707: np.add.at of
// coefficient x weight onto the virtual lattice; duplicate targets sum).  The
// geometry-only plan lists, per touched lattice cell, its (point, weight)
// contributions (CSR, host-built); one thread per touched cell sums them in
// fixed order for every value set, so the result is deterministic without
// atomics.  Untouched cells are zeroed by the caller.
__global__ void k_scatter_csr(const int* __restrict__ cell_start, const long long* __restrict__ cells,
                              const int* __restrict__ ent_pt, const float* __restrict__ ent_w,
                              int n_cells, const float2* __restrict__ vals, long long val_stride,
                              int nv, float2* __restrict__ out, long long out_stride) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cells; c += gridDim.x * blockDim.x) {
    const int e0 = cell_start[c], e1 = cell_start[c + 1];
    const long long dst = cells[c];
    for (int v = 0; v < nv; v++) {
      const float2* vv = vals + (long long)v * val_stride;
      float2 acc = make_float2(0.f, 0.f);
      for (int e = e0; e < e1; e++) {
        const float w = ent_w[e];
        const float2 x = vv[ent_pt[e]];
        acc.x = fmaf(w, x.x, acc.x);
        acc.y = fmaf(w, x.y, acc.y);
      }
      out[(long long)v * out_stride + dst] = acc;
    }
  }
}

extern "C" int pf_scatter_csr(const int32_t* cell_start, const int64_t* cells,
                              const int32_t* ent_pt, const float* ent_w, int n_cells,
                              const void* vals, int64_t val_stride, int nv, void* out,
                              int64_t out_stride, void* stream) {
  PF_ARG_CHECK(n_cells >= 0 && nv >= 1, "pf_scatter_csr: bad sizes");
  if (n_cells == 0) return 0;
  const int grid = pf_cdiv(n_cells, 256) < 148 * 16 ? pf_cdiv(n_cells, 256) : 148 * 16;
  k_scatter_csr<<<grid, 256, 0, (cudaStream_t)stream>>>(
      cell_start, (const long long*)cells, ent_pt, ent_w, n_cells, (const float2*)vals,
      val_stride, nv, (float2*)out, out_stride);
  PF_LAUNCH_CHECK("k_scatter_csr");
  return 0;
}

// ---- FP32 peak probe (bench.py roofline denominator; "FP32 peak measured on
// the box"): 8 independent FFMA chains per thread, `iters` rounds, result stored so the
// chains are live.  Flops = 2 * 8 * iters * threads.
__global__ void __launch_bounds__(256) k_fp32_probe(float* out, int iters, float a, float b) {
  float c0 = threadIdx.x, c1 = c0 + 1.f, c2 = c0 + 2.f, c3 = c0 + 3.f;
  float c4 = c0 + 4.f, c5 = c0 + 5.f, c6 = c0 + 6.f, c7 = c0 + 7.f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      c0 = fmaf(c0, a, b); c1 = fmaf(c1, a, b); c2 = fmaf(c2, a, b); c3 = fmaf(c3, a, b);
      c4 = fmaf(c4, a, b); c5 = fmaf(c5, a, b); c6 = fmaf(c6, a, b); c7 = fmaf(c7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
}

extern "C" int pf_fp32_probe(void* out, int blocks, int iters, void* stream) {
  PF_ARG_CHECK(out && blocks > 0 && iters > 0, "pf_fp32_probe: bad args");
  k_fp32_probe<<<blocks, 256, 0, (cudaStream_t)stream>>>((float*)out, iters, 0.9999f, 1e-4f);
  PF_LAUNCH_CHECK("k_fp32_probe");
  return 0;
}
