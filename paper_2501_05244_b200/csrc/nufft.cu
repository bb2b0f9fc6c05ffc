// Gaussian-gridding NUFFT, types 1 and 2, in 2D and 3D.
//
// Reference: spectral.py:230-381 (NufftPlan / nufft1 / nufft2).  Same
// geometry-only plan (spread half-width w, fine grid mr = next_fast_len(2m),
// Gaussian variance tau, DISCRETE deconvolution ker = DFT of the truncated
// stencil, so on-lattice points are exact) -- built on the host in float64 by
// the Python layer and uploaded as per-point (i0, d0) pairs.
//
// Type 1 (reference spectral.py:351-358, a Python loop over points) becomes a
// deterministic tiled GATHER: points are bucketed (CSR) by the fine-grid tiles
// their (2w+1)^d stencil touches; one CTA owns one tile, stages its points and
// their per-axis window weights in shared memory and every thread accumulates
// its own cell in fixed point order (no atomics, bit-reproducible).  It then
// writes every cell of its tile exactly once, so no zero-fill pass is needed.
// Type 2 (spectral.py:374-380) interpolates with one thread per target point.
#include <stdlib.h>

#include "fft.cuh"

// pf_nufft_geom: see include/pfgpu.h

namespace {

constexpr int NT = 256;
constexpr int SP_CHUNK = 32;   // points staged per pass
// value sets (complex) accumulated per CTA: 16 when there are at least 16 (every
// frequency of a capture shares one staging of the tile's points), else 8

__device__ __forceinline__ int wrap_off(int d, int mr) {
  // representative of d mod mr in [-mr/2, mr - mr/2), for d in (-mr, 2 mr)
  // (offsets between natural slots plus a tile-local index: no division needed)
  if (d >= mr) d -= mr;
  if (d < -(mr / 2)) d += mr;
  if (d >= mr - mr / 2) d -= mr;
  return d;
}

// Window weight of a tap dl (radians) from the point on axis a.  window 0: the reference's
// Gaussian exp(-dl^2 / 4 tau) (spectral.py:303).  window 1: the exponential of semicircle
// exp(beta (sqrt(1 - (dl / (w h))^2) - 1)) on |dl| < w h, zero outside: 2 w taps in support
// where the Gaussian needs 2 w + 1 = 17 for the same eps = 1e-6 (w = 4 against 8).
__device__ __forceinline__ float pf_win(const pf_nufft_geom& G, int a, float dl) {
  if (G.window == 0) return __expf(-dl * dl * G.inv4tau[a]);
  const float z = dl * G.inv_hw[a];
  const float q = 1.0f - z * z;
  return q > 0.f ? __expf(G.beta * (sqrtf(q) - 1.0f)) : 0.f;
}

// grid: (total tiles, ceil(nv / SP_V)); block: tile cells (<= 256 threads)
template <int SP_V>
__global__ void __launch_bounds__(NT)
k_spread(pf_nufft_geom G, const int* __restrict__ i0, const float* __restrict__ d0,
         const int* __restrict__ tile_start, const int* __restrict__ tile_pts,
         const float2* __restrict__ vals, long long val_stride, int nv,
         float2* __restrict__ fine, long long fine_stride) {
  __shared__ float wgt[SP_CHUNK][3][2 * 16 + 1];
  __shared__ int pi0[SP_CHUNK][3];
  __shared__ float2 pv[SP_V][SP_CHUNK];
  const int tid = threadIdx.x;
  const int tile = blockIdx.x;
  const int tz = tile / (G.ntiles[1] * G.ntiles[2]);
  const int ty = (tile / G.ntiles[2]) % G.ntiles[1];
  const int tx = tile % G.ntiles[2];
  const int cx = tx * G.tile[2] + tid % G.tile[2];
  const int cy = ty * G.tile[1] + (tid / G.tile[2]) % G.tile[1];
  const int cz = tz * G.tile[0] + tid / (G.tile[2] * G.tile[1]);
  const bool inside = tid < G.tile[0] * G.tile[1] * G.tile[2] && cx < G.mr[2] && cy < G.mr[1] &&
                      cz < G.mr[0];
  const int v0 = blockIdx.y * SP_V;
  const int nvv = min(SP_V, nv - v0);
  const int W = 2 * G.w + 1;
  float2 acc[SP_V];
#pragma unroll
  for (int v = 0; v < SP_V; v++) acc[v] = make_float2(0.f, 0.f);
  const int s0 = tile_start[tile], s1 = tile_start[tile + 1];
  // tile origin per axis: a point's offset to every cell of the tile is its
  // offset to the origin (wrapped once, when staged) plus the cell's local index
  const int tile0z = tz * G.tile[0], tile0y = ty * G.tile[1], tile0x = tx * G.tile[2];
  const int lz = cz - tile0z, ly = cy - tile0y, lx = cx - tile0x;
  for (int c0 = s0; c0 < s1; c0 += SP_CHUNK) {
    const int nc = min(SP_CHUNK, s1 - c0);
    __syncthreads();
    for (int e = tid; e < nc * 3; e += NT) {
      const int p = e / 3, a = e - 3 * p;
      const int pt = tile_pts[c0 + p];
      if (a >= 3 - G.dim) {
        const float base = d0[3 * pt + a];
        for (int o = 0; o < W; o++) {
          const float dl = base + (float)(o - G.w) * G.h[a];
          wgt[p][a][o] = pf_win(G, a, dl);
        }
        const int t0 = a == 0 ? tile0z : (a == 1 ? tile0y : tile0x);
        pi0[p][a] = wrap_off(t0 - natural(i0[3 * pt + a], G.mr[a]), G.mr[a]);
      } else {
        for (int o = 0; o < W; o++) wgt[p][a][o] = 1.0f;
        pi0[p][a] = 0;      // unused axis of a 2D grid
      }
    }
    for (int e = tid; e < nc * nvv; e += NT) {
      const int p = e % nc, v = e / nc;
      pv[v][p] = vals[(long long)(v0 + v) * val_stride + tile_pts[c0 + p]];
    }
    __syncthreads();
    if (inside) {
      for (int p = 0; p < nc; p++) {
        // pi0 holds (tile origin - anchor) wrapped; + local index, wrapped once more
        const int ox = wrap_off(pi0[p][2] + lx, G.mr[2]);
        const int oy = wrap_off(pi0[p][1] + ly, G.mr[1]);
        const int oz = G.dim == 3 ? wrap_off(pi0[p][0] + lz, G.mr[0]) : 0;
        if (abs(ox) > G.w || abs(oy) > G.w || abs(oz) > G.w) continue;
        float wv = wgt[p][2][ox + G.w] * wgt[p][1][oy + G.w];
        if (G.dim == 3) wv *= wgt[p][0][oz + G.w];
#pragma unroll
        for (int v = 0; v < SP_V; v++) {
          if (v < nvv) {
            acc[v].x = fmaf(wv, pv[v][p].x, acc[v].x);
            acc[v].y = fmaf(wv, pv[v][p].y, acc[v].y);
          }
        }
      }
    }
  }
  if (inside) {
    const long long cell = ((long long)cz * G.mr[1] + cy) * G.mr[2] + cx;
#pragma unroll
    for (int v = 0; v < SP_V; v++)   // constant indices: acc stays in registers
      if (v < nvv) fine[(long long)(v0 + v) * fine_stride + cell] = acc[v];
  }
}

// type-1 finish: modes (natural order on the m-grid) = fine_hat[c mod mr] / prod ker
// transpose (2D only): write [v][x][y]
__global__ void k_deconv_gather(pf_nufft_geom G, const float2* __restrict__ fine,
                                long long fine_stride, const float* __restrict__ kz,
                                const float* __restrict__ ky, const float* __restrict__ kx,
                                int nv, float2* __restrict__ out, long long out_stride,
                                int transpose) {
  const long long per = (long long)G.m[0] * G.m[1] * G.m[2];
  const long long total = per * nv;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(e / per);
    const long long rem = e - (long long)v * per;
    int jz, jy, jx;
    if (transpose) {
      jy = (int)(rem % G.m[1]);
      jx = (int)((rem / G.m[1]) % G.m[2]);
      jz = 0;
    } else {
      jx = (int)(rem % G.m[2]);
      jy = (int)((rem / G.m[2]) % G.m[1]);
      jz = (int)(rem / ((long long)G.m[2] * G.m[1]));
    }
    const int czc = centred(jz, G.m[0]), cyc = centred(jy, G.m[1]), cxc = centred(jx, G.m[2]);
    const long long cell = ((long long)natural(czc, G.mr[0]) * G.mr[1] + natural(cyc, G.mr[1])) *
                               G.mr[2] + natural(cxc, G.mr[2]);
    const float den = kz[czc + G.m[0] / 2] * ky[cyc + G.m[1] / 2] * kx[cxc + G.m[2] / 2];
    const float2 f = fine[(long long)v * fine_stride + cell];
    out[(long long)v * out_stride + rem] = make_float2(f.x / den, f.y / den);
  }
}

// type-2 start: fine[v][cell] = S[v][mode] / prod ker on mode slots, 0 elsewhere.
// S is natural order on the m-grid (or transposed [x][y] in 2D).
__global__ void k_place(pf_nufft_geom G, const float2* __restrict__ S, long long s_stride,
                        const float* __restrict__ kz, const float* __restrict__ ky,
                        const float* __restrict__ kx, int nv, float2* __restrict__ fine,
                        long long fine_stride, int transpose) {
  const long long per = (long long)G.mr[0] * G.mr[1] * G.mr[2];
  const long long total = per * nv;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(e / per);
    const long long cell = e - (long long)v * per;
    const int fx = (int)(cell % G.mr[2]);
    const int fy = (int)((cell / G.mr[2]) % G.mr[1]);
    const int fz = (int)(cell / ((long long)G.mr[2] * G.mr[1]));
    // centred mode of each fine slot, or out of band
    int c[3];
    const int f3[3] = {fz, fy, fx};
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const int m = G.m[a], mr = G.mr[a];
      int cc = f3[a] < mr - mr / 2 ? f3[a] : f3[a] - mr;
      if (cc < -(m / 2) || cc >= m - m / 2) ok = false;
      c[a] = cc;
    }
    float2 val = make_float2(0.f, 0.f);
    if (ok) {
      const int jz = natural(c[0], G.m[0]), jy = natural(c[1], G.m[1]), jx = natural(c[2], G.m[2]);
      const long long idx = transpose ? ((long long)jx * G.m[1] + jy)
                                      : (((long long)jz * G.m[1] + jy) * G.m[2] + jx);
      const float den = kz[c[0] + G.m[0] / 2] * ky[c[1] + G.m[1] / 2] * kx[c[2] + G.m[2] / 2];
      const float2 s = S[(long long)v * s_stride + idx];
      val = make_float2(s.x / den, s.y / den);
    }
    fine[(long long)v * fine_stride + cell] = val;
  }
}

// type-2 finish (2D): out = sum_stencil fine * wy * wx, then * scale * exp(1j khat r_ill),
// accumulated into vol[frame][dst0 + perm[l]] (frames: exp(1j w t) weights).
// One WARP per target point: lane = stencil column (W = 2w+1 <= 32), a loop over
// the W stencil rows reads one contiguous row segment per step, and a shuffle
// reduction forms the point's value.  Wrap-around is resolved once per row /
// column (no per-tap modulo).
__device__ __forceinline__ int wrap_once(int c, int mr) { return c < 0 ? c + mr : (c >= mr ? c - mr : c); }

__global__ void __launch_bounds__(256)
k_interp2_warp(pf_nufft_geom G, const int* __restrict__ i0, const float* __restrict__ d0,
               const double* __restrict__ xyz, int npts, const float2* __restrict__ fine,
               long long fine_stride, int n_illum, const double* __restrict__ ill, double kturns,
               int include_illum, float scale, const float2* __restrict__ frame_w, int n_frames,
               float2* __restrict__ vol, long long vol_frame_stride, long long dst0,
               const int* __restrict__ perm) {
  const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (l >= npts) return;
  const int W = 2 * G.w + 1;
  const int mry = G.mr[1], mrx = G.mr[2];
  const bool on = lane < W;
  const float dyl = d0[3 * l + 1], dxl = d0[3 * l + 2];
  const float dx = dxl + (float)(lane - G.w) * G.h[2];
  const float wx = on ? pf_win(G, 2, dx) : 0.f;
  // row weights: lane o forms row o's weight once; the row loop broadcasts it
  const float dyo = dyl + (float)(lane - G.w) * G.h[1];
  const float wy_lane = on ? pf_win(G, 1, dyo) : 0.f;
  const int cx = wrap_once(natural((long long)i0[3 * l + 2] - G.w, mrx) + (on ? lane : 0), mrx);
  const int cy0 = natural((long long)i0[3 * l + 1] - G.w, mry);
  float2 tot = make_float2(0.f, 0.f);
  for (int p = 0; p < n_illum; p++) {
    const float2* fp = fine + (long long)p * fine_stride + cx;
    float2 acc = make_float2(0.f, 0.f);
    int cy = cy0;
    for (int oy = 0; oy < W; oy++) {
      const float w = wx * __shfl_sync(0xffffffffu, wy_lane, oy);
      const float2 f = __ldg(fp + (long long)cy * mrx);
      acc.x = fmaf(w, f.x, acc.x);
      acc.y = fmaf(w, f.y, acc.y);
      if (++cy == mry) cy = 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    float2 val = cscale(acc, scale);
    if (include_illum) {
      const double ex = xyz[3 * l] - ill[3 * p], ey = xyz[3 * l + 1] - ill[3 * p + 1];
      const double ez = xyz[3 * l + 2] - ill[3 * p + 2];
      val = cmul(val, expi_reduced(PF_TWO_PI * kturns * sqrt(ex * ex + ey * ey + ez * ez)));
    }
    tot = cadd(tot, val);
  }
  if (lane == 0) {
    const long long lo = perm ? perm[l] : l;   // points may be stored cell-sorted
    for (int f = 0; f < n_frames; f++) {
      float2* d = vol + f * vol_frame_stride + dst0 + lo;
      *d = cadd(*d, cmul(tot, frame_w[f]));
    }
  }
}

// Batched readout: the points of several planes in one launch.  Point l belongs to
// plane plane_idx[l] (fine grids of the launch's planes are fine + (plane - plane0) *
// fine_plane_stride, illumination p at + p * fine_stride) and accumulates into
// vol[frame][dst_idx[l]].  Same per-point arithmetic as k_interp2_warp.
__global__ void __launch_bounds__(256)
k_interp2_batch(pf_nufft_geom G, const int* __restrict__ i0, const float* __restrict__ d0,
                const double* __restrict__ xyz, const int* __restrict__ plane_idx,
                const long long* __restrict__ dst_idx, int npts, int plane0,
                const float2* __restrict__ fine, long long fine_plane_stride,
                long long fine_stride, int n_illum, const double* __restrict__ ill, double kturns,
                int include_illum, float scale, const float2* __restrict__ frame_w, int n_frames,
                float2* __restrict__ vol, long long vol_frame_stride) {
  const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (l >= npts) return;
  const int W = 2 * G.w + 1;
  const int mry = G.mr[1], mrx = G.mr[2];
  const bool on = lane < W;
  const float dyl = d0[3 * l + 1], dxl = d0[3 * l + 2];
  const float dx = dxl + (float)(lane - G.w) * G.h[2];
  const float wx = on ? pf_win(G, 2, dx) : 0.f;
  // row weights: lane o forms row o's weight once; the row loop broadcasts it
  const float dyo = dyl + (float)(lane - G.w) * G.h[1];
  const float wy_lane = on ? pf_win(G, 1, dyo) : 0.f;
  const int cx = wrap_once(natural((long long)i0[3 * l + 2] - G.w, mrx) + (on ? lane : 0), mrx);
  const int cy0 = natural((long long)i0[3 * l + 1] - G.w, mry);
  const float2* fplane = fine + (long long)(plane_idx[l] - plane0) * fine_plane_stride;
  float2 tot = make_float2(0.f, 0.f);
  for (int p = 0; p < n_illum; p++) {
    const float2* fp = fplane + (long long)p * fine_stride + cx;
    float2 acc = make_float2(0.f, 0.f);
    int cy = cy0;
    for (int oy = 0; oy < W; oy++) {
      const float w = wx * __shfl_sync(0xffffffffu, wy_lane, oy);
      const float2 f = __ldg(fp + (long long)cy * mrx);
      acc.x = fmaf(w, f.x, acc.x);
      acc.y = fmaf(w, f.y, acc.y);
      if (++cy == mry) cy = 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    float2 val = cscale(acc, scale);
    if (include_illum) {
      const double ex = xyz[3 * l] - ill[3 * p], ey = xyz[3 * l + 1] - ill[3 * p + 1];
      const double ez = xyz[3 * l + 2] - ill[3 * p + 2];
      val = cmul(val, expi_reduced(PF_TWO_PI * kturns * sqrt(ex * ex + ey * ey + ez * ez)));
    }
    tot = cadd(tot, val);
  }
  if (lane == 0) {
    const long long dst = dst_idx[l];
    for (int f = 0; f < n_frames; f++) {
      float2* d = vol + f * vol_frame_stride + dst;
      *d = cadd(*d, cmul(tot, frame_w[f]));
    }
  }
}

// The batched readout with a half-warp per point (W = 2w + 1 <= 32): lane c of a half
// serves stencil columns c and c + 16 (when c + 16 < W), so a warp interpolates two
// points where the warp-per-point kernel left 32 - W lanes idle; per-point arithmetic
// and summation order per column pair as k_interp2_batch (the column partial sums of a
// row are combined in a different order, fp32 rounding only).
// nodes > 1 (arbitrary voxel depths, z-Chebyshev readout): the voxel's value is the sum
// over its slab's `nodes` consecutive fine grids (first at plane_idx[l]) weighted by its
// Lagrange weights lw[l][m] -- the same stencil on every node grid.
__global__ void __launch_bounds__(256)
k_interp2_batch_h(pf_nufft_geom G, const int* __restrict__ i0, const float* __restrict__ d0,
                  const double* __restrict__ xyz, const int* __restrict__ plane_idx,
                  const long long* __restrict__ dst_idx, int npts, int plane0,
                  const float2* __restrict__ fine, long long fine_plane_stride,
                  long long fine_stride, int n_illum, const double* __restrict__ ill,
                  double kturns, int include_illum, float scale,
                  const float2* __restrict__ frame_w, int n_frames, float2* __restrict__ vol,
                  long long vol_frame_stride, int nodes = 1,
                  const float* __restrict__ lw = nullptr) {
  const int lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4;
  const int l = blockIdx.x * (blockDim.x >> 4) + ((threadIdx.x >> 5) << 1) + half;
  const bool live = l < npts;
  const int lc = live ? l : 0;
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  const int W = 2 * G.w + 1;
  const int mry = G.mr[1], mrx = G.mr[2];
  const bool on1 = hl < W, on2 = hl + 16 < W;
  const float dyl = d0[3 * lc + 1], dxl = d0[3 * lc + 2];
  const float dx1 = dxl + (float)(hl - G.w) * G.h[2];
  const float dx2 = dxl + (float)(hl + 16 - G.w) * G.h[2];
  const float wx1 = on1 ? pf_win(G, 2, dx1) : 0.f;
  const float wx2 = on2 ? pf_win(G, 2, dx2) : 0.f;
  // row weights: lane c forms rows c and c + 16; the row loop broadcasts them
  const float dy1 = dyl + (float)(hl - G.w) * G.h[1];
  const float dy2 = dyl + (float)(hl + 16 - G.w) * G.h[1];
  const float wy1 = on1 ? pf_win(G, 1, dy1) : 0.f;
  const float wy2 = on2 ? pf_win(G, 1, dy2) : 0.f;
  const int cxb = natural((long long)i0[3 * lc + 2] - G.w, mrx);
  const int cx1 = wrap_once(cxb + (on1 ? hl : 0), mrx);
  const int cx2 = wrap_once(cxb + (on2 ? hl + 16 : 0), mrx);
  const int cy0 = natural((long long)i0[3 * lc + 1] - G.w, mry);
  const float2* fplane = fine + (long long)(plane_idx[lc] - plane0) * fine_plane_stride;
  float2 tot = make_float2(0.f, 0.f);
  for (int p = 0; p < n_illum; p++) {
    float2 acc = make_float2(0.f, 0.f);
    for (int m = 0; m < nodes; m++) {
      const float2* fp = fplane + (long long)m * fine_plane_stride + (long long)p * fine_stride;
      const float lwm = lw ? __ldg(lw + (long long)lc * nodes + m) : 1.0f;
      const float wx1m = wx1 * lwm, wx2m = wx2 * lwm;
      int cy = cy0;
      for (int oy = 0; oy < W; oy++) {
        const int src = (half << 4) + (oy & 15);
        const float wa = __shfl_sync(0xffffffffu, wy1, src);
        const float wb = __shfl_sync(0xffffffffu, wy2, src);
        const float wy = oy < 16 ? wa : wb;
        const float2* rowp = fp + (long long)cy * mrx;
        const float2 f1 = __ldg(rowp + cx1);
        const float w1 = wx1m * wy;
        acc.x = fmaf(w1, f1.x, acc.x);
        acc.y = fmaf(w1, f1.y, acc.y);
        if (on2) {
          const float2 f2 = __ldg(rowp + cx2);
          const float w2 = wx2m * wy;
          acc.x = fmaf(w2, f2.x, acc.x);
          acc.y = fmaf(w2, f2.y, acc.y);
        }
        if (++cy == mry) cy = 0;
      }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    float2 val = cscale(acc, scale);
    if (include_illum && hl == 0) {
      const double ex = xyz[3 * lc] - ill[3 * p], ey = xyz[3 * lc + 1] - ill[3 * p + 1];
      const double ez = xyz[3 * lc + 2] - ill[3 * p + 2];
      val = cmul(val, expi_reduced(PF_TWO_PI * kturns * sqrt(ex * ex + ey * ey + ez * ez)));
    }
    tot = cadd(tot, val);
  }
  (void)hmask;
  if (hl == 0 && live) {
    const long long dst = dst_idx[l];
    for (int f = 0; f < n_frames; f++) {
      float2* d = vol + f * vol_frame_stride + dst;
      *d = cadd(*d, cmul(tot, frame_w[f]));
    }
  }
}


// The half-warp readout specialised for W = 17 (w = 8: the reference's default accuracy
// eps = 1e-6), trimmed to the instructions a tap needs: lane c owns stencil column c for
// rows 0..15 (row weights broadcast by shuffle) and row 16 (its weight formed in every
// lane); column 16 is spread over the lanes after the row loop (lane r takes tap (r, 16),
// lane 0 also (16, 16)) instead of a predicated second column in every row.  32-bit cell
// offsets (the fine grid has < 2^31 cells), the torus wrap-around by one compare per row.
// Same weights as k_interp2_batch_h; the column-16 taps join each lane's sum last (fp32
// summation order only).
__global__ void __launch_bounds__(256)
k_interp2_h17(pf_nufft_geom G, const int* __restrict__ i0, const float* __restrict__ d0,
              const double* __restrict__ xyz, const int* __restrict__ plane_idx,
              const long long* __restrict__ dst_idx, int npts, int plane0,
              const float2* __restrict__ fine, long long fine_plane_stride,
              long long fine_stride, int n_illum, const double* __restrict__ ill,
              double kturns, int include_illum, float scale,
              const float2* __restrict__ frame_w, int n_frames, float2* __restrict__ vol,
              long long vol_frame_stride, int nodes, const float* __restrict__ lw) {
  constexpr int w = 8;
  const int lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4;
  const int l = blockIdx.x * (blockDim.x >> 4) + ((threadIdx.x >> 5) << 1) + half;
  const bool live = l < npts;
  const int lc = live ? l : 0;
  const int mry = G.mr[1], mrx = G.mr[2], fe = mry * mrx;
  const float dyl = d0[3 * lc + 1], dxl = d0[3 * lc + 2];
  const float dx = dxl + (float)(hl - w) * G.h[2];
  const float wx = __expf(-dx * dx * G.inv4tau[2]);
  const float dx16 = dxl + (float)(16 - w) * G.h[2];
  const float wx16 = __expf(-dx16 * dx16 * G.inv4tau[2]);
  const float dy = dyl + (float)(hl - w) * G.h[1];
  const float wy_own = __expf(-dy * dy * G.inv4tau[1]);
  const float dy16 = dyl + (float)(16 - w) * G.h[1];
  const float wy16 = __expf(-dy16 * dy16 * G.inv4tau[1]);
  // anchors lie in [0, mr]: the stencil origin wraps at most once
  const int cxb = wrap_once(i0[3 * lc + 2] - w, mrx);
  const int cx = wrap_once(cxb + hl, mrx), cx16 = wrap_once(cxb + 16, mrx);
  const int cy0 = wrap_once(i0[3 * lc + 1] - w, mry);
  const int r0 = cy0 * mrx;                                   // row 0's offset
  const int r_own = wrap_once(cy0 + hl, mry) * mrx;           // this lane's row (column 16)
  const int r16 = wrap_once(cy0 + 16, mry) * mrx;
  const float2* fplane = fine + (long long)(plane_idx[lc] - plane0) * fine_plane_stride;
  float2 tot = make_float2(0.f, 0.f);
  for (int p = 0; p < n_illum; p++) {
    float2 acc = make_float2(0.f, 0.f);
    for (int m = 0; m < nodes; m++) {
      const float2* g = fplane + (long long)m * fine_plane_stride + (long long)p * fine_stride;
      const float lwm = lw ? __ldg(lw + (long long)lc * nodes + m) : 1.0f;
      const float wxm = wx * lwm;
      const float2* col = g + cx;
      int ro = r0;
#pragma unroll 4
      for (int oy = 0; oy < 16; oy++) {
        const float wy = __shfl_sync(0xffffffffu, wy_own, (half << 4) + oy);
        const float2 f = __ldg(col + ro);
        const float ww = wxm * wy;
        acc.x = fmaf(ww, f.x, acc.x);
        acc.y = fmaf(ww, f.y, acc.y);
        ro += mrx;
        if (ro >= fe) ro -= fe;
      }
      {
        const float2 f = __ldg(col + ro);                      // row 16
        const float ww = wxm * wy16;
        acc.x = fmaf(ww, f.x, acc.x);
        acc.y = fmaf(ww, f.y, acc.y);
      }
      const float wx16m = wx16 * lwm;
      {   // column 16: lane r takes row r, lane 0 also row 16
        const float2 f = __ldg(g + r_own + cx16);
        const float ww = wx16m * wy_own;
        acc.x = fmaf(ww, f.x, acc.x);
        acc.y = fmaf(ww, f.y, acc.y);
        if (hl == 0) {
          const float2 f2 = __ldg(g + r16 + cx16);
          const float w2 = wx16m * wy16;
          acc.x = fmaf(w2, f2.x, acc.x);
          acc.y = fmaf(w2, f2.y, acc.y);
        }
      }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    float2 val = cscale(acc, scale);
    if (include_illum && hl == 0) {
      const double ex = xyz[3 * lc] - ill[3 * p], ey = xyz[3 * lc + 1] - ill[3 * p + 1];
      const double ez = xyz[3 * lc + 2] - ill[3 * p + 2];
      val = cmul(val, expi_reduced(PF_TWO_PI * kturns * sqrt(ex * ex + ey * ey + ez * ez)));
    }
    tot = cadd(tot, val);
  }
  if (hl == 0 && live) {
    const long long dst = dst_idx[l];
    for (int f = 0; f < n_frames; f++) {
      float2* d = vol + f * vol_frame_stride + dst;
      *d = cadd(*d, cmul(tot, frame_w[f]));
    }
  }
}

// W = 17 trimmed to 16 x 16 taps.  The reference's Gaussian (tau = pi w / (s (s - 1/2) m^2),
// w = 8, s = 2) weighs a tap j cells from the point by exp(-(3 pi / 32) j^2): of the two
// edge taps of an axis the one on the far side of the anchor lies >= 8 cells away and weighs
// <= 6.5e-9 of the centre tap, i.e. <= 2e-9 of the stencil's sum -- a factor 30 under the
// float32 rounding of the 289-term sum itself.  It is not loaded: each axis keeps the 16
// taps nearest the point (origin i0 - 8 when the anchor lies right of the point, i0 - 7
// otherwise), lane c owns column c for all 16 rows, and the row-16 / column-16 special
// cases of k_interp2_h17 disappear (16 loads per lane per point instead of 18-19).
template <int UNR>
__global__ void __launch_bounds__(256)
k_interp2_h16(pf_nufft_geom G, const int* __restrict__ i0, const float* __restrict__ d0,
              const double* __restrict__ xyz, const int* __restrict__ plane_idx,
              const long long* __restrict__ dst_idx, int npts, int plane0,
              const float2* __restrict__ fine, long long fine_plane_stride,
              long long fine_stride, int n_illum, const double* __restrict__ ill,
              double kturns, int include_illum, float scale,
              const float2* __restrict__ frame_w, int n_frames, float2* __restrict__ vol,
              long long vol_frame_stride, int nodes, const float* __restrict__ lw) {
  constexpr int w = 8;
  const int lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4;
  const int l = blockIdx.x * (blockDim.x >> 4) + ((threadIdx.x >> 5) << 1) + half;
  const bool live = l < npts;
  const int lc = live ? l : 0;
  const int mry = G.mr[1], mrx = G.mr[2], fe = mry * mrx;
  const float dyl = d0[3 * lc + 1], dxl = d0[3 * lc + 2];
  // d0 = anchor - point: anchor right of the point -> the far edge tap is j = +8
  const int sx = dxl > 0.f ? 0 : 1, sy = dyl > 0.f ? 0 : 1;
  const float dx = dxl + (float)(hl - w + sx) * G.h[2];
  const float wx = __expf(-dx * dx * G.inv4tau[2]);
  const float dy = dyl + (float)(hl - w + sy) * G.h[1];
  const float wy_own = __expf(-dy * dy * G.inv4tau[1]);
  // anchors lie in [0, mr]: the stencil origin wraps at most once
  const int cx = wrap_once(wrap_once(i0[3 * lc + 2] - w + sx, mrx) + hl, mrx);
  const int r0 = wrap_once(i0[3 * lc + 1] - w + sy, mry) * mrx;   // row 0's offset
  const float2* fplane = fine + (long long)(plane_idx[lc] - plane0) * fine_plane_stride;
  float2 tot = make_float2(0.f, 0.f);
  for (int p = 0; p < n_illum; p++) {
    float2 acc = make_float2(0.f, 0.f);
    for (int m = 0; m < nodes; m++) {
      const float2* col = fplane + (long long)m * fine_plane_stride +
                          (long long)p * fine_stride + cx;
      const float wxm = lw ? wx * __ldg(lw + (long long)lc * nodes + m) : wx;
      int ro = r0;
#pragma unroll UNR
      for (int oy = 0; oy < 16; oy++) {
        const float wy = __shfl_sync(0xffffffffu, wy_own, (half << 4) + oy);
        const float2 f = __ldg(col + ro);
        const float ww = wxm * wy;
        acc.x = fmaf(ww, f.x, acc.x);
        acc.y = fmaf(ww, f.y, acc.y);
        ro += mrx;
        if (ro >= fe) ro -= fe;
      }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    float2 val = cscale(acc, scale);
    if (include_illum && hl == 0) {
      const double ex = xyz[3 * lc] - ill[3 * p], ey = xyz[3 * lc + 1] - ill[3 * p + 1];
      const double ez = xyz[3 * lc + 2] - ill[3 * p + 2];
      val = cmul(val, expi_reduced(PF_TWO_PI * kturns * sqrt(ex * ex + ey * ey + ez * ez)));
    }
    tot = cadd(tot, val);
  }
  if (hl == 0 && live) {
    const long long dst = dst_idx[l];
    for (int f = 0; f < n_frames; f++) {
      float2* d = vol + f * vol_frame_stride + dst;
      *d = cadd(*d, cmul(tot, frame_w[f]));
    }
  }
}

// Exponential-of-semicircle readout for w = 4 (the default accuracy eps = 1e-6): the window
// vanishes at |d| >= 4 h, so of the taps -4..4 about the nearest node the one on the far side
// of the anchor has weight exactly zero and each axis keeps 8 taps -- a quarter warp per
// point (lane c owns column c, 64-byte row segments), four points per warp, 8 loads per lane
// per point and node.  Same weights as the general kernels; float32 summation order only.
template <int UNR>
__global__ void __launch_bounds__(256)
k_interp2_es8(pf_nufft_geom G, const int* __restrict__ i0, const float* __restrict__ d0,
              const double* __restrict__ xyz, const int* __restrict__ plane_idx,
              const long long* __restrict__ dst_idx, int npts, int plane0,
              const float2* __restrict__ fine, long long fine_plane_stride,
              long long fine_stride, int n_illum, const double* __restrict__ ill,
              double kturns, int include_illum, float scale,
              const float2* __restrict__ frame_w, int n_frames, float2* __restrict__ vol,
              long long vol_frame_stride, int nodes, const float* __restrict__ lw) {
  constexpr int w = 4;
  const int lane = threadIdx.x & 31, ql = lane & 7, grp = lane >> 3;
  const int l = blockIdx.x * (blockDim.x >> 3) + ((threadIdx.x >> 5) << 2) + grp;
  const bool live = l < npts;
  const int lc = live ? l : 0;
  const int mry = G.mr[1], mrx = G.mr[2], fe = mry * mrx;
  const float dyl = d0[3 * lc + 1], dxl = d0[3 * lc + 2];
  // d0 = anchor - point: anchor right of the point -> tap +4 lies outside the support
  const int sx = dxl > 0.f ? 0 : 1, sy = dyl > 0.f ? 0 : 1;
  const float wx = pf_win(G, 2, dxl + (float)(ql - w + sx) * G.h[2]);
  const float wy_own = pf_win(G, 1, dyl + (float)(ql - w + sy) * G.h[1]);
  const int cx = wrap_once(wrap_once(i0[3 * lc + 2] - w + sx, mrx) + ql, mrx);
  const int r0 = wrap_once(i0[3 * lc + 1] - w + sy, mry) * mrx;
  const float2* fplane = fine + (long long)(plane_idx[lc] - plane0) * fine_plane_stride;
  // the point's tail data (lane 0 of its quarter warp) is requested ahead of the gathers,
  // so the position, target index and target value arrive while the stencil is summed
  const bool tail = ql == 0 && live;
  double px = 0.0, py = 0.0, pz = 0.0;
  long long dst = 0;
  float2 old = make_float2(0.f, 0.f);
  if (tail) {
    dst = dst_idx[l];
    if (include_illum) {
      px = xyz[3 * lc];
      py = xyz[3 * lc + 1];
      pz = xyz[3 * lc + 2];
    }
    old = vol[dst];
  }
  float2 tot = make_float2(0.f, 0.f);
  for (int p = 0; p < n_illum; p++) {
    float2 acc = make_float2(0.f, 0.f);
    for (int m = 0; m < nodes; m++) {
      const float2* col = fplane + (long long)m * fine_plane_stride +
                          (long long)p * fine_stride + cx;
      const float wxm = lw ? wx * __ldg(lw + (long long)lc * nodes + m) : wx;
      int ro = r0;
#pragma unroll UNR
      for (int oy = 0; oy < 8; oy++) {
        const float wy = __shfl_sync(0xffffffffu, wy_own, (grp << 3) + oy);
        const float2 f = __ldg(col + ro);
        const float ww = wxm * wy;
        acc.x = fmaf(ww, f.x, acc.x);
        acc.y = fmaf(ww, f.y, acc.y);
        ro += mrx;
        if (ro >= fe) ro -= fe;
      }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    float2 val = cscale(acc, scale);
    if (include_illum && tail) {
      const double ex = px - ill[3 * p], ey = py - ill[3 * p + 1], ez = pz - ill[3 * p + 2];
      val = cmul(val, expi_reduced(PF_TWO_PI * kturns * sqrt(ex * ex + ey * ey + ez * ez)));
    }
    tot = cadd(tot, val);
  }
  if (tail) {
    vol[dst] = cadd(old, cmul(tot, frame_w[0]));   // each target belongs to one point
    for (int f = 1; f < n_frames; f++) {
      float2* d = vol + f * vol_frame_stride + dst;
      *d = cadd(*d, cmul(tot, frame_w[f]));
    }
  }
}

// The node-gathering readout (arbitrary voxel depths) on node-interleaved fine grids: the M
// node grids of a depth slab are stored cell by cell (fine_il[slab][cell][node], written by
// pf_nufft_type2_start_2d_il), so a tap's M node values are 8 M contiguous bytes and a lane
// reads them with 16-byte loads -- every sector fetched is fully used, where the per-grid
// layout fetches a 64-byte row segment (2-3 partly used sectors) per node and row.  Quarter
// warp per voxel as k_interp2_es8 (w = 4, one illumination); the Lagrange-weighted node sum
// of a tap is formed first, then weighted by the stencil.
template <int M>
__global__ void __launch_bounds__(256, 4)
k_interp2_es8_il(pf_nufft_geom G, const int* __restrict__ i0, const float* __restrict__ d0,
                 const double* __restrict__ xyz, const int* __restrict__ plane_idx,
                 const long long* __restrict__ dst_idx, int npts, int plane0,
                 const float2* __restrict__ fine_il, long long slab_stride,
                 const double* __restrict__ ill, double kturns, int include_illum, float scale,
                 const float2* __restrict__ frame_w, int n_frames, float2* __restrict__ vol,
                 long long vol_frame_stride, const float* __restrict__ lw) {
  static_assert(M % 2 == 0, "node pairs are read as float4");
  constexpr int w = 4;
  const int lane = threadIdx.x & 31, ql = lane & 7, grp = lane >> 3;
  const int l = blockIdx.x * (blockDim.x >> 3) + ((threadIdx.x >> 5) << 2) + grp;
  const bool live = l < npts;
  const int lc = live ? l : 0;
  const int mry = G.mr[1], mrx = G.mr[2], fe = mry * mrx;
  const float dyl = d0[3 * lc + 1], dxl = d0[3 * lc + 2];
  const int sx = dxl > 0.f ? 0 : 1, sy = dyl > 0.f ? 0 : 1;
  const float wx = pf_win(G, 2, dxl + (float)(ql - w + sx) * G.h[2]) * scale;
  const float wy_own = pf_win(G, 1, dyl + (float)(ql - w + sy) * G.h[1]);
  const int cx = wrap_once(wrap_once(i0[3 * lc + 2] - w + sx, mrx) + ql, mrx);
  const int r0 = wrap_once(i0[3 * lc + 1] - w + sy, mry) * mrx;
  const float2* base = fine_il + (long long)((plane_idx[lc] - plane0) / M) * slab_stride;
  const bool tail = ql == 0 && live;
  double px = 0.0, py = 0.0, pz = 0.0;
  long long dst = 0;
  float2 old = make_float2(0.f, 0.f);
  if (tail) {
    dst = dst_idx[l];
    if (include_illum) {
      px = xyz[3 * lc];
      py = xyz[3 * lc + 1];
      pz = xyz[3 * lc + 2];
    }
    old = vol[dst];
  }
  // A row of the stencil is 8 columns x M nodes = 8 M contiguous float2.  The quarter warp
  // reads it as NP 128-byte pieces (lane ql takes the 16 bytes at 128 q + 16 ql: one cache
  // line per piece and voxel instead of eight), so lane ql's piece q holds node pair
  // (8 q + ql) % (M / 2) of column (8 q + ql) / (M / 2); its weights are fetched once.
  constexpr int NP = M / 2;                  // 16-byte pieces per lane and row (8 M / 2 / 8)
  float wq[NP];
  float2 lq[NP];
#pragma unroll
  for (int q = 0; q < NP; q++) {
    const int t = 8 * q + ql;
    const int colq = t / NP, pair = t - colq * NP;
    wq[q] = __shfl_sync(0xffffffffu, wx, (grp << 3) + colq);
    lq[q] = __ldg(reinterpret_cast<const float2*>(lw + (long long)lc * M) + pair);
  }
  // the row's first byte: column 0 of the stencil (the columns wrap with the torus: a row
  // whose 8 columns straddle the seam falls back to per-column addresses)
  const int cx0 = wrap_once(i0[3 * lc + 2] - w + sx, mrx);
  const bool straddle = cx0 + 8 > mrx;
  float2 acc = make_float2(0.f, 0.f);
  int ro = r0;
  if (!straddle) {
#pragma unroll 2
    for (int oy = 0; oy < 8; oy++) {
      const float wy = __shfl_sync(0xffffffffu, wy_own, (grp << 3) + oy);
      const float4* p4 = reinterpret_cast<const float4*>(base + (long long)(ro + cx0) * M) + ql;
      float4 v[NP];
#pragma unroll
      for (int q = 0; q < NP; q++) v[q] = __ldg(p4 + 8 * q);
      float sxr = 0.f, syr = 0.f;
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const float a0 = wq[q] * lq[q].x, a1 = wq[q] * lq[q].y;
        sxr = fmaf(a0, v[q].x, sxr);
        syr = fmaf(a0, v[q].y, syr);
        sxr = fmaf(a1, v[q].z, sxr);
        syr = fmaf(a1, v[q].w, syr);
      }
      acc.x = fmaf(wy, sxr, acc.x);
      acc.y = fmaf(wy, syr, acc.y);
      ro += mrx;
      if (ro >= fe) ro -= fe;
    }
  } else {
    for (int oy = 0; oy < 8; oy++) {
      const float wy = __shfl_sync(0xffffffffu, wy_own, (grp << 3) + oy);
      float sxr = 0.f, syr = 0.f;
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const int t = 8 * q + ql;
        const int colq = t / NP, pair = t - colq * NP;
        const int cxq = wrap_once(cx0 + colq, mrx);
        const float4 v =
            __ldg(reinterpret_cast<const float4*>(base + (long long)(ro + cxq) * M) + pair);
        const float a0 = wq[q] * lq[q].x, a1 = wq[q] * lq[q].y;
        sxr = fmaf(a0, v.x, sxr);
        syr = fmaf(a0, v.y, syr);
        sxr = fmaf(a1, v.z, sxr);
        syr = fmaf(a1, v.w, syr);
      }
      acc.x = fmaf(wy, sxr, acc.x);
      acc.y = fmaf(wy, syr, acc.y);
      ro += mrx;
      if (ro >= fe) ro -= fe;
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if (tail) {
    float2 val = acc;
    if (include_illum) {
      const double ex = px - ill[0], ey = py - ill[1], ez = pz - ill[2];
      val = cmul(val, expi_reduced(PF_TWO_PI * kturns * sqrt(ex * ex + ey * ey + ez * ez)));
    }
    vol[dst] = cadd(old, cmul(val, frame_w[0]));
    for (int f = 1; f < n_frames; f++) {
      float2* d = vol + f * vol_frame_stride + dst;
      *d = cadd(*d, cmul(val, frame_w[f]));
    }
  }
}

// The plane readout over all frequencies at once, on frequency-interleaved fine grids
// (fine_f[group][plane][cell][16], written by pf_nufft_type2_start_2d_ilm with il = 16 and
// member = f % 16): a stencil row is 8 columns x 16 frequencies = 1024 contiguous bytes, read
// by the quarter warp as eight 128-byte pieces in which lane ql holds frequencies 2 ql and
// 2 ql + 1 of one column.  Each lane sums the stencil for its two frequencies, applies their
// illumination phases and frame weights (all eight lanes work on phases, where the
// per-frequency kernels use one), and the frequency sum is a shuffle reduction; the voxel's
// indices, weights and target update are formed once instead of once per frequency.
// ES window at w = 4, one illumination, one frame.
__global__ void __launch_bounds__(256, 4)
k_interp2_es8_f16(pf_nufft_geom G, const int* __restrict__ i0, const float* __restrict__ d0,
                  const double* __restrict__ xyz, const int* __restrict__ plane_idx,
                  const long long* __restrict__ dst_idx, int npts, int plane0,
                  const float2* __restrict__ fine_f, long long plane_stride,
                  long long group_stride, int F, const double* __restrict__ kturns_f,
                  const double* __restrict__ ill, int include_illum, float scale,
                  const float2* __restrict__ frame_w, float2* __restrict__ vol) {
  constexpr int w = 4;
  const int lane = threadIdx.x & 31, ql = lane & 7, grp = lane >> 3;
  const int l = blockIdx.x * (blockDim.x >> 3) + ((threadIdx.x >> 5) << 2) + grp;
  const bool live = l < npts;
  const int lc = live ? l : 0;
  const int mry = G.mr[1], mrx = G.mr[2], fe = mry * mrx;
  const float dyl = d0[3 * lc + 1], dxl = d0[3 * lc + 2];
  const int sx = dxl > 0.f ? 0 : 1, sy = dyl > 0.f ? 0 : 1;
  const float wx_own = pf_win(G, 2, dxl + (float)(ql - w + sx) * G.h[2]) * scale;
  const float wy_own = pf_win(G, 1, dyl + (float)(ql - w + sy) * G.h[1]);
  float wxs[8];
#pragma unroll
  for (int q = 0; q < 8; q++) wxs[q] = __shfl_sync(0xffffffffu, wx_own, (grp << 3) + q);
  const int cx0 = wrap_once(i0[3 * lc + 2] - w + sx, mrx);
  const bool straddle = cx0 + 8 > mrx;
  const int r0 = wrap_once(i0[3 * lc + 1] - w + sy, mry) * mrx;
  const float2* base = fine_f + (long long)(plane_idx[lc] - plane0) * plane_stride;
  const bool tail = ql == 0 && live;
  long long dst = 0;
  float2 old = make_float2(0.f, 0.f);
  if (tail) {
    dst = dst_idx[l];
    old = vol[dst];
  }
  double dist = 0.0;
  if (include_illum) {
    const double ex = xyz[3 * lc] - ill[0], ey = xyz[3 * lc + 1] - ill[1];
    const double ez = xyz[3 * lc + 2] - ill[2];
    dist = sqrt(ex * ex + ey * ey + ez * ez);
  }
  float2 tot = make_float2(0.f, 0.f);
  for (int f0 = 0; f0 < F; f0 += 16, base += group_stride) {
    float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
    int ro = r0;
#pragma unroll 2
    for (int oy = 0; oy < 8; oy++) {
      const float wy = __shfl_sync(0xffffffffu, wy_own, (grp << 3) + oy);
      float4 v[8];
      if (!straddle) {
        const float4* p4 = reinterpret_cast<const float4*>(base + (long long)(ro + cx0) * 16) + ql;
#pragma unroll
        for (int q = 0; q < 8; q++) v[q] = __ldg(p4 + 8 * q);
      } else {
#pragma unroll
        for (int q = 0; q < 8; q++)
          v[q] = __ldg(reinterpret_cast<const float4*>(
                           base + (long long)(ro + wrap_once(cx0 + q, mrx)) * 16) + ql);
      }
      float sx0 = 0.f, sy0 = 0.f, sx1 = 0.f, sy1 = 0.f;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        sx0 = fmaf(wxs[q], v[q].x, sx0);
        sy0 = fmaf(wxs[q], v[q].y, sy0);
        sx1 = fmaf(wxs[q], v[q].z, sx1);
        sy1 = fmaf(wxs[q], v[q].w, sy1);
      }
      a0.x = fmaf(wy, sx0, a0.x);
      a0.y = fmaf(wy, sy0, a0.y);
      a1.x = fmaf(wy, sx1, a1.x);
      a1.y = fmaf(wy, sy1, a1.y);
      ro += mrx;
      if (ro >= fe) ro -= fe;
    }
    const int fa = f0 + 2 * ql;
    if (fa < F) {
      float2 val = a0;
      if (include_illum) val = cmul(val, expi_reduced(PF_TWO_PI * kturns_f[fa] * dist));
      tot = cadd(tot, cmul(val, frame_w[fa]));
    }
    if (fa + 1 < F) {
      float2 val = a1;
      if (include_illum) val = cmul(val, expi_reduced(PF_TWO_PI * kturns_f[fa + 1] * dist));
      tot = cadd(tot, cmul(val, frame_w[fa + 1]));
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    tot.x += __shfl_xor_sync(0xffffffffu, tot.x, o);
    tot.y += __shfl_xor_sync(0xffffffffu, tot.y, o);
  }
  if (tail) vol[dst] = cadd(old, tot);
}

// PF_INTERP_H17: 2 (default) the 16 x 16 trimmed kernel for W = 17, 1 the full 17 x 17
// specialisation, 0 the general half-warp kernel (A/B measurements)
int g_interp_mode = -1;
int interp_h17_mode() {
  if (g_interp_mode < 0) {
    const char* e = getenv("PF_INTERP_H17");
    g_interp_mode = e == nullptr ? 2 : atoi(e);
  }
  return g_interp_mode;
}
bool interp_h17_enabled() { return interp_h17_mode() != 0; }
// row-loop unroll of the quarter / half warp readouts (PF_INTERP_UNROLL overrides): 8 rows
// in flight for the many-node gathers, 4 (fewer registers, more resident warps) for the
// single-grid readout -- measured: config 2 20.2 -> 18.9 ms with 4, config 7 51.9 -> 49.5 with 8
int interp_unroll(int nodes = 2) {
  static int u = -1;
  if (u < 0) {
    const char* e = getenv("PF_INTERP_UNROLL");
    u = e ? atoi(e) : 0;
  }
  return u ? u : (nodes > 1 ? 8 : 4);
}
// PF_INTERP_ES8=0 keeps the general kernels for the w = 4 exponential-of-semicircle stencil
bool interp_es8_ok(const pf_nufft_geom& g) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("PF_INTERP_ES8");
    on = (e == nullptr || atoi(e) != 0) ? 1 : 0;
  }
  return on && g.window == 1 && g.w == 4 && (long long)g.mr[1] * g.mr[2] < (1LL << 31);
}
// the far edge tap (8 cells away) must weigh < 2e-8 of the centre tap on both axes
bool interp_trim_ok(const pf_nufft_geom& g) {
  if (interp_h17_mode() != 2) return false;
  for (int a = 1; a <= 2; a++) {
    const float d = 8.0f * g.h[a];
    if (d * d * g.inv4tau[a] < 17.75f) return false;
  }
  return true;
}

extern "C" int pf_nufft_interp2_nodes(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                                      const double* xyz, const int32_t* plane_idx,
                                      const int64_t* dst_idx, int npts, int plane0,
                                      const void* fine, int64_t fine_plane_stride,
                                      int64_t fine_stride, int n_illum, const double* ill,
                                      double khat, int include_illum, float scale,
                                      const void* frame_w, int n_frames, void* vol,
                                      int64_t vol_frame_stride, int nodes, const float* lw,
                                      void* stream);

// w = 16 (W = 33 > 32 lanes): one thread per point.
__global__ void k_interp2_acc(pf_nufft_geom G, const int* __restrict__ i0,
                              const float* __restrict__ d0, const double* __restrict__ xyz,
                              int npts, const float2* __restrict__ fine, long long fine_stride,
                              int n_illum, const double* __restrict__ ill, double kturns,
                              int include_illum, float scale, const float2* __restrict__ frame_w,
                              int n_frames, float2* __restrict__ vol, long long vol_frame_stride,
                              long long dst0, const int* __restrict__ perm) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= npts) return;
  const int W = 2 * G.w + 1;
  const int mry = G.mr[1], mrx = G.mr[2];
  const int cx0 = natural((long long)i0[3 * l + 2] - G.w, mrx);
  int cy = natural((long long)i0[3 * l + 1] - G.w, mry);
  float2 tot = make_float2(0.f, 0.f);
  for (int p = 0; p < n_illum; p++) {
    const float2* fp = fine + (long long)p * fine_stride;
    float2 acc = make_float2(0.f, 0.f);
    int y = cy;
    for (int oy = 0; oy < W; oy++) {
      const float dy = d0[3 * l + 1] + (float)(oy - G.w) * G.h[1];
      const float wy = pf_win(G, 1, dy);
      float2 row = make_float2(0.f, 0.f);
      int x = cx0;
      for (int ox = 0; ox < W; ox++) {
        const float dx = d0[3 * l + 2] + (float)(ox - G.w) * G.h[2];
        const float wx = pf_win(G, 2, dx);
        const float2 f = fp[(long long)y * mrx + x];
        row.x = fmaf(wx, f.x, row.x);
        row.y = fmaf(wx, f.y, row.y);
        if (++x == mrx) x = 0;
      }
      acc.x = fmaf(wy, row.x, acc.x);
      acc.y = fmaf(wy, row.y, acc.y);
      if (++y == mry) y = 0;
    }
    float2 val = cscale(acc, scale);
    if (include_illum) {
      const double ex = xyz[3 * l] - ill[3 * p], ey = xyz[3 * l + 1] - ill[3 * p + 1];
      const double ez = xyz[3 * l + 2] - ill[3 * p + 2];
      val = cmul(val, expi_reduced(PF_TWO_PI * kturns * sqrt(ex * ex + ey * ey + ez * ez)));
    }
    tot = cadd(tot, val);
  }
  const long long lo = perm ? perm[l] : l;
  for (int f = 0; f < n_frames; f++) {
    float2* d = vol + f * vol_frame_stride + dst0 + lo;
    *d = cadd(*d, cmul(tot, frame_w[f]));
  }
}

// Plain type-2 finish for any dimension (spectral.nufft2, reference spectral.py:376-380):
// out[l] = sum over the (2w+1)^dim stencil of fine * prod(axis windows).  One warp per
// point: lane = x tap (W <= 32), loops over the z and y taps (1 for missing axes).
__global__ void __launch_bounds__(256)
k_interp_any(pf_nufft_geom G, const int* __restrict__ i0, const float* __restrict__ d0, int npts,
             const float2* __restrict__ fine, float2* __restrict__ out) {
  const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (l >= npts) return;
  const int W = 2 * G.w + 1;
  const int Wz = G.dim == 3 ? W : 1, Wy = G.dim >= 2 ? W : 1;
  const int mrz = G.mr[0], mry = G.mr[1], mrx = G.mr[2];
  const bool on = lane < W;
  const float dx = d0[3 * l + 2] + (float)(lane - G.w) * G.h[2];
  const float wx = on ? pf_win(G, 2, dx) : 0.f;
  const int cx = wrap_once(natural((long long)i0[3 * l + 2] - G.w, mrx) + (on ? lane : 0), mrx);
  const int cy0 = Wy > 1 ? natural((long long)i0[3 * l + 1] - G.w, mry) : 0;
  int cz = Wz > 1 ? natural((long long)i0[3 * l] - G.w, mrz) : 0;
  float2 acc = make_float2(0.f, 0.f);
  for (int oz = 0; oz < Wz; oz++) {
    float wz = 1.f;
    if (Wz > 1) {
      const float dz = d0[3 * l] + (float)(oz - G.w) * G.h[0];
      wz = pf_win(G, 0, dz);
    }
    int cy = cy0;
    for (int oy = 0; oy < Wy; oy++) {
      float wy = 1.f;
      if (Wy > 1) {
        const float dy = d0[3 * l + 1] + (float)(oy - G.w) * G.h[1];
        wy = pf_win(G, 1, dy);
      }
      const float w = wx * wy * wz;
      const float2 f = __ldg(fine + ((long long)cz * mry + cy) * mrx + cx);
      acc.x = fmaf(w, f.x, acc.x);
      acc.y = fmaf(w, f.y, acc.y);
      if (++cy == mry) cy = 0;
    }
    if (++cz == mrz) cz = 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if (lane == 0) out[l] = acc;
}

int grid1d(long long total) {
  long long g = (total + 255) / 256;
  return (int)(g < 148 * 32 ? (g < 1 ? 1 : g) : 148 * 32);
}

}  // namespace

extern "C" int pf_nufft_spread(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                               const int32_t* tile_start, const int32_t* tile_pts,
                               const void* vals, int64_t val_stride, int nv, void* fine,
                               int64_t fine_stride, void* stream) {
  PF_ARG_CHECK(g && (g->dim == 2 || g->dim == 3) && g->w >= 1 && g->w <= 16 && nv >= 1,
               "pf_nufft_spread: bad geometry");
  PF_ARG_CHECK(g->tile[0] * g->tile[1] * g->tile[2] <= NT, "pf_nufft_spread: tile too large");
  const int ntiles = g->ntiles[0] * g->ntiles[1] * g->ntiles[2];
  if (nv >= 16) {
    k_spread<16><<<dim3(ntiles, pf_cdiv(nv, 16)), NT, 0, (cudaStream_t)stream>>>(
        *g, i0, d0, tile_start, tile_pts, (const float2*)vals, val_stride, nv, (float2*)fine,
        fine_stride);
  } else {
    k_spread<8><<<dim3(ntiles, pf_cdiv(nv, 8)), NT, 0, (cudaStream_t)stream>>>(
        *g, i0, d0, tile_start, tile_pts, (const float2*)vals, val_stride, nv, (float2*)fine,
        fine_stride);
  }
  PF_LAUNCH_CHECK("k_spread");
  return 0;
}

extern "C" int pf_nufft_deconv(const pf_nufft_geom* g, const void* fine, int64_t fine_stride,
                               const float* kz, const float* ky, const float* kx, int nv,
                               void* out, int64_t out_stride, int transpose, void* stream) {
  PF_ARG_CHECK(g && nv >= 1, "pf_nufft_deconv: bad args");
  const long long total = (long long)g->m[0] * g->m[1] * g->m[2] * nv;
  k_deconv_gather<<<grid1d(total), 256, 0, (cudaStream_t)stream>>>(
      *g, (const float2*)fine, fine_stride, kz, ky, kx, nv, (float2*)out, out_stride, transpose);
  PF_LAUNCH_CHECK("k_deconv_gather");
  return 0;
}

extern "C" int pf_nufft_place(const pf_nufft_geom* g, const void* S, int64_t s_stride,
                              const float* kz, const float* ky, const float* kx, int nv,
                              void* fine, int64_t fine_stride, int transpose, void* stream) {
  PF_ARG_CHECK(g && nv >= 1, "pf_nufft_place: bad args");
  const long long total = (long long)g->mr[0] * g->mr[1] * g->mr[2] * nv;
  k_place<<<grid1d(total), 256, 0, (cudaStream_t)stream>>>(*g, (const float2*)S, s_stride, kz, ky,
                                                           kx, nv, (float2*)fine, fine_stride,
                                                           transpose);
  PF_LAUNCH_CHECK("k_place");
  return 0;
}

extern "C" int pf_nufft_interp2_acc(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                                    const double* xyz, int npts, const void* fine,
                                    int64_t fine_stride, int n_illum, const double* ill,
                                    double khat, int include_illum, float scale,
                                    const void* frame_w, int n_frames, void* vol,
                                    int64_t vol_frame_stride, int64_t dst0, const int32_t* perm,
                                    void* stream) {
  PF_ARG_CHECK(g && g->dim == 2 && g->w <= 16 && npts >= 0, "pf_nufft_interp2_acc: bad args");
  if (npts == 0) return 0;
  if (2 * g->w + 1 <= 32) {
    k_interp2_warp<<<pf_cdiv(npts, 8), 256, 0, (cudaStream_t)stream>>>(
        *g, i0, d0, xyz, npts, (const float2*)fine, fine_stride, n_illum, ill, khat / PF_TWO_PI,
        include_illum, scale, (const float2*)frame_w, n_frames, (float2*)vol, vol_frame_stride,
        dst0, perm);
    PF_LAUNCH_CHECK("k_interp2_warp");
    return 0;
  }
  k_interp2_acc<<<pf_cdiv(npts, 128), 128, 0, (cudaStream_t)stream>>>(
      *g, i0, d0, xyz, npts, (const float2*)fine, fine_stride, n_illum, ill, khat / PF_TWO_PI,
      include_illum, scale, (const float2*)frame_w, n_frames, (float2*)vol, vol_frame_stride,
      dst0, perm);
  PF_LAUNCH_CHECK("k_interp2_acc");
  return 0;
}

extern "C" int pf_nufft_interp(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                               int npts, const void* fine, void* out, void* stream) {
  PF_ARG_CHECK(g && g->dim >= 1 && g->dim <= 3 && 2 * g->w + 1 <= 32 && npts >= 0,
               "pf_nufft_interp: bad args (stencil width must be <= 32)");
  if (npts == 0) return 0;
  k_interp_any<<<pf_cdiv(npts, 8), 256, 0, (cudaStream_t)stream>>>(
      *g, i0, d0, npts, (const float2*)fine, (float2*)out);
  PF_LAUNCH_CHECK("k_interp_any");
  return 0;
}

extern "C" int pf_nufft_interp_mode(int mode) {
  const int prev = interp_h17_mode();
  if (mode >= 0 && mode <= 2) g_interp_mode = mode;
  return prev;
}

extern "C" int pf_nufft_interp2_batch(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                                      const double* xyz, const int32_t* plane_idx,
                                      const int64_t* dst_idx, int npts, int plane0,
                                      const void* fine, int64_t fine_plane_stride,
                                      int64_t fine_stride, int n_illum, const double* ill,
                                      double khat, int include_illum, float scale,
                                      const void* frame_w, int n_frames, void* vol,
                                      int64_t vol_frame_stride, void* stream) {
  PF_ARG_CHECK(g && g->dim == 2 && 2 * g->w + 1 <= 32 && npts >= 0,
               "pf_nufft_interp2_batch: bad args (2D, stencil width <= 32)");
  if (npts == 0) return 0;
  static int half = -1;
  if (half < 0) {
    const char* e = getenv("PF_INTERP_HALF");
    half = (e == nullptr || atoi(e) != 0) ? 1 : 0;
  }
  if (interp_es8_ok(*g)) {
    if (interp_unroll(1) == 4)
      k_interp2_es8<4><<<pf_cdiv(npts, 32), 256, 0, (cudaStream_t)stream>>>(
          *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0,
          (const float2*)fine, fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI,
          include_illum, scale, (const float2*)frame_w, n_frames, (float2*)vol,
          vol_frame_stride, 1, nullptr);
    else
      k_interp2_es8<8><<<pf_cdiv(npts, 32), 256, 0, (cudaStream_t)stream>>>(
          *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0,
          (const float2*)fine, fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI,
          include_illum, scale, (const float2*)frame_w, n_frames, (float2*)vol,
          vol_frame_stride, 1, nullptr);
    PF_LAUNCH_CHECK("k_interp2_es8");
    return 0;
  }
  if (half && g->window == 0 && g->w == 8 && (long long)g->mr[1] * g->mr[2] < (1LL << 31) &&
      interp_h17_enabled()) {   // W = 17
    if (interp_trim_ok(*g)) {
      if (interp_unroll() == 8)
        k_interp2_h16<8><<<pf_cdiv(npts, 16), 256, 0, (cudaStream_t)stream>>>(
            *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0,
            (const float2*)fine, fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI,
            include_illum, scale, (const float2*)frame_w, n_frames, (float2*)vol,
            vol_frame_stride, 1, nullptr);
      else
        k_interp2_h16<4><<<pf_cdiv(npts, 16), 256, 0, (cudaStream_t)stream>>>(
            *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0,
            (const float2*)fine, fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI,
            include_illum, scale, (const float2*)frame_w, n_frames, (float2*)vol,
            vol_frame_stride, 1, nullptr);
      PF_LAUNCH_CHECK("k_interp2_h16");
      return 0;
    }
    k_interp2_h17<<<pf_cdiv(npts, 16), 256, 0, (cudaStream_t)stream>>>(
        *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0, (const float2*)fine,
        fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI, include_illum, scale,
        (const float2*)frame_w, n_frames, (float2*)vol, vol_frame_stride, 1, nullptr);
    PF_LAUNCH_CHECK("k_interp2_h17");
    return 0;
  }
  if (half) {   // two points per warp (half a warp each)
    k_interp2_batch_h<<<pf_cdiv(npts, 16), 256, 0, (cudaStream_t)stream>>>(
        *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0, (const float2*)fine,
        fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI, include_illum, scale,
        (const float2*)frame_w, n_frames, (float2*)vol, vol_frame_stride);
    PF_LAUNCH_CHECK("k_interp2_batch_h");
    return 0;
  }
  k_interp2_batch<<<pf_cdiv(npts, 8), 256, 0, (cudaStream_t)stream>>>(
      *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0, (const float2*)fine,
      fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI, include_illum, scale,
      (const float2*)frame_w, n_frames, (float2*)vol, vol_frame_stride);
  PF_LAUNCH_CHECK("k_interp2_batch");
  return 0;
}

extern "C" int pf_nufft_interp2_nodes(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                                      const double* xyz, const int32_t* plane_idx,
                                      const int64_t* dst_idx, int npts, int plane0,
                                      const void* fine, int64_t fine_plane_stride,
                                      int64_t fine_stride, int n_illum, const double* ill,
                                      double khat, int include_illum, float scale,
                                      const void* frame_w, int n_frames, void* vol,
                                      int64_t vol_frame_stride, int nodes, const float* lw,
                                      void* stream) {
  PF_ARG_CHECK(g && g->dim == 2 && 2 * g->w + 1 <= 32 && npts >= 0 && nodes >= 1 &&
                   (nodes == 1 || lw != nullptr),
               "pf_nufft_interp2_nodes: bad args (2D, stencil width <= 32, weights for nodes > 1)");
  if (npts == 0) return 0;
  if (interp_es8_ok(*g)) {
    if (interp_unroll(nodes) == 4)
      k_interp2_es8<4><<<pf_cdiv(npts, 32), 256, 0, (cudaStream_t)stream>>>(
          *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0,
          (const float2*)fine, fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI,
          include_illum, scale, (const float2*)frame_w, n_frames, (float2*)vol,
          vol_frame_stride, nodes, lw);
    else
      k_interp2_es8<8><<<pf_cdiv(npts, 32), 256, 0, (cudaStream_t)stream>>>(
          *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0,
          (const float2*)fine, fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI,
          include_illum, scale, (const float2*)frame_w, n_frames, (float2*)vol,
          vol_frame_stride, nodes, lw);
    PF_LAUNCH_CHECK("k_interp2_es8");
    return 0;
  }
  if (g->window == 0 && g->w == 8 && (long long)g->mr[1] * g->mr[2] < (1LL << 31) &&
      interp_h17_enabled()) {
    if (interp_trim_ok(*g)) {
      if (interp_unroll() == 8)
        k_interp2_h16<8><<<pf_cdiv(npts, 16), 256, 0, (cudaStream_t)stream>>>(
            *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0,
            (const float2*)fine, fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI,
            include_illum, scale, (const float2*)frame_w, n_frames, (float2*)vol,
            vol_frame_stride, nodes, lw);
      else
        k_interp2_h16<4><<<pf_cdiv(npts, 16), 256, 0, (cudaStream_t)stream>>>(
            *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0,
            (const float2*)fine, fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI,
            include_illum, scale, (const float2*)frame_w, n_frames, (float2*)vol,
            vol_frame_stride, nodes, lw);
      PF_LAUNCH_CHECK("k_interp2_h16");
      return 0;
    }
    k_interp2_h17<<<pf_cdiv(npts, 16), 256, 0, (cudaStream_t)stream>>>(
        *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0, (const float2*)fine,
        fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI, include_illum, scale,
        (const float2*)frame_w, n_frames, (float2*)vol, vol_frame_stride, nodes, lw);
    PF_LAUNCH_CHECK("k_interp2_h17");
    return 0;
  }
  k_interp2_batch_h<<<pf_cdiv(npts, 16), 256, 0, (cudaStream_t)stream>>>(
      *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0, (const float2*)fine,
      fine_plane_stride, fine_stride, n_illum, ill, khat / PF_TWO_PI, include_illum, scale,
      (const float2*)frame_w, n_frames, (float2*)vol, vol_frame_stride, nodes, lw);
  PF_LAUNCH_CHECK("k_interp2_nodes");
  return 0;
}

// Node-gathering readout on node-interleaved fine grids (pf_nufft_type2_start_2d_il with
// il = nodes): fine_il[slab][cell][node], slab s of the batch at fine_il + s * slab_stride.
// ES window at w = 4, 12 nodes, one illumination; other cases: pf_nufft_interp2_nodes.
extern "C" int pf_nufft_interp2_nodes_il(const pf_nufft_geom* g, const int32_t* i0,
                                         const float* d0, const double* xyz,
                                         const int32_t* plane_idx, const int64_t* dst_idx,
                                         int npts, int plane0, const void* fine_il,
                                         int64_t slab_stride, const double* ill, double khat,
                                         int include_illum, float scale, const void* frame_w,
                                         int n_frames, void* vol, int64_t vol_frame_stride,
                                         int nodes, const float* lw, void* stream) {
  PF_ARG_CHECK(g && g->dim == 2 && g->window == 1 && g->w == 4 && nodes == 12 && lw && npts >= 0 &&
                   (long long)g->mr[1] * g->mr[2] * nodes < (1LL << 31),
               "pf_nufft_interp2_nodes_il: needs the ES window at w = 4 and 12 nodes");
  if (npts == 0) return 0;
  k_interp2_es8_il<12><<<pf_cdiv(npts, 32), 256, 0, (cudaStream_t)stream>>>(
      *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0, (const float2*)fine_il,
      slab_stride, ill, khat / PF_TWO_PI, include_illum, scale, (const float2*)frame_w, n_frames,
      (float2*)vol, vol_frame_stride, lw);
  PF_LAUNCH_CHECK("k_interp2_es8_il");
  return 0;
}

// Plane readout over all frequencies in one launch on frequency-interleaved fine grids:
// fine_f[group][plane][cell][16] (group g = frequencies 16 g .. 16 g + 15; plane p of the
// batch at + p * plane_stride, group g at + g * group_stride; slots of frequencies >= F must
// be zero).  kturns_f [F] = k_f / (2 pi) (device), frame_w [F].  ES window at w = 4, one
// illumination, one frame.
extern "C" int pf_nufft_interp2_freqs(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                                      const double* xyz, const int32_t* plane_idx,
                                      const int64_t* dst_idx, int npts, int plane0,
                                      const void* fine_f, int64_t plane_stride,
                                      int64_t group_stride, int n_freq, const double* kturns_f,
                                      const double* ill, int include_illum, float scale,
                                      const void* frame_w, void* vol, void* stream) {
  PF_ARG_CHECK(g && g->dim == 2 && g->window == 1 && g->w == 4 && n_freq >= 1 && npts >= 0 &&
                   kturns_f && frame_w && (long long)g->mr[1] * g->mr[2] * 16 < (1LL << 31),
               "pf_nufft_interp2_freqs: needs the ES window at w = 4");
  if (npts == 0) return 0;
  k_interp2_es8_f16<<<pf_cdiv(npts, 32), 256, 0, (cudaStream_t)stream>>>(
      *g, i0, d0, xyz, plane_idx, (const long long*)dst_idx, npts, plane0, (const float2*)fine_f,
      plane_stride, group_stride, n_freq, kturns_f, ill, include_illum, scale,
      (const float2*)frame_w, (float2*)vol);
  PF_LAUNCH_CHECK("k_interp2_es8_f16");
  return 0;
}
