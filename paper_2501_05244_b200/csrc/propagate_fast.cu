// Register-FFT propagation path for square power-of-two pads P = 32 L
// (L = 4..32: P = 128 .. 1024; configs 0, 3 and 4).
//
// Same math as propagate.cu (reference rsd reconstruct.py:254-266 and its
// siblings), restructured around warp_fft.cuh so each 1D transform lives in
// registers (one shared-memory exchange per transform) and every global
// access is a contiguous run:
//   (A) line = kernel row jy in [0, P/2]: synthesise G, x-FFT, keep kx <= P/2,
//       stage through shared memory, store transposed  At[plane][kx][jy].
//   (B) line = (plane, kx):  read At row (mirrored to P), y-FFT -> Ghat column;
//       for each illumination and each of the columns kx, P-kx: * Uhat^T row,
//       y-IFFT, store the cropped rows to Tt[plane][p][col][i] (contiguous i).
//   (C) tile of output rows i: load Tt[.][.][col][i0..i0+R) (contiguous runs),
//       transpose in shared memory, x-IFFT per row, crop, illumination phase,
//       sum illuminations, accumulate frames into the volume.
// Uhat is consumed TRANSPOSED (Uhat^T[col][jy]) on this path; the host asks
// pf_prop_fast() before building it.
#include <stdlib.h>

#include "prop_stages.cuh"

namespace {

constexpr int FT = 256;  // 8 warps

// Frequency batching (small configs): blockIdx.z indexes the frequency; per-f
// kernel wavenumbers (turns/m) and per-f workspace / spectrum strides.
struct FBatch {
  const double* kturns;   // nullptr: single frequency (scalar argument)
  long long ws_a_fs, ws_b_fs, uhat_fs;
  int nf;
};

// A for every plane of a batch (blockIdx.y) and, batched, every frequency (blockIdx.z).
template <int L>
__global__ void __launch_bounds__(FT, 2)
k_pa(const pf_plane* __restrict__ planes, double kturns_s, pf_prop_geom g,
     const float2* __restrict__ tw, float2* __restrict__ ws_a, FBatch fb) {
  extern __shared__ float2 sm[];
  constexpr int NA = 32 * L / 2 + 1;
  const double kturns = fb.kturns ? fb.kturns[blockIdx.z] : kturns_s;
  st_a<L>(sm, planes[blockIdx.y], kturns, tw,
          ws_a + blockIdx.z * fb.ws_a_fs + (long long)blockIdx.y * NA * NA, blockIdx.x);
}

// C for every plane of a batch (blockIdx.y).  MULTI: more than one illumination
// (summed in registers first).  PRE: single frame, the CTA's volume rows prefetched
// with cp.async at entry so the accumulate is load-free at the end.
template <int L, bool MULTI, bool PRE, bool CENT>
__global__ void __launch_bounds__(FT, MULTI ? 1 : 2)
k_pc(const pf_plane* __restrict__ planes, double kturns, pf_prop_geom g,
     const float2* __restrict__ tw, const float2* __restrict__ ws_b,
     const double* __restrict__ ill, const float2* __restrict__ frame_w, int n_frames,
     float2* __restrict__ vol, long long vol_frame_stride) {
  extern __shared__ float2 sm[];
  const long long wb_plane = (long long)g.n_illum * 32 * L * g.ny;
  st_c<L, MULTI, PRE, CENT>(sm, planes[blockIdx.y], kturns, g, tw, ws_b + blockIdx.y * wb_plane, ill,
                      frame_w, n_frames, vol, vol_frame_stride, blockIdx.x);
}

// C with the illumination phase by Horner's rule over descending frequencies (st_c HOR)
template <int L, int HOR>
__global__ void __launch_bounds__(FT, 2)
k_pc_h(const pf_plane* __restrict__ planes, double kturns, float dturns, pf_prop_geom g,
       const float2* __restrict__ tw, const float2* __restrict__ ws_b,
       const double* __restrict__ ill, const float2* __restrict__ frame_w,
       float2* __restrict__ vol, float2* __restrict__ ws_o, double zturns,
       float2* __restrict__ vol_out) {
  extern __shared__ float2 sm[];
  const long long wb_plane = 32LL * L * g.ny;
  st_c<L, false, true, true, HOR>(sm, planes[blockIdx.y], kturns, g, tw,
                                  ws_b + blockIdx.y * wb_plane, ill, frame_w, 1, vol, 0,
                                  blockIdx.x, dturns, ws_o, zturns, vol_out);
  if ((HOR == 2 || HOR == 4) && vol_out) __threadfence_system();
}

// ---- B split in two register-light kernels (128 registers, 16 warps/SM):
// B1: in place on ws_a, each line = one At row (plane b, kx): mirror, y-FFT,
//     keep ky <= P/2  ->  Ghat quadrant Gq[b][kx][ky] (Ghat is even in ky too).
// B2: line = (plane b, side): Gq row (mirrored) * Uhat^T column, y-IFFT, crop.
template <int L>
__global__ void __launch_bounds__(FT, 2)
k_pb1(int nplanes, const float2* __restrict__ tw, float2* __restrict__ ws_a, FBatch fb) {
  extern __shared__ float2 sm[];
  constexpr int NA = 32 * L / 2 + 1;
  st_b1<L>(sm, tw, ws_a + blockIdx.z * fb.ws_a_fs + (long long)blockIdx.y * NA * NA, blockIdx.x);
}

template <int L, bool MULTI, bool CENT>
__global__ void __launch_bounds__(FT, 2)
k_pb2(const pf_plane* __restrict__ planes, int nplanes, pf_prop_geom g,
      const float2* __restrict__ tw, const float2* __restrict__ ws_a,
      const float2* __restrict__ uhat_t, float2* __restrict__ ws_b, FBatch fb) {
  ws_a += blockIdx.z * fb.ws_a_fs;
  uhat_t += blockIdx.z * fb.uhat_fs;
  ws_b += blockIdx.z * fb.ws_b_fs;
  constexpr int P = 32 * L, H = P / 2, NA = H + 1;
  constexpr int LPW = 32 / L;
  extern __shared__ float2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int kx = blockIdx.x;
  const int li = (blockIdx.y * 8 + warp) * LPW + line;
  const int b = li >> 1, side = li & 1;
  const int col = side == 0 ? kx : (P - kx) % P;
  const bool active = b < nplanes && !(side == 1 && col == kx);
  const int bb = b < nplanes ? b : nplanes - 1;
  const pf_plane pl = planes[bb];
  const float2* grow = ws_a + ((long long)bb * NA + kx) * NA;
  const int ny = g.ny;
  const int n_ill = MULTI ? g.n_illum : 1;
  // crop offset and height multiples of L: row i = t + base(m), kept iff base(m) < ny
  const bool aligned = ((g.nu0y | ny) & (L - 1)) == 0;
#pragma unroll 1
  for (int p = 0; p < n_ill; p++) {
    const float2* ucol = uhat_t + pl.uhat_off + (long long)p * g.uhat_illum_stride +
                         (long long)col * P;
    float2 w[32];
#pragma unroll
    for (int m = 0; m < 32; m++) {
      const int ky = t + L * m;
      // mirrored row: ky <= P/2 exactly for m < 16 (m = 16 only at t = 0, where
      // P - ky = ky), so the index form is fixed per unrolled m
      w[m] = cmul(__ldg(m < 16 ? grow + ky : grow + (P - ky)), __ldg(ucol + ky));
    }
    wfft<L, 1>(w, sm + warp * WFFT_XCH, tw);
    if (active) {
      float2* dcol = ws_b + ((long long)bb * g.n_illum + p) * (long long)P * ny + (long long)col * ny;
      if (CENT) {      // centred crop: kept rows t + L ((m + 8) mod 32), compile time
        float2* dt = dcol + t;
#pragma unroll
        for (int m = 0; m < 32; m++)
          if (cent_keep(m)) dt[L * cent_base(m)] = w[m];
      } else if (aligned) {   // crop decided per m for the whole warp: no per-lane index math
        float2* dt = dcol + t;
#pragma unroll
        for (int m = 0; m < 32; m++) {
          const int base = (L * m - g.nu0y) & (P - 1);
          if (base < ny) dt[base] = w[m];
        }
      } else {
#pragma unroll
        for (int m = 0; m < 32; m++) {
          const int i = (t + L * m - g.nu0y) & (P - 1);
          if (i < ny) dcol[i] = w[m];
        }
      }
    }
  }
}

// B1 and B2 fused: line = (plane b, kx) of the kernel quadrant.  The mirrored At row is
// y-transformed to the Ghat column kx (even in ky: lanes keep the ky <= P/2 outputs and
// take the rest from the mirror lane by shuffle), then for each illumination and each of
// the output columns kx and P - kx it is multiplied by the Uhat^T column, y-inverted and
// stored row-cropped to Tt.  The Ghat quadrant never leaves the SM (B1's in-place
// quadrant write and B2's two mirrored reads of it are gone, and so is one launch).
// CTA lines: pbc planes x (NL / pbc) consecutive kx, so the lines of one kx (same Uhat^T
// columns) run in the same CTA.
template <int L, bool MULTI, bool CENT>
__global__ void __launch_bounds__(FT, 2)
k_pb12(const pf_plane* __restrict__ planes, int nplanes, int pbc, pf_prop_geom g,
       const float2* __restrict__ tw, const float2* __restrict__ ws_a,
       const float2* __restrict__ uhat_t, float2* __restrict__ ws_b, FBatch fb) {
  ws_a += blockIdx.z * fb.ws_a_fs;
  uhat_t += blockIdx.z * fb.uhat_fs;
  ws_b += blockIdx.z * fb.ws_b_fs;
  constexpr int P = 32 * L, H = P / 2, NA = H + 1;
  constexpr int LPW = 32 / L, NL = 8 * LPW;
  extern __shared__ float2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int li = warp * LPW + line;
  const int kxc = NL / pbc;
  const int bl = li % pbc, kxl = li / pbc;
  const int b = blockIdx.y * pbc + bl;
  const int kx_raw = blockIdx.x * kxc + kxl;
  const bool valid = b < nplanes && kxl < kxc && kx_raw < NA;
  const int bb = b < nplanes ? b : nplanes - 1;
  const int kx = kx_raw < H ? kx_raw : H;
  const pf_plane pl = planes[bb];
  float2 gq[17];   // Ghat[t + L m], m <= 16 (ky <= P/2 for m < 16, and m = 16 at t = 0)
  {
    const float2* arow = ws_a + ((long long)bb * NA + kx) * NA;
    float2 v[32];
#pragma unroll
    for (int m = 0; m < 32; m++) {
      const int jy = t + L * m;
      v[m] = __ldg(m < 16 ? arow + jy : arow + (P - jy));
    }
    wfft<L, -1>(v, sm + warp * WFFT_XCH, tw);
#pragma unroll
    for (int m = 0; m <= 16; m++) gq[m] = v[m];
  }
  // Ghat[t + L m] for m > 16 = Ghat[P - t - L m] = lane (L - t)'s gq[31 - m] (t > 0), or
  // this lane's gq[32 - m] (t = 0)
  const int mirror = (lane - t) + ((L - t) & (L - 1));
  const int ny = g.ny;
  const int n_ill = MULTI ? g.n_illum : 1;
  const bool aligned = ((g.nu0y | ny) & (L - 1)) == 0;
#pragma unroll 1
  for (int p = 0; p < n_ill; p++) {
#pragma unroll 1
    for (int side = 0; side < 2; side++) {
      const int col = side == 0 ? kx : (P - kx) & (P - 1);
      if (LPW == 1 && side == 1 && col == kx) break;   // warp-uniform (one line per warp)
      const bool active = valid && !(side == 1 && col == kx);
      const float2* ucol = uhat_t + pl.uhat_off + (long long)p * g.uhat_illum_stride +
                           (long long)col * P;
      float2 w[32];
#pragma unroll
      for (int m = 0; m < 32; m++) {
        float2 gm;
        if (m <= 16) {
          gm = gq[m];
        } else {
          const float2 o = make_float2(__shfl_sync(0xffffffffu, gq[31 - m].x, mirror),
                                       __shfl_sync(0xffffffffu, gq[31 - m].y, mirror));
          gm = t == 0 ? gq[32 - m] : o;
        }
        w[m] = cmul(gm, __ldg(ucol + t + L * m));
      }
      wfft<L, 1>(w, sm + warp * WFFT_XCH, tw);
      if (active) {
        float2* dcol = ws_b + ((long long)bb * g.n_illum + p) * (long long)P * ny +
                       (long long)col * ny;
        if (CENT) {
          float2* dt = dcol + t;
#pragma unroll
          for (int m = 0; m < 32; m++)
            if (cent_keep(m)) dt[L * cent_base(m)] = w[m];
        } else if (aligned) {
          float2* dt = dcol + t;
#pragma unroll
          for (int m = 0; m < 32; m++) {
            const int base = (L * m - g.nu0y) & (P - 1);
            if (base < ny) dt[base] = w[m];
          }
        } else {
#pragma unroll
          for (int m = 0; m < 32; m++) {
            const int i = (t + L * m - g.nu0y) & (P - 1);
            if (i < ny) dcol[i] = w[m];
          }
        }
      }
    }
  }
}

static bool b12_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("PF_B12");
    on = (e == nullptr || atoi(e) != 0) ? 1 : 0;
  }
  return on == 1;
}

// C over all frequencies of the batch in one launch: per (plane, row tile) the
// ascending-frequency sum is formed in registers and written once.
// NW warps per CTA (RPC = NW * 32/L rows): small volumes (config 0: 64 planes x
// 64 rows) take fewer rows per CTA so the grid still covers the SMs.  The
// (frequency, illumination) tiles are double-buffered: the cp.async load of the
// next tile is in flight while the current one is transformed.
template <int L, bool MULTI, int NW = 8>
__global__ void __launch_bounds__(32 * NW, 1)
k_pcf(const pf_plane* __restrict__ planes, pf_prop_geom g, const float2* __restrict__ tw,
      const float2* __restrict__ ws_b, const double* __restrict__ ill,
      const float2* __restrict__ frame_w, float2* __restrict__ vol, FBatch fb,
      float2* __restrict__ part) {
  constexpr int P = 32 * L;
  constexpr int LPW = 32 / L, RPC = NW * LPW, SLD = RPC + 1, TILE = P * SLD;
  extern __shared__ float2 sm[];
  float2* xch = sm + 2 * TILE;   // per-warp FFT exchange, disjoint from the two tiles
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int r = warp * LPW + line;
  const int ny = g.ny, nx = g.nx;
  const int i0 = blockIdx.x * RPC;
  const int i = i0 + r;
  const int nr = min(RPC, ny - i0);
  const pf_plane pl = planes[blockIdx.y];
  const float scale = 1.0f / ((float)P * (float)P);
  const double yv = pl.y0 + pl.dy * i;
  const int n_ill = MULTI ? g.n_illum : 1;
  // frequency group blockIdx.z of gridDim.z (part != nullptr: partial sums)
  const int f_lo = (int)((long long)blockIdx.z * fb.nf / gridDim.z);
  const int f_hi = (int)((long long)(blockIdx.z + 1) * fb.nf / gridDim.z);
  const int n_tiles = (f_hi - f_lo) * n_ill;
  // full tile of an even-height crop at even offsets: 16-byte copies (see load_tile)
  const bool pairs = nr == RPC && (ny & 1) == 0 && (fb.ws_b_fs & 1) == 0;
  const int sh = pairs ? (t & 1) : 0;   // (t + L m) & 1 == t & 1 (L even)
  auto load_tile = [&](int idx, float2* dst) {
    const int f = f_lo + idx / n_ill, p = idx % n_ill;
    const float2* src = ws_b + f * fb.ws_b_fs +
                        ((long long)blockIdx.y * g.n_illum + p) * (long long)P * ny + i0;
    if (pairs) {
      // 16-byte row pairs; odd columns sit one slot later in the padded tile so both
      // sides stay 16-byte aligned (the reads below add the same offset)
      constexpr int PSTEP = 32 * NW / (RPC / 2);
      const int pr = threadIdx.x % (RPC / 2), c0p = threadIdx.x / (RPC / 2);
      const float4* q = reinterpret_cast<const float4*>(src + (long long)c0p * ny + 2 * pr);
      float4* d = reinterpret_cast<float4*>(dst + c0p * SLD + (c0p & 1) + 2 * pr);
#pragma unroll 8
      for (int col = c0p; col < P; col += PSTEP) {
        cp_async16(d, q);
        q += (long long)PSTEP * ny / 2;
        d += PSTEP * SLD / 2;
      }
    } else {
      constexpr int CSTEP = 32 * NW / RPC;
      const int rr = threadIdx.x % RPC, c0 = threadIdx.x / RPC;
      if (rr < nr) {
        const float2* q = src + (long long)c0 * ny + rr;
        float2* d = dst + c0 * SLD + rr;
#pragma unroll 8
        for (int col = c0; col < P; col += CSTEP) {
          cp_async8(d, q);
          q += (long long)CSTEP * ny;
          d += CSTEP * SLD;
        }
      }
    }
    cp_async_commit();
  };
  float2 acc[32];
#pragma unroll
  for (int m = 0; m < 32; m++) acc[m] = make_float2(0.f, 0.f);
  load_tile(0, sm);
#pragma unroll 1
  for (int idx = 0; idx < n_tiles; idx++) {
    const int f = f_lo + idx / n_ill, p = idx % n_ill;
    float2* cur = sm + (idx & 1) * TILE;
    if (idx + 1 < n_tiles) {
      load_tile(idx + 1, sm + ((idx + 1) & 1) * TILE);
      cp_async_wait_1();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    float2 v[32];
#pragma unroll
    for (int m = 0; m < 32; m++) v[m] = cur[(t + L * m) * SLD + sh + r];
    __syncthreads();   // the tile is refilled by the load issued in the next iteration
    wfft<L, 1>(v, xch + warp * WFFT_XCH, tw);
    const double kturns = fb.kturns[f];
    const float2 fw = frame_w[f];
    const double sx = ill[3 * p], sy = ill[3 * p + 1], sz = ill[3 * p + 2];
    const double dy = yv - sy, dz = pl.z - sz;
    const double byz = fma(dy, dy, dz * dz);
#pragma unroll
    for (int m = 0; m < 32; m++) {
      const int mo = (t + L * m - g.nu0x) & (P - 1);
      float2 val = cscale(v[m], scale);
      if (g.include_illum && mo < nx) {
        const double dx = pl.x0 + pl.dx * mo - sx;
        val = cmul(val, phase_turns(fma(dx, dx, byz), kturns, (float)kturns));
      }
      acc[m] = cadd(acc[m], cmul(val, fw));
    }
  }
  if (i < ny) {
    if (part) {
      float2* prow = part + (((long long)blockIdx.z * gridDim.y + blockIdx.y) * ny + i) * nx;
#pragma unroll
      for (int m = 0; m < 32; m++) {
        const int mo = (t + L * m - g.nu0x) & (P - 1);
        if (mo < nx) prow[mo] = acc[m];
      }
      return;
    }
    float2* drow = vol + (pl.vol_plane * ny + i) * (long long)nx;
#pragma unroll
    for (int m = 0; m < 32; m++) {
      const int mo = (t + L * m - g.nu0x) & (P - 1);
      if (mo < nx) drow[mo] = cadd(drow[mo], acc[m]);
    }
  }
}

// vol[plane] += sum over groups z (ascending) of part[z][plane]
__global__ void k_pcf_sum(const pf_plane* __restrict__ planes, int nplanes, int ny, int nx,
                          const float2* __restrict__ part, int groups, float2* __restrict__ vol) {
  const long long per = (long long)ny * nx, total = per * nplanes;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e / per);
    const long long o = e - b * per;
    float2 s = part[e];
    for (int z = 1; z < groups; z++) s = cadd(s, part[z * total + e]);
    float2* d = vol + planes[b].vol_plane * per + o;
    *d = cadd(*d, s);
  }
}

template <int L, int NW = 8>
size_t smem_a() {
  constexpr int P = 32 * L, NA = P / 2 + 1, RPC = NW * (32 / L);
  size_t x = NW * WFFT_XCH, s = (size_t)NA * (RPC + 1);
  return (x > s ? x : s) * sizeof(float2);
}
// k_pcf: two tiles + the per-warp exchange buffers
template <int L, int NW = 8>
size_t smem_cf() {
  constexpr int P = 32 * L, RPC = NW * (32 / L);
  return ((size_t)2 * P * (RPC + 1) + (size_t)NW * WFFT_XCH) * sizeof(float2);
}
template <int L, int NW = 8>
size_t smem_c(int nx, bool pre) {
  constexpr int P = 32 * L, RPC = NW * (32 / L);
  size_t x = NW * WFFT_XCH, s = (size_t)P * (RPC + 1);
  return ((x > s ? x : s) + (pre ? (size_t)RPC * nx : 0)) * sizeof(float2);
}

template <int L>
int run_stage(int stage, const pf_plane* planes, int nplanes, double khat, const pf_prop_geom& g,
              const float2* tw, const float2* ws_a, float2* ws_a_out, const float2* uhat,
              const float2* ws_b, float2* ws_b_out, const double* ill, const float2* frame_w,
              int n_frames, float2* vol, long long vfs, cudaStream_t st,
              FBatch fb = FBatch{nullptr, 0, 0, 0, 1}) {
  constexpr int NA = 32 * L / 2 + 1, RPC = 8 * (32 / L), LPW = 32 / L;
  static PfDevOnce attr;  
  if (attr.first()) {
    const int big = 200 * 1024;
    cudaFuncSetAttribute(k_pa<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_pb1<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_pb2<L, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_pb2<L, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_pb2<L, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_pb2<L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_pb12<L, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_pb12<L, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_pb12<L, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_pb12<L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
#define PF_PC_ATTR(M, PR, C) \
    cudaFuncSetAttribute(k_pc<L, M, PR, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    PF_PC_ATTR(false, false, false) PF_PC_ATTR(true, false, false)
    PF_PC_ATTR(false, true, false) PF_PC_ATTR(true, true, false)
    PF_PC_ATTR(false, false, true) PF_PC_ATTR(true, false, true)
    PF_PC_ATTR(false, true, true) PF_PC_ATTR(true, true, true)
#undef PF_PC_ATTR
    const int most = 227 * 1024;   // k_pcf at P = 1024 with 8 warps: 215 KB
    cudaFuncSetAttribute(k_pcf<L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
    cudaFuncSetAttribute(k_pcf<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
    cudaFuncSetAttribute(k_pcf<L, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
    cudaFuncSetAttribute(k_pcf<L, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
  }
  const double kturns = khat / PF_TWO_PI;
  if (stage == 0) {   // A: kernel rows -> At
    dim3 grid(pf_cdiv(NA, RPC), nplanes, fb.nf);
    k_pa<L><<<grid, FT, smem_a<L>(), st>>>(planes, kturns, g, tw, ws_a_out, fb);
    PF_LAUNCH_CHECK("k_pa");
  } else if (stage == 1) {   // B1 (Ghat quadrant in place) + B2 (product, y-IFFT, crop)
    const size_t sm = 8 * WFFT_XCH * sizeof(float2);
    const bool cent_y = 2 * g.ny == 32 * L && 2 * g.nu0y == -g.ny;
    if (b12_enabled()) {   // B1 + B2 fused
      const int pbc = nplanes < 8 * LPW ? nplanes : 8 * LPW;
      dim3 g12(pf_cdiv(NA, (8 * LPW) / pbc), pf_cdiv(nplanes, pbc), fb.nf);
      if (g.n_illum > 1) {
        if (cent_y) k_pb12<L, true, true><<<g12, FT, sm, st>>>(planes, nplanes, pbc, g, tw, ws_a, uhat, ws_b_out, fb);
        else k_pb12<L, true, false><<<g12, FT, sm, st>>>(planes, nplanes, pbc, g, tw, ws_a, uhat, ws_b_out, fb);
      } else {
        if (cent_y) k_pb12<L, false, true><<<g12, FT, sm, st>>>(planes, nplanes, pbc, g, tw, ws_a, uhat, ws_b_out, fb);
        else k_pb12<L, false, false><<<g12, FT, sm, st>>>(planes, nplanes, pbc, g, tw, ws_a, uhat, ws_b_out, fb);
      }
      PF_LAUNCH_CHECK("k_pb12");
      return 0;
    }
    dim3 g1(pf_cdiv(NA, 8 * LPW), nplanes, fb.nf);
    k_pb1<L><<<g1, FT, sm, st>>>(nplanes, tw, const_cast<float2*>(ws_a), fb);
    PF_LAUNCH_CHECK("k_pb1");
    dim3 g2(NA, pf_cdiv(2 * nplanes, 8 * LPW), fb.nf);
    // centred row crop (output lattice = relay lattice): compile-time kept rows
    if (g.n_illum > 1) {
      if (cent_y) k_pb2<L, true, true><<<g2, FT, sm, st>>>(planes, nplanes, g, tw, ws_a, uhat, ws_b_out, fb);
      else k_pb2<L, true, false><<<g2, FT, sm, st>>>(planes, nplanes, g, tw, ws_a, uhat, ws_b_out, fb);
    } else {
      if (cent_y) k_pb2<L, false, true><<<g2, FT, sm, st>>>(planes, nplanes, g, tw, ws_a, uhat, ws_b_out, fb);
      else k_pb2<L, false, false><<<g2, FT, sm, st>>>(planes, nplanes, g, tw, ws_a, uhat, ws_b_out, fb);
    }
    PF_LAUNCH_CHECK("k_pb2");
  } else if (fb.kturns != nullptr) {   // C over all frequencies of the batch
    // 8 warps per CTA unless that leaves fewer than two CTAs per SM; then 2
    const bool narrow = (long long)pf_cdiv(g.ny, RPC) * nplanes < 2LL * pf_sm_count();
    if (narrow) {
      constexpr int RPC2 = 2 * (32 / L);
      // few (plane, row tile) CTAs: split the frequencies into groups whose partial
      // sums go to the (now free) kernel-spectrum workspace, then add them in order
      const long long ctas = (long long)pf_cdiv(g.ny, RPC2) * nplanes;
      int groups = (int)((8LL * pf_sm_count() + ctas - 1) / ctas);
      if (groups > fb.nf) groups = fb.nf;
      if (groups > 8) groups = 8;
      const long long need = (long long)groups * nplanes * g.ny * g.nx;
      if (groups < 2 || need > (long long)fb.nf * fb.ws_a_fs) groups = 1;
      float2* part = groups > 1 ? const_cast<float2*>(ws_a) : nullptr;
      dim3 grid(pf_cdiv(g.ny, RPC2), nplanes, groups);
      const size_t sm = smem_cf<L, 2>();
      if (g.n_illum > 1)
        k_pcf<L, true, 2><<<grid, 64, sm, st>>>(planes, g, tw, ws_b, ill, frame_w, vol, fb, part);
      else
        k_pcf<L, false, 2><<<grid, 64, sm, st>>>(planes, g, tw, ws_b, ill, frame_w, vol, fb, part);
      if (part) {
        const long long total = (long long)nplanes * g.ny * g.nx;
        const int blocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
        k_pcf_sum<<<blocks, 256, 0, st>>>(planes, nplanes, g.ny, g.nx, part, groups, vol);
        PF_LAUNCH_CHECK("k_pcf_sum");
      }
    } else {
      dim3 grid(pf_cdiv(g.ny, RPC), nplanes);
      const size_t sm = smem_cf<L>();
      if (g.n_illum > 1)
        k_pcf<L, true><<<grid, FT, sm, st>>>(planes, g, tw, ws_b, ill, frame_w, vol, fb, nullptr);
      else
        k_pcf<L, false><<<grid, FT, sm, st>>>(planes, g, tw, ws_b, ill, frame_w, vol, fb, nullptr);
    }
    PF_LAUNCH_CHECK("k_pcf");
  } else {   // C: x-IFFT, crop, illumination phase, volume accumulate
    dim3 grid(pf_cdiv(g.ny, RPC), nplanes);
    const bool pre = n_frames == 1 && frame_w != nullptr && (size_t)RPC * g.nx * 8 <= 64 * 1024;
    const size_t sm = smem_c<L>(g.nx, pre);
    // centred column crop: compile-time kept columns
    const bool cent_x = 2 * g.nx == 32 * L && 2 * g.nu0x == -g.nx &&
                        2 * g.ny == 32 * L && 2 * g.nu0y == -g.ny;   // both crops centred
#define PF_PC_LAUNCH(M)                                                                        \
  if (pre) {                                                                                   \
    if (cent_x) k_pc<L, M, true, true><<<grid, FT, sm, st>>>(planes, kturns, g, tw, ws_b, ill, frame_w, n_frames, vol, vfs); \
    else k_pc<L, M, true, false><<<grid, FT, sm, st>>>(planes, kturns, g, tw, ws_b, ill, frame_w, n_frames, vol, vfs); \
  } else {                                                                                     \
    if (cent_x) k_pc<L, M, false, true><<<grid, FT, sm, st>>>(planes, kturns, g, tw, ws_b, ill, frame_w, n_frames, vol, vfs); \
    else k_pc<L, M, false, false><<<grid, FT, sm, st>>>(planes, kturns, g, tw, ws_b, ill, frame_w, n_frames, vol, vfs); \
  }
    if (g.n_illum > 1) {
      PF_PC_LAUNCH(true)
    } else {
      PF_PC_LAUNCH(false)
    }
#undef PF_PC_LAUNCH
    PF_LAUNCH_CHECK("k_pc");
  }
  return 0;
}

// ---- Relay spectra on the register path (reference reconstruct.py:259-260:
// Uhat = cfft2(_pad_embed(u)), with the centred embed of :113-119 as an index map).
// Output TRANSPOSED natural-order spectrum Uhat^T[b][kx][ky] (what B2 consumes).
// Rows: only the ny relay rows are transformed (zero rows transform to zero) and
// stored transposed through a padded shared tile; columns: one line per kx,
// reading only the relay rows' slots (the rest are zero), contiguous in ky.
template <int L>
__global__ void __launch_bounds__(FT, 2)
k_us_rows(const float2* __restrict__ src, int ny, int nx, long long sbs,
          const float2* __restrict__ tw, float2* __restrict__ dst) {
  constexpr int P = 32 * L, LPW = 32 / L, RPC = 8 * LPW, SLD = RPC + 1;
  extern __shared__ float2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int r = warp * LPW + line;
  const int jy0 = blockIdx.x * RPC;
  // rows jy0 .. jy0 + RPC - 1 hold relay rows iff centred(jy) + ny/2 in [0, ny);
  // a tile without any is never read by the column pass (uniform exit, before syncs)
  bool any = false;
#pragma unroll 1
  for (int q = 0; q < RPC; q++) any |= (unsigned)(centred(jy0 + q, P) + ny / 2) < (unsigned)ny;
  if (!any) return;
  const int iy = centred(jy0 + r, P) + ny / 2;
  const bool vrow = (unsigned)iy < (unsigned)ny;
  const float2* row = src + blockIdx.y * sbs + (long long)(vrow ? iy : 0) * nx;
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; m++) {
    const int ix = centred(t + L * m, P) + nx / 2;
    v[m] = (vrow && (unsigned)ix < (unsigned)nx) ? __ldg(row + ix) : make_float2(0.f, 0.f);
  }
  wfft<L, -1>(v, sm + warp * WFFT_XCH, tw);
  __syncthreads();
#pragma unroll
  for (int m = 0; m < 32; m++) sm[(t + L * m) * SLD + r] = v[m];
  __syncthreads();
  constexpr int KSTEP = FT / RPC;
  const int rr = threadIdx.x % RPC, k0 = threadIdx.x / RPC;
  float2* d = dst + (long long)blockIdx.y * P * P + (long long)k0 * P + jy0 + rr;
  const float2* q = sm + k0 * SLD + rr;
#pragma unroll 4
  for (int kx = k0; kx < P; kx += KSTEP) {
    *d = *q;
    d += (long long)KSTEP * P;
    q += KSTEP * SLD;
  }
}

template <int L>
__global__ void __launch_bounds__(FT, 2)
k_us_cols(int ny, const float2* __restrict__ tw, float2* __restrict__ dst) {
  constexpr int P = 32 * L, LPW = 32 / L;
  extern __shared__ float2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int kx = (blockIdx.x * 8 + warp) * LPW + line;
  float2* col = dst + blockIdx.y * (long long)P * P + (long long)kx * P;
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; m++) {
    const int jy = t + L * m;
    v[m] = (unsigned)(centred(jy, P) + ny / 2) < (unsigned)ny ? col[jy] : make_float2(0.f, 0.f);
  }
  wfft<L, -1>(v, sm + warp * WFFT_XCH, tw);
#pragma unroll
  for (int m = 0; m < 32; m++) col[t + L * m] = v[m];
}

template <int L>
int run_relay_spectra(const float2* src, long long nb, int ny, int nx, long long sbs,
                      const float2* tw, float2* dst, cudaStream_t st) {
  constexpr int P = 32 * L, LPW = 32 / L, RPC = 8 * LPW;
  const size_t sm_r = (size_t)(8 * WFFT_XCH > P * (RPC + 1) ? 8 * WFFT_XCH : P * (RPC + 1)) *
                      sizeof(float2);
  const size_t sm_c = 8 * WFFT_XCH * sizeof(float2);
  static PfDevOnce attr;  
  if (attr.first()) {
    cudaFuncSetAttribute(k_us_rows<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_us_cols<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  for (long long b0 = 0; b0 < nb; b0 += 65535) {
    const int n = (int)(nb - b0 < 65535 ? nb - b0 : 65535);
    k_us_rows<L><<<dim3(P / RPC, n), FT, sm_r, st>>>(src + b0 * sbs, ny, nx, sbs, tw,
                                                     dst + b0 * (long long)P * P);
    PF_LAUNCH_CHECK("k_us_rows");
    k_us_cols<L><<<dim3(P / (8 * LPW), n), FT, sm_c, st>>>(ny, tw, dst + b0 * (long long)P * P);
    PF_LAUNCH_CHECK("k_us_cols");
  }
  return 0;
}

}  // namespace

// 32*L when the register path applies (square power-of-two pad 128..1024), else 0
int pf_prop_fast_L(const pf_prop_geom* g) {
  if ((g->flags & 1) || g->px != g->py) return 0;
  switch (g->px) {
    case 128: return 4;
    case 256: return 8;
    case 512: return 16;
    case 1024: return 32;
    default: return 0;
  }
}

int pf_prop_fast_stage(int stage, const pf_plane* planes, int nplanes, double khat,
                       const pf_prop_geom* g, const pf_fft_plan* plan, const void* ws_a_in,
                       void* ws_a_out, const void* uhat, const void* ws_b_in, void* ws_b_out,
                       const double* ill, const void* frame_w, int n_frames, void* vol,
                       long long vfs, cudaStream_t st) {
  const float2* tw = (const float2*)plan->tw;
#define PF_FAST_CASE(LL)                                                                      \
  case LL:                                                                                    \
    return run_stage<LL>(stage, planes, nplanes, khat, *g, tw, (const float2*)ws_a_in,        \
                         (float2*)ws_a_out, (const float2*)uhat, (const float2*)ws_b_in,      \
                         (float2*)ws_b_out, ill, (const float2*)frame_w, n_frames,            \
                         (float2*)vol, vfs, st);
  switch (pf_prop_fast_L(g)) {
    PF_FAST_CASE(4)
    PF_FAST_CASE(8)
    PF_FAST_CASE(16)
    PF_FAST_CASE(32)
    default: break;
  }
#undef PF_FAST_CASE
  pf_set_error("pf_prop_fast_stage: geometry not eligible");
  return -1;
}

// Frequency-batched stages (all nf frequencies of a plane batch in one launch
// per stage; kernel C sums them in registers).  Register path only.
int pf_prop_fbatch_stage(int stage, const pf_plane* planes, int nplanes, const double* kturns,
                         int nf, const pf_prop_geom* g, const pf_fft_plan* plan, void* ws_a,
                         long long ws_a_fs, const void* uhat, long long uhat_fs, void* ws_b,
                         long long ws_b_fs, const double* ill, const void* frame_w, void* vol,
                         cudaStream_t st) {
  const float2* tw = (const float2*)plan->tw;
  FBatch fb{kturns, ws_a_fs, ws_b_fs, uhat_fs, nf};
#define PF_FB_CASE(LL)                                                                        \
  case LL:                                                                                    \
    return run_stage<LL>(stage, planes, nplanes, 0.0, *g, tw, (const float2*)ws_a,            \
                         (float2*)ws_a, (const float2*)uhat, (const float2*)ws_b,             \
                         (float2*)ws_b, ill, (const float2*)frame_w, 1, (float2*)vol, 0, st,  \
                         fb);
  switch (pf_prop_fast_L(g)) {
    PF_FB_CASE(4)
    PF_FB_CASE(8)
    PF_FB_CASE(16)
    PF_FB_CASE(32)
    default: break;
  }
#undef PF_FB_CASE
  pf_set_error("pf_prop_fbatch: geometry not eligible for the register path");
  return -1;
}

// Transposed relay spectra for the register path: dst[b][kx][ky] = cfft2 of the
// centred embed of src[b] (ny x nx, row-major) into P x P (P = pf_prop_fast).
extern "C" int pf_relay_spectra_fast(const void* src, int64_t nb, int ny, int nx,
                                     int64_t src_batch_stride, void* dst, int P,
                                     const pf_fft_plan* plan, void* stream) {
  PF_ARG_CHECK(plan != nullptr && plan->n == P, "pf_relay_spectra_fast: plan length != P");
  PF_ARG_CHECK(nb >= 0 && ny >= 1 && nx >= 1 && ny <= P && nx <= P,
               "pf_relay_spectra_fast: bad sizes");
  if (nb == 0) return 0;
  const float2* tw = (const float2*)plan->tw;
  cudaStream_t st = (cudaStream_t)stream;
  switch (P) {
    case 128: return run_relay_spectra<4>((const float2*)src, nb, ny, nx, src_batch_stride, tw, (float2*)dst, st);
    case 256: return run_relay_spectra<8>((const float2*)src, nb, ny, nx, src_batch_stride, tw, (float2*)dst, st);
    case 512: return run_relay_spectra<16>((const float2*)src, nb, ny, nx, src_batch_stride, tw, (float2*)dst, st);
    case 1024: return run_relay_spectra<32>((const float2*)src, nb, ny, nx, src_batch_stride, tw, (float2*)dst, st);
    default: break;
  }
  pf_set_error("pf_relay_spectra_fast: P must be 128, 256, 512 or 1024");
  return -1;
}

// Stage C with Horner's rule (see st_c): frequencies must be visited in descending order;
// dkhat = k_{f+1} - k_f (uniform spacing).  mode: 1 inner step, 2 last step of a
// single-block sum (f = 0, khat = k_0), 3 lowest frequency of a block (not f = 0),
// 4 f = 0 of a multi-block sum; modes 3/4 use ws_o (nplanes x ny x nx complex64, the
// batch's outer accumulator) and zkhat = B dkhat (B = block length).
// Eligible: register path, both crops centred, one illumination, illumination phase on,
// single frame.  Returns 1 (and does nothing) when the geometry is not eligible.
extern "C" int pf_prop_rows_out_horner(const pf_plane* planes, int nplanes, double khat,
                                       double dkhat, int mode, const pf_prop_geom* g,
                                       const pf_fft_plan* plan_x, const void* ws_b,
                                       const double* ill_xyz, const void* frame_w, void* vol,
                                       void* ws_o, double zkhat, void* vol_out, void* stream) {
  PF_ARG_CHECK(g && plan_x && plan_x->n == g->px && nplanes >= 1 && frame_w && vol &&
               mode >= 1 && mode <= 4 && (mode < 3 || ws_o),
               "pf_prop_rows_out_horner: bad args");
  const int L = pf_prop_fast_L(g);
  const int P = 32 * L;
  if (L == 0 || g->n_illum != 1 || !g->include_illum || 2 * g->nx != P || 2 * g->ny != P ||
      2 * g->nu0x != -g->nx || 2 * g->nu0y != -g->ny) {
    pf_set_error("pf_prop_rows_out_horner: geometry not eligible (register pad, one "
                 "illumination, centred crop of half the pad)");
    return 1;
  }
  const float2* tw = (const float2*)plan_x->tw;
  const double kturns = khat / PF_TWO_PI;
  const float dturns = (float)(dkhat / PF_TWO_PI);
  const double zturns = zkhat / PF_TWO_PI;
  cudaStream_t st = (cudaStream_t)stream;
#define PF_H_CASE(LL)                                                                          \
  case LL: {                                                                                   \
    constexpr int RPC = 8 * (32 / LL);                                                         \
    static PfDevOnce attr;                                                                    \
    if (attr.first()) {                                                                               \
      cudaFuncSetAttribute(k_pc_h<LL, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
      cudaFuncSetAttribute(k_pc_h<LL, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
      cudaFuncSetAttribute(k_pc_h<LL, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
      cudaFuncSetAttribute(k_pc_h<LL, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
    }                                                                                          \
    dim3 grid(pf_cdiv(g->ny, RPC), nplanes);                                                   \
    const size_t sm = smem_c<LL>(g->nx, true);                                                 \
    const float2* wb = (const float2*)ws_b;                                                    \
    const float2* fw = (const float2*)frame_w;                                                 \
    float2* vo = (float2*)vol;                                                                 \
    float2* wo = (float2*)ws_o;                                                                \
    float2* vout = (float2*)vol_out;                                                           \
    switch (mode) {                                                                            \
      case 1: k_pc_h<LL, 1><<<grid, FT, sm, st>>>(planes, kturns, dturns, *g, tw, wb, ill_xyz, fw, vo, wo, zturns, vout); break; \
      case 2: k_pc_h<LL, 2><<<grid, FT, sm, st>>>(planes, kturns, dturns, *g, tw, wb, ill_xyz, fw, vo, wo, zturns, vout); break; \
      case 3: k_pc_h<LL, 3><<<grid, FT, sm, st>>>(planes, kturns, dturns, *g, tw, wb, ill_xyz, fw, vo, wo, zturns, vout); break; \
      default: k_pc_h<LL, 4><<<grid, FT, sm, st>>>(planes, kturns, dturns, *g, tw, wb, ill_xyz, fw, vo, wo, zturns, vout); break; \
    }                                                                                          \
    PF_LAUNCH_CHECK("k_pc_h");                                                                 \
    return 0;                                                                                  \
  }
  switch (L) {
    PF_H_CASE(4)
    PF_H_CASE(8)
    PF_H_CASE(16)
    PF_H_CASE(32)
    default: break;
  }
#undef PF_H_CASE
  pf_set_error("pf_prop_rows_out_horner: no register FFT for L = %d", L);
  return 1;
}
