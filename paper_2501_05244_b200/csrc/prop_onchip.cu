// On-chip propagation for the reference pad P = 140 (= 35 x 4; config 1, off-lattice nursd1,
// whose result depends on the pad so the reference's next_fast_len pad is kept: SURVEY F3).
//
// Reference: nursd1 reconstruct.py:372-383 (and rsd :254-266): for every (frequency f,
// plane k)  plane = cifft2(Uhat_f * cfft2(G_fk))[rows, cols] * mask_fk,  vol[k] += plane.
//
// A 140 x 140 complex plane is 157 KB, so one CTA holds a whole (f, k) unit in shared
// memory and no stage round-trips through L2 (the generic path's kernels A/B/C write and
// re-read the x-transformed kernel quadrant and the column-pass output per unit).  One CTA
// owns one plane and a range of frequencies (ascending; the sum stays in shared memory),
// so a plane's frequency sum has a fixed order for any grid.  Per frequency:
//   1  kernel columns jx <= P/2 (G is even in both lags): synthesise along y (float64
//      radius, g_kernel), y-FFT in registers, store rows ky <= P/2 at x = jx and P - jx
//      (Ghat_y is even in ky; the mirror in x makes each row the full even x-line)
//   2  x-FFT of rows ky <= P/2 in place  -> Ghat[ky][kx] (Ghat even in ky)
//   3  rows ky and P - ky together in one warp (both read Ghat row ky before either
//      writes): * Uhat[ky][:] (natural layout, read once per unit from L2), x-IFFT, keep
//      the cropped output columns
//   4  y-IFFT of the kept columns (strided in place), keep the cropped rows, scale,
//      illumination phase, * frame weight, acc += (ascending f)
// Line FFTs are the 35 x 4 mixed-radix register FFT (xfft.cuh): 4 lanes per line, 35
// points per lane, one exchange through the line's own row (or column) of the plane; the
// row pitch 140 = 12 (mod 16) float2 puts the 4 lanes x 4 lines of a half-warp in distinct
// bank quads for both the row and the strided column accesses.
#include <algorithm>

#include "fft.cuh"
#include "prop_math.cuh"

namespace {

constexpr int OC_L = 4, OC_R = XFFT_R, OC_P = OC_R * OC_L;   // 140
constexpr int OC_J = xfft_J(OC_L);                            // 9
constexpr int OC_H = OC_P / 2;
constexpr int OC_LD = OC_P;
constexpr int OC_ROWS = OC_P + 2;   // rows P/2+1 .. P+1: exchange rows of stage 1
constexpr int OC_LPW = 32 / OC_L;

// natural slot of c in (-P, 2P)
__device__ __forceinline__ int oc_wrap(int c) {
  c += c < 0 ? OC_P : 0;
  return c - (c >= OC_P ? OC_P : 0);
}

// 140-point line transform, Cooley-Tukey 35 x 4 in natural order (the prime-factor form
// has no twiddles but its CRT / Ruritanian index maps put the 4 lanes of a line on the same
// bank quad for either the loads or the stores: measured slower): lane t of the line holds
// v[m] = x[t + 4 m]; 35-point DFT in registers (itself prime-factor 5 x 7), twiddles
// W_140^{k1 t} (tw, shared memory), one exchange through the line's own storage (element e
// at row[e * ES]), 4-point DFTs; on return w[j][k2] = X[k1 + 35 k2] with k1 = t + 4 j < 35.
// `active` lanes write the exchange; every lane calls it.
// lane within the line, re-read per stage (volatile: the compiler cannot hoist the 35
// t-dependent element offsets of every stage out of the frequency loop, which would pin
// ~70 registers for the whole kernel)
__device__ __forceinline__ int oc_t() {
  unsigned l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return (int)(l & (OC_L - 1));
}
__device__ __forceinline__ int oc_in(int m, int t) { return t + OC_L * m; }
__device__ __forceinline__ int oc_out(int k1, int k2) { return k1 + OC_R * k2; }

template <int DIR, int ES>
__device__ __forceinline__ void oc_fft(float2 (&v)[OC_R], float2 (&w)[OC_J][OC_L],
                                       float2* row, const float2* tw, int t, bool active) {
  Dft<OC_R, DIR>::run(v);
  if (t != 0) {
#pragma unroll
    for (int k1 = 1; k1 < OC_R; k1++) {
      const float2 c = tw[k1 * OC_L + t];
      v[k1] = DIR < 0 ? cmul(v[k1], c) : cmulc(v[k1], c);
    }
  }
  __syncwarp();
  if (active) {
#pragma unroll
    for (int k1 = 0; k1 < OC_R; k1++) row[(t * OC_R + k1) * ES] = v[k1];
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < OC_J; j++) {
    const int k1 = t + OC_L * j;
    if (k1 < OC_R) {
#pragma unroll
      for (int tp = 0; tp < OC_L; tp++) w[j][tp] = row[(tp * OC_R + k1) * ES];
      Dft<OC_L, DIR>::run(w[j]);
    }
  }
  __syncwarp();
}

template <int NW>
__device__ __forceinline__ void oc_body(const pf_plane* __restrict__ planes,
                                        const double* __restrict__ kturns_f, int nf, int fpc,
                                        const pf_prop_geom& g, const float2* __restrict__ uhat,
                                        long long uhat_fs, const double* __restrict__ ill,
                                        const float2* __restrict__ frame_w,
                                        float2* __restrict__ vol, float2* __restrict__ ws_part,
                                        int acc_ld) {
  extern __shared__ float2 sm[];
  const int nx = g.nx, ny = g.ny;
  float2* S = sm;                               // [OC_ROWS][OC_LD]
  float2* acc = sm + OC_ROWS * OC_LD;           // [nx][acc_ld]: acc[m][i]
  float2* tw = acc + (size_t)nx * acc_ld;       // [35][4] = W_140^{k1 t}
  for (int e = threadIdx.x; e < OC_R * OC_L; e += NW * 32) {
    double sn, cs;
    sincospi(-2.0 * (double)((e / OC_L) * (e % OC_L)) / OC_P, &sn, &cs);
    tw[e] = make_float2((float)cs, (float)sn);
  }
  const pf_plane pl = planes[blockIdx.x];
  const int f0 = blockIdx.y * fpc, f1 = min(nf, f0 + fpc);
  for (int e = threadIdx.x; e < nx * acc_ld; e += NW * 32) acc[e] = make_float2(0.f, 0.f);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int line = lane / OC_L;
  const float scale = 1.0f / ((float)OC_P * (float)OC_P);
  const double sx = ill[0], sy = ill[1], sz = ill[2];
  const float2* up = uhat + pl.uhat_off;
  for (int f = f0; f < f1; f++) {
    const double kt = kturns_f[f];
    const float ktf = (float)kt;
    __syncthreads();   // previous frequency's stage 4 is done with S (and acc zeroed)
    // ---- 1: kernel columns jx = slot <= P/2, synthesised along y, y-FFT
    for (int s0 = warp * OC_LPW; s0 <= OC_H; s0 += NW * OC_LPW) {   // warp-uniform
      const int t = oc_t();
      const int sl = s0 + line;
      const bool act = sl <= OC_H;
      const int jx = act ? sl : OC_H;
      const double lx = (double)centred(jx, OC_P) * pl.lag_dx;
      const double bx = fma(lx, lx, pl.dz * pl.dz);
      // synthesised into the line's exchange row (rows P/2+1 .. P+1) first, lags 0..P/2
      // once each (G is even in the y lag): the float64 radius of 35 points at once in
      // registers would not fit the register budget
      float2* xrow = S + (OC_H + 1 + jx) * OC_LD;
      if (act) {
#pragma unroll 3
        for (int jy = t; jy <= OC_H; jy += OC_L) {
          const double ly = (double)jy * pl.lag_dy;
          const float2 gv = g_kernel(fma(ly, ly, bx), kt, ktf);
          xrow[jy] = gv;
          if (jy != 0 && jy != OC_H) xrow[OC_P - jy] = gv;
        }
      }
      __syncwarp();
      float2 v[OC_R];
#pragma unroll
      for (int n1 = 0; n1 < OC_R; n1++) v[n1] = xrow[oc_in(n1, t)];
      float2 w[OC_J][OC_L];
      oc_fft<-1, 1>(v, w, xrow, tw, t, act);
      if (act) {
        const bool mir = jx != 0 && jx != OC_H;
#pragma unroll
        for (int j = 0; j < OC_J; j++) {
          const int k1 = t + OC_L * j;
#pragma unroll
          for (int k2 = 0; k2 < OC_L; k2++) {
            const int ky = oc_out(k1, k2);
            if (k1 < OC_R && ky <= OC_H) {
              S[ky * OC_LD + jx] = w[j][k2];
              if (mir) S[ky * OC_LD + OC_P - jx] = w[j][k2];
            }
          }
        }
      }
    }
    __syncthreads();
    // ---- 2: x-FFT of rows ky <= P/2 in place
    for (int s0 = warp * OC_LPW; s0 <= OC_H; s0 += NW * OC_LPW) {
      const int t = oc_t();
      const int sl = s0 + line;
      const bool act = sl <= OC_H;
      float2* row = S + min(sl, OC_H) * OC_LD;
      float2 v[OC_R];
#pragma unroll
      for (int n1 = 0; n1 < OC_R; n1++) v[n1] = row[oc_in(n1, t)];
      float2 w[OC_J][OC_L];
      oc_fft<-1, 1>(v, w, row, tw, t, act);
      if (act) {
#pragma unroll
        for (int j = 0; j < OC_J; j++) {
          const int k1 = t + OC_L * j;
          if (k1 < OC_R) {
#pragma unroll
            for (int k2 = 0; k2 < OC_L; k2++) row[oc_out(k1, k2)] = w[j][k2];
          }
        }
      }
    }
    __syncthreads();
    // ---- 3: rows ky, P - ky: * Uhat, x-IFFT, keep the cropped columns (pairs in one warp)
    for (int s0 = warp * OC_LPW; s0 < 2 * (OC_H + 1); s0 += NW * OC_LPW) {   // warp-uniform
      const int t = oc_t();
      const int s = min(s0 + line, 2 * OC_H + 1);
      const int q = s >> 1, side = s & 1;
      const bool act = s0 + line <= 2 * OC_H + 1 && (side == 0 || (q != 0 && q != OC_H));
      const int ky = side == 0 ? q : OC_P - q;
      float2* row = S + (act ? ky : q) * OC_LD;
      const float2* grow = S + q * OC_LD;
      const float2* urow = up + (long long)f * uhat_fs + (long long)(act ? ky : q) * OC_P;
      float2 v[OC_R];
#pragma unroll
      for (int n1 = 0; n1 < OC_R; n1++) v[n1] = __ldg(urow + oc_in(n1, t));
#pragma unroll
      for (int n1 = 0; n1 < OC_R; n1++) v[n1] = cmul(grow[oc_in(n1, t)], v[n1]);
      float2 w[OC_J][OC_L];
      oc_fft<1, 1>(v, w, row, tw, t, act);
      if (act) {
#pragma unroll
        for (int j = 0; j < OC_J; j++) {
          const int k1 = t + OC_L * j;
#pragma unroll
          for (int k2 = 0; k2 < OC_L; k2++) {
            const int xn = oc_out(k1, k2);
            if (k1 < OC_R && oc_wrap(xn - g.nu0x) < nx) row[xn] = w[j][k2];
          }
        }
      }
    }
    __syncthreads();
    // ---- 4: y-IFFT of output column m (x = nu0x + m), rows cropped, acc += (ascending f)
    const float2 fw = cscale(frame_w[f], scale);
    for (int m0 = warp * OC_LPW; m0 < nx; m0 += NW * OC_LPW) {
      const int t = oc_t();
      const int mr = m0 + line;
      const bool act = mr < nx;
      const int m = act ? mr : m0;
      float2* col = S + oc_wrap(g.nu0x + m);
      float2 v[OC_R];
#pragma unroll
      for (int n1 = 0; n1 < OC_R; n1++) v[n1] = col[oc_in(n1, t) * OC_LD];
      float2 w[OC_J][OC_L];
      oc_fft<1, OC_LD>(v, w, col, tw, t, act);
      if (act) {
        const double dx = fma(pl.dx, (double)m, pl.x0 - sx);
        const double dz = pl.z - sz;
        const double bxz = fma(dx, dx, dz * dz);
#pragma unroll
        for (int j = 0; j < OC_J; j++) {
          const int k1 = t + OC_L * j;
#pragma unroll
          for (int k2 = 0; k2 < OC_L; k2++) {
            const int i = oc_wrap(oc_out(k1, k2) - g.nu0y);
            if (k1 < OC_R && i < ny) {
              float2 val = w[j][k2];
              if (g.include_illum) {
                const double dy = fma(pl.dy, (double)i, pl.y0 - sy);
                val = cmul(val, phase_turns(fma(dy, dy, bxz), kt, ktf));
              }
              float2& a = acc[m * acc_ld + i];
              a = cadd(a, cmul(val, fw));
            }
          }
        }
      }
    }
  }
  __syncthreads();
  // the plane's sum over this CTA's frequencies: straight into the volume (one group) or
  // into the group's partial plane (k_onchip_sum adds the groups in ascending order)
  const long long plane_elems = (long long)ny * nx;
  for (int i = warp; i < ny; i += NW) {
    for (int m = lane; m < nx; m += 32) {
      const float2 a = acc[m * acc_ld + i];
      const long long e = (long long)i * nx + m;
      if (gridDim.y == 1) {
        float2* d = vol + pl.vol_plane * plane_elems + e;
        *d = cadd(*d, a);
      } else {
        ws_part[((long long)blockIdx.y * gridDim.x + blockIdx.x) * plane_elems + e] = a;
      }
    }
  }
}

#define OC_KARGS                                                                              \
  const pf_plane *__restrict__ planes, const double *__restrict__ kturns_f, int nf, int fpc,  \
      pf_prop_geom g, const float2 *__restrict__ uhat, long long uhat_fs,                      \
      const double *__restrict__ ill, const float2 *__restrict__ frame_w,                      \
      float2 *__restrict__ vol, float2 *__restrict__ ws_part, int acc_ld
// 12 / 16 warps: the launch bound caps registers at 168 / 128 (fewer warps cannot use more
// registers: each SM sub-partition holds 16 K registers for its share of the warps)
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_prop_onchip(OC_KARGS) {
  oc_body<NW>(planes, kturns_f, nf, fpc, g, uhat, uhat_fs, ill, frame_w, vol, ws_part, acc_ld);
}
#undef OC_KARGS

// vol[plane k] += sum over groups g (ascending) of ws_part[g][k]
__global__ void k_onchip_sum(const pf_plane* __restrict__ planes, int nplanes, int groups,
                             long long plane_elems, const float2* __restrict__ ws_part,
                             float2* __restrict__ vol) {
  const long long n = (long long)nplanes * plane_elems;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e / plane_elems);
    const long long r = e - k * plane_elems;
    float2 s = ws_part[e];
    for (int gi = 1; gi < groups; gi++) s = cadd(s, ws_part[gi * n + e]);
    float2* d = vol + planes[k].vol_plane * plane_elems + r;
    *d = cadd(*d, s);
  }
}

constexpr int OC_NW = 12;

int acc_pitch(int ny) {
  int k = ny;
  while (k % 16 != 4) k++;   // acc[m][i]: 4 lines x 4 lanes of a half-warp in distinct bank quads
  return k;
}

size_t onchip_smem(const pf_prop_geom& g) {
  return ((size_t)OC_ROWS * OC_LD + (size_t)g.nx * acc_pitch(g.ny) + OC_R * OC_L) *
         sizeof(float2);
}

}  // namespace

extern "C" int pf_prop_onchip_ok(const pf_prop_geom* g) {
  if (!g) return 0;
  int d = 0, smax = 0;
  cudaGetDevice(&d);
  if (cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, d) != cudaSuccess)
    smax = 232448;
  return g->px == OC_P && g->py == OC_P && g->n_illum == 1 && g->nx >= 1 && g->ny >= 1 &&
         g->nx <= OC_P && g->ny <= OC_P && onchip_smem(*g) <= (size_t)smax;
}

extern "C" int pf_prop_fbatch_onchip(const pf_plane* planes, int nplanes, const double* kturns,
                                     int nf, const pf_prop_geom* g, const void* uhat,
                                     int64_t uhat_fs, const double* ill_xyz, const void* frame_w,
                                     void* vol, void* ws_part, int groups, int warps,
                                     void* stream) {
  PF_ARG_CHECK(g && planes && kturns && uhat && ill_xyz && frame_w && vol && nplanes >= 1 &&
                   nf >= 1 && groups >= 1 && groups <= nf,
               "pf_prop_fbatch_onchip: bad args");
  PF_ARG_CHECK(pf_prop_onchip_ok(g),
               "pf_prop_fbatch_onchip: needs px = py = 140, one illumination and a plane that "
               "fits shared memory");
  if (warps <= 0) warps = OC_NW;
  PF_ARG_CHECK(warps == 8 || warps == 9 || warps == 10 || warps == 12 || warps == 16,
               "pf_prop_fbatch_onchip: warps per CTA must be 8, 9, 10, 12 or 16 (0: default)");
  const int fpc = pf_cdiv(nf, groups);
  const int gy = pf_cdiv(nf, fpc);   // groups actually populated
  PF_ARG_CHECK(gy == 1 || ws_part, "pf_prop_fbatch_onchip: ws_part needed for groups > 1");
  cudaStream_t st = (cudaStream_t)stream;
  static PfDevOnce attr;
  const size_t smem = onchip_smem(*g);
  if (attr.first()) {
    int d = 0, smax = 232448;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
    cudaFuncSetAttribute(k_prop_onchip<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
    cudaFuncSetAttribute(k_prop_onchip<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
    cudaFuncSetAttribute(k_prop_onchip<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
    cudaFuncSetAttribute(k_prop_onchip<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
    cudaFuncSetAttribute(k_prop_onchip<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
  }
  const dim3 grid(nplanes, gy);
#define OC_LAUNCH(KERN, NWV)                                                                  \
  KERN<<<grid, NWV * 32, smem, st>>>(planes, kturns, nf, fpc, *g,                             \
                                                    (const float2*)uhat, uhat_fs, ill_xyz,     \
                                                    (const float2*)frame_w, (float2*)vol,      \
                                                    (float2*)ws_part, acc_pitch(g->ny))
  if (warps == 16) OC_LAUNCH(k_prop_onchip<16>, 16);
  else if (warps == 8) OC_LAUNCH(k_prop_onchip<8>, 8);
  else if (warps == 9) OC_LAUNCH(k_prop_onchip<9>, 9);
  else if (warps == 10) OC_LAUNCH(k_prop_onchip<10>, 10);
  else OC_LAUNCH(k_prop_onchip<12>, 12);
#undef OC_LAUNCH
  PF_LAUNCH_CHECK("k_prop_onchip");
  if (gy > 1) {
    const long long pe = (long long)g->ny * g->nx;
    const int blocks = (int)std::min<long long>(pf_cdiv(nplanes * pe, 256), 4LL * pf_sm_count());
    k_onchip_sum<<<blocks, 256, 0, st>>>(planes, nplanes, gy, pe, (const float2*)ws_part,
                                         (float2*)vol);
    PF_LAUNCH_CHECK("k_onchip_sum");
  }
  return 0;
}
