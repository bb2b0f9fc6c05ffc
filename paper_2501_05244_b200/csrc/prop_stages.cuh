// Stage bodies of the register-FFT propagation, one CTA each (tile = the CTA's
// block of lines within the stage), shared by the per-stage kernels
// (propagate_fast.cu) and the single-launch streaming kernel (prop_mega.cu).
// Reference rsd reconstruct.py:254-266 (and srsd :312-325, nursd1 :372-383):
//   A  synthesise kernel rows jy <= P/2 (G even: mirror lanes), x-FFT, store At[kx][jy]
//   B1 y-FFT of At rows in place -> Ghat quadrant (Ghat even in ky)
//   B2 Ghat column * Uhat^T column, y-IFFT, row crop -> Tt[col][i]
//   C  transposed tile, x-IFFT, column crop, illumination phase, volume +=
#pragma once
#include "prop_math.cuh"
#include "warp_fft.cuh"

constexpr int PROP_MT = 256;   // 8 warps per CTA

template <int L>
__device__ __forceinline__ void st_a(float2* sm, const pf_plane& pl, double kturns,
                                     const float2* __restrict__ tw, float2* __restrict__ wa,
                                     int tile) {
  constexpr int P = 32 * L, H = P / 2, NA = H + 1;
  constexpr int LPW = 32 / L, RPC = 8 * LPW, SLD = RPC + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int r = warp * LPW + line;
  const int jy0 = tile * RPC;
  const int jy = jy0 + r;
  const double ly = (double)jy * pl.lag_dy;
  const double base = fma(ly, ly, pl.dz * pl.dz);
  float2 v[32];
  const double lx_t = (double)t * pl.lag_dx;
#pragma unroll
  for (int m = 0; m <= 16; m++) {
    // lag of centred(t + L m, P): t + L m below P/2 for m < 16, t - P/2 at m = 16
    const double lx = fma((double)(m < 16 ? L * m : -H), pl.lag_dx, lx_t);
    v[m] = g_kernel(fma(lx, lx, base), kturns, (float)kturns);
  }
  const int mirror = (lane - t) + ((L - t) & (L - 1));
#pragma unroll
  for (int m = 17; m < 32; m++) {
    const float2 o = make_float2(__shfl_sync(0xffffffffu, v[31 - m].x, mirror),
                                 __shfl_sync(0xffffffffu, v[31 - m].y, mirror));
    v[m] = (t == 0) ? v[32 - m] : o;
  }
  wfft<L, -1>(v, sm + warp * WFFT_XCH, tw);
  __syncthreads();
  if (jy <= H) {
#pragma unroll
    for (int m = 0; m <= 16; m++) {
      // kx = t + L m <= P/2: every m < 16, and m = 16 at t = 0 only
      if (m < 16 || t == 0) sm[(t + L * m) * SLD + r] = v[m];
    }
  }
  __syncthreads();
  const int nr = min(RPC, NA - jy0);
  constexpr int KSTEP = PROP_MT / RPC;
  const int rr = threadIdx.x % RPC, k0 = threadIdx.x / RPC;
  if (rr < nr) {
    float2* d = wa + (long long)k0 * NA + jy0 + rr;
    const float2* q = sm + k0 * SLD + rr;
#pragma unroll 4
    for (int kx = k0; kx < NA; kx += KSTEP) {
      *d = *q;
      d += (long long)KSTEP * NA;
      q += KSTEP * SLD;
    }
  }
}

template <int L>
__device__ __forceinline__ void st_b1(float2* sm, const float2* __restrict__ tw,
                                      float2* __restrict__ wa, int tile) {
  constexpr int P = 32 * L, H = P / 2, NA = H + 1;
  constexpr int LPW = 32 / L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int row = (tile * 8 + warp) * LPW + line;
  const bool active = row < NA;
  float2* arow = wa + (long long)(active ? row : 0) * NA;
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; m++) {
    const int jy = t + L * m;
    v[m] = m < 16 ? arow[jy] : arow[P - jy];   // jy <= P/2 iff m < 16 (or m = 16, t = 0)
  }
  wfft<L, -1>(v, sm + warp * WFFT_XCH, tw);
  if (active) {
#pragma unroll
    for (int m = 0; m <= 16; m++) {
      if (m < 16 || t == 0) arow[t + L * m] = v[m];   // ky <= P/2
    }
  }
}

template <int L, bool MULTI>
__device__ __forceinline__ void st_b2(float2* sm, const pf_plane& pl, const pf_prop_geom& g,
                                      const float2* __restrict__ tw, const float2* __restrict__ wa,
                                      const float2* __restrict__ uhat_f, float2* __restrict__ wb,
                                      int tile) {
  constexpr int P = 32 * L, H = P / 2, NA = H + 1;
  constexpr int LPW = 32 / L, NL = 8 * LPW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int li = warp * LPW + line;
  const int kx_raw = tile * (NL / 2) + (li >> 1), side = li & 1;
  const int kx = min(kx_raw, H);
  const int col = side == 0 ? kx : (P - kx) % P;
  const bool active = kx_raw < NA && !(side == 1 && col == kx);
  const float2* grow = wa + (long long)kx * NA;
  const int ny = g.ny;
  const int n_ill = MULTI ? g.n_illum : 1;
#pragma unroll 1
  for (int p = 0; p < n_ill; p++) {
    const float2* ucol = uhat_f + pl.uhat_off + (long long)p * g.uhat_illum_stride +
                         (long long)col * P;
    float2 w[32];
#pragma unroll
    for (int m = 0; m < 32; m++) {
      const int ky = t + L * m;
      w[m] = cmul(m < 16 ? grow[ky] : grow[P - ky], __ldg(ucol + ky));
    }
    wfft<L, 1>(w, sm + warp * WFFT_XCH, tw);
    if (active) {
      float2* dcol = wb + (long long)p * P * ny + (long long)col * ny;
#pragma unroll
      for (int m = 0; m < 32; m++) {
        const int i = (t + L * m - g.nu0y) & (P - 1);
        if (i < ny) dcol[i] = w[m];
      }
    }
  }
}

// Centred crop (the output lattice is the relay lattice: n = P/2, nu0 = -n/2): the
// kept outputs of lane t are t + L ((m + 8) mod 32) for m in [0, 8) and [24, 32),
// known at compile time, so the crop and its addresses need no per-element tests.
__host__ __device__ constexpr bool cent_keep(int m) { return ((m + 8) & 31) < 16; }
__host__ __device__ constexpr int cent_base(int m) { return (m + 8) & 31; }

// HOR (single illumination, centred crop, prefetched single-frame volume): frequencies
// arrive in DESCENDING order and the illumination phase exp(i k_f d) is applied by
// Horner's rule, vol <- vol * z + v_f with z = exp(i dk d) (uniformly spaced k_f; dk d
// is a few radians, so z is formed in float32), and on the last step (f = 0, HOR = 2,
// kturns = k_0 / 2 pi) the sum is multiplied by exp(i k_0 d) in the float64-reduced form.
// Same sum as the ascending per-frequency phases, in nested order.
// Many frequencies (F > block): the nesting restarts every block of B frequencies so z is
// raised to at most B - 1, and the blocks are chained by Z = exp(i B dk d) formed from a
// float64-reduced phase (the outer accumulator o lives in ws_o, one row set per plane of
// the batch):  HOR = 3 at a block's lowest frequency: o <- o Z + (h z + v), h <- 0;
// HOR = 4 at f = 0: vol <- (o Z + (h z + v)) exp(i k_0 d).
template <int L, bool MULTI, bool PRE, bool CENT = false, int HOR = 0>
__device__ __forceinline__ void st_c(float2* sm, const pf_plane& pl, double kturns,
                                     const pf_prop_geom& g, const float2* __restrict__ tw,
                                     const float2* __restrict__ wb, const double* __restrict__ ill,
                                     const float2* __restrict__ frame_w, int n_frames,
                                     float2* __restrict__ vol, long long vfs, int tile,
                                     float dturns = 0.f, float2* __restrict__ ws_o = nullptr,
                                     double zturns = 0.0, float2* __restrict__ vol_out = nullptr) {
  static_assert(HOR == 0 || (!MULTI && PRE && CENT), "Horner variant: one illumination, "
                "centred crop, prefetched volume");
  constexpr int P = 32 * L;
  constexpr int LPW = 32 / L, RPC = 8 * LPW, SLD = RPC + 1;
  constexpr int UNION = (8 * WFFT_XCH > P * SLD) ? 8 * WFFT_XCH : P * SLD;
  float2* volbuf = sm + UNION;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = lane % L, line = lane / L;
  const int r = warp * LPW + line;
  // CENT: both crops centred, so ny = nx = P/2 at compile time (RPC divides P/2)
  const int ny = CENT ? P / 2 : g.ny, nx = CENT ? P / 2 : g.nx;
  const int i0 = tile * RPC;
  const int i = i0 + r;
  const int nr = CENT ? RPC : min(RPC, ny - i0);
  const float scale = 1.0f / ((float)P * (float)P);
  const long long vol_row0 = (pl.vol_plane * ny + i0) * (long long)nx;
  const bool aligned = ((g.nu0x | nx) & (L - 1)) == 0;   // column crop uniform per m
  // rows of P/2 elements starting at a multiple of P/2: 16-byte copies.  One illumination:
  // issued after the tile (LATE_VOL), so the transform waits only for the tile and the
  // volume rows arrive while it runs
  constexpr bool LATE_VOL = PRE && CENT && !MULTI;
  auto prefetch_vol = [&]() {
    const float4* src = reinterpret_cast<const float4*>(vol + vol_row0);
    float4* dst = reinterpret_cast<float4*>(volbuf);
#pragma unroll
    for (int e = threadIdx.x; e < RPC * (P / 4); e += PROP_MT) cp_async16(dst + e, src + e);
    cp_async_commit();
  };
  if (PRE && CENT && !LATE_VOL) {
    prefetch_vol();
  } else if (PRE && !CENT) {
    for (int rr = 0; rr < nr; rr++) {
      const float2* src = vol + vol_row0 + (long long)rr * nx;
#pragma unroll 4
      for (int mo = threadIdx.x; mo < nx; mo += PROP_MT) cp_async8(volbuf + rr * nx + mo, src + mo);
    }
    cp_async_commit();
  }
  float2 acc[MULTI ? 32 : 1];
  float2 v[32];
  const double yv = pl.y0 + pl.dy * i;
  const int n_ill = MULTI ? g.n_illum : 1;
#pragma unroll 1
  for (int p = 0; p < n_ill; p++) {
    const float2* src = wb + (long long)p * P * ny + i0;
    if (p > 0) __syncthreads();
    {
      constexpr int CSTEP = PROP_MT / RPC;
      const int rr = threadIdx.x % RPC, c0 = threadIdx.x / RPC;
      if (CENT) {
        // 16-byte copies of row pairs: odd columns sit one slot later in the padded tile
        // (col * SLD + (col & 1) + row), so every pair is 16-byte aligned on both sides;
        // compile-time strides, every copy is base + immediate offset
        constexpr int PSTEP = PROP_MT / (RPC / 2);
        const int pr = threadIdx.x % (RPC / 2), c0p = threadIdx.x / (RPC / 2);
        const float4* q = reinterpret_cast<const float4*>(src + c0p * (P / 2) + 2 * pr);
        float4* d = reinterpret_cast<float4*>(sm + c0p * SLD + (c0p & 1) + 2 * pr);
#pragma unroll
        for (int k = 0; k < P / PSTEP; k++)
          cp_async16(d + k * PSTEP * SLD / 2, q + k * PSTEP * (P / 2) / 2);
      } else if (rr < nr) {
        const float2* q = src + (long long)c0 * ny + rr;
        float2* d = sm + c0 * SLD + rr;
#pragma unroll 8
        for (int col = c0; col < P; col += CSTEP) {
          cp_async8(d, q);
          q += (long long)CSTEP * ny;
          d += CSTEP * SLD;
        }
      }
    }
    cp_async_commit();
    if (LATE_VOL) {
      prefetch_vol();
      cp_async_wait_1();   // the tile group; the volume group stays in flight
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 32; m++) v[m] = sm[(t + L * m) * SLD + (CENT ? (t & 1) : 0) + r];
    __syncthreads();
    wfft<L, 1>(v, sm + warp * WFFT_XCH, tw);
    const double sx = ill[3 * p], sy = ill[3 * p + 1], sz = ill[3 * p + 2];
    const double dy = yv - sy, dz = pl.z - sz;
    const double byz = fma(dy, dy, dz * dz);
    // x of output column t + base(m) (aligned crop): x0 - sx + dx * t once per lane
    const double xt = pl.x0 - sx + pl.dx * t;
    if (CENT && g.include_illum) {
#pragma unroll
      for (int m = 0; m < 32; m++) {
        float2 val = v[m];   // 1/P^2 (a power of two: exact) is folded into the frame weight
        if (HOR == 0 && cent_keep(m)) {
          const double dx = fma(pl.dx, (double)(L * cent_base(m)), xt);
          val = cmul(val, phase_turns(fma(dx, dx, byz), kturns, (float)kturns));
        }
        if (MULTI) {
          if (p == 0) acc[m] = val; else acc[m] = cadd(acc[m], val);
        } else {
          v[m] = val;
        }
      }
      continue;
    }
#pragma unroll
    for (int m = 0; m < 32; m++) {
      const int mo = (t + L * m - g.nu0x) & (P - 1);
      float2 val = v[m];   // 1/P^2 (a power of two: exact) is folded into the frame weight
      if (aligned) {
        const int base = (L * m - g.nu0x) & (P - 1);
        if (g.include_illum && base < nx) {
          const double dx = fma(pl.dx, (double)base, xt);
          val = cmul(val, phase_turns(fma(dx, dx, byz), kturns, (float)kturns));
        }
      } else if (g.include_illum && mo < nx) {
        const double dx = pl.x0 + pl.dx * mo - sx;
        val = cmul(val, phase_turns(fma(dx, dx, byz), kturns, (float)kturns));
      }
      if (MULTI) {
        if (p == 0) acc[m] = val; else acc[m] = cadd(acc[m], val);
      } else {
        v[m] = val;
      }
    }
  }
  if (LATE_VOL) {   // volume rows copied by other threads: complete and visible
    cp_async_wait_all();
    __syncthreads();
  }
  if (i < ny) {
    const long long off = vol_row0 + (long long)r * nx;
    if (PRE) {
      const float2* old = volbuf + r * nx;
      const float2 fw = cscale(frame_w[0], scale);
      if (CENT && HOR) {
        // the final step (HOR 2 / 4) may store the finished plane elsewhere: the fused
        // volume gather writes it straight into rank 0's volume (peer memory)
        float2* dt = ((HOR == 2 || HOR == 4) && vol_out ? vol_out : vol) + off + t;
        const float2* ot = old + t;
        const double dy = yv - ill[1], dz = pl.z - ill[2];
        const double byz = fma(dy, dy, dz * dz);
        const double xt = pl.x0 - ill[0] + pl.dx * t;
        const float byzf = (float)byz;
#pragma unroll
        for (int m = 0; m < 32; m++) {
          if (cent_keep(m)) {
            const int base = L * cent_base(m);
            const double dx = fma(pl.dx, (double)base, xt);
            const float dxf = (float)dx;
            const float d2 = fmaf(dxf, dxf, byzf);
            const float tz = dturns * (d2 * rsqrtf(d2));
            float zs, zc;
            __sincosf(6.28318530717958647692f * (tz - rintf(tz)), &zs, &zc);
            float2 nv = cadd(cmul(ot[base], make_float2(zc, zs)), cmul(v[m], fw));
            if (HOR >= 3) {   // chain the block: o Z + h (o row of this batch plane)
              const double d2 = fma(dx, dx, byz);
              float2* op = ws_o + ((long long)blockIdx.y * ny + i) * nx + t + base;
              nv = cadd(cmul(*op, phase_turns(d2, zturns, (float)zturns)), nv);
              if (HOR == 3) {
                *op = nv;
                nv = make_float2(0.f, 0.f);
              } else {
                nv = cmul(nv, phase_turns(d2, kturns, (float)kturns));
              }
            }
            if (HOR == 2) nv = cmul(nv, phase_turns(fma(dx, dx, byz), kturns, (float)kturns));
            dt[base] = nv;
          }
        }
      } else if (CENT) {
        float2* dt = vol + off + t;
        const float2* ot = old + t;
#pragma unroll
        for (int m = 0; m < 32; m++) {
          if (cent_keep(m)) {
            const int base = L * cent_base(m);
            dt[base] = cadd(ot[base], cmul(MULTI ? acc[m] : v[m], fw));
          }
        }
      } else if (aligned) {
        float2* dt = vol + off + t;
        const float2* ot = old + t;
#pragma unroll
        for (int m = 0; m < 32; m++) {
          const int base = (L * m - g.nu0x) & (P - 1);
          if (base < nx) dt[base] = cadd(ot[base], cmul(MULTI ? acc[m] : v[m], fw));
        }
      } else {
#pragma unroll
        for (int m = 0; m < 32; m++) {
          const int mo = (t + L * m - g.nu0x) & (P - 1);
          if (mo < nx) vol[off + mo] = cadd(old[mo], cmul(MULTI ? acc[m] : v[m], fw));
        }
      }
    } else {
      // frames innermost: each element's offset is formed once and reused for every
      // frame (hoisting 32 offsets out of a frame loop spilled)
#pragma unroll
      for (int m = 0; m < 32; m++) {
        const int mo = (t + L * m - g.nu0x) & (P - 1);
        if (mo < nx) {
          const float2 val = MULTI ? acc[m] : v[m];
          float2* d = vol + off + mo;
#pragma unroll 1
          for (int fr = 0; fr < n_frames; fr++) {
            float2* q = d + fr * vfs;
            *q = cadd(*q, cmul(val, cscale(__ldg(frame_w + fr), scale)));
          }
        }
      }
    }
  }
}

