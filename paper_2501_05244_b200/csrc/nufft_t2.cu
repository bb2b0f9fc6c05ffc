// Type-2 NUFFT start for 2D plans, fused (reference spectral.py:373-375):
//   fine = ifftn(place(S / (ker_y ker_x)))       (unnormalised inverse, natural order)
// in two passes instead of place + two pruned line passes (pf_nufft_place + pf_fft_lines):
//
//   rows:    for every KEPT fine row (the my slots holding centred modes) build the row
//            in shared memory straight from the mode grid -- S / deconvolution on the mx
//            kept slots, zero elsewhere -- inverse-transform it along x and store it;
//   columns: for every fine column read only the kept rows (the other rows are zero by
//            construction and are never written nor read), inverse-transform along y and
//            store the whole column.
//
// Per fine grid this moves S (my mx) + kept rows (my mrx, written then read) + the grid
// (mry mrx, written) instead of S + a zero-filled grid written + kept rows read / written
// + the grid read / written: 9 instead of 17 bytes-units at mr = 2m.  Same arithmetic and
// operation order as the unfused sequence (the FFT kernels are the same), so the fine
// grid is bit-identical to it.
#include "fft.cuh"

namespace {

constexpr int T2_THREADS = 256;
constexpr size_t T2_SMEM = 200 * 1024;

template <int XL>
__global__ void __launch_bounds__(T2_THREADS, XL > 0 ? 2 : 1)
k_t2_rows(pf_nufft_geom G, const float2* __restrict__ S, long long s_stride,
          const float* __restrict__ ky, const float* __restrict__ kx, int nv,
          float2* __restrict__ fine, long long fine_stride, pf_fft_plan plan_x, int cnt) {
  extern __shared__ float2 sm[];
  const int mrx = G.mr[2], mx = G.m[2], my = G.m[1], mry = G.mr[1];
  const int ld = pf_ld(mrx);
  float2* a = sm;
  float2* b = sm + (size_t)cnt * ld;
  const long long nlines = (long long)nv * my;
  const long long l0 = (long long)blockIdx.x * cnt;
  const int nl = (int)(nlines - l0 < cnt ? nlines - l0 : cnt);
  const FastDiv dmrx(mrx);
  for (int e = threadIdx.x; e < nl * mrx; e += T2_THREADS) {
    const int c = dmrx.div(e), fx = e - c * mrx;
    const long long l = l0 + c;
    const int v = (int)(l / my), i = (int)(l - (long long)v * my);
    const int cy = i - my / 2;
    const int cx = fx < mrx - mrx / 2 ? fx : fx - mrx;
    float2 val = make_float2(0.f, 0.f);
    if (cx >= -(mx / 2) && cx < mx - mx / 2) {
      const int jy = natural(cy, my), jx = natural(cx, mx);
      // k_place's denominator: kz[0] (= 1) * ky * kx
      const float den = 1.0f * ky[cy + my / 2] * kx[cx + mx / 2];
      const float2 s = S[(long long)v * s_stride + (long long)jy * mx + jx];
      val = make_float2(s.x / den, s.y / den);
    }
    a[c * ld + fx] = val;
  }
  __syncthreads();
  const float2* res = fft_any<XL, 1>(a, b, ld, nl, plan_x);
  for (int e = threadIdx.x; e < nl * mrx; e += T2_THREADS) {
    const int c = dmrx.div(e), fx = e - c * mrx;
    const long long l = l0 + c;
    const int v = (int)(l / my), i = (int)(l - (long long)v * my);
    const int cy = i - my / 2;
    const int fy = cy < 0 ? cy + mry : cy;
    fine[(long long)v * fine_stride + (long long)fy * mrx + fx] = res[c * ld + fx];
  }
}

template <int XL>
__global__ void __launch_bounds__(T2_THREADS, XL > 0 ? 2 : 1)
k_t2_cols(pf_nufft_geom G, int nv, float2* __restrict__ fine, long long fine_stride,
          pf_fft_plan plan_y, int cnt) {
  extern __shared__ float2 sm[];
  __shared__ long long lbase[64];
  const int mrx = G.mr[2], my = G.m[1], mry = G.mr[1];
  const int ld = pf_ld(mry);
  float2* a = sm;
  float2* b = sm + (size_t)cnt * ld;
  const long long nlines = (long long)nv * mrx;
  const long long l0 = (long long)blockIdx.x * cnt;
  const int nl = (int)(nlines - l0 < cnt ? nlines - l0 : cnt);
  for (int c = threadIdx.x; c < nl; c += T2_THREADS) {
    const long long l = l0 + c;
    const long long v = l / mrx;
    lbase[c] = v * fine_stride + (l - v * mrx);
  }
  __syncthreads();
  const FastDiv dnl(nl);
  const int lo_hi = my - my / 2;          // kept slots [0, lo_hi) and [mry - my/2, mry)
  const int hi_lo = mry - my / 2;
  for (int e = threadIdx.x; e < nl * mry; e += T2_THREADS) {
    const int fy = dnl.div(e), c = e - fy * nl;
    float2 val = make_float2(0.f, 0.f);
    if (fy < lo_hi || fy >= hi_lo) val = fine[lbase[c] + (long long)fy * mrx];
    a[c * ld + fy] = val;
  }
  __syncthreads();
  const float2* res = fft_any<XL, 1>(a, b, ld, nl, plan_y);
  for (int e = threadIdx.x; e < nl * mry; e += T2_THREADS) {
    const int fy = dnl.div(e), c = e - fy * nl;
    fine[lbase[c] + (long long)fy * mrx] = res[c * ld + fy];
  }
}

// ---- split passes for mr = 2 m (the reference's fine grid whenever 2 m is a fast length) --
// A fine line holds the m centred modes c[k], k in [-m/2, m - m/2), and zeros elsewhere, so
// its 2 m-point inverse transform splits by output parity into two m-point transforms of
// the modes alone:
//     X[2 j]     = sum_k c[k]                    e^{2 pi i j k / m}
//     X[2 j + 1] = sum_k c[k] e^{i pi k / m}     e^{2 pi i j k / m}
// (the radix-2 decimation-in-frequency step whose other half of the inputs is zero).  Each
// fine line becomes two half-lines of length m = 35 L' run by the register FFT with L'
// lanes: no zero is loaded or transformed, and for 700 = 2 x 350 the lines fill 30 of a
// warp's 32 lanes (3 lines x 10 lanes) where the 700-point transform fills 20.  The
// half-length twiddle table W_m^{k1 t} is formed in shared memory from the 2 m plan's
// unit roots.  Results differ from the unsplit passes by float32 rounding only.
template <int HL, int NT>
__device__ __forceinline__ void t2_half_table(float2* tw2, int m, const float2* __restrict__ roots2m) {
  for (int e = threadIdx.x; e < XFFT_R * HL; e += NT) {
    const int k1 = e / HL, t = e - k1 * HL;
    tw2[e] = __ldg(roots2m + 2 * ((k1 * t) % m));
  }
}

template <int HL, int NT>
__global__ void __launch_bounds__(NT, 512 / NT)
k_t2_rows_split(pf_nufft_geom G, const float2* __restrict__ S, long long s_stride,
                const float* __restrict__ ky, const float* __restrict__ kx, int nv,
                float2* __restrict__ fine, long long fine_stride, pf_fft_plan plan_x, int cnt,
                int col0, int ncols) {
  extern __shared__ float2 sm[];
  const int mrx = G.mr[2], mx = G.m[2], my = G.m[1], mry = G.mr[1];
  const int ld = pf_ld(mx);
  float2* a = sm;                                   // [2 cnt][ld]: line c -> rows 2c (even), 2c + 1
  float2* tw2 = sm + (size_t)2 * cnt * ld;          // [35][HL]
  const float2* roots = reinterpret_cast<const float2*>(plan_x.tw);
  t2_half_table<HL, NT>(tw2, mx, roots);
  const long long nlines = (long long)nv * my;
  const long long l0 = (long long)blockIdx.x * cnt;
  const int nl = (int)(nlines - l0 < cnt ? nlines - l0 : cnt);
  // per line: source row of S, target row of the fine grid, 1 / ker_y (the 64-bit divisions
  // once per line, not per element); per column: 1 / ker_x
  __shared__ long long src_row[32], dst_row[32];
  __shared__ float rky[32];
  float* rkx = reinterpret_cast<float*>(tw2 + XFFT_R * HL);   // [mx]
  for (int c = threadIdx.x; c < nl; c += NT) {
    const long long l = l0 + c;
    const int v = (int)(l / my), i = (int)(l - (long long)v * my);
    const int cy = i - my / 2;
    src_row[c] = (long long)v * s_stride + (long long)natural(cy, my) * mx;
    dst_row[c] = (long long)v * fine_stride + (long long)(cy < 0 ? cy + mry : cy) * mrx;
    rky[c] = 1.0f / ky[i];
  }
  for (int q = threadIdx.x; q < mx; q += NT) rkx[q] = 1.0f / kx[q];
  __syncthreads();
  const FastDiv dmx(mx);
  for (int e = threadIdx.x; e < nl * mx; e += NT) {
    const int c = dmx.div(e), q = e - c * mx;
    const int cx = q - mx / 2;
    const int jx = cx < 0 ? cx + mx : cx;
    const float inv = rky[c] * rkx[q];
    const float2 sv = S[src_row[c] + jx];
    const float2 val = make_float2(sv.x * inv, sv.y * inv);
    a[(2 * c) * ld + jx] = val;
    a[(2 * c + 1) * ld + jx] = cmulc(val, __ldg(roots + (cx < 0 ? cx + mrx : cx)));
  }
  __syncthreads();
  xfft_tile<HL, 1, true>(a, ld, 2 * nl, tw2);
  // only the columns some readout stencil touches are stored (window [col0, col0 + ncols) on
  // the torus; the column pass transforms no others): output pairs (2 j, 2 j + 1) from
  // j = col0 / 2 on, around the seam
  const int j0 = col0 >> 1;
  const int npairs = min(mx, ((col0 + ncols - 1) >> 1) - j0 + 1);
  const FastDiv dnp(npairs);
  for (int e = threadIdx.x; e < nl * npairs; e += NT) {
    const int c = dnp.div(e);
    int j = j0 + (e - c * npairs);
    j -= j >= mx ? mx : 0;
    int d0 = 2 * j - col0, d1 = 2 * j + 1 - col0;
    d0 += d0 < 0 ? mrx : 0;
    d1 += d1 < 0 ? mrx : 0;
    const bool in0 = d0 < ncols, in1 = d1 < ncols;
    if (!in0 && !in1) continue;
    const float2 ev = a[(2 * c) * ld + j], od = a[(2 * c + 1) * ld + j];
    float2* dst = fine + dst_row[c] + 2 * j;
    if (in0 && in1) {
      *reinterpret_cast<float4*>(dst) = make_float4(ev.x, ev.y, od.x, od.y);
    } else if (in0) {
      dst[0] = ev;
    } else {
      dst[1] = od;
    }
  }
}

template <int HL, int NT>
__global__ void __launch_bounds__(NT, 512 / NT)
k_t2_cols_split(pf_nufft_geom G, int nv, float2* __restrict__ fine, long long fine_stride,
                pf_fft_plan plan_y, int cnt, int col0, int ncols, int row0, int nrows,
                float2* __restrict__ out, int il, int member) {
  // out / il: the transformed columns go to `out` with every il consecutive grids
  // interleaved cell by cell, out[(v / il) (fine_stride il) + cell il + v % il] (il = 1,
  // out = fine: in place) -- the layout the node-gathering readout reads with wide loads;
  // member >= 0: every grid v of this call is slot `member` of its own group v (the call
  // holds one frequency of every plane: out[v (fine_stride il) + cell il + member])
  extern __shared__ float2 sm[];
  __shared__ long long lbase[64], obase[64];
  const int mrx = G.mr[2], my = G.m[1], mry = G.mr[1];
  const int ld = pf_ld(my);
  float2* a = sm;                                   // [2 cnt][ld]
  float2* tw2 = sm + (size_t)2 * cnt * ld;
  const float2* roots = reinterpret_cast<const float2*>(plan_y.tw);
  t2_half_table<HL, NT>(tw2, my, roots);
  // only the columns of the window [col0, col0 + ncols) (torus) are transformed, and of each
  // only the rows of [row0, row0 + nrows) are stored: the cells the readout stencils touch
  const long long nlines = (long long)nv * ncols;
  const long long l0 = (long long)blockIdx.x * cnt;
  const int nl = (int)(nlines - l0 < cnt ? nlines - l0 : cnt);
  for (int c = threadIdx.x; c < nl; c += NT) {
    const long long l = l0 + c;
    const long long v = l / ncols;
    int col = col0 + (int)(l - v * ncols);
    col -= col >= mrx ? mrx : 0;
    lbase[c] = v * fine_stride + col;
    const long long vg = member >= 0 ? v : v / il;
    obase[c] = vg * (fine_stride * il) + (long long)col * il + (member >= 0 ? member : v - vg * il);
  }
  __syncthreads();
  const FastDiv dnl(nl);
  for (int e = threadIdx.x; e < nl * my; e += NT) {
    const int q = dnl.div(e), c = e - q * nl;
    const int cy = q - my / 2;
    const int fy = cy < 0 ? cy + mry : cy;      // the kept fine row holding mode cy
    const int jy = natural(cy, my);
    const float2 val = fine[lbase[c] + (long long)fy * mrx];
    a[(2 * c) * ld + jy] = val;
    a[(2 * c + 1) * ld + jy] = cmulc(val, __ldg(roots + fy));
  }
  __syncthreads();
  xfft_tile<HL, 1, true>(a, ld, 2 * nl, tw2);
  for (int e = threadIdx.x; e < nl * nrows; e += NT) {
    const int r = dnl.div(e), c = e - r * nl;
    int fy = row0 + r;
    fy -= fy >= mry ? mry : 0;
    out[obase[c] + (long long)fy * mrx * il] = a[(2 * c + (fy & 1)) * ld + (fy >> 1)];
  }
}

// lines per CTA: register FFT: 32 / L lines per warp, `rounds` passes of the 8 warps;
// Stockham: enough lines to keep the 256 threads busy.  Both within the smem budget.
size_t t2_per_line(int n, int xl) { return (xl ? 1 : 2) * (size_t)pf_ld(n) * sizeof(float2); }

int t2_cnt(int n, int xl, int rounds, int want_min) {
  const size_t per = t2_per_line(n, xl);
  int cnt = xl ? rounds * (T2_THREADS / 32) * (32 / xl) : (4 * T2_THREADS + n - 1) / n;
  if (cnt < want_min) cnt = want_min;
  const int fit = (int)(T2_SMEM / per);
  if (cnt > fit) cnt = fit;
  if (cnt > 64) cnt = 64;
  return cnt < 1 ? 1 : cnt;
}

template <typename K>
void t2_allow(K k) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T2_SMEM);
}

template <int XL>
void t2_allow_all() {
  t2_allow(k_t2_rows<XL>);
  t2_allow(k_t2_cols<XL>);
  if constexpr (XL > 0) {
    t2_allow(k_t2_rows_split<XL, 128>);
    t2_allow(k_t2_cols_split<XL, 128>);
    t2_allow(k_t2_rows_split<XL, 256>);
    t2_allow(k_t2_cols_split<XL, 256>);
  }
}

// PF_T2_SPLIT=0 keeps the full-length passes (A/B measurements)
int t2_split_L(int m) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("PF_T2_SPLIT");
    on = (e == nullptr || atoi(e) != 0) ? 1 : 0;
  }
  return on ? xfft_L(m) : 0;
}
// threads per CTA of the split passes (PF_T2_THREADS_ROWS / PF_T2_THREADS_COLS: 128 or 256)
int t2_split_threads(bool cols) {
  static int tr = -1, tc = -1;
  if (tr < 0) {
    const char* e = getenv("PF_T2_THREADS_ROWS");
    tr = (e && atoi(e) == 256) ? 256 : 128;
    e = getenv("PF_T2_THREADS_COLS");
    tc = (e && atoi(e) == 128) ? 128 : 256;
  }
  return cols ? tc : tr;
}
// fine lines per CTA: one round of the warps' 32 / L' half-lines each
int t2_split_cnt(int nt, int hl) {
  int cnt = (nt / 32) * (32 / hl) / 2;
  return cnt < 1 ? 1 : (cnt > 32 ? 32 : cnt);
}
size_t t2_split_smem(int m, int hl, int cnt) {   // lines + half-length twiddles + 1 / ker (m floats)
  return ((size_t)2 * cnt * pf_ld(m) + (size_t)XFFT_R * hl + (size_t)(m + 1) / 2) * sizeof(float2);
}
template <int HL, typename... A>
void t2_launch_rows_split(int nt, unsigned grid, size_t smem, cudaStream_t st, A... args) {
  if constexpr (HL > 0) {
    if (nt == 128) k_t2_rows_split<HL, 128><<<grid, 128, smem, st>>>(args...);
    else k_t2_rows_split<HL, 256><<<grid, 256, smem, st>>>(args...);
  }
}
template <int HL, typename... A>
void t2_launch_cols_split(int nt, unsigned grid, size_t smem, cudaStream_t st, A... args) {
  if constexpr (HL > 0) {
    if (nt == 128) k_t2_cols_split<HL, 128><<<grid, 128, smem, st>>>(args...);
    else k_t2_cols_split<HL, 256><<<grid, 256, smem, st>>>(args...);
  }
}

}  // namespace

extern "C" int pf_nufft_type2_start_2d_ilm(const pf_nufft_geom* g, const void* S,
                                           int64_t s_stride, const float* ky, const float* kx,
                                           int nv, void* fine, int64_t fine_stride,
                                           const pf_fft_plan* plan_x, const pf_fft_plan* plan_y,
                                           int col0, int ncols, int row0, int nrows, void* out,
                                           int il, int member, void* stream) {
  PF_ARG_CHECK(g && g->dim == 2 && g->mr[0] == 1 && nv >= 1 && plan_x && plan_y &&
                   plan_x->n == g->mr[2] && plan_y->n == g->mr[1] && g->m[2] <= g->mr[2] &&
                   g->m[1] <= g->mr[1],
               "pf_nufft_type2_start_2d: bad args (2D plan, plans of the fine-grid lengths)");
  PF_ARG_CHECK(S && fine && ky && kx, "pf_nufft_type2_start_2d: null buffer");
  PF_ARG_CHECK(col0 >= 0 && col0 < g->mr[2] && ncols >= 1 && ncols <= g->mr[2] && row0 >= 0 &&
                   row0 < g->mr[1] && nrows >= 1 && nrows <= g->mr[1],
               "pf_nufft_type2_start_2d_win: window outside the fine grid");
  PF_ARG_CHECK(out && il >= 1 && member < il && (il == 1 || member >= 0 || nv % il == 0),
               "pf_nufft_type2_start_2d_il: nv must be a multiple of the interleave");
  static PfDevOnce attr;
  if (attr.first()) {   // every instantiation: later calls may take other lengths
    for (int xl : {0, 4, 5, 8, 10, 15, 20, 30}) PF_XL_DISPATCH(xl, (t2_allow_all<XL>()));
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int xlx = plan_xl(*plan_x), xly = plan_xl(*plan_y);
  // split passes (two half-length register FFTs per fine line) when mr = 2 m = 70 L'
  const int hlx = g->mr[2] == 2 * g->m[2] ? t2_split_L(g->m[2]) : 0;
  const int hly = g->mr[1] == 2 * g->m[1] ? t2_split_L(g->m[1]) : 0;
  if (hlx) {
    const int nt = t2_split_threads(false);
    const int cnt = t2_split_cnt(nt, hlx);
    const long long nl = (long long)nv * g->m[1];
    const size_t smem = t2_split_smem(g->m[2], hlx, cnt);
    PF_XL_DISPATCH(hlx, (t2_launch_rows_split<XL>(nt, (unsigned)((nl + cnt - 1) / cnt), smem, st, *g,
                                                  (const float2*)S, s_stride, ky, kx, nv,
                                                  (float2*)fine, fine_stride, *plan_x, cnt,
                                                  hly ? col0 : 0, hly ? ncols : g->mr[2])));
    PF_LAUNCH_CHECK("k_t2_rows_split");
  } else {
    const int cnt = t2_cnt(g->mr[2], xlx, 1, 1);
    const long long nl = (long long)nv * g->m[1];
    const size_t smem = cnt * t2_per_line(g->mr[2], xlx);
    PF_XL_DISPATCH(xlx, (k_t2_rows<XL><<<(unsigned)((nl + cnt - 1) / cnt), T2_THREADS, smem, st>>>(
                             *g, (const float2*)S, s_stride, ky, kx, nv, (float2*)fine,
                             fine_stride, *plan_x, cnt)));
    PF_LAUNCH_CHECK("k_t2_rows");
  }
  if (hly) {
    const int nt = t2_split_threads(true);
    const int cnt = t2_split_cnt(nt, hly);
    const long long nl = (long long)nv * ncols;
    const size_t smem = t2_split_smem(g->m[1], hly, cnt);
    PF_XL_DISPATCH(hly, (t2_launch_cols_split<XL>(nt, (unsigned)((nl + cnt - 1) / cnt), smem, st, *g,
                                                  nv, (float2*)fine, fine_stride, *plan_y, cnt,
                                                  col0, ncols, row0, nrows, (float2*)out, il,
                                                  member)));
    PF_LAUNCH_CHECK("k_t2_cols_split");
  } else {
    PF_ARG_CHECK(il == 1 && out == fine,
                 "pf_nufft_type2_start_2d_il: interleaved output needs the split column pass "
                 "(mr = 2 m = 70 L)");
    // columns: >= 16 adjacent columns per CTA for 128-byte row segments
    const int cnt = t2_cnt(g->mr[1], xly, 2, 16);
    const long long nl = (long long)nv * g->mr[2];
    const size_t smem = cnt * t2_per_line(g->mr[1], xly);
    PF_XL_DISPATCH(xly, (k_t2_cols<XL><<<(unsigned)((nl + cnt - 1) / cnt), T2_THREADS, smem, st>>>(
                             *g, nv, (float2*)fine, fine_stride, *plan_y, cnt)));
    PF_LAUNCH_CHECK("k_t2_cols");
  }
  return 0;
}

extern "C" int pf_nufft_type2_start_2d_il(const pf_nufft_geom* g, const void* S,
                                          int64_t s_stride, const float* ky, const float* kx,
                                          int nv, void* fine, int64_t fine_stride,
                                          const pf_fft_plan* plan_x, const pf_fft_plan* plan_y,
                                          int col0, int ncols, int row0, int nrows, void* out,
                                          int il, void* stream) {
  return pf_nufft_type2_start_2d_ilm(g, S, s_stride, ky, kx, nv, fine, fine_stride, plan_x, plan_y,
                                     col0, ncols, row0, nrows, out, il, -1, stream);
}

extern "C" int pf_nufft_type2_start_2d_win(const pf_nufft_geom* g, const void* S,
                                           int64_t s_stride, const float* ky, const float* kx,
                                           int nv, void* fine, int64_t fine_stride,
                                           const pf_fft_plan* plan_x, const pf_fft_plan* plan_y,
                                           int col0, int ncols, int row0, int nrows,
                                           void* stream) {
  return pf_nufft_type2_start_2d_il(g, S, s_stride, ky, kx, nv, fine, fine_stride, plan_x, plan_y,
                                    col0, ncols, row0, nrows, fine, 1, stream);
}

// 1 when the column pass of this plan is split (interleaved output available)
extern "C" int pf_nufft_type2_il_ok(const pf_nufft_geom* g) {
  return g && g->dim == 2 && g->mr[1] == 2 * g->m[1] && t2_split_L(g->m[1]) > 0 ? 1 : 0;
}

extern "C" int pf_nufft_type2_start_2d(const pf_nufft_geom* g, const void* S, int64_t s_stride,
                                       const float* ky, const float* kx, int nv, void* fine,
                                       int64_t fine_stride, const pf_fft_plan* plan_x,
                                       const pf_fft_plan* plan_y, void* stream) {
  PF_ARG_CHECK(g, "pf_nufft_type2_start_2d: null geometry");
  return pf_nufft_type2_start_2d_win(g, S, s_stride, ky, kx, nv, fine, fine_stride, plan_x,
                                     plan_y, 0, g->mr[2], 0, g->mr[1], stream);
}
