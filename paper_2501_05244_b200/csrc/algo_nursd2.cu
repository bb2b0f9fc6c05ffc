// Whole-algorithm C entry point for nursd2 (reference reconstruct.py:413-459): detections
// on a uniform relay lattice -> explicit voxels on planes of constant depth, through the
// relay spectra, the per-plane product with the kernel spectrum and a type-2 NUFFT read
// out at each plane's voxels.  The same plan and launch sequence as the Python engine
// (algorithms.Nursd2Engine + _Type2Readout), in C++ behind the C-ABI.
//
//   pf_nursd2_workspace_bytes(args)            device scratch the call needs
//   pf_nursd2(args, slices, vol, ws, bytes, s) slices [F][I][ny*nx] c64 -> vol [frames][N]
//
// Host side: validation with the reference's messages; the reference pad rule (the
// voxels' fractional lattice indices make the result depend on it, reconstruct.py:425-433);
// the NufftPlan (nufft_host.cuh); every plane's voxels cell-sorted within the plane and
// concatenated in plane order, each carrying (x, y, z), its plane and its output slot;
// all of it copied into the caller's workspace.  Device side: relay spectra (embed +
// natural-order 2D FFT), then per frequency and plane batch: kernel rows, product-only
// columns (Uhat * Ghat_k), the fused place / deconvolution + inverse fine-grid FFT
// (pf_nufft_type2_start_2d) and one interpolation launch for the batch's voxels (scale
// 1 / (px py), illumination phase at each voxel, frame weights).
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "nufft_host.cuh"

namespace {

using namespace pfalgo;

constexpr int64_t READOUT_BYTES = 256LL << 20;   // algorithms._READOUT_BYTES
constexpr int64_t READOUT_FUSED_BYTES = 2048LL << 20;   // algorithms._READOUT_FUSED_BYTES

struct Plan {
  int px, py, nb;
  int64_t n_vox;
  pf_prop_geom g;
  Nufft2Plan nu;
  std::vector<int32_t> i0, plane;
  std::vector<float> d0;
  std::vector<double> xyz;
  std::vector<int64_t> dst, pt_lo;
  int win[4];        // col0, ncols, row0, nrows: the fine cells the voxels' stencils touch
  bool fused;        // readout over all frequencies per launch (frequency-interleaved grids)
  int n_groups;      // groups of 16 frequencies
  int64_t off_fine_f, off_kturns;
  int64_t n_tw[4];   // px, py, mry, mrx tables (0 = shared with an earlier one)
  int64_t off_tw[4], off_planes, off_ill, off_fw, off_ker[3], off_i0, off_d0, off_xyz, off_pl,
      off_dst, off_uhat, off_wa, off_spec, off_fine, total;
};

int fail(const char* msg) {
  pf_set_error("%s", msg);
  return -1;
}

int plan(const pf_nursd2_args* a, Plan* P) {
  if (!a || a->n_freq < 1 || a->n_illum < 1 || a->relay_nx < 1 || a->relay_ny < 1 ||
      a->n_planes < 1 || !a->plane_z || !a->plane_count || !a->voxel_xy || !a->frequencies ||
      !a->ill_xyz || (a->n_frames > 0 && !a->times))
    return fail("pf_nursd2: bad arguments");
  for (int k = 0; k < a->n_planes; k++)
    if (!(a->plane_z[k] > a->relay_z))
      return fail("every voxel plane must lie strictly beyond the relay plane");
  int64_t N = 0;
  for (int k = 0; k < a->n_planes; k++) {
    if (a->plane_count[k] < 0) return fail("pf_nursd2: negative plane count");
    N += a->plane_count[k];
  }
  if (N < 1) return fail("pf_nursd2: no voxels");
  P->n_vox = N;
  // fractional lattice indices about the relay centre (reconstruct.py:393-410)
  const double cx = a->relay_x0 + (a->relay_nx / 2) * a->relay_dx;
  const double cy = a->relay_y0 + (a->relay_ny / 2) * a->relay_dy;
  std::vector<double> nux(N), nuy(N);
  double mnx = INFINITY, mxx = -INFINITY, mny = INFINITY, mxy = -INFINITY, ax = 0, ay = 0;
  for (int64_t l = 0; l < N; l++) {
    const double x = a->voxel_xy[2 * l], y = a->voxel_xy[2 * l + 1];
    if (!(isfinite(x) && isfinite(y))) return fail("point coordinates must be finite");
    nux[l] = (x - cx) / a->relay_dx;
    nuy[l] = (y - cy) / a->relay_dy;
    mnx = fmin(mnx, nux[l]); mxx = fmax(mxx, nux[l]);
    mny = fmin(mny, nuy[l]); mxy = fmax(mxy, nuy[l]);
    ax = fmax(ax, fabs(nux[l])); ay = fmax(ay, fabs(nuy[l]));
  }
  const int gx = a->relay_nx, gy = a->relay_ny;
  const int jx_lo = -(gx / 2), jx_hi = gx - gx / 2 - 1, jy_lo = -(gy / 2), jy_hi = gy - gy / 2 - 1;
  const long px = ref_pad(fmax(mxx - jx_lo, jx_hi - mnx), fmax(ax, gx / 2), gx);
  const long py = ref_pad(fmax(mxy - jy_lo, jy_hi - mny), fmax(ay, gy / 2), gy);
  int rad[PF_MAX_STAGES];
  if (radices(px, rad) < 0 || radices(py, rad) < 0) return fail("pf_nursd2: pad is not 11-smooth");
  P->px = (int)px;
  P->py = (int)py;
  if (nufft2_plan((int)py, (int)px, a->eps, &P->nu) != 0) return -1;
  const int I = a->n_illum, F = a->n_freq, frames = a->n_frames > 0 ? a->n_frames : 1;
  // voxels plane by plane, cell-sorted within the plane
  P->pt_lo.assign(1, 0);
  int64_t start = 0;
  for (int k = 0; k < a->n_planes; k++) {
    const int64_t cnt = a->plane_count[k];
    std::vector<double> tx(cnt), ty(cnt);
    for (int64_t l = 0; l < cnt; l++) {
      tx[l] = 2.0 * M_PI * nux[start + l] / px;
      ty[l] = 2.0 * M_PI * nuy[start + l] / py;
    }
    std::vector<int64_t> order;
    if (nufft2_points(P->nu, tx.data(), ty.data(), cnt, true, &P->i0, &P->d0, &order) != 0)
      return -1;
    for (int64_t o : order) {
      P->xyz.push_back(a->voxel_xy[2 * (start + o)]);
      P->xyz.push_back(a->voxel_xy[2 * (start + o) + 1]);
      P->xyz.push_back(a->plane_z[k]);
      P->plane.push_back(k);
      P->dst.push_back(start + o);
    }
    start += cnt;
    P->pt_lo.push_back(start);
  }
  nufft2_stencil_window(P->nu, P->i0, N, P->win);
  // product-only propagation geometry over the whole pad (reconstruct.py:441-449)
  pf_prop_geom& g = P->g;
  g = pf_prop_geom{};
  g.px = (int)px;
  g.py = (int)py;
  g.nx = (int)px;
  g.ny = (int)py;
  g.n_illum = I;
  g.include_illum = a->include_illum ? 1 : 0;
  g.flags = 1;   // register path off: generic product-only columns
  g.uhat_illum_stride = px * py;
  const int64_t per_plane = 8 * (int64_t)I * (P->nu.fine_elems + px * py);
  int64_t nb = READOUT_BYTES / per_plane;
  if (nb > a->n_planes) nb = a->n_planes;
  // algorithms._Type2Readout.fused_f: ES window at w = 4, one illumination, static scene,
  // split column pass -> one readout launch per plane batch over all frequencies
  P->n_groups = (F + 15) / 16;
  P->fused = P->nu.g.window == 1 && P->nu.g.w == 4 && I == 1 && a->n_frames <= 0 &&
             P->nu.fine_elems * 16 < (1LL << 31) && pf_nufft_type2_il_ok(&P->nu.g) &&
             !(getenv("PF_READOUT_FUSED") && atoi(getenv("PF_READOUT_FUSED")) == 0);
  if (P->fused) {
    const int64_t per_f = 8LL * 16 * P->n_groups * P->nu.fine_elems;
    const int64_t cap = READOUT_FUSED_BYTES / per_f;
    if (nb > cap) nb = cap;
  }
  P->nb = nb < 1 ? 1 : (int)nb;
  // workspace layout
  const long lens[4] = {px, py, P->nu.g.mr[1], P->nu.g.mr[2]};
  for (int i = 0; i < 4; i++) {
    P->n_tw[i] = (int64_t)twiddles(lens[i]).size();
    for (int j = 0; j < i; j++)
      if (lens[j] == lens[i]) P->n_tw[i] = 0;
  }
  int64_t o = 0;
  for (int i = 0; i < 4; i++) {
    P->off_tw[i] = o;
    o = align256(o + 8 * P->n_tw[i]);
  }
  P->off_planes = o; o = align256(o + (int64_t)sizeof(pf_plane) * a->n_planes);
  P->off_ill = o; o = align256(o + 8 * 3 * I);
  P->off_fw = o; o = align256(o + 8 * (int64_t)F * frames);
  for (int i = 0; i < 3; i++) {
    P->off_ker[i] = o;
    o = align256(o + 4 * (int64_t)P->nu.ker[i].size());
  }
  P->off_i0 = o; o = align256(o + 4 * (int64_t)P->i0.size());
  P->off_d0 = o; o = align256(o + 4 * (int64_t)P->d0.size());
  P->off_xyz = o; o = align256(o + 8 * (int64_t)P->xyz.size());
  P->off_pl = o; o = align256(o + 4 * (int64_t)P->plane.size());
  P->off_dst = o; o = align256(o + 8 * (int64_t)P->dst.size());
  P->off_uhat = o; o = align256(o + 8 * (int64_t)F * I * px * py);
  P->off_wa = o; o = align256(o + 8 * pf_prop_ws_a(&g, P->nb));
  P->off_spec = o; o = align256(o + 8 * (int64_t)P->nb * I * px * py);
  P->off_fine = o; o = align256(o + 8 * (int64_t)P->nb * I * P->nu.fine_elems);
  P->off_fine_f = o;
  if (P->fused) o = align256(o + 8LL * 16 * P->n_groups * P->nb * P->nu.fine_elems);
  P->off_kturns = o; o = align256(o + 8 * (int64_t)F);
  P->total = o;
  return 0;
}

#define UPLOAD(off, src, bytes)                                                          \
  PF_CUDA_CHECK(cudaMemcpyAsync(w + (off), (src), (bytes), cudaMemcpyHostToDevice, st), \
                "pf_nursd2: upload")

}  // namespace

extern "C" int64_t pf_nursd2_workspace_bytes(const pf_nursd2_args* a) {
  Plan P;
  if (plan(a, &P) != 0) return -1;
  return P.total;
}

extern "C" int pf_nursd2(const pf_nursd2_args* a, const void* slices, void* vol, void* ws,
                         int64_t ws_bytes, void* stream) {
  Nvtx range("pf_nursd2");
  Plan P;
  if (plan(a, &P) != 0) return -1;
  PF_ARG_CHECK(slices && vol && ws && ws_bytes >= P.total,
               "pf_nursd2: null buffer or workspace smaller than pf_nursd2_workspace_bytes");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  const int F = a->n_freq, I = a->n_illum, frames = a->n_frames > 0 ? a->n_frames : 1;
  const int px = P.px, py = P.py;
  const int mry = P.nu.g.mr[1], mrx = P.nu.g.mr[2];
  const int64_t fe = P.nu.fine_elems;
  // ---- tables -> workspace; plans px, py, mry, mrx
  const long lens[4] = {px, py, mry, mrx};
  pf_fft_plan pl[4];
  for (int i = 0; i < 4; i++) {
    int src = i;
    for (int j = 0; j < i; j++)
      if (lens[j] == lens[i]) {
        src = j;
        break;
      }
    if (src == i) {
      std::vector<float2> t = twiddles(lens[i]);
      UPLOAD(P.off_tw[i], t.data(), 8 * t.size());
      pl[i] = make_plan(lens[i], w + P.off_tw[i], t.size());
    } else {
      pl[i] = pl[src];
    }
  }
  std::vector<pf_plane> planes(a->n_planes);
  for (int k = 0; k < a->n_planes; k++)
    planes[k] = pf_plane{a->plane_z[k] - a->relay_z, a->relay_dx, a->relay_dy, 0.0, 1.0, 0.0, 1.0,
                         a->plane_z[k], 0, k};
  UPLOAD(P.off_planes, planes.data(), sizeof(pf_plane) * a->n_planes);
  UPLOAD(P.off_ill, a->ill_xyz, 8 * 3 * I);
  std::vector<float2> fw((size_t)F * frames);
  for (int f = 0; f < F; f++)
    for (int j = 0; j < frames; j++) {
      const double ph = a->n_frames > 0 ? a->frequencies[f] * a->times[j] : 0.0;
      fw[(size_t)f * frames + j] = make_float2((float)cos(ph), (float)sin(ph));
    }
  UPLOAD(P.off_fw, fw.data(), 8 * fw.size());
  for (int i = 0; i < 3; i++) UPLOAD(P.off_ker[i], P.nu.ker[i].data(), 4 * P.nu.ker[i].size());
  UPLOAD(P.off_i0, P.i0.data(), 4 * P.i0.size());
  UPLOAD(P.off_d0, P.d0.data(), 4 * P.d0.size());
  UPLOAD(P.off_xyz, P.xyz.data(), 8 * P.xyz.size());
  UPLOAD(P.off_pl, P.plane.data(), 4 * P.plane.size());
  UPLOAD(P.off_dst, P.dst.data(), 8 * P.dst.size());
  PF_CUDA_CHECK(cudaMemsetAsync(vol, 0, 8 * (size_t)frames * P.n_vox, st), "pf_nursd2: zero volume");
  // ---- relay spectra Uhat_f = cfft2(pad_embed(u_f)), natural order (reconstruct.py:441-443)
  float2* uhat = (float2*)(w + P.off_uhat);
  int rc = pf_embed_centered(slices, (int64_t)F * I, a->relay_ny, a->relay_nx,
                             (int64_t)a->relay_ny * a->relay_nx, uhat, py, px, 0, stream);
  if (rc == 0) rc = pf_fft_lines(uhat, &pl[0], (int64_t)F * I * py, 1, 0, px, 1, -1, 1.0f, stream);
  if (rc == 0)
    rc = pf_fft_lines(uhat, &pl[1], (int64_t)F * I * px, px, 1, (int64_t)py * px, px, -1, 1.0f,
                      stream);
  if (rc != 0) return rc;
  const pf_plane* planes_d = (const pf_plane*)(w + P.off_planes);
  const float* ky = (const float*)(w + P.off_ker[1]);
  const float* kx = (const float*)(w + P.off_ker[2]);
  float2* wa = (float2*)(w + P.off_wa);
  float2* spec = (float2*)(w + P.off_spec);
  float2* fine = (float2*)(w + P.off_fine);
  const int64_t per_f = (int64_t)I * px * py;
  if (P.fused) {
    // per plane batch: every frequency's product spectra and type-2 start into the
    // frequency-interleaved fine grids, then one readout launch over all frequencies
    float2* fine_f = (float2*)(w + P.off_fine_f);
    const int64_t gstride = (int64_t)P.nb * fe * 16;
    std::vector<double> kt(F);
    for (int f = 0; f < F; f++) kt[f] = a->frequencies[f] / C_LIGHT / (2.0 * M_PI);
    UPLOAD(P.off_kturns, kt.data(), 8 * (size_t)F);
    if (F % 16)   // the unused frequency slots of the last group are read: zero them
      PF_CUDA_CHECK(cudaMemsetAsync(fine_f + (int64_t)(P.n_groups - 1) * gstride, 0,
                                    8 * (size_t)gstride, st),
                    "pf_nursd2: zero fine grids");
    for (int b0 = 0; b0 < a->n_planes && rc == 0; b0 += P.nb) {
      const int n = a->n_planes - b0 < P.nb ? a->n_planes - b0 : P.nb;
      const pf_plane* pp = planes_d + b0;
      for (int f = 0; f < F && rc == 0; f++) {
        const double khat = a->frequencies[f] / C_LIGHT;
        rc = pf_prop_kernel_rows(pp, n, khat, &P.g, &pl[0], wa, stream);
        if (rc == 0)
          rc = pf_prop_columns(pp, n, &P.g, &pl[1], wa, uhat + f * per_f, spec, 1, stream);
        if (rc == 0)
          rc = pf_nufft_type2_start_2d_ilm(&P.nu.g, spec, (int64_t)py * px, ky, kx, n, fine, fe,
                                           &pl[3], &pl[2], P.win[0], P.win[1], P.win[2],
                                           P.win[3], fine_f + (int64_t)(f / 16) * gstride, 16,
                                           f % 16, stream);
      }
      const int64_t lo = P.pt_lo[b0], hi = P.pt_lo[b0 + n];
      if (rc == 0 && hi > lo)
        rc = pf_nufft_interp2_freqs(
            &P.nu.g, (const int32_t*)(w + P.off_i0) + 3 * lo, (const float*)(w + P.off_d0) + 3 * lo,
            (const double*)(w + P.off_xyz) + 3 * lo, (const int32_t*)(w + P.off_pl) + lo,
            (const int64_t*)(w + P.off_dst) + lo, (int)(hi - lo), b0, fine_f, fe * 16, gstride, F,
            (const double*)(w + P.off_kturns), (const double*)(w + P.off_ill),
            a->include_illum ? 1 : 0, (float)(1.0 / ((double)px * py)),
            (const float2*)(w + P.off_fw), vol, stream);
    }
    return rc;
  }
  for (int f = 0; f < F && rc == 0; f++) {
    const double khat = a->frequencies[f] / C_LIGHT;
    for (int b0 = 0; b0 < a->n_planes && rc == 0; b0 += P.nb) {
      const int n = a->n_planes - b0 < P.nb ? a->n_planes - b0 : P.nb;
      const pf_plane* pp = planes_d + b0;
      const int nv = n * I;
      rc = pf_prop_kernel_rows(pp, n, khat, &P.g, &pl[0], wa, stream);
      if (rc == 0) rc = pf_prop_columns(pp, n, &P.g, &pl[1], wa, uhat + f * per_f, spec, 1, stream);
      // type-2 first half (spectral.py:373-375): place (spectrum / deconvolution) and the
      // inverse fine-grid FFT, fused (pf_nufft_type2_start_2d)
      if (rc == 0)
        rc = pf_nufft_type2_start_2d_win(&P.nu.g, spec, (int64_t)py * px, ky, kx, nv, fine, fe,
                                         &pl[3], &pl[2], P.win[0], P.win[1], P.win[2], P.win[3],
                                         stream);
      const int64_t lo = P.pt_lo[b0], hi = P.pt_lo[b0 + n];
      if (rc == 0 && hi > lo)
        rc = pf_nufft_interp2_batch(
            &P.nu.g, (const int32_t*)(w + P.off_i0) + 3 * lo, (const float*)(w + P.off_d0) + 3 * lo,
            (const double*)(w + P.off_xyz) + 3 * lo, (const int32_t*)(w + P.off_pl) + lo,
            (const int64_t*)(w + P.off_dst) + lo, (int)(hi - lo), b0, fine, I * fe, fe, I,
            (const double*)(w + P.off_ill), khat, a->include_illum ? 1 : 0,
            (float)(1.0 / ((double)px * py)), (const float2*)(w + P.off_fw) + (int64_t)f * frames,
            frames, vol, P.n_vox, stream);
    }
  }
  return rc;
}
