// Whole-algorithm C entry point for nursd1 (reference reconstruct.py:335-385): scattered
// detections on one relay plane -> cuboid grid through a type-1 NUFFT of the relay
// coefficients onto the padded lattice's spectrum, then the rsd propagation.  The same
// plan and launch sequence as the Python engine (algorithms.Nursd1Engine +
// nufft.NufftPlan / NufftPoints / type1), in C++ behind the C-ABI.
//
//   pf_nursd1_workspace_bytes(args)            device scratch the call needs
//   pf_nursd1(args, slices, vol, ws, bytes, s) slices [F][I][n_points] c64 -> vol [frames][V]
//
// Host side: validation with the reference's messages; the pad (the reference rule
// next_fast_len(2 ceil(lag) + 10) when a detection is off the voxel lattice -- the
// result then depends on P, SURVEY F3 -- else the exact pad, F4); the NUFFT plan of
// reference NufftPlan (spectral.py:230-315: w = max(2, ceil(log10 1/eps) + 2), fine grid
// next_fast_len(max(2m, 2w + 2)), tau = pi w / (s (s - 1/2) m^2), the discrete
// deconvolution 1 + 2 sum_j exp(-(j h)^2 / 4 tau) cos(k j h)); the stencil anchors of
// spectral.py:281-303 and the tile buckets of the gather-spread kernel.  All of it is
// copied into the caller's workspace.  Device side: spreading, the type-1 finish (the
// register-path split FFT for square power-of-two modes with mr = 2m, else the pruned
// fine-grid FFT + deconvolution), then the propagation loop shared with pf_rsd.
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "nufft_host.cuh"

namespace {

using namespace pfalgo;

struct Plan {
  // propagation
  int px, py, batch, lanes;
  bool fast, horner;
  double dkhat;
  pf_prop_geom g;
  // NUFFT (modes (py, px), 2D)
  Nufft2Plan nu;
  std::vector<int32_t> i0, tstart, tpts;
  int win[4];   // col0, ncols, row0, nrows: fine cells the relay points' stencils touch
  std::vector<float> d0;
  // workspace
  int64_t n_tw[4];   // px, py, mry, mrx tables (0 = shared with an earlier one)
  int64_t off_tw[4], off_planes, off_ill, off_fw, off_ker[3], off_i0, off_d0, off_ts, off_tp,
      off_fine, off_rt, off_uhat, off_wa, off_wb, off_wo, total;
};

int fail(const char* msg) {
  pf_set_error("%s", msg);
  return -1;
}

int plan(const pf_nursd1_args* a, Plan* P) {
  if (!a || a->n_freq < 1 || a->n_illum < 1 || a->n_points < 1 || a->nx < 1 || a->ny < 1 ||
      a->nz < 1 || !a->frequencies || !a->ill_xyz || !a->relay_xy ||
      (a->n_frames > 0 && !a->times))
    return fail("pf_nursd1: bad arguments");
  for (int k = 0; k < a->nz; k++)
    if (!(a->z0 + k * a->dz > a->relay_z))
      return fail("every voxel plane must lie strictly beyond the relay plane");
  const int Lp = a->n_points;
  // fractional lattice indices of the detections about the grid centre
  const double cx = a->x0 + (a->nx / 2) * a->dx, cy = a->y0 + (a->ny / 2) * a->dy;
  std::vector<double> nux(Lp), nuy(Lp);
  double mnx = INFINITY, mxx = -INFINITY, mny = INFINITY, mxy = -INFINITY, ax = 0, ay = 0;
  bool on_lattice = true;
  for (int l = 0; l < Lp; l++) {
    const double x = a->relay_xy[2 * l], y = a->relay_xy[2 * l + 1];
    if (!(isfinite(x) && isfinite(y))) return fail("point coordinates must be finite");
    nux[l] = (x - cx) / a->dx;
    nuy[l] = (y - cy) / a->dy;
    mnx = fmin(mnx, nux[l]); mxx = fmax(mxx, nux[l]);
    mny = fmin(mny, nuy[l]); mxy = fmax(mxy, nuy[l]);
    ax = fmax(ax, fabs(nux[l])); ay = fmax(ay, fabs(nuy[l]));
    if (fabs(nux[l] - nearbyint(nux[l])) >= 1e-9 || fabs(nuy[l] - nearbyint(nuy[l])) >= 1e-9)
      on_lattice = false;
  }
  const int lo_x = -(a->nx / 2), hi_x = a->nx - a->nx / 2 - 1;
  const int lo_y = -(a->ny / 2), hi_y = a->ny - a->ny / 2 - 1;
  const double lx = fmax(hi_x - mnx, mxx - lo_x), ly = fmax(hi_y - mny, mxy - lo_y);
  const long px = on_lattice ? exact_pad(lx, fmax(ax, a->nx / 2), a->nx)
                             : ref_pad(lx, fmax(ax, a->nx / 2), a->nx);
  const long py = on_lattice ? exact_pad(ly, fmax(ay, a->ny / 2), a->ny)
                             : ref_pad(ly, fmax(ay, a->ny / 2), a->ny);
  int rad[PF_MAX_STAGES];
  if (radices(px, rad) < 0 || radices(py, rad) < 0) return fail("pf_nursd1: pad is not 11-smooth");
  P->px = (int)px;
  P->py = (int)py;
  // ---- NUFFT plan (nufft.NufftPlan, modes (py, px)), anchors and tile buckets
  if (nufft2_plan((int)py, (int)px, a->eps, &P->nu) != 0) return -1;
  {
    std::vector<double> tx(Lp), ty(Lp);
    for (int l = 0; l < Lp; l++) {
      tx[l] = 2.0 * M_PI * nux[l] / px;
      ty[l] = 2.0 * M_PI * nuy[l] / py;
    }
    if (nufft2_points(P->nu, tx.data(), ty.data(), Lp, false, &P->i0, &P->d0, nullptr) != 0)
      return -1;
  }
  nufft2_tiles(P->nu, P->i0, Lp, &P->tstart, &P->tpts);
  nufft2_stencil_window(P->nu, P->i0, Lp, P->win);
  const int mry = P->nu.g.mr[1], mrx = P->nu.g.mr[2];
  // ---- propagation geometry (algorithms._UhatPropEngine: centred output windows)
  pf_prop_geom& g = P->g;
  g = pf_prop_geom{};
  g.px = (int)px;
  g.py = (int)py;
  g.nx = a->nx;
  g.ny = a->ny;
  g.nu0x = -(a->nx / 2);
  g.nu0y = -(a->ny / 2);
  g.n_illum = a->n_illum;
  g.include_illum = a->include_illum ? 1 : 0;
  g.uhat_illum_stride = px * py;
  P->fast = pf_prop_fast(&g) != 0;
  P->batch = prop_batch(&g, a->nz, P->fast);
  const int nb = (a->nz + P->batch - 1) / P->batch;
  P->lanes = nb < LANES ? nb : LANES;
  const int F = a->n_freq, I = a->n_illum, frames = a->n_frames > 0 ? a->n_frames : 1;
  P->dkhat = 0.0;
  P->horner = horner_ok(&g, P->fast, a->frequencies, F, a->n_frames, a->include_illum, &P->dkhat);
  // ---- workspace layout
  const long lens[4] = {px, py, mry, mrx};
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
  P->off_planes = o; o = align256(o + (int64_t)sizeof(pf_plane) * a->nz);
  P->off_ill = o; o = align256(o + 8 * 3 * I);
  P->off_fw = o; o = align256(o + 8 * (int64_t)F * frames);
  for (int i = 0; i < 3; i++) {
    P->off_ker[i] = o;
    o = align256(o + 4 * (int64_t)P->nu.ker[i].size());
  }
  P->off_i0 = o; o = align256(o + 4 * (int64_t)P->i0.size());
  P->off_d0 = o; o = align256(o + 4 * (int64_t)P->d0.size());
  P->off_ts = o; o = align256(o + 4 * (int64_t)P->tstart.size());
  P->off_tp = o; o = align256(o + 4 * (int64_t)std::max<size_t>(1, P->tpts.size()));
  P->off_fine = o; o = align256(o + 8 * (int64_t)F * I * P->nu.fine_elems);
  P->off_rt = o;
  if (P->fast && P->nu.pow2_finish) o = align256(o + 8 * (int64_t)F * I * px * 2 * px);
  P->off_uhat = o; o = align256(o + 8 * (int64_t)F * I * px * py);
  P->off_wa = o; o = align256(o + 8 * P->lanes * pf_prop_ws_a(&g, P->batch));
  P->off_wb = o; o = align256(o + 8 * P->lanes * pf_prop_ws_b(&g, P->batch));
  P->off_wo = o;
  if (P->horner && F > HORNER_BLOCK)
    o = align256(o + 8 * (int64_t)P->lanes * P->batch * a->nx * a->ny);
  P->total = o;
  return 0;
}

#define UPLOAD(off, src, bytes)                                                          \
  PF_CUDA_CHECK(cudaMemcpyAsync(w + (off), (src), (bytes), cudaMemcpyHostToDevice, st), \
                "pf_nursd1: upload")

}  // namespace

extern "C" int pf_nufft_window(int mode) {
  int& w = pfalgo::nufft_window_ref();
  const int prev = w;
  if (mode == 0 || mode == 1) w = mode;
  return prev;
}

extern "C" int64_t pf_nursd1_workspace_bytes(const pf_nursd1_args* a) {
  Plan P;
  if (plan(a, &P) != 0) return -1;
  return P.total;
}

extern "C" int pf_nursd1(const pf_nursd1_args* a, const void* slices, void* vol, void* ws,
                         int64_t ws_bytes, void* stream) {
  Nvtx range("pf_nursd1");
  Plan P;
  if (plan(a, &P) != 0) return -1;
  PF_ARG_CHECK(slices && vol && ws && ws_bytes >= P.total,
               "pf_nursd1: null buffer or workspace smaller than pf_nursd1_workspace_bytes");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  const int F = a->n_freq, I = a->n_illum, frames = a->n_frames > 0 ? a->n_frames : 1;
  const int64_t V = (int64_t)a->nz * a->ny * a->nx;
  const int nv = F * I;
  // ---- tables (host, fp64 twiddles) -> workspace; plans px, py, mry, mrx
  const long lens[4] = {P.px, P.py, P.nu.g.mr[1], P.nu.g.mr[2]};
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
  std::vector<pf_plane> planes(a->nz);
  for (int k = 0; k < a->nz; k++) {
    const double z = a->z0 + k * a->dz;
    planes[k] = pf_plane{z - a->relay_z, a->dx, a->dy, a->x0, a->dx, a->y0, a->dy, z, 0, k};
  }
  UPLOAD(P.off_planes, planes.data(), sizeof(pf_plane) * a->nz);
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
  UPLOAD(P.off_ts, P.tstart.data(), 4 * P.tstart.size());
  if (!P.tpts.empty()) UPLOAD(P.off_tp, P.tpts.data(), 4 * P.tpts.size());
  PF_CUDA_CHECK(cudaMemsetAsync(vol, 0, 8 * (size_t)frames * V, st), "pf_nursd1: zero volume");
  // ---- type-1 NUFFT: Uhat[f][i] at the P x P centred modes (transposed on the register path)
  float2* fine = (float2*)(w + P.off_fine);
  float2* uhat = (float2*)(w + P.off_uhat);
  const float* kz = (const float*)(w + P.off_ker[0]);
  const float* ky = (const float*)(w + P.off_ker[1]);
  const float* kx = (const float*)(w + P.off_ker[2]);
  int rc = pf_nufft_spread(&P.nu.g, (const int32_t*)(w + P.off_i0), (const float*)(w + P.off_d0),
                           (const int32_t*)(w + P.off_ts), (const int32_t*)(w + P.off_tp), slices,
                           a->n_points, nv, fine, P.nu.fine_elems, stream);
  if (rc != 0) return rc;
  const int64_t out_stride = (int64_t)P.px * P.py;
  if (P.fast && P.nu.pow2_finish) {
    rc = pf_nufft_type1_finish_pow2(&P.nu.g, fine, P.nu.fine_elems, nv, w + P.off_rt, &pl[3], &pl[0],
                                    ky, kx, uhat, out_stride, stream);
  } else {
    // pruned fine-grid FFT (_device.fftn_pruned, outputs=True): every row along x, then
    // along y only the columns holding kept modes
    const int mry = P.nu.g.mr[1], mrx = P.nu.g.mr[2];
    // (x pass: only the rows the spreading touched; the other rows are zero and stay zero)
    const int r0 = P.win[2], nr = P.win[3];
    const int runs[2][2] = {{r0, r0 + nr <= mry ? nr : mry - r0}, {0, r0 + nr <= mry ? 0 : r0 + nr - mry}};
    for (int q = 0; q < 2 && rc == 0; q++)
      if (runs[q][1] > 0)
        rc = pf_fft_lines(fine + (int64_t)runs[q][0] * mrx, &pl[3], (int64_t)nv * runs[q][1],
                          runs[q][1], mrx, P.nu.fine_elems, 1, -1, 1.0f, stream);
    for (auto r : kept_ranges(P.px, mrx)) {
      if (rc != 0 || r.second == 0) continue;
      rc = pf_fft_lines(fine + r.first, &pl[2], (int64_t)nv * r.second, r.second, 1,
                        P.nu.fine_elems, mrx, -1, 1.0f, stream);
    }
    if (rc == 0)
      rc = pf_nufft_deconv(&P.nu.g, fine, P.nu.fine_elems, kz, ky, kx, nv, uhat, out_stride,
                           P.fast ? 1 : 0, stream);
  }
  if (rc != 0) return rc;
  PropLoop p{&P.g, &pl[0], &pl[1], (const pf_plane*)(w + P.off_planes), a->nz, P.batch, P.lanes,
             frames, (const double*)(w + P.off_ill), (const float2*)(w + P.off_fw), P.horner,
             P.dkhat, w + P.off_wa, w + P.off_wb,
             (P.horner && F > HORNER_BLOCK) ? w + P.off_wo : nullptr};
  return prop_loop(p, uhat, a->frequencies, F, vol, V, st);
}
