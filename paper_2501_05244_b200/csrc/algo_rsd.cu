// Whole-algorithm C entry point for rsd (reference reconstruct.py:208-268): the same
// plan and launch sequence as the Python engine (reconstruct.RsdEngine), in C++ behind
// the C-ABI, for a caller that binds the library directly.
//
//   pf_rsd_workspace_bytes(args)            device scratch the call needs
//   pf_rsd(args, slices, vol, ws, bytes, s) slices [F][I][ny*nx] c64 -> vol [frames][V] c64
//
// Host side: validation with the reference's messages, pad sizes (reference pad rule
// without the +8 margin, a power of two when within 1.6x: rsd is pad independent once no
// lag wraps), fp64 twiddle tables, plane specs, frame weights; all of it is copied into
// the caller's workspace.  Device side: relay spectra, then per plane batch and frequency
// the A / fused B / C kernels (Horner's rule in C when the geometry allows), with plane
// batches spread over three lanes (streams forked from and joined back to the caller's
// stream).  No allocation, no global mutable state; not capturable into a CUDA graph
// (the tables are uploaded from pageable host memory).
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "algo_host.cuh"

namespace {

using namespace pfalgo;

struct Layout {
  int px, py, nu0x, nu0y, batch, lanes;
  bool fast, horner;
  double dkhat;
  int64_t off_twx, off_twy, off_planes, off_ill, off_fw, off_uhat, off_wa, off_wb, off_wo, total;
  int64_t n_twx, n_twy;
};


// validation + plan; returns 0 or -1 with pf_set_error
int plan(const pf_rsd_args* a, Layout* L) {
  if (!a || a->n_freq < 1 || a->n_illum < 1 || a->relay_nx < 1 || a->relay_ny < 1 ||
      a->nx < 1 || a->ny < 1 || a->nz < 1 || !a->frequencies || !a->ill_xyz ||
      (a->n_frames > 0 && !a->times)) {
    pf_set_error("pf_rsd: bad arguments");
    return -1;
  }
  if (!(close_rel(a->dx, a->relay_dx) && close_rel(a->dy, a->relay_dy))) {
    pf_set_error("output lateral pitch must equal the relay pitch");
    return -1;
  }
  const double cx = a->relay_x0 + (a->relay_nx / 2) * a->relay_dx;
  const double cy = a->relay_y0 + (a->relay_ny / 2) * a->relay_dy;
  const double qx = (a->x0 - cx) / a->relay_dx, qy = (a->y0 - cy) / a->relay_dy;
  const double rx = nearbyint(qx), ry = nearbyint(qy);
  if (fabs(qx - rx) > 1e-9 * fmax(1.0, fabs(qx))) {
    pf_set_error("output grid x origin offset must be an integer multiple of the lattice pitch");
    return -1;
  }
  if (fabs(qy - ry) > 1e-9 * fmax(1.0, fabs(qy))) {
    pf_set_error("output grid y origin offset must be an integer multiple of the lattice pitch");
    return -1;
  }
  for (int k = 0; k < a->nz; k++)
    if (!(a->z0 + k * a->dz > a->relay_z)) {
      pf_set_error("every voxel plane must lie strictly beyond the relay plane");
      return -1;
    }
  const int nu0x = (int)rx, nu0y = (int)ry;
  const int gx = a->relay_nx, gy = a->relay_ny;
  const int jx_lo = -(gx / 2), jx_hi = gx - gx / 2 - 1, jy_lo = -(gy / 2), jy_hi = gy - gy / 2 - 1;
  const int nux_lo = nu0x, nux_hi = nu0x + a->nx - 1, nuy_lo = nu0y, nuy_hi = nu0y + a->ny - 1;
  long px, py;
  if (a->padding_none) {
    if (!(a->nx == gx && a->ny == gy && nu0x == jx_lo && nu0y == jy_lo)) {
      pf_set_error("padding='none' requires the output lattice to coincide with the relay "
                   "lattice");
      return -1;
    }
    px = gx;
    py = gy;
  } else {
    const double lx = fmax(abs(nux_lo - jx_hi), abs(nux_hi - jx_lo));
    const double ly = fmax(abs(nuy_lo - jy_hi), abs(nuy_hi - jy_lo));
    px = exact_pad(lx, fmax(fmax(abs(nux_lo), abs(nux_hi)), gx / 2), gx);
    py = exact_pad(ly, fmax(fmax(abs(nuy_lo), abs(nuy_hi)), gy / 2), gy);
  }
  int rad[PF_MAX_STAGES];
  if (radices(px, rad) < 0 || radices(py, rad) < 0) {
    pf_set_error("pf_rsd: pad is not 11-smooth");
    return -1;
  }
  pf_prop_geom g{};
  g.px = (int)px;
  g.py = (int)py;
  g.nx = a->nx;
  g.ny = a->ny;
  g.nu0x = nu0x;
  g.nu0y = nu0y;
  g.n_illum = a->n_illum;
  g.include_illum = a->include_illum ? 1 : 0;
  g.uhat_illum_stride = px * py;
  L->px = (int)px;
  L->py = (int)py;
  L->nu0x = nu0x;
  L->nu0y = nu0y;
  L->fast = pf_prop_fast(&g) != 0;
  L->batch = prop_batch(&g, a->nz, L->fast);
  const int nb = (a->nz + L->batch - 1) / L->batch;
  L->lanes = nb < LANES ? nb : LANES;
  const int F = a->n_freq;
  L->dkhat = 0.0;
  L->horner = horner_ok(&g, L->fast, a->frequencies, F, a->n_frames, a->include_illum, &L->dkhat);
  const int batch = L->batch;
  const int frames = a->n_frames > 0 ? a->n_frames : 1;
  L->n_twx = (int64_t)twiddles(px).size();
  L->n_twy = py == px ? 0 : (int64_t)twiddles(py).size();
  int64_t o = 0;
  L->off_twx = o; o = align256(o + 8 * L->n_twx);
  L->off_twy = o; o = align256(o + 8 * L->n_twy);
  L->off_planes = o; o = align256(o + (int64_t)sizeof(pf_plane) * a->nz);
  L->off_ill = o; o = align256(o + 8 * 3 * a->n_illum);
  L->off_fw = o; o = align256(o + 8 * (int64_t)F * frames);
  L->off_uhat = o; o = align256(o + 8 * (int64_t)F * a->n_illum * px * py);
  L->off_wa = o; o = align256(o + 8 * L->lanes * pf_prop_ws_a(&g, batch));
  L->off_wb = o; o = align256(o + 8 * L->lanes * pf_prop_ws_b(&g, batch));
  L->off_wo = o;
  if (L->horner && F > HORNER_BLOCK) o = align256(o + 8 * (int64_t)L->lanes * batch * a->nx * a->ny);
  L->total = o;
  return 0;
}

}  // namespace

extern "C" int64_t pf_rsd_workspace_bytes(const pf_rsd_args* a) {
  Layout L;
  if (plan(a, &L) != 0) return -1;
  return L.total;
}

extern "C" int pf_rsd(const pf_rsd_args* a, const void* slices, void* vol, void* ws,
                      int64_t ws_bytes, void* stream) {
  Nvtx range("pf_rsd");
  Layout L;
  if (plan(a, &L) != 0) return -1;
  PF_ARG_CHECK(slices && vol && ws && ws_bytes >= L.total,
               "pf_rsd: null buffer or workspace smaller than pf_rsd_workspace_bytes");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  const int F = a->n_freq, I = a->n_illum, frames = a->n_frames > 0 ? a->n_frames : 1;
  const int64_t V = (int64_t)a->nz * a->ny * a->nx;
  // ---- tables (host, fp64) -> workspace
  pf_fft_plan plx{}, ply{};
  {
    std::vector<float2> tx = twiddles(L.px);
    PF_CUDA_CHECK(cudaMemcpyAsync(w + L.off_twx, tx.data(), 8 * tx.size(),
                                  cudaMemcpyHostToDevice, st), "pf_rsd: upload");
    plx.n = L.px;
    plx.nst = radices(L.px, plx.radix);
    plx.tw = w + L.off_twx;
    if (L.n_twx > L.px && !(L.px == 128 || L.px == 256 || L.px == 512 || L.px == 1024))
      plx.radix[PF_MAX_STAGES - 1] = PF_XFFT_TAG;
    if (L.py != L.px) {
      std::vector<float2> ty = twiddles(L.py);
      PF_CUDA_CHECK(cudaMemcpyAsync(w + L.off_twy, ty.data(), 8 * ty.size(),
                                    cudaMemcpyHostToDevice, st), "pf_rsd: upload");
      ply.n = L.py;
      ply.nst = radices(L.py, ply.radix);
      ply.tw = w + L.off_twy;
      if (L.n_twy > L.py && !(L.py == 128 || L.py == 256 || L.py == 512 || L.py == 1024))
        ply.radix[PF_MAX_STAGES - 1] = PF_XFFT_TAG;
    } else {
      ply = plx;
    }
  }
  std::vector<pf_plane> planes(a->nz);
  for (int k = 0; k < a->nz; k++) {
    const double z = a->z0 + k * a->dz;
    planes[k] = pf_plane{z - a->relay_z, a->relay_dx, a->relay_dy, a->x0, a->dx, a->y0, a->dy,
                         z, 0, k};
  }
  PF_CUDA_CHECK(cudaMemcpyAsync(w + L.off_planes, planes.data(), sizeof(pf_plane) * a->nz,
                                cudaMemcpyHostToDevice, st), "pf_rsd: upload");
  PF_CUDA_CHECK(cudaMemcpyAsync(w + L.off_ill, a->ill_xyz, 8 * 3 * I, cudaMemcpyHostToDevice, st),
                "pf_rsd: upload");
  std::vector<float2> fw((size_t)F * frames);
  for (int f = 0; f < F; f++)
    for (int j = 0; j < frames; j++) {
      const double ph = a->n_frames > 0 ? a->frequencies[f] * a->times[j] : 0.0;
      fw[(size_t)f * frames + j] = make_float2((float)cos(ph), (float)sin(ph));
    }
  PF_CUDA_CHECK(cudaMemcpyAsync(w + L.off_fw, fw.data(), 8 * fw.size(), cudaMemcpyHostToDevice, st),
                "pf_rsd: upload");
  PF_CUDA_CHECK(cudaMemsetAsync(vol, 0, 8 * (size_t)frames * V, st), "pf_rsd: zero volume");

  pf_prop_geom g{};
  g.px = L.px;
  g.py = L.py;
  g.nx = a->nx;
  g.ny = a->ny;
  g.nu0x = L.nu0x;
  g.nu0y = L.nu0y;
  g.n_illum = I;
  g.include_illum = a->include_illum ? 1 : 0;
  g.uhat_illum_stride = (int64_t)L.px * L.py;
  float2* uhat = (float2*)(w + L.off_uhat);
  // ---- relay spectra Uhat_f = cfft2(pad_embed(u_f)) (transposed on the register path)
  int rc;
  if (L.fast) {
    rc = pf_relay_spectra_fast(slices, (int64_t)F * I, a->relay_ny, a->relay_nx,
                               (int64_t)a->relay_ny * a->relay_nx, uhat, L.px, &plx, stream);
  } else {
    rc = pf_embed_centered(slices, (int64_t)F * I, a->relay_ny, a->relay_nx,
                           (int64_t)a->relay_ny * a->relay_nx, uhat, L.py, L.px, 0, stream);
    if (rc == 0)
      rc = pf_fft_lines(uhat, &plx, (int64_t)F * I * L.py, 1, 0, L.px, 1, -1, 1.0f, stream);
    if (rc == 0)
      rc = pf_fft_lines(uhat, &ply, (int64_t)F * I * L.px, L.px, 1, (int64_t)L.py * L.px, L.px,
                        -1, 1.0f, stream);
  }
  if (rc != 0) return rc;
  PropLoop p{&g, &plx, &ply, (const pf_plane*)(w + L.off_planes), a->nz, L.batch, L.lanes,
             frames, (const double*)(w + L.off_ill), (const float2*)(w + L.off_fw), L.horner,
             L.dkhat, w + L.off_wa, w + L.off_wb,
             (L.horner && F > HORNER_BLOCK) ? w + L.off_wo : nullptr};
  return prop_loop(p, uhat, a->frequencies, F, vol, V, st);
}
