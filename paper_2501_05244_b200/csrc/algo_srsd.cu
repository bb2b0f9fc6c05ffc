// Whole-algorithm C entry point for srsd (reference reconstruct.py:276-327): the plan and
// launch sequence of the Python engine (algorithms.SrsdEngine) behind one C call.
//
//   pf_srsd_workspace_bytes(args)             device scratch the call needs
//   pf_srsd(args, slices, vol, ws, bytes, s)  slices [F][I][ny*nx] c64 -> vol [frames][V] c64
//
// Host side: the reference's validation (frustum base = relay lattice, planes beyond the
// relay), P = next_fast_len(2N) (the SRSD result depends on it), Q =
// next_fast_len(2P - 1), fp64 twiddle tables, plane specs (kernel lag pitch dx / alpha_k,
// output pitch dx / alpha_k about the base centre, reconstruct.py:307-308 and core.py
// FrustumGrid.plane_xy), frame weights.  Device side: the per-plane scaled-FFT tables
// (chirps exp(-i pi a (n - o)^2 / M) with float64 phases, and the Q-point FFT of the
// embedded kernel exp(+i pi a l^2 / M), reference spectral.py:143-158), then per plane
// batch and frequency the Bluestein x / y passes into the batch's spectra and the A /
// fused B / C propagation (Horner's rule in C where eligible), plane batches on three lanes
// forked from and joined back to the caller's stream.  No allocation, no global state.
#include "algo_host.cuh"

namespace {

using namespace pfalgo;

constexpr int64_t SRSD_BATCH_BYTES = 96LL << 20;
constexpr int SRSD_MINQ = 8;

// chirp[b][n] = exp(-i pi a_b (n - o)^2 / M) (n < M); kern[b][q] = exp(+i pi a_b l^2 / M)
// at q = l mod Q for |l| < M, else 0.  Phases in float64 (up to ~pi M), reduced before the
// float32 sincos (common.cuh expi_reduced).
__global__ void k_srsd_tables(int M, int Q, int o, const double* __restrict__ scale, int nplanes,
                              float2* __restrict__ chirp, float2* __restrict__ kern) {
  const long long total = (long long)nplanes * (M + Q);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e / (M + Q));
    const int j = (int)(e - (long long)b * (M + Q));
    const double a = scale[b];
    if (j < M) {
      const double n = (double)(j - o);
      chirp[(long long)b * M + j] = expi_reduced(-M_PI * a * n * n / (double)M);
    } else {
      const int q = j - M;
      // lag l with l mod Q == q and |l| < M: l = q (q < M) or l = q - Q (q > Q - M)
      float2 v = make_float2(0.f, 0.f);
      if (q < M) {
        v = expi_reduced(M_PI * a * (double)q * (double)q / (double)M);
      } else if (q > Q - M) {
        const double l = (double)(q - Q);
        v = expi_reduced(M_PI * a * l * l / (double)M);
      }
      kern[(long long)b * Q + q] = v;
    }
  }
}

struct SLayout {
  int px, py, qx, qy, batch, lanes, nb_batches;
  bool fast, bwarp, horner;
  double dkhat;
  int64_t off_tw[4], n_tw[4];   // plans px, py, qx, qy
  int64_t off_planes, off_ill, off_fw, off_sc, off_chx, off_khx, off_chy, off_khy;
  int64_t off_uhat, off_xbuf, off_wa, off_wb, off_wo, total;
};

int splan(const pf_srsd_args* a, SLayout* L) {
  if (!a || a->n_freq < 1 || a->n_illum < 1 || a->nx < 1 || a->ny < 1 || a->nz < 1 ||
      !a->frequencies || !a->ill_xyz || !a->zs || !a->alphas || !a->betas ||
      (a->n_frames > 0 && !a->times)) {
    pf_set_error("pf_srsd: bad arguments");
    return -1;
  }
  for (int k = 0; k < a->nz; k++) {
    if (!(a->zs[k] > a->relay_z)) {
      pf_set_error("every voxel plane must lie strictly beyond the relay plane");
      return -1;
    }
    if (!(a->alphas[k] > 0 && a->betas[k] > 0)) {
      pf_set_error("frustum scale factors must be > 0");
      return -1;
    }
  }
  const long px = next_fast_len(2L * a->nx), py = next_fast_len(2L * a->ny);
  const long qx = next_fast_len(2 * px - 1), qy = next_fast_len(2 * py - 1);
  L->px = (int)px;
  L->py = (int)py;
  L->qx = (int)qx;
  L->qy = (int)qy;
  pf_prop_geom g{};
  g.px = (int)px;
  g.py = (int)py;
  g.nx = a->nx;
  g.ny = a->ny;
  g.nu0x = -(a->nx / 2);
  g.nu0y = -(a->ny / 2);
  g.n_illum = a->n_illum;
  g.include_illum = a->include_illum ? 1 : 0;
  g.uhat_illum_stride = px * py;
  L->fast = pf_prop_fast(&g) != 0;
  auto pow2 = [](long n) { return n == 128 || n == 256 || n == 512 || n == 1024; };
  L->bwarp = L->fast && pow2(qx) && pow2(qy);
  const int I = a->n_illum;
  const int64_t per = 8 * (2LL * I * py * px + (int64_t)I * a->ny * px);
  int batch = (int)fmax(1.0, fmin((double)a->nz, (double)(SRSD_BATCH_BYTES / per)));
  if (L->fast) {
    const int q = SRSD_MINQ * (32 / (int)(px / 32));
    int b = (batch / q) * q;
    batch = b < q ? q : b;
    if (batch > a->nz) batch = a->nz;
  }
  L->batch = batch;
  L->nb_batches = (a->nz + batch - 1) / batch;
  L->lanes = L->nb_batches < 3 ? L->nb_batches : 3;
  const int F = a->n_freq;
  L->horner = L->fast && F >= 2 && a->n_frames <= 1 && I == 1 && a->include_illum &&
              2 * a->nx == px && 2 * a->ny == py;
  if (L->horner) {
    const double d0 = a->frequencies[1] - a->frequencies[0];
    for (int f = 1; f < F; f++)
      if (fabs((a->frequencies[f] - a->frequencies[f - 1]) - d0) > 1e-9 * fabs(d0))
        L->horner = false;
    L->dkhat = d0 / 299792458.0;
  }
  const long ns[4] = {px, py, qx, qy};
  int64_t o = 0;
  for (int i = 0; i < 4; i++) {
    L->n_tw[i] = (int64_t)twiddles(ns[i]).size();
    L->off_tw[i] = o;
    o = align256(o + 8 * L->n_tw[i]);
  }
  const int frames = a->n_frames > 0 ? a->n_frames : 1;
  L->off_planes = o; o = align256(o + (int64_t)sizeof(pf_plane) * a->nz);
  L->off_ill = o; o = align256(o + 8 * 3 * I);
  L->off_fw = o; o = align256(o + 8 * (int64_t)F * frames);
  L->off_sc = o; o = align256(o + 8 * 2 * (int64_t)a->nz);
  L->off_chx = o; o = align256(o + 8 * (int64_t)a->nz * px);
  L->off_khx = o; o = align256(o + 8 * (int64_t)a->nz * qx);
  L->off_chy = o; o = align256(o + 8 * (int64_t)a->nz * py);
  L->off_khy = o; o = align256(o + 8 * (int64_t)a->nz * qy);
  L->off_uhat = o; o = align256(o + 8 * (int64_t)L->lanes * batch * I * py * px);
  L->off_xbuf = o; o = align256(o + 8 * (int64_t)L->lanes * batch * a->ny * px);
  L->off_wa = o; o = align256(o + 8 * L->lanes * pf_prop_ws_a(&g, batch));
  L->off_wb = o; o = align256(o + 8 * L->lanes * pf_prop_ws_b(&g, batch));
  L->off_wo = o;
  if (L->horner && F > 32) o = align256(o + 8 * (int64_t)L->lanes * batch * a->nx * a->ny);
  L->total = o;
  return 0;
}

}  // namespace

extern "C" int64_t pf_srsd_workspace_bytes(const pf_srsd_args* a) {
  SLayout L;
  if (splan(a, &L) != 0) return -1;
  return L.total;
}

extern "C" int pf_srsd(const pf_srsd_args* a, const void* slices, void* vol, void* ws,
                       int64_t ws_bytes, void* stream) {
  Nvtx range("pf_srsd");
  SLayout L;
  if (splan(a, &L) != 0) return -1;
  PF_ARG_CHECK(slices && vol && ws && ws_bytes >= L.total,
               "pf_srsd: null buffer or workspace smaller than pf_srsd_workspace_bytes");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  const int F = a->n_freq, I = a->n_illum, frames = a->n_frames > 0 ? a->n_frames : 1;
  const int nx = a->nx, ny = a->ny, px = L.px, py = L.py;
  const int64_t V = (int64_t)a->nz * ny * nx;
  // ---- fp64 tables from the host
  const long ns[4] = {px, py, L.qx, L.qy};
  pf_fft_plan plans[4];
  for (int i = 0; i < 4; i++) {
    std::vector<float2> t = twiddles(ns[i]);
    PF_CUDA_CHECK(cudaMemcpyAsync(w + L.off_tw[i], t.data(), 8 * t.size(), cudaMemcpyHostToDevice,
                                  st), "pf_srsd: upload");
    plans[i] = make_plan(ns[i], w + L.off_tw[i], t.size());
  }
  const double cx = a->relay_x0 + (nx / 2) * a->relay_dx;
  const double cy = a->relay_y0 + (ny / 2) * a->relay_dy;
  std::vector<pf_plane> planes(a->nz);
  std::vector<double> sc(2 * (size_t)a->nz);
  for (int k = 0; k < a->nz; k++) {
    const double pxk = a->relay_dx / a->alphas[k], pyk = a->relay_dy / a->betas[k];
    planes[k] = pf_plane{a->zs[k] - a->relay_z, pxk, pyk, cx - (nx / 2) * pxk, pxk,
                         cy - (ny / 2) * pyk, pyk, a->zs[k],
                         (int64_t)(k % L.batch) * I * py * px, k};
    sc[k] = a->alphas[k];
    sc[a->nz + k] = a->betas[k];
  }
  PF_CUDA_CHECK(cudaMemcpyAsync(w + L.off_planes, planes.data(), sizeof(pf_plane) * a->nz,
                                cudaMemcpyHostToDevice, st), "pf_srsd: upload");
  PF_CUDA_CHECK(cudaMemcpyAsync(w + L.off_ill, a->ill_xyz, 8 * 3 * I, cudaMemcpyHostToDevice, st),
                "pf_srsd: upload");
  PF_CUDA_CHECK(cudaMemcpyAsync(w + L.off_sc, sc.data(), 8 * sc.size(), cudaMemcpyHostToDevice, st),
                "pf_srsd: upload");
  std::vector<float2> fw((size_t)F * frames);
  for (int f = 0; f < F; f++)
    for (int j = 0; j < frames; j++) {
      const double ph = a->n_frames > 0 ? a->frequencies[f] * a->times[j] : 0.0;
      fw[(size_t)f * frames + j] = make_float2((float)cos(ph), (float)sin(ph));
    }
  PF_CUDA_CHECK(cudaMemcpyAsync(w + L.off_fw, fw.data(), 8 * fw.size(), cudaMemcpyHostToDevice, st),
                "pf_srsd: upload");
  PF_CUDA_CHECK(cudaMemsetAsync(vol, 0, 8 * (size_t)frames * V, st), "pf_srsd: zero volume");
  // ---- scaled-FFT tables on the device: chirps and Khat = FFT_Q(kernel) per plane and axis
  const double* sc_d = (const double*)(w + L.off_sc);
  float2* chx = (float2*)(w + L.off_chx);
  float2* khx = (float2*)(w + L.off_khx);
  float2* chy = (float2*)(w + L.off_chy);
  float2* khy = (float2*)(w + L.off_khy);
  k_srsd_tables<<<1024, 256, 0, st>>>(px, L.qx, px / 2, sc_d, a->nz, chx, khx);
  PF_LAUNCH_CHECK("k_srsd_tables");
  k_srsd_tables<<<1024, 256, 0, st>>>(py, L.qy, py / 2, sc_d + a->nz, a->nz, chy, khy);
  PF_LAUNCH_CHECK("k_srsd_tables");
  int rc = pf_fft_lines(khx, &plans[2], a->nz, 1, 0, L.qx, 1, -1, 1.0f, stream);
  if (rc == 0) rc = pf_fft_lines(khy, &plans[3], a->nz, 1, 0, L.qy, 1, -1, 1.0f, stream);
  if (rc != 0) return rc;
  // ---- lanes forked from the caller's stream
  pf_prop_geom g{};
  g.px = px;
  g.py = py;
  g.nx = nx;
  g.ny = ny;
  g.nu0x = -(nx / 2);
  g.nu0y = -(ny / 2);
  g.n_illum = I;
  g.include_illum = a->include_illum ? 1 : 0;
  g.uhat_illum_stride = (int64_t)px * py;
  cudaStream_t lane_st[3];
  cudaEvent_t ev_fork, ev_join[3];
  PF_CUDA_CHECK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "pf_srsd: event");
  PF_CUDA_CHECK(cudaEventRecord(ev_fork, st), "pf_srsd: event");
  for (int l = 0; l < L.lanes; l++) {
    PF_CUDA_CHECK(cudaStreamCreateWithFlags(&lane_st[l], cudaStreamNonBlocking), "pf_srsd: stream");
    PF_CUDA_CHECK(cudaEventCreateWithFlags(&ev_join[l], cudaEventDisableTiming), "pf_srsd: event");
    PF_CUDA_CHECK(cudaStreamWaitEvent(lane_st[l], ev_fork, 0), "pf_srsd: fork");
  }
  const pf_plane* planes_d = (const pf_plane*)(w + L.off_planes);
  const double* ill_d = (const double*)(w + L.off_ill);
  const float2* fw_d = (const float2*)(w + L.off_fw);
  const float2* sl = (const float2*)slices;
  const int64_t D = (int64_t)nx * ny;
  const int64_t uh_n = (int64_t)L.batch * I * py * px, xb_n = (int64_t)L.batch * ny * px;
  const int64_t wa_n = pf_prop_ws_a(&g, L.batch), wb_n = pf_prop_ws_b(&g, L.batch);
  const int64_t wo_n = (int64_t)L.batch * nx * ny;
  rc = 0;
  for (int b0 = 0, bi = 0; b0 < a->nz && rc == 0; b0 += L.batch, bi++) {
    const int lane = bi % L.lanes;
    void* ls = (void*)lane_st[lane];
    const int nb = a->nz - b0 < L.batch ? a->nz - b0 : L.batch;
    const pf_plane* pp = planes_d + b0;
    float2* uhat = (float2*)(w + L.off_uhat) + lane * uh_n;
    float2* xbuf = (float2*)(w + L.off_xbuf) + lane * xb_n;
    float2* wa = (float2*)(w + L.off_wa) + lane * wa_n;
    float2* wb = (float2*)(w + L.off_wb) + lane * wb_n;
    float2* wo = (float2*)(w + L.off_wo) + lane * wo_n;
    for (int s = 0; s < F && rc == 0; s++) {
      const int f = L.horner ? F - 1 - s : s;
      for (int p = 0; p < I && rc == 0; p++) {
        const float2* u = sl + ((int64_t)f * I + p) * D;
        float2* uo = uhat + (int64_t)p * py * px;
        if (L.bwarp) {   // register Bluestein passes, spectra transposed for the register path
          rc = pf_bluestein_warp(1, u, 0, nx, nx, px / 2 - nx / 2, xbuf, (int64_t)px * ny, ny, px,
                                 ny, nb, &plans[2], chx + (int64_t)b0 * px,
                                 khx + (int64_t)b0 * L.qx, ls);
          if (rc == 0)
            rc = pf_bluestein_warp(0, xbuf, (int64_t)px * ny, ny, ny, py / 2 - ny / 2, uo,
                                   (int64_t)I * py * px, py, py, px, nb, &plans[3],
                                   chy + (int64_t)b0 * py, khy + (int64_t)b0 * L.qy, ls);
        } else {
          rc = pf_bluestein_lines(u, 0, nx, 1, nx, px / 2 - nx / 2, xbuf, (int64_t)ny * px, px, 1,
                                  1, px, ny, nb, &plans[2], chx + (int64_t)b0 * px,
                                  khx + (int64_t)b0 * L.qx, ls);
          if (rc == 0) {
            if (L.fast)   // transposed spectra
              rc = pf_bluestein_lines(xbuf, (int64_t)ny * px, 1, px, ny, py / 2 - ny / 2, uo,
                                      (int64_t)I * py * px, py, 1, 1, py, px, nb, &plans[3],
                                      chy + (int64_t)b0 * py, khy + (int64_t)b0 * L.qy, ls);
            else
              rc = pf_bluestein_lines(xbuf, (int64_t)ny * px, 1, px, ny, py / 2 - ny / 2, uo,
                                      (int64_t)I * py * px, 1, px, 1, py, px, nb, &plans[3],
                                      chy + (int64_t)b0 * py, khy + (int64_t)b0 * L.qy, ls);
          }
        }
      }
      if (rc != 0) break;
      const double khat = a->frequencies[f] / 299792458.0;
      rc = pf_prop_kernel_rows(pp, nb, khat, &g, &plans[0], wa, ls);
      if (rc == 0) rc = pf_prop_columns(pp, nb, &g, &plans[1], wa, uhat, wb, 0, ls);
      if (rc != 0) break;
      if (L.horner) {
        int mode;
        if (F <= 32) {
          mode = f == 0 ? 2 : 1;
        } else {
          mode = f == 0 ? 4 : (f % 32 == 0 ? 3 : 1);
          if (f == F - 1)
            PF_CUDA_CHECK(cudaMemsetAsync(wo, 0, 8 * (size_t)nb * nx * ny, lane_st[lane]),
                          "pf_srsd: zero");
        }
        rc = pf_prop_rows_out_horner(pp, nb, khat, L.dkhat, mode, &g, &plans[0], wb, ill_d,
                                     fw_d + (int64_t)f * frames, vol, wo, 32 * L.dkhat, nullptr, ls);
      } else {
        rc = pf_prop_rows_out(pp, nb, khat, &g, &plans[0], wb, ill_d, fw_d + (int64_t)f * frames,
                              frames, vol, V, ls);
      }
    }
  }
  for (int l = 0; l < L.lanes; l++) {
    cudaEventRecord(ev_join[l], lane_st[l]);
    cudaStreamWaitEvent(st, ev_join[l], 0);
    cudaEventDestroy(ev_join[l]);
    cudaStreamDestroy(lane_st[l]);
  }
  cudaEventDestroy(ev_fork);
  return rc;
}
