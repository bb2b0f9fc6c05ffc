// Host-side helpers shared by the whole-algorithm C entry points (algo_rsd.cu,
// algo_srsd.cu): pad rules, FFT plan radices and fp64-built twiddle tables.
#pragma once
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "xfft.cuh"

namespace pfalgo {

constexpr double C_LIGHT = 299792458.0;
constexpr int LANES = 3;
constexpr int HORNER_BLOCK = 32;
constexpr int64_t BATCH_BYTES = 64LL << 20;

inline bool close_rel(double a, double b) {
  return fabs(a - b) <= fmax(1e-9 * fmax(fabs(a), fabs(b)), 1e-12);
}

inline bool smooth11(long n) {
  if (n < 1) return false;
  const int ps[5] = {2, 3, 5, 7, 11};
  for (int p : ps)
    while (n % p == 0) n /= p;
  return n == 1;
}

inline long next_fast_len(long n) {
  if (n < 1) n = 1;
  while (!smooth11(n)) n++;
  return n;
}

inline long exact_pad(double lag_max, double nu_max, long n_min) {
  long need = 2 * (long)ceil(fmax(lag_max, nu_max)) + 2;
  if (need < n_min) need = n_min;
  long p2 = 1;
  while (p2 < need) p2 *= 2;
  if (64 < need && p2 <= 1024 && p2 * 5 <= need * 8) return p2;
  return next_fast_len(need);
}

// stage radices: powers of two merged into as few even stages as possible, then odd primes
// in descending order (_device.radices_for)
inline int radices(long n, int* out) {
  std::vector<int> f;
  long m = n;
  for (int p : {2, 3, 5, 7, 11})
    while (m % p == 0) {
      f.push_back(p);
      m /= p;
    }
  if (m != 1) return -1;
  int k = 0;
  std::vector<int> odd;
  for (int p : f) (p == 2 ? k++ : (odd.push_back(p), 0));
  int ns = 0;
  if (k) {
    const int s = (k + 3) / 4;
    for (int i = 0; i < s; i++) out[ns++] = 1 << (k / s + (i < k % s ? 1 : 0));
  }
  for (int i = (int)odd.size() - 1; i >= 0; i--) out[ns++] = odd[i];   // descending
  return ns;
}

// unit roots exp(-2 pi i m / n) in fp64, rounded to c64; the register-FFT lengths append
// the k1-major twiddles [k1][t] = exp(-2 pi i ((k1 t) mod n) / n), n = 32 L
inline std::vector<float2> twiddles(long n) {
  std::vector<float2> w;
  for (long m = 0; m < n; m++) {
    const double a = -2.0 * M_PI * (double)m / (double)n;
    w.push_back(make_float2((float)cos(a), (float)sin(a)));
  }
  // register FFT tables as the Python plans (_device.xfft_plan_L): L >= 10 by default
  const char* ev = getenv("PF_XFFT");
  long xl = xfft_L((int)n);
  if (ev && strcmp(ev, "0") == 0) xl = 0;
  long lmin = 10;   // _device.xfft_plan_L: "all", an integer minimum, or "large" (10)
  if (ev && strcmp(ev, "all") == 0) lmin = 1;
  else if (ev && ev[0] >= '1' && ev[0] <= '9') lmin = atol(ev);
  if (xl < lmin) xl = 0;
  if (xl) {   // mixed-radix register FFT: k1-major [35][L]
    for (long k1 = 0; k1 < 35; k1++)
      for (long t = 0; t < xl; t++) {
        const double a = -2.0 * M_PI * (double)((k1 * t) % n) / (double)n;
        w.push_back(make_float2((float)cos(a), (float)sin(a)));
      }
  }
  if (n == 128 || n == 256 || n == 512 || n == 1024) {
    const long L = n / 32;
    for (long k1 = 0; k1 < 32; k1++)
      for (long t = 0; t < L; t++) {
        const double a = -2.0 * M_PI * (double)((k1 * t) % n) / (double)n;
        w.push_back(make_float2((float)cos(a), (float)sin(a)));
      }
  }
  return w;
}


// NVTX range over a host scope (a profiler shows the C entry points' phases; no cost
// without one attached)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

inline int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }

// a pf_fft_plan over a table already in device memory (tw), tagged for the register
// FFT when its table carries the 35 L extension
inline pf_fft_plan make_plan(long n, const void* tw_dev, size_t n_tw) {
  pf_fft_plan p{};
  p.n = (int)n;
  p.nst = radices(n, p.radix);
  p.tw = tw_dev;
  if ((long)n_tw > n && !(n == 128 || n == 256 || n == 512 || n == 1024))
    p.radix[PF_MAX_STAGES - 1] = PF_XFFT_TAG;
  return p;
}

}  // namespace pfalgo

namespace pfalgo {

// plane batch of the propagation loop (reconstruct.Propagator): ws_a + ws_b within
// BATCH_BYTES; register path: a multiple of 4 (32 / L) planes, at most 4 (32 / L)
inline int prop_batch(const pf_prop_geom* g, int nz, bool fast) {
  const int64_t per = 8 * ((int64_t)(g->py / 2 + 1) * (g->px / 2 + 1) +
                           (int64_t)g->n_illum * g->ny * g->px);
  int batch = (int)fmax(1.0, fmin((double)nz, (double)(BATCH_BYTES / per)));
  if (fast) {
    const int l = g->px / 32, q = 4 * (32 / l);
    int b = (batch / q) * q;
    if (b < q) b = q;
    batch = b;
    if (batch > 4 * (32 / l)) batch = 4 * (32 / l);
    if (batch > nz) batch = nz;
  }
  return batch;
}

// Horner's rule in kernel C: register path, centred crops, one illumination, one frame,
// uniformly spaced frequencies (reconstruct.Propagator.freq_order); *dkhat = spacing / c
inline bool horner_ok(const pf_prop_geom* g, bool fast, const double* freqs, int F,
                      int n_frames, int include_illum, double* dkhat) {
  if (!(fast && F >= 2 && n_frames <= 1 && g->n_illum == 1 && include_illum &&
        2 * g->nx == g->px && 2 * g->ny == g->py && 2 * g->nu0x == -g->nx &&
        2 * g->nu0y == -g->ny))
    return false;
  const double d0 = freqs[1] - freqs[0];
  for (int f = 1; f < F; f++)
    if (fabs((freqs[f] - freqs[f - 1]) - d0) > 1e-9 * fabs(d0)) return false;
  *dkhat = d0 / C_LIGHT;
  return true;
}

// The per plane batch, per frequency A / fused B / C launches of the propagation, plane
// batches round-robin over `lanes` streams forked from and joined back to `st`.
// uhat: [F][I][P^2] relay spectra; vol: [frames][V] (accumulated into, zeroed by the caller).
struct PropLoop {
  const pf_prop_geom* g;
  const pf_fft_plan* plx;
  const pf_fft_plan* ply;
  const pf_plane* planes;   // device [nz]
  int nz, batch, lanes, frames;
  const double* ill;        // device [I][3]
  const float2* fw;         // device [F][frames]
  bool horner;
  double dkhat;
  char* wa;                 // device lanes x pf_prop_ws_a(g, batch) c64
  char* wb;                 // device lanes x pf_prop_ws_b(g, batch) c64
  char* wo;                 // device lanes x batch x nx x ny c64 (Horner blocks), or null
};

inline int prop_loop(const PropLoop& p, const float2* uhat, const double* freqs, int F,
                     void* vol, int64_t V, cudaStream_t st) {
  const pf_prop_geom& g = *p.g;
  cudaStream_t lane_st[LANES];
  cudaEvent_t ev_fork, ev_join[LANES];
  PF_CUDA_CHECK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "prop: event");
  PF_CUDA_CHECK(cudaEventRecord(ev_fork, st), "prop: event");
  for (int l = 0; l < p.lanes; l++) {
    PF_CUDA_CHECK(cudaStreamCreateWithFlags(&lane_st[l], cudaStreamNonBlocking), "prop: stream");
    PF_CUDA_CHECK(cudaEventCreateWithFlags(&ev_join[l], cudaEventDisableTiming), "prop: event");
    PF_CUDA_CHECK(cudaStreamWaitEvent(lane_st[l], ev_fork, 0), "prop: fork");
  }
  const int64_t per_f = (int64_t)g.n_illum * g.px * g.py;
  const int64_t wa_n = pf_prop_ws_a(&g, p.batch), wb_n = pf_prop_ws_b(&g, p.batch);
  const int64_t wo_n = (int64_t)p.batch * g.nx * g.ny;
  int rc = 0;
  for (int b0 = 0, bi = 0; b0 < p.nz && rc == 0; b0 += p.batch, bi++) {
    const int lane = bi % p.lanes;
    void* ls = (void*)lane_st[lane];
    const int nb = p.nz - b0 < p.batch ? p.nz - b0 : p.batch;
    const pf_plane* pp = p.planes + b0;
    float2* wa = (float2*)p.wa + lane * wa_n;
    float2* wb = (float2*)p.wb + lane * wb_n;
    float2* wo = p.wo ? (float2*)p.wo + lane * wo_n : nullptr;
    for (int s = 0; s < F && rc == 0; s++) {
      const int f = p.horner ? F - 1 - s : s;   // Horner: descending frequencies
      const double khat = freqs[f] / C_LIGHT;
      const float2* uh = uhat + f * per_f;
      rc = pf_prop_kernel_rows(pp, nb, khat, &g, p.plx, wa, ls);
      if (rc == 0) rc = pf_prop_columns(pp, nb, &g, p.ply, wa, uh, wb, 0, ls);
      if (rc != 0) break;
      if (p.horner) {
        int mode;
        if (F <= HORNER_BLOCK) {
          mode = f == 0 ? 2 : 1;
        } else {
          mode = f == 0 ? 4 : (f % HORNER_BLOCK == 0 ? 3 : 1);
          if (f == F - 1)
            PF_CUDA_CHECK(cudaMemsetAsync(wo, 0, 8 * (size_t)nb * g.nx * g.ny, lane_st[lane]),
                          "prop: zero");
        }
        rc = pf_prop_rows_out_horner(pp, nb, khat, p.dkhat, mode, &g, p.plx, wb, p.ill,
                                     p.fw + (int64_t)f * p.frames, vol, wo,
                                     HORNER_BLOCK * p.dkhat, nullptr, ls);
      } else {
        rc = pf_prop_rows_out(pp, nb, khat, &g, p.plx, wb, p.ill, p.fw + (int64_t)f * p.frames,
                              p.frames, vol, V, ls);
      }
    }
  }
  for (int l = 0; l < p.lanes; l++) {
    cudaEventRecord(ev_join[l], lane_st[l]);
    cudaStreamWaitEvent(st, ev_join[l], 0);
    cudaEventDestroy(ev_join[l]);
    cudaStreamDestroy(lane_st[l]);
  }
  cudaEventDestroy(ev_fork);
  return rc;
}

}  // namespace pfalgo
