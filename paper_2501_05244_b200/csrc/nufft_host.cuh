// Host planning of the 2D GPU NUFFT for the whole-algorithm C entry points
// (algo_nursd1.cu, algo_nursd2.cu); the C++ counterpart of nufft.NufftPlan /
// NufftPoints, following reference NufftPlan (spectral.py:230-315): fine grid
// mr = next_fast_len(max(2m, 2w + 2)) (h = 2 pi / mr), the per-point stencil anchors of
// spectral.py:281-303, and one of two windows (pf_nufft_window / PF_NUFFT_WINDOW):
//   1 (default) exponential of semicircle exp(beta (sqrt(1 - (d / (w h))^2) - 1)),
//     2w = max(6, ceil(log10(1/eps)) + 2) taps, beta = 2.30 * 2w, deconvolved by its continuous
//     transform (64-node Gauss-Legendre);
//   0 the reference's Gaussian: w = max(2, ceil(log10(1/eps)) + 2),
//     tau = pi w / (s (s - 1/2) m^2) with s = mr/m, the DISCRETE deconvolution
//     ker[k] = 1 + 2 sum_j exp(-(j h)^2 / 4 tau) cos(k j h).
#pragma once
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <utility>
#include <vector>

#include "algo_host.cuh"

namespace pfalgo {

constexpr double NUFFT_EPS_MIN = 1e-14, NUFFT_EPS_MAX = 1e-1, NUFFT_COORD_TOL = 1e-9;
constexpr int NUFFT_TILE = 16;   // nufft.TILE_2D = (1, 16, 16)

// reference pad rule (reconstruct.py:102-110), used where results depend on the pad
inline long ref_pad(double lag_max, double nu_max, long n_min) {
  const long need = 2 * (long)ceil(fmax(lag_max, nu_max)) + 2;
  return next_fast_len(n_min > need + 8 ? n_min : need + 8);
}

// natural slots of the centred modes [-m/2, m - m/2) on a length-mr axis (_device.kept_ranges)
inline std::vector<std::pair<int, int>> kept_ranges(int m, int mr) {
  if (m >= mr) return {{0, mr}};
  if (m / 2) return {{0, m - m / 2}, {mr - m / 2, m / 2}};
  return {{0, m - m / 2}};
}

// default window of the C++ planner: PF_NUFFT_WINDOW ("es" | "gaussian"), or pf_nufft_window
inline int& nufft_window_ref() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PF_NUFFT_WINDOW");
    v = (e && strcmp(e, "gaussian") == 0) ? 0 : 1;
  }
  return v;
}

// n-node Gauss-Legendre rule on [-1, 1] (Newton on P_n from the Chebyshev guess)
inline void gauss_legendre(int n, std::vector<double>* x, std::vector<double>* wt) {
  x->assign(n, 0.0);
  wt->assign(n, 0.0);
  for (int i = 0; i < (n + 1) / 2; i++) {
    double z = cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 1.0;
    for (int it = 0; it < 100; it++) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; k++) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (fabs(dz) < 1e-15) break;
    }
    (*x)[i] = -z;
    (*x)[n - 1 - i] = z;
    (*wt)[i] = (*wt)[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

constexpr double ES_BETA_PER_TAP = 2.30;

struct Nufft2Plan {
  pf_nufft_geom g;
  std::vector<float> ker[3];   // z (= {1}), y, x deconvolution factors
  int64_t fine_elems;
  bool pow2_finish;            // type-1 register finish: square m in 128..1024, mr = 2m
};

// plan for modes (my, mx); 0, or -1 with pf_set_error
inline int nufft2_plan(int my, int mx, double eps, Nufft2Plan* N) {
  if (!(isfinite(eps) && eps >= NUFFT_EPS_MIN && eps <= NUFFT_EPS_MAX)) {
    pf_set_error("accuracy target must lie in [1e-14, 0.1]");
    return -1;
  }
  const int window = nufft_window_ref();
  const int digits = (int)ceil(log10(1.0 / eps)) + 2;
  const int w = window == 1 ? std::max(3, (digits + 1) / 2) : std::max(2, digits);
  if (w > 16) {
    pf_set_error("accuracy target too tight for the GPU stencil (w <= 16)");
    return -1;
  }
  pf_nufft_geom& g = N->g;
  g = pf_nufft_geom{};
  g.dim = 2;
  g.w = w;
  g.window = window;
  g.beta = (float)(ES_BETA_PER_TAP * 2 * w);
  std::vector<double> gx, gw;
  if (window == 1) gauss_legendre(64, &gx, &gw);
  const int modes[3] = {1, my, mx};
  for (int a = 0; a < 3; a++) {
    const int m = modes[a];
    int mr;
    double tau;
    if (a == 0) {
      mr = 1;
      tau = 1.0;
      N->ker[0].assign(1, 1.0f);
    } else {
      mr = (int)next_fast_len(std::max(2 * m, 2 * w + 2));
      const double s = (double)mr / m;
      tau = M_PI * w / (s * (s - 0.5) * m * m);
      const double h = 2.0 * M_PI / mr;
      N->ker[a].resize(m);
      for (int i = 0; i < m; i++) {
        const double k = i - m / 2;
        double acc = 0.0;
        if (window == 1) {
          for (size_t q = 0; q < gx.size(); q++)
            acc += exp(ES_BETA_PER_TAP * 2 * w * (sqrt(1.0 - gx[q] * gx[q]) - 1.0)) * gw[q] * w *
                   cos(k * h * gx[q] * w);
          N->ker[a][i] = (float)acc;
        } else {
          for (int j = 1; j <= w; j++)
            acc += exp(-(j * h) * (j * h) / (4.0 * tau)) * cos(k * (j * h));
          N->ker[a][i] = (float)(1.0 + 2.0 * acc);
        }
      }
    }
    g.mr[a] = mr;
    g.m[a] = m;
    g.h[a] = (float)(2.0 * M_PI / mr);
    g.inv4tau[a] = (float)(1.0 / (4.0 * tau));
    g.inv_hw[a] = (float)(1.0 / (w * (2.0 * M_PI / mr)));
    g.tile[a] = a == 0 ? 1 : NUFFT_TILE;
    g.ntiles[a] = (mr + g.tile[a] - 1) / g.tile[a];
  }
  N->fine_elems = (int64_t)g.mr[1] * g.mr[2];
  N->pow2_finish = mx == my && (mx == 128 || mx == 256 || mx == 512 || mx == 1024) &&
                   g.mr[1] == 2 * my && g.mr[2] == 2 * mx;
  return 0;
}

// stencil anchors of L points at torus coordinates (tx, ty) in [-pi, pi): i0 [L][3] int32
// (nearest fine node), d0 [L][3] float32 (= i0 h - x).  cell_sorted: points ordered by
// anchor (y, then x; stable), `order` maps stored position -> caller's index.
// Appends to i0 / d0 / order.  0, or -1 with pf_set_error.
inline int nufft2_points(const Nufft2Plan& N, const double* tx, const double* ty, int64_t L,
                         bool cell_sorted, std::vector<int32_t>* i0, std::vector<float>* d0,
                         std::vector<int64_t>* order) {
  std::vector<int32_t> ai((size_t)3 * L, 0);
  std::vector<float> ad((size_t)3 * L, 0.0f);
  for (int64_t l = 0; l < L; l++) {
    const double tor[2] = {tx[l], ty[l]};
    for (int c = 0; c < 2; c++)
      if (!(isfinite(tor[c]) && tor[c] >= -M_PI - NUFFT_COORD_TOL &&
            tor[c] < M_PI + NUFFT_COORD_TOL)) {
        pf_set_error("point coordinates must lie in [-pi, pi)");
        return -1;
      }
    for (int a = 1; a < 3; a++) {
      const double x = tor[2 - a];   // mode axis a pairs with point column 2 - a
      const double h = 2.0 * M_PI / N.g.mr[a];
      const double xi = x - 2.0 * M_PI * floor(x / (2.0 * M_PI));
      const long k = (long)floor(xi / h + 0.5);
      ai[3 * (size_t)l + a] = (int32_t)k;
      ad[3 * (size_t)l + a] = (float)(k * h - xi);
    }
  }
  std::vector<int64_t> ord((size_t)L);
  std::iota(ord.begin(), ord.end(), (int64_t)0);
  if (cell_sorted)
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t p, int64_t q) {
      const int32_t py = ai[3 * p + 1], qy = ai[3 * q + 1];
      return py != qy ? py < qy : ai[3 * p + 2] < ai[3 * q + 2];
    });
  for (int64_t l : ord) {
    i0->insert(i0->end(), ai.begin() + 3 * l, ai.begin() + 3 * l + 3);
    d0->insert(d0->end(), ad.begin() + 3 * l, ad.begin() + 3 * l + 3);
    if (order) order->push_back(l);
  }
  return 0;
}

// (col0, ncols, row0, nrows): per axis the shortest arc of the fine-grid torus holding every
// stencil cell (anchor - w .. anchor + w) of the points i0 [L][3] (nufft.stencil_window):
// all a type-2 readout of these points reads
inline void nufft2_stencil_window(const Nufft2Plan& N, const std::vector<int32_t>& i0, int64_t L,
                                  int win[4]) {
  for (int s = 0; s < 2; s++) {
    const int a = s == 0 ? 2 : 1;
    const int mr = N.g.mr[a], w = N.g.w;
    std::vector<char> touched((size_t)mr, 0);
    for (int64_t l = 0; l < L; l++)
      for (int j = -w; j <= w; j++) touched[(size_t)((((i0[3 * l + a] + j) % mr) + mr) % mr)] = 1;
    int first = -1, best_gap = -1, best_after = 0, prev = -1;
    for (int c = 0; c < mr; c++) {
      if (!touched[c]) continue;
      if (first < 0) first = c;
      if (prev >= 0 && c - prev - 1 > best_gap) {
        best_gap = c - prev - 1;
        best_after = c;
      }
      prev = c;
    }
    if (first < 0) {   // no points
      win[2 * s] = 0;
      win[2 * s + 1] = mr;
      continue;
    }
    const int wrap_gap = first + mr - prev - 1;   // the run across the seam
    if (wrap_gap > best_gap) {
      best_gap = wrap_gap;
      best_after = first;
    }
    win[2 * s] = best_gap > 0 ? best_after : 0;
    win[2 * s + 1] = mr - (best_gap > 0 ? best_gap : 0);
  }
}

// tile buckets of the gather-spread kernel (NufftPoints.tiles): CSR over the fine-grid
// tiles each point's (2w + 1)^2 stencil touches, points ascending within a tile
inline void nufft2_tiles(const Nufft2Plan& N, const std::vector<int32_t>& i0, int64_t L,
                         std::vector<int32_t>* start, std::vector<int32_t>* pts) {
  const int w = N.g.w, mry = N.g.mr[1], mrx = N.g.mr[2];
  const int nty = N.g.ntiles[1], ntx = N.g.ntiles[2];
  std::vector<std::vector<int>> per_pt((size_t)L);
  std::vector<int32_t> count((size_t)nty * ntx + 1, 0);
  for (int64_t l = 0; l < L; l++) {
    int ty[64], tx[64], ny = 0, nx = 0;
    for (int j = -w; j <= w; j++) {
      const int cy = ((i0[3 * l + 1] + j) % mry + mry) % mry / NUFFT_TILE;
      const int cx = ((i0[3 * l + 2] + j) % mrx + mrx) % mrx / NUFFT_TILE;
      if (std::find(ty, ty + ny, cy) == ty + ny) ty[ny++] = cy;
      if (std::find(tx, tx + nx, cx) == tx + nx) tx[nx++] = cx;
    }
    for (int i = 0; i < ny; i++)
      for (int k = 0; k < nx; k++) {
        const int t = ty[i] * ntx + tx[k];
        per_pt[l].push_back(t);
        count[t + 1]++;
      }
  }
  start->assign((size_t)nty * ntx + 1, 0);
  for (size_t t = 0; t < (size_t)nty * ntx; t++) (*start)[t + 1] = (*start)[t] + count[t + 1];
  pts->assign(start->back(), 0);
  std::vector<int32_t> fill(start->begin(), start->end() - 1);
  for (int64_t l = 0; l < L; l++)
    for (int t : per_pt[l]) (*pts)[fill[t]++] = (int32_t)l;
}

}  // namespace pfalgo
