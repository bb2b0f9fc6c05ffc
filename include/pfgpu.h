/*
 * libpfgpu - B200 (sm_100a) kernels for the phasor-field NLOS reconstruction hot path.
 *
 * Drop-in boundary: the reference is the pure-Python
 * package `phasorfield` (/root/reference/pkg/src/phasorfield).  Its hot-path
 * entry points are Python functions; the Python shim
 * `paper_2501_05244_b200` keeps their names/signatures and calls these C
 * entry points through ctypes.  Every function below cites the reference
 * code it replaces.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless the parameter says "host".
 *    Buffers are allocated by the caller (torch); the library never allocates.
 *  - Complex data is interleaved float32 pairs (complex64, "c64").
 *  - `stream` is a cudaStream_t (may be NULL = legacy default stream).
 *    Every call is asynchronous on `stream`; there is no global mutable state.
 *  - Return value: 0 ok, <0 argument error, >0 CUDA error code.  The message
 *    is available from pf_last_error() (thread-local).  No C++ exception ever
 *    crosses this boundary.
 *  - Spectra are kept in NATURAL FFT order internally; the reference's
 *    centred-index convention (spectral.py:77-124) is applied by index maps
 *    at the load/store of each kernel, never by separate shift passes.
 */
#ifndef PFGPU_H
#define PFGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_MAX_STAGES 24

/* Mixed-radix plan for one transform length (host struct, passed by pointer).
 * radix[] lists the stage radices (2,3,4,5,7,8,11,16); tw is a DEVICE table of
 * n complex64 unit roots W_n^m = exp(-2 pi i m / n) built in float64. */
typedef struct pf_fft_plan {
  int n;
  int nst;
  int radix[PF_MAX_STAGES];
  const void* tw;
} pf_fft_plan;

int pf_version(void);
/* Copy the calling thread's last error message into buf (always NUL-terminated). */
int pf_last_error(char* buf, size_t len);

/* ---------------------------------------------------------------- K1
 * Temporal phasor transform: replaces phasor.to_frequency (phasor.py:107-127,
 * the FFT-gather-weight-phase of lines 119-121).
 *   out[f * out_stride + trace] = (sum_t hist[trace][t] W_T^{bins[f] t}) * wphase[f]
 * hist: float32 [n_traces][n_bins]; twiddle: c64 [n_bins/64][n_freq] with
 * entry [r][f] = W_T^{bins[f] r} (fp64-built); wphase: c64 [n_freq] =
 * weight_f * exp(-1j w_f t0).  Requires n_bins = 64*M, M a power of two <= 256. */
int pf_temporal_dft(const float* hist, int64_t n_traces, int n_bins, const int32_t* bins,
                    const void* twiddle, const void* wphase, int n_freq, void* out,
                    int64_t out_stride, void* stream);
/* Same transform for any n_bins (direct sum); unit_roots: c64 [n_bins] W_T^m. */
int pf_temporal_dft_direct(const float* hist, int64_t n_traces, int n_bins,
                           const int32_t* bins, const void* unit_roots, const void* wphase,
                           int n_freq, void* out, int64_t out_stride, void* stream);

/* ---------------------------------------------------------------- FFT core
 * Batched in-place 1D FFT of c64 lines; replaces numpy.fft.fftn/ifftn inside
 * cfft_n/cifft_n (spectral.py:107-124) and the NUFFT/SFFT inner FFTs
 * (spectral.py:156,167,356,375).  Line l starts at
 *   (l / inner) * outer_stride + (l % inner) * inner_stride
 * and its element i sits at + i * elem_stride (all in elements).
 * dir = -1 forward (exp(-1j..)), +1 inverse (unnormalised); result *= scale. */
int pf_fft_lines(void* data, const pf_fft_plan* plan, int64_t nlines, int64_t inner,
                 int64_t inner_stride, int64_t outer_stride, int64_t elem_stride, int dir,
                 float scale, void* stream);

/* Embed relay planes into zero-padded natural-order grids (the reference's
 * _pad_embed + ifftshift, reconstruct.py:113-119 with spectral.py:107-109).
 * src: c64 [nb][ny][nx] (row pitch src_ld), dst: c64 [nb][py][px].  Centred
 * relay index i - n//2 lands at natural slot (i - n//2) mod p.  transpose=1 writes
 * the transposed grid [nb][px][py] (the register path consumes Uhat^T). */
int pf_embed_centered(const void* src, int64_t nb, int ny, int nx, int64_t src_batch_stride,
                      void* dst, int py, int px, int transpose, void* stream);

/* ---------------------------------------------------------------- propagation
 * Plane-to-plane RSD propagation, the per-(frequency, plane) inner loop of
 * rsd (reconstruct.py:254-266), srsd (:312-325), nursd1 (:372-383) and the
 * nursd3d stage 2 (:641-659):
 *   plane_k = cifft2(Uhat * cfft2(G_k))[rows, cols] * mask_k
 * with G_k = exp(1j khat r) / r synthesised on the fly (never read from HBM).
 * Three kernels: (A) kernel rows + x-FFT, keeping the non-redundant quadrant
 * (G is even on the torus, so Ghat(-k) = Ghat(k)); (B) kernel y-FFT, product
 * with Uhat, y-IFFT, crop rows; (C) x-IFFT, crop columns, illumination phase,
 * accumulate into the volume in ascending frequency order. */
typedef struct pf_plane {
  double dz;             /* plane z minus source-plane z (> 0) */
  double lag_dx, lag_dy; /* kernel lag pitch (relay pitch / scale) */
  double x0, dx, y0, dy; /* output sample m,n at (x0 + m dx, y0 + n dy) */
  double z;              /* plane z (illumination mask) */
  int64_t uhat_off;      /* element offset of this plane's spectrum in uhat */
  int64_t vol_plane;     /* output plane index in the volume */
} pf_plane;

typedef struct pf_prop_geom {
  int px, py;            /* padded transform sizes */
  int nx, ny;            /* output plane size */
  int nu0x, nu0y;        /* centred index of output column / row 0 */
  int n_illum;
  int include_illum;
  int64_t uhat_illum_stride; /* elements between illuminations inside uhat */
} pf_prop_geom;

/* Pad size handled by the register-FFT path (square power-of-two 128..1024), else 0.
 * When nonzero, the three stages expect uhat TRANSPOSED: Uhat^T[col][row]. */
int pf_prop_fast(const pf_prop_geom* g);

/* workspace element counts (c64) for a batch of nplanes */
int64_t pf_prop_ws_a(const pf_prop_geom* g, int nplanes);
int64_t pf_prop_ws_b(const pf_prop_geom* g, int nplanes);

int pf_prop_kernel_rows(const pf_plane* planes, int nplanes, double khat,
                        const pf_prop_geom* g, const pf_fft_plan* plan_x, void* ws_a,
                        void* stream);
int pf_prop_columns(const pf_plane* planes, int nplanes, const pf_prop_geom* g,
                    const pf_fft_plan* plan_y, const void* ws_a, const void* uhat,
                    void* ws_b, void* stream);
/* ill_xyz: device float64 [n_illum][3]; frame_w: device c64 [n_frames]
 * (exp(1j w t_j) for time-resolved output, or {1} for static); vol: c64
 * [n_frames][vol_frame_stride] with plane k at k*ny*nx; accumulates (+=). */
int pf_prop_rows_out(const pf_plane* planes, int nplanes, double khat,
                     const pf_prop_geom* g, const pf_fft_plan* plan_x, const void* ws_b,
                     const double* ill_xyz, const void* frame_w, int n_frames, void* vol,
                     int64_t vol_frame_stride, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PFGPU_H */
