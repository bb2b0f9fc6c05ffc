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
/* A plan whose radix[PF_MAX_STAGES - 1] holds PF_XFFT_TAG carries, after its n unit
 * roots, the k1-major twiddle table [35][L] (W_n^{k1 t}) of the mixed-radix register FFT
 * for n = 35 L, L in {4, 5, 8, 10, 15, 20, 30} (pf_fft_lines then takes that kernel). */
#define PF_XFFT_TAG 0x35F7
typedef struct pf_fft_plan {
  int n;
  int nst;
  int radix[PF_MAX_STAGES];
  const void* tw;
} pf_fft_plan;

int pf_version(void);
/* Copy the calling thread's last error message into buf (always NUL-terminated). */
int pf_last_error(char* buf, size_t len);
/* Kernels launched by this library in this process (a stream-captured launch counts
 * once, at capture).  Used by the bench's gpu_launches figure. */
int64_t pf_launch_count(void);

/* ---------------------------------------------------------------- K1
 * Temporal phasor transform: replaces phasor.to_frequency (phasor.py:107-127,
 * the FFT-gather-weight-phase of lines 119-121).
 *   out[f * out_stride + trace] = (sum_t hist[trace][t] W_T^{bins[f] t}) * wphase[f]
 * hist: float32 [n_traces][n_bins]; twiddle: c64 [n_bins/64][n_freq] with
 * entry [r][f] = W_T^{bins[f] r} (fp64-built); wphase: c64 [n_freq] =
 * weight_f * exp(-1j w_f t0).  Requires n_bins = 64*M, M a power of two <= 256.
 * inner_mask: bit k set for every inner bin k = min(b mod 64, 64 - b mod 64) of the
 * retained bins (sizes shared memory and selects the bins formed; 0 = unknown:
 * the kernel derives it, shared memory for all 33; a set missing a bin traps). */
int pf_temporal_dft(const float* hist, int64_t n_traces, int n_bins, const int32_t* bins,
                    const void* twiddle, const void* wphase, int n_freq, void* out,
                    int64_t out_stride, uint64_t inner_mask, void* stream);
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
/* The same over a three-level line set: line l has inner index l % inner (stride
 * inner_stride), middle index (l / inner) % mid (stride mid_stride) and outer index
 * l / (inner mid) (stride outer_stride) -- e.g. the lines of a sub-block of the two other
 * axes of every array of a batch in one launch (the NUFFT's pruned 3D transforms). */
int pf_fft_lines3(void* data, const pf_fft_plan* plan, int64_t nlines, int64_t inner,
                  int64_t inner_stride, int64_t mid, int64_t mid_stride, int64_t outer_stride,
                  int64_t elem_stride, int dir, float scale, void* stream);

/* Embed relay planes into zero-padded natural-order grids (the reference's
 * _pad_embed + ifftshift, reconstruct.py:113-119 with spectral.py:107-109).
 * src: c64 [nb][ny][nx] (row pitch src_ld), dst: c64 [nb][py][px].  Centred
 * relay index i - n//2 lands at natural slot (i - n//2) mod p.  transpose=1 writes
 * the transposed grid [nb][px][py] (the register path consumes Uhat^T). */
int pf_embed_centered(const void* src, int64_t nb, int ny, int nx, int64_t src_batch_stride,
                      void* dst, int py, int px, int transpose, void* stream);

/* Register-path relay spectra (replaces _pad_embed + cfft_2d, reference
 * reconstruct.py:113-119,259-260): dst[b][kx][ky] = the TRANSPOSED natural-order
 * forward 2D FFT of src[b] (ny x nx, row-major) embedded centred in P x P, for
 * P in {128, 256, 512, 1024} (plan: pf_fft_plan of length P).  Only the ny relay
 * rows are transformed; the zero rows cost nothing.  Two launches. */
int pf_relay_spectra_fast(const void* src, int64_t nb, int ny, int nx,
                          int64_t src_batch_stride, void* dst, int P,
                          const pf_fft_plan* plan, void* stream);

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
  int flags;             /* bit 0: never take the register-FFT path */
  int reserved;
  int64_t uhat_illum_stride; /* elements between illuminations inside uhat */
} pf_prop_geom;

/* Pad size handled by the register-FFT path (square power-of-two 128..1024), else 0.
 * When nonzero, the three stages expect uhat TRANSPOSED: Uhat^T[col][row]. */
int pf_prop_fast(const pf_prop_geom* g);

/* workspace element counts (c64) for a batch of nplanes */
int64_t pf_prop_ws_a(const pf_prop_geom* g, int nplanes);
int64_t pf_prop_ws_b(const pf_prop_geom* g, int nplanes);
/* full product spectra [nplanes][n_illum][py][px] (product_only mode) */
int64_t pf_prop_ws_spectrum(const pf_prop_geom* g, int nplanes);

int pf_prop_kernel_rows(const pf_plane* planes, int nplanes, double khat,
                        const pf_prop_geom* g, const pf_fft_plan* plan_x, void* ws_a,
                        void* stream);
/* product_only=1 (type-2 readouts: nursd2 reconstruct.py:453, nursd3 :519,
 * srsd_nursd2 :580): write the full natural-order product Uhat * Ghat_k to ws_b
 * ([nplanes][n_illum][py][px]) instead of the y-IFFT + row crop.  Requires
 * flags bit 0 (register path off). */
int pf_prop_columns(const pf_plane* planes, int nplanes, const pf_prop_geom* g,
                    const pf_fft_plan* plan_y, const void* ws_a, const void* uhat,
                    void* ws_b, int product_only, void* stream);
/* ill_xyz: device float64 [n_illum][3]; frame_w: device c64 [n_frames]
 * (exp(1j w t_j) for time-resolved output, or {1} for static); vol: c64
 * [n_frames][vol_frame_stride] with plane k at k*ny*nx; accumulates (+=). */
int pf_prop_rows_out(const pf_plane* planes, int nplanes, double khat,
                     const pf_prop_geom* g, const pf_fft_plan* plan_x, const void* ws_b,
                     const double* ill_xyz, const void* frame_w, int n_frames, void* vol,
                     int64_t vol_frame_stride, void* stream);

/* Stage C with the illumination phase by Horner's rule (register path, both crops
 * centred, one illumination, single frame): call it for the frequencies in DESCENDING
 * order; dkhat = the uniform frequency spacing in rad/m.  vol <- vol * exp(i dk d) + v_f,
 * and at f = 0 the sum is multiplied by exp(i k_0 d): the same sum as
 * reconstruct.py:160-168 (ascending f, per-frequency phases) in nested order.
 * mode 1: inner step; 2: f = 0 of a single-block sum (khat = k_0).  Sums longer than a
 * block of B frequencies restart the nesting per block (z is raised to at most B - 1) and
 * chain the blocks with Z = exp(i B dk d) from a float64-reduced phase: mode 3 at the
 * lowest frequency of a block other than the first (o <- o Z + (vol z + v), vol <- 0),
 * mode 4 at f = 0 (vol <- (o Z + (vol z + v)) exp(i k_0 d)); ws_o = the batch's outer
 * accumulator (nplanes x ny x nx complex64), zkhat = B dkhat.  vol_out (NULL: vol) receives the
 * finished planes of the final step (modes 2 and 4) at the same offsets: the fused volume
 * gather points it at rank 0's volume (peer memory, distributed.PeerVolume).
 * Returns 1 without work when the geometry is not eligible. */
int pf_prop_rows_out_horner(const pf_plane* planes, int nplanes, double khat, double dkhat,
                            int mode, const pf_prop_geom* g, const pf_fft_plan* plan_x,
                            const void* ws_b, const double* ill_xyz, const void* frame_w,
                            void* vol, void* ws_o, double zkhat, void* vol_out, void* stream);

/* All nf frequencies of a plane batch at once (register path, static volume):
 * kturns: device float64 [nf] = khat_f / (2 pi); ws_a / uhat / ws_b advance by
 * the given per-frequency strides (elements); frame_w: device c64 [nf] weights
 * (ones for a static volume); kernel C sums the frequencies in ascending order
 * in registers and adds the result to vol once.  For small configurations
 * (config 0/1) where per-launch latency dominates. */
int pf_prop_fbatch(const pf_plane* planes, int nplanes, const double* kturns, int nf,
                   const pf_prop_geom* g, const pf_fft_plan* plan, void* ws_a, int64_t ws_a_fs,
                   const void* uhat, int64_t uhat_fs, void* ws_b, int64_t ws_b_fs,
                   const double* ill_xyz, const void* frame_w, void* vol, void* stream);

/* pf_prop_fbatch for any pad (Stockham shared-memory path; e.g. the reference's
 * P = 140 of config 1): khat_f: device float64 [nf] wavenumbers (rad/m); plan_x /
 * plan_y: length px / py plans; otherwise as pf_prop_fbatch.  Three launches:
 * A and B over (tiles, planes, frequencies), C looping the frequencies in
 * ascending order per (row tile, plane) with the sum kept in shared memory. */
int pf_prop_fbatch_generic(const pf_plane* planes, int nplanes, const double* khat_f, int nf,
                           const pf_prop_geom* g, const pf_fft_plan* plan_x,
                           const pf_fft_plan* plan_y, void* ws_a, int64_t ws_a_fs,
                           const void* uhat, int64_t uhat_fs, void* ws_b, int64_t ws_b_fs,
                           const double* ill_xyz, const void* frame_w, void* vol, void* stream);

/* pf_prop_fbatch for the reference pad P = 140 (config 1's off-lattice nursd1, reference
 * reconstruct.py:372-383) with every stage of a (frequency, plane) unit in one CTA's shared
 * memory (the 140 x 140 plane, 157 KB, never leaves the SM): grid (nplanes, groups), each
 * CTA sums its contiguous range of ceil(nf / groups) frequencies in ascending order;
 * with groups > 1 the partial planes go to ws_part ([groups][nplanes][ny][nx] c64) and a
 * second launch adds them to vol in ascending group order.  kturns: device float64 [nf]
 * = khat_f / (2 pi); uhat natural layout [py][px] per plane offset, uhat_fs elements per
 * frequency; frame_w: device c64 [nf]; warps: warps per CTA (12 or 16; 0 = default).
 * Requires pf_prop_onchip_ok(g) (px = py = 140, one illumination, output plane within the
 * shared-memory budget). */
int pf_prop_onchip_ok(const pf_prop_geom* g);
int pf_prop_fbatch_onchip(const pf_plane* planes, int nplanes, const double* kturns, int nf,
                          const pf_prop_geom* g, const void* uhat, int64_t uhat_fs,
                          const double* ill_xyz, const void* frame_w, void* vol, void* ws_part,
                          int groups, int warps, void* stream);

/* K1 with the slice all-gather fused into its store (distributed.PeerSlices): each retained
 * bin of this rank's traces is written to peers[j][f * peer_stride + peer_col + trace] for
 * every rank's full [F][I][D] slice buffer (device array of n_peers device pointers, peer
 * memory mapped with pf_ipc_open); n_bins = 64 M with M in {32, 64, 128, 256}. */
int pf_temporal_dft_peers(const float* hist, int64_t n_traces, int n_bins, const int32_t* bins,
                          const void* twiddle, const void* wphase, int n_freq,
                          uint64_t inner_mask, const uint64_t* peers, int n_peers,
                          int64_t peer_stride, int64_t peer_col, void* stream);
/* CUDA IPC for the peer-memory collectives: the 64-byte handle of the allocation holding
 * ptr plus ptr's offset in it; the mapping of that allocation in another process (same
 * device, or a peer over NVLink / NVSwitch) with the offset applied; unmapping (pass the
 * mapped pointer minus its offset). */
int pf_ipc_handle(const void* ptr, void* handle_out, int64_t* offset_out);
int pf_ipc_open(const void* handle, int64_t offset, void** ptr_out);
int pf_ipc_close(void* base);

/* out (device int32[2]) = {number of non-finite, number of negative} float32
 * values in x[0..n): the payload checks of reference read_dataset
 * (core.py:727-728, NaN/inf) and TransientMeasurement (counts >= 0) for
 * histograms read straight into device memory.  x must be 16-byte aligned. */
int pf_count_nonfinite(const float* x, int64_t n, int32_t* out, void* stream);

/* rsd3d stage-1 gridding (reconstruct.py:680-707, np.add.at onto the virtual
 * lattice): for touched cell c, out[v][cells[c]] = sum_{e in [cell_start[c],
 * cell_start[c+1])} ent_w[e] * vals[v][ent_pt[e]] (fixed order, no atomics).
 * Cells not listed are left untouched (the caller zeroes the lattice). */
int pf_scatter_csr(const int32_t* cell_start, const int64_t* cells, const int32_t* ent_pt,
                   const float* ent_w, int n_cells, const void* vals, int64_t val_stride, int nv,
                   void* out, int64_t out_stride, void* stream);

/* Measurement helper (bench.py): FP32 FFMA throughput probe, blocks x 256 threads,
 * 8 chains x 16 unrolled FMAs x iters each; flops = 256 * blocks * iters * 256. */
int pf_fp32_probe(void* out, int blocks, int iters, void* stream);

/* ---------------------------------------------------------------- SFFT (Bluestein)
 * Scaled-DFT lines, replacing SfftPlan.apply (spectral.py:160-168) inside
 * sfft_2d_centered (:209-218): per plane b (grid y) the tables chirp[b][M] and
 * khat[b][Q] (float64-built; Q = plan_q->n >= 2M-1).  Input element i < n_in of
 * line l is at src + b*src_ps + l*src_ls + i*src_es and occupies slot o_in + i;
 * output slot k goes to dst + b*dst_ps + l*dst_ls + pos(k)*dst_es with
 * pos(k) = k, or natural(k - M/2) when natural_out (centred -> FFT order). */
int pf_bluestein_lines(const void* src, int64_t src_ps, int64_t src_ls, int64_t src_es,
                       int n_in, int o_in, void* dst, int64_t dst_ps, int64_t dst_ls,
                       int64_t dst_es, int natural_out, int M, int nlines, int nplanes,
                       const pf_fft_plan* plan_q, const void* chirp, const void* khat,
                       void* stream);

/* Register-FFT Bluestein pass for Q = plan_q->n in {128,256,512,1024} (plan_q->tw
 * must carry the warp-FFT twiddle extension).  Lines are contiguous input rows
 * (element i at src + b*src_ps + l*src_ls + i, slot o_in + i).  xpass=1 stores
 * the pass TRANSPOSED with natural column order: dst[b*dst_ps + col*dst_ls + l];
 * xpass=0 stores dst[b*dst_ps + l*dst_ls + row_nat] (Uhat^T for the register
 * propagation path). */
int pf_bluestein_warp(int xpass, const void* src, int64_t src_ps, int64_t src_ls, int n_in,
                      int o_in, void* dst, int64_t dst_ps, int64_t dst_ls, int M, int nlines,
                      int nplanes, const pf_fft_plan* plan_q, const void* chirp,
                      const void* khat, void* stream);

/* ---------------------------------------------------------------- NUFFT
 * Gridding NUFFT (spectral.py:230-381): the reference's Gaussian stencil (window 0) or the
 * exponential-of-semicircle window on the same 2x-oversampled fine grid (window 1, the
 * default of the Python layer; same eps contract, half the stencil width).  Axis order
 * (z, y, x); 2D uses mr[0] = m[0] = 1.  Per point (device): i0[L][3] int32 nearest fine
 * node, d0[L][3] float32 = i0*h - x (the offset of the centre tap); taps -w..w.  */
typedef struct pf_nufft_geom {
  int dim;
  int w;
  int mr[3];
  int m[3];
  float h[3];
  float inv4tau[3];
  int tile[3];
  int ntiles[3];
  int window;      /* 0: Gaussian (the reference's stencil), 1: exponential of semicircle */
  float beta;      /* window 1: exp(beta (sqrt(1 - (d / (w h))^2) - 1)), beta = 2.30 * 2 w */
  float inv_hw[3]; /* window 1: 1 / (w h[a]) */
} pf_nufft_geom;

/* type-1 spreading (spectral.py:353-355) as a tiled gather: fine[v][cell] =
 * sum over points in tile_pts[tile_start[t]..] of vals[v][pt] * window.
 * Writes every fine cell. */
int pf_nufft_spread(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                    const int32_t* tile_start, const int32_t* tile_pts, const void* vals,
                    int64_t val_stride, int nv, void* fine, int64_t fine_stride, void* stream);
/* type-1 finish (spectral.py:357-358): centred modes / discrete deconvolution,
 * written in natural order on the mode grid ([x][y] when transpose, 2D). */
/* Type-1 finish on the register path (replaces the fine-grid fftn + pf_nufft_deconv,
 * reference spectral.py:356-358) for 2D plans with square modes m in {128, 256, 512,
 * 1024} and fine grid mr = 2m: out[v][c_x][c_y] (TRANSPOSED natural-order modes) =
 * FFT(fine[v]) at the centred modes / (ker_y * ker_x).  rt: scratch of nv * m * 2m
 * complex64.  plan_mr / plan_h: pf_fft_plan of lengths 2m and m.  Two launches. */
int pf_nufft_type1_finish_pow2(const pf_nufft_geom* g, const void* fine, int64_t fine_stride,
                               int nv, void* rt, const pf_fft_plan* plan_mr,
                               const pf_fft_plan* plan_h, const float* ky, const float* kx,
                               void* out, int64_t out_stride, void* stream);
int pf_nufft_deconv(const pf_nufft_geom* g, const void* fine, int64_t fine_stride,
                    const float* kz, const float* ky, const float* kx, int nv, void* out,
                    int64_t out_stride, int transpose, void* stream);
/* Type-2 start for 2D plans in two fused passes (spectral.py:373-375, = pf_nufft_place +
 * the pruned inverse fine-grid FFT, bit for bit): fine[v] = unnormalised inverse FFT of
 * S[v] / (ker_y ker_x) placed on the fine slots, S natural order [v][my][mx].  The x pass
 * builds each kept fine row from S in shared memory; the y pass reads only the kept rows.
 * plan_x / plan_y: pf_fft_plan of lengths mr[2] / mr[1]. */
int pf_nufft_type2_start_2d(const pf_nufft_geom* g, const void* S, int64_t s_stride,
                            const float* ky, const float* kx, int nv, void* fine,
                            int64_t fine_stride, const pf_fft_plan* plan_x,
                            const pf_fft_plan* plan_y, void* stream);
/* The same with an output window: only the fine cells of columns [col0, col0 + ncols) and
 * rows [row0, row0 + nrows) (indices on the torus: they may wrap past mr) are needed by the
 * caller -- the cells its readout stencils touch.  With the split passes (mr = 2 m = 70 L)
 * the y pass transforms only the window's columns and stores only its rows; cells outside
 * the window are left unwritten.  (Without them the whole grid is formed.) */
int pf_nufft_type2_start_2d_win(const pf_nufft_geom* g, const void* S, int64_t s_stride,
                                const float* ky, const float* kx, int nv, void* fine,
                                int64_t fine_stride, const pf_fft_plan* plan_x,
                                const pf_fft_plan* plan_y, int col0, int ncols, int row0,
                                int nrows, void* stream);
/* The same with the column pass writing to `out` with every il consecutive grids interleaved
 * cell by cell: out[(v / il) * (fine_stride * il) + cell * il + v % il] (il = 1, out = fine:
 * pf_nufft_type2_start_2d_win).  Needs the split column pass (pf_nufft_type2_il_ok). */
int pf_nufft_type2_start_2d_il(const pf_nufft_geom* g, const void* S, int64_t s_stride,
                               const float* ky, const float* kx, int nv, void* fine,
                               int64_t fine_stride, const pf_fft_plan* plan_x,
                               const pf_fft_plan* plan_y, int col0, int ncols, int row0,
                               int nrows, void* out, int il, void* stream);
/* ... and with every grid v of the call stored as slot `member` of its own group v
 * (out[v * (fine_stride * il) + cell * il + member]): one frequency of every plane per call,
 * the frequencies of a plane interleaved (member < 0: pf_nufft_type2_start_2d_il). */
int pf_nufft_type2_start_2d_ilm(const pf_nufft_geom* g, const void* S, int64_t s_stride,
                                const float* ky, const float* kx, int nv, void* fine,
                                int64_t fine_stride, const pf_fft_plan* plan_x,
                                const pf_fft_plan* plan_y, int col0, int ncols, int row0,
                                int nrows, void* out, int il, int member, void* stream);
int pf_nufft_type2_il_ok(const pf_nufft_geom* g);
/* type-2 start (spectral.py:374): modes / deconvolution onto their fine slots, 0 elsewhere. */
int pf_nufft_place(const pf_nufft_geom* g, const void* S, int64_t s_stride, const float* kz,
                   const float* ky, const float* kx, int nv, void* fine, int64_t fine_stride,
                   int transpose, void* stream);
/* pf_nufft_interp2_acc for the points of several planes in one launch: point l reads
 * the fine grids of plane plane_idx[l] (at fine + (plane_idx[l] - plane0) *
 * fine_plane_stride, illumination p at + p * fine_stride) and accumulates into
 * vol[f][dst_idx[l]] (nursd2 family readouts, reconstruct.py:453-457). */
int pf_nufft_interp2_batch(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                           const double* xyz, const int32_t* plane_idx, const int64_t* dst_idx,
                           int npts, int plane0, const void* fine, int64_t fine_plane_stride,
                           int64_t fine_stride, int n_illum, const double* ill, double khat,
                           int include_illum, float scale, const void* frame_w, int n_frames,
                           void* vol, int64_t vol_frame_stride, void* stream);
/* pf_nufft_interp2_nodes on node-interleaved fine grids (pf_nufft_type2_start_2d_il with
 * il = nodes): a tap's node values are contiguous, read with 16-byte loads.  ES window at
 * w = 4, 12 nodes, one illumination. */
int pf_nufft_interp2_nodes_il(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                              const double* xyz, const int32_t* plane_idx,
                              const int64_t* dst_idx, int npts, int plane0, const void* fine_il,
                              int64_t slab_stride, const double* ill, double khat,
                              int include_illum, float scale, const void* frame_w, int n_frames,
                              void* vol, int64_t vol_frame_stride, int nodes, const float* lw,
                              void* stream);
/* The plane readout (pf_nufft_interp2_batch) over all n_freq frequencies in one launch, on
 * frequency-interleaved fine grids fine_f[group][plane][cell][16] (pf_nufft_type2_start_2d_ilm
 * with il = 16, member = f % 16; unused slots zero): vol[dst] += sum_f frame_w[f]
 * exp(i k_f |x - s|) scale * stencil(fine_f).  kturns_f [n_freq] = k_f / (2 pi) on the device.
 * ES window at w = 4, one illumination, one frame. */
int pf_nufft_interp2_freqs(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                           const double* xyz, const int32_t* plane_idx, const int64_t* dst_idx,
                           int npts, int plane0, const void* fine_f, int64_t plane_stride,
                           int64_t group_stride, int n_freq, const double* kturns_f,
                           const double* ill, int include_illum, float scale,
                           const void* frame_w, void* vol, void* stream);
/* Readout kernel for the reference's default stencil (w = 8, 17 x 17 taps): 2 (default)
 * the 16 x 16 trimmed kernel (the far edge tap of each axis, <= 6.5e-9 of the centre
 * weight, is not loaded), 1 the full 17 x 17 kernel, 0 the general kernel; mode < 0 only
 * queries.  Returns the previous mode (also PF_INTERP_H17 in the environment). */
int pf_nufft_interp_mode(int mode);
/* The same readout for voxels at arbitrary depths (z-Chebyshev): voxel l takes the
 * Lagrange-weighted sum lw[l][m] over its slab's `nodes` consecutive fine grids (the
 * first at plane_idx[l]) of the same stencil; nodes = 1, lw = NULL is
 * pf_nufft_interp2_batch.  One half warp per point. */
int pf_nufft_interp2_nodes(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                           const double* xyz, const int32_t* plane_idx, const int64_t* dst_idx,
                           int npts, int plane0, const void* fine, int64_t fine_plane_stride,
                           int64_t fine_stride, int n_illum, const double* ill, double khat,
                           int include_illum, float scale, const void* frame_w, int n_frames,
                           void* vol, int64_t vol_frame_stride, int nodes, const float* lw,
                           void* stream);
/* type-2 finish for any dimension (spectral.py:376-380): out[l] = stencil sum of the
 * fine grid (after pf_nufft_place + inverse FFT) at point l; stencil width 2w+1 <= 32. */
int pf_nufft_interp(const pf_nufft_geom* g, const int32_t* i0, const float* d0, int npts,
                    const void* fine, void* out, void* stream);
/* type-2 finish (spectral.py:377-380) fused with the per-voxel scale, the
 * illumination phase (reconstruct.py:140-144) and the ascending-frequency
 * accumulation (reconstruct.py:163-177): vol[f][dst0 + perm[l]] += sum_p(...) * frame_w[f]
 * (perm may be NULL; points stored cell-sorted for gather locality use it). */
int pf_nufft_interp2_acc(const pf_nufft_geom* g, const int32_t* i0, const float* d0,
                         const double* xyz, int npts, const void* fine, int64_t fine_stride,
                         int n_illum, const double* ill, double khat, int include_illum,
                         float scale, const void* frame_w, int n_frames, void* vol,
                         int64_t vol_frame_stride, int64_t dst0, const int32_t* perm,
                         void* stream);

/* ---------------------------------------------------------------- elementwise
 * _kernel_3d (reconstruct.py:624-638) on the natural 3D grid (zero lag -> 0). */
int pf_kernel3d(void* out, int pz, int py, int px, double dx, double dy, double dz, double khat,
                void* stream);
/* a[i] = a[i] * b[i % b_period] * scale */
int pf_cmul(void* a, const void* b, int64_t n, int64_t b_period, float scale, void* stream);
/* Even 3D kernels (the lattice stages' G3 is even in every lag, so is its transform): the
 * mirrored half of an axis filled by copy before that axis' pass -- axis 1: rows y > py/2
 * for z <= lim, x <= xmax; axis 0: planes z > pz/2 for y <= lim, x <= xmax -- and the
 * product a[f][i][z][y][x] *= g[f][z][min(y, py - y)][min(x, px - x)] * scale with g formed
 * on that octant only (_kernel_3d and the product of reconstruct.py:624-638, 758). */
int pf_mirror_fill(void* buf, int nb, int pz, int py, int px, int axis, int lim, int xmax,
                   void* stream);
int pf_cmul_even(void* a, const void* g, int nf, int ni, int pz, int py, int px, float scale,
                 void* stream);
/* dst[b][:] = src[b*src_stride + plane_off + :plane_elems] (slab extraction, :760) */
/* One output plane of an inverse DFT along the leading axis: dst[b][j] = scale *
 * sum_z src[b][z][j] * w[z] (w = exp(+2 pi i z slab / nz), complex64, host-built in
 * float64); replaces the z pass of cifft_n + slab extraction (reconstruct.py:758-759). */
int pf_zslab(const void* src, int nb, int nz, int64_t nyx, const void* w, float scale,
             void* dst, void* stream);
int pf_copy_planes(const void* src, int nb, int64_t src_stride, int64_t plane_off,
                   int64_t plane_elems, void* dst, void* stream);
/* Centred nx x ny window of nb natural-order py x px planes (inverse of the centred
 * embed): dst[b][i][j] = src[b][(i - ny/2) mod py][(j - nx/2) mod px]; the virtual plane
 * of the 3D stage 1 on the frustum-base lattice (3D RSD / NURSD + SRSD). */
int pf_crop_centered(const void* src, int64_t nb, int py, int px, void* dst, int ny, int nx,
                     void* stream);

/* circular shift of the trailing axes (n0, n1, n2) of nb arrays:
 * dst[b][j] = src[b][(j + s) mod n] per axis (ifftshift: s = n/2, fftshift: s = n - n/2;
 * the index maps of cfft_n / cifft_n, spectral.py:107-114). */
int pf_roll(const void* src, void* dst, int64_t nb, int n0, int n1, int n2, int s0, int s1, int s2,
            void* stream);

/* ---------------------------------------------------------------- whole algorithm
 * rsd (reference reconstruct.py:208-268, rsd(slices, grid, padding, times, threads,
 * include_illumination)) in one call: relay lattice and output cuboid as the reference's
 * UniformGrid2D / UniformGrid3D fields (x0/y0 = first sample, not the centre); host
 * arrays frequencies [n_freq] (rad/s, ascending, FrequencySlices.frequencies),
 * ill_xyz [n_illum][3] (illumination_coordinates, core.py), times [n_frames] or
 * n_frames = 0 for a static volume.  slices: device c64 [n_freq][n_illum][relay_ny *
 * relay_nx] (frequency-major, row-major lattice); vol: device c64 [max(1, n_frames)]
 * [nz * ny * nx], x fastest (written, not accumulated); ws: device scratch of at least
 * pf_rsd_workspace_bytes(args) bytes.  Validation errors (status -1, pf_last_error) carry
 * the reference's ValidationError messages ("pitch", "origin", "beyond the relay",
 * "padding='none'").  Asynchronous on `stream`; plane batches run on three internal
 * lanes forked from and joined back to it. */
typedef struct pf_rsd_args {
  int relay_nx, relay_ny;
  double relay_dx, relay_dy, relay_x0, relay_y0, relay_z;
  int nx, ny, nz;
  double dx, dy, dz, x0, y0, z0;
  int n_freq, n_illum;
  const double* frequencies;
  const double* ill_xyz;
  int n_frames;
  const double* times;
  int padding_none;
  int include_illum;
} pf_rsd_args;

int64_t pf_rsd_workspace_bytes(const pf_rsd_args* args);
int pf_rsd(const pf_rsd_args* args, const void* slices, void* vol, void* ws, int64_t ws_bytes,
           void* stream);

/* srsd (reference reconstruct.py:276-327, srsd(slices, grid, times, threads,
 * include_illumination)) in one call.  The frustum's base is the relay lattice (the
 * reference requires them to coincide, :291-294); zs / alphas / betas (host, [nz]) are
 * FrustumGrid.zs / alphas / betas.  Same conventions as pf_rsd otherwise; the output
 * planes keep nx x ny samples at pitch dx / alpha_k about the base centre. */
typedef struct pf_srsd_args {
  int nx, ny;
  double relay_dx, relay_dy, relay_x0, relay_y0, relay_z;
  int nz;
  const double* zs;
  const double* alphas;
  const double* betas;
  int n_freq, n_illum;
  const double* frequencies;
  const double* ill_xyz;
  int n_frames;
  const double* times;
  int include_illum;
} pf_srsd_args;

int64_t pf_srsd_workspace_bytes(const pf_srsd_args* args);
int pf_srsd(const pf_srsd_args* args, const void* slices, void* vol, void* ws, int64_t ws_bytes,
            void* stream);

/* Spreading window of the plans the C entry points build (pf_nursd1, pf_nursd2): 1 (default)
 * the exponential of semicircle, 0 the reference's Gaussian stencil (spectral.py:230-315);
 * any other value only queries.  Returns the previous setting (initially from
 * PF_NUFFT_WINDOW = "es" | "gaussian"). */
int pf_nufft_window(int mode);
/* nursd1 (reference reconstruct.py:335-385, nursd1(slices, grid, eps, times, threads,
 * include_illumination)) in one call: detections scattered on the plane z = relay_z
 * (relay_xy host [n_points][2], x then y) -> cuboid grid, via a type-1 NUFFT at accuracy
 * eps onto the padded lattice spectrum and the rsd propagation.  slices: device
 * [F][I][n_points] c64 (a frequency-major transpose of FrequencySlices.coefficients);
 * vol: device [frames][nz*ny*nx] c64.  Pad: the reference rule when a detection is off
 * the voxel lattice (the result depends on it), else the exact pad.  Same conventions
 * as pf_rsd otherwise. */
typedef struct pf_nursd1_args {
  int n_points;
  const double* relay_xy;
  double relay_z;
  int nx, ny, nz;
  double dx, dy, dz, x0, y0, z0;
  int n_freq, n_illum;
  const double* frequencies;
  const double* ill_xyz;
  int n_frames;
  const double* times;
  double eps;
  int include_illum;
} pf_nursd1_args;

int64_t pf_nursd1_workspace_bytes(const pf_nursd1_args* args);
int pf_nursd1(const pf_nursd1_args* args, const void* slices, void* vol, void* ws,
              int64_t ws_bytes, void* stream);

/* nursd2 (reference reconstruct.py:413-459, nursd2(slices, grid, eps, times, threads,
 * include_illumination)) in one call: detections on a uniform relay lattice -> explicit
 * voxels on planes of constant depth (ExplicitGrid: plane_z / plane_count host
 * [n_planes], voxel_xy host [sum plane_count][2], plane-major, x then y).  slices:
 * device [F][I][relay_ny*relay_nx] c64; vol: device [frames][sum plane_count] c64 in
 * the grid's voxel order.  Reference pad rule; type-2 NUFFT at accuracy eps.  Same
 * conventions as pf_rsd otherwise. */
typedef struct pf_nursd2_args {
  int relay_nx, relay_ny;
  double relay_dx, relay_dy, relay_x0, relay_y0, relay_z;
  int n_planes;
  const double* plane_z;
  const int64_t* plane_count;
  const double* voxel_xy;
  int n_freq, n_illum;
  const double* frequencies;
  const double* ill_xyz;
  int n_frames;
  const double* times;
  double eps;
  int include_illum;
} pf_nursd2_args;

int64_t pf_nursd2_workspace_bytes(const pf_nursd2_args* args);
int pf_nursd2(const pf_nursd2_args* args, const void* slices, void* vol, void* ws,
              int64_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PFGPU_H */
