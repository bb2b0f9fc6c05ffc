// Standalone micro-benchmark: throughput of 1024-point line FFTs (load -> FFT -> store)
// with the 32-lane register FFT (32 elements/thread) vs a 64-thread variant
// (16 elements/thread, two exchanges).  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -std=c++17 -o gpurun_out/fftbench tools/fftbench.cu
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2501_05244_b200/csrc/warp_fft.cuh"

void pf_set_error(const char*, ...) {}

// ---- A: current warp FFT (L = 32), 8 warps per CTA, 1 line per warp
__global__ void __launch_bounds__(256, 2) k_a(float2* data, const float2* tw, int nlines, int REPS) {
  extern __shared__ float2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int line = blockIdx.x * 8 + warp;
  if (line >= nlines) return;
  float2* d = data + (long long)line * 1024;
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; m++) v[m] = d[lane + 32 * m];
  for (int r = 0; r < REPS; r++) wfft<32, -1>(v, sm + warp * WFFT_XCH, tw);
#pragma unroll
  for (int m = 0; m < 32; m++) d[lane + 32 * m] = v[m];
}
__device__ int REPS_dummy;

// ---- B: 64 threads per line, 16 elements per thread.
// x index n = t + 64 m (t < 64, m < 16).  Step 1: DFT16 over m, twiddle W1024^{t k1}.
// exchange -> thread (k1, t1), t1 < 4: holds y[t1 + 4 t2][k1], t2 < 16; DFT16 over t2,
// twiddle W64^{t1 k2}; DFT4 over t1 across the 4 lanes (shuffles) -> thread (k1, k3)
// holds X[k1 + 16 k2 + 256 k3] for k2 < 16.
template <int DIR>
__device__ __forceinline__ void fft1024_64(float2 (&v)[16], float2* xch /*64*17 float2*/,
                                           const float2* tw /*W_1024^m table*/) {
  const int t = threadIdx.x & 63;
  Dft<16, DIR>::run(v);
#pragma unroll
  for (int k1 = 1; k1 < 16; k1++) {
    const float2 w = __ldg(tw + ((t * k1) & 1023));
    v[k1] = DIR < 0 ? cmul(v[k1], w) : cmulc(v[k1], w);
  }
  // write y[t][k1] at xch[t*17 + k1]
#pragma unroll
  for (int k1 = 0; k1 < 16; k1++) xch[t * 17 + k1] = v[k1];
  __syncthreads();
  const int k1 = t >> 2, t1 = t & 3;
#pragma unroll
  for (int t2 = 0; t2 < 16; t2++) v[t2] = xch[(t1 + 4 * t2) * 17 + k1];
  __syncthreads();
  Dft<16, DIR>::run(v);   // v[k2]
  if (t1) {
#pragma unroll
    for (int k2 = 1; k2 < 16; k2++) {
      const float2 w = __ldg(tw + ((t1 * k2 * 16) & 1023));   // W64^{t1 k2}
      v[k2] = DIR < 0 ? cmul(v[k2], w) : cmulc(v[k2], w);
    }
  }
  // DFT4 over t1 across lanes (xor 1, 2 partners within the group of 4)
#pragma unroll
  for (int k2 = 0; k2 < 16; k2++) {
    float2 a[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      a[j].x = __shfl_sync(0xffffffffu, v[k2].x, (threadIdx.x & ~3) | j);
      a[j].y = __shfl_sync(0xffffffffu, v[k2].y, (threadIdx.x & ~3) | j);
    }
    Dft<4, DIR>::run(a);
    v[k2] = a[t1];   // k3 = t1
  }
}

__global__ void __launch_bounds__(256, 4) k_b(float2* data, const float2* tw, int nlines) {
  __shared__ float2 sm[4][64 * 17];
  const int grp = threadIdx.x >> 6, t = threadIdx.x & 63;
  const int line = blockIdx.x * 4 + grp;
  const bool act = line < nlines;
  float2* d = data + (long long)(act ? line : 0) * 1024;
  float2 v[16];
#pragma unroll
  for (int m = 0; m < 16; m++) v[m] = d[t + 64 * m];
  fft1024_64<-1>(v, sm[grp], tw);
  const int k1 = t >> 2, k3 = t & 3;
  if (act) {
#pragma unroll
    for (int k2 = 0; k2 < 16; k2++) d[k1 + 16 * k2 + 256 * k3] = v[k2];
  }
}

int main() {
  const int nlines = 1 << 17;   // 131072 lines x 8 KB = 1 GB
  std::vector<float2> h((size_t)nlines * 1024), tw(2048);
  for (int m = 0; m < 1024; m++) {
    double a = -2.0 * M_PI * m / 1024.0;
    tw[m] = make_float2((float)cos(a), (float)sin(a));
  }
  // k1-major extension for wfft<32>: tw2[k1 * 32 + t] = W^{t k1}
  for (int k1 = 0; k1 < 32; k1++)
    for (int t = 0; t < 32; t++) {
      double a = -2.0 * M_PI * ((k1 * t) % 1024) / 1024.0;
      tw[1024 + k1 * 32 + t] = make_float2((float)cos(a), (float)sin(a));
    }
  for (size_t i = 0; i < h.size(); i++) h[i] = make_float2((float)((i * 7919) % 1000) / 1000.f, 0.f);
  float2 *d, *dt;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&dt, tw.size() * 8);
  cudaMemcpy(dt, tw.data(), tw.size() * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_a, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int reps = 1; reps <= 8; reps *= 2) {
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    float best = 1e30f;
    for (int it = 0; it < 4; it++) {
      cudaEventRecord(e0);
      k_a<<<(nlines + 7) / 8, 256, 8 * WFFT_XCH * 8>>>(d, dt, nlines, reps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it) best = ms < best ? ms : best;
    }
    printf("A reps=%d: %.3f ms -> %.3f ns per line-FFT\n", reps, best, best * 1e6 / nlines / reps);
  }
  int reps = 1;
  for (int variant = 0; variant < 2; variant++) {
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    float best = 1e30f;
    for (int it = 0; it < 6; it++) {
      cudaEventRecord(e0);
      if (variant == 0)
        k_a<<<(nlines + 7) / 8, 256, 8 * WFFT_XCH * 8>>>(d, dt, nlines, reps);
      else
        k_b<<<(nlines + 3) / 4, 256>>>(d, dt, nlines);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it) best = ms < best ? ms : best;
    }
    // correctness of one line vs direct DFT (first iteration's input)
    std::vector<float2> o(1024);
    cudaMemcpy(d, h.data(), 1024 * 8, cudaMemcpyHostToDevice);
    if (variant == 0) k_a<<<1, 256, 8 * WFFT_XCH * 8>>>(d, dt, 1, 1);
    else k_b<<<1, 256>>>(d, dt, 1);
    cudaMemcpy(o.data(), d, 1024 * 8, cudaMemcpyDeviceToHost);
    double err = 0, nrm = 0;
    for (int k = 0; k < 1024; k++) {
      double re = 0, im = 0;
      for (int n = 0; n < 1024; n++) {
        double a = -2.0 * M_PI * ((long long)n * k % 1024) / 1024.0;
        re += h[n].x * cos(a) - h[n].y * sin(a);
        im += h[n].x * sin(a) + h[n].y * cos(a);
      }
      err += (o[k].x - re) * (o[k].x - re) + (o[k].y - im) * (o[k].y - im);
      nrm += re * re + im * im;
    }
    printf("variant %s: %.3f ms for %d lines (%.2f ns/line, %.1f GB/s)  relerr %.2e  %s\n",
           variant == 0 ? "A warp32x32" : "B 64thr x16", best, nlines, best * 1e6 / nlines,
           2.0 * nlines * 8192 / (best * 1e6), sqrt(err / nrm), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
