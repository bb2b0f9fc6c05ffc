// Streaming propagation: every (plane, frequency) job of an rsd-family
// reconstruction in ONE persistent kernel launch.
//
// Same math and the same four stages as propagate_fast.cu (reference rsd
// reconstruct.py:254-266 and its siblings srsd :312-325, nursd1 :372-383):
//   A  (65 tasks at P=1024)  synthesise kernel rows jy <= P/2, x-FFT, store At[kx][jy]
//   B1 (65)                  y-FFT of At rows in place -> Ghat quadrant
//   B2 (129)                 Ghat column * Uhat^T column, y-IFFT, crop -> Tt[col][i]
//   C  (64)                  transposed tile, x-IFFT, crop, illumination phase, vol +=
// A task is one CTA's worth of lines (8 warps).  Tasks are handed out in a
// fixed global order by an atomic ticket: step s carries A(job s), B1(job
// s-lag), B2(job s-2 lag) and C(job s-3 lag), so each task depends only on
// tasks with smaller tickets (deadlock-free with any number of resident CTAs),
// and by the time a task is fetched its inputs are normally complete.  Per-job
// completion counters enforce the dependencies; workspaces live in a ring of
// R >= 3 lag + 2 job slots (~50 MB at P=1024: L2-resident).  Volume rows of a
// plane are accumulated in ascending frequency order (C waits on the previous
// frequency's C of the same plane), so the sum order matches the stage path.
//
// Compared with one launch per stage and plane batch, no SM idles at kernel
// boundaries and the stages of different jobs overlap on every SM.
#include "prop_stages.cuh"

namespace {

constexpr int MT = 256;   // 8 warps per CTA

struct MegaJob {
  int plane;   // index into planes[]
  int f;       // frequency index
  int prev;    // job index of (plane, f - 1), or -1
  int pad;
};

struct MegaArgs {
  const pf_plane* planes;
  const MegaJob* jobs;
  int njobs;
  const double* kturns;      // [F] khat_f / (2 pi)
  const float2* uhat;        // Uhat^T, per frequency uhat_fs elements
  long long uhat_fs;
  const float2* frame_w;     // [F][n_frames]
  int n_frames;
  const double* ill;         // [n_illum][3]
  pf_prop_geom g;
  const float2* tw;
  float2* ws_a;              // [R][NA*NA]
  float2* ws_b;              // [R][n_illum*P*ny]
  long long ws_b_slot;
  int R, lag;
  int* ctr;                  // [njobs][4] stage completions, then ticket, abort
  float2* vol;
  long long vfs;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Spin (thread 0) until *p >= target; false (and the abort flag set) after ~2 s.
// ld.acquire.gpu invalidates the SM's L1 (CCTL.IVALL), and the CTA barrier that
// follows orders every thread's loads after it.
__device__ bool wait_geq(const int* p, int target, int* abort_flag) {
  if (ld_acquire(p) >= target) return true;
  for (int it = 0;; it++) {
    __nanosleep(128);
    if (ld_acquire(p) >= target) return true;
    if ((it & 255) == 255 && ld_acquire(abort_flag)) return false;
    if (it > (1 << 24)) {
      atomicExch(abort_flag, 1);
      return false;
    }
  }
}

template <int L>
struct MegaShape {
  static constexpr int P = 32 * L, NA = P / 2 + 1, LPW = 32 / L, RPC = 8 * LPW;
  static constexpr int nA = (NA + RPC - 1) / RPC;
  static constexpr int nB1 = (NA + RPC - 1) / RPC;
  static constexpr int nB2 = (NA + RPC / 2 - 1) / (RPC / 2);
  static __host__ __device__ int nC(int ny) { return (ny + RPC - 1) / RPC; }
};

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// A decoded ticket: stage (-1: no job at this slot, -2: past the end), job,
// tile, and up to two "counter >= target" dependencies.
struct Tk {
  int stage, job, tile;
  const int* d0;
  int t0;
  const int* d1;
  int t1;
};

template <int L>
__device__ __forceinline__ Tk decode(long long tk, const MegaArgs& a, int TPS, int nC,
                                     long long total) {
  using S = MegaShape<L>;
  Tk r{-2, 0, 0, nullptr, 0, nullptr, 0};
  if (tk >= total) return r;
  const int step = (int)(tk / TPS);
  int k = (int)(tk - (long long)step * TPS);
  int st, jb;
  if (k < S::nA) { st = 0; jb = step; }
  else if ((k -= S::nA) < S::nB1) { st = 1; jb = step - a.lag; }
  else if ((k -= S::nB1) < S::nB2) { st = 2; jb = step - 2 * a.lag; }
  else { k -= S::nB2; st = 3; jb = step - 3 * a.lag; }
  r.stage = (jb < 0 || jb >= a.njobs) ? -1 : st;
  if (r.stage < 0) return r;
  r.job = jb;
  r.tile = k;
  if (st == 0) {
    if (jb >= a.R) {   // ring slot free: previous occupant's B2 and C done
      r.d0 = a.ctr + 4 * (jb - a.R) + 2; r.t0 = S::nB2;
      r.d1 = a.ctr + 4 * (jb - a.R) + 3; r.t1 = nC;
    }
  } else if (st == 1) {
    r.d0 = a.ctr + 4 * jb + 0; r.t0 = S::nA;
  } else if (st == 2) {
    r.d0 = a.ctr + 4 * jb + 1; r.t0 = S::nB1;
  } else {
    r.d0 = a.ctr + 4 * jb + 2; r.t0 = S::nB2;
    const int pv = a.jobs[jb].prev;
    if (pv >= 0) { r.d1 = a.ctr + 4 * pv + 3; r.t1 = nC; }
  }
  return r;
}

// Scheduling (thread 0 only) runs two tickets ahead of the task being executed:
// the ticket after next is fetched with an atomic whose result is consumed one
// task later, and the next task's dependency counters are read (relaxed) at the
// previous scheduling point; the fence that publishes a finished task then also
// serves as the acquire for those reads.  Tickets held by a CTA are increasing
// and every dependency points to a smaller ticket, so the smallest unfinished
// ticket can always run: no deadlock, whatever the number of resident CTAs.
template <int L, bool MULTI, bool PRE>
__global__ void __launch_bounds__(MT, MULTI ? 1 : 2) k_prop_mega(MegaArgs a) {
  using S = MegaShape<L>;
  constexpr int NA = S::NA;
  extern __shared__ float2 sm[];
  __shared__ int s_task[3];   // stage, job, tile (stage < 0: finished)
  const int nC = S::nC(a.g.ny);
  const int TPS = S::nA + S::nB1 + S::nB2 + nC;
  const long long total = (long long)(a.njobs + 3 * a.lag) * TPS;
  int* ticket = a.ctr + 4 * a.njobs;
  int* abort_flag = ticket + 1;
  // Scheduler state: in-flight values stay in registers (3), the rest in shared.
  __shared__ int s_q0, s_done, s_fenced;
  int v0 = 0, v1 = 0;         // relaxed reads of the next task's counters
  int q1 = 0;                 // the ticket after it (atomic in flight)
  if (threadIdx.x == 0) {
    s_q0 = atomicAdd(ticket, 1);
    const Tk n = decode<L>(s_q0, a, TPS, nC, total);
    if (n.d0) v0 = ld_relaxed(n.d0);
    if (n.d1) v1 = ld_relaxed(n.d1);
    q1 = atomicAdd(ticket, 1);
    s_done = -1;
    s_fenced = 0;
  }
  for (;;) {
    __syncthreads();            // every thread's stores of the finished task are issued
    if (threadIdx.x == 0) {
      if (s_done >= 0) {        // release: cumulative over the CTA through the barrier
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        s_fenced = 1;
        atomicAdd(a.ctr + s_done, 1);
      }
      Tk cur;
      for (;;) {
        cur = decode<L>(s_q0, a, TPS, nC, total);
        bool ok = true;
        if (cur.stage >= 0) {
          const bool ready = (!cur.d0 || v0 >= cur.t0) && (!cur.d1 || v1 >= cur.t1);
          if (ready) {
            if (!s_fenced) asm volatile("fence.acq_rel.gpu;" ::: "memory");
          } else {
            ok = (!cur.d0 || wait_geq(cur.d0, cur.t0, abort_flag)) &&
                 (!cur.d1 || wait_geq(cur.d1, cur.t1, abort_flag));
          }
        }
        if (!ok || ld_relaxed(abort_flag)) { cur.stage = -2; break; }
        if (cur.stage == -2) break;
        s_q0 = q1;
        const Tk n = decode<L>(q1, a, TPS, nC, total);
        v0 = n.d0 ? ld_relaxed(n.d0) : 0;
        v1 = n.d1 ? ld_relaxed(n.d1) : 0;
        s_fenced = 0;
        q1 = atomicAdd(ticket, 1);
        if (cur.stage >= 0) break;
      }
      s_task[0] = cur.stage; s_task[1] = cur.job; s_task[2] = cur.tile;
      s_done = cur.stage >= 0 ? 4 * cur.job + cur.stage : -1;
    }
    __syncthreads();
    const int stage = s_task[0], job = s_task[1], tile = s_task[2];
    if (stage < 0) break;
    const MegaJob jd = a.jobs[job];
    const pf_plane pl = a.planes[jd.plane];
    const int slot = job % a.R;
    float2* wa = a.ws_a + (long long)slot * NA * NA;
    float2* wb = a.ws_b + (long long)slot * a.ws_b_slot;
    const double kturns = a.kturns[jd.f];
    switch (stage) {
      case 0: st_a<L>(sm, pl, kturns, a.tw, wa, tile); break;
      case 1: st_b1<L>(sm, a.tw, wa, tile); break;
      case 2: st_b2<L, MULTI>(sm, pl, a.g, a.tw, wa, a.uhat + jd.f * a.uhat_fs, wb, tile); break;
      default:
        st_c<L, MULTI, PRE>(sm, pl, kturns, a.g, a.tw, wb, a.ill, a.frame_w + jd.f * a.n_frames,
                            a.n_frames, a.vol, a.vfs, tile);
        break;
    }
  }
}

template <int L>
size_t mega_smem(int nx, bool pre) {
  constexpr int P = 32 * L, RPC = 8 * (32 / L), NA = P / 2 + 1;
  size_t x = 8 * WFFT_XCH, sa = (size_t)NA * (RPC + 1), sc = (size_t)P * (RPC + 1);
  size_t u = x > sa ? x : sa;
  u = u > sc ? u : sc;
  return (u + (pre ? (size_t)RPC * nx : 0)) * sizeof(float2);
}

template <int L, bool MULTI, bool PRE>
int launch_mega(const MegaArgs& a, cudaStream_t st) {
  static int attr = 0;
  const size_t smem = mega_smem<L>(a.g.nx, PRE);
  if (!attr) {
    cudaFuncSetAttribute(k_prop_mega<L, MULTI, PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         220 * 1024);
    attr = 1;
  }
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_prop_mega<L, MULTI, PRE>, MT, smem);
  if (per_sm < 1) {
    pf_set_error("pf_prop_mega: kernel does not fit on an SM (smem %zu)", smem);
    return -1;
  }
  k_prop_mega<L, MULTI, PRE><<<nsm * per_sm, MT, smem, st>>>(a);
  PF_LAUNCH_CHECK("k_prop_mega");
  return 0;
}

template <int L>
int mega_dispatch(const MegaArgs& a, cudaStream_t st) {
  constexpr int RPC = 8 * (32 / L);
  const bool pre = a.n_frames == 1 && (size_t)RPC * a.g.nx * 8 <= 64 * 1024;
  const bool multi = a.g.n_illum > 1;
  if (multi) return pre ? launch_mega<L, true, true>(a, st) : launch_mega<L, true, false>(a, st);
  return pre ? launch_mega<L, false, true>(a, st) : launch_mega<L, false, false>(a, st);
}

}  // namespace

int pf_prop_fast_L(const pf_prop_geom* g);

extern "C" int64_t pf_prop_mega_ws(const pf_prop_geom* g, int slots, int which) {
  const long long P = g->px, NA = P / 2 + 1;
  if (which == 0) return (int64_t)slots * NA * NA;
  return (int64_t)slots * g->n_illum * P * g->ny;
}

extern "C" int pf_prop_mega(const pf_plane* planes, const int32_t* jobs, int njobs,
                            const double* kturns, const pf_prop_geom* g, const pf_fft_plan* plan,
                            const void* uhat, int64_t uhat_fs, const double* ill_xyz,
                            const void* frame_w, int n_frames, void* vol,
                            int64_t vol_frame_stride, void* ws_a, void* ws_b, int slots, int lag,
                            int32_t* counters, void* stream) {
  PF_ARG_CHECK(njobs >= 1 && lag >= 1 && slots >= 3 * lag + 2,
               "pf_prop_mega: need njobs >= 1, lag >= 1, slots >= 3 lag + 2");
  const int L = pf_prop_fast_L(g);
  PF_ARG_CHECK(L != 0 && plan && plan->n == g->px,
               "pf_prop_mega: geometry not eligible for the register path");
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(counters, 0, (size_t)(4 * njobs + 2) * sizeof(int32_t), st);
  MegaArgs a;
  a.planes = planes;
  a.jobs = (const MegaJob*)jobs;
  a.njobs = njobs;
  a.kturns = kturns;
  a.uhat = (const float2*)uhat;
  a.uhat_fs = uhat_fs;
  a.frame_w = (const float2*)frame_w;
  a.n_frames = n_frames;
  a.ill = ill_xyz;
  a.g = *g;
  a.tw = (const float2*)plan->tw;
  a.ws_a = (float2*)ws_a;
  a.ws_b = (float2*)ws_b;
  a.ws_b_slot = (long long)g->n_illum * g->px * g->ny;
  a.R = slots;
  a.lag = lag;
  a.ctr = counters;
  a.vol = (float2*)vol;
  a.vfs = vol_frame_stride;
  switch (L) {
    case 4: return mega_dispatch<4>(a, st);
    case 8: return mega_dispatch<8>(a, st);
    case 16: return mega_dispatch<16>(a, st);
    case 32: return mega_dispatch<32>(a, st);
    default: break;
  }
  pf_set_error("pf_prop_mega: unsupported pad");
  return -1;
}

// Host check after the stream has synchronised: nonzero if the kernel gave up
// waiting on a dependency (never expected; a guard against a hung launch).
extern "C" int pf_prop_mega_aborted(const int32_t* counters, int njobs) {
  int32_t v = 0;
  if (cudaMemcpy(&v, counters + 4 * njobs + 1, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return v;
}
