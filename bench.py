#!/usr/bin/env python
"""Bench: reconstructed voxels/s for BASELINE config 4 (RSD, 512x512 relay, 256 planes).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]

A step = one pass of the hot path over one capture: the temporal phasor
transform of all 262,144 x 4,096 float32 transients (K1) followed by RSD
propagation to the 512x512x256 complex volume.  ``value`` is device-timed with
inputs resident in HBM; ``e2e`` goes through the public host API
(``TransientReconstructor``: pinned host transients -> H2D -> K1 -> rsd ->
D2H volume) with the copies inside the timed region.

Multi-GPU (torchrun, one rank per GPU, NCCL): detectors are sharded for K1
and the slices all-gathered; depth planes are sharded contiguously for the
propagation and the finished plane blocks gathered to rank 0.  Total work is
fixed, so scaling is "strong".  Timing is max over ranks of CUDA-event time.

``--impl reference`` times the reference algorithm on the host CPU (the
oracle port of the pure-Python reference; /root/reference cannot travel to
the GPU box), process-parallel over (frequency, plane) units on all cores,
each step a bounded sample extrapolated to the full workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reconstructed voxels/sec (device-timed, 1/2/4/8 B200) + % HBM roofline vs CPU ref"
UNIT = "voxel/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        # NVML in-process (no fork of this large process every sample: a forking sampler
        # stalled the launching thread for milliseconds, which device events count as gaps
        # in launch-bound steps); nvidia-smi only when NVML is unavailable
        nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwPowerCap]
        except Exception:
            nv = None
        while not self._stop.is_set():
            try:
                if nv is not None:
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append([str(sm), str(mx)] +
                                        ["Active" if r & b else "Not Active" for b in bits])
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          "--query-gpu=" + self.Q, "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05 if nv is not None else 0.2)

    def __enter__(self):
        # the sampler (NVML init, first query) is up before the caller's timed region starts
        self._t.start()
        t0 = time.perf_counter()
        while not self.samples and time.perf_counter() - t0 < 3.0:
            time.sleep(0.01)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples else None,
                "reasons": reasons, "samples": len(self.samples)}


def _n_planes(grid):
    return {"frustum": lambda g: g.n_planes, "explicit": lambda g: len(g.planes),
            "voxels": lambda g: 1}.get(
        grid.kind, lambda g: g.grid.nz)(grid)


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2501_05244_b200 as pf
    from paper_2501_05244_b200 import _lib, configs
    from paper_2501_05244_b200.distributed import SliceGather, VolumeGather, shard_range
    from paper_2501_05244_b200.pipeline import TransientReconstructor

    world, rank, local = _dist_env()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("PF_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:   # gloo: CPU-staged collectives (used to exercise N>1 logic on one GPU)
            dist.init_process_group(backend)
    cfg = configs.config(args.config)
    kernel = configs.kernel(cfg)
    hist = configs.transients(cfg, device=device)            # [1, D, T] float32, identical per rank
    I, D, T = hist.shape
    F = kernel.n_freq
    nz = _n_planes(cfg.grid)
    explicit = cfg.grid.kind in ("explicit", "voxels")
    if explicit and world > 1:
        raise SystemExit("bench: config %d (explicit voxels) runs on one GPU" % args.config)
    d_lo, d_hi = shard_range(D, world, rank)
    k_lo, k_hi = shard_range(nz, world, rank)
    hist_shard = hist[:, d_lo:d_hi].contiguous()
    del hist
    torch.cuda.empty_cache()
    plane_vox = cfg.n_voxels // nz
    sgather = vgather = None
    if world > 1:
        sgather = SliceGather(F, I, D, world, device)
        vgather = VolumeGather(nz, plane_vox, 1, world, rank, device)
    rec = TransientReconstructor(kernel, cfg.relay, cfg.illuminations, cfg.grid, t0=cfg.t0,
                                 plane_range=(k_lo, k_hi), device=device,
                                 trace_range=(d_lo, d_hi), slice_gather=sgather,
                                 volume_gather=vgather, algorithm=cfg.algorithm,
                                 lattice=getattr(cfg, "lattice", None))
    eng = rec.engine
    local_shard = rec.coeff
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]

    # N > 1: the rank's planes run in chunks; each finished chunk is gathered to rank 0
    # on a side stream while the next chunk computes
    n_chunks = rec.gather_chunks

    # N > 1 on the Horner register path: the collectives fused into the kernels over peer
    # memory (K1 stores every rank's slices, kernel C stores rank 0's volume; CUDA IPC over
    # NVLink / NVSwitch) -- no NCCL data transfer, two one-element all-reduces for order
    peer = None
    if (world > 1 and os.environ.get("PF_PEER", "1") != "0" and I == 1 and T % 2048 == 0
            and hasattr(eng, "fused_gather_ok") and eng.fused_gather_ok()):
        from paper_2501_05244_b200.distributed import open_peer_collectives
        from paper_2501_05244_b200.phasor import temporal_peers
        # every rank maps the others' buffers; if any rank cannot (no peer access), all fall
        # back to the NCCL gathers together
        peer = open_peer_collectives(F, I, D, nz, plane_vox, world, rank, device)

    final = {}

    def step_peer():
        ps, pv = peer
        ev[0].record(stream)
        temporal_peers(rec.temporal, hist_shard.view(-1, T), ps, stream)
        ev[1].record(stream)
        ps.sync(stream)
        ev[2].record(stream)
        eng.run_graphed(ps.full, rec.vol, stream, vol_out=pv.out_ptr)
        ev[3].record(stream)
        final["vol"] = pv.sync(stream)
        ev[4].record(stream)

    def step():
        if peer is not None:
            return step_peer()
        ev[0].record(stream)
        rec.temporal.run(hist_shard.view(-1, T), local_shard.view(F, -1), stream)
        ev[1].record(stream)
        coeff = sgather(local_shard) if world > 1 else local_shard
        ev[2].record(stream)
        if n_chunks > 1:
            final["vol"] = rec.propagate_and_gather(coeff, rec.vol, stream)
            ev[3].record(stream)
        else:
            eng.run_graphed(coeff, rec.vol, stream)
            final["vol"] = rec.vol
            ev[3].record(stream)
            if world > 1:
                final["vol"] = vgather(rec.vol)
        ev[4].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    fp32_meas = _fp32_peak(device)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_k1, t_s3, t_step = [], [], []
    # the timing rule: inputs larger than L2, or an L2 flush between timed steps
    in_bytes = hist_shard.numel() * 4
    l2_bytes = torch.cuda.get_device_properties(device).L2_cache_size
    flush = None
    if in_bytes < 2 * l2_bytes:
        flush = torch.empty(4 * l2_bytes // 4, dtype=torch.float32, device=device)
    if flush is not None:   # the timed loop's exact sequence once, untimed (first-use costs)
        flush.fill_(1.0)
        torch.cuda._sleep(100_000)
        step()
        torch.cuda.synchronize()
    launches0 = _lib.launches()
    # no Python garbage collection inside the timed region: a collection pause between two
    # enqueued events of a short step is timed by the device as an idle gap
    import gc
    gc.collect()
    gc.disable()
    with ClockSampler(local) as clk:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for _ in range(args.steps):
            if flush is not None:
                flush.fill_(1.0)   # evict the previous step's data (not inside ev[0]..ev[4])
                # ~50 us of device work ahead of the step's first event, so the whole step
                # is enqueued before the device reaches it (per-step events: host jitter is
                # not timed as a gap in these launch-bound small steps)
                torch.cuda._sleep(100_000)
            step()
            torch.cuda.synchronize()
            t_k1.append(ev[0].elapsed_time(ev[1]))
            t_s3.append(ev[2].elapsed_time(ev[3]))
            t_step.append(ev[0].elapsed_time(ev[4]))
        end.record(stream)
        torch.cuda.synchronize()
    gc.enable()
    vol_digest = None
    if rank == 0 and final.get("vol") is not None:
        import hashlib
        # bytes of the last timed step's (gathered) volume: identical for every N
        vol_digest = hashlib.sha256(final["vol"].cpu().numpy().tobytes()).hexdigest()[:16]
    launches = (_lib.launches() - launches0) // max(1, args.steps)
    launches += eng_graph_launches(eng, n_chunks)
    # with flushes between steps the region also holds the flush writes: use the
    # per-step events (first kernel of the step to its last) instead
    total_ms = sum(t_step) if flush is not None else start.elapsed_time(end)
    if world > 1:
        dist.barrier()
        tt = torch.tensor([total_ms])
        if dist.get_backend() == "nccl":
            tt = tt.to(device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    value = cfg.n_voxels / (ms_per_step * 1e-3)

    # ---- end-to-end through the public host API ---------------------------------------
    # a stream of captures through TransientReconstructor.submit/result: every step
    # copies its transients host->device and its volume device->host; two captures
    # are in flight, so step i's upload overlaps step i-1's propagation
    e2e_line = None if args.no_e2e else _e2e_leg(rec, hist_shard, cfg, world, device)
    dropin = None
    if not args.no_e2e and world == 1 and cfg.algorithm in ("rsd", "srsd", "nursd1"):
        dropin = _dropin_leg(cfg, kernel, hist_shard, device)

    hbm_peak, sm_max, peak_src = _peaks()
    k1_ms = statistics.mean(t_k1)
    s3_ms = statistics.mean(t_s3)
    k1_bytes = (d_hi - d_lo) * I * T * 4 + F * I * (d_hi - d_lo) * 8
    P = eng.px
    units = F * (k_hi - k_lo) * I
    s3_flops = (2 * units + F * I) * 5.0 * P * P * math.log2(P * P)
    if cfg.algorithm == "srsd":   # + per-unit Bluestein x (N rows) and y (P columns) passes
        Q = 2 * P
        s3_flops += units * (cfg.relay.grid.ny + P) * 2 * 5.0 * Q * math.log2(Q)
    if cfg.algorithm == "nursd1":   # + per-(f, p) type-1 NUFFT: fine-grid FFT + 17x17 spread
        s3_flops += F * I * (5.0 * (2 * P) ** 2 * math.log2((2 * P) ** 2) + cfg.relay.count * 17 * 17 * 8)
    kernel_name = ("propagation k_pa + k_pb12 + k_pc_h (pf_prop_kernel_rows / columns / "
                   "rows_out_horner, S3)")
    if explicit:
        s3_flops, kernel_name = _explicit_flops(eng, F, I, cfg)
    fp32_nominal = 148 * 128 * 2 * sm_max * 1e6 / 1e12
    fp32_peak = fp32_meas if fp32_meas > 0 else fp32_nominal
    clocks = clk.summary()
    roof_k1 = {"bound": "hbm", "achieved": k1_bytes / (k1_ms * 1e-3) / 1e9, "peak": hbm_peak,
               "unit": "GB/s", "traffic": _traffic("k_temporal_dft", args.config, world),
               "kernel": "k_temporal_dft (K1)",
               "ms": k1_ms, "peak_source": peak_src}
    roof_k1["frac"] = roof_k1["achieved"] / hbm_peak
    roof_s3 = {"bound": "fp32", "achieved": s3_flops / (s3_ms * 1e-3) / 1e12, "peak": fp32_peak,
               "unit": "TFLOP/s", "traffic": _prop_traffic(F, k_hi - k_lo, args.config),
               "kernel": kernel_name,
               "ms": s3_ms, "peak_source": "measured on this GPU before the timed region: FFMA probe "
                                           "(pf_fp32_probe, best of 6); nominal %.1f TFLOP/s = "
                                           "148 SM x 128 lanes x 2 x sm_max_mhz; MEASURED_PEAKS.json "
                                           "has no FP32 entry" % fp32_nominal,
               "flops_model": _flops_model(cfg.algorithm, P),
               "traffic_note": "steady-state DRAM bytes per step of the propagation kernels "
                               "(ncu application replay, no cache control, kernels serialised "
                               "by the profiler; profiles/r2_traffic_steady.json): ~70x the "
                               "0.6 GB compulsory (slices in, volume out), mostly write-back "
                               "of the per-batch stage workspaces and the volume slices"}
    roof_s3["frac"] = roof_s3["achieved"] / fp32_peak
    ex = _executed_flops(cfg, eng, F, k_hi - k_lo, I)
    if ex is not None:
        roof_s3["executed"] = {
            "flops": ex[0], "achieved": ex[0] / (s3_ms * 1e-3) / 1e12,
            "frac": ex[0] / (s3_ms * 1e-3) / 1e12 / fp32_peak, "unit": "TFLOP/s",
            "model": ex[1]}
    dominant, other = (roof_s3, roof_k1) if s3_ms >= k1_ms else (roof_k1, roof_s3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c64 (fp32 arithmetic, fp64 phases)",
        "data": f"synthetic (seeded GPU three-bounce renderer, Poisson noise; BASELINE config "
                f"{args.config})",
        "config": {"workload": f"config{args.config}-{cfg.algorithm}", "relay": cfg.relay.count,
                   "n_bins": T, "n_freq": F, "planes": nz,
                   "voxels": cfg.n_voxels, "pad": P, "parallelism": f"planes+detectors x{world}",
                   "l2": ("inputs (%.2f GB transients) exceed the %d MB L2; no flush needed"
                          % (in_bytes / 1e9, l2_bytes >> 20)) if flush is None else
                         ("inputs (%.1f MB transients) fit the %d MB L2: a %d MB buffer is written "
                          "between timed steps (outside the step events)"
                          % (in_bytes / 1e6, l2_bytes >> 20, flush.numel() * 4 >> 20)),
                   "timed": "K1 + slice gather + propagation + volume gather"},
        "roofline": dominant, "roofline_other": other,
        "stage_ms": {"k1": k1_ms, "propagation": s3_ms, "step_event": statistics.mean(t_step),
                     "k1_min": min(t_k1), "propagation_min": min(t_s3),
                     "step_event_max": max(t_step)},
        "e2e": e2e_line,
        "e2e_dropin": dropin,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "volume_sha256_16": vol_digest,
        "dist_backend": (dist.get_backend() if world > 1 else None),
        "collectives": (None if world == 1 else
                        "fused into K1 and kernel C over peer memory (CUDA IPC)" if peer is not None
                        else "NCCL all-gather + chunked gather"),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_sample(cfg, kernel, hist_shard, rec, args)
    if peer is not None:
        torch.cuda.synchronize()
        dist.barrier()
        for pb in peer:
            pb.close()
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def _e2e_leg(rec, hist_shard, cfg, world, device):
    """Stream of captures through TransientReconstructor.submit/result: every step copies
    its transients host->device and its volume device->host; two captures are in flight,
    so step i's upload overlaps step i-1's propagation."""
    import torch
    import torch.distributed as dist
    hist_host = torch.empty(hist_shard.shape, dtype=torch.float32, pin_memory=True)
    hist_host.copy_(hist_shard)
    n_e2e = 16   # captures in the timed window (the pipeline fill is part of it)
    for _ in range(2):
        rec.result(rec.submit(hist_host))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    handles = [rec.submit(hist_host) for _ in range(2)]
    done_at = []
    for _ in range(n_e2e - 2):
        rec.result(handles.pop(0))
        done_at.append(time.perf_counter())
        handles.append(rec.submit(hist_host))
    for h in handles:
        rec.result(h)
        done_at.append(time.perf_counter())
    torch.cuda.synchronize()
    e2e = (time.perf_counter() - t0) * 1e3 / n_e2e      # whole window, pipeline fill included
    e2e_steady = (done_at[-1] - done_at[0]) * 1e3 / (len(done_at) - 1)
    h2d_gbs = _h2d_probe(hist_host, device)
    # single-capture latency through the blocking call, for reference
    for _ in range(2):
        rec(hist_host)
    torch.cuda.synchronize()
    a = time.perf_counter()
    rec(hist_host)
    torch.cuda.synchronize()
    e2e_latency = (time.perf_counter() - a) * 1e3
    if world > 1:
        tt = torch.tensor([e2e, e2e_latency])
        if dist.get_backend() == "nccl":
            tt = tt.to(device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e, e2e_latency = float(tt[0].item()), float(tt[1].item())

    return {"value": cfg.n_voxels / (e2e * 1e-3), "unit": UNIT, "ms_per_step": e2e,
            "single_capture_latency_ms": e2e_latency, "captures": n_e2e,
            "steady_ms_per_step": e2e_steady,
            "h2d_gbs_measured": h2d_gbs,
            "h2d_floor_ms": hist_host.numel() * 4 / (h2d_gbs * 1e6),
            "h2d_bytes_per_step": int(hist_host.numel() * 4 * world),
            "d2h_bytes_per_step": int(cfg.n_voxels * 8),
            "path": "TransientReconstructor.submit/result stream (pinned host f32 -> chunked "
                    "H2D||K1 -> propagation -> D2H; 2 captures in flight; wall clock)"}


def _dropin_leg(cfg, kernel, hist_dev, device, reps=3):
    """The call a reference user makes, timed end to end on the wall clock:
    ``pf.reconstruct(pf.to_frequency(measurement, kernel), grid, algorithm)`` with the
    measurement's float32 histograms in (pageable) numpy host memory and the
    ReconstructionVolume (complex128 numpy field) back on the host.  The measurement is
    built once, outside the timed region (reference core.py TransientMeasurement)."""
    import torch

    import paper_2501_05244_b200 as pf
    hist_np = hist_dev.cpu().numpy()
    m = pf.TransientMeasurement(cfg.relay, cfg.illuminations, hist_np, cfg.delta_t, cfg.t0)
    del hist_np

    def call():
        return pf.reconstruct(pf.to_frequency(m, kernel), cfg.grid, cfg.algorithm)

    call()          # plans (engine cache miss + graph capture) once, as a user's first call
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        v = call()
        ts.append(time.perf_counter() - t)
    ms = statistics.median(ts) * 1e3
    return {"value": cfg.n_voxels / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "reps": reps, "all_ms": [x * 1e3 for x in ts],
            "h2d_bytes_per_step": int(m.histograms.nbytes),
            "d2h_bytes_per_step": int(cfg.n_voxels * 8),
            "host_field_bytes": int(v.field.nbytes),
            "path": "pf.reconstruct(pf.to_frequency(m, k), grid, '%s'): numpy float32 "
                    "histograms -> H2D -> K1 -> propagation (cached engine, graph replay) -> "
                    "D2H -> complex128 ReconstructionVolume; wall clock, median" % cfg.algorithm}


def eng_graph_launches(eng, n_chunks=1):
    """libpfgpu kernels replayed per step from the engine's captured CUDA graph(s)."""
    if n_chunks > 1:
        per = getattr(eng, "chunk_graph_kernels", {})
        return int(sum(per.get((j, n_chunks), 0) for j in range(n_chunks)))
    return int(getattr(eng, "graph_kernels", 0))


def _executed_flops(cfg, eng, F, nz, I):
    """FFT work the register path actually executes per step (5 n log2 n per executed
    length-P line): per (f, plane, illumination) unit A transforms P/2 + 1 kernel rows,
    the fused B1/B2 kernel P/2 + 1 Ghat columns plus 2 (P/2 + 1) - 2 product columns,
    C ny output rows; per (f, illumination) the relay spectrum ny rows + P columns.
    The nominal model counts 4P lines per unit (two full 2D transforms)."""
    P = getattr(eng, "px", None)
    if cfg.algorithm != "rsd" or P is None or P & (P - 1):
        return None
    ny = cfg.grid.grid.ny
    line = 5.0 * P * math.log2(P)
    per_unit = (P // 2 + 1) + (P // 2 + 1) + (2 * (P // 2 + 1) - 2) + ny
    per_f = ny + P
    flops = (F * nz * I * per_unit + F * I * per_f) * line
    return flops, ("(F*Nz*I*((P/2+1) + (P/2+1) + (P) + ny) + F*I*(ny + P)) * 5 P log2 P, "
                   "P=%d, ny=%d: executed line-FFTs after the kernel symmetry and crop "
                   "pruning" % (P, ny))


def _explicit_flops(eng, F, I, cfg):
    """Config 2 (nursd3d stage 1 + nursd2 readout), standard counts: stage 1 per frequency
    = 3D type-1 spreading (L points x 17^3 x 8) + the 3D fine-grid FFT; stage 2 per
    (frequency, plane) = the kernel's 2D FFT on the P x P pad + the fine-grid inverse FFT
    + the 17 x 17 interpolation of every voxel (8 flops per tap)."""
    s1, s2 = eng.stage1, eng.stage2.ro
    fine3 = int(s1.plan.fine_elems) if hasattr(s1, "plan") else 0
    f1 = F * I * (cfg.relay.count * 17 ** 3 * 8 + (5.0 * fine3 * math.log2(fine3) if fine3 else 0))
    P2 = s2.px * s2.py
    fine2 = s2.plan.fine_elems
    # voxel clouds: every slab's Chebyshev node is a plane, every voxel reads all its nodes
    nodes = getattr(s2, "nodes", 1)
    nplanes = s2.n_slabs * nodes if hasattr(s2, "n_slabs") else s2.n_planes
    f2 = F * I * nplanes * (5.0 * P2 * math.log2(P2) + 5.0 * fine2 * math.log2(fine2))
    f2 += F * I * cfg.n_voxels * 17 * 17 * 8 * nodes
    return f1 + f2, ("stage 1 + stage 2 (type-1 spread + 3D FFT; kernel 2D FFT + fine-grid "
                     "IFFT + 17x17 interpolation; 5 n log2 n per FFT, 8 flops per tap)")


def _flops_model(alg, P):
    base = "(2*F*Nz*I + F*I) * 5 P^2 log2(P^2)"
    if alg == "srsd":
        base += " + F*Nz*I * (N + P) * 2 * 5 Q log2(Q), Q=2P (Bluestein x and y passes)"
    elif alg == "nursd1":
        base += " + F*I * (5 (2P)^2 log2((2P)^2) + L * 17^2 * 8) (type-1 NUFFT)"
    return base + ", P=%d" % P


def _steady():
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic_steady.json")) as f:
            return json.load(f)
    except Exception:
        return None


def _prop_traffic(n_freq, n_planes, config):
    """Steady-state DRAM bytes per step of the propagation kernels (A, fused B, C and the
    relay spectra) from the committed ncu application-replay capture without cache control
    (profiles/r2_traffic_steady.json, config 4, F = 32, all 256 planes); null for other
    configurations (not measured)."""
    t = _steady()
    if t is None or int(config) != 4 or n_freq != 32 or n_planes != 256:
        return None
    return t["propagation_dram_bytes_per_step"]


def _traffic(kernel_prefix, config, world=1):
    """K1's DRAM bytes per launch from the same capture (config 4, one GPU)."""
    t = _steady()
    if t is None or int(config) != 4 or world != 1:
        return None
    for name, d in t["kernels"].items():
        if name.startswith(kernel_prefix):
            return d["dram_read_bytes_per_step"] + d["dram_write_bytes_per_step"]
    return None


# ---------------------------------------------------------------------------
# CPU baselines (oracle port of the reference; test infrastructure)
# ---------------------------------------------------------------------------


def _fp32_peak(device) -> float:
    """FP32 FFMA throughput measured on this GPU (TFLOP/s; best of 5), the roofline
    denominator SURVEY 8(d) asks for (MEASURED_PEAKS.json has no FP32 entry)."""
    import torch
    from paper_2501_05244_b200 import _device as dev
    from paper_2501_05244_b200 import _lib
    nsm = torch.cuda.get_device_properties(device).multi_processor_count
    blocks, iters = nsm * 8, 2048
    out = torch.empty(blocks * 256, dtype=torch.float32, device=device)
    best = 0.0
    for _ in range(6):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _lib.call("pf_fp32_probe", dev.ptr(out), blocks, iters, dev.stream_ptr())
        e.record()
        torch.cuda.synchronize()
        flops = 2.0 * 8 * 16 * iters * blocks * 256
        best = max(best, flops / (s.elapsed_time(e) * 1e-3) / 1e12)
    return best


def _h2d_probe(hist_host, device) -> float:
    """Pinned host -> device copy bandwidth (GB/s) of one capture-sized transfer: the
    floor of the e2e step when the capture does not fit the PCIe budget."""
    import torch
    dst = torch.empty_like(hist_host, device=device)
    dst.copy_(hist_host, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(2):
        dst.copy_(hist_host, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    del dst
    return 2 * hist_host.numel() * 4 / (s.elapsed_time(e) * 1e-3) / 1e9


def _cpu_units(cfg, n_f, n_k):
    """Bounded sample: all-detector slices for n_f frequencies x n_k planes."""
    return n_f, n_k


def cpu_baseline_sample(cfg, kernel, hist_dev, rec, args):
    from oracle import pf_oracle as O

    F = kernel.n_freq
    nz = _n_planes(cfg.grid)
    n_tr = 4096
    h = hist_dev.view(-1, cfg.n_bins)[:n_tr].cpu().numpy().astype(np.float64)
    t = time.perf_counter()
    O.to_frequency(h, kernel.bin_indices, kernel.frequencies, kernel.weights, cfg.t0)
    t1 = (time.perf_counter() - t) * (hist_dev.shape[1] / n_tr)
    coeff = rec.coeff.permute(1, 2, 0).cpu().numpy().astype(np.complex128)
    sl = _HostSlices(kernel.frequencies, coeff, cfg.relay, cfg.illuminations)
    if cfg.algorithm == "nursd3d-explicit":
        # composed oracle (stage 1 + nursd2) on one frequency, single core, times F; a voxel
        # cloud is one reference plane per voxel: a voxel subsample, extrapolated per voxel
        from oracle.pool import _OneFreq
        grid, scale = _oracle_voxels(cfg.grid, 200)
        t = time.perf_counter()
        O.nursd3d_explicit(_OneFreq(sl, 0), grid, cfg.lattice,
                           z_pitch=sl.shortest_wavelength / 2.0)
        t3 = (time.perf_counter() - t) * F * scale
        return {"value": cfg.n_voxels / (t1 + t3), "unit": UNIT, "cores": 1, "kind": "port",
                "sample": f"oracle.to_frequency on {n_tr} of {hist_dev.shape[1]} traces + the "
                          f"composed oracle (nursd3d stage 1 + nursd2) for 1 of {F} frequencies"
                          + (f" on {grid.count} of {cfg.n_voxels} voxels (one plane each)"
                             if scale != 1.0 else "") +
                          "; per-trace, per-frequency (and per-voxel) linear extrapolation",
                "s1_s": t1, "s3_s": t3}
    fn = {"rsd": O.rsd, "srsd": O.srsd, "nursd1": O.nursd1}[cfg.algorithm]
    # per-frequency setup (relay spectrum / NUFFT) and per-plane cost separated by
    # timing 1 and 3 planes per frequency, then extrapolated to F x Nz
    n_f = 2
    per_f, per_k = [], []
    for f in range(n_f):
        t = time.perf_counter()
        fn(sl, cfg.grid, freq_range=(f, f + 1), plane_range=(0, 1))
        a = time.perf_counter() - t
        t = time.perf_counter()
        fn(sl, cfg.grid, freq_range=(f, f + 1), plane_range=(0, 3))
        b = time.perf_counter() - t
        per_k.append(max(b - a, 1e-9) / 2)
        per_f.append(max(a - per_k[-1], 0.0))
    t3 = F * (statistics.mean(per_f) + nz * statistics.mean(per_k))
    n_k = 3
    return {"value": cfg.n_voxels / (t1 + t3), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle.to_frequency on {n_tr} of {hist_dev.shape[1]} traces + oracle."
                      f"{cfg.algorithm} (reference pads) on {n_f} freqs x (1 and 3) planes of "
                      f"{F}x{nz}; per-trace and per-frequency + per-plane linear extrapolation",
            "s1_s": t1, "s3_s": t3}


class _HostSlices:
    def __init__(self, freqs, coeff, relay, ill):
        self.frequencies = np.asarray(freqs)
        self.coefficients = coeff
        self.relay = relay
        self.illuminations = ill
        self.n_freq = self.frequencies.size

    @property
    def shortest_wavelength(self):
        return 2.0 * math.pi * 299792458.0 / float(self.frequencies.max())


_REF_STATE = {}


def _ref_unit(unit):
    """Worker: oracle on 1 and 3 planes of one frequency -> (per-frequency, per-plane) seconds."""
    from oracle import pf_oracle as O
    f, k0 = unit
    fn = {"rsd": O.rsd, "srsd": O.srsd, "nursd1": O.nursd1}[_REF_STATE["alg"]]
    sl, grid = _REF_STATE["slices"], _REF_STATE["grid"]
    t = time.perf_counter()
    fn(sl, grid, freq_range=(f, f + 1), plane_range=(k0, k0 + 1))
    a = time.perf_counter() - t
    t = time.perf_counter()
    fn(sl, grid, freq_range=(f, f + 1), plane_range=(k0, k0 + 3))
    b = time.perf_counter() - t
    per_k = max(b - a, 1e-9) / 2
    return max(a - per_k, 0.0), per_k


def _ref_task(task):
    """Worker of the reference arm: one task of a step's bounded sub-workload, either
    ("s3", f, k0, k1): the reference algorithm's term of frequency f on planes [k0, k1), or
    ("s1", n): to_frequency on n traces.  Returns the seconds it took."""
    from oracle import pf_oracle as O
    t = time.perf_counter()
    if task[0] == "s3":
        _, f, k0, k1 = task
        fn = {"rsd": O.rsd, "srsd": O.srsd, "nursd1": O.nursd1}[_REF_STATE["alg"]]
        fn(_REF_STATE["slices"], _REF_STATE["grid"], freq_range=(f, f + 1), plane_range=(k0, k1))
    else:
        k = _REF_STATE["kernel"]
        O.to_frequency(_REF_STATE["hist"][:task[1]], k.bin_indices, k.frequencies, k.weights,
                       _REF_STATE["t0"])
    return time.perf_counter() - t


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    import multiprocessing as mp

    import paper_2501_05244_b200 as pf
    from oracle import pf_oracle as O
    from paper_2501_05244_b200 import configs

    cfg = configs.config(args.config)
    kernel = configs.kernel(cfg)
    F = kernel.n_freq
    nz = _n_planes(cfg.grid)
    D = cfg.relay.count
    rng = np.random.default_rng(cfg.seed)
    # S3 cost is data-independent FFT work: seeded random-phase coefficients stand in
    coeff = np.exp(2j * np.pi * rng.random((1, D, F)))
    sl = _HostSlices(kernel.frequencies, coeff, cfg.relay, cfg.illuminations)
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    if cfg.algorithm == "nursd3d-explicit":
        return _run_reference_explicit(args, cfg, kernel, sl, ncores, world)
    # A step = the reference algorithm's complete work for a bounded part of the capture: n_s
    # of the nz depth planes with every frequency term (tasks of one frequency x a block of
    # planes, shared by all host cores) and to_frequency on the same fraction n_s / nz of the
    # traces.  value = the voxels of those planes / the step's measured wall time: measured,
    # not extrapolated.  n_s is sized from one calibration task so a step takes a few seconds.
    _REF_STATE.update(slices=sl, grid=cfg.grid, alg=cfg.algorithm, kernel=kernel, t0=cfg.t0)
    # tasks = (frequency, block of the step's planes): as few plane blocks as balance the F
    # frequencies over the cores, so the per-frequency work (relay spectrum, type-1 NUFFT) is
    # repeated as little as possible (once per frequency when F is a multiple of the cores)
    nblk = min(range(1, 5), key=lambda b: (-(-F * b // ncores) * ncores / (F * b), b))
    _ref_task(("s3", 0, 0, 1))               # first call: imports, plan caches
    t = time.perf_counter()
    _ref_task(("s3", 0, 0, 1))
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    _ref_task(("s3", 0, 0, 3))
    t3 = time.perf_counter() - t
    per_k = max((t3 - t1) / 2, 1e-6)
    per_f = max(t1 - per_k, 0.0)
    target_s = float(os.environ.get("PF_REF_STEP_SECONDS", "5"))
    # step ~ 1.5 (cores sharing memory bandwidth) x F (nblk per_f + n_s per_k) / ncores
    n_s = int((target_s * ncores / (1.5 * F) - nblk * per_f) / per_k)
    n_s = max(nblk, min(nz, n_s)) // nblk * nblk
    pb = n_s // nblk
    blocks = [(k0, k0 + pb) for k0 in range(0, n_s, pb)]
    n_tr = max(ncores, int(round(D * n_s / nz)))
    per = -(-n_tr // ncores)
    _REF_STATE["hist"] = rng.poisson(2.0, size=(per, cfg.n_bins)).astype(np.float64)
    tasks = [("s3", f, k0, k1) for (k0, k1) in blocks for f in range(F)]
    tasks += [("s1", min(per, n_tr - i * per)) for i in range(ncores) if n_tr - i * per > 0]
    plane_vox = cfg.n_voxels // nz
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(ncores) as pool:
        for it in range(args.warmup + args.steps):
            t = time.perf_counter()
            list(pool.imap_unordered(_ref_task, tasks, chunksize=1))
            dt = time.perf_counter() - t
            if it >= args.warmup:
                times.append(dt)
    est = statistics.mean(times)
    value = n_s * plane_vox / est
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": est * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c128 (float64)", "data": "synthetic (seeded random-phase slices, Poisson hist)",
        "config": {"workload": f"config{args.config}-{cfg.algorithm}", "voxels": cfg.n_voxels,
                   "pad": "reference pad rule",
                   "step": f"{n_s} of {nz} planes x all {F} frequencies + to_frequency on "
                           f"{n_tr} of {D} traces ({n_s * plane_vox} voxels per step)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ncores, "kind": "port",
                         "sample": f"per step, measured (not extrapolated): oracle.{cfg.algorithm} "
                                   f"for {n_s} of {nz} planes, every frequency term ({len(blocks) * F} "
                                   f"tasks of 1 frequency x {pb} planes over {ncores} processes; the "
                                   f"cross-process sum of the terms is not formed) + to_frequency on "
                                   f"{n_tr} of {D} traces; value = those planes' voxels / step time"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def _respawn(args) -> bool:
    """``--gpus N`` without a launcher: re-exec this script under torch.distributed.run with
    N ranks (one per GPU, rendezvous on 127.0.0.1). Returns True when it did (the caller
    exits with the launcher's status)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stderr.write("bench: --gpus %d without WORLD_SIZE: %s\n" % (args.gpus, " ".join(cmd)))
    rc = subprocess.call(cmd)
    sys.exit(rc)


def _oracle_voxels(grid, n):
    """The oracle's view of an output grid: explicit planes as they are; a voxel cloud as
    one reference plane per voxel (reconstruct.py:393-410), subsampled to n voxels plus the
    lateral extremes (the nursd2 pad depends on them) -> (grid, extrapolation factor)."""
    if grid.kind != "voxels":
        return grid, 1.0
    from paper_2501_05244_b200.core import VoxelCloud
    pts = np.asarray(grid.points)
    rng = np.random.default_rng(11)
    keep = np.unique(np.concatenate([rng.choice(pts.shape[0], size=min(n, pts.shape[0]),
                                                replace=False),
                                     [pts[:, 0].argmin(), pts[:, 0].argmax(),
                                      pts[:, 1].argmin(), pts[:, 1].argmax()]]))
    return VoxelCloud(pts[keep]).as_explicit(), pts.shape[0] / keep.size


def _run_reference_explicit(args, cfg, kernel, sl, ncores, world):
    """Config 2: the whole composed oracle (nursd3d stage 1 + nursd2, every frequency,
    every voxel) per step, frequencies spread over the host cores and added in ascending
    order (oracle.pool); plus to_frequency on a trace sample."""
    from oracle import pf_oracle as O
    from oracle.pool import oracle_freq_terms
    F, D = kernel.n_freq, cfg.relay.count
    n_tr = 2048
    h = np.random.default_rng(1).poisson(2.0, size=(n_tr, cfg.n_bins)).astype(np.float64)
    grid, scale = _oracle_voxels(cfg.grid, 400)
    times = []
    for it in range(args.warmup + args.steps):
        t = time.perf_counter()
        oracle_freq_terms("nursd3d_explicit", sl, (grid, cfg.lattice), procs=ncores,
                          z_pitch=sl.shortest_wavelength / 2.0)
        t3 = (time.perf_counter() - t) * scale
        t = time.perf_counter()
        O.to_frequency(h, kernel.bin_indices, kernel.frequencies, kernel.weights, cfg.t0)
        t1 = (time.perf_counter() - t) * D / n_tr / ncores
        if it >= args.warmup:
            times.append(t3 + t1)
    est = statistics.mean(times)
    value = cfg.n_voxels / est
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": est * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c128 (float64)", "data": "synthetic (seeded random-phase slices, Poisson hist)",
        "config": {"workload": f"config{args.config}-{cfg.algorithm}", "voxels": cfg.n_voxels,
                   "pad": "reference pad rules"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ncores, "kind": "port",
                         "sample": (f"per step: the full composed oracle over all {F} frequencies "
                                    f"and {cfg.n_voxels} voxels " if scale == 1.0 else
                                    f"per step: the composed oracle over all {F} frequencies on "
                                    f"{grid.count} of {cfg.n_voxels} voxels (one reference plane "
                                    f"each), extrapolated per voxel, ") +
                                   f"({min(ncores, F)} processes, one frequency each) + "
                                   f"to_frequency on {n_tr} traces, extrapolated to {D} traces"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true",
                    help="skip the end-to-end leg (for ncu launch lists of the device step)")
    args = ap.parse_args()
    _respawn(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
