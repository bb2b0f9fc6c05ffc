"""Time BASELINE config 2 (non-planar relay -> 1e6 arbitrary voxels) on one GPU.

Planning (geometry only: pads, NUFFT plans, point buckets) is built once, as an
engine; each capture then runs K1 + stage 1 + the nursd2 readout.  Reported:
planning seconds, device time per capture (CUDA events, eager and CUDA-graph
replay) and the wall clock of a capture through the public function (planning
included) for reference.
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_05244_b200 as pf  # noqa: E402
from paper_2501_05244_b200 import configs  # noqa: E402
from paper_2501_05244_b200.algorithms import Nursd3dExplicitEngine, nursd3d_explicit  # noqa: E402

cfg = configs.config(2)
hist = configs.transients(cfg, device=torch.device("cuda"))
k = pf.build_kernel(cfg.lambda_c, cfg.n_bins, cfg.delta_t)
coeff = pf.to_frequency_device(hist, k, cfg.t0)
sl = pf.DeviceFrequencySlices(k.frequencies, coeff, cfg.relay, cfg.illuminations)
torch.cuda.synchronize()
t = time.perf_counter()
eng = Nursd3dExplicitEngine(sl, cfg.grid, cfg.lattice)
torch.cuda.synchronize()
plan_s = time.perf_counter() - t
vol = torch.zeros((1, cfg.grid.count), dtype=torch.complex64, device="cuda")


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e))
    return min(out)


def capture():
    c = pf.to_frequency_device(hist, k, cfg.t0)
    eng.run(c, vol)


eager_ms = timed(capture)
graph_ms = timed(lambda: eng.run_graphed(sl.device_coefficients, vol))
k1_ms = timed(lambda: pf.to_frequency_device(hist, k, cfg.t0))
torch.cuda.synchronize()
t = time.perf_counter()
nursd3d_explicit(sl, cfg.grid, cfg.lattice)
torch.cuda.synchronize()
wall_s = time.perf_counter() - t
print(json.dumps({"config": "config2-nursd3d-explicit", "voxels": cfg.grid.count,
                  "n_freq": k.n_freq, "planning_s": plan_s,
                  "device_ms_k1_plus_reconstruct_eager": eager_ms,
                  "device_ms_reconstruct_graphed_plus_k1": graph_ms + k1_ms,
                  "voxels_per_s_device": cfg.grid.count / ((graph_ms + k1_ms) * 1e-3),
                  "public_call_wall_s_incl_planning": wall_s}))
