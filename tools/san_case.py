"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck): rsd through both
the frequency-batched and the per-frequency (A, fused B, C Horner) launches, srsd
(Bluestein register passes), nursd1 (type-1 spreading + register finish), nursd2 (type-2
readout) and K1."""
import importlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_05244_b200 as pf  # noqa: E402

R = importlib.import_module("paper_2501_05244_b200.reconstruct")
rng = np.random.default_rng(3)
n, T, dt, lam = 64, 512, 16e-12, 0.06
p = 2.0 / n
g = pf.UniformGrid2D(n, n, p, p, -1 + p / 2, -1 + p / 2, 0.0)
relay = pf.UniformRelay(g)
ill = pf.PointList(np.array([[0.0, 0.0]]))
hist = rng.uniform(0.0, 3.0, size=(1, n * n, T)).astype(np.float32)
k = pf.build_kernel(lam, T, dt)
sl = pf.to_frequency(pf.TransientMeasurement(relay, ill, hist, dt, t0=1e-10), k)
grid = pf.CuboidGrid(pf.UniformGrid3D(n, n, 6, p, p, 0.2, g.x0, g.y0, 0.6))
pf.rsd(sl, grid)
R._FBATCH_BYTES = 0
pf.rsd(sl, grid)
zs = np.linspace(0.6, 1.6, 4)
pf.srsd(sl, pf.FrustumGrid(g, zs, zs[0] / zs, zs[0] / zs))
pts = rng.uniform(-1, 1, size=(1500, 2))
c = rng.normal(size=(1, 1500, k.n_freq)) + 1j * rng.normal(size=(1, 1500, k.n_freq))
sl1 = pf.FrequencySlices(k.frequencies, c, pf.NonUniformPlanarRelay(pf.PointList(pts), 0.0), ill)
pf.nursd1(sl1, grid)
planes = tuple(pf.VoxelPlane(z, pf.PointList(rng.uniform(-0.5, 0.5, size=(200, 2))))
               for z in (0.7, 0.9))
pf.nursd2(sl, pf.ExplicitVoxels(planes))
torch.cuda.synchronize()
print("san case ok")
