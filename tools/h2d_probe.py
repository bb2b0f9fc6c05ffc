"""Host-side rates that bound the drop-in path: pageable H2D of a numpy array, threaded
memcpy into pinned memory, pinned H2D, cudaHostRegister of the numpy buffer, and the
drop-in call split into to_frequency / reconstruct / volume construction (config 4)."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = 4 << 30
a = np.ones(n // 4, dtype=np.float32)
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(torch.from_numpy(a)); torch.cuda.synchronize()
    print("pageable H2D 4 GiB: %.1f ms (%.1f GB/s)" % ((time.perf_counter() - t) * 1e3, n / (time.perf_counter() - t) / 1e9))
pin = torch.empty(256 << 20 >> 2, dtype=torch.float32, pin_memory=True)
pn = pin.numpy()
for th in (1, 4, 8, 16):
    ex = ThreadPoolExecutor(th)
    t = time.perf_counter()
    step = pn.size // th
    for rep in range(4):
        src = a[rep * pn.size:(rep + 1) * pn.size]
        list(ex.map(lambda i: np.copyto(pn[i * step:(i + 1) * step], src[i * step:(i + 1) * step]), range(th)))
    dt = time.perf_counter() - t
    print("memcpy numpy->pinned 1 GiB, %d threads: %.1f ms (%.1f GB/s)" % (th, dt * 1e3, (1 << 30) / dt / 1e9))
    ex.shutdown()
torch.cuda.synchronize(); t = time.perf_counter()
for rep in range(4):
    d[:pin.numel()].copy_(pin, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("pinned H2D 1 GiB: %.1f ms (%.1f GB/s)" % (dt * 1e3, (1 << 30) / dt / 1e9))
cr = torch.cuda.cudart()
t = time.perf_counter()
r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
dt = time.perf_counter() - t
print("cudaHostRegister 4 GiB: rc=%s %.1f ms" % (r, dt * 1e3))
torch.cuda.synchronize(); t = time.perf_counter()
d.copy_(torch.from_numpy(a), non_blocking=True); torch.cuda.synchronize()
dt = time.perf_counter() - t
print("registered H2D 4 GiB: %.1f ms (%.1f GB/s)" % (dt * 1e3, n / dt / 1e9))
t = time.perf_counter()
cr.cudaHostUnregister(a.ctypes.data)
print("unregister: %.1f ms" % ((time.perf_counter() - t) * 1e3))

import paper_2501_05244_b200 as pf  # noqa: E402
from paper_2501_05244_b200 import configs  # noqa: E402
cfg = configs.config(4)
k = pf.build_kernel(cfg.lambda_c, cfg.n_bins, cfg.delta_t)
h = configs.transients(cfg, device=torch.device("cuda")).cpu().numpy()
m = pf.TransientMeasurement(cfg.relay, cfg.illuminations, h, cfg.delta_t, cfg.t0)
pf.reconstruct(pf.to_frequency(m, k), cfg.grid, "rsd")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sl = pf.to_frequency(m, k); torch.cuda.synchronize(); t1 = time.perf_counter()
    v = pf.reconstruct(sl, cfg.grid, "rsd"); t2 = time.perf_counter()
    print("drop-in: to_frequency %.1f ms, reconstruct (incl. volume) %.1f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
R = sys.modules["paper_2501_05244_b200.reconstruct"]
eng = next(iter(R._ENGINES.values()))
from paper_2501_05244_b200.phasor import device_coefficients  # noqa: E402
c = device_coefficients(sl)
torch.cuda.synchronize(); t = time.perf_counter()
vol = eng.run_dropin(c); torch.cuda.synchronize(); t1 = time.perf_counter()
vv = R._volume(cfg.grid, vol, None); t2 = time.perf_counter()
print("run_dropin %.1f ms, _volume %.1f ms" % ((t1 - t) * 1e3, (t2 - t1) * 1e3))
