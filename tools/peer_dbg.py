import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2501_05244_b200 as pf
from paper_2501_05244_b200.phasor import TemporalPlan, to_frequency_device
from paper_2501_05244_b200 import _lib, _device as dev
rng = np.random.default_rng(9)
n, T, dt = 64, 2048, 8e-12
hist = rng.poisson(2.0, size=(1, n * n, T)).astype(np.float32)
k = pf.build_kernel(0.06, T, dt)
d = torch.device('cuda', 0)
h = torch.from_numpy(hist).to(d)
ref = to_frequency_device(h, k, 1e-10)
plan = TemporalPlan(k, 1e-10, d)
full = torch.zeros_like(ref)
peers = torch.tensor([full.data_ptr()], dtype=torch.int64, device=d)
for lo, hi in ((0, 2048), (2048, 4096)):
    _lib.call("pf_temporal_dft_peers", h[0, lo:hi].data_ptr(), hi - lo, T, dev.ptr(plan.bins), dev.ptr(plan.tw), dev.ptr(plan.wphase), plan.n_freq, plan.inner_mask, peers.data_ptr(), 1, n * n, lo, 0)
torch.cuda.synchronize()
bad = (full != ref).nonzero()
print('F', k.n_freq, 'bins', k.bin_indices, 'bad rows', sorted(set(bad[:, 0].tolist())), len(bad))
