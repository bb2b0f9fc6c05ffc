for c in "3 4" "4 4" "2 4" "3 2" "4 2" "6 2"; do
  set -- $c
  echo "lanes=$1 cap=$2: $(PF_LANES=$1 PF_BATCH_CAP=$2 python - <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2501_05244_b200 as pf
from paper_2501_05244_b200 import configs
from paper_2501_05244_b200.pipeline import _Meta
cfg = configs.config(4)
k = pf.build_kernel(cfg.lambda_c, cfg.n_bins, cfg.delta_t)
meta = _Meta(k, cfg.relay, cfg.illuminations)
coeff = torch.from_numpy(np.exp(2j*np.pi*np.random.default_rng(0).random((k.n_freq,1,cfg.relay.count))).astype(np.complex64)).cuda()
res = []
for n in (8, 4, 2):
    eng = pf.RsdEngine(meta, cfg.grid, plane_range=(0, 256 // n))
    vol = torch.zeros((1, eng.n_voxels), dtype=torch.complex64, device="cuda")
    eng.run_graphed(coeff, vol); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); eng.run_graphed(coeff, vol); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    res.append(f"N={n}:{best:.2f}")
print(" ".join(res))
PY
)"
done
