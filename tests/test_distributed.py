"""Multi-rank host logic on CPU (gloo, world_size 2): sharding, slice all-gather, volume gather.

Each rank transforms its detector shard and propagates its depth-plane shard with the CPU
oracle standing in for the kernels; rank 0 must reassemble exactly the single-process result.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_05244_b200.distributed import SliceGather, VolumeGather, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    import paper_2501_05244_b200 as pf
    rng = np.random.default_rng(11)
    n, T, dt = 12, 256, 16e-12
    p = 0.03
    g = pf.UniformGrid2D(n, n, p, p, -(n - 1) * p / 2, -(n - 1) * p / 2, 0.0)
    hist = rng.poisson(2.0, size=(1, n * n, T)).astype(np.float64)
    k = pf.build_kernel(0.08, T, dt)
    grid = pf.CuboidGrid(pf.UniformGrid3D(n, n, 5, p, p, 0.07, g.x0, g.y0, 0.4))
    return pf, g, hist, k, grid


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pf_oracle as O
    pf, g, hist, k, grid = _scene()
    D = g.count
    d_lo, d_hi = shard_range(D, world, rank)
    loc = O.to_frequency(hist[:, d_lo:d_hi], k.bin_indices, k.frequencies, k.weights, 0.0)
    local = torch.from_numpy(np.ascontiguousarray(loc.transpose(2, 0, 1)).astype(np.complex64))
    sg = SliceGather(k.n_freq, 1, D, world, torch.device("cpu"))
    full = sg(local)
    coeff = full.numpy().transpose(1, 2, 0).astype(np.complex128)
    sl = pf.FrequencySlices(k.frequencies, coeff, pf.UniformRelay(g), pf.PointList(np.zeros((1, 2))))
    nz = grid.grid.nz
    k_lo, k_hi = shard_range(nz, world, rank)
    vol_local = O.rsd(sl, grid, plane_range=(k_lo, k_hi)).astype(np.complex64)[None, :]
    vg = VolumeGather(nz, g.nx * g.ny, 1, world, rank, torch.device("cpu"))
    res = vg(torch.from_numpy(vol_local))
    if rank == 0:
        out_q.put((full.numpy(), res.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_cover_in_order():
    for n in (1, 5, 64, 256, 262144):
        for w in (1, 2, 3, 8):
            r = [shard_range(n, w, k) for k in range(w)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert max(h - l for l, h in r) - min(h - l for l, h in r) <= 1


def test_two_rank_gloo_reassembles_single_process_result():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, vol = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from oracle import pf_oracle as O
    pf, g, hist, k, grid = _scene()
    ref_c = O.to_frequency(hist, k.bin_indices, k.frequencies, k.weights, 0.0)
    assert np.array_equal(full, ref_c.transpose(2, 0, 1).astype(np.complex64))
    sl = pf.FrequencySlices(k.frequencies, full.transpose(1, 2, 0).astype(np.complex128),
                            pf.UniformRelay(g), pf.PointList(np.zeros((1, 2))))
    ref_v = O.rsd(sl, grid).astype(np.complex64)
    # per-plane results do not depend on the shard: bit-identical reassembly
    assert np.array_equal(vol[0], ref_v)


def _pipeline_scene(n_caps=3):
    import paper_2501_05244_b200 as pf
    rng = np.random.default_rng(5)
    n, T, dt = 32, 1024, 8e-12
    p = 2.0 / n
    g = pf.UniformGrid2D(n, n, p, p, -1 + p / 2, -1 + p / 2, 0.0)
    caps = [rng.poisson(1.0 + c, size=(1, n * n, T)).astype(np.float32) for c in range(n_caps)]
    k = pf.build_kernel(0.06, T, dt)
    grid = pf.CuboidGrid(pf.UniformGrid3D(n, n, 7, p, p, 0.1, g.x0, g.y0, 0.5))
    return pf, g, caps, k, grid


def _pipeline_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_05244_b200.pipeline import TransientReconstructor
    pf, g, caps, k, grid = _pipeline_scene()
    dev = torch.device("cuda", 0)
    D, nz = g.count, grid.grid.nz
    d_lo, d_hi = shard_range(D, world, rank)
    k_lo, k_hi = shard_range(nz, world, rank)
    rec = TransientReconstructor(k, pf.UniformRelay(g), pf.PointList(np.zeros((1, 2))), grid,
                                 plane_range=(k_lo, k_hi), trace_range=(d_lo, d_hi), device=dev,
                                 slice_gather=SliceGather(k.n_freq, 1, D, world, dev),
                                 volume_gather=VolumeGather(nz, g.count, 1, world, rank, dev))
    hosts = [torch.from_numpy(c[:, d_lo:d_hi].copy()).pin_memory() for c in caps]
    hs = [rec.submit(hosts[0]), rec.submit(hosts[1])]
    outs = [rec.result(hs[0])]
    outs[0] = None if outs[0] is None else outs[0].clone()
    hs.append(rec.submit(hosts[2]))
    for h in hs[1:]:
        r = rec.result(h)
        outs.append(None if r is None else r.clone())
    if rank == 0:
        out_q.put([o.numpy() for o in outs])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_pipelined_captures_match_single_gpu():
    """Detector + plane sharded streaming (submit/result, two captures in flight, gathers
    host-staged over gloo, both ranks on cuda:0): every capture's reassembled volume equals
    the single-process volume bit for bit (no buffer reuse race between captures)."""
    from paper_2501_05244_b200.pipeline import TransientReconstructor
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    pf, g, caps, k, grid = _pipeline_scene()
    rec = TransientReconstructor(k, pf.UniformRelay(g), pf.PointList(np.zeros((1, 2))), grid)
    for c, h in enumerate(caps):
        ref = rec(torch.from_numpy(h).pin_memory()).numpy()
        assert np.array_equal(got[c], ref), c


def _part_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nz, pv, nf = 11, 6, 2
    lo, hi = shard_range(nz, world, rank)
    g = torch.Generator().manual_seed(100 + rank)
    local = torch.randn((nf, (hi - lo) * pv), dtype=torch.complex64, generator=g)
    vg = VolumeGather(nz, pv, nf, world, rank, torch.device("cpu"))
    full_once = vg(local)
    full_once = None if full_once is None else full_once.clone()
    vg2 = VolumeGather(nz, pv, nf, world, rank, torch.device("cpu"))
    for j in range(2):                       # 2 chunks on 2-plane units (uneven shards 4/4/3)
        res = vg2.gather_part(local, j, 2, 2)
    if rank == 0:
        out_q.put((full_once.numpy(), res.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_chunked_volume_gather_equals_single_gather():
    """Overlapped (per-chunk) gathers reassemble exactly the one-shot gather (world 3,
    uneven shards)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_part_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    once, parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(once, parts)


def test_chunk_split_units():
    from paper_2501_05244_b200.distributed import chunk_split, max_chunks
    for n, c, u in [(32, 4, 12), (64, 4, 12), (128, 4, 12), (11, 2, 2), (7, 3, 1), (5, 1, 12)]:
        c = min(c, max_chunks(n, c, u))
        parts = chunk_split(n, c, u)
        assert parts[0][0] == 0 and parts[-1][1] == n and len(parts) == c
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        assert all(b > a for a, b in parts)
        assert all(b % u == 0 for _, b in parts[:-1])
    assert chunk_split(32, 3, 12) == [(0, 12), (12, 24), (24, 32)]


def _peer_worker(rank, world, port, out_q):
    """Two ranks on cuda:0 exchanging CUDA IPC mappings (the mechanism NVLink peers use):
    K1 with the slice all-gather fused into its store, kernel C storing the finished planes
    straight into rank 0's volume."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import importlib
    R = importlib.import_module("paper_2501_05244_b200.reconstruct")
    R._FBATCH_BYTES = 0                      # per-frequency launches (the config-4 sequence)
    from paper_2501_05244_b200.distributed import PeerSlices, PeerVolume
    from paper_2501_05244_b200.phasor import TemporalPlan, temporal_peers
    from paper_2501_05244_b200.pipeline import _Meta
    pf, g, hist, k, grid = _peer_scene()
    dev = torch.device("cuda", 0)
    D, nz, T = g.count, grid.grid.nz, hist.shape[-1]
    d_lo, d_hi = shard_range(D, world, rank)
    k_lo, k_hi = shard_range(nz, world, rank)
    ps = PeerSlices(k.n_freq, 1, D, world, rank, dev)
    pv = PeerVolume(nz, g.count, world, rank, dev)
    h = torch.from_numpy(hist[0, d_lo:d_hi].copy()).to(dev)
    temporal_peers(TemporalPlan(k, 1e-10, dev), h, ps)
    full = ps.sync()
    ill = pf.PointList(np.zeros((1, 2)))
    eng = R.RsdEngine(_Meta(k, pf.UniformRelay(g), ill), grid, plane_range=(k_lo, k_hi),
                      device=dev)
    assert eng.fused_gather_ok()
    vol = torch.zeros((1, eng.n_voxels), dtype=torch.complex64, device=dev)
    eng.run_graphed(full, vol, vol_out=pv.out_ptr)
    out = pv.sync()
    if rank == 0:
        out_q.put((full.cpu().numpy(), out.cpu().numpy()))
    dist.barrier()
    ps.close()
    pv.close()
    dist.destroy_process_group()


def _peer_scene():
    import paper_2501_05244_b200 as pf
    rng = np.random.default_rng(9)
    n, T, dt = 64, 2048, 8e-12
    p = 2.0 / n
    g = pf.UniformGrid2D(n, n, p, p, -1 + p / 2, -1 + p / 2, 0.0)
    hist = rng.poisson(2.0, size=(1, n * n, T)).astype(np.float32)
    k = pf.build_kernel(0.06, T, dt)
    grid = pf.CuboidGrid(pf.UniformGrid3D(n, n, 6, p, p, 0.2, g.x0, g.y0, 0.5))
    return pf, g, hist, k, grid


@pytest.mark.gpu
def test_two_rank_peer_memory_collectives_match_single_gpu():
    """The fused collectives (K1 writing every rank's slice buffer, kernel C writing rank 0's
    volume, CUDA IPC mappings; two gloo ranks on cuda:0 only for the host handshake and the
    barriers) give the single-process slices and volume bit for bit."""
    import importlib
    R = importlib.import_module("paper_2501_05244_b200.reconstruct")
    from paper_2501_05244_b200.phasor import to_frequency_device
    from paper_2501_05244_b200.pipeline import _Meta
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, vol = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    pf, g, hist, k, grid = _peer_scene()
    dev = torch.device("cuda", 0)
    coeff = to_frequency_device(torch.from_numpy(hist).to(dev), k, 1e-10)
    ref_c = coeff.cpu().numpy()
    bad = np.argwhere(full != ref_c)
    assert bad.size == 0, (bad[:5].tolist(), len(bad), np.abs(full - ref_c).max())
    keep = R._FBATCH_BYTES
    R._FBATCH_BYTES = 0
    try:
        eng = R.RsdEngine(_Meta(k, pf.UniformRelay(g), pf.PointList(np.zeros((1, 2)))), grid,
                          device=dev)
        ref = eng.run(coeff).cpu().numpy()
    finally:
        R._FBATCH_BYTES = keep
    assert np.array_equal(vol, ref)
