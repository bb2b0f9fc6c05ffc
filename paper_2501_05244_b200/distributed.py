"""Multi-GPU plumbing: depth-plane sharding, slice all-gather, volume gather.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch on the box,
gloo in the CPU tests).  The work partitions without a data-path exchange
inside the propagation: every voxel's frequency sum (in the fixed order the
whole-grid geometry selects) lives on the rank that owns its depth plane, so
results are bitwise independent of the number of GPUs.  The two exchanges are at the edges of the path:

* K1 shards the detectors; the frequency slices (64 MiB at config 4) are
  all-gathered so every rank holds ``[F, I, D]`` (the north star's "frequency
  slices broadcast over NVLink");
* the finished plane blocks are gathered to rank 0.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items owned by ``rank`` (balanced, in order)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def chunk_split(n: int, n_chunks: int, unit: int = 1) -> list[tuple[int, int]]:
    """Cut [0, n) into n_chunks contiguous pieces whose boundaries fall on multiples of
    ``unit`` (the propagation's lanes x planes-per-batch, so a chunk keeps every stream
    lane busy); n_chunks must not exceed ceil(n / unit)."""
    units = -(-n // unit)
    base, extra = divmod(units, n_chunks)
    out, u = [], 0
    for j in range(n_chunks):
        nu = base + (1 if j < extra else 0)
        out.append((min(n, u * unit), min(n, (u + nu) * unit)))
        u += nu
    return out


def max_chunks(n: int, want: int, unit: int = 1) -> int:
    return max(1, min(int(want), -(-n // unit))) if n else 1


def _real(t: torch.Tensor) -> torch.Tensor:
    return torch.view_as_real(t) if t.is_complex() else t


def _host_staged(group) -> bool:
    """gloo cannot reduce/gather device tensors: stage those collectives through the host."""
    return dist.get_backend(group) == "gloo"


class SliceGather:
    """All-gather detector-sharded slices [F, I, D_r] into [F, I, D] on every rank."""

    def __init__(self, n_freq: int, n_illum: int, n_det: int, world: int, device, group=None):
        self.world, self.group = world, group
        self.F, self.I, self.D = n_freq, n_illum, n_det
        self.ranges = [shard_range(n_det, world, r) for r in range(world)]
        self.maxd = max(h - l for l, h in self.ranges)
        self.send = torch.zeros((n_freq * n_illum * self.maxd,), dtype=torch.complex64, device=device)
        self.recv = [torch.empty_like(self.send) for _ in range(world)]
        self.full = torch.empty((n_freq, n_illum, n_det), dtype=torch.complex64, device=device)

    def __call__(self, local: torch.Tensor) -> torch.Tensor:
        n = local.numel()
        self.send[:n].copy_(local.reshape(-1))
        if self.send.is_cuda and _host_staged(self.group):
            send = self.send.cpu()
            recv = [torch.empty_like(send) for _ in self.recv]
            dist.all_gather([_real(r) for r in recv], _real(send), group=self.group)
            for d, h in zip(self.recv, recv):
                d.copy_(h)
        else:
            dist.all_gather([_real(r) for r in self.recv], _real(self.send), group=self.group)
        for r, (lo, hi) in enumerate(self.ranges):
            cnt = self.F * self.I * (hi - lo)
            self.full[:, :, lo:hi].copy_(self.recv[r][:cnt].view(self.F, self.I, hi - lo))
        return self.full


class VolumeGather:
    """Gather plane-sharded volumes [frames, V_r] into [frames, V] on rank 0."""

    def __init__(self, n_planes: int, plane_voxels: int, n_frames: int, world: int, rank: int,
                 device, group=None):
        self.world, self.rank, self.group = world, rank, group
        self.ranges = [shard_range(n_planes, world, r) for r in range(world)]
        self.pv, self.nf = plane_voxels, n_frames
        self.maxv = max(h - l for l, h in self.ranges) * plane_voxels
        self.send = torch.zeros((n_frames, self.maxv), dtype=torch.complex64, device=device)
        self.recv = ([torch.empty_like(self.send) for _ in range(world)] if rank == 0 else None)
        self.full = (torch.empty((n_frames, n_planes * plane_voxels), dtype=torch.complex64,
                                 device=device) if rank == 0 else None)

    def __call__(self, local: torch.Tensor):
        self.send[:, :local.shape[1]].copy_(local)
        if self.send.is_cuda and _host_staged(self.group):
            send = self.send.cpu()
            recv = [torch.empty_like(send) for _ in range(self.world)] if self.rank == 0 else None
            dist.gather(_real(send), [_real(r) for r in recv] if recv else None, dst=0,
                        group=self.group)
            if self.rank == 0:
                for d, h in zip(self.recv, recv):
                    d.copy_(h)
        else:
            dist.gather(_real(self.send), [_real(r) for r in self.recv] if self.rank == 0 else None,
                        dst=0, group=self.group)
        if self.rank != 0:
            return None
        for r, (lo, hi) in enumerate(self.ranges):
            n = (hi - lo) * self.pv
            self.full[:, lo * self.pv:hi * self.pv].copy_(self.recv[r][:, :n])
        return self.full

    def part_ranges(self, j: int, n_chunks: int, unit: int = 1):
        """Per rank: local plane range of chunk j when each shard is cut by
        ``chunk_split(shard, n_chunks, unit)`` (the split ``GraphedRun.chunk_bounds`` uses)."""
        return [chunk_split(hi - lo, n_chunks, unit)[j] for lo, hi in self.ranges]

    def gather_part(self, local: torch.Tensor, j: int, n_chunks: int, unit: int = 1):
        """Gather chunk j of every rank's shard into ``full`` on rank 0 (call on the stream
        that must order it: after chunk j's planes are final on this rank)."""
        parts = self.part_ranges(j, n_chunks, unit)
        maxp = max(1, max(b - a for a, b in parts)) * self.pv
        a, b = parts[self.rank]
        send = self.send[:, :maxp]
        send[:, :(b - a) * self.pv].copy_(local.view(self.nf, -1)[:, a * self.pv:b * self.pv])
        send = send.contiguous()
        recv = [r[:, :maxp].contiguous() for r in self.recv] if self.rank == 0 else None
        if send.is_cuda and _host_staged(self.group):
            hs = send.cpu()
            hr = [torch.empty_like(hs) for _ in range(self.world)] if self.rank == 0 else None
            dist.gather(_real(hs), [_real(x) for x in hr] if hr else None, dst=0, group=self.group)
            if self.rank == 0:
                for d, h in zip(recv, hr):
                    d.copy_(h)
        else:
            dist.gather(_real(send), [_real(x) for x in recv] if recv else None, dst=0,
                        group=self.group)
        if self.rank != 0:
            return None
        for r, ((lo, _), (pa, pb)) in enumerate(zip(self.ranges, parts)):
            n = (pb - pa) * self.pv
            self.full[:, (lo + pa) * self.pv:(lo + pb) * self.pv].copy_(recv[r][:, :n])
        return self.full


# ---------------------------------------------------------------------------
# peer-memory collectives: the exchange is fused into the producing kernel
# ---------------------------------------------------------------------------


def _ipc_handle(t: torch.Tensor) -> tuple:
    """(64-byte handle of the allocation holding t, t's offset in it)."""
    import ctypes

    from . import _lib
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    _lib.call("pf_ipc_handle", t.data_ptr(), buf, ctypes.byref(off))
    return buf.raw, int(off.value)


def _ipc_open(h: tuple) -> tuple:
    """Map a peer's allocation: (pointer to the peer tensor, mapping base to close)."""
    import ctypes

    from . import _lib
    p = ctypes.c_void_p()
    _lib.call("pf_ipc_open", ctypes.create_string_buffer(h[0], 64), h[1], ctypes.byref(p))
    return int(p.value), int(p.value) - h[1]


def stream_barrier(group=None, device=None, stream=None) -> None:
    """Order every rank's later device work after every rank's earlier device work without
    a host round trip: a one-element all-reduce enqueued on the stream (NCCL).  gloo (CPU
    tests, one GPU shared by the ranks): drain the device, then a host barrier."""
    if dist.get_backend(group) == "gloo":
        torch.cuda.synchronize(device)
        dist.barrier(group=group)
        return
    flag = torch.ones(1, dtype=torch.float32, device=device)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    with torch.cuda.stream(s):
        dist.all_reduce(flag, group=group)


class PeerSlices:
    """The slice all-gather fused into K1: every rank owns a full
    ``[F, I, D]`` slice buffer; the ranks exchange CUDA IPC handles of those buffers once,
    and each rank's K1 (``pf_temporal_dft_peers``) writes its detector shard's bins
    straight into all of them over NVLink / NVSwitch (peer stores tile by tile, no NCCL
    transfer); ``sync`` orders the reads after every rank's K1."""

    def __init__(self, n_freq: int, n_illum: int, n_det: int, world: int, rank: int, device,
                 group=None):
        if n_illum != 1:   # a rank's traces are contiguous columns only for one illumination
            raise ValueError("the fused slice all-gather takes one illumination")
        self.F, self.I, self.D = n_freq, n_illum, n_det
        self.world, self.rank, self.group, self.device = world, rank, group, device
        self.ranges = [shard_range(n_det, world, r) for r in range(world)]
        self.full = torch.zeros((n_freq, n_illum, n_det), dtype=torch.complex64, device=device)
        torch.cuda.synchronize(device)   # zeroed before any peer can write into it
        # every rank reaches every collective of the handshake; failures only clear self.ok
        # (open_peer_collectives agrees on the outcome across ranks)
        self.ok, self.error = True, None
        try:
            mine = _ipc_handle(self.full)
        except Exception as e:
            mine, self.ok, self.error = None, False, e
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        self._opened = []
        ptrs = []
        for r, h in enumerate(handles):
            if r == rank:
                ptrs.append(self.full.data_ptr())
                continue
            if h is None or not self.ok:
                self.ok = False
                ptrs.append(0)
                continue
            try:
                p, base = _ipc_open(h)
                self._opened.append(base)
                ptrs.append(p)
            except Exception as e:
                self.ok, self.error = False, e
                ptrs.append(0)
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=device)
        lo, _ = self.ranges[rank]
        # column of this rank's first trace in the [F][I*D] view (illumination-major rows)
        self.peer_stride = n_illum * n_det
        self.col = lo

    def sync(self, stream=None):
        stream_barrier(self.group, self.device, stream)
        return self.full

    def close(self):
        from . import _lib
        for p in self._opened:
            _lib.call("pf_ipc_close", p)
        self._opened = []


class PeerVolume:
    """The volume gather fused into kernel C: rank 0 owns the full
    volume; the other ranks map it once (CUDA IPC) and their final Horner step of every
    plane batch stores the finished planes straight into it (``vol_out`` of
    ``pf_prop_rows_out_horner``), so each plane batch's transfer overlaps the rest of the
    propagation with no separate gather; ``sync`` orders rank 0's reads after every
    rank's last store."""

    def __init__(self, n_planes: int, plane_voxels: int, world: int, rank: int, device,
                 group=None):
        self.world, self.rank, self.group, self.device = world, rank, group, device
        self.ranges = [shard_range(n_planes, world, r) for r in range(world)]
        self.pv = plane_voxels
        full = torch.zeros((1, n_planes * plane_voxels), dtype=torch.complex64, device=device) \
            if rank == 0 else torch.zeros(1, dtype=torch.complex64, device=device)
        self.full = full if rank == 0 else None
        torch.cuda.synchronize(device)   # zeroed before any peer can write into it
        self.ok, self.error = True, None
        handles = [None]
        if rank == 0:
            try:
                handles = [_ipc_handle(full)]
            except Exception as e:
                self.ok, self.error = False, e
        dist.broadcast_object_list(handles, src=0, group=group)
        self._opened = None
        base = 0
        if rank == 0:
            base = full.data_ptr()
        elif handles[0] is None:
            self.ok = False
        else:
            try:
                base, self._opened = _ipc_open(handles[0])
            except Exception as e:
                self.ok, self.error = False, e
        lo, _ = self.ranges[rank]
        self.out_ptr = base + 8 * lo * plane_voxels     # this shard's first plane in rank 0

    def sync(self, stream=None):
        stream_barrier(self.group, self.device, stream)
        return self.full

    def close(self):
        from . import _lib
        if self._opened:
            _lib.call("pf_ipc_close", self._opened)
            self._opened = None


def open_peer_collectives(n_freq, n_illum, n_det, n_planes, plane_voxels, world, rank, device,
                          group=None):
    """(PeerSlices, PeerVolume) when every rank can map the others' buffers, else None on
    every rank (the decision is all-reduced so no rank is left waiting in a collective the
    others skipped).  The reason a rank failed is printed once."""
    made = (PeerSlices(n_freq, n_illum, n_det, world, rank, device, group),
            PeerVolume(n_planes, plane_voxels, world, rank, device, group))
    good = all(m.ok for m in made)
    err = next((m.error for m in made if m.error is not None), None)
    ok = torch.tensor([1 if good else 0], dtype=torch.int32)
    if dist.get_backend(group) != "gloo":
        ok = ok.to(device)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
    if int(ok.item()) == 1:
        return made
    for m in made:
        m.close()
    if err is not None:
        print(f"peer-memory collectives unavailable on rank {rank}: {err}; using NCCL",
              flush=True)
    return None
