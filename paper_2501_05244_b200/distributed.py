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
