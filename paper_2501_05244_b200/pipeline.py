"""End-to-end public API: host transients in, host volume out.

``TransientReconstructor`` is what a user of the reference calls as
``to_frequency`` + ``reconstruct`` (reference phasor.py:107-127,
reconstruct.py:776-809) when the capture sits in host memory: it streams the
float32 histograms to the GPU in chunks on a copy stream, overlapping each
chunk's host->device transfer with the temporal transform (K1) of the previous
chunk, runs the propagation on the device and returns the volume to (pinned)
host memory.  The device-resident sub-steps are exposed for benchmarking.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _device as dev
from .core import SPEED_OF_LIGHT, ReconstructionVolume
from .phasor import TemporalPlan
from .reconstruct import RsdEngine


class _Meta:
    """Slices geometry without coefficients (what the engines need to plan)."""

    def __init__(self, kernel, relay, illuminations):
        self.frequencies = np.asarray(kernel.frequencies)
        self.relay = relay
        self.illuminations = illuminations
        self.n_freq = int(self.frequencies.size)

    @property
    def shortest_wavelength(self) -> float:
        return 2.0 * np.pi * SPEED_OF_LIGHT / float(self.frequencies.max())


def make_engine(algorithm, meta, grid, device, plane_range=None, times=None,
                include_illumination=True, padding="exact", eps=1e-6, lattice=None):
    """Device engine (``run(coeff, vol, stream)``) for a cuboid/frustum algorithm, or the
    non-planar relay -> explicit voxels composition ("nursd3d-explicit", needs the stage-1
    ``lattice``; one GPU, no plane sharding)."""
    name = algorithm.replace("_", "-").lower()
    if name == "nursd3d-explicit":
        from .algorithms import Nursd3dExplicitEngine
        n_pl = len(grid.planes) if grid.kind == "explicit" else 1
        if plane_range is not None and tuple(plane_range) != (0, n_pl):
            raise ValueError("nursd3d-explicit does not shard depth planes")
        return Nursd3dExplicitEngine(meta, grid, lattice, eps, None, times,
                                     include_illumination, device=device)
    if name == "rsd":
        return RsdEngine(meta, grid, padding, include_illumination, times, device=device,
                         plane_range=plane_range)
    from .algorithms import Nursd1Engine, SrsdEngine
    if name == "srsd":
        return SrsdEngine(meta, grid, include_illumination, times, device=device,
                          plane_range=plane_range)
    if name == "nursd1":
        return Nursd1Engine(meta, grid, eps, include_illumination, times, device=device,
                            plane_range=plane_range)
    raise ValueError(f"no streaming engine for {algorithm!r}")


class TransientReconstructor:
    """rsd / srsd / nursd1 from host histograms [I, D, T] (float32) to a host volume.

    ``plane_range`` restricts the planes (multi-GPU sharding); ``trace_range``
    restricts the detectors this instance transforms (K1 sharding).
    """

    def __init__(self, kernel, relay, illuminations, grid, t0: float = 0.0, padding="exact",
                 include_illumination=True, times=None, plane_range=None, chunks: int = 8,
                 device=None, trace_range=None, slice_gather=None, volume_gather=None,
                 algorithm="rsd", eps=1e-6, lattice=None):
        self.device = device or dev.require_cuda()
        self.kernel = kernel
        self.grid = grid
        self.meta = _Meta(kernel, relay, illuminations)
        self.engine = make_engine(algorithm, self.meta, grid, self.device, plane_range, times,
                                  include_illumination, padding, eps, lattice)
        self.temporal = TemporalPlan(kernel, t0, self.device)
        self.n_illum = illuminations.count
        self.n_det = relay.count
        lo, hi = trace_range or (0, self.n_det)
        self.n_det_local = hi - lo
        self.slice_gather, self.volume_gather = slice_gather, volume_gather
        self.coeff = torch.empty((kernel.n_freq, self.n_illum, self.n_det_local),
                                 dtype=torch.complex64, device=self.device)
        self.vol = torch.zeros((self.engine.n_frames, self.engine.n_voxels), dtype=torch.complex64,
                               device=self.device)
        self.chunks = max(1, int(chunks))
        self.use_graphs = True
        # multi-GPU: planes in chunks, each gathered while the next computes
        nloc = getattr(self.engine, "n_planes_local", 0)
        want = int(os.environ.get("PF_GATHER_CHUNKS", "4"))
        self.gather_chunks, self.chunk_unit = 1, 1
        if volume_gather is not None and hasattr(self.engine, "run_chunk") and want > 1:
            from .distributed import max_chunks
            self.chunk_unit = self.engine.chunk_unit
            self.gather_chunks = min(max_chunks(hi - lo, want, self.chunk_unit)
                                     for lo, hi in volume_gather.ranges)
        self.gather_stream = torch.cuda.Stream(device=self.device)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self._hist_dev = None
        self._vol_host = None

    # -- device-resident pieces -------------------------------------------------
    def transform(self, hist_dev: torch.Tensor, stream=None) -> torch.Tensor:
        """K1 over device histograms [I, D, T] -> self.coeff [F, I, D]."""
        i_n, d_n, t_n = hist_dev.shape
        self.temporal.run(hist_dev.view(i_n * d_n, t_n), self.coeff.view(self.kernel.n_freq, -1),
                          stream)
        return self.coeff

    def propagate(self, coeff: torch.Tensor, stream=None) -> torch.Tensor:
        if self.use_graphs:
            return self.engine.run_graphed(coeff, self.vol, stream)
        return self.engine.run(coeff, self.vol, stream)

    def propagate_and_gather(self, coeff: torch.Tensor, vol: torch.Tensor, stream=None,
                             after=None):
        """Chunked propagation; chunk j's planes are gathered to rank 0 on the gather
        stream while chunk j+1 computes.  ``after``: event the first gather must wait
        for (the previous capture's read of the gathered volume).  Returns the
        gathered volume on rank 0 (None elsewhere); ``stream`` waits for the gathers."""
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        gs = self.gather_stream
        if after is not None:
            gs.wait_event(after)
        res = None
        for j in range(self.gather_chunks):
            self.engine.run_graphed_chunk(coeff, vol, j, self.gather_chunks, main)
            done = torch.cuda.Event()
            done.record(main)
            gs.wait_event(done)
            with torch.cuda.stream(gs):
                res = self.volume_gather.gather_part(vol, j, self.gather_chunks,
                                                     self.chunk_unit)
        main.wait_stream(gs)
        return res

    # -- host in, host out ------------------------------------------------------
    def __call__(self, hist_host: torch.Tensor) -> torch.Tensor:
        """hist_host: pinned float32 [I, D, T]; returns pinned host complex64 [frames, V]."""
        i_n, d_n, t_n = hist_host.shape
        n_tr = i_n * d_n
        if self._hist_dev is None or self._hist_dev.shape != hist_host.shape:
            self._hist_dev = torch.empty_like(hist_host, device=self.device)
        if self._vol_host is None:
            shape = self.vol.shape
            if self.volume_gather is not None:
                shape = (self.vol.shape[0], self.grid.count)
            self._vol_host = torch.empty(shape, dtype=self.vol.dtype, pin_memory=True)
        src = hist_host.view(n_tr, t_n)
        dst = self._hist_dev.view(n_tr, t_n)
        out = self.coeff.view(self.kernel.n_freq, n_tr)
        main = torch.cuda.current_stream(self.device)
        step = (n_tr + self.chunks - 1) // self.chunks
        with dev.nvtx("pf: h2d + K1"):
            for c0 in range(0, n_tr, step):
                c1 = min(n_tr, c0 + step)
                with torch.cuda.stream(self.copy_stream):
                    dst[c0:c1].copy_(src[c0:c1], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(self.copy_stream)
                main.wait_event(ev)
                self.temporal.run(dst[c0:c1], out[:, c0:c1], main)
        with dev.nvtx("pf: slice gather"):
            coeff = self.slice_gather(self.coeff) if self.slice_gather is not None else self.coeff
        vol = self.vol
        with dev.nvtx("pf: propagation + volume gather"):
            if self.gather_chunks > 1:
                vol = self.propagate_and_gather(coeff, self.vol, main)
            else:
                self.propagate(coeff, main)
                if self.volume_gather is not None:
                    vol = self.volume_gather(self.vol)   # full volume on rank 0, None elsewhere
        if self.volume_gather is not None and vol is None:
            main.synchronize()
            return None
        with dev.nvtx("pf: d2h"):
            self._vol_host.copy_(vol, non_blocking=True)
            main.synchronize()
        return self._vol_host

    # -- pipelined streaming of successive captures -----------------------------------
    def submit(self, hist_host: torch.Tensor):
        """Enqueue one capture; returns a handle for :meth:`result`.

        Two captures are in flight: the host->device copy of capture i+1 (copy
        stream) overlaps the propagation of capture i (compute stream) and the
        device->host read of volume i-1 (d2h stream).  Each capture still pays its
        own H2D and D2H; only their overlap with compute changes.
        """
        if not hasattr(self, "_slots"):
            self._init_slots(hist_host)
        k = self._next
        self._next ^= 1
        sl = self._slots[k]
        i_n, d_n, t_n = hist_host.shape
        n_tr = i_n * d_n
        main = torch.cuda.current_stream(self.device)
        src = hist_host.view(n_tr, t_n)
        dst = sl["hist"].view(n_tr, t_n)
        out = sl["coeff"].view(self.kernel.n_freq, n_tr)
        step = (n_tr + self.chunks - 1) // self.chunks
        self.copy_stream.wait_event(sl["hist_free"])
        for c0 in range(0, n_tr, step):
            c1 = min(n_tr, c0 + step)
            with torch.cuda.stream(self.copy_stream):
                dst[c0:c1].copy_(src[c0:c1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
            main.wait_event(ev)
            self.temporal.run(dst[c0:c1], out[:, c0:c1], main)
        sl["hist_free"].record(main)
        coeff = self.slice_gather(sl["coeff"]) if self.slice_gather is not None else sl["coeff"]
        main.wait_event(sl["vol_free"])
        vol = sl["vol"]
        if self.gather_chunks > 1:
            # the gathered volume lives in one buffer (rank 0): the previous capture's
            # device->host read of it must finish before this capture's gathers write it
            vol = self.propagate_and_gather(coeff, sl["vol"], main, after=self._last_d2h)
        else:
            if self.use_graphs:
                self.engine.run_graphed(coeff, sl["vol"], main)
            else:
                self.engine.run(coeff, sl["vol"], main)
            if self.volume_gather is not None:
                if self._last_d2h is not None:
                    main.wait_event(self._last_d2h)
                vol = self.volume_gather(sl["vol"])
        done = torch.cuda.Event()
        if vol is not None:
            sl["vol_ready"].record(main)
            self.d2h_stream.wait_event(sl["vol_ready"])
            with torch.cuda.stream(self.d2h_stream):
                sl["host"].copy_(vol, non_blocking=True)
                sl["vol_free"].record(self.d2h_stream)
                done.record(self.d2h_stream)
            self._last_d2h = done
        else:
            sl["vol_free"].record(main)
            done.record(main)
        return (k, done)

    def result(self, handle):
        k, done = handle
        done.synchronize()
        return self._slots[k]["host"] if self.volume_gather is None or \
            self.volume_gather.rank == 0 else None

    def _init_slots(self, hist_host):
        self.d2h_stream = torch.cuda.Stream(device=self.device)
        self._last_d2h = None
        self._next = 0
        self._slots = []
        vshape = self.vol.shape
        if self.volume_gather is not None:
            vshape = (self.vol.shape[0], self.grid.count)
        for _ in range(2):
            sl = {"hist": torch.empty_like(hist_host, device=self.device),
                  "coeff": torch.empty_like(self.coeff),
                  "vol": torch.zeros_like(self.vol),
                  "host": torch.empty(vshape, dtype=self.vol.dtype, pin_memory=True),
                  "hist_free": torch.cuda.Event(), "vol_free": torch.cuda.Event(),
                  "vol_ready": torch.cuda.Event()}
            sl["hist_free"].record()
            sl["vol_free"].record()
            self._slots.append(sl)

    def volume(self, host_vol: torch.Tensor) -> ReconstructionVolume:
        field = host_vol.numpy().astype(np.complex128)
        times = self.engine.times
        return ReconstructionVolume(self.grid, field[0] if times is None else field, times)
