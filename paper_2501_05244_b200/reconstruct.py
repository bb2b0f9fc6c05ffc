"""GPU drop-ins for the reference reconstruction entry points (reference ``reconstruct.py``).

Every public function keeps the reference signature, argument meaning and
``ValidationError`` messages; the arithmetic runs in ``libpfgpu.so``:

==============  =========================================  ==========================
reference       device pipeline                            reference lines
==============  =========================================  ==========================
rsd             embed -> 2D FFT -> propagate (A,B,C)        reconstruct.py:208-268
srsd            embed -> Bluestein x/y -> propagate         reconstruct.py:276-327
nursd1          type-1 NUFFT -> propagate                   reconstruct.py:335-385
nursd2/3, hyb.  ... -> product -> type-2 NUFFT readout      reconstruct.py:413-586
nursd3d         3D type-1 -> 3D conv -> slab -> propagate   reconstruct.py:722-765
==============  =========================================  ==========================

Accumulation order per voxel is fixed by the geometry: ascending frequency then
illumination (reference order), or descending frequency when kernel C applies the
illumination phase by Horner's rule (one illumination, uniform bins, register pads).
Every path choice is made from the whole grid, never from a shard, so results are
bit-reproducible run to run and independent of how depth planes are batched or
sharded across GPUs; different paths (e.g. frequency-batched vs per-frequency
launches) round differently in fp32.  ``threads`` is accepted and ignored (the
reference uses it only to parallelise the per-frequency terms).
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

from . import _device as dev
from . import _lib
from ._fastlen import next_fast_len
from .core import (SPEED_OF_LIGHT, ReconstructionVolume, ValidationError, _require,
                   illumination_coordinates)
from .phasor import device_coefficients

ALGORITHM_NAMES = ("rsd", "srsd", "nursd1", "nursd2", "nursd3", "rsd3d", "nursd3d",
                   "srsd-nursd2")

# workspace budget per propagation batch: keep ws_a + ws_b L2-resident (126 MB L2)
_BATCH_BYTES = 64 << 20
_LANES = int(os.environ.get("PF_LANES", "3"))
_FAST_BATCH_CAP = int(os.environ.get("PF_BATCH_CAP", "4"))
_FBATCH_BYTES = int(os.environ.get("PF_FBATCH_MB", "256")) << 20
_FBATCH_GENERIC = os.environ.get("PF_FBATCH_GENERIC", "1") != "0"
_ONCHIP = os.environ.get("PF_ONCHIP", "1") != "0"   # P = 140: whole units in shared memory
_ONCHIP_GROUPS = int(os.environ.get("PF_ONCHIP_GROUPS", "0"))   # 0: from the geometry
_ONCHIP_WARPS = int(os.environ.get("PF_ONCHIP_WARPS", "0"))     # 0: the library default
_HORNER = os.environ.get("PF_HORNER", "1") != "0"   # kernel C phases by Horner's rule
_HORNER_BLOCK = int(os.environ.get("PF_HORNER_BLOCK", "32"))   # frequencies per nested block


# ---------------------------------------------------------------------------
# validation helpers (reference reconstruct.py:90-200)
# ---------------------------------------------------------------------------


def _close(a: float, b: float) -> bool:
    return math.isclose(a, b, rel_tol=1e-9, abs_tol=1e-12)


def _integer_offset(value: float, pitch: float, what: str) -> int:
    q = value / pitch
    qi = round(q)
    _require(abs(q - qi) <= 1e-9 * max(1.0, abs(q)),
             f"{what} must be an integer multiple of the lattice pitch")
    return int(qi)


def _pad_size(lag_max: float, nu_max: float, n_min: int) -> int:
    """Reference pad rule (reconstruct.py:102-110), needed where results depend on it."""
    need = 2 * math.ceil(max(lag_max, nu_max)) + 2
    return next_fast_len(max(n_min, need + 8))


def _exact_pad(lag_max: float, nu_max: float, n_min: int) -> int:
    """Smallest 11-smooth length whose centred index set holds every lag.

    rsd is pad-size independent once no lag wraps (forcing other pads
    changes the volume by <= 6e-16), so the GPU drops the reference's +8 margin
    (140 -> 128 at config 0, 1050 -> 1024 at config 4).
    """
    need = max(n_min, 2 * math.ceil(max(lag_max, nu_max)) + 2)
    p2 = dev.pow2_ceil(need)
    if 64 < need and p2 <= 1024 and p2 * 5 <= need * 8:
        return p2   # square power-of-two pads take the register-FFT path
    return next_fast_len(need)


def _uniform_relay(slices):
    _require(getattr(slices.relay, "kind", None) == "uniform",
             "this algorithm needs detections on a uniform relay grid")
    return slices.relay


def _planar_relay(slices):
    _require(getattr(slices.relay, "kind", None) == "nonuniform_planar",
             "this algorithm needs scattered detections on a single plane")
    return slices.relay


def _nonplanar_relay(slices):
    _require(getattr(slices.relay, "kind", None) == "nonplanar",
             "this algorithm needs detections scattered in 3D")
    return slices.relay


def _check_depths(zs, z_relay: float) -> None:
    _require(bool((np.asarray(zs) > z_relay).all()),
             "every voxel plane must lie strictly beyond the relay plane")


def _check_times(times):
    if times is None:
        return None
    t = np.asarray(times, dtype=np.float64)
    _require(t.ndim == 1 and t.size >= 1, "frame times must be a nonempty vector")
    return t


def _kind(grid) -> str:
    return getattr(grid, "kind", "")


# ---------------------------------------------------------------------------
# device propagation engine (kernels A, B, C of propagate.cu)
# ---------------------------------------------------------------------------


class PlaneSpec:
    """One output plane: kernel depth/pitch, output sampling, spectrum offset."""

    __slots__ = ("dz", "lag_dx", "lag_dy", "x0", "dx", "y0", "dy", "z", "uhat_off", "vol_plane")

    def __init__(self, dz, lag_dx, lag_dy, x0, dx, y0, dy, z, uhat_off=0, vol_plane=0):
        self.dz, self.lag_dx, self.lag_dy = float(dz), float(lag_dx), float(lag_dy)
        self.x0, self.dx, self.y0, self.dy, self.z = (float(x0), float(dx), float(y0), float(dy),
                                                     float(z))
        self.uhat_off, self.vol_plane = int(uhat_off), int(vol_plane)


class Propagator:
    """Buffers and per-plane geometry for cifft2(Uhat * cfft2(G_k))[crop] * mask_k.

    Built once per (relay, grid) geometry and reused across frequencies and
    calls; ``run_frequency`` enqueues kernels A/B/C for every plane batch.
    """

    def __init__(self, device, px, py, nx, ny, nu0x, nu0y, n_illum, include_illum,
                 planes: list, uhat_illum_stride: int, batch: int | None = None,
                 n_planes_total: int | None = None):
        self.device = device
        # path choices (frequency batching) follow the whole grid, not this shard, so a
        # plane-sharded engine runs the same arithmetic as the single-GPU one
        self.n_planes_total = int(n_planes_total or len(planes))
        g = _lib.PfPropGeom()
        g.px, g.py, g.nx, g.ny = int(px), int(py), int(nx), int(ny)
        g.nu0x, g.nu0y = int(nu0x), int(nu0y)
        g.n_illum, g.include_illum = int(n_illum), int(bool(include_illum))
        g.uhat_illum_stride = int(uhat_illum_stride)
        self.geom = g
        self.nplanes = len(planes)
        per_plane = 8 * ((py // 2 + 1) * (px // 2 + 1) + n_illum * ny * px)
        fast_l = px // 32 if (px == py and px in (128, 256, 512, 1024)) else 0
        if batch is None:
            batch = max(1, min(self.nplanes, _BATCH_BYTES // per_plane))
            if fast_l:   # kernel B packs 8 warps x (32/L) lines of planes per CTA
                q = 4 * (32 // fast_l)
                batch = min(self.nplanes, max(q, (batch // q) * q), _FAST_BATCH_CAP * (32 // fast_l))
        self.batch = int(batch)
        arr = (_lib.PfPlane * self.nplanes)()
        for i, p in enumerate(planes):
            for name in PlaneSpec.__slots__:
                setattr(arr[i], name, getattr(p, name))
        raw = np.frombuffer(bytes(arr), dtype=np.uint8).copy()
        self.planes_dev = torch.from_numpy(raw).to(device)
        self.plane_size = ctypes.sizeof(_lib.PfPlane)
        # two independent lanes (workspace + stream): consecutive plane batches run
        # concurrently so the synthesis-bound kernel A of one batch overlaps the
        # load-bound kernels B/C of the other on the same SMs
        nlanes = min(_LANES, -(-self.nplanes // self.batch))
        self.ws_a_l = [torch.empty(_lib.call("pf_prop_ws_a", ctypes.byref(g), self.batch),
                                   dtype=torch.complex64, device=device) for _ in range(nlanes)]
        self.ws_b_l = [torch.empty(_lib.call("pf_prop_ws_b", ctypes.byref(g), self.batch),
                                   dtype=torch.complex64, device=device) for _ in range(nlanes)]
        self.ws_a, self.ws_b = self.ws_a_l[0], self.ws_b_l[0]
        self.lane_streams = [torch.cuda.Stream(device=device) for _ in range(nlanes)]
        self.plan_x = dev.fft_plan(px, device)
        self.plan_y = dev.fft_plan(py, device)
        # register-FFT path (square power-of-two pads) consumes Uhat transposed
        self.transposed = bool(_lib.call("pf_prop_fast", ctypes.byref(g)))
        # P = 140 (config 1's reference pad): every stage of a unit in one CTA's shared memory
        self.onchip = (_ONCHIP and not self.transposed
                       and bool(_lib.call("pf_prop_onchip_ok", ctypes.byref(g))))

    def freq_order(self, freqs: np.ndarray, n_frames: int):
        """(frequency visiting order, Horner spacing): descending with kernel C applying the
        illumination phase by Horner's rule (pf_prop_rows_out_horner) when the geometry
        allows it (register path, centred crops, one illumination, one frame, uniformly
        spaced frequencies), else ascending and None."""
        F = int(freqs.size)
        g = self.geom
        P = g.px
        ok = (_HORNER and self.transposed and F >= 2 and n_frames == 1 and g.n_illum == 1
              and g.include_illum and 2 * g.nx == P and 2 * g.ny == P
              and 2 * g.nu0x == -g.nx and 2 * g.nu0y == -g.ny)
        if ok:
            d = np.diff(np.asarray(freqs, dtype=np.float64))
            ok = bool(np.all(np.abs(d - d[0]) <= 1e-9 * abs(d[0])))
        if not ok:
            return list(range(F)), None
        return list(range(F - 1, -1, -1)), float(d[0]) / SPEED_OF_LIGHT

    def run_frequency(self, uhat_ptr: int, khat: float, ill_ptr: int, frame_w_ptr: int,
                      n_frames: int, vol: torch.Tensor, vol_frame_stride: int,
                      plane_lo: int = 0, plane_hi: int | None = None, stream=None,
                      uhat_ptr_for_batch=None, lane: int = 0, horner=None,
                      vol_out=None) -> None:
        """One frequency over planes [plane_lo, plane_hi).  horner=(dkhat, f, F): kernel C
        by Horner's rule (frequencies visited in ``freq_order``)."""
        plane_hi = self.nplanes if plane_hi is None else plane_hi
        s = dev.stream_ptr(stream)
        gref = ctypes.byref(self.geom)
        base = dev.ptr(self.planes_dev)
        wa, wb = dev.ptr(self.ws_a_l[lane]), dev.ptr(self.ws_b_l[lane])
        for b0 in range(plane_lo, plane_hi, self.batch):
            nb = min(self.batch, plane_hi - b0)
            pp = base + b0 * self.plane_size
            up = uhat_ptr if uhat_ptr_for_batch is None else uhat_ptr_for_batch(b0, nb)
            _lib.call("pf_prop_kernel_rows", pp, nb, khat, gref, self.plan_x.ref, wa, s)
            _lib.call("pf_prop_columns", pp, nb, gref, self.plan_y.ref, wa, up, wb, 0, s)
            if horner is not None:
                dk, fi, nf = horner
                B = _HORNER_BLOCK
                if nf <= B:
                    mode, wo = (2 if fi == 0 else 1), 0
                else:   # blocks of B frequencies chained through the outer accumulator
                    mode = 4 if fi == 0 else (3 if fi % B == 0 else 1)
                    wo_t = self._ws_o(lane, nb)
                    if fi == nf - 1:
                        wo_t.zero_()
                    wo = dev.ptr(wo_t)
                # a nonzero status (geometry not eligible) raises PfError in _lib.call
                _lib.call("pf_prop_rows_out_horner", pp, nb, khat, dk, mode, gref,
                          self.plan_x.ref, wb, ill_ptr, frame_w_ptr, dev.ptr(vol), wo, B * dk,
                          vol_out, s)
                continue
            _lib.call("pf_prop_rows_out", pp, nb, khat, gref, self.plan_x.ref, wb, ill_ptr,
                      frame_w_ptr, n_frames, dev.ptr(vol), vol_frame_stride, s)

    def _ws_o(self, lane: int, nb: int) -> torch.Tensor:
        """Outer Horner accumulator of a lane's plane batch (nb x ny x nx complex64)."""
        lst = self.__dict__.setdefault("ws_o_l", {})
        t = lst.get(lane)
        if t is None:
            t = lst[lane] = torch.empty((self.batch * self.geom.ny * self.geom.nx,),
                                        dtype=torch.complex64, device=self.device)
        return t[:nb * self.geom.ny * self.geom.nx]

    def fbatch_ok(self, n_freq: int, n_frames: int) -> bool:
        """All frequencies in one launch per stage (small configs, static volume);
        register path or, for other pads (config 1's P = 140), the Stockham path."""
        if n_frames != 1 or (not self.transposed and not _FBATCH_GENERIC):
            return False
        g = self.geom
        per = 8 * ((g.py // 2 + 1) * (g.px // 2 + 1) + g.n_illum * g.ny * g.px)
        return n_freq * self.n_planes_total * per <= _FBATCH_BYTES

    def onchip_groups(self, nf: int) -> int:
        """Frequency groups of the on-chip path: the count minimising (CTA waves over 148
        SMs) x (frequencies per CTA), fewest groups on ties; from the whole grid's plane
        count, so a plane-sharded engine sums each plane in the same order."""
        if _ONCHIP_GROUPS > 0:
            return max(1, min(nf, _ONCHIP_GROUPS))
        best = None
        for gr in range(1, nf + 1):
            fpc = -(-nf // gr)
            cost = -(-self.n_planes_total * (-(-nf // fpc)) // 148) * fpc
            if best is None or cost < best[0]:
                best = (cost, gr)
        return best[1]

    def run_fbatch(self, uhat: torch.Tensor, uhat_fs: int, freqs: np.ndarray, ill_ptr: int,
                   frame_w: torch.Tensor, vol: torch.Tensor, stream=None) -> None:
        g = self.geom
        nf = int(freqs.size)
        key = ("fb", nf)
        if getattr(self, "_fb_key", None) != key:
            na = (g.py // 2 + 1) * (g.px // 2 + 1)
            self._fb_ws_a = torch.empty((nf * self.nplanes * na,), dtype=torch.complex64,
                                        device=self.device)
            nb = self.nplanes * g.n_illum * g.ny * g.px
            self._fb_ws_b = torch.empty((nf * nb,), dtype=torch.complex64, device=self.device)
            self._fb_kt = torch.from_numpy(np.asarray(freqs, dtype=np.float64)
                                           / (SPEED_OF_LIGHT * 2 * np.pi)).to(self.device)
            # rad/m, formed exactly as the per-frequency launches form khat
            self._fb_kh = torch.tensor([float(f) / SPEED_OF_LIGHT for f in freqs],
                                       dtype=torch.float64).to(self.device)
            self._fb_strides = (self.nplanes * na, nb)
            self._fb_key = key
        fa, fbs = self._fb_strides
        if self.onchip:
            groups = self.onchip_groups(nf)
            if getattr(self, "_oc_key", None) != (nf, groups):
                ng = -(-nf // -(-nf // groups))
                self._oc_part = (torch.empty((ng * self.nplanes * g.ny * g.nx,),
                                             dtype=torch.complex64, device=self.device)
                                 if ng > 1 else None)
                self._oc_key = (nf, groups)
            part = 0 if self._oc_part is None else dev.ptr(self._oc_part)
            _lib.call("pf_prop_fbatch_onchip", dev.ptr(self.planes_dev), self.nplanes,
                      dev.ptr(self._fb_kt), nf, ctypes.byref(g), dev.ptr(uhat), uhat_fs, ill_ptr,
                      dev.ptr(frame_w), dev.ptr(vol), part, groups, _ONCHIP_WARPS,
                      dev.stream_ptr(stream))
            return
        if not self.transposed:
            _lib.call("pf_prop_fbatch_generic", dev.ptr(self.planes_dev), self.nplanes,
                      dev.ptr(self._fb_kh), nf, ctypes.byref(g), self.plan_x.ref, self.plan_y.ref,
                      dev.ptr(self._fb_ws_a), fa, dev.ptr(uhat), uhat_fs, dev.ptr(self._fb_ws_b),
                      fbs, ill_ptr, dev.ptr(frame_w), dev.ptr(vol), dev.stream_ptr(stream))
            return
        _lib.call("pf_prop_fbatch", dev.ptr(self.planes_dev), self.nplanes, dev.ptr(self._fb_kt),
                  nf, ctypes.byref(g), self.plan_x.ref, dev.ptr(self._fb_ws_a), fa, dev.ptr(uhat),
                  uhat_fs, dev.ptr(self._fb_ws_b), fbs, ill_ptr, dev.ptr(frame_w), dev.ptr(vol),
                  dev.stream_ptr(stream))

    def run_batches(self, body, stream=None, lo: int = 0, hi: int | None = None) -> None:
        """Call ``body(b0, b1, lane, lane_stream)`` for every plane batch of [lo, hi),
        alternating lanes.  Lanes wait for ``stream`` (inputs ready) and ``stream``
        waits for every lane."""
        hi = self.nplanes if hi is None else hi
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        for ls in self.lane_streams:
            ls.wait_stream(main)
        for i, b0 in enumerate(range(lo, hi, self.batch)):
            lane = i % len(self.lane_streams)
            ls = self.lane_streams[lane]
            with torch.cuda.stream(ls):
                body(b0, min(hi, b0 + self.batch), lane, ls)
        for ls in self.lane_streams:
            main.wait_stream(ls)


def _frame_weights(freqs: np.ndarray, times, device) -> torch.Tensor:
    if times is None:
        w = np.ones((freqs.size, 1), dtype=np.complex64)
    else:
        w = dev.phase_factors(freqs, times)
    return torch.from_numpy(np.ascontiguousarray(w)).to(device)


def _ill_tensor(slices, device) -> torch.Tensor:
    ill = illumination_coordinates(slices.relay, slices.illuminations)
    return torch.from_numpy(np.array(ill, dtype=np.float64, copy=True)).to(device)


_PINNED: dict = {}


_D2H_CHUNK = 1 << 22     # complex64 elements per device->host chunk (32 MB)


def _host_c128(vol: torch.Tensor) -> np.ndarray:
    """Device complex64 [frames, V] -> fresh host complex128 array (the reference's field
    dtype).  The volume goes device->host in 32 MB chunks into a cached pinned buffer on a
    side stream; host threads upcast each chunk into the output as soon as its copy lands
    (numpy releases the GIL), so the transfer and the upcast overlap."""
    n = vol.numel()
    buf = _PINNED.get("vol")
    if buf is None or buf.numel() < n:
        _PINNED.pop("vol", None)
        buf = torch.empty((n,), dtype=torch.complex64, pin_memory=True)
        _PINNED["vol"] = buf
    if "pool" not in _PINNED:
        from concurrent.futures import ThreadPoolExecutor
        _PINNED["pool"] = ThreadPoolExecutor(8)
        _PINNED["stream"] = {}
    side = _PINNED["stream"].get(vol.device.index)
    if side is None:
        side = _PINNED["stream"][vol.device.index] = torch.cuda.Stream(device=vol.device)
    side.wait_stream(torch.cuda.current_stream(vol.device))
    flat_dev = vol.reshape(-1)
    edges = list(range(0, n, _D2H_CHUNK)) + [n]
    events = []
    with torch.cuda.stream(side):
        for a, b in zip(edges[:-1], edges[1:]):
            buf[a:b].copy_(flat_dev[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
            events.append(ev)
    src = buf[:n].numpy()
    out = np.empty(vol.shape, dtype=np.complex128)
    flat = out.reshape(-1)

    def upcast(j):
        events[j].synchronize()
        flat[edges[j]:edges[j + 1]] = src[edges[j]:edges[j + 1]]

    list(_PINNED["pool"].map(upcast, range(len(events))))
    return out


def _volume(grid, vol: torch.Tensor, times) -> ReconstructionVolume:
    """ReconstructionVolume from the device result (reference semantics: complex128, finite,
    read-only).  The finiteness check runs on the device; the host array is freshly made
    here and handed over without the defensive copy."""
    _require(bool(torch.isfinite(torch.view_as_real(vol)).all()), "field must be finite")
    field = _host_c128(vol)
    if times is None:
        field = field[0]
    return ReconstructionVolume._owned(grid, field, times)


# ---------------------------------------------------------------------------
# engine cache: the drop-in functions plan once per geometry (like an FFT plan cache)
# ---------------------------------------------------------------------------

_ENGINES: "dict" = {}
_ENGINE_CACHE = int(os.environ.get("PF_ENGINE_CACHE", "2"))


def _fingerprint(obj):
    """Hashable value-identity of geometry objects (dataclasses of scalars / arrays)."""
    import dataclasses
    import hashlib
    if obj is None or isinstance(obj, (bool, int, float, str)):
        return obj
    if isinstance(obj, (np.floating, np.integer)):
        return obj.item()
    if isinstance(obj, np.ndarray):
        a = np.ascontiguousarray(obj)
        return ("nd", a.shape, a.dtype.str, hashlib.sha1(a.tobytes()).hexdigest())
    if isinstance(obj, (list, tuple)):
        return tuple(_fingerprint(x) for x in obj)
    if dataclasses.is_dataclass(obj):
        return (type(obj).__name__,) + tuple(
            (f.name, _fingerprint(getattr(obj, f.name))) for f in dataclasses.fields(obj))
    return ("id", id(obj))


def _slices_geometry(slices):
    return (_fingerprint(np.asarray(slices.frequencies, dtype=np.float64)),
            _fingerprint(slices.relay), _fingerprint(slices.illuminations))


def _nufft_window() -> str:
    from . import nufft
    return nufft.DEFAULT_WINDOW


def cached_engine(kind: str, slices, grid, options: tuple, factory):
    """Engine for (kind, slices geometry, grid, options) from a small LRU cache; ``factory``
    builds it on a miss.  Engines hold only geometry-derived plans and workspaces, so a
    hit is exactly what a rebuild would produce."""
    if _ENGINE_CACHE <= 0:
        return factory()
    # the module's path switches are part of the key: an engine captured under other
    # switches would replay their launch sequence
    flags = (_LANES, _FAST_BATCH_CAP, _FBATCH_BYTES, _FBATCH_GENERIC, _HORNER, _HORNER_BLOCK,
             _BATCH_BYTES, _ONCHIP, _ONCHIP_GROUPS, _ONCHIP_WARPS, _nufft_window())
    devi = torch.cuda.current_device() if torch.cuda.is_available() else -1
    key = (kind, devi, _slices_geometry(slices), _fingerprint(grid),
           _fingerprint(options), flags)
    eng = _ENGINES.pop(key, None)
    if eng is None:
        eng = factory()
    _ENGINES[key] = eng
    while len(_ENGINES) > _ENGINE_CACHE:
        _ENGINES.pop(next(iter(_ENGINES)))
    return eng


def clear_engine_cache() -> None:
    _ENGINES.clear()


# ---------------------------------------------------------------------------
# rsd: uniform relay -> cuboid at the relay pitch
# ---------------------------------------------------------------------------


class GraphedRun:
    """CUDA-graph replay of an engine's ``run(coeff, vol, stream)``.

    The propagation enqueues thousands of small kernels (config 4: ~6k per
    step); replaying a captured graph removes the per-launch host cost so the
    GPU runs them back to back.  One graph is captured per (coeff, vol) buffer
    pair; inputs and outputs are used in place.
    """

    def run_graphed(self, coeff: torch.Tensor, vol: torch.Tensor, stream=None, vol_out=None):
        graphs = self.__dict__.setdefault("_graphs", {})
        key = (coeff.data_ptr(), vol.data_ptr(), vol_out)
        kw = {} if vol_out is None else {"vol_out": vol_out}
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        g = graphs.get(key)
        if g is None:
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                self.run(coeff, vol, side, **kw)    # warm-up: plans, attributes, caches
            main.wait_stream(side)
            g = torch.cuda.CUDAGraph()
            n0 = _lib.launches()
            with torch.cuda.graph(g, stream=side):
                self.run(coeff, vol, side, **kw)
            main.wait_stream(side)
            self.graph_kernels = _lib.launches() - n0   # libpfgpu launches per replay
            graphs[key] = g
        with torch.cuda.stream(main):
            g.replay()
        return vol

    def run_dropin(self, coeff: torch.Tensor, stream=None) -> torch.Tensor:
        """Graph replay on engine-owned input/output buffers (the drop-in functions' path:
        ``coeff`` is copied into the captured input, the returned volume is reused by the
        next call)."""
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        inp = self.__dict__.get("_dropin_in")
        if inp is None or inp.shape != coeff.shape:
            inp = torch.empty_like(coeff, device=self.device)
            self._dropin_in = inp
            self._dropin_out = torch.zeros((self.n_frames, self.n_voxels),
                                           dtype=torch.complex64, device=self.device)
        with torch.cuda.stream(main):
            inp.copy_(coeff, non_blocking=True)
        return self.run_graphed(inp, self._dropin_out, main)

    @property
    def chunk_unit(self) -> int:
        """Plane granularity of chunks: one round of plane batches over all stream lanes."""
        return self.prop.batch * len(self.prop.lane_streams)

    def chunk_bounds(self, n_chunks: int) -> list:
        """Contiguous local plane ranges of ``run_chunk`` (distributed.chunk_split)."""
        from .distributed import chunk_split
        return chunk_split(self.n_planes_local, n_chunks, self.chunk_unit)

    def run_graphed_chunk(self, coeff: torch.Tensor, vol: torch.Tensor, j: int, n_chunks: int,
                          stream=None):
        """Graph replay of chunk j of ``n_chunks``: chunk 0 also builds the relay spectra;
        chunk j leaves planes ``chunk_bounds(n_chunks)[j]`` of ``vol`` final, so their
        transfer can start while later chunks compute (multi-GPU volume gather)."""
        graphs = self.__dict__.setdefault("_chunk_graphs", {})
        key = (coeff.data_ptr(), vol.data_ptr(), j, n_chunks)
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        lo, hi = self.chunk_bounds(n_chunks)[j]
        g = graphs.get(key)
        if g is None:
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                self.run_chunk(coeff, vol, lo, hi, j == 0, side)
            main.wait_stream(side)
            g = torch.cuda.CUDAGraph()
            n0 = _lib.launches()
            with torch.cuda.graph(g, stream=side):
                self.run_chunk(coeff, vol, lo, hi, j == 0, side)
            main.wait_stream(side)
            # libpfgpu launches per replay of chunk j of n_chunks
            self.__dict__.setdefault("chunk_graph_kernels", {})[(j, n_chunks)] = \
                _lib.launches() - n0
            graphs[key] = g
        with torch.cuda.stream(main):
            g.replay()
        return vol


class RsdEngine(GraphedRun):
    """Device plan of :func:`rsd` for one (slices geometry, grid); reusable.

    ``run(coeff)`` takes the frequency-major device coefficients [F, I, D]
    and returns the device volume [n_frames, Nz*Ny*Nx] (complex64).
    Reference: reconstruct.py:208-268.
    """

    def __init__(self, slices, grid, padding="exact", include_illumination=True, times=None,
                 device=None, plane_range=None):
        _require(_kind(grid) == "cuboid", "rsd reconstructs onto a cuboid grid")
        _require(padding in ("exact", "none"), "padding must be 'exact' or 'none'")
        relay = _uniform_relay(slices)
        g = relay.grid
        vg = grid.grid
        _require(_close(vg.dx, g.dx) and _close(vg.dy, g.dy),
                 "output lateral pitch must equal the relay pitch")
        cx, cy = g.center()
        nu0x = _integer_offset(vg.x0 - cx, g.dx, "output grid x origin offset")
        nu0y = _integer_offset(vg.y0 - cy, g.dy, "output grid y origin offset")
        zs = vg.z_coords()
        _check_depths(zs, g.z)
        self.times = _check_times(times)
        jx_lo, jx_hi = -(g.nx // 2), g.nx - g.nx // 2 - 1
        jy_lo, jy_hi = -(g.ny // 2), g.ny - g.ny // 2 - 1
        nux_lo, nux_hi = nu0x, nu0x + vg.nx - 1
        nuy_lo, nuy_hi = nu0y, nu0y + vg.ny - 1
        if padding == "none":
            _require(vg.nx == g.nx and vg.ny == g.ny and nu0x == jx_lo and nu0y == jy_lo,
                     "padding='none' requires the output lattice to coincide with "
                     "the relay lattice")
            px, py = g.nx, g.ny
        else:
            lx = max(abs(nux_lo - jx_hi), abs(nux_hi - jx_lo))
            ly = max(abs(nuy_lo - jy_hi), abs(nuy_hi - jy_lo))
            px = _exact_pad(lx, max(abs(nux_lo), abs(nux_hi), g.nx // 2), g.nx)
            py = _exact_pad(ly, max(abs(nuy_lo), abs(nuy_hi), g.ny // 2), g.ny)
        self.device = device or dev.require_cuda()
        self.relay_grid, self.grid = g, grid
        self.px, self.py = px, py
        self.freqs = np.asarray(slices.frequencies, dtype=np.float64)
        self.n_illum = int(slices.illuminations.count)
        k_lo, k_hi = plane_range or (0, vg.nz)
        self.k_lo, self.k_hi = k_lo, k_hi
        planes = [PlaneSpec(zs[k] - g.z, g.dx, g.dy, vg.x0, vg.dx, vg.y0, vg.dy, zs[k],
                            0, k - k_lo) for k in range(k_lo, k_hi)]
        self.prop = Propagator(self.device, px, py, vg.nx, vg.ny, nu0x, nu0y, self.n_illum,
                               include_illumination, planes, py * px, n_planes_total=vg.nz)
        self.ill = _ill_tensor(slices, self.device)
        self.frame_w = _frame_weights(self.freqs, self.times, self.device)
        self.n_frames = 1 if self.times is None else self.times.size
        self.plane_voxels = vg.nx * vg.ny
        self.uhat = torch.empty((self.freqs.size, self.n_illum, py, px), dtype=torch.complex64,
                                device=self.device)

    @property
    def n_voxels(self) -> int:
        return (self.k_hi - self.k_lo) * self.plane_voxels

    @property
    def n_planes_local(self) -> int:
        return self.k_hi - self.k_lo

    def run_chunk(self, coeff, vol, lo: int, hi: int, first: bool, stream=None):
        """Local planes [lo, hi) only (lanes path; chunk 0 builds the spectra)."""
        if first:
            self.relay_spectra(coeff, stream)
        pv = self.plane_voxels
        vol.view(self.n_frames, -1)[:, lo * pv:hi * pv].zero_()
        per_f = self.n_illum * self.py * self.px
        uhat = self.uhat

        def body(b0, b1, lane, ls):
            order, dk = self.prop.freq_order(self.freqs, self.n_frames)
            for fi in order:
                khat = float(self.freqs[fi]) / SPEED_OF_LIGHT
                self.prop.run_frequency(dev.ptr(uhat) + 8 * fi * per_f, khat, dev.ptr(self.ill),
                                        dev.ptr(self.frame_w) + 8 * fi * self.n_frames,
                                        self.n_frames, vol, self.n_voxels, plane_lo=b0,
                                        plane_hi=b1, stream=ls, lane=lane,
                                        horner=None if dk is None else (dk, fi, len(order)))

        self.prop.run_batches(body, stream, lo, hi)
        return vol

    def relay_spectra(self, coeff: torch.Tensor, stream=None) -> torch.Tensor:
        """Uhat_f = cfft2(pad_embed(u_f)) for all (f, p), natural order (reconstruct.py:259-260)."""
        g = self.relay_grid
        F, I = self.freqs.size, self.n_illum
        if self.prop.transposed:   # register path: embed + row FFT + column FFT, Uhat^T
            _lib.call("pf_relay_spectra_fast", dev.ptr(coeff), F * I, g.ny, g.nx, g.ny * g.nx,
                      dev.ptr(self.uhat), self.px, self.prop.plan_x.ref, dev.stream_ptr(stream))
            return self.uhat
        _lib.call("pf_embed_centered", dev.ptr(coeff), F * I, g.ny, g.nx, g.ny * g.nx,
                  dev.ptr(self.uhat), self.py, self.px, 0, dev.stream_ptr(stream))
        dev.fft2_natural(self.uhat, self.py, self.px, F * I, -1, 1.0, stream)
        return self.uhat

    def fused_gather_ok(self) -> bool:
        """Kernel C's final Horner step can store the finished planes elsewhere (the fused
        volume gather of distributed.PeerVolume): register path, Horner geometry, no
        frequency-batched launches."""
        return (not self.prop.fbatch_ok(self.freqs.size, self.n_frames)
                and self.prop.freq_order(self.freqs, self.n_frames)[1] is not None)

    def run(self, coeff: torch.Tensor, vol: torch.Tensor | None = None, stream=None,
            vol_out: int | None = None):
        """``vol_out``: device address the finished planes go to instead of ``vol`` (rank 0's
        volume at this shard's first plane, peer memory); ``vol`` then only accumulates."""
        if vol is None:
            vol = torch.zeros((self.n_frames, self.n_voxels), dtype=torch.complex64,
                              device=self.device)
        else:
            vol.zero_()
        if vol_out is not None and not self.fused_gather_ok():
            raise ValueError("the fused volume gather needs the Horner register path")
        uhat = self.relay_spectra(coeff, stream)
        per_f = self.n_illum * self.py * self.px
        if self.prop.fbatch_ok(self.freqs.size, self.n_frames):
            self.prop.run_fbatch(uhat, per_f, self.freqs, dev.ptr(self.ill), self.frame_w, vol,
                                 stream)
            return vol

        # plane batches outer, frequencies inner: the batch's volume slice stays
        # L2-resident across its ascending-frequency accumulation
        def body(b0, b1, lane, ls):
            order, dk = self.prop.freq_order(self.freqs, self.n_frames)
            for fi in order:
                khat = float(self.freqs[fi]) / SPEED_OF_LIGHT
                self.prop.run_frequency(dev.ptr(uhat) + 8 * fi * per_f, khat, dev.ptr(self.ill),
                                        dev.ptr(self.frame_w) + 8 * fi * self.n_frames,
                                        self.n_frames, vol, self.n_voxels, plane_lo=b0,
                                        plane_hi=b1, stream=ls, lane=lane,
                                        horner=None if dk is None else (dk, fi, len(order)),
                                        vol_out=vol_out)

        self.prop.run_batches(body, stream)
        return vol


def rsd(slices, grid, padding: str = "exact", times=None, threads: int = 1,
        include_illumination: bool = True) -> ReconstructionVolume:
    """Plane-to-plane propagation onto a cuboid sharing the relay pitch (reconstruct.py:208-268)."""
    eng = cached_engine("rsd", slices, grid, (padding, bool(include_illumination),
                                              None if times is None else np.asarray(times)),
                        lambda: RsdEngine(slices, grid, padding, include_illumination, times))
    vol = eng.run_dropin(device_coefficients(slices))
    return _volume(grid, vol, eng.times)


# ---------------------------------------------------------------------------
# dispatcher, video, projection
# ---------------------------------------------------------------------------


def reconstruct(slices, grid, algorithm: str, *, eps: float = 1e-6, padding: str = "exact",
                alpha: float | None = None, beta: float | None = None,
                lattice_pitch: float | None = None, z_pitch: float | None = None,
                scatter: str = "trilinear", times=None, threads: int = 1,
                include_illumination: bool = True) -> ReconstructionVolume:
    """Run one algorithm selected by name (reference reconstruct.py:776-809)."""
    name = algorithm.replace("_", "-").lower()
    common = dict(times=times, threads=threads, include_illumination=include_illumination)
    if name == "rsd":
        return rsd(slices, grid, padding=padding, **common)
    table = _ALGORITHMS()
    if name == "srsd-nursd2":
        _require(alpha is not None, "srsd-nursd2 needs a scale factor (alpha)")
        return table[name](slices, grid, alpha=alpha, beta=beta, eps=eps, **common)
    if name == "srsd":
        return table[name](slices, grid, **common)
    if name in ("nursd1", "nursd2"):
        return table[name](slices, grid, eps=eps, **common)
    if name == "nursd3":
        return table[name](slices, grid, eps=eps, lattice_pitch=lattice_pitch, **common)
    if name == "nursd3d":
        return table[name](slices, grid, eps=eps, z_pitch=z_pitch, **common)
    if name == "rsd3d":
        return table[name](slices, grid, scatter=scatter, z_pitch=z_pitch, **common)
    raise ValidationError(
        f"unknown algorithm {algorithm!r}; choose from {', '.join(ALGORITHM_NAMES)}")


def _ALGORITHMS():
    from . import algorithms as A
    return {"srsd": A.srsd, "nursd1": A.nursd1, "nursd2": A.nursd2, "nursd3": A.nursd3,
            "nursd3d": A.nursd3d, "srsd-nursd2": A.srsd_nursd2, "rsd3d": A.rsd3d}


def light_transport_video(slices, grid, times, algorithm: str = "rsd", threads: int = 1,
                          include_illumination: bool = True, **options) -> ReconstructionVolume:
    """Frame t = sum_w exp(1j w t) V_w (reference reconstruct.py:812-831)."""
    name = algorithm.replace("_", "-").lower()
    _require(name in ("rsd", "srsd"),
             "time-resolved rendering supports the plane-to-plane propagators "
             "('rsd' and 'srsd')")
    return reconstruct(slices, grid, name, times=np.asarray(times, dtype=np.float64),
                       threads=threads, include_illumination=include_illumination, **options)


def project_max_depth(volume: ReconstructionVolume, frame: int = 0) -> np.ndarray:
    """Maximum-intensity projection of |field| along depth (reconstruct.py:834-836)."""
    return np.abs(volume.as_array3d(frame)).max(axis=0)
