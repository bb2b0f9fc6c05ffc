"""Phasor kernel (host) and the temporal phasor transform (GPU, kernel K1).

Drop-in for reference ``phasor.py``: ``build_kernel`` (:72-104) is the same
closed-form host computation; ``to_frequency`` (:107-127) runs on the GPU
(``pf_temporal_dft``) and returns a :class:`DeviceFrequencySlices`, which
behaves like the reference ``FrequencySlices`` (same attributes; the host
``coefficients`` array is materialised lazily) while keeping the
frequency-major complex64 tensor resident on the device for the propagators.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .core import SPEED_OF_LIGHT, FrequencySlices, ValidationError, _readonly, _require


@dataclass(frozen=True)
class PhasorKernel:
    """Gaussian packet on the DFT bins (reference ``phasor.py:42-69``)."""

    lambda_c: float
    delta_t: float
    n_bins: int
    threshold: float
    omega_c: float
    sigma: float
    bin_indices: np.ndarray
    frequencies: np.ndarray
    weights: np.ndarray

    @property
    def n_freq(self) -> int:
        return int(self.bin_indices.size)

    @property
    def lambda_star(self) -> float:
        return 2.0 * math.pi * SPEED_OF_LIGHT / float(self.frequencies[-1])


def build_kernel(lambda_c: float, n_bins: int, delta_t: float,
                 threshold: float = 0.01) -> PhasorKernel:
    """Retain positive bins whose Gaussian weight reaches ``threshold`` (phasor.py:72-104).

    omega_c = 2 pi c / lambda_c, sigma = c / (5 lambda_c); bin k in 1..T/2.
    """
    _require(lambda_c > 0 and math.isfinite(lambda_c), "virtual wavelength must be > 0")
    _require(n_bins >= 2, "need at least two time bins")
    _require(delta_t > 0 and math.isfinite(delta_t), "bin width must be > 0")
    _require(0.0 < threshold < 1.0, "retention threshold must lie in (0, 1)")
    omega_c = 2.0 * math.pi * SPEED_OF_LIGHT / lambda_c
    sigma = SPEED_OF_LIGHT / (5.0 * lambda_c)
    k = np.arange(1, n_bins // 2 + 1)
    om = 2.0 * math.pi * k / (n_bins * delta_t)
    wt = np.exp(-((om - omega_c) ** 2) / (2.0 * sigma * sigma))
    sel = wt >= threshold
    if not sel.any():
        raise ValidationError("no DFT bin reaches the retention threshold; the time window is "
                              "too short or the virtual wavelength is outside the sampled band")
    return PhasorKernel(float(lambda_c), float(delta_t), int(n_bins), float(threshold), omega_c,
                        sigma, _readonly(k[sel]), _readonly(om[sel]), _readonly(wt[sel]))


class DeviceFrequencySlices:
    """Frequency slices resident on the GPU, frequency-major: ``device_coefficients[F, I, D]``.

    Exposes the reference ``FrequencySlices`` attribute set (``frequencies``,
    ``coefficients`` [I, D, F] complex128 materialised on first access,
    ``relay``, ``illuminations``, ``n_freq``, ``n_illum``, ``max_frequency``,
    ``shortest_wavelength``) so it can be handed to reference-style callers.
    """

    def __init__(self, frequencies, device_coefficients: torch.Tensor, relay, illuminations):
        w = np.asarray(frequencies, dtype=np.float64)
        _require(w.ndim == 1 and w.size >= 1, "frequencies must be a nonempty vector")
        _require(bool(np.all(np.diff(w) > 0)), "frequencies must be strictly increasing")
        _require(device_coefficients.dtype == torch.complex64 and device_coefficients.dim() == 3
                 and device_coefficients.shape[0] == w.size,
                 "device coefficients must be complex64 [F, n_illum, n_detect]")
        _require(device_coefficients.shape[2] == relay.count,
                 "detection axis must match relay point count")
        _require(device_coefficients.shape[1] == illuminations.count,
                 "illumination axis must match illumination point count")
        self.frequencies = _readonly(w)
        self.device_coefficients = device_coefficients
        self.relay = relay
        self.illuminations = illuminations
        self._host = None

    @property
    def coefficients(self) -> np.ndarray:
        if self._host is None:
            h = self.device_coefficients.permute(1, 2, 0).cpu().numpy().astype(np.complex128)
            self._host = _readonly(h)
        return self._host

    def to_host(self) -> FrequencySlices:
        return FrequencySlices(self.frequencies, self.coefficients, self.relay, self.illuminations)

    @property
    def n_freq(self) -> int:
        return int(self.frequencies.size)

    @property
    def n_illum(self) -> int:
        return int(self.device_coefficients.shape[1])

    @property
    def max_frequency(self) -> float:
        return float(self.frequencies[-1])

    @property
    def shortest_wavelength(self) -> float:
        return 2.0 * math.pi * SPEED_OF_LIGHT / self.max_frequency


def device_coefficients(slices) -> torch.Tensor:
    """Frequency-major complex64 device tensor [F, I, D] for any slices object."""
    if isinstance(slices, DeviceFrequencySlices):
        return slices.device_coefficients
    device = dev.require_cuda()
    c = np.asarray(slices.coefficients)
    host = torch.from_numpy(np.ascontiguousarray(c.transpose(2, 0, 1)).astype(np.complex64))
    return host.to(device, non_blocking=False)


class TemporalPlan:
    """Device tables of the retained-bin transform for one (kernel, t0)."""

    def __init__(self, kernel, t0: float, device: torch.device):
        T = int(kernel.n_bins)
        bins = np.asarray(kernel.bin_indices, dtype=np.int64)
        om = np.asarray(kernel.frequencies, dtype=np.float64)
        wt = np.asarray(kernel.weights, dtype=np.float64)
        self.n_bins, self.n_freq = T, int(bins.size)
        self.bins = torch.from_numpy(bins.astype(np.int32)).to(device)
        self.wphase = torch.from_numpy((wt * np.exp(-1j * om * t0)).astype(np.complex64)).to(device)
        m = T // 64 if T % 64 == 0 else 0
        self.fast = m in (1, 2, 4, 8, 16, 32, 64, 128, 256)
        if self.fast:
            r = np.arange(m, dtype=np.int64)
            ph = (np.outer(r, bins) % T).astype(np.float64) / T   # [M, F], exact integer reduction
            self.tw = torch.from_numpy(np.exp(-2j * np.pi * ph).astype(np.complex64)).to(device)
            k = bins % 64
            # inner bins the retained bins fold to (K1 forms and parks only these)
            self.inner_mask = sum(1 << int(j) for j in set(np.minimum(k, 64 - k).tolist()))
        else:
            ph = np.arange(T, dtype=np.float64) / T
            self.tw = torch.from_numpy(np.exp(-2j * np.pi * ph).astype(np.complex64)).to(device)

    def run(self, hist: torch.Tensor, out: torch.Tensor, stream=None) -> None:
        """hist float32 [n_traces, T] (contiguous) -> out complex64 [F, n_traces]."""
        n_traces = hist.shape[0]
        if self.fast:
            _lib.call("pf_temporal_dft", dev.ptr(hist), n_traces, self.n_bins, dev.ptr(self.bins),
                      dev.ptr(self.tw), dev.ptr(self.wphase), self.n_freq, dev.ptr(out),
                      out.stride(0), self.inner_mask, dev.stream_ptr(stream))
        else:
            _lib.call("pf_temporal_dft_direct", dev.ptr(hist), n_traces, self.n_bins,
                      dev.ptr(self.bins), dev.ptr(self.tw), dev.ptr(self.wphase), self.n_freq,
                      dev.ptr(out), out.stride(0), dev.stream_ptr(stream))


_PLANS: dict = {}


def _plan_for(kernel, t0: float, device) -> "TemporalPlan":
    """TemporalPlan cache keyed by the kernel's bins / frequencies / weights and t0."""
    key = (int(kernel.n_bins), np.asarray(kernel.bin_indices).tobytes(),
           np.asarray(kernel.frequencies, dtype=np.float64).tobytes(),
           np.asarray(kernel.weights, dtype=np.float64).tobytes(), float(t0), str(device))
    plan = _PLANS.pop(key, None) or TemporalPlan(kernel, t0, device)
    _PLANS[key] = plan
    while len(_PLANS) > 4:
        _PLANS.pop(next(iter(_PLANS)))
    return plan


class _HostStager:
    """Host histograms -> K1 without a pageable copy: the rows are cut into chunks; host
    threads copy chunk c into pinned buffer c % 2 (numpy releases the GIL) while chunk c - 1
    is in flight host->device on the copy stream and chunk c - 2 is in K1, whose device
    ring slot c % 2 is reused once its K1 has run.  Float64 payloads are narrowed to
    float32 by the same copy."""

    CHUNK_BYTES = int(os.environ.get("PF_STAGE_MB", "64")) << 20
    BUFS = int(os.environ.get("PF_STAGE_BUFS", "2"))
    THREADS = int(os.environ.get("PF_STAGE_THREADS", "8"))

    def __init__(self, device):
        from concurrent.futures import ThreadPoolExecutor
        self.device = device
        n = self.CHUNK_BYTES // 4
        nb = self.BUFS
        self.pinned = [torch.empty((n,), dtype=torch.float32, pin_memory=True) for _ in range(nb)]
        self.ring = [torch.empty((n,), dtype=torch.float32, device=device) for _ in range(nb)]
        self.h2d_done = [torch.cuda.Event() for _ in range(nb)]
        self.k1_done = [torch.cuda.Event() for _ in range(nb)]
        self.copy_stream = torch.cuda.Stream(device=device)
        self.pool = ThreadPoolExecutor(self.THREADS)

    def run(self, host: np.ndarray, plan: "TemporalPlan", out: torch.Tensor) -> None:
        n_tr, T = host.shape
        rows = max(1, self.CHUNK_BYTES // (4 * T))
        main = torch.cuda.current_stream(self.device)
        th = self.THREADS
        for c, r0 in enumerate(range(0, n_tr, rows)):
            k = c % self.BUFS
            r1 = min(n_tr, r0 + rows)
            n = (r1 - r0) * T
            # pinned[k] no longer read by an earlier transfer (this call's or the previous
            # call's; an event never recorded returns at once)
            self.h2d_done[k].synchronize()
            dst = self.pinned[k].numpy()[:n].reshape(r1 - r0, T)
            src = host[r0:r1]
            edges = np.linspace(0, r1 - r0, th + 1).astype(np.int64)
            list(self.pool.map(lambda i: np.copyto(dst[edges[i]:edges[i + 1]],
                                                   src[edges[i]:edges[i + 1]],
                                                   casting="same_kind"), range(th)))
            self.copy_stream.wait_event(self.k1_done[k])   # ring[k] consumed by its K1
            with torch.cuda.stream(self.copy_stream):
                self.ring[k][:n].copy_(self.pinned[k][:n], non_blocking=True)
                self.h2d_done[k].record(self.copy_stream)
            main.wait_event(self.h2d_done[k])
            plan.run(self.ring[k][:n].view(r1 - r0, T), out[:, r0:r1], main)
            self.k1_done[k].record(main)


_STAGERS: dict = {}


def temporal_peers(plan: "TemporalPlan", hist: torch.Tensor, peers, stream=None) -> None:
    """K1 of this rank's traces with the slice all-gather fused into its store
    (``distributed.PeerSlices``): hist float32 [n_traces, T] of the rank's detectors."""
    _lib.call("pf_temporal_dft_peers", dev.ptr(hist), hist.shape[0], plan.n_bins,
              dev.ptr(plan.bins), dev.ptr(plan.tw), dev.ptr(plan.wphase), plan.n_freq,
              plan.inner_mask, dev.ptr(peers.peers), peers.world, peers.peer_stride, peers.col,
              dev.stream_ptr(stream))


def to_frequency_device(histograms: torch.Tensor, kernel, t0: float = 0.0,
                        out: torch.Tensor | None = None, plan: TemporalPlan | None = None,
                        stream=None) -> torch.Tensor:
    """Device-resident K1: float32 [I, D, T] -> complex64 [F, I, D]."""
    _require(histograms.dim() == 3 and histograms.shape[2] == kernel.n_bins,
             "measurement and kernel disagree on the number of time bins")
    h = histograms if histograms.dtype == torch.float32 else histograms.float()
    h = h.contiguous()
    i_n, d_n, _ = h.shape
    plan = plan or TemporalPlan(kernel, t0, h.device)
    if out is None:
        out = torch.empty((plan.n_freq, i_n, d_n), dtype=torch.complex64, device=h.device)
    plan.run(h.view(i_n * d_n, -1), out.view(plan.n_freq, i_n * d_n), stream)
    return out


def to_frequency(measurement, kernel) -> DeviceFrequencySlices:
    """GPU drop-in for reference ``to_frequency`` (phasor.py:107-127).

    ``coeff[p, c, k] = FFT(h[p, c])[b_k] * w_k * exp(-1j w_k t0)``.
    """
    _require(measurement.n_bins == kernel.n_bins,
             "measurement and kernel disagree on the number of time bins")
    _require(math.isclose(measurement.delta_t, kernel.delta_t, rel_tol=1e-12),
             "measurement and kernel disagree on the bin width")
    device = dev.require_cuda()
    h = measurement.histograms
    plan = _plan_for(kernel, float(measurement.t0), device)
    if isinstance(h, torch.Tensor):
        ht = h.to(device=device, dtype=torch.float32)
        coeff = to_frequency_device(ht, kernel, float(measurement.t0), plan=plan)
    else:
        # host payload: staged through pinned chunks straight into K1 (no device copy of
        # the whole capture, no pageable transfer)
        host = np.asarray(h)
        i_n, d_n, t_n = host.shape
        host2 = host.reshape(i_n * d_n, t_n)
        if not host2.flags.c_contiguous:
            host2 = np.ascontiguousarray(host2)
        coeff = torch.empty((plan.n_freq, i_n, d_n), dtype=torch.complex64, device=device)
        st = _STAGERS.get(str(device))
        if st is None:
            st = _STAGERS[str(device)] = _HostStager(device)
        st.run(host2, plan, coeff.view(plan.n_freq, i_n * d_n))
    return DeviceFrequencySlices(kernel.frequencies, coeff, measurement.relay,
                                 measurement.illuminations)


def lateral_resolution(lambda_c: float, z: float, aperture: float) -> float:
    """Diffraction-limited lateral resolution ``1.22 lambda_c z / aperture``
    (reference phasor.py:130-134)."""
    _require(lambda_c > 0 and z > 0 and aperture > 0, "wavelength, depth, and aperture must be > 0")
    return 1.22 * lambda_c * z / aperture
