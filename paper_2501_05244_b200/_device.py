"""Device plumbing: CUDA checks, streams, FFT plans (radix choice + fp64 twiddle tables).

PyTorch is used only for device memory, streams and collectives; every
arithmetic kernel on the path lives in ``libpfgpu.so``.
"""

from __future__ import annotations

import contextlib
import ctypes
import math
import os

import numpy as np
import torch

from . import _lib
from ._fastlen import factorize


class DeviceUnavailable(RuntimeError):
    """No CUDA device / no built extension: the engine has no CPU fallback."""


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceUnavailable("paper_2501_05244_b200 needs a CUDA device (sm_100a); "
                                "there is no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor) -> int:
    return int(t.data_ptr())


def radices_for(n: int) -> list[int]:
    """Stage radices: powers of two merged into as few even stages as possible."""
    f = factorize(n)
    k = f.count(2)
    odd = [p for p in f if p != 2]
    pow2 = []
    if k:
        s = (k + 3) // 4
        bits = [k // s + (1 if i < k % s else 0) for i in range(s)]
        pow2 = [1 << b for b in bits]
    return pow2 + sorted(odd, reverse=True)


PF_MAX_STAGES = 24
PF_XFFT_TAG = 0x35F7     # include/pfgpu.h


def xfft_L(n: int) -> int:
    """Lanes of the mixed-radix register FFT for n = 35 L (xfft.cuh), else 0."""
    if n % 35:
        return 0
    L = n // 35
    return L if L in (4, 5, 8, 10, 15, 20, 30) else 0


def xfft_plan_L(n: int) -> int:
    """Lanes of the register FFT a plan of length n is tagged for (0: Stockham stages).
    PF_XFFT = "large" (default): only L >= 10 (n = 350, 525, 700, 1050), where it measured faster
    (config 2's 700-point fine-grid lines); "all": every 35 L length (slower at 140 and 280:
    the generic propagation kernels drop to one CTA per SM); an integer: L at least that;
    "0": never."""
    mode = os.environ.get("PF_XFFT", "large")
    L = xfft_L(n)
    if mode == "0":
        return 0
    lmin = 1 if mode == "all" else (int(mode) if mode.isdigit() else 10)
    return L if L >= lmin else 0


class FftPlan:
    """Mixed-radix plan for one length on one device (twiddles built in float64)."""

    def __init__(self, n: int, device: torch.device):
        self.n = int(n)
        rad = radices_for(self.n) if self.n > 1 else []
        m = np.arange(self.n, dtype=np.float64)
        w = np.exp(-2j * np.pi * m / self.n)
        if self.n in (128, 256, 512, 1024):
            # register-FFT twiddles laid out k1-major ([k1][t], n = 32 L) right after
            # the unit-root table, so a warp's 32 lanes read one contiguous run
            L = self.n // 32
            k1 = np.arange(32)[:, None]
            t = np.arange(L)[None, :]
            w = np.concatenate([w, np.exp(-2j * np.pi * ((k1 * t) % self.n) / self.n).ravel()])
        xl = xfft_plan_L(self.n)
        if xl:
            # mixed-radix register FFT (n = 35 L): k1-major table [35][L] after the roots
            k1 = np.arange(35)[:, None]
            t = np.arange(xl)[None, :]
            w = np.concatenate([w, np.exp(-2j * np.pi * ((k1 * t) % self.n) / self.n).ravel()])
        self.tw = torch.from_numpy(w.astype(np.complex64)).to(device)
        self.c = _lib.PfFftPlan()
        self.c.n = self.n
        self.c.nst = len(rad)
        for i, r in enumerate(rad):
            self.c.radix[i] = r
        self.c.tw = ctypes.c_void_p(ptr(self.tw))
        if xl:
            self.c.radix[PF_MAX_STAGES - 1] = PF_XFFT_TAG

    @property
    def ref(self):
        return ctypes.byref(self.c)


_PLANS: dict[tuple[int, int], FftPlan] = {}


def fft_plan(n: int, device: torch.device) -> FftPlan:
    key = (int(n), device.index or 0)
    p = _PLANS.get(key)
    if p is None:
        p = FftPlan(n, device)
        _PLANS[key] = p
    return p


def fft_lines(data: torch.Tensor, n: int, nlines: int, inner: int, inner_stride: int,
              outer_stride: int, elem_stride: int, direction: int, scale: float = 1.0,
              stream=None) -> None:
    plan = fft_plan(n, data.device)
    _lib.call("pf_fft_lines", ptr(data), plan.ref, nlines, inner, inner_stride, outer_stride,
              elem_stride, direction, scale, stream_ptr(stream))


def fft2_natural(buf: torch.Tensor, ny: int, nx: int, nbatch: int, direction: int,
                 scale: float = 1.0, stream=None) -> None:
    """In-place 2D FFT of ``nbatch`` contiguous [ny, nx] c64 planes (natural order)."""
    if nx > 1:
        fft_lines(buf, nx, nbatch * ny, 1, 0, nx, 1, direction, 1.0, stream)
    if ny > 1:
        fft_lines(buf, ny, nbatch * nx, nx, 1, ny * nx, nx, direction, scale, stream)
    elif scale != 1.0:
        buf.mul_(scale)


def fftn_natural(buf: torch.Tensor, shape: tuple[int, ...], nbatch: int, direction: int,
                 scale: float = 1.0, stream=None) -> None:
    """In-place N-D FFT (N = 1..3) of ``nbatch`` contiguous arrays of ``shape``."""
    total = int(np.prod(shape))
    d = len(shape)
    done_scale = False
    for ax in range(d - 1, -1, -1):
        n = shape[ax]
        if n == 1:
            continue
        inner = int(np.prod(shape[ax + 1:])) if ax + 1 < d else 1
        outer_block = inner * n
        nlines = nbatch * total // n
        s = scale if not done_scale else 1.0
        done_scale = True
        if inner == 1:
            fft_lines(buf, n, nlines, 1, 0, n, 1, direction, s, stream)
        else:
            fft_lines(buf, n, nlines, inner, 1, outer_block, inner, direction, s, stream)
    if not done_scale and scale != 1.0:
        buf.mul_(scale)


def kept_ranges(m: int, mr: int) -> list[tuple[int, int]]:
    """Natural slots on a length-mr axis holding the centred modes [-m//2, m - m//2):
    (start, length) runs (reference NufftPlan.slots, spectral.py:287-295)."""
    if m >= mr:
        return [(0, mr)]
    return [(0, m - m // 2), (mr - m // 2, m // 2)] if m // 2 else [(0, m - m // 2)]


def fftn_pruned(buf: torch.Tensor, shape: tuple[int, ...], nbatch: int, direction: int,
                kept: list, outputs: bool, stream=None, nonzero: list | None = None) -> None:
    """In-place 2D/3D FFT of ``nbatch`` contiguous arrays computing only the lines a
    NUFFT needs.  ``kept[a]``: (start, length) runs of the kept slots on axis a.
    outputs=True (type 1, forward): only kept outputs are read afterwards, so an axis
    is transformed only along lines whose already-transformed coordinates are kept.
    outputs=False (type 2, inverse): the input is zero off the kept slots, so an axis
    is transformed only along lines whose not-yet-transformed coordinates are kept
    (the other lines are zero and stay zero).  Axes run last to first, as in
    ``fftn_natural``; line sets map onto pf_fft_lines' (inner, istr, ostr) indexing.
    ``nonzero[a]`` (outputs=True only): runs of the slots of axis a that can be nonzero on
    input (the cells a type-1 spreading touched); lines through all-zero slots of a
    not-yet-transformed axis are zero and stay zero, so they are skipped as well."""
    d = len(shape)
    assert d in (2, 3)
    strides = [int(np.prod(shape[a + 1:])) for a in range(d)]
    total = int(np.prod(shape))
    base = ptr(buf)

    def run(off, n, nl, inner, istr, ostr, estr):
        if nl > 0:
            _lib.call("pf_fft_lines", base + 8 * off, fft_plan(n, buf.device).ref, nl, inner,
                      istr, ostr, estr, direction, 1.0, stream_ptr(stream))

    for ax in range(d - 1, -1, -1):
        n = shape[ax]
        if n == 1:
            continue
        others = [a for a in range(d) if a != ax]
        full = [(nonzero[a] if (outputs and nonzero is not None) else [(0, shape[a])])
                for a in range(d)]
        runs = [kept[a] if (a > ax) == outputs else full[a] for a in others]
        if d == 2:
            (o,) = others
            for s0, ln in runs[0]:
                # lines along the other axis o, batches folded in with stride `total`
                run(s0 * strides[o], n, nbatch * ln, ln, strides[o], total, strides[ax])
            continue
        oa, ia = others
        for so, lo in runs[0]:
            for si, li in runs[1]:
                # the block's lines of every array of the batch in one launch: inner run on
                # axis ia, middle run on axis oa, outer level = the batch
                if lo > 0 and li > 0:
                    _lib.call("pf_fft_lines3", base + 8 * (so * strides[oa] + si * strides[ia]),
                              fft_plan(n, buf.device).ref, nbatch * lo * li, li, strides[ia], lo,
                              strides[oa], total, strides[ax], direction, 1.0, stream_ptr(stream))


def c64(t: torch.Tensor) -> torch.Tensor:
    """View a complex64 tensor; ensures contiguity."""
    assert t.dtype == torch.complex64
    return t.contiguous()


def phase_factors(omega: np.ndarray, times: np.ndarray) -> np.ndarray:
    """exp(1j w t) in float64, rounded to complex64 [F, n_frames]."""
    return np.exp(1j * np.outer(omega, times)).astype(np.complex64)


def pow2_ceil(x: int) -> int:
    return 1 << max(0, math.ceil(math.log2(max(1, x))))


@contextlib.contextmanager
def nvtx(name: str):
    """NVTX range around a host scope (pipeline stages show up named in a profiler's
    timeline; free when none is attached)."""
    torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()
