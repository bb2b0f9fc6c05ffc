"""Process-parallel CPU oracle (TEST INFRASTRUCTURE: the full-size parity tests and the
reference arm of bench.py; never imported by the product package).

The float64 oracle (``oracle/pf_oracle.py``) computes every (frequency, plane) unit
independently, so a full BASELINE-size volume is split across the host cores:

* ``oracle_planes``: contiguous depth-plane blocks, one oracle call per block with
  ``plane_range``; the blocks are concatenated in plane order.  Each block's voxels see
  exactly the arithmetic of the unsplit call (per-plane work never mixes planes).
* ``oracle_freq_terms``: one oracle call per frequency on a single-frequency view of the
  slices; the caller adds the terms in ascending frequency order, which is the
  reference's own reduction (``reconstruct.py:163-168``, ``_reduce``), so the sum is the
  unsplit result bit for bit.

Workers are forked (the slices and grid are inherited, not pickled); they run numpy only
and never touch CUDA.
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from oracle import pf_oracle as O

_STATE: dict = {}


def n_procs() -> int:
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    return max(1, min(int(os.environ.get("PF_ORACLE_PROCS", n)), 64))


def _blocks(n: int, parts: int) -> list[tuple[int, int]]:
    base, rem = divmod(n, parts)
    out, lo = [], 0
    for i in range(parts):
        hi = lo + base + (1 if i < rem else 0)
        if hi > lo:
            out.append((lo, hi))
        lo = hi
    return out


def _plane_block(task):
    name, lo, hi, kw = task
    fn = getattr(O, name)
    return lo, np.asarray(fn(_STATE["slices"], _STATE["grid"], plane_range=(lo, hi), **kw))


def oracle_planes(name: str, slices, grid, n_planes: int, procs: int | None = None,
                  blocks_per_proc: int = 1, **kw) -> np.ndarray:
    """``O.<name>(slices, grid, **kw)`` over all ``n_planes`` planes, flattened [V]."""
    procs = procs or n_procs()
    tasks = [(name, lo, hi, kw) for lo, hi in _blocks(n_planes, procs * blocks_per_proc)]
    _STATE.update(slices=slices, grid=grid)
    try:
        with mp.get_context("fork").Pool(min(procs, len(tasks))) as pool:
            res = pool.map(_plane_block, tasks, chunksize=1)
    finally:
        _STATE.clear()
    res.sort(key=lambda r: r[0])
    return np.concatenate([r[1].reshape(-1) for r in res])


class _OneFreq:
    """Single-frequency view of host slices (the reference FrequencySlices fields)."""

    def __init__(self, sl, fi):
        self.frequencies = np.asarray(sl.frequencies)[fi:fi + 1]
        self.coefficients = np.asarray(sl.coefficients)[:, :, fi:fi + 1]
        self.relay = sl.relay
        self.illuminations = sl.illuminations
        self.n_freq = 1
        self.shortest_wavelength = sl.shortest_wavelength


def _freq_term(task):
    name, fi, kw = task
    fn = getattr(O, name)
    view = _OneFreq(_STATE["slices"], fi)
    return fi, np.asarray(fn(view, *_STATE["args"], **kw))


def oracle_freq_terms(name: str, slices, args: tuple, procs: int | None = None,
                      **kw) -> np.ndarray:
    """Ascending-frequency sum of ``O.<name>(one-frequency view, *args, **kw)`` terms.

    Geometry that the reference derives from the whole frequency set (e.g. nursd3d's
    z pitch = shortest wavelength / 2) must be passed explicitly in ``kw``; the view
    also carries the full set's ``shortest_wavelength``."""
    procs = procs or n_procs()
    F = int(np.asarray(slices.frequencies).size)
    tasks = [(name, fi, kw) for fi in range(F)]
    _STATE.update(slices=slices, args=args)
    try:
        with mp.get_context("fork").Pool(min(procs, F)) as pool:
            res = pool.map(_freq_term, tasks, chunksize=1)
    finally:
        _STATE.clear()
    res.sort(key=lambda r: r[0])
    out = np.zeros_like(res[0][1])
    for _, term in res:
        out += term
    return out
