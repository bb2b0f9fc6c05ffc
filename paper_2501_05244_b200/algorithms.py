"""SRSD / NURSD family on the GPU (filled in next)."""

from __future__ import annotations


def _todo(*a, **k):
    raise NotImplementedError("not yet ported to the GPU engine")


srsd = nursd1 = nursd2 = nursd3 = nursd3d = srsd_nursd2 = rsd3d = _todo
