"""Rebuild slices / grids from the golden ``.npz`` fixtures into the engine's types."""

from __future__ import annotations

import os

import numpy as np

from paper_2501_05244_b200 import core

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))


def relay_from(d, prefix="relay"):
    kind = str(d[f"{prefix}_kind"])
    if kind == "uniform":
        nx, ny, dx, dy, x0, y0, z = d[f"{prefix}_grid"]
        return core.UniformRelay(core.UniformGrid2D(int(nx), int(ny), dx, dy, x0, y0, z))
    if kind == "nonuniform_planar":
        return core.NonUniformPlanarRelay(core.PointList(d[f"{prefix}_points"]),
                                          float(d[f"{prefix}_z"]))
    return core.NonPlanarRelay(core.PointList(d[f"{prefix}_points"]))


def slices_from(d):
    return core.FrequencySlices(d["frequencies"], d["coefficients"], relay_from(d),
                                core.PointList(d["illuminations"]))


def grid_from(d):
    kind = str(d["grid_kind"])
    if kind == "cuboid":
        nx, ny, nz, dx, dy, dz, x0, y0, z0 = d["grid_cuboid"]
        return core.CuboidGrid(core.UniformGrid3D(int(nx), int(ny), int(nz), dx, dy, dz,
                                                  x0, y0, z0))
    if kind == "frustum":
        nx, ny, dx, dy, x0, y0, z = d["grid_base"]
        base = core.UniformGrid2D(int(nx), int(ny), dx, dy, x0, y0, z)
        return core.FrustumGrid(base, d["grid_zs"], d["grid_alphas"], d["grid_betas"])
    planes, s = [], 0
    for z, n in zip(d["grid_plane_z"], d["grid_plane_n"]):
        planes.append(core.VoxelPlane(float(z), core.PointList(d["grid_points"][s:s + int(n)])))
        s += int(n)
    return core.ExplicitVoxels(tuple(planes))


REC_CASES = [
    "rsd_small", "rsd_small_noill", "rsd_full16", "rsd_none16", "rsd_video", "chain_rsd",
    "chain_srsd_unit", "chain_srsd_08", "chain_nursd1", "chain_nursd2", "chain_nursd3",
    "chain_hybrid", "chain_nursd3d_flat", "nursd1_random", "nursd2_random", "nursd3_random",
    "hybrid_random", "srsd_linear16", "srsd_aniso16", "nursd3d_curved", "rsd_odd", "rsd_odd_none",
    "rsd3d_curved_tri", "rsd3d_curved_near",
]


def case_call(name):
    """(algorithm, kwargs) the golden case was generated with (see make_golden.py)."""
    table = {
        "rsd_small": ("rsd", {}),
        "rsd_small_noill": ("rsd", {"include_illumination": False}),
        "rsd_full16": ("rsd", {}),
        "rsd_none16": ("rsd", {"padding": "none"}),
        "rsd_video": ("rsd", {"times": "times"}),
        "chain_rsd": ("rsd", {}),
        "chain_srsd_unit": ("srsd", {}),
        "chain_srsd_08": ("srsd", {}),
        "chain_nursd1": ("nursd1", {"eps": 1e-8}),
        "chain_nursd2": ("nursd2", {"eps": 1e-8}),
        "chain_nursd3": ("nursd3", {"eps": 1e-8, "lattice_pitch": 0.02}),
        "chain_hybrid": ("srsd-nursd2", {"alpha": 1.0, "eps": 1e-8}),
        "chain_nursd3d_flat": ("nursd3d", {"eps": 1e-8}),
        "nursd1_random": ("nursd1", {"eps": 1e-6}),
        "nursd2_random": ("nursd2", {"eps": 1e-6}),
        "nursd3_random": ("nursd3", {"eps": 1e-6}),
        "hybrid_random": ("srsd-nursd2", {"alpha": 0.7, "beta": 0.55, "eps": 1e-6}),
        "srsd_linear16": ("srsd", {}),
        "srsd_aniso16": ("srsd", {}),
        "nursd3d_curved": ("nursd3d", {"eps": 1e-6}),
        "rsd_odd": ("rsd", {}),
        "rsd_odd_none": ("rsd", {"padding": "none"}),
        "rsd3d_curved_tri": ("rsd3d", {"scatter": "trilinear"}),
        "rsd3d_curved_near": ("rsd3d", {"scatter": "nearest"}),
    }
    return table[name]
