"""ctypes binding of ``libpfgpu.so`` (the C-ABI declared in ``include/pfgpu.h``).

The shared library is built in-tree by ``paper_2501_05244_b200.build`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no CPU fallback: if the
library or a CUDA device is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpfgpu.so")

PF_MAX_STAGES = 24


class PfFftPlan(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("nst", ctypes.c_int),
                ("radix", ctypes.c_int * PF_MAX_STAGES), ("tw", ctypes.c_void_p)]


class PfPlane(ctypes.Structure):
    _fields_ = [("dz", ctypes.c_double), ("lag_dx", ctypes.c_double), ("lag_dy", ctypes.c_double),
                ("x0", ctypes.c_double), ("dx", ctypes.c_double), ("y0", ctypes.c_double),
                ("dy", ctypes.c_double), ("z", ctypes.c_double), ("uhat_off", ctypes.c_int64),
                ("vol_plane", ctypes.c_int64)]


class PfPropGeom(ctypes.Structure):
    _fields_ = [("px", ctypes.c_int), ("py", ctypes.c_int), ("nx", ctypes.c_int),
                ("ny", ctypes.c_int), ("nu0x", ctypes.c_int), ("nu0y", ctypes.c_int),
                ("n_illum", ctypes.c_int), ("include_illum", ctypes.c_int),
                ("flags", ctypes.c_int), ("reserved", ctypes.c_int),
                ("uhat_illum_stride", ctypes.c_int64)]


class PfNufftGeom(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("w", ctypes.c_int), ("mr", ctypes.c_int * 3),
                ("m", ctypes.c_int * 3), ("h", ctypes.c_float * 3),
                ("inv4tau", ctypes.c_float * 3), ("tile", ctypes.c_int * 3),
                ("ntiles", ctypes.c_int * 3), ("window", ctypes.c_int), ("beta", ctypes.c_float),
                ("inv_hw", ctypes.c_float * 3)]


class PfRsdArgs(ctypes.Structure):
    _fields_ = [("relay_nx", ctypes.c_int), ("relay_ny", ctypes.c_int),
                ("relay_dx", ctypes.c_double), ("relay_dy", ctypes.c_double),
                ("relay_x0", ctypes.c_double), ("relay_y0", ctypes.c_double),
                ("relay_z", ctypes.c_double),
                ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double),
                ("x0", ctypes.c_double), ("y0", ctypes.c_double), ("z0", ctypes.c_double),
                ("n_freq", ctypes.c_int), ("n_illum", ctypes.c_int),
                ("frequencies", ctypes.c_void_p), ("ill_xyz", ctypes.c_void_p),
                ("n_frames", ctypes.c_int), ("times", ctypes.c_void_p),
                ("padding_none", ctypes.c_int), ("include_illum", ctypes.c_int)]


class PfSrsdArgs(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int),
                ("relay_dx", ctypes.c_double), ("relay_dy", ctypes.c_double),
                ("relay_x0", ctypes.c_double), ("relay_y0", ctypes.c_double),
                ("relay_z", ctypes.c_double), ("nz", ctypes.c_int),
                ("zs", ctypes.c_void_p), ("alphas", ctypes.c_void_p), ("betas", ctypes.c_void_p),
                ("n_freq", ctypes.c_int), ("n_illum", ctypes.c_int),
                ("frequencies", ctypes.c_void_p), ("ill_xyz", ctypes.c_void_p),
                ("n_frames", ctypes.c_int), ("times", ctypes.c_void_p),
                ("include_illum", ctypes.c_int)]


class PfNursd1Args(ctypes.Structure):
    _fields_ = [("n_points", ctypes.c_int), ("relay_xy", ctypes.c_void_p),
                ("relay_z", ctypes.c_double), ("nx", ctypes.c_int), ("ny", ctypes.c_int),
                ("nz", ctypes.c_int), ("dx", ctypes.c_double), ("dy", ctypes.c_double),
                ("dz", ctypes.c_double), ("x0", ctypes.c_double), ("y0", ctypes.c_double),
                ("z0", ctypes.c_double), ("n_freq", ctypes.c_int), ("n_illum", ctypes.c_int),
                ("frequencies", ctypes.c_void_p), ("ill_xyz", ctypes.c_void_p),
                ("n_frames", ctypes.c_int), ("times", ctypes.c_void_p),
                ("eps", ctypes.c_double), ("include_illum", ctypes.c_int)]


class PfNursd2Args(ctypes.Structure):
    _fields_ = [("relay_nx", ctypes.c_int), ("relay_ny", ctypes.c_int),
                ("relay_dx", ctypes.c_double), ("relay_dy", ctypes.c_double),
                ("relay_x0", ctypes.c_double), ("relay_y0", ctypes.c_double),
                ("relay_z", ctypes.c_double), ("n_planes", ctypes.c_int),
                ("plane_z", ctypes.c_void_p), ("plane_count", ctypes.c_void_p),
                ("voxel_xy", ctypes.c_void_p), ("n_freq", ctypes.c_int),
                ("n_illum", ctypes.c_int), ("frequencies", ctypes.c_void_p),
                ("ill_xyz", ctypes.c_void_p), ("n_frames", ctypes.c_int),
                ("times", ctypes.c_void_p), ("eps", ctypes.c_double),
                ("include_illum", ctypes.c_int)]


_vp, _i, _i64, _d, _f = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_float
_P = ctypes.POINTER

# name -> argtypes (restype int unless listed in _RESTYPES)
_SIGNATURES = {
    "pf_version": [],
    "pf_last_error": [ctypes.c_char_p, ctypes.c_size_t],
    "pf_launch_count": [],
    "pf_temporal_dft": [_vp, _i64, _i, _vp, _vp, _vp, _i, _vp, _i64, ctypes.c_uint64, _vp],
    "pf_temporal_dft_direct": [_vp, _i64, _i, _vp, _vp, _vp, _i, _vp, _i64, _vp],
    "pf_fft_lines": [_vp, _P(PfFftPlan), _i64, _i64, _i64, _i64, _i64, _i, _f, _vp],
    "pf_fft_lines3": [_vp, _P(PfFftPlan), _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i, _f, _vp],
    "pf_embed_centered": [_vp, _i64, _i, _i, _i64, _vp, _i, _i, _i, _vp],
    "pf_prop_fast": [_P(PfPropGeom)],
    "pf_rsd_workspace_bytes": [_P(PfRsdArgs)],
    "pf_crop_centered": [_vp, _i64, _i, _i, _vp, _i, _i, _vp],
    "pf_rsd": [_P(PfRsdArgs), _vp, _vp, _vp, _i64, _vp],
    "pf_srsd_workspace_bytes": [_P(PfSrsdArgs)],
    "pf_srsd": [_P(PfSrsdArgs), _vp, _vp, _vp, _i64, _vp],
    "pf_nursd1_workspace_bytes": [_P(PfNursd1Args)],
    "pf_nursd1": [_P(PfNursd1Args), _vp, _vp, _vp, _i64, _vp],
    "pf_nursd2_workspace_bytes": [_P(PfNursd2Args)],
    "pf_nursd2": [_P(PfNursd2Args), _vp, _vp, _vp, _i64, _vp],
    "pf_nufft_type1_finish_pow2": [_P(PfNufftGeom), _vp, _i64, _i, _vp, _P(PfFftPlan),
                                   _P(PfFftPlan), _vp, _vp, _vp, _i64, _vp],
    "pf_relay_spectra_fast": [_vp, _i64, _i, _i, _i64, _vp, _i, _P(PfFftPlan), _vp],
    "pf_prop_ws_a": [_P(PfPropGeom), _i],
    "pf_prop_ws_b": [_P(PfPropGeom), _i],
    "pf_prop_kernel_rows": [_vp, _i, _d, _P(PfPropGeom), _P(PfFftPlan), _vp, _vp],
    "pf_prop_columns": [_vp, _i, _P(PfPropGeom), _P(PfFftPlan), _vp, _vp, _vp, _i, _vp],
    "pf_prop_ws_spectrum": [_P(PfPropGeom), _i],
    "pf_prop_fbatch": [_vp, _i, _vp, _i, _P(PfPropGeom), _P(PfFftPlan), _vp, _i64, _vp, _i64, _vp,
                       _i64, _vp, _vp, _vp, _vp],
    "pf_prop_fbatch_generic": [_vp, _i, _vp, _i, _P(PfPropGeom), _P(PfFftPlan), _P(PfFftPlan),
                               _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp],
    "pf_prop_onchip_ok": [_P(PfPropGeom)],
    "pf_prop_fbatch_onchip": [_vp, _i, _vp, _i, _P(PfPropGeom), _vp, _i64, _vp, _vp, _vp, _vp,
                              _i, _i, _vp],
    "pf_count_nonfinite": [_vp, _i64, _vp, _vp],
    "pf_fp32_probe": [_vp, _i, _i, _vp],
    "pf_nufft_interp_mode": [_i],
    "pf_nufft_window": [_i],
    "pf_nufft_interp": [_P(PfNufftGeom), _vp, _vp, _i, _vp, _vp, _vp],
    "pf_nufft_interp2_batch": [_P(PfNufftGeom), _vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _i64, _i64,
                               _i, _vp, _d, _i, _f, _vp, _i, _vp, _i64, _vp],
    "pf_nufft_interp2_nodes": [_P(PfNufftGeom), _vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _i64, _i64,
                               _i, _vp, _d, _i, _f, _vp, _i, _vp, _i64, _i, _vp, _vp],
    "pf_scatter_csr": [_vp, _vp, _vp, _vp, _i, _vp, _i64, _i, _vp, _i64, _vp],
    "pf_bluestein_lines": [_vp, _i64, _i64, _i64, _i, _i, _vp, _i64, _i64, _i64, _i, _i, _i, _i,
                           _P(PfFftPlan), _vp, _vp, _vp],
    "pf_bluestein_warp": [_i, _vp, _i64, _i64, _i, _i, _vp, _i64, _i64, _i, _i, _i, _P(PfFftPlan),
                          _vp, _vp, _vp],
    "pf_nufft_spread": [_P(PfNufftGeom), _vp, _vp, _vp, _vp, _vp, _i64, _i, _vp, _i64, _vp],
    "pf_nufft_deconv": [_P(PfNufftGeom), _vp, _i64, _vp, _vp, _vp, _i, _vp, _i64, _i, _vp],
    "pf_nufft_type2_start_2d": [_P(PfNufftGeom), _vp, _i64, _vp, _vp, _i, _vp, _i64, _P(PfFftPlan), _P(PfFftPlan), _vp],
    "pf_nufft_type2_start_2d_win": [_P(PfNufftGeom), _vp, _i64, _vp, _vp, _i, _vp, _i64, _P(PfFftPlan), _P(PfFftPlan), _i, _i, _i, _i, _vp],
    "pf_nufft_type2_start_2d_il": [_P(PfNufftGeom), _vp, _i64, _vp, _vp, _i, _vp, _i64, _P(PfFftPlan), _P(PfFftPlan), _i, _i, _i, _i, _vp, _i, _vp],
    "pf_nufft_type2_il_ok": [_P(PfNufftGeom)],
    "pf_nufft_type2_start_2d_ilm": [_P(PfNufftGeom), _vp, _i64, _vp, _vp, _i, _vp, _i64, _P(PfFftPlan), _P(PfFftPlan), _i, _i, _i, _i, _vp, _i, _i, _vp],
    "pf_nufft_interp2_freqs": [_P(PfNufftGeom), _vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _i64, _i64, _i, _vp, _vp, _i, _f, _vp, _vp, _vp],
    "pf_nufft_interp2_nodes_il": [_P(PfNufftGeom), _vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _i64, _vp, _d, _i, _f, _vp, _i, _vp, _i64, _i, _vp, _vp],
    "pf_nufft_place": [_P(PfNufftGeom), _vp, _i64, _vp, _vp, _vp, _i, _vp, _i64, _i, _vp],
    "pf_nufft_interp2_acc": [_P(PfNufftGeom), _vp, _vp, _vp, _i, _vp, _i64, _i, _vp, _d, _i, _f,
                             _vp, _i, _vp, _i64, _i64, _vp, _vp],
    "pf_kernel3d": [_vp, _i, _i, _i, _d, _d, _d, _d, _vp],
    "pf_cmul": [_vp, _vp, _i64, _i64, _f, _vp],
    "pf_mirror_fill": [_vp, _i, _i, _i, _i, _i, _i, _i, _vp],
    "pf_cmul_even": [_vp, _vp, _i, _i, _i, _i, _i, _f, _vp],
    "pf_copy_planes": [_vp, _i, _i64, _i64, _i64, _vp, _vp],
    "pf_zslab": [_vp, _i, _i, _i64, _vp, _f, _vp, _vp],
    "pf_roll": [_vp, _vp, _i64, _i, _i, _i, _i, _i, _i, _vp],
    "pf_prop_rows_out_horner": [_vp, _i, _d, _d, _i, _P(PfPropGeom), _P(PfFftPlan), _vp, _vp,
                                _vp, _vp, _vp, _d, _vp, _vp],
    "pf_temporal_dft_peers": [_vp, _i64, _i, _vp, _vp, _vp, _i, ctypes.c_uint64, _vp, _i,
                              _i64, _i64, _vp],
    "pf_ipc_handle": [_vp, _vp, _P(ctypes.c_int64)],
    "pf_ipc_open": [_vp, _i64, _P(ctypes.c_void_p)],
    "pf_ipc_close": [_vp],
    "pf_prop_rows_out": [_vp, _i, _d, _P(PfPropGeom), _P(PfFftPlan), _vp, _vp, _vp, _i, _vp,
                         _i64, _vp],
}
_RESTYPES = {"pf_launch_count": ctypes.c_int64, "pf_prop_ws_a": ctypes.c_int64, "pf_prop_ws_b": ctypes.c_int64,
             "pf_prop_ws_spectrum": ctypes.c_int64, "pf_rsd_workspace_bytes": ctypes.c_int64,
             "pf_srsd_workspace_bytes": ctypes.c_int64, "pf_nursd1_workspace_bytes": ctypes.c_int64,
             "pf_nursd2_workspace_bytes": ctypes.c_int64,
             "pf_prop_fast": ctypes.c_int, "pf_prop_onchip_ok": ctypes.c_int,
             "pf_nufft_interp_mode": ctypes.c_int, "pf_nufft_window": ctypes.c_int, "pf_nufft_type2_il_ok": ctypes.c_int}

_lib = None



def launches() -> int:
    """Kernels libpfgpu has launched in this process (native counter, one per launch
    site that ran; a launch captured into a CUDA graph counts once, at capture)."""
    return int(load().pf_launch_count())


class PfError(RuntimeError):
    """A libpfgpu call failed (argument or CUDA error)."""


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def load(path: str = LIB_PATH):
    """Load the library (no device needed) and bind every declared entry point."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise PfError(f"libpfgpu.so not built at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    for name, args in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    _lib = lib
    return lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    load().pf_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def call(name: str, *args) -> int:
    rc = getattr(load(), name)(*args)
    if name in _RESTYPES:
        return rc
    if rc != 0:
        raise PfError(f"{name} failed ({rc}): {last_error()}")
    return rc
