"""NLS1 containers against files written by the reference.

The fixtures under tests/golden/nls1 were produced by the reference's own
writers (tests/golden/make_golden.py, ``gen_containers``): our readers must
parse them and our writers must reproduce them byte for byte.
"""
import os
import shutil
import struct

import numpy as np
import pytest
import torch

from paper_2501_05244_b200 import container as K
from paper_2501_05244_b200.core import (ContainerFormatError, InvalidMagicError,
                                        NonFiniteDataError, TruncatedPayloadError,
                                        UnsupportedVersionError, ValidationError)

D = os.path.join(os.path.dirname(__file__), "golden", "nls1")
DATASETS = ["uniform", "planar", "nonplanar"]
VOLUMES = ["cuboid", "frustum", "explicit", "video"]


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


@pytest.mark.parametrize("name", DATASETS)
def test_dataset_roundtrip_is_byte_identical(tmp_path, name):
    src = os.path.join(D, f"dataset_{name}.nls1")
    m = K.read_dataset(src)
    assert m.histograms.dtype == np.float32
    out = str(tmp_path / "d.nls1")
    K.write_dataset(m, out)
    assert _bytes(out) == _bytes(src)
    assert _bytes(out + ".json") == _bytes(src + ".json")


@pytest.mark.parametrize("name", VOLUMES)
def test_volume_roundtrip_is_byte_identical(tmp_path, name):
    src = os.path.join(D, f"volume_{name}.nls1")
    v = K.read_volume(src)
    out = str(tmp_path / "v.nls1")
    K.write_volume(v, out)
    assert _bytes(out) == _bytes(src)
    # the raw complex64 tensor path writes the same bytes
    field = v.field if v.times is not None else v.field[None, :]
    out2 = str(tmp_path / "v2.nls1")
    K.write_volume(torch.from_numpy(field.astype(np.complex64)), out2, grid=v.grid, times=v.times)
    assert _bytes(out2) == _bytes(src)


def test_reader_errors(tmp_path):
    src = _bytes(os.path.join(D, "dataset_uniform.nls1"))
    cases = {
        "magic": (b"XLS1" + src[4:], InvalidMagicError, "magic"),
        "version": (src[:4] + struct.pack("<I", 2) + src[8:], UnsupportedVersionError, "version"),
        "trunc": (src[:-5], TruncatedPayloadError, "file ends"),
    }
    for key, (data, exc, msg) in cases.items():
        p = tmp_path / f"{key}.nls1"
        p.write_bytes(data)
        with pytest.raises(exc, match=msg):
            K.read_dataset(str(p))
    # a volume file is not a dataset and vice versa
    with pytest.raises(ContainerFormatError, match="volume file"):
        K.read_dataset(os.path.join(D, "volume_cuboid.nls1"))
    with pytest.raises(ContainerFormatError, match="not a volume grid"):
        K.read_volume(os.path.join(D, "dataset_uniform.nls1"))
    # NaN in the payload
    hist_off = len(src) - 4 * 2 * 12 * 8
    bad = bytearray(src)
    bad[hist_off:hist_off + 4] = struct.pack("<f", float("nan"))
    p = tmp_path / "nan.nls1"
    p.write_bytes(bytes(bad))
    with pytest.raises(NonFiniteDataError):
        K.read_dataset(str(p))


def test_raw_volume_needs_grid():
    with pytest.raises(ValidationError):
        K.write_volume(torch.zeros(4, dtype=torch.complex64), "/dev/null")


@pytest.mark.gpu
@pytest.mark.parametrize("name", DATASETS)
def test_dataset_to_device_matches_host_read(name, monkeypatch):
    src = os.path.join(D, f"dataset_{name}.nls1")
    monkeypatch.setattr(K, "CHUNK_BYTES", 64)       # many chunks: exercise the double buffer
    md = K.read_dataset_device(src)
    mh = K.read_dataset(src)
    assert md.histograms.is_cuda and md.histograms.dtype == torch.float32
    assert np.array_equal(md.histograms.cpu().numpy(), mh.histograms)
    assert (md.delta_t, md.t0, md.relay.count) == (mh.delta_t, mh.t0, mh.relay.count)


@pytest.mark.gpu
def test_device_read_rejects_nan_and_negative(tmp_path):
    src = _bytes(os.path.join(D, "dataset_uniform.nls1"))
    hist_off = len(src) - 4 * 2 * 12 * 8
    for val, exc in ((float("inf"), NonFiniteDataError), (-1.0, ValidationError)):
        bad = bytearray(src)
        bad[hist_off + 40:hist_off + 44] = struct.pack("<f", val)
        p = tmp_path / "bad.nls1"
        p.write_bytes(bytes(bad))
        with pytest.raises(exc):
            K.read_dataset_device(str(p))


@pytest.mark.gpu
def test_device_dataset_through_to_frequency_and_volume_writer(tmp_path):
    """File -> device -> K1 -> rsd -> device volume -> file, against the oracle."""
    import paper_2501_05244_b200 as pf
    from oracle import pf_oracle as O
    from paper_2501_05244_b200.core import TransientMeasurement
    from paper_2501_05244_b200.reconstruct import RsdEngine
    rng = np.random.default_rng(11)
    g = pf.UniformGrid2D(16, 16, 0.05, 0.05, -0.375, -0.375, 0.0)
    ill = pf.PointList(np.array([[0.0, 0.0]]))
    hist = rng.poisson(2.0, size=(1, 256, 1024)).astype(np.float32)
    m = TransientMeasurement(pf.UniformRelay(g), ill, hist, 8e-12, 1e-9)
    src = str(tmp_path / "cap.nls1")
    K.write_dataset(m, src)
    md = K.read_dataset_device(src)
    assert torch.equal(md.histograms.cpu(), torch.from_numpy(hist))
    k = pf.build_kernel(0.06, md.n_bins, md.delta_t)
    sl = pf.to_frequency(md, k)
    ref = O.to_frequency(hist.astype(np.float64), np.asarray(k.bin_indices),
                         np.asarray(k.frequencies), np.asarray(k.weights), m.t0)
    assert O.rel_l2(np.asarray(sl.coefficients), ref) < 1e-5
    grid = pf.CuboidGrid(pf.UniformGrid3D(16, 16, 2, 0.05, 0.05, 0.2, g.x0, g.y0, 0.5))
    vol = RsdEngine(sl, grid).run(pf.phasor.device_coefficients(sl))
    out = str(tmp_path / "vol.nls1")
    K.write_volume(vol, out, grid=grid)
    back = K.read_volume(out)
    assert np.array_equal(back.field, vol[0].cpu().numpy().astype(np.complex128))
    host = pf.rsd(sl, grid)
    assert O.rel_l2(back.field, host.field) < 1e-6
