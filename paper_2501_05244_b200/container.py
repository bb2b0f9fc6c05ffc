"""NLS1 containers read straight into device memory and volumes written from it.

SURVEY §8(f) rank 2: the reference reads a transient dataset into host memory,
inflates the float32 payload to float64 (reference ``core.py:709-731``) and the
caller then copies it to wherever the transform runs.  Here the header is
parsed on the host, the float32 payload streams from the file through two
pinned staging buffers into a device tensor (disk read of chunk i+1 overlaps
the host->device copy of chunk i), and the NaN/inf and sign checks run on the
GPU (``pf_count_nonfinite``).  The volume writer takes the complex64 device
volume and produces the reference's container byte for byte
(``write_volume`` ``core.py:783-806``: same header, interleaved ``<c8``
payload), without the complex128 round trip.

File layout (little endian), shared by both container kinds:
``b"NLS1"``, u32 version=1, u32 x3 counts, f64 x2, u8 kind tag, kind-specific
geometry, then the payload.  Transient kind tags 0/1/2 (uniform, planar
points, 3D points); volume kind tags 16/17/18 (cuboid, frustum, explicit).
"""

from __future__ import annotations

import json
import struct

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .core import (ContainerFormatError, CuboidGrid, ExplicitVoxels, FrustumGrid,
                   InvalidMagicError, NonFiniteDataError, NonPlanarRelay, NonUniformPlanarRelay,
                   UnsupportedVersionError,
                   PointList, ReconstructionVolume, TransientMeasurement, TruncatedPayloadError,
                   UniformGrid2D, UniformGrid3D, UniformRelay, ValidationError, VoxelPlane)

MAGIC = b"NLS1"
VERSION = 1
RELAY_TAGS = {"uniform": 0, "nonuniform_planar": 1, "nonplanar": 2}
VOLUME_TAGS = {"cuboid": 16, "frustum": 17, "explicit": 18}
CHUNK_BYTES = 256 << 20


# ---------------------------------------------------------------- byte helpers
class _Cursor:
    """Sequential little-endian reader over a binary file object."""

    def __init__(self, f):
        self.f = f
        self.pos = 0
        f.seek(0, 2)
        self.size = f.tell()
        f.seek(0)

    def raw(self, n: int) -> bytes:
        if self.pos + n > self.size:
            raise TruncatedPayloadError(
                f"file ends at byte {self.size} but {self.pos + n} are needed")
        b = self.f.read(n)
        self.pos += n
        return b

    def fields(self, fmt: str):
        fmt = "<" + fmt
        return struct.unpack(fmt, self.raw(struct.calcsize(fmt)))

    def f64(self, count: int) -> np.ndarray:
        return np.frombuffer(self.raw(8 * count), dtype="<f8").astype(np.float64)


def _f64_bytes(a) -> bytes:
    return np.ascontiguousarray(a, dtype="<f8").tobytes()


def _preamble(c: _Cursor):
    magic = c.raw(4)
    if magic != MAGIC:
        raise InvalidMagicError(f"expected magic {MAGIC!r}, found {magic!r}")
    (version,) = c.fields("I")
    if version != VERSION:
        raise UnsupportedVersionError(f"container version {version} is not supported")


# ---------------------------------------------------------------- geometry codecs
def _relay_bytes(relay) -> bytes:
    parts = [struct.pack("<B", RELAY_TAGS[relay.kind])]
    if relay.kind == "uniform":
        g = relay.grid
        parts += [struct.pack("<II", g.nx, g.ny), struct.pack("<5d", g.dx, g.dy, g.x0, g.y0, g.z)]
    elif relay.kind == "nonuniform_planar":
        parts += [struct.pack("<d", relay.z), struct.pack("<I", relay.points.count),
                  _f64_bytes(relay.points.points)]
    else:
        parts += [struct.pack("<I", relay.points.count), _f64_bytes(relay.points.points)]
    return b"".join(parts)


def _relay_read(c: _Cursor):
    (tag,) = c.fields("B")
    if tag == 0:
        nx, ny = c.fields("II")
        dx, dy, x0, y0, z = c.fields("5d")
        return UniformRelay(UniformGrid2D(nx, ny, dx, dy, x0, y0, z))
    if tag == 1:
        (z,) = c.fields("d")
        (n,) = c.fields("I")
        return NonUniformPlanarRelay(PointList(c.f64(2 * n).reshape(n, 2)), z)
    if tag == 2:
        (n,) = c.fields("I")
        return NonPlanarRelay(PointList(c.f64(3 * n).reshape(n, 3)))
    raise ContainerFormatError(f"unknown relay kind tag {tag} (is this a volume file?)")


def _relay_json(relay) -> dict:
    if relay.kind == "uniform":
        g = relay.grid
        return {"kind": "uniform", "nx": g.nx, "ny": g.ny, "dx": g.dx, "dy": g.dy,
                "x0": g.x0, "y0": g.y0, "z": g.z}
    if relay.kind == "nonuniform_planar":
        return {"kind": "points_planar", "z": relay.z, "points": relay.points.points.tolist()}
    return {"kind": "points_3d", "points": relay.points.points.tolist()}


def _grid_bytes(grid) -> bytes:
    if grid.kind == "cuboid":
        g = grid.grid
        return struct.pack("<III", g.nx, g.ny, g.nz) + struct.pack(
            "<6d", g.dx, g.dy, g.dz, g.x0, g.y0, g.z0)
    if grid.kind == "frustum":
        b = grid.base
        return b"".join([struct.pack("<III", b.nx, b.ny, grid.n_planes),
                         struct.pack("<5d", b.dx, b.dy, b.x0, b.y0, b.z),
                         _f64_bytes(grid.zs), _f64_bytes(grid.alphas), _f64_bytes(grid.betas)])
    parts = [struct.pack("<I", len(grid.planes))]
    for pl in grid.planes:
        parts += [struct.pack("<dI", pl.z, pl.points.count), _f64_bytes(pl.points.points)]
    return b"".join(parts)


def _grid_read(c: _Cursor, tag: int):
    if tag == 16:
        nx, ny, nz = c.fields("III")
        return CuboidGrid(UniformGrid3D(nx, ny, nz, *c.fields("6d")))
    if tag == 17:
        nx, ny, n = c.fields("III")
        dx, dy, x0, y0, z = c.fields("5d")
        zs, al, be = c.f64(n), c.f64(n), c.f64(n)
        return FrustumGrid(UniformGrid2D(nx, ny, dx, dy, x0, y0, z), zs, al, be)
    if tag == 18:
        (n,) = c.fields("I")
        planes = []
        for _ in range(n):
            z, cnt = c.fields("dI")
            planes.append(VoxelPlane(z, PointList(c.f64(2 * cnt).reshape(cnt, 2))))
        return ExplicitVoxels(tuple(planes))
    raise ContainerFormatError(f"unknown voxel grid kind tag {tag}")


# ---------------------------------------------------------------- transient datasets
class DeviceTransientMeasurement:
    """A transient capture whose float32 histograms ``[I, D, T]`` live on the GPU.

    Duck-types reference ``TransientMeasurement`` for :func:`to_frequency`.
    """

    def __init__(self, relay, illuminations, histograms: torch.Tensor, delta_t: float, t0: float):
        self.relay, self.illuminations = relay, illuminations
        self.histograms, self.delta_t, self.t0 = histograms, float(delta_t), float(t0)

    @property
    def n_illum(self) -> int:
        return int(self.histograms.shape[0])

    @property
    def n_detect(self) -> int:
        return int(self.histograms.shape[1])

    @property
    def n_bins(self) -> int:
        return int(self.histograms.shape[2])


def _dataset_header(c: _Cursor):
    _preamble(c)
    n_illum, n_det, n_bins = c.fields("III")
    delta_t, t0 = c.fields("dd")
    relay = _relay_read(c)
    dim, n_pts = c.fields("BI")
    if dim not in (2, 3):
        raise ContainerFormatError(f"illumination dimensionality {dim} invalid")
    ill = PointList(c.f64(n_pts * dim).reshape(n_pts, dim))
    return n_illum, n_det, n_bins, delta_t, t0, relay, ill


def _check_geometry(relay, ill, n_illum, n_det, n_bins, delta_t, t0):
    """The TransientMeasurement preconditions that do not need the payload."""
    if n_bins < 1:
        raise ValidationError("need at least one time bin")
    if not delta_t > 0:
        raise ValidationError("bin width must be > 0")
    if not np.isfinite(t0):
        raise ValidationError("t0 must be finite")
    if n_det != relay.count:
        raise ValidationError("detector axis must match relay point count")
    if n_illum != ill.count:
        raise ValidationError("illumination axis must match illumination point count")


def read_dataset_device(path: str, device=None) -> DeviceTransientMeasurement:
    """Read an NLS1 transient dataset into device memory (float32, no host inflation)."""
    device = device or dev.require_cuda()
    with open(path, "rb") as f:
        c = _Cursor(f)
        n_illum, n_det, n_bins, delta_t, t0, relay, ill = _dataset_header(c)
        _check_geometry(relay, ill, n_illum, n_det, n_bins, delta_t, t0)
        n = n_illum * n_det * n_bins
        if c.pos + 4 * n > c.size:
            raise TruncatedPayloadError(
                f"file ends at byte {c.size} but {c.pos + 4 * n} are needed")
        out = torch.empty(n, dtype=torch.float32, device=device)
        _stream_in(f, out, n)
    counts = torch.empty(2, dtype=torch.int32, device=device)
    _lib.call("pf_count_nonfinite", dev.ptr(out), n, dev.ptr(counts), dev.stream_ptr())
    bad, negative = (int(v) for v in counts.cpu())
    if bad:
        raise NonFiniteDataError("histogram payload contains non-finite values")
    if negative:
        raise ValidationError("histogram values are photon counts and must be >= 0")
    return DeviceTransientMeasurement(relay, ill, out.view(n_illum, n_det, n_bins), delta_t, t0)


def _stream_in(f, out: torch.Tensor, n: int) -> None:
    """File -> two pinned chunks -> device, the read of chunk i+1 under the copy of chunk i."""
    per = max(1, min(n, CHUNK_BYTES // 4))
    stage = [torch.empty(per, dtype=torch.float32, pin_memory=True) for _ in range(2)]
    done = [None, None]
    side = torch.cuda.Stream(device=out.device)
    side.wait_stream(torch.cuda.current_stream(out.device))
    for k, lo in enumerate(range(0, n, per)):
        cnt = min(per, n - lo)
        b = k & 1
        if done[b] is not None:
            done[b].synchronize()
        view = stage[b][:cnt].numpy().view(np.uint8)
        got = f.readinto(memoryview(view))
        if got != 4 * cnt:
            raise TruncatedPayloadError("file ended inside the histogram payload")
        with torch.cuda.stream(side):
            out[lo:lo + cnt].copy_(stage[b][:cnt], non_blocking=True)
            done[b] = torch.cuda.Event()
            done[b].record(side)
    torch.cuda.current_stream(out.device).wait_stream(side)
    side.synchronize()


def read_dataset(path: str) -> TransientMeasurement:
    """Host read (reference ``read_dataset`` core.py:709-731) keeping the float32 payload."""
    with open(path, "rb") as f:
        c = _Cursor(f)
        n_illum, n_det, n_bins, delta_t, t0, relay, ill = _dataset_header(c)
        n = n_illum * n_det * n_bins
        hist = np.frombuffer(c.raw(4 * n), dtype="<f4").astype(np.float32)
    if not np.isfinite(hist).all():
        raise NonFiniteDataError("histogram payload contains non-finite values")
    return TransientMeasurement(relay, ill, hist.reshape(n_illum, n_det, n_bins), delta_t, t0)


def write_dataset(m, path: str) -> None:
    """Reference ``write_dataset`` (core.py:676-706): container plus JSON sidecar.

    ``m.histograms`` may be a numpy array or a (device) tensor; the payload is
    written as little-endian float32 either way.
    """
    h = m.histograms
    if isinstance(h, torch.Tensor):
        h = h.detach().to("cpu", torch.float32).numpy()
    head = b"".join([MAGIC, struct.pack("<I", VERSION),
                     struct.pack("<III", m.n_illum, m.n_detect, m.n_bins),
                     struct.pack("<dd", m.delta_t, m.t0), _relay_bytes(m.relay),
                     struct.pack("<BI", m.illuminations.dim, m.illuminations.count),
                     _f64_bytes(m.illuminations.points)])
    with open(path, "wb") as f:
        f.write(head)
        f.write(np.ascontiguousarray(h, dtype="<f4").tobytes())
    side = {"format": "NLS1 transient dataset", "version": VERSION, "n_illum": m.n_illum,
            "n_detect": m.n_detect, "n_bins": m.n_bins, "delta_t": m.delta_t, "t0": m.t0,
            "relay": _relay_json(m.relay), "n_illumination_points": m.illuminations.count}
    with open(path + ".json", "w", encoding="utf-8") as f:
        json.dump(side, f, indent=2, sort_keys=True)
        f.write("\n")


# ---------------------------------------------------------------- volumes
def _volume_head(grid, n_frames: int, times) -> bytes:
    t = np.zeros(1) if times is None else np.asarray(times, dtype=np.float64)
    return b"".join([MAGIC, struct.pack("<I", VERSION),
                     struct.pack("<III", n_frames, grid.count, 0), struct.pack("<dd", 0.0, 0.0),
                     struct.pack("<B", VOLUME_TAGS[grid.kind]), _grid_bytes(grid), _f64_bytes(t)])


def write_volume(volume, path: str, grid=None, times=None) -> None:
    """Write a volume container (reference ``write_volume`` core.py:783-806).

    ``volume`` is a :class:`ReconstructionVolume`, or a complex64 tensor
    ``[n_frames, n_voxels]`` (device or host) together with ``grid`` /
    ``times``; device tensors are streamed out through a pinned buffer in
    chunks, never widened to complex128.
    """
    if isinstance(volume, ReconstructionVolume):
        grid, times = volume.grid, volume.times
        field = volume.field if times is not None else volume.field[None, :]
        with open(path, "wb") as f:
            f.write(_volume_head(grid, field.shape[0], times))
            f.write(np.ascontiguousarray(field, dtype="<c8").tobytes())
        return
    if grid is None:
        raise ValidationError("a raw volume tensor needs its grid")
    t = volume.reshape(-1, grid.count)
    n_frames = t.shape[0]
    if times is None and n_frames != 1:
        raise ValidationError("time-resolved field must be [n_frames, n_voxels]")
    if times is not None and np.asarray(times).size != n_frames:
        raise ValidationError("time-resolved field must be [n_frames, n_voxels]")
    flat = t.reshape(-1)
    if flat.dtype != torch.complex64:
        flat = flat.to(torch.complex64)
    with open(path, "wb") as f:
        f.write(_volume_head(grid, n_frames, times))
        if flat.device.type == "cpu":
            f.write(flat.contiguous().numpy().tobytes())
            return
        per = max(1, CHUNK_BYTES // 8)
        buf = torch.empty(min(per, flat.numel()), dtype=torch.complex64, pin_memory=True)
        for lo in range(0, flat.numel(), per):
            cnt = min(per, flat.numel() - lo)
            buf[:cnt].copy_(flat[lo:lo + cnt])
            f.write(memoryview(buf[:cnt].numpy().view(np.uint8)))


def read_volume(path: str) -> ReconstructionVolume:
    """Reference ``read_volume`` (core.py:809-832)."""
    with open(path, "rb") as f:
        c = _Cursor(f)
        _preamble(c)
        n_frames, n_vox, _ = c.fields("III")
        c.fields("dd")
        (tag,) = c.fields("B")
        if tag not in VOLUME_TAGS.values():
            raise ContainerFormatError(
                f"kind tag {tag} is not a volume grid (is this a transient dataset?)")
        grid = _grid_read(c, tag)
        if grid.count != n_vox:
            raise ContainerFormatError("declared voxel count does not match grid geometry")
        times = c.f64(n_frames)
        field = np.frombuffer(c.raw(8 * n_frames * n_vox), dtype="<c8").reshape(n_frames, n_vox)
    if not np.isfinite(field).all():
        raise NonFiniteDataError("volume payload contains non-finite values")
    if n_frames == 1:
        return ReconstructionVolume(grid, field[0].astype(np.complex128))
    return ReconstructionVolume(grid, field.astype(np.complex128), times)
