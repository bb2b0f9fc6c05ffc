"""B200-native phasor-field NLOS reconstruction engine (drop-in for the reference hot path).

Public names mirror the reference package ``phasorfield`` (reference
``__init__.py:19-89``) for the hot path: the phasor kernel and temporal
transform, the eight reconstruction algorithms, the dispatcher, the video
renderer and the depth projection, the boundary types, and the NLS1
containers on either side of the path (read straight to device memory,
volumes written from it).  Compute runs in
``libpfgpu.so`` (hand-written sm_100a CUDA); there is no CPU fallback.
"""

from .container import (DeviceTransientMeasurement, read_dataset, read_dataset_device,
                        read_volume, write_dataset, write_volume)
from .core import (PROPAGATION_SIGN, SPEED_OF_LIGHT, ContainerFormatError, CuboidGrid,
                   ExplicitVoxels, FrequencySlices, FrustumGrid, InvalidMagicError,
                   NonFiniteDataError, NonPlanarRelay, NonUniformPlanarRelay, PointList,
                   ReconstructionVolume, TransientMeasurement, TruncatedPayloadError,
                   TorusMap, UniformGrid2D, UniformGrid3D, UniformRelay, UnsupportedVersionError,
                   ValidationError, VoxelCloud, VoxelPlane, grid_coordinates,
                   illumination_coordinates,
                   rescale_to_torus)
from .phasor import (DeviceFrequencySlices, PhasorKernel, build_kernel, lateral_resolution,
                     to_frequency, to_frequency_device)
from .reconstruct import (ALGORITHM_NAMES, RsdEngine, light_transport_video, project_max_depth,
                          reconstruct, rsd)

__version__ = "0.1.0"


def __getattr__(name):
    # the non-rsd algorithms live in .algorithms (loaded on first use)
    if name in ("srsd", "nursd1", "nursd2", "nursd3", "nursd3d", "srsd_nursd2", "rsd3d",
                "nursd3d_explicit", "nursd3d_srsd", "rsd3d_srsd", "nursd2_voxels"):
        from . import algorithms
        return getattr(algorithms, name)
    if name in ("cfft_n", "cifft_n", "cfft_2d", "cifft_2d", "sfft_1d", "sfft_2d",
                "sfft_2d_centered", "nufft1", "nufft2", "next_fast_len", "fft_2d", "ifft_2d",
                "dft_2d", "idft_2d"):
        from . import spectral
        return getattr(spectral, name)
    if name in ("Scatterer", "Scene", "simulate", "add_poisson_noise"):
        from . import sim
        return getattr(sim, name)
    raise AttributeError(name)
