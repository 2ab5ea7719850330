"""B200-native differentiable RF Gaussian-splatting rasterizer (GSRF, arXiv 2502.01826).

Drop-in for the hot path of the reference package `rfsplat`: projection onto
the receiver's azimuth/elevation grid, 16x16 tile binning, a 64-bit key radix
sort, complex front-to-back compositing and the analytic backward, as
hand-written sm_100a CUDA behind a C ABI (include/rfsplat_b200.h).

Public API:
    RFSplat / rfsplat                       torch.autograd.Function (autograd.py)
    api.render_complex_frame(s) / backward_frame(s) / build_tiles_for_render /
    project_scene                           reference-shaped host functions (api.py)
    raster.*                                device-level pipeline (raster.py)
    scene.HostScene, bench_scene, random_scene, cube_init
    parallel.*                              TX-sharded data parallelism (parallel.py)
    loss.*                                  spectrum / scalar losses on the device (loss.py)
    train.*                                 SGD, density control, training loop on the device (train.py)
    io.*                                    dataset / checkpoint formats, device dataset loading (io.py)

Importing the package does not need a GPU; calling any compute entry point
without the built library or a CUDA device raises NativeLibraryError.
"""

from .errors import (  # noqa: F401
    ConfigError, ContractViolationError, CudaError, DataError, DegenerateCovarianceError, GeometryError,
    NativeLibraryError, NonFiniteGradientError, RFSplatError, ShapeError,
)
from .scene import HostScene, bench_scene, cube_init, default_txs, random_scene, round_to_f32  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # lazy: torch-dependent modules load on first use
    if name in ("RFSplat", "rfsplat"):
        from . import autograd

        return getattr(autograd, name)
    if name in ("api", "raster", "autograd", "parallel", "loss", "train", "io"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
