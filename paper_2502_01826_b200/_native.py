"""ctypes binding of the sm_100a library (include/rfsplat_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every entry point raises NativeLibraryError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import NativeLibraryError, raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
# RFS_LIB_PATH: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("RFS_LIB_PATH") or os.path.join(_HERE, "lib", "librfsplat_b200.so")
# RFS_NVTX=1: NVTX ranges named after the entry points around every call
# (e.g. `ncu --nvtx --nvtx-include "rfs_hits/"`, or a timeline profiler)
NVTX = os.environ.get("RFS_NVTX", "") == "1"
_lock = threading.Lock()
_lib = None

vp = C.c_void_p
i32 = C.c_int
f64 = C.c_double
sz = C.c_size_t

# name -> (restype, argtypes)
_SIGS = {
    "rfs_project": (i32, [i32, vp, vp, vp, vp, vp, vp, f64, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "rfs_scan_temp_elems": (sz, [i32]),
    "rfs_exclusive_scan_u32": (i32, [vp, i32, vp, vp, vp, vp]),
    "rfs_bin_fill": (i32, [i32, vp, vp, vp, i32, i32, vp, vp, vp]),
    "rfs_expand_keys": (i32, [vp, i32, vp, vp]),
    "rfs_sort_temp_bytes": (sz, [i32, i32]),
    "rfs_sort_pairs_u64": (i32, [vp, vp, vp, vp, i32, i32, vp, sz, C.POINTER(i32), vp, vp]),
    "rfs_sort_cub_temp_bytes": (sz, [i32, i32]),
    "rfs_sort_pairs_u64_cub": (i32, [vp, vp, vp, vp, i32, i32, vp, sz, C.POINTER(i32), vp]),
    "rfs_tile_ranges": (i32, [vp, i32, vp, i32, vp, vp]),
    "rfs_bin_bucket_temp_bytes": (sz, [i32, i32, i32, i32]),
    "rfs_bin_bucket": (i32, [i32, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "rfs_lower_bounds": (i32, [vp, i32, vp, vp, vp, vp]),
    "rfs_ray_dirs": (i32, [i32, i32, vp, vp]),
    "rfs_hits": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, vp, f64, i32, i32, i32, i32, vp, vp, vp, vp, vp, i32, i32, i32,
                       vp]),
    "rfs_hits_slow": (i32, [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, f64, i32, i32, i32, vp, vp, vp, vp, vp, i32,
                            vp, vp, i32, vp]),
    "rfs_psi": (i32, [i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "rfs_forward": (i32, [vp, vp, i32, vp, i32, i32, i32, vp, vp]),
    "rfs_lam_transpose": (i32, [vp, i32, i32, vp, vp]),
    "rfs_bwd_part_elems": (sz, [i32, i32]),
    "rfs_bwd_gauss": (i32, [i32, i32, vp, i32, vp, vp, i32, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp]),
    "rfs_bwd_rays": (i32, [vp, vp, i32, i32, vp, vp, vp, vp, vp]),
    "rfs_hit_keys": (i32, [vp, vp, vp, i32, i32, vp, vp, vp, vp]),
    "rfs_gather_sorted": (i32, [vp, i32, vp, i32, vp, vp, vp, vp, vp, vp, vp]),
    "rfs_gauss_ranges": (i32, [vp, i32, vp, i32, vp, vp]),
    "rfs_used_list": (i32, [i32, vp, vp, i32, vp, vp]),
    "rfs_geom_part_elems": (sz, [i32]),
    "rfs_grad_geom": (i32, [i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, f64, vp, vp, vp, i32, vp, vp, vp, vp, vp,
                            vp, vp, vp, vp, vp, vp, vp, vp, i32, vp]),
    "rfs_grad_tx": (i32, [i32, vp, vp, i32, vp, i32, i32, vp, vp, vp, vp, i32, i32, vp, vp, vp]),
    "rfs_loss_scratch_bytes": (sz, [i32, i32, i32]),
    "rfs_spectrum_loss": (i32, [i32, i32, i32, vp, vp, vp, f64, f64, vp, vp, vp, vp, vp, sz, vp, vp]),
    "rfs_frame_range_elems": (sz, [i32]),
    "rfs_frame_range": (i32, [i32, i32, i32, vp, vp, vp]),
    "rfs_scalar_loss": (i32, [i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "rfs_sgd_step": (i32, [i32, i32, vp, C.c_float, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "rfs_density_flags": (i32, [i32, i32, vp, vp, vp, f64, f64, f64, vp, vp, vp, vp]),
    "rfs_density_apply": (i32, [i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, C.c_float, C.c_float, C.c_ulonglong, i32,
                                vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "rfs_datagen_path_bytes": (sz, []),
    "rfs_spectrum_dataset": (i32, [i32, vp, i32, vp, vp, f64, i32, i32, f64, i32, vp, vp, vp, vp, vp, vp]),
    "rfs_scalar_dataset": (i32, [i32, vp, i32, vp, vp, f64, i32, i32, f64, i32, vp, vp, vp, vp]),
    "rfs_version": (i32, []),
    "rfs_device_arch": (i32, []),
}

EXPORTED = tuple(_SIGS)


def load(require_cuda: bool = True):
    """Load (once) and return the ctypes library handle."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"{LIB_PATH} is missing; run `python -m paper_2502_01826_b200.build` (no CPU fallback)"
                )
            try:
                lib = C.CDLL(LIB_PATH)
            except OSError as e:  # pragma: no cover - environment specific
                raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_cuda:
        import torch

        if not torch.cuda.is_available():
            raise NativeLibraryError("no CUDA device visible: the rasterizer runs only on sm_100a GPUs")
    return _lib


# kernels launched per entry-point call (sort: 2 + passes, added by raster.sort_pairs)
KERNELS_PER_CALL = {
    "rfs_project": 1, "rfs_exclusive_scan_u32": 2, "rfs_bin_fill": 1, "rfs_expand_keys": 1,
    "rfs_tile_ranges": 1, "rfs_lower_bounds": 1, "rfs_bin_bucket": 8, "rfs_hits": 6, "rfs_hits_slow": 3, "rfs_psi": 1,
    "rfs_forward": 1, "rfs_lam_transpose": 1, "rfs_bwd_gauss": 2, "rfs_bwd_rays": 1, "rfs_hit_keys": 1, "rfs_gauss_ranges": 2, "rfs_used_list": 1, "rfs_grad_geom": 0,
    "rfs_grad_tx": 1, "rfs_gather_sorted": 1,
    "rfs_ray_dirs": 1, "rfs_spectrum_loss": 4, "rfs_frame_range": 1, "rfs_sgd_step": 3, "rfs_scalar_loss": 1, "rfs_density_flags": 1,
    "rfs_density_apply": 1, "rfs_spectrum_dataset": 3, "rfs_scalar_dataset": 2,
}
launch_counter = {"kernels": 0}


_FN: dict = {}
_CUDA_OK = False


def call(name: str, *args) -> None:
    """Call an entry point; raises the rfsplat error class of a non-zero status.

    Hot path (tens of calls per step): the bound ctypes function is cached
    after the first (checked) load, so a call costs the ctypes dispatch only.
    """
    global _CUDA_OK
    fn = _FN.get(name)
    if fn is None or not _CUDA_OK:
        fn = getattr(load(), name)
        _FN[name] = fn
        _CUDA_OK = True
    if NVTX:  # one NVTX range per entry point: its kernels group under the C-ABI name
        import torch

        torch.cuda.nvtx.range_push(name)
        rc = fn(*args)
        torch.cuda.nvtx.range_pop()
    else:
        rc = fn(*args)
    if rc:
        raise_for_status(int(rc), name)
    launch_counter["kernels"] += KERNELS_PER_CALL.get(name, 0)
