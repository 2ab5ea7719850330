"""CPU-side boundary checks: the C-ABI library loads and exports every symbol
include/rfsplat_b200.h declares; host logic fails loudly without a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2502_01826_b200 import _native, build
from paper_2502_01826_b200.errors import (
    ContractViolationError, GeometryError, NativeLibraryError, ShapeError, raise_for_status,
)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "rfsplat_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t)\s+(rfs_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return ctypes.CDLL(_native.LIB_PATH)


def test_header_declares_the_kernel_abi():
    names = _declared()
    for n in ("rfs_project", "rfs_exclusive_scan_u32", "rfs_bin_fill", "rfs_sort_pairs_u64", "rfs_sort_pairs_u64_cub",
              "rfs_tile_ranges", "rfs_lower_bounds", "rfs_bin_bucket_temp_bytes", "rfs_bin_bucket", "rfs_hits", "rfs_psi", "rfs_forward", "rfs_lam_transpose", "rfs_bwd_gauss", "rfs_bwd_rays",
              "rfs_hit_keys", "rfs_gather_sorted", "rfs_gauss_ranges", "rfs_used_list", "rfs_grad_geom", "rfs_grad_tx"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    assert sorted(_native.EXPORTED) == _declared()


def test_library_is_sm100a(lib):
    out = os.popen(f"cuobjdump --list-elf {_native.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_size_queries_without_gpu(lib):
    lib.rfs_sort_temp_bytes.restype = ctypes.c_size_t
    lib.rfs_scan_temp_elems.restype = ctypes.c_size_t
    assert lib.rfs_sort_temp_bytes(483_032, 40) > 0
    assert lib.rfs_scan_temp_elems(100_000) >= 25
    assert lib.rfs_version() == 1 and lib.rfs_device_arch() == 100


def test_compute_without_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2502_01826_b200 import api
    from paper_2502_01826_b200.scene import random_scene

    with pytest.raises((NativeLibraryError, RuntimeError, AssertionError)):
        api.render_complex_frame(random_scene(np.random.default_rng(0), 4), [1.0, 2.0, 3.0])


def test_status_codes_map_to_reference_errors():
    raise_for_status(0, "ok")
    with pytest.raises(GeometryError):
        raise_for_status(1, "x")
    with pytest.raises(ShapeError):
        raise_for_status(2, "x")
    with pytest.raises(ContractViolationError):
        raise_for_status(3, "x")


def test_product_does_not_import_oracle():
    pkg = os.path.join(REPO, "paper_2502_01826_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src/rfsplat"), reason="reference not present")
def test_errors_are_the_reference_classes_when_installed():
    """With the reference importable, callers catching rfsplat.errors.* catch
    what this package raises (the classes are the reference's own)."""
    import subprocess
    import sys

    code = ("import paper_2502_01826_b200.errors as e, rfsplat.errors as r;"
            "assert e.GeometryError is r.GeometryError and e.ShapeError is r.ShapeError;"
            "assert issubclass(e.CudaError, r.RFSplatError);"
            "import rfsplat; assert rfsplat.GeometryError is e.GeometryError")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join(["/root/reference/pkg/src", REPO]),
               NUMBA_CACHE_DIR="/tmp/nb")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=300)


def test_pcap_evict_flag_matches_header():
    """rfs_hits' ring flag: the header's value is the one the kernels and raster.py use."""
    from paper_2502_01826_b200 import raster

    hdr = re.search(r"#define RFS_PCAP_EVICT (0x[0-9a-fA-F]+)", open(HEADER).read())
    common = re.search(r"#define RFS_PCAP_EVICT (0x[0-9a-fA-F]+)",
                       open(os.path.join(REPO, "paper_2502_01826_b200", "csrc", "rfs_common.cuh")).read())
    assert hdr and common and int(hdr.group(1), 16) == int(common.group(1), 16) == raster.RFS_PCAP_EVICT
