"""C-ABI boundary checks that need no GPU: the library loads, exports every
entry point include/svdk.h declares (and the ctypes table binds them all),
the host-side Gaussian sampler is bit-identical to the reference's, and the
engine fails loudly (no CPU fallback) when no GPU is present."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1906_12085_b200 import _lib, errors
from tests.conftest import HAS_GPU, ROOT

HEADER = os.path.join(ROOT, "include", "svdk.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(svdk_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    assert len(names) >= 30
    for must in ("svdk_gram", "svdk_eig_sym", "svdk_truncated_svd", "svdk_randomized_pca", "svdk_krylov_svd",
                 "svdk_lanczos_svd", "svdk_select_components", "svdk_fit_pca", "svdk_dev_pca", "svdk_qr_thin"):
        assert must in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(_lib.LIB_PATH), "libsvdk.so not built"
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (svdk_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_ctypes_table_matches_header():
    assert sorted(_lib.SIGNATURES) == declared()
    lib = _lib.load()
    for name in declared():
        assert getattr(lib, name) is not None
    assert b"sm_100a" in lib.svdk_version()


def test_status_mapping():
    with pytest.raises(errors.DimensionError):
        errors.raise_for_status(1, "x")
    with pytest.raises(errors.ParamError):
        errors.raise_for_status(2, "x")
    with pytest.raises(errors.NumericalError) as e:
        errors.raise_for_status(3, "x", 0.25)
    assert e.value.residual() == 0.25
    with pytest.raises(errors.EngineError):
        errors.raise_for_status(4, "x")


@pytest.mark.parametrize("shape,seed", [((3, 2), 42), ((7, 5), 0), ((1, 1), 3), ((513, 301), 77)])
def test_host_sampler_bit_identical(port, shape, seed):
    """svdk_gaussian_matrix (host, threaded Box-Muller) == reference sampler bit for bit."""
    from paper_1906_12085_b200 import svdkit
    g = svdkit.gaussian_matrix(*shape, seed)
    assert np.array_equal(g, port.gaussian_matrix(*shape, seed))


def test_host_sampler_param_error():
    from paper_1906_12085_b200 import svdkit
    with pytest.raises(errors.ParamError):
        svdkit.gaussian_matrix(0, 3, 1)


def test_python_mirror_validates_shapes_before_device():
    from paper_1906_12085_b200 import svdkit
    with pytest.raises(errors.DimensionError):
        svdkit.matmul(np.ones((2, 3)), np.ones((2, 3)))
    with pytest.raises(errors.DimensionError):
        svdkit.matmul_transposed_left(np.ones((2, 3)), np.ones((3, 3)))
    with pytest.raises(errors.ParamError):
        svdkit.truncated_svd(np.array([[1.0, np.nan], [0, 1]]))


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    with pytest.raises(errors.EngineError):
        _lib.Context(0)


FACADE_API = ["svdkit::matmul(", "svdkit::matmul_transposed_left(", "svdkit::transpose(", "svdkit::gram(",
              "svdkit::frobenius_norm_sq(", "svdkit::qr_thin(", "svdkit::eig_sym(", "svdkit::gaussian_matrix(",
              "svdkit::truncated_svd(", "svdkit::randomized_pca(", "svdkit::krylov_svd(", "svdkit::lanczos_svd(",
              "svdkit::truncate_rank(", "svdkit::compute_svd(", "svdkit::compute_svd_any(", "svdkit::center(",
              "svdkit::total_variance(", "svdkit::select_components(", "svdkit::fit_pca(", "svdkit::transform(",
              "svdkit::residual_delta(", "svdkit::method_name(", "svdkit::method_from_name(",
              "svdkit::MethodParams::defaults_for(", "svdkit::DenseMatrix::DenseMatrix(", "svdkit::shape_string"]


def test_facade_exports_reference_api():
    lib = os.path.join(ROOT, "facade", "libsvdkit.so")
    assert os.path.exists(lib), "facade not built"
    out = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    missing = [f for f in FACADE_API if f not in out]
    assert not missing, missing


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure path")
def test_facade_fails_loudly_without_gpu():
    exe = os.path.join(ROOT, "facade", "facade_test")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
