"""Full-size parity at BASELINE.json's configs against the compiled reference.

Each case generates the config's A in HBM with the shared generator (the same
bytes the fixture script fed the reference — test_gpu_synth.py checks that),
runs the engine's PCA pipeline through the C-ABI (svdk_dev_pca: centre ->
total variance -> method -> select_components) and compares with the golden
fixture (tests/golden/make_golden.py, SURVEY §8c oracles):

  eigenvalues within 1e-10 relative, K exact, top-K subspace sine <= 1e-8,
  per-vector sines <= 1e-8 for gap-separated vectors (relative gap >= 1e-6),
  clusters compared as subspaces.

The engine methods are checked against the exact (truncated) oracle; the
sketch methods also against the reference's own sketch run where the fixture
holds one (same Omega seed). Fixtures missing from tests/golden skip.
"""
import gc
import os

import numpy as np
import pytest

from paper_1906_12085_b200 import synth
from tests.parity import fixture_parity, parity_ok

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
METHOD = {"truncated": 0, "randomized": 1, "krylov": 2, "lanczos": 3}
# (fixture, method, l, q)
CASES = [
    ("c1", "truncated", 0, 0), ("c1", "randomized", 256, 2), ("c1", "krylov", 128, 1), ("c1", "lanczos", 0, 0),
    ("c2mid", "truncated", 0, 0), ("c2mid", "randomized", 1024, 2), ("c2mid", "lanczos", 0, 0),
    ("c2", "randomized", 1024, 2), ("c2", "truncated", 0, 0), ("c2", "lanczos", 0, 0),
    ("c3", "lanczos", 0, 0), ("c3", "truncated", 0, 0),
    ("c4", "truncated", 0, 0),
    ("c5", "truncated", 0, 0), ("c5", "randomized", 4096, 3), ("c5", "lanczos", 0, 0),
    # the same c5 bytes against LAPACK on the reference's Gram (a labelled cross-check oracle, minutes to make)
    ("c5lapack", "truncated", 0, 0), ("c5lapack", "randomized", 4096, 3), ("c5lapack", "lanczos", 0, 0),
]

_state = {"name": None, "a": None}


@pytest.fixture(scope="module")
def eng(sk):
    from paper_1906_12085_b200.engine import Engine
    return Engine(0)


def _fixture(name):
    p = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(p):
        pytest.skip(f"fixture {name}.npz not generated")
    gz = np.load(p)
    if "a_rows" not in gz:
        pytest.skip(f"{name}.npz predates the shared generator")
    return gz


def _matrix(eng, name, gz):
    import torch
    key = str(gz["cfg"]) + ":" + str(int(gz["m"]))  # fixtures of the same input share the matrix
    if _state["name"] != key:
        _state["a"] = None
        gc.collect()
        torch.cuda.empty_cache()
        cfg = synth.CONFIGS[str(gz["cfg"])]
        _state["a"] = synth.device_matrix(eng, int(gz["m"]), int(gz["n"]), cfg.spectrum(int(gz["n"])),
                                          float(gz["sigma"]), seed=int(gz["seed"]))
        _state["name"] = key
    return _state["a"]


@pytest.mark.parametrize("name,method,l,q", CASES, ids=[f"{c[0]}-{c[1]}" for c in CASES])
def test_config_parity(eng, name, method, l, q):
    gz = _fixture(name)
    a = _matrix(eng, name, gz)
    m, n = a.shape
    big = 8 * m * n > 40e9  # c4: centre in place (A 64 GB + U 64 GB)
    out = eng.pca(a, method=METHOD[method], l=l, q=q, seed=synth.METHOD_SEED, center=2 if big else 1,
                  threshold=float(gz["threshold"]))
    sigma = out.sigma[:out.rank].cpu().numpy()
    lam = sigma * sigma  # fit_pca's eigenvalues (pca.cpp:110-113)
    basis = out.v[:, :out.rank].cpu().numpy()
    total = float(gz["total"])
    # the total variance is a sum of m n squares: two summation orders differ by
    # ~sqrt(m n) eps relative (c4: 8.6e9 terms); it only matters through K
    assert abs(out.total - total) <= 1e-10 * total
    p = fixture_parity(gz, "truncated", lam, basis, out.k)
    print(name, method, p)
    assert parity_ok(p), p
    if f"{method}_lambda" in gz and method != "truncated":  # the reference's own sketch, same seed
        p2 = fixture_parity(gz, method, lam, basis, out.k)
        print(name, method, "vs reference", method, p2)
        assert parity_ok(p2), p2
    if big:
        _state["name"] = None  # A was centred in place
