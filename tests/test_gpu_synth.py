"""The shared synthetic-input generator (paper_1906_12085_b200/synth.py,
csrc/synth.h): the GPU produces the same bytes as the CPU, any row shard is
byte-identical to those rows of the unsharded matrix, and every golden
fixture's input regenerates on the device (probe rows + mixing checksum) —
so the full-size parity tests and bench.py's parity block compare against
the reference on the SAME input bytes."""
import glob
import hashlib
import os

import numpy as np
import pytest

from paper_1906_12085_b200 import synth
from tests.datagen import config_matrix

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def eng(sk):
    from paper_1906_12085_b200.engine import Engine
    return Engine(0)


def _np(t):
    return t.cpu().numpy()


def test_device_equals_host_c1(eng):
    a_dev = synth.config_device_matrix(eng, "c1")
    a_host = config_matrix("c1")
    assert np.array_equal(_np(a_dev), a_host)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_shards_equal_unsharded(eng, world):
    """Rank r of `world` generates rows [r m/world, (r+1) m/world) with its partial
    X^T X allreduced (here: summed on one device): the same bytes as N = 1."""
    import torch
    cfg = synth.CONFIGS["c1"]
    m, n = 20002, cfg.n  # not a multiple of world: ragged shards
    full = _np(synth.device_matrix(eng, m, n, cfg.spectrum(), cfg.sigma))
    bounds = [m * r // world for r in range(world + 1)]
    parts = [synth.device_gram_x(eng, m, n, row0=bounds[r], rows=bounds[r + 1] - bounds[r])
             for r in range(world)]
    g = torch.zeros_like(parts[0])
    for p in reversed(parts):  # any order: the partial Grams are exact
        g += p
    assert torch.equal(g, synth.device_gram_x(eng, m, n))
    mix, _ = synth.mixing(g.cpu().numpy(), cfg.spectrum(), synth.MATRIX_SEED)
    for r in range(world):
        a_r = synth.device_rows(eng, mix, m, n, cfg.sigma, row0=bounds[r], rows=bounds[r + 1] - bounds[r])
        assert np.array_equal(_np(a_r), full[bounds[r]:bounds[r + 1]]), r


def _fixtures():
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        with np.load(p) as z:
            if "a_rows" in z:
                out.append(os.path.basename(p))
    return out


@pytest.mark.parametrize("name", _fixtures())
def test_fixture_input_regenerates_on_device(eng, name):
    gz = np.load(os.path.join(GOLDEN, name))
    cfg = synth.CONFIGS[str(gz["cfg"])]
    m, n = int(gz["m"]), int(gz["n"])
    g = synth.device_gram_x(eng, m, n, seed=int(gz["seed"]))
    mix, _ = synth.mixing(g.cpu().numpy(), cfg.spectrum(n), int(gz["seed"]))
    assert hashlib.sha256(np.ascontiguousarray(mix).tobytes()).hexdigest() == str(gz["mix_sha256"])
    for k, i in enumerate(np.asarray(gz["a_rows_idx"])):
        row = synth.device_rows(eng, mix, m, n, float(gz["sigma"]), seed=int(gz["seed"]), row0=int(i), rows=1)
        assert np.array_equal(_np(row)[0], np.asarray(gz["a_rows"])[k]), (name, int(i))
