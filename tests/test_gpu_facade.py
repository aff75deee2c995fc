"""The C++ drop-in facade (libsvdkit.so) through a reference-style caller, plus
the engine's NCCL row-sharded path at world size 1 (a real communicator)."""
import os
import subprocess

import numpy as np
import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu


def test_facade_reference_caller():
    exe = os.path.join(ROOT, "facade", "facade_test")
    assert os.path.exists(exe), "facade not built"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "facade_test: ok" in r.stdout


def test_facade_tools_gpu():
    """facade/tools_test gpu: images_to_matrix kernel + run_grid through the C++ API."""
    exe = os.path.join(ROOT, "facade", "tools_test")
    assert os.path.exists(exe), "facade not built"
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "tools_test gpu: ok" in r.stdout
    assert r.stdout.startswith("method,m,n,repeats,mean_seconds,std_seconds,delta,model_flops,")


def test_nccl_world1_matches_local():
    import torch

    from paper_1906_12085_b200 import _lib
    from paper_1906_12085_b200.engine import Engine, colmajor
    from tests.datagen import make_matrix
    a_np = make_matrix(6000, 128, "c2", seed=9)
    a = colmajor(*a_np.shape)
    a.copy_(torch.from_numpy(np.array(a_np)).cuda())
    e_local = Engine(0)
    e_nccl = Engine(0)
    e_nccl.ctx.attach_nccl(_lib.nccl_unique_id(), 0, 1)
    for method, l, q in ((0, 0, 0), (1, 128, 2), (3, 0, 0)):
        with torch.cuda.stream(e_local.stream):
            o1 = e_local.pca(a, method=method, l=l, q=q, seed=5, threshold=0.95)
        with torch.cuda.stream(e_nccl.stream):
            o2 = e_nccl.pca(a, method=method, l=l, q=q, seed=5, threshold=0.95)
        torch.cuda.synchronize()
        assert o1.rank == o2.rank and o1.k == o2.k
        s1, s2 = o1.sigma[:o1.rank].cpu().numpy(), o2.sigma[:o2.rank].cpu().numpy()
        assert np.max(np.abs(s1 - s2) / s1) <= 1e-13
