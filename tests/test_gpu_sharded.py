"""The engine's row-sharded path, executed: `world` ranks = contexts on host
threads joined by the in-process host-staged collective group (comm.cu), so
every sharded branch of svdk_dev_pca (allreduced column sums / total / Gram /
A^T Y / CholeskyQR Grams / Lanczos w, rank-0 eigensolve + broadcast, local U
shards) runs on one GPU. No kernel waits on another rank (each collective is
stream-sync + host sum), so ranks sharing the GPU cannot deadlock it.

Bars: world 2/3/4 match world 1 — sigma <= 1e-13
relative, same K, V subspace <= 1e-10 — and the golden fixture's reference
bars hold for the sharded result too. Also: an empty shard, ragged shards,
and argument disagreement failing on EVERY rank instead of hanging.
"""
import threading

import numpy as np
import pytest

from paper_1906_12085_b200 import errors, synth
from tests.parity import eig_rel_err, subspace_sine, topk_sine

pytestmark = pytest.mark.gpu
METHODS = {"truncated": (0, 0, 0), "randomized": (1, 256, 2), "krylov": (2, 128, 1), "lanczos": (3, 0, 0)}


@pytest.fixture(scope="module")
def base(sk):
    import torch

    from paper_1906_12085_b200.engine import Engine
    eng = Engine(0)
    cfg = synth.CONFIGS["c1"]
    a = synth.config_device_matrix(eng, cfg)
    torch.cuda.synchronize()
    return eng, a, cfg


def _copy_rows(a, r0, r1):
    from paper_1906_12085_b200.engine import colmajor
    out = colmajor(max(r1 - r0, 0), a.shape[1], a.device)
    if r1 > r0:
        out.copy_(a[r0:r1])
    return out


def run_sharded(a, bounds, method, threshold, args_override=None):
    """One svdk_dev_pca per rank on its own thread; returns per-rank outputs or exceptions."""
    import torch

    from paper_1906_12085_b200._lib import HostGroup
    from paper_1906_12085_b200.engine import Engine
    world = len(bounds) - 1
    group = HostGroup(world)
    engines = [Engine(0) for _ in range(world)]
    for r, e in enumerate(engines):
        e.ctx.attach_host_group(group, r)
    shards = [_copy_rows(a, bounds[r], bounds[r + 1]) for r in range(world)]
    torch.cuda.synchronize()
    mid, l, q = METHODS[method]
    results = [None] * world

    def work(r):
        try:
            kw = dict(method=mid, l=l, q=q, seed=synth.METHOD_SEED, center=1, threshold=threshold)
            if args_override and r in args_override:
                kw.update(args_override[r])
            results[r] = engines[r].pca(shards[r], **kw)
            # this rank's stream only: a device-wide synchronize is illegal while another
            # rank's thread is capturing its sweep graph (it invalidates that capture)
            engines[r].ctx.sync()
        except Exception as e:  # collected and asserted by the caller
            results[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a rank hung"
    for e in engines:
        e.ctx.detach_comm()
    group.close()
    return results


@pytest.mark.parametrize("method", list(METHODS))
@pytest.mark.parametrize("layout", ["2", "4", "3-ragged", "3-empty"])
def test_sharded_matches_single(base, method, layout):
    eng, a, cfg = base
    m = a.shape[0]
    bounds = {"2": [0, m // 2, m], "4": [0, m // 4, m // 2, 3 * m // 4, m],
              "3-ragged": [0, 6667, 13001, m], "3-empty": [0, 0, 9999, m]}[layout]
    mid, l, q = METHODS[method]
    one = eng.pca(a, method=mid, l=l, q=q, seed=synth.METHOD_SEED, center=1, threshold=cfg.t)
    outs = run_sharded(a, bounds, method, cfg.t)
    for r, o in enumerate(outs):
        assert not isinstance(o, Exception), (r, o)
    s1 = one.sigma[:one.rank].cpu().numpy()
    v1 = one.v[:, :one.rank].cpu().numpy()
    u1 = one.u[:, :one.rank].cpu().numpy()
    for r, o in enumerate(outs):
        assert o.rank == one.rank and o.k == one.k, (r, o.rank, o.k)
        s = o.sigma[:o.rank].cpu().numpy()
        assert eig_rel_err(s, s1) <= 1e-13, r
        v = o.v[:, :o.rank].cpu().numpy()
        # V is replicated: every rank holds the same bits
        assert np.array_equal(v, outs[0].v[:, :o.rank].cpu().numpy())
        kk = one.k
        assert subspace_sine(v[:, :kk], v1[:, :kk]) <= 1e-10
        assert abs(o.total - one.total) <= 1e-13 * one.total
    # the stacked U shards span the single-GPU U's top-K subspace, with the same
    # signs (the sketch methods' U = Q W carries CholeskyQR's ~1e-10 rounding)
    u = np.vstack([o.u[:, :o.rank].cpu().numpy() for o in outs])
    kk = one.k
    assert topk_sine(u[:, :kk], u1[:, :kk]) <= (1e-10 if method in ("truncated", "lanczos") else 1e-8)
    assert np.all(np.sum(u[:, :kk] * u1[:, :kk], axis=0) > 0.5)


def test_sharded_vs_reference_fixture(base):
    """world 4 against the compiled reference's c1 fixture (same input bytes)."""
    import os
    eng, a, cfg = base
    path = os.path.join(os.path.dirname(__file__), "golden", "c1.npz")
    gz = np.load(path)
    from tests.parity import fixture_parity, parity_ok
    m = a.shape[0]
    outs = run_sharded(a, [0, 5000, 10000, 15000, m], "truncated", cfg.t)
    o = outs[2]
    s = o.sigma[:o.rank].cpu().numpy()
    p = fixture_parity(gz, "truncated", s * s, o.v[:, :o.rank].cpu().numpy(), o.k)
    assert parity_ok(p), p


def test_sharded_argument_disagreement_fails_everywhere(base):
    """Rank 1 passes a different sketch width: every rank raises ParamError
    (agreed before any data collective) instead of hanging in a reduction."""
    eng, a, cfg = base
    m = a.shape[0]
    outs = run_sharded(a, [0, m // 2, m], "randomized", cfg.t, {1: dict(l=128)})
    assert all(isinstance(o, errors.ParamError) for o in outs), outs


def test_sharded_sketch_param_error_everywhere(base):
    """An invalid replicated parameter (l > n) fails identically on every rank."""
    eng, a, cfg = base
    m = a.shape[0]
    outs = run_sharded(a, [0, m // 3, m], "randomized", cfg.t, {0: dict(l=512), 1: dict(l=512)})
    assert all(isinstance(o, errors.ParamError) for o in outs), outs


def test_c4_world2_vs_reference_fixture(sk):
    """BASELINE c4 itself, row-sharded over 2 ranks (host-staged group, both on
    this GPU): each rank generates ITS half of the rows (synth.device_rows with
    the allreduced X^T X), runs svdk_dev_pca on it (centre in place), and the
    result must meet the full-size reference bars of tests/golden/c4.npz."""
    import os

    import torch

    from paper_1906_12085_b200._lib import HostGroup
    from paper_1906_12085_b200.engine import Engine
    from tests.parity import fixture_parity, parity_ok
    path = os.path.join(os.path.dirname(__file__), "golden", "c4.npz")
    if not os.path.exists(path):
        pytest.skip("c4 fixture not generated")
    free, _ = torch.cuda.mem_get_info()
    if free < 150e9:
        pytest.skip("needs ~140 GB of free HBM")
    gz = np.load(path)
    cfg = synth.CONFIGS["c4"]
    world = 2
    bounds = [cfg.m * r // world for r in range(world + 1)]
    group = HostGroup(world)
    engines = [Engine(0) for _ in range(world)]
    for r, e in enumerate(engines):
        e.ctx.attach_host_group(group, r)
    # the allreduce of the per-rank partial X^T X (exact on the generator's grid)
    parts = [synth.device_gram_x(engines[r], cfg.m, cfg.n, row0=bounds[r], rows=bounds[r + 1] - bounds[r])
             for r in range(world)]
    g = parts[0] + parts[1]
    mix, _ = synth.mixing(g.cpu().numpy(), cfg.spectrum(), synth.MATRIX_SEED)
    del parts, g
    shards = [synth.device_rows(engines[r], mix, cfg.m, cfg.n, cfg.sigma, row0=bounds[r],
                                rows=bounds[r + 1] - bounds[r]) for r in range(world)]
    torch.cuda.synchronize()
    outs = [None] * world

    def work(r):
        try:
            outs[r] = engines[r].pca(shards[r], method=0, center=2, threshold=cfg.t)
        except Exception as e:
            outs[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join(timeout=900) for t in th]
    assert not any(t.is_alive() for t in th)
    for o in outs:
        assert not isinstance(o, Exception), o
    o = outs[1]
    s = o.sigma[:o.rank].cpu().numpy()
    p = fixture_parity(gz, "truncated", s * s, o.v[:, :o.rank].cpu().numpy(), o.k)
    print("c4 world 2", p)
    assert abs(o.total - float(gz["total"])) <= 1e-10 * float(gz["total"])
    assert parity_ok(p), p
    for e in engines:
        e.ctx.detach_comm()
    group.close()
