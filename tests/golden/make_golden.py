"""Generate the golden fixtures from the COMPILED REFERENCE (oracle/_ref) — test infrastructure.

Run here, where /root/reference exists (oracle/Makefile builds oracle/_ref from
its sources):

    python tests/golden/make_golden.py small c1 c2mid      # minutes
    python tests/golden/make_golden.py c2 [--threads T]     # ~1 h  (full reference truncated + randomized)
    python tests/golden/make_golden.py c4 c3 c5             # hours (c5: eig_sym(4096) > 4 h)
    python tests/golden/make_golden.py c5lapack             # 8 min: c5's reference Gram + LAPACK (cross-check)

Inputs come from the generator shared with bench.py (paper_1906_12085_b200/
synth.py): the GPU regenerates the same bytes, checked through `a_rows` (a few
rows of A stored verbatim) and `mix_sha256` (the host-built mixing matrix).
Outputs are what the unmodified reference computes on those bytes:

* c1, c2mid, c2, small: the reference pipeline itself on the whole matrix —
  center (pca.cpp:13-55), total_variance (pca.cpp:57-59), truncated_svd
  (svd_methods.cpp:121-158) and the sketch methods with the config's l, q and
  seed (svd_methods.cpp:160-196), eigenvalues = sigma^2 (pca.cpp:110-113),
  select_components (pca.cpp:61-89). Phase wall times are recorded (one core).
* c3, c4, c5 (SURVEY §8c's labelled alternative — the whole reference
  truncated_svd would also form the unused m x n U for hours): reference
  center semantics (sequential column sums, pca.cpp:37-53), reference `gram`
  (kernels.cpp:80-97) on fixed row blocks summed in block order, reference
  `eig_sym` (kernels.cpp:241-346) on that Gram, sigma = sqrt(max(lambda, 0))
  and the rank cut exactly as truncated_svd does, eigenvalues = sigma^2.
  c3 / c5 materialise A and run the reference center + frobenius_norm_sq
  whole; c4 (64 GB) is processed in row blocks (its total variance is the
  sum of the blocks' reference frobenius_norm_sq — rounding-level different).

Eigenvectors stored: every column at c1; V[:, :K] at the headline configs c2
and c4 (every per-vector sine is checked); elsewhere the smaller of V[:, :K]
and the complement V[:, K:] (the top-K subspace sine is ||V_K^T V_perp_ref||_2)
plus 128 sampled gap-separated top-K vectors for the per-vector sines.
"""
import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Oracle  # noqa: E402
from paper_1906_12085_b200 import synth  # noqa: E402
from tests.datagen import make_matrix  # noqa: E402
from tests.parity import gap_groups  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
GEN = "synth-v1"  # generator version (csrc/synth.h)
TIMES = os.path.join(ROOT, "profiles", "r2_reference_fixture_times.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def record_times(name, times):
    data = {}
    if os.path.exists(TIMES):
        data = json.load(open(TIMES))
    data[name] = times
    json.dump(data, open(TIMES, "w"), indent=1, sort_keys=True)


def row_probe(m):
    idx = sorted({0, 1, max(m // 8 - 1, 0), m // 8, m // 2 + 1, m - 1})
    return np.array([i for i in idx if 0 <= i < m], dtype=np.int64)


def small(ref):
    m, n, seed = 300, 24, 7
    a = make_matrix(m, n, "c1", seed=seed)
    l, q, kl, ki, rseed = 24, 2, 8, 2, 1234
    t = ref.truncated_svd(a)
    r = ref.randomized_pca(a, l, q, rseed)
    k = ref.krylov_svd(a, kl, ki, rseed)
    g = ref.gram(a)
    w, v = ref.eig_sym(g)
    np.savez_compressed(os.path.join(OUT, "small.npz"), gen=GEN, m=m, n=n, seed=seed, a=a, l=l, q=q, kl=kl,
                        ki=ki, rseed=rseed, trunc_sigma=t.sigma, trunc_u=t.u, trunc_v=t.v, rand_sigma=r.sigma,
                        rand_u=r.u, rand_v=r.v, kry_sigma=k.sigma, kry_u=k.u, kry_v=k.v, gram=g, eig_w=w,
                        eig_v=v)


def k_margin(lam, total, t, k):
    cum = np.cumsum(lam) / total
    lo = abs(cum[k - 2] - t) if k >= 2 else np.inf
    return float(min(abs(cum[k - 1] - t), lo))


def store_basis(out, prefix, lam, v, k, n, full=False, force_vk=False):
    """Every column (full), V[:, :K] (force_vk, or when smaller), else the complement
    V[:, K:] plus 128 sampled gap-separated top-K vectors for the per-vector sines."""
    if full:
        out[f"{prefix}_v"] = v
        return
    singles = [g[0] for g in gap_groups(lam) if len(g) == 1 and g[0] < k]
    nsample = min(128, len(singles))
    if force_vk or k <= (n - k) + nsample:
        out[f"{prefix}_vk"] = np.asfortranarray(v[:, :k])
        return
    out[f"{prefix}_vperp"] = np.asfortranarray(v[:, k:])
    pick = np.array(singles, dtype=np.int64)[np.linspace(0, len(singles) - 1, nsample).astype(int)]
    out[f"{prefix}_vidx"] = pick
    out[f"{prefix}_vsample"] = np.asfortranarray(v[:, pick])


def header(cfg, m, n, seed, mix, a_rows_src):
    rows = row_probe(m)
    return dict(gen=GEN, cfg=cfg.name, m=m, n=n, seed=seed, sigma=cfg.sigma, threshold=cfg.t,
                mix_sha256=sha(mix), a_rows_idx=rows, a_rows=a_rows_src(rows))


def sweep_trajectory(ref, c, cap_max=30):
    """off(A) after each sweep of the reference eig_sym on c's Gram (kernels.cpp:
    321-326: the NumericalError residual with max_sweeps = cap), SURVEY 8a."""
    from oracle.pyoracle import OracleError
    g = ref.gram(c)
    offs = []
    for cap in range(1, cap_max + 1):
        try:
            ref.eig_sym(g, cap)
            return np.array(offs), cap
        except OracleError as e:
            offs.append(e.residual)
    return np.array(offs), -1


def finish_lambda(w):
    """truncated_svd's sigma = sqrt(max(lambda, 0)) + rank cut; eigenvalues = sigma^2 (pca.cpp:110-113)."""
    sigma = np.sqrt(np.maximum(w, 0.0))
    rank = 0
    while rank < len(sigma) and sigma[rank] > 1e-12 * sigma[0]:
        rank += 1
    return sigma[:rank] * sigma[:rank], rank


# --------------------------------------------------------------------------- whole-matrix reference runs
def full(ref, name, cfg, m, seed, methods, full_v=False, force_vk=False, trajectory=False):
    n = cfg.n
    t0 = time.time()
    gx = synth.host_gram_x(m, n, seed)
    mix, _ = synth.mixing(gx, cfg.spectrum(), seed)
    a = synth.host_matrix(m, n, cfg.spectrum(), cfg.sigma, seed, mix=mix)
    log(name, "generated", a.shape, f"{time.time() - t0:.1f}s")
    out = header(cfg, m, n, seed, mix, lambda r: a[r, :])
    times = {"m": m, "n": n, "threads": 1, "host": os.uname().nodename}
    t0 = time.perf_counter()
    c, mean = ref.center(a, 1)
    times["center_s"] = time.perf_counter() - t0
    del a
    t0 = time.perf_counter()
    total = ref.frobenius_norm_sq(c)
    times["total_variance_s"] = time.perf_counter() - t0
    out.update(total=total, mean=mean, oracle="svdkit_ref: center + total_variance + "
               + " / ".join(methods) + " on the whole matrix (compiled reference)")
    if trajectory:
        offs, conv = sweep_trajectory(ref, c)
        out.update(ref_sweep_off=offs, ref_sweeps=conv)
        log(name, "reference sweep trajectory", offs, "converged at", conv)
    for meth, (l, q, rs) in methods.items():
        t0 = time.perf_counter()
        if meth == "truncated":
            s = ref.truncated_svd(c)
        elif meth == "randomized":
            s = ref.randomized_pca(c, l, q, rs)
        else:
            s = ref.krylov_svd(c, l, q, rs)
        times[f"{meth}_s"] = time.perf_counter() - t0
        lam = s.sigma * s.sigma
        k = ref.select_components(lam, total, cfg.t) or 0
        out[f"{meth}_lambda"] = lam
        out[f"{meth}_k"] = k
        out[f"{meth}_margin"] = k_margin(lam, total, cfg.t, k)
        out[f"{meth}_params"] = np.array([l, q, rs])
        if meth == "truncated" or full_v:
            store_basis(out, meth, lam, s.v, k, n, full=full_v, force_vk=force_vk)
        else:  # method-level cross-check: the top-K subspace via the smaller side
            if k <= n - k:
                out[f"{meth}_vk"] = np.asfortranarray(s.v[:, :k])
            else:
                out[f"{meth}_vperp"] = np.asfortranarray(s.v[:, k:])
        log(name, meth, f"{times[f'{meth}_s']:.1f}s K={k} margin={out[f'{meth}_margin']:.2e}")
        del s
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    record_times(name, times)


# --------------------------------------------------------------------------- row-blocked reference runs
def block_gram(ref, c_rows_iter, threads):
    """sum over fixed row blocks (in block order) of the reference gram of each block."""
    g = None
    pool = ThreadPoolExecutor(max_workers=threads)
    for blocks in c_rows_iter:
        parts = list(pool.map(ref.gram, blocks))  # ctypes releases the GIL
        for p in parts:
            g = p if g is None else g + p
    pool.shutdown()
    return g


def blocked(ref, name, cfg, seed, threads, sub_rows=32768, gen_rows=262144, force_vk=False,
            materialise_max=12e9, eig="ref"):
    m, n = cfg.m, cfg.n
    times = {"m": m, "n": n, "threads": threads, "sub_rows": sub_rows, "host": os.uname().nodename}
    t0 = time.time()
    gx = synth.host_gram_x(m, n, seed, chunk=gen_rows)
    mix, _ = synth.mixing(gx, cfg.spectrum(), seed)
    times["gen_mix_s"] = time.time() - t0
    log(name, "mixing ready", f"{time.time() - t0:.1f}s")
    materialise = 8 * m * n <= materialise_max
    if materialise:
        a = synth.host_matrix(m, n, cfg.spectrum(), cfg.sigma, seed, mix=mix)
        out = header(cfg, m, n, seed, mix, lambda r: a[r, :])
        t0 = time.perf_counter()
        c, mean = ref.center(a, 1)
        del a
        total = ref.frobenius_norm_sq(c)
        times["center_total_s"] = time.perf_counter() - t0

        def blocks():
            for r0 in range(0, m, sub_rows * threads):
                yield [np.asfortranarray(c[r:min(r + sub_rows, m)]) for r in
                       range(r0, min(r0 + sub_rows * threads, m), sub_rows)]
        total_note = "reference center + frobenius_norm_sq on the whole matrix"
    else:
        def gen(r0):
            return synth.host_matrix(m, n, cfg.spectrum(), cfg.sigma, seed, row0=r0,
                                     rows=min(gen_rows, m - r0), mix=mix)
        probe = row_probe(m)
        rows_out = np.empty((len(probe), n))
        carry = np.zeros(n)
        t0 = time.perf_counter()
        for r0 in range(0, m, gen_rows):
            ab = gen(r0)
            sel = (probe >= r0) & (probe < r0 + ab.shape[0])
            rows_out[sel] = ab[probe[sel] - r0]
            # the reference's sequential column sums, carried across blocks
            carry = np.add.accumulate(np.vstack([carry[None, :], ab]), axis=0)[-1]
            del ab
        mean = carry / float(m)
        times["colsum_pass_s"] = time.perf_counter() - t0
        out = header(cfg, m, n, seed, mix, lambda r: rows_out)
        log(name, "column means ready")
        tot = [0.0]

        def blocks():
            for r0 in range(0, m, gen_rows):
                cb = gen(r0)
                cb -= mean[None, :]
                cb = np.asfortranarray(cb)
                tot[0] += ref.frobenius_norm_sq(cb)
                yield [np.asfortranarray(cb[r:min(r + sub_rows, cb.shape[0])])
                       for r in range(0, cb.shape[0], sub_rows)]
                log(name, f"rows {r0 + cb.shape[0]}/{m}")
        total = None
        total_note = "sum over 262144-row blocks of the reference frobenius_norm_sq (rounding-level different)"
    t0 = time.perf_counter()
    g = block_gram(ref, blocks(), threads)
    times["block_gram_s"] = time.perf_counter() - t0
    if total is None:
        total = tot[0]
    log(name, f"gram done {times['block_gram_s']:.1f}s; eig_sym({n}) ...")
    t0 = time.perf_counter()
    if eig == "lapack":  # labelled weaker oracle: LAPACK dsyevd on the reference's Gram (minutes instead of hours)
        w, v = np.linalg.eigh(g)
        w, v = w[::-1].copy(), v[:, ::-1].copy()
    else:
        w, v = ref.eig_sym(g)
    times["eig_sym_s"] = time.perf_counter() - t0
    lam, rank = finish_lambda(w)
    k = ref.select_components(lam, total, cfg.t) or 0
    log(name, f"eig_sym {times['eig_sym_s']:.1f}s rank={rank} K={k}")
    out.update(total=total, mean=mean, truncated_lambda=lam, truncated_k=k,
               truncated_margin=k_margin(lam, total, cfg.t, k), gram_sha256=sha(g),
               oracle=(f"svdkit_ref::gram on {sub_rows}-row blocks summed in block order + "
                       + ("LAPACK dsyevd (numpy.linalg.eigh) on that Gram — NOT the reference eig_sym; a labelled "
                          "cross-check oracle" if eig == "lapack" else "svdkit_ref::eig_sym")
                       + f" (SURVEY 8c alternative); total: {total_note}"))
    store_basis(out, "truncated", lam, v, k, n, force_vk=force_vk)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    record_times(name, times)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="*", default=["small", "c1"])
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 4)
    args = ap.parse_args()
    ref = Oracle("ref")
    C = synth.CONFIGS
    for w in args.which:
        log("==", w)
        if w == "small":
            small(ref)
        elif w == "c1":
            full(ref, "c1", C["c1"], C["c1"].m, synth.MATRIX_SEED,
                 {"truncated": (0, 0, 0), "randomized": (256, 2, synth.METHOD_SEED),
                  "krylov": (128, 1, synth.METHOD_SEED)}, full_v=True, trajectory=True)
        elif w == "c2mid":
            # c2's spectrum and method at a height the reference finishes in minutes
            full(ref, "c2mid", C["c2"], 20000, synth.MATRIX_SEED,
                 {"truncated": (0, 0, 0), "randomized": (1024, 2, synth.METHOD_SEED)})
        elif w == "c2":
            full(ref, "c2", C["c2"], C["c2"].m, synth.MATRIX_SEED,
                 {"truncated": (0, 0, 0), "randomized": (1024, 2, synth.METHOD_SEED)}, force_vk=True)
        elif w in ("c3", "c4", "c5"):
            blocked(ref, w, C[w], synth.MATRIX_SEED, args.threads, force_vk=(w == "c4"))
        elif w == "c5lapack":  # c5 with LAPACK on the reference's Gram: a cross-check of the c5 fixture
            blocked(ref, "c5lapack", C["c5"], synth.MATRIX_SEED, args.threads, eig="lapack")
        else:
            raise SystemExit(f"unknown fixture {w}")
