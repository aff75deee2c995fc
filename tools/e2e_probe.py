"""Host-buffer fit_pca timing (development probe): plain vs streamed upload, and
the raw H2D of the same pinned buffer (contiguous and in 2-D row chunks).
  python tools/e2e_probe.py [config]"""
import ctypes as C
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1906_12085_b200 import _lib  # noqa: E402
from paper_1906_12085_b200.engine import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = dict(bench.CONFIGS[name])
m, n = cfg["m"], cfg["n"]
mid = bench.METHOD_ID[cfg["method"]]
eng = Engine(0)
torch.cuda.set_stream(eng.stream)
A = bench.generate(cfg, m, torch.device("cuda", 0), 0)
host = torch.empty(n, m, dtype=torch.float64, pin_memory=True).t()
host.copy_(A)
del A
torch.cuda.synchronize()
torch.cuda.empty_cache()
lib = _lib.load()
width = cfg["l"] if cfg["method"] == "randomized" else n
basis = torch.empty(width, n, dtype=torch.float64, pin_memory=True)
eig = torch.empty(width, dtype=torch.float64, pin_memory=True)
mean = torch.empty(n, dtype=torch.float64, pin_memory=True)
total, rank = C.c_double(0), C.c_int64(0)
for mode in ["1", "0", "1", "0"]:
    os.environ["SVDK_STREAM"] = mode
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(lib.svdk_fit_pca(eng.ctx.handle, C.c_void_p(host.data_ptr()), m, n, 1, mid, cfg["l"], cfg["q"],
                                    4242, 1, C.c_void_p(basis.data_ptr()), C.c_void_p(eig.data_ptr()), C.byref(total),
                                    C.c_void_p(mean.data_ptr()), C.byref(rank)))
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"fit_pca stream={mode}: {min(ts) * 1e3:.1f} ms (best of 3), all {[round(t * 1e3, 1) for t in ts]}", flush=True)
    eng.ctx.set_timing(True)
    eng.ctx.timing_reset()
    t0 = time.perf_counter()
    _lib.check(lib.svdk_fit_pca(eng.ctx.handle, C.c_void_p(host.data_ptr()), m, n, 1, mid, cfg["l"], cfg["q"],
                                4242, 1, C.c_void_p(basis.data_ptr()), C.c_void_p(eig.data_ptr()), C.byref(total),
                                C.c_void_p(mean.data_ptr()), C.byref(rank)))
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    print("   phases (device ms):", {k: round(eng.ctx.timing(k)["ms"], 2) for k in eng.ctx.timing_names()},
          f"wall {wall:.1f} ms", flush=True)
    eng.ctx.set_timing(False)
dev = torch.empty(n, m, dtype=torch.float64, device="cuda").t()
for label, chunk in (("contiguous", m), ("2-D chunks of 32768 rows", 32768)):
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for r0 in range(0, m, chunk):
            dev[r0:r0 + chunk].copy_(host[r0:r0 + chunk], non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    gb = 8 * m * n / 1e9
    print(f"H2D {label}: {min(ts) * 1e3:.1f} ms = {gb / min(ts):.1f} GB/s", flush=True)
