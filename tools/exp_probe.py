"""eig_sym(n) timing + pair-solve clock64 stamps for a development build
(SVDK_LIB=build/exp<k>/libsvdk.so, see tools/exp_pair.sh); timing-only
variants may not converge, so a NumericalError is reported, not raised."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1906_12085_b200 import _lib  # noqa: E402
from paper_1906_12085_b200.engine import Engine, colmajor  # noqa: E402

eng = Engine(0)
torch.cuda.set_stream(eng.stream)
for n in [int(a) for a in sys.argv[1:]] or [256, 1024]:
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    s = colmajor(n, n, ld=n)
    s.copy_(x + x.t())
    ms, err, note = [], None, ""
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        try:
            w, v = eng.eig_sym(s)
        except Exception as ex:  # timing-only variants
            note = type(ex).__name__
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    if not note:
        ref = torch.linalg.eigvalsh(s.contiguous()).flip(0)
        err = float((w - ref).abs().max() / torch.linalg.norm(s))
    buf = (ctypes.c_longlong * 16)()
    _lib.load().svdk_debug_jacobi_probe(buf)
    st = list(buf)
    print(f"{os.environ.get('SVDK_LIB', 'prod')} n={n}: {min(ms):.2f} ms sweeps={eng.ctx.last_sweeps()} "
          f"err={err} {note} | CTA0 round5: load {st[1] - st[0]} inner {st[2] - st[1]} "
          f"(per inner round {(st[2] - st[1]) / 16:.0f}) LA entries {st[3]} rot {st[4]} to-bar {st[6]} bar {st[7]} "
          f"| from round start: LA look word landed {st[12]}, LA loads landed {st[11]}, M thread 0 done {st[9]}, Q lane 0 done {st[10]}",
          flush=True)
