"""cuBLAS (torch.matmul / torch.bmm) on the BASELINE shapes, timed like
bench.py (L2 flushed before every call, CUDA events): the library-GEMM
reference point for this repo's kernels.  Dev tool."""
import sys

import torch

flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=20):
    for _ in range(3):
        fn()
    ev = []
    for _ in range(reps):
        flush_buf.fill_(1)
        clean.view(torch.int64).sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return v[len(v) // 2]


torch.backends.cuda.matmul.allow_tf32 = False
for dt, name in ((torch.float16, "H"), (torch.float32, "S")):
    for (m, n, k, batch) in ((1024, 1024, 1024, 1), (4096, 128, 9216, 1), (64, 3136, 576, 1),
                             (8192, 8192, 8192, 1), (32, 32, 32, 16384), (64, 64, 64, 16384)):
        a = torch.rand(batch, m, k, device="cuda").to(dt)
        b = torch.rand(batch, k, n, device="cuda").to(dt)
        fn = (lambda: torch.matmul(a[0], b[0])) if batch == 1 else (lambda: torch.bmm(a, b))
        us = t(fn)
        fl = 2.0 * m * n * k * batch
        print(f"cuBLAS {name} {m}x{n}x{k} batch {batch}: {us:9.2f} us  {fl / us / 1e6:8.1f} TF/s", flush=True)
