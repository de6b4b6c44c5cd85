"""PCIe copy rates on the box (pinned host memory, CUDA events): H2D 256 MB,
D2H 128 MB, both at once on two streams; then netlib_call HGEMM 8192^3 on
pinned arrays (the bench's e2e).  Dev tool."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.routines import netlib  # noqa: E402

h_in = torch.empty(128 << 20, dtype=torch.float16, pin_memory=True)
h_out = torch.empty(64 << 20, dtype=torch.float16, pin_memory=True)
d_in = torch.empty(128 << 20, dtype=torch.float16, device="cuda")
d_out = torch.empty(64 << 20, dtype=torch.float16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t = timed(h2d)
print(f"H2D 256 MB: {t:.3f} ms  {256 / 1024 / t * 1e3:.1f} GB/s", flush=True)


def h2d_two():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    half = h_in.numel() // 2
    with torch.cuda.stream(s1):
        d_in[:half].copy_(h_in[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        d_in[half:].copy_(h_in[half:], non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t = timed(h2d_two)
print(f"H2D 256 MB as two halves on two streams: {t:.3f} ms  {256 / 1024 / t * 1e3:.1f} GB/s", flush=True)
t = timed(d2h)
print(f"D2H 128 MB: {t:.3f} ms  {128 / 1024 / t * 1e3:.1f} GB/s", flush=True)
t = timed(both)
print(f"H2D 256 MB + D2H 128 MB concurrently: {t:.3f} ms", flush=True)

S = 8192
ctx = tb.context_create(tb.host_device())
H = tb.Precision.H
ha, hb, hc = (netlib.pinned_empty(S * S, H) for _ in range(3))
ha[:] = 0.5
hb[:] = 0.25
for chunk_mb, maxc in ((32, 8), (16, 16), (8, 32)):
    netlib.CHUNK_BYTES, netlib.MAX_CHUNKS = chunk_mb << 20, maxc

    def step():
        tb.netlib_call("hgemm", tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.NO, S, S, S, 1.0, ha, hb, 0.0, hc,
                       ctx=ctx)
    t = timed(step, reps=6)
    print(f"netlib hgemm 8192^3 pinned, chunks of {chunk_mb} MB (max {maxc}): {t:.3f} ms  "
          f"{2 * S ** 3 / t / 1e9:.1f} TFLOP/s", flush=True)
