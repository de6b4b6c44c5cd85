"""Netlib's copy pattern without the GEMMs: B whole, then 8 chunks of A
H2D, each followed (after an event) by a D2H chunk of C; optionally a GEMM
between.  Timeline from the torch profiler.  Dev tool.
usage: python tools/copy_pattern_probe.py [gemm] [alt]   (alt: H2D chunks alternate between two streams)"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with_gemm = "gemm" in sys.argv[1:]
alt = "alt" in sys.argv[1:]
S, CH = 8192, 8
hA, hB, hC = (torch.empty(S * S, dtype=torch.float16, pin_memory=True) for _ in range(3))
dA, dB, dC = (torch.zeros(S * S, dtype=torch.float16, device="cuda") for _ in range(3))
h2d, d2h, h2d_b = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
cur = torch.cuda.current_stream()
rows = S // CH


def step():
    h2d.wait_stream(cur)
    h2d_b.wait_stream(cur)
    d2h.wait_stream(cur)
    with torch.cuda.stream(h2d):
        dB.copy_(hB, non_blocking=True)
    for i in range(CH):
        lo, hi = i * rows * S, (i + 1) * rows * S
        hs = h2d_b if (alt and i % 2) else h2d
        if alt and i == 1:
            h2d_b.wait_stream(h2d)  # after B
        with torch.cuda.stream(hs):
            dA[lo:hi].copy_(hA[lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(hs)
        cur.wait_event(ev)
        if with_gemm:
            torch.matmul(dA[lo:hi].view(rows, S), dB.view(S, S), out=dC[lo:hi].view(rows, S))
        d2h.wait_stream(cur)
        with torch.cuda.stream(d2h):
            hC[lo:hi].copy_(dC[lo:hi], non_blocking=True)
    cur.wait_stream(h2d)
    cur.wait_stream(h2d_b)
    cur.wait_stream(d2h)


for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    step()
e1.record()
torch.cuda.synchronize()
print(f"{'with' if with_gemm else 'without'} GEMM, alt={alt}: {e0.elapsed_time(e1) / 5:.3f} ms per step", flush=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in evs)
for e in sorted(evs, key=lambda e: e.time_range.start):
    s, f = e.time_range.start - t0, e.time_range.end - t0
    print(f"{s:9.1f} {f:9.1f} {f - s:8.1f} {e.name[:50]}")
