"""Netlib's copy pattern without the GEMMs: B whole, then 8 chunks of A
H2D, each followed (after an event) by a D2H chunk of C; optionally a GEMM
between.  Timeline from the torch profiler.  Dev tool.
usage: python tools/copy_pattern_probe.py [gemm] [alt]   (alt: H2D chunks alternate between two streams)"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with_gemm = "gemm" in sys.argv[1:]
elementwise = "ew" in sys.argv[1:]
ours = "tb" in sys.argv[1:] or "tb1" in sys.argv[1:]  # this library's GEMM (tb1: single-CTA kernel, no cluster)  # a plain (non-cluster) elementwise kernel instead of the GEMM
alt = "alt" in sys.argv[1:]
xy = "xy" in sys.argv[1:]  # each chunk's GEMM on its own copy stream (two alternating), no event wait
S, CH = 8192, 8
hA, hB, hC = (torch.empty(S * S, dtype=torch.float16, pin_memory=True) for _ in range(3))
dA, dB, dC = (torch.zeros(S * S, dtype=torch.float16, device="cuda") for _ in range(3))
h2d, d2h, h2d_b = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
cur = torch.cuda.current_stream()
rows = S // CH
if ours:
    import paper_1705_05249_b200 as tb
    from paper_1705_05249_b200.kernels import native
    from paper_1705_05249_b200.kernels.dispatch import gemm_native
    ctx = tb.context_create(tb.host_device())
    H = tb.Precision.H
    ba, bb, bc = (tb.buffer_from_tensor(ctx, H, x) for x in (dA, dB, dC))
    flags = native.FLAG_NO_2SM if "tb1" in sys.argv[1:] else 0

    def tb_gemm(r0, r1):
        gemm_native(ctx, H, tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.NO, r1 - r0, S, S, 1.0, ba, r0 * S, S,
                    bb, 0, S, 0.0, bc, r0 * S, S, None, flags)


def step():
    h2d.wait_stream(cur)
    h2d_b.wait_stream(cur)
    d2h.wait_stream(cur)
    with torch.cuda.stream(h2d):
        dB.copy_(hB, non_blocking=True)
    for i in range(CH):
        lo, hi = i * rows * S, (i + 1) * rows * S
        hs = h2d_b if ((alt or xy) and i % 2) else h2d
        if (alt or xy) and i == 1:
            h2d_b.wait_stream(h2d)  # after B
        with torch.cuda.stream(hs):
            dA[lo:hi].copy_(hA[lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(hs)
        if xy:
            with torch.cuda.stream(hs):
                torch.matmul(dA[lo:hi].view(rows, S), dB.view(S, S), out=dC[lo:hi].view(rows, S))
                ev = torch.cuda.Event()
                ev.record(hs)
            d2h.wait_event(ev)
        else:
            cur.wait_event(ev)
            if with_gemm:
                torch.matmul(dA[lo:hi].view(rows, S), dB.view(S, S), out=dC[lo:hi].view(rows, S))
            if ours:
                tb_gemm(lo // S, hi // S)
            if elementwise:
                torch.mul(dA[lo:hi], 2.0, out=dC[lo:hi])
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
print(f"{'with' if with_gemm else 'without'} GEMM, ew={elementwise}, alt={alt} xy={xy}: {e0.elapsed_time(e1) / 5:.3f} ms per step", flush=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in evs)
for e in sorted(evs, key=lambda e: e.time_range.start):
    s, f = e.time_range.start - t0, e.time_range.end - t0
    print(f"{s:9.1f} {f:9.1f} {f - s:8.1f} {e.name[:50]}")
