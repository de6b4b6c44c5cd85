import os, sys, subprocess
sizes = [(8192,), (32768,)]
for gm in (8, 16):
    for no2 in ("", "1"):
        env = dict(os.environ, TBGEMM_GROUP_M=str(gm))
        if no2: env["TBGEMM_NO_2SM"] = "1"
        out = subprocess.run([sys.executable, "-c", """
import sys, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200.kernels.dispatch import gemm_native
ctx = tb.context_create(tb.host_device())
T = tb.Transpose
cfg = tb.routines.common.get_store(ctx).resolve('gemm', tb.Precision.H, ctx.device, (1, 1, 1))[0]
for N in (8192, 32768):
    a = tb.buffer_from_tensor(ctx, tb.Precision.H, (torch.rand(N*N, device='cuda')*2-1).half())
    b = tb.buffer_from_tensor(ctx, tb.Precision.H, (torch.rand(N*N, device='cuda')*2-1).half())
    c = tb.buffer_alloc(ctx, tb.Precision.H, N*N)
    rec = {}
    fn = lambda: rec.update(gemm_native(ctx, tb.Precision.H, tb.Layout.ROW_MAJOR, T.NO, T.NO, N, N, N, 1.0, a, 0, N, b, 0, N, 0.0, c, 0, N, cfg))
    fn(); torch.cuda.synchronize()
    reps = 10 if N == 8192 else 2
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(N, rec['kernel'], f'{ms:.3f} ms', f'{2*N**3/ms/1e9:.1f} TFLOPS', flush=True)
    del a, b, c
    torch.cuda.empty_cache()
"""], env=env, capture_output=True, text=True).stdout
        for line in out.splitlines():
            print("gm", gm, "no2sm" if no2 else "2sm  ", line, flush=True)
