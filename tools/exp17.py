"""Timing of the structured level-3 routines (events around the whole routine)."""
import sys, torch
sys.path.insert(0, '.')
import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Side, Triangle, Transpose, Diagonal
ctx = tb.context_create(tb.host_device())
COL = Layout.COL_MAJOR
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3
for prec in (tb.Precision.H, tb.Precision.S):
    n = 4096
    dt = prec.torch_dtype
    mk = lambda cnt: tb.buffer_from_tensor(ctx, prec, (torch.rand(cnt, device='cuda') * 2 - 1).to(dt))
    a, b, c = mk(n * n), mk(n * n), mk(n * n)
    # well-conditioned triangular A for trsm: scale off-diagonals, big diagonal
    at = torch.rand(n, n, device='cuda') * 2 - 1
    at = at / n ** 0.5
    at.diagonal().add_(2.0)
    atri = tb.buffer_from_tensor(ctx, prec, at.to(dt).reshape(-1))
    gemm_s = t(lambda: tb.gemm(ctx, COL, Transpose.NO, Transpose.NO, n, n, n, 1.0, a, b, 0.0, c))
    symm_s = t(lambda: tb.symm(ctx, COL, Side.LEFT, Triangle.UPPER, n, n, 1.0, a, b, 0.0, c))
    syrk_s = t(lambda: tb.syrk(ctx, COL, Triangle.LOWER, Transpose.NO, n, n, 1.0, a, 0.0, c))
    syr2k_s = t(lambda: tb.syr2k(ctx, COL, Triangle.LOWER, Transpose.NO, n, n, 1.0, a, b, 0.0, c))
    trmm_s = t(lambda: tb.trmm(ctx, COL, Side.LEFT, Triangle.LOWER, Transpose.NO, Diagonal.NON_UNIT, n, n, 1.0, a, b))
    trsm_s = t(lambda: tb.trsm(ctx, COL, Side.LEFT, Triangle.LOWER, Transpose.NO, Diagonal.NON_UNIT, n, n, 1.0, atri, b), 2)
    f = 2 * n ** 3
    print(f"{prec.value} n={n}: gemm {gemm_s*1e3:.3f} ms ({f/gemm_s/1e12:.0f} TF) | symm {symm_s*1e3:.3f} ms ({f/symm_s/1e12:.0f}) | "
          f"syrk {syrk_s*1e3:.3f} ms ({n**3/syrk_s/1e12:.0f} useful TF) | syr2k {syr2k_s*1e3:.3f} ms | "
          f"trmm {trmm_s*1e3:.3f} ms ({n**3/trmm_s/1e12:.0f} useful) | trsm {trsm_s*1e3:.2f} ms ({n**3/trsm_s/1e12:.1f} useful TF)", flush=True)
