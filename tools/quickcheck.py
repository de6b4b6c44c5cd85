"""First-contact GPU check of libtbgemm.so (self-contained; dev tool)."""
import ctypes, sys, time
import numpy as np
import torch

so = ctypes.CDLL(sys.argv[1] if len(sys.argv) > 1 else "paper_1705_05249_b200/_lib/libtbgemm.so")
i32, i64, f32, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p
so.tb_gemm.restype = i32
so.tb_gemm.argtypes = [i32, i32, i32, i32, i64, i64, i64, f32, vp, i64, i64, vp, i64, i64, f32, vp, i64, i64, vp, i32, vp]
so.tb_last_error.restype = ctypes.c_char_p
class Rec(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_char * 64), ("grid", ctypes.c_int64 * 3), ("block", ctypes.c_int32 * 3),
                ("cluster", ctypes.c_int32 * 3), ("smem_bytes", ctypes.c_int32), ("launches", ctypes.c_int32), ("tiles", ctypes.c_int64)]

def run(prec, layout, ta, tb, m, n, k, alpha=1.0, beta=0.0, flags=0, pad=0):
    dt = torch.float16 if prec == 0 else torch.float32
    g = torch.Generator(device="cpu").manual_seed(m * 7 + n * 3 + k)
    ar, ac = (m, k) if ta == 0 else (k, m)
    br, bc = (k, n) if tb == 0 else (n, k)
    A = (torch.rand(ar, ac, generator=g) * 2 - 1).to(dt)
    B = (torch.rand(br, bc, generator=g) * 2 - 1).to(dt)
    C = (torch.rand(m, n, generator=g) * 2 - 1).to(dt)
    def store(X):  # flatten to layout storage, with ld = rows(col) or cols(row) + pad
        r, c = X.shape
        if layout == 0:
            ld = r + pad; buf = torch.zeros(ld * c, dtype=dt); buf.view(c, ld)[:, :r] = X.T
        else:
            ld = c + pad; buf = torch.zeros(ld * r, dtype=dt); buf.view(r, ld)[:, :c] = X
        return buf.cuda(), ld
    a, lda = store(A); b, ldb = store(B); c, ldc = store(C)
    opA = A.double() if ta == 0 else A.double().T
    opB = B.double() if tb == 0 else B.double().T
    want = alpha * (opA @ opB) + (beta * C.double() if beta != 0 else 0)
    st = so.tb_gemm(prec, layout, ta, tb, m, n, k, alpha, a.data_ptr(), 0, lda, b.data_ptr(), 0, ldb, beta,
                    c.data_ptr(), 0, ldc, None, flags, None)
    torch.cuda.synchronize()
    rec = Rec(); so.tb_last_launch(ctypes.byref(rec))
    if st != 0:
        return False, f"status {st} {so.tb_last_error().decode()}"
    cc = c.cpu()
    got = (cc.view(n, ldc)[:, :m].T if layout == 0 else cc.view(m, ldc)[:, :n]).double()
    eps = 2.0 ** -10 if prec == 0 else 2.0 ** -23
    tol = 4 * eps * k * (opA.abs().max(1).values[:, None] * opB.abs().max(0).values[None, :]) * abs(alpha) + 1e-6 + (2 * eps * abs(beta) if prec == 0 else 0)
    if prec == 0:
        tol = tol + 2.0 ** -11 * want.abs()
    err = (got - want).abs()
    ok = bool((err <= tol).all())
    return ok, f"{rec.kernel.decode()} maxerr={err.max().item():.3e} maxtol={tol.max().item():.3e}"

fails = 0
cases = []
for prec in (1, 0):
    for layout in (0, 1):
        for ta in (0, 1):
            for tb in (0, 1):
                cases.append((prec, layout, ta, tb, 200, 300, 130, 1.0, 0.0, 0, 0))
                cases.append((prec, layout, ta, tb, 257, 129, 77, 1.5, 0.5, 0, 0))
    cases.append((prec, 0, 0, 0, 1024, 1024, 1024, 1.0, 0.0, 0, 0))
    cases.append((prec, 1, 0, 0, 512, 512, 512, 1.0, 0.0, 0, 0))
    cases.append((prec, 0, 1, 0, 129, 129, 129, 1.0, 0.0, 0, 0))
    cases.append((prec, 0, 0, 0, 100, 70, 33, 1.0, 0.0, 0, 3))
    cases.append((prec, 1, 1, 1, 300, 200, 100, -1.0, 2.0, 0, 5))
for prec in (0,):
    for layout in (0, 1):
        for ta in (0, 1):
            for tb in (0, 1):
                cases.append((prec, layout, ta, tb, 256, 512, 192, 1.0, 0.0, 2, 0))
for cs in cases:
    try:
        ok, msg = run(*cs)
    except Exception as e:
        ok, msg = False, repr(e)
    fails += not ok
    print(("PASS" if ok else "FAIL"), cs, msg, flush=True)
print("FAILS", fails)

# quick timing
for prec, N in ((0, 8192), (1, 4096), (1, 8192)):
    dt = torch.float16 if prec == 0 else torch.float32
    a = torch.randn(N * N, device="cuda", dtype=dt); b = torch.randn(N * N, device="cuda", dtype=dt); c = torch.empty(N * N, device="cuda", dtype=dt)
    for _ in range(3):
        so.tb_gemm(prec, 1, 0, 0, N, N, N, 1.0, a.data_ptr(), 0, N, b.data_ptr(), 0, N, 0.0, c.data_ptr(), 0, N, None, 0, None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    R = 10
    for _ in range(R):
        so.tb_gemm(prec, 1, 0, 0, N, N, N, 1.0, a.data_ptr(), 0, N, b.data_ptr(), 0, N, 0.0, c.data_ptr(), 0, N, None, 0, None)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    rec = Rec(); so.tb_last_launch(ctypes.byref(rec))
    print(f"prec={prec} N={N} {rec.kernel.decode()} {ms:.3f} ms  {2*N**3/ms/1e9:.1f} TFLOPS", flush=True)
