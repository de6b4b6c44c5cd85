"""Per-CTA phase timeline of the cluster split-K HGEMM (debug build with
-DTB_SPLITK_TIMING).  Build here:
    python tools/splitk_timeline.py --build
run on the GPU:
    python tools/splitk_timeline.py 4096 128 9216
or for convgemm (channels, height, width, filters; 3x3, pad 1):
    python tools/splitk_timeline.py conv 64 56 56 64
--build-tag X / --lib X build / load tools/dbg/libtbgemm_dbg_X.so (extra
-D flags after --defs, comma separated).
"""
import ctypes
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
def _opt(name, default=""):
    if name in sys.argv:
        i = sys.argv.index(name)
        v = sys.argv[i + 1]
        del sys.argv[i:i + 2]
        return v
    return default


TAG = _opt("--tag")
DEFS = [f"-D{d}" for d in _opt("--defs").split(",") if d]
DBG = ROOT / "tools" / "dbg" / (f"libtbgemm_dbg_{TAG}.so" if TAG else "libtbgemm_dbg.so")

if "--build" in sys.argv:
    sys.path.insert(0, str(ROOT))
    from paper_1705_05249_b200 import build_native as bn

    objs = []
    (ROOT / "tools" / "dbg").mkdir(exist_ok=True)
    for src in bn.SOURCES:
        obj = ROOT / "tools" / "dbg" / (src.stem + TAG + ".o")
        subprocess.run([bn.nvcc(), *bn.NVCC_FLAGS, "-DTB_SPLITK_TIMING", *DEFS, f"-I{ROOT / 'include'}", "-c", "-o",
                        str(obj), str(src)], check=True)
        objs.append(str(obj))
    subprocess.run([bn.nvcc(), *bn.ARCH, "-shared", "-o", str(DBG), *objs], check=True)
    print(DBG)
    sys.exit(0)

os.environ["TBGEMM_LIB"] = str(DBG)
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_1705_05249_b200 as tb  # noqa: E402
from paper_1705_05249_b200.kernels import native  # noqa: E402

conv = sys.argv[1] == "conv"
ctx = tb.context_create(tb.host_device())
prec = tb.Precision.H
if conv:
    ch, hh, ww, nf = (int(x) for x in sys.argv[2:6])
    im = tb.buffer_from_tensor(ctx, prec, (torch.rand(ch * hh * ww, device="cuda") * 2 - 1).half())
    kern = tb.buffer_from_tensor(ctx, prec, (torch.rand(nf * ch * 9, device="cuda") * 2 - 1).half())
    res = tb.buffer_alloc(ctx, prec, nf * hh * ww)
    ks = 0

    def call():
        tb.convgemm(ctx, ch, hh, ww, 3, 3, 1, 1, 1, 1, 1, 1, nf, 1, im, kern, res)
else:
    m, n, k = (int(x) for x in sys.argv[1:4])
    ks = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    a = tb.buffer_from_tensor(ctx, prec, (torch.rand(m * k, device="cuda") * 2 - 1).half())
    b = tb.buffer_from_tensor(ctx, prec, (torch.rand(k * n, device="cuda") * 2 - 1).half())
    c = tb.buffer_alloc(ctx, prec, m * n)

    def call():
        tb.gemm(ctx, tb.Layout.ROW_MAJOR, tb.Transpose.NO, tb.Transpose.NO, m, n, k, 1.0, a, b, 0.0, c)
if ks:
    store = tb.routines.common.get_store(ctx)
    store.set_override("gemm_b200", prec, ctx.device, (m, n, k), tb.Configuration.make(
        "gemm_b200", dict(MWG=128, NWG=128, KWG=64, STAGES=0, CTA_GROUP=1, SPLIT_K=ks, GROUP_M=0)))
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
so = native.lib()
so.tb_debug_splitk_times.restype = ctypes.c_int
so.tb_debug_splitk_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
for rep in range(3):
    flush_buf.fill_(1)
    clean.view(torch.int64).sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call()
    e1.record()
    torch.cuda.synchronize()
grid = ctx.last_launch.native["grid"][0]
buf = (ctypes.c_ulonglong * (grid * 16))()
so.tb_debug_splitk_times(buf, grid * 16)
import numpy as np  # noqa: E402

t = np.array(buf, dtype=np.float64).reshape(grid, 16)[:, :11]
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
print(f"{ctx.last_launch.native['kernel']} grid {grid}  event time {e0.elapsed_time(e1) * 1e3:.2f} us")
names = ["start", "cl_sync", "tma0", "data0", "last_kb", "mma_done", "red_full", "red_done", "end",
         "red_loads", "red_arrive"]
for i, nm in enumerate(names):
    col = rel[:, i]
    print(f"{nm:9s} min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f} us")
