"""The public routines are CUDA-graph capturable (no allocation, no host
sync on the call path; work is stream-ordered on the caller's stream): a
captured sequence replays with results identical to eager calls."""

import pytest

import paper_1705_05249_b200 as tb
from paper_1705_05249_b200 import Layout, Precision, Transpose

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", [Precision.H, Precision.S])
def test_gemm_and_batched_capture_replay(ctx, prec):
    import torch

    g = torch.Generator(device="cuda").manual_seed(4)
    m, n, k = 640, 384, 512
    dt = prec.torch_dtype
    a = tb.buffer_from_tensor(ctx, prec, (torch.rand(m * k, device="cuda", generator=g) * 2 - 1).to(dt))
    b = tb.buffer_from_tensor(ctx, prec, (torch.rand(k * n, device="cuda", generator=g) * 2 - 1).to(dt))
    c_eager, c_graph = tb.buffer_alloc(ctx, prec, m * n), tb.buffer_alloc(ctx, prec, m * n)
    s, e = 32, 32 * 32
    ab = tb.buffer_from_tensor(ctx, prec, (torch.rand(64 * e, device="cuda", generator=g) * 2 - 1).to(dt))
    bb = tb.buffer_from_tensor(ctx, prec, (torch.rand(64 * e, device="cuda", generator=g) * 2 - 1).to(dt))
    cb_eager, cb_graph = tb.buffer_alloc(ctx, prec, 64 * e), tb.buffer_alloc(ctx, prec, 64 * e)

    def work(c, cb):
        tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.YES, m, n, k, 1.0, a, b, 0.0, c, ldb=k)
        tb.gemm_strided_batched(ctx, Layout.COL_MAJOR, Transpose.NO, Transpose.NO, s, s, s, 0.5, ab, e,
                                bb, e, 0.0, cb, e, 64)

    work(c_eager, cb_eager)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        work(c_graph, cb_graph)          # warm-up on the capture stream
        torch.cuda.synchronize()
        c_graph.device_tensor().zero_()
        cb_graph.device_tensor().zero_()
        with torch.cuda.graph(graph, stream=stream):
            work(c_graph, cb_graph)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(c_graph.device_tensor(), c_eager.device_tensor())
    assert torch.equal(cb_graph.device_tensor(), cb_eager.device_tensor())


def test_capture_on_fresh_stream_large_hgemm_and_splitk(ctx):
    """capture on a stream that never ran a call before, with an
    HGEMM above the wave-barrier threshold (> 6 TFLOP: the pair kernel's
    counters) and a split-K HGEMM (its partial workspace): nothing may be
    allocated during capture.  The wave-barrier counters come from the
    per-device pool tb_prepare_device allocated when the context first
    launched, so the captured pair kernel keeps its barrier; the split-K
    workspace is per stream and absent, so the captured kernel exchanges
    partials through DSMEM.  The replay equals the eager calls bitwise (the
    per-element arithmetic does not depend on either)."""
    import torch

    prec = Precision.H
    g = torch.Generator(device="cuda").manual_seed(12)
    big_m, big_n, big_k = 16384, 12288, 16384            # 6.6 TFLOP: wave barrier on
    a = tb.buffer_from_tensor(ctx, prec, (torch.rand(big_m * big_k, device="cuda", generator=g) * 2 - 1).half())
    b = tb.buffer_from_tensor(ctx, prec, (torch.rand(big_k * big_n, device="cuda", generator=g) * 2 - 1).half())
    sm, sn, sk = 4096, 128, 9216                         # C3: cluster split-K
    a2 = tb.buffer_from_tensor(ctx, prec, (torch.rand(sm * sk, device="cuda", generator=g) * 2 - 1).half())
    b2 = tb.buffer_from_tensor(ctx, prec, (torch.rand(sk * sn, device="cuda", generator=g) * 2 - 1).half())

    def work(c, c2):
        tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, big_m, big_n, big_k, 1.0, a, b, 0.0, c)
        k1 = ctx.last_launch.native["kernel"]
        tb.gemm(ctx, Layout.ROW_MAJOR, Transpose.NO, Transpose.NO, sm, sn, sk, 1.0, a2, b2, 0.0, c2)
        return k1, ctx.last_launch.native["kernel"]

    c_e, c2_e = tb.buffer_alloc(ctx, prec, big_m * big_n), tb.buffer_alloc(ctx, prec, sm * sn)
    eager_kernels = work(c_e, c2_e)
    torch.cuda.synchronize()
    assert eager_kernels[0].endswith("_ws") and "splitk" in eager_kernels[1], eager_kernels
    c_g, c2_g = tb.buffer_alloc(ctx, prec, big_m * big_n), tb.buffer_alloc(ctx, prec, sm * sn)
    stream = torch.cuda.Stream()                         # fresh: no per-stream state yet
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        graph_kernels = work(c_g, c2_g)
    assert graph_kernels[0].endswith("_ws"), graph_kernels           # pooled counter, no allocation
    assert graph_kernels[1].endswith("_dsmem"), graph_kernels        # no workspace during capture
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(c_g.device_tensor(), c_e.device_tensor())
    assert torch.equal(c2_g.device_tensor(), c2_e.device_tensor())
