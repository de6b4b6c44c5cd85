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
