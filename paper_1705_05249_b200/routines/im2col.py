"""``im2col`` on the GPU: the reference's routine
(pkg/src/tunedblas/routines/extras.py:56-109) with the same signature, checks,
error text and launch record, over the gather kernel in csrc/im2col.cuh.

The reference gathered the patches with NumPy and copied them through a
``copy_pad`` transform launch (extras.py:98-109 -> transforms.py:21-76); here
one CUDA kernel writes the column matrix straight into ``col``.  It is pure
data movement, so results are bit-identical to the reference.
"""

from __future__ import annotations

from ..core import Buffer, Context
from ..errors import UsageError
from ..kernels import native
from ..kernels.dispatch import prec_code, require_gpu
from ..kernels.engine import WorkGrid, launch_grid, pre_launch, record_launch, reference_grid
from .common import check_precision, get_store

__all__ = ["im2col", "im2col_geometry", "convgemm"]


def im2col_geometry(channels, height, width, kernel_h, kernel_w, pad_h, pad_w,
                    stride_h, stride_w, dilation_h, dilation_w) -> tuple[int, int, int, int]:
    """(out_h, out_w, rows, cols), with the reference's checks and messages
    in its order (extras.py:71-84)."""
    if channels < 1 or height < 1 or width < 1 or kernel_h < 1 or kernel_w < 1:
        raise UsageError("image and kernel dimensions must be >= 1")
    if stride_h < 1 or stride_w < 1 or dilation_h < 1 or dilation_w < 1:
        raise UsageError("strides and dilations must be >= 1")
    span_h = dilation_h * (kernel_h - 1) + 1
    span_w = dilation_w * (kernel_w - 1) + 1
    out_h = (height + 2 * pad_h - span_h) // stride_h + 1
    out_w = (width + 2 * pad_w - span_w) // stride_w + 1
    if out_h <= 0 or out_w <= 0:
        raise UsageError("convolution output dimensions are not positive")
    return out_h, out_w, channels * kernel_h * kernel_w, out_h * out_w


def im2col(ctx: Context, channels: int, height: int, width: int,
           kernel_h: int, kernel_w: int, pad_h: int, pad_w: int,
           stride_h: int, stride_w: int, dilation_h: int, dilation_w: int,
           im: Buffer, col: Buffer, *, im_offset: int = 0, col_offset: int = 0) -> None:
    """Rearrange image patches into columns so convolution becomes a matmul.

    The image is channel-major with row-major h x w planes.  The output is the
    (channels*kernel_h*kernel_w) x (out_h*out_w) column matrix, stored
    column-major, with column q = oy*out_w + ox holding the patch at output
    position (oy, ox); a weights-as-rows GEMM against it equals direct
    cross-correlation.  Asynchronous on the context's stream.
    """
    precision = im.precision
    check_precision(ctx, precision, im, col)
    out_h, out_w, rows, cols = im2col_geometry(
        channels, height, width, kernel_h, kernel_w, pad_h, pad_w,
        stride_h, stride_w, dilation_h, dilation_w)
    im.check_range(im_offset, channels * height * width)
    col.check_range(col_offset, rows * cols)
    pcode = prec_code(precision)  # H and S on this path

    store = get_store(ctx)
    cfg, _ = store.resolve("transform", precision, ctx.device, (rows, cols, 0))
    grid = launch_grid("transform", (max(rows, 1), max(cols, 1)), cfg)
    pre_launch(ctx, "transform", cfg, grid, precision)
    require_gpu(ctx)
    so = native.lib()
    st = so.tb_im2col(pcode, channels, height, width, kernel_h, kernel_w, pad_h, pad_w,
                      stride_h, stride_w, dilation_h, dilation_w, im.data_ptr(), im_offset,
                      col.data_ptr(), col_offset, ctx.stream_handle())
    col.mark_device_written()
    native.check(st, "tb_im2col")
    record_launch(ctx, "transform", cfg, grid, native.last_launch())


def convgemm(ctx: Context, channels: int, height: int, width: int,
             kernel_h: int, kernel_w: int, pad_h: int, pad_w: int,
             stride_h: int, stride_w: int, dilation_h: int, dilation_w: int,
             num_kernels: int, batch_count: int, im: Buffer, kernel: Buffer, result: Buffer, *,
             im_offset: int = 0, kernel_offset: int = 0, result_offset: int = 0) -> None:
    """Convolution as an implicit GEMM: for each of
    ``batch_count`` channel-major images,

        result[b][f][q] = sum_r kernel[f][r] * im2col(image_b)[r][q]

    — exactly ``im2col`` (same geometry, checks and column order) followed by
    the weights-as-rows GEMM its docstring describes (extras.py:56-66), but
    the column matrix is never materialised: the GEMM's A-operand producer
    gathers it from the image tile by tile (csrc/hgemm_tc.cuh
    conv_fill_tile, csrc/sgemm_simt.cuh simt_conv_stage).

    ``kernel`` holds num_kernels rows of channels*kernel_h*kernel_w weights
    (row-major); image b starts at im_offset + b*channels*height*width and
    its output plane block at result_offset + b*num_kernels*out_h*out_w
    (NCHW).  S results equal im2col + gemm bitwise (sequential-k chain); H
    accumulates in FP32 on the tensor cores and rounds once to FP16.
    Asynchronous on the context's stream.
    """
    precision = im.precision
    check_precision(ctx, precision, im, kernel, result)
    out_h, out_w, rows, cols = im2col_geometry(
        channels, height, width, kernel_h, kernel_w, pad_h, pad_w,
        stride_h, stride_w, dilation_h, dilation_w)
    if num_kernels < 0:
        raise UsageError("num_kernels must be >= 0")
    if batch_count < 1:
        raise UsageError("batch_count must be >= 1")
    im.check_range(im_offset, batch_count * channels * height * width)
    kernel.check_range(kernel_offset, num_kernels * rows)
    result.check_range(result_offset, batch_count * num_kernels * cols)
    pcode = prec_code(precision)
    if num_kernels == 0:
        return
    store = get_store(ctx)
    cfg, _ = store.resolve("gemm", precision, ctx.device, (cols, num_kernels, rows))
    grid1 = reference_grid("gemm", cols, num_kernels, cfg)
    grid = WorkGrid((batch_count,) + grid1.work_groups, grid1.work_group_size)
    pre_launch(ctx, "gemm", cfg, grid, precision)
    require_gpu(ctx)
    so = native.lib()
    st = so.tb_convgemm(pcode, channels, height, width, kernel_h, kernel_w, pad_h, pad_w,
                        stride_h, stride_w, dilation_h, dilation_w, num_kernels, batch_count,
                        im.data_ptr(), im_offset, kernel.data_ptr(), kernel_offset,
                        result.data_ptr(), result_offset, 0, ctx.stream_handle())
    result.mark_device_written()
    native.check(st, "tb_convgemm")
    record_launch(ctx, "convgemm", cfg, grid, native.last_launch())
