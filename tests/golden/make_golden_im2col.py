"""Generate golden im2col vectors by running the REFERENCE implementation.

Run in the build container (needs /root/reference, absent on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_im2col.py

Writes tests/golden/im2col_golden.npz + im2col_golden.json: per case the
image buffer, the routine arguments, and the whole output buffer the
reference's ``tunedblas.im2col`` (extras.py:56-109) produced from a
sentinel-filled ``col`` (so untouched regions are pinned too).
"""

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tunedblas as tb  # noqa: E402  (the reference, read-only)

OUT = Path(__file__).resolve().parent
SENTINEL = 7.25  # exactly representable in FP16 and FP32


def main():
    ctx = tb.context_create(tb.host_device())
    rng = np.random.default_rng(20240607)
    P = {"S": tb.Precision.S, "H": tb.Precision.H}
    cases, arrays = [], {}

    def add(prec, c, h, w, kh, kw, ph, pw, sh, sw, dh, dw, im_off=0, col_off=0):
        dt = P[prec].dtype
        span_h, span_w = dh * (kh - 1) + 1, dw * (kw - 1) + 1
        oh = (h + 2 * ph - span_h) // sh + 1
        ow = (w + 2 * pw - span_w) // sw + 1
        rows, cols = c * kh * kw, oh * ow
        im = rng.uniform(-1, 1, im_off + c * h * w + 5).astype(dt)
        col = np.full(col_off + rows * cols + 5, SENTINEL, dt)
        ib = tb.buffer_alloc(ctx, P[prec], im.size)
        ib.data[:] = im
        cb = tb.buffer_alloc(ctx, P[prec], col.size)
        cb.data[:] = col
        tb.im2col(ctx, c, h, w, kh, kw, ph, pw, sh, sw, dh, dw, ib, cb,
                  im_offset=im_off, col_offset=col_off)
        i = len(cases)
        arrays[f"i{i}_im"] = im
        arrays[f"i{i}_col_in"] = col
        arrays[f"i{i}_col_out"] = cb.data.copy()
        cases.append(dict(prec=prec, c=c, h=h, w=w, kh=kh, kw=kw, ph=ph, pw=pw, sh=sh, sw=sw,
                          dh=dh, dw=dw, im_off=im_off, col_off=col_off, rows=rows, cols=cols,
                          out_h=oh, out_w=ow))

    for prec in ("S", "H"):
        # geometries of the reference's own tests (tests/test_extras.py:78-138)
        add(prec, 2, 3, 4, 1, 1, 0, 0, 1, 1, 1, 1)
        add(prec, 1, 4, 4, 3, 3, 0, 0, 1, 1, 1, 1)
        add(prec, 1, 3, 3, 3, 3, 1, 1, 1, 1, 1, 1)
        add(prec, 3, 7, 8, 3, 2, 1, 0, 2, 1, 2, 1)
        # random cases in the style of routine_cases.case_im2col (793-819)
        for _ in range(6):
            c, h, w = int(rng.integers(1, 4)), int(rng.integers(3, 9)), int(rng.integers(3, 9))
            kh, kw = int(rng.integers(1, min(4, h + 1))), int(rng.integers(1, min(4, w + 1)))
            ph, pw = int(rng.integers(0, 2)), int(rng.integers(0, 2))
            sh, sw = int(rng.integers(1, 3)), int(rng.integers(1, 3))
            if (h + 2 * ph - kh) // sh + 1 <= 0 or (w + 2 * pw - kw) // sw + 1 <= 0:
                continue
            add(prec, c, h, w, kh, kw, ph, pw, sh, sw, 1, 1)
        # offsets, negative padding (cropping), larger planes, dilation > 1
        add(prec, 2, 9, 11, 3, 3, 1, 2, 2, 3, 1, 2, im_off=13, col_off=7)
        add(prec, 3, 10, 10, 2, 2, -1, 0, 1, 2, 1, 1, im_off=4, col_off=9)
        add(prec, 8, 20, 17, 3, 3, 1, 1, 2, 2, 2, 2)
        add(prec, 5, 33, 40, 5, 4, 2, 1, 1, 1, 1, 1)
        add(prec, 1, 1, 64, 1, 7, 0, 3, 1, 1, 1, 1)

    np.savez_compressed(OUT / "im2col_golden.npz", **arrays)
    (OUT / "im2col_golden.json").write_text(json.dumps({"sentinel": SENTINEL, "cases": cases}, indent=1))
    print(f"wrote {len(cases)} im2col cases")


if __name__ == "__main__":
    main()
