/*
 * oracle/gemm_seqk.c — TEST INFRASTRUCTURE ONLY (parity checker).
 *
 * Plain-C restatement of the reference GEMM semantics
 *   C = alpha * op(A) * op(B) + beta * C
 * (pkg/src/tunedblas/routines/level3.py:94-149 for the argument model,
 *  kernels/compute.py:408-412 / 458-463 for the epilogue,
 *  core.py:345-362 + level3.py:41-45 for the addressing of layouts,
 *  level3.py:125-132 for the alpha == 0 / k == 0 early-out)
 * with the summation order FIXED to a sequential-k FMA chain:
 *     acc = 0; for kk in 0..k-1: acc = fmaf(opA(i,kk), opB(kk,j), acc)
 * That order is the B200 SGEMM kernels' documented contract, so for
 * precision S this checker must agree with the GPU BITWISE; the reference's
 * own summation order is OpenBLAS-internal (np.matmul) and is matched only
 * to the reference tolerance (tests pin both).
 *
 * Precision H: FP16 inputs widened exactly to FP32, the same FP32 chain and
 * epilogue, one round-to-nearest-even to FP16 (level3.py:91).  Tensor cores
 * sum in their own order, so H is a tolerance checker.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library (oracle/_build/liboracle.so).
 *
 * Build: make -C oracle   (gcc -O2 -ffp-contract=off; fmaf is correctly rounded)
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* ---- IEEE binary16 <-> binary32 (exact widening, RNE narrowing) -------- */
static float h2f(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t exp = (h >> 10) & 0x1Fu;
  uint32_t man = h & 0x3FFu;
  uint32_t bits;
  if (exp == 0) {
    if (man == 0) {
      bits = sign;
    } else { /* subnormal: normalise */
      int e = -1;
      do { man <<= 1; ++e; } while ((man & 0x400u) == 0);
      man &= 0x3FFu;
      bits = sign | (uint32_t)(127 - 15 - e) << 23 | (man << 13);
    }
  } else if (exp == 0x1F) {
    bits = sign | 0x7F800000u | (man << 13);
  } else {
    bits = sign | (exp - 15 + 127) << 23 | (man << 13);
  }
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

static uint16_t f2h(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t absx = x & 0x7FFFFFFFu;
  if (absx >= 0x7F800000u) { /* inf / nan */
    return (uint16_t)(sign | 0x7C00u | (absx > 0x7F800000u ? 0x200u | ((absx >> 13) & 0x3FFu) : 0));
  }
  if (absx >= 0x477FF000u) return (uint16_t)(sign | 0x7C00u); /* rounds to >= 65520 -> inf */
  if (absx < 0x38800000u) {                                     /* half subnormal or zero */
    /* value = absx as float; scale to units of 2^-24 and round to nearest even */
    float a;
    memcpy(&a, &absx, 4);
    float scaled = a * 16777216.0f; /* exact (power of two) */
    float r = rintf(scaled);        /* default rounding mode: nearest-even */
    return (uint16_t)(sign | (uint32_t)r);
  }
  uint32_t exp = ((absx >> 23) - 127 + 15);
  uint32_t man = absx & 0x7FFFFFu;
  uint32_t h = (exp << 10) | (man >> 13);
  uint32_t rem = man & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h += 1; /* may carry into exponent: ok */
  return (uint16_t)(sign | h);
}

/* Element (i, j) of a logical rows x cols matrix stored in `layout`
 * (0 = column-major, 1 = row-major) with leading dimension ld. */
static int64_t at(int layout, int64_t i, int64_t j, int64_t ld) {
  return layout == 0 ? i + j * ld : i * ld + j;
}

static float epi(float alpha, float beta, int skip_ab, float acc, float cval) {
  if (skip_ab) return beta == 0.0f ? 0.0f : beta * cval;
  float v = alpha * acc;
  if (beta != 0.0f) {
    float t = beta * cval;
    v = v + t;
  }
  return v;
}

/*
 * prec: 0 = H (uint16 storage), 1 = S (float storage)
 * trans: 0 = NO, 1/2 = YES/CONJUGATE (identical for real types)
 * Offsets / ld in elements, exactly as the routine arguments.
 */
int oracle_gemm(int prec, int layout, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                float alpha, const void* a, int64_t a_off, int64_t lda, const void* b,
                int64_t b_off, int64_t ldb, float beta, void* c, int64_t c_off, int64_t ldc) {
  if (m < 0 || n < 0 || k < 0) return 1;
  if (m == 0 || n == 0) return 0;
  const int skip_ab = (k == 0 || alpha == 0.0f);
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = 0; i < m; ++i) {
      float acc = 0.0f;
      if (!skip_ab) {
        for (int64_t kk = 0; kk < k; ++kk) {
          /* op(A)(i,kk): stored A is (m,k) if NO else (k,m) */
          int64_t ia = trans_a == 0 ? at(layout, i, kk, lda) : at(layout, kk, i, lda);
          int64_t ib = trans_b == 0 ? at(layout, kk, j, ldb) : at(layout, j, kk, ldb);
          float av, bv;
          if (prec == 1) {
            av = ((const float*)a)[a_off + ia];
            bv = ((const float*)b)[b_off + ib];
          } else {
            av = h2f(((const uint16_t*)a)[a_off + ia]);
            bv = h2f(((const uint16_t*)b)[b_off + ib]);
          }
          acc = fmaf(av, bv, acc);
        }
      }
      int64_t ic = c_off + at(layout, i, j, ldc);
      if (prec == 1) {
        float* cp = (float*)c + ic;
        float cv = (beta != 0.0f) ? *cp : 0.0f;
        *cp = epi(alpha, beta, skip_ab, acc, cv);
      } else {
        uint16_t* cp = (uint16_t*)c + ic;
        float cv = (beta != 0.0f) ? h2f(*cp) : 0.0f;
        *cp = f2h(epi(alpha, beta, skip_ab, acc, cv));
      }
    }
  }
  return 0;
}

/* Strided batched: instance z uses offset + z * stride (extras.py:309-348). */
int oracle_gemm_strided_batched(int prec, int layout, int trans_a, int trans_b, int64_t m, int64_t n,
                                int64_t k, float alpha, const void* a, int64_t a_off, int64_t lda,
                                int64_t stride_a, const void* b, int64_t b_off, int64_t ldb,
                                int64_t stride_b, float beta, void* c, int64_t c_off, int64_t ldc,
                                int64_t stride_c, int64_t batch) {
  for (int64_t z = 0; z < batch; ++z) {
    int rc = oracle_gemm(prec, layout, trans_a, trans_b, m, n, k, alpha, a, a_off + z * stride_a, lda,
                         b, b_off + z * stride_b, ldb, beta, c, c_off + z * stride_c, ldc);
    if (rc) return rc;
  }
  return 0;
}

/* Exposed for tests of the conversion helpers. */
float oracle_h2f(uint16_t h) { return h2f(h); }
uint16_t oracle_f2h(float f) { return f2h(f); }
