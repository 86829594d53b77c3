/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE ONLY -- the CPU restatement of the reference's GEMM
 * hot path, used by tests/ (parity checker), __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg. Never linked into or called by the product.
 *
 * Parity pinned: tests/test_oracle.py checks this restatement bit-for-bit
 * against golden vectors produced by the unmodified reference library
 * (oracle/_ref, built from /root/reference/proj by oracle/Makefile; script
 * oracle/make_golden.py, fixtures tests/golden/).
 *
 * Restated from (reference paths under /root/reference/proj):
 *   runGemm<T>            src/kernels.cpp:445-558   acc = beta*C (skipped when
 *                         beta == 0, :463), then per element ascending k:
 *                         acc += (alpha * a_ik) * b_kj, separate multiply and
 *                         add (no FMA; the reference is built without -march),
 *                         stored in C's precision (:555-557).
 *   computePrecision      src/kernels.cpp:136-140   Double iff any operand is
 *                         Double, else Single (float).
 *   floatToHalf/halfToFloat include/gridmath/precision.hpp:42-100
 *   loadScalar/storeScalar  include/gridmath/precision.hpp:105-149
 * The 256-wide k-panels of the reference do not change the per-element
 * order (every element still accumulates k = 0..K-1 in order), so the
 * restatement is a plain triple loop. Compiled with -ffp-contract=off.
 *
 * FC-layer neighbours of the GEMM, same conventions:
 *   runElementwise<T>     src/kernels.cpp:741-815   relu / mulScalar / add /
 *                         sub / axpy / reluGrad / copy / biasAdd, T from
 *                         execElementwise :817-829
 *   runRowColSumDet<T>    src/kernels.cpp:570-614   ascending-index sums,
 *                         acc = acc + alpha * sum
 *   execSetConst          src/kernels.cpp:435-443   storeScalar<double>
 *
 * Precision tags: 0 half, 1 single, 2 double, 3 bf16 (bf16 is not a
 * reference type; it is widened exactly like half and stored RNE via float).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* precision.hpp:42-74: RNE; e >= 31 -> inf; subnormals by shifted RNE. */
uint16_t oracle_float_to_half(float f) {
  const uint32_t x = f2u(f);
  const uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t mant = x & 0x007FFFFFu;
  const int32_t exp = (int32_t)((x >> 23) & 0xFFu);
  if (exp == 255) {
    uint32_t m = mant >> 13;
    if (mant == 0) return (uint16_t)(sign | 0x7C00u);
    return (uint16_t)(sign | 0x7C00u | (m ? m : 1u));
  }
  const int32_t e = exp - 127 + 15;
  if (e >= 31) return (uint16_t)(sign | 0x7C00u);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    mant |= 0x00800000u;
    const int shift = 14 - e;
    const uint32_t out = mant >> shift;
    const uint32_t rem = mant & ((1u << shift) - 1u);
    const uint32_t half = 1u << (shift - 1);
    uint32_t r = out;
    if (rem > half || (rem == half && (out & 1u))) ++r;
    return (uint16_t)(sign | r);
  }
  {
    const uint32_t out = mant >> 13;
    const uint32_t rem = mant & 0x1FFFu;
    uint32_t h = sign | ((uint32_t)e << 10) | out;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
    return (uint16_t)h;
  }
}

/* precision.hpp:77-100. Restated bug-for-bug: for subnormal halves the
 * reference uses exponent 112 - shift where IEEE needs 113 - shift, so every
 * subnormal widens to half its IEEE value (the product keeps IEEE semantics;
 * see DESIGN.md "Known reference deviations"). */
float oracle_half_to_float(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu, out;
  if (e == 0) {
    if (m == 0) {
      out = sign;
    } else {
      int shift = 0;
      while (!(m & 0x400u)) { m <<= 1; ++shift; }
      m &= 0x3FFu;
      out = sign | ((uint32_t)(112 - shift) << 23) | (m << 13);
    }
  } else if (e == 31) {
    out = sign | 0x7F800000u | (m << 13);
  } else {
    out = sign | ((e + 112) << 23) | (m << 13);
  }
  return u2f(out);
}

/* Bulk variants (keep NaN payload bits intact, unlike a scalar ctypes round trip). */
void oracle_half_to_float_n(const uint16_t* in, float* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = oracle_half_to_float(in[i]);
}

void oracle_float_to_half_n(const float* in, uint16_t* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = oracle_float_to_half(in[i]);
}

uint16_t oracle_float_to_bf16(float f) {
  uint32_t u = f2u(f);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FFFu;
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float oracle_bf16_to_float(uint16_t b) { return u2f((uint32_t)b << 16); }

static double load_d(const void* base, int prec, size_t i) {
  switch (prec) {
    case 0: return (double)oracle_half_to_float(((const uint16_t*)base)[i]);
    case 1: return (double)((const float*)base)[i];
    case 2: return ((const double*)base)[i];
    default: return (double)oracle_bf16_to_float(((const uint16_t*)base)[i]);
  }
}

static float load_f(const void* base, int prec, size_t i) {
  switch (prec) {
    case 0: return oracle_half_to_float(((const uint16_t*)base)[i]);
    case 1: return ((const float*)base)[i];
    case 2: return (float)((const double*)base)[i];
    default: return oracle_bf16_to_float(((const uint16_t*)base)[i]);
  }
}

static void store_d(void* base, int prec, size_t i, double v) {
  switch (prec) {
    case 0: ((uint16_t*)base)[i] = oracle_float_to_half((float)v); break;
    case 1: ((float*)base)[i] = (float)v; break;
    case 2: ((double*)base)[i] = v; break;
    default: ((uint16_t*)base)[i] = oracle_float_to_bf16((float)v); break;
  }
}

/* C (m x n, row-major, pitch n) = alpha*op(A)*op(B) + beta*C, full images.
 * A is m x k (k x m when trans_a), B is k x n (n x k when trans_b).
 * rows [r0, r1) only (lets callers sample rows of a large product). */
int oracle_gemm(uint64_t m, uint64_t n, uint64_t k, const void* a, int pa, const void* b, int pb,
                void* c, int pc, double alpha, double beta, int trans_a, int trans_b,
                uint64_t r0, uint64_t r1) {
  const int dbl = (pa == 2 || pb == 2 || pc == 2);
  if (r1 > m) r1 = m;
  for (uint64_t i = r0; i < r1; ++i) {
    for (uint64_t j = 0; j < n; ++j) {
      const size_t ci = (size_t)(i * n + j);
      if (dbl) {
        double acc = 0.0;
        if (beta != 0.0) acc = beta * load_d(c, pc, ci);
        if (alpha != 0.0)
          for (uint64_t kk = 0; kk < k; ++kk) {
            const double av = load_d(a, pa, (size_t)(trans_a ? kk * m + i : i * k + kk));
            const double bv = load_d(b, pb, (size_t)(trans_b ? j * k + kk : kk * n + j));
            const double aa = alpha * av;
            const double prod = aa * bv;
            acc = acc + prod;
          }
        store_d(c, pc, ci, acc);
      } else {
        const float al = (float)alpha, be = (float)beta;
        float acc = 0.0f;
        if (be != 0.0f) acc = be * load_f(c, pc, ci);
        if (al != 0.0f)
          for (uint64_t kk = 0; kk < k; ++kk) {
            const float av = load_f(a, pa, (size_t)(trans_a ? kk * m + i : i * k + kk));
            const float bv = load_f(b, pb, (size_t)(trans_b ? j * k + kk : kk * n + j));
            const float aa = al * av;
            const float prod = aa * bv;
            acc = acc + prod;
          }
        store_d(c, pc, ci, (double)acc);
      }
    }
  }
  return 0;
}

/* SplitMix64 draw i of seed (common.hpp:37-50) -> U[lo, hi) -> storage. */
static uint64_t avalanche64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

void oracle_fill_uniform(void* dst, int prec, uint64_t rows, uint64_t cols, uint64_t seed,
                         double lo, double hi) {
  for (uint64_t i = 0; i < rows * cols; ++i) {
    const uint64_t x = avalanche64(seed + (i + 1) * 0x9E3779B97F4A7C15ull);
    const double u = (double)(x >> 11) * 0x1.0p-53;
    store_d(dst, prec, (size_t)i, lo + (hi - lo) * u);
  }
}

/* layout.cpp:13-27: near-equal split, earliest parts take the remainder. */
uint32_t oracle_split(uint64_t n, uint64_t parts, uint64_t* starts, uint64_t* lens) {
  uint32_t cnt = 0;
  uint64_t at = 0;
  for (uint64_t p = 0; p < parts; ++p) {
    const uint64_t len = n / parts + (p < n % parts ? 1 : 0);
    if (len == 0) continue;
    starts[cnt] = at;
    lens[cnt] = len;
    at += len;
    ++cnt;
  }
  return cnt;
}

/* ---- FC-layer neighbours ---------------------------------------------- */

static void store_f(void* base, int prec, size_t i, float v) { store_d(base, prec, i, (double)v); }

/* Elementwise op over full row-major images (kernels.cpp:741-815).
 * unary: kind 0 Relu, 1 MulScalar (y unused). binary: kind 0 Add, 1 Sub,
 * 2 Axpy (alpha*x + y), 3 ReluGrad (x > 0 ? y : 0), 4 Copy, 5 BiasAdd
 * (x + y[0, j], y is 1 x cols). Compute type: Double iff any of x, y (binary
 * only), dst is Double (:817-829). dst may alias x or y (elementwise). */
void oracle_elementwise(int unary, int kind, double alpha, uint64_t rows, uint64_t cols,
                        const void* x, int xp, const void* y, int yp, void* dst, int dp) {
  const int dbl = xp == 2 || dp == 2 || (!unary && yp == 2);
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t j = 0; j < cols; ++j) {
      const size_t e = (size_t)(i * cols + j);
      const size_t ye = (!unary && kind == 5) ? (size_t)j : e;
      if (dbl) {
        const double xv = load_d(x, xp, e);
        double out;
        if (unary) {
          out = kind == 0 ? (xv > 0.0 ? xv : 0.0) : alpha * xv;
        } else {
          const double yv = kind == 4 ? 0.0 : load_d(y, yp, ye);
          switch (kind) {
            case 0: out = xv + yv; break;
            case 1: out = xv - yv; break;
            case 2: { const double ax = alpha * xv; out = ax + yv; break; }
            case 3: out = xv > 0.0 ? yv : 0.0; break;
            case 5: out = xv + yv; break;
            default: out = xv; break;
          }
        }
        store_d(dst, dp, e, out);
      } else {
        const float al = (float)alpha;
        const float xv = load_f(x, xp, e);
        float out;
        if (unary) {
          out = kind == 0 ? (xv > 0.0f ? xv : 0.0f) : al * xv;
        } else {
          const float yv = kind == 4 ? 0.0f : load_f(y, yp, ye);
          switch (kind) {
            case 0: out = xv + yv; break;
            case 1: out = xv - yv; break;
            case 2: { const float ax = al * xv; out = ax + yv; break; }
            case 3: out = xv > 0.0f ? yv : 0.0f; break;
            case 5: out = xv + yv; break;
            default: out = xv; break;
          }
        }
        store_f(dst, dp, e, out);
      }
    }
}

/* Deterministic addRowColSum (kernels.cpp:570-614): racc[i] += alpha *
 * sum_j a[i][j], then cacc[j] += alpha * sum_i a[i][j], each sum in
 * ascending index order in T. racc is rows x 1, cacc is 1 x cols. */
void oracle_row_col_sum(double alpha, uint64_t rows, uint64_t cols, const void* a, int ap,
                        void* racc, int rp, void* cacc, int cp) {
  const int dbl = ap == 2 || rp == 2 || cp == 2;
  for (uint64_t i = 0; i < rows; ++i) {
    if (dbl) {
      double sum = 0.0;
      for (uint64_t j = 0; j < cols; ++j) sum += load_d(a, ap, (size_t)(i * cols + j));
      const double cur = load_d(racc, rp, (size_t)i), add = alpha * sum;
      store_d(racc, rp, (size_t)i, cur + add);
    } else {
      float sum = 0.0f;
      for (uint64_t j = 0; j < cols; ++j) sum += load_f(a, ap, (size_t)(i * cols + j));
      const float cur = load_f(racc, rp, (size_t)i), add = (float)alpha * sum;
      store_f(racc, rp, (size_t)i, cur + add);
    }
  }
  for (uint64_t j = 0; j < cols; ++j) {
    if (dbl) {
      double sum = 0.0;
      for (uint64_t i = 0; i < rows; ++i) sum += load_d(a, ap, (size_t)(i * cols + j));
      const double cur = load_d(cacc, cp, (size_t)j), add = alpha * sum;
      store_d(cacc, cp, (size_t)j, cur + add);
    } else {
      float sum = 0.0f;
      for (uint64_t i = 0; i < rows; ++i) sum += load_f(a, ap, (size_t)(i * cols + j));
      const float cur = load_f(cacc, cp, (size_t)j), add = (float)alpha * sum;
      store_f(cacc, cp, (size_t)j, cur + add);
    }
  }
}

/* execSetConst (kernels.cpp:435-443): storeScalar<double>(value). */
void oracle_set_const(void* dst, int prec, uint64_t n, double value) {
  for (uint64_t i = 0; i < n; ++i) store_d(dst, prec, (size_t)i, value);
}
