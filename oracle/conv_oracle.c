/*
 * TEST INFRASTRUCTURE ONLY — the CPU fp32 checker for super-kernel activations.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * Restates the operator semantics the reference models but never computes
 * (it has no tensor numerics: SURVEY §0, "activation parity unpinned"):
 *   - conv lowered to its im2col GEMM: rows = output positions (n, p, q),
 *     cols = C_out, inner = the unrolled (r, s, c) filter patch
 *     (proj/include/gpumux/gemm.hpp:42-51), input batching multiplies the rows
 *     (gemm.hpp:54-56);
 *   - GEMM C[m, n] = sum_k A[m, k] * B[n, k]  (gemm.hpp:11-16, B stored K-major).
 * Layouts match the product: X NHWC, W KRSC with row stride ldw, Y NHWC.
 * Accumulation is in double, so the oracle is at least as accurate as any fp32
 * reference path; inputs are the same bf16-rounded values the GPU reads.
 * Cross-checked against torch.nn.functional.conv2d in tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* Round-to-nearest-even fp32 -> bf16 -> fp32 (the rounding torch applies in
 * tensor.to(torch.bfloat16)); NaN stays NaN. */
void oracle_round_bf16(float* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u;
    memcpy(&u, &v[i], 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) continue;
    const uint32_t lsb = (u >> 16) & 1u;
    u = (u + 0x7fffu + lsb) & 0xffff0000u;
    memcpy(&v[i], &u, 4);
  }
}

/* y[b, p, q, o] = sum_{r,s,c} x[b, p*st - pad + r, q*st - pad + s, c] * w[o, (r*S + s)*Cin + c] */
void oracle_conv2d_nhwc(const float* x, const float* w, float* y, int64_t batch, int64_t H, int64_t W,
                        int64_t Cin, int64_t Cout, int64_t R, int64_t S, int64_t stride, int64_t pad,
                        int64_t ldw, int32_t relu) {
  const int64_t P = (H + 2 * pad - R) / stride + 1;
  const int64_t Q = (W + 2 * pad - S) / stride + 1;
  if (ldw <= 0) ldw = R * S * Cin;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t b = 0; b < batch; ++b) {
    for (int64_t p = 0; p < P; ++p) {
      for (int64_t q = 0; q < Q; ++q) {
        float* out = y + ((b * P + p) * Q + q) * Cout;
        for (int64_t o = 0; o < Cout; ++o) {
          double acc = 0.0;
          const float* wo = w + o * ldw;
          for (int64_t r = 0; r < R; ++r) {
            const int64_t ih = p * stride - pad + r;
            if (ih < 0 || ih >= H) continue;
            for (int64_t s = 0; s < S; ++s) {
              const int64_t iw = q * stride - pad + s;
              if (iw < 0 || iw >= W) continue;
              const float* xi = x + ((b * H + ih) * W + iw) * Cin;
              const float* wi = wo + (r * S + s) * Cin;
              for (int64_t c = 0; c < Cin; ++c) acc += (double)xi[c] * (double)wi[c];
            }
          }
          float v = (float)acc;
          out[o] = (relu && v < 0.0f) ? 0.0f : v;
        }
      }
    }
  }
}

/* c[m, n] = sum_k a[m*lda + k] * b[n*ldb + k] */
void oracle_gemm_nt(const float* a, const float* b, float* c, int64_t M, int64_t N, int64_t K, int64_t lda,
                    int64_t ldb, int32_t relu) {
  if (lda <= 0) lda = K;
  if (ldb <= 0) ldb = K;
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < M; ++m) {
    for (int64_t n = 0; n < N; ++n) {
      double acc = 0.0;
      const float* am = a + m * lda;
      const float* bn = b + n * ldb;
      for (int64_t k = 0; k < K; ++k) acc += (double)am[k] * (double)bn[k];
      float v = (float)acc;
      c[m * N + n] = (relu && v < 0.0f) ? 0.0f : v;
    }
  }
}

/* Explicit im2col of one NHWC tensor into [M, ldk] rows (zero padding),
 * k = (r*S + s)*Cin + c — the layout the GPU pre-pass writes. */
void oracle_im2col_nhwc(const float* x, float* out, int64_t batch, int64_t H, int64_t W, int64_t Cin, int64_t R,
                        int64_t S, int64_t stride, int64_t pad, int64_t ldk) {
  const int64_t P = (H + 2 * pad - R) / stride + 1;
  const int64_t Q = (W + 2 * pad - S) / stride + 1;
  const int64_t K = R * S * Cin;
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < batch * P * Q; ++m) {
    const int64_t b = m / (P * Q), p = (m / Q) % P, q = m % Q;
    float* row = out + m * ldk;
    for (int64_t k = 0; k < ldk; ++k) row[k] = 0.0f;
    for (int64_t r = 0; r < R; ++r)
      for (int64_t s = 0; s < S; ++s) {
        const int64_t ih = p * stride - pad + r, iw = q * stride - pad + s;
        if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
        memcpy(row + (r * S + s) * Cin, x + ((b * H + ih) * W + iw) * Cin, (size_t)Cin * sizeof(float));
      }
    (void)K;
  }
}

/* Depthwise conv (groups = C): y[b, p, q, c] = sum_{r,s} x[b, p*st - pad + r, q*st - pad + s, c] * w[c*ldw + r*S + s].
 * The reference models it only as a K = R*S GEMM (proj/src/workload.cpp:66: (M, C, 9)); the
 * semantics restated here are torchvision's MobileNet-v2 depthwise 3x3 (conv2d, groups = C). */
void oracle_dwconv2d_nhwc(const float* x, const float* w, float* y, int64_t batch, int64_t H, int64_t W, int64_t C,
                          int64_t R, int64_t S, int64_t stride, int64_t pad, int64_t ldw, int32_t relu) {
  const int64_t P = (H + 2 * pad - R) / stride + 1;
  const int64_t Q = (W + 2 * pad - S) / stride + 1;
  if (ldw <= 0) ldw = R * S;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t b = 0; b < batch; ++b) {
    for (int64_t p = 0; p < P; ++p) {
      for (int64_t q = 0; q < Q; ++q) {
        float* out = y + ((b * P + p) * Q + q) * C;
        for (int64_t c = 0; c < C; ++c) {
          double acc = 0.0;
          for (int64_t r = 0; r < R; ++r) {
            const int64_t ih = p * stride - pad + r;
            if (ih < 0 || ih >= H) continue;
            for (int64_t s = 0; s < S; ++s) {
              const int64_t iw = q * stride - pad + s;
              if (iw < 0 || iw >= W) continue;
              acc += (double)x[((b * H + ih) * W + iw) * C + c] * (double)w[c * ldw + r * S + s];
            }
          }
          float v = (float)acc;
          out[c] = (relu && v < 0.0f) ? 0.0f : v;
        }
      }
    }
  }
}

/* ---------------------------------------------------------------------------
 * Dataflow operators (a tenant graph where each layer reads an earlier
 * layer's output): fused residual add and activation, pooling, and row
 * sampling for the large configurations.
 *
 *   y[m, o] = act(sum(...) + res[m * ldr + o])   (res == NULL: no add)
 *   act: 0 none, 1 relu, 2 relu6 (MobileNet-v2), 3 gelu (erf form, BERT FFN)
 *   rows: the output rows m to compute (y then holds n_rows rows, in order);
 *         rows == NULL computes every row (y holds all M rows).
 * The residual add and activation are the torchvision block semantics
 * (ResNet: relu(conv3(x) + identity/downsample); MobileNet-v2: project(x) + x);
 * pooling is torch.nn.MaxPool2d (padded taps ignored) / AvgPool2d (global, no
 * padding).  The reference models none of these (it has no tensors). */

static float oracle_act(double v, int32_t act) {
  if (act == 1) return v < 0.0 ? 0.0f : (float)v;
  if (act == 2) return v < 0.0 ? 0.0f : (v > 6.0 ? 6.0f : (float)v);
  if (act == 3) return (float)(0.5 * v * (1.0 + erf(v * 0.70710678118654752440)));
  return (float)v;
}

void oracle_conv2d_ex(const float* x, const float* w, const float* res, int64_t ldr, float* y, const int64_t* rows,
                      int64_t n_rows, int64_t batch, int64_t H, int64_t W, int64_t Cin, int64_t Cout, int64_t R,
                      int64_t S, int64_t stride, int64_t pad, int64_t ldw, int32_t act) {
  const int64_t P = (H + 2 * pad - R) / stride + 1;
  const int64_t Q = (W + 2 * pad - S) / stride + 1;
  const int64_t M = batch * P * Q;
  if (ldw <= 0) ldw = R * S * Cin;
  if (ldr <= 0) ldr = Cout;
  const int64_t n = rows ? n_rows : M;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t m = rows ? rows[i] : i;
    const int64_t b = m / (P * Q), p = (m / Q) % P, q = m % Q;
    float* out = y + i * Cout;
    for (int64_t o = 0; o < Cout; ++o) {
      double acc = 0.0;
      const float* wo = w + o * ldw;
      for (int64_t r = 0; r < R; ++r) {
        const int64_t ih = p * stride - pad + r;
        if (ih < 0 || ih >= H) continue;
        for (int64_t s = 0; s < S; ++s) {
          const int64_t iw = q * stride - pad + s;
          if (iw < 0 || iw >= W) continue;
          const float* xi = x + ((b * H + ih) * W + iw) * Cin;
          const float* wi = wo + (r * S + s) * Cin;
          for (int64_t c = 0; c < Cin; ++c) acc += (double)xi[c] * (double)wi[c];
        }
      }
      if (res) acc += (double)res[m * ldr + o];
      out[o] = oracle_act(acc, act);
    }
  }
}

void oracle_gemm_ex(const float* a, const float* b, const float* res, int64_t ldr, float* c, const int64_t* rows,
                    int64_t n_rows, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int32_t act) {
  if (lda <= 0) lda = K;
  if (ldb <= 0) ldb = K;
  if (ldr <= 0) ldr = N;
  const int64_t n = rows ? n_rows : M;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t m = rows ? rows[i] : i;
    const float* am = a + m * lda;
    for (int64_t j = 0; j < N; ++j) {
      double acc = 0.0;
      const float* bn = b + j * ldb;
      for (int64_t k = 0; k < K; ++k) acc += (double)am[k] * (double)bn[k];
      if (res) acc += (double)res[m * ldr + j];
      c[i * N + j] = oracle_act(acc, act);
    }
  }
}

void oracle_dwconv2d_ex(const float* x, const float* w, float* y, const int64_t* rows, int64_t n_rows, int64_t batch,
                        int64_t H, int64_t W, int64_t C, int64_t R, int64_t S, int64_t stride, int64_t pad,
                        int64_t ldw, int32_t act) {
  const int64_t P = (H + 2 * pad - R) / stride + 1;
  const int64_t Q = (W + 2 * pad - S) / stride + 1;
  const int64_t M = batch * P * Q;
  if (ldw <= 0) ldw = R * S;
  const int64_t n = rows ? n_rows : M;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t m = rows ? rows[i] : i;
    const int64_t b = m / (P * Q), p = (m / Q) % P, q = m % Q;
    for (int64_t c = 0; c < C; ++c) {
      double acc = 0.0;
      for (int64_t r = 0; r < R; ++r) {
        const int64_t ih = p * stride - pad + r;
        if (ih < 0 || ih >= H) continue;
        for (int64_t s = 0; s < S; ++s) {
          const int64_t iw = q * stride - pad + s;
          if (iw < 0 || iw >= W) continue;
          acc += (double)x[((b * H + ih) * W + iw) * C + c] * (double)w[c * ldw + r * S + s];
        }
      }
      y[i * C + c] = oracle_act(acc, act);
    }
  }
}

/* is_max: torch MaxPool2d (padded taps never win); else AvgPool2d over the
 * full R x S window (count_include_pad: divisor R*S). */
void oracle_pool2d(const float* x, float* y, const int64_t* rows, int64_t n_rows, int64_t batch, int64_t H, int64_t W,
                   int64_t C, int64_t R, int64_t S, int64_t stride, int64_t pad, int32_t is_max) {
  const int64_t P = (H + 2 * pad - R) / stride + 1;
  const int64_t Q = (W + 2 * pad - S) / stride + 1;
  const int64_t M = batch * P * Q;
  const int64_t n = rows ? n_rows : M;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t m = rows ? rows[i] : i;
    const int64_t b = m / (P * Q), p = (m / Q) % P, q = m % Q;
    for (int64_t c = 0; c < C; ++c) {
      double acc = is_max ? -INFINITY : 0.0;
      for (int64_t r = 0; r < R; ++r) {
        const int64_t ih = p * stride - pad + r;
        if (ih < 0 || ih >= H) continue;
        for (int64_t s = 0; s < S; ++s) {
          const int64_t iw = q * stride - pad + s;
          if (iw < 0 || iw >= W) continue;
          const double v = (double)x[((b * H + ih) * W + iw) * C + c];
          if (is_max)
            acc = v > acc ? v : acc;
          else
            acc += v;
        }
      }
      y[i * C + c] = is_max ? (float)acc : (float)(acc / (double)(R * S));
    }
  }
}
