/*
 * axq_oracle.c -- plain, slow, obviously-correct CPU oracle for the AdaPT approximate
 * LUT layer (arXiv 2203.04071).  TEST INFRASTRUCTURE ONLY: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load it.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2203_04071_b200/csrc), and neither side includes or links the other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; "S:n" = SPEC.md line n;
 * "Ax"/"Ox" = the readings listed in DESIGN.md §3.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 * (no intrinsics, no blocking).  fp32 steps are pinned to IEEE single precision with
 * round-to-nearest-even because the paper's quantizer works on fp32 PyTorch tensors
 * (§III.A) and a quantized code is an integer decided by fp32 arithmetic; integer
 * sums use int64 and are checked to fit the int32 accumulator the path uses (A12).
 *
 * Pins (tests/test_oracle_pins.py): exact-multiplier LUT == numpy int64 matmul; indicator /
 * row-sum / column-sum LUT probes; bincount reformulation; brute force at b=2; conv with
 * the exact LUT == float64 torch conv2d; conv == explicit im2col + GEMM; padding probe;
 * quantizer worked examples (tests/golden/) and round-trip / tie / symmetry properties.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- threads (cpu_baseline only: OpenMP parallel for over the outermost loop) ---- */
void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- O2: amax = max_i |x_i| ("the max absolute number of our values"; BJ:ns max
 *      calibration).  Exact: a max of absolute values has no rounding. ---- */
float orc_amax(const float* x, int64_t n) {
    float m = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
        float a = fabsf(x[i]);
        if (a > m) m = a;
    }
    return m;
}

/* ---- O3: scale A = amax / (2^(b-1) - 1) ("real_value = A x quantized_value + B",
 *      B = 0; "scale = calib_max / (2^(b-1)-1)"); amax == 0 -> 1 (A4). ---- */
float orc_scale(float amax, int bits) {
    float qmax = (float)((1 << (bits - 1)) - 1);
    if (amax == 0.0f) return 1.0f;
    return amax / qmax;
}

/* ---- O4: q = clamp(round(x / A)), round half to even (A1), symmetric clamp
 *      to +-(2^(b-1)-1) (A2), IEEE division (A3). ---- */
void orc_quantize(const float* x, int64_t n, float s, int bits, int8_t* q) {
    float qmax = (float)((1 << (bits - 1)) - 1);
    for (int64_t i = 0; i < n; ++i) {
        float t = x[i] / s;
        if (t > qmax) t = qmax;
        if (t < -qmax) t = -qmax;
        q[i] = (int8_t)rintf(t);
    }
}

/* b-bit two's-complement pattern of an operand ("ubits masks the operand's
 * two's-complement bit pattern to its bitwidth"). */
static inline int64_t ubits(int v, int bits) { return (int64_t)(v & ((1 << bits) - 1)); }

/* ---- O5: acc[m][n] = sum_k LUT[a[m][k]][w[k][n]] ("the inner multiplications
 *      between each input and filter values using a LUT"; BJ:ns).  A is [M][K],
 *      W is stored [N][K] because the layer is y = x A^T + b.  Table index
 *      (ua << b) | uw, first index = activation (A8).  Returns the number of outputs
 *      whose exact sum does not fit int32 (0 when the int32 accumulator is exact). ---- */
int64_t orc_lut_gemm(int64_t M, int64_t N, int64_t K, const int8_t* A, const int8_t* W,
                     int bits, const int32_t* T, int32_t* C) {
    int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t n = 0; n < N; ++n) {
            int64_t acc = 0;
            for (int64_t k = 0; k < K; ++k) {
                int64_t idx = (ubits(A[m * K + k], bits) << bits) | ubits(W[n * K + k], bits);
                acc += T[idx];
            }
            if (acc > INT32_MAX || acc < INT32_MIN) bad++;
            C[m * N + n] = (int32_t)acc;
        }
    }
    return bad;
}

/* ---- O6: direct convolution, X (N, C_in, H_in, W_in) -> Y (N, C_out, H_out, W_out) with
 *      kernel size, padding, stride, groups (§III.B.1), every multiply a LUT
 *      lookup.  "multiplying these 2 matrices would compute the same dot product as the
 *      original 2D convolution": the im2col matrix holds zeros at padded taps and
 *      those zeros are multiplied too, so a padded tap contributes LUT[0][w] (A11).
 *      Weights are (C_out, C_in/groups, R, S) as in PyTorch.  Output int32 NCHW. ---- */
int64_t orc_lut_conv2d(int64_t Nb, int64_t Cin, int64_t H, int64_t Wd, int64_t Cout,
                       int64_t R, int64_t S, int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                       int64_t dh, int64_t dw, int64_t groups, const int8_t* X,
                       const int8_t* Wt, int bits, const int32_t* T, int32_t* Y) {
    int64_t Ho = (H + 2 * ph - dh * (R - 1) - 1) / sh + 1;
    int64_t Wo = (Wd + 2 * pw - dw * (S - 1) - 1) / sw + 1;
    int64_t cin_g = Cin / groups, cout_g = Cout / groups;
    int64_t bad = 0;
#pragma omp parallel for collapse(2) schedule(static) reduction(+ : bad)
    for (int64_t img = 0; img < Nb; ++img) {
        for (int64_t co = 0; co < Cout; ++co) {
            int64_t g = co / cout_g;
            for (int64_t ho = 0; ho < Ho; ++ho) {
                for (int64_t wo = 0; wo < Wo; ++wo) {
                    int64_t acc = 0;
                    for (int64_t ci = 0; ci < cin_g; ++ci) {
                        int64_t c = g * cin_g + ci;
                        for (int64_t r = 0; r < R; ++r) {
                            for (int64_t s = 0; s < S; ++s) {
                                int64_t hi = ho * sh - ph + r * dh;
                                int64_t wi = wo * sw - pw + s * dw;
                                int a = 0; /* padded tap: a = 0, still looked up */
                                if (hi >= 0 && hi < H && wi >= 0 && wi < Wd)
                                    a = X[((img * Cin + c) * H + hi) * Wd + wi];
                                int w = Wt[((co * cin_g + ci) * R + r) * S + s];
                                acc += T[(ubits(a, bits) << bits) | ubits(w, bits)];
                            }
                        }
                    }
                    if (acc > INT32_MAX || acc < INT32_MIN) bad++;
                    Y[((img * Cout + co) * Ho + ho) * Wo + wo] = (int32_t)acc;
                }
            }
        }
    }
    return bad;
}

/* ---- O7: dequantize with bias: y = acc * (A_a * A_w) + b (P:74 real = A x q with both
 *      operands' scales; "y = xA^T + b" plus "an optional bias vector").  Pinned
 *      fp32 order (A14): y = fl(fl((float)acc * fl(s_a * s_w)) + bias[ch]), no FMA.
 *      Element i belongs to channel (i / inner) % nch ([M][N]: inner=1; NCHW: inner=HW). */
void orc_dequantize(int64_t count, const int32_t* acc, float s_a, float s_w,
                    const float* bias, int64_t nch, int64_t inner, float* y) {
    float sc = s_a * s_w;
    for (int64_t i = 0; i < count; ++i) {
        float v = (float)acc[i];
        v = v * sc;
        if (bias) v = v + bias[(i / inner) % nch];
        y[i] = v;
    }
}

/* ===================== NEXT-1: the paper's own quantizer =====================
 * "weight ranges are per channel while activation ranges are per tensor"; activations
 * are calibrated by "the histogram calibrator for a 99.9% percentile" which "learns
 * offline calib_max, the absolute maximum input value representable in the quantized space"
 * (P:94).  Readings A30-A32 fix what the paper leaves open. */

/* Per-output-channel amax of a weight tensor stored [rows][cols] (rows = output channels;
 * conv weights flattened per output channel).  Max-abs statistic (A31). */
void orc_amax_rows(const float* W, int64_t rows, int64_t cols, float* amax_r) {
    for (int64_t r = 0; r < rows; ++r) amax_r[r] = orc_amax(W + r * cols, cols);
}

/* q[r][c] = clamp(rint(W[r][c] / s[r])) -- O4 with the row's own scale. */
void orc_quantize_rows(const float* W, int64_t rows, int64_t cols, const float* s_r, int bits,
                       int8_t* q) {
    for (int64_t r = 0; r < rows; ++r) orc_quantize(W + r * cols, cols, s_r[r], bits, q + r * cols);
}

/* Histogram percentile calib_max (A30): bins of width w = fl(amax / bins) over [0, amax];
 * |x| falls in bin min(trunc(fl(|x| / w)), bins - 1); calib_max is the upper edge
 * fl((i + 1) * w) of the first bin i whose cumulative count c satisfies
 * c * p_den >= n * p_num (percentile p = p_num / p_den, 99.9 % = 999 / 1000).  amax == 0 gives
 * calib_max = 0 (the scale rule then returns 1, A4).  Also returns the bin index. */
int64_t orc_hist_calib(const float* x, int64_t n, int bins, int64_t p_num, int64_t p_den,
                       float* calib_max) {
    float a = orc_amax(x, n);
    *calib_max = 0.0f;
    if (a == 0.0f || n == 0) return -1;
    float w = a / (float)bins;
    int64_t* cnt = (int64_t*)calloc((size_t)bins, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        float t = fabsf(x[i]) / w;
        int64_t b = (int64_t)t;          /* t >= 0: truncation is floor */
        if (b > bins - 1) b = bins - 1;
        cnt[b] += 1;
    }
    int64_t cum = 0, hit = bins - 1;
    for (int64_t b = 0; b < bins; ++b) {
        cum += cnt[b];
        if (cum * p_den >= n * p_num) { hit = b; break; }
    }
    free(cnt);
    *calib_max = (float)(hit + 1) * w;
    return hit;
}

/* O7 with per-channel weight scales (A32): y = fl(fl((float)acc * fl(s_a * s_w[ch])) + b[ch]). */
void orc_dequantize_pc(int64_t count, const int32_t* acc, float s_a, const float* s_w,
                       const float* bias, int64_t nch, int64_t inner, float* y) {
    for (int64_t i = 0; i < count; ++i) {
        int64_t ch = (i / inner) % nch;
        float sc = s_a * s_w[ch];
        float v = (float)acc[i];
        v = v * sc;
        if (bias) v = v + bias[ch];
        y[i] = v;
    }
}

/* ===================== NEXT-2: wide ACUs (b = 9..12) =====================
 * The paper also emulates 12-bit multipliers (mul12s, "one with 12-bit precision").
 * Codes no longer fit int8, so operands are int16 two's-complement codes; everything else is
 * O4 / O5 unchanged: q = clamp(rint(x / s)) with qmax = 2^(b-1) - 1, and
 * acc = sum_k T[(u(a) << b) | u(w)] with u = the b-bit pattern. */
void orc_quantize16(const float* x, int64_t n, float s, int bits, int16_t* q) {
    float qmax = (float)((1 << (bits - 1)) - 1);
    for (int64_t i = 0; i < n; ++i) {
        float t = x[i] / s;
        if (t > qmax) t = qmax;
        if (t < -qmax) t = -qmax;
        q[i] = (int16_t)rintf(t);
    }
}

int64_t orc_lut_gemm16(int64_t M, int64_t N, int64_t K, const int16_t* A, const int16_t* W,
                       int bits, const int32_t* T, int32_t* C) {
    int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t n = 0; n < N; ++n) {
            int64_t acc = 0;
            for (int64_t k = 0; k < K; ++k) {
                int64_t idx = (ubits(A[m * K + k], bits) << bits) | ubits(W[n * K + k], bits);
                acc += T[idx];
            }
            if (acc > INT32_MAX || acc < INT32_MIN) bad++;
            C[m * N + n] = (int32_t)acc;
        }
    }
    return bad;
}
