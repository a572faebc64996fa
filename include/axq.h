/*
 * axq.h -- C ABI of the B200-native approximate-multiplier LUT layer (AdaPT,
 * arXiv 2203.04071).  Every multiply of a quantized convolution / linear layer is
 * replaced by a lookup into an approximate multiplier's 2^b x 2^b product table.
 *
 * Citations: "P:n" = PAPER.md line n; "S:n" = SPEC.md line n;
 * readings "A1".."A23" are listed in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *   - extern "C", plain pointers and sizes; no CUDA or torch types.  `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Tensor pointers are DEVICE pointers on the current CUDA device unless the argument
 *     name says host_.  The caller owns every buffer; hot calls never allocate, never
 *     synchronize and are asynchronous on `stream`.
 *   - Arguments are validated on the host before any launch.  Errors are returned as
 *     axq_status codes (no exceptions, no abort, no printing).  On an error no kernel was
 *     launched, except AXQ_ERR_CUDA (a launch failed; axq_last_cuda_error() has the code).
 *   - Integer outputs are exact: int32 accumulation is associative, so results are
 *     bit-identical for every tiling, split-K factor and GPU count (A23).
 *   - fp32 steps are pinned (IEEE division, round-half-even, no FMA contraction) so that
 *     quantized codes match the oracle bit for bit (A1, A3, A14).
 *   - Reentrant: calls from several host threads, and launches in flight on several
 *     streams, never share library-owned mutable state.  LUT and weight-pack handles are
 *     immutable after creation (one per device) and usable from any stream.  The only
 *     per-call scratch is the caller's epilogue workspace (axq_epilogue.workspace): one
 *     workspace must not be used by two launches that may run concurrently.
 */
#ifndef AXQ_H
#define AXQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    AXQ_OK = 0,
    AXQ_ERR_INVALID = 1,     /* null pointer, extent < 0, bad leading dimension, bits not in
                                [2,8], misaligned pointer where alignment is documented */
    AXQ_ERR_OVERFLOW = 2,    /* K * max|LUT| >= 2^31: an int32 accumulator could overflow */
    AXQ_ERR_UNSUPPORTED = 3, /* a documented-but-unimplemented case (e.g. groups > 1 on _wp) */
    AXQ_ERR_CUDA = 4         /* a CUDA call failed; see axq_last_cuda_error() */
} axq_status;

/* Device representation chosen by axq_lut_create. */
typedef enum {
    AXQ_LUT_DELTA8 = 0, /* int8 E = LUT - a*w, shared-memory resident (64 KiB), exact part
                           added with dp4a */
    AXQ_LUT_I16 = 1,    /* int16 LUT values, shared-memory resident (128 KiB) */
    AXQ_LUT_I32 = 2,    /* int32 values: gathered through L1 (default) or SM-resident as two
                           128 KiB halves by the activation's high bit (axq_lut_set_i32_resident) */
    AXQ_LUT_WIDE16 = 3, /* b = 9..12 (NEXT-2): int16 E = LUT - a*w, [uw][ua] in b-bit patterns,
                           read through L1/L2 (2^(2b+1) bytes: 32 MiB at b = 12) */
    AXQ_LUT_WIDE32 = 4  /* b = 9..12 with E beyond int16: int32 LUT values through L1/L2 */
} axq_lut_repr;

typedef struct axq_lut* axq_lut_t;

/* Kernel family of the last LUT launch made by the calling thread (axq_last_path): low byte
 * the kernel, plus flags.  Observability for tests and measurement; no effect on results. */
#define AXQ_PATH_V1 1         /* lut_mm_kernel: per-lane gather from the resident table */
#define AXQ_PATH_P4 2         /* lut_p4_kernel: packed tables, mma.sync exact part */
#define AXQ_PATH_P4W 3        /* lut_p4w_kernel: packed tables, tcgen05 exact part, warp roles */
#define AXQ_PATH_GCONV 4      /* grouped / depthwise resident-table kernels (NEXT-3) */
#define AXQ_PATH_WIDE 5       /* wide (b = 9..12) kernels (NEXT-2) */
#define AXQ_PATH_LSTM_REC 6   /* persistent LSTM recurrence */
#define AXQ_PATH_F32A 7       /* quantize-on-load kernel (axq_lut_gemm_f32a / axq_lut_conv2d_f32) */
#define AXQ_PATH_P4W16 8      /* lut_p4w_kernel<E16>: packed int16 E tables (|E| beyond int8) */
#define AXQ_PATH_WIDEPK 9     /* lut_widepk_kernel: packed wide (b = 9..12) tables (NEXT-2) */
#define AXQ_PATH_SPLITK 0x100 /* K split across CTAs (int32 atomics + epilogue pass) */
#define AXQ_PATH_STREAMK 0x200/* stream-K pieces in the caller's workspace */
#define AXQ_PATH_TMA 0x400    /* P4W activation planes by TMA, 2D tiled (GEMM rows) */
#define AXQ_PATH_TMA_IM2COL 0x800 /* P4W activation planes by TMA, im2col mode (convs) */
axq_status axq_last_path(int* out);

/* Returns the CUDA error code of the last AXQ_ERR_CUDA on this thread (0 if none). */
int axq_last_cuda_error(void);
/* Static string for a status code. */
const char* axq_status_string(axq_status s);
/* Library version: major*10000 + minor*100 + patch. */
int axq_version(void);

/* ---------------------------------------------------------------------------------
 * ACU table.  "the corresponding LUT is produced from AdaPT's Look-up Table (LUT)
 * generator" (§III.C); any deterministic multiplier is allowed.
 *
 * axq_lut_create: host_table is a HOST int32 array of 2^(2*bits) entries, entry
 *   (ua << bits) | uw = ACU(a, w), ua / uw the b-bit two's-complement patterns of the
 *   activation a and the weight w (first index = ACTIVATION, A8).  bits in [2,12];
 *   bits 9..12 (NEXT-2, the paper's 12-bit multipliers) give a WIDE16 / WIDE32 handle that
 *   only axq_lut_gemm16 accepts (the int8 entry points return AXQ_ERR_UNSUPPORTED).
 *   The library copies the table, picks the device representation (axq_lut_repr),
 *   uploads it to the current device and synchronizes.  *out receives the handle.
 * axq_lut_destroy: frees the handle (synchronizes the device first).  NULL is a no-op.
 * axq_lut_info: bits, representation and the min / max table value (any out-pointer
 *   may be NULL).
 * ------------------------------------------------------------------------------- */
axq_status axq_lut_create(int bits, const int32_t* host_table, axq_lut_t* out);
axq_status axq_lut_destroy(axq_lut_t lut);
axq_status axq_lut_info(axq_lut_t lut, int* bits, int* repr, int32_t* tmin, int32_t* tmax);

/*
 * axq_lut_set_i32_resident: for an AXQ_LUT_I32 table, choose how the LUT kernel holds it
 * (north_star "int32 split across SM-resident halves"):
 * resident = 1 stages it in shared memory as two 128 KiB halves by the activation's high bit
 * (a tile's second pass runs only when its codes need the other half); 0 (the default, or
 * AXQ_I32_RESIDENT in the environment at the first table creation) gathers it through L1.
 * Results are identical.  Not synchronised with launches in flight on the same table.
 * Errors: AXQ_ERR_INVALID (null), AXQ_ERR_UNSUPPORTED (not an int32 table).
 */
axq_status axq_lut_set_i32_resident(axq_lut_t lut, int resident);

/* ---------------------------------------------------------------------------------
 * Quantizer.  "real_value = A x quantized_value + B where A is the scale and B is the
 * zero point (often set to zero)" (§III.A); per-tensor max calibration (BJ:ns,
 * overriding P:93-95's histogram, A5/A6).
 *
 * axq_amax:   *d_amax = max_i |x_i| over n fp32 values (exact).  n >= 0 (n = 0 -> 0).
 * axq_scale:  *d_scale = fl32(*d_amax / (2^(bits-1)-1)), or 1.0 if *d_amax == 0 (A4).
 * axq_quantize: q_i = clamp(rint(fl32(x_i / *d_scale)), -(2^(b-1)-1), 2^(b-1)-1), rint =
 *   round half to even (A1), symmetric clamp (A2), IEEE division (A3).  q is int8 holding
 *   the sign-extended b-bit code.  Layout-preserving.
 * axq_quantize_nchw_to_nhwc: the same map on an fp32 NCHW tensor [N][C][H][W], writing int8
 *   NHWC [N][H][W][Cq] (the layout axq_lut_conv2d reads); Cq >= C, channels C..Cq-1 are
 *   written as 0 (storage padding, see axq_conv_desc.c_valid).
 * ------------------------------------------------------------------------------- */
axq_status axq_amax(const float* x, int64_t n, float* d_amax, void* stream);
axq_status axq_scale(const float* d_amax, int bits, float* d_scale, void* stream);
axq_status axq_quantize(const float* x, int64_t n, const float* d_scale, int bits,
                        int8_t* q, void* stream);

/* ---------------------------------------------------------------------------------
 * NEXT-1: the paper's own quantizer ("we implemented the histogram calibrator for a
 * 99.9% percentile ... weight ranges are per channel while activation ranges are per
 * tensor"; readings A30-A32).  All device pointers, asynchronous on `stream`.
 * axq_amax_rows: d_amax[r] = max_c |W[r][c]| for W fp32 [rows][cols] (row = output channel,
 *   conv weights flattened KRSC or KCRS per output channel).
 * axq_scale_vec: d_scale[i] = d_amax[i] / (2^(bits-1)-1), 0 -> 1 (axq_scale per element).
 * axq_quantize_rows: q[r][c] = clamp(rint(W[r][c] / d_scale_rows[r])) (axq_quantize per row).
 * axq_calib_histogram: d_hist[bins] (uint32, zeroed by the call) = counts of |x| over the
 *   bins of width fl(*d_amax / bins) on [0, *d_amax]: bin = min(trunc(fl(|x| / w)), bins-1).
 *   d_amax must hold max|x| (axq_amax).  bins <= 8192; n < 2^32.
 * axq_calib_percentile: calib_max = fl((i+1) * w) for the first bin i whose cumulative count c
 *   has c * p_den >= n * p_num (99.9 % = 999 / 1000); writes it to d_calib_max (nullable) and
 *   the scale calib_max / qmax (0 -> 1) to d_scale (nullable). */
axq_status axq_amax_rows(const float* W, int64_t rows, int64_t cols, float* d_amax, void* stream);
axq_status axq_scale_vec(const float* d_amax, int64_t n, int bits, float* d_scale, void* stream);
axq_status axq_quantize_rows(const float* W, int64_t rows, int64_t cols, const float* d_scale_rows,
                             int bits, int8_t* q, void* stream);
axq_status axq_calib_histogram(const float* x, int64_t n, const float* d_amax, int bins,
                               uint32_t* d_hist, void* stream);
axq_status axq_calib_percentile(const uint32_t* d_hist, int bins, int64_t n, const float* d_amax,
                                int64_t p_num, int64_t p_den, int bits, float* d_calib_max,
                                float* d_scale, void* stream);
axq_status axq_quantize_nchw_to_nhwc(const float* x, int64_t N, int64_t C, int64_t H,
                                     int64_t W, int64_t Cq, const float* d_scale, int bits,
                                     int8_t* q, void* stream);

/* ---------------------------------------------------------------------------------
 * LUT-GEMM.  Linear layer y = x A^T + b (§III.B.3) with "the inner
 * multiplications between each input and filter values using a LUT" (§IV):
 *     C[m][n] = sum_{k<K} LUT[A[m][k]][W[n][k]]    (int32; BJ:ns acc[m,n])
 * A: int8 activations, element (m,k) at A[m*lda + k], lda >= K.
 * W: int8 weights stored [N][K] (PyTorch Linear layout), element (n,k) at W[n*ldw + k].
 * C: int32 [M][ldc], ldc >= N, overwritten.
 * M, N, K >= 0 (any zero extent: C gets zeros for K == 0, nothing otherwise).
 * Operands must be b-bit codes (sign-extended in int8) of the LUT's bit width; other
 * values index the table by their low b bits.
 * Errors: AXQ_ERR_OVERFLOW if K * max|LUT| >= 2^31.
 * ------------------------------------------------------------------------------- */
axq_status axq_lut_gemm(int64_t M, int64_t N, int64_t K, const int8_t* A, int64_t lda,
                        const int8_t* W, int64_t ldw, axq_lut_t lut, int32_t* C, int64_t ldc,
                        void* stream);

/* Fused dequantize epilogue (P:74 with both operands' scales; "+ b"), applied per
 * output element in this pinned fp32 order (A13/A14/A17):
 *     v = fl(fl((float)acc) * fl(*d_scale_a * *d_scale_w))
 *     v = fl(v + bias[n])            if bias
 *     v = fl(v + residual[m][n])     if residual   (row / NHWC layout, stride ldr)
 *     v = max(v, 0)                  if relu
 *     y = v                          if y
 *     q_out[m][n] = clamp(rint(fl(v / *d_scale_out)))   if q_out  (requantize for the next
 *                                    layer with bits_out, same rule as axq_quantize)
 * Zero-initialise the struct and set what is needed.  workspace: NULL, or device int32
 * scratch (16-byte aligned) of workspace_elems elements (0 = M*N, the minimum) owned by the
 * caller.  It lets the library split K across CTAs when the M*N outputs alone cannot fill
 * the GPU (needs >= M*N elements), or let the packed-table P4W kernel cut tiles at stream-K
 * boundaries (needs >= axq_workspace_elems(M, N) elements: 256 tile counters, then per-CTA
 * partial slots).  Results are identical with or without it.  A workspace must be
 * ZERO-FILLED when first passed; every call leaves its first 256 elements zero again (the
 * rest is scratch), so one buffer can be reused across calls and layers ON ONE STREAM -- two
 * launches that may run concurrently need two workspaces.  Layout of y: GEMM -> [M][ldy];
 * conv -> NCHW unless y_nhwc = 1 ([N*Ho*Wo][ldy]).  q_out is always [M][ldq] (conv: NHWC). */
typedef struct axq_epilogue {
    const float* d_scale_a;   /* device fp32 scalar: activation scale (required) */
    const float* d_scale_w;   /* device fp32 scalar: weight scale (required) */
    const float* bias;        /* device fp32 [N] or NULL */
    float* y;                 /* device fp32 output or NULL */
    int64_t ldy;              /* row stride of y (GEMM, or conv with y_nhwc) */
    int32_t* workspace;       /* device int32 [M*N] or NULL */
    const float* residual;    /* device fp32 [M][ldr] or NULL */
    int64_t ldr;
    int32_t relu;             /* nonzero: ReLU after the residual add */
    int32_t y_nhwc;           /* conv only: 1 -> y is NHWC [M][ldy] */
    int8_t* q_out;            /* device int8 [M][ldq] requantized output or NULL */
    int64_t ldq;
    const float* d_scale_out; /* device fp32 scalar, required with q_out */
    int32_t bits_out;         /* 2..8, required with q_out */
    const float* d_scale_w_ch;/* device fp32 [N] per-output-channel weight scales or NULL
                                 (NEXT-1, "weight ranges are per channel"): column n then
                                 uses fl(s_a * s_w[n]) in place of fl(s_a * s_w) (A32) */
    int64_t workspace_elems;  /* int32 elements of workspace; 0 = M*N */
} axq_epilogue;

/* axq_workspace_elems: the epilogue workspace size (int32 elements) that enables every
 * work decomposition for an M x N output on the current device: max(M*N, 256 + 2 * SMs *
 * 896 * 16).  -1 for negative extents. */
int64_t axq_workspace_elems(int64_t M, int64_t N);

axq_status axq_lut_gemm_dq(int64_t M, int64_t N, int64_t K, const int8_t* A, int64_t lda,
                           const int8_t* W, int64_t ldw, axq_lut_t lut,
                           const axq_epilogue* ep, void* stream);

/* ---------------------------------------------------------------------------------
 * LUT convolution.  X (N, C_in, H_in, W_in) -> Y (N, C_out, H_out, W_out) with kernel
 * size, padding, stride and groups (§III.B.1), computed as the im2col GEMM of P:119
 * without materialising the im2col matrix (implicit im2col):
 *     Y[img][ho][wo][co] = sum_{r,s,c} LUT[x(img, ho*sh-ph+r*dh, wo*sw-pw+s*dw, c)][Wt[co][r][s][c]]
 * where x(...) = X value inside the image and 0 at a padded tap -- the 0 is still looked
 * up (A11), exactly as the zero entries of the paper's im2col matrix are multiplied.
 * X: int8 NHWC [N][H][W][C];  Wt: int8 [C_out][R][S][C] (KRSC);  Y: int32 NHWC
 * [N][H_out][W_out][C_out].
 * groups = G > 1 (NEXT-3: grouped and depthwise convolution): C and C_out divisible by G,
 *   Wt is [C_out][R][S][C/G], output channel co reads input channels g*C/G .. (g+1)*C/G - 1
 *   with g = co / (C_out/G); the sum runs over those C/G channels only.  c_valid must be 0.
 *   Runs on a resident-table kernel (a grouped layer has too few lookups per output to
 *   amortise packed tables); the _wp entry points require groups == 1.
 * ------------------------------------------------------------------------------- */
typedef struct axq_conv_desc {
    int64_t N, H, W, C;       /* input (C = channels as stored, i.e. the NHWC row length) */
    int64_t K, R, S;          /* output channels, filter height / width */
    int64_t stride_h, stride_w, pad_h, pad_w, dil_h, dil_w, groups;
    int64_t c_valid;          /* 0, or the number of real channels (< C): channels >= c_valid
                                 are STORAGE padding holding a = 0 and w = 0; their lookups
                                 are removed exactly (they are not the paper's padding) */
} axq_conv_desc;

axq_status axq_conv2d_out_hw(const axq_conv_desc* d, int64_t* Ho, int64_t* Wo);
axq_status axq_lut_conv2d(const axq_conv_desc* d, const int8_t* X, const int8_t* Wt,
                          axq_lut_t lut, int32_t* Y, void* stream);
/* Fused dequant epilogue writing fp32 NCHW y[img][co][ho][wo] (the paper's layout). */
axq_status axq_lut_conv2d_dq(const axq_conv_desc* d, const int8_t* X, const int8_t* Wt,
                             axq_lut_t lut, const axq_epilogue* ep, void* stream);

/* ---------------------------------------------------------------------------------
 * Quantize-on-load variants: the quantizer of P:74 ("real_value = A x quantized_value") fused
 * into the operand load of the LUT-GEMM / LUT-conv, so the fp32 activations are read once and
 * no int8 copy is written (the paper puts quantize + dequantize at ~10 % of the time).
 * axq_lut_gemm_f32a: A fp32 [M][lda] (row m at A + m*lda) with its device scale *d_scale_a
 *   (e.g. from axq_amax + axq_scale); every element is quantized exactly as axq_quantize does
 *   (A1-A3: IEEE x / s, symmetric clamp to the LUT's bit width, round half to even) inside the
 *   load, then summed as axq_lut_gemm.  ep NULL -> raw int32 C [M][ldc]; else the fused
 *   epilogue of axq_lut_gemm_dq (ep->d_scale_a is normally the same scale pointer).
 * axq_lut_conv2d_f32: X fp32 NCHW [N][C][H][W] (the paper's layout; d->c_valid must be
 *   0), quantized on load with *d_scale_a; padded taps are the code 0 (A11).  Wt int8 KRSC.
 *   ep NULL -> raw int32 Y NHWC [N][Ho][Wo][K]; else the fused epilogue (NCHW fp32 y unless
 *   ep->y_nhwc).  groups must be 1.
 * Results are bit-identical to axq_quantize(_nchw_to_nhwc) followed by the int8 entry point
 * (tested).  Errors as the int8 entry points; AXQ_ERR_INVALID if d_scale_a is NULL.
 * ------------------------------------------------------------------------------- */
axq_status axq_lut_gemm_f32a(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                             const float* d_scale_a, const int8_t* W, int64_t ldw, axq_lut_t lut,
                             const axq_epilogue* ep, int32_t* C, int64_t ldc, void* stream);
axq_status axq_lut_conv2d_f32(const axq_conv_desc* d, const float* X, const float* d_scale_a,
                              const int8_t* Wt, axq_lut_t lut, const axq_epilogue* ep, int32_t* Y,
                              void* stream);

/* ---------------------------------------------------------------------------------
 * Prepared weights for the packed-table kernel.  For a delta8 table
 * (LUT = a*w + E with E in int8) the weights of a layer are known before inference ("learns
 * offline"), so the product row E[.][w] of every weight can be laid out once:
 *     tables[n_block][k][q][ua] = 4 x int8 E[ua][w(16 n_block + 4q + j, k)], j = 0..3
 * which lets one 32-bit shared-memory load serve four lookups; the exact part sum a*w runs on
 * the tensor cores.  Results are bit-identical to axq_lut_gemm / axq_lut_conv2d.
 * axq_wpack_create: W device int8 [N][ldw] (N x K, conv: KRSC flattened, K = R*S*C); the
 *   LUT handle must have representation AXQ_LUT_DELTA8 (else AXQ_ERR_UNSUPPORTED).
 *   a_nonneg = 1 promises that every activation code the handle will be used with is >= 0
 *   (e.g. quantized ReLU outputs): the tables then hold ua = 0..127 only (half the bytes, a
 *   deeper pipeline).  A negative code with such a handle gives unspecified (but memory-safe)
 *   results.  Allocates N/16 * K/16 * 64 KiB (32 KiB with a_nonneg) plus a packed weight copy
 *   of device memory, synchronizes.  The handle keeps no reference to W or lut.
 * axq_lut_gemm_wp / axq_lut_conv2d_wp: as axq_lut_gemm_dq / axq_lut_conv2d_dq (same epilogue
 *   semantics; with ep->workspace the library may split K when the tiles alone cannot fill
 *   the GPU).  With ep == NULL the raw int32 result goes to C ([M][ldc]) / Y (NHWC), which is
 *   then also used as the split-K accumulator.  Requirements (else AXQ_ERR_UNSUPPORTED): A / X 16-byte
 *   aligned, lda % 16 == 0 (GEMM); conv: C % 4 == 0 and X 4-byte aligned (C % 16 == 0 with a
 *   16-byte aligned X takes 16-byte operand copies, otherwise 4-byte ones); grouped conv
 *   (groups > 1, NEXT-3): wp packs the weights [K][R][S][C/groups] as an N = K,
 *   K = R*S*C/groups GEMM operand; C/groups and K/groups multiples of 16, X 16-byte aligned,
 *   c_valid 0, int8-E tables (each 16-column tile lies in one group and reads that group's
 *   input channels).
 * ------------------------------------------------------------------------------- */
typedef struct axq_wpack* axq_wpack_t;
axq_status axq_wpack_create(axq_lut_t lut, const int8_t* W, int64_t N, int64_t K, int64_t ldw,
                            int a_nonneg, axq_wpack_t* out);
/* a_nonneg is a flag word: AXQ_WPACK_NONNEG (= 1, the promise above) and
 * AXQ_WPACK_ACTIVATIONS (= 2): W holds ACTIVATION codes x [N][K] (a small matrix, e.g. a
 * 256-row linear-layer input) and the tables are specialised on them (byte = E[x][u] for a
 * weight code u) for axq_lut_gemm_xs.
 * axq_wpack_repack: re-packs new codes W [N][ldw] (same N, K) into wp, asynchronously on
 *   `stream` (no allocation: the per-call activation tables of axq_lut_gemm_xs).
 * axq_lut_gemm_xs: acc[m][n] = sum_k LUT[x[m][k]][W[n][k]] for the activations x packed in
 *   xp (AXQ_WPACK_ACTIVATIONS) and weight codes W [N][ldw] (16-byte aligned, ldw % 16 == 0):
 *   the packed-table kernel with the weights as its row operand, written back in the normal
 *   layout -- raw int32 C [M][ldc] or the fused epilogue (bias / per-channel scale indexed by
 *   n, y [M][ldy], q_out [M][ldq]).  Results identical to axq_lut_gemm_dq.  Suits small M
 *   with large N*K: the tables are M x K x 1 KiB / 4 and are built per call. */
#define AXQ_WPACK_NONNEG 1
#define AXQ_WPACK_ACTIVATIONS 2
axq_status axq_wpack_repack(axq_wpack_t wp, const int8_t* W, int64_t ldw, void* stream);
axq_status axq_lut_gemm_xs(int64_t N, const int8_t* W, int64_t ldw, axq_wpack_t xp,
                           const axq_epilogue* ep, int32_t* C, int64_t ldc, void* stream);
axq_status axq_wpack_destroy(axq_wpack_t wp);
axq_status axq_wpack_info(axq_wpack_t wp, int64_t* N, int64_t* K, int64_t* device_bytes);
axq_status axq_lut_gemm_wp(int64_t M, const int8_t* A, int64_t lda, axq_wpack_t wp,
                           const axq_epilogue* ep, int32_t* C, int64_t ldc, void* stream);
axq_status axq_lut_conv2d_wp(const axq_conv_desc* d, const int8_t* X, axq_wpack_t wp,
                             const axq_epilogue* ep, int32_t* Y, void* stream);
/* axq_wpack_kernel: selects the kernel behind axq_lut_gemm_wp / axq_lut_conv2d_wp for the
 *   calling process (all results are bit-identical; this is a performance switch for
 *   measurement): 0 = default (P4W; P4 for the 4-byte-tap conv loader), 1 = P4 (exact part on
 *   mma.sync, 16 warps, 512- or 1024-row tiles), 3 = P4W (exact part on tcgen05.mma with TMEM
 *   accumulators, warp-specialised: 4 producer warps stream the operands, 16-28 consumer warps
 *   look up, 512- or 896-row tiles).  Returns the previous setting, or -1 for an unknown value
 *   (unchanged). */
int axq_wpack_kernel(int variant);   /* 2 (the former P4T variant) is retired: returns -1 */
/* axq_wpack_shapes: consumer-warp counts of the P4W shapes for the calling process (tile rows =
 *   32 x warps; a performance switch, all results bit-identical).  main_cw: non-residual layers
 *   with half-range 32-k tables -- 28 (default), 24 or 20; res_cw: layers with a residual
 *   epilogue (half-range 32-k) -- 16 (default), 20, 24 or 28; small_cw: non-residual layers
 *   with M <= 1024 -- 16 (default) or 28 (off).  0 leaves a value unchanged.  The environment
 *   (AXQ_P4W_MAIN_CW, AXQ_P4W_RES_CW, AXQ_P4W_CW) is read before the first call applies.
 *   Returns AXQ_ERR_INVALID (nothing changed) for any other value. */
axq_status axq_wpack_shapes(int main_cw, int res_cw, int small_cw);

/* ---------------------------------------------------------------------------------
 * NEXT-4: straight-through-estimator backward of an approximate linear layer
 * (§III.A.2 "Retraining": QAT "based on Straight Through Estimator (STE)
 * derivative approximation", "fake quantization modules which work with quantized floating
 * point values").  Under the STE the quantizer and the ACU are the identity in the backward
 * pass (A36), so with the fake-quantized operands fq(q) = fl32(s * q):
 *   gx[m][k] = [|x[m][k]| <= clip_a] * sum_n gy[m][n] * fq(qw[n][k])      (fp32 [M][K])
 *   gw[n][k] = [|w[n][k]| <= clip_w] * sum_m gy[m][n] * fq(qa[m][k])      (fp32 [N][K])
 *   gb[n]    = sum_m gy[m][n]                                             (fp32 [N])
 * gy: fp32 [M][N] dL/dy; qa int8 [M][K] / qw int8 [N][K]: the codes the forward used, with
 * their device scales; x fp32 [M][K] / w fp32 [N][K]: the unquantized operands, with the
 * calibrated clip ranges (device scalars, e.g. amax; a value with |v| > clip gets no gradient);
 * x / w null: no mask.  All buffers contiguous, on the current device; gx / gw / gb nullable
 * (not computed).  workspace (nullable, workspace_elems floats, 16-byte aligned, caller-owned,
 * no contents required, one per concurrently running call): with at least
 * axq_ste_linear_workspace_elems(M, N, K) elements each product first converts its operands
 * once into the tensor cores' tiled bf16 layout there and streams them with bulk copies
 * (several times faster); K-split slices are added inside a thread-block cluster through
 * distributed shared memory, beyond 8 slices through partial slots in the workspace; with less
 * room the operands are converted tile by tile inside the GEMM (fewer or no K slices).  The
 * slices are always added in a fixed order: deterministic for a given (shape, workspace size).
 * fp32 accumulation on the tensor cores (not bit-exact against a different summation order:
 * within the fp32 dot-product bound).  Asynchronous on stream.  AXQ_ERR_INVALID for negative extents or a
 * missing operand of a requested gradient.
 * --------------------------------------------------------------------------------- */
axq_status axq_ste_linear_backward(int64_t M, int64_t N, int64_t K, const float* gy,
                                   const int8_t* qa, const float* d_scale_a, const float* x,
                                   const float* d_clip_a, const int8_t* qw, const float* d_scale_w,
                                   const float* w, const float* d_clip_w, float* gx, float* gw,
                                   float* gb, float* workspace, int64_t workspace_elems,
                                   void* stream);

/* axq_ste_linear_workspace_elems / axq_ste_conv2d_workspace_elems: the workspace (fp32
 * elements) that enables the fastest decomposition of every product of the backward on the
 * current device (pre-converted operands + partial slots + two-pass column sums).  -1 for
 * negative extents or an invalid descriptor. */
int64_t axq_ste_linear_workspace_elems(int64_t M, int64_t N, int64_t K);
int64_t axq_ste_conv2d_workspace_elems(const axq_conv_desc* d);

/* axq_ste_conv2d_backward: the same STE backward for a convolution (groups = 1, dilation 1,
 *   c_valid 0; the conv is the GEMM of its im2col matrix).  gy fp32 NHWC [N][Ho][Wo][K]
 *   (dL/dy), qx int8 NHWC [N][H][W][C] / qw int8 [K][R][S][C]: the forward's codes with their
 *   device scales; x fp32 NHWC / w fp32 [K][R][S][C] + clips: the STE masks (nullable).
 *     gw[k][(r,s,c)] = [|w| <= clip_w] * sum_m gy[m][k] * fq(im2col(qx)[m][(r,s,c)])
 *     gx[n][h][w][c] = [|x| <= clip_a] * sum over the (m, r, s) whose window places tap (r, s)
 *                      on (h, w) of sum_k gy[m][k] * fq(qw[k][(r,s,c)])   (the adjoint of im2col)
 *     gb[k] = sum_m gy[m][k]
 *   Workspaces (caller-owned): cols int8 [M][ldcols] (ldcols >= R*S*C, multiple of 16; needed
 *   for gw), gcols fp32 [M][R*S*C] (needed for gx), workspace / workspace_elems as
 *   axq_ste_linear_backward (optional).  fp32 accumulation, deterministic.  AXQ_ERR_INVALID for
 *   other conv shapes or a missing operand of a requested gradient. */
axq_status axq_ste_conv2d_backward(const axq_conv_desc* d, const float* gy, const int8_t* qx,
                                   const float* d_scale_a, const float* x, const float* d_clip_a,
                                   const int8_t* qw, const float* d_scale_w, const float* w,
                                   const float* d_clip_w, float* gx, float* gw, float* gb,
                                   int8_t* cols, int64_t ldcols, float* gcols, float* workspace,
                                   int64_t workspace_elems, void* stream);

/* The same backwards with per-output-channel weight quantization (the paper's quantizer,
 * P:95 "weight ranges are per channel"; NEXT-1): d_scale_w_ch [N] (conv: [K]) replaces the
 * scalar d_scale_w when non-NULL -- fq(qw)[n] = fl32(s_w[n] * qw[n]) -- and d_clip_w_ch [N]
 * replaces d_clip_w (gw[n][k] masked by |w[n][k]| <= clip_w[n]).  The plain entry points are
 * these with both NULL.  Both products run on the tensor cores (tcgen05 kind::f16: the fp32
 * operand split exactly into three bf16 terms, the int8 codes exact in bf16, fp32
 * accumulation in TMEM; A36'); AXQ_ERR_UNSUPPORTED when a product has more than
 * 65535 x 128 output columns. */
axq_status axq_ste_linear_backward_pc(int64_t M, int64_t N, int64_t K, const float* gy,
                                      const int8_t* qa, const float* d_scale_a, const float* x,
                                      const float* d_clip_a, const int8_t* qw, const float* d_scale_w,
                                      const float* d_scale_w_ch, const float* w, const float* d_clip_w,
                                      const float* d_clip_w_ch, float* gx, float* gw, float* gb,
                                      float* workspace, int64_t workspace_elems, void* stream);
axq_status axq_ste_conv2d_backward_pc(const axq_conv_desc* d, const float* gy, const int8_t* qx,
                                      const float* d_scale_a, const float* x, const float* d_clip_a,
                                      const int8_t* qw, const float* d_scale_w,
                                      const float* d_scale_w_ch, const float* w, const float* d_clip_w,
                                      const float* d_clip_w_ch, float* gx, float* gw, float* gb,
                                      int8_t* cols, int64_t ldcols, float* gcols, float* workspace,
                                      int64_t workspace_elems, void* stream);

/* ---------------------------------------------------------------------------------
 * Dequantize (unfused), same pinned formula as the epilogue.
 * axq_dequantize: acc int32 [M][ldacc] -> y fp32 [M][ldy], bias[n] (nullable).
 * axq_dequantize_nhwc_to_nchw: acc int32 NHWC [N][HW][C] -> y fp32 NCHW [N][C][HW].
 * axq_epilogue_apply: the full axq_epilogue on an int32 [M][ldacc] accumulator (y in row
 *   layout [M][ldy]).
 * ------------------------------------------------------------------------------- */
axq_status axq_dequantize(int64_t M, int64_t N, const int32_t* acc, int64_t ldacc,
                          const float* d_scale_a, const float* d_scale_w, const float* bias,
                          float* y, int64_t ldy, void* stream);
axq_status axq_dequantize_nhwc_to_nchw(int64_t N, int64_t HW, int64_t C, const int32_t* acc,
                                       const float* d_scale_a, const float* d_scale_w,
                                       const float* bias, float* y, void* stream);
axq_status axq_epilogue_apply(int64_t M, int64_t N, const int32_t* acc, int64_t ldacc,
                              const axq_epilogue* ep, void* stream);

/* ---------------------------------------------------------------------------------
 * Model glue for the ResNet-50-shaped forward (BASELINE.json configs[3]; A16/A17).
 * axq_maxpool2d_nhwc_i8: max pooling on int8 codes NHWC [N][H][W][C] -> [N][Ho][Wo][C],
 *   window R x S, stride, padding; out-of-image taps are ignored (-inf padding).  Pooling
 *   codes equals quantizing the pooled fp32 values because quantization is monotone
 *   (A17).
 * axq_avgpool_nhwc: global average pool fp32 NHWC [N][HW][C] -> y fp32 [N][C]: a sequential
 *   fp32 sum over hw = 0..HW-1, then one IEEE division by (float)HW (A17).  If q is given,
 *   also writes q = quantize(y) with *d_scale / bits (int8 [N][C]).
 * ------------------------------------------------------------------------------- */
axq_status axq_maxpool2d_nhwc_i8(const int8_t* x, int64_t N, int64_t H, int64_t W, int64_t C,
                                 int64_t R, int64_t S, int64_t stride, int64_t pad, int8_t* y,
                                 void* stream);
/* axq_im2col_nhwc_i8: the explicit im2col matrix of P:119 from int8 NHWC codes X [N][H][W][C]
 *   (only channels 0..c_valid-1 used; 0 = all): A[m][k], m = (img, ho, wo), k = (r*S + s)*cv + c
 *   for k < K = R*S*cv, the code at (ho*stride_h - pad_h + r, wo*stride_w - pad_w + s) or 0 at a
 *   padded tap; A[m][K..lda) = 0.  lda % 16 == 0, lda >= K, A 16-byte aligned.  Used for the
 *   3-channel stem, whose implicit im2col would pad C to 4 (33 % more lookups): the matrix then
 *   goes through axq_lut_gemm_wp with K = R*S*3. */
axq_status axq_im2col_nhwc_i8(const int8_t* X, int64_t N, int64_t H, int64_t W, int64_t C, int64_t c_valid,
                              int64_t R, int64_t S, int64_t stride_h, int64_t stride_w, int64_t pad_h,
                              int64_t pad_w, int8_t* A, int64_t lda, void* stream);
/* axq_maxpool2d_nhwc_f32: the same pooling on fp32 NHWC (used by the paper quantizer's
 *   calibration pass, where the pooled real values are histogrammed). */
axq_status axq_maxpool2d_nhwc_f32(const float* x, int64_t N, int64_t H, int64_t W, int64_t C,
                                  int64_t R, int64_t S, int64_t stride, int64_t pad, float* y,
                                  void* stream);
axq_status axq_avgpool_nhwc(const float* x, int64_t N, int64_t HW, int64_t C, float* y,
                            int8_t* q, const float* d_scale, int bits, void* stream);

/* ---------------------------------------------------------------------------------
 * LSTM cell (BASELINE.json configs[4]; "mathematically equivalent with the vanilla
 * Pytorch RNN layer", gates i, f, g, o; A18).  For b in [0,B), j in [0,Hd):
 *   gate_x = fl(gates_ih[b][x*Hd + j] + gates_hh[b][x*Hd + j])   x = i, f, g, o
 *   i = sigma(gate_i), f = sigma(gate_f), g = tanh(gate_g), o = sigma(gate_o)
 *   c[b][j] = fl(fl(f*c) + fl(i*g));  h = fl(o * tanh(c))
 * with the pinned fp32 exp of A18 inside sigma / tanh.  gates_* are fp32 [B][4*Hd] (bias
 * already added by the GEMM epilogues).  c is updated in place; h is written to h_out
 * [B][Hd] (fp32) and, if q_h is given, quantized with *d_scale_h / bits into q_h [B][Hd].
 * ------------------------------------------------------------------------------- */
axq_status axq_lstm_cell(int64_t B, int64_t Hd, const float* gates_ih, const float* gates_hh,
                         float* c, float* h_out, int8_t* q_h, const float* d_scale_h, int bits,
                         void* stream);

/* axq_lstm_recurrent: the whole static-scale recurrence of BASELINE.json configs[4] in one
 *   persistent (cooperative) launch -- per step t = 0..T-1 exactly the chain
 *   axq_lut_gemm_dq(hq_{t-1}, W_hh; bias b_hh) -> axq_lstm_cell (A18),
 *   with h_{-1} = c_{-1} = 0 and hq_t = quantize(h_t, *d_scale_h, bits).
 *   gates_ih: fp32 [T][B][4H] = fl(x_t W_ih^T dequantized + b_ih) (the hoisted input GEMM);
 *   qw_hh: int8 [4H][H] codes; d_scale_w_hh, d_scale_h: device fp32 scalars; b_hh fp32 [4H];
 *   lut: delta8 handle of the same bit width; hs: fp32 [T][B][H] (all h_t); c_out: fp32
 *   [B][H] (c_{T-1}); workspace: device bytes >= 2*B*H + 256, no contents required.
 *   Needs H % 16 == 0 and a grid of ceil(H / #SMs) * ceil(B / 32) <= 16 warps per SM that
 *   fits co-resident (else AXQ_ERR_UNSUPPORTED: use the per-step calls). */
/* ---------------------------------------------------------------------------------
 * NEXT-2: wide ACUs (b = 9..12, "one with 12-bit precision") with int16
 * operand codes.
 * axq_quantize16: q = clamp(rint(x / *d_scale)) to +-(2^(bits-1)-1) as int16 (axq_quantize's
 *   rule, A1-A3), bits in [2, 16].  (axq_scale accepts bits up to 16.)
 * axq_lut_gemm16: acc[m][n] = sum_k LUT[A[m*lda+k]][W[n*ldw+k]] with int16 codes and a WIDE16 /
 *   WIDE32 handle; ep NULL -> raw int32 C [M][ldc], else the fused epilogue of axq_lut_gemm_dq
 *   (row layout; no workspace used).  Guard: K * max|LUT| < 2^31 (else AXQ_ERR_OVERFLOW).
 * ------------------------------------------------------------------------------- */
axq_status axq_quantize16(const float* x, int64_t n, const float* d_scale, int bits, int16_t* q,
                          void* stream);
axq_status axq_lut_gemm16(int64_t M, int64_t N, int64_t K, const int16_t* A, int64_t lda,
                          const int16_t* W, int64_t ldw, axq_lut_t lut, const axq_epilogue* ep,
                          int32_t* C, int64_t ldc, void* stream);

/* NEXT-2 packed ("populate the CPU cores cache with the LUTs", P:322 wider = slower):
 * the wide table tiled by the weights.  For every k and every quad of 4 output columns the four
 * weights select a 2^b-entry slab of the table, T[k][q][ua] = 4 x (E[ua][w(4q+j,k)] + 2^15),
 * staged into shared memory by bulk copies and read with one 64-bit load per 4 lookups.
 * axq_wpack16_create: W int16 codes [N][ldw] (N x K) and a WIDE16 handle (else
 *   AXQ_ERR_UNSUPPORTED; also for K >= 65528).  Allocates N * Kp * 2^(b+1) bytes of tables
 *   (512 MiB for N = K = 256 at b = 12) plus packed weights; synchronizes.
 * axq_lut_gemm16_wp: acc[m][n] = sum_k LUT[A[m][k]][W[n][k]] for int16 codes A [M][lda]
 *   (bit-identical to axq_lut_gemm16); raw int32 C [M][ldc] (ep NULL) or the fused epilogue
 *   (row layout).  Free the pack with axq_wpack_destroy. */
axq_status axq_wpack16_create(axq_lut_t lut, const int16_t* W, int64_t N, int64_t K, int64_t ldw,
                              axq_wpack_t* out);
axq_status axq_lut_gemm16_wp(int64_t M, const int16_t* A, int64_t lda, axq_wpack_t wp,
                             const axq_epilogue* ep, int32_t* C, int64_t ldc, void* stream);

axq_status axq_lstm_recurrent(int64_t T, int64_t B, int64_t H, const float* gates_ih,
                              const int8_t* qw_hh, const float* d_scale_w_hh, const float* b_hh,
                              const float* d_scale_h, int bits, axq_lut_t lut, float* hs,
                              float* c_out, int8_t* workspace, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AXQ_H */
