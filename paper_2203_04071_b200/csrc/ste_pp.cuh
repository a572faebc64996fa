// ste_pp.cuh -- the pre-converted ("pp") tensor-core path of the NEXT-4 STE backward products
// (A36', §4.6).  Included by mm_ste.cu after ste_desc / bf16_rn_bits /
// ste_reduce_kernel.
//
// Each product C[Mg][Ng] = mask * A(Mg x Kg) . fq(B)(Kg x Ng) first converts its operands ONCE
// into the tiled canonical K-major layout the MMA reads, so a pipeline stage of the GEMM is two
// bulk copies and the tensor cores are not starved by a per-tile fp32 -> bf16 conversion:
//   A' = [m tile][k tile][term hi / mid / lo][chunk 0..3][128 rows][8 bf16]   (24 KiB per tile pair)
//   B' = [n tile][k tile][chunk 0..3][128 rows][8 bf16]                      (8 KiB)
// (row = the GEMM's M resp. N index, chunk = 8 consecutive summed indices p; the fp32 operand is
// split exactly into hi + mid + lo bf16 terms, the int8 codes are exact in bf16).
//
// Launch structure of one backward: ONE prep launch converts every operand of both products
// (and runs the first column-sum pass of gb) from a job table; ONE GEMM launch (programmatic
// dependent launch: its prologue overlaps the prep's tail) computes both products, 128 x 128
// output tiles, K split into up to 8 slices that a thread-block cluster reduces through
// distributed shared memory.  A product whose K needs more than 8 slices (a conv's weight
// gradient) runs alone, clusters of 8 writing partial slots that ste_reduce_kernel adds.
#pragma once

namespace axq {
namespace stepp {
constexpr int BM = 128, BN = 128, BK = 32;
constexpr int TILE_A = 3 * BM * BK * 2;        // 24 KiB: hi, mid, lo
constexpr int TILE_B = BN * BK * 2;            // 8 KiB
constexpr int STAGE = TILE_A + TILE_B;         // 32 KiB
constexpr int STAGES = 3;                      // 2 CTAs per SM: one's epilogue overlaps the other's main loop
constexpr int TS = BN + 4;                     // epilogue row stride (floats): conflict-free float4 rows
constexpr int SMEM = STAGES * STAGE + 128;
static_assert(BM * TS * 4 <= STAGES * STAGE, "epilogue tile must fit the stage buffers");
// instruction descriptor: D f32, A / B bf16, K-major, N >> 3, M >> 4
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

enum PrepKind { PREP_A = 0, PREP_B = 1, PREP_COLSUM = 2, PREP_B_CONV = 3 };
// implicit im2col for PREP_B_CONV: B[p][j] = x[n][ho*sh - ph + r][wo*sw - pw + s][c] (0 outside)
// with p = (n, ho, wo) an output pixel and j = (r, s, c) a tap (the conv is the GEMM of
// its im2col matrix) -- the gw operand read straight from the NHWC codes
struct ConvGeo {
    int H, W, C, Ho, Wo, sh, sw, ph, pw, S;
};
// one job of the prep launch (blocks: its share of the grid)
struct PrepJob {
    int kind;
    int ta, pcs, vec;       // A: operand stored transposed (A[p][i]), per-p scale folded in, 16-byte loads
    int64_t rows, K, ld;    // A: Mg x Kg, lda; B: Ng columns x Kg, ldb; colsum: M rows x N columns, ldg
    int64_t KT;             // k tiles (colsum: row blocks RB)
    const void* src;
    const float* s_b;
    void* out;
    int64_t blocks;
    ConvGeo cg;             // PREP_B_CONV only
};
struct PrepArgs {
    PrepJob job[5];
    int njobs;
};
// one product of the GEMM launch: CTAs [cta0, cta0 + Mt * Nt * S), slice z fastest
struct GemmJob {
    int64_t M, N, KT, kps, ldc, Mt, Nt, S, cta0;
    const uint4* Ap;
    const uint4* Bp;
    const float* s_b;
    float* C;
    const float* R;
    const float* clip;
    int clip_vec, pcs;
};
struct GemmArgs {
    GemmJob job[2];
    int njobs;
};
}  // namespace stepp

// A' of one (m tile, k tile), thread -> (row, chunk): 8 consecutive p of row i split into 3
// terms.  TA (A[p][i]): row fastest, a warp reads 32 consecutive i per p; else chunk fastest,
// 4 threads read one row's 32 consecutive p (two float4 each when aligned).
__device__ __forceinline__ void pp_prep_a(const stepp::PrepJob& J, int64_t g0, int64_t gs) {
    const int64_t M = J.rows, K = J.K, lda = J.ld, KT = J.KT;
    const float* __restrict__ A = static_cast<const float*>(J.src);
    uint4* __restrict__ out = static_cast<uint4*>(J.out);
    const bool ta = J.ta != 0;
    const int64_t total = ((M + 127) / 128) * KT * 4 * 128;
    for (int64_t g = g0; g < total; g += gs) {
        const int row = ta ? (int)(g & 127) : (int)((g >> 2) & 127);
        const int c = ta ? (int)((g >> 7) & 3) : (int)(g & 3);
        const int64_t tk = g >> 9;                       // (m tile, k tile)
        const int64_t kt = tk % KT, mt = tk / KT;
        const int64_t i = mt * 128 + row, p0 = kt * 32 + c * 8;
        float a[8];
        if (!ta && J.vec && i < M && p0 + 8 <= K) {
            const float4 f0 = __ldg(reinterpret_cast<const float4*>(A + i * lda + p0));
            const float4 f1 = __ldg(reinterpret_cast<const float4*>(A + i * lda + p0) + 1);
            a[0] = f0.x; a[1] = f0.y; a[2] = f0.z; a[3] = f0.w;
            a[4] = f1.x; a[5] = f1.y; a[6] = f1.z; a[7] = f1.w;
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int64_t p = p0 + e;
                a[e] = (i < M && p < K) ? (ta ? __ldg(A + p * lda + i) : __ldg(A + i * lda + p)) : 0.f;
            }
        }
        if (J.pcs) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (p0 + e < K) a[e] = __fmul_rn(a[e], __ldg(J.s_b + p0 + e));   // per-channel scale of p
        }
        uint32_t hw[4], mw[4], lw[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
            uint16_t h[2], md[2], l[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const float x = a[e + u];
                h[u] = bf16_rn_bits(x);
                const float r1 = __fsub_rn(x, __bfloat162float(__ushort_as_bfloat16(h[u])));
                md[u] = bf16_rn_bits(r1);
                const float r2 = __fsub_rn(r1, __bfloat162float(__ushort_as_bfloat16(md[u])));
                l[u] = bf16_rn_bits(r2);
            }
            hw[e / 2] = (uint32_t)h[0] | ((uint32_t)h[1] << 16);
            mw[e / 2] = (uint32_t)md[0] | ((uint32_t)md[1] << 16);
            lw[e / 2] = (uint32_t)l[0] | ((uint32_t)l[1] << 16);
        }
        uint4* base = out + tk * (3 * 4 * 128) + c * 128 + row;      // in 16-byte units
        base[0] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        base[4 * 128] = make_uint4(mw[0], mw[1], mw[2], mw[3]);
        base[8 * 128] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

// B' of one (n tile, k tile), thread -> (4 columns j .. j + 3, chunk): the int8 codes B[p][j] of
// 8 consecutive p (one 4-byte load per p when aligned) as bf16 into 4 rows of the tile
__device__ __forceinline__ void pp_prep_b(const stepp::PrepJob& J, int64_t g0, int64_t gs) {
    const int64_t N = J.rows, K = J.K, ldb = J.ld, KT = J.KT;
    const int8_t* __restrict__ B = static_cast<const int8_t*>(J.src);
    uint4* __restrict__ out = static_cast<uint4*>(J.out);
    const int64_t total = ((N + 127) / 128) * KT * 4 * 32;
    for (int64_t g = g0; g < total; g += gs) {
        const int rq = (int)(g & 31), c = (int)((g >> 5) & 3);
        const int64_t tk = g >> 7;
        const int64_t kt = tk % KT, nt = tk / KT;
        const int64_t j0 = nt * 128 + rq * 4, p0 = kt * 32 + c * 8;
        uint32_t q[8];     // q[e] = bytes of B[p0 + e][j0 .. j0 + 3]
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int64_t p = p0 + e;
            uint32_t v = 0u;
            if (p < K) {
                if (J.vec && j0 + 4 <= N) {
                    v = __ldg(reinterpret_cast<const unsigned int*>(B + p * ldb + j0));
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (j0 + u < N) v |= (uint32_t)(uint8_t)B[p * ldb + j0 + u] << (8 * u);
                }
            }
            q[e] = v;
        }
        uint4* base = out + tk * (4 * 128) + c * 128 + rq * 4;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
                const float f0 = (float)(int8_t)(q[e] >> (8 * u)), f1 = (float)(int8_t)(q[e + 1] >> (8 * u));
                w[e / 2] = (uint32_t)bf16_rn_bits(f0) | ((uint32_t)bf16_rn_bits(f1) << 16);
            }
            base[u] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

// B' from the NHWC codes through the implicit im2col (PREP_B_CONV; rows = R*S*C taps, K = the
// output pixels, < 2^31): thread -> (4 taps j .. j + 3, chunk of 8 pixels); with C % 4 == 0 the 4
// taps are 4 channels of one (r, s): one 4-byte load per pixel
__device__ __forceinline__ void pp_prep_b_conv(const stepp::PrepJob& J, int64_t g0, int64_t gs) {
    const int64_t Nc = J.rows, K = J.K, KT = J.KT;
    const stepp::ConvGeo& g = J.cg;
    const int8_t* __restrict__ X = static_cast<const int8_t*>(J.src);
    uint4* __restrict__ out = static_cast<uint4*>(J.out);
    const int64_t total = ((Nc + 127) / 128) * KT * 4 * 32;
    const int hw = g.Ho * g.Wo;
    const bool c4 = (g.C & 3) == 0 && J.vec;
    for (int64_t gi = g0; gi < total; gi += gs) {
        const int rq = (int)(gi & 31), c = (int)((gi >> 5) & 3);
        const int64_t tk = gi >> 7;
        const int64_t kt = tk % KT, nt = tk / KT;
        const int64_t j0 = nt * 128 + rq * 4;
        const int p0 = (int)(kt * 32 + c * 8);
        // taps of j0 .. j0 + 3
        int tr[4], ts[4], tc[4];
        bool tv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = (int)(j0 + u < Nc ? j0 + u : Nc - 1);
            const int rs = j / g.C;
            tc[u] = j - rs * g.C;
            tr[u] = rs / g.S;
            ts[u] = rs - tr[u] * g.S;
            tv[u] = j0 + u < Nc;
        }
        int n = p0 / hw, rem = p0 - n * hw;
        int ho = rem / g.Wo, wo = rem - ho * g.Wo;
        uint32_t q[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            uint32_t v = 0u;
            if (p0 + e < K) {
                const int hb = ho * g.sh - g.ph, wb = wo * g.sw - g.pw;
                const int8_t* xb = X + (int64_t)n * g.H * g.W * g.C;
                if (c4 && tv[3]) {
                    const int hi = hb + tr[0], wi = wb + ts[0];
                    if ((unsigned)hi < (unsigned)g.H && (unsigned)wi < (unsigned)g.W)
                        v = __ldg(reinterpret_cast<const unsigned int*>(xb + ((int64_t)hi * g.W + wi) * g.C + tc[0]));
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int hi = hb + tr[u], wi = wb + ts[u];
                        if (tv[u] && (unsigned)hi < (unsigned)g.H && (unsigned)wi < (unsigned)g.W)
                            v |= (uint32_t)(uint8_t)xb[((int64_t)hi * g.W + wi) * g.C + tc[u]] << (8 * u);
                    }
                }
            }
            q[e] = v;
            if (++wo == g.Wo) {
                wo = 0;
                if (++ho == g.Ho) {
                    ho = 0;
                    ++n;
                }
            }
        }
        uint4* base = out + tk * (4 * 128) + c * 128 + rq * 4;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
                const float f0 = (float)(int8_t)(q[e] >> (8 * u)), f1 = (float)(int8_t)(q[e + 1] >> (8 * u));
                w[e / 2] = (uint32_t)bf16_rn_bits(f0) | ((uint32_t)bf16_rn_bits(f1) << 16);
            }
            base[u] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

// column sums, first pass (the ste_colsum_part_kernel order): block (column group x, row block
// y) of RB row blocks -> out[y][n] (RB = 1: out = gb)
__device__ __forceinline__ void pp_colsum(const stepp::PrepJob& J, int64_t bid, float (*red)[33]) {
    const int64_t M = J.rows, N = J.K, ldg = J.ld, RB = J.KT;
    const float* __restrict__ gy = static_cast<const float*>(J.src);
    float* __restrict__ part = static_cast<float*>(J.out);
    const int64_t cg = (N + 31) / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t b = bid; b < cg * RB; b += J.blocks) {
        const int64_t bx = b % cg, by = b / cg;
        const int64_t n = bx * 32 + lane;
        const int64_t rows = (M + RB - 1) / RB, r0 = by * rows, r1 = min(M, r0 + rows);
        float s = 0.f;
        if (n < N) {
#pragma unroll 8
            for (int64_t m = r0 + warp; m < r1; m += 8) s = __fadd_rn(s, __ldg(gy + m * ldg + n));
        }
        __syncthreads();
        red[warp][lane] = s;
        __syncthreads();
        if (warp == 0 && n < N) {
            float t = red[0][lane];
            for (int w = 1; w < 8; ++w) t = __fadd_rn(t, red[w][lane]);
            part[by * N + n] = t;
        }
    }
}

__global__ void __launch_bounds__(256) ste_prep_kernel(const __grid_constant__ stepp::PrepArgs args) {
    __shared__ float red[8][33];
    int jb = 0;
    int64_t b0 = 0;
    while (jb + 1 < args.njobs && (int64_t)blockIdx.x >= b0 + args.job[jb].blocks) b0 += args.job[jb++].blocks;
    const stepp::PrepJob& J = args.job[jb];
    const int64_t bid = (int64_t)blockIdx.x - b0;
    if (J.kind == stepp::PREP_A) pp_prep_a(J, bid * 256 + threadIdx.x, J.blocks * 256);
    else if (J.kind == stepp::PREP_B) pp_prep_b(J, bid * 256 + threadIdx.x, J.blocks * 256);
    else if (J.kind == stepp::PREP_B_CONV) pp_prep_b_conv(J, bid * 256 + threadIdx.x, J.blocks * 256);
    else pp_colsum(J, bid, red);
    // the GEMM launch (programmatic dependent launch) may start its prologue now; its producer
    // waits (griddepcontrol.wait) for this grid's completion before the first bulk copy
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// One 128 x 128 output tile, K slice z, of product job[jb]: thread 0 streams the stages (two bulk
// copies each), thread 32 issues the MMAs (3 terms x 2 K steps of 16 per stage into one TMEM
// accumulator).  Epilogue: the 4 warps move the accumulator into a padded shared-memory tile;
// the CZ CTAs of a cluster (the slices z = CZ * c .. CZ * c + CZ - 1 of one tile) then reduce
// their tiles through distributed shared memory, CTA rank q owning rows [q * 128 / CZ,
// (q + 1) * 128 / CZ), adding the slices in rank order (deterministic), and write those rows with
// 512-byte row stores -- to C (scaled, masked) when the cluster covers every slice, else
// (scaled) to partial slot c of the workspace for ste_reduce_kernel.
template <int CZ>
__global__ void __launch_bounds__(128) ste_pp_kernel(const __grid_constant__ stepp::GemmArgs args) {
    using namespace stepp;
    extern __shared__ __align__(1024) uint8_t pp_smem[];
    const int jb = (args.njobs > 1 && (int64_t)blockIdx.x >= args.job[1].cta0) ? 1 : 0;
    const GemmJob& J = args.job[jb];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t local = (int64_t)blockIdx.x - J.cta0;
    const int64_t z = local % J.S, tile = local / J.S;
    const bool valid = tile < J.Mt * J.Nt;             // CTAs padding the job to whole clusters: no work
    const int64_t nt = tile % J.Nt, mt = tile / J.Nt;
    const int64_t M = J.M, N = J.N, KT = J.KT, ldc = J.ldc;
    const int64_t kt0 = z * J.kps, kt1 = valid ? min(KT, kt0 + J.kps) : kt0;
    const int nkt = (int)max((int64_t)0, kt1 - kt0);
    // reduction group: the G = min(S, CZ) consecutive cluster ranks holding the slices of one tile
    // (S <= CZ: every slice, the result is final; S > CZ: slot z / CZ of the partials)
    const int G = (int)min(J.S, (int64_t)CZ);
    const bool final_out = J.S <= CZ;
    float* C = final_out ? J.C : J.C + (z / CZ) * M * ldc;
    const uint32_t s_base = smem_u32(pp_smem);
    const uint32_t bar_full = s_base + STAGES * STAGE, bar_mma = bar_full + 8 * STAGES;
    const uint32_t bar_done = bar_mma + 8 * STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pp_smem + STAGES * STAGE + 16 * STAGES + 8);
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_mma + 8 * s, 1);
        }
        mbar_init(bar_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(BN) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (tid == 0) {
        // A' / B' come from the preceding prep grid (programmatic dependent launch)
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
        for (int s = 0; s < nkt; ++s) {
            const int buf = s % STAGES;
            if (s >= STAGES) mbar_wait(bar_mma + 8 * buf, ((s / STAGES) - 1) & 1u);
            const uint32_t bar = bar_full + 8 * buf;
            mbar_expect_tx(bar, STAGE);
            const int64_t kt = kt0 + s;
            bulk_g2s(s_base + buf * STAGE, J.Ap + (mt * KT + kt) * (3 * 4 * 128), TILE_A, bar);
            bulk_g2s(s_base + buf * STAGE + TILE_A, J.Bp + (nt * KT + kt) * (4 * BN), TILE_B, bar);
        }
    } else if (tid == 32) {
        for (int s = 0; s < nkt; ++s) {
            const int buf = s % STAGES;
            mbar_wait(bar_full + 8 * buf, (s / STAGES) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint32_t sa = s_base + buf * STAGE, sbb = sa + TILE_A;
#pragma unroll
            for (int t = 0; t < 3; ++t)
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk) {
                    // K step of 16 = chunks 2kk, 2kk+1: LBO = one chunk (rows x 16 B), SBO = 128 B
                    const uint64_t ad = ste_desc(sa + t * (TILE_A / 3) + kk * 2 * BM * 16, BM * 16, 128);
                    const uint64_t bd = ste_desc(sbb + kk * 2 * BN * 16, BN * 16, 128);
                    const uint32_t acc = (s > 0 || t > 0 || kk > 0) ? 1u : 0u;
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                                 "l"(ad), "l"(bd), "r"(IDESC), "r"(acc)
                                 : "memory");
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             bar_mma + 8 * buf) : "memory");
        }
        if (nkt > 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             bar_done) : "memory");
    }
    // everyone waits for all MMAs: one more commit onto bar_done (single phase; a per-stage
    // barrier's parity would alias with its phase STAGES stages earlier)
    if (nkt > 0) mbar_wait(bar_done, 0u);
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // TMEM -> shared tile T[128][TS] (row = TMEM lane; the stage buffers are idle now)
    float* T = reinterpret_cast<float*>(pp_smem);
    {
        const int r = warp * 32 + lane;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t v[16];
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (nkt == 0) {
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = 0u;
            }
            float4* dst = reinterpret_cast<float4*>(T + r * TS + c0);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                dst[e] = make_float4(__uint_as_float(v[4 * e]), __uint_as_float(v[4 * e + 1]),
                                     __uint_as_float(v[4 * e + 2]), __uint_as_float(v[4 * e + 3]));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    uint32_t q = 0;
    if (CZ > 1) {
        asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(q));
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
        __syncthreads();
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(BN) : "memory");
    // rows [r0, r1): a warp writes one 128-column row per step (lane l: columns 4l .. 4l + 3), the
    // CZ slices of RB rows loaded before any is added (one DSMEM round trip per RB rows)
    constexpr int RB = CZ >= 8 ? 1 : 8 / CZ;
    const int qg = (int)q % G, gbase = (int)q - qg;      // rank within the group, the group's first rank
    const int r0 = valid ? qg * BM / G : 0, r1 = valid ? (qg + 1) * BM / G : 0;
    const float sb = J.pcs ? 1.f : *J.s_b;
    const bool apply_mask = J.R && final_out;
    const uint32_t t_base = smem_u32(T);
    const int col = 4 * lane;
    const int64_t j = nt * BN + col;
    const bool vec = (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0 && j + 4 <= N;
    for (int rb = r0 + warp; rb < r1; rb += 4 * RB) {
        float4 y[RB][CZ];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const int r = rb + 4 * u;
            if (r < r1) {
                const uint32_t a = t_base + (uint32_t)(r * TS + col) * 4u;
#pragma unroll
                for (int zz = 0; zz < CZ; ++zz) {
                    if (CZ == 1) {
                        y[u][zz] = *reinterpret_cast<const float4*>(T + r * TS + col);
                    } else if (zz < G) {
                        uint32_t ra;
                        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(a), "r"(gbase + zz));
                        asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                                     : "=f"(y[u][zz].x), "=f"(y[u][zz].y), "=f"(y[u][zz].z), "=f"(y[u][zz].w)
                                     : "r"(ra));
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const int r = rb + 4 * u;
            const int64_t i = mt * BM + r;
            if (r >= r1 || i >= M || j >= N) continue;
            float4 x = y[u][0];
#pragma unroll
            for (int zz = 1; zz < CZ; ++zz) {
                if (zz >= G) break;
                x.x = __fadd_rn(x.x, y[u][zz].x); x.y = __fadd_rn(x.y, y[u][zz].y);
                x.z = __fadd_rn(x.z, y[u][zz].z); x.w = __fadd_rn(x.w, y[u][zz].w);
            }
            if (!J.pcs) {
                x.x = __fmul_rn(x.x, sb); x.y = __fmul_rn(x.y, sb);
                x.z = __fmul_rn(x.z, sb); x.w = __fmul_rn(x.w, sb);
            }
            if (apply_mask) {
                const float cl = J.clip_vec ? J.clip[i] : *J.clip;
                const float* rr = J.R + i * ldc + j;
                if (j + 0 < N && !(fabsf(rr[0]) <= cl)) x.x = 0.f;
                if (j + 1 < N && !(fabsf(rr[1]) <= cl)) x.y = 0.f;
                if (j + 2 < N && !(fabsf(rr[2]) <= cl)) x.z = 0.f;
                if (j + 3 < N && !(fabsf(rr[3]) <= cl)) x.w = 0.f;
            }
            float* crow = C + i * ldc + j;
            if (vec) {
                *reinterpret_cast<float4*>(crow) = x;
            } else {
                if (j + 0 < N) crow[0] = x.x;
                if (j + 1 < N) crow[1] = x.y;
                if (j + 2 < N) crow[2] = x.z;
                if (j + 3 < N) crow[3] = x.w;
            }
        }
    }
    if (CZ > 1)   // keep this CTA's tile alive until every rank of the cluster has read it
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// ---- host side ----
// Plan of one product: tiles, K slices (S), cluster size (CZ in 1, 2, 4, 8), partial slots.
// S: ~2 CTAs per SM, >= 4 k tiles per slice; S <= 8 rounds up to a power of two (one cluster per
// tile), S > 8: clusters of 8 and S / 8 partial slots (room permitting).
struct PrepPlan {
    int64_t Mt, Nt, KT, a_elems, b_elems, S0, S, CZ, slots, kps, part;
};
static inline int64_t round32(int64_t e) { return (e + 31) / 32 * 32; }
static inline int64_t pp_ab_elems(const PrepPlan& p) { return round32(p.a_elems) + round32(p.b_elems); }

// largest cluster (a power of two): 8-CTA clusters of these 98 KiB CTAs fit only ~15 at a time
// on a 148-SM part (measured: cudaOccupancyMaxActiveClusters), 4-CTA ones fill the SMs
static int64_t pp_max_cz() {
    static const int64_t v = [] {
        const char* e = std::getenv("AXQ_STE_MAXCZ");
        const int64_t x = e ? std::atoll(e) : 4;
        return x >= 8 ? 8 : x >= 4 ? 4 : x >= 2 ? 2 : 1;
    }();
    return v;
}
static bool pp_plan(int64_t Mg, int64_t Ng, int64_t Kg, int64_t ldc, int sms, int64_t room_for_slots, PrepPlan& pl) {
    using namespace stepp;
    pl.Mt = (Mg + BM - 1) / BM;
    pl.Nt = (Ng + BN - 1) / BN;
    pl.KT = (Kg + BK - 1) / BK;
    if (pl.Mt <= 0 || pl.Nt <= 0 || pl.KT <= 0 || pl.Nt > 65535) return false;
    pl.a_elems = pl.Mt * pl.KT * (TILE_A / 4);
    pl.b_elems = pl.Nt * pl.KT * (TILE_B / 4);
    const int64_t tiles = pl.Mt * pl.Nt, mcz = pp_max_cz();
    int64_t S = std::min<int64_t>({(2 * (int64_t)sms + tiles - 1) / tiles, 128, std::max<int64_t>(1, pl.KT / 4)});
    pl.S0 = S;
    if (S <= mcz) {
        S = S <= 1 ? 1 : S <= 2 ? 2 : S <= 4 ? 4 : 8;
        pl.CZ = S;
    } else {
        pl.CZ = mcz;
        const int64_t slots = std::min<int64_t>((S + mcz - 1) / mcz, room_for_slots / std::max<int64_t>(1, round32(Mg * ldc)));
        S = slots >= 2 ? slots * mcz : mcz;
    }
    pl.kps = (pl.KT + S - 1) / S;
    if (S > mcz) {   // drop whole clusters that would hold no k tile
        S = (pl.KT + pl.kps - 1) / pl.kps;
        S = std::max<int64_t>(mcz, (S + mcz - 1) / mcz * mcz);
    }
    pl.S = S;
    pl.slots = S / pl.CZ;
    pl.part = pl.slots > 1 ? round32(pl.slots * Mg * ldc) : 0;
    if (pl.Mt * pl.Nt * pl.S > 0x7fffffff) return false;
    return true;
}
// S slices in one cluster of S CTAs (S a power of two <= pp_max_cz()), no partial slots
static void pp_set_s(PrepPlan& pl, int64_t S) {
    pl.S = S;
    pl.CZ = S;
    pl.kps = (pl.KT + S - 1) / S;
    pl.slots = 1;
    pl.part = 0;
}
// CTAs of a product in a launch with cluster size cz: whole clusters (S <= cz: cz / S tiles per
// cluster, the last one padded with idle CTAs)
static int64_t pp_ctas(const PrepPlan& pl, int64_t cz) {
    const int64_t n = pl.Mt * pl.Nt * pl.S;
    return (n + cz - 1) / cz * cz;
}

static stepp::PrepJob pp_job_a(bool ta, int64_t Mg, int64_t Kg, const float* A, int64_t lda, const float* sB,
                               bool pcs, int64_t KT, uint4* out, int sms) {
    stepp::PrepJob j{};
    j.kind = stepp::PREP_A;
    j.ta = ta;
    j.pcs = pcs;
    j.vec = ((lda & 3) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) ? 1 : 0;
    j.rows = Mg;
    j.K = Kg;
    j.ld = lda;
    j.KT = KT;
    j.src = A;
    j.s_b = sB;
    j.out = out;
    j.blocks = std::max<int64_t>(1, std::min<int64_t>(((Mg + 127) / 128 * KT * 512 + 255) / 256, 8 * (int64_t)sms));
    return j;
}
static stepp::PrepJob pp_job_b(int64_t Ng, int64_t Kg, const int8_t* B, int64_t ldb, int64_t KT, uint4* out, int sms) {
    stepp::PrepJob j{};
    j.kind = stepp::PREP_B;
    j.vec = ((ldb & 3) == 0 && (reinterpret_cast<uintptr_t>(B) & 3) == 0) ? 1 : 0;
    j.rows = Ng;
    j.K = Kg;
    j.ld = ldb;
    j.KT = KT;
    j.src = B;
    j.out = out;
    j.blocks = std::max<int64_t>(1, std::min<int64_t>(((Ng + 127) / 128 * KT * 128 + 255) / 256, 8 * (int64_t)sms));
    return j;
}
static stepp::PrepJob pp_job_b_conv(int64_t Nc, int64_t Mp, const int8_t* X, const stepp::ConvGeo& cg, int64_t KT,
                                    uint4* out, int sms) {
    stepp::PrepJob j = pp_job_b(Nc, Mp, X, 0, KT, out, sms);
    j.kind = stepp::PREP_B_CONV;
    j.vec = (reinterpret_cast<uintptr_t>(X) & 3) == 0 ? 1 : 0;
    j.cg = cg;
    return j;
}
static stepp::PrepJob pp_job_colsum(int64_t M, int64_t N, const float* gy, int64_t RB, float* out, int sms) {
    stepp::PrepJob j{};
    j.kind = stepp::PREP_COLSUM;
    j.rows = M;
    j.K = N;
    j.ld = N;
    j.KT = RB;
    j.src = gy;
    j.out = out;
    j.blocks = std::max<int64_t>(1, std::min<int64_t>((N + 31) / 32 * RB, 8 * (int64_t)sms));
    return j;
}
static stepp::GemmJob pp_job_gemm(const PrepPlan& pl, int64_t Mg, int64_t Ng, int64_t ldc, const uint4* Ap,
                                  const uint4* Bp, const float* sB, bool pcs, float* out, const float* R,
                                  const float* clip, bool clip_vec, int64_t cta0) {
    stepp::GemmJob g{};
    g.M = Mg;
    g.N = Ng;
    g.KT = pl.KT;
    g.kps = pl.kps;
    g.ldc = ldc;
    g.Mt = pl.Mt;
    g.Nt = pl.Nt;
    g.S = pl.S;
    g.cta0 = cta0;
    g.Ap = Ap;
    g.Bp = Bp;
    g.s_b = sB;
    g.C = out;
    g.R = R;
    g.clip = clip;
    g.clip_vec = clip_vec ? 1 : 0;
    g.pcs = pcs ? 1 : 0;
    return g;
}

static void pp_launch_prep(const stepp::PrepArgs& a, cudaStream_t st) {
    int64_t blocks = 0;
    for (int i = 0; i < a.njobs; ++i) blocks += a.job[i].blocks;
    ste_prep_kernel<<<(unsigned)blocks, 256, 0, st>>>(a);
}

template <int CZ>
static void pp_launch_gemm_cz(const stepp::GemmArgs& a, int64_t ctas, cudaStream_t st) {
    auto kern = ste_pp_kernel<CZ>;
    static unsigned configured = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(configured & (1u << (dev & 31)))) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, stepp::SMEM);
        configured |= 1u << (dev & 31);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ctas, 1, 1);
    cfg.blockDim = dim3(128, 1, 1);
    cfg.dynamicSmemBytes = stepp::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CZ;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, kern, a);
}
static void pp_launch_gemm(const stepp::GemmArgs& a, int64_t cz, int64_t ctas, cudaStream_t st) {
    switch (cz) {
        case 1: pp_launch_gemm_cz<1>(a, ctas, st); break;
        case 2: pp_launch_gemm_cz<2>(a, ctas, st); break;
        case 4: pp_launch_gemm_cz<4>(a, ctas, st); break;
        default: pp_launch_gemm_cz<8>(a, ctas, st); break;
    }
}
}  // namespace axq
