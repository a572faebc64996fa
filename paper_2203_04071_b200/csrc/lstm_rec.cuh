// lstm_rec.cuh -- the whole recurrence of the approximate LSTM (BASELINE.json configs[4]) in
// one persistent kernel (sm_100a).
//
// Per step t ("the feedback loop in the recurrent layer ... utilizes our custom
// Linear layer"; A18 fixes the arithmetic):
//   acc[b][n] = sum_k LUT[hq_{t-1}[b][k]][W_hh[n][k]]                  (int32, exact)
//   ghh = fl(fl((float)acc * fl(s_h * s_w)) + b_hh[n]);  gate = fl(gih[t][b][n] + ghh)
//   i, f, o = sigma(gate), g = tanh(gate);  c = fl(fl(f*c) + fl(i*g));  h = fl(o * tanh(c))
//   hs[t][b][j] = h;  hq_t[b][j] = clamp(rint(fl(h / s_h)))      (static scale, A7')
// which is exactly what the per-step chain LUT-GEMM + epilogue + lstm_cell_kernel computes.
//
// Design: CTA c owns the hidden units j in [c*H/G, (c+1)*H/G) -- all four gate columns of each
// -- so the cell update needs no exchange of gate values; only the int8 codes of h_t (B x H
// bytes) go through global memory (double-buffered), followed by a grid-wide barrier.  The
// CTA's W_hh rows (4 x units x H codes) and the ACU table (delta8, 64 KiB, transposed
// [uw][ua]) stay in shared memory for all T steps; h_{t-1} is staged per step.  A warp owns
// one unit and 32 batch rows (one per lane); a lookup is the v1 per-lane gather (lanes share
// the weight, so a gather reads one 256-byte table row), the exact part a*w one dp4a per 4 k.
// c stays in a register for the whole sequence.  Launched cooperatively (all CTAs resident).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "epilogue.cuh"
#include "pinned_math.cuh"
#include "lstm_rec_args.h"

namespace axq {


namespace lstmr {
constexpr int NT = 1024;                   // 32 warps: units x row groups x K splits
constexpr int TABLE = 65536;
// h_{t-1} rows in shared memory are H + 16 bytes apart: the lanes of a warp (consecutive batch
// rows) read 16 bytes of their own rows at the same k; at a multiple-of-128-byte stride all of
// them hit the same 4 banks (8-way replays per quarter warp), at H + 16 they spread over all 32
constexpr int H_PAD = 16;
}

__global__ void __launch_bounds__(lstmr::NT, 1) lstm_rec_kernel(const __grid_constant__ LstmRecArgs a) {
    using namespace lstmr;
    extern __shared__ __align__(16) int8_t lr_smem[];
    const int H = a.H, B = a.B, H4 = 4 * a.H;
    const int G = gridDim.x, cta = blockIdx.x;
    const int u0 = (int)(((int64_t)cta * H) / G), u1 = (int)(((int64_t)(cta + 1) * H) / G), nu = u1 - u0;
    const int rg = (B + 31) / 32;
    int8_t* tab_s = lr_smem;                           // 64 KiB
    int8_t* w_s = tab_s + TABLE;                       // [nu][4][H]
    int8_t* h_s = w_s + (size_t)nu * 4 * H;            // [B][H + H_PAD]
    const int HS = H + H_PAD;                          // h_s row stride (bytes)
    int* red_s = reinterpret_cast<int*>(h_s + (size_t)B * HS);  // [32 warps][4][32 lanes]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // warp -> (unit u, row group r, K part ks): the K loop of a (unit, row group) is split
    // over KSP warps (more warps in flight per SM), partial sums reduced through shared memory
    const int KSP = (NT / 32) / (nu * rg) > 0 ? (NT / 32) / (nu * rg) : 1;

    {
        const uint4* src = reinterpret_cast<const uint4*>(a.table);
        uint4* dst = reinterpret_cast<uint4*>(tab_s);
        for (int i = tid; i < TABLE / 16; i += NT) dst[i] = __ldg(src + i);
        const int hv = H / 16;
        for (int i = tid; i < nu * 4 * hv; i += NT) {
            const int row = i / hv, kc = i - row * hv;        // row = u * 4 + gate
            const int u = row >> 2, g = row & 3;
            reinterpret_cast<uint4*>(w_s)[i] =
                __ldg(reinterpret_cast<const uint4*>(a.qw + ((int64_t)g * H + u0 + u) * H) + kc);
        }
    }
    const int ks = warp % KSP, ur = warp / KSP;
    const int u = ur / rg, r = ur - u * rg;
    const int b = r * 32 + lane;
    const bool live = u < nu && b < B;
    const int j = u0 + u;
    const float sc = __fmul_rn(*a.sh, *a.sw);
    const float s_h = *a.sh;
    const float qm = (float)((1 << (a.bits - 1)) - 1);
    float bias[4] = {0.f, 0.f, 0.f, 0.f};
    if (live)
        for (int g = 0; g < 4; ++g) bias[g] = a.b_hh[g * H + j];
    float c = 0.f;
    const int hv = H / 16;

    for (int t = 0; t < a.T; ++t) {
        // h_{t-1} codes -> shared (h_{-1} = 0); L2 reads: other CTAs wrote them this launch
        {
            const int n16 = B * hv;
            const int hsv = HS / 16;
            uint4* dst = reinterpret_cast<uint4*>(h_s);
            if (t == 0) {
                for (int i = tid; i < n16; i += NT) {
                    const int bb = i / hv, kc = i - bb * hv;
                    dst[bb * hsv + kc] = make_uint4(0, 0, 0, 0);
                }
            } else {
                const uint4* src = reinterpret_cast<const uint4*>(a.hq + (size_t)((t - 1) & 1) * B * H);
                for (int i = tid; i < n16; i += NT) {
                    const int bb = i / hv, kc = i - bb * hv;
                    dst[bb * hsv + kc] = __ldcg(src + i);
                }
            }
        }
        __syncthreads();
        int acc[4] = {0, 0, 0, 0};
        if (live) {
            const uint4* hrow = reinterpret_cast<const uint4*>(h_s + (size_t)b * HS);
            const uint4* wrow = reinterpret_cast<const uint4*>(w_s + (size_t)u * 4 * H);
            const int kc0 = (ks * hv) / KSP, kc1 = ((ks + 1) * hv) / KSP;
#pragma unroll 2
            for (int kc = kc0; kc < kc1; ++kc) {
                const uint4 av = hrow[kc];
                uint4 wv[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) wv[g] = wrow[g * hv + kc];
#pragma unroll
                for (int kq = 0; kq < 4; ++kq) {
                    const uint32_t a4 = kq == 0 ? av.x : kq == 1 ? av.y : kq == 2 ? av.z : av.w;
                    const uint32_t alo = __byte_perm(a4, 0u, 0x4140), ahi = __byte_perm(a4, 0u, 0x4342);
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const uint32_t w4 = kq == 0 ? wv[g].x : kq == 1 ? wv[g].y : kq == 2 ? wv[g].z : wv[g].w;
                        const int e0 = tab_s[__byte_perm(alo, w4, 0x1140)];
                        const int e1 = tab_s[__byte_perm(alo, w4, 0x3352)];
                        const int e2 = tab_s[__byte_perm(ahi, w4, 0x1160)];
                        const int e3 = tab_s[__byte_perm(ahi, w4, 0x3372)];
                        acc[g] = __dp4a((int)a4, (int)w4, acc[g]) + e0 + e1 + e2 + e3;
                    }
                }
            }
        }
        if (KSP > 1) {
#pragma unroll
            for (int g = 0; g < 4; ++g) red_s[(warp * 4 + g) * 32 + lane] = acc[g];
            __syncthreads();
            if (ks == 0)
                for (int q = 1; q < KSP; ++q)
#pragma unroll
                    for (int g = 0; g < 4; ++g) acc[g] += red_s[((warp + q) * 4 + g) * 32 + lane];
        }
        if (live && ks == 0) {
            // epilogue (pinned order) + cell, as axq_lut_gemm_dq + lstm_cell_kernel
            const float* gi = a.gih + ((size_t)t * B + b) * H4 + j;
            float gate[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const float hh = __fadd_rn(__fmul_rn(__int2float_rn(acc[g]), sc), bias[g]);
                gate[g] = __fadd_rn(__ldg(gi + g * H), hh);
            }
            const float ig = pinned_sigmoid(gate[0]), fg = pinned_sigmoid(gate[1]);
            const float gg = pinned_tanh(gate[2]), og = pinned_sigmoid(gate[3]);
            c = __fadd_rn(__fmul_rn(fg, c), __fmul_rn(ig, gg));
            const float h = __fmul_rn(og, pinned_tanh(c));
            a.hs[((size_t)t * B + b) * H + j] = h;
            a.hq[(size_t)(t & 1) * B * H + (size_t)b * H + j] = epi_quant(h, s_h, qm);
        }
        // grid barrier: every CTA's h_t codes are written before anyone reads them
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicAdd(a.bar, 1u);
            const unsigned int target = (unsigned int)(t + 1) * (unsigned int)G;
            unsigned int v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(a.bar) : "memory");
            } while (v < target);
        }
        __syncthreads();
    }
    if (live && ks == 0) a.c_out[(size_t)b * H + j] = c;
}

}  // namespace axq
