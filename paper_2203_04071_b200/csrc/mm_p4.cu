// mm_p4.cu -- host side of the P4 LUT kernel (lut_p4.cuh): weight packing and launch.
#include "lut_p4.cuh"
#include "lut_p4w.cuh"
#include "mm_launch.h"

namespace axq {

int p4_pack(const int8_t* W, int64_t N, int64_t K, int64_t ldw, int64_t Kp, const int8_t* dtab,
            uint32_t* tables, int8_t* wpk, int half, int swap, cudaStream_t st) {
    const int64_t nb = (N + p4::TN - 1) / p4::TN;
    const int rows = half ? 128 : 256;
    const int64_t t2 = nb * Kp * p4::TN;
    static unsigned pack_configured = 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    if (!(pack_configured & (1u << (dev & 31)))) {
        cudaError_t e = cudaFuncSetAttribute(p4_pack_tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        if (e != cudaSuccess) return (int)e;
        pack_configured |= 1u << (dev & 31);
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t items = nb * ((Kp + PACK_KC - 1) / PACK_KC);
    p4_pack_tables_kernel<<<(unsigned)std::min<int64_t>(items, (int64_t)(sms > 0 ? sms : 148) * 3), PACK_THREADS,
                            65536, st>>>(W, N, K, ldw, Kp, dtab, tables, rows, swap);
    p4_pack_w_kernel<<<(unsigned)std::min<int64_t>((t2 + 255) / 256, 148 * 16), 256, 0, st>>>(W, N, K, ldw, Kp, wpk);
    return (int)cudaGetLastError();
}

int p4_pack_w(const int8_t* W, int64_t N, int64_t K, int64_t ldw, int64_t Kp, int8_t* wpk, cudaStream_t st) {
    const int64_t t2 = ((N + p4::TN - 1) / p4::TN) * Kp * p4::TN;
    p4_pack_w_kernel<<<(unsigned)std::min<int64_t>((t2 + 255) / 256, 148 * 16), 256, 0, st>>>(W, N, K, ldw, Kp, wpk);
    return (int)cudaGetLastError();
}

int p4_pack16(const int8_t* W, int64_t N, int64_t K, int64_t ldw, int64_t Kp, const int16_t* e16,
              uint32_t* tables, cudaStream_t st) {
    static unsigned configured = 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    if (!(configured & (1u << (dev & 31)))) {
        cudaError_t e = cudaFuncSetAttribute(p4_pack16_tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             131072);
        if (e != cudaSuccess) return (int)e;
        configured |= 1u << (dev & 31);
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nb = (N + p4::TN - 1) / p4::TN;
    const int64_t items = nb * ((Kp + PACK_KC - 1) / PACK_KC);
    p4_pack16_tables_kernel<<<(unsigned)std::min<int64_t>(items, (int64_t)(sms > 0 ? sms : 148)), PACK_THREADS,
                              131072, st>>>(W, N, K, ldw, Kp, e16, tables);
    return (int)cudaGetLastError();
}

template <int RPL, bool HALF>
static int launch_p4_t(const P4Args& a, cudaStream_t st) {
    static unsigned configured = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 31;
    if (!(configured & (1u << dev))) {
        cudaError_t e = cudaFuncSetAttribute(lut_p4_kernel<RPL, HALF>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             p4::Geo<HALF>::SMEM_BYTES);
        if (e != cudaSuccess) return (int)e;
        configured |= 1u << dev;
    }
    const int64_t bm = (int64_t)p4::WARPS * 32 * RPL;
    const int64_t work = ((a.mm.M + bm - 1) / bm) * ((a.mm.N + p4::TN - 1) / p4::TN) * a.splits;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned g = (unsigned)std::min<int64_t>(work, sms > 0 ? sms : 148);
    lut_p4_kernel<RPL, HALF><<<g, p4::NT, p4::Geo<HALF>::SMEM_BYTES, st>>>(a);
    return (int)cudaGetLastError();
}

int g_p4w_pdl = 1;   // programmatic dependent launch of P4W (AXQ_P4W_PDL=0 disables)

template <bool HALF, int KSX, bool RES = false, int CWX = 28, bool E16 = false>
static int launch_p4w_t(const P4Args& a, cudaStream_t st) {
    using G = p4w::Geo<HALF, KSX, CWX, E16, RES>;
    using S = p4w::Shape<CWX>;
    static unsigned configured = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 31;
    if (!(configured & (1u << dev))) {
        cudaError_t e = cudaFuncSetAttribute(lut_p4w_kernel<HALF, KSX, RES, CWX, E16>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM_BYTES);
        if (e != cudaSuccess) return (int)e;
        configured |= 1u << dev;
    }
    const int64_t tiles = ((a.mm.M + S::BM - 1) / S::BM) * ((a.mm.N + p4::TN - 1) / p4::TN);
    const int64_t work = a.streamk ? tiles * (a.Kp / KSX) : tiles * a.splits;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned g = (unsigned)std::min<int64_t>(work, sms > 0 ? sms : 148);
    // launched with programmatic stream serialization: the kernel's griddepcontrol.wait (after
    // its prologue) orders it after the previous kernel on the stream
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(S::NT + G::NT_EXTRA);
    cfg.dynamicSmemBytes = G::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_p4w_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    P4Args args = a;
    cudaError_t e = cudaLaunchKernelEx(&cfg, lut_p4w_kernel<HALF, KSX, RES, CWX, E16>, args);
    return (int)(e != cudaSuccess ? e : cudaGetLastError());
}

int p4w_bm(int cw) { return cw * 32; }

int launch_p4w(const P4Args& a, cudaStream_t st) {
    const bool res = a.mm.ep.residual != nullptr && a.mm.C_out == nullptr;
    const int cw = a.cw ? a.cw : 28;
    constexpr int BAD = (int)cudaErrorInvalidValue;
    if (a.c4 && cw != 28) return BAD;           // the 4-byte-tap table lives in the 28-warp shapes
    if (a.e16) {                                // P4W16: half-range int16-E tables, 16-k stages
        if (!a.half || a.c4 || a.ks != 16) return BAD;
        if (res) return launch_p4w_t<true, 16, true, 16, true>(a, st);
        return cw == 16 ? launch_p4w_t<true, 16, false, 16, true>(a, st) : launch_p4w_t<true, 16, false, 28, true>(a, st);
    }
    if (!a.half) {                              // full-range tables, 16-k stages
        if (cw == 16 && !res) return launch_p4w_t<false, 16, false, 16>(a, st);
        return cw == 28 ? launch_p4w_t<false, 16>(a, st) : BAD;
    }
    if (a.ks == 16) return cw == 28 ? launch_p4w_t<true, 16>(a, st) : BAD;
    if (res) {
        // residual epilogue: fewer consumer warps leave more registers per thread, so the row's
        // residual loaded before the tile's MMA wait does not spill
        switch (cw) {
            case 16: return launch_p4w_t<true, 32, true, 16>(a, st);
            case 20: return launch_p4w_t<true, 32, true, 20>(a, st);
            case 24: return launch_p4w_t<true, 32, true, 24>(a, st);
            case 28: return launch_p4w_t<true, 32, true>(a, st);
            default: return BAD;
        }
    }
    switch (cw) {
        case 16: return launch_p4w_t<true, 32, false, 16>(a, st);
        case 20: return launch_p4w_t<true, 32, false, 20>(a, st);
        case 24: return launch_p4w_t<true, 32, false, 24>(a, st);
        case 28: return launch_p4w_t<true, 32>(a, st);
        default: return BAD;
    }
}

// Tensor-core packed-table tiles (P4W, bm rows): split K (exact, int32 atomics) only when they cannot fill the SMs.
void p4w_plan(int64_t M, int64_t N, int64_t Kp, int ks, int bm, int sms, bool can_split, int& splits, int& sps) {
    const int64_t nst = Kp / ks, nb = (N + p4::TN - 1) / p4::TN;
    const int64_t t = ((M + bm - 1) / bm) * nb;
    splits = 1;
    sps = (int)nst;
    if (t >= sms || !can_split) return;
    int64_t s = (sms + t - 1) / t;
    s = std::min<int64_t>(s, std::max<int64_t>(1, nst / 2));
    const int64_t per = (nst + s - 1) / s;
    sps = (int)per;
    splits = (int)((nst + per - 1) / per);
}

int launch_p4(const P4Args& a, cudaStream_t st) {
    if (a.half) return a.rpl == 1 ? launch_p4_t<1, true>(a, st) : launch_p4_t<2, true>(a, st);
    return a.rpl == 1 ? launch_p4_t<1, false>(a, st) : launch_p4_t<2, false>(a, st);
}

// Tile shape and K split.  Large problems: 1024- or 512-row tiles, whichever needs fewer
// persistent-CTA waves per row (512-row tiles cost ~8% more per lookup: the table fill is
// amortised over half the rows); no split (measured: its atomics and extra epilogue pass cost
// more than a partial wave).  Problems whose 512-row tiles cannot fill the SMs: split K
// (exact, int32 atomics) until they do, keeping >= 4 stages (64 k) per split.
void p4_plan(int64_t M, int64_t N, int64_t Kp, int sms, bool can_split, int& rpl, int& splits,
             int& sps) {
    const int64_t nst = Kp / p4::KS, nb = (N + p4::TN - 1) / p4::TN;
    const int64_t t2 = ((M + 1023) / 1024) * nb, t1 = ((M + 511) / 512) * nb;
    splits = 1;
    sps = (int)nst;
    if (t1 >= sms || !can_split) {
        const double c2 = (double)((t2 + sms - 1) / sms) * 1024.0;
        const double c1 = (double)((t1 + sms - 1) / sms) * 512.0 * 1.08;
        rpl = (c1 < c2) ? 1 : 2;
        return;
    }
    rpl = 1;
    int64_t s = (sms + t1 - 1) / t1;                   // enough parts to cover every SM
    s = std::min<int64_t>(s, std::max<int64_t>(1, nst / 4));
    const int64_t per = (nst + s - 1) / s;
    sps = (int)per;
    splits = (int)((nst + per - 1) / per);
}

}  // namespace axq
