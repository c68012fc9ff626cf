// kernels.cu -- host side of the kernel layer: table sizes and images, the
// TMA shape choice, and dispatch to the per-step launchers
// (kernels_private.cu / kernels_shared.cu / kernels_global.cu).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "kernels.hpp"
#include "kernels_impl.cuh"

namespace sfa {

size_t table_smem_bytes(Res mode, const DevTables& t) {
    switch (mode) {
        case Res::Private: return StepPrivate::supported(t) ? table_bytes<StepPrivate>(t) + t.aux_bytes : SIZE_MAX / 2;
        case Res::Shared: return StepShared::supported(t) ? table_bytes<StepShared>(t) + t.aux_bytes : SIZE_MAX / 2;
        case Res::Hot: return StepHot::supported(t) ? table_bytes<StepHot>(t) + t.aux_bytes : SIZE_MAX / 2;
        default: return table_bytes<StepGlobal>(t) + t.aux_bytes;
    }
}
// HOT residency: the number of renumbered rows that fit in smem next to what
// the launch kind needs (kind 0: the TMA scan with K=1, 32-byte stages and a
// 2-deep ring; 1: k_scan_direct; 2: the batch kernels), capped at nS.
void build_private_pairs(const uint16_t* Trange, uint32_t nS, uint32_t W, uint32_t R, uint32_t* pairs) {
    StepPrivate::build_pairs(Trange, nS, W, R, pairs);
}

uint32_t hot_rows_for(int kind, const DevTables& t, size_t smem_optin) {
    size_t other = t.aux_bytes + t.dwin_bytes + 32;
    if (kind == 0) {
        using Sh = TmaShape<1, 32>;
        other += Sh::kFixed + 2 * Sh::kStageBytes;
    } else if (kind == 1) {
        other += kDirectRed + 16;
    }
    if (other >= smem_optin) return 0;
    size_t rows = (smem_optin - other) / (2 * static_cast<size_t>(t.W));
    if (const char* e = getenv("SFA_HOT_ROWS")) rows = std::min<size_t>(rows, std::max(1l, atol(e)));  // tests: force cold rows
    return static_cast<uint32_t>(std::min<size_t>(rows, t.nS));
}

size_t direct_smem_bytes(Res mode, const DevTables& t) { return kDirectRed + 16 + table_smem_bytes(mode, t); }
uint32_t direct_threads_per_cta() { return kDirectWarps * 32; }

static int Sh_NB_host(int K) { return K == 1 ? Sh_NB<1>() : Sh_NB<2>(); }

// (K, ROWB) candidates in order of preference; the ring takes what is left.
// SFA_TMA_CONFIG="K,ROWB,ring[,pf[,promo]]" forces a shape (diagnostic sweeps
// and tests): ring 0 = as deep as fits, pf = L2 prefetch distance in 256-B
// lines (-1 = none), promo = L2 promotion bytes of the load map (0/64/128/256).
static bool tma_choose_once(Res mode, const DevTables& t, size_t smem_optin, TmaConfig* out, bool staged);

// Prefers staging the compact table in smem (one bulk copy) when it fits
// next to the table and a ring; else the table is built from global memory.
bool tma_choose(Res mode, const DevTables& t, size_t smem_optin, TmaConfig* out) {
    return tma_choose_once(mode, t, smem_optin, out, true) || tma_choose_once(mode, t, smem_optin, out, false);
}

static bool tma_choose_once(Res mode, const DevTables& t, size_t smem_optin, TmaConfig* out, bool staged) {
    size_t tb = table_smem_bytes(mode, t);
    size_t sb = 0;
    if (staged && mode == Res::Private) sb = StepPrivate::staged_bytes(t);
    if (staged && mode == Res::Shared) sb = StepShared::staged_bytes(t);
    if (staged && sb == 0) return false;
    tb += sb;
    if (tb > smem_optin) return false;
    static const int cand[][2] = {{1, 32}, {2, 32}, {1, 64}, {2, 16}, {1, 16}};
    const char* env = getenv("SFA_TMA_CONFIG");
    int fk = 0, fr = 0, fn = 0, fpf = -2, fpromo = -1;
    if (env) sscanf(env, "%d,%d,%d,%d,%d", &fk, &fr, &fn, &fpf, &fpromo);
    const bool forced = fk && (fk == 1 || fk == 2) && (fr == 16 || fr == 32 || fr == 64);
    for (int pass = 0; pass < 2; ++pass) {
        for (size_t ci = 0; ci < sizeof(cand) / sizeof(cand[0]); ++ci) {
            int K = cand[ci][0], rowb = cand[ci][1];
            if (forced) {
                if (ci) break;
                K = fk;
                rowb = fr;
            }
            const size_t R = static_cast<size_t>(K) * kNW * 32;
            const size_t stage = R * rowb;
            const size_t fixed = (((K * kNW + 2) * 32 + 15) & ~15u) + 16 + (2 * kMaxRing + 3) * 8 + 1024;
            if (tb + fixed + 2 * stage > smem_optin) continue;
            uint32_t ring = static_cast<uint32_t>(std::min<size_t>(kMaxRing, (smem_optin - tb - fixed) / stage));
            if (fn) ring = std::min<uint32_t>(ring, static_cast<uint32_t>(fn));
            if (pass == 0 && ring < 3 && !forced) continue;
            out->K = K;
            out->rowb = rowb;
            out->nring = ring;
            out->rows_per_cta = static_cast<uint32_t>(R);
            out->nb = Sh_NB_host(K);
            // No L2 prefetch by default: with ~1000 rows per SM, lines fetched
            // ahead of the TMA loads were evicted before use (1.6x DRAM reads).
            out->pf_lines = fpf >= -1 ? fpf : -1;
            out->promo = fpromo >= 0 ? fpromo : 0;
            out->staged = staged;
            return true;
        }
    }
    return false;
}

__global__ void k_combine_maps(const uint32_t* __restrict__ maps, uint32_t count, uint32_t nD,
                               const uint8_t* __restrict__ dfinal, sfa_result* result) {
    uint32_t q = 0;  // q0 (C3)
    for (uint32_t r = 0; r < count; ++r) q = maps[static_cast<size_t>(r) * nD + q];
    result->final_state = q;
    result->accept = dfinal[q];
}

cudaError_t launch_combine_maps(const uint32_t* maps, uint32_t count, uint32_t nD, const uint8_t* dfinal,
                                sfa_result* result, cudaStream_t stream) {
    k_combine_maps<<<1, 1, 0, stream>>>(maps, count, nD, dfinal, result);
    return cudaGetLastError();
}

cudaError_t launch_scan_tma(Res mode, bool vec, const ScanArgs& a, const TmaConfig& cfg, cudaStream_t stream) {
    switch (mode) {
        case Res::Private: return StepLaunch<StepPrivate>::scan_tma(vec, a, cfg, stream);
        case Res::Shared: return StepLaunch<StepShared>::scan_tma(vec, a, cfg, stream);
        case Res::Hot: return StepLaunch<StepHot>::scan_tma(vec, a, cfg, stream);
        default: return StepLaunch<StepGlobal>::scan_tma(vec, a, cfg, stream);
    }
}

cudaError_t launch_scan_direct(Res mode, bool vec, const DirectArgs& a, cudaStream_t stream) {
    switch (mode) {
        case Res::Private: return StepLaunch<StepPrivate>::scan_direct(vec, a, stream);
        case Res::Shared: return StepLaunch<StepShared>::scan_direct(vec, a, stream);
        case Res::Hot: return StepLaunch<StepHot>::scan_direct(vec, a, stream);
        default: return StepLaunch<StepGlobal>::scan_direct(vec, a, stream);
    }
}

cudaError_t launch_batch(Res mode, bool vec, const BatchArgs& a, int sm_count, cudaStream_t stream) {
    switch (mode) {
        case Res::Private: return StepLaunch<StepPrivate>::batch(vec, a, sm_count, stream);
        case Res::Shared: return StepLaunch<StepShared>::batch(vec, a, sm_count, stream);
        case Res::Hot: return StepLaunch<StepHot>::batch(vec, a, sm_count, stream);
        default: return StepLaunch<StepGlobal>::batch(vec, a, sm_count, stream);
    }
}

}  // namespace sfa
