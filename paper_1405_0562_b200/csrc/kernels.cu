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
void build_private_pairs(const uint16_t* Trange, uint32_t nS, uint32_t W, uint32_t R, uint32_t* pairs) {
    StepPrivate::build_pairs(Trange, nS, W, R, pairs);
}

// HOT residency: the number of renumbered rows that fit in smem next to what
// the launch kind needs (kind 0: the TMA scan with K=1, 32-byte stages and a
// 2-deep ring; 1: k_scan_direct), capped at nS and at `cap` (> 0: a tuning
// knob; tests force cold rows with it).
uint32_t hot_rows_for(int kind, const DevTables& t, size_t smem_optin, uint32_t cap) {
    size_t other = t.aux_bytes + t.dwin_bytes + 32;
    if (kind == 0) {
        using Sh = TmaShape<1, 32>;
        // FACTORED (a DFA window in smem): the SFA rows only serve the first
        // stages of a row, the ring of 32-byte stages comes first (3 deep)
        other += Sh::kFixed + (t.dwin_bytes ? 3 : 2) * Sh::kStageBytes;
    } else if (kind == 1) {
        other += kDirectRed + 16;
    }
    if (other >= smem_optin) return 0;
    size_t rows = (smem_optin - other) / (2 * static_cast<size_t>(t.W));
    if (cap) rows = std::min<size_t>(rows, cap);
    return static_cast<uint32_t>(std::min<size_t>(rows, t.nS));
}

size_t factored_mixed_budget(size_t smem_optin, uint32_t W) {
    using Sh = TmaShape<1, 32>;
    const size_t keep = Sh::kFixed + 3 * Sh::kStageBytes + 64u * 2u * W + 64;
    return smem_optin > keep ? smem_optin - keep : 0;
}

size_t direct_smem_bytes(Res mode, const DevTables& t) { return kDirectRed + 16 + table_smem_bytes(mode, t); }
uint32_t direct_threads_per_cta() { return kDirectWarps * 32; }

static int Sh_NB_host(int K) { return K == 1 ? Sh_NB<1>() : Sh_NB<2>(); }

// (K, ROWB) candidates in order of preference; the ring takes what is left.
// Tuning (sfa_set_tuning) may force K, ROWB, the ring depth and the L2
// promotion of the loads (shape only: results never change).
static bool tma_choose_once(Res mode, const DevTables& t, size_t smem_optin, const Tuning& tu, TmaConfig* out,
                            bool staged);

// Prefers staging the compact table in smem (one bulk copy) when it fits
// next to the table and a ring; else the table is built from global memory.
bool tma_choose(Res mode, const DevTables& t, size_t smem_optin, const Tuning& tu, TmaConfig* out) {
    return tma_choose_once(mode, t, smem_optin, tu, out, true) || tma_choose_once(mode, t, smem_optin, tu, out, false);
}

static bool tma_choose_once(Res mode, const DevTables& t, size_t smem_optin, const Tuning& tu, TmaConfig* out,
                            bool staged) {
    size_t tb = table_smem_bytes(mode, t);
    size_t sb = 0;
    if (staged && mode == Res::Private) sb = StepPrivate::staged_bytes(t);
    if (staged && mode == Res::Shared) sb = StepShared::staged_bytes(t);
    if (staged && sb == 0) return false;
    tb += sb;
    if (tb > smem_optin) return false;
    static const int cand[][2] = {{1, 32}, {2, 32}, {1, 64}, {2, 16}, {1, 16}};
    const bool forced = (tu.tma_k == 1 || tu.tma_k == 2) && (tu.tma_rowb == 16 || tu.tma_rowb == 32 || tu.tma_rowb == 64);
    for (int pass = 0; pass < 2; ++pass) {
        for (size_t ci = 0; ci < sizeof(cand) / sizeof(cand[0]); ++ci) {
            int K = cand[ci][0], rowb = cand[ci][1];
            if (forced) {
                if (ci) break;
                K = tu.tma_k;
                rowb = tu.tma_rowb;
            }
            const size_t R = static_cast<size_t>(K) * kNW * 32;
            const size_t stage = R * rowb;
            const size_t fixed = (((K * kNW + 2) * 32 + 15) & ~15u) + 16 + (2 * kMaxRing + 3) * 8 + 1024;
            if (tb + fixed + 2 * stage > smem_optin) continue;
            uint32_t ring = static_cast<uint32_t>(std::min<size_t>(kMaxRing, (smem_optin - tb - fixed) / stage));
            if (tu.tma_ring > 0) ring = std::min<uint32_t>(ring, static_cast<uint32_t>(std::max(2, tu.tma_ring)));
            if (pass == 0 && ring < 3 && !forced) continue;
            out->K = K;
            out->rowb = rowb;
            out->nring = ring;
            out->rows_per_cta = static_cast<uint32_t>(R);
            out->nb = Sh_NB_host(K);
            out->promo = tu.tma_promo >= 0 ? tu.tma_promo : 0;
            out->staged = staged;
            return true;
        }
    }
    return false;
}

// ------------------------------------------------------------------------------------------
// k_batch_plan -- the batch's launch plan on the device (SURVEY s8(b):
// sfa_match_batch is asynchronous, so the host never reads the offsets).
// Every thread checks its texts' offsets (a decreasing pair -> *err = epoch:
// the scan then reports every result as invalid), answers empty texts
// ((q0 = 0, [eps in L])) and tracks the text lengths; the last block to finish
// plans the scan of [off[0], off[count]) as one range -- rows of len / mm
// bytes when every text has the same length (make_plan_uniform: no boundary
// inside a row), else make_plan -- and rewrites the tensor maps in global memory
// from the host-encoded template (tensormap.replace: base, dims, row stride,
// box height; three maps for the box heights bh, rc_hi % bh, rc_lo % bh), then
// publishes them to the TMA proxy.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void tmap_store(void* dst, const CUtensorMap& src) {
    const uint4* s = reinterpret_cast<const uint4*>(&src);
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = s[i];
}
__device__ __forceinline__ void tmap_retarget(void* m, uint64_t addr, uint32_t L, uint32_t rows, uint32_t bh) {
    asm volatile("tensormap.replace.tile.global_address.global.b1024.b64 [%0], %1;" ::"l"(m), "l"(addr) : "memory");
    asm volatile("tensormap.replace.tile.global_dim.global.b1024.b32 [%0], 0, %1;" ::"l"(m), "r"(L) : "memory");
    asm volatile("tensormap.replace.tile.global_dim.global.b1024.b32 [%0], 1, %1;" ::"l"(m), "r"(rows) : "memory");
    asm volatile("tensormap.replace.tile.global_stride.global.b1024.b64 [%0], 0, %1;" ::"l"(m), "l"(static_cast<uint64_t>(L))
                 : "memory");
    asm volatile("tensormap.replace.tile.box_dim.global.b1024.b32 [%0], 1, %1;" ::"l"(m), "r"(bh) : "memory");
}

static __global__ void __launch_bounds__(1024) k_batch_plan(const __grid_constant__ TmaMaps tmpl, const BatchPlanArgs a) {
    pdl_launch_dependents();
    __shared__ unsigned long long s_min, s_max;
    __shared__ uint32_t s_bad, s_last;
    if (threadIdx.x == 0) {
        s_min = ~0ull;
        s_max = 0;
        s_bad = 0;
    }
    __syncthreads();
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t mn = ~0ull, mx = 0;
    uint32_t bad = 0;
    for (uint64_t i = tid; i < a.count; i += nth) {
        const uint64_t s = __ldg(a.off + i), e = __ldg(a.off + i + 1);
        if (e < s) {
            bad = 1;
            continue;
        }
        if (e == s) a.results[i] = sfa_result{0u, a.eps_accept};
        mn = min(mn, e - s);
        mx = max(mx, e - s);
    }
    atomicMin(&s_min, mn);
    atomicMax(&s_max, mx);
    if (bad) atomicOr(&s_bad, 1u);
    __syncthreads();
    // the last block to finish reduces the blocks' (min, max, bad) and plans
    if (threadIdx.x == 0) {
        a.slots[blockIdx.x] = make_uint4(static_cast<uint32_t>(s_min), static_cast<uint32_t>(s_min >> 32),
                                         static_cast<uint32_t>(s_max), static_cast<uint32_t>(s_max >> 32) | (s_bad << 31));
        __threadfence();
        s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    uint64_t gmin = ~0ull, gmax = 0;
    uint32_t gbad = 0;
    for (uint32_t b = 0; b < gridDim.x; ++b) {
        const uint4 v = __ldcg(a.slots + b);
        gmin = min(gmin, static_cast<uint64_t>(v.x) | (static_cast<uint64_t>(v.y) << 32));
        gmax = max(gmax, static_cast<uint64_t>(v.z) | (static_cast<uint64_t>(v.w & 0x7fffffffu) << 32));
        gbad |= v.w >> 31;
    }
    *a.ticket = 0;  // self-resetting
    const uint64_t s = __ldg(a.off), e = __ldg(a.off + a.count);
    if (e < s) gbad = 1;
    TmaPlan p;
    const uint64_t addr = reinterpret_cast<uint64_t>(a.texts + s);
    // equal texts: rows of len / mm bytes (no boundary inside a row); else the general cut
    if (gbad || gmin != gmax || !make_plan_uniform(addr, gmin, a.count, a.G, a.R, a.NB, a.rowb, &p))
        make_plan(addr, !gbad ? e - s : 0, a.G, a.R, a.NB, a.rowb, a.row_align, &p);
    *a.dplan = p;
    uint64_t base = reinterpret_cast<uint64_t>(a.texts + s + p.head);
    if (p.nchunks == 0) base &= ~uint64_t(255);
    const uint32_t rows = p.nchunks ? p.nchunks : 1u;
    uint8_t* m = static_cast<uint8_t*>(a.gmaps);
    uint32_t heights[3];
    detail::box_heights(p, heights);
    for (int k = 0; k < 3; ++k) {
        tmap_store(m + k * sizeof(CUtensorMap), tmpl.load);
        tmap_retarget(m + k * sizeof(CUtensorMap), base, static_cast<uint32_t>(p.L), rows, heights[k]);
    }
    asm volatile("fence.proxy.tensormap::generic.release.gpu;" ::: "memory");
    if (gbad) *a.err = a.epoch;
}

cudaError_t launch_batch_plan(const BatchPlanArgs& a, const TmaConfig& cfg, int sm_count, cudaStream_t stream) {
    // the template: any valid 16-B aligned base; everything but the element
    // type, swizzle, box width and L2 promotion is replaced on the device
    struct Key {
        int dev, rowb, promo;
        void* base;
    };
    static thread_local Key last{-1, 0, -9, nullptr};
    static thread_local TmaMaps tmpl;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(last.dev == dev && last.rowb == cfg.rowb && last.promo == cfg.promo && last.base == a.gmaps)) {
        cudaError_t e = detail::encode_map(&tmpl.load, a.gmaps, 256, 1, cfg.rowb, 8, cfg.promo);
        if (e != cudaSuccess) return e;
        last = Key{dev, cfg.rowb, cfg.promo, a.gmaps};
    }
    const uint64_t want = (a.count + 1023) / 1024;
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, static_cast<uint64_t>(sm_count))));
    k_batch_plan<<<grid, 1024, 0, stream>>>(tmpl, a);
    return cudaGetLastError();
}

static __global__ void k_fill_result(sfa_result* r, uint32_t q, uint32_t acc, uint32_t* map, uint32_t nD) {
    if (r && threadIdx.x == 0 && blockIdx.x == 0) *r = sfa_result{q, acc};
    if (map)
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nD; i += gridDim.x * blockDim.x) map[i] = i;
}

static __global__ void k_fill_results(sfa_result* r, uint64_t count, uint32_t q, uint32_t acc) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        r[i] = sfa_result{q, acc};
}

cudaError_t launch_fill_results(sfa_result* r, uint64_t count, uint32_t q, uint32_t acc, cudaStream_t stream) {
    const uint64_t want = (count + 255) / 256;
    k_fill_results<<<static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, 1024))), 256, 0, stream>>>(r, count, q, acc);
    return cudaGetLastError();
}

cudaError_t launch_fill_result(sfa_result* r, uint32_t q, uint32_t acc, uint32_t* map, uint32_t nD, cudaStream_t stream) {
    k_fill_result<<<map ? std::max<uint32_t>(1, std::min<uint32_t>(64, (nD + 255) / 256)) : 1, 256, 0, stream>>>(r, q, acc, map, nD);
    return cudaGetLastError();
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

cudaError_t launch_scan_seg(Res mode, const ScanArgs& a, const TmaConfig& cfg, unsigned grid, cudaStream_t stream) {
    switch (mode) {
        case Res::Private: return StepLaunch<StepPrivate>::scan_seg(a, cfg, grid, stream);
        case Res::Shared: return StepLaunch<StepShared>::scan_seg(a, cfg, grid, stream);
        case Res::Hot: return StepLaunch<StepHot>::scan_seg(a, cfg, grid, stream);
        default: return StepLaunch<StepGlobal>::scan_seg(a, cfg, grid, stream);
    }
}

}  // namespace sfa
