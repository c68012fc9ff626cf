// device.cuh -- sm_100a device helpers and the per-byte step policies of the
// SFA chunk run (Alg. 5 lines 1-5).
//
// A "step policy" owns where the SFA transition table delta_s lives (A6,
// residency) and how one text byte advances a chunk's SFA state (A1 + A2).
// Every table sits at dynamic shared-memory offset 0 so its base is a
// compile-time immediate of the LDS.
//
//   StepPrivate  byte -> column by arithmetic on a byte window [lo, lo+W-2]
//                (every other byte shares column W-1); table in shared memory
//                as 32 bank-private u16 copies (lane L only touches bank L):
//                per byte  PRMT (byte) + VIADDMNMX (column) + IMAD (address)
//                + LDS.U16, one conflict-free wavefront per warp.
//   StepShared   one copy of the [nS x W] window table in shared memory, u32
//                entries premultiplied to row offsets: per byte PRMT +
//                VIADDMNMX + LEA + LDS (random banks: conflicts possible).
//   StepGlobal   the u16 window table read through L1/L2 (any |S|).
//
// Interface:  fill(t, tid, nthreads)  builds the smem table from t.Trange;
//             params(t)  per-thread constants;
//             init(lane) -> state of f_I;  step(state, byte) -> state;
//             id(state, lane) -> SFA id;   from_id(id, lane) -> state.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "plan.hpp"

namespace sfa {

// The kernels' dynamic shared memory.  Tables are indexed through this symbol
// (not through a cvta'd address) so the shared-window base folds into the LDS
// immediate instead of costing an add per byte.
extern __shared__ __align__(1024) uint8_t dsmem[];

__device__ __forceinline__ uint32_t ld_tbl_u16(uint32_t off) { return *reinterpret_cast<const uint16_t*>(dsmem + off); }
__device__ __forceinline__ uint32_t ld_tbl_u8(uint32_t off) { return dsmem[off]; }
__device__ __forceinline__ uint32_t ld_tbl_u32(uint32_t off) { return *reinterpret_cast<const uint32_t*>(dsmem + off); }

// ------------------------------------------------------------------------------------------
// PTX wrappers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
// 32 bytes (one L2 sector) per thread in one request: LDG.E.NA.ENL2.256 on sm_100a
struct U8x32 {
    uint4 lo, hi;
};
__device__ __forceinline__ U8x32 ldg_stream32(const void* p) {
    U8x32 v;
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v.lo.x), "=r"(v.lo.y), "=r"(v.lo.z), "=r"(v.lo.w), "=r"(v.hi.x), "=r"(v.hi.y), "=r"(v.hi.z),
                   "=r"(v.hi.w)
                 : "l"(p));
    return v;
}
// byte k of w, zero-extended: one PRMT
template <int K>
__device__ __forceinline__ uint32_t byte_of(uint32_t w) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "n"(0x4440 | K));
    return r;
}

// mbarrier (shared::cta)
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// TMA: 2-D tile global -> shared, completion counted on an mbarrier; `policy`
// is an L2 cache policy (createpolicy), evict-first for the streamed text so
// the table images stay L2-resident across launches.
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, uint32_t bar, int x, int y,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;"
        ::"r"(dst), "l"(tmap), "r"(bar), "r"(x), "r"(y), "l"(policy) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Programmatic dependent launch: let the next kernel of the stream start its
// prologue now / wait until the previous kernel of the stream has completed
// (and its memory is visible) before touching shared scratch.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// 1-D bulk copy global -> shared (bytes a multiple of 16), completion on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// 1-D bulk prefetch of [src, src + bytes) into L2 (16-B aligned, bytes a multiple of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const void* tmap, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(tmap), "r"(x), "r"(y) : "memory");
}
// A tensor map another kernel rewrote in global memory (tensormap.replace):
// order the generic-proxy writes before this kernel's TMA uses of it.
__device__ __forceinline__ void tmap_acquire(const void* tmap) {
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(tmap) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// named barrier among the compute warps only (the producer warp never joins)
__device__ __forceinline__ void bar_compute(uint32_t nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
constexpr unsigned kFull = 0xffffffffu;
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// column of a byte in the window table: min(byte - lo (mod 2^32), W - 1)
__device__ __forceinline__ uint32_t window_col(uint32_t byte, uint32_t neg_lo, uint32_t wmax) {
    return __viaddmin_u32(byte, neg_lo, wmax);
}

// Cooperative global -> smem copy of n16 16-byte words, 4 loads in flight per
// thread before their stores.
__device__ __forceinline__ void copy16(uint4* dst, const uint4* src, size_t n16, int tid, int nthreads) {
    size_t i = tid;
    for (; i + 3 * nthreads < n16; i += 4 * nthreads) {
        const uint4 a = __ldg(src + i), b = __ldg(src + i + nthreads), c = __ldg(src + i + 2 * nthreads),
                    d = __ldg(src + i + 3 * nthreads);
        dst[i] = a;
        dst[i + nthreads] = b;
        dst[i + 2 * nthreads] = c;
        dst[i + 3 * nthreads] = d;
    }
    for (; i < n16; i += nthreads) dst[i] = __ldg(src + i);
}

// ------------------------------------------------------------------------------------------
// Step policies
// ------------------------------------------------------------------------------------------
struct StepPrivate {
    static constexpr bool kFactor = false;
    static constexpr bool kStaged = true;  // TMA kernel: bulk-copy the pair words, expand in smem
    // R lane-group copies of the window table (plan.hpp dfa_enc; R = t.priv_R,
    // 32 = one bank-private copy per lane, 16 when 32 copies do not fit):
    // cell (s, j) of lane L's copy is the u16 at j*X + dfa_enc(s, L % R, R)
    // and holds dfa_enc(delta_s(s, j), L % R, R), the column-0 offset of the
    // next state, so the next address is one IMAD: col*X + state.
    uint32_t X, neg_lo, wmax, R;

    static __host__ __device__ uint32_t lines(const DevTables& t) {
        return t.priv_R ? (t.nS + 64u / t.priv_R - 1) / (64u / t.priv_R) : 0u;
    }
    static __host__ __device__ uint32_t col_bytes(const DevTables& t) { return t.priv_R ? dfa_X(t.nS, t.priv_R) : 0u; }
    static __host__ __device__ size_t smem_bytes(const DevTables& t) { return static_cast<size_t>(t.W) * col_bytes(t); }
    static __host__ __device__ bool supported(const DevTables& t) { return t.priv_R != 0 && t.pairs != nullptr; }
    static __host__ __device__ uint32_t npairs(const DevTables& t) { return t.priv_R ? t.W * lines(t) * (32u / t.priv_R) : 0u; }
    static __host__ __device__ uint32_t staged_bytes(const DevTables& t) { return (npairs(t) * 4 + 15) & ~15u; }
    static __host__ __device__ const void* staged_src(const DevTables& t) { return t.pairs; }

    // The copies from the lane-independent pair words (built on the host):
    // pairs[(j * lines + l) * (32/R) + k] = b(s0') | b(s1') << 16 with s0'/s1'
    // the next states of states l*spl + 2k, +1 in column j and b(x) =
    // dfa_enc(x, 0, R); word w of line l of column j (copy c = w % R, k = w / R)
    // = pairs[...] + 4c * 0x10001.  The skew gap after each column is zero.
    // `src_s`: shared-window address of an smem copy of t.pairs (the TMA
    // kernel stages it), else 0 (global).  Generic stores (see k_scan_tma:
    // they keep the smem base foldable into the hot loop's LDS).
    __device__ static void fill(const DevTables& t, int tid, int nthreads, uint32_t src_s) {
        const uint32_t R = t.priv_R, lgR = __ffs(R) - 1, lgk = 5 - lgR, nl = lines(t);
        const uint32_t L = tid & 31, w = tid >> 5, nw = nthreads >> 5, units = t.W * nl, add = (L & (R - 1)) * 0x40004u;
        uint32_t* tbl = reinterpret_cast<uint32_t*>(dsmem);
        // Staged pair words: the C++ load (not volatile asm) lets the loads of
        // several iterations be in flight at once.
        const uint32_t* sp = src_s ? reinterpret_cast<const uint32_t*>(dsmem + (src_s - smem_u32(dsmem))) : nullptr;
        // one warp per line unit u = j * nl + l: word L of line l of column j
        // sits at word 32u + jR + L (X/4 = 32 nl + R); the skew gap is never read
        if (R == 32) {  // no skew: line unit u is line u
#pragma unroll 4
            for (uint32_t u = w; u < units; u += nw) tbl[32 * u + L] = (sp ? sp[u] : __ldg(t.pairs + u)) + add;
            return;
        }
        uint32_t j = w / nl, l = w - j * nl;
        const uint32_t dj = nw / nl, dl = nw - dj * nl;
#pragma unroll 4
        for (uint32_t u = w; u < units; u += nw) {
            const uint32_t pi = (u << lgk) + (L >> lgR);
            const uint32_t a = sp ? sp[pi] : __ldg(t.pairs + pi);
            tbl[32 * u + j * R + L] = a + add;
            j += dj;
            l += dl;
            if (l >= nl) {
                l -= nl;
                ++j;
            }
        }
    }
    // host: the pair words of Trange [nS x W] for R copies
    static __host__ void build_pairs(const uint16_t* Trange, uint32_t nS, uint32_t W, uint32_t R, uint32_t* pairs) {
        const uint32_t spl = 64u / R, nl = (nS + spl - 1) / spl, kpl = 32u / R;
        for (uint32_t j = 0; j < W; ++j)
            for (uint32_t l = 0; l < nl; ++l)
                for (uint32_t k = 0; k < kpl; ++k) {
                    const uint32_t g0 = l * spl + 2 * k, g1 = g0 + 1;
                    const uint32_t b0 = g0 < nS ? dfa_enc(Trange[g0 * W + j], 0, R) : 0u;
                    const uint32_t b1 = g1 < nS ? dfa_enc(Trange[g1 * W + j], 0, R) : 0u;
                    pairs[(j * nl + l) * kpl + k] = b0 | (b1 << 16);
                }
    }
    __device__ void params(const DevTables& t) {
        X = col_bytes(t);
        neg_lo = 0u - t.lo;
        wmax = t.W - 1;
        R = t.priv_R;
    }
    __device__ __forceinline__ uint32_t init(uint32_t lane) const { return dfa_enc(0, lane % R, R); }
    __device__ __forceinline__ uint32_t step(uint32_t st, uint32_t byte) const {
        const uint32_t col = window_col(byte, neg_lo, wmax);
        return ld_tbl_u16(col * X + st);
    }
    __device__ __forceinline__ uint32_t id(uint32_t st, uint32_t lane) const { return dfa_dec(st, lane % R, R); }
    __device__ __forceinline__ uint32_t from_id(uint32_t s, uint32_t lane) const { return dfa_enc(s, lane % R, R); }
};


struct StepShared {
    static constexpr bool kFactor = false;
    static constexpr bool kStaged = true;  // TMA kernel: bulk-copy the compact table, expand in smem
    // bytes the TMA kernel stages (16-B padded: Trange is allocated padded) and their source
    static __host__ __device__ uint32_t staged_bytes(const DevTables& t) { return (t.nS * t.W * 2 + 15) & ~15u; }
    static __host__ __device__ const void* staged_src(const DevTables& t) { return t.Trange; }
    // one copy of the window table, u32 entries premultiplied to byte offsets:
    // state = 4*W*s (offset of row s), cell (s, j) holds 4*W*delta_s(s, j).
    uint32_t neg_lo, wmax, row;

    static __host__ __device__ size_t smem_bytes(const DevTables& t) { return static_cast<size_t>(t.nS) * t.W * 4; }
    static __host__ __device__ bool supported(const DevTables& t) { return static_cast<uint64_t>(t.nS) * t.W * 4 < (1u << 24); }
    __device__ static void fill(const DevTables& t, int tid, int nthreads, uint32_t src_s) {
        uint32_t* tbl = reinterpret_cast<uint32_t*>(dsmem);
        const uint32_t row = 4 * t.W, total = t.nS * t.W;
#pragma unroll 4
        for (uint32_t i = tid; i < total; i += nthreads)
            tbl[i] = (src_s ? lds_u16(src_s + 2 * i) : static_cast<uint32_t>(__ldg(t.Trange + i))) * row;
    }
    __device__ void params(const DevTables& t) {
        neg_lo = 0u - t.lo;
        wmax = t.W - 1;
        row = 4 * t.W;
    }
    __device__ __forceinline__ uint32_t init(uint32_t) const { return 0; }
    __device__ __forceinline__ uint32_t step(uint32_t st, uint32_t byte) const {
        const uint32_t col = window_col(byte, neg_lo, wmax);
        return ld_tbl_u32(st + 4 * col);
    }
    __device__ __forceinline__ uint32_t id(uint32_t st, uint32_t) const { return st / row; }
    __device__ __forceinline__ uint32_t from_id(uint32_t s, uint32_t) const { return s * row; }
};

struct StepGlobal {
    static constexpr bool kFactor = false;
    static constexpr bool kStaged = false;
    static __host__ __device__ uint32_t staged_bytes(const DevTables&) { return 0; }
    static __host__ __device__ const void* staged_src(const DevTables&) { return nullptr; }
    // the u16 window table through L1/L2: state = s*W (element offset of row s)
    uint32_t neg_lo, wmax, W;
    const uint16_t* T;

    static __host__ __device__ size_t smem_bytes(const DevTables&) { return 0; }
    static __host__ __device__ bool supported(const DevTables&) { return true; }
    __device__ static void fill(const DevTables&, int, int, uint32_t) {}
    __device__ void params(const DevTables& t) {
        neg_lo = 0u - t.lo;
        wmax = t.W - 1;
        W = t.W;
        T = t.Trange;
    }
    __device__ __forceinline__ uint32_t init(uint32_t) const { return 0; }
    __device__ __forceinline__ uint32_t step(uint32_t st, uint32_t byte) const {
        const uint32_t col = window_col(byte, neg_lo, wmax);
        return static_cast<uint32_t>(__ldg(T + st + col)) * W;
    }
    __device__ __forceinline__ uint32_t id(uint32_t st, uint32_t) const { return st / W; }
    __device__ __forceinline__ uint32_t from_id(uint32_t s, uint32_t) const { return s * W; }
};

struct StepHot {
    static constexpr bool kStaged = false;
    static __host__ __device__ uint32_t staged_bytes(const DevTables&) { return 0; }
    static __host__ __device__ const void* staged_src(const DevTables&) { return nullptr; }
    // HOT residency (A6): SFA states renumbered by expected visit frequency
    // (host ranking, DevTables::perm / iperm); rows [0, H) of the renumbered
    // u16 window table DevTables::Tdev sit in smem, the other rows are read
    // from global memory (L2).  state = device id.
    uint32_t neg_lo, wmax, W, H, init_dev, sbase;
    const uint16_t* Tdev;
    const uint16_t* perm;
    const uint16_t* iperm;

    static constexpr bool kFactor = true;  // kernels may switch warps to the factored step (StepDfa)
    // smem: [DFA table copies (t.dwin_bytes, StepDfa) | hot rows]
    static __host__ __device__ size_t hot_bytes(const DevTables& t) { return (static_cast<size_t>(t.hotH) * t.W * 2 + 15) & ~size_t(15); }
    static __host__ __device__ size_t smem_bytes(const DevTables& t) { return hot_bytes(t) + t.dwin_bytes; }
    static __host__ __device__ bool supported(const DevTables& t) { return t.Tdev != nullptr && t.hotH > 0; }
    __device__ static void fill(const DevTables& t, int tid, int nthreads, uint32_t) {  // hot rows = Tdev's prefix
        copy16(reinterpret_cast<uint4*>(dsmem + t.dwin_bytes), reinterpret_cast<const uint4*>(t.Tdev), hot_bytes(t) / 16,
               tid, nthreads);
        if (t.dwin_cpt) {  // bank-private rows expanded from the compact source (plan.hpp DevTables::dwin_cpt)
            uint32_t* tbl = reinterpret_cast<uint32_t*>(dsmem);
            const uint32_t L = tid & 31, w = tid >> 5, nw = nthreads >> 5, X4 = t.dwin_X >> 2, hl = t.dwin_hl;
            const uint32_t units = t.W * hl;
            // warp w: units [32 b, 32 b + 32) for b = w, w + nw, ...: one load per lane
            // (one L2 round trip per 32 units), each unit broadcast to the 32 lanes
            for (uint32_t u0 = 32 * w; u0 < units; u0 += 32 * nw) {
                const uint32_t mine = u0 + L < units ? __ldg(t.dwin_cpt + u0 + L) : 0u;
                const uint32_t n = min(32u, units - u0);
                uint32_t j = u0 / hl, k = u0 - j * hl;
                for (uint32_t i = 0; i < n; ++i) {
                    const uint32_t c = __shfl_sync(0xffffffffu, mine, i);
                    tbl[j * X4 + k * 32 + L] = cpt_expand(c, L);
                    if (++k == hl) {
                        k = 0;
                        ++j;
                    }
                }
            }
            if (t.dwin_tw) {  // the shared twin copy, as is: 4 loads in flight per thread
                const uint32_t tw = t.dwin_tw, hb4 = t.dwin_hotb >> 2, total = t.W * tw;
                for (uint32_t i0 = tid; i0 < total; i0 += 4 * nthreads) {
                    uint32_t v[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const uint32_t i = i0 + r * nthreads;
                        v[r] = i < total ? __ldg(t.dwin_twin + i) : 0u;
                    }
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const uint32_t i = i0 + r * nthreads;
                        if (i < total) {
                            const uint32_t j = i / tw;
                            tbl[j * X4 + hb4 + (i - j * tw)] = v[r];
                        }
                    }
                }
            }
        } else if (t.dwin_bytes) {  // the DFA window table's smem image (lane-group copies, built on the host)
            copy16(reinterpret_cast<uint4*>(dsmem), reinterpret_cast<const uint4*>(t.dwin), t.dwin_bytes / 16, tid, nthreads);
        }
    }
    __device__ void params(const DevTables& t) {
        neg_lo = 0u - t.lo;
        wmax = t.W - 1;
        W = t.W;
        H = t.hotH;
        Tdev = t.Tdev;
        perm = t.perm;
        iperm = t.iperm;
        init_dev = __ldg(t.perm);  // f_I (canonical id 0)
        sbase = smem_u32(dsmem) + t.dwin_bytes;
    }
    __device__ __forceinline__ uint32_t init(uint32_t) const { return init_dev; }
    // One predicated LDS (hot row) and one predicated LDG (cold row): no
    // branch, no reconvergence; only the lanes whose state is cold touch L2.
    __device__ __forceinline__ uint32_t step(uint32_t st, uint32_t byte) const {
        const uint32_t idx = st * W + window_col(byte, neg_lo, wmax);
        // "+r" from st: ptxas cannot tell that the two predicated loads cover
        // every case, so an output-only register would stay live (and spill)
        uint32_t r = st;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %0, %1;\n\t"
            "@p ld.shared.u16 %0, [%2];\n\t@!p ld.global.nc.u16 %0, [%3];\n\t}"
            : "+r"(r) : "r"(H), "r"(sbase + 2 * idx), "l"(Tdev + idx) : "memory");
        return r;
    }
    __device__ __forceinline__ uint32_t id(uint32_t st, uint32_t) const { return __ldg(iperm + st); }
    __device__ __forceinline__ uint32_t from_id(uint32_t s, uint32_t) const { return __ldg(perm + s); }
};

// The factored SFA step.  If every q that f does not send to an absorbing DFA
// state goes to one state g, then f . delta^c (Def. 3) keeps the
// absorbing part and sends those q to delta(g, c): the SFA state is (family,
// g) and one transition is one lookup in the DFA window table (smem, after the
// hot rows).  state = 2W * g.  Entered per warp once all its lanes' states are
// factorable (k_scan_tma, k_batch_scan); converted back to the canonical SFA
// id through DevTables::fact_tab at the end of the chunk.
struct StepDfa {
    // state = dfa_enc(g, lane % R): the column-0 offset of DFA state g in the
    // lane's copy; one step = PRMT + VIADDMNMX + IMAD + LDS, as StepPrivate.
    uint32_t neg_lo, wmax, X;
    __device__ void params(const DevTables& t) {
        neg_lo = 0u - t.lo;
        wmax = t.W - 1;
        X = t.dwin_X;
    }
    __device__ __forceinline__ uint32_t step(uint32_t st, uint32_t byte) const {
        return ld_tbl_u16(window_col(byte, neg_lo, wmax) * X + st);
    }
};

// The MIXED layout (plan.hpp mix_hot / mix_twin): the same one-IMAD step --
// a hot state's cells are lane L's bank-private copy, a twin's the shared
// copy -- plus fix(), run every 16 bytes off the byte loop: a lane whose
// state is the twin of a hot state moves back to its own copy (arithmetic
// only; the twin of a cold state stays).
struct StepDfaMix {
    uint32_t neg_lo, wmax, X, hotb, lane4;
    __device__ void params(const DevTables& t) {
        neg_lo = 0u - t.lo;
        wmax = t.W - 1;
        X = t.dwin_X;
        hotb = t.dwin_hotb;
        lane4 = 4u * lane_id();
    }
    __device__ __forceinline__ uint32_t step(uint32_t st, uint32_t byte) const {
        return ld_tbl_u16(window_col(byte, neg_lo, wmax) * X + st);
    }
    __device__ __forceinline__ uint32_t fix(uint32_t st) const { return mix_fix(st, hotb, lane4); }
};

// Steps that re-normalise their state between 16-byte pieces (StepDfaMix)
template <class T, class = void>
struct HasFix : std::false_type {};
template <class T>
struct HasFix<T, std::void_t<decltype(&T::fix)>> : std::true_type {};
template <class Step>
__device__ __forceinline__ uint32_t maybe_fix(const Step& S, uint32_t st) {
    if constexpr (HasFix<Step>::value) return S.fix(st);
    else return st;
}

// The same with the u8 layout (plan.hpp col8): 32 bank-private byte copies,
// state = the DFA id; one step = PRMT + VIADDMNMX + 2 ALU ops for the column
// term (off the chain) + IMAD + LDS.U8 (the chain), conflict-free where the
// u16 layout only fits 16 copies (2-way conflicts).
struct StepDfa8 {
    uint32_t neg_lo, wmax, RB, lanebase;
    __device__ void params(const DevTables& t) {
        neg_lo = 0u - t.lo;
        wmax = t.W - 1;
        RB = t.dwin_X;
        lanebase = smem_u32(dsmem) + (lane_id() << 2);  // the table sits at dsmem offset 0
    }
    __device__ __forceinline__ uint32_t step(uint32_t st, uint32_t byte) const {
        const uint32_t x = window_col(byte, neg_lo, wmax);
        // the column term (x >> 2) * 128 + (x & 3) = 31 (x & ~3) + x, plus
        // the lane and base bits -- all off the chain
        const uint32_t c = (x & ~3u) * 31u + x + lanebase;
        uint32_t a, v;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(a) : "r"(st), "r"(RB), "r"(c));  // the chain: one IMAD
        asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));                        // non-volatile: freely scheduled
        return v;
    }
};

// SFA id -> factored state and family; false if s is not factorable
__device__ __forceinline__ bool fact_from_id(const DevTables& t, uint32_t s, uint32_t& fam, uint32_t& st) {
    fam = __ldg(t.fact_fam + s);
    st = dw_enc(t, __ldg(t.fact_g + s), lane_id());
    return fam != 0xffffu;
}
__device__ __forceinline__ uint32_t fact_to_id(const DevTables& t, uint32_t fam, uint32_t st) {
    return __ldg(t.fact_tab + fam * t.nD + dw_dec(t, st, lane_id()));
}

// Factored chunk values (DevTables::fam_bits / fam_img): bit 30 tags (F, g),
// F in bits 16..29, g (a DFA id) in bits 0..15; untagged values are SFA ids.
constexpr uint32_t kFact = 0x40000000u;
__device__ __forceinline__ bool fact_values(const DevTables& t) { return t.fam_bits || t.fam_img; }
__device__ __forceinline__ uint32_t fact_pack(uint32_t fam, uint32_t g) { return kFact | (fam << 16) | g; }
// f_(F, g)(q): the absorbing image of a marked q, else g
__device__ __forceinline__ uint32_t fam_apply(const DevTables& t, uint32_t F, uint32_t g, uint32_t q) {
    if (t.aux_fam) return (lds_u32(smem_u32(dsmem) + t.aux_off + 4u * (F * t.fam_w + (q >> 5))) >> (q & 31)) & 1u ? t.fam_a0 : g;
    if (t.fam_bits) return (__ldg(t.fam_bits + F * t.fam_w + (q >> 5)) >> (q & 31)) & 1u ? t.fam_a0 : g;
    const uint32_t m = __ldg(t.fam_img + F * t.nD + q);
    return m != 0xffffu ? m : g;
}
// Diagnostic builds with -DSFA_COUNTERS: count an event (sfa_diag_counters):
// 0 combine_fact, 1 combine_ids, 2 combine_slow, 3 replay (per warp; the
// atomics perturb the timings, so the stamp build leaves them out)
#if defined(SFA_STAMPS) && defined(SFA_COUNTERS)
#define SFA_CTR(t, i)                                 \
    do {                                              \
        if ((t).diag && (threadIdx.x & 31) == 0) atomicAdd((t).diag + (i), 1ull); \
    } while (0)
#else
#define SFA_CTR(t, i) \
    do {              \
    } while (0)
#endif

// an SFA id as a factored value when it is factorable
__device__ __forceinline__ uint32_t fact_of_id(const DevTables& t, uint32_t s) {
    const uint32_t fa = __ldg(t.fact_fam + s);
    return fa != 0xffffu ? fact_pack(fa, __ldg(t.fact_g + s)) : s;
}
// a factored value's canonical SFA id
__device__ __forceinline__ uint32_t fact_value_id(const DevTables& t, uint32_t v) {
    return __ldg(t.fact_tab + ((v >> 16) & 0x3fffu) * t.nD + (v & 0xffffu));
}

// 4 text bytes of one word, in text order (little-endian)
template <class Step>
__device__ __forceinline__ uint32_t step4(const Step& S, uint32_t st, uint32_t w) {
    st = S.step(st, byte_of<0>(w));
    st = S.step(st, byte_of<1>(w));
    st = S.step(st, byte_of<2>(w));
    st = S.step(st, byte_of<3>(w));
    return st;
}
template <class Step>
__device__ __forceinline__ uint32_t step16(const Step& S, uint32_t st, const uint4& v) {
    st = step4(S, st, v.x);
    st = step4(S, st, v.y);
    st = step4(S, st, v.z);
    return maybe_fix(S, step4(S, st, v.w));
}

// Bytes [lo, hi) (offsets within the 16-byte block v) through S.
template <class Step>
__device__ __forceinline__ uint32_t step_part16(const Step& S, uint32_t st, const uint4& v, uint32_t lo, uint32_t hi) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (uint32_t j = 0; j < 16; ++j)
        if (j >= lo && j < hi) st = S.step(st, (w[j >> 2] >> (8 * (j & 3))) & 0xffu);
    return st;
}

// A byte range [a, b) of `t`, from state st, with 16-byte loads only: the
// ragged ends come from the aligned 16-byte blocks that hold them (a block
// holding a byte of the text lies in the same page as that byte), so a short
// unaligned piece costs one or two parallel loads, not one dependent load per
// byte (head pieces, the tail).
template <class Step>
__device__ uint32_t run_range(const Step& S, uint32_t st, const uint8_t* __restrict__ t, uint64_t a, uint64_t b) {
    if (a >= b) return st;
    const uintptr_t pa = reinterpret_cast<uintptr_t>(t + a), pb = reinterpret_cast<uintptr_t>(t + b);
    uintptr_t blk = pa & ~uintptr_t(15);
    const uintptr_t last = (pb - 1) & ~uintptr_t(15);
    if (blk == last)  // one block
        return step_part16(S, st, ldg_stream(reinterpret_cast<const void*>(blk)), static_cast<uint32_t>(pa - blk),
                           static_cast<uint32_t>(pb - blk));
    const uint4 vl = ldg_stream(reinterpret_cast<const void*>(last));  // in flight while the rest runs
    if (pa != blk) {
        st = step_part16(S, st, ldg_stream(reinterpret_cast<const void*>(blk)), static_cast<uint32_t>(pa - blk), 16u);
        blk += 16;
    }
    if (blk < last) {
        uint4 v = ldg_stream(reinterpret_cast<const void*>(blk));
        blk += 16;
        while (blk < last) {
            const uint4 nx = ldg_stream(reinterpret_cast<const void*>(blk));  // next 16 bytes in flight while v is consumed
            blk += 16;
            st = step16(S, st, v);
            v = nx;
        }
        st = step16(S, st, v);
    }
    return step_part16(S, st, vl, 0u, static_cast<uint32_t>(pb - last));
}

// ------------------------------------------------------------------------------------------
// Composition (Alg. 5 line 6).  '.' is reverse composition: (f.g)(q) = g(f(q)).
// ------------------------------------------------------------------------------------------
// Vector form (|D| <= 32): lane q holds g(q).  maps32[s*32 + q] = f_s(q)
// (identity-padded for q >= |D|).
__device__ __forceinline__ uint32_t vec_compose(uint32_t g1, uint32_t g2) {
    return __shfl_sync(kFull, g2, g1);  // (g1 . g2)(q) = g2(g1(q))
}
// fold the 32 lanes' SFA ids in lane order into a vector
__device__ __forceinline__ uint32_t vec_fold_ids(const uint8_t* __restrict__ maps32, uint32_t s_lane) {
    uint32_t g = lane_id();
#pragma unroll 8
    for (int l = 0; l < 32; ++l) {
        uint32_t s = __shfl_sync(kFull, s_lane, l);
        g = maps32[s * 32 + g];  // smem copy when small (DevTables::aux), else global
    }
    return g;
}

// Replay form (any |D|): s_a . s_b = delta_s^(s_a, w) for any word w with
// f_I -w-> s_b (Lemma 1), w = the representative word of s_b.
template <class Step>
__device__ __forceinline__ uint32_t replay(const Step& S, const DevTables& t, uint32_t sa, uint32_t sb, uint32_t lane) {
    SFA_CTR(t, 3);
    uint32_t st = S.from_id(sa, lane);
    if (t.rep16) {  // depth <= 15: the word in one 16-byte slot, its length in byte 15
        const uint4 w = __ldg(t.rep16 + sb);
        const uint32_t len = w.w >> 24;
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (uint32_t k = 0; k < 15; ++k)
            if (k < len) st = S.step(st, (ws[k >> 2] >> (8 * (k & 3))) & 0xffu);
        return S.id(st, lane);
    }
    const uint32_t e = t.rep_off[sb + 1];
    for (uint32_t k = t.rep_off[sb]; k < e; ++k) st = S.step(st, t.rep[k]);
    return S.id(st, lane);
}
// tree-fold the 32 lanes' ids in lane order; result valid in lane 0
template <class Step>
__device__ uint32_t replay_fold(const Step& S, const DevTables& t, uint32_t s) {
    const uint32_t lane = lane_id();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t o = __shfl_down_sync(kFull, s, d);
        if ((lane & (2 * d - 1)) == 0) s = replay(S, t, s, o, lane);
    }
    return s;
}

}  // namespace sfa
