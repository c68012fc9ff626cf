// device.cuh -- sm_100a device helpers and the per-byte step policies of the
// SFA chunk run (Alg. 5 lines 1-5).
//
// A "step policy" owns where the SFA transition table delta_s lives (A6,
// residency) and how one text byte advances a chunk's SFA state (A1 + A2):
//
//   StepPrivate  byte -> column by arithmetic on a byte window [lo, lo+W-2]
//                (all other bytes share column W-1), table in shared memory as
//                32 bank-private copies with premultiplied lane addresses:
//                per byte  PRMT/SHF + VIADDMNMX + LEA + LDS.32, 1 conflict-free
//                shared wavefront.
//   StepShared   class map (u16, 2*class) + one u16 table in shared memory:
//                per byte  LDS.U16 (class) + IMAD + LDS.U16 (next state).
//   StepGlobal   class map in shared memory, u16 table read through L1/L2.
//
// Every policy exposes the same interface so the kernels are generic:
//   init(lane) -> state of f_I;  step(state, byte) -> state;
//   id(state, lane) -> SFA id;   from_id(id, lane) -> state.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "plan.hpp"

namespace sfa {

// ------------------------------------------------------------------------------------------
// PTX wrappers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    uint16_t v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
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
__device__ __forceinline__ uint32_t ldg_u16(const uint16_t* p) { return __ldg(p); }

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
// TMA: 2-D tile global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, uint32_t bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(dst), "l"(tmap), "r"(bar), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const void* tmap, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(tmap), "r"(x), "r"(y) : "memory");
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

// ------------------------------------------------------------------------------------------
// Step policies
// ------------------------------------------------------------------------------------------
struct StepPrivate {
    // table: nS * W * 32 words; word ((s*W + j)*32 + L) of lane L's copy holds
    // the shared-memory byte address of row delta_s(s, column j) in lane L's
    // copy, so one LEA + one LDS advances the state.
    uint32_t base;     // shared address of the table
    uint32_t neg_lo;   // -lo (mod 2^32)
    uint32_t wmax;     // W - 1 (the "every other byte" column)
    uint32_t row_words;  // W * 32

    static __host__ __device__ size_t smem_bytes(const DevTables& t) {
        return static_cast<size_t>(t.nS) * t.W * 32 * 4;
    }
    __device__ void setup(const DevTables& t, uint8_t* smem, int tid, int nthreads) {
        base = smem_u32(smem);
        neg_lo = 0u - t.lo;
        wmax = t.W - 1;
        row_words = t.W * 32;
        uint32_t* tbl = reinterpret_cast<uint32_t*>(smem);
        const uint32_t total = t.nS * row_words;
        for (uint32_t i = tid; i < total; i += nthreads) {
            uint32_t cell = i >> 5, L = i & 31;  // cell = s*W + j
            uint32_t nxt = t.Trange[cell];
            tbl[i] = base + (nxt * row_words + L) * 4u;
        }
    }
    __device__ __forceinline__ uint32_t init(uint32_t lane) const { return base + lane * 4u; }
    __device__ __forceinline__ uint32_t step(uint32_t st, uint32_t byte) const {
        uint32_t col = __viaddmin_u32(byte, neg_lo, wmax);  // min(byte - lo, W-1), wrapping below lo
        return lds_u32(st + (col << 7));
    }
    __device__ __forceinline__ uint32_t id(uint32_t st, uint32_t) const { return ((st - base) >> 2) / row_words; }
    __device__ __forceinline__ uint32_t from_id(uint32_t s, uint32_t lane) const {
        return base + (s * row_words + lane) * 4u;
    }
};

struct StepShared {
    // cls: 256 x u16 holding 2*class; T: nS*C u16 SFA ids.
    uint32_t cls_base, t_base, two_c;

    static __host__ __device__ size_t smem_bytes(const DevTables& t) {
        return 512 + ((static_cast<size_t>(t.nS) * t.C * 2 + 15) & ~size_t(15));
    }
    __device__ void setup(const DevTables& t, uint8_t* smem, int tid, int nthreads) {
        cls_base = smem_u32(smem);
        t_base = cls_base + 512;
        two_c = 2 * t.C;
        uint16_t* c16 = reinterpret_cast<uint16_t*>(smem);
        for (int b = tid; b < 256; b += nthreads) c16[b] = static_cast<uint16_t>(2 * t.cls[b]);
        uint16_t* T16 = reinterpret_cast<uint16_t*>(smem + 512);
        const uint32_t total = t.nS * t.C;
        for (uint32_t i = tid; i < total; i += nthreads) T16[i] = t.T[i];
    }
    __device__ __forceinline__ uint32_t init(uint32_t) const { return 0; }
    __device__ __forceinline__ uint32_t step(uint32_t s, uint32_t byte) const {
        uint32_t c2 = lds_u16(cls_base + 2 * byte);
        return lds_u16(t_base + s * two_c + c2);
    }
    __device__ __forceinline__ uint32_t id(uint32_t s, uint32_t) const { return s; }
    __device__ __forceinline__ uint32_t from_id(uint32_t s, uint32_t) const { return s; }
};

struct StepGlobal {
    uint32_t cls_base, C;
    const uint16_t* T;

    static __host__ __device__ size_t smem_bytes(const DevTables&) { return 512; }
    __device__ void setup(const DevTables& t, uint8_t* smem, int tid, int nthreads) {
        cls_base = smem_u32(smem);
        C = t.C;
        T = t.T;
        uint16_t* c16 = reinterpret_cast<uint16_t*>(smem);
        for (int b = tid; b < 256; b += nthreads) c16[b] = static_cast<uint16_t>(t.cls[b]);
    }
    __device__ __forceinline__ uint32_t init(uint32_t) const { return 0; }
    __device__ __forceinline__ uint32_t step(uint32_t s, uint32_t byte) const {
        uint32_t c = lds_u16(cls_base + 2 * byte);
        return ldg_u16(T + s * C + c);
    }
    __device__ __forceinline__ uint32_t id(uint32_t s, uint32_t) const { return s; }
    __device__ __forceinline__ uint32_t from_id(uint32_t s, uint32_t) const { return s; }
};

// 16 text bytes in text order (little-endian words)
template <class Step>
__device__ __forceinline__ uint32_t step16(const Step& S, uint32_t st, const uint4& v) {
#pragma unroll
    for (int k = 0; k < 4; ++k) st = S.step(st, (v.x >> (8 * k)) & 0xffu);
#pragma unroll
    for (int k = 0; k < 4; ++k) st = S.step(st, (v.y >> (8 * k)) & 0xffu);
#pragma unroll
    for (int k = 0; k < 4; ++k) st = S.step(st, (v.z >> (8 * k)) & 0xffu);
#pragma unroll
    for (int k = 0; k < 4; ++k) st = S.step(st, (v.w >> (8 * k)) & 0xffu);
    return st;
}

// A byte range [a, b) of `t`, from state st, with 16-byte loads where aligned.
template <class Step>
__device__ uint32_t run_range(const Step& S, uint32_t st, const uint8_t* __restrict__ t, uint64_t a, uint64_t b) {
    while (a < b && (reinterpret_cast<uintptr_t>(t + a) & 15)) st = S.step(st, __ldg(t + a++));
    if (a + 16 <= b) {
        uint4 v = ldg_stream(t + a);
        a += 16;
        while (a + 16 <= b) {
            uint4 nx = ldg_stream(t + a);  // next 16 bytes in flight while v is consumed
            a += 16;
            st = step16(S, st, v);
            v = nx;
        }
        st = step16(S, st, v);
    }
    while (a < b) st = S.step(st, __ldg(t + a++));
    return st;
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
        g = __ldg(maps32 + s * 32 + g);
    }
    return g;
}

// Replay form (any |D|): s_a . s_b = delta_s^(s_a, w) for any word w with
// f_I -w-> s_b (Lemma 1), w = the representative word of s_b.
template <class Step>
__device__ __forceinline__ uint32_t replay(const Step& S, const DevTables& t, uint32_t sa, uint32_t sb, uint32_t lane) {
    uint32_t st = S.from_id(sa, lane);
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
