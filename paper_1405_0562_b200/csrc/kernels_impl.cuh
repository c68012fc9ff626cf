// kernels_impl.cuh -- sm_100a kernels of the SFA hot path (Alg. 5)
// and their host launch templates.  Included by one kernels_<step>.cu per step
// policy (parallel build); kernels.cu holds the host-side planning/dispatch.
//
//   k_scan_tma     a long byte range.  One CTA per SM: kNW compute warps + 1
//                  TMA producer warp.  The 256-aligned body of the range is
//                  viewed as a 2-D tensor [nchunks rows x L bytes]; every stage
//                  the producer loads a ROWB-byte column slice of all of the
//                  CTA's rows (TMA 2-D boxes, mbarrier ring), each compute
//                  thread owns K rows (= K chunks of Alg. 5 lines 1-5,
//                  interleaved for ILP), so every byte of HBM is read once and
//                  the smem reads of the staged text are conflict-free.
//                  Two modes:
//                    one text (SEG = false): chunk states are composed warp ->
//                      block -> grid (line 6); the last CTA to finish folds the
//                      per-CTA partials (plus the head piece and the ragged
//                      tail) and finalises (line 7).
//                    a batch (SEG = true, A5): the texts lie back to back in
//                      the range; a row may hold several text boundaries.  A
//                      chunk's value is then a segmented element (the piece
//                      before its first boundary, the piece after its last),
//                      texts that start and end inside a row are finished in
//                      place, and the same warp -> block -> grid tree composes
//                      the elements with a segmented operator that finishes a
//                      text where its first and last pieces meet.
//   k_scan_direct  short texts and the forced-chunking test knob: one piece
//                  per thread (SPEC's chunk rule), same composition tree.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "device.cuh"
#include "kernels.hpp"

namespace sfa {

// Diagnostic builds (libsfa_diag.so, -DSFA_STAMPS): per-CTA phase times of
// k_scan_tma (scripts/stamps.py).  The product library compiles them out.
#ifdef SFA_STAMPS
#define SFA_STAMP(i)                                                                 \
    do {                                                                             \
        if (a.stamps && threadIdx.x == 0) a.stamps[blockIdx.x * 16 + (i)] = globaltimer(); \
    } while (0)
#define SFA_STAMP_P(i)                                                               \
    do {                                                                             \
        if (a.stamps) a.stamps[blockIdx.x * 16 + (i)] = globaltimer();                \
    } while (0)
#define SFA_STAMP_AT(ptr, i)                                                         \
    do {                                                                             \
        if ((ptr) && threadIdx.x == 0) (ptr)[blockIdx.x * 16 + (i)] = globaltimer(); \
    } while (0)
#else
#define SFA_STAMP_AT(ptr, i) \
    do {                     \
    } while (0)
#define SFA_STAMP(i) \
    do {             \
    } while (0)
#define SFA_STAMP_P(i) \
    do {               \
    } while (0)
#endif

template <class Step>
__host__ __device__ size_t table_bytes(const DevTables& t) {
    return (Step::smem_bytes(t) + 15) & ~size_t(15);
}

// ------------------------------------------------------------------------------------------
// Composition (Alg. 5 line 6): f . g := g o f, associative
// (PAPER.md:150), so chunk states fold in text order under any bracketing.
//
//   ID  (VEC = false)  a value is an SFA id, the same in every lane.
//                      s_a . s_b = comp[s_a][s_b], the D-SFA's composition
//                      table built on the host (closed: f_u . f_v = f_uv is a
//                      state again, Lemma 1), copied into smem
//                      when small; without a table (|S|^2 too large) by
//                      Lemma-1 replay: delta_s run from s_a over rep(s_b), a
//                      shortest word with f_I -rep(s_b)-> s_b (<= depth lookups).
//   VEC (VEC = true)   |Q| <= 32: lane q holds f(q); f . g = shfl(g, f) (the
//                      north_star's warp-shuffle form); ids become vectors
//                      through maps32 (smem when small).
// A warp folds its 32 lane values with a 5-level shuffle tree (ID) or a
// 32-step sequential application (VEC, one dependent LDS per step).
// ------------------------------------------------------------------------------------------
template <class Step, bool VEC>
struct Comp;

template <class Step>
struct Comp<Step, true> {
    static constexpr int kSlot = 32;  // bytes per stored value
    __device__ static uint32_t identity() { return lane_id(); }
    // maps32: its smem copy when the aux image holds it
    __device__ static const uint8_t* maps(const DevTables& t) {
        return t.aux_maps ? dsmem + t.aux_off + t.aux_maps_off : t.maps32;
    }
    __device__ static uint32_t fold_states(const Step&, const DevTables& t, uint32_t s) { return vec_fold_ids(maps(t), s); }
    __device__ static uint32_t combine(const Step&, const DevTables&, uint32_t a, uint32_t b) { return vec_compose(a, b); }
    __device__ static void store(uint8_t* slot, uint32_t v) { slot[lane_id()] = static_cast<uint8_t>(v); }
    __device__ static uint32_t load(const uint8_t* slot) { return slot[lane_id()]; }
    __device__ static uint32_t load_global(const uint8_t* p) { return __ldcg(p + lane_id()); }
    // fold `count` stored values in order into acc
    __device__ static uint32_t fold_slots(const Step& S, const DevTables& t, const uint8_t* base, uint32_t count,
                                          uint32_t acc, bool global) {
        for (uint32_t u = 0; u < count; ++u) {
            uint32_t v = global ? load_global(base + u * kSlot) : load(base + u * kSlot);
            acc = combine(S, t, acc, v);
        }
        return acc;
    }
    // f_fin(q): lane q holds f_fin(q)
    __device__ static uint32_t q_final(const DevTables&, uint32_t v, uint32_t q) { return __shfl_sync(kFull, v, q); }
};

template <class Step>
struct Comp<Step, false> {
    static constexpr int kSlot = 4;
    __device__ static uint32_t identity() { return 0; }  // f_I has id 0 (C3)
    __device__ __forceinline__ static uint32_t combine(const Step& S, const DevTables& t, uint32_t a, uint32_t b) {
        if (a == 0) return b;  // f_I . f = f
        if (b == 0) return a;
        // factored values stay factored (and SFA ids become factored when they
        // can) unless the composition table sits in smem
        if (a & b & kFact)  // both factored: (F1, g1) . (F2, g2) = (F1, f_(F2, g2)(g1)), inline
            return (a & 0xffff0000u) | fam_apply(t, (b >> 16) & 0x3fffu, b & 0xffffu, a & 0xffffu);
        if (((a | b) & kFact) || (fact_values(t) && !t.aux_comp)) return combine_fact(S, t, a, b);
        return combine_ids(S, t, a, b);
    }
    // two canonical SFA ids
    __device__ __forceinline__ static uint32_t combine_ids(const Step& S, const DevTables& t, uint32_t a, uint32_t b) {
        SFA_CTR(t, 1);
        if (t.comp) {  // its smem copy when the aux image holds it
            const void* c = t.aux_comp ? static_cast<const void*>(dsmem + t.aux_off) : t.comp;
            const uint32_t i = a * t.nS + b;
            return t.comp_u8 ? static_cast<const uint8_t*>(c)[i] : static_cast<const uint16_t*>(c)[i];
        }
        return combine_slow(S, t, a, b);
    }
    // A factored value on either side (Step policies with FACTORED chunk values):
    // (F1, g1) . b = (F1, f_b(g1)) -- f_b(g1) from b's family when b is factored
    // (fam_apply, L1-resident), else from maps16; an SFA id a on the left is
    // factored first when it can be, else b goes back to its canonical id.
    __device__ __noinline__ static uint32_t combine_fact(const Step& S, const DevTables& t, uint32_t a, uint32_t b) {
        SFA_CTR(t, 0);
        if (!(a & kFact)) {
            const uint32_t fa = __ldg(t.fact_fam + a);
            if (fa == 0xffffu) return combine_ids(S, t, a, (b & kFact) ? fact_value_id(t, b) : b);
            a = fact_pack(fa, __ldg(t.fact_g + a));
        }
        if (!(b & kFact) && !t.maps16) return combine_ids(S, t, fact_value_id(t, a), b);
        const uint32_t g1 = a & 0xffffu;
        const uint32_t g = (b & kFact) ? fam_apply(t, (b >> 16) & 0x3fffu, b & 0xffffu, g1)
                                       : __ldg(t.maps16 + static_cast<uint64_t>(b) * t.nD + g1);
        return (a & 0xffff0000u) | g;
    }
    // no composition table (|S| > 4096): a call, so the folds stay small
    __device__ __noinline__ static uint32_t combine_slow(const Step& S, const DevTables& t, uint32_t a, uint32_t b) {
        SFA_CTR(t, 2);
        if (t.fact_fam && t.maps16) {
            // a factorable: f_a = (family F, g) sends its unmarked q to g and the
            // marked ones to absorbing states, which f_b fixes; so f_a . f_b =
            // (F, f_b(g)) -- one mapping lookup instead of a replay of rep(b).
            const uint32_t fa = __ldg(t.fact_fam + a);
            if (fa != 0xffffu) {
                const uint32_t gb = __ldg(t.maps16 + static_cast<uint64_t>(b) * t.nD + __ldg(t.fact_g + a));
                const uint32_t r = __ldg(t.fact_tab + fa * t.nD + gb);
                if (r != 0xffffu) return r;
            }
        }
        return replay(S, t, a, b, lane_id());
    }
    // the 32 lanes' ids, in lane order, folded by a shuffle tree; result in every lane
    // __noinline__: one copy of the fold code, so the last CTA's final fold runs
    // instructions its own CTA fold has just brought into the I-cache
    __device__ __noinline__ static uint32_t fold_states(const Step& S, const DevTables& t, uint32_t s) {
        const uint32_t lane = lane_id();
        if (t.aux_comp && !fact_values(t)) {  // ids through the smem composition table: a tight LDS tree
            const uint32_t base = smem_u32(dsmem) + t.aux_off, nS = t.nS;
            const bool u8 = t.comp_u8 != 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_down_sync(kFull, s, d);
                const uint32_t i = s * nS + o;
                const uint32_t v = u8 ? lds_u8(base + i) : lds_u16(base + 2 * i);
                const uint32_t c = s == 0 ? o : (o == 0 ? s : v);
                s = (lane & (2 * d - 1)) == 0 ? c : s;
            }
            return __shfl_sync(kFull, s, 0);
        }
        if (t.aux_fam && __all_sync(kFull, s == 0 || (s & kFact))) {
            // every value factored (or f_I): branch-free tree over the smem marked sets
            const uint32_t base = smem_u32(dsmem) + t.aux_off, fw = t.fam_w, a0 = t.fam_a0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_down_sync(kFull, s, d);
                const uint32_t F = (o >> 16) & 0x3fffu, g = s & 0xffffu;
                const uint32_t w = lds_u32(base + 4u * (F * fw + (g >> 5)));
                uint32_t c = (s & 0xffff0000u) | (((w >> (g & 31)) & 1u) ? a0 : (o & 0xffffu));
                c = s == 0 ? o : (o == 0 ? s : c);
                s = (lane & (2 * d - 1)) == 0 ? c : s;
            }
            return __shfl_sync(kFull, s, 0);
        }
        if (t.aux_fam) SFA_CTR(t, 4);  // diag: a fold with an SFA id among factored values
        if (fact_values(t)) {  // factored values: the inline (F, g) rule, the rest by combine
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_down_sync(kFull, s, d);
                if ((lane & (2 * d - 1)) == 0) {
                    if (s & o & kFact) s = (s & 0xffff0000u) | fam_apply(t, (o >> 16) & 0x3fffu, o & 0xffffu, s & 0xffffu);
                    else s = combine(S, t, s, o);
                }
            }
            return __shfl_sync(kFull, s, 0);
        }
        if (t.comp) {  // a table lookup: every lane combines (no divergence), the tree keeps its lanes
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_down_sync(kFull, s, d);
                const uint32_t c = combine(S, t, s, o);
                s = (lane & (2 * d - 1)) == 0 ? c : s;
            }
        } else {
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_down_sync(kFull, s, d);
                if ((lane & (2 * d - 1)) == 0) s = combine(S, t, s, o);
            }
        }
        return __shfl_sync(kFull, s, 0);
    }
    __device__ static void store(uint8_t* slot, uint32_t v) {
        if (lane_id() == 0) *reinterpret_cast<uint32_t*>(slot) = v;
    }
    __device__ static uint32_t load(const uint8_t* slot) { return *reinterpret_cast<const uint32_t*>(slot); }
    __device__ __noinline__ static uint32_t fold_slots(const Step& S, const DevTables& t, const uint8_t* base,
                                                       uint32_t count, uint32_t acc, bool global) {
        for (uint32_t c0 = 0; c0 < count; c0 += 32) {
            uint32_t u = c0 + lane_id();
            uint32_t x = 0;
            if (u < count)
                x = global ? __ldcg(reinterpret_cast<const unsigned int*>(base) + u)
                           : reinterpret_cast<const uint32_t*>(base)[u];
            uint32_t r = fold_states(S, t, x);
            acc = combine(S, t, acc, r);
        }
        return acc;
    }
    __device__ static uint32_t q_final(const DevTables& t, uint32_t v, uint32_t q) {
        if (v & kFact) return fam_apply(t, (v >> 16) & 0x3fffu, v & 0xffffu, q);
        return q == 0 ? (t.img0[v] & 0x7fffffffu) : t.maps16[static_cast<uint64_t>(v) * t.nD + q];
    }
};

// Kernel prologue: the step table -> dsmem[0, tbl) (expanded from the compact
// window table), the aux image (composition table and/or maps32,
// DevTables::aux) -> dsmem[tbl, tbl + aux) unless `aux_async` (the caller
// bulk-copies it), cooperatively by `nthreads` threads.  `t` stays the
// kernel parameter (no local copy): Comp finds the smem copies by offset.
template <class Step>
__device__ __forceinline__ void load_tables(const DevTables& t, int tid, int nthreads, bool aux_async = false,
                                            uint32_t compact_s = 0) {
    Step::fill(t, tid, nthreads, compact_s);
    const uint32_t tb = static_cast<uint32_t>((Step::smem_bytes(t) + 15) & ~size_t(15));
    if (t.aux_bytes && !aux_async)
        copy16(reinterpret_cast<uint4*>(dsmem + tb), reinterpret_cast<const uint4*>(t.aux), t.aux_bytes / 16, tid,
               nthreads);
}

template <class Step, bool VEC>
__device__ void grid_epilogue(const Step& S, const DevTables& t, const Scratch& sc, sfa_result* result,
                              const uint8_t* text, uint64_t head, uint32_t nslots, uint64_t tail0, uint64_t tail1,
                              const uint32_t* q_in, int nwarps, uint8_t* red, uint32_t* flag, uint32_t* map_out,
                              uint64_t* stamps = nullptr) {
    using CP = Comp<Step, VEC>;
    (void)stamps;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nthreads = nwarps * 32;
    if (warp == 0 && lane == 0) {  // the partial (stored by this thread) is released with the ticket
        uint32_t old;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(sc.ticket) : "memory");
        *flag = old == gridDim.x - 1 ? 1u : 0u;
    }
    bar_compute(nthreads);
    if (*flag == 0) return;
    __threadfence();  // acquire the other CTAs' partials
    SFA_STAMP_AT(stamps, 11);  // last CTA: ticket taken
    // The last CTA, all warps at once: warps [0, np) fold the CTA partials,
    // warp np runs the head [0, head), the other warps the tail [tail0,
    // tail1) in 16-byte pieces (its bytes were prefetched into L2 at entry);
    // slots in text order: head | partials | tail pieces.
    const int np = min(nwarps - 2, max(1, static_cast<int>((nslots + 31) / 32)));
    const uint32_t per = (nslots + np - 1) / np;
    const int tw = nwarps - 1 - np;  // tail warps
    uint32_t acc;
    if (warp < np) {
        const uint32_t b0 = min(nslots, warp * per), b1 = min(nslots, b0 + per);
        acc = CP::fold_slots(S, t, sc.partials + b0 * CP::kSlot, b1 - b0, CP::identity(), true);
        CP::store(red + (1 + warp) * CP::kSlot, acc);
    } else if (warp == np) {  // head, split over the 32 lanes
        const uint64_t hp = (head + 31) / 32;
        const uint64_t h0 = min(head, lane * hp), h1 = min(head, h0 + hp);
        uint32_t s = S.id(run_range(S, S.init(lane), text, h0, h1), lane);
        if (!VEC && fact_values(t) && s) s = fact_of_id(t, s);
        CP::store(red, CP::fold_states(S, t, s));
    } else {
        const uint64_t len = tail1 - tail0, ti = static_cast<uint64_t>(threadIdx.x - (np + 1) * 32);
        const uint64_t pp = 16 * ((len + 16 * 32 * tw - 1) / (16 * 32 * tw));
        const uint64_t p0 = min(tail1, tail0 + ti * pp), p1 = min(tail1, p0 + pp);
        uint32_t s = S.id(run_range(S, S.init(lane), text, p0, p1), lane);
        if (!VEC && fact_values(t) && s) s = fact_of_id(t, s);
        CP::store(red + warp * CP::kSlot, CP::fold_states(S, t, s));
    }
    bar_compute(nthreads);
    SFA_STAMP_AT(stamps, 12);  // partials, head and tail folded
    if (warp == 0) {
        acc = CP::fold_slots(S, t, red, nwarps, CP::identity(), false);
        SFA_STAMP_AT(stamps, 13);  // final fold
#ifdef SFA_STAMPS
        {  // diagnostic: the same fold again (warm caches)
            const uint32_t again = CP::fold_slots(S, t, red, nwarps, CP::identity(), false);
            SFA_STAMP_AT(stamps, 14);
            if (again != acc) acc = 0xdeadbeefu;
        }
#endif
        const uint32_t q0 = q_in ? *q_in : 0u;
        if (map_out)  // the whole mapping f_fin (sfa_match_map: shards of a text compose by Lemma 1)
            for (uint32_t b = 0; b < t.nD; b += 32) {
                const uint32_t qq = b + lane;
                const uint32_t v = CP::q_final(t, acc, qq < t.nD ? qq : 0u);
                if (qq < t.nD) map_out[qq] = v;
            }
        if (!VEC && q0 == 0 && !(acc & kFact)) {  // f_fin(q0) and its accept bit in one load (DevTables::img0)
            if (lane == 0) {
                const uint32_t x = t.img0[acc];
                if (result) *result = sfa_result{x & 0x7fffffffu, x >> 31};
                *sc.ticket = 0;  // ready for the next launch (stream-ordered)
            }
        } else {
            const uint32_t q = CP::q_final(t, acc, q0);
            if (lane == 0) {
                if (result) {
                    result->final_state = q;
                    result->accept = t.dfinal[q];
                }
                *sc.ticket = 0;
            }
        }
    }
}

// Fold one state per thread of `nwarps` warps, in thread order, into a CTA
// value; valid in warp 0 (all lanes).  Uses red[0 .. nwarps) slots.
template <class Step, bool VEC>
__device__ uint32_t block_fold(const Step& S, const DevTables& t, uint32_t s, int nwarps, uint8_t* red) {
    using CP = Comp<Step, VEC>;
    const int warp = threadIdx.x >> 5;
    CP::store(red + warp * CP::kSlot, CP::fold_states(S, t, s));
    bar_compute(nwarps * 32);
    uint32_t acc = CP::identity();
    if (warp == 0) acc = CP::fold_slots(S, t, red, nwarps, acc, false);
    bar_compute(nwarps * 32);
    return acc;
}

template <bool VEC>
__device__ __forceinline__ void store_partial(uint8_t* partials, uint32_t slot, uint32_t acc) {
    if (VEC) partials[slot * 32 + lane_id()] = static_cast<uint8_t>(acc);
    else if (lane_id() == 0) reinterpret_cast<uint32_t*>(partials)[slot] = acc;
}

// ------------------------------------------------------------------------------------------
// Batches (A5, SEG kernels): the texts back to back form one range; text
// boundaries may fall anywhere in a chunk.
//
// A chunk (row, head/tail piece, warp, CTA, ...) folds to a segmented element
//   (h, b, tl, t):  b = the chunk contains a text boundary (its start counts);
//                   h = the SFA state of the piece before the first boundary
//                       (the whole chunk if !b; f_I if the chunk starts a text);
//                   tl, t = the text of the piece after the last boundary and
//                       that piece's value.
// Elements compose in text order by
//   (h1,0)      . (h2,0)      = (h1.h2, 0)
//   (h1,0)      . (h2,1,l2,t2)= (h1.h2, 1, l2, t2)
//   (h1,1,l1,t1). (h2,0)      = (h1, 1, l1, t1.h2)
//   (h1,1,l1,t1). (h2,1,l2,t2)= (h1, 1, l2, t2)   and text l1 = t1.h2 is complete
// (associative: it is the composition of Alg. 5 line 6 restricted to each
// text).  A complete text's result is written where its two ends meet, so
// every text is finished exactly once; the range's last text when the whole
// range is folded.
//
// A value is an SFA id, or, for the piece that starts a text, possibly a DFA
// state tagged with kTag: a text always starts in q0, so its first piece only
// needs f(q0) -- which the FACTORED step (a warp running the DFA on each
// chunk's surviving image) computes directly.  (kTag | q) . s = kTag | f_s(q).
// ------------------------------------------------------------------------------------------
constexpr uint32_t kTag = 0x80000000u;
constexpr uint32_t kTagFam = 0xfffeu;  // FACTORED step: the lane runs the DFA from q0 (a text's first piece)

struct SegEl {
    uint32_t h, t, tl, b;
};

__device__ __forceinline__ SegEl seg_identity() { return SegEl{0u, 0u, 0u, 0u}; }

__device__ __forceinline__ SegEl shfl_down_el(const SegEl& e, int d) {
    return SegEl{__shfl_down_sync(kFull, e.h, d), __shfl_down_sync(kFull, e.t, d), __shfl_down_sync(kFull, e.tl, d),
                 __shfl_down_sync(kFull, e.b, d)};
}

// The tables the folds and the epilogue read from global memory, bulk-
// prefetched into L2 at kernel entry (the streamed text is evict-first, so
// they stay): otherwise each dependent lookup of the last CTA's fold can be
// a DRAM miss.  CTA 0 takes the small tables, CTAs 1.. the large ones in
// 1 MiB pieces (<= 8 MiB each).
__device__ __forceinline__ void prefetch_span(const void* p, uint64_t bytes, uint32_t piece, uint32_t npieces) {
    if (!p || !bytes) return;
    bytes = (bytes + 15) & ~uint64_t(15);
    const uint64_t per = 1u << 20, n = (bytes + per - 1) / per;
    for (uint64_t j = piece; j < n; j += npieces) {
        const uint64_t o = j * per;
        bulk_prefetch_l2(static_cast<const uint8_t*>(p) + o, static_cast<uint32_t>(min(per, bytes - o)));
    }
}
__device__ inline void prefetch_fold_tables(const DevTables& t, uint32_t cta, uint32_t nctas) {
    const uint64_t nS = t.nS, nD = t.nD;
    if (cta == 0) {
        prefetch_span(t.img0, nS * 4, 0, 1);
        prefetch_span(t.dfinal, nD, 0, 1);
        prefetch_span(t.fam_bits, static_cast<uint64_t>(t.fam_n) * t.fam_w * 4, 0, 1);
        prefetch_span(t.fam_img, static_cast<uint64_t>(t.fam_n) * nD * 2, 0, 1);
        prefetch_span(t.dwin_unrank, nD * 2, 0, 1);
        prefetch_span(t.dwin_rank, nD * 2, 0, 1);
        prefetch_span(t.fact_fam, nS * 2, 0, 1);
        prefetch_span(t.fact_g, nS * 2, 0, 1);
        prefetch_span(t.fact_tab, static_cast<uint64_t>(t.fam_n) * nD * 2, 0, 1);
        return;
    }
    const uint64_t m16 = nS * nD * 2, cb = nS * nS * (t.comp_u8 ? 1 : 2);
    if (m16 <= (8u << 20)) prefetch_span(t.maps16, m16, cta - 1, nctas - 1);
    if (t.comp && !t.aux_comp && cb <= (8u << 20)) prefetch_span(t.comp, cb, cta - 1, nctas - 1);
}

// The boundaries of a batch range: text i = [start(i), start(i+1)).
struct Bounds {
    const uint64_t* off;  // count + 1 absolute offsets; nullptr: equal texts of `len` bytes
    uint64_t off0, count, len;
    __device__ __forceinline__ uint64_t start(uint64_t i) const {
        return off ? __ldg(off + i) - off0 : i * len;
    }
    // the nonempty text that holds byte x (x < range length): the last i with start(i) <= x
    __device__ uint32_t text_at(uint64_t x) const {
        if (!off) return static_cast<uint32_t>(x / len);
        uint64_t lo = 0, hi = count;  // start(lo) <= x < start(hi)
        const uint64_t ax = x + off0;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (__ldg(off + mid) <= ax) lo = mid;
            else hi = mid;
        }
        return static_cast<uint32_t>(lo);
    }
    // the nonempty text that starts where text i ends (empty texts skipped)
    __device__ __noinline__ uint32_t next(uint32_t i) const {
        if (!off) return i + 1;
        const uint64_t e = __ldg(off + i + 1);
        ++i;
        while (__ldg(off + i + 1) == e) ++i;
        return i;
    }
};

template <class Step>
struct Seg {
    // f_s(q): the mapping table, else Lemma-1 replay of rep(s) through the DFA
    // window table (smem; kTag values only come from FACTORED warps, which have it)
    __device__ __noinline__ static uint32_t apply(const DevTables& t, uint32_t s, uint32_t q) {
        if (s & kFact) return fam_apply(t, (s >> 16) & 0x3fffu, s & 0xffffu, q);
        if (t.maps16) return __ldg(t.maps16 + static_cast<uint64_t>(s) * t.nD + q);
        const uint32_t lane = lane_id();
        uint32_t st = dw_enc(t, q, lane);
        const uint32_t e = __ldg(t.rep_off + s + 1);
        if (t.dwin_u8) {
            StepDfa8 D;
            D.params(t);
            for (uint32_t k = __ldg(t.rep_off + s); k < e; ++k) st = D.step(st, __ldg(t.rep + k));
        } else if (t.dwin_H) {
            StepDfaMix D;
            D.params(t);
            for (uint32_t k = __ldg(t.rep_off + s); k < e; ++k) st = D.step(st, __ldg(t.rep + k));
        } else {
            StepDfa D;
            D.params(t);
            for (uint32_t k = __ldg(t.rep_off + s); k < e; ++k) st = D.step(st, __ldg(t.rep + k));
        }
        return dw_dec(t, st, lane);
    }
    // a . b for two values of one text in order (b is never tagged)
    __device__ static uint32_t cval(const Step& S, const DevTables& t, uint32_t a, uint32_t b) {
        if (a & kTag) return b == 0 ? a : (kTag | apply(t, b, a & ~kTag));
        return Comp<Step, false>::combine(S, t, a, b);
    }
    __device__ __noinline__ static void emit(const DevTables& t, sfa_result* res, uint32_t ti, uint32_t v) {
        if (v & (kTag | kFact)) {
            const uint32_t q = (v & kTag) ? v & ~kTag : fam_apply(t, (v >> 16) & 0x3fffu, v & 0xffffu, 0u);
            res[ti] = sfa_result{q, t.dfinal[q]};
        } else {
            const uint32_t x = t.img0[v];
            res[ti] = sfa_result{x & 0x7fffffffu, x >> 31};
        }
    }
    __device__ __noinline__ static SegEl comb(const Step& S, const DevTables& t, sfa_result* res, const SegEl x,
                                              const SegEl y) {
        SegEl r;
        if (!x.b) {
            r.h = cval(S, t, x.h, y.h);
            r.b = y.b;
            r.tl = y.tl;
            r.t = y.t;
        } else {
            const uint32_t m = cval(S, t, x.t, y.h);
            r.h = x.h;
            r.b = 1;
            if (y.b) {
                emit(t, res, x.tl, m);
                r.tl = y.tl;
                r.t = y.t;
            } else {
                r.tl = x.tl;
                r.t = m;
            }
        }
        return r;
    }
    // the 32 lanes' elements in lane order; result in lane 0
    __device__ static SegEl fold_warp(const Step& S, const DevTables& t, sfa_result* res, SegEl e) {
        const uint32_t lane = lane_id();
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const SegEl o = shfl_down_el(e, d);
            if ((lane & (2 * d - 1)) == 0) e = comb(S, t, res, e, o);
        }
        return e;
    }
    // fold `count` stored elements (smem or global) in order into acc (valid in lane 0)
    __device__ static SegEl fold_slots(const Step& S, const DevTables& t, sfa_result* res, const uint4* base,
                                       uint32_t count, SegEl acc, bool global) {
        for (uint32_t c0 = 0; c0 < count; c0 += 32) {
            const uint32_t u = c0 + lane_id();
            SegEl x = seg_identity();
            if (u < count) {
                const uint4 v = global ? __ldcg(base + u) : base[u];
                x = SegEl{v.x, v.y, v.z, v.w};
            }
            x = fold_warp(S, t, res, x);
            if (lane_id() == 0) acc = comb(S, t, res, acc, x);
        }
        return acc;
    }
    // a piece [x0, x1) of the range run byte by byte by one thread (head and tail pieces)
    __device__ __noinline__ static SegEl run_piece(const Step& S, const DevTables& t, sfa_result* res, const Bounds B,
                                      const uint8_t* text, uint64_t x0, uint64_t x1) {
        SegEl e = seg_identity();
        if (x0 >= x1) return e;
        const uint32_t lane = lane_id();
        uint32_t ti = B.text_at(x0);
        e.b = B.start(ti) == x0;
        uint64_t nb = B.start(static_cast<uint64_t>(ti) + 1);
        uint32_t st = S.init(lane);
        uint64_t p = x0;
        for (;;) {
            const uint64_t q = nb < x1 ? nb : x1;
            st = run_range(S, st, text, p, q);
            p = q;
            if (p == x1) break;
            const uint32_t v = S.id(st, lane);  // a boundary inside the piece
            if (!e.b) {
                e.h = v;
                e.b = 1;
            } else {
                emit(t, res, ti, v);
            }
            ti = B.next(ti);
            nb = B.start(static_cast<uint64_t>(ti) + 1);
            st = S.init(lane);
        }
        if (e.b) {  // the running piece is the last one
            e.tl = ti;
            e.t = S.id(st, lane);
        } else {    // no boundary: the whole piece is h
            e.h = S.id(st, lane);
        }
        return e;
    }
};

// ------------------------------------------------------------------------------------------
// k_scan_tma
//
// Shared memory (dynamic):  [table | staging | red slots | flag | mbarriers | stage ring]
// The table is first so its base is an immediate of every LDS.  A stage holds
// ROWB bytes of each of the CTA's rows (row-major, ROWB per row), loaded by
// NB 2-D TMA boxes; the ring depth is chosen at launch from the shared memory
// left after the table.
// ------------------------------------------------------------------------------------------
constexpr int kNW = 31;        // compute warps
constexpr int kMaxRing = 8;    // max smem ring depth

template <int K>
__host__ __device__ constexpr int Sh_NB() { return (K * kNW * 32 + 255) / 256; }

template <int K, int ROWB>
struct TmaShape {
    static constexpr int R = K * kNW * 32;            // rows (chunks) per CTA at most
    static constexpr int NB = (R + 255) / 256;        // TMA boxes per stage (box dim <= 256)
    static_assert(ROWB % 16 == 0 && 256 % ROWB == 0, "row slice must be 16-B granular");
    // TMA swizzle matched to the row slice (16 B: none, 32 B: SWIZZLE_32B,
    // 64 B: SWIZZLE_64B): 16-byte chunk bits [4, 4+log2(ROWB/16)) of a smem
    // address are XORed with bits [7, ...).  With it, the 8 lanes of one LDS.128
    // wavefront (8 consecutive rows, same chunk) hit 8 distinct 16-B bank groups.
    static constexpr uint32_t kSwzMask = ROWB / 16 - 1;
    static_assert(R * ROWB % 1024 == 0 || kSwzMask == 0, "stages must keep the 1024-B swizzle phase");
    static constexpr uint32_t kStageBytes = R * ROWB;
    static constexpr uint32_t kRedBytes = ((K * kNW + 2) * 32 + 15) & ~15u;
    // bytes besides the table and the ring
    static constexpr uint32_t kFixed = kRedBytes + 16 + (2 * kMaxRing + 3) * 8 + 1024;
    // physical offset of logical stage offset `o` (rows of ROWB bytes)
    __host__ __device__ static constexpr uint32_t swz(uint32_t o) { return o ^ (((o >> 7) & kSwzMask) << 4); }
};

struct TmaMaps {
    CUtensorMap load;      // box [ROWB x bh]: the full boxes of a stage
    CUtensorMap part_hi;   // box [ROWB x (rc_hi % bh)]: the last box of CTAs with rc_hi rows
    CUtensorMap part_lo;   // box [ROWB x (rc_lo % bh)]: ... with rc_lo rows
};

// The consumer side of the stage ring: full/empty mbarriers, slot, phase.
struct Ring {
    uint32_t full0, empty0, base, n, slot, phase;
    __device__ __forceinline__ uint32_t src(uint32_t stage_bytes) const { return base + slot * stage_bytes; }
    // Release the slot only after every lane has consumed its loaded bytes,
    // so no LDS of this stage can still be in flight when the producer's next
    // TMA write lands (an arrive right after issuing the LDS raced).
    __device__ __forceinline__ void release(uint32_t lane) {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * slot);
        if (++slot == n) {
            slot = 0;
            phase ^= 1;
        }
    }
};

template <int K, int ROWB, class Sh>
__device__ __forceinline__ void load_stage(uint4 (&v)[K][ROWB / 16], const uint32_t (&rsrc)[K][ROWB / 16], Ring& ring) {
    mbar_wait(ring.full0 + 8 * ring.slot, ring.phase);
    const uint32_t src = ring.base + ring.slot * Sh::kStageBytes;
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int c = 0; c < ROWB / 16; ++c) v[k][c] = lds_v4(src + rsrc[k][c]);
}

// Stages [i0, i1) of the K rows of this thread through `S` (Alg. 5 lines 3-5):
// wait for the stage, read each row's ROWB bytes (swizzled LDS.128), step the
// K chains byte by byte (interleaved for ILP), release the slot.
template <int K, int ROWB, class Sh, class StepT>
__device__ __forceinline__ void scan_stages(const StepT& S, uint32_t (&st)[K], const uint32_t (&rsrc)[K][ROWB / 16],
                                            Ring& ring, uint32_t i0, uint32_t i1, uint32_t lane) {
    for (uint32_t i = i0; i < i1; ++i) {
        uint4 v[K][ROWB / 16];
        load_stage<K, ROWB, Sh>(v, rsrc, ring);
#pragma unroll
        for (int c = 0; c < ROWB / 16; ++c) {
            const uint32_t* w[K];
#pragma unroll
            for (int k = 0; k < K; ++k) w[k] = reinterpret_cast<const uint32_t*>(&v[k][c]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
#pragma unroll
                for (int k = 0; k < K; ++k) st[k] = S.step(st[k], byte_of<0>(w[k][q]));
#pragma unroll
                for (int k = 0; k < K; ++k) st[k] = S.step(st[k], byte_of<1>(w[k][q]));
#pragma unroll
                for (int k = 0; k < K; ++k) st[k] = S.step(st[k], byte_of<2>(w[k][q]));
#pragma unroll
                for (int k = 0; k < K; ++k) st[k] = S.step(st[k], byte_of<3>(w[k][q]));
            }
#pragma unroll
            for (int k = 0; k < K; ++k) st[k] = maybe_fix(S, st[k]);
        }
        ring.release(lane);
    }
}

// A warp without rows: keeps the ring's empty-barrier count (kNW arrivals per
// stage) without reading the stages.
__device__ __forceinline__ void follow_stages(Ring& ring, uint32_t nstages, uint32_t lane) {
    for (uint32_t i = 0; i < nstages; ++i) {
        mbar_wait(ring.full0 + 8 * ring.slot, ring.phase);
        ring.release(lane);
    }
}

// Per-row segment state of a SEG scan (row-relative positions).
template <int K>
struct RowSegs {
    uint64_t x0[K];   // row start in the range
    uint32_t nb[K];   // next boundary (row-relative); >= L: none inside the row
    uint32_t h[K], tl[K];
    uint32_t b[K], ts[K];  // ts: the running piece starts a text
};

// The same for a batch: a stage in which some row of the warp meets a text
// boundary runs byte by byte (LDS.U8 from the stage) and `close(k)` ends row
// k's running piece after the byte that reaches its boundary nb[k].
template <int K, int ROWB, class Sh, class StepT, class Close>
__device__ __forceinline__ void scan_stages_seg(const StepT& S, uint32_t (&st)[K], const uint32_t (&rsrc)[K][ROWB / 16],
                                                const uint32_t (&rrow)[K], Ring& ring, uint32_t i0, uint32_t i1,
                                                uint32_t lane, const uint32_t (&nb)[K], Close&& close) {
    for (uint32_t i = i0; i < i1; ++i) {
        // the stages before the warp's next text boundary run as a plain scan
        // (no per-stage test); a boundary at row position nb lies in stage (nb - 1) / ROWB
        uint32_t m = nb[0];
#pragma unroll
        for (int k = 1; k < K; ++k) m = min(m, nb[k]);
        m = __reduce_min_sync(kFull, m);
        const uint32_t j = m == 0xffffffffu ? i1 : min(i1, (m - 1) / ROWB);
        if (j > i) {
            scan_stages<K, ROWB, Sh>(S, st, rsrc, ring, i, j, lane);
            i = j - 1;
            continue;
        }
        const uint32_t pend = (i + 1) * ROWB;
        bool need = false;
#pragma unroll
        for (int k = 0; k < K; ++k) need |= nb[k] <= pend;
        if (!__any_sync(kFull, need)) {
            uint4 v[K][ROWB / 16];
            load_stage<K, ROWB, Sh>(v, rsrc, ring);
#pragma unroll
            for (int c = 0; c < ROWB / 16; ++c) {
                const uint32_t* w[K];
#pragma unroll
                for (int k = 0; k < K; ++k) w[k] = reinterpret_cast<const uint32_t*>(&v[k][c]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
#pragma unroll
                    for (int k = 0; k < K; ++k) st[k] = S.step(st[k], byte_of<0>(w[k][q]));
#pragma unroll
                    for (int k = 0; k < K; ++k) st[k] = S.step(st[k], byte_of<1>(w[k][q]));
#pragma unroll
                    for (int k = 0; k < K; ++k) st[k] = S.step(st[k], byte_of<2>(w[k][q]));
#pragma unroll
                    for (int k = 0; k < K; ++k) st[k] = S.step(st[k], byte_of<3>(w[k][q]));
                }
#pragma unroll
                for (int k = 0; k < K; ++k) st[k] = maybe_fix(S, st[k]);
            }
        } else {
            mbar_wait(ring.full0 + 8 * ring.slot, ring.phase);
            const uint32_t src = ring.src(Sh::kStageBytes);
#pragma unroll 1
            for (uint32_t j = 0; j < ROWB; ++j) {
                const uint32_t pos = i * ROWB + j + 1;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    st[k] = S.step(st[k], lds_u8(src + Sh::swz(rrow[k] * ROWB + j)));
                    if (pos == nb[k]) close(k);
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k) st[k] = maybe_fix(S, st[k]);
        }
        ring.release(lane);
    }
}

template <class Step, int K, int ROWB, bool VEC, bool SEG>
__global__ void __launch_bounds__((kNW + 1) * 32, 1)
k_scan_tma(const __grid_constant__ TmaMaps maps, const __grid_constant__ ScanArgs a, const uint32_t tbl_bytes,
           const uint32_t stage_bytes,
           const uint32_t nring) {
    using Sh = TmaShape<K, ROWB>;
    using CP = Comp<Step, VEC>;
    using SG = Seg<Step>;
    // [step table + aux (tbl_bytes) | compact table staging (stage_bytes) | red | flag | bars | ring]
    uint8_t* const staging = dsmem + ((tbl_bytes + 15) & ~15u);
    uint8_t* red = staging + stage_bytes;
    uint32_t* flag = reinterpret_cast<uint32_t*>(red + Sh::kRedBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + Sh::kRedBytes + 16);
    const uint32_t abar = smem_u32(bars + 2 * kMaxRing);      // aux image landed
    const uint32_t cbar = smem_u32(bars + 2 * kMaxRing + 1);  // compact table landed
    const uint32_t rbar = smem_u32(bars + 2 * kMaxRing + 2);  // compute warps built their table part
    const uint32_t ring0 = (smem_u32(bars + 2 * kMaxRing + 3) + 1023) & ~1023u;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t full0 = smem_u32(bars), empty0 = full0 + kMaxRing * 8;
    pdl_launch_dependents();
    SFA_STAMP(0);
#ifdef SFA_STAMPS
    if (a.stamps && threadIdx.x == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.stamps[blockIdx.x * 16 + 6] = smid;
    }
#endif
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < nring; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, kNW);
        }
        mbar_init(abar, 1);
        mbar_init(cbar, 1);
        mbar_init(rbar, kNW);
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kNW) {  // ---- TMA producer ----
        if (lane == 0) {
            if (stage_bytes) {  // the compact table (the handle's), expanded in smem by the compute warps
                mbar_expect_tx(cbar, stage_bytes);
                bulk_g2s(smem_u32(staging), Step::staged_src(a.t), stage_bytes, cbar);
            }
            if (gridDim.x > 1) prefetch_fold_tables(a.t, blockIdx.x, gridDim.x);
            if (a.t.aux_bytes) {  // composition aux image: needed only at the fold
                const uint32_t tb = static_cast<uint32_t>((Step::smem_bytes(a.t) + 15) & ~size_t(15));
                mbar_expect_tx(abar, a.t.aux_bytes);
                bulk_g2s(smem_u32(dsmem + tb), a.t.aux, a.t.aux_bytes, abar);
            }
            // The text (and a batch's plan) may come from the previous kernel of
            // the stream: nothing of it is read before that kernel completed.
            pdl_wait();
            if (SEG && a.err && *a.err == a.epoch) return;  // bad offsets: the compute warps report
            const TmaPlan P = a.dplan ? *a.dplan : a.plan;
            if (blockIdx.x == gridDim.x - 1) {  // the tail this CTA runs after its rows, and the head: into L2 now
                const uint8_t* base = a.text + (a.off ? __ldg(a.off) : 0ull);
                const uint32_t tb = static_cast<uint32_t>((P.n - P.tail_start) & ~uint64_t(15));
                if (tb) bulk_prefetch_l2(base + P.tail_start, tb);
                // the 16-B blocks holding [0, head): the whole blocks lie in the text's pages
                const uintptr_t h0 = reinterpret_cast<uintptr_t>(base) & ~uintptr_t(15);
                const uintptr_t h1 = (reinterpret_cast<uintptr_t>(base) + P.head + 15) & ~uintptr_t(15);
                if (P.head && h1 > h0) bulk_prefetch_l2(reinterpret_cast<const void*>(h0), static_cast<uint32_t>(h1 - h0));
            }
            const uint32_t rc = P.cta_rows(blockIdx.x);
            if (rc == 0) return;
            const CUtensorMap* gm = static_cast<const CUtensorMap*>(a.gmaps);
            const CUtensorMap* mload = gm ? gm : &maps.load;
            const CUtensorMap* mpart = gm ? gm + (rc == P.rc_hi ? 1 : 2) : (rc == P.rc_hi ? &maps.part_hi : &maps.part_lo);
            const uint32_t nfull = rc / P.bh, part = rc - nfull * P.bh;  // boxes of bh rows, then one of `part`
            if (gm) {
                tmap_acquire(mload);
                tmap_acquire(mpart);
            }
            prefetch_tmap(mload);
            if (part) prefetch_tmap(mpart);
            SFA_STAMP_P(7);  // producer: first TMA about to be issued
            const uint64_t policy = policy_evict_first();
            const int y0 = static_cast<int>(P.cta_row0(blockIdx.x));
            const uint32_t nstages = static_cast<uint32_t>(P.L / ROWB);
            uint32_t slot = 0, phase = 0;
            for (uint32_t i = 0; i < nstages; ++i) {
                // Only the first stage is requested before the compute warps
                // have built the table: their table reads would otherwise
                // queue behind the whole ring fill (~20 MB device-wide).
                if (i == 1) mbar_wait(rbar, 0);
                if (i >= nring) mbar_wait(empty0 + 8 * slot, phase ^ 1);
                mbar_expect_tx(full0 + 8 * slot, rc * ROWB);
                const uint32_t dst = ring0 + slot * Sh::kStageBytes;
                for (uint32_t j = 0; j < nfull; ++j)
                    tma_load_2d(dst + j * P.bh * ROWB, mload, full0 + 8 * slot, i * ROWB, y0 + j * P.bh, policy);
                if (part)
                    tma_load_2d(dst + nfull * P.bh * ROWB, mpart, full0 + 8 * slot, i * ROWB, y0 + nfull * P.bh, policy);
                if (++slot == nring) {
                    slot = 0;
                    phase ^= 1;
                }
            }
        }
        return;
    }

    // ---- compute warps ----
    Step S;
    const DevTables& t = a.t;
    S.params(t);
    // The table images (built on the host at upload) -> smem.  A cooperative
    // copy through generic stores (not a bulk copy): with it ptxas keeps the
    // smem base in a uniform register and folds it into every LDS.U16 of the
    // hot loop ([R+UR]), one IADD per byte less.
    if (stage_bytes) mbar_wait(cbar, 0);
    load_tables<Step>(t, threadIdx.x, kNW * 32, true, stage_bytes ? smem_u32(staging) : 0u);
    if (t.aux_fam) mbar_wait(abar, 0);  // the marked sets: a batch may finish texts (emit) mid-scan
    __syncwarp();
    if (lane == 0) mbar_arrive(rbar);
    bar_compute(kNW * 32);
    SFA_STAMP(1);  // tables built
    // Everything below reads the text, the plan or the scratch shared with
    // the previous launch of the stream: wait for it (the prologue above
    // overlapped its tail).
    pdl_wait();
    if (SEG && a.err && *a.err == a.epoch) {  // k_batch_plan found decreasing offsets: every result is invalid
        if (t.aux_bytes) mbar_wait(abar, 0);  // no bulk copy may land after the CTA exits
        for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kNW * 32 + threadIdx.x; i < a.count;
             i += static_cast<uint64_t>(gridDim.x) * kNW * 32)
            a.results[i] = sfa_result{0xffffffffu, 0u};
        return;
    }
    const TmaPlan P = a.dplan ? *a.dplan : a.plan;
    const uint32_t rc = P.cta_rows(blockIdx.x);
    const uint64_t crow0 = P.cta_row0(blockIdx.x);
    const uint32_t nstages = rc ? static_cast<uint32_t>(P.L / ROWB) : 0u;
    // boundaries by arithmetic when the texts have equal length (plan.len), else from the offsets
    const uint64_t off0 = a.off ? __ldg(a.off) : 0ull;
    const Bounds B{P.len ? nullptr : a.off, off0, a.count, P.len};
    const uint8_t* const text = a.text + off0;  // the range: one text, or the batch's texts back to back
    SFA_STAMP(2);  // after griddepcontrol.wait

    // The last CTA also runs the ragged tail [tail_start, n) (< L bytes) after
    // its rows (its bytes were prefetched to L2 by the producer), split over
    // its compute threads in 16-byte pieces; its value goes to slot gridDim.x
    // of the partials.
    uint32_t tail_acc = 0;
    SegEl tail_el = seg_identity();
    auto run_tail = [&]() {
        if (t.aux_bytes) mbar_wait(abar, 0);
        // 16-byte pieces from the (16-aligned) tail start: one vector load each
        const uint64_t len = P.n - P.tail_start;
        const uint64_t per = 16 * ((len + 16 * kNW * 32 - 1) / (16 * kNW * 32));
        const uint64_t p0 = min(P.n, P.tail_start + threadIdx.x * per), p1 = min(P.n, p0 + per);
        if constexpr (SEG) {
            SegEl e = SG::fold_warp(S, t, a.results, SG::run_piece(S, t, a.results, B, text, p0, p1));
            if (lane == 0) *reinterpret_cast<uint4*>(red + warp * 16) = make_uint4(e.h, e.t, e.tl, e.b);
            bar_compute(kNW * 32);
            if (warp == 0)
                tail_el = SG::fold_slots(S, t, a.results, reinterpret_cast<const uint4*>(red), kNW, seg_identity(), false);
            bar_compute(kNW * 32);
        } else {
            const uint32_t s = S.id(run_range(S, S.init(lane), text, p0, p1), lane);
            tail_acc = block_fold<Step, VEC>(S, t, s, kNW, red);
        }
    };

    uint32_t st[K];
#pragma unroll
    for (int k = 0; k < K; ++k) st[k] = S.init(lane);
    const uint32_t row0 = warp * 32 + lane;
    uint32_t rsrc[K][ROWB / 16];  // swizzled stage offset of each 16-B piece of this thread's rows
    uint32_t rrow[K];             // the rows in the stage (0 for rows past the CTA's)
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t r = k * kNW * 32 + row0;
        rrow[k] = r < rc ? r : 0u;
#pragma unroll
        for (int c = 0; c < ROWB / 16; ++c) rsrc[k][c] = Sh::swz(rrow[k] * ROWB + c * 16);
    }
    bool valid[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t r = k * kNW * 32 + row0;
        valid[k] = r < rc && crow0 + r < P.nchunks;
    }
    RowSegs<K> rs{};
    if constexpr (SEG) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            rs.x0[k] = P.head + (crow0 + k * kNW * 32 + row0) * P.L;
            rs.h[k] = 0;
            rs.b[k] = rs.ts[k] = 0;
            rs.tl[k] = 0;
            rs.nb[k] = 0xffffffffu;
            if (valid[k]) {
                const uint32_t ti = B.text_at(rs.x0[k]);
                rs.tl[k] = ti;
                rs.b[k] = rs.ts[k] = B.start(ti) == rs.x0[k];
                const uint64_t e = B.start(static_cast<uint64_t>(ti) + 1) - rs.x0[k];
                rs.nb[k] = e < P.L ? static_cast<uint32_t>(e) : 0xffffffffu;  // a boundary at the row end is the next row's
            }
        }
    }
    // row k's running piece ends at its boundary nb[k] (v = its value): the
    // first boundary of the row closes h; later ones finish a whole text
    auto seg_close = [&](int k, uint32_t v) {
        if (!rs.b[k]) {
            rs.h[k] = v;
            rs.b[k] = 1;
        } else {
            SG::emit(t, a.results, rs.tl[k], v);
        }
        const uint32_t ti = B.next(rs.tl[k]);
        rs.tl[k] = ti;
        const uint64_t e = B.start(static_cast<uint64_t>(ti) + 1) - rs.x0[k];
        rs.nb[k] = e < P.L ? static_cast<uint32_t>(e) : 0xffffffffu;
        rs.ts[k] = 1;
    };

    Ring ring{full0, empty0, ring0, nring, 0, 0};
    uint32_t fam[K], g[K];  // FACTORED: (family, DFA state) of each row
    bool factored = false;
    auto close_sfa = [&](int k) {
        seg_close(k, S.id(st[k], lane));
        st[k] = S.init(lane);
    };
    // A warp none of whose rows exists (the CTA has fewer rows than threads)
    // only follows the ring: wait for each stage, release it.
    bool any_valid = false;
#pragma unroll
    for (int k = 0; k < K; ++k) any_valid |= valid[k];
    if (!__any_sync(kFull, any_valid)) {
        follow_stages(ring, nstages, lane);
    } else if constexpr (Step::kFactor) {
        // Stages through the SFA table until every lane's state is factorable
        // (<= 1 non-absorbing image; the image count never grows along a
        // walk), checked after stages 1, 2, 4, 8, ...; the rest with the
        // factored DFA step.  A batch row's piece that starts a text needs
        // only f(q0): it continues as the DFA run from q0 (kTagFam).
        // every lane factorable?  (a batch row's text-start piece: its f(q0) as a tagged DFA state)
        auto check = [&]() -> bool {
            bool ok = true;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const uint32_t sid = S.id(st[k], lane);
                if (SEG && rs.ts[k]) {
                    fam[k] = kTagFam;
                    g[k] = dw_enc(t, t.img0[sid] & 0x7fffffffu, lane);
                } else {
                    ok &= fact_from_id(t, sid, fam[k], g[k]);
                }
            }
            return __all_sync(kFull, ok);
        };
        // stages [i0, nstages) through the DFA window table (u8 or u16 layout)
        auto run_dfa = [&](const auto& D, uint32_t i0) {
            if constexpr (SEG) {
                const uint32_t g0 = dw_enc(t, 0u, lane);
                auto close_fact = [&](int k) {
                    const uint32_t v = fam[k] == kTagFam ? (kTag | dw_dec(t, g[k], lane))
                                       : fact_values(t) ? fact_pack(fam[k], dw_dec(t, g[k], lane))
                                                        : fact_to_id(t, fam[k], g[k]);
                    seg_close(k, v);
                    fam[k] = kTagFam;
                    g[k] = g0;
                };
                scan_stages_seg<K, ROWB, Sh>(D, g, rsrc, rrow, ring, i0, nstages, lane, rs.nb, close_fact);
            } else {
                scan_stages<K, ROWB, Sh>(D, g, rsrc, ring, i0, nstages, lane);
            }
        };
        auto with_dfa_step = [&](auto&& fn) {
            if (t.dwin_u8) {
                StepDfa8 D;
                D.params(t);
                fn(D);
            } else if (t.dwin_H) {
                StepDfaMix D;
                D.params(t);
                fn(D);
            } else {
                StepDfa D;
                D.params(t);
                fn(D);
            }
        };
        uint32_t i = 0, next_check = 1;
        // The first stage: its first 8 bytes through the SFA table, then the
        // check -- chunks of most automata synchronise within a few bytes
        // (cfg3: <= 4 bytes for all but 5e-5 of them) and the SFA table's
        // rows for those first bytes are mostly cold (L2) -- and the rest of
        // the stage through whichever step applies.  Skipped when a text
        // boundary of the warp falls in the first stage (batch).
        bool boundary0 = false;
        if constexpr (SEG) {
#pragma unroll
            for (int k = 0; k < K; ++k) boundary0 |= rs.nb[k] <= static_cast<uint32_t>(ROWB);
            boundary0 = __any_sync(kFull, boundary0);
        }
        if (t.fact_fam && nstages > 1 && !boundary0) {
            uint4 v[K][ROWB / 16];
            load_stage<K, ROWB, Sh>(v, rsrc, ring);
#pragma unroll
            for (int k = 0; k < K; ++k) st[k] = step4(S, step4(S, st[k], v[k][0].x), v[k][0].y);
            // bytes 8 .. ROWB of the stage from the registers
            auto rest = [&](const auto& X, uint32_t(&s)[K]) {
#pragma unroll
                for (int k = 0; k < K; ++k) s[k] = maybe_fix(X, step4(X, step4(X, s[k], v[k][0].z), v[k][0].w));
#pragma unroll
                for (int c = 1; c < ROWB / 16; ++c)
#pragma unroll
                    for (int k = 0; k < K; ++k) s[k] = step16(X, s[k], v[k][c]);
            };
            if (check()) {
                with_dfa_step([&](const auto& D) {
                    rest(D, g);
                    ring.release(lane);
                    SFA_STAMP(15);  // thread 0: first stage done
                    run_dfa(D, 1);
                });
                factored = true;
            } else {
                rest(S, st);
                ring.release(lane);
                SFA_STAMP(15);
                i = 1;
                next_check = 2;
            }
        }
        while (!factored && i < nstages) {
            if constexpr (SEG) scan_stages_seg<K, ROWB, Sh>(S, st, rsrc, rrow, ring, i, i + 1, lane, rs.nb, close_sfa);
            else scan_stages<K, ROWB, Sh>(S, st, rsrc, ring, i, i + 1, lane);
            ++i;
            if (!t.fact_fam || i != next_check || i == nstages) continue;
            next_check *= 2;
            if (check()) {  // the rest of the rows through the DFA window table
                with_dfa_step([&](const auto& D) { run_dfa(D, i); });
                factored = true;
            }
        }
    } else {
        if constexpr (SEG) scan_stages_seg<K, ROWB, Sh>(S, st, rsrc, rrow, ring, 0, nstages, lane, rs.nb, close_sfa);
        else scan_stages<K, ROWB, Sh>(S, st, rsrc, ring, 0, nstages, lane);
    }
    SFA_STAMP(3);  // thread 0's rows scanned
    if (t.aux_bytes) mbar_wait(abar, 0);  // the composition image (bulk copy issued at entry)
    if (SEG && blockIdx.x == gridDim.x - 1) run_tail();  // single texts: the tail is the epilogue's
    SFA_STAMP(8);  // thread 0: composition image and tail done
    // canonical value of each row's running piece
    uint32_t val[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (factored) {
            if (SEG && fam[k] == kTagFam) val[k] = kTag | dw_dec(t, g[k], lane);
            else if (!VEC && fact_values(t) && !a.row_ids) val[k] = fact_pack(fam[k], dw_dec(t, g[k], lane));
            else val[k] = fact_to_id(t, fam[k], g[k]);
        } else {
            val[k] = S.id(st[k], lane);
        }
    }
    SFA_STAMP(9);  // thread 0: canonical values

    if constexpr (SEG) {
        // ---- segmented composition: warp -> block -> grid ----
        uint4* slots = reinterpret_cast<uint4*>(red);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            SegEl e = seg_identity();  // rows past the range: f_I
            if (valid[k]) e = rs.b[k] ? SegEl{rs.h[k], val[k], rs.tl[k], 1u} : SegEl{val[k], 0u, 0u, 0u};
            e = SG::fold_warp(S, t, a.results, e);
            if (lane == 0) slots[k * kNW + warp] = make_uint4(e.h, e.t, e.tl, e.b);
        }
        bar_compute(kNW * 32);
        SFA_STAMP(10);  // every warp folded
        uint4* parts = reinterpret_cast<uint4*>(a.sc.partials);
        if (warp == 0) {
            const SegEl e = SG::fold_slots(S, t, a.results, slots, K * kNW, seg_identity(), false);
            if (lane == 0) {
                parts[blockIdx.x] = make_uint4(e.h, e.t, e.tl, e.b);
                if (blockIdx.x == gridDim.x - 1) parts[gridDim.x] = make_uint4(tail_el.h, tail_el.t, tail_el.tl, tail_el.b);
            }
        }
        SFA_STAMP(4);  // CTA folded
        // last CTA to finish: head piece . CTA 0 . ... . CTA G-1 . tail
        if (warp == 0) {
            __threadfence();
            if (lane == 0) *flag = (atomicAdd(a.sc.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
        }
        bar_compute(kNW * 32);
        if (*flag == 0) return;
        __threadfence();
        // two levels: warp w folds parts [w*per, (w+1)*per) (warp 0 after the
        // head piece), then warp 0 folds the kNW warp values
        const uint32_t nparts = gridDim.x + 1, per = (nparts + kNW - 1) / kNW;  // <= 32
        SegEl e = seg_identity();
        const uint32_t u = warp * per + lane;
        if (lane < per && u < nparts) {
            const uint4 v = __ldcg(parts + u);
            e = SegEl{v.x, v.y, v.z, v.w};
        }
        e = SG::fold_warp(S, t, a.results, e);
        if (warp == 0) {
            const uint64_t hp = (P.head + 31) / 32;
            const uint64_t h0 = min(P.head, lane * hp), h1 = min(P.head, h0 + hp);
            const SegEl hd = SG::fold_warp(S, t, a.results, SG::run_piece(S, t, a.results, B, text, h0, h1));
            if (lane == 0) e = SG::comb(S, t, a.results, hd, e);
        }
        if (lane == 0) slots[warp] = make_uint4(e.h, e.t, e.tl, e.b);
        bar_compute(kNW * 32);
        if (warp == 0) {
            const SegEl acc = SG::fold_slots(S, t, a.results, slots, kNW, seg_identity(), false);
            if (lane == 0) {
                if (acc.b) SG::emit(t, a.results, acc.tl, acc.t);  // the range's last text
                *a.sc.ticket = 0;
            }
        }
        SFA_STAMP(5);  // epilogue done (last CTA)
        return;
    } else {
        if (a.row_ids) {
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (valid[k]) a.row_ids[crow0 + k * kNW * 32 + row0] = val[k];
        }
        // ---- composition: warp -> block (rows are ordered k-major, then warp, then lane) ----
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t s = valid[k] ? val[k] : 0u;  // rows past the text: f_I
            CP::store(red + (k * kNW + warp) * CP::kSlot, CP::fold_states(S, t, s));
        }
        bar_compute(kNW * 32);
        SFA_STAMP(10);  // every warp folded
        if (warp == 0) {
            uint32_t acc = CP::fold_slots(S, t, red, K * kNW, CP::identity(), false);
            store_partial<VEC>(a.sc.partials, blockIdx.x, acc);
        }
        bar_compute(kNW * 32);
        SFA_STAMP(4);  // CTA folded
        grid_epilogue<Step, VEC>(S, t, a.sc, a.result, a.text, P.head, gridDim.x, P.tail_start, P.n, a.q_in, kNW, red, flag,
                                 a.map_out, a.stamps);
        SFA_STAMP(5);
    }
}

// ------------------------------------------------------------------------------------------
// k_scan_direct: piece g = [start(g), start(g+1)) by SPEC's rule (C6).
// ------------------------------------------------------------------------------------------
constexpr int kDirectWarps = 8;
constexpr uint32_t kDirectRed = ((kDirectWarps + 2) * 32 + 15) & ~15u;

__device__ __forceinline__ uint64_t piece_start(uint64_t g, uint64_t n, uint64_t p) {
    const uint64_t q = n / p, r = n % p;
    return g * q + (g < r ? g : r);
}

template <class Step, bool VEC>
__global__ void __launch_bounds__(kDirectWarps * 32)
k_scan_direct(const __grid_constant__ DirectArgs a) {
    uint8_t* red = dsmem + table_bytes<Step>(a.t) + a.t.aux_bytes;
    uint32_t* flag = reinterpret_cast<uint32_t*>(red + kDirectRed);
    pdl_launch_dependents();
    Step S;
    const DevTables& t = a.t;
    S.params(t);
    load_tables<Step>(t, threadIdx.x, blockDim.x);
    __syncthreads();
    pdl_wait();  // the text and the scratch may belong to the previous kernel of the stream
    const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    uint32_t s = 0;
    if (g < a.npieces) {
        uint64_t b0 = piece_start(g, a.n, a.npieces), b1 = piece_start(g + 1, a.n, a.npieces);
        s = S.id(run_range(S, S.init(lane), a.text, b0, b1), lane);
    }
    if (g < a.npieces && a.piece_ids) a.piece_ids[g] = s;
    const uint32_t acc = block_fold<Step, VEC>(S, t, s, kDirectWarps, red);
    if ((threadIdx.x >> 5) == 0) store_partial<VEC>(a.sc.partials, blockIdx.x, acc);
    bar_compute(kDirectWarps * 32);
    grid_epilogue<Step, VEC>(S, t, a.sc, a.result, a.text, 0, gridDim.x, 0, 0, a.q_in, kDirectWarps, red, flag, a.map_out);
}

// ------------------------------------------------------------------------------------------
// Host launchers
// ------------------------------------------------------------------------------------------
namespace detail {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a kernel needs
// more than it was last given on this device (host overhead per launch).
template <class F>
cudaError_t ensure_smem(F kern, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> granted;  // (kernel, device) -> bytes
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_pair(reinterpret_cast<const void*>(kern), dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = granted.find(key);
    if (it != granted.end() && it->second >= static_cast<int>(smem)) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e == cudaSuccess) granted[key] = static_cast<int>(smem);
    return e;
}

// Launch with programmatic stream serialization (PDL): the kernel may begin
// while the previous kernel of the stream finishes; it calls pdl_wait()
// before it touches the text or state the previous kernel may still use.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

// One 2-D u8 tensor map [rows x L] at `base` with a [rowb x bh] box, swizzle matched to rowb.
inline cudaError_t encode_map(CUtensorMap* m, void* base, uint64_t L, uint64_t rows, uint32_t rowb, uint32_t bh, int promo) {
    EncodeFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    cuuint64_t dims[2] = {L, rows ? rows : 1};
    cuuint64_t strides[1] = {L};
    cuuint32_t box[2] = {rowb, bh ? bh : 8};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle swz = rowb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : rowb == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    const CUtensorMapL2promotion pr = promo == 64    ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                    : promo == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                                   : CU_TENSOR_MAP_L2_PROMOTION_NONE;
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Box heights of a plan's three maps (0: unused, encoded as 8).
__host__ __device__ inline void box_heights(const TmaPlan& P, uint32_t h[3]) {
    h[0] = P.bh;
    h[1] = P.bh ? P.rc_hi % P.bh : 0;
    h[2] = P.bh ? P.rc_lo % P.bh : 0;
    for (int k = 0; k < 3; ++k)
        if (h[k] == 0) h[k] = 8;
}

// The host's maps for a host plan: the last encoding is reused when the
// geometry repeats (repeated matches of one buffer: host overhead).
inline cudaError_t host_maps(const ScanArgs& a, const TmaConfig& cfg, TmaMaps* out) {
    struct Key {
        const void* base;
        uint64_t L, rows;
        uint32_t h0, h1, h2, rowb;
        int promo;
        bool operator==(const Key& o) const {
            return base == o.base && L == o.L && rows == o.rows && h0 == o.h0 && h1 == o.h1 && h2 == o.h2 &&
                   rowb == o.rowb && promo == o.promo;
        }
    };
    static thread_local Key last{nullptr, 0, 0, 0, 0, 0, 0, -9};
    static thread_local TmaMaps maps;
    const TmaPlan& P = a.plan;
    void* base = const_cast<uint8_t*>(a.text + P.head);
    if (P.nchunks == 0) base = reinterpret_cast<void*>(reinterpret_cast<uintptr_t>(base) & ~uintptr_t(255));
    uint32_t h[3];
    box_heights(P, h);
    const Key key{base, P.L, P.nchunks, h[0], h[1], h[2], static_cast<uint32_t>(cfg.rowb), cfg.promo};
    if (!(key == last)) {
        last = Key{nullptr, 0, 0, 0, 0, 0, 0, -9};
        cudaError_t e = encode_map(&maps.load, base, P.L, P.nchunks, cfg.rowb, h[0], cfg.promo);
        if (e == cudaSuccess) e = encode_map(&maps.part_hi, base, P.L, P.nchunks, cfg.rowb, h[1], cfg.promo);
        if (e == cudaSuccess) e = encode_map(&maps.part_lo, base, P.L, P.nchunks, cfg.rowb, h[2], cfg.promo);
        if (e != cudaSuccess) return e;
        last = key;
    }
    *out = maps;
    return cudaSuccess;
}

template <class Step, int K, int ROWB, bool VEC, bool SEG>
cudaError_t tma_launch_t(const ScanArgs& a, const TmaConfig& cfg, unsigned grid, cudaStream_t stream) {
    using Sh = TmaShape<K, ROWB>;
    auto kern = k_scan_tma<Step, K, ROWB, VEC, SEG>;
    ScanArgs a2 = a;
    a2.t.aux_off = static_cast<uint32_t>(table_bytes<Step>(a.t));
    const uint32_t tbytes = static_cast<uint32_t>(table_bytes<Step>(a.t) + a.t.aux_bytes);
    const uint32_t sbytes = cfg.staged ? Step::staged_bytes(a.t) : 0u;
    const size_t smem = tbytes + sbytes + Sh::kFixed + static_cast<size_t>(cfg.nring) * Sh::kStageBytes;
    cudaError_t e = ensure_smem(kern, smem);
    if (e != cudaSuccess) return e;
    TmaMaps maps;
    if (a.dplan) {
        std::memset(&maps, 0, sizeof(maps));  // unused: the kernel reads a.gmaps
    } else {
        const TmaPlan& P = a.plan;
        if (P.nchunks && (P.bh == 0 || P.bh > 256 || P.bh % 8)) return cudaErrorInvalidValue;
        e = host_maps(a, cfg, &maps);
        if (e != cudaSuccess) return e;
    }
    return launch_pdl(kern, grid, (kNW + 1) * 32, smem, stream, maps, a2, tbytes, sbytes, cfg.nring);
}

template <class Step, bool VEC, bool SEG>
cudaError_t tma_launch(const ScanArgs& a, const TmaConfig& cfg, unsigned grid, cudaStream_t stream) {
    switch (cfg.K * 1000 + cfg.rowb) {
        case 1016: return tma_launch_t<Step, 1, 16, VEC, SEG>(a, cfg, grid, stream);
        case 1032: return tma_launch_t<Step, 1, 32, VEC, SEG>(a, cfg, grid, stream);
        case 2016: return tma_launch_t<Step, 2, 16, VEC, SEG>(a, cfg, grid, stream);
        case 2032: return tma_launch_t<Step, 2, 32, VEC, SEG>(a, cfg, grid, stream);
        case 1064: return tma_launch_t<Step, 1, 64, VEC, SEG>(a, cfg, grid, stream);
        case 2064: return tma_launch_t<Step, 2, 64, VEC, SEG>(a, cfg, grid, stream);
    }
    return cudaErrorInvalidValue;
}

template <class Step, bool VEC>
cudaError_t direct_launch(const DirectArgs& a, cudaStream_t stream) {
    auto kern = k_scan_direct<Step, VEC>;
    const size_t smem = kDirectRed + 16 + table_bytes<Step>(a.t) + a.t.aux_bytes;
    cudaError_t e = ensure_smem(kern, smem);
    if (e != cudaSuccess) return e;
    const uint64_t ctas = (a.npieces + kDirectWarps * 32 - 1) / (kDirectWarps * 32);
    DirectArgs a2 = a;
    a2.t.aux_off = static_cast<uint32_t>(table_bytes<Step>(a.t));
    return launch_pdl(kern, static_cast<unsigned>(ctas), kDirectWarps * 32, smem, stream, a2);
}

}  // namespace detail

// One step policy's launchers: single-text kernels in kernels_<step>.cu, the
// batch (SEG) kernels in kernels_<step>_seg.cu.
#define SFA_DEFINE_STEP_LAUNCHERS(STEP)                                                                      \
    template <>                                                                                              \
    cudaError_t StepLaunch<STEP>::scan_tma(bool vec, const ScanArgs& a, const TmaConfig& cfg, cudaStream_t s) { \
        return vec ? detail::tma_launch<STEP, true, false>(a, cfg, a.plan.ctas, s)                          \
                   : detail::tma_launch<STEP, false, false>(a, cfg, a.plan.ctas, s);                        \
    }                                                                                                        \
    template <>                                                                                              \
    cudaError_t StepLaunch<STEP>::scan_direct(bool vec, const DirectArgs& a, cudaStream_t s) {               \
        return vec ? detail::direct_launch<STEP, true>(a, s) : detail::direct_launch<STEP, false>(a, s);     \
    }
#define SFA_DEFINE_STEP_SEG_LAUNCHER(STEP)                                                                   \
    template <>                                                                                              \
    cudaError_t StepLaunch<STEP>::scan_seg(const ScanArgs& a, const TmaConfig& cfg, unsigned grid, cudaStream_t s) { \
        return detail::tma_launch<STEP, false, true>(a, cfg, grid, s);                                       \
    }

}  // namespace sfa
