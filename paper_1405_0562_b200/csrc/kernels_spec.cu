// kernels_spec.cu -- Alg. 3: parallel computation of the
// DFA by speculative simulation, the paper's baseline for the SFA (its cost,
// O(|D| n / p + |D| log p), against the SFA's O(n / p + ...),
// Table II).  SURVEY.md s8(f) NEXT-1: the same text, the
// same byte window, one GPU -- |D| dependent DFA lookups per byte instead of 1.
//
// Mapping to the GPU.  A "chain" is one pair (chunk i, start state q) of
// Alg. 3 lines 2-6: T_i[q] <- q, then T_i[q] <- delta(T_i[q], sigma_ij) for
// every byte of chunk i.  The |D| chains of a chunk are consecutive threads
// (they read the same text bytes, which L1 serves), a CTA runs `cpc` chunks
// per pass, and the CTA's chunks are contiguous in the text so it can fold
// them in order: the pass's maps are tree-composed in shared memory (the
// parallel reduction, Alg. 3 line 9, `.` associative) and the
// result appended to the CTA's running map R <- R . G.  The last CTA to
// finish folds the per-CTA maps the same way and applies the result to q0
// (Alg. 3 line 10).  '.' is reverse composition: (f . g)(q) = g(f(q)).
//
// The DFA window table lives in shared memory when it fits (u32 entries
// premultiplied to row byte offsets, as StepShared), else it is read through
// L1/L2.  Chunk boundaries follow SPEC's rule (C6).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device.cuh"
#include "kernels.hpp"

namespace sfa {

namespace {

__device__ __forceinline__ uint64_t spec_piece(uint64_t g, uint64_t n, uint64_t p) {
    const uint64_t q = n / p, r = n % p;
    return g * q + (g < r ? g : r);
}

// state = byte offset of DFA row q (4 W q); cell (q, j) holds 4 W delta_d(q, byte_j)
template <bool SMEM>
struct DfaStep {
    const uint32_t* Tg;
    uint32_t neg_lo, wmax;
    __device__ __forceinline__ uint32_t step(uint32_t st, uint32_t byte) const {
        const uint32_t col = window_col(byte, neg_lo, wmax);
        return SMEM ? ld_tbl_u32(st + 4 * col) : __ldg(Tg + (st >> 2) + col);
    }
};

// Alg. 3 lines 4-6 for one chain: bytes [a, b) of the text from state st.
template <bool SMEM>
__device__ uint32_t spec_run(const DfaStep<SMEM>& S, uint32_t st, const uint8_t* __restrict__ t, uint64_t a, uint64_t b) {
    while (a < b && (reinterpret_cast<uintptr_t>(t + a) & 15)) st = S.step(st, __ldg(t + a++));
    if (a + 16 <= b) {
        uint4 v = __ldg(reinterpret_cast<const uint4*>(t + a));  // L1-allocating: |D| chains read each line
        a += 16;
        while (a + 16 <= b) {
            const uint4 nx = __ldg(reinterpret_cast<const uint4*>(t + a));
            a += 16;
            st = step16(S, st, v);
            v = nx;
        }
        st = step16(S, st, v);
    }
    while (a < b) st = S.step(st, __ldg(t + a++));
    return st;
}

// gm[0..nc) (nD entries each, in text order) -> gm[0] = gm[0] . gm[1] . ... ;
// then R <- R . gm[0].  All threads of the CTA; ends synchronised.
__device__ void fold_group(uint32_t* gm, uint32_t nc, uint32_t nD, uint32_t* R) {
    const uint32_t tid = threadIdx.x, nth = blockDim.x;
    for (uint32_t d = 1; d < nc; d <<= 1) {
        for (uint32_t k = tid; k < nc * nD; k += nth) {
            const uint32_t ci = k / nD;
            if ((ci & (2 * d - 1)) == 0 && ci + d < nc) gm[k] = gm[(ci + d) * nD + gm[k]];
        }
        __syncthreads();
    }
    for (uint32_t q = tid; q < nD; q += nth) R[q] = gm[R[q]];
    __syncthreads();
}

template <bool SMEM>
__global__ void __launch_bounds__(1024) k_spec_scan(const SpecArgs a) {
    const uint32_t nD = a.nD, tid = threadIdx.x, nth = blockDim.x, row = 4 * a.W;
    uint32_t* gm = reinterpret_cast<uint32_t*>(dsmem + a.tbl_smem);  // gcap maps of nD entries
    uint32_t* R = gm + static_cast<size_t>(a.gcap) * nD;                // the CTA's running map
    uint32_t* flag = R + nD;
    if (SMEM) copy16(reinterpret_cast<uint4*>(dsmem), reinterpret_cast<const uint4*>(a.Td), a.tbl_smem / 16, tid, nth);
    for (uint32_t q = tid; q < nD; q += nth) R[q] = q;  // f_I: the identity (Alg. 3 lines 2-3)
    __syncthreads();
    DfaStep<SMEM> S{a.Td, 0u - a.lo, a.W - 1};
    const uint64_t c_begin = static_cast<uint64_t>(blockIdx.x) * a.cpb;
    const uint64_t c_end = min(c_begin + a.cpb, a.nchunks);
    for (uint64_t c0 = c_begin; c0 < c_end; c0 += a.cpc) {
        const uint32_t nc = static_cast<uint32_t>(c_end - c0 < a.cpc ? c_end - c0 : a.cpc);
        for (uint32_t k = tid; k < nc * nD; k += nth) {
            const uint32_t ci = k / nD, q = k - ci * nD;
            const uint64_t c = c0 + ci;
            const uint64_t b0 = spec_piece(c, a.n, a.nchunks), b1 = spec_piece(c + 1, a.n, a.nchunks);
            const uint32_t s = spec_run(S, q * row, a.text, b0, b1) / row;  // T_i[q]
            gm[k] = s;
            if (a.chunk_maps) a.chunk_maps[c * nD + q] = s;
        }
        __syncthreads();
        fold_group(gm, nc, nD, R);
    }
    for (uint32_t q = tid; q < nD; q += nth) a.cta_maps[static_cast<size_t>(blockIdx.x) * nD + q] = R[q];
    // last CTA to finish folds the per-CTA maps (grid-level reduction)
    __threadfence();
    __syncthreads();
    if (tid == 0) *flag = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!*flag) return;
    __threadfence();
    for (uint32_t q = tid; q < nD; q += nth) R[q] = q;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < gridDim.x; b0 += a.gcap) {
        const uint32_t nc = min(a.gcap, gridDim.x - b0);
        for (uint32_t k = tid; k < nc * nD; k += nth) gm[k] = __ldcg(a.cta_maps + static_cast<size_t>(b0) * nD + k);
        __syncthreads();
        fold_group(gm, nc, nD, R);
    }
    if (tid == 0) {
        const uint32_t q = R[0];  // q_final = T[q0], q0 = 0 (C3)
        a.result->final_state = q;
        a.result->accept = a.dfinal[q];
        *a.ticket = 0;  // self-resetting for the next launch
    }
    if (a.map_out)
        for (uint32_t q = tid; q < nD; q += nth) a.map_out[q] = R[q];
}

}  // namespace

cudaError_t spec_plan(const SpecArgs& proto, int sm_count, size_t smem_optin, uint64_t n, uint64_t nchunks,
                      SpecArgs* out, uint32_t* threads, size_t* smem) {
    SpecArgs a = proto;
    const uint32_t nD = a.nD;
    a.cpc = std::max<uint32_t>(1u, 1024u / nD);
    const uint32_t nth = std::min<uint32_t>(1024u, ((a.cpc * nD + 31) / 32) * 32);
    const size_t tbl = (static_cast<size_t>(nD) * a.W * 4 + 15) & ~size_t(15);
    // group capacity: at least one pass's chunks, more (for the final fold) if it fits in 48 KB
    a.gcap = std::max<uint32_t>(a.cpc, static_cast<uint32_t>(std::min<size_t>(4096, (48u << 10) / (4u * nD))));
    const size_t fixed = (static_cast<size_t>(a.gcap) + 1) * nD * 4 + 16;
    a.tbl_smem = (tbl + fixed <= std::min<size_t>(smem_optin, 160u << 10)) ? static_cast<uint32_t>(tbl) : 0u;
    const size_t sm = a.tbl_smem + fixed;
    if (sm > smem_optin) return cudaErrorInvalidConfiguration;
    auto kern = a.tbl_smem ? k_spec_scan<true> : k_spec_scan<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, static_cast<int>(nth), sm);
    if (e != cudaSuccess) return e;
    const uint64_t max_ctas = static_cast<uint64_t>(std::max(per_sm, 1)) * static_cast<uint64_t>(sm_count);
    a.n = n;
    // auto: 4 passes per CTA at full occupancy (fewer chunks for short texts)
    a.nchunks = nchunks ? nchunks : std::max<uint64_t>(1, std::min<uint64_t>(n, max_ctas * a.cpc * 4));
    if (a.nchunks > n) a.nchunks = std::max<uint64_t>(n, 1);  // SPEC's rule: n one-byte chunks (C6)
    const uint64_t passes = (a.nchunks + a.cpc - 1) / a.cpc;
    const uint64_t ctas = std::min<uint64_t>(max_ctas, passes);
    a.cpb = ((passes + ctas - 1) / ctas) * a.cpc;
    a.ctas = static_cast<uint32_t>((a.nchunks + a.cpb - 1) / a.cpb);
    *out = a;
    *threads = nth;
    *smem = sm;
    return cudaSuccess;
}

cudaError_t launch_spec(const SpecArgs& a, uint32_t threads, size_t smem, cudaStream_t stream) {
    auto kern = a.tbl_smem ? k_spec_scan<true> : k_spec_scan<false>;
    kern<<<a.ctas, threads, smem, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace sfa
