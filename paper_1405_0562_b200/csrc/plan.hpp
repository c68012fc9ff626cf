// plan.hpp -- device-table descriptors and launch plans shared by host and device code.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/sfa.h"

namespace sfa {

// Device copies of the compiled automata (all owned by the handle).
struct DevTables {
    const uint16_t* T = nullptr;        // nS * C   next SFA id per (state, class)
    const uint8_t* cls = nullptr;       // 256      byte -> class
    const uint16_t* Trange = nullptr;   // nS * W   next SFA id per (state, window column)
    const uint32_t* pairs = nullptr;    // PRIVATE: lane-independent pair words (device.cuh StepPrivate)
    uint32_t priv_R = 0;                // PRIVATE: lane-group copies (32 = bank-private), 0 = unavailable
    const uint8_t* maps32 = nullptr;    // nS * 32  f_s(q) for |D| <= 32 (identity-padded)
    const uint16_t* maps16 = nullptr;   // nS * nD  f_s(q) (any |D|; used to apply f_fin to q_in != q0)
    const uint32_t* img0 = nullptr;     // nS       f_s(q0)
    const uint8_t* dfinal = nullptr;    // nD       q in F_d
    const uint32_t* rep_off = nullptr;  // nS + 1
    const uint8_t* rep = nullptr;       // representative words (bytes)
    // composition (kernels.cu Comp): table comp[a * nS + b] = id(f_a . f_b), u8 if comp_u8 else
    // u16 (nullptr: Lemma-1 replay); rep16[s] = rep(s) in bytes 0..14, |rep(s)| in byte 15 (depth <= 15)
    const void* comp = nullptr;
    uint32_t comp_u8 = 0;
    const uint4* rep16 = nullptr;
    // aux smem image copied after the step table: [comp table if aux_comp][maps32 at aux_maps_off if aux_maps]
    // HOT residency: renumbered window table (u16 device ids, nS x W, padded to 16 B), canonical <-> device
    // id permutations, and the number of rows H kept in smem for this launch
    const uint16_t* Tdev = nullptr;
    const uint16_t* perm = nullptr;    // canonical -> device
    const uint16_t* iperm = nullptr;   // device -> canonical
    uint32_t hotH = 0;
    // FACTORED step (HOT residency): SFA states whose mapping has at most one
    // non-absorbing image g are (family, g); fact_fam / fact_g by canonical id (0xFFFF: not
    // factorable), fact_tab[fam * nD + g] = canonical id, dwin = the DFA window table
    // copied into smem (before the hot rows) as dwin_R copies, lane L using copy L % dwin_R.
    const uint16_t* fact_fam = nullptr;
    const uint16_t* fact_g = nullptr;
    const uint16_t* fact_tab = nullptr;
    const uint16_t* dwin = nullptr;     // smem image of the DFA window table: dwin_R lane-group copies
    uint32_t dwin_bytes = 0;            // (StepDfa, dfa_enc), copied to smem offset 0
    uint32_t dwin_R = 0, dwin_X = 0;
    const uint32_t* aux = nullptr;
    uint32_t aux_bytes = 0, aux_comp = 0, aux_maps = 0, aux_maps_off = 0;
    uint32_t nS = 0, C = 0, nD = 0;
    uint32_t lo = 0, W = 0;             // byte window: columns lo..lo+W-2, column W-1 = every other byte
};

// R lane-group copies of a u16 table (R | 32; lane L uses copy L % R, which
// owns the banks c, c+R, c+2R, ... -- 32/R banks).  Entry (g, column j) of
// copy c lives at j*X + dfa_enc(g, c, R):
//   dfa_enc(g, c, R) = (g / spl) * 128 + 4 * (c + R * ((g % spl) / 2)) + 2 * (g & 1),  spl = 64 / R,
// and X = 128 * ceil(nD / spl) + 4R (R < 32), so consecutive columns of one
// state rotate through the copy's banks (lanes of one copy at the same state
// but on different bytes do not conflict).  R = 32 is a bank-private layout.
__host__ __device__ __forceinline__ uint32_t dfa_enc(uint32_t g, uint32_t c, uint32_t R) {
    const uint32_t spl = 64u / R, k = g % spl;
    return (g / spl) * 128u + 4u * (c + R * (k >> 1)) + 2u * (k & 1u);
}
__host__ __device__ __forceinline__ uint32_t dfa_dec(uint32_t e, uint32_t c, uint32_t R) {
    const uint32_t spl = 64u / R, w = (e & 127u) >> 2;
    return (e >> 7) * spl + 2u * ((w - c) / R) + ((e >> 1) & 1u);
}
__host__ __device__ __forceinline__ uint32_t dfa_X(uint32_t nD, uint32_t R) {
    return 128u * ((nD + 64u / R - 1) / (64u / R)) + (R < 32 ? 4u * R : 0u);  // R = 32: one lane per copy, no skew needed
}

// Residency modes that have a kernel (sfa_residency without AUTO).
enum class Res : int { Private = SFA_RES_SMEM_PRIVATE, Shared = SFA_RES_SMEM_SHARED, Hot = SFA_RES_HOT_L2, Global = SFA_RES_L2 };

// Per-launch scratch owned by the handle.
struct Scratch {
    uint8_t* partials = nullptr;   // per CTA (+1 tail slot): 32 B vector or 4 B id
    uint32_t* ticket = nullptr;    // last-CTA-done counter (self-resetting)
    uint32_t max_ctas = 0;         // slots available in partials (excluding the tail slot)
};

// Single-text scan through the TMA pipeline.  The text [0, n) is cut into
//   head  [0, head)                           < 256 bytes, up to 256-B alignment
//   rows  [head + r*L, head + (r+1)*L), r < nchunks   (the 2-D TMA tensor;
//         L a multiple of 256, so each row's 256-B L2 lines are whole)
//   tail  [tail_start, n)                     < L bytes
// CTA b runs rows [b*rows_per_cta, (b+1)*rows_per_cta).
// Every piece is a chunk of Alg. 5 (any division, Theorem 3).
struct TmaPlan {
    uint64_t head = 0;
    uint64_t L = 0;           // row length, multiple of 16
    uint32_t nchunks = 0;     // rows
    uint32_t ctas = 0;
    uint32_t rows_per_cta = 0;
    uint64_t tail_start = 0;  // head + nchunks * L
};

}  // namespace sfa
