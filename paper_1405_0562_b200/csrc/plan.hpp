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
    const uint32_t* img0 = nullptr;     // nS       f_s(q0) | [f_s(q0) in F_d] << 31 (the accept bit: one load at the end)
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
    uint32_t dwin_u8 = 0;               // 1: 32 bank-private u8 copies (StepDfa8, col8), |D| <= 256
    // MIXED u16 layout (dwin_H > 0, StepDfaMix, mix_enc): the dwin_H most visited DFA states in
    // 32 bank-private copies, every state once more in one shared copy; ranks by visit frequency
    uint32_t dwin_H = 0, dwin_hotb = 0;
    const uint16_t* dwin_rank = nullptr;    // DFA id -> rank
    const uint16_t* dwin_unrank = nullptr;  // rank -> DFA id
    // compact source of a bank-private u16 window (32 u16 copies, or MIXED): per column j and
    // 128-byte line k (dwin_hl lines) one word = the pair of cells of lane 0 with bit 15 of each
    // half set where lane L adds 4L (a private target); then the shared twin words (dwin_tw per
    // column).  The kernels expand it in smem (StepHot::fill) instead of copying the image.
    // Factored composition (kernels_impl.cuh Comp): a chunk value (F, g) = fact_pack(F, g) keeps
    // its form through the folds; (F1, g1) . (F2, g2) = (F1, marked_F2(g1) ? img_F2(g1) : g2).
    // fam_bits[F * fam_w + q / 32] bit q % 32 = q marked in F (every marked q goes to the one
    // absorbing state fam_a0), else fam_img[F * nD + q] = img_F(q) or 0xFFFF (unmarked).
    const uint32_t* fam_bits = nullptr;
    const uint16_t* fam_img = nullptr;
    uint32_t fam_w = 0, fam_a0 = 0, fam_n = 0;  // fam_n: families
    const uint32_t* dwin_cpt = nullptr;
    uint32_t dwin_hl = 0;
    const uint32_t* dwin_twin = nullptr;
    uint32_t dwin_tw = 0;
    const uint32_t* aux = nullptr;
    uint32_t aux_bytes = 0, aux_comp = 0, aux_maps = 0, aux_maps_off = 0;
    uint32_t aux_off = 0;               // dsmem offset of the aux image (= the step table's bytes; set per launch)
    uint32_t aux_fam = 0;               // the aux image is fam_bits (factored handles without an smem table)
    uint32_t nS = 0, C = 0, nD = 0;
    uint32_t lo = 0, W = 0;             // byte window: columns lo..lo+W-2, column W-1 = every other byte
#ifdef SFA_STAMPS
    unsigned long long* diag = nullptr;  // diagnostic builds: event counters (sfa_diag_counters)
#endif
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

// The u8 DFA window layout (|D| <= 256): 32 bank-private byte copies,
// state-major: cell (q, j) of lane L is the byte at q*RB + col8(j) + 4L with
// col8(j) = ((j >> 2) << 7) | (j & 3) and RB = 128 * ceil(W / 4) -- four
// columns share lane L's word in bank L, so every lookup is conflict-free at
// half the bytes of 32 u16 copies.  The cell holds the next DFA id, which is
// also the carried state: one IMAD and one LDS.U8 on the dependency chain,
// the column term computed off it.
__host__ __device__ __forceinline__ uint32_t enc8(uint32_t q, uint32_t) { return q; }
__host__ __device__ __forceinline__ uint32_t dec8(uint32_t e) { return e; }
__host__ __device__ __forceinline__ uint32_t col8(uint32_t j) { return ((j >> 2) << 7) | (j & 3u); }
__host__ __device__ __forceinline__ uint32_t dfa8_RB(uint32_t W) { return 128u * ((W + 3) / 4); }
// The MIXED u16 layout (|D| too large for 32 u16 copies): DFA states ranked by
// visit frequency; ranks r < H (even) are "hot" and every rank has a "twin",
// a lane-independent cell any lane may run in.
// Column j occupies [j*X, (j+1)*X), X = hotb + 128 * ceil(nD / 64):
//   hot  (r, lane L): j*X + mix_hot(r, L),  mix_hot(r, L) = (r >> 1) * 128 + 4L + 2 (r & 1)
//                     (32 bank-private copies: lane L only touches bank L; hotb = 64 H)
//   twin (r):         j*X + mix_twin(r):    a hot state's twin is lane 31's private cell,
//                     mix_hot(r, 31) -- lane 31's copy doubles as the shared copy -- and a
//                     cold state's (r >= H) the u16 at hotb + 2r (one copy for all lanes)
// A hot cell of lane L holds the next state as mix_hot(., L) if it is hot, else
// as its twin; lane 31's cells and the cold cells therefore hold twins only
// (lane-independent).  Every encoding addresses a complete table, so any mix of
// them runs the DFA exactly; a lane running in lane 31's copy is moved back to
// its own every 16 bytes (StepDfaMix::fix: the lane field of the address, one
// LOP3 + compare + select) -- only the bank conflicts depend on where it runs.
__host__ __device__ __forceinline__ uint32_t mix_hot(uint32_t r, uint32_t lane) {
    return (r >> 1) * 128u + 4u * lane + 2u * (r & 1u);
}
__host__ __device__ __forceinline__ uint32_t mix_twin(uint32_t r, uint32_t hotb, uint32_t H) {
    return r < H ? mix_hot(r, 31u) : hotb + 2u * r;
}
__host__ __device__ __forceinline__ uint32_t mix_X(uint32_t nD, uint32_t H) { return 64u * H + 128u * ((nD + 63) / 64); }
__host__ __device__ __forceinline__ uint32_t mix_rank_of(uint32_t e, uint32_t hotb) {
    return e < hotb ? 2u * (e >> 7) + ((e >> 1) & 1u) : (e - hotb) >> 1;
}
// StepDfaMix::fix: a hot state's cell in any lane's copy (its twin included)
// -> the cell of lane L (lane4 = 4L); a cold state's twin unchanged
__host__ __device__ __forceinline__ uint32_t mix_fix(uint32_t e, uint32_t hotb, uint32_t lane4) {
    return e < hotb ? ((e & ~124u) | lane4) : e;
}
// The compact source of a bank-private window (DevTables::dwin_cpt): a pair
// word of lane 0's cells with bit 15 set on private targets -> lane L's word
__host__ __device__ __forceinline__ uint32_t cpt_expand(uint32_t c, uint32_t lane) {
    return (c & 0x7fff7fffu) + ((c >> 15) & 0x00010001u) * (4u * lane);
}
__host__ __device__ __forceinline__ uint32_t cpt_cell(uint32_t enc_lane0, bool private_target) {
    return enc_lane0 | (private_target ? 0x8000u : 0u);
}
// a DFA state in the factored step's encoding (any layout) and back
__device__ __forceinline__ uint32_t dw_enc(const DevTables& t, uint32_t q, uint32_t lane) {
    if (t.dwin_u8) return enc8(q, lane);
    if (t.dwin_H) {
        const uint32_t r = t.dwin_rank[q];
        return r < t.dwin_H ? mix_hot(r, lane) : mix_twin(r, t.dwin_hotb, t.dwin_H);
    }
    return dfa_enc(q, lane % t.dwin_R, t.dwin_R);
}
__device__ __forceinline__ uint32_t dw_dec(const DevTables& t, uint32_t e, uint32_t lane) {
    if (t.dwin_u8) return dec8(e);
    if (t.dwin_H) return t.dwin_unrank[mix_rank_of(e, t.dwin_hotb)];
    return dfa_dec(e, lane % t.dwin_R, t.dwin_R);
}

// Residency modes that have a kernel (sfa_residency without AUTO).
enum class Res : int { Private = SFA_RES_SMEM_PRIVATE, Shared = SFA_RES_SMEM_SHARED, Hot = SFA_RES_HOT_L2, Global = SFA_RES_L2 };

// Per-launch scratch owned by the handle.
struct Scratch {
    uint8_t* partials = nullptr;   // per CTA (+1 tail slot): 32 B vector or 4 B id
    uint32_t* ticket = nullptr;    // last-CTA-done counter (self-resetting)
    uint32_t max_ctas = 0;         // slots available in partials (excluding the tail slot)
};

// The TMA scan's cut of a byte range [0, n) (one text, or a batch's texts
// back to back):
//   head  [0, head)                           < 256 bytes, up to 256-B alignment
//   rows  [head + r*L, head + (r+1)*L), r < nchunks   (the 2-D TMA tensor;
//         L a multiple of 64 and >= 256)
//   tail  [tail_start, n)                     < L bytes
// Every piece is a chunk of Alg. 5 (any division, Theorem 3).
// The rows are split over the CTAs as evenly as possible (the launch lasts as
// long as its busiest CTA): the first m CTAs get rc_hi = ceil(rows / G) rows,
// the others rc_lo = floor(rows / G).  A CTA loads its rc rows per stage as
// rc / bh TMA boxes of bh rows (bh a multiple of 8, the swizzle atom) and one
// last box of rc % bh rows (any height: nothing follows it in the stage).
struct TmaPlan {
    uint64_t n = 0;
    uint64_t head = 0;
    uint64_t L = 0;            // row length
    uint32_t nchunks = 0;      // rows
    uint32_t ctas = 0;         // CTAs that own rows (the launch may have more)
    uint32_t rc_hi = 0, rc_lo = 0, m = 0;
    uint32_t bh = 0;           // full box height; the last box of a CTA is rc % bh rows
    uint64_t tail_start = 0;   // head + nchunks * L
    uint64_t len = 0;          // batch of equal texts: their length (0: offsets / one text)
    __host__ __device__ uint32_t cta_rows(uint32_t b) const { return b < m ? rc_hi : (b < ctas ? rc_lo : 0u); }
    __host__ __device__ uint64_t cta_row0(uint32_t b) const {
        return b < m ? static_cast<uint64_t>(b) * rc_hi : static_cast<uint64_t>(m) * rc_hi + static_cast<uint64_t>(b - m) * rc_lo;
    }
};

// rows (<= G * R) over G CTAs: ceil / floor of rows / G each; full boxes of bh rows.
__host__ __device__ inline void split_rows(uint64_t rows, uint32_t G, uint32_t NB, TmaPlan* p) {
    p->nchunks = static_cast<uint32_t>(rows);
    p->tail_start = p->head + rows * p->L;
    if (rows == 0) return;
    p->rc_lo = static_cast<uint32_t>(rows / G);
    p->m = static_cast<uint32_t>(rows - static_cast<uint64_t>(p->rc_lo) * G);
    p->rc_hi = p->rc_lo + (p->m ? 1u : 0u);
    if (!p->m) p->m = G;  // every CTA rc_hi (= rc_lo) rows
    p->ctas = p->rc_lo ? G : p->m;
    p->bh = 8 * ((p->rc_hi + 8 * NB - 1) / (8 * NB));
}

// The plan of a TMA scan of n bytes starting at device address `addr` on G
// CTAs of at most R rows (NB boxes per stage, rowb bytes per row per stage).
// row_align: 0 = choose (256/128/64 B, the fewest idle compute rows after a
// measured DRAM cost of 64-B rows), else force.  Host and device (the batch
// plan kernel runs it on the GPU).
__host__ __device__ inline void make_plan(uint64_t addr, uint64_t n, uint32_t G, uint32_t R, uint32_t NB, uint32_t rowb,
                                          uint32_t row_align, TmaPlan* p) {
    *p = TmaPlan{};
    p->n = n;
    uint64_t head = (256 - (addr & 255)) & 255;
    if (head > n) head = n;
    const uint64_t body = n - head;
    const uint64_t GR = static_cast<uint64_t>(G) * R;
    uint64_t L = 256;
    double best = -1;
    const uint64_t cand[3] = {256, 128, 64};
    for (int ci = 0; ci < 3; ++ci) {
        if (row_align && ci) break;
        uint64_t al = row_align ? row_align : cand[ci];
        if (al < rowb) al = rowb;
        uint64_t Lc = al * ((body + al * GR - 1) / (al * GR));
        if (Lc < 256) Lc = 256;
        const double used = static_cast<double>(body / Lc) / static_cast<double>(GR);
        const double score = used * (al >= 128 ? 1.0 : 0.977);
        if (score > best + 1e-9) {
            best = score;
            L = Lc;
        }
    }
    p->head = head;
    p->L = L;
    split_rows(body / L, G, NB, p);
}

// Equal texts of `len` bytes back to back (count of them at `addr`): rows of
// L = len / mm bytes, so every text is mm whole rows and no text boundary
// falls inside a row (the batch scan then never takes its byte-by-byte
// boundary path).  mm is the largest divisor of len with count * mm <= G * R
// (the most rows in flight) and L >= 256 a multiple of rowb and 16; needs
// addr % 32 == 0 (each 32-B stage piece one DRAM sector).  false: no such cut
// (use make_plan).
__host__ __device__ inline bool make_plan_uniform(uint64_t addr, uint64_t len, uint64_t count, uint32_t G, uint32_t R,
                                                  uint32_t NB, uint32_t rowb, TmaPlan* p) {
    if (len == 0 || count == 0 || (addr & 31) != 0) return false;
    const uint64_t GR = static_cast<uint64_t>(G) * R;
    if (count > GR) return false;
    uint64_t mm = GR / count;
    if (mm > len / 256) mm = len / 256;
    for (; mm >= 1; --mm) {
        if (len % mm) continue;
        const uint64_t L = len / mm;
        if (L % rowb || L % 16) continue;
        *p = TmaPlan{};
        p->n = len * count;
        p->head = 0;
        p->L = L;
        p->len = len;
        split_rows(count * mm, G, NB, p);
        return true;
    }
    return false;
}

}  // namespace sfa
