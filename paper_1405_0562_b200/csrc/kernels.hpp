// kernels.hpp -- launch interface of the sm_100a kernels (host side).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "plan.hpp"

namespace sfa {

// q_in (device, nullable): the DFA state the text is run from.  NULL means q0
// (Alg. 5 line 7).  A non-NULL q_in chains slices of one text:
// q_final = f_slice(q_in), the sequential reduction of Alg. 5 (right column,
// PAPER.md:567-573) applied across slices.

struct ScanArgs {
    DevTables t;
    const uint8_t* text;  // base of the scanned range (device): one text, or a batch's texts back to back
    uint64_t n;
    TmaPlan plan;         // the host's plan (dplan == nullptr)
    const TmaPlan* dplan; // batch: the plan k_batch_plan wrote (read after griddepcontrol.wait)
    const void* gmaps;    // batch: its three tensor maps in global memory (load, part_hi, part_lo), else nullptr
    Scratch sc;
    const uint32_t* q_in;
    sfa_result* result;
    uint32_t* map_out;    // optional: f_fin(q) for every DFA state q (nD u32, device)
    uint32_t* row_ids;    // optional: canonical SFA id of every row (plan.nchunks u32, device)
    // batch (SEG kernels): text i = [off[i] - off[0], off[i+1] - off[0]) of the range, or
    // [i * plan.len, (i+1) * plan.len) when off == nullptr
    const uint64_t* off;
    uint64_t count;
    sfa_result* results;
    const uint32_t* err;  // batch error word: == epoch when k_batch_plan found bad offsets
    uint32_t epoch;
    uint64_t* stamps;     // diagnostic builds (-DSFA_STAMPS) only: 8 %globaltimer stamps per CTA
};

struct DirectArgs {
    DevTables t;
    const uint8_t* text;
    uint64_t n;
    uint64_t npieces;
    Scratch sc;
    const uint32_t* q_in;
    sfa_result* result;
    uint32_t* piece_ids;  // optional, npieces entries (device SFA ids)
    uint32_t* map_out;    // optional: f_fin(q) for every DFA state q (nD u32, device)
};

// k_batch_plan: validates the offsets, answers the empty texts and plans the
// batch's TMA scan on the device (no host round trip).
struct BatchPlanArgs {
    const uint8_t* texts;
    const uint64_t* off;
    uint64_t count;
    uint32_t G, R, NB, rowb, row_align;
    TmaPlan* dplan;
    void* gmaps;           // 3 x 128-B tensor maps, rewritten from the template (tensormap.replace)
    uint32_t* err;
    uint32_t epoch;
    sfa_result* results;
    uint32_t eps_accept;   // [eps in L]: the result of an empty text is (q0 = 0, eps_accept)
    uint4* slots;          // scratch: one (min len, max len | bad) per block (>= G)
    uint32_t* ticket;      // scratch: last-block-done counter (self-resetting, starts 0)
};

// Shape of a k_scan_tma launch: K chunks per compute thread, ROWB bytes of
// every row per pipeline stage, nring stages in the smem ring.
struct TmaConfig {
    int K = 1, rowb = 16;
    uint32_t nring = 2, rows_per_cta = 0;
    int promo = 0;        // L2 promotion of the TMA loads (bytes; 0 = none)
    bool staged = false;  // bulk-copy the step's compact table into smem before building it
    uint32_t nb = 4;      // TMA boxes per stage
};

// Shape knobs (sfa_set_tuning); 0 = automatic.  None of them changes a result.
struct Tuning {
    int tma_k = 0, tma_rowb = 0, tma_ring = 0, tma_promo = -1;
    uint32_t hot_rows = 0;
    uint32_t row_align = 0;
    uint32_t direct_piece = 0;
};

uint32_t hot_rows_for(int kind, const DevTables& t, size_t smem_optin, uint32_t cap);
// smem the MIXED DFA window may take: what is left after a 3-deep ring of
// 32-byte stages, the fixed part and 64 SFA hot rows (kernels.cu)
size_t factored_mixed_budget(size_t smem_optin, uint32_t W);
// Host: the PRIVATE layout's lane-independent pair words for R copies (StepPrivate::npairs u32).
void build_private_pairs(const uint16_t* Trange, uint32_t nS, uint32_t W, uint32_t R, uint32_t* pairs);
size_t direct_smem_bytes(Res mode, const DevTables& t);
size_t table_smem_bytes(Res mode, const DevTables& t);   // SIZE_MAX/2 if the layout cannot hold t
uint32_t direct_threads_per_cta();
// false if `mode` cannot run the TMA scan within smem_optin bytes
bool tma_choose(Res mode, const DevTables& t, size_t smem_optin, const Tuning& tu, TmaConfig* out);

// Per-step-policy launchers, specialised in kernels_<step>.cu.
template <class Step>
struct StepLaunch {
    static cudaError_t scan_tma(bool vec, const ScanArgs& a, const TmaConfig& cfg, cudaStream_t s);
    static cudaError_t scan_direct(bool vec, const DirectArgs& a, cudaStream_t s);
    // batch (SEG) scan: host plan (a.dplan == nullptr, maps encoded here) or device plan
    static cudaError_t scan_seg(const ScanArgs& a, const TmaConfig& cfg, unsigned grid, cudaStream_t s);
};

// Sequential reduction over shard mappings (Alg. 5, right column):
// q = q0 = 0; q = maps[r * nD + q] for r = 0..count-1; result = (q, dfinal[q]).
cudaError_t launch_combine_maps(const uint32_t* maps, uint32_t count, uint32_t nD, const uint8_t* dfinal,
                                sfa_result* result, cudaStream_t stream);

// Alg. 3, speculative DFA simulation (kernels_spec.cu).
struct SpecArgs {
    const uint32_t* Td = nullptr;   // nD * W: 4 W delta_d(q, byte of column j), padded to 16 B
    uint32_t nD = 0, W = 0, lo = 0;
    const uint8_t* dfinal = nullptr;
    const uint8_t* text = nullptr;
    uint64_t n = 0, nchunks = 0;
    uint64_t cpb = 0;               // chunks per CTA (a multiple of cpc)
    uint32_t cpc = 0;               // chunks per pass (their |D| chains are the CTA's threads)
    uint32_t gcap = 0;              // maps the smem group buffer holds
    uint32_t tbl_smem = 0;          // bytes of the table in smem (0: read through L1/L2)
    uint32_t ctas = 0;
    uint32_t* cta_maps = nullptr;   // scratch: ctas * nD
    uint32_t* ticket = nullptr;     // scratch: last-CTA-done counter (self-resetting, starts 0)
    uint32_t* chunk_maps = nullptr; // optional: nchunks * nD, T_i[q] (Alg. 3 line 6)
    uint32_t* map_out = nullptr;    // optional: nD, the text's mapping T
    sfa_result* result = nullptr;
};
// Fills the launch shape (chunks, CTAs, smem) of a speculative run of n bytes
// in nchunks chunks (0 = auto) into *out from proto's table fields.
cudaError_t spec_plan(const SpecArgs& proto, int sm_count, size_t smem_optin, uint64_t n, uint64_t nchunks,
                      SpecArgs* out, uint32_t* threads, size_t* smem);
cudaError_t launch_spec(const SpecArgs& a, uint32_t threads, size_t smem, cudaStream_t stream);

// On-the-fly construction (kernels_lazy.cu): chunk runs that stop at unbuilt transitions,
// the gather of the text windows the host builds from, the mapping-vector fold.
struct LazyScanArgs {
    const uint32_t* T = nullptr;      // nS * C: next id | kFactBit, 0xFFFFFFFF = not built
    const uint32_t* fg = nullptr;     // nS: the factored image g_s, 0xFFFFFFFF = not factorable
    const uint16_t* drow = nullptr;   // nD * C: byte offset 2 C delta(q, class) of the next row (factored runs)
    const uint8_t* cls = nullptr;     // 256
    uint32_t C = 0, nD = 0;
    int factor = 0;                   // switch to the DFA at the first factorable state
    const uint8_t* text = nullptr;
    uint64_t n = 0, p = 0;
    uint32_t* state = nullptr;        // p: SFA state (the factorable one once switched)
    uint64_t* pos = nullptr;          // p: next byte
    uint32_t* fd = nullptr;           // p: the DFA state of a factored chunk, 0xFFFFFFFF = not factored
    uint32_t* counts = nullptr;       // 2, zeroed by the caller: chunks stalled, chunks finished unfactored
};
constexpr uint32_t kLazyFactorSmem = 48u << 10;  // the factored run's DFA table lives in smem
cudaError_t lazy_init(uint64_t n, uint64_t p, uint32_t* state, uint64_t* pos, uint32_t* fd, int sm_count,
                      cudaStream_t s);
cudaError_t lazy_scan(const LazyScanArgs& a, cudaStream_t s);
cudaError_t lazy_gather(const uint8_t* text, uint64_t n, uint64_t p, const uint64_t* pos, const uint32_t* idx,
                        uint32_t count, uint32_t K, uint8_t* out, cudaStream_t s);
// f_fin = f_{c_0} . ... . f_{c_{p-1}}, c_g the chunk states (state, fd); absorbing: nD flags
cudaError_t lazy_fold(const uint16_t* maps, const uint32_t* state, const uint32_t* fd, const uint8_t* absorbing,
                      uint64_t p, uint32_t nD, uint16_t* buf, uint16_t* out, int sm_count, cudaStream_t s);
// the same when every chunk is factored, by one lookup per composition (buf: 4 * ceil(p / 1024) u32)
cudaError_t lazy_cfold(const uint16_t* maps, const uint8_t* absorbing, uint32_t nD, const uint32_t* state,
                       const uint32_t* fd, uint64_t p, uint32_t* buf, uint16_t* out, cudaStream_t s);

cudaError_t launch_scan_tma(Res mode, bool vec, const ScanArgs& a, const TmaConfig& cfg, cudaStream_t stream);
cudaError_t launch_scan_direct(Res mode, bool vec, const DirectArgs& a, cudaStream_t stream);
cudaError_t launch_scan_seg(Res mode, const ScanArgs& a, const TmaConfig& cfg, unsigned grid, cudaStream_t stream);
// k_batch_plan (plain launch: it waits for all earlier work of the stream, e.g. the kernel that wrote the offsets)
cudaError_t launch_batch_plan(const BatchPlanArgs& a, const TmaConfig& cfg, int sm_count, cudaStream_t stream);
// n == 0 answers and the identity mapping without a host round trip
cudaError_t launch_fill_result(sfa_result* r, uint32_t q, uint32_t acc, uint32_t* map, uint32_t nD, cudaStream_t stream);
cudaError_t launch_fill_results(sfa_result* r, uint64_t count, uint32_t q, uint32_t acc, cudaStream_t stream);

}  // namespace sfa
