// api.cpp -- the C-ABI of include/sfa.h: handle lifecycle, table residency
// (A6), launch planning and the host<->device crossings.  All arithmetic of
// the hot path runs in kernels.cu; this file only plans and launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/sfa.h"
#include "compile.hpp"
#include "kernels.hpp"
#include "lazy.hpp"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* where) {
    return fail(e == cudaErrorMemoryAllocation ? SFA_ERR_OOM : SFA_ERR_CUDA,
                std::string(where) + ": " + cudaGetErrorString(e));
}
#define CU(call)                                                 \
    do {                                                         \
        cudaError_t e_ = (call);                                 \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);      \
    } while (0)

constexpr uint64_t kTmaMin = 4ull << 20;       // below: k_scan_direct
constexpr uint64_t kDirectPiece = 64;          // bytes per thread in k_scan_direct (at least)
constexpr uint64_t kDirectPieceMax = 512;      // ... and at most (texts < kTmaMin)
constexpr uint32_t kMaxSlots = (1u << 16) + 2; // partial slots (CTAs + tail)
constexpr uint64_t kSlice = 64ull << 20;       // sfa_match_host slice
constexpr uint32_t kCompMaxStates = 4096;      // composition table up to |S|^2 = 16M entries
constexpr size_t kAuxMax = 16u << 10;          // comp / maps32 copied into smem up to this size
constexpr uint64_t kDfaMax = 132u << 10;       // FACTORED: the DFA table copies take at most this much smem

template <class T>
cudaError_t upload(T** dst, const T* src, size_t count) {
    *dst = nullptr;
    if (count == 0) return cudaSuccess;
    // padded to 256 B: the kernels bulk-prefetch whole 16-B granules of the tables into L2
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), (count * sizeof(T) + 255) & ~size_t(255));
    if (e != cudaSuccess) return e;
    return cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
}

}  // namespace

// Device state of the on-the-fly construction (sfa_compile_lazy / sfa_match_lazy).
struct LazyDev {
    uint32_t* T = nullptr;   // transition table copy (u32, cap_rows * C)
    uint16_t* maps = nullptr;  // mapping vectors (cap_rows * nD)
    uint32_t* fg = nullptr;    // factored images (cap_rows)
    uint16_t* dfa = nullptr;   // nD * C DFA table (factored runs)
    uint8_t* absorbing = nullptr;  // nD
    uint8_t* cls = nullptr;
    size_t cap_rows = 0, maps_rows = 0;
    uint32_t* state = nullptr;
    uint64_t* pos = nullptr;
    uint32_t* idx = nullptr;
    uint32_t* fd = nullptr;    // p: DFA state of factored chunks
    uint32_t* counts = nullptr;  // 2: chunks stalled / finished unfactored in the last scan
    uint32_t* cbuf = nullptr;  // compact-fold scratch (4 * ceil(cap_p / 1024))
    uint8_t* win = nullptr;
    uint16_t* fold = nullptr;
    uint16_t* fin = nullptr;
    size_t cap_p = 0, cap_win = 0;
    void release() {
        for (void* q : {(void*)T, (void*)maps, (void*)fg, (void*)dfa, (void*)absorbing, (void*)cls, (void*)state,
                        (void*)pos, (void*)idx, (void*)fd, (void*)counts, (void*)cbuf, (void*)win, (void*)fold,
                        (void*)fin})
            if (q) cudaFree(q);
        *this = LazyDev{};
    }
};

struct sfa_handle {
    sfa::Automata A;
    std::unique_ptr<sfa::LazySFA> lazy;  // sfa_compile_lazy handles
    LazyDev ld;
    double lazy_build_s = 0;             // host time spent building states while matching
    // byte window of the range tables (DevTables::lo / W)
    uint32_t lo = 0, W = 1, other = 0;
    int forced = SFA_RES_AUTO;

    std::mutex mu;
    bool uploaded = false;
    int device = -1, sm_count = 0;
    size_t smem_optin = 0;
    // device tables
    uint16_t* dT = nullptr;
    uint8_t* dcls = nullptr;
    uint16_t* dTrange = nullptr;
    uint8_t* dmaps32 = nullptr;
    uint16_t* dmaps16 = nullptr;
    uint32_t* dimg0 = nullptr;
    uint8_t* dfinal = nullptr;
    uint32_t* drep_off = nullptr;
    uint8_t* drep = nullptr;
    void* dcomp = nullptr;                    // composition table (u8 if nS <= 256, else u16)
    uint32_t* dpairs = nullptr;               // PRIVATE: pair words (device.cuh StepPrivate)
    uint32_t priv_R = 0;                      // PRIVATE: lane-group copies (0: no PRIVATE layout)
    uint16_t* dTdev = nullptr;                // HOT: window table renumbered by visit frequency
    uint16_t* dperm = nullptr;                // HOT: canonical -> device id
    uint16_t* diperm = nullptr;               // HOT: device -> canonical id
    uint16_t *dfam = nullptr, *dfg = nullptr, *dftab = nullptr, *ddwin = nullptr;  // FACTORED step tables
    uint32_t dwin_bytes = 0, nfam = 0, dwin_R = 0, dwin_X = 0, dwin_u8 = 0;
    uint32_t dwin_H = 0, dwin_hotb = 0;                     // MIXED layout (plan.hpp mix_*)
    uint16_t *ddrank = nullptr, *ddunrank = nullptr;        // MIXED: DFA id <-> rank
    uint32_t *ddcpt = nullptr, *ddtwin = nullptr;           // compact source of a bank-private window
    uint32_t* dfam_bits = nullptr;                          // factored values: marked sets (one absorbing state)
    uint16_t* dfam_img = nullptr;                           //   or absorbing images per family
    uint32_t fam_w = 0, fam_a0 = 0;
    uint32_t dwin_hl = 0, dwin_tw = 0;
    sfa_tuning_t tuning{};                    // shape knobs (sfa_set_tuning); zero = automatic
    // The last single-text TMA launch's decisions (residency, tables, shape,
    // plan) for the same text and size: a repeated call skips them (host cost
    // per call).  Any setter that can change them bumps cfg_epoch.
    uint64_t cfg_epoch = 1;
    struct LaunchCache {
        uint64_t epoch = 0;
        const uint8_t* text = nullptr;
        uint64_t n = 0;
        sfa::Res mode{};
        sfa::DevTables t{};
        sfa::TmaConfig cfg{};
        sfa::TmaPlan plan{};
    } lcache;
    bool factor_on() const { return tuning.no_factor == 0; }
    sfa::Tuning ktune() const {
        sfa::Tuning k;
        k.tma_k = tuning.tma_k;
        k.tma_rowb = tuning.tma_rowb;
        k.tma_ring = tuning.tma_ring;
        k.tma_promo = tuning.tma_promo;
        k.hot_rows = tuning.hot_rows;
        k.row_align = tuning.row_align;
        k.direct_piece = tuning.direct_piece;
        return k;
    }
    uint32_t* dspecT = nullptr;               // Alg. 3 baseline: DFA window table (kernels_spec.cu)
    uint32_t* spec_maps = nullptr;            // Alg. 3: per-CTA maps (spec_cap entries)
    uint32_t* spec_ticket = nullptr;
    size_t spec_cap = 0;
    uint4* drep16 = nullptr;                  // rep(s) slots (depth <= 15)
    uint32_t* daux[2] = {nullptr, nullptr};   // aux smem images: [0] comp (TABLE), [1] maps32 (VEC)
    uint32_t aux_bytes[2] = {0, 0};
    int compose = SFA_COMPOSE_AUTO;
    uint64_t dev_bytes = 0;
    // scratch
    uint8_t* partials = nullptr;
    uint32_t* ticket = nullptr;
    sfa_result* dres = nullptr;       // 2 results (single-text matches and the slice ring)
    sfa_result* hres = nullptr;       // pinned
#ifdef SFA_STAMPS
    uint64_t* dstamps = nullptr;      // diagnostic builds: 16 stamps per CTA of the last TMA scan
#endif
    sfa::TmaPlan* dplan = nullptr;    // batch: the plan k_batch_plan writes
    void* gmaps = nullptr;            // batch: 3 tensor maps rewritten on the device
    uint32_t* berr = nullptr;         // batch: error word (== epoch: bad offsets)
    uint32_t epoch = 0;
    uint8_t* stage[2] = {nullptr, nullptr};   // sfa_match_host / sfa_match_batch_host staging
    size_t stage_cap = 0;
    uint64_t* soff[2] = {nullptr, nullptr};   // sfa_match_batch_host: offsets of the staged slices
    size_t soff_cap = 0;
    sfa_result* bres = nullptr;               // sfa_match_batch_host: device results
    size_t bres_cap = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
    cudaEvent_t ev_done = nullptr;    // orders uses of the shared scratch across streams

    ~sfa_handle() { release_device(); }

    // Frees every device table and scratch buffer (after the device work that
    // used them); the next device call uploads again.
    void release_device() {
        ++cfg_epoch;
        if (!uploaded) return;
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        cudaDeviceSynchronize();
        for (void** pp : {(void**)&dT, (void**)&dcls, (void**)&dTrange, (void**)&dmaps32, (void**)&dmaps16, (void**)&dimg0,
                          (void**)&dfinal, (void**)&drep_off, (void**)&drep, (void**)&partials, (void**)&ticket, (void**)&dres,
                          (void**)&dplan, (void**)&gmaps, (void**)&berr, (void**)&stage[0], (void**)&stage[1], (void**)&soff[0], (void**)&soff[1], (void**)&bres,
                          (void**)&dcomp, (void**)&dpairs, (void**)&dTdev, (void**)&dfam, (void**)&dfg, (void**)&dftab,
                          (void**)&ddwin, (void**)&ddrank, (void**)&ddunrank, (void**)&ddcpt, (void**)&ddtwin, (void**)&dfam_bits, (void**)&dfam_img, (void**)&dperm, (void**)&diperm, (void**)&drep16, (void**)&dspecT,
                          (void**)&spec_maps, (void**)&spec_ticket, (void**)&daux[0], (void**)&daux[1]}) {
            if (*pp) cudaFree(*pp);
            *pp = nullptr;
        }
        if (hres) cudaFreeHost(hres);
        hres = nullptr;
        ld.release();
        for (int i = 0; i < 2; ++i) {
            if (ev_copied[i]) cudaEventDestroy(ev_copied[i]);
            if (ev_used[i]) cudaEventDestroy(ev_used[i]);
            ev_copied[i] = ev_used[i] = nullptr;
        }
        if (ev_done) cudaEventDestroy(ev_done);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        ev_done = nullptr;
        copy_stream = nullptr;
        priv_R = dwin_bytes = nfam = dwin_R = dwin_X = dwin_u8 = dwin_H = dwin_hotb = dwin_hl = dwin_tw = fam_w = fam_a0 = 0;
        aux_bytes[0] = aux_bytes[1] = 0;
        spec_cap = 0;
        stage_cap = soff_cap = bres_cap = 0;
        dev_bytes = 0;
        has_last = false;
        uploaded = false;
        cudaSetDevice(prev);
    }

    bool has_comp() const { return A.nS <= kCompMaxStates; }
    // bytes of the families' marked sets as an smem aux image (0: too large, or none)
    uint32_t fam_aux_bytes() const {
        const uint64_t b = (static_cast<uint64_t>(nfam) * fam_w * 4 + 15) & ~uint64_t(15);
        return b <= 8192 ? static_cast<uint32_t>(b) : 0u;
    }
    // mapping vectors (VEC composition, sfa_match_map, q_in chaining): D-SFA only
    bool can_vec() const { return !A.nsfa && A.nD <= 32; }
    // effective composition mode
    int compose_mode() const {
        if (compose != SFA_COMPOSE_AUTO) return compose;
        if (has_comp()) return SFA_COMPOSE_TABLE;
        return can_vec() ? SFA_COMPOSE_VEC : SFA_COMPOSE_REPLAY;
    }
    bool vec() const { return compose_mode() == SFA_COMPOSE_VEC; }

    // device tables as seen by a kernel (aux = the composition mode's smem image)
    // id_only: the batch (SEG) kernels compose SFA ids (TABLE or REPLAY), never vectors
    sfa::DevTables tables(sfa::Res mode = sfa::Res::Global, int kind = 0, bool id_only = false) const {
        sfa::DevTables t;
        int cm = compose_mode();
        if (id_only && cm == SFA_COMPOSE_VEC) cm = has_comp() ? SFA_COMPOSE_TABLE : SFA_COMPOSE_REPLAY;
        t.comp = cm == SFA_COMPOSE_TABLE ? dcomp : nullptr;
        t.comp_u8 = A.nS <= 256 ? 1u : 0u;
        t.rep16 = drep16;
        if (cm == SFA_COMPOSE_TABLE && daux[0]) {
            t.aux = daux[0];
            t.aux_bytes = aux_bytes[0];
            t.aux_comp = 1;
        } else if (cm == SFA_COMPOSE_VEC && daux[1]) {
            t.aux = daux[1];
            t.aux_bytes = aux_bytes[1];
            t.aux_maps = 1;
            t.aux_maps_off = 0;
        }
        t.T = dT;
        t.cls = dcls;
        t.Trange = dTrange;
        t.maps32 = dmaps32;
        t.maps16 = dmaps16;
        t.img0 = dimg0;
        t.dfinal = dfinal;
        t.rep_off = drep_off;
        t.rep = drep;
        t.nS = A.nS;
        t.C = A.C;
        t.nD = A.nD;
        t.lo = lo;
        t.W = W;
        t.pairs = dpairs;
        t.priv_R = priv_R;
        t.Tdev = dTdev;
        t.perm = dperm;
        t.iperm = diperm;
        if (mode == sfa::Res::Hot && dfam && factor_on()) {
            t.fact_fam = dfam;
            t.fact_g = dfg;
            t.fact_tab = dftab;
            t.dwin = ddwin;
            t.dwin_bytes = dwin_bytes;
            t.dwin_R = dwin_R;
            t.dwin_X = dwin_X;
            t.dwin_u8 = dwin_u8;
            t.dwin_H = dwin_H;
            t.dwin_hotb = dwin_hotb;
            t.dwin_rank = ddrank;
            t.dwin_unrank = ddunrank;
            t.dwin_cpt = ddcpt;
            if (tuning.fact_fold != 2) {  // tuning fact_fold = 2: the folds use canonical SFA ids
                t.fam_bits = dfam_bits;
                t.fam_img = dfam_img;
            }
            if (!t.aux && t.fam_bits && fam_aux_bytes() && tuning.fact_fold == 0) {  // the marked sets in smem for the folds
                t.aux = dfam_bits;
                t.aux_bytes = fam_aux_bytes();
                t.aux_fam = 1;
            }
            t.fam_w = fam_w;
            t.fam_n = nfam;
            t.fam_a0 = fam_a0;
            t.dwin_hl = dwin_hl;
            t.dwin_twin = ddtwin;
            t.dwin_tw = dwin_tw;
        }
        t.hotH = (mode == sfa::Res::Hot && dTdev) ? sfa::hot_rows_for(kind, t, smem_optin, tuning.hot_rows) : 0;
        return t;
    }

    // HOT residency: rank SFA states by visit frequency.  Static part: a
    // random walk drawing every window column (byte class of the table)
    // uniformly, restarting from f_I every 2048 steps (chunks start from f_I,
    // Alg. 5 line 2).  Profile part (sample != NULL): the SFA run over
    // 2048-byte chunks of a sample of real text, weighted 16x.  Device ids =
    // ranks, so the hot rows are a prefix of the renumbered table.
    void hot_ranking(std::vector<uint32_t>& perm, const uint8_t* sample, size_t ns) const {
        const uint32_t nS = A.nS;
        std::vector<uint64_t> cnt(nS, 0);
        std::vector<uint32_t> colcls(W);
        for (uint32_t j = 0; j + 1 < W; ++j) colcls[j] = A.cls[lo + j];
        colcls[W - 1] = other;
        uint64_t x = 0x9e3779b97f4a7c15ull;
        for (int walk = 0; walk < 2048; ++walk) {
            uint32_t st = 0;
            ++cnt[st];
            for (int k = 0; k < 2048; ++k) {
                x ^= x << 13;
                x ^= x >> 7;
                x ^= x << 17;
                st = A.T[static_cast<size_t>(st) * A.C + colcls[(x >> 11) % W]];
                ++cnt[st];
            }
        }
        for (size_t c0 = 0; sample && c0 < ns; c0 += 2048) {
            uint32_t st = 0;
            for (size_t i = c0; i < std::min(ns, c0 + 2048); ++i) {
                st = A.T[static_cast<size_t>(st) * A.C + A.cls[sample[i]]];
                cnt[st] += 16;
            }
        }
        std::vector<uint32_t> order(nS);
        for (uint32_t i = 0; i < nS; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cnt[a] > cnt[b]; });
        perm.assign(nS, 0);
        for (uint32_t r = 0; r < nS; ++r) perm[order[r]] = r;
    }

    // DFA states by visit frequency (the MIXED DFA window layout): the same
    // static walk over the window columns as hot_ranking, on the minimal DFA
    // from q0 (a factored warp runs the DFA once its chunks have synchronised).
    // order[r] = the DFA id of rank r; cnt = visits per DFA id.
    void dfa_ranking(std::vector<uint32_t>& order, std::vector<uint64_t>& cnt) const {
        const uint32_t nD = A.nD;
        cnt.assign(nD, 0);
        const uint32_t ob = lo + W - 1 < 256 ? lo + W - 1 : lo - 1;  // a byte of column W-1
        // The walk stays out of absorbing DFA states while some column avoids
        // them: a uniform walk over r_n's digits is dead after a few steps and
        // would call every other state cold, while an accepted text visits them
        // all.  The absorbing states themselves rank first (a text that reaches
        // one keeps its rows there -- cfg5's texts after their planted word --
        // and a lane left in the shared copy conflicts on every byte).
        std::vector<uint8_t> sink(nD, 1);
        for (uint32_t q = 0; q < nD; ++q)
            for (uint32_t b = 0; b < 256 && sink[q]; ++b)
                if (A.dfa[static_cast<size_t>(q) * 256 + b] != q) sink[q] = 0;
        uint64_t x = 0x2545f4914f6cdd1dull;
        auto next = [&](uint32_t q, uint32_t j) { return A.dfa[static_cast<size_t>(q) * 256 + (j + 1 < W ? lo + j : ob)]; };
        auto rnd = [&]() {
            x ^= x << 13;
            x ^= x >> 7;
            x ^= x << 17;
            return static_cast<uint32_t>((x >> 11) % W);
        };
        for (int walk = 0; walk < 1024; ++walk) {
            uint32_t q = 0;
            for (int k = 0; k < 2048; ++k) {
                uint32_t nx = next(q, rnd());
                for (int tries = 0; tries < 4 && sink[nx] && nx != q; ++tries) nx = next(q, rnd());
                if (sink[nx] && nx != q)
                    for (uint32_t j = 0; j < W; ++j)
                        if (!sink[next(q, j)]) {
                            nx = next(q, j);
                            break;
                        }
                q = nx;
                ++cnt[q];
                if (sink[q]) break;
            }
        }
        uint64_t top = 0;
        for (uint32_t q = 0; q < nD; ++q) top = std::max(top, cnt[q]);
        for (uint32_t q = 0; q < nD; ++q)
            if (sink[q]) cnt[q] = top + 1;
        order.resize(nD);
        for (uint32_t i = 0; i < nD; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cnt[a] > cnt[b]; });
    }

    // (Re)builds the HOT tables from a ranking and writes them to the device
    // buffers (allocated on first use).  Synchronous.
    int upload_hot(const uint8_t* sample, size_t ns) {
        ++cfg_epoch;
        const uint32_t nS = A.nS;
        std::vector<uint32_t> perm;
        hot_ranking(perm, sample, ns);
        std::vector<uint16_t> p16(nS), ip16(nS), Td((static_cast<size_t>(nS) * W + 7) & ~size_t(7), 0);
        for (uint32_t st = 0; st < nS; ++st) {
            p16[st] = static_cast<uint16_t>(perm[st]);
            ip16[perm[st]] = static_cast<uint16_t>(st);
        }
        for (uint32_t st = 0; st < nS; ++st)
            for (uint32_t j = 0; j < W; ++j) {
                const uint32_t c = j + 1 < W ? A.cls[lo + j] : other;
                Td[static_cast<size_t>(perm[st]) * W + j] = p16[A.T[static_cast<size_t>(st) * A.C + c]];
            }
        if (!dTdev) {
            CU(cudaMalloc(&dTdev, Td.size() * 2));
            CU(cudaMalloc(&dperm, nS * 2));
            CU(cudaMalloc(&diperm, nS * 2));
        }
        CU(cudaMemcpy(dTdev, Td.data(), Td.size() * 2, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(dperm, p16.data(), nS * 2, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(diperm, ip16.data(), nS * 2, cudaMemcpyHostToDevice));
        return SFA_OK;
    }

    // FACTORED step tables.  A DFA state a is absorbing if
    // delta(a, b) = a for every byte.  An SFA state s is factorable if all q
    // with f_s(q) not absorbing share one image g_s; its family is f_s with
    // those q marked.  fact_tab[family][g] = the SFA state (family, g).  Built
    // when most states are factorable and the tables are small.
    int upload_fact() {
        const uint32_t nS = A.nS, nD = A.nD;
        if (static_cast<uint64_t>(nD) * W * 2 > 32768) return SFA_OK;
        std::vector<uint8_t> absorbing(nD, 1);
        for (uint32_t q = 0; q < nD; ++q)
            for (int b = 0; b < 256 && absorbing[q]; ++b)
                if (A.dfa[static_cast<size_t>(q) * 256 + b] != q) absorbing[q] = 0;
        uint32_t abs0 = UINT32_MAX;
        for (uint32_t q = 0; q < nD; ++q)
            if (absorbing[q]) {
                abs0 = q;
                break;
            }
        std::vector<uint16_t> fam(nS, 0xffff), g(nS, 0);
        std::map<std::vector<uint16_t>, uint32_t> fams;
        uint32_t nfact = 0;
        for (uint32_t st = 0; st < nS; ++st) {
            const uint32_t* m = &A.maps[static_cast<size_t>(st) * nD];
            uint32_t gg = UINT32_MAX;
            bool ok = true;
            std::vector<uint16_t> key(nD);
            for (uint32_t q = 0; q < nD && ok; ++q) {
                if (absorbing[m[q]]) {
                    key[q] = static_cast<uint16_t>(m[q]);
                } else {
                    key[q] = 0xffff;
                    if (gg == UINT32_MAX) gg = m[q];
                    else if (gg != m[q]) ok = false;
                }
            }
            if (!ok) continue;
            if (gg == UINT32_MAX) {  // frozen: every image absorbing
                if (abs0 == UINT32_MAX) continue;
                gg = abs0;
            }
            auto it = fams.emplace(key, static_cast<uint32_t>(fams.size())).first;
            fam[st] = static_cast<uint16_t>(it->second);
            g[st] = static_cast<uint16_t>(gg);
            ++nfact;
        }
        if (nfact * 2 < nS || fams.size() >= 0xffff || static_cast<uint64_t>(fams.size()) * nD > (8u << 20)) return SFA_OK;
        std::vector<uint16_t> tab(fams.size() * static_cast<size_t>(nD), 0xffff);
        for (uint32_t st = 0; st < nS; ++st)
            if (fam[st] != 0xffff) tab[static_cast<size_t>(fam[st]) * nD + g[st]] = static_cast<uint16_t>(st);
        // g reaching an absorbing state a freezes the mapping: (family, a) is the
        // frozen state whose mapping is the family's with the marked q sent to a
        for (const auto& kv : fams) {
            bool marked = false;
            for (uint16_t x : kv.first) marked |= x == 0xffff;
            if (!marked) continue;
            for (uint32_t a = 0; a < nD; ++a) {
                if (!absorbing[a]) continue;
                std::vector<uint16_t> k2(kv.first);
                for (uint16_t& x : k2)
                    if (x == 0xffff) x = static_cast<uint16_t>(a);
                auto f2 = fams.find(k2);
                if (f2 != fams.end())
                    tab[static_cast<size_t>(kv.second) * nD + a] = tab[static_cast<size_t>(f2->second) * nD + abs0];
            }
        }
        // factored chunk values (DevTables::fam_bits / fam_img): a family's marked
        // states and their absorbing images, read by the folds (F < 2^14)
        if (fams.size() < (1u << 14)) {
            uint32_t nabs = 0;
            for (uint32_t q = 0; q < nD; ++q) nabs += absorbing[q];
            if (nabs <= 1) {
                const uint32_t w = (nD + 31) / 32;
                std::vector<uint32_t> bits(fams.size() * static_cast<size_t>(w), 0);
                for (const auto& kv : fams)
                    for (uint32_t q = 0; q < nD; ++q)
                        if (kv.first[q] != 0xffff) bits[static_cast<size_t>(kv.second) * w + q / 32] |= 1u << (q % 32);
                CU(upload(&dfam_bits, bits.data(), bits.size()));
                fam_w = w;
                fam_a0 = nabs ? abs0 : 0u;
            } else {
                std::vector<uint16_t> img(fams.size() * static_cast<size_t>(nD));
                for (const auto& kv : fams)
                    std::memcpy(&img[static_cast<size_t>(kv.second) * nD], kv.first.data(), nD * 2);
                CU(upload(&dfam_img, img.data(), img.size()));
            }
        }
        // compact DFA window table (next state ids); in smem as R lane-group copies,
        // R the largest of 32, 16, ..., 1 whose copies take <= 80 KB (StepDfa)
        const uint32_t ob = lo + W - 1 < 256 ? lo + W - 1 : lo - 1;  // a byte outside the window (class `other`)
        std::vector<uint16_t> dw((static_cast<size_t>(nD) * W + 7) & ~size_t(7), 0);
        for (uint32_t q = 0; q < nD; ++q)
            for (uint32_t j = 0; j < W; ++j) {
                const uint32_t b = j + 1 < W ? lo + j : ob;
                dw[static_cast<size_t>(q) * W + j] = static_cast<uint16_t>(A.dfa[static_cast<size_t>(q) * 256 + b]);
            }
        // Layout: the largest R of 32, 16, ... lane-group u16 copies that fits
        // (cfg4: R = 32, conflict-free, 4 instr/byte; cfg3/5: R = 16, 2-way
        // conflicts).  Tuning dfa_u8 = 1 takes 32 bank-private u8 copies instead
        // when |D| <= 256 and 32 u16 copies do not fit (plan.hpp col8):
        // conflict-free, 2 more ALU ops per byte off the dependency chain.
        uint32_t R = 32, X = 0, H = 0;
        const uint32_t Rmax = tuning.dfa_copies ? tuning.dfa_copies : 32u;  // tuning: cap R
        const bool u16_32 = Rmax >= 32 && static_cast<uint64_t>(sfa::dfa_X(nD, 32)) * W <= kDfaMax;
        const bool u8_fits = !u16_32 && Rmax >= 32 && nD <= 256 && static_cast<uint64_t>(nD) * sfa::dfa8_RB(W) <= kDfaMax;
        bool u8_32 = tuning.dfa_u8 && u8_fits;
        // MIXED candidate (plan.hpp mix_*): DFA states ranked by visit frequency,
        // the largest even H whose 32 private copies + the shared copy fit
        std::vector<uint32_t> order, rank;
        uint32_t Hm = 0;
        double cold = 1.0;  // walk visits outside the H hot states
        if (!u16_32 && !u8_32 && tuning.dfa_layout != 1 && !tuning.dfa_copies) {
            std::vector<uint64_t> cnt;
            dfa_ranking(order, cnt);
            const uint32_t hcap = tuning.dfa_hot ? std::max(2u, tuning.dfa_hot & ~1u) : nD;
            // (less the families' marked sets, which sit in smem as the aux image)
            const uint64_t fb = (static_cast<uint64_t>(fams.size()) * fam_w * 4 + 15) & ~uint64_t(15);
            const uint64_t budget = sfa::factored_mixed_budget(smem_optin, W) - (dfam_bits && fb <= 8192 ? fb : 0);
            for (uint32_t h = 2; h < nD && h <= hcap; h += 2) {
                const uint64_t xm = sfa::mix_X(nD, h);
                if (xm * W > budget || xm > 65535u) break;
                Hm = h;
            }
            if (Hm) {
                uint64_t tot = 0, hot = 0;
                for (uint32_t r = 0; r < nD; ++r) {
                    tot += cnt[order[r]];
                    if (r < Hm) hot += cnt[order[r]];
                }
                cold = tot ? 1.0 - static_cast<double>(hot) / static_cast<double>(tot) : 1.0;
            }
        }
        if (!u8_32) {
            for (; R >= 1; R /= 2) {
                X = sfa::dfa_X(nD, R);
                if (R <= Rmax && static_cast<uint64_t>(X) * W <= (kDfaMax) && X <= 65535u) break;
            }
            // smem wavefronts per warp lookup: R lane-group copies ~ 1 + log2(32/R)
            // (two lanes per copy at R = 16: nearly always a 2-way conflict); MIXED
            // ~ 1 + P(some lane of the warp runs in the shared copy), a lane staying
            // there ~8.5 bytes (to the next 16-byte fix) per entry
            if (Hm) {
                const double est_u = R >= 1 ? 1.0 + std::log2(32.0 / R) : 1e9;
                const double est_m = 1.0 + std::min(1.0, 1.0 - std::pow(1.0 - std::min(1.0, 8.5 * cold), 32.0));
                if (tuning.dfa_layout == 2 || est_m < est_u) {
                    H = Hm;
                    R = 32;
                    X = sfa::mix_X(nD, H);
                }
            }
            // AUTO: neither 32 u16 copies nor a MIXED window with few visits outside
            // its hot states (r_100, r_127: an accepted text visits every DFA state
            // equally) -- the conflict-free u8 copies beat R = 16 lane-group copies
            // (measured: r_100 3.15 vs 3.00 TB/s, r_127 3.30 vs 3.14; MIXED 2.33 / 2.61)
            if (!H && R < 32 && u8_fits && tuning.dfa_layout == 0 && !tuning.dfa_copies) u8_32 = true;
            if (R == 0 && !u8_32) return SFA_OK;
        }
        if (u8_32) {
            R = 32;
            X = sfa::dfa8_RB(W);  // bytes per state row
        }
        dwin_R = R;
        dwin_X = X;
        dwin_u8 = u8_32 ? 1u : 0u;
        dwin_H = H;
        dwin_hotb = 64u * H;
        CU(upload(&dfam, fam.data(), fam.size()));
        CU(upload(&dfg, g.data(), g.size()));
        CU(upload(&dftab, tab.data(), tab.size()));
        dwin_bytes = ((u8_32 ? X * nD : X * W) + 15) & ~15u;
        std::vector<uint8_t> img(dwin_bytes, 0);
        auto put16 = [&](size_t at, uint32_t v) {
            const uint16_t v16 = static_cast<uint16_t>(v);
            std::memcpy(&img[at], &v16, 2);
        };
        if (H) {  // MIXED: ranks; hot cells per lane, twin cells shared (plan.hpp)
            rank.assign(nD, 0);
            for (uint32_t r = 0; r < nD; ++r) rank[order[r]] = r;
            const uint32_t hotb = dwin_hotb;
            for (uint32_t j = 0; j < W; ++j)
                for (uint32_t r = 0; r < nD; ++r) {
                    const uint32_t nr = rank[dw[static_cast<size_t>(order[r]) * W + j]];
                    put16(static_cast<size_t>(j) * X + sfa::mix_twin(r, hotb, H), sfa::mix_twin(nr, hotb, H));
                    if (r < H)
                        for (uint32_t L = 0; L < 32; ++L)
                            put16(static_cast<size_t>(j) * X + sfa::mix_hot(r, L),
                                  nr < H ? sfa::mix_hot(nr, L) : sfa::mix_twin(nr, hotb, H));
                }
            std::vector<uint16_t> rk(nD), ur(nD);
            for (uint32_t q = 0; q < nD; ++q) {
                rk[q] = static_cast<uint16_t>(rank[q]);
                ur[rank[q]] = static_cast<uint16_t>(q);
            }
            CU(upload(&ddrank, rk.data(), rk.size()));
            CU(upload(&ddunrank, ur.data(), ur.size()));
        } else {
            for (uint32_t j = 0; j < W; ++j)
                for (uint32_t q = 0; q < nD; ++q) {
                    const uint32_t nq = dw[static_cast<size_t>(q) * W + j];
                    for (uint32_t c = 0; c < R; ++c) {
                        if (u8_32) img[q * X + sfa::col8(j) + 4 * c] = static_cast<uint8_t>(nq);
                        else put16(j * X + sfa::dfa_enc(q, c, R), sfa::dfa_enc(nq, c, R));
                    }
                }
        }
        CU(upload(reinterpret_cast<uint8_t**>(&ddwin), img.data(), img.size()));
        // compact source of a bank-private window (32 u16 copies or MIXED; the
        // kernels expand it in smem): per (column, 128-B line) the pair word of
        // lane 0 with bit 15 set on private targets (values < 32768), then the twin words
        if (!u8_32 && R == 32 && X <= 32768u) {
            const uint32_t hl = H ? H / 2 : X / 128u, hotb = dwin_hotb;
            std::vector<uint32_t> cpt(static_cast<size_t>(W) * hl, 0);
            auto cell = [&](uint32_t j, uint32_t r) -> uint32_t {  // lane-0 value of rank/state r, flagged
                if (r >= (H ? H : nD)) return 0u;
                const uint32_t q = H ? order[r] : r;
                const uint32_t nq = dw[static_cast<size_t>(q) * W + j];
                const uint32_t nr = H ? rank[nq] : nq;
                if (H && nr >= H) return sfa::cpt_cell(sfa::mix_twin(nr, hotb, H), false);
                return sfa::cpt_cell(sfa::mix_hot(nr, 0), true);
            };
            for (uint32_t j = 0; j < W; ++j)
                for (uint32_t k = 0; k < hl; ++k) cpt[static_cast<size_t>(j) * hl + k] = cell(j, 2 * k) | (cell(j, 2 * k + 1) << 16);
            CU(upload(&ddcpt, cpt.data(), cpt.size()));
            dwin_hl = hl;
            if (H) {
                const uint32_t tw = (X - hotb) / 4;
                std::vector<uint32_t> twin(static_cast<size_t>(W) * tw);
                for (uint32_t j = 0; j < W; ++j) std::memcpy(&twin[static_cast<size_t>(j) * tw], &img[static_cast<size_t>(j) * X + hotb], tw * 4);
                CU(upload(&ddtwin, twin.data(), twin.size()));
                dwin_tw = tw;
            }
        }
        nfam = static_cast<uint32_t>(fams.size());
        dev_bytes += fam.size() * 4 + tab.size() * 2 + dw.size() * 2;
        return SFA_OK;
    }

    // Profile-guided HOT ranking from (a prefix of) a device text
    // (sfa_tune_residency only: a match never blocks on it).  Waits for all
    // earlier work of the handle (the tables are rewritten in place).  Results
    // never depend on the ranking.
    int tune_hot(const uint8_t* d_text, size_t n, cudaStream_t stream) {
        const size_t ns = std::min<size_t>(n, 8u << 20);
        std::vector<uint8_t> sample(ns);
        if (has_last) CU(cudaStreamSynchronize(last_stream));
        CU(cudaMemcpyAsync(sample.data(), d_text, ns, cudaMemcpyDeviceToHost, stream));
        CU(cudaStreamSynchronize(stream));
        return upload_hot(sample.data(), ns);
    }

    // Device state for the DFA-only calls of an on-the-fly handle (Alg. 3).
    int ensure_dfa_only() {
        if (!uploaded) {
            CU(cudaGetDevice(&device));
            int v = 0;
            CU(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
            sm_count = v;
            uploaded = true;
        }
        if (!smem_optin) {
            int v = 0;
            CU(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
            smem_optin = static_cast<size_t>(v);
        }
        if (!dfinal) CU(upload(&dfinal, A.dfa_final.data(), A.dfa_final.size()));
        return SFA_OK;
    }

    // Lazy upload: sfa_compile works without a GPU (host tests); the first
    // device call uploads to the then-current device.
    int ensure_uploaded() {
        if (uploaded) return SFA_OK;
        CU(cudaGetDevice(&device));
        int v = 0;
        CU(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
        sm_count = v;
        CU(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        smem_optin = static_cast<size_t>(v);
        uploaded = true;  // from here on the destructor frees what was allocated

        const uint32_t nS = A.nS, C = A.C, nD = A.nD;
        std::vector<uint16_t> T16(static_cast<size_t>(nS) * C), R16(static_cast<size_t>(nS) * W);
        for (size_t i = 0; i < T16.size(); ++i) T16[i] = static_cast<uint16_t>(A.T[i]);
        for (uint32_t s = 0; s < nS; ++s) {
            for (uint32_t j = 0; j + 1 < W; ++j) R16[static_cast<size_t>(s) * W + j] = T16[static_cast<size_t>(s) * C + A.cls[lo + j]];
            R16[static_cast<size_t>(s) * W + W - 1] = T16[static_cast<size_t>(s) * C + other];
        }
        CU(upload(&dT, T16.data(), T16.size()));
        {  // PRIVATE: R lane-group copies, R the largest of 32, 16, 8 whose table
           // leaves room for a 3-deep ring of 32-byte stages (else <= 200 KB)
            const uint32_t Rcap = tuning.private_copies ? tuning.private_copies : 32u;  // tuning: cap R
            uint32_t R = 0;
            for (int pass = 0; pass < 2 && !R; ++pass)
                for (uint32_t r = 32; r >= 8; r /= 2) {
                    const uint64_t X = sfa::dfa_X(nS, r);
                    if (r > Rcap || X > 65535u) continue;
                    if (X * W <= (pass == 0 ? (112u << 10) : (200u << 10))) {
                        R = r;
                        break;
                    }
                }
            if (R) {
                const uint32_t spl = 64u / R, nl = (nS + spl - 1) / spl;
                std::vector<uint32_t> pw(static_cast<size_t>(W) * nl * (32u / R));
                sfa::build_private_pairs(R16.data(), nS, W, R, pw.data());
                pw.resize((pw.size() + 3) & ~size_t(3), 0);
                CU(upload(&dpairs, pw.data(), pw.size()));
                priv_R = R;
            }
        }
        {  // padded to 16 bytes: the TMA kernel bulk-copies it
            std::vector<uint16_t> padded(R16);
            padded.resize((padded.size() + 7) & ~size_t(7), 0);
            CU(upload(&dTrange, padded.data(), padded.size()));
        }
        CU(upload(&dcls, A.cls, 256));
        if (can_vec()) {
            std::vector<uint8_t> m32(static_cast<size_t>(nS) * 32);
            for (uint32_t s = 0; s < nS; ++s)
                for (uint32_t q = 0; q < 32; ++q)
                    m32[static_cast<size_t>(s) * 32 + q] = static_cast<uint8_t>(q < nD ? A.maps[static_cast<size_t>(s) * nD + q] : q);
            CU(upload(&dmaps32, m32.data(), m32.size()));
        }
        if (!A.nsfa && nD <= 65535 && static_cast<uint64_t>(nS) * nD * 2 <= (1ull << 30)) {
            std::vector<uint16_t> m16(static_cast<size_t>(nS) * nD);
            for (size_t i = 0; i < m16.size(); ++i) m16[i] = static_cast<uint16_t>(A.maps[i]);
            CU(upload(&dmaps16, m16.data(), m16.size()));
            dev_bytes += m16.size() * 2;
        }
        // composition table comp[a][b] = id(f_a . f_b) = delta_s^(a, rep(b)) (Lemma 1)
        if (has_comp()) {
            const bool u8 = nS <= 256;
            const size_t cells = static_cast<size_t>(nS) * nS;
            std::vector<uint16_t> comp(cells);
            for (uint32_t a = 0; a < nS; ++a)
                for (uint32_t b = 0; b < nS; ++b) {
                    uint32_t st = a;
                    if (!A.comp.empty()) {  // N-SFA: the logical matrix products of compile_nsfa
                        st = A.comp[static_cast<size_t>(a) * nS + b];
                    } else {
                        for (uint32_t k = A.rep_off[b]; k < A.rep_off[b + 1]; ++k)
                            st = A.T[static_cast<size_t>(st) * C + A.cls[A.rep[k]]];
                    }
                    comp[static_cast<size_t>(a) * nS + b] = static_cast<uint16_t>(st);
                }
            std::vector<uint8_t> bytes(cells * (u8 ? 1 : 2));
            for (size_t i = 0; i < cells; ++i) {
                if (u8) bytes[i] = static_cast<uint8_t>(comp[i]);
                else std::memcpy(&bytes[2 * i], &comp[i], 2);
            }
            bytes.resize((bytes.size() + 15) & ~size_t(15), 0);
            CU(upload(reinterpret_cast<uint8_t**>(&dcomp), bytes.data(), bytes.size()));
            dev_bytes += bytes.size();
            if (bytes.size() <= kAuxMax) {
                CU(upload(&daux[0], reinterpret_cast<const uint32_t*>(bytes.data()), bytes.size() / 4));
                aux_bytes[0] = static_cast<uint32_t>(bytes.size());
            }
        }
        if (A.depth <= 15) {  // rep(s) in one 16-byte slot, |rep(s)| in byte 15
            std::vector<uint8_t> slots(static_cast<size_t>(nS) * 16, 0);
            for (uint32_t st = 0; st < nS; ++st) {
                const uint32_t len = A.rep_off[st + 1] - A.rep_off[st];
                std::memcpy(&slots[static_cast<size_t>(st) * 16], A.rep.data() + A.rep_off[st], len);
                slots[static_cast<size_t>(st) * 16 + 15] = static_cast<uint8_t>(len);
            }
            CU(upload(reinterpret_cast<uint8_t**>(&drep16), slots.data(), slots.size()));
        }
        if (can_vec() && static_cast<size_t>(nS) * 32 <= kAuxMax) {
            std::vector<uint8_t> m32(static_cast<size_t>(nS) * 32);
            for (uint32_t st = 0; st < nS; ++st)
                for (uint32_t q = 0; q < 32; ++q)
                    m32[static_cast<size_t>(st) * 32 + q] = static_cast<uint8_t>(q < nD ? A.maps[static_cast<size_t>(st) * nD + q] : q);
            CU(upload(&daux[1], reinterpret_cast<const uint32_t*>(m32.data()), m32.size() / 4));
            aux_bytes[1] = static_cast<uint32_t>(m32.size());
        }
        // HOT residency tables (AUTO uses them when neither smem layout holds the whole table)
        {
            int rc = upload_hot(nullptr, 0);
            if (rc) return rc;
            if (!A.nsfa) rc = upload_fact();
            if (rc) return rc;
            dev_bytes += static_cast<uint64_t>(nS) * W * 2 + 4ull * nS;
        }
        {  // f_s(q0) with its accept bit (bit 31): the epilogue's last lookup is one load
            std::vector<uint32_t> ia(A.img0.size());
            for (size_t i = 0; i < ia.size(); ++i) ia[i] = A.img0[i] | (A.dfa_final[A.img0[i]] ? 0x80000000u : 0u);
            CU(upload(&dimg0, ia.data(), ia.size()));
        }
        CU(upload(&dfinal, A.dfa_final.data(), A.dfa_final.size()));
        CU(upload(&drep_off, A.rep_off.data(), A.rep_off.size()));
        if (!A.rep.empty()) CU(upload(&drep, A.rep.data(), A.rep.size()));
        dev_bytes += T16.size() * 2 + R16.size() * 2 + 256 + (vec() ? static_cast<uint64_t>(nS) * 32 : 0) +
                     A.img0.size() * 4 + A.dfa_final.size() + A.rep_off.size() * 4 + A.rep.size();

        CU(cudaMalloc(&partials, static_cast<size_t>(kMaxSlots) * 32));
        CU(cudaMalloc(&ticket, sizeof(uint32_t)));
        CU(cudaMemset(ticket, 0, sizeof(uint32_t)));
        CU(cudaMalloc(&dres, 2 * sizeof(sfa_result)));
#ifdef SFA_STAMPS
        CU(cudaMalloc(&dstamps, (kMaxSlots + 1) * 16 * sizeof(uint64_t)));
#endif
        CU(cudaMalloc(&dplan, sizeof(sfa::TmaPlan)));
        CU(cudaMalloc(&gmaps, 512));
        CU(cudaMalloc(&berr, 16));
        CU(cudaMemset(berr, 0, 16));
        CU(cudaMallocHost(&hres, 2 * sizeof(sfa_result)));
        CU(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
        return SFA_OK;
    }

    // does `mode` fit for this launch kind?
    bool fits(sfa::Res mode, int kind /*0 tma, 1 direct*/) const {
        const sfa::DevTables t = tables(mode, kind);
        if (mode == sfa::Res::Hot && t.hotH == 0) return false;
        if (kind == 0) {
            sfa::TmaConfig c;
            return sfa::tma_choose(mode, t, smem_optin, ktune(), &c);
        }
        return sfa::direct_smem_bytes(mode, t) <= smem_optin;
    }
    int resolve(int kind, sfa::Res* out) const {
        if (forced != SFA_RES_AUTO) {
            const sfa::Res m = static_cast<sfa::Res>(forced);
            if (!fits(m, kind)) return fail(SFA_ERR_CAPACITY, "forced residency does not fit in shared memory");
            *out = m;
            return SFA_OK;
        }
        // TMA scan: a factorable automaton whose DFA window gets more lane copies
        // than the PRIVATE SFA table (fewer bank conflicts per lookup) runs
        // HOT + FACTORED (cfg4: R = 32 DFA copies against R = 16 SFA copies).
        if (kind == 0 && dfam && factor_on() && dwin_R > priv_R && fits(sfa::Res::Hot, kind)) {
            *out = sfa::Res::Hot;
            return SFA_OK;
        }
        for (sfa::Res m : {sfa::Res::Private, sfa::Res::Shared, sfa::Res::Hot, sfa::Res::Global})
            if (fits(m, kind)) {
                *out = m;
                return SFA_OK;
            }
        return fail(SFA_ERR_CAPACITY, "no residency mode fits");
    }

    sfa::Scratch scratch() const {
        sfa::Scratch s;
        s.partials = partials;
        s.ticket = ticket;
        s.max_ctas = kMaxSlots - 2;
        return s;
    }

    // The TMA scan's launch shape and plan for n bytes at d_text.
    int tma_plan(sfa::Res mode, const sfa::DevTables& t, const uint8_t* d_text, uint64_t n, sfa::TmaConfig* cfg,
                 sfa::TmaPlan* plan) const {
        if (!sfa::tma_choose(mode, t, smem_optin, ktune(), cfg)) return fail(SFA_ERR_CAPACITY, "no TMA shape fits");
        sfa::make_plan(reinterpret_cast<uintptr_t>(d_text), n, static_cast<uint32_t>(sm_count), cfg->rows_per_cta,
                       cfg->nb, static_cast<uint32_t>(cfg->rowb), tuning.row_align, plan);
        if (plan->nchunks == 0 || plan->ctas == 0 || plan->ctas > kMaxSlots - 2)
            return fail(SFA_ERR_INVALID_ARG, "text too short for the TMA scan");
        return SFA_OK;
    }

    // One text on the device -> result (device), stream-ordered.  force_tma:
    // the TMA scan even below kTmaMin (sfa_match_rows); row_ids / plan_out:
    // its per-row SFA ids and geometry.
    int launch_one(const uint8_t* d_text, uint64_t n, cudaStream_t stream, const uint32_t* q_in, sfa_result* d_result,
                   uint64_t force_pieces = 0, uint32_t* piece_ids = nullptr, uint32_t* map_out = nullptr,
                   bool force_tma = false, uint32_t* row_ids = nullptr, size_t row_cap = 0,
                   sfa::TmaPlan* plan_out = nullptr) {
        const bool direct = !force_tma && (force_pieces > 0 || n < kTmaMin);
        sfa::Res mode;
        int rc = SFA_OK;
        if (!direct && lcache.epoch == cfg_epoch && lcache.text == d_text && lcache.n == n && !row_ids)
            mode = lcache.mode;  // the same text again: the cached decisions below
        else
            rc = resolve(direct ? 1 : 0, &mode);
        if (rc) return rc;
        cudaError_t e;
        if (direct) {
            sfa::DirectArgs a;
            a.t = tables(mode, 1);
            a.text = d_text;
            a.n = n;
            // Bytes per thread: about 8192 threads (32 CTAs) until pieces reach
            // 512 B.  Every CTA builds its own smem table, so more, shorter pieces
            // cost more than their shorter chains save (3 MiB, cfg2: 12.3 us at
            // 64-B pieces, 6.5 us at 384-512).  Tuning direct_piece forces one.
            const uint64_t forced_piece =
                tuning.direct_piece >= 16 && tuning.direct_piece <= 4096 ? tuning.direct_piece : 0u;
            const uint64_t piece =
                forced_piece ? forced_piece : std::min<uint64_t>(kDirectPieceMax, std::max<uint64_t>(kDirectPiece, n / 8192));
            a.npieces = force_pieces ? force_pieces : std::max<uint64_t>(1, (n + piece - 1) / piece);
            a.sc = scratch();
            a.q_in = q_in;
            a.result = d_result;
            a.piece_ids = piece_ids;
            a.map_out = map_out;
            const uint64_t ctas = (a.npieces + sfa::direct_threads_per_cta() - 1) / sfa::direct_threads_per_cta();
            if (ctas > a.sc.max_ctas) return fail(SFA_ERR_INVALID_ARG, "too many chunks");
            e = sfa::launch_scan_direct(mode, vec(), a, stream);
        } else {
            sfa::ScanArgs a{};
            const bool cached = lcache.epoch == cfg_epoch && lcache.text == d_text && lcache.n == n && !row_ids;
            a.t = cached ? lcache.t : tables(mode, 0);
            a.text = d_text;
            a.n = n;
            a.sc = scratch();
            a.q_in = q_in;
            a.result = d_result;
            a.map_out = map_out;
            a.row_ids = row_ids;
#ifdef SFA_STAMPS
            a.stamps = dstamps;
            a.t.diag = reinterpret_cast<unsigned long long*>(dstamps + kMaxSlots * 16);
            CU(cudaMemsetAsync(dstamps, 0, (kMaxSlots + 1) * 16 * sizeof(uint64_t), stream));
#endif
            sfa::TmaConfig cfg;
            if (cached) {
                cfg = lcache.cfg;
                a.plan = lcache.plan;
            } else {
                rc = tma_plan(mode, a.t, d_text, n, &cfg, &a.plan);
                if (rc) return rc;
                lcache.epoch = cfg_epoch;
                lcache.text = d_text;
                lcache.n = n;
                lcache.mode = mode;
                lcache.t = a.t;
                lcache.cfg = cfg;
                lcache.plan = a.plan;
            }
            if (row_ids && a.plan.nchunks > row_cap) return fail(SFA_ERR_CAPACITY, "row_cap is smaller than the row count");
            if (plan_out) *plan_out = a.plan;
            e = sfa::launch_scan_tma(mode, vec(), a, cfg, stream);
        }
        if (e != cudaSuccess) return cuda_fail(e, "scan launch");
        return SFA_OK;
    }

    // Host-call staging: two device slices of >= bytes each, the copy stream and its events.
    int ensure_staging(size_t bytes) {
        if (!copy_stream) {
            for (int i = 0; i < 2; ++i) {
                CU(cudaEventCreateWithFlags(&ev_copied[i], cudaEventDisableTiming));
                CU(cudaEventCreateWithFlags(&ev_used[i], cudaEventDisableTiming));
            }
            CU(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
        }
        if (stage_cap < bytes) {
            if (has_last) CU(cudaStreamSynchronize(last_stream));
            for (int i = 0; i < 2; ++i) {
                if (stage[i]) CU(cudaFree(stage[i]));
                stage[i] = nullptr;
            }
            stage_cap = 0;
            for (int i = 0; i < 2; ++i) CU(cudaMalloc(&stage[i], bytes));
            stage_cap = bytes;
        }
        return SFA_OK;
    }

    int launch_seg_empty(sfa_result* d_results, uint64_t count, cudaStream_t stream) {
        cudaError_t e = sfa::launch_fill_results(d_results, count, 0, A.dfa_final[0], stream);
        return e == cudaSuccess ? SFA_OK : cuda_fail(e, "fill launch");
    }

    // A batch through the SEG scan: texts back to back at `base`; host plan
    // for equal texts of `len` bytes (off == nullptr), else the device plan.
    int launch_seg(const uint8_t* base, const uint64_t* d_off, uint64_t len, uint64_t count, sfa_result* d_results,
                   cudaStream_t stream) {
        sfa::Res mode;
        int rc = resolve(0, &mode);
        if (rc) return rc;
        sfa::ScanArgs a{};
        a.t = tables(mode, 0, true);
        a.text = base;
        a.sc = scratch();
        a.off = d_off;
        a.count = count;
        a.results = d_results;
#ifdef SFA_STAMPS
        a.stamps = dstamps;
        a.t.diag = reinterpret_cast<unsigned long long*>(dstamps + kMaxSlots * 16);
        CU(cudaMemsetAsync(dstamps, 0, (kMaxSlots + 1) * 16 * sizeof(uint64_t), stream));
#endif
        sfa::TmaConfig cfg;
        if (!sfa::tma_choose(mode, a.t, smem_optin, ktune(), &cfg)) return fail(SFA_ERR_CAPACITY, "no TMA shape fits");
        const uint32_t G = static_cast<uint32_t>(sm_count);
        cudaError_t e;
        if (d_off) {
            sfa::BatchPlanArgs p;
            p.texts = base;
            p.off = d_off;
            p.count = count;
            p.G = G;
            p.R = cfg.rows_per_cta;
            p.NB = cfg.nb;
            p.rowb = static_cast<uint32_t>(cfg.rowb);
            p.row_align = tuning.row_align;
            p.dplan = dplan;
            p.gmaps = gmaps;
            p.err = berr;
            p.epoch = ++epoch ? epoch : ++epoch;  // never 0 (the error word starts at 0)
            p.results = d_results;
            p.eps_accept = A.dfa_final[0];
            p.slots = reinterpret_cast<uint4*>(partials);  // the scan uses them only after griddepcontrol.wait
            p.ticket = berr + 1;
            e = sfa::launch_batch_plan(p, cfg, sm_count, stream);
            if (e != cudaSuccess) return cuda_fail(e, "batch plan launch");
            a.dplan = dplan;
            a.gmaps = gmaps;
            a.err = berr;
            a.epoch = p.epoch;
            e = sfa::launch_scan_seg(mode, a, cfg, G, stream);
        } else {
            a.n = len * count;
            if (!sfa::make_plan_uniform(reinterpret_cast<uintptr_t>(base), len, count, G, cfg.rows_per_cta, cfg.nb,
                                        static_cast<uint32_t>(cfg.rowb), &a.plan))
                sfa::make_plan(reinterpret_cast<uintptr_t>(base), a.n, G, cfg.rows_per_cta, cfg.nb,
                               static_cast<uint32_t>(cfg.rowb), tuning.row_align, &a.plan);
            a.plan.len = len;
            e = sfa::launch_scan_seg(mode, a, cfg, G, stream);
        }
        if (e != cudaSuccess) return cuda_fail(e, "batch scan launch");
        return SFA_OK;
    }

    // Serialise the shared scratch across streams.  Launches on the stream of
    // the previous call are ordered by the stream itself (and may overlap
    // through PDL, the kernels wait before touching scratch); a different
    // stream first waits for everything enqueued on the previous one.
    cudaStream_t last_stream = nullptr;
    bool has_last = false;
    // Alg. 3 baseline: the DFA window table, u32 cells premultiplied to row
    // byte offsets (4 W delta_d(q, byte)); column W-1 = every byte outside the
    // window (one class, so any such byte represents it).
    int upload_spec() {
        if (dspecT) return SFA_OK;
        if (!A.has_dfa || A.nsfa) return fail(SFA_ERR_CAPACITY, "Alg. 3 needs a D-SFA handle");
        const uint32_t nD = A.nD;
        uint32_t ob = 0;
        while (ob >= lo && ob + 1 < lo + W) ++ob;  // a byte outside [lo, lo + W - 2]
        std::vector<uint32_t> Td((static_cast<size_t>(nD) * W + 3) & ~size_t(3), 0);
        for (uint32_t q = 0; q < nD; ++q) {
            for (uint32_t j = 0; j + 1 < W; ++j) Td[static_cast<size_t>(q) * W + j] = 4 * W * A.dfa[q * 256u + lo + j];
            Td[static_cast<size_t>(q) * W + W - 1] = 4 * W * A.dfa[q * 256u + ob];
        }
        CU(upload(&dspecT, Td.data(), Td.size()));
        CU(cudaMalloc(&spec_ticket, 16));
        CU(cudaMemset(spec_ticket, 0, 16));
        return SFA_OK;
    }

    int begin(cudaStream_t stream) {
        if (lazy) return fail(SFA_ERR_INVALID_ARG, "an on-the-fly handle (sfa_compile_lazy) matches with sfa_match_lazy");
        int rc = ensure_uploaded();
        if (rc) return rc;
        if (has_last && stream != last_stream) {
            CU(cudaEventRecord(ev_done, last_stream));
            CU(cudaStreamWaitEvent(stream, ev_done, 0));
        }
        return SFA_OK;
    }
    int end(cudaStream_t stream) {
        last_stream = stream;
        has_last = true;
        return SFA_OK;
    }
};

extern "C" {

const char* sfa_last_error(void) { return g_err.c_str(); }

// Byte window: the smallest [lo, hi] such that every byte outside it has one
// class ("other"); table columns are lo..hi, then W-1 = other.  With cand = 0
// the window never contains byte 0, with cand = 255 never byte 255, so W <= 256.
static void set_window(sfa_handle* h) {
    const uint8_t* cls = h->A.cls;
    h->W = 257;
    for (int cand : {0, 255}) {
        const uint8_t o = cls[cand];
        int lo = -1, hi = -1;
        for (int b = 0; b < 256; ++b)
            if (cls[b] != o) {
                if (lo < 0) lo = b;
                hi = b;
            }
        const uint32_t W = lo < 0 ? 1u : static_cast<uint32_t>(hi - lo + 2);
        if (W < h->W) {
            h->W = W;
            h->lo = lo < 0 ? 0u : static_cast<uint32_t>(lo);
            h->other = o;
        }
    }
}

static int compile_any(bool nsfa, const char* regex, const uint8_t* alphabet, int alphabet_len, uint32_t max_sfa,
                       sfa_handle** out) {
    if (!out) return fail(SFA_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!regex) return fail(SFA_ERR_INVALID_ARG, "regex is NULL");
    if (alphabet && alphabet_len < 0) return fail(SFA_ERR_INVALID_ARG, "alphabet_len < 0");
    sfa_handle* h = new (std::nothrow) sfa_handle;
    if (!h) return fail(SFA_ERR_OOM, "host allocation failed");
    try {
        h->A = nsfa ? sfa::compile_nsfa(regex, alphabet, alphabet ? alphabet_len : -1, max_sfa)
                    : sfa::compile_regex(regex, alphabet, alphabet ? alphabet_len : -1, max_sfa);
    } catch (const sfa::CompileError& e) {
        delete h;
        return fail(e.code, e.what());
    } catch (const std::bad_alloc&) {
        delete h;
        return fail(SFA_ERR_OOM, "host allocation failed during compile");
    }
    set_window(h);
    *out = h;
    return SFA_OK;
}

int sfa_compile(const char* regex, const uint8_t* alphabet, int alphabet_len, uint32_t max_sfa, sfa_handle** out) {
    return compile_any(false, regex, alphabet, alphabet_len, max_sfa, out);
}

int sfa_compile_lazy(const char* regex, const uint8_t* alphabet, int alphabet_len, uint32_t max_states,
                     sfa_handle** out) {
    if (!out) return fail(SFA_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!regex) return fail(SFA_ERR_INVALID_ARG, "regex is NULL");
    if (alphabet && alphabet_len < 0) return fail(SFA_ERR_INVALID_ARG, "alphabet_len < 0");
    sfa_handle* h = new (std::nothrow) sfa_handle;
    if (!h) return fail(SFA_ERR_OOM, "host allocation failed");
    try {
        h->A = sfa::compile_regex(regex, alphabet, alphabet ? alphabet_len : -1, 0, false);
        h->lazy.reset(new sfa::LazySFA(h->A, max_states ? max_states : (1u << 24)));
        set_window(h);  // for Alg. 3 (sfa_match_speculative) on the same DFA
    } catch (const sfa::CompileError& e) {
        delete h;
        return fail(e.code, e.what());
    } catch (const std::bad_alloc&) {
        delete h;
        return fail(SFA_ERR_OOM, "host allocation failed during compile");
    }
    *out = h;
    return SFA_OK;
}

int sfa_compile_nsfa(const char* regex, const uint8_t* alphabet, int alphabet_len, uint32_t max_sfa,
                     sfa_handle** out) {
    return compile_any(true, regex, alphabet, alphabet_len, max_sfa, out);
}

void sfa_free(sfa_handle* h) { delete h; }

int sfa_info(const sfa_handle* h, sfa_info_t* info) {
    if (!h || !info) return fail(SFA_ERR_INVALID_ARG, "NULL argument");
    std::memset(info, 0, sizeof(*info));
    const auto& A = h->A;
    info->nfa_positions = A.nfa_positions;
    info->dfa_subset_states = A.subset_states;
    info->dfa_states = A.nD;
    info->dfa_live = A.dead >= 0 ? A.nD - 1 : A.nD;
    info->dead_state = A.dead >= 0 ? static_cast<uint32_t>(A.dead) : UINT32_MAX;
    info->sfa_states = A.nS;
    info->classes = A.C;
    info->sfa_depth = A.depth;
    info->compose_mode = static_cast<uint32_t>(h->compose_mode());
    info->range_lo = h->lo;
    info->range_width = h->W;
    info->residency = 0;
    if (h->uploaded) {
        sfa::Res m;
        if (h->resolve(0, &m) == SFA_OK) info->residency = static_cast<uint32_t>(m);
    }
    info->device_table_bytes = h->dev_bytes;
    info->dfa_seconds = A.dfa_seconds;
    info->sfa_seconds = A.sfa_seconds;
    info->kind = h->lazy ? 2u : (A.nsfa ? 1u : 0u);
    if (h->lazy) {
        info->compose_mode = 0;
        info->residency = SFA_RES_L2;
        info->sfa_states = h->lazy->nS;
        info->lazy_transitions = h->lazy->transitions;
        info->lazy_seconds = h->lazy_build_s;
    }
    info->nfa_states = A.nfa_states;
    info->has_dfa = A.has_dfa ? 1u : 0u;
    info->dfa_window_copies = h->dfam ? h->dwin_R : 0u;
    info->dfa_window_hot = h->dfam ? h->dwin_H : 0u;
    return SFA_OK;
}

int sfa_set_residency(sfa_handle* h, int mode) {
    if (!h) return fail(SFA_ERR_INVALID_ARG, "NULL handle");
    if (mode < SFA_RES_AUTO || mode > SFA_RES_L2) return fail(SFA_ERR_INVALID_ARG, "bad residency mode");
    std::lock_guard<std::mutex> lk(h->mu);
    if (mode == SFA_RES_AUTO) {
        h->forced = mode;
        ++h->cfg_epoch;
        return SFA_OK;
    }
    int rc = h->ensure_uploaded();
    if (rc) return rc;
    const int prev = h->forced;
    h->forced = mode;
    ++h->cfg_epoch;
    sfa::Res m;
    rc = h->resolve(1, &m);
    if (rc) {
        h->forced = prev;
        ++h->cfg_epoch;
    }
    return rc;
}

int sfa_tune_residency(sfa_handle* h, const uint8_t* d_sample, size_t n, sfa_stream_t stream) {
    if (!h) return fail(SFA_ERR_INVALID_ARG, "NULL handle");
    if (!d_sample && n > 0) return fail(SFA_ERR_INVALID_ARG, "d_sample is NULL with n > 0");
    std::lock_guard<std::mutex> lk(h->mu);
    int rc = h->ensure_uploaded();
    if (rc) return rc;
    if (n == 0) {  // back to the static ranking
        if (h->has_last) CU(cudaStreamSynchronize(h->last_stream));
        return h->upload_hot(nullptr, 0);
    }
    return h->tune_hot(d_sample, n, reinterpret_cast<cudaStream_t>(stream));
}

int sfa_set_compose(sfa_handle* h, int mode) {
    if (!h) return fail(SFA_ERR_INVALID_ARG, "NULL handle");
    if (mode < SFA_COMPOSE_AUTO || mode > SFA_COMPOSE_REPLAY) return fail(SFA_ERR_INVALID_ARG, "bad compose mode");
    if (mode == SFA_COMPOSE_VEC && !h->can_vec()) return fail(SFA_ERR_CAPACITY, "VEC composition needs a D-SFA with |D| <= 32");
    if (mode == SFA_COMPOSE_TABLE && !h->has_comp()) return fail(SFA_ERR_CAPACITY, "composition table needs |S| <= 4096");
    std::lock_guard<std::mutex> lk(h->mu);
    h->compose = mode;
    ++h->cfg_epoch;
    return SFA_OK;
}

int sfa_set_tuning(sfa_handle* h, const sfa_tuning_t* tu) {
    if (!h) return fail(SFA_ERR_INVALID_ARG, "NULL handle");
    sfa_tuning_t t{};
    if (tu) t = *tu;
    if (t.tma_k < 0 || t.tma_k > 2 || (t.tma_rowb && t.tma_rowb != 16 && t.tma_rowb != 32 && t.tma_rowb != 64) ||
        (t.tma_rowb && !t.tma_k) || t.tma_ring < 0 || t.tma_ring > 8 ||
        (t.tma_promo != -1 && t.tma_promo != 0 && t.tma_promo != 64 && t.tma_promo != 128 && t.tma_promo != 256) ||
        (t.row_align && t.row_align != 64 && t.row_align != 128 && t.row_align != 256) ||
        (t.dfa_copies & (t.dfa_copies - 1)) || t.dfa_copies > 32 ||
        (t.private_copies & (t.private_copies - 1)) || t.private_copies > 32 ||
        (t.direct_piece && (t.direct_piece < 16 || t.direct_piece > 4096)) || t.dfa_u8 > 1 || t.dfa_layout > 2 || t.fact_fold > 2)
        return fail(SFA_ERR_INVALID_ARG, "bad tuning value");
    if (!tu) t.tma_promo = -1;
    std::lock_guard<std::mutex> lk(h->mu);
    // the table layouts depend on the copy caps and the factoring switch: rebuild lazily
    h->release_device();
    h->tuning = t;
    ++h->cfg_epoch;
    return SFA_OK;
}

int sfa_export_dfa(const sfa_handle* h, uint32_t* table, uint8_t* finals) {
    if (!h) return fail(SFA_ERR_INVALID_ARG, "NULL handle");
    if (!h->A.has_dfa) return fail(SFA_ERR_CAPACITY, "this N-SFA handle has no DFA (more than 2^20 states)");
    if (table) std::memcpy(table, h->A.dfa.data(), h->A.dfa.size() * sizeof(uint32_t));
    if (finals) std::memcpy(finals, h->A.dfa_final.data(), h->A.dfa_final.size());
    return SFA_OK;
}

int sfa_export_sfa(const sfa_handle* h, uint32_t* table, uint32_t* maps, uint8_t* finals) {
    if (!h) return fail(SFA_ERR_INVALID_ARG, "NULL handle");
    if (h->lazy) {  // the states built so far; transitions not built yet are UINT32_MAX
        const sfa::LazySFA& Z = *h->lazy;
        if (table)
            for (uint32_t st = 0; st < Z.nS; ++st)
                for (int b = 0; b < 256; ++b) {
                    const uint32_t t = Z.next(st, Z.cls[b]);
                    table[static_cast<size_t>(st) * 256 + b] = t == sfa::kUnknown ? t : t & ~sfa::kFactBit;
                }
        if (maps)
            for (size_t i = 0; i < Z.maps.size(); ++i) maps[i] = Z.maps[i];
        if (finals)
            for (uint32_t st = 0; st < Z.nS; ++st) finals[st] = Z.dfinal[Z.img0(st)];
        return SFA_OK;
    }
    const auto& A = h->A;
    if (table)
        for (uint32_t s = 0; s < A.nS; ++s)
            for (int b = 0; b < 256; ++b) table[static_cast<size_t>(s) * 256 + b] = A.T[static_cast<size_t>(s) * A.C + A.cls[b]];
    if (maps && A.nsfa) return fail(SFA_ERR_CAPACITY, "N-SFA states are set-valued mappings (no |D| map)");
    if (maps) std::memcpy(maps, A.maps.data(), A.maps.size() * sizeof(uint32_t));
    if (finals) std::memcpy(finals, A.acc.data(), A.acc.size());
    return SFA_OK;
}

int sfa_match_async(const sfa_handle* hc, const uint8_t* d_text, size_t n, sfa_stream_t stream, sfa_result* d_result) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h || !d_result) return fail(SFA_ERR_INVALID_ARG, "NULL handle or result");
    if (!d_text && n > 0) return fail(SFA_ERR_INVALID_ARG, "d_text is NULL with n > 0");
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = h->begin(s);
    if (rc) return rc;
    if (n == 0) {  // (q0, [eps in L]) written by a one-thread kernel: no host round trip
        cudaError_t e = sfa::launch_fill_result(d_result, 0, h->A.dfa_final[0], nullptr, 0, s);
        if (e != cudaSuccess) return cuda_fail(e, "fill launch");
        return h->end(s);
    }
    rc = h->launch_one(d_text, n, s, nullptr, d_result);
    if (rc) return rc;
    return h->end(s);
}

int sfa_match(const sfa_handle* hc, const uint8_t* d_text, size_t n, sfa_stream_t stream, uint32_t* final_state,
              int* accept) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h || !final_state || !accept) return fail(SFA_ERR_INVALID_ARG, "NULL argument");
    if (!d_text && n > 0) return fail(SFA_ERR_INVALID_ARG, "d_text is NULL with n > 0");
    if (n == 0) {  // (q0, [eps in L]) without a launch
        *final_state = 0;
        *accept = h->A.dfa_final[0];
        return SFA_OK;
    }
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = h->begin(s);
    if (rc) return rc;
    rc = h->launch_one(d_text, n, s, nullptr, h->dres);
    if (rc) return rc;
    CU(cudaMemcpyAsync(h->hres, h->dres, sizeof(sfa_result), cudaMemcpyDeviceToHost, s));
    rc = h->end(s);
    if (rc) return rc;
    CU(cudaStreamSynchronize(s));
    *final_state = h->hres[0].final_state;
    *accept = static_cast<int>(h->hres[0].accept);
    return SFA_OK;
}

int sfa_match_chunked(const sfa_handle* hc, const uint8_t* d_text, size_t n, uint32_t nchunks, sfa_stream_t stream,
                      uint32_t* final_state, int* accept, uint32_t* h_chunk_states) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h || !final_state || !accept || nchunks == 0) return fail(SFA_ERR_INVALID_ARG, "bad argument");
    if (!d_text && n > 0) return fail(SFA_ERR_INVALID_ARG, "d_text is NULL with n > 0");
    if (n == 0) {
        *final_state = 0;
        *accept = h->A.dfa_final[0];
        if (h_chunk_states) h_chunk_states[0] = 0;
        return SFA_OK;
    }
    const uint64_t p = std::min<uint64_t>(nchunks, n);  // n < p: n one-byte chunks (C6)
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = h->begin(s);
    if (rc) return rc;
    uint32_t* dids = nullptr;
    if (h_chunk_states) CU(cudaMallocAsync(&dids, p * sizeof(uint32_t), s));
    rc = h->launch_one(d_text, n, s, nullptr, h->dres, p, dids);
    if (rc) {
        if (dids) cudaFreeAsync(dids, s);
        return rc;
    }
    CU(cudaMemcpyAsync(h->hres, h->dres, sizeof(sfa_result), cudaMemcpyDeviceToHost, s));
    if (dids) {
        CU(cudaMemcpyAsync(h_chunk_states, dids, p * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        CU(cudaFreeAsync(dids, s));
    }
    rc = h->end(s);
    if (rc) return rc;
    CU(cudaStreamSynchronize(s));
    *final_state = h->hres[0].final_state;
    *accept = static_cast<int>(h->hres[0].accept);
    return SFA_OK;
}

int sfa_match_rows(const sfa_handle* hc, const uint8_t* d_text, size_t n, sfa_stream_t stream, uint32_t* d_row_ids,
                   size_t row_cap, sfa_rows_plan* plan, sfa_result* d_result) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h || !d_text || !d_row_ids || !plan || !d_result) return fail(SFA_ERR_INVALID_ARG, "NULL argument");
    if (n < (64u << 10)) return fail(SFA_ERR_INVALID_ARG, "sfa_match_rows needs n >= 64 KiB");
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = h->begin(s);
    if (rc) return rc;
    sfa::TmaPlan p;
    rc = h->launch_one(d_text, n, s, nullptr, d_result, 0, nullptr, nullptr, true, d_row_ids, row_cap, &p);
    if (rc) return rc;
    plan->head = p.head;
    plan->row_len = p.L;
    plan->rows = p.nchunks;
    plan->tail_start = p.tail_start;
    plan->ctas = p.ctas;
    plan->rows_hi = p.rc_hi;
    plan->rows_lo = p.rc_lo;
    plan->ctas_hi = p.m;
    return h->end(s);
}

int sfa_match_map(const sfa_handle* hc, const uint8_t* d_text, size_t n, sfa_stream_t stream, uint32_t* d_map) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h || !d_map) return fail(SFA_ERR_INVALID_ARG, "NULL handle or map");
    if (!d_text && n > 0) return fail(SFA_ERR_INVALID_ARG, "d_text is NULL with n > 0");
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = h->begin(s);
    if (rc) return rc;
    if (!h->vec() && !h->dmaps16) return fail(SFA_ERR_CAPACITY, "no mapping table for sfa_match_map (N-SFA or too large)");
    if (n == 0) {  // f_eps = identity
        cudaError_t e = sfa::launch_fill_result(nullptr, 0, 0, d_map, h->A.nD, s);
        if (e != cudaSuccess) return cuda_fail(e, "fill launch");
        return h->end(s);
    }
    rc = h->launch_one(d_text, n, s, nullptr, nullptr, 0, nullptr, d_map);
    if (rc) return rc;
    return h->end(s);
}

int sfa_combine_maps(const sfa_handle* hc, const uint32_t* d_maps, size_t count, sfa_stream_t stream,
                     sfa_result* d_result) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h || !d_result || (count > 0 && !d_maps)) return fail(SFA_ERR_INVALID_ARG, "NULL argument");
    if (count > 0xffffffffull) return fail(SFA_ERR_INVALID_ARG, "count too large");
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = h->begin(s);
    if (rc) return rc;
    cudaError_t e = sfa::launch_combine_maps(d_maps, static_cast<uint32_t>(count), h->A.nD, h->dfinal, d_result, s);
    if (e != cudaSuccess) return cuda_fail(e, "combine launch");
    return h->end(s);
}

int sfa_match_batch(const sfa_handle* hc, const uint8_t* d_texts, const uint64_t* d_offsets, size_t count,
                    sfa_stream_t stream, sfa_result* d_results) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h) return fail(SFA_ERR_INVALID_ARG, "NULL handle");
    if (count == 0) return SFA_OK;
    if (!d_offsets || !d_results || !d_texts) return fail(SFA_ERR_INVALID_ARG, "NULL texts, offsets or results");
    if (count > (1ull << 31)) return fail(SFA_ERR_INVALID_ARG, "count too large");
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = h->begin(s);
    if (rc) return rc;
    rc = h->launch_seg(d_texts, d_offsets, 0, count, d_results, s);
    if (rc) return rc;
    return h->end(s);
}

// `count` back-to-back texts of `len` bytes: the same SEG scan with the
// boundaries at multiples of len and the plan made on the host.
int sfa_match_batch_uniform(const sfa_handle* hc, const uint8_t* d_texts, size_t len, size_t count, sfa_stream_t stream,
                            sfa_result* d_results) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h || (count && !d_results)) return fail(SFA_ERR_INVALID_ARG, "NULL handle or results");
    if (count == 0) return SFA_OK;
    if (!d_texts && len > 0) return fail(SFA_ERR_INVALID_ARG, "d_texts is NULL");
    if (count > (1ull << 31) || (len && count > UINT64_MAX / len)) return fail(SFA_ERR_INVALID_ARG, "count too large");
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = h->begin(s);
    if (rc) return rc;
    if (len == 0) {  // every text empty: (q0, [eps in L]) each
        rc = h->launch_seg_empty(d_results, count, s);
        if (rc) return rc;
        return h->end(s);
    }
    rc = h->launch_seg(d_texts, nullptr, len, count, d_results, s);
    if (rc) return rc;
    return h->end(s);
}

int sfa_match_speculative(const sfa_handle* hc, const uint8_t* d_text, size_t n, uint64_t nchunks, sfa_stream_t stream,
                          uint32_t* d_chunk_maps, sfa_result* d_result) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h || !d_result) return fail(SFA_ERR_INVALID_ARG, "NULL handle or result");
    if (!d_text && n > 0) return fail(SFA_ERR_INVALID_ARG, "d_text is NULL with n > 0");
    if (d_chunk_maps && nchunks == 0)  // the caller must know how many rows it receives
        return fail(SFA_ERR_INVALID_ARG, "d_chunk_maps needs an explicit nchunks");
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = h->lazy ? h->ensure_dfa_only() : h->begin(s);
    if (rc) return rc;
    if (n == 0) {  // no chunk: T = identity, q_final = q0
        cudaError_t e = sfa::launch_fill_result(d_result, 0, h->A.dfa_final[0], d_chunk_maps, h->A.nD, s);
        if (e != cudaSuccess) return cuda_fail(e, "fill launch");
        return h->end(s);
    }
    rc = h->upload_spec();
    if (rc) return rc;
    sfa::SpecArgs p, a;
    p.Td = h->dspecT;
    p.nD = h->A.nD;
    p.W = h->W;
    p.lo = h->lo;
    p.dfinal = h->dfinal;
    p.text = d_text;
    uint32_t threads = 0;
    size_t smem = 0;
    cudaError_t e = sfa::spec_plan(p, h->sm_count, h->smem_optin, n, nchunks, &a, &threads, &smem);
    if (e == cudaErrorInvalidConfiguration) return fail(SFA_ERR_CAPACITY, "DFA too large for the speculative kernel");
    if (e != cudaSuccess) return cuda_fail(e, "speculative plan");
    const size_t need = static_cast<size_t>(a.ctas) * h->A.nD;
    if (h->spec_cap < need) {
        if (h->spec_maps) CU(cudaFree(h->spec_maps));
        h->spec_maps = nullptr;
        h->spec_cap = 0;
        CU(cudaMalloc(&h->spec_maps, need * 4));
        h->spec_cap = need;
    }
    a.cta_maps = h->spec_maps;
    a.ticket = h->spec_ticket;
    a.chunk_maps = d_chunk_maps;
    a.result = d_result;
    e = sfa::launch_spec(a, threads, smem, s);
    if (e != cudaSuccess) return cuda_fail(e, "speculative launch");
    return h->end(s);
}

int sfa_match_host(const sfa_handle* hc, const uint8_t* h_text, size_t n, sfa_stream_t stream, uint32_t* final_state,
                   int* accept) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h || !final_state || !accept) return fail(SFA_ERR_INVALID_ARG, "NULL argument");
    if (!h_text && n > 0) return fail(SFA_ERR_INVALID_ARG, "h_text is NULL with n > 0");
    if (n == 0) {
        *final_state = 0;
        *accept = h->A.dfa_final[0];
        return SFA_OK;
    }
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = h->begin(s);
    if (rc) return rc;
    if (!h->dmaps16) return fail(SFA_ERR_CAPACITY, "mapping table too large for sliced host matching");
    rc = h->ensure_staging(kSlice);
    if (rc) return rc;
    // The copy stream must not overwrite a staging buffer before earlier work
    // on `s` (from a previous call) is done with it.
    CU(cudaEventRecord(h->ev_used[0], s));
    CU(cudaEventRecord(h->ev_used[1], s));
    const uint64_t m = (n + kSlice - 1) / kSlice;
    for (uint64_t k = 0; k < m; ++k) {
        const int b = static_cast<int>(k & 1);
        const uint64_t off = k * kSlice, len = std::min<uint64_t>(kSlice, n - off);
        CU(cudaStreamWaitEvent(h->copy_stream, h->ev_used[b], 0));
        CU(cudaMemcpyAsync(h->stage[b], h_text + off, len, cudaMemcpyHostToDevice, h->copy_stream));
        CU(cudaEventRecord(h->ev_copied[b], h->copy_stream));
        CU(cudaStreamWaitEvent(s, h->ev_copied[b], 0));
        // slice k runs from q_{k-1} = result of slice k-1 (sequential reduction across slices)
        const uint32_t* q_in = k == 0 ? nullptr : &h->dres[(k - 1) & 1].final_state;
        rc = h->launch_one(h->stage[b], len, s, q_in, &h->dres[k & 1]);
        if (rc) return rc;
        CU(cudaEventRecord(h->ev_used[b], s));
    }
    CU(cudaMemcpyAsync(h->hres, &h->dres[(m - 1) & 1], sizeof(sfa_result), cudaMemcpyDeviceToHost, s));
    rc = h->end(s);
    if (rc) return rc;
    CU(cudaStreamSynchronize(s));
    *final_state = h->hres[0].final_state;
    *accept = static_cast<int>(h->hres[0].accept);
    return SFA_OK;
}

int sfa_match_batch_host(const sfa_handle* hc, const uint8_t* h_texts, const uint64_t* h_offsets, size_t count,
                         sfa_stream_t stream, sfa_result* h_results) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h) return fail(SFA_ERR_INVALID_ARG, "NULL handle");
    if (count == 0) return SFA_OK;
    if (!h_offsets || !h_results) return fail(SFA_ERR_INVALID_ARG, "NULL offsets or results");
    if (count > (1ull << 31)) return fail(SFA_ERR_INVALID_ARG, "count too large");
    uint64_t longest = 0;
    for (size_t i = 0; i < count; ++i) {
        if (h_offsets[i + 1] < h_offsets[i]) return fail(SFA_ERR_INVALID_ARG, "offsets decrease");
        longest = std::max<uint64_t>(longest, h_offsets[i + 1] - h_offsets[i]);
    }
    if (!h_texts && h_offsets[count] > h_offsets[0]) return fail(SFA_ERR_INVALID_ARG, "h_texts is NULL");
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = h->begin(s);
    if (rc) return rc;
    // slices of whole texts, at most max(kSlice, longest text) bytes and 2^20 texts
    const uint64_t cap = std::max<uint64_t>(kSlice, (longest + 255) & ~uint64_t(255));
    rc = h->ensure_staging(cap);
    if (rc) return rc;
    const size_t kMaxTexts = 1u << 20;
    const size_t ntexts_cap = std::min<size_t>(count, kMaxTexts) + 1;
    if (h->soff_cap < ntexts_cap) {
        if (h->has_last) CU(cudaStreamSynchronize(h->last_stream));
        for (int i = 0; i < 2; ++i) {
            if (h->soff[i]) CU(cudaFree(h->soff[i]));
            h->soff[i] = nullptr;
        }
        h->soff_cap = 0;
        for (int i = 0; i < 2; ++i) CU(cudaMalloc(&h->soff[i], ntexts_cap * sizeof(uint64_t)));
        h->soff_cap = ntexts_cap;
    }
    if (h->bres_cap < count) {
        if (h->has_last) CU(cudaStreamSynchronize(h->last_stream));
        if (h->bres) CU(cudaFree(h->bres));
        h->bres = nullptr;
        h->bres_cap = 0;
        CU(cudaMalloc(&h->bres, count * sizeof(sfa_result)));
        h->bres_cap = count;
    }
    // the copy stream must not overwrite a staging slice before earlier work on `s` is done with it
    CU(cudaEventRecord(h->ev_used[0], s));
    CU(cudaEventRecord(h->ev_used[1], s));
    size_t i0 = 0;
    for (int k = 0; i0 < count; ++k) {
        const int b = k & 1;
        size_t i1 = i0 + 1;
        while (i1 < count && i1 - i0 < kMaxTexts && h_offsets[i1 + 1] - h_offsets[i0] <= cap) ++i1;
        const uint64_t a0 = h_offsets[i0], bytes = h_offsets[i1] - a0;
        CU(cudaStreamWaitEvent(h->copy_stream, h->ev_used[b], 0));
        if (bytes) CU(cudaMemcpyAsync(h->stage[b], h_texts + a0, bytes, cudaMemcpyHostToDevice, h->copy_stream));
        CU(cudaMemcpyAsync(h->soff[b], h_offsets + i0, (i1 - i0 + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                           h->copy_stream));
        CU(cudaEventRecord(h->ev_copied[b], h->copy_stream));
        CU(cudaStreamWaitEvent(s, h->ev_copied[b], 0));
        // text i of the slice = stage[b][off[i] - a0 ...): the kernels only add off[i] to the base
        rc = h->launch_seg(h->stage[b] - a0, h->soff[b], 0, i1 - i0, h->bres + i0, s);
        if (rc) return rc;
        CU(cudaEventRecord(h->ev_used[b], s));
        i0 = i1;
    }
    CU(cudaMemcpyAsync(h_results, h->bres, count * sizeof(sfa_result), cudaMemcpyDeviceToHost, s));
    rc = h->end(s);
    if (rc) return rc;
    CU(cudaStreamSynchronize(s));
    return SFA_OK;
}

// sfa_match_lazy: Alg. 5 with the SFA built on the fly.
// Rounds of: the device runs every unfinished chunk until it meets a
// transition not built yet; the host builds the transitions the stalled
// chunks need by running its construction over the next K bytes of each
// (Alg. 4 lines 6-8 per (f, sigma) met); the table copy is refreshed.  Then
// the chunk states are folded as mapping vectors (pairwise tree on the
// device) and applied to q0.  States persist in the handle: a later match
// of similar text builds little or nothing.
int sfa_match_lazy(const sfa_handle* hc, const uint8_t* d_text, size_t n, sfa_stream_t stream, uint32_t* final_state,
                   int* accept) {
    sfa_handle* h = const_cast<sfa_handle*>(hc);
    if (!h || !final_state || !accept) return fail(SFA_ERR_INVALID_ARG, "NULL argument");
    if (!h->lazy) return fail(SFA_ERR_INVALID_ARG, "not an on-the-fly handle (sfa_compile_lazy)");
    if (!d_text && n > 0) return fail(SFA_ERR_INVALID_ARG, "d_text is NULL with n > 0");
    sfa::LazySFA& Z = *h->lazy;
    if (n == 0) {
        *final_state = 0;
        *accept = Z.dfinal[0];
        return SFA_OK;
    }
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc0 = h->ensure_dfa_only();
    if (rc0) return rc0;
    LazyDev& D = h->ld;
    const uint32_t nD = Z.nD, C = Z.C;
    // chunks: SPEC's rule (C6); at most 1024 per SM and 256 MiB of fold vectors
    uint64_t p = std::min<uint64_t>(n, 1024ull * static_cast<uint64_t>(h->sm_count));
    p = std::max<uint64_t>(1, std::min<uint64_t>(p, (128ull << 20) / nD));
    if (!D.cls) {
        CU(cudaMalloc(&D.cls, 256));
        CU(cudaMemcpy(D.cls, Z.cls, 256, cudaMemcpyHostToDevice));
        CU(cudaMalloc(&D.fin, nD * sizeof(uint16_t)));
        // the factored runs' table: row offsets 2 C delta(q, class) (C24)
        std::vector<uint16_t> dw(static_cast<size_t>(nD) * C);
        if (dw.size() * 2 <= sfa::kLazyFactorSmem)
            for (size_t i = 0; i < dw.size(); ++i) dw[i] = static_cast<uint16_t>(2u * C * Z.dcls[i]);
        CU(cudaMalloc(&D.dfa, dw.size() * sizeof(uint16_t)));
        CU(cudaMemcpy(D.dfa, dw.data(), dw.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
        CU(cudaMalloc(&D.absorbing, nD));
        CU(cudaMemcpy(D.absorbing, Z.absorbing.data(), nD, cudaMemcpyHostToDevice));
        CU(cudaMalloc(&D.counts, 2 * sizeof(uint32_t)));
    }
    // factored runs (C24): the DFA table must fit the scan's shared memory; the
    // host stops building at factorable states exactly when the device switches
    const bool factor = !h->tuning.no_factor && static_cast<uint64_t>(nD) * C * 2 <= sfa::kLazyFactorSmem;
    if (D.cap_p < p) {
        for (void* q : {(void*)D.state, (void*)D.pos, (void*)D.idx, (void*)D.fd, (void*)D.cbuf, (void*)D.fold})
            if (q) CU(cudaFree(q));
        D.state = nullptr, D.pos = nullptr, D.idx = nullptr, D.fd = nullptr, D.cbuf = nullptr, D.fold = nullptr;
        D.cap_p = 0;
        CU(cudaMalloc(&D.state, p * sizeof(uint32_t)));
        CU(cudaMalloc(&D.pos, p * sizeof(uint64_t)));
        CU(cudaMalloc(&D.idx, p * sizeof(uint32_t)));
        CU(cudaMalloc(&D.fd, p * sizeof(uint32_t)));
        CU(cudaMalloc(&D.cbuf, 4 * ((p + 1023) / 1024) * sizeof(uint32_t)));
        CU(cudaMalloc(&D.fold, 2 * p * nD * sizeof(uint16_t)));
        D.cap_p = p;
    }
    auto sync_tables = [&]() -> int {  // the device copies of T (all rows) and maps (new rows)
        if (D.cap_rows < Z.nS) {
            size_t cap = std::max<size_t>(1024, D.cap_rows);
            while (cap < Z.nS) cap *= 2;
            uint32_t* nT = nullptr;
            uint16_t* nM = nullptr;
            uint32_t* nF = nullptr;
            CU(cudaMalloc(&nT, cap * C * sizeof(uint32_t)));
            CU(cudaMalloc(&nM, cap * nD * sizeof(uint16_t)));
            CU(cudaMalloc(&nF, cap * sizeof(uint32_t)));
            if (D.maps_rows) {
                CU(cudaMemcpyAsync(nM, D.maps, D.maps_rows * nD * sizeof(uint16_t), cudaMemcpyDeviceToDevice, s));
                CU(cudaMemcpyAsync(nF, D.fg, D.maps_rows * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
            }
            CU(cudaStreamSynchronize(s));
            if (D.T) CU(cudaFree(D.T));
            if (D.maps) CU(cudaFree(D.maps));
            if (D.fg) CU(cudaFree(D.fg));
            D.T = nT;
            D.maps = nM;
            D.fg = nF;
            D.cap_rows = cap;
        }
        CU(cudaMemcpyAsync(D.T, Z.T.data(), static_cast<size_t>(Z.nS) * C * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        if (D.maps_rows < Z.nS) {
            CU(cudaMemcpyAsync(D.maps + D.maps_rows * nD, Z.maps.data() + D.maps_rows * nD,
                               (Z.nS - D.maps_rows) * nD * sizeof(uint16_t), cudaMemcpyHostToDevice, s));
            CU(cudaMemcpyAsync(D.fg + D.maps_rows, Z.fg.data() + D.maps_rows, (Z.nS - D.maps_rows) * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, s));
            D.maps_rows = Z.nS;
        }
        return SFA_OK;
    };
    cudaError_t e = sfa::lazy_init(n, p, D.state, D.pos, D.fd, h->sm_count, s);
    if (e != cudaSuccess) return cuda_fail(e, "lazy init");
    std::vector<uint64_t> hpos(p), hend(p);
    std::vector<uint32_t> hstate(p), stalled;
    for (uint64_t g = 0; g < p; ++g) hend[g] = (g + 1) * (n / p) + std::min<uint64_t>(g + 1, n % p);
    const uint32_t K = 4096;  // bytes of text the host builds ahead per stalled chunk and round
    std::vector<uint8_t> hwin;
    uint32_t counts[2] = {0, 0};
    for (int round = 0;; ++round) {
        int rc = sync_tables();
        if (rc) return rc;
        sfa::LazyScanArgs la;
        la.T = D.T, la.fg = D.fg, la.drow = D.dfa, la.cls = D.cls, la.C = C, la.nD = nD, la.factor = factor;
        la.text = d_text, la.n = n, la.p = p, la.state = D.state, la.pos = D.pos, la.fd = D.fd, la.counts = D.counts;
        CU(cudaMemsetAsync(D.counts, 0, 2 * sizeof(uint32_t), s));
        e = sfa::lazy_scan(la, s);
        if (e != cudaSuccess) return cuda_fail(e, "lazy scan");
        CU(cudaMemcpyAsync(counts, D.counts, sizeof(counts), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (counts[0] == 0) break;  // nothing stalled
        CU(cudaMemcpyAsync(hpos.data(), D.pos, p * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hstate.data(), D.state, p * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        stalled.clear();
        for (uint64_t g = 0; g < p; ++g)
            if (hpos[g] < hend[g]) stalled.push_back(static_cast<uint32_t>(g));
        if (stalled.empty()) break;
        // the windows the host builds from (at most 128 MiB of them per round:
        // the other stalled chunks wait for the next round)
        const size_t max_chunks = std::max<size_t>(1, (128u << 20) / K);
        if (stalled.size() > max_chunks) stalled.resize(max_chunks);
        const size_t need = stalled.size() * static_cast<size_t>(K);
        if (D.cap_win < need) {
            if (D.win) CU(cudaFree(D.win));
            D.win = nullptr;
            D.cap_win = 0;
            CU(cudaMalloc(&D.win, need));
            D.cap_win = need;
        }
        hwin.resize(need);
        CU(cudaMemcpyAsync(D.idx, stalled.data(), stalled.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        e = sfa::lazy_gather(d_text, n, p, D.pos, D.idx, static_cast<uint32_t>(stalled.size()), K, D.win, s);
        if (e != cudaSuccess) return cuda_fail(e, "lazy gather");
        CU(cudaMemcpyAsync(hwin.data(), D.win, need, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        const auto t0 = std::chrono::steady_clock::now();
        try {
            for (size_t j = 0; j < stalled.size(); ++j) {
                const uint32_t g = stalled[j];
                const uint64_t len = std::min<uint64_t>(K, hend[g] - hpos[g]);
                Z.run(hstate[g], hwin.data() + j * static_cast<size_t>(K), len, factor);
            }
        } catch (const sfa::CompileError& ce) {
            return fail(ce.code, ce.what());
        } catch (const std::bad_alloc&) {
            return fail(SFA_ERR_OOM, "host allocation failed while building SFA states");
        }
        h->lazy_build_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    // f_fin = f_1 . ... . f_p on the device, q_final = f_fin(q0): by single
    // lookups when every chunk ended factored, else as mapping vectors
    e = counts[1] == 0 ? sfa::lazy_cfold(D.maps, D.absorbing, nD, D.state, D.fd, p, D.cbuf, D.fin, s)
                       : sfa::lazy_fold(D.maps, D.state, D.fd, D.absorbing, p, nD, D.fold, D.fin, h->sm_count, s);
    if (e != cudaSuccess) return cuda_fail(e, "lazy fold");
    uint16_t q16 = 0;
    CU(cudaMemcpyAsync(&q16, D.fin, sizeof(uint16_t), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    *final_state = q16;
    *accept = Z.dfinal[q16];
    return SFA_OK;
}

#ifdef SFA_STAMPS
// Diagnostic builds only (include/sfa_diag.h): the stamps of the last TMA scan.
SFA_API int sfa_diag_counters(const sfa_handle* h, uint64_t* host, size_t n) {
    if (!h || !h->dstamps) return fail(SFA_ERR_INVALID_ARG, "no stamps");
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(host, h->dstamps + kMaxSlots * 16, std::min<size_t>(n, 16) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return SFA_OK;
}
SFA_API int sfa_diag_stamps(const sfa_handle* h, uint64_t* host, size_t n) {
    if (!h || !h->dstamps) return fail(SFA_ERR_INVALID_ARG, "no stamps");
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(host, h->dstamps, std::min<size_t>(n, kMaxSlots * 16) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return SFA_OK;
}
#endif

}  // extern "C"
