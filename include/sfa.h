/*
 * sfa.h -- C-ABI of the B200-native SFA matcher (arXiv 1405.0562).
 *
 * The library (paper_1405_0562_b200/_lib/libsfa.so) runs the data-parallel hot
 * path of Alg. 5 of the paper ("Parallel computation of
 * SFA") on one NVIDIA B200 (sm_100a):
 *
 *   A1  byte -> table column                 (implementation; the paper indexes
 *                                             a 256-wide table)
 *   A2  chunk run from f_I, one lookup/byte  (Alg. 5 lines 1-5, PAPER.md:560-565,
 *                                             "looks up the transition table once
 *                                             for each character")
 *   A3  f_fin = f_1 . ... . f_p              (line 6; '.' is reverse
 *                                             composition f.g := g o f, PAPER.md:149,
 *                                             associative)
 *   A4  q_final = f_fin(q0), accept          (line 7; F_s)
 *   A5  batches of independent texts        ("naive" parallelism)
 *   A6  table residency (smem / L2)          (cache-miss cost)
 *
 * Any division of the text gives the same result (Theorem 3),
 * so results are bit-exact against the sequential DFA run (Alg. 2,
 * PAPER.md:259-272) of the canonical minimal complete DFA (C2/C3).
 *
 * Conventions
 *   - All functions return an sfa_status (0 = SFA_OK) except sfa_free and
 *     sfa_last_error.  No exception crosses the ABI.  On error a message is
 *     available from sfa_last_error() (thread-local, valid until the next call
 *     on the same thread).
 *   - "d_" pointers are CUDA device pointers on the handle's device; "h_"
 *     pointers and the plain output pointers are host memory.
 *   - stream is a cudaStream_t (0 = legacy default stream).
 *   - The handle owns its host tables, device tables and reusable device
 *     scratch.  The caller owns texts, offsets, results and streams.
 *   - A handle is immutable after sfa_compile except for sfa_set_residency.
 *     Matches on one handle may be issued from any host thread and stream:
 *     the library orders them on the device (a per-handle event makes each
 *     launch wait for the previous one's use of the shared scratch).
 */
#ifndef SFA_H
#define SFA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SFA_API __attribute__((visibility("default")))
#else
#define SFA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sfa_stream_t; /* == cudaStream_t */

typedef enum {
    SFA_OK = 0,
    SFA_ERR_SYNTAX = 1,        /* malformed regex; message has the byte position      */
    SFA_ERR_UNSUPPORTED = 2,   /* back-references, look-around, anchors */
    SFA_ERR_CAPACITY = 3,      /* NFA/DFA/SFA over the caps; |S| > 65535 (uint16 ids)  */
    SFA_ERR_INVALID_ARG = 4,   /* NULL handle/output, d_text NULL with n > 0, ...      */
    SFA_ERR_CUDA = 5,          /* a CUDA runtime/driver call failed                    */
    SFA_ERR_OOM = 6            /* host or device allocation failed                    */
} sfa_status;

/* Table residency (A6).  AUTO picks the fastest mode that fits. */
typedef enum {
    SFA_RES_AUTO = 0,
    SFA_RES_SMEM_PRIVATE = 1,  /* bank-private per-lane copies in shared memory     */
    SFA_RES_SMEM_SHARED = 2,   /* one copy of the class-compressed table in smem     */
    SFA_RES_HOT_L2 = 3,        /* frequent rows in smem, the rest from L2            */
    SFA_RES_L2 = 4             /* whole table from global memory (L2-resident)       */
} sfa_residency;

/* Composition of chunk states (A3).  AUTO: TABLE when |S| <= 4096, else VEC
 * when |D| <= 32, else REPLAY. */
typedef enum {
    SFA_COMPOSE_AUTO = 0,
    SFA_COMPOSE_VEC = 1,       /* mapping vectors, one lane per DFA state, warp shuffles (|D| <= 32) */
    SFA_COMPOSE_TABLE = 2,     /* SFA ids; composition table comp[a][b] built on the host (|S| <= 4096) */
    SFA_COMPOSE_REPLAY = 3     /* SFA ids; s_a . s_b = delta_s^(s_a, rep(s_b)) (Lemma 1) */
} sfa_compose;

typedef struct sfa_handle sfa_handle;

/* One result per text: the DFA state q_final (canonical id, C3) and
 * accept = [q_final in F_d] (0/1).  8 bytes. */
typedef struct {
    uint32_t final_state;
    uint32_t accept;
} sfa_result;

typedef struct {
    uint32_t nfa_positions;    /* Glushkov positions (McNaughton-Yamada) */
    uint32_t dfa_subset_states;/* Alg. 1 output before minimisation              */
    uint32_t dfa_states;       /* complete minimal |D| (dead state counted)      */
    uint32_t dfa_live;         /* |D| without the dead state                     */
    uint32_t dead_state;       /* canonical id of the dead state, UINT32_MAX if none */
    uint32_t sfa_states;       /* |S| by Alg. 4 (constant-dead mapping counted)  */
    uint32_t classes;          /* byte classes C (table columns)                 */
    uint32_t sfa_depth;        /* longest shortest word f_I -> f (replay bound)  */
    uint32_t residency;        /* effective sfa_residency for single texts       */
    uint32_t compose_mode;     /* effective sfa_compose (VEC, TABLE or REPLAY)   */
    uint32_t range_lo, range_width; /* byte window of the PRIVATE layout (0 if n/a) */
    uint64_t device_table_bytes;    /* bytes of SFA tables held on the device    */
    double   dfa_seconds, sfa_seconds; /* host construction times (not the target) */
    uint32_t kind;             /* 0: D-SFA (sfa_compile), 1: N-SFA (sfa_compile_nsfa), 2: on the fly (sfa_compile_lazy) */
    uint32_t nfa_states;       /* N-SFA: |Q_N| of the Glushkov NFA (positions + initial) */
    uint32_t has_dfa;          /* 1: results carry the minimal DFA's canonical state */
    uint64_t lazy_transitions; /* on the fly: SFA transitions built so far (sfa_states: states built) */
    double   lazy_seconds;     /* on the fly: host time spent building them inside sfa_match_lazy */
    uint32_t dfa_window_copies;/* FACTORED step: lane-group copies of the DFA window (32: bank-private
                                  or MIXED; 0 before the first device call or without it)       */
    uint32_t dfa_window_hot;   /* MIXED layout: DFA states in 32 bank-private copies (0: not MIXED) */
} sfa_info_t;

/*
 * sfa_compile -- regex -> Glushkov NFA -> Alg. 1 subset construction
 * -> minimisation -> canonical numbering ->
 * Alg. 4 correspondence construction in its DFA form ->
 * byte classes, device tables (uploaded to the current CUDA device).
 *
 *   regex        NUL-terminated pattern, grammar of DESIGN.md C10; full-match.
 *   alphabet     bytes of Sigma; NULL = all 256 bytes (C2).
 *   alphabet_len number of bytes at `alphabet`; ignored when alphabet is NULL.
 *   max_sfa      cap on |S| (0 = default 65535, the uint16 id limit).
 *   out          receives the handle; *out = NULL on error.
 * Errors: SYNTAX, UNSUPPORTED, CAPACITY, INVALID_ARG, CUDA, OOM.
 */
SFA_API int sfa_compile(const char* regex, const uint8_t* alphabet, int alphabet_len,
                uint32_t max_sfa, sfa_handle** out);

/*
 * sfa_compile_nsfa -- the N-SFA: Alg. 4 in its general form
 * over the regex's Glushkov NFA N, a state being a mapping
 * Q_N -> 2^Q_N (|Q_N| bitset rows), with no DFA in between; the composition
 * '.' is the logical matrix product, built on the host into the
 * composition table when |S| <= 4096 (else Lemma-1 replay on the device).
 * Matching runs through the same kernels and calls as a D-SFA handle.  The
 * minimal DFA is also built when it has <= 2^20 states (info.has_dfa): results
 * then carry its canonical state (the DFA state of f_fin(I)); otherwise
 * final_state is the N-SFA id and accept = [f_fin in F_s].  Not available on
 * N-SFA handles (CAPACITY): VEC composition, sfa_match_map, sfa_match_host,
 * sfa_match_speculative, sfa_export_sfa's maps.  Arguments and errors as
 * sfa_compile.
 */
SFA_API int sfa_compile_nsfa(const char* regex, const uint8_t* alphabet, int alphabet_len,
                             uint32_t max_sfa, sfa_handle** out);

/*
 * On-the-fly construction.
 *
 * sfa_compile_lazy -- builds only the minimal DFA (Alg. 1 + minimisation);
 * the D-SFA is built while matching, one state and one transition at a time
 * (Alg. 4 lines 6-8 for the (f, sigma) a chunk of text meets), with 32-bit ids
 * in discovery order, so SFAs far beyond the eager tables' 65,535 states
 * (r_500: 1,000,999) match with only their visited part
 * built.  max_states: cap on states built (0 = 2^24; CAPACITY when reached
 * during a match).  Needs |D| <= 65535.  Such a handle only matches with
 * sfa_match_lazy (the other calls return INVALID_ARG); sfa_info reports kind
 * 2, the states and transitions built, and the host time spent building.
 *
 * sfa_match_lazy -- one text in device memory (d_text, n bytes, caller-owned),
 * blocking: rounds of a device scan of every unfinished chunk (SPEC's rule,
 * <= 1024 chunks per SM) that stops at the first transition not built yet,
 * and host construction of the transitions the stalled chunks need (the next
 * 4 KiB of text of each); then the chunk states are folded as mapping vectors
 * (a pairwise tree of (f . g)(q) = g(f(q))) and applied to q0.
 * Factored chunk runs (C24; on unless tuning no_factor, and only
 * when |D| x classes x 2 B <= 48 KiB): a chunk that reaches a factorable
 * state s (every non-absorbing image equal to one g) runs the DFA alone from
 * g to its end and no state past s is built; when every chunk ends factored
 * the fold takes one lookup per composition.  Results are the canonical
 * (q_final, accept) of Alg. 2 (Theorem 2) either way.  Built states persist
 * in the handle.
 */
SFA_API int sfa_compile_lazy(const char* regex, const uint8_t* alphabet, int alphabet_len, uint32_t max_states,
                             sfa_handle** out);
SFA_API int sfa_match_lazy(const sfa_handle* h, const uint8_t* d_text, size_t n, sfa_stream_t stream,
                           uint32_t* final_state, int* accept);

/* Releases the handle and its device memory (synchronises the device work
 * that used it).  NULL is a no-op. */
SFA_API void sfa_free(sfa_handle* h);

/* Thread-local message of the last failing call on this thread ("" if none). */
SFA_API const char* sfa_last_error(void);

SFA_API int sfa_info(const sfa_handle* h, sfa_info_t* info);

/*
 * sfa_match -- one text in device memory (Alg. 5 with the device tree
 * reduction).  Blocking: returns after the result is on the host (it
 * synchronises `stream`).  n == 0 returns (q0 = 0, [eps in L]) with no launch.
 *   d_text       device pointer to n bytes (any alignment), caller-owned.
 *   final_state  host out: q_final.   accept: host out, 0/1.
 */
SFA_API int sfa_match(const sfa_handle* h, const uint8_t* d_text, size_t n, sfa_stream_t stream,
              uint32_t* final_state, int* accept);

/* Same work as sfa_match, stream-ordered and non-blocking: the result is
 * written to device memory d_result (8 bytes, caller-owned) when the stream
 * reaches it (n == 0 included: a one-thread kernel writes it).  No host
 * synchronisation, no host<->device copy: suitable for CUDA-event timing and
 * graph capture. */
SFA_API int sfa_match_async(const sfa_handle* h, const uint8_t* d_text, size_t n, sfa_stream_t stream,
                    sfa_result* d_result);

/*
 * sfa_match_batch -- count independent texts (A5, the "naive" parallelism over
 * data of PAPER.md:67-70), text i = d_texts[d_offsets[i] : d_offsets[i+1]).
 *   d_texts    device pointer the offsets index (any alignment), caller-owned.
 *   d_offsets  count+1 uint64, device, caller-owned; must be non-decreasing.
 *   d_results  count sfa_result, device, caller-owned.
 * Async and stream-ordered: the call only enqueues work (no host read of the
 * offsets, no synchronisation).  The texts, back to back, are scanned as one
 * range by the TMA pipeline with every text boundary honoured in place; a
 * device-side plan kernel validates the offsets.  If any pair decreases (or
 * d_offsets[count] < d_offsets[0]) EVERY result is written as
 * {SFA_INVALID_STATE, 0}.  count == 0 is a no-op; an empty text gives
 * (0, [eps in L]).  Scratch is per handle (matches on one handle serialise).
 * Errors (returned): INVALID_ARG (NULL pointers, count > 2^31), CAPACITY, CUDA.
 */
#define SFA_INVALID_STATE 0xffffffffu
SFA_API int sfa_match_batch(const sfa_handle* h, const uint8_t* d_texts, const uint64_t* d_offsets,
                    size_t count, sfa_stream_t stream, sfa_result* d_results);

/*
 * sfa_match_batch_uniform -- `count` texts of `len` bytes each, back to back
 * at d_texts (device, any alignment; text i = d_texts[i*len : (i+1)*len)).
 * Same results as sfa_match_batch with offsets i*len and the same kernel; the
 * plan is made on the host (no offsets array).  Async, stream-ordered.
 */
SFA_API int sfa_match_batch_uniform(const sfa_handle* h, const uint8_t* d_texts, size_t len, size_t count,
                            sfa_stream_t stream, sfa_result* d_results);

/*
 * Sharded matching (one text split over several GPUs / streams; Theorem 3,
 * PAPER.md:469-479, and Lemma 1).
 *
 * sfa_match_map -- like sfa_match_async, but writes the text's whole SFA
 * state as its mapping: d_map[q] = f_text(q) = delta^_d(q, text) for every
 * DFA state q (|D| = sfa_info().dfa_states u32 entries, device, caller-owned).
 * Async, stream-ordered.  n == 0 writes the identity (f_I).  CAPACITY if the
 * handle keeps no mapping table (|S| * |D| > 2^29).
 *
 * sfa_combine_maps -- the reduction over `count` shard mappings in text
 * order (d_maps: count * |D| u32, device; e.g. an all-gather of every rank's
 * sfa_match_map): q = q0; q = d_maps[r * |D| + q] for r = 0..count-1, the
 * sequential reduction of Alg. 5 (right column); writes
 * (q, [q in F_d]) to d_result (device).  Async, stream-ordered.
 */
SFA_API int sfa_match_map(const sfa_handle* h, const uint8_t* d_text, size_t n, sfa_stream_t stream, uint32_t* d_map);
SFA_API int sfa_combine_maps(const sfa_handle* h, const uint32_t* d_maps, size_t count, sfa_stream_t stream,
                     sfa_result* d_result);

/*
 * sfa_match_speculative -- the paper's BASELINE, not the SFA: Alg. 3
 * (PAPER.md:293-328), the DFA run speculatively from every state.  The text
 * is cut into `nchunks` chunks by SPEC's rule (0 = as many as fill the GPU;
 * > n means n one-byte chunks, C6); chunk i yields the mapping
 * T_i[q] = delta^_d(q, chunk_i) for every DFA state q (|D| dependent lookups
 * per byte), the T_i are composed in text order and
 * (q_final = T[q0], [q_final in F_d]) is written to d_result (device).
 * d_chunk_maps (device, nullable): receives T_i as min(nchunks, max(n, 1)) * |D|
 * u32, row i = chunk i; it needs nchunks > 0 (INVALID_ARG otherwise: the
 * automatic count is not reported).  Async, stream-ordered.  n == 0:
 * (0, [eps in L]) and, with d_chunk_maps, the identity in row 0.
 * Same result as sfa_match_async for every input (Theorem 2).
 */
SFA_API int sfa_match_speculative(const sfa_handle* h, const uint8_t* d_text, size_t n, uint64_t nchunks,
                          sfa_stream_t stream, uint32_t* d_chunk_maps, sfa_result* d_result);

/*
 * sfa_match_host -- end-to-end call on a HOST buffer (pinned or pageable):
 * the text is copied to the device in slices on `stream` while earlier slices
 * are matched (each slice yields one SFA state; slices compose by Lemma 1,
 * PAPER.md:441), then the result is read back.  Blocking.
 */
SFA_API int sfa_match_host(const sfa_handle* h, const uint8_t* h_text, size_t n, sfa_stream_t stream,
                   uint32_t* final_state, int* accept);

/*
 * sfa_match_batch_host -- end-to-end sfa_match_batch on HOST buffers (pinned
 * or pageable): texts h_texts[h_offsets[i] : h_offsets[i+1]) (h_offsets:
 * count+1 uint64, host, non-decreasing: checked, INVALID_ARG otherwise), the
 * results to h_results (count entries, host).  The texts go to the device in
 * slices of whole texts (<= max(64 MiB, the longest text), <= 2^20 texts) on a
 * copy stream while the previous slice is matched on `stream`.  Blocking.
 */
SFA_API int sfa_match_batch_host(const sfa_handle* h, const uint8_t* h_texts, const uint64_t* h_offsets, size_t count,
                                 sfa_stream_t stream, sfa_result* h_results);

/*
 * Test / diagnostic knobs.
 *
 * sfa_match_chunked -- divides the text into exactly `nchunks` chunks by
 * SPEC's rule (floor(n/p) bytes, the remainder to the leading chunks; if
 * n < p, n one-byte chunks; C6), runs each from f_I on the device,
 * reduces on the device, and optionally returns the per-chunk SFA states
 * (canonical ids, host array of min(nchunks, max(n,1)) entries).  Blocking.
 */
SFA_API int sfa_match_chunked(const sfa_handle* h, const uint8_t* d_text, size_t n, uint32_t nchunks,
                      sfa_stream_t stream, uint32_t* final_state, int* accept, uint32_t* h_chunk_states);

/*
 * sfa_match_rows -- diagnostic view of the TMA scan (the kernel sfa_match
 * times for texts >= 4 MiB), forced for any n >= 64 KiB: writes the canonical
 * SFA id of every row (chunk) to d_row_ids (device, row_cap u32, caller-owned;
 * CAPACITY if the plan has more rows), the result to d_result (device) and the
 * row geometry to *plan (host): head piece [0, head), rows [head + r*row_len,
 * head + (r+1)*row_len) for r < rows, tail [tail_start, n).  The ids are
 * Alg. 5 lines 1-5 per chunk (Lemma 1 / Thm. 3,
 * PAPER.md:434-479).  Async, stream-ordered.
 */
typedef struct {
    uint64_t head, row_len, rows, tail_start;
    uint32_t ctas, rows_hi, rows_lo, ctas_hi;  /* the first ctas_hi CTAs scan rows_hi rows, the rest rows_lo */
} sfa_rows_plan;
SFA_API int sfa_match_rows(const sfa_handle* h, const uint8_t* d_text, size_t n, sfa_stream_t stream,
                           uint32_t* d_row_ids, size_t row_cap, sfa_rows_plan* plan, sfa_result* d_result);

/* Forces a residency mode (SFA_RES_*); CAPACITY if it does not fit. */
SFA_API int sfa_set_residency(sfa_handle* h, int mode);

/* HOT residency: re-ranks the SFA states by their visit frequency on a
 * sample of text (the first min(n, 8 MiB) bytes of d_sample, device memory,
 * caller-owned; copied to the host on `stream`), so the most visited rows sit
 * in shared memory.  Blocking: waits for earlier work of the handle, then
 * rewrites the HOT tables.  n == 0 restores the static ranking (the default:
 * no match call ever tunes on its own).  Results never depend on the ranking. */
SFA_API int sfa_tune_residency(sfa_handle* h, const uint8_t* d_sample, size_t n, sfa_stream_t stream);

/* Forces a composition mode (SFA_COMPOSE_*); CAPACITY if the handle cannot
 * use it (VEC needs |D| <= 32, TABLE |S| <= 4096).  Results do not depend on
 * it (composition is exact); only the epilogue cost does. */
SFA_API int sfa_set_compose(sfa_handle* h, int mode);

/*
 * sfa_set_tuning -- launch-shape knobs for measurements and tests (NULL or a
 * zeroed struct = automatic).  None of them can change a result: every shape
 * computes the same exact Alg. 5.  Blocking: waits for the handle's device
 * work and drops its device tables (rebuilt by the next device call).
 * INVALID_ARG for a value out of range.  The library reads no environment
 * variable.
 */
typedef struct {
    int32_t tma_k;            /* chunks per compute thread of the TMA scan: 0 auto, 1 or 2     */
    int32_t tma_rowb;         /* bytes per row per pipeline stage: 0 auto, 16/32/64 (needs tma_k) */
    int32_t tma_ring;         /* cap on the stage-ring depth: 0 = as deep as fits, 2..8        */
    int32_t tma_promo;        /* L2 promotion of the TMA loads: 0 none (auto), 64, 128, 256    */
    uint32_t hot_rows;        /* HOT residency: cap on the rows kept in smem (0 = all that fit) */
    uint32_t no_factor;       /* 1: never use the FACTORED step (nor factored on-the-fly runs)  */
    uint32_t dfa_copies;      /* FACTORED: cap on lane-group copies of the DFA window (0 = 32)  */
    uint32_t private_copies;  /* PRIVATE: cap on lane-group copies of the SFA table (0 = 32)    */
    uint32_t row_align;       /* TMA row length alignment: 0 auto, 64, 128 or 256              */
    uint32_t direct_piece;    /* bytes per thread of the short-text kernel: 0 auto, 16..4096   */
    uint32_t dfa_u8;          /* FACTORED: 1 = 32 bank-private u8 copies of the DFA window when
                                 32 u16 copies do not fit (|D| <= 256, state-major); 0 = auto:
                                 u16 layouts, the u8 copies only where MIXED is not chosen      */
    uint32_t dfa_layout;      /* FACTORED u16 layout when 32 copies do not fit: 0 auto, 1 = R
                                 lane-group copies, 2 = MIXED (the most visited DFA states in 32
                                 bank-private copies, every state in one shared copy)          */
    uint32_t dfa_hot;         /* MIXED: cap on the bank-private DFA states (0 = all that fit)   */
    uint32_t fact_fold;       /* FACTORED chunk values in the folds: 0 auto (marked sets in smem
                                 when small), 1 = marked sets read from global memory, 2 = off
                                 (canonical SFA ids, as before round 2b)                         */
} sfa_tuning_t;
SFA_API int sfa_set_tuning(sfa_handle* h, const sfa_tuning_t* t);

/* Minimal DFA over all 256 bytes: table |D|*256 canonical ids, finals |D| (0/1). */
SFA_API int sfa_export_dfa(const sfa_handle* h, uint32_t* table, uint8_t* finals);

/* D-SFA: table |S|*256 canonical SFA ids, maps |S|*|D| (row s = f_s),
 * finals |S| (s in F_s).  Any pointer may be NULL.  On-the-fly handles: the
 * states built so far (sfa_info().sfa_states, discovery order), transitions
 * not built yet as UINT32_MAX. */
SFA_API int sfa_export_sfa(const sfa_handle* h, uint32_t* table, uint32_t* maps, uint8_t* finals);

#ifdef __cplusplus
}
#endif
#endif /* SFA_H */
