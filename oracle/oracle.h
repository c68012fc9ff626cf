/*
 * oracle.h -- CPU ORACLE for the SFA matcher.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load, call or execute anything under oracle/.
 * The product (paper_1405_0562_b200/) never includes, links or imports it,
 * and this file includes nothing from the product: the two share no code.
 *
 * What the oracle computes: for a regex and an alphabet
 * Sigma, the canonical minimal complete DFA and, for a text,
 *     q_final = delta^_d(q0, text)        (Alg. 2)
 *     accept  = [q_final in F_d]          (Def. 4/5)
 * plus, for SFA-level pins only, a plain D-SFA by correspondence construction
 * (Alg. 4) and a plain Alg. 5 run.
 *
 * Conventions:
 *   C2  Sigma = alphabet (NULL/-1 = all 256 bytes); '.' and [^..] range over
 *       Sigma; the DFA is complete over all 256 bytes, out-of-Sigma bytes go
 *       to an absorbing non-final dead state.
 *   C3  canonical ids: BFS from q0 over Sigma bytes in ascending byte value,
 *       numbering on first discovery; a dead state reachable only via
 *       out-of-Sigma bytes gets the last id.  Same rule for SFA mappings.
 *   C5  compose(f1,f2)[q] = f2[f1[q]]   (f1 . f2 := f2 o f1)
 *
 * Error codes: 0 ok, 1 syntax, 2 unsupported, 3 capacity, 4 invalid argument.
 */
#ifndef SFA_ORACLE_H
#define SFA_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_dfa oracle_dfa;
typedef struct oracle_sfa oracle_sfa;

/* regex -> Thompson NFA -> subset construction (Alg. 1) -> Moore minimisation
 * -> canonical numbering.  sigma_len < 0 means Sigma = all 256 bytes. */
int oracle_compile(const char* regex, const uint8_t* sigma, int sigma_len,
                   oracle_dfa** out, char* err, int errlen);
void oracle_free(oracle_dfa* d);

uint32_t oracle_nfa_states(const oracle_dfa* d);     /* Thompson NFA size   */
uint32_t oracle_subset_states(const oracle_dfa* d);  /* Alg. 1 output size  */
uint32_t oracle_dfa_states(const oracle_dfa* d);     /* complete minimal |D| */
int32_t  oracle_dfa_dead(const oracle_dfa* d);       /* dead id or -1       */
/* table: |D|*256 state ids (row-major), finals: |D| bytes (0/1) */
void oracle_dfa_export(const oracle_dfa* d, uint32_t* table, uint8_t* finals);

/* Alg. 2: sequential DFA run.  Returns accept (0/1), writes q_final. */
int oracle_run(const oracle_dfa* d, const uint8_t* text, uint64_t n, uint32_t* q_final);
/* Alg. 2 on each text i = texts[off[i] : off[i+1]). */
void oracle_run_batch(const oracle_dfa* d, const uint8_t* texts, const uint64_t* off,
                      uint64_t count, uint32_t* q_final, uint8_t* accept);

/* Alg. 3: speculative DFA per chunk [bounds[i], bounds[i+1]), i < p, with the
 * sequential reduction.  Returns accept (0/1) or -1 (allocation), writes
 * q_final and (maps != NULL) T_i[q] = delta^(q, chunk i) as p * |D| entries. */
int oracle_run_spec(const oracle_dfa* d, const uint8_t* text, const uint64_t* bounds, uint64_t p,
                    uint32_t* maps, uint32_t* q_final);

/* Brute-force language evaluator on the AST (position-set semantics), for
 * strings of length <= 62.  Returns 1 match, 0 no match, -code on error. */
int oracle_brute(const char* regex, const uint8_t* sigma, int sigma_len,
                 const uint8_t* s, int n);

/* oracle_brute on every string over chars[0..nchars) of length 0..maxlen in
 * shortlex order; out[i] = 0/1.  Returns the count or -code. */
int64_t oracle_brute_all(const char* regex, const uint8_t* sigma, int sigma_len,
                         const uint8_t* chars, int nchars, int maxlen, uint8_t* out);

/* Alg. 4 (correspondence construction, DFA simplification PAPER.md:495-499).
 * Returns 0 or 3 (capacity: more than cap mappings). */
int oracle_sfa_build(const oracle_dfa* d, uint32_t cap, oracle_sfa** out);
void oracle_sfa_free(oracle_sfa* s);
uint32_t oracle_sfa_states(const oracle_sfa* s);
/* table: |S|*256 SFA ids; maps: |S|*|D| DFA ids (row s = mapping f_s);
 * finals: |S| bytes, s in F_s (Def. 3). */
void oracle_sfa_export(const oracle_sfa* s, uint32_t* table, uint32_t* maps, uint8_t* finals);
/* Alg. 5 with explicit chunk boundaries bounds[0]=0 < ... bounds[p]=n
 * (non-decreasing).  Writes the per-chunk SFA ids (lines 1-5), the DFA state
 * from the sequential reduction (right column) and from the parallel
 * reduction f_fin = f_1 . ... . f_p, f_fin(q0) (left column). */
int oracle_sfa_run_chunked(const oracle_sfa* s, const uint8_t* text, const uint64_t* bounds,
                           int p, uint32_t* chunk_ids, uint32_t* q_seq, uint32_t* q_par);

/* NFA and N-SFA (NEXT-3).  The NFA: the Thompson NFA of a regex seen
 * eps-free (delta(q, b) = closure(move({q}, b)), I = closure({start}),
 * F = {end}), or an explicit eps-free NFA (n <= 64, delta[q*256+b] successor
 * bitsets).  The N-SFA: Alg. 4 in its general form (mappings Q -> 2^Q,
 * PAPER.md:501-521), canonical BFS ids (C3); Alg. 5 with both reductions,
 * the parallel one by logical matrix products.  Sets are
 * bitsets of ceil(n/64) words. */
typedef struct oracle_nfa oracle_nfa;
typedef struct oracle_nsfa oracle_nsfa;
int oracle_nfa_compile(const char* regex, const uint8_t* sigma, int sigma_len,
                       oracle_nfa** out, char* err, int errlen);
int oracle_nfa_explicit(int n, const uint64_t* delta, uint64_t I, uint64_t F, const uint8_t* sigma,
                        int sigma_len, oracle_nfa** out);
void oracle_nfa_free(oracle_nfa* a);
uint32_t oracle_nfa_size(const oracle_nfa* a);
int oracle_nfa_run(const oracle_nfa* a, const uint8_t* text, uint64_t n, uint64_t* final_set);
void oracle_nfa_word_map(const oracle_nfa* a, const uint8_t* w, int len, uint64_t* out);
int oracle_nsfa_build(const oracle_nfa* a, uint32_t cap, oracle_nsfa** out);
void oracle_nsfa_free(oracle_nsfa* s);
uint32_t oracle_nsfa_states(const oracle_nsfa* s);
int oracle_nsfa_run_chunked(const oracle_nsfa* s, const uint8_t* text, const uint64_t* bounds, int p,
                            uint32_t* chunk_ids, uint64_t* set_seq, uint64_t* set_par);

#ifdef __cplusplus
}
#endif
#endif
