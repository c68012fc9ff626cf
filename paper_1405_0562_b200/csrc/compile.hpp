// compile.hpp -- host-side automaton construction for the SFA matcher.
//
// regex --(parse, C10)--> tree --(Glushkov / McNaughton-Yamada,
// PAPER.md:644-645)--> position NFA --(Alg. 1)--> DFA
// --(Hopcroft minimisation; "minimized DFA")--> canonical
// numbering (C3) --(byte classes)--> D-SFA by Alg. 4 in its DFA form
// with canonical numbering of the mappings.
//
// Host only, not timed.  Shares no code with oracle/.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace sfa {

struct CompileError : std::runtime_error {
    int code;  // sfa_status
    CompileError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct Automata {
    // ---- minimal complete DFA over all 256 bytes (canonical ids) ----
    uint32_t nD = 0;                 // |D| (dead state counted)
    int32_t dead = -1;               // canonical dead id or -1
    std::vector<uint32_t> dfa;       // nD * 256
    std::vector<uint8_t> dfa_final;  // nD
    uint32_t nfa_positions = 0, subset_states = 0;

    // ---- byte classes of the minimal DFA (columns of the SFA table) ----
    uint32_t C = 0;
    uint8_t cls[256] = {};           // byte -> class; classes numbered by smallest byte
    uint8_t rep_byte[256] = {};      // class -> representative byte (smallest Sigma byte, else smallest)
    uint8_t sigma[32] = {};          // Sigma bitset

    // ---- D-SFA (Alg. 4), canonical ids, f_I = 0 ----
    uint32_t nS = 0;
    std::vector<uint32_t> T;         // nS * C   next SFA id
    std::vector<uint32_t> maps;      // nS * nD  mapping f_s (row s)
    std::vector<uint32_t> img0;      // nS       f_s(q0)
    std::vector<uint8_t> acc;        // nS       f_s in F_s
    std::vector<uint32_t> rep_off;   // nS + 1   representative word of s (bytes)
    std::vector<uint8_t> rep;        //          a shortest word with f_I -w-> s
    uint32_t depth = 0;              // max |rep(s)|

    double dfa_seconds = 0, sfa_seconds = 0;

    // ---- N-SFA (compile_nsfa): T/rep/acc as above, but a state is a mapping
    // Q_N -> 2^Q_N of the Glushkov NFA (no `maps`); img0[s] = the minimal DFA's
    // state after rep(s) when the DFA was built (has_dfa), else s (and then
    // nD = nS, dfa_final = acc).  comp: the composition table by logical
    // matrix products (|S| <= 4096), else empty.
    bool nsfa = false, has_dfa = true;
    uint32_t nfa_states = 0;        // |Q_N| (Glushkov positions + the initial state)
    std::vector<uint32_t> comp;     // nS * nS
};

// Throws CompileError.  sigma == nullptr means all 256 bytes.
// build_sfa = false: the minimal DFA and its byte classes only.
Automata compile_regex(const std::string& regex, const uint8_t* sigma, int sigma_len, uint32_t max_sfa,
                       bool build_sfa = true);
// The N-SFA of the regex's Glushkov NFA by Alg. 4 in its general form
// (PAPER.md:481-521); the minimal DFA too when it has <= 2^20 states.
Automata compile_nsfa(const std::string& regex, const uint8_t* sigma, int sigma_len, uint32_t max_sfa);

}  // namespace sfa
