// lazy.hpp -- on-the-fly D-SFA construction (SURVEY s8(f)
// NEXT-4): the SFA is not built before matching; a state and a transition
// are created (Alg. 4 lines 6-8 for one (f, sigma)) only when a chunk of the
// text needs them.  Ids are 32-bit and in discovery order (f_I = 0), so an
// SFA far past the 65,535 states of the eager tables (r_500: 1,000,999,
// PAPER.md:754-756) can be matched with only its visited part built.
//
// Host side: the DFA (compile_regex without the SFA), the states built so far
// as u16 mapping vectors, their transition table (kUnknown = not built yet).
// Host only, shares no code with oracle/.
#pragma once

#include <cstdint>
#include <vector>

#include "compile.hpp"

namespace sfa {

constexpr uint32_t kUnknown = 0xffffffffu;
// T entries carry this bit when the target state is factorable (fg != kUnknown)
constexpr uint32_t kFactBit = 0x80000000u;

class LazySFA {
public:
    // A: the minimal DFA and its byte classes (compile_regex(..., build_sfa = false)); |D| <= 65535.
    LazySFA(const Automata& A, uint32_t max_states);

    uint32_t nD, C;
    uint8_t cls[256];
    std::vector<uint8_t> dfinal;      // nD
    uint32_t nS = 0;                  // states built
    std::vector<uint16_t> maps;       // nS * nD: f_s(q)
    std::vector<uint32_t> T;          // nS * C: next id | kFactBit, kUnknown = not built yet
    // Factored form (C24): fg[s] = g if every q whose image f_s(q)
    // is not absorbing has f_s(q) = g (all images absorbing: the first
    // absorbing state), else kUnknown.  From a factorable s the chunk runs on
    // the DFA alone: f_{s.w}(q) = absorbing[f_s(q)] ? f_s(q) : delta*(g, w).
    std::vector<uint32_t> fg;         // nS
    std::vector<uint8_t> absorbing;   // nD: delta(a, b) = a for every byte
    std::vector<uint16_t> dcls;       // nD * C: delta_d(q, class)
    uint64_t transitions = 0;         // transitions built
    uint32_t max_states;

    // Alg. 4 lines 6-8 for (s, c): f_next(q) = delta(f_s(q), c), interned; fills T[s][c].
    // Throws CompileError(capacity) past max_states.
    uint32_t step(uint32_t s, uint32_t c);
    // The SFA from state s over text[0, n), building every transition it meets;
    // with stop_factored it returns at the first factorable state.
    uint32_t run(uint32_t s, const uint8_t* text, size_t n, bool stop_factored);
    uint32_t next(uint32_t s, uint32_t c) const { return T[static_cast<size_t>(s) * C + c]; }  // raw entry
    uint32_t img0(uint32_t s) const { return maps[static_cast<size_t>(s) * nD]; }

private:
    uint32_t abs0 = kUnknown;         // the first absorbing state
    std::vector<uint32_t> slots;      // open addressing over maps
    uint64_t hash(const uint16_t* f) const;
    uint32_t intern(const uint16_t* f);
    std::vector<uint16_t> scratch;
};

}  // namespace sfa
