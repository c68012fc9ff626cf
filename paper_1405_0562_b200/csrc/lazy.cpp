// lazy.cpp -- on-the-fly D-SFA construction (see lazy.hpp).
#include "lazy.hpp"

#include <cstring>
#include <string>

namespace sfa {

LazySFA::LazySFA(const Automata& A, uint32_t max_states_) : nD(A.nD), C(A.C), max_states(max_states_) {
    if (nD > 65535) throw CompileError(3, "on-the-fly SFA needs |D| <= 65535");
    if (max_states > 0x7fffffffu) max_states = 0x7fffffffu;  // ids keep kFactBit free
    std::memcpy(cls, A.cls, 256);
    dfinal = A.dfa_final;
    dcls.resize(static_cast<size_t>(nD) * C);
    for (uint32_t q = 0; q < nD; ++q)
        for (uint32_t c = 0; c < C; ++c)
            dcls[static_cast<size_t>(q) * C + c] = static_cast<uint16_t>(A.dfa[static_cast<size_t>(q) * 256 + A.rep_byte[c]]);
    absorbing.assign(nD, 1);
    for (uint32_t q = 0; q < nD; ++q)
        for (int b = 0; b < 256 && absorbing[q]; ++b)
            if (A.dfa[static_cast<size_t>(q) * 256 + b] != q) absorbing[q] = 0;
    for (uint32_t q = 0; q < nD && abs0 == kUnknown; ++q)
        if (absorbing[q]) abs0 = q;
    slots.assign(1024, kUnknown);
    scratch.resize(nD);
    for (uint32_t q = 0; q < nD; ++q) scratch[q] = static_cast<uint16_t>(q);  // f_I (Def. 3)
    intern(scratch.data());
}

uint64_t LazySFA::hash(const uint16_t* f) const {
    uint64_t h = 0x9E3779B97F4A7C15ull;
    for (uint32_t q = 0; q < nD; ++q) h = (h ^ f[q]) * 0xBF58476D1CE4E5B9ull, h ^= h >> 29;
    return h;
}

uint32_t LazySFA::intern(const uint16_t* f) {
    if ((static_cast<size_t>(nS) + 1) * 2 > slots.size()) {
        std::vector<uint32_t> ns(slots.size() * 2, kUnknown);
        for (uint32_t s = 0; s < nS; ++s) {
            size_t k = hash(&maps[static_cast<size_t>(s) * nD]) & (ns.size() - 1);
            while (ns[k] != kUnknown) k = (k + 1) & (ns.size() - 1);
            ns[k] = s;
        }
        slots.swap(ns);
    }
    size_t k = hash(f) & (slots.size() - 1);
    while (slots[k] != kUnknown) {
        if (std::memcmp(&maps[static_cast<size_t>(slots[k]) * nD], f, nD * sizeof(uint16_t)) == 0) return slots[k];
        k = (k + 1) & (slots.size() - 1);
    }
    if (nS >= max_states) throw CompileError(3, "on-the-fly SFA reached " + std::to_string(max_states) + " states");
    slots[k] = nS;
    maps.insert(maps.end(), f, f + nD);
    uint32_t g = kUnknown;
    bool ok = true;
    for (uint32_t q = 0; q < nD && ok; ++q)
        if (!absorbing[f[q]]) {
            if (g == kUnknown) g = f[q];
            else ok = g == f[q];
        }
    fg.push_back(!ok ? kUnknown : g != kUnknown ? g : abs0);
    T.resize(T.size() + C, kUnknown);
    return nS++;
}

uint32_t LazySFA::step(uint32_t s, uint32_t c) {
    uint32_t& t = T[static_cast<size_t>(s) * C + c];
    if (t != kUnknown) return t & ~kFactBit;
    // line 6 (DFA form): f_next(q) = delta(f(q), sigma)
    const uint16_t* f = &maps[static_cast<size_t>(s) * nD];
    for (uint32_t q = 0; q < nD; ++q) scratch[q] = dcls[static_cast<size_t>(f[q]) * C + c];
    const uint32_t id = intern(scratch.data());  // may grow T: index again
    T[static_cast<size_t>(s) * C + c] = fg[id] != kUnknown ? id | kFactBit : id;  // line 7
    ++transitions;
    return id;
}

uint32_t LazySFA::run(uint32_t s, const uint8_t* text, size_t n, bool stop_factored) {
    for (size_t i = 0; i < n; ++i) {
        if (stop_factored && fg[s] != kUnknown) break;
        const uint32_t c = cls[text[i]];
        const uint32_t t = T[static_cast<size_t>(s) * C + c];
        s = t != kUnknown ? t & ~kFactBit : step(s, c);
    }
    return s;
}

}  // namespace sfa
