// compile.cpp -- regex -> minimal DFA -> D-SFA (host, C++17).  See compile.hpp.
#include "compile.hpp"

#include <algorithm>
#include <array>
#include <cctype>
#include <chrono>
#include <cstring>
#include <deque>
#include <unordered_map>

namespace sfa {
namespace {

constexpr int kSyntax = 1, kUnsupported = 2, kCapacity = 3;
constexpr int kMaxRepeat = 1000;
constexpr uint32_t kMaxPositions = 16384;
constexpr uint32_t kMaxDfa = 1u << 20;
constexpr size_t kMaxNodes = 4u << 20;

using ByteSet = std::array<uint64_t, 4>;

inline bool bs_has(const ByteSet& s, int b) { return (s[b >> 6] >> (b & 63)) & 1; }
inline void bs_set(ByteSet& s, int b) { s[b >> 6] |= 1ull << (b & 63); }
inline ByteSet bs_range(int lo, int hi) {
    ByteSet s{};
    for (int b = lo; b <= hi; ++b) bs_set(s, b);
    return s;
}
inline ByteSet bs_not(ByteSet s) {
    for (auto& w : s) w = ~w;
    return s;
}
inline ByteSet bs_or(ByteSet a, const ByteSet& b) {
    for (int i = 0; i < 4; ++i) a[i] |= b[i];
    return a;
}

// ------------------------------------------------------------------------------------------
// Regex tree.  Bounded repeats are expanded into copies so every leaf is one
// Glushkov position.
// ------------------------------------------------------------------------------------------
enum class K : uint8_t { Chars, Eps, Cat, Alt, Star };
struct Node {
    K k;
    ByteSet set{};          // Chars: bytes (intersected with Sigma)
    std::vector<int> kids;  // Cat / Alt: >= 2 children; Star: 1
};

class Parser {
public:
    Parser(const std::string& src, const ByteSet& sigma, std::vector<Node>& out)
        : s_(src), sigma_(sigma), nodes_(out) {}

    int parse() {
        int r = alternation(0);
        if (i_ != s_.size()) fail(kSyntax, s_[i_] == ')' ? "unbalanced ')'" : "unexpected character");
        return r;
    }

private:
    const std::string& s_;
    ByteSet sigma_;
    std::vector<Node>& nodes_;
    size_t i_ = 0;

    [[noreturn]] void fail(int code, const char* what) const {
        throw CompileError(code, std::string(what) + " at " + std::to_string(i_));
    }
    bool done() const { return i_ >= s_.size(); }
    int cur() const { return done() ? -1 : static_cast<unsigned char>(s_[i_]); }

    int make(K k, std::vector<int> kids = {}, ByteSet set = {}) {
        if (nodes_.size() >= kMaxNodes) fail(kCapacity, "regex too large after repeat expansion");
        Node n;
        n.k = k;
        n.kids = std::move(kids);
        if (k == K::Chars)
            for (int w = 0; w < 4; ++w) n.set[w] = set[w] & sigma_[w];
        nodes_.push_back(std::move(n));
        return static_cast<int>(nodes_.size()) - 1;
    }
    int clone(int x) {
        Node n = nodes_[x];  // copy (the vector may reallocate below)
        for (auto& c : n.kids) c = clone(c);
        if (nodes_.size() >= kMaxNodes) fail(kCapacity, "regex too large after repeat expansion");
        nodes_.push_back(std::move(n));
        return static_cast<int>(nodes_.size()) - 1;
    }

    int alternation(int depth) {
        if (depth > 1000) fail(kCapacity, "nesting too deep");
        std::vector<int> alts{sequence(depth)};
        while (cur() == '|') {
            ++i_;
            alts.push_back(sequence(depth));
        }
        return alts.size() == 1 ? alts[0] : make(K::Alt, std::move(alts));
    }

    static bool quantifier(int c) { return c == '*' || c == '+' || c == '?' || c == '{'; }

    int sequence(int depth) {
        std::vector<int> items;
        for (;;) {
            int c = cur();
            if (c < 0 || c == '|' || c == ')') break;
            if (quantifier(c)) fail(kSyntax, "dangling quantifier");
            items.push_back(postfix(depth));
        }
        if (items.empty()) return make(K::Eps);
        return items.size() == 1 ? items[0] : make(K::Cat, std::move(items));
    }

    int number() {
        if (!(cur() >= '0' && cur() <= '9')) fail(kSyntax, "bad repeat");
        long v = 0;
        while (cur() >= '0' && cur() <= '9') {
            v = std::min<long>(v * 10 + (cur() - '0'), 1000000);
            ++i_;
        }
        return static_cast<int>(v);
    }

    // x{lo,hi} (hi < 0: unbounded): lo copies, then x* or nested optionals.
    int repeat(int x, int lo, int hi) {
        std::vector<int> parts;
        for (int j = 0; j < lo; ++j) parts.push_back(j == 0 ? x : clone(x));
        if (hi < 0) {
            parts.push_back(make(K::Star, {lo == 0 ? x : clone(x)}));
        } else if (hi > lo) {
            // (x(x(x)?)?)? with hi-lo copies
            int tail = -1;
            for (int j = 0; j < hi - lo; ++j) {
                int xc = (lo == 0 && j == hi - lo - 1) ? x : clone(x);
                int body = tail < 0 ? xc : make(K::Cat, {xc, tail});
                tail = make(K::Alt, {body, make(K::Eps)});
            }
            parts.push_back(tail);
        }
        if (parts.empty()) return make(K::Eps);
        return parts.size() == 1 ? parts[0] : make(K::Cat, std::move(parts));
    }

    int postfix(int depth) {
        int x = primary(depth);
        for (;;) {
            int c = cur();
            if (c == '*') { ++i_; x = make(K::Star, {x}); }
            else if (c == '+') { ++i_; x = repeat(x, 1, -1); }
            else if (c == '?') { ++i_; x = repeat(x, 0, 1); }
            else if (c == '{') {
                ++i_;
                int lo = number(), hi;
                if (cur() == '}') hi = lo;
                else if (cur() == ',') {
                    ++i_;
                    hi = (cur() == '}') ? -1 : number();
                } else fail(kSyntax, "bad repeat");
                if (cur() != '}') fail(kSyntax, "bad repeat");
                ++i_;
                if (hi >= 0 && hi < lo) fail(kSyntax, "repeat {m,n} with m > n");
                if (lo > kMaxRepeat || hi > kMaxRepeat) fail(kCapacity, "repeat count too large");
                x = repeat(x, lo, hi);
            } else break;
        }
        return x;
    }

    static bool class_escape(int c, ByteSet& out) {
        switch (c) {
            case 'd': out = bs_range('0', '9'); return true;
            case 'D': out = bs_not(bs_range('0', '9')); return true;
            case 'w': case 'W': {
                ByteSet w = bs_or(bs_or(bs_range('0', '9'), bs_range('a', 'z')), bs_range('A', 'Z'));
                bs_set(w, '_');
                out = c == 'w' ? w : bs_not(w);
                return true;
            }
            case 's': case 'S': {
                ByteSet w{};
                for (int b : {' ', '\t', '\n', '\r', '\f', '\v'}) bs_set(w, b);
                out = c == 's' ? w : bs_not(w);
                return true;
            }
        }
        return false;
    }
    static int hex(int c) {
        if (c >= '0' && c <= '9') return c - '0';
        if (c >= 'a' && c <= 'f') return c - 'a' + 10;
        if (c >= 'A' && c <= 'F') return c - 'A' + 10;
        return -1;
    }
    // After '\'.  Returns a byte, or -1 with `set` filled for \d-style escapes.
    int escape(ByteSet& set) {
        if (done()) fail(kSyntax, "trailing backslash");
        int c = cur();
        ++i_;
        if (class_escape(c, set)) return -1;
        switch (c) {
            case 'n': return '\n';
            case 't': return '\t';
            case 'r': return '\r';
            case 'f': return '\f';
            case 'v': return '\v';
            case 'x': {
                int h = i_ + 1 < s_.size() ? hex(static_cast<unsigned char>(s_[i_])) : -1;
                int l = i_ + 1 < s_.size() ? hex(static_cast<unsigned char>(s_[i_ + 1])) : -1;
                if (h < 0 || l < 0) fail(kSyntax, "bad \\x escape");
                i_ += 2;
                return h * 16 + l;
            }
        }
        if (c >= '1' && c <= '9') fail(kUnsupported, "back-reference");
        if (c == 'b' || c == 'B' || c == 'A' || c == 'Z' || c == 'z') fail(kUnsupported, "assertion escape");
        if (std::isalnum(c)) fail(kSyntax, "unknown escape");
        return c;
    }

    int bracket() {  // after '['
        bool neg = false;
        if (cur() == '^') { neg = true; ++i_; }
        ByteSet set{};
        bool first = true;
        for (;;) {
            if (done()) fail(kSyntax, "unterminated class");
            int c = cur();
            if (c == ']' && !first) { ++i_; break; }
            first = false;
            ++i_;
            int lo = c;
            if (c == '\\') {
                ByteSet e{};
                lo = escape(e);
                if (lo < 0) {
                    if (cur() == '-' && i_ + 1 < s_.size() && s_[i_ + 1] != ']') fail(kSyntax, "class escape as range endpoint");
                    set = bs_or(set, e);
                    continue;
                }
            }
            int hi = lo;
            if (cur() == '-' && i_ + 1 < s_.size() && s_[i_ + 1] != ']') {
                ++i_;
                int d = cur();
                ++i_;
                if (d == '\\') {
                    ByteSet e{};
                    d = escape(e);
                    if (d < 0) fail(kSyntax, "class escape as range endpoint");
                }
                if (d < lo) fail(kSyntax, "bad range");
                hi = d;
            }
            set = bs_or(set, bs_range(lo, hi));
        }
        return make(K::Chars, {}, neg ? bs_not(set) : set);
    }

    int primary(int depth) {
        int c = cur();
        if (c == '(') {
            ++i_;
            if (cur() == '?') fail(kUnsupported, "group extension / look-around");
            int x = alternation(depth + 1);
            if (cur() != ')') fail(kSyntax, "missing ')'");
            ++i_;
            return x;
        }
        if (c == '[') { ++i_; return bracket(); }
        if (c == '.') { ++i_; return make(K::Chars, {}, bs_not(ByteSet{})); }
        if (c == '^' || c == '$') fail(kUnsupported, "anchor");
        if (c == '\\') {
            ++i_;
            ByteSet e{};
            int b = escape(e);
            if (b < 0) return make(K::Chars, {}, e);
            ByteSet one{};
            bs_set(one, b);
            return make(K::Chars, {}, one);
        }
        ++i_;
        ByteSet one{};
        bs_set(one, c);
        return make(K::Chars, {}, one);
    }
};

// ------------------------------------------------------------------------------------------
// Glushkov position automaton: state 0 = initial, positions 1..m = leaves.
// ------------------------------------------------------------------------------------------
struct Glushkov {
    uint32_t m = 0;                        // positions
    std::vector<ByteSet> chars;            // [m+1], chars[0] unused
    std::vector<std::vector<uint64_t>> follow;  // [m+1] bitsets over 0..m
    std::vector<uint64_t> finals;          // bitset
    uint32_t W = 0;                        // words per bitset
};

struct GInfo {
    bool nullable;
    std::vector<uint32_t> first, last;
};

class GlushkovBuilder {
public:
    GlushkovBuilder(const std::vector<Node>& nodes, Glushkov& g) : n_(nodes), g_(g) {}

    void build(int root) {
        // number the leaves left to right
        g_.m = 0;
        g_.chars.assign(1, ByteSet{});
        number(root);
        if (g_.m > kMaxPositions) throw CompileError(kCapacity, "too many NFA positions");
        g_.W = (g_.m + 1 + 63) / 64;
        g_.follow.assign(g_.m + 1, std::vector<uint64_t>(g_.W, 0));
        next_pos_ = 1;
        GInfo r = info(root);
        add_follow({0}, r.first);
        g_.finals.assign(g_.W, 0);
        for (uint32_t p : r.last) g_.finals[p >> 6] |= 1ull << (p & 63);
        if (r.nullable) g_.finals[0] |= 1;
    }

private:
    const std::vector<Node>& n_;
    Glushkov& g_;
    uint32_t next_pos_ = 1;

    void number(int x) {
        const Node& nd = n_[x];
        if (nd.k == K::Chars) {
            ++g_.m;
            if (g_.m > kMaxPositions) throw CompileError(kCapacity, "too many NFA positions");
            g_.chars.push_back(nd.set);
            return;
        }
        for (int c : nd.kids) number(c);
    }
    void add_follow(const std::vector<uint32_t>& from, const std::vector<uint32_t>& to) {
        if (to.empty()) return;
        std::vector<uint64_t> mask(g_.W, 0);
        for (uint32_t q : to) mask[q >> 6] |= 1ull << (q & 63);
        for (uint32_t p : from)
            for (uint32_t w = 0; w < g_.W; ++w) g_.follow[p][w] |= mask[w];
    }
    static std::vector<uint32_t> unite(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
        std::vector<uint32_t> r;
        r.reserve(a.size() + b.size());
        std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(r));
        return r;
    }
    GInfo info(int x) {
        const Node& nd = n_[x];
        switch (nd.k) {
            case K::Chars: {
                uint32_t p = next_pos_++;
                return {false, {p}, {p}};
            }
            case K::Eps: return {true, {}, {}};
            case K::Star: {
                GInfo a = info(nd.kids[0]);
                add_follow(a.last, a.first);
                a.nullable = true;
                return a;
            }
            case K::Alt: {
                GInfo a = info(nd.kids[0]);
                for (size_t j = 1; j < nd.kids.size(); ++j) {
                    GInfo b = info(nd.kids[j]);
                    a.nullable = a.nullable || b.nullable;
                    a.first = unite(a.first, b.first);
                    a.last = unite(a.last, b.last);
                }
                return a;
            }
            case K::Cat: {
                GInfo a = info(nd.kids[0]);
                for (size_t j = 1; j < nd.kids.size(); ++j) {
                    GInfo b = info(nd.kids[j]);
                    add_follow(a.last, b.first);
                    if (a.nullable) a.first = unite(a.first, b.first);
                    a.last = b.nullable ? unite(a.last, b.last) : std::move(b.last);
                    a.nullable = a.nullable && b.nullable;
                }
                return a;
            }
        }
        return {true, {}, {}};
    }
};

struct VecHash {
    size_t operator()(const std::vector<uint64_t>& v) const {
        uint64_t h = 0x243F6A8885A308D3ull;
        for (uint64_t w : v) h = (h ^ w) * 0x100000001B3ull + (h >> 31);
        return static_cast<size_t>(h);
    }
};

// ------------------------------------------------------------------------------------------
// Hopcroft partition refinement (block worklist variant).
// ------------------------------------------------------------------------------------------
std::vector<uint32_t> hopcroft(uint32_t N, uint32_t K, const std::vector<uint32_t>& delta,
                               const std::vector<uint8_t>& fin, uint32_t& nblocks) {
    // inverse transitions: for symbol k, target t -> sources
    std::vector<uint32_t> inv_off(static_cast<size_t>(K) * N + 1, 0), inv;
    for (uint32_t q = 0; q < N; ++q)
        for (uint32_t k = 0; k < K; ++k) ++inv_off[static_cast<size_t>(k) * N + delta[static_cast<size_t>(q) * K + k] + 1];
    for (size_t i = 1; i < inv_off.size(); ++i) inv_off[i] += inv_off[i - 1];
    inv.resize(inv_off.back());
    {
        std::vector<uint32_t> fill(inv_off.begin(), inv_off.end() - 1);
        for (uint32_t q = 0; q < N; ++q)
            for (uint32_t k = 0; k < K; ++k) inv[fill[static_cast<size_t>(k) * N + delta[static_cast<size_t>(q) * K + k]]++] = q;
    }
    std::vector<uint32_t> blk(N);
    std::vector<std::vector<uint32_t>> members;
    {
        std::vector<uint32_t> f, nf;
        for (uint32_t q = 0; q < N; ++q) (fin[q] ? f : nf).push_back(q);
        if (!nf.empty()) members.push_back(std::move(nf));
        if (!f.empty()) members.push_back(std::move(f));
        for (uint32_t b = 0; b < members.size(); ++b)
            for (uint32_t q : members[b]) blk[q] = b;
    }
    std::vector<uint8_t> in_work(members.size(), 0);
    std::deque<uint32_t> work;
    if (members.size() == 2) {
        uint32_t s = members[0].size() <= members[1].size() ? 0 : 1;
        work.push_back(s);
        in_work[s] = 1;
    }
    std::vector<uint32_t> mark_cnt;
    std::vector<uint8_t> marked(N, 0);
    std::vector<uint32_t> touched, X;
    while (!work.empty()) {
        uint32_t A = work.front();
        work.pop_front();
        in_work[A] = 0;
        const std::vector<uint32_t> splitter = members[A];  // snapshot
        for (uint32_t k = 0; k < K; ++k) {
            X.clear();
            for (uint32_t t : splitter) {
                size_t o = static_cast<size_t>(k) * N + t;
                for (uint32_t j = inv_off[o]; j < inv_off[o + 1]; ++j) {
                    uint32_t q = inv[j];
                    if (!marked[q]) { marked[q] = 1; X.push_back(q); }
                }
            }
            if (X.empty()) continue;
            mark_cnt.resize(members.size(), 0);
            touched.clear();
            for (uint32_t q : X) {
                if (mark_cnt[blk[q]]++ == 0) touched.push_back(blk[q]);
            }
            for (uint32_t Y : touched) {
                uint32_t cnt = mark_cnt[Y];
                mark_cnt[Y] = 0;
                if (cnt == members[Y].size()) continue;
                std::vector<uint32_t> in, out;
                for (uint32_t q : members[Y]) (marked[q] ? in : out).push_back(q);
                uint32_t Z = static_cast<uint32_t>(members.size());
                members[Y] = std::move(out);
                members.push_back(std::move(in));
                in_work.push_back(0);
                mark_cnt.push_back(0);
                for (uint32_t q : members[Z]) blk[q] = Z;
                if (in_work[Y]) {
                    work.push_back(Z);
                    in_work[Z] = 1;
                } else {
                    uint32_t s = members[Z].size() <= members[Y].size() ? Z : Y;
                    work.push_back(s);
                    in_work[s] = 1;
                }
            }
            for (uint32_t q : X) marked[q] = 0;
        }
    }
    nblocks = static_cast<uint32_t>(members.size());
    return blk;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// The parts of a compile shared by the D-SFA and the N-SFA: Sigma, the
// Glushkov NFA and its byte classes (bytes no position set distinguishes).
struct Front {
    ByteSet sig{};
    Glushkov g;
    std::array<uint32_t, 256> ncls{};
    uint32_t K = 1;
    std::vector<int> krep;
    std::vector<std::vector<uint64_t>> posmask;  // positions whose set contains class k
};

Front make_front(Automata& A, const std::string& regex, const uint8_t* sigma, int sigma_len) {
    Front F;
    ByteSet& sig = F.sig;
    if (sigma == nullptr || sigma_len < 0) sig = bs_not(ByteSet{});
    else
        for (int i = 0; i < sigma_len; ++i) bs_set(sig, sigma[i]);
    for (int b = 0; b < 256; ++b)
        if (bs_has(sig, b)) A.sigma[b >> 3] |= static_cast<uint8_t>(1u << (b & 7));

    // ---- parse + Glushkov ----
    std::vector<Node> nodes;
    int root = Parser(regex, sig, nodes).parse();
    Glushkov& g = F.g;
    GlushkovBuilder(nodes, g).build(root);
    nodes.clear();
    nodes.shrink_to_fit();
    A.nfa_positions = g.m;

    // ---- NFA byte classes: bytes indistinguishable by every position's set ----
    std::array<uint32_t, 256>& ncls = F.ncls;
    uint32_t K = 1;
    for (uint32_t p = 1; p <= g.m; ++p) {
        std::unordered_map<uint64_t, uint32_t> remap;
        std::array<uint32_t, 256> nc{};
        uint32_t k2 = 0;
        for (int b = 0; b < 256; ++b) {
            uint64_t key = (static_cast<uint64_t>(ncls[b]) << 1) | (bs_has(g.chars[p], b) ? 1 : 0);
            auto it = remap.find(key);
            if (it == remap.end()) it = remap.emplace(key, k2++).first;
            nc[b] = it->second;
        }
        ncls = nc;
        K = k2;
    }
    F.K = K;
    F.krep.assign(K, -1);
    for (int b = 0; b < 256; ++b)
        if (F.krep[ncls[b]] < 0) F.krep[ncls[b]] = b;
    F.posmask.assign(K, std::vector<uint64_t>(g.W, 0));
    for (uint32_t k = 0; k < K; ++k)
        for (uint32_t p = 1; p <= g.m; ++p)
            if (bs_has(g.chars[p], F.krep[k])) F.posmask[k][p >> 6] |= 1ull << (p & 63);
    return F;
}

// Alg. 1 (subset construction over the NFA classes) ->
// Hopcroft minimisation -> canonical numbering (C3): the DFA fields of A.
// Throws CompileError(capacity) past kMaxDfa subsets.
void build_min_dfa(Automata& A, const Front& F) {
    const ByteSet& sig = F.sig;
    const Glushkov& g = F.g;
    const std::array<uint32_t, 256>& ncls = F.ncls;
    const uint32_t K = F.K;
    const std::vector<std::vector<uint64_t>>& posmask = F.posmask;
    // ---- Alg. 1: subset construction over NFA classes ----
    std::vector<std::vector<uint64_t>> dstates;
    std::unordered_map<std::vector<uint64_t>, uint32_t, VecHash> index;
    std::vector<uint32_t> sdelta;  // subset DFA: id * K + k
    std::vector<uint8_t> sfin;
    {
        std::vector<uint64_t> start(g.W, 0);
        start[0] = 1;  // {initial}
        index.emplace(start, 0);
        dstates.push_back(std::move(start));
        std::vector<uint64_t> U(g.W), nx(g.W);
        for (size_t i = 0; i < dstates.size(); ++i) {
            if (dstates.size() > kMaxDfa) throw CompileError(kCapacity, "DFA too large");
            std::fill(U.begin(), U.end(), 0);
            const std::vector<uint64_t> S = dstates[i];
            for (uint32_t w = 0; w < g.W; ++w)
                for (uint64_t bits = S[w]; bits; bits &= bits - 1) {
                    uint32_t p = w * 64 + __builtin_ctzll(bits);
                    for (uint32_t v = 0; v < g.W; ++v) U[v] |= g.follow[p][v];
                }
            bool fin = false;
            for (uint32_t w = 0; w < g.W; ++w) fin = fin || (S[w] & g.finals[w]);
            sfin.push_back(fin ? 1 : 0);
            for (uint32_t k = 0; k < K; ++k) {
                for (uint32_t w = 0; w < g.W; ++w) nx[w] = U[w] & posmask[k][w];
                auto it = index.find(nx);
                uint32_t id;
                if (it == index.end()) {
                    id = static_cast<uint32_t>(dstates.size());
                    index.emplace(nx, id);
                    dstates.push_back(nx);
                } else id = it->second;
                sdelta.push_back(id);
            }
        }
    }
    const uint32_t NS = static_cast<uint32_t>(dstates.size());
    A.subset_states = NS;
    dstates.clear();
    index.clear();

    // ---- minimisation ----
    uint32_t nb = 0;
    std::vector<uint32_t> blk = hopcroft(NS, K, sdelta, sfin, nb);

    // ---- canonical BFS numbering over Sigma bytes (C3) ----
    std::vector<uint32_t> bdelta(static_cast<size_t>(nb) * K);
    std::vector<uint8_t> bfin(nb);
    for (uint32_t q = 0; q < NS; ++q) {
        for (uint32_t k = 0; k < K; ++k) bdelta[static_cast<size_t>(blk[q]) * K + k] = blk[sdelta[static_cast<size_t>(q) * K + k]];
        bfin[blk[q]] = sfin[q];
    }
    std::vector<uint32_t> canon(nb, UINT32_MAX), order;
    order.reserve(nb);
    canon[blk[0]] = 0;
    order.push_back(blk[0]);
    for (size_t h = 0; h < order.size(); ++h) {
        uint32_t c = order[h];
        for (int b = 0; b < 256; ++b) {
            if (!bs_has(sig, b)) continue;
            uint32_t t = bdelta[static_cast<size_t>(c) * K + ncls[b]];
            if (canon[t] == UINT32_MAX) {
                canon[t] = static_cast<uint32_t>(order.size());
                order.push_back(t);
            }
        }
    }
    for (uint32_t c = 0; c < nb; ++c)
        if (canon[c] == UINT32_MAX) {
            canon[c] = static_cast<uint32_t>(order.size());
            order.push_back(c);
        }
    A.nD = nb;
    A.dfa.resize(static_cast<size_t>(nb) * 256);
    A.dfa_final.resize(nb);
    for (uint32_t i = 0; i < nb; ++i) {
        uint32_t c = order[i];
        for (int b = 0; b < 256; ++b) A.dfa[static_cast<size_t>(i) * 256 + b] = canon[bdelta[static_cast<size_t>(c) * K + ncls[b]]];
        A.dfa_final[i] = bfin[c];
    }
    for (uint32_t i = 0; i < nb && A.dead < 0; ++i) {
        if (A.dfa_final[i]) continue;
        bool absorbing = true;
        for (int b = 0; b < 256 && absorbing; ++b) absorbing = A.dfa[static_cast<size_t>(i) * 256 + b] == i;
        if (absorbing) A.dead = static_cast<int32_t>(i);
    }
}

}  // namespace

Automata compile_regex(const std::string& regex, const uint8_t* sigma, int sigma_len, uint32_t max_sfa, bool build_sfa) {
    auto t0 = std::chrono::steady_clock::now();
    Automata A;
    Front F = make_front(A, regex, sigma, sigma_len);
    const ByteSet& sig = F.sig;
    build_min_dfa(A, F);
    const uint32_t nb = A.nD;
    A.dfa_seconds = seconds_since(t0);
    auto t1 = std::chrono::steady_clock::now();

    // ---- byte classes of the minimal DFA (equal columns) ----
    {
        std::unordered_map<std::vector<uint64_t>, uint32_t, VecHash> colmap;
        std::vector<uint64_t> col(nb);
        for (int b = 0; b < 256; ++b) {
            for (uint32_t q = 0; q < nb; ++q) col[q] = A.dfa[static_cast<size_t>(q) * 256 + b];
            auto it = colmap.find(col);
            if (it == colmap.end()) it = colmap.emplace(col, static_cast<uint32_t>(colmap.size())).first;
            A.cls[b] = static_cast<uint8_t>(it->second);
        }
        A.C = static_cast<uint32_t>(colmap.size());
        std::vector<int> rep(A.C, -1), any(A.C, -1);
        for (int b = 0; b < 256; ++b) {
            if (any[A.cls[b]] < 0) any[A.cls[b]] = b;
            if (bs_has(sig, b) && rep[A.cls[b]] < 0) rep[A.cls[b]] = b;
        }
        for (uint32_t c = 0; c < A.C; ++c) A.rep_byte[c] = static_cast<uint8_t>(rep[c] >= 0 ? rep[c] : any[c]);
    }
    if (!build_sfa) return A;  // the on-the-fly construction (lazy.cpp) builds the SFA while matching

    // ---- Alg. 4 (DFA form), canonical numbering ----
    const uint32_t D = nb, C = A.C;
    std::vector<uint32_t> dcls(static_cast<size_t>(D) * C);
    for (uint32_t q = 0; q < D; ++q)
        for (uint32_t c = 0; c < C; ++c) dcls[static_cast<size_t>(q) * C + c] = A.dfa[static_cast<size_t>(q) * 256 + A.rep_byte[c]];
    std::vector<uint32_t> sig_order;  // classes by first Sigma byte
    std::vector<uint8_t> has_sigma(C, 0);
    for (int b = 0; b < 256; ++b)
        if (bs_has(sig, b) && !has_sigma[A.cls[b]]) {
            has_sigma[A.cls[b]] = 1;
            sig_order.push_back(A.cls[b]);
        }
    const uint32_t cap = max_sfa ? std::min<uint32_t>(max_sfa, 65535u) : 65535u;
    // open-addressing table over mappings stored in A.maps
    std::vector<uint32_t> slots(1024, UINT32_MAX);
    auto hash_map = [&](const uint32_t* f) {
        uint64_t h = 0x9E3779B97F4A7C15ull;
        for (uint32_t q = 0; q < D; ++q) h = (h ^ f[q]) * 0xBF58476D1CE4E5B9ull, h ^= h >> 29;
        return h;
    };
    std::vector<uint32_t> parent, pclass;
    auto intern = [&](const uint32_t* f, uint32_t from, uint32_t via) -> uint32_t {
        if ((A.nS + 1) * 2 > slots.size()) {
            std::vector<uint32_t> ns(slots.size() * 2, UINT32_MAX);
            for (uint32_t s = 0; s < A.nS; ++s) {
                size_t k = hash_map(&A.maps[static_cast<size_t>(s) * D]) & (ns.size() - 1);
                while (ns[k] != UINT32_MAX) k = (k + 1) & (ns.size() - 1);
                ns[k] = s;
            }
            slots.swap(ns);
        }
        size_t k = hash_map(f) & (slots.size() - 1);
        while (slots[k] != UINT32_MAX) {
            if (std::memcmp(&A.maps[static_cast<size_t>(slots[k]) * D], f, D * sizeof(uint32_t)) == 0) return slots[k];
            k = (k + 1) & (slots.size() - 1);
        }
        if (A.nS >= cap) throw CompileError(kCapacity, "SFA has more than " + std::to_string(cap) + " states");
        slots[k] = A.nS;
        A.maps.insert(A.maps.end(), f, f + D);
        A.T.resize(A.T.size() + C, UINT32_MAX);
        parent.push_back(from);
        pclass.push_back(via);
        return A.nS++;
    };
    {
        std::vector<uint32_t> f(D), gnext(D);
        for (uint32_t q = 0; q < D; ++q) f[q] = q;  // f_I
        intern(f.data(), UINT32_MAX, UINT32_MAX);
        for (int pass = 0; pass < 2; ++pass) {
            // pass 0: BFS over Sigma (classes in order of their first Sigma
            // byte); pass 1: out-of-Sigma columns, and every column of the
            // mappings first met in pass 1 (only the constant-dead one).
            const uint32_t n0 = A.nS;
            for (uint32_t i = 0; i < A.nS; ++i) {
                auto visit = [&](uint32_t c) {
                    const uint32_t* fm = &A.maps[static_cast<size_t>(i) * D];
                    // line 6, DFA form: f_next(q) = delta(f(q), sigma)
                    for (uint32_t q = 0; q < D; ++q) gnext[q] = dcls[static_cast<size_t>(fm[q]) * C + c];
                    uint32_t id = intern(gnext.data(), i, c);
                    A.T[static_cast<size_t>(i) * C + c] = id;  // line 7
                };
                if (pass == 0) {
                    for (uint32_t c : sig_order) visit(c);
                } else {
                    for (uint32_t c = 0; c < C; ++c)
                        if (!(has_sigma[c] && i < n0)) visit(c);
                }
            }
        }
    }
    A.img0.resize(A.nS);
    A.acc.resize(A.nS);
    A.rep_off.assign(A.nS + 1, 0);
    std::vector<uint32_t> len(A.nS, 0);
    for (uint32_t s = 1; s < A.nS; ++s) len[s] = len[parent[s]] + 1;
    for (uint32_t s = 0; s < A.nS; ++s) {
        A.img0[s] = A.maps[static_cast<size_t>(s) * D + 0];
        A.acc[s] = A.dfa_final[A.img0[s]];
        A.rep_off[s + 1] = A.rep_off[s] + len[s];
        A.depth = std::max(A.depth, len[s]);
    }
    A.rep.resize(A.rep_off[A.nS]);
    for (uint32_t s = 1; s < A.nS; ++s) {
        // rep(s) = rep(parent) + representative byte of the class taken
        uint32_t p = parent[s];
        std::copy(A.rep.begin() + A.rep_off[p], A.rep.begin() + A.rep_off[p + 1], A.rep.begin() + A.rep_off[s]);
        A.rep[A.rep_off[s + 1] - 1] = A.rep_byte[pclass[s]];
    }
    A.sfa_seconds = seconds_since(t1);
    return A;
}

// ------------------------------------------------------------------------------------------
// N-SFA: Alg. 4 over the Glushkov NFA N = (Q, Sigma,
// delta, I = {0}, F): a state is a mapping f: Q -> 2^Q stored as |Q| bitset
// rows; f_I(q) = {q}; line 6: f_next(q) = U_{q' in f(q)} delta(q', sigma),
// delta(q', k) = follow(q') & positions of class k; line 11: f in F_s iff
// f(0) meets F.  Canonical numbering as the D-SFA (C3).  The composition
// f . g is the logical matrix product
// (f . g)(q) = U_{p in f(q)} g(p).
// ------------------------------------------------------------------------------------------
Automata compile_nsfa(const std::string& regex, const uint8_t* sigma, int sigma_len, uint32_t max_sfa) {
    auto t0 = std::chrono::steady_clock::now();
    Automata A;
    Front F = make_front(A, regex, sigma, sigma_len);
    const Glushkov& g = F.g;
    try {  // the minimal DFA, for canonical final states (C3); optional
        build_min_dfa(A, F);
    } catch (const CompileError& e) {
        if (e.code != kCapacity) throw;
        A.has_dfa = false;
        A.nD = 0;
        A.dfa.clear();
        A.dfa_final.clear();
        A.dead = -1;
    }
    A.dfa_seconds = seconds_since(t0);
    auto t1 = std::chrono::steady_clock::now();
    A.nsfa = true;
    const uint32_t Q = g.m + 1, W = g.W, MW = Q * W, K = F.K;
    A.nfa_states = Q;
    // table columns: the NFA byte classes; representative bytes prefer Sigma
    A.C = K;
    for (int b = 0; b < 256; ++b) A.cls[b] = static_cast<uint8_t>(F.ncls[b]);
    {
        std::vector<int> rep(K, -1);
        for (int b = 0; b < 256; ++b)
            if (bs_has(F.sig, b) && rep[F.ncls[b]] < 0) rep[F.ncls[b]] = b;
        for (uint32_t k = 0; k < K; ++k) A.rep_byte[k] = static_cast<uint8_t>(rep[k] >= 0 ? rep[k] : F.krep[k]);
    }
    // delta(q, k) as W-word bitsets
    std::vector<uint64_t> dq(static_cast<size_t>(Q) * K * W);
    for (uint32_t q = 0; q < Q; ++q)
        for (uint32_t k = 0; k < K; ++k)
            for (uint32_t w = 0; w < W; ++w) dq[(static_cast<size_t>(q) * K + k) * W + w] = g.follow[q][w] & F.posmask[k][w];
    std::vector<uint32_t> sig_order;
    std::vector<uint8_t> has_sigma(K, 0);
    for (int b = 0; b < 256; ++b)
        if (bs_has(F.sig, b) && !has_sigma[F.ncls[b]]) {
            has_sigma[F.ncls[b]] = 1;
            sig_order.push_back(F.ncls[b]);
        }
    const uint32_t cap = max_sfa ? std::min<uint32_t>(max_sfa, 65535u) : 65535u;
    std::vector<uint64_t> mp;  // nS * MW
    std::vector<uint32_t> slots(1024, UINT32_MAX), parent, pclass;
    auto hash_m = [&](const uint64_t* f) {
        uint64_t h = 0x9E3779B97F4A7C15ull;
        for (uint32_t i = 0; i < MW; ++i) h = (h ^ f[i]) * 0xBF58476D1CE4E5B9ull, h ^= h >> 29;
        return h;
    };
    auto find = [&](const uint64_t* f) -> uint32_t {
        size_t k = hash_m(f) & (slots.size() - 1);
        while (slots[k] != UINT32_MAX) {
            if (std::memcmp(&mp[static_cast<size_t>(slots[k]) * MW], f, MW * sizeof(uint64_t)) == 0) return slots[k];
            k = (k + 1) & (slots.size() - 1);
        }
        return UINT32_MAX;
    };
    auto intern = [&](const uint64_t* f, uint32_t from, uint32_t via) -> uint32_t {
        if ((A.nS + 1) * 2 > slots.size()) {
            std::vector<uint32_t> ns(slots.size() * 2, UINT32_MAX);
            for (uint32_t s = 0; s < A.nS; ++s) {
                size_t k = hash_m(&mp[static_cast<size_t>(s) * MW]) & (ns.size() - 1);
                while (ns[k] != UINT32_MAX) k = (k + 1) & (ns.size() - 1);
                ns[k] = s;
            }
            slots.swap(ns);
        }
        size_t k = hash_m(f) & (slots.size() - 1);
        while (slots[k] != UINT32_MAX) {
            if (std::memcmp(&mp[static_cast<size_t>(slots[k]) * MW], f, MW * sizeof(uint64_t)) == 0) return slots[k];
            k = (k + 1) & (slots.size() - 1);
        }
        if (A.nS >= cap) throw CompileError(kCapacity, "N-SFA has more than " + std::to_string(cap) + " states");
        slots[k] = A.nS;
        mp.insert(mp.end(), f, f + MW);
        A.T.resize(A.T.size() + K, UINT32_MAX);
        parent.push_back(from);
        pclass.push_back(via);
        return A.nS++;
    };
    {
        std::vector<uint64_t> f(MW, 0), gn(MW);
        for (uint32_t q = 0; q < Q; ++q) f[static_cast<size_t>(q) * W + (q >> 6)] = 1ull << (q & 63);  // f_I(q) = {q}
        intern(f.data(), UINT32_MAX, UINT32_MAX);
        for (int pass = 0; pass < 2; ++pass) {
            const uint32_t n0 = A.nS;
            for (uint32_t i = 0; i < A.nS; ++i) {
                auto visit = [&](uint32_t c) {
                    const uint64_t* fm = &mp[static_cast<size_t>(i) * MW];
                    std::fill(gn.begin(), gn.end(), 0);
                    for (uint32_t q = 0; q < Q; ++q)  // line 6: f_next(q) = U_{q' in f(q)} delta(q', sigma)
                        for (uint32_t w = 0; w < W; ++w)
                            for (uint64_t bits = fm[static_cast<size_t>(q) * W + w]; bits; bits &= bits - 1) {
                                const uint32_t p = w * 64 + __builtin_ctzll(bits);
                                const uint64_t* d = &dq[(static_cast<size_t>(p) * K + c) * W];
                                for (uint32_t v = 0; v < W; ++v) gn[static_cast<size_t>(q) * W + v] |= d[v];
                            }
                    const uint32_t id = intern(gn.data(), i, c);
                    A.T[static_cast<size_t>(i) * K + c] = id;  // line 7
                };
                if (pass == 0) {
                    for (uint32_t c : sig_order) visit(c);
                } else {
                    for (uint32_t c = 0; c < K; ++c)
                        if (!(has_sigma[c] && i < n0)) visit(c);
                }
            }
        }
    }
    // rep words (Lemma 1 replay), F_s (line 11), the final-state map
    A.rep_off.assign(A.nS + 1, 0);
    std::vector<uint32_t> len(A.nS, 0);
    for (uint32_t s = 1; s < A.nS; ++s) len[s] = len[parent[s]] + 1;
    for (uint32_t s = 0; s < A.nS; ++s) {
        A.rep_off[s + 1] = A.rep_off[s] + len[s];
        A.depth = std::max(A.depth, len[s]);
    }
    A.rep.resize(A.rep_off[A.nS]);
    for (uint32_t s = 1; s < A.nS; ++s) {
        const uint32_t p = parent[s];
        std::copy(A.rep.begin() + A.rep_off[p], A.rep.begin() + A.rep_off[p + 1], A.rep.begin() + A.rep_off[s]);
        A.rep[A.rep_off[s + 1] - 1] = A.rep_byte[pclass[s]];
    }
    A.acc.resize(A.nS);
    A.img0.resize(A.nS);
    for (uint32_t s = 0; s < A.nS; ++s) {
        bool fin = false;
        for (uint32_t w = 0; w < W; ++w) fin = fin || (mp[static_cast<size_t>(s) * MW + w] & g.finals[w]);  // f(0) cap F
        A.acc[s] = fin ? 1 : 0;
        if (A.has_dfa) {  // the minimal DFA's state after rep(s): f_s(I) is that state's subset
            uint32_t q = 0;
            for (uint32_t k = A.rep_off[s]; k < A.rep_off[s + 1]; ++k) q = A.dfa[static_cast<size_t>(q) * 256 + A.rep[k]];
            A.img0[s] = q;
        } else {
            A.img0[s] = s;
        }
    }
    if (!A.has_dfa) {  // results are (N-SFA id, [id in F_s])
        A.nD = A.nS;
        A.dfa_final = A.acc;
    }
    // composition table by logical matrix products (|S| <= 4096)
    if (A.nS <= 4096) {
        A.comp.assign(static_cast<size_t>(A.nS) * A.nS, 0);
        std::vector<uint64_t> h(MW);
        for (uint32_t a = 0; a < A.nS; ++a)
            for (uint32_t b = 0; b < A.nS; ++b) {
                const uint64_t* fa = &mp[static_cast<size_t>(a) * MW];
                const uint64_t* fb = &mp[static_cast<size_t>(b) * MW];
                std::fill(h.begin(), h.end(), 0);
                for (uint32_t q = 0; q < Q; ++q)
                    for (uint32_t w = 0; w < W; ++w)
                        for (uint64_t bits = fa[static_cast<size_t>(q) * W + w]; bits; bits &= bits - 1) {
                            const uint32_t p = w * 64 + __builtin_ctzll(bits);
                            for (uint32_t v = 0; v < W; ++v) h[static_cast<size_t>(q) * W + v] |= fb[static_cast<size_t>(p) * W + v];
                        }
                const uint32_t id = find(h.data());  // the transition monoid is closed (Lemma 1)
                if (id == UINT32_MAX) throw CompileError(kCapacity, "N-SFA composition not closed");
                A.comp[static_cast<size_t>(a) * A.nS + b] = id;
            }
    }
    A.sfa_seconds = seconds_since(t1);
    return A;
}

}  // namespace sfa
