/*
 * oracle.c -- CPU ORACLE for the SFA matcher.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct C.  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU legs may load it; the product never does.  It shares no code
 * with paper_1405_0562_b200/ (own parser, Thompson NFA instead of the
 * product's Glushkov NFA, Moore instead of Hopcroft minimisation).
 *
 * Passages followed (PAPER.md = /root/reference/PAPER.md):
 *   NFA quintuple                 Def. 1
 *   DFA (complete, |I| = 1)       Def. 2
 *   extended transition delta^
 *   acceptance / L(A)             Def. 4-5
 *   subset construction           Alg. 1
 *   sequential DFA run            Alg. 2
 *   minimised DFA                 PAPER.md:672 (algorithm unnamed -> Moore)
 *   composition o, reverse .
 *   SFA definition                Def. 3
 *   correspondence construction   Alg. 4, PAPER.md:501-521 (+ DFA form 495-499)
 *   parallel SFA run              Alg. 5, PAPER.md:552-576 (both reductions)
 * Readings (C2, C3, C5, C8, C10) are listed in DESIGN.md.
 *
 * Pins (tests/test_oracle.py): brute force on every short string, Python's
 * `re` library, closed forms per config, the paper's printed sizes and
 * Table I / Examples 1-2.
 */
#include "oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define E_OK 0
#define E_SYNTAX 1
#define E_UNSUP 2
#define E_CAP 3
#define E_ARG 4

#define MAX_REPEAT 1000
#define MAX_NFA (1u << 21)
#define MAX_DFA (1u << 20)

/* ------------------------------------------------------------------------ */
/* AST                                                                       */
/* ------------------------------------------------------------------------ */

enum { K_NONE = 0, K_EPS, K_SET, K_CAT, K_ALT, K_STAR };

typedef struct {
    int kind;
    int l, r;              /* children (K_CAT, K_ALT: l r; K_STAR: l) */
    uint8_t set[32];       /* K_SET: byte set, already intersected with Sigma */
} Node;

typedef struct {
    Node* v;
    int n, cap;
    const uint8_t* p;
    size_t len, pos;
    uint8_t sigma[32];
    int err;
    char msg[160];
} Parser;

static int set_has(const uint8_t* s, int b) { return (s[b >> 3] >> (b & 7)) & 1; }
static void set_add(uint8_t* s, int b) { s[b >> 3] |= (uint8_t)(1u << (b & 7)); }

static void perr(Parser* P, int code, const char* what) {
    if (P->err) return;
    P->err = code;
    snprintf(P->msg, sizeof P->msg, "%s at %zu", what, P->pos);
}

static int new_node(Parser* P, int kind, int l, int r) {
    if (P->n == P->cap) {
        int nc = P->cap ? P->cap * 2 : 64;
        Node* nv = (Node*)realloc(P->v, (size_t)nc * sizeof(Node));
        if (!nv) { perr(P, E_CAP, "out of memory"); return 0; }
        P->v = nv;
        P->cap = nc;
    }
    Node* x = &P->v[P->n];
    memset(x, 0, sizeof *x);
    x->kind = kind;
    x->l = l;
    x->r = r;
    return P->n++;
}

/* a set node holding (bytes & Sigma) */
static int set_node(Parser* P, const uint8_t* bytes) {
    int id = new_node(P, K_SET, -1, -1);
    if (P->err) return id;
    for (int i = 0; i < 32; i++) P->v[id].set[i] = (uint8_t)(bytes[i] & P->sigma[i]);
    return id;
}

static int peek(Parser* P) { return P->pos < P->len ? P->p[P->pos] : -1; }

static int parse_alt(Parser* P, int depth);

/* \d \w \s families (ASCII), used both outside and inside classes */
static int escape_class(int c, uint8_t* out) {
    memset(out, 0, 32);
    int neg = 0;
    switch (c) {
        case 'D': neg = 1; /* fallthrough */
        case 'd': for (int b = '0'; b <= '9'; b++) set_add(out, b); break;
        case 'W': neg = 1; /* fallthrough */
        case 'w':
            for (int b = '0'; b <= '9'; b++) set_add(out, b);
            for (int b = 'a'; b <= 'z'; b++) set_add(out, b);
            for (int b = 'A'; b <= 'Z'; b++) set_add(out, b);
            set_add(out, '_');
            break;
        case 'S': neg = 1; /* fallthrough */
        case 's': {
            const char* ws = " \t\n\r\f\v";
            for (const char* q = ws; *q; q++) set_add(out, (uint8_t)*q);
            break;
        }
        default: return 0;
    }
    if (neg)
        for (int i = 0; i < 32; i++) out[i] = (uint8_t)~out[i];
    return 1;
}

static int hexval(int c) {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    return -1;
}

/* Parses the character after a backslash (pos points at it).  Returns a
 * single byte (>= 0), or -2 when a class escape was written into `cls`. */
static int parse_escape(Parser* P, uint8_t* cls) {
    int c = peek(P);
    if (c < 0) { perr(P, E_SYNTAX, "trailing backslash"); return 0; }
    P->pos++;
    if (escape_class(c, cls)) return -2;
    switch (c) {
        case 'n': return '\n';
        case 't': return '\t';
        case 'r': return '\r';
        case 'f': return '\f';
        case 'v': return '\v';
        case 'x': {
            int h1 = P->pos < P->len ? hexval(P->p[P->pos]) : -1;
            int h2 = P->pos + 1 < P->len ? hexval(P->p[P->pos + 1]) : -1;
            if (h1 < 0 || h2 < 0) { perr(P, E_SYNTAX, "bad \\x escape"); return 0; }
            P->pos += 2;
            return h1 * 16 + h2;
        }
        default: break;
    }
    if (c >= '1' && c <= '9') { perr(P, E_UNSUP, "back-reference"); return 0; }
    if (c == 'b' || c == 'B' || c == 'A' || c == 'Z' || c == 'z') {
        perr(P, E_UNSUP, "assertion escape");
        return 0;
    }
    if ((c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || (c >= '0' && c <= '9')) {
        perr(P, E_SYNTAX, "unknown escape");
        return 0;
    }
    return c; /* escaped punctuation / any other byte: itself */
}

static int parse_class(Parser* P) {
    /* '[' already consumed */
    uint8_t s[32];
    memset(s, 0, 32);
    int neg = 0;
    if (peek(P) == '^') { neg = 1; P->pos++; }
    int first = 1;
    for (;;) {
        int c = peek(P);
        if (c < 0) { perr(P, E_SYNTAX, "unterminated class"); return 0; }
        if (c == ']' && !first) { P->pos++; break; }
        first = 0;
        P->pos++;
        int lo;
        if (c == '\\') {
            uint8_t cls[32];
            lo = parse_escape(P, cls);
            if (P->err) return 0;
            if (lo == -2) {
                if (peek(P) == '-' && P->pos + 1 < P->len && P->p[P->pos + 1] != ']') {
                    perr(P, E_SYNTAX, "class escape as range endpoint");
                    return 0;
                }
                for (int i = 0; i < 32; i++) s[i] |= cls[i];
                continue;
            }
        } else {
            lo = c;
        }
        int hi = lo;
        if (peek(P) == '-' && P->pos + 1 < P->len && P->p[P->pos + 1] != ']') {
            P->pos++;
            int d = peek(P);
            P->pos++;
            if (d == '\\') {
                uint8_t cls[32];
                d = parse_escape(P, cls);
                if (P->err) return 0;
                if (d == -2) { perr(P, E_SYNTAX, "class escape as range endpoint"); return 0; }
            }
            hi = d;
            if (hi < lo) { perr(P, E_SYNTAX, "bad range"); return 0; }
        }
        for (int b = lo; b <= hi; b++) set_add(s, b);
    }
    if (neg)
        for (int i = 0; i < 32; i++) s[i] = (uint8_t)~s[i];
    return set_node(P, s);
}

static int parse_atom(Parser* P, int depth) {
    int c = peek(P);
    uint8_t s[32];
    if (c == '(') {
        P->pos++;
        if (peek(P) == '?') { perr(P, E_UNSUP, "group extension / look-around"); return 0; }
        int x = parse_alt(P, depth + 1);
        if (P->err) return 0;
        if (peek(P) != ')') { perr(P, E_SYNTAX, "missing )"); return 0; }
        P->pos++;
        return x;
    }
    if (c == '[') { P->pos++; return parse_class(P); }
    if (c == '.') {
        P->pos++;
        memset(s, 0xff, 32);
        return set_node(P, s);
    }
    if (c == '^' || c == '$') { perr(P, E_UNSUP, "anchor"); return 0; }
    if (c == '\\') {
        P->pos++;
        uint8_t cls[32];
        int b = parse_escape(P, cls);
        if (P->err) return 0;
        if (b == -2) return set_node(P, cls);
        memset(s, 0, 32);
        set_add(s, b);
        return set_node(P, s);
    }
    P->pos++;
    memset(s, 0, 32);
    set_add(s, c);
    return set_node(P, s);
}

static int read_int(Parser* P, int* out) {
    int v = 0, any = 0;
    while (peek(P) >= '0' && peek(P) <= '9') {
        v = v * 10 + (peek(P) - '0');
        if (v > 100000) v = 100000;
        P->pos++;
        any = 1;
    }
    *out = v;
    return any;
}

/* x{lo,hi}: lo copies, then (hi-lo) nested optionals; hi<0 means unbounded */
static int repeat_node(Parser* P, int x, int lo, int hi) {
    int eps = new_node(P, K_EPS, -1, -1);
    int tail;
    if (hi < 0) {
        tail = new_node(P, K_STAR, x, -1);
    } else {
        tail = eps; /* x{0} = eps */
        for (int i = 0; i < hi - lo && !P->err; i++) {
            int cat = new_node(P, K_CAT, x, tail);
            tail = new_node(P, K_ALT, cat, eps);
        }
    }
    int res = tail;
    for (int i = 0; i < lo && !P->err; i++) res = new_node(P, K_CAT, x, res);
    return res;
}

static int parse_rep(Parser* P, int depth) {
    int x = parse_atom(P, depth);
    for (;;) {
        if (P->err) return 0;
        int c = peek(P);
        if (c == '*') { P->pos++; x = new_node(P, K_STAR, x, -1); }
        else if (c == '+') { P->pos++; x = repeat_node(P, x, 1, -1); }
        else if (c == '?') { P->pos++; x = repeat_node(P, x, 0, 1); }
        else if (c == '{') {
            P->pos++;
            int lo, hi;
            if (!read_int(P, &lo)) { perr(P, E_SYNTAX, "bad repeat"); return 0; }
            if (peek(P) == '}') { hi = lo; }
            else if (peek(P) == ',') {
                P->pos++;
                if (peek(P) == '}') hi = -1;
                else if (!read_int(P, &hi)) { perr(P, E_SYNTAX, "bad repeat"); return 0; }
            } else { perr(P, E_SYNTAX, "bad repeat"); return 0; }
            if (peek(P) != '}') { perr(P, E_SYNTAX, "bad repeat"); return 0; }
            P->pos++;
            if (hi >= 0 && hi < lo) { perr(P, E_SYNTAX, "repeat {m,n} with m > n"); return 0; }
            if (lo > MAX_REPEAT || hi > MAX_REPEAT) { perr(P, E_CAP, "repeat count too large"); return 0; }
            x = repeat_node(P, x, lo, hi);
        } else break;
    }
    return x;
}

static int is_quant(int c) { return c == '*' || c == '+' || c == '?' || c == '{'; }

static int parse_cat(Parser* P, int depth) {
    int c = peek(P);
    if (c < 0 || c == '|' || c == ')') return new_node(P, K_EPS, -1, -1);
    if (is_quant(c)) { perr(P, E_SYNTAX, "dangling quantifier"); return 0; }
    /* left-to-right list, folded to the right */
    int n = 0, cap = 16;
    int* it = (int*)malloc((size_t)cap * sizeof(int));
    if (!it) { perr(P, E_CAP, "out of memory"); return 0; }
    while (!P->err) {
        c = peek(P);
        if (c < 0 || c == '|' || c == ')') break;
        if (is_quant(c)) { perr(P, E_SYNTAX, "dangling quantifier"); break; }
        int x = parse_rep(P, depth);
        if (n == cap) {
            cap *= 2;
            int* nh = (int*)realloc(it, (size_t)cap * sizeof(int));
            if (!nh) { perr(P, E_CAP, "out of memory"); break; }
            it = nh;
        }
        it[n++] = x;
    }
    int res = 0;
    if (!P->err) {
        res = it[n - 1];
        for (int i = n - 2; i >= 0; i--) res = new_node(P, K_CAT, it[i], res);
    }
    free(it);
    return res;
}

static int parse_alt(Parser* P, int depth) {
    if (depth > 2000) { perr(P, E_CAP, "nesting too deep"); return 0; }
    int x = parse_cat(P, depth);
    while (!P->err && peek(P) == '|') {
        P->pos++;
        int y = parse_cat(P, depth);
        x = new_node(P, K_ALT, x, y);
    }
    return x;
}

static void sigma_init(uint8_t* sig, const uint8_t* sigma, int sigma_len) {
    if (sigma_len < 0 || sigma == NULL) { memset(sig, 0xff, 32); return; }
    memset(sig, 0, 32);
    for (int i = 0; i < sigma_len; i++) set_add(sig, sigma[i]);
}

/* returns root or -1; fills P (caller frees P->v) */
static int parse_regex(Parser* P, const char* re, const uint8_t* sigma, int sigma_len) {
    memset(P, 0, sizeof *P);
    P->p = (const uint8_t*)re;
    P->len = strlen(re);
    sigma_init(P->sigma, sigma, sigma_len);
    int root = parse_alt(P, 0);
    if (!P->err && P->pos != P->len) {
        if (peek(P) == ')') perr(P, E_SYNTAX, "unbalanced )");
        else perr(P, E_SYNTAX, "unexpected character");
    }
    return P->err ? -1 : root;
}

/* ------------------------------------------------------------------------ */
/* Brute-force evaluator: ends(node, S) = set of end positions reachable     */
/* from start positions S (bitmask over 0..n), read off the regex's meaning. */
/* ------------------------------------------------------------------------ */

static uint64_t ends(const Node* v, int x, uint64_t S, const uint8_t* s, int n) {
    const Node* nd = &v[x];
    switch (nd->kind) {
        case K_NONE: return 0;
        case K_EPS: return S;
        case K_SET: {
            uint64_t R = 0;
            for (int i = 0; i < n; i++)
                if (((S >> i) & 1) && set_has(nd->set, s[i])) R |= 1ull << (i + 1);
            return R;
        }
        case K_CAT: return ends(v, nd->r, ends(v, nd->l, S, s, n), s, n);
        case K_ALT: return ends(v, nd->l, S, s, n) | ends(v, nd->r, S, s, n);
        case K_STAR: {
            uint64_t R = S;
            for (;;) {
                uint64_t R2 = R | ends(v, nd->l, R, s, n);
                if (R2 == R) return R;
                R = R2;
            }
        }
    }
    return 0;
}

int oracle_brute(const char* regex, const uint8_t* sigma, int sigma_len, const uint8_t* s, int n) {
    if (n < 0 || n > 62) return -E_ARG;
    Parser P;
    int root = parse_regex(&P, regex, sigma, sigma_len);
    if (root < 0) { free(P.v); return -P.err; }
    uint64_t R = ends(P.v, root, 1ull, s, n);
    free(P.v);
    return (int)((R >> n) & 1);
}

/* Every string over chars[0..nchars) of length 0..maxlen, in shortlex order
 * (length first, then lexicographic by position in `chars`); out[i] = match.
 * Returns the number of strings, or -code on a parse error. */
int64_t oracle_brute_all(const char* regex, const uint8_t* sigma, int sigma_len,
                         const uint8_t* chars, int nchars, int maxlen, uint8_t* out) {
    if (nchars < 1 || maxlen < 0 || maxlen > 62) return -E_ARG;
    Parser P;
    int root = parse_regex(&P, regex, sigma, sigma_len);
    if (root < 0) { free(P.v); return -P.err; }
    int64_t k = 0;
    uint8_t s[64];
    int idx[64];
    for (int len = 0; len <= maxlen; len++) {
        for (int i = 0; i < len; i++) idx[i] = 0;
        for (;;) {
            for (int i = 0; i < len; i++) s[i] = chars[idx[i]];
            out[k++] = (uint8_t)((ends(P.v, root, 1ull, s, len) >> len) & 1);
            int i = len - 1;
            while (i >= 0 && ++idx[i] == nchars) idx[i--] = 0;
            if (i < 0) break;
        }
    }
    free(P.v);
    return k;
}

/* ------------------------------------------------------------------------ */
/* Thompson NFA: every fragment has one entry and one exit (an EPS state).   */
/* ------------------------------------------------------------------------ */

enum { S_EPS = 0, S_SPLIT, S_SET };
typedef struct {
    int type;
    int out1, out2; /* -1 = none */
    int node;       /* S_SET: AST node holding the byte set */
} NState;

typedef struct {
    NState* v;
    int n, cap;
    int err;
} Nfa;

static int nfa_new(Nfa* N, int type, int o1, int o2, int node) {
    if (N->err) return 0;
    if ((unsigned)N->n >= MAX_NFA) { N->err = E_CAP; return 0; }
    if (N->n == N->cap) {
        int nc = N->cap ? N->cap * 2 : 256;
        NState* nv = (NState*)realloc(N->v, (size_t)nc * sizeof(NState));
        if (!nv) { N->err = E_CAP; return 0; }
        N->v = nv;
        N->cap = nc;
    }
    NState* s = &N->v[N->n];
    s->type = type;
    s->out1 = o1;
    s->out2 = o2;
    s->node = node;
    return N->n++;
}

typedef struct { int start, end; } Frag;

static Frag build(Nfa* N, const Node* v, int x) {
    Frag f = {0, 0};
    if (N->err) return f;
    const Node* nd = &v[x];
    switch (nd->kind) {
        case K_NONE: {
            int e = nfa_new(N, S_EPS, -1, -1, -1);
            int s = nfa_new(N, S_SET, e, -1, x); /* set is empty: never fires */
            f.start = s; f.end = e;
            return f;
        }
        case K_EPS: {
            int s = nfa_new(N, S_EPS, -1, -1, -1);
            f.start = s; f.end = s;
            return f;
        }
        case K_SET: {
            int e = nfa_new(N, S_EPS, -1, -1, -1);
            int s = nfa_new(N, S_SET, e, -1, x);
            f.start = s; f.end = e;
            return f;
        }
        case K_CAT: {
            Frag a = build(N, v, nd->l);
            Frag b = build(N, v, nd->r);
            if (N->err) return f;
            N->v[a.end].out1 = b.start;
            f.start = a.start; f.end = b.end;
            return f;
        }
        case K_ALT: {
            Frag a = build(N, v, nd->l);
            Frag b = build(N, v, nd->r);
            int e = nfa_new(N, S_EPS, -1, -1, -1);
            int s = nfa_new(N, S_SPLIT, a.start, b.start, -1);
            if (N->err) return f;
            N->v[a.end].out1 = e;
            N->v[b.end].out1 = e;
            f.start = s; f.end = e;
            return f;
        }
        case K_STAR: {
            Frag a = build(N, v, nd->l);
            int e = nfa_new(N, S_EPS, -1, -1, -1);
            int s = nfa_new(N, S_SPLIT, a.start, e, -1);
            if (N->err) return f;
            N->v[a.end].out1 = s;
            f.start = s; f.end = e;
            return f;
        }
    }
    return f;
}

/* ------------------------------------------------------------------------ */
/* Bitsets of NFA states                                                     */
/* ------------------------------------------------------------------------ */

typedef uint64_t word;

static void closure(const Nfa* N, word* S, int* stack) {
    int sp = 0;
    int W = (N->n + 63) / 64;
    for (int w = 0; w < W; w++)
        for (word m = S[w]; m; m &= m - 1) stack[sp++] = w * 64 + __builtin_ctzll(m);
    while (sp) {
        int q = stack[--sp];
        const NState* s = &N->v[q];
        int outs[2] = {-1, -1};
        if (s->type == S_EPS) outs[0] = s->out1;
        else if (s->type == S_SPLIT) { outs[0] = s->out1; outs[1] = s->out2; }
        for (int k = 0; k < 2; k++) {
            int t = outs[k];
            if (t < 0) continue;
            if (!((S[t >> 6] >> (t & 63)) & 1)) {
                S[t >> 6] |= 1ull << (t & 63);
                stack[sp++] = t;
            }
        }
    }
}

/* hash set of bitsets -> id */
typedef struct {
    word* sets;      /* n * W words */
    uint32_t n, cap;
    int W;
    uint32_t* slot;  /* hash slots: id+1, 0 = empty */
    uint32_t nslot;
} SetTab;

static uint64_t hash_words(const word* w, int W) {
    uint64_t h = 1469598103934665603ull;
    for (int i = 0; i < W; i++) { h ^= w[i]; h *= 1099511628211ull; h ^= h >> 29; }
    return h;
}

static int settab_grow(SetTab* T) {
    uint32_t ns = T->nslot ? T->nslot * 2 : 1024;
    uint32_t* sl = (uint32_t*)calloc(ns, sizeof(uint32_t));
    if (!sl) return 0;
    for (uint32_t i = 0; i < T->n; i++) {
        uint64_t h = hash_words(T->sets + (size_t)i * T->W, T->W);
        uint32_t k = (uint32_t)(h & (ns - 1));
        while (sl[k]) k = (k + 1) & (ns - 1);
        sl[k] = i + 1;
    }
    free(T->slot);
    T->slot = sl;
    T->nslot = ns;
    return 1;
}

/* returns id; *is_new set when inserted; UINT32_MAX on failure */
static uint32_t settab_get(SetTab* T, const word* s, int* is_new) {
    if ((T->n + 1) * 2 > T->nslot && !settab_grow(T)) return UINT32_MAX;
    uint64_t h = hash_words(s, T->W);
    uint32_t k = (uint32_t)(h & (T->nslot - 1));
    while (T->slot[k]) {
        uint32_t id = T->slot[k] - 1;
        if (memcmp(T->sets + (size_t)id * T->W, s, (size_t)T->W * sizeof(word)) == 0) {
            *is_new = 0;
            return id;
        }
        k = (k + 1) & (T->nslot - 1);
    }
    if (T->n == T->cap) {
        uint32_t nc = T->cap ? T->cap * 2 : 256;
        word* ns = (word*)realloc(T->sets, (size_t)nc * T->W * sizeof(word));
        if (!ns) return UINT32_MAX;
        T->sets = ns;
        T->cap = nc;
    }
    memcpy(T->sets + (size_t)T->n * T->W, s, (size_t)T->W * sizeof(word));
    T->slot[k] = T->n + 1;
    *is_new = 1;
    return T->n++;
}

/* ------------------------------------------------------------------------ */
/* The oracle DFA                                                            */
/* ------------------------------------------------------------------------ */

struct oracle_dfa {
    uint32_t n;          /* complete minimal |D| */
    uint32_t* table;     /* n * 256 */
    uint8_t* finals;     /* n */
    int32_t dead;
    uint32_t nfa_states, subset_states;
    uint8_t sigma[32];
};

void oracle_free(oracle_dfa* d) {
    if (!d) return;
    free(d->table);
    free(d->finals);
    free(d);
}

uint32_t oracle_nfa_states(const oracle_dfa* d) { return d->nfa_states; }
uint32_t oracle_subset_states(const oracle_dfa* d) { return d->subset_states; }
uint32_t oracle_dfa_states(const oracle_dfa* d) { return d->n; }
int32_t oracle_dfa_dead(const oracle_dfa* d) { return d->dead; }

void oracle_dfa_export(const oracle_dfa* d, uint32_t* table, uint8_t* finals) {
    if (table) memcpy(table, d->table, (size_t)d->n * 256 * sizeof(uint32_t));
    if (finals) memcpy(finals, d->finals, d->n);
}

static void seterr(char* err, int errlen, const char* msg) {
    if (err && errlen > 0) snprintf(err, (size_t)errlen, "%s", msg);
}

/* Moore minimisation: refine {F, Q\F} by successor classes until stable. */
static uint32_t* moore(uint32_t n, const uint32_t* T, const uint8_t* fin, uint32_t* ncls_out) {
    uint32_t* cls = (uint32_t*)malloc(n * sizeof(uint32_t));
    uint32_t* ncl = (uint32_t*)malloc(n * sizeof(uint32_t));
    uint32_t* sig = (uint32_t*)malloc((size_t)n * 257 * sizeof(uint32_t));
    uint32_t nslot = 1;
    while (nslot < 2 * n + 2) nslot <<= 1;
    uint32_t* slot = (uint32_t*)malloc(nslot * sizeof(uint32_t));
    if (!cls || !ncl || !sig || !slot) { free(cls); free(ncl); free(sig); free(slot); return NULL; }
    /* initial partition by finality, ids in order of first appearance */
    int seen[2] = {-1, -1};
    uint32_t k = 0;
    for (uint32_t q = 0; q < n; q++) {
        int f = fin[q] ? 1 : 0;
        if (seen[f] < 0) seen[f] = (int)k++;
        cls[q] = (uint32_t)seen[f];
    }
    uint32_t ncls = k;
    for (;;) {
        for (uint32_t q = 0; q < n; q++) {
            uint32_t* sg = sig + (size_t)q * 257;
            sg[0] = cls[q];
            for (int b = 0; b < 256; b++) sg[1 + b] = cls[T[(size_t)q * 256 + b]];
        }
        memset(slot, 0, nslot * sizeof(uint32_t));
        uint32_t nn = 0;
        for (uint32_t q = 0; q < n; q++) {
            const uint32_t* sg = sig + (size_t)q * 257;
            uint64_t h = 1469598103934665603ull;
            for (int j = 0; j < 257; j++) { h ^= sg[j]; h *= 1099511628211ull; }
            uint32_t s = (uint32_t)(h & (nslot - 1));
            for (;;) {
                if (!slot[s]) { slot[s] = q + 1; ncl[q] = nn++; break; }
                uint32_t r = slot[s] - 1;
                if (memcmp(sig + (size_t)r * 257, sg, 257 * sizeof(uint32_t)) == 0) { ncl[q] = ncl[r]; break; }
                s = (s + 1) & (nslot - 1);
            }
        }
        uint32_t* t = cls; cls = ncl; ncl = t;
        if (nn == ncls) break;
        ncls = nn;
    }
    free(ncl);
    free(sig);
    free(slot);
    *ncls_out = ncls;
    return cls;
}

int oracle_compile(const char* regex, const uint8_t* sigma, int sigma_len,
                   oracle_dfa** out, char* err, int errlen) {
    if (!regex || !out) { seterr(err, errlen, "null argument"); return E_ARG; }
    *out = NULL;
    Parser P;
    int root = parse_regex(&P, regex, sigma, sigma_len);
    if (root < 0) {
        seterr(err, errlen, P.msg);
        int e = P.err;
        free(P.v);
        return e;
    }
    /* Thompson NFA (I = {start}, F = {end}) */
    Nfa N;
    memset(&N, 0, sizeof N);
    Frag f = build(&N, P.v, root);
    if (N.err) { seterr(err, errlen, "NFA too large"); free(P.v); free(N.v); return E_CAP; }
    int W = (N.n + 63) / 64;
    int* stack = (int*)malloc((size_t)N.n * sizeof(int));
    word* cur = (word*)calloc((size_t)W, sizeof(word));
    word* nxt = (word*)calloc((size_t)W, sizeof(word));
    SetTab T;
    memset(&T, 0, sizeof T);
    T.W = W;
    uint32_t* tab = NULL;
    size_t tabcap = 0;
    int rc = E_OK;
    if (!stack || !cur || !nxt) { rc = E_CAP; goto done; }

    /* Alg. 1: Q_tmp <- {I}; process subsets in discovery order */
    cur[f.start >> 6] |= 1ull << (f.start & 63);
    closure(&N, cur, stack);
    int isnew;
    if (settab_get(&T, cur, &isnew) == UINT32_MAX) { rc = E_CAP; goto done; }
    for (uint32_t i = 0; i < T.n; i++) {
        if (T.n > MAX_DFA) { rc = E_CAP; goto done; }
        if ((size_t)T.n * 256 > tabcap) {
            size_t nc = tabcap ? tabcap * 2 : 256 * 256;
            while (nc < (size_t)T.n * 256) nc *= 2;
            uint32_t* nt = (uint32_t*)realloc(tab, nc * sizeof(uint32_t));
            if (!nt) { rc = E_CAP; goto done; }
            tab = nt;
            tabcap = nc;
        }
        for (int b = 0; b < 256; b++) {
            /* S_next <- U_{q in S} delta(q, sigma) (Alg. 1 line 6), then eps-closure */
            memcpy(cur, T.sets + (size_t)i * W, (size_t)W * sizeof(word));
            memset(nxt, 0, (size_t)W * sizeof(word));
            for (int w = 0; w < W; w++)
                for (word m = cur[w]; m; m &= m - 1) {
                    int q = w * 64 + __builtin_ctzll(m);
                    const NState* s = &N.v[q];
                    if (s->type == S_SET && set_has(P.v[s->node].set, b))
                        nxt[s->out1 >> 6] |= 1ull << (s->out1 & 63);
                }
            closure(&N, nxt, stack);
            uint32_t id = settab_get(&T, nxt, &isnew);
            if (id == UINT32_MAX) { rc = E_CAP; goto done; }
            tab[(size_t)i * 256 + b] = id;
        }
    }
    {
        uint32_t n = T.n;
        uint8_t* fin = (uint8_t*)malloc(n);
        if (!fin) { rc = E_CAP; goto done; }
        /* F_d = {S | S cap F != 0} (Alg. 1 line 11), F = {f.end} */
        for (uint32_t i = 0; i < n; i++) fin[i] = (uint8_t)((T.sets[(size_t)i * W + (f.end >> 6)] >> (f.end & 63)) & 1);
        uint32_t ncls;
        uint32_t* cls = moore(n, tab, fin, &ncls);
        if (!cls) { free(fin); rc = E_CAP; goto done; }
        /* quotient automaton, then canonical BFS numbering (C3) */
        uint32_t* qt = (uint32_t*)malloc((size_t)ncls * 256 * sizeof(uint32_t));
        uint8_t* qf = (uint8_t*)calloc(ncls, 1);
        uint32_t* canon = (uint32_t*)malloc(ncls * sizeof(uint32_t));
        uint32_t* order = (uint32_t*)malloc(ncls * sizeof(uint32_t));
        oracle_dfa* d = (oracle_dfa*)calloc(1, sizeof(oracle_dfa));
        if (!qt || !qf || !canon || !order || !d) {
            free(qt); free(qf); free(canon); free(order); free(d); free(cls); free(fin);
            rc = E_CAP; goto done;
        }
        for (uint32_t q = 0; q < n; q++) {
            for (int b = 0; b < 256; b++) qt[(size_t)cls[q] * 256 + b] = cls[tab[(size_t)q * 256 + b]];
            qf[cls[q]] = fin[q];
        }
        for (uint32_t c = 0; c < ncls; c++) canon[c] = UINT32_MAX;
        uint32_t start = cls[0], cnt = 0, head = 0;
        canon[start] = cnt; order[cnt++] = start;
        while (head < cnt) {
            uint32_t c = order[head++];
            for (int b = 0; b < 256; b++) {
                if (!set_has(P.sigma, b)) continue;
                uint32_t t = qt[(size_t)c * 256 + b];
                if (canon[t] == UINT32_MAX) { canon[t] = cnt; order[cnt++] = t; }
            }
        }
        /* states not reached over Sigma: only the dead state can be one */
        for (uint32_t c = 0; c < ncls; c++)
            if (canon[c] == UINT32_MAX) { canon[c] = cnt; order[cnt++] = c; }
        d->n = ncls;
        d->table = (uint32_t*)malloc((size_t)ncls * 256 * sizeof(uint32_t));
        d->finals = (uint8_t*)malloc(ncls);
        if (!d->table || !d->finals) { oracle_free(d); free(qt); free(qf); free(canon); free(order); free(cls); free(fin); rc = E_CAP; goto done; }
        for (uint32_t i = 0; i < ncls; i++) {
            uint32_t c = order[i];
            for (int b = 0; b < 256; b++) d->table[(size_t)i * 256 + b] = canon[qt[(size_t)c * 256 + b]];
            d->finals[i] = qf[c];
        }
        d->dead = -1;
        for (uint32_t i = 0; i < ncls; i++) {
            if (d->finals[i]) continue;
            int all = 1;
            for (int b = 0; b < 256 && all; b++) all = d->table[(size_t)i * 256 + b] == i;
            if (all) { d->dead = (int32_t)i; break; }
        }
        d->nfa_states = (uint32_t)N.n;
        d->subset_states = n;
        memcpy(d->sigma, P.sigma, 32);
        *out = d;
        free(qt); free(qf); free(canon); free(order); free(cls); free(fin);
    }
done:
    if (rc == E_CAP) seterr(err, errlen, "capacity exceeded");
    free(stack); free(cur); free(nxt);
    free(T.sets); free(T.slot);
    free(tab);
    free(N.v);
    free(P.v);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Alg. 2                                                                    */
/* ------------------------------------------------------------------------ */

int oracle_run(const oracle_dfa* d, const uint8_t* text, uint64_t n, uint32_t* q_final) {
    const uint32_t* T = d->table;
    uint32_t q = 0;                           /* q <- q0 (line 1) */
    for (uint64_t i = 0; i < n; i++)          /* for i = 1 -> n   */
        q = T[(size_t)q * 256 + text[i]];     /*   q <- delta_d[q, sigma_i] */
    if (q_final) *q_final = q;                /* q_final <- q     */
    return d->finals[q];
}

void oracle_run_batch(const oracle_dfa* d, const uint8_t* texts, const uint64_t* off,
                      uint64_t count, uint32_t* q_final, uint8_t* accept) {
    for (uint64_t i = 0; i < count; i++) {
        uint32_t q;
        int a = oracle_run(d, texts + off[i], off[i + 1] - off[i], &q);
        if (q_final) q_final[i] = q;
        if (accept) accept[i] = (uint8_t)a;
    }
}

/* Alg. 3, parallel computation of the DFA by speculative
 * simulation, written out sequentially: chunk i = text[bounds[i], bounds[i+1]);
 * lines 2-3: T_i[q] <- q for every q; lines 4-6: for every byte sigma_ij and
 * every q, T_i[q] <- delta(T_i[q], sigma_ij); then the sequential reduction
 * (right column, lines 9-11; reading C8): q_final <- q0; q_final <- T_i[q_final]
 * for i = 1..p.  maps (nullable) receives T_i as row i (p * |D| entries). */
int oracle_run_spec(const oracle_dfa* d, const uint8_t* text, const uint64_t* bounds, uint64_t p,
                    uint32_t* maps, uint32_t* q_final) {
    const uint32_t* T = d->table;
    const uint32_t nd = d->n;
    uint32_t* Ti = malloc(sizeof(uint32_t) * (nd ? nd : 1));
    if (!Ti) return -1;
    uint32_t qf = 0;                                       /* q_final <- q0 */
    for (uint64_t i = 0; i < p; i++) {
        for (uint32_t q = 0; q < nd; q++) Ti[q] = q;        /* T_i[q] <- q */
        for (uint64_t j = bounds[i]; j < bounds[i + 1]; j++)
            for (uint32_t q = 0; q < nd; q++)
                Ti[q] = T[(size_t)Ti[q] * 256 + text[j]];   /* T_i[q] <- delta(T_i[q], sigma_ij) */
        if (maps) memcpy(maps + (size_t)i * nd, Ti, sizeof(uint32_t) * nd);
        qf = Ti[qf];                                       /* q_final <- T_i[q_final] */
    }
    free(Ti);
    if (q_final) *q_final = qf;
    return d->finals[qf];
}

/* ------------------------------------------------------------------------ */
/* Alg. 4 (D-SFA) and Alg. 5                                                 */
/* ------------------------------------------------------------------------ */

struct oracle_sfa {
    uint32_t n, nd;
    uint32_t* maps;   /* n * nd */
    uint32_t* table;  /* n * 256 */
    uint8_t* finals;  /* n */
};

void oracle_sfa_free(oracle_sfa* s) {
    if (!s) return;
    free(s->maps);
    free(s->table);
    free(s->finals);
    free(s);
}

uint32_t oracle_sfa_states(const oracle_sfa* s) { return s->n; }

void oracle_sfa_export(const oracle_sfa* s, uint32_t* table, uint32_t* maps, uint8_t* finals) {
    if (table) memcpy(table, s->table, (size_t)s->n * 256 * sizeof(uint32_t));
    if (maps) memcpy(maps, s->maps, (size_t)s->n * s->nd * sizeof(uint32_t));
    if (finals) memcpy(finals, s->finals, s->n);
}

int oracle_sfa_build(const oracle_dfa* d, uint32_t cap, oracle_sfa** out) {
    *out = NULL;
    uint32_t D = d->n;
    /* mappings stored as bitset-hash entries: reuse SetTab on u32 vectors
     * packed into 64-bit words */
    SetTab T;
    memset(&T, 0, sizeof T);
    T.W = (int)((D + 1) / 2);
    word* f = (word*)calloc((size_t)T.W, sizeof(word));
    word* g = (word*)calloc((size_t)T.W, sizeof(word));
    uint32_t* tab = NULL;
    size_t tabcap = 0;
    int rc = E_OK, isnew;
    if (!f || !g) { rc = E_CAP; goto fail; }
    /* f_I(q) = q  (Def. 3) */
    for (uint32_t q = 0; q < D; q++) ((uint32_t*)f)[q] = q;
    if (settab_get(&T, f, &isnew) == UINT32_MAX) { rc = E_CAP; goto fail; }
    /* Alg. 4 with FIFO worklist and Sigma bytes in ascending order (C3).
     * pass 0: BFS over Sigma; pass 1: the out-of-Sigma bytes of those
     * mappings, and every byte of mappings first found in pass 1 (only the
     * constant-dead mapping can be one). */
    uint32_t n0 = 0;
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1) n0 = T.n;
        for (uint32_t i = 0; i < T.n; i++) {
            if ((size_t)T.n * 256 > tabcap || tab == NULL) {
                size_t nc = tabcap ? tabcap : 256 * 64;
                while (nc < (size_t)(T.n + 1) * 256) nc *= 2;
                uint32_t* nt = (uint32_t*)realloc(tab, nc * sizeof(uint32_t));
                if (!nt) { rc = E_CAP; goto fail; }
                tab = nt;
                tabcap = nc;
            }
            for (int b = 0; b < 256; b++) {
                int in_sigma = set_has(d->sigma, b);
                if (pass == 0 && !in_sigma) continue;
                if (pass == 1 && in_sigma && i < n0) continue;
                const uint32_t* fm = (const uint32_t*)(T.sets + (size_t)i * T.W);
                uint32_t* gm = (uint32_t*)g;
                /* line 6 (DFA form): f_next(q) = delta(f(q), sigma) */
                for (uint32_t q = 0; q < D; q++) gm[q] = d->table[(size_t)fm[q] * 256 + b];
                uint32_t id = settab_get(&T, g, &isnew);
                if (id == UINT32_MAX) { rc = E_CAP; goto fail; }
                if (T.n > cap) { rc = E_CAP; goto fail; }
                tab[(size_t)i * 256 + b] = id;   /* line 7: delta_s[f, sigma] <- f_next */
            }
        }
    }
    {
        oracle_sfa* s = (oracle_sfa*)calloc(1, sizeof(oracle_sfa));
        if (!s) { rc = E_CAP; goto fail; }
        s->n = T.n;
        s->nd = D;
        s->maps = (uint32_t*)malloc((size_t)T.n * D * sizeof(uint32_t));
        s->table = (uint32_t*)malloc((size_t)T.n * 256 * sizeof(uint32_t));
        s->finals = (uint8_t*)malloc(T.n);
        if (!s->maps || !s->table || !s->finals) { oracle_sfa_free(s); rc = E_CAP; goto fail; }
        for (uint32_t i = 0; i < T.n; i++) {
            const uint32_t* fm = (const uint32_t*)(T.sets + (size_t)i * T.W);
            memcpy(s->maps + (size_t)i * D, fm, D * sizeof(uint32_t));
            /* F_s = {f | exists q in I: f(q) cap F != 0}, I = {q0 = 0} (line 11) */
            s->finals[i] = d->finals[fm[0]];
        }
        memcpy(s->table, tab, (size_t)T.n * 256 * sizeof(uint32_t));
        *out = s;
    }
fail:
    free(f); free(g); free(tab);
    free(T.sets); free(T.slot);
    return rc;
}

int oracle_sfa_run_chunked(const oracle_sfa* s, const uint8_t* text, const uint64_t* bounds,
                           int p, uint32_t* chunk_ids, uint32_t* q_seq, uint32_t* q_par) {
    if (p < 1) return -E_ARG;
    uint32_t D = s->nd;
    /* lines 1-5: each chunk from f_I (id 0), one table lookup per byte */
    uint32_t* ids = (uint32_t*)malloc((size_t)p * sizeof(uint32_t));
    if (!ids) return -E_CAP;
    for (int i = 0; i < p; i++) {
        uint32_t f = 0;
        for (uint64_t j = bounds[i]; j < bounds[i + 1]; j++) f = s->table[(size_t)f * 256 + text[j]];
        ids[i] = f;
        if (chunk_ids) chunk_ids[i] = f;
    }
    /* right column: S_fin <- I; for i: S_fin <- U_{p in S_fin} f_i(p) */
    uint32_t q = 0;
    for (int i = 0; i < p; i++) q = s->maps[(size_t)ids[i] * D + q];
    if (q_seq) *q_seq = q;
    /* left column: f_fin <- f_1 . ... . f_p (left fold; . is associative),
     * S_fin <- f_fin(q0) */
    uint32_t* ff = (uint32_t*)malloc(D * sizeof(uint32_t));
    uint32_t* tmp = (uint32_t*)malloc(D * sizeof(uint32_t));
    if (!ff || !tmp) { free(ids); free(ff); free(tmp); return -E_CAP; }
    for (uint32_t k = 0; k < D; k++) ff[k] = k;
    for (int i = 0; i < p; i++) {
        const uint32_t* g = s->maps + (size_t)ids[i] * D;
        for (uint32_t k = 0; k < D; k++) tmp[k] = g[ff[k]];   /* (f . g)(k) = g(f(k)) */
        memcpy(ff, tmp, D * sizeof(uint32_t));
    }
    if (q_par) *q_par = ff[0];
    free(ids); free(ff); free(tmp);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* NFA and N-SFA                                       */
/*                                                                          */
/* The NFA is either the Thompson NFA of a regex, seen eps-free (PAPER.md:   */
/* 156-169): Q = the Thompson states, delta(q, b) = closure(move({q}, b)),   */
/* I = closure({start}), F = {end}; or an explicit eps-free NFA given by its */
/* transition bitsets (the paper's Ex. 3 NFA).            */
/* The N-SFA is Alg. 4 in its general form: a state is a  */
/* mapping f: Q -> 2^Q, f_I(q) = {q}, line 6: f_next(q) = U_{q' in f(q)}     */
/* delta(q', sigma), line 11: F_s = {f | exists q in I: f(q) cap F != 0};    */
/* its composition f . g is the logical matrix product.      */
/* ------------------------------------------------------------------------ */

struct oracle_nfa {
    int n, W;            /* states, words per bitset */
    word* delta;         /* n * 256 * W: delta(q, b) */
    word* I;             /* W */
    word* F;             /* W */
    uint8_t sigma[32];
};

void oracle_nfa_free(oracle_nfa* a) {
    if (!a) return;
    free(a->delta); free(a->I); free(a->F);
    free(a);
}

uint32_t oracle_nfa_size(const oracle_nfa* a) { return (uint32_t)a->n; }

static oracle_nfa* nfa_alloc(int n) {
    oracle_nfa* a = (oracle_nfa*)calloc(1, sizeof(oracle_nfa));
    if (!a) return NULL;
    a->n = n;
    a->W = (n + 63) / 64;
    a->delta = (word*)calloc((size_t)n * 256 * a->W, sizeof(word));
    a->I = (word*)calloc((size_t)a->W, sizeof(word));
    a->F = (word*)calloc((size_t)a->W, sizeof(word));
    if (!a->delta || !a->I || !a->F) { oracle_nfa_free(a); return NULL; }
    return a;
}

int oracle_nfa_compile(const char* regex, const uint8_t* sigma, int sigma_len,
                       oracle_nfa** out, char* err, int errlen) {
    if (!regex || !out) { seterr(err, errlen, "null argument"); return E_ARG; }
    *out = NULL;
    Parser P;
    int root = parse_regex(&P, regex, sigma, sigma_len);
    if (root < 0) {
        seterr(err, errlen, P.msg);
        int e = P.err;
        free(P.v);
        return e;
    }
    Nfa N;
    memset(&N, 0, sizeof N);
    Frag f = build(&N, P.v, root);
    if (N.err || N.n > 4096) { seterr(err, errlen, "NFA too large"); free(P.v); free(N.v); return E_CAP; }
    oracle_nfa* a = nfa_alloc(N.n);
    int* stack = (int*)malloc((size_t)N.n * sizeof(int));
    if (!a || !stack) { oracle_nfa_free(a); free(stack); free(P.v); free(N.v); return E_CAP; }
    int W = a->W;
    for (int q = 0; q < N.n; q++) {
        const NState* s = &N.v[q];
        if (s->type != S_SET) continue;   /* eps / split states have no byte move */
        for (int b = 0; b < 256; b++) {
            if (!set_has(P.v[s->node].set, b)) continue;
            word* d = a->delta + ((size_t)q * 256 + b) * W;
            d[s->out1 >> 6] |= 1ull << (s->out1 & 63);
            closure(&N, d, stack);
        }
    }
    a->I[f.start >> 6] |= 1ull << (f.start & 63);
    closure(&N, a->I, stack);
    a->F[f.end >> 6] |= 1ull << (f.end & 63);
    memcpy(a->sigma, P.sigma, 32);
    free(stack); free(P.v); free(N.v);
    *out = a;
    return E_OK;
}

/* An explicit eps-free NFA of n <= 64 states: delta[q * 256 + b] = bitset of
 * successors, I and F bitsets; Sigma as for oracle_compile. */
int oracle_nfa_explicit(int n, const uint64_t* delta, uint64_t I, uint64_t F, const uint8_t* sigma,
                        int sigma_len, oracle_nfa** out) {
    *out = NULL;
    if (n < 1 || n > 64 || !delta) return E_ARG;
    oracle_nfa* a = nfa_alloc(n);
    if (!a) return E_CAP;
    for (size_t i = 0; i < (size_t)n * 256; i++) a->delta[i] = delta[i];
    a->I[0] = I;
    a->F[0] = F;
    sigma_init(a->sigma, sigma, sigma_len);
    *out = a;
    return E_OK;
}

/* S <- U_{q in S} delta(q, b) */
static void nfa_step(const oracle_nfa* a, const word* S, int b, word* out) {
    memset(out, 0, (size_t)a->W * sizeof(word));
    for (int w = 0; w < a->W; w++)
        for (word m = S[w]; m; m &= m - 1) {
            int q = w * 64 + __builtin_ctzll(m);
            const word* d = a->delta + ((size_t)q * 256 + b) * a->W;
            for (int v = 0; v < a->W; v++) out[v] |= d[v];
        }
}

static int meets(const word* S, const word* F, int W) {
    for (int w = 0; w < W; w++)
        if (S[w] & F[w]) return 1;
    return 0;
}

/* The NFA run (the definition): S <- I, then S <- U delta(q, b) per byte.
 * Returns accept (0/1) or -E_CAP; final_set (W words, nullable). */
int oracle_nfa_run(const oracle_nfa* a, const uint8_t* text, uint64_t n, uint64_t* final_set) {
    word* S = (word*)malloc((size_t)a->W * sizeof(word));
    word* T = (word*)malloc((size_t)a->W * sizeof(word));
    if (!S || !T) { free(S); free(T); return -E_CAP; }
    memcpy(S, a->I, (size_t)a->W * sizeof(word));
    for (uint64_t i = 0; i < n; i++) {
        nfa_step(a, S, text[i], T);
        word* x = S; S = T; T = x;
    }
    int acc = meets(S, a->F, a->W);
    if (final_set) memcpy(final_set, S, (size_t)a->W * sizeof(word));
    free(S); free(T);
    return acc;
}

struct oracle_nsfa {
    const oracle_nfa* a;
    uint32_t ns;
    word* maps;        /* ns mappings of n rows of W words: maps + (s*n + q)*W = f_s(q) */
    uint32_t* table;   /* ns * 256 */
    uint8_t* finals;   /* ns */
};

void oracle_nsfa_free(oracle_nsfa* s) {
    if (!s) return;
    free(s->maps); free(s->table); free(s->finals);
    free(s);
}

uint32_t oracle_nsfa_states(const oracle_nsfa* s) { return s->ns; }

/* Alg. 4, general form; mapping rows as bitsets; canonical BFS numbering
 * (C3: Sigma bytes ascending, then the out-of-Sigma bytes).  cap: at most
 * that many mappings (3 = capacity otherwise). */
int oracle_nsfa_build(const oracle_nfa* a, uint32_t cap, oracle_nsfa** out) {
    *out = NULL;
    const int n = a->n, W = a->W, MW = n * W;    /* words per mapping */
    SetTab T;
    memset(&T, 0, sizeof T);
    T.W = MW;
    word* f = (word*)calloc((size_t)MW, sizeof(word));
    word* g = (word*)calloc((size_t)MW, sizeof(word));
    uint32_t* tab = NULL;
    size_t tabcap = 0;
    int rc = E_OK, isnew;
    if (!f || !g) { rc = E_CAP; goto fail; }
    for (int q = 0; q < n; q++) f[(size_t)q * W + (q >> 6)] = 1ull << (q & 63);   /* f_I(q) = {q} */
    if (settab_get(&T, f, &isnew) == UINT32_MAX) { rc = E_CAP; goto fail; }
    uint32_t n0 = 0;
    for (int pass = 0; pass < 2; pass++) {
        if (pass == 1) n0 = T.n;
        for (uint32_t i = 0; i < T.n; i++) {
            if ((size_t)(T.n + 1) * 256 > tabcap) {
                size_t nc = tabcap ? tabcap : 256 * 64;
                while (nc < (size_t)(T.n + 1) * 256) nc *= 2;
                uint32_t* nt = (uint32_t*)realloc(tab, nc * sizeof(uint32_t));
                if (!nt) { rc = E_CAP; goto fail; }
                tab = nt;
                tabcap = nc;
            }
            for (int b = 0; b < 256; b++) {
                int in_sigma = set_has(a->sigma, b);
                if (pass == 0 && !in_sigma) continue;
                if (pass == 1 && in_sigma && i < n0) continue;
                /* line 6: f_next(q) = U_{q' in f(q)} delta(q', sigma) */
                for (int q = 0; q < n; q++) nfa_step(a, T.sets + (size_t)i * MW + (size_t)q * W, b, g + (size_t)q * W);
                uint32_t id = settab_get(&T, g, &isnew);
                if (id == UINT32_MAX) { rc = E_CAP; goto fail; }
                if (T.n > cap) { rc = E_CAP; goto fail; }
                tab[(size_t)i * 256 + b] = id;   /* line 7 */
            }
        }
    }
    {
        oracle_nsfa* s = (oracle_nsfa*)calloc(1, sizeof(oracle_nsfa));
        if (!s) { rc = E_CAP; goto fail; }
        s->a = a;
        s->ns = T.n;
        s->maps = (word*)malloc((size_t)T.n * MW * sizeof(word));
        s->table = (uint32_t*)malloc((size_t)T.n * 256 * sizeof(uint32_t));
        s->finals = (uint8_t*)malloc(T.n);
        word* S = (word*)calloc((size_t)W, sizeof(word));
        if (!s->maps || !s->table || !s->finals || !S) { free(S); oracle_nsfa_free(s); rc = E_CAP; goto fail; }
        memcpy(s->maps, T.sets, (size_t)T.n * MW * sizeof(word));
        memcpy(s->table, tab, (size_t)T.n * 256 * sizeof(uint32_t));
        for (uint32_t i = 0; i < T.n; i++) {
            /* line 11: F_s = {f | exists q in I: f(q) cap F != 0} */
            memset(S, 0, (size_t)W * sizeof(word));
            for (int w = 0; w < W; w++)
                for (word m = a->I[w]; m; m &= m - 1) {
                    int q = w * 64 + __builtin_ctzll(m);
                    for (int v = 0; v < W; v++) S[v] |= s->maps[(size_t)i * MW + (size_t)q * W + v];
                }
            s->finals[i] = (uint8_t)meets(S, a->F, W);
        }
        free(S);
        *out = s;
    }
fail:
    free(f); free(g); free(tab);
    free(T.sets); free(T.slot);
    return rc;
}

/* (f . g)(q) = U_{p in f(q)} g(p): the logical matrix product */
static void bool_compose(const word* f, const word* g, int n, int W, word* out) {
    memset(out, 0, (size_t)n * W * sizeof(word));
    for (int q = 0; q < n; q++)
        for (int w = 0; w < W; w++)
            for (word m = f[(size_t)q * W + w]; m; m &= m - 1) {
                int p = w * 64 + __builtin_ctzll(m);
                for (int v = 0; v < W; v++) out[(size_t)q * W + v] |= g[(size_t)p * W + v];
            }
}

/* Alg. 5 over an N-SFA with chunks [bounds[i], bounds[i+1]): per-chunk ids
 * (lines 1-5), the sequential reduction S <- I, S <- U_{p in S} f_i(p)
 * (right column) and the parallel one f_fin = f_1 . ... . f_p,
 * S <- U_{q in I} f_fin(q) (left column).  Writes both final sets (W words
 * each, nullable) and returns acc_seq | acc_par << 1, or -code. */
int oracle_nsfa_run_chunked(const oracle_nsfa* s, const uint8_t* text, const uint64_t* bounds, int p,
                            uint32_t* chunk_ids, uint64_t* set_seq, uint64_t* set_par) {
    if (p < 1) return -E_ARG;
    const oracle_nfa* a = s->a;
    const int n = a->n, W = a->W, MW = n * W;
    uint32_t* ids = (uint32_t*)malloc((size_t)p * sizeof(uint32_t));
    word* S = (word*)malloc((size_t)W * sizeof(word));
    word* T = (word*)malloc((size_t)W * sizeof(word));
    word* ff = (word*)malloc((size_t)MW * sizeof(word));
    word* tmp = (word*)malloc((size_t)MW * sizeof(word));
    if (!ids || !S || !T || !ff || !tmp) { free(ids); free(S); free(T); free(ff); free(tmp); return -E_CAP; }
    for (int i = 0; i < p; i++) {
        uint32_t f = 0;
        for (uint64_t j = bounds[i]; j < bounds[i + 1]; j++) f = s->table[(size_t)f * 256 + text[j]];
        ids[i] = f;
        if (chunk_ids) chunk_ids[i] = f;
    }
    memcpy(S, a->I, (size_t)W * sizeof(word));
    for (int i = 0; i < p; i++) {
        memset(T, 0, (size_t)W * sizeof(word));
        for (int w = 0; w < W; w++)
            for (word m = S[w]; m; m &= m - 1) {
                int q = w * 64 + __builtin_ctzll(m);
                for (int v = 0; v < W; v++) T[v] |= s->maps[(size_t)ids[i] * MW + (size_t)q * W + v];
            }
        memcpy(S, T, (size_t)W * sizeof(word));
    }
    int acc_seq = meets(S, a->F, W);
    if (set_seq) memcpy(set_seq, S, (size_t)W * sizeof(word));
    memcpy(ff, s->maps, (size_t)MW * sizeof(word));   /* id 0 = f_I */
    for (int i = 0; i < p; i++) {
        bool_compose(ff, s->maps + (size_t)ids[i] * MW, n, W, tmp);
        memcpy(ff, tmp, (size_t)MW * sizeof(word));
    }
    memset(S, 0, (size_t)W * sizeof(word));
    for (int w = 0; w < W; w++)
        for (word m = a->I[w]; m; m &= m - 1) {
            int q = w * 64 + __builtin_ctzll(m);
            for (int v = 0; v < W; v++) S[v] |= ff[(size_t)q * W + v];
        }
    int acc_par = meets(S, a->F, W);
    if (set_par) memcpy(set_par, S, (size_t)W * sizeof(word));
    free(ids); free(S); free(T); free(ff); free(tmp);
    return acc_seq | (acc_par << 1);
}

/* f_w for a word w by direct simulation from every state (brute-force pin
 * for |N-SFA|: the distinct f_w over all words up to some length). */
void oracle_nfa_word_map(const oracle_nfa* a, const uint8_t* w, int len, uint64_t* out) {
    const int n = a->n, W = a->W;
    word* S = (word*)malloc((size_t)W * sizeof(word));
    word* T = (word*)malloc((size_t)W * sizeof(word));
    for (int q = 0; q < n; q++) {
        memset(S, 0, (size_t)W * sizeof(word));
        S[q >> 6] = 1ull << (q & 63);
        for (int i = 0; i < len; i++) {
            nfa_step(a, S, w[i], T);
            word* x = S; S = T; T = x;
        }
        memcpy(out + (size_t)q * W, S, (size_t)W * sizeof(word));
    }
    free(S); free(T);
}
