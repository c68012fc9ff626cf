"""Pins for the CPU oracle (oracle/), independent of the CUDA path.

Each test ties the oracle to something other than itself (ADVICE/prompt (3)):
values the paper prints (tests/golden/, each line cited), the regex's meaning
evaluated by brute force on every short string, Python's ``re`` library, closed
forms of the configs' languages, and algebraic invariants of the SFA
(Lemma 1, Theorem 3).
"""
import re

import numpy as np
import pytest

import oracle as O
import workloads as W
from conftest import golden_lines

CFG1 = ("(ab|ba)*c", b"abc")
CFG2 = ("([0-4]{5}[5-9]{5})*", b"0123456789")
CFG4 = (".*a[ab]{8}", b"ab")


# --------------------------------------------------------------------------- paper worked examples
def _table1():
    maps = {}
    for line in golden_lines("table1_ab_star.txt"):
        name, *img = line.split()
        maps[name] = [int(x) for x in img]
    return maps


def test_table1_dfa_and_sfa_mappings():
    """Fig. 1 DFA and Table I under the canonical numbering C3."""
    d = O.OracleDFA("(ab)*", "ab")
    assert d.n == 3 and d.dead == 2
    a, b = ord("a"), ord("b")
    assert d.table[:, [a, b]].tolist() == [[1, 2], [2, 0], [2, 2]]
    assert d.finals.tolist() == [1, 0, 0]
    s = O.OracleSFA(d)
    t1 = _table1()
    assert s.n == 6
    for i in range(6):
        assert s.maps[i].tolist() == t1[f"f{i}"], f"f{i}"


def test_example1_and_example2():
    lines = list(golden_lines("example1_2.txt"))
    d = O.OracleDFA("(ab)*", "ab")
    s = O.OracleSFA(d)
    name = {f"f{i}": i for i in range(6)}
    inv = {v: k for k, v in name.items()}
    compose = lambda f, g: [s.maps[g][s.maps[f][q]] for q in range(3)]   # (f . g)(q) = g(f(q))
    for line in lines:
        kind, *rest = line.split()
        if kind == "trace":
            word, *states = rest
            f = 0
            seen = [inv[f]]
            for ch in word.encode():
                f = int(s.table[f, ch])
                seen.append(inv[f])
            assert seen == states
        elif kind == "accepting":
            assert s.finals[name[rest[0]]] == 1
        elif kind == "chunks":
            chunks = [c.encode() for c in rest]
        elif kind == "chunk_states":
            text = b"".join(chunks)
            bounds = np.cumsum([0] + [len(c) for c in chunks])
            ids, q_seq, q_par = s.run_chunked(text, bounds)
            assert [inv[int(i)] for i in ids] == rest
            assert q_seq == q_par == d.run(text)[0]
        elif kind == "compose":
            f, g, h = (name[x] for x in rest)
            assert compose(f, g) == s.maps[h].tolist()
        elif kind == "sequential":
            assert q_seq == int(rest[0])


def test_paper_sizes():
    """|D| and |S_d| printed in the paper (C4: dead state counted or not)."""
    for line in golden_lines("paper_sizes.txt"):
        name, regex, alpha, nd, ns, dead_counted, _cite = line.split("\t")
        d = O.OracleDFA(regex, None if alpha == "-" else alpha)
        s = O.OracleSFA(d)
        if dead_counted == "yes":
            assert (d.n, s.n) == (int(nd), int(ns)), name
        else:
            assert d.dead >= 0
            # the dead state and the constant-dead mapping are not counted
            assert (d.live, s.n - 1) == (int(nd), int(ns)), name


def test_example3_fact1_dfa_sizes():
    for line in golden_lines("example3_fact1.txt"):
        n, nd = (int(x) for x in line.split())
        d = O.OracleDFA(f"[ap]*[al][alp]{{{n - 2}}}", "alp")
        assert d.n == nd == 2 ** n


def test_example4_fact2_sfa_is_full_transformation_monoid():
    for n in (3, 4):
        d = O.OracleDFA(f"(m|(t|c([mt]*c){{{n - 2}}})[cmt])*", "cmt")
        s = O.OracleSFA(d)
        live = [q for q in range(d.n) if q != d.dead]
        assert len(live) == n
        # every mapping of the live states into themselves occurs (|S_d| = |D|^|D|)
        imgs = {tuple(s.maps[i, live]) for i in range(s.n) if d.dead not in s.maps[i, live]}
        assert len(imgs) == n ** n


@pytest.mark.parametrize("n", [2, 5, 50])
def test_rn_square_law(n):
    """r_n: |S| = |D|^2 + |D| - 1 in the live convention."""
    d = O.OracleDFA(f"([0-4]{{{n}}}[5-9]{{{n}}})*", "0123456789")
    s = O.OracleSFA(d)
    assert d.live == 2 * n
    assert s.n - 1 == d.live ** 2 + d.live - 1


def test_canonical_ids_of_configs():
    """Reading C3 applied to configs 1, 2, 4."""
    d = O.OracleDFA(*CFG1)
    assert d.n == 5 and d.dead == 4
    assert [int(d.table[0, ord(c)]) for c in "abc"] == [1, 2, 3]
    assert np.flatnonzero(d.finals).tolist() == [3]
    d = O.OracleDFA(*CFG2)
    assert d.n == 11 and d.dead == 2 and np.flatnonzero(d.finals).tolist() == [0]
    d = O.OracleDFA(*CFG4)
    assert d.n == 513 and d.dead == 512
    d = O.OracleDFA(CFG4[0], None)
    assert d.n == 512 and d.dead == -1


# --------------------------------------------------------------------------- brute force
def _check_brute(regex, alphabet, chars, maxlen):
    texts, off = O.all_strings(chars, maxlen)
    expect = O.brute_all(regex, alphabet, chars, maxlen)
    d = O.OracleDFA(regex, alphabet)
    q, acc = d.run_batch(texts, off)
    bad = np.flatnonzero(expect != acc.astype(bool))
    assert bad.size == 0, (regex, [bytes(texts[off[i]:off[i + 1]]) for i in bad[:5]])
    return d, q, acc


def test_brute_cfg1_all_strings_len8():
    _check_brute(*CFG1, b"abcx", 8)


def test_brute_cfg2_all_strings_len8():
    # class representatives of both halves plus one out-of-Sigma byte
    _check_brute(*CFG2, b"0459x", 8)


def test_brute_cfg4_all_strings_len12():
    d, q, acc = _check_brute(*CFG4, b"ab", 12)
    _check_brute(*CFG4, b"abc", 8)
    assert acc[:2 ** 9 - 1].sum() == 0       # every string shorter than 9 is rejected


def test_brute_cfg3_scaled_word_set():
    words = ("abca", "bcab", "cabba", "aaab", "ccc")
    regex = ".*(" + "|".join(words) + ").*"
    _check_brute(regex, None, b"abcd", 7)


def test_brute_paper_examples():
    _check_brute("(ab)*", b"ab", b"abx", 10)
    _check_brute("([0-4]{2}[5-9]{2})*", b"0123456789", b"05x", 9)
    _check_brute("[ap]*[al][alp]{3}", b"alp", b"alp", 8)
    _check_brute("(m|(t|c([mt]*c){2})[cmt])*", b"cmt", b"cmt", 8)
    _check_brute("(([02468][13579]){5})*", b"0123456789", b"01", 12)


def _random_regex(rng, depth):
    if depth == 0 or rng.random() < 0.25:
        k = rng.integers(0, 6)
        if k < 3:
            return "abcd"[rng.integers(0, 4)]
        if k == 3:
            return "[" + "".join(sorted(set(rng.choice(list("abcd"), size=2)))) + "]"
        if k == 4:
            return "[^" + "abcd"[rng.integers(0, 4)] + "]"
        return "."
    k = rng.integers(0, 7)
    sub = lambda: _random_regex(rng, depth - 1)
    if k == 0:
        return sub() + sub()
    if k == 1:
        return "(" + sub() + "|" + sub() + ")"
    if k == 2:
        return "(" + sub() + ")*"
    if k == 3:
        return "(" + sub() + ")+"
    if k == 4:
        return "(" + sub() + ")?"
    if k == 5:
        lo = int(rng.integers(0, 3))
        hi = lo + int(rng.integers(0, 2))
        return "(" + sub() + "){%d,%d}" % (lo, hi)
    return sub() + sub() + sub()


def test_brute_random_regexes():
    """SPEC AC 6: random ASTs of depth <= 6 over {a,b,c,d}; every
    string of length <= 5 over {a,b,c,d} plus one out-of-Sigma byte."""
    rng = np.random.default_rng(1234)
    for _ in range(300):
        rx = _random_regex(rng, 6)
        _check_brute(rx, b"abcd", b"abcde", 5)


# --------------------------------------------------------------------------- library cross-check
def test_python_re_agrees():
    rng = np.random.default_rng(7)
    cases = [CFG1, CFG2, CFG4, ("(ab)*", b"ab"), ("[ap]*[al][alp]{4}", b"alp")]
    for _ in range(150):
        # shallow: Python's backtracking matcher is exponential on nested stars
        cases.append((_random_regex(rng, 3), b"abcd"))
    for rx, alpha in cases:
        d = O.OracleDFA(rx, alpha)
        pat = re.compile(rx.encode(), re.DOTALL)
        al = np.frombuffer(alpha, np.uint8)
        for _ in range(40):
            t = bytes(al[rng.integers(0, al.size, size=int(rng.integers(0, 16)))])
            assert d.run(t)[1] == (pat.fullmatch(t) is not None), (rx, t)


def test_python_re_on_long_texts():
    for rx, alpha, t in [(*CFG1, W.cfg1_accepted(50_000)), (*CFG2, W.cfg2_accepted(100_000)),
                         (*CFG4, W.cfg4_text(1 << 20))]:
        d = O.OracleDFA(rx, alpha)
        assert d.run(t)[1] == (re.fullmatch(rx.encode(), t.tobytes(), re.DOTALL) is not None)


# --------------------------------------------------------------------------- closed forms
def test_closed_forms_cfg1():
    d = O.OracleDFA(*CFG1)
    assert d.run(W.cfg1_accepted(10_000)) == (3, True)
    assert d.run(W.cfg1_random(1 << 16)) == (4, False)
    assert d.run(b"") == (0, False) and d.run(b"c") == (3, True)


def test_closed_forms_cfg2():
    d = O.OracleDFA(*CFG2)
    t = W.cfg2_accepted(3000)
    assert d.run(t) == (0, True)
    # the state after a prefix depends only on its length mod 10 (10 live states)
    rng = np.random.default_rng(0)
    by_phase = {}
    for L in rng.integers(0, t.size, size=400).tolist():
        by_phase.setdefault(L % 10, set()).add(d.run(t[:L])[0])
    assert all(len(v) == 1 for v in by_phase.values())
    assert len({next(iter(v)) for v in by_phase.values()}) == 10
    assert d.run(W.cfg2_rejected(3000)) == (2, False)


def test_closed_forms_cfg4():
    d = O.OracleDFA(*CFG4)
    rng = np.random.default_rng(3)
    for _ in range(50):
        t = W.cfg4_text(1000)[rng.integers(0, 500):]
        q, acc = d.run(t)
        assert acc == (t[-9] == ord("a"))
        pre = rng.integers(97, 99, size=int(rng.integers(1, 50)), dtype=np.uint8)
        assert d.run(np.concatenate([pre, t]))[0] == q        # depends on the last 9 bytes only


def test_closed_form_cfg3_contains():
    words = W.cfg3_words()
    d = O.OracleDFA(W.cfg3_regex(words), None)
    rng = np.random.default_rng(5)
    for i in range(20):
        t = W.letters(rng, 20_000)
        if i % 2:
            w = words[i]
            o = int(rng.integers(0, t.size - len(w)))
            t[o:o + len(w)] = np.frombuffer(w, np.uint8)
        tb = t.tobytes()
        assert d.run(t)[1] == any(w in tb for w in words)


# --------------------------------------------------------------------------- SFA algebra (Alg. 4 oracle)
SFA_CASES = [("(ab)*", b"ab"), CFG1, CFG2, ("([0-4]{2}[5-9]{2})*", b"0123456789"),
             (".*a[ab]{4}", b"ab"), (".*(abc|bca|cab).*", None), ("(m|(t|c([mt]*c){1})[cmt])*", b"cmt")]


@pytest.mark.parametrize("rx,alpha", SFA_CASES)
def test_sfa_lemma1_identity_associativity(rx, alpha):
    d = O.OracleDFA(rx, alpha)
    s = O.OracleSFA(d)
    M = s.maps.astype(np.int64)
    assert M[0].tolist() == list(range(d.n))                       # f_I
    comp = lambda f, g: M[g][M[f]]                                 # (f . g) = g o f
    # Lemma 1 coherence: map[T[s,b]] == map[s] . map[T[0,b]]
    for b in range(256):
        assert (M[s.table[:, b]] == M[s.table[0, b]][M]).all()
    rng = np.random.default_rng(11)
    for _ in range(2000):
        f, g, h = rng.integers(0, s.n, size=3)
        assert (comp(f, 0) == M[f]).all() and (comp(0, f) == M[f]).all()
        assert (M[h][M[g][M[f]]] == M[h][comp(f, g)]).all()        # (f.g).h == f.(g.h)
    # F_s (Def. 3): f accepting iff f(q0) is final
    assert (s.finals == d.finals[M[:, 0]]).all()


@pytest.mark.parametrize("rx,alpha", SFA_CASES)
def test_alg5_any_division(rx, alpha):
    """Theorem 3: every division gives Alg. 2's state, with
    both the sequential and the parallel reduction (Alg. 5)."""
    d = O.OracleDFA(rx, alpha)
    s = O.OracleSFA(d)
    rng = np.random.default_rng(2)
    al = np.frombuffer(alpha if alpha else b"abcx", np.uint8)
    for _ in range(60):
        n = int(rng.integers(0, 64))
        t = al[rng.integers(0, al.size, size=n)]
        q_ref = d.run(t)[0]
        for p in (1, 2, 3, 4, 7):
            cuts = np.sort(rng.integers(0, n + 1, size=p - 1))
            bounds = np.concatenate([[0], cuts, [n]])
            ids, q_seq, q_par = s.run_chunked(t, bounds)
            assert q_seq == q_par == q_ref


# --------------------------------------------------------------------------- errors and conventions
@pytest.mark.parametrize("rx,code", [("(ab", 1), ("ab)", 1), ("[z-a]", 1), ("a{3,2}", 1), ("*a", 1),
                                     ("a|*", 1), ("[abc", 1), ("a\\", 1), ("a{x}", 1), ("\\q", 1),
                                     ("(a)\\1", 2), ("(?=a)", 2), ("^a", 2), ("a$", 2), ("\\b", 2),
                                     ("a{1001}", 3)])
def test_parse_errors(rx, code):
    with pytest.raises(O.OracleError) as e:
        O.OracleDFA(rx, None)
    assert e.value.code == code


def test_sigma_and_empty_pattern():
    d = O.OracleDFA("(ab)*", None)          # Sigma = all bytes: byte 0x00 is visited first (C3)
    assert d.n == 3 and d.dead == 1 and d.table[0, ord("a")] == 2
    assert d.run(b"ab\x00") == (1, False)
    d = O.OracleDFA("", b"ab")              # empty pattern: only epsilon
    assert d.n == 2 and d.run(b"") == (0, True) and d.run(b"a") == (1, False)
    d = O.OracleDFA(".*", b"ab")            # out-of-Sigma byte -> dead (C2)
    assert d.run(b"abba")[1] and not d.run(b"abca")[1]
    d = O.OracleDFA("[^a]", b"abc")         # negation ranges over Sigma
    assert d.run(b"b")[1] and d.run(b"c")[1] and not d.run(b"a")[1] and not d.run(b"d")[1]


# --------------------------------------------------------------------------- input recipes
def test_workload_recipes():
    assert W.cfg1_accepted().size == (1 << 20) - 1
    assert W.cfg1_random().size == 1 << 20
    t = W.cfg2_accepted(1000)
    assert t.size == 10_000 and (t.reshape(-1, 10)[:, :5] < 53).all() and (t.reshape(-1, 10)[:, 5:] >= 53).all()
    words = W.cfg3_words()
    assert len(words) == 32 and len(set(words)) == 32 and all(4 <= len(w) <= 8 for w in words)
    t = W.cfg3_text(1 << 22)
    assert W.find_occurrences(t, words) == []
    tb = W.cfg3_text(1 << 22, plant=True).tobytes()
    assert any(w in tb for w in words)
    texts, off, idx = W.cfg5_batch(count=512, length=4096)
    assert idx.size == 51
    tb = texts.tobytes()
    hits = [any(w in tb[off[i]:off[i + 1]] for w in words) for i in range(512)]
    assert np.flatnonzero(hits).tolist() == idx.tolist()


# --------------------------------------------------------------------------- Alg. 3 (speculative DFA)
def _bounds(rng, n, p):
    cuts = np.sort(rng.integers(0, n + 1, size=p - 1))
    return np.concatenate([[0], cuts, [n]]).astype(np.uint64)


@pytest.mark.parametrize("rx,alpha", [CFG1, CFG2, CFG4, ("(ab)*", b"ab")])
def test_spec_equals_alg2_on_any_chunking(rx, alpha):
    """Alg. 3's ENSURE: q_final = delta^(q0, w), for any division
    of w (empty chunks included) -- against Alg. 2 and, on short words, against
    the brute-force evaluator of the regex."""
    d = O.OracleDFA(rx, alpha)
    rng = np.random.default_rng(31)
    chars = np.frombuffer(alpha + b"x", np.uint8)
    for n in (0, 1, 2, 9, 40, 333):
        t = rng.choice(chars, size=n).astype(np.uint8)
        for p in (1, 2, 5, 17):
            q, acc, maps = d.run_spec(t, _bounds(rng, n, p))
            assert (q, acc) == d.run(t)
            assert maps.shape == (p, d.n)
        if n <= 9:
            assert d.run_spec(t, [0, n])[1] == O.brute(rx, alpha, bytes(t))


def test_spec_maps_single_bytes_and_empty_chunk():
    """Lines 2-6 on a one-byte chunk give the DFA column (T_i[q] = delta(q, b),
    the DFA of Alg. 1 checked by the brute-force pins above); an empty chunk
    gives the identity (lines 2-3)."""
    d = O.OracleDFA(*CFG2)
    t = np.frombuffer(b"07x", np.uint8)
    _, _, maps = d.run_spec(t, [0, 1, 1, 2, 3])
    q = np.arange(d.n)
    assert (maps[0] == d.table.reshape(d.n, 256)[q, ord("0")]).all()
    assert (maps[1] == q).all()
    assert (maps[2] == d.table.reshape(d.n, 256)[q, ord("7")]).all()
    assert (maps[3] == d.dead).all()  # 'x' is outside Sigma: every state to the dead state (C2)


def test_spec_maps_compose_homomorphically():
    """T_{uv} = T_u . T_v with (f . g)(q) = g(f(q)): the chunk
    map of a concatenation is the composition of the chunk maps, in order."""
    d = O.OracleDFA(*CFG4)
    rng = np.random.default_rng(5)
    t = rng.choice(np.frombuffer(b"ab", np.uint8), size=200).astype(np.uint8)
    _, _, whole = d.run_spec(t, [0, 200])
    _, _, parts = d.run_spec(t, [0, 61, 200])
    assert (whole[0] == parts[1][parts[0]]).all()
    # closed form: cfg4's DFA remembers the last 9 bytes, so after >= 9 bytes
    # every live start state lands in the same state; the dead state (reached
    # only by out-of-Sigma bytes, C2) stays dead
    live = np.arange(d.n) != d.dead
    assert (whole[0][live] == whole[0][0]).all() and whole[0][d.dead] == d.dead


def test_spec_cfg2_block_closed_form():
    """Config 2: one accepted 10-byte block sends q0 back to q0 (the language
    is (block)*) and the dead state to itself; a full accepted text is accepted
    from q0 on any chunking."""
    d = O.OracleDFA(*CFG2)
    blk = W.cfg2_accepted(1)
    _, _, m = d.run_spec(blk, [0, 10])
    assert m[0][0] == 0 and m[0][d.dead] == d.dead
    t = W.cfg2_accepted(1000)
    assert d.run_spec(t, np.linspace(0, t.size, 8).astype(np.uint64)) [:2] == (0, True)


def test_rn_dfa_sizes_printed_for_r500_and_ra():
    """The r_500 and r_a captions (|D| = 1000 and 1002, no dead state, C4)."""
    for line in golden_lines("rn_dfa_sizes.txt"):
        name, regex, alpha, nd, _cite = line.split("\t")
        d = O.OracleDFA(regex, alpha)
        assert d.dead >= 0 and d.live == int(nd), name
