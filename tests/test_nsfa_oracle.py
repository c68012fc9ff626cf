"""The oracle's NFA and N-SFA, pinned to the paper and
to independent computations, no GPU.

* The NFA run accepts exactly the regex's language:
  the oracle DFA (Alg. 1 + Alg. 2, separate code) and the brute-force AST
  evaluator agree on every string up to length 7/8.
* Theorem 3 for the N-SFA: any division of the text, both
  reductions of Alg. 5 (sequential, and the parallel one by logical matrix
  products), give the NFA run's final set.
* Example 3: the paper's n-state NFA for [ap]*[al][alp]{n-2}
  (transitions as the text describes them: 'a' arithmetic shift, 'l' logical
  shift, 'p' a shift from the second bit) has 2^n reachable state sets (Fact 1,
  counted here by a plain Python BFS); its N-SFA has exactly as many states as
  the distinct word mappings f_w (brute force over all words up to a length
  that reaches them) and as the D-SFA of the regex's minimal DFA (Alg. 4 in
  DFA form, separate code): both are the syntactic monoid, 2^(n+1) - n - 1.
"""
import itertools

import numpy as np
import pytest

import oracle as O
import workloads as W


def ex3_nfa(n):
    """The NFA of PAPER.md Fig./Ex. 3: state 0 loops on a,p; 0 -a,l-> 1; i -[alp]-> i+1; final n-1."""
    delta = {(0, ord("a")): {0, 1}, (0, ord("p")): {0}, (0, ord("l")): {1}}
    for q in range(1, n - 1):
        for c in b"alp":
            delta[(q, c)] = {q + 1}
    return O.OracleNFA.explicit(n, delta, {0}, {n - 1}, b"alp"), delta


def ex3_regex(n):
    return "[ap]*[al][alp]{%d}" % (n - 2)


@pytest.mark.parametrize("rx,alpha,chars,maxlen", [("(ab|ba)*c", b"abc", b"abc", 7),
                                                    ("([0-4]{2}[5-9]{2})*", b"0123456789", b"05x", 7),
                                                    (ex3_regex(5), b"alp", b"alp", 7),
                                                    ("a(b|c)*d?|e+", None, b"abcde", 6),
                                                    (".*a[ab]{3}", b"ab", b"ab", 8)])
def test_nfa_run_language(rx, alpha, chars, maxlen):
    nfa = O.OracleNFA(rx, alpha)
    dfa = O.OracleDFA(rx, alpha)
    for L in range(maxlen + 1):
        for w in itertools.product(chars, repeat=L):
            s = bytes(w)
            acc, _ = nfa.run(s)
            assert acc == dfa.run(s)[1] == bool(O.brute(rx, alpha, s)), (rx, s)


def test_nfa_run_random_regexes():
    from test_oracle import _random_regex
    rng = np.random.default_rng(5)
    for _ in range(60):
        rx = _random_regex(rng, 5)
        alpha = b"abcd"
        nfa = O.OracleNFA(rx, alpha)
        dfa = O.OracleDFA(rx, alpha)
        for _ in range(20):
            s = bytes(rng.choice(list(b"abcde"), size=int(rng.integers(0, 12))).tolist())
            assert nfa.run(s)[0] == dfa.run(s)[1], (rx, s)


@pytest.mark.parametrize("rx,alpha,gen", [("(ab|ba)*c", b"abc", lambda n: W.cfg1_accepted(n // 2)),
                                           ("([0-4]{5}[5-9]{5})*", b"0123456789", lambda n: W.cfg2_accepted(n // 10)),
                                           (".*a[ab]{8}", b"ab", W.cfg4_text),
                                           (ex3_regex(9), b"alp", lambda n: np.frombuffer(b"alp", np.uint8)[
                                               np.random.default_rng(1).integers(0, 3, size=n)])])
def test_nsfa_theorem3_both_reductions(rx, alpha, gen):
    """Any division, both reductions == the NFA run's final set and accept."""
    nfa = O.OracleNFA(rx, alpha)
    s = O.OracleNSFA(nfa)
    rng = np.random.default_rng(2)
    text = gen(20_000)
    for _ in range(8):
        n = int(rng.integers(0, text.size + 1))
        t = text[:n]
        acc, final = nfa.run(t)
        p = int(rng.integers(1, 40))
        cuts = np.sort(rng.integers(0, n + 1, size=p - 1))
        bounds = np.concatenate([[0], cuts, [n]]).astype(np.uint64)
        ids, (acc_s, set_s), (acc_p, set_p) = s.run_chunked(t, bounds)
        assert set_s == set_p == final and acc_s == acc_p == acc
        assert ids.size == p


@pytest.mark.parametrize("n", [3, 4, 5, 6, 8, 10])
def test_example3_sizes(n):
    nfa, delta = ex3_nfa(n)
    assert nfa.n == n
    # Fact 1: the subsets reachable from I = {0} -- all 2^n (plain BFS, independent of the C code)
    seen, todo = {frozenset({0})}, [frozenset({0})]
    while todo:
        S = todo.pop()
        for c in b"alp":
            T = frozenset(t for q in S for t in delta.get((q, c), ()))
            if T not in seen:
                seen.add(T)
                todo.append(T)
    assert len(seen) == 2 ** n
    # the regex's minimal DFA has 2^n states too (its dead state among them)
    dfa = O.OracleDFA(ex3_regex(n), b"alp")
    assert dfa.n == 2 ** n
    # N-SFA of the paper's NFA == D-SFA of the minimal DFA == 2^(n+1) - n - 1
    ns = O.OracleNSFA(nfa).n
    assert ns == O.OracleSFA(dfa).n == 2 ** (n + 1) - n - 1
    # brute force: the distinct word mappings f_w over all words up to length 2n + 1
    if n <= 5:
        maps = {nfa.word_map(bytes(w)) for L in range(2 * n + 2) for w in itertools.product(b"alp", repeat=L)}
        assert len(maps) == ns


def test_example3_nfa_language():
    """The explicit NFA of Ex. 3 accepts exactly [ap]*[al][alp]{n-2}."""
    n = 6
    nfa, _ = ex3_nfa(n)
    dfa = O.OracleDFA(ex3_regex(n), b"alp")
    for L in range(9):
        for w in itertools.product(b"alp", repeat=L):
            s = bytes(w)
            assert nfa.run(s)[0] == dfa.run(s)[1], s
