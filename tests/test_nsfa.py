"""The product's N-SFA (sfa_compile_nsfa).

CPU (the host construction, no compute call): its transition table and F_s
accept exactly the regex's language (the oracle DFA and brute force on every
short string), and for the paper's Ex. 3 its size is the oracle's N-SFA of the
paper's NFA = the oracle's D-SFA = 2^(n+1) - n - 1.
GPU: the same kernels and calls as the D-SFA, results bit-exact against the
oracle's Alg. 2 (canonical final state and accept), any chunking (Thm. 3),
batches, residency modes.
"""
import itertools

import numpy as np
import pytest

import oracle as O
import paper_1405_0562_b200 as P
import workloads as W
from test_nsfa_oracle import ex3_nfa, ex3_regex

CASES = [("(ab|ba)*c", b"abc", b"abc", 7), ("([0-4]{2}[5-9]{2})*", b"0123456789", b"05x", 6),
         (".*a[ab]{4}", b"ab", b"ab", 9), ("a(b|c)*d?|e+", None, b"abcde", 6)]


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1405_0562_b200 import _build
    _build.build()


@pytest.mark.parametrize("rx,alpha,chars,maxlen", CASES + [(ex3_regex(6), b"alp", b"alp", 8)])
def test_nsfa_table_language(rx, alpha, chars, maxlen):
    """Alg. 4 (general form) output run as an automaton: delta_s from f_I, accept
    = [f in F_s] -- equal to the oracle DFA and the brute-force AST evaluator."""
    h = P.sfa_compile(rx, alpha, 0, True)
    try:
        info = P.sfa_info(h)
        assert info["kind"] == 1 and info["nfa_states"] == info["nfa_positions"] + 1
        table, _, finals = P.sfa_export_sfa_table(h)
    finally:
        P.sfa_free(h)
    d = O.OracleDFA(rx, alpha)
    for L in range(maxlen + 1):
        for w in itertools.product(chars, repeat=L):
            s = 0
            for b in w:
                s = table[s, b]
            acc = bool(finals[s])
            assert acc == d.run(bytes(w))[1] == bool(O.brute(rx, alpha, bytes(w))), (rx, bytes(w))


@pytest.mark.parametrize("n", [3, 4, 5, 6, 7, 8, 9])
def test_nsfa_example3_size(n):
    h = P.sfa_compile(ex3_regex(n), b"alp", 0, True)
    try:
        info = P.sfa_info(h)
    finally:
        P.sfa_free(h)
    nfa, _ = ex3_nfa(n)
    assert info["sfa_states"] == O.OracleNSFA(nfa).n == 2 ** (n + 1) - n - 1
    assert info["dfa_states"] == 2 ** n and info["has_dfa"] == 1


def test_nsfa_refuses_mapping_calls():
    h = P.sfa_compile("(ab|ba)*c", b"abc", 0, True)
    try:
        with pytest.raises(P.SFAError) as e:
            P.sfa_set_compose(h, P.COMPOSE_VEC)
        assert e.value.code == P.SFA_ERR_CAPACITY
        with pytest.raises(P.SFAError):
            P.sfa_export_sfa(h)      # maps are set-valued
    finally:
        P.sfa_free(h)


# --------------------------------------------------------------------------- GPU
def _dev(torch, a, pad=0):
    buf = torch.empty(a.size + pad + 16, dtype=torch.uint8, device="cuda")
    v = buf[pad:pad + a.size]
    if a.size:
        v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return buf, v


@pytest.mark.gpu
@pytest.mark.parametrize("rx,alpha,gen", [("(ab|ba)*c", b"abc", lambda n: W.cfg1_accepted(n // 2)),
                                           ("([0-4]{5}[5-9]{5})*", b"0123456789", lambda n: W.cfg2_accepted(n // 10)),
                                           (".*a[ab]{8}", b"ab", W.cfg4_text),
                                           (ex3_regex(10), b"alp", lambda n: np.frombuffer(b"alp", np.uint8)[
                                               np.random.default_rng(3).integers(0, 3, size=n)])])
def test_nsfa_gpu_parity(cuda_ok, rx, alpha, gen):
    import torch
    d = O.OracleDFA(rx, alpha)
    sfa = P.SFA(rx, alpha, nsfa=True)
    assert sfa.info()["kind"] == 1
    text = gen(9 << 20)
    rng = np.random.default_rng(7)
    for n in (0, 1, 17, 70_001, 3 << 20, text.size - 3, text.size):
        t = text[:n].copy()
        if n > 100 and rng.random() < 0.5:
            t[rng.integers(0, n)] = t[rng.integers(0, n)]
        buf, v = _dev(torch, t, int(rng.integers(0, 16)))
        assert sfa.match(v) == d.run(t), (rx, n)
    buf, v = _dev(torch, text[:200_003])
    for p in (1, 7, 777, 5000):
        q, acc, ids = sfa.match_chunked(v, p)
        assert (q, acc) == d.run(text[:200_003])
    texts, off = W.ragged_batch(5, 400, 50_000, alpha)
    res = torch.zeros(800, dtype=torch.int32, device="cuda")
    sfa.match_batch(torch.from_numpy(texts).cuda(), torch.from_numpy(off.astype(np.int64)).cuda(), 400, res)
    torch.cuda.synchronize()
    got = res.cpu().numpy().view(np.uint32).reshape(400, 2)
    qo, ao = d.run_batch(texts, off)
    assert (got[:, 0] == qo).all() and (got[:, 1] == ao).all()
    for m in (P.RES_SMEM_SHARED, P.RES_L2, P.RES_HOT_L2):
        sfa.set_residency(m)
        buf, v = _dev(torch, text[:5 << 20], 3)
        assert sfa.match(v) == d.run(text[:5 << 20]), m
