"""On-the-fly SFA construction (sfa_compile_lazy / sfa_match_lazy; PAPER.md:
532-542) and, through it, the paper's r_500 and r_a
(NEXT-2), whose D-SFA (1,000,999 / 1,001,000 states) is far
beyond the eager tables.

Checked against the oracle: results equal Alg. 2 of the oracle DFA (Theorem
2); every state built is a mapping of the oracle's full D-SFA (Alg. 4, where
that is small enough to build) and every transition built is coherent with
Lemma 1 (f_{T[s][b]} = f_s . delta(., b)); a second match of the same text
builds nothing; only the visited part of an exploding SFA (Ex. 4, |S| = n^n,
PAPER.md:893-906) is built.  Both with the factored chunk runs (C24:
a chunk that reaches a factorable state runs the DFA alone; no state past it
is built) and without them (tuning no_factor: every visited state is built).
"""
import numpy as np
import pytest

import oracle as O
import paper_1405_0562_b200 as P
import workloads as W

CFG2 = ("([0-4]{5}[5-9]{5})*", b"0123456789")


def test_lazy_handle_host_only():
    """Compile without a GPU: only the DFA; the SFA holds f_I; eager calls refuse."""
    sfa = P.SFA(W.rn_regex(500), b"0123456789", lazy=True)
    info = sfa.info()
    assert info["kind"] == 2 and info["sfa_states"] == 1 and info["dfa_states"] == 1001
    table, maps, finals = P.sfa_export_sfa(sfa.h)
    assert (maps[0] == np.arange(1001)).all()          # f_I (Def. 3)
    assert (table[0] == 0xFFFFFFFF).all()               # nothing built yet


def _lazy_coherent(sfa, d):
    """Lemma 1 on what was built: maps[T[s][b]][q] == dfa[maps[s][q]][b]."""
    table, maps, finals = P.sfa_export_sfa(sfa.h)
    dt, dfin = d.table, d.finals
    built = np.argwhere(table != 0xFFFFFFFF)
    for s, b in built[:: max(1, len(built) // 5000)]:
        assert (maps[table[s, b]] == dt[maps[s], b]).all(), (s, b)
    assert (finals == dfin[maps[:, 0]]).all()
    return table, maps


@pytest.mark.gpu
@pytest.mark.parametrize("no_factor", [0, 1])
@pytest.mark.parametrize("rx,alpha,gen", [("(ab|ba)*c", b"abc", lambda n: W.cfg1_accepted(n // 2)),
                                           (*CFG2, lambda n: W.cfg2_accepted(n // 10)),
                                           (".*a[ab]{8}", b"ab", W.cfg4_text),
                                           (W.rn_regex(20), b"0123456789", lambda n: W.rn_accepted(20, n))])
def test_lazy_parity_small(cuda_ok, rx, alpha, gen, no_factor):
    import torch
    d = O.OracleDFA(rx, alpha)
    full = O.OracleSFA(d)
    sfa = P.SFA(rx, alpha, lazy=True)
    sfa.set_tuning(no_factor=no_factor)
    text = gen(20 << 20)
    rng = np.random.default_rng(4)
    for n in (1, 100, 70_001, 5 << 20, text.size):
        t = text[:n].copy()
        if n > 1000 and rng.random() < 0.5:
            t[rng.integers(0, n)] = t[rng.integers(0, n)]
        assert sfa.match_lazy(torch.from_numpy(t).cuda()) == d.run(t), (rx, n)
    before = sfa.info()["lazy_transitions"]
    assert sfa.match_lazy(torch.from_numpy(text).cuda()) == d.run(text)
    assert sfa.info()["lazy_transitions"] == before          # the second pass builds nothing
    table, maps = _lazy_coherent(sfa, d)
    fm = {tuple(r) for r in full.maps.tolist()}
    assert all(tuple(r) in fm for r in maps.tolist())        # every built state is a D-SFA state
    assert sfa.info()["sfa_states"] <= full.n


@pytest.mark.gpu
@pytest.mark.parametrize("no_factor", [0, 1])
def test_lazy_r500_and_ra(cuda_ok, no_factor):
    """r_500 (|D| = 1001 with the dead state, |S| = 1,000,999) and r_a = r_500|a*
    on accepted / rejected texts: the oracle's Alg. 2, with only the visited
    states built (factored: only the states before each chunk's first
    factorable one -- a few per 1000-byte phase, far fewer)."""
    import torch
    rx, alpha = W.rn_regex(500), b"0123456789"
    d = O.OracleDFA(rx, alpha)
    assert d.n == 1001
    sfa = P.SFA(rx, alpha, lazy=True)
    sfa.set_tuning(no_factor=no_factor)
    t = W.rn_accepted(500, 64 << 20)
    r = t.copy()
    r[len(r) // 3] = ord("9") if r[len(r) // 3] < ord("5") else ord("0")
    for x in (t, r, t[:12_345_678], t[1:]):
        assert sfa.match_lazy(torch.from_numpy(x).cuda()) == d.run(x)
    info = sfa.info()
    assert 1 < info["sfa_states"] < (1_000_999 if no_factor else 300_000)
    _lazy_coherent(sfa, d)
    rxa = W.ra_regex(500)
    da = O.OracleDFA(rxa, b"0123456789a")
    sa = P.SFA(rxa, b"0123456789a", lazy=True)
    sa.set_tuning(no_factor=no_factor)
    for x in (W.ra_text(32 << 20), t[:5 << 20]):
        assert sa.match_lazy(torch.from_numpy(x).cuda()) == da.run(x)


@pytest.mark.gpu
def test_lazy_example4_explosion(cuda_ok):
    """Ex. 4: (m|(t|c([mt]*c){n-2})[cmt])* whose D-SFA has
    n^n states (8^8 = 16.7M for n = 8): matched with only the visited states."""
    import torch
    n = 8
    rx = "(m|(t|c([mt]*c){%d})[cmt])*" % (n - 2)
    d = O.OracleDFA(rx, b"cmt")
    sfa = P.SFA(rx, b"cmt", lazy=True)
    rng = np.random.default_rng(8)
    text = np.frombuffer(b"cmt", np.uint8)[rng.integers(0, 3, size=8 << 20)]
    assert sfa.match_lazy(torch.from_numpy(text).cuda()) == d.run(text)
    assert sfa.info()["sfa_states"] < n ** n
    _lazy_coherent(sfa, d)
