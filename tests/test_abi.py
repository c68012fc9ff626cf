"""The C-ABI library without a GPU: it loads, exports every symbol
include/sfa.h declares, and its host compiler (sfa_compile: Glushkov + Alg. 1 +
Hopcroft + Alg. 4) produces exactly the oracle's
canonical minimal DFA (Thompson + Alg. 1 + Moore, independent code) and the
paper's SFA worked examples.  No compute call is made (tables upload lazily)."""
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1405_0562_b200 as P
import workloads as W
from conftest import ROOT, golden_lines
from test_oracle import _random_regex

CFG1 = ("(ab|ba)*c", b"abc")
CFG2 = ("([0-4]{5}[5-9]{5})*", b"0123456789")
CFG4 = (".*a[ab]{8}", b"ab")


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1405_0562_b200 import _build
    _build.build()


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "sfa.h")).read()
    return sorted(set(re.findall(r"^\s*SFA_API\s+(?:int|void|const char\*)\s+(sfa_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    L = P.lib()
    syms = _header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(P.EXPORTS)


def test_library_exports_only_the_abi():
    out = os.popen(f"nm -D --defined-only {P.LIB_PATH}").read().split("\n")
    ours = sorted({l.split()[-1] for l in out if l.strip() and l.split()[-1].startswith("sfa")})
    assert ours == _header_symbols()


def _same_dfa(rx, alpha):
    d = O.OracleDFA(rx, alpha)
    h = P.sfa_compile(rx, alpha)
    try:
        table, finals = P.sfa_export_dfa(h)
        info = P.sfa_info(h)
    finally:
        P.sfa_free(h)
    assert info["dfa_states"] == d.n, rx
    assert int(info["dead_state"]) == (d.dead if d.dead >= 0 else 0xFFFFFFFF), rx
    assert (table == d.table).all(), rx
    assert (finals == d.finals).all(), rx
    return info


@pytest.mark.parametrize("rx,alpha", [CFG1, CFG2, CFG4, ("(ab)*", b"ab"), ("(ab)*", None),
                                      ("([0-4]{50}[5-9]{50})*", b"0123456789"),
                                      ("(([02468][13579]){5})*", b"0123456789"),
                                      ("[ap]*[al][alp]{6}", b"alp"), ("", b"ab"), (".*", b"ab"),
                                      ("[^a]", b"abc"), ("a{2,5}b+c?", None), ("\\d+\\.\\d*", None),
                                      ("[\\x00-\\x1f]x|\\n", None)])
def test_compiler_dfa_equals_oracle(rx, alpha):
    _same_dfa(rx, alpha)


def test_compiler_dfa_equals_oracle_cfg3():
    info = _same_dfa(W.cfg3_regex(), None)
    assert info["classes"] == 27 and 100 < info["dfa_states"] < 200


def test_compiler_dfa_equals_oracle_random_regexes():
    rng = np.random.default_rng(99)
    for _ in range(200):
        rx = _random_regex(rng, 6)
        _same_dfa(rx, b"abcd" if rng.random() < 0.7 else None)


@pytest.mark.parametrize("rx,alpha", [CFG1, CFG2, ("([0-4]{2}[5-9]{2})*", b"0123456789"), (".*a[ab]{4}", b"ab"),
                                      (".*(abc|bca|cab).*", None), ("(m|(t|c([mt]*c){1})[cmt])*", b"cmt"),
                                      ("(ab)*", b"ab")])
def test_compiler_sfa_equals_oracle(rx, alpha):
    """Alg. 4 in the product == Alg. 4 in the oracle, ids and all (C3)."""
    s = O.OracleSFA(O.OracleDFA(rx, alpha))
    h = P.sfa_compile(rx, alpha)
    try:
        table, maps, finals = P.sfa_export_sfa(h)
    finally:
        P.sfa_free(h)
    assert table.shape == s.table.shape
    assert (table == s.table).all() and (maps == s.maps).all() and (finals == s.finals).all()


def test_table1_through_product():
    """Table I from sfa_compile."""
    t1 = {}
    for line in golden_lines("table1_ab_star.txt"):
        name, *img = line.split()
        t1[name] = [int(x) for x in img]
    h = P.sfa_compile("(ab)*", b"ab")
    table, maps, finals = P.sfa_export_sfa(h)
    P.sfa_free(h)
    assert maps.shape == (6, 3)
    for i in range(6):
        assert maps[i].tolist() == t1[f"f{i}"]
    # Example 1 trace: f0 -a-> f1 -b-> f4 -a-> f1 -b-> f4
    f, seen = 0, []
    for ch in b"abab":
        f = int(table[f, ch])
        seen.append(f)
    assert seen == [1, 4, 1, 4] and finals[4] == 1


def test_paper_sizes_through_product():
    for line in golden_lines("paper_sizes.txt"):
        name, rx, alpha, d_pr, s_pr, dead_counted, _cite = line.split("\t")
        h = P.sfa_compile(rx, None if alpha == "-" else alpha.encode())
        info = P.sfa_info(h)
        P.sfa_free(h)
        off = 0 if dead_counted == "yes" else 1
        assert info["dfa_states"] - off == int(d_pr), name
        assert info["sfa_states"] - off == int(s_pr), name


def test_example3_sizes_through_product():
    """Example 3 / Fact 1: |D| = 2^n (the SFA must also fit the cap)."""
    for line in golden_lines("example3_fact1.txt"):
        n, d = map(int, line.split())
        if n > 5:
            continue
        h = P.sfa_compile("[ap]*[al][alp]{%d}" % (n - 2), b"alp")
        assert P.sfa_info(h)["dfa_states"] == d
        P.sfa_free(h)


def test_errors_and_capacity():
    for rx, code in [("(ab", P.SFA_ERR_SYNTAX), ("a{3,2}", P.SFA_ERR_SYNTAX), ("(a)\\1", P.SFA_ERR_UNSUPPORTED),
                     ("^a", P.SFA_ERR_UNSUPPORTED), ("a{1001}", P.SFA_ERR_CAPACITY)]:
        with pytest.raises(P.SFAError) as e:
            P.sfa_compile(rx, None)
        assert e.value.code == code, rx
    # Example 4 n=4 has 257 SFA states (complete): a cap of 100 must refuse
    with pytest.raises(P.SFAError) as e:
        P.sfa_compile("(m|(t|c([mt]*c){2})[cmt])*", b"cmt", max_sfa=100)
    assert e.value.code == P.SFA_ERR_CAPACITY
    # r_500 exceeds the uint16 id space (|S| ~ 10^6)
    with pytest.raises(P.SFAError) as e:
        P.sfa_compile("([0-4]{300}[5-9]{300})*", b"0123456789")
    assert e.value.code == P.SFA_ERR_CAPACITY


def test_info_and_byte_window():
    """A1: the column window of each config (kernel section)."""
    T = P.COMPOSE_TABLE
    for (rx, alpha), lo, w, cm in [(CFG1, ord("a"), 4, T), (CFG2, ord("0"), 11, T), (CFG4, ord("a"), 3, T)]:
        h = P.sfa_compile(rx, alpha)
        info = P.sfa_info(h)
        P.sfa_free(h)
        assert (info["range_lo"], info["range_width"]) == (lo, w), rx
        assert info["compose_mode"] == cm
    h = P.sfa_compile(W.cfg3_regex(), None)
    info = P.sfa_info(h)
    P.sfa_free(h)
    # |S| ~ 20k > 4096: no composition table, |D| > 32: no vectors -> Lemma-1 replay
    assert (info["range_lo"], info["range_width"], info["compose_mode"]) == (ord("a"), 27, P.COMPOSE_REPLAY)
    assert 1 <= info["sfa_depth"] <= 16


def test_window_columns_cover_every_byte():
    """Every byte b maps to column min(b - lo mod 2^32, W-1) whose SFA column equals its class column."""
    rng = np.random.default_rng(5)
    for _ in range(50):
        rx = _random_regex(rng, 5)
        h = P.sfa_compile(rx, None)
        info = P.sfa_info(h)
        table, maps, finals = P.sfa_export_sfa(h)
        P.sfa_free(h)
        lo, w = info["range_lo"], info["range_width"]
        cols = [min((b - lo) % (1 << 32), w - 1) for b in range(256)]
        # bytes sharing a column must share the SFA transition column
        rep = {}
        for b, c in enumerate(cols):
            if c in rep:
                assert (table[:, b] == table[:, rep[c]]).all() or c < w - 1, (rx, b)
            else:
                rep[c] = b
        other = [b for b, c in enumerate(cols) if c == w - 1 and not (0 <= b - lo < w - 1)]
        for b in other:
            assert (table[:, b] == table[:, other[0]]).all(), (rx, b)


def test_set_compose_capacity():
    """sfa_set_compose refuses modes the automaton cannot use (no device needed)."""
    h = P.sfa_compile(*CFG4)          # |D| = 513 > 32
    with pytest.raises(P.SFAError) as e:
        P.sfa_set_compose(h, P.COMPOSE_VEC)
    assert e.value.code == P.SFA_ERR_CAPACITY
    P.sfa_set_compose(h, P.COMPOSE_REPLAY)
    assert P.sfa_info(h)["compose_mode"] == P.COMPOSE_REPLAY
    with pytest.raises(P.SFAError) as e:
        P.sfa_set_compose(h, 7)
    assert e.value.code == P.SFA_ERR_INVALID_ARG
    P.sfa_free(h)
    h = P.sfa_compile(W.cfg3_regex(), None)   # |S| ~ 20k > 4096
    with pytest.raises(P.SFAError) as e:
        P.sfa_set_compose(h, P.COMPOSE_TABLE)
    assert e.value.code == P.SFA_ERR_CAPACITY
    P.sfa_free(h)
    h = P.sfa_compile(*CFG2)
    for m in (P.COMPOSE_VEC, P.COMPOSE_TABLE, P.COMPOSE_REPLAY, P.COMPOSE_AUTO):
        P.sfa_set_compose(h, m)
    assert P.sfa_info(h)["compose_mode"] == P.COMPOSE_TABLE
    P.sfa_free(h)


def test_rn_family_through_product():
    """r_n: |S| = |D|^2 + |D| - 1 (live) up to the largest n
    whose D-SFA fits u16 ids (n = 127: 64,770 states); r_500's D-SFA
    (1,000,999 states) is refused with CAPACITY (reading C16)."""
    for n in (10, 100, 127):
        h = P.sfa_compile("([0-4]{%d}[5-9]{%d})*" % (n, n), b"0123456789")
        info = P.sfa_info(h)
        P.sfa_free(h)
        live = info["dfa_states"] - 1
        assert live == 2 * n and info["sfa_states"] - 1 == live * live + live - 1
    with pytest.raises(P.SFAError) as e:
        P.sfa_compile("([0-4]{500}[5-9]{500})*", b"0123456789")
    assert e.value.code == 3


def test_argument_checks_before_any_device_work():
    """Host-side argument checks of the async calls (no device call is made):
    Alg. 3 chunk maps need an explicit chunk count (the automatic
    count was not reported, the buffer could be overrun); NULL pointers and
    out-of-range tuning values are INVALID_ARG; an on-the-fly handle refuses
    the eager calls."""
    import ctypes as C
    L = P.lib()
    h = P.sfa_compile("(ab|ba)*c", b"abc")
    try:
        fake = C.c_void_p(0x1000)
        res = C.c_void_p(0x2000)
        assert L.sfa_match_speculative(h, fake, 100, 0, None, fake, res) == P.SFA_ERR_INVALID_ARG
        assert "explicit nchunks" in L.sfa_last_error().decode()
        assert L.sfa_match_batch(h, None, fake, 3, None, res) == P.SFA_ERR_INVALID_ARG
        assert L.sfa_match_async(h, None, 5, None, res) == P.SFA_ERR_INVALID_ARG
        assert L.sfa_match_rows(h, fake, 1000, None, fake, 10, None, res) == P.SFA_ERR_INVALID_ARG
        for bad in (dict(tma_k=3), dict(tma_rowb=32), dict(tma_k=1, tma_rowb=48), dict(row_align=96),
                    dict(dfa_copies=3), dict(direct_piece=8), dict(tma_promo=100), dict(dfa_u8=2)):
            with pytest.raises(P.SFAError) as e:
                P.sfa_set_tuning(h, **bad)
            assert e.value.code == P.SFA_ERR_INVALID_ARG, bad
        P.sfa_set_tuning(h, tma_k=2, tma_rowb=16, hot_rows=7, no_factor=1)
        P.sfa_set_tuning(h)
    finally:
        P.sfa_free(h)
    lz = P.sfa_compile("(ab|ba)*c", b"abc", lazy=True)
    try:
        assert L.sfa_match_async(lz, C.c_void_p(0x1000), 5, None, C.c_void_p(0x2000)) == P.SFA_ERR_INVALID_ARG
        assert "sfa_match_lazy" in L.sfa_last_error().decode()
    finally:
        P.sfa_free(lz)
