"""GPU parity for the paper's baseline, Alg. 3: the DFA run
speculatively from every state per chunk.

Bit-exact against the oracle's plain Alg. 3 (``OracleDFA.run_spec``): the
per-chunk mappings T_i[q] = delta^(q, chunk i) under SPEC's chunk rule
(C6) and (q_final, accept); and against Alg. 2 (``OracleDFA.run``)
with the automatic chunking, at sizes spanning many CTAs with ragged tails,
every alignment, empty texts, n < chunks, and full-size config 2.
"""
import numpy as np
import pytest

import oracle as O
import paper_1405_0562_b200 as P
import workloads as W

pytestmark = pytest.mark.gpu

CFG1 = ("(ab|ba)*c", b"abc")
CFG2 = ("([0-4]{5}[5-9]{5})*", b"0123456789")
CFG4 = (".*a[ab]{8}", b"ab")

_oracles = {}


def oracle_of(rx, alpha):
    if (rx, alpha) not in _oracles:
        _oracles[(rx, alpha)] = O.OracleDFA(rx, alpha)
    return _oracles[(rx, alpha)]


def spec_bounds(n, p):
    """SPEC's chunk rule (C6): floor(n/p), remainder to the leading chunks; n < p: n chunks."""
    p = min(p, n) if n else 1
    q, r = divmod(n, p)
    return np.array([g * q + min(g, r) for g in range(p + 1)], np.uint64)


def run_spec(torch, sfa, text, nchunks=0, want_maps=False, pad=0):
    buf = torch.empty(text.size + pad + 16, dtype=torch.uint8, device="cuda")
    v = buf[pad:pad + text.size]
    if text.size:
        v.copy_(torch.from_numpy(np.ascontiguousarray(text)))
    nd = sfa.info()["dfa_states"]
    p = min(nchunks, text.size) if text.size else 1
    maps = torch.full((max(p, 1) * nd,), 0xFFFF, dtype=torch.int32, device="cuda") if want_maps else None
    res = torch.zeros(2, dtype=torch.int32, device="cuda")
    sfa.match_speculative(v, res, nchunks, maps)
    torch.cuda.synchronize()
    r = res.cpu().numpy().view(np.uint32)
    out = (int(r[0]), bool(r[1]))
    if want_maps:
        return out, maps.cpu().numpy().view(np.uint32).reshape(max(p, 1), nd)
    return out


@pytest.fixture(scope="module")
def torch_cuda(cuda_ok):
    import torch
    return torch


@pytest.mark.parametrize("rx,alpha", [CFG1, CFG2, CFG4, (None, None)])
@pytest.mark.parametrize("nchunks", [1, 7, 64, 1000, 5000])
def test_chunk_maps_equal_oracle_alg3(torch_cuda, rx, alpha, nchunks):
    torch = torch_cuda
    if rx is None:
        rx, alpha = W.cfg3_regex(), None
        t = W.cfg3_text(1 << 16, plant=True)
    elif alpha == b"abc":
        t = W.cfg1_accepted(20_000)
    elif alpha == b"ab":
        t = W.cfg4_text(1 << 16)
    else:
        t = W.cfg2_accepted(6_001)
    t = t[: t.size - 3]  # ragged against every chunk count
    sfa = P.SFA(rx, alpha)
    d = oracle_of(rx, alpha)
    got, maps = run_spec(torch, sfa, t, nchunks, want_maps=True, pad=nchunks % 16)
    q, acc, emaps = d.run_spec(t, spec_bounds(t.size, nchunks))
    assert got == (q, acc) == d.run(t)
    np.testing.assert_array_equal(maps, emaps)


@pytest.mark.parametrize("rx,alpha,gen", [
    (*CFG1, lambda: W.cfg1_random()),
    (*CFG2, lambda: W.cfg2_accepted(1_600_003)),
    (*CFG4, lambda: W.cfg4_text(3 << 20)),
    (None, None, lambda: W.cfg3_text(1 << 21, plant=True)),
])
def test_auto_chunking_equals_alg2(torch_cuda, rx, alpha, gen):
    torch = torch_cuda
    if rx is None:
        rx = W.cfg3_regex()
    sfa = P.SFA(rx, alpha)
    d = oracle_of(rx, alpha)
    t = gen()
    rng = np.random.default_rng(9)
    for trial in range(4):
        n = t.size if trial == 0 else int(rng.integers(1, t.size))
        got = run_spec(torch, sfa, t[:n], pad=int(rng.integers(0, 16)))
        assert got == d.run(t[:n]) == sfa.match(torch.from_numpy(t[:n].copy()).cuda()), (n, got)


def test_empty_and_tiny_texts(torch_cuda):
    torch = torch_cuda
    for rx, alpha in (CFG1, CFG2, ("a*", b"a")):
        sfa = P.SFA(rx, alpha)
        d = oracle_of(rx, alpha)
        assert run_spec(torch, sfa, np.zeros(0, np.uint8)) == d.run(b"")
        got, maps = run_spec(torch, sfa, np.zeros(0, np.uint8), 4, want_maps=True)
        assert (maps[0] == np.arange(d.n)).all()          # T of no bytes = identity (Alg. 3 l.2-3)
        for s in (b"a", b"ab", b"abc", b"0", b"x", b"01234"):
            t = np.frombuffer(s, np.uint8)
            for p in (1, 3, 64):                            # p > n: n one-byte chunks (C6)
                got, maps = run_spec(torch, sfa, t, p, want_maps=True)
                q, acc, em = d.run_spec(t, spec_bounds(t.size, p))
                assert got == (q, acc) == d.run(t)
                np.testing.assert_array_equal(maps, em)


def test_cfg2_full_size_accept_and_reject(torch_cuda):
    torch = torch_cuda
    sfa = P.SFA(*CFG2)
    d = oracle_of(*CFG2)
    a = W.cfg2_accepted()
    assert run_spec(torch, sfa, a) == d.run(a) == (0, True)
    r = W.cfg2_rejected(text=a)
    assert run_spec(torch, sfa, r) == d.run(r) == (d.dead, False)


def test_repeated_launches_reuse_scratch(torch_cuda):
    """The grid fold's ticket resets itself: back-to-back launches of different
    shapes on one stream stay correct."""
    torch = torch_cuda
    sfa = P.SFA(*CFG4)
    d = oracle_of(*CFG4)
    t = W.cfg4_text(1 << 20)
    for n in (1 << 20, 12_345, 999_999, 17, 1 << 20):
        assert run_spec(torch, sfa, t[:n]) == d.run(t[:n])
