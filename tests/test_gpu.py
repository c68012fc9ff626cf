"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bit-exact on (final DFA state, accept bit) per text, and on the per-chunk SFA
ids where the chunking is forced (canonical ids, C3), for all five
BASELINE.json configs at full size, scaled sizes spanning several tiles with
ragged tails, every residency mode, batches with empty and ragged texts, and
the host-buffer end-to-end call.  The oracle is Alg. 2 of
an independently built DFA; chunk ids come from the oracle's plain Alg. 5.
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


@pytest.fixture(scope="module")
def torch_cuda(cuda_ok):
    import torch
    return torch


def dev(torch, a: np.ndarray, pad_front: int = 0):
    """Device copy of a uint8 array, starting `pad_front` bytes into a buffer
    (so the text's address has any alignment)."""
    buf = torch.empty(a.size + pad_front + 16, dtype=torch.uint8, device="cuda")
    v = buf[pad_front:pad_front + a.size]
    if a.size:
        v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return buf, v


def spec_bounds(n, p):
    """SPEC's chunk rule (C6): floor(n/p), remainder to the leading chunks."""
    p = min(p, n) if n else 1
    q, r = divmod(n, p)
    return np.array([g * q + min(g, r) for g in range(p + 1)], np.uint64)


_cache = {}


def oracle_pair(rx, alpha):
    key = (rx, alpha)
    if key not in _cache:
        d = O.OracleDFA(rx, alpha)
        _cache[key] = d
    return _cache[key]


def check_text(torch, sfa, d, text, pad=0):
    buf, v = dev(torch, text, pad)
    got = sfa.match(v)
    exp = d.run(text)
    assert got == exp, (len(text), pad, got, exp)
    return got


# --------------------------------------------------------------------------- config 1
def test_cfg1_full_size_and_forced_chunk_counts(torch_cuda):
    torch = torch_cuda
    sfa = P.SFA(*CFG1)
    d = oracle_pair(*CFG1)
    s = O.OracleSFA(d)
    for text, exp in [(W.cfg1_random(), (4, False)), (W.cfg1_accepted(), (3, True))]:
        assert d.run(text) == exp                          # closed form
        assert check_text(torch, sfa, d, text) == exp
        buf, v = dev(torch, text)
        for p in (1, 7, 64, 4096):
            q, acc, ids = sfa.match_chunked(v, p)
            assert (q, acc) == exp, p
            o_ids, q_seq, q_par = s.run_chunked(text, spec_bounds(text.size, p))
            assert q_seq == q_par == exp[0]
            assert ids.tolist() == o_ids.tolist(), p           # bit-exact per-chunk SFA ids


def test_cfg1_random_chunkings(torch_cuda):
    torch = torch_cuda
    sfa = P.SFA(*CFG1)
    d = oracle_pair(*CFG1)
    s = O.OracleSFA(d)
    rng = np.random.default_rng(3)
    for _ in range(20):
        n = int(rng.integers(1, 5000))
        # mostly-accepted texts so the state is not stuck in the dead state
        t = W.cfg1_accepted(n // 2)
        if rng.random() < 0.5:
            t = t.copy()
            t[rng.integers(0, t.size)] = np.uint8(rng.integers(97, 100))
        buf, v = dev(torch, t, int(rng.integers(0, 16)))
        for p in (1, 2, 3, 7, int(rng.integers(1, n + 2))):
            q, acc, ids = sfa.match_chunked(v, p)
            o_ids, q_seq, _ = s.run_chunked(t, spec_bounds(t.size, p))
            assert (q, acc) == d.run(t)
            assert ids.tolist() == o_ids.tolist()


# --------------------------------------------------------------------------- config 2
def test_cfg2_full_size_accept_and_reject(torch_cuda):
    torch = torch_cuda
    sfa = P.SFA(*CFG2)
    d = oracle_pair(*CFG2)
    a = W.cfg2_accepted()
    assert a.size == 268_435_450
    assert check_text(torch, sfa, d, a) == (0, True)
    r = W.cfg2_rejected(text=a)
    assert check_text(torch, sfa, d, r) == (2, False)
    # same text at every 16-byte misalignment (head piece), and prefixes (ragged tail)
    buf, v = dev(torch, a, 5)
    assert sfa.match(v) == (0, True)
    for cut in (1, 9, 15, 17, 12345, 1 << 20):
        t = a[:a.size - cut]
        assert sfa.match(v[:a.size - cut]) == d.run(t), cut


def test_cfg2_scaled_sizes_every_alignment(torch_cuda):
    """Sizes around the direct/TMA switch and the per-SM row count, all 16 alignments."""
    torch = torch_cuda
    sfa = P.SFA(*CFG2)
    d = oracle_pair(*CFG2)
    base = W.cfg2_accepted(1_200_000)          # 12 MB
    rng = np.random.default_rng(8)
    sizes = [0, 1, 15, 16, 17, 255, 4096, 65537, (4 << 20) - 1, 4 << 20, (4 << 20) + 1, 4_757_011,
             10 * 148 * 992 + 7, 12_000_000]
    for n in sizes:
        t = base[:n].copy()
        if n > 100 and rng.random() < 0.5:
            t[rng.integers(0, n)] = np.uint8(48 + rng.integers(0, 10))   # maybe rejected
        for pad in (0, 1, 7, 15):
            check_text(torch, sfa, d, t, pad)


def test_cfg2_text_beyond_4_gib(torch_cuda):
    """Maximum sizes: one text (and a batch) past 2^32 bytes, so every offset,
    row start and row length of the plan needs 64 bits.  cfg2's DFA does not
    synchronise (the state is the position mod 10), so a row that starts at a
    truncated offset, or a byte past 4 GiB that is never read, changes the
    result.  Expected values: the oracle's Alg. 2 over the whole host text."""
    torch = torch_cuda
    sfa = P.SFA(*CFG2)
    d = oracle_pair(*CFG2)
    a = W.cfg2_accepted()                       # 268,435,450 bytes, a multiple of the 10-byte block
    reps = 17                                   # 4,563,402,650 bytes > 2^32
    n = reps * a.size + 7                       # ragged: ends 7 bytes into a block
    host = np.empty(n, np.uint8)
    for k in range(reps):
        host[k * a.size:(k + 1) * a.size] = a
    host[reps * a.size:] = a[:7]
    assert n > (1 << 32)
    buf, v = dev(torch, host, 3)
    exp = d.run(host)
    assert exp[0] != 2 and not exp[1]           # 7 bytes into a block: a live, non-final state
    assert sfa.match(v) == exp
    assert sfa.match(v[:reps * a.size]) == (0, True)      # whole blocks: accepted (closed form, C12)
    # one wrong-half digit past 2^32: dead state 2 (closed form) -- the bytes past 4 GiB are read
    pos = (1 << 32) + 123_456_789
    old = int(host[pos])
    host[pos] = 48 + (old - 48 + 5) % 10
    v[pos:pos + 1].copy_(torch.from_numpy(host[pos:pos + 1]))
    exp_r = d.run(host)
    assert exp_r == (2, False)
    assert sfa.match(v) == exp_r
    host[pos] = old
    v[pos:pos + 1].copy_(torch.from_numpy(host[pos:pos + 1]))
    # a batch over the same buffer whose offsets pass 2^32 (an empty text among them)
    off = np.array([0, 10, (1 << 32) + 5, (1 << 32) + 5, n - 7, n], np.uint64)
    count = off.size - 1
    do = torch.from_numpy(off.astype(np.int64)).cuda()
    res = torch.zeros(2 * count, dtype=torch.int32, device="cuda")
    sfa.match_batch(v, do, count, res)
    torch.cuda.synchronize()
    r = res.cpu().numpy().view(np.uint32).reshape(count, 2)
    qo, acco = d.run_batch(host, off)
    assert (r[:, 0] == qo).all() and (r[:, 1] == acco).all(), (r, qo, acco)


# --------------------------------------------------------------------------- config 3
def test_cfg3_full_size_contains_match(torch_cuda):
    torch = torch_cuda
    rx = W.cfg3_regex()
    sfa = P.SFA(rx, None)
    d = oracle_pair(rx, None)
    t = W.cfg3_text()
    assert check_text(torch, sfa, d, t)[1] is False
    words = W.cfg3_words()
    s = W._streams(3)
    w = words[int(s[3].integers(0, len(words)))]
    off = int(s[2].integers(0, t.size - len(w) + 1))
    t[off:off + len(w)] = np.frombuffer(w, np.uint8)          # == cfg3_text(plant=True)
    assert check_text(torch, sfa, d, t)[1] is True


def test_cfg3_scaled_with_planted_words(torch_cuda):
    torch = torch_cuda
    rx = W.cfg3_regex()
    sfa = P.SFA(rx, None)
    d = oracle_pair(rx, None)
    t0 = W.cfg3_text(1 << 23)
    rng = np.random.default_rng(4)
    words = W.cfg3_words()
    for trial in range(12):
        t = t0[: int(rng.integers(1, t0.size))].copy()
        if trial % 2:
            w = words[int(rng.integers(0, 32))]
            if len(w) <= t.size:
                o = int(rng.integers(0, t.size - len(w) + 1))
                t[o:o + len(w)] = np.frombuffer(w, np.uint8)
        if trial % 3 == 0:
            t[rng.integers(0, t.size)] = np.uint8(rng.integers(0, 256))   # out-of-window byte
        check_text(torch, sfa, d, t, int(rng.integers(0, 16)))


# --------------------------------------------------------------------------- config 4
def test_cfg4_full_size(torch_cuda):
    torch = torch_cuda
    sfa = P.SFA(*CFG4)
    d = oracle_pair(*CFG4)
    t = W.cfg4_text()
    q, acc = check_text(torch, sfa, d, t)
    assert acc == (t[-9] == ord("a"))                         # closed form


# --------------------------------------------------------------------------- config 5 (batch)
def _batch(torch, sfa, texts, off):
    count = off.size - 1
    bt, vt = dev(torch, texts)
    do = torch.from_numpy(off.astype(np.int64)).cuda()
    res = torch.zeros(2 * count, dtype=torch.int32, device="cuda")
    sfa.match_batch(vt if texts.size else bt, do, count, res)
    torch.cuda.synchronize()
    r = res.cpu().numpy().view(np.uint32).reshape(count, 2)
    return r[:, 0], r[:, 1]


def test_cfg5_full_size_batch(torch_cuda):
    torch = torch_cuda
    rx = W.cfg3_regex()
    sfa = P.SFA(rx, None)
    d = oracle_pair(rx, None)
    texts, off, idx = W.cfg5_batch()
    q, acc = _batch(torch, sfa, texts, off)
    qo, acco = d.run_batch(texts, off)
    assert (q == qo).all() and (acc == acco).all()
    assert np.flatnonzero(acc).tolist() == idx.tolist()        # exactly the planted texts
    # the launch configuration bench.py times: equal texts through sfa_match_batch_uniform
    count, length = off.size - 1, int(off[1] - off[0])
    dt = torch.from_numpy(texts).cuda()
    res = torch.zeros(2 * count, dtype=torch.int32, device="cuda")
    sfa.match_batch_uniform(dt, length, count, res)
    torch.cuda.synchronize()
    r = res.cpu().numpy().view(np.uint32).reshape(count, 2)
    assert (r[:, 0] == qo).all() and (r[:, 1] == acco).all()


@pytest.mark.parametrize("rx,alpha", [CFG1, CFG2, CFG4, (W.cfg3_regex(), None)])
def test_batch_ragged_with_empty_texts(torch_cuda, rx, alpha):
    torch = torch_cuda
    sfa = P.SFA(rx, alpha)
    d = oracle_pair(rx, alpha)
    for seed, count, max_len in [(1, 1, 0), (2, 3, 10), (3, 500, 3000), (4, 40, 300_000)]:
        texts, off = W.ragged_batch(seed, count, max_len, alpha if alpha else b"abcdefghijklmnopqrstuvwxyz")
        q, acc = _batch(torch, sfa, texts, off)
        qo, acco = d.run_batch(texts, off)
        assert (q == qo).all() and (acc == acco).all(), (seed, count)


def test_batch_count_zero_is_noop(torch_cuda):
    sfa = P.SFA(*CFG1)
    sfa.match_batch(0, 0, 0, 0)


# --------------------------------------------------------------------------- residency modes
@pytest.mark.parametrize("factor", [1, 0])
@pytest.mark.parametrize("hot_rows", [0, 7])
@pytest.mark.parametrize("rx,alpha,modes", [(*CFG1, (P.RES_SMEM_PRIVATE, P.RES_SMEM_SHARED, P.RES_HOT_L2, P.RES_L2)),
                                            (*CFG2, (P.RES_SMEM_PRIVATE, P.RES_SMEM_SHARED, P.RES_HOT_L2, P.RES_L2)),
                                            (*CFG4, (P.RES_SMEM_PRIVATE, P.RES_SMEM_SHARED, P.RES_HOT_L2, P.RES_L2)),
                                            (W.cfg3_regex(), None, (P.RES_HOT_L2, P.RES_L2))])
def test_every_residency_mode(torch_cuda, rx, alpha, modes, hot_rows, factor):
    """A6: every table placement gives the oracle's result; hot_rows=7 keeps
    only 7 renumbered rows in smem so nearly every HOT lookup takes the
    global (L2) path; factor=0 disables the FACTORED step."""
    torch = torch_cuda
    d = oracle_pair(rx, alpha)
    sfa = P.SFA(rx, alpha)
    sfa.set_tuning(hot_rows=hot_rows, no_factor=1 - factor)
    rng = np.random.default_rng(6)
    al = np.frombuffer(alpha if alpha else b"abcdefghijklmnopqrstuvwxyz", np.uint8)
    texts = [al[rng.integers(0, al.size, size=n)] for n in (1, 1000, 5_000_000)]
    if rx == CFG2[0]:
        texts.append(W.cfg2_accepted(700_000))
    if rx == CFG1[0]:
        texts.append(W.cfg1_accepted(3_000_000))
    for m in modes:
        sfa.set_residency(m)
        assert P.sfa_info(sfa.h)["residency"] == m
        for t in texts:
            check_text(torch, sfa, d, t, 3)


def test_private_capacity_refused_for_big_table(torch_cuda):
    sfa = P.SFA(W.cfg3_regex(), None)
    with pytest.raises(P.SFAError) as e:
        sfa.set_residency(P.RES_SMEM_PRIVATE)
    assert e.value.code == P.SFA_ERR_CAPACITY


# --------------------------------------------------------------------------- random regexes
def test_random_regexes_small_texts(torch_cuda):
    torch = torch_cuda
    from test_oracle import _random_regex
    rng = np.random.default_rng(21)
    for _ in range(40):
        rx = _random_regex(rng, 5)
        alpha = b"abcd" if rng.random() < 0.6 else None
        d = O.OracleDFA(rx, alpha)
        sfa = P.SFA(rx, alpha)
        for n in (0, 1, 2, 33, 700, 20_000):
            t = np.frombuffer(b"abcde", np.uint8)[rng.integers(0, 5, size=n)]
            check_text(torch, sfa, d, t, int(rng.integers(0, 16)))


# --------------------------------------------------------------------------- API entry points
def test_empty_text_and_async_and_host(torch_cuda):
    torch = torch_cuda
    sfa = P.SFA("(ab)*", b"ab")
    empty = torch.empty(0, dtype=torch.uint8, device="cuda")
    assert sfa.match(empty) == (0, True)
    res = torch.zeros(2, dtype=torch.int32, device="cuda")
    t = np.frombuffer(b"ab" * 3_000_000, np.uint8)
    buf, v = dev(torch, t)
    sfa.match_async(v, res)
    torch.cuda.synchronize()
    assert res.cpu().tolist() == [0, 1]
    sfa.match_async(empty, res)
    torch.cuda.synchronize()
    assert res.cpu().tolist() == [0, 1]
    assert sfa.match_host(t) == (0, True)
    assert sfa.match_host(t[:-1]) == (1, False)


def test_match_host_slices_full_cfg2(torch_cuda):
    """sfa_match_host: 64 MiB slices chained by q_in (sequential reduction across
    slices) from pinned memory == Alg. 2."""
    torch = torch_cuda
    sfa = P.SFA(*CFG2)
    d = oracle_pair(*CFG2)
    a = W.cfg2_accepted()
    pinned = torch.from_numpy(a).pin_memory()
    assert sfa.match_host(pinned) == (0, True)
    for n in (a.size - 3, (64 << 20) + 5, (128 << 20) - 1):
        assert sfa.match_host(pinned[:n]) == d.run(a[:n]), n
    r = W.cfg2_rejected(text=a)
    assert sfa.match_host(r) == (2, False)


def test_match_host_replay_mode(torch_cuda):
    """q_in chaining through maps16 (|D| > 32)."""
    torch = torch_cuda
    sfa = P.SFA(*CFG4)
    d = oracle_pair(*CFG4)
    t = W.cfg4_text(150 << 20)
    assert sfa.match_host(t) == d.run(t)
    rx = W.cfg3_regex()
    sfa3 = P.SFA(rx, None)
    d3 = oracle_pair(rx, None)
    t3 = W.cfg3_text(130 << 20, plant=True)
    assert sfa3.match_host(t3) == d3.run(t3)


# --------------------------------------------------------------------------- every TMA pipeline shape
@pytest.mark.parametrize("shape", ["1,16,0", "1,32,0", "2,16,0", "2,32,0", "1,64,0", "1,16,2", "2,16,2",
                                   "1,32,3", "1,32,0,256", "1,64,0,128", "2,32,0,0"])
def test_every_tma_shape(torch_cuda, shape):
    """k_scan_tma for each (K chunks/thread, bytes/row/stage, ring depth, L2
    promotion) the launcher can pick (sfa_set_tuning forces one), on texts
    spanning several rows per thread and ragged tails, and a batch."""
    torch = torch_cuda
    v = [int(x) for x in shape.split(",")]
    knobs = dict(tma_k=v[0], tma_rowb=v[1], tma_ring=v[2])
    if len(v) > 3:
        knobs["tma_promo"] = v[3]
    for rx, alpha, text in [(*CFG2, W.cfg2_accepted(2_000_000)), (*CFG1, W.cfg1_accepted(5_000_000)),
                            (*CFG4, W.cfg4_text(20_000_000))]:
        d = oracle_pair(rx, alpha)
        sfa = P.SFA(rx, alpha)
        sfa.set_tuning(**knobs)
        for n in (text.size, text.size - 1, 4_200_001, 9_999_937):
            t = text[:n]
            for pad in (0, 5):
                check_text(torch, sfa, d, t, pad)
        texts, off = W.ragged_batch(17, 300, 60_000, alpha)
        q, acc = _batch(torch, sfa, texts, off)
        qo, ao = d.run_batch(texts, off)
        assert (q == qo).all() and (acc == ao).all(), shape


# --------------------------------------------------------------------------- every composition mode
@pytest.mark.parametrize("rx,alpha,modes", [(*CFG1, (P.COMPOSE_VEC, P.COMPOSE_TABLE, P.COMPOSE_REPLAY)),
                                            (*CFG2, (P.COMPOSE_VEC, P.COMPOSE_TABLE, P.COMPOSE_REPLAY)),
                                            (*CFG4, (P.COMPOSE_TABLE, P.COMPOSE_REPLAY))])
def test_every_compose_mode(torch_cuda, rx, alpha, modes):
    """A3 by shuffled mapping vectors, by the composition table and by Lemma-1
    replay: the same exact result on the direct and TMA scans, the forced
    chunkings (per-chunk ids included) and batches."""
    torch = torch_cuda
    d = oracle_pair(rx, alpha)
    gen = {CFG1: W.cfg1_random, CFG2: lambda n: W.cfg2_accepted(n // 10), CFG4: W.cfg4_text}[(rx, alpha)]
    text = gen(6_000_011)
    for m in modes:
        sfa = P.SFA(rx, alpha)
        sfa.set_compose(m)
        for n in (text.size, 5_000_003, 70_001, 13):
            check_text(torch, sfa, d, text[:n], pad=3)
        _, v = dev(torch, text[:100_003])
        q, acc, ids = sfa.match_chunked(v, 777)
        assert (q, acc) == d.run(text[:100_003])
        o_ids, _, _ = O.OracleSFA(d).run_chunked(text[:100_003], spec_bounds(100_003, 777))
        assert ids.tolist() == o_ids.tolist(), m
        texts, off = W.ragged_batch(11, 40, 200_000, alpha)
        res = torch.zeros(80, dtype=torch.int32, device="cuda")
        sfa.match_batch(torch.from_numpy(texts).cuda(), torch.from_numpy(off.astype(np.int64)).cuda(), 40, res)
        torch.cuda.synchronize()
        got = res.cpu().numpy().view(np.uint32).reshape(40, 2)
        qo, ao = d.run_batch(texts, off)
        assert (got[:, 0] == qo).all() and (got[:, 1] == ao).all(), m


def test_tune_residency_keeps_results(torch_cuda):
    """The HOT ranking (static, profiled on a sample, auto-tuned) only moves
    rows between smem and L2: results stay the oracle's."""
    torch = torch_cuda
    rx = W.cfg3_regex()
    d = oracle_pair(rx, None)
    text = W.cfg3_text(9 << 20, plant=True)
    sfa = P.SFA(rx, None)
    sfa.set_residency(P.RES_HOT_L2)
    buf, v = dev(torch, text)
    for sample in (None, v[:1 << 20], v):
        sfa.tune_residency(sample)
        for n in (text.size, 4_194_319, 300_001):
            check_text(torch, sfa, d, text[:n], 1)
    rng = np.random.default_rng(12)
    junk = torch.from_numpy(rng.integers(0, 256, size=1 << 20, dtype=np.uint8)).cuda()
    sfa.tune_residency(junk)          # a misleading sample: slower, never wrong
    check_text(torch, sfa, d, text, 0)


def test_factored_step_contains_match_boundaries(torch_cuda):
    """FACTORED step (HOT residency): a word completed anywhere -- inside a
    chunk's first 32 bytes (SFA-table phase), just after it, across chunk
    boundaries, at the very end -- freezes the mapping into the accepting sink
    (the (family, absorbing g) entries of fact_tab)."""
    torch = torch_cuda
    rx = W.cfg3_regex()
    d = oracle_pair(rx, None)
    sfa = P.SFA(rx, None)
    base = W.cfg3_text(6 << 20, plant=False)
    assert d.run(base)[1] is False
    word = np.frombuffer(W.cfg3_words()[5], np.uint8)
    rng = np.random.default_rng(21)
    for off in [0, 3, 29, 31, 32, 33, 255, 4096, 7424 - 2, base.size - word.size] + rng.integers(0, base.size - 8, 12).tolist():
        t = base.copy()
        t[off:off + word.size] = word
        exp = d.run(t)
        assert exp[1] is True
        check_text(torch, sfa, d, t, 0)
    texts, offs = [], [0]
    for i in range(64):
        t = base[i * 65536:(i + 1) * 65536].copy()
        if i % 3 == 0:
            o = int(rng.integers(0, 65536 - 8))
            t[o:o + word.size] = word
        texts.append(t)
        offs.append(offs[-1] + t.size)
    cat = np.concatenate(texts)
    off = np.array(offs, np.uint64)
    res = torch.zeros(128, dtype=torch.int32, device="cuda")
    sfa.match_batch(torch.from_numpy(cat).cuda(), torch.from_numpy(off.astype(np.int64)).cuda(), 64, res)
    torch.cuda.synchronize()
    got = res.cpu().numpy().view(np.uint32).reshape(64, 2)
    qo, ao = d.run_batch(cat, off)
    assert (got[:, 0] == qo).all() and (got[:, 1] == ao).all()


@pytest.mark.parametrize("rx,alpha,compose", [(W.cfg3_regex(), None, None), (*CFG2, None), (*CFG4, None),
                                               (*CFG1, None), (*CFG1, P.COMPOSE_VEC), (*CFG2, P.COMPOSE_REPLAY)])
def test_batch_uniform(torch_cuda, rx, alpha, compose):
    """sfa_match_batch_uniform: equal texts through the TMA scan with a per-text
    segmented fold (or the offsets path for VEC / unaligned / odd lengths)."""
    torch = torch_cuda
    d = oracle_pair(rx, alpha)
    sfa = P.SFA(rx, alpha)
    if compose:
        sfa.set_compose(compose)
    al = np.frombuffer(alpha if alpha else b"abcdefghijklmnopqrstuvwxyz", np.uint8)
    rng = np.random.default_rng(31)
    for length, count, pad in [(65536, 300, 0), (4096, 5000, 0), (768, 20000, 0), (65536, 3, 0), (1000, 77, 0),
                               (4096, 64, 8)]:
        if rx == CFG2[0]:
            body = W.cfg2_accepted(length * count // 10 + 1)[:length * count]
            body = body.copy()
            flips = rng.integers(0, body.size, size=count // 3)
            body[flips] = np.uint8(ord("7"))
        elif rx == CFG1[0]:
            body = np.tile(W.cfg1_accepted(length // 2)[:length], count)[:length * count].copy()
        else:
            body = al[rng.integers(0, al.size, size=length * count)]
        if rx == W.cfg3_regex():
            word = np.frombuffer(W.cfg3_words()[7], np.uint8)
            for i in rng.choice(count, size=max(1, count // 10), replace=False):
                o = int(i) * length + int(rng.integers(0, length - word.size))
                body[o:o + word.size] = word
        buf = torch.empty(body.size + pad + 16, dtype=torch.uint8, device="cuda")
        v = buf[pad:pad + body.size]
        v.copy_(torch.from_numpy(body))
        res = torch.zeros(2 * count, dtype=torch.int32, device="cuda")
        sfa.match_batch_uniform(v, length, count, res)
        torch.cuda.synchronize()
        got = res.cpu().numpy().view(np.uint32).reshape(count, 2)
        off = np.arange(count + 1, dtype=np.uint64) * length
        qo, ao = d.run_batch(body, off)
        assert (got[:, 0] == qo).all() and (got[:, 1] == ao).all(), (length, count, pad)


def test_row_alignment_choices(torch_cuda):
    """Text sizes for which the TMA plan picks 256-, 128- and 64-byte row
    lengths (rows used vs DRAM cost, api.cpp), with ragged heads and tails,
    for the PRIVATE (cfg2) and HOT + FACTORED (cfg4) scans."""
    torch = torch_cuda
    rng = np.random.default_rng(21)
    for (rx, alpha), gen in ((CFG2, lambda n: W.cfg2_accepted(n // 10 + 1)), (CFG4, W.cfg4_text)):
        sfa = P.SFA(rx, alpha)
        d = oracle_pair(rx, alpha)
        big = gen(300 << 20)
        for n in (40_000_003, 97_000_000, 150 << 20, 268_435_450, 299_999_999):
            t = big[:n]
            if rng.random() < 0.5:
                t = t.copy()
                t[rng.integers(0, n)] ^= np.uint8(1)
            check_text(torch, sfa, d, t, int(rng.integers(0, 16)))
