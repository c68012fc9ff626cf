"""GPU parity, round 2: the timed kernels' interiors and the batch path.

* k_scan_tma's per-row SFA ids (sfa_match_rows) against the oracle's plain
  Alg. 5 on the same chunk bounds (Lemma 1 / Thm. 3,
  PAPER.md:434-479), on the PRIVATE path (cfg2; R = 32, 16 and 8 lane-group
  copies) and the HOT + FACTORED path (cfg3, cfg4), at >= 64 MiB: a final
  state alone cannot see an interior-chunk error when the DFA synchronises.
* sfa_match_batch (one segmented TMA scan over the texts back to back, with a
  device-side plan): boundaries at every position of a row, many texts per
  row, one text over many CTAs, empty texts everywhere, decreasing offsets
  (every result invalid), and no host synchronisation.
* random regexes at TMA sizes with out-of-window bytes.
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
AZ = b"abcdefghijklmnopqrstuvwxyz"


@pytest.fixture(scope="module")
def torch_cuda(cuda_ok):
    import torch
    return torch


_dfa, _sfa = {}, {}


def odfa(rx, alpha):
    if (rx, alpha) not in _dfa:
        _dfa[(rx, alpha)] = O.OracleDFA(rx, alpha)
    return _dfa[(rx, alpha)]


def osfa(rx, alpha):
    if (rx, alpha) not in _sfa:
        _sfa[(rx, alpha)] = O.OracleSFA(odfa(rx, alpha))
    return _sfa[(rx, alpha)]


def dev(torch, a, pad=0):
    buf = torch.empty(a.size + pad + 16, dtype=torch.uint8, device="cuda")
    v = buf[pad:pad + a.size]
    if a.size:
        v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return buf, v


def rows_vs_oracle(torch, sfa, rx, alpha, text, pad):
    buf, v = dev(torch, text, pad)
    ids = torch.zeros(148 * 2048, dtype=torch.int32, device="cuda")
    res = torch.zeros(2, dtype=torch.int32, device="cuda")
    plan = sfa.match_rows(v, ids, res)
    torch.cuda.synchronize()
    got = ids[:plan["rows"]].cpu().numpy().view(np.uint32)
    head, L, rows = plan["head"], plan["row_len"], plan["rows"]
    assert head < 256 and rows > 0 and plan["tail_start"] == head + rows * L <= text.size
    bounds = head + np.arange(rows + 1, dtype=np.uint64) * np.uint64(L)
    o_ids, _, _ = osfa(rx, alpha).run_chunked(text, bounds)
    bad = np.flatnonzero(got != o_ids)
    assert bad.size == 0, (bad[:10], got[bad[:10]], o_ids[bad[:10]], plan)
    q, acc = res.cpu().numpy().view(np.uint32)
    assert (int(q), bool(acc)) == odfa(rx, alpha).run(text)
    return plan


@pytest.mark.parametrize("copies", [0, 16, 8])
def test_rows_private_cfg2(torch_cuda, copies):
    """PRIVATE step, R = 32 (auto), 16 and 8 lane-group copies of the SFA table."""
    torch = torch_cuda
    sfa = P.SFA(*CFG2)
    if copies:   # AUTO would then pick HOT + FACTORED (more DFA copies than SFA copies)
        sfa.set_tuning(private_copies=copies)
        sfa.set_residency(P.RES_SMEM_PRIVATE)
    t = W.cfg2_rejected(text=W.cfg2_accepted((80 << 20) // 10))   # one flipped digit: a dead chunk in the middle
    plan = rows_vs_oracle(torch, sfa, *CFG2, t, 5)
    assert plan["ctas"] == 148                      # every SM scans (uneven split)
    assert P.sfa_info(sfa.h)["residency"] == P.RES_SMEM_PRIVATE


def test_rows_private_cfg4_r16(torch_cuda):
    """cfg4's 1024-state SFA in PRIVATE with R = 16 copies (AUTO picks HOT+FACTORED)."""
    torch = torch_cuda
    sfa = P.SFA(*CFG4)
    sfa.set_residency(P.RES_SMEM_PRIVATE)
    rows_vs_oracle(torch, sfa, *CFG4, W.cfg4_text(64 << 20), 3)


@pytest.mark.parametrize("which", ["cfg3", "cfg4", "cfg3-u8", "cfg3-lanes", "cfg3-hot8", "cfg3-hot2"])
def test_rows_hot_factored(torch_cuda, which):
    """HOT + FACTORED: rows switch to the DFA step after their first stages;
    their canonical ids come back through fact_tab.  DFA window layouts: AUTO
    (cfg3: MIXED -- hot states in 32 bank-private copies, every state in one
    shared copy; cfg4: 32 u16 copies), R = 16 lane-group copies ("lanes"), the
    u8 bank-private layout, and MIXED with only 8 / 2 hot states (most bytes
    run in the shared copy and move back to the private copies at every
    16-byte fix)."""
    torch = torch_cuda
    if which.startswith("cfg3"):
        rx, alpha = W.cfg3_regex(), None
        t = W.cfg3_text(64 << 20, plant=True)
        words = W.cfg3_words()
        rng = np.random.default_rng(5)
        for _ in range(200):                        # words everywhere: some rows end in the accepting sink
            w = np.frombuffer(words[int(rng.integers(0, 32))], np.uint8)
            o = int(rng.integers(0, t.size - w.size))
            t[o:o + w.size] = w
    else:
        rx, alpha = CFG4
        t = W.cfg4_text(64 << 20)
    sfa = P.SFA(rx, alpha)
    knobs = {"cfg3-u8": dict(dfa_u8=1), "cfg3-lanes": dict(dfa_layout=1), "cfg3-hot8": dict(dfa_layout=2, dfa_hot=8),
             "cfg3-hot2": dict(dfa_layout=2, dfa_hot=2)}.get(which)
    if knobs:
        sfa.set_tuning(**knobs)
    rows_vs_oracle(torch, sfa, rx, alpha, t, 0)
    info = P.sfa_info(sfa.h)
    assert info["residency"] == P.RES_HOT_L2
    hot = {"cfg3": None, "cfg4": 0, "cfg3-u8": 0, "cfg3-lanes": 0, "cfg3-hot8": 8, "cfg3-hot2": 2}[which]
    if hot is None:
        assert 0 < info["dfa_window_hot"] < info["dfa_states"]      # AUTO picks MIXED for cfg3
    else:
        assert info["dfa_window_hot"] == hot
    assert info["dfa_window_copies"] == (16 if which == "cfg3-lanes" else 32)
    if which != "cfg4":   # and a batch through the same layout
        texts, off = W.ragged_batch(19, 2000, 40_000, b"abcdefghijklmnopqrstuvwxyz")
        check_batch(torch, sfa, odfa(rx, alpha), texts, off)


# --------------------------------------------------------------------------- batches (segmented scan)
def batch(torch, sfa, texts, off, pad=0):
    count = off.size - 1
    bt, vt = dev(torch, texts, pad)
    do = torch.from_numpy(off.astype(np.int64)).cuda()
    res = torch.full((2 * count,), 7, dtype=torch.int32, device="cuda")
    sfa.match_batch(vt if texts.size else bt, do, count, res)
    torch.cuda.synchronize()
    r = res.cpu().numpy().view(np.uint32).reshape(count, 2)
    return r[:, 0], r[:, 1]


def check_batch(torch, sfa, d, texts, off, pad=0):
    q, acc = batch(torch, sfa, texts, off, pad)
    qo, ao = d.run_batch(texts, off)
    bad = np.flatnonzero((q != qo) | (acc != ao))
    assert bad.size == 0, (bad[:10], q[bad[:10]], qo[bad[:10]])


@pytest.mark.parametrize("rx,alpha", [CFG1, CFG2, CFG4, (W.cfg3_regex(), None)])
def test_batch_boundaries_everywhere(torch_cuda, rx, alpha):
    """Texts of 0..300 bytes (tens per TMA row, empty ones in runs), texts
    larger than a row, and one text spanning many CTAs, in one batch."""
    torch = torch_cuda
    d = odfa(rx, alpha)
    sfa = P.SFA(rx, alpha)
    al = np.frombuffer(alpha or AZ, np.uint8)
    rng = np.random.default_rng(77)
    for case in range(4):
        if case == 0:
            lens = rng.integers(0, 300, size=200_000)
            lens[rng.random(lens.size) < 0.2] = 0
        elif case == 1:
            lens = rng.integers(0, 30_000, size=3000)
        elif case == 2:
            lens = np.array([5, 0, 0, 40 << 20, 0, 17, 3 << 20, 1])
        else:
            lens = np.concatenate([rng.integers(1, 9, size=100_000), [25 << 20], rng.integers(0, 2, size=1000)])
        texts = al[rng.integers(0, al.size, size=int(lens.sum()))]
        if rx == CFG2[0]:
            texts = W.cfg2_accepted(texts.size // 10 + 1)[:texts.size].copy()
            texts[rng.integers(0, texts.size, size=texts.size // 100000 + 1)] = ord("7")
        if rx == CFG1[0]:
            texts = np.tile(W.cfg1_accepted(1 << 16), texts.size // (1 << 17) + 2)[:texts.size].copy()
        off = np.zeros(lens.size + 1, np.uint64)
        off[1:] = np.cumsum(lens)
        check_batch(torch, sfa, d, texts, off, int(rng.integers(0, 16)))


def test_batch_offsets_not_from_zero_and_gaps_in_buffer(torch_cuda):
    """Offsets start anywhere in the buffer (text i = texts[off[i]:off[i+1]])."""
    torch = torch_cuda
    rx = W.cfg3_regex()
    d = odfa(rx, None)
    sfa = P.SFA(rx, None)
    buf = W.cfg3_text(30 << 20, plant=False)
    word = np.frombuffer(W.cfg3_words()[3], np.uint8)
    rng = np.random.default_rng(9)
    for o in rng.integers(0, buf.size - 8, size=40):
        buf[o:o + 8] = word[:8] if word.size >= 8 else np.resize(word, 8)
    for start in (0, 1, 255, 12_345_677):
        lens = rng.integers(0, 70_000, size=300)
        off = np.concatenate([[start], start + np.cumsum(lens)]).astype(np.uint64)
        off = off[off <= buf.size]
        check_batch(torch, sfa, d, buf, off)




def test_batch_decreasing_offsets_invalidates_every_result(torch_cuda):
    """A decreasing offset pair (it used to overrun the task buffer):
    the device plan flags it, every result is {INVALID_STATE, 0}, nothing else
    is written, and the next good batch on the handle is exact again."""
    torch = torch_cuda
    sfa = P.SFA(*CFG2)
    d = odfa(*CFG2)
    texts = W.cfg2_accepted((64 << 20) // 10)
    for off in ([0, 64 << 20, 0, 64 << 20], [0, 10, 5, 20], [100, 50], [5, 6, 7, 3]):
        off = np.array(off, np.uint64)
        q, acc = batch(torch, sfa, texts, off)
        assert (q == P.INVALID_STATE).all() and (acc == 0).all(), off
    off = np.array([0, 10, 10, 64 << 20], np.uint64)
    check_batch(torch, sfa, d, texts, off)


def test_batch_async_does_not_synchronise(torch_cuda):
    """sfa_match_batch and sfa_match_async only enqueue: both return while a
    long kernel enqueued before them is still running."""
    torch = torch_cuda
    sfa = P.SFA(*CFG2)
    d = odfa(*CFG2)
    texts = W.cfg2_accepted(1 << 20)
    bt, vt = dev(torch, texts)
    off = torch.tensor([0, 1000, 5000, texts.size], dtype=torch.int64, device="cuda")
    res = torch.zeros(6, dtype=torch.int32, device="cuda")
    r1 = torch.zeros(2, dtype=torch.int32, device="cuda")
    empty = torch.empty(0, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    # first calls upload the tables and load the kernels (CUDA lazy loading): outside the check
    sfa.match(vt, s)
    sfa.match_batch(vt, off, 3, res, s)
    sfa.match_async(vt, r1, s)
    sfa.match_async(empty, r1, s)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        torch.cuda._sleep(2_000_000_000)             # ~1 s of GPU time
        done = torch.cuda.Event()
        sfa.match_batch(vt, off, 3, res, s)
        sfa.match_async(vt, r1, s)
        sfa.match_async(empty, r1, s)
        done.record(s)
    assert not done.query(), "a call synchronised with the stream"
    done.synchronize()
    got = res.cpu().numpy().view(np.uint32).reshape(3, 2)
    qo, ao = d.run_batch(texts, np.array([0, 1000, 5000, texts.size], np.uint64))
    assert (got[:, 0] == qo).all() and (got[:, 1] == ao).all()
    assert r1.cpu().tolist() == [0, int(d.run(np.zeros(0, np.uint8))[1])]


def test_cuda_graph_capture_and_replay(torch_cuda):
    """sfa_match_async and sfa_match_batch inside a CUDA graph (include/sfa.h:
    no host synchronisation, no allocation after a handle's first call): the
    graph is captured once and replayed on a changed text and on changed device
    offsets -- the batch plan is made on the device, so a replay follows them."""
    torch = torch_cuda
    sfa = P.SFA(*CFG2)
    d = odfa(*CFG2)
    text = W.cfg2_accepted(800_000)                       # 8 MB: the TMA scan
    host = text.copy()
    bt, vt = dev(torch, host)
    offs = [np.array([0, 10, 4_000_000, 4_000_000, host.size], np.uint64),
            np.array([0, 1_000_000, 1_000_020, 7_999_990, host.size], np.uint64)]
    off = torch.from_numpy(offs[0].astype(np.int64)).cuda()
    res = torch.zeros(8, dtype=torch.int32, device="cuda")
    r1 = torch.zeros(2, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    sfa.match_async(vt, r1, s)                            # first calls: tables, scratch, kernel loading
    sfa.match_batch(vt, off, 4, res, s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sfa.match_async(vt, r1, s)
        sfa.match_batch(vt, off, 4, res, s)
    r1.zero_()
    res.zero_()
    for trial in range(3):
        if trial:                                         # change the text and the offsets in place
            pos = 123_457 * trial
            host[pos] = 48 + (int(host[pos]) - 48 + 5) % 10
            vt.copy_(torch.from_numpy(host))
            off.copy_(torch.from_numpy(offs[trial % 2].astype(np.int64)))
        g.replay()
        torch.cuda.synchronize()
        assert tuple(r1.cpu().tolist()) == tuple(int(x) for x in d.run(host)), trial
        got = res.cpu().numpy().view(np.uint32).reshape(4, 2)
        qo, ao = d.run_batch(host, offs[trial % 2] if trial else offs[0])
        assert (got[:, 0] == qo).all() and (got[:, 1] == ao).all(), (trial, got, qo, ao)


@pytest.mark.parametrize("length,count,pad", [(65536, 300, 0), (1000, 777, 3), (1, 100_000, 0), (7, 50_000, 1),
                                              (4 << 20, 5, 0), (65537, 513, 9)])
def test_batch_uniform_any_length(torch_cuda, length, count, pad):
    torch = torch_cuda
    rx = W.cfg3_regex()
    d = odfa(rx, None)
    sfa = P.SFA(rx, None)
    rng = np.random.default_rng(length)
    al = np.frombuffer(AZ, np.uint8)
    body = al[rng.integers(0, 26, size=length * count)]
    word = np.frombuffer(W.cfg3_words()[1], np.uint8)
    if length >= word.size:
        for i in rng.choice(count, size=max(1, count // 10), replace=False):
            o = int(i) * length + int(rng.integers(0, length - word.size + 1))
            body[o:o + word.size] = word
    bt, v = dev(torch, body, pad)
    res = torch.zeros(2 * count, dtype=torch.int32, device="cuda")
    sfa.match_batch_uniform(v, length, count, res)
    torch.cuda.synchronize()
    got = res.cpu().numpy().view(np.uint32).reshape(count, 2)
    qo, ao = d.run_batch(body, np.arange(count + 1, dtype=np.uint64) * length)
    assert (got[:, 0] == qo).all() and (got[:, 1] == ao).all()


# --------------------------------------------------------------------------- random regexes at TMA sizes
def test_random_regexes_tma_sizes(torch_cuda):
    torch = torch_cuda
    from test_oracle import _random_regex
    rng = np.random.default_rng(2024)
    for i in range(12):
        rx = _random_regex(rng, 6)
        alpha = b"abcd" if i % 2 else None
        try:
            sfa = P.SFA(rx, alpha)
        except P.SFAError:
            continue
        d = O.OracleDFA(rx, alpha)
        n = int(rng.integers(5 << 20, 9 << 20))
        t = np.frombuffer(b"abcde", np.uint8)[rng.integers(0, 5, size=n)]
        t[rng.integers(0, n, size=3)] = rng.integers(0, 256, size=3).astype(np.uint8)   # out-of-window bytes
        buf, v = dev(torch, t, int(rng.integers(0, 16)))
        assert sfa.match(v) == d.run(t), rx
        lens = rng.integers(0, 200_000, size=50)
        off = np.zeros(51, np.uint64)
        off[1:] = np.minimum(np.cumsum(lens), n)
        check_batch(torch, sfa, d, t, off)


def test_batch_host_end_to_end(torch_cuda):
    """sfa_match_batch_host: host texts in slices of whole texts (one text longer
    than a 64 MiB slice included), pinned and pageable, == Alg. 2 per text;
    decreasing host offsets are refused with INVALID_ARG."""
    torch = torch_cuda
    rx = W.cfg3_regex()
    d = odfa(rx, None)
    sfa = P.SFA(rx, None)
    rng = np.random.default_rng(41)
    lens = np.concatenate([rng.integers(0, 100_000, size=3000), [70 << 20], rng.integers(0, 50, size=5000)])
    off = np.zeros(lens.size + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    texts = W.cfg3_text(int(off[-1]), plant=True)
    word = np.frombuffer(W.cfg3_words()[9], np.uint8)
    for o in rng.integers(0, texts.size - 8, size=500):
        texts[o:o + word.size] = word
    qo, ao = d.run_batch(texts, off)
    q, a = sfa.match_batch_host(texts, off)
    assert (q == qo).all() and (a == ao).all()
    ht = torch.from_numpy(texts).pin_memory()
    ho = torch.from_numpy(off.view(np.int64)).pin_memory()
    q, a = sfa.match_batch_host(ht, ho)
    assert (q == qo).all() and (a == ao).all()
    bad = off.copy()
    bad[5], bad[6] = bad[6], bad[5]
    with pytest.raises(P.SFAError) as e:
        sfa.match_batch_host(texts, bad)
    assert e.value.code == P.SFA_ERR_INVALID_ARG


def _guarded(torch, n_i32, fill=0x5A5A5A5A):
    """A device int32 buffer of n_i32 entries inside 4 KiB guard regions."""
    g = 1024
    buf = torch.full((n_i32 + 2 * g,), fill - (1 << 32) if fill >= (1 << 31) else fill, dtype=torch.int32,
                     device="cuda")
    return buf, buf[g:g + n_i32], g


def test_guard_bytes_and_determinism(torch_cuda):
    """compute-sanitizer is closed on this GPU pool, so: every output buffer
    (results, per-row ids, maps) sits between guard regions that must stay
    untouched, and every kernel is run 12 times with different shapes (ring
    depth, K, stage width) and back-to-back launches; the outputs must be
    identical every time and equal to the oracle (results must not depend on
    scheduling)."""
    torch = torch_cuda
    n = (4 << 20) + 4097
    for rx, alpha, text in [(*CFG2, W.cfg2_accepted(n // 10 + 1)[:n]), (W.cfg3_regex(), None, W.cfg3_text(n, plant=True))]:
        d = odfa(rx, alpha)
        texts, off = W.ragged_batch(3, 300, 30_000, alpha or AZ)
        qo, ao = d.run_batch(texts, off)
        dt = torch.from_numpy(text).cuda()
        dtx = torch.from_numpy(texts).cuda()
        do = torch.from_numpy(off.astype(np.int64)).cuda()
        first = None
        for i, knobs in enumerate([{}, dict(tma_k=1, tma_rowb=16, tma_ring=2), dict(tma_k=1, tma_rowb=32, tma_ring=3),
                                   dict(tma_k=2, tma_rowb=16), dict(tma_k=1, tma_rowb=64)] * 2 + [{}, {}]):
            sfa = P.SFA(rx, alpha)
            try:
                sfa.set_tuning(**knobs)
                buf, res, g = _guarded(torch, 600)
                rbuf, r1, _ = _guarded(torch, 2)
                ibuf, ids, _ = _guarded(torch, 148 * 2048)
                for _ in range(3):   # back to back on one stream
                    sfa.match_batch(dtx, do, 300, res)
                    sfa.match_async(dt, r1)
                plan = sfa.match_rows(dt, ids, r1)
                torch.cuda.synchronize()
            except P.SFAError as e:     # a forced shape that does not fit this automaton
                assert e.code == P.SFA_ERR_CAPACITY, knobs
                continue
            finally:
                sfa.close()
            for b in (buf, rbuf, ibuf):
                gv = b.cpu().numpy().view(np.uint32)
                assert (gv[:g] == 0x5A5A5A5A).all() and (gv[-g:] == 0x5A5A5A5A).all(), ("guard overwritten", knobs)
            got = res.cpu().numpy().view(np.uint32).reshape(300, 2)
            assert (got[:, 0] == qo).all() and (got[:, 1] == ao).all(), knobs
            assert tuple(r1.cpu().numpy().view(np.uint32)) == (d.run(text)[0], int(d.run(text)[1])), knobs
            rows = ids[:plan["rows"]].cpu().numpy().view(np.uint32).copy()
            if not knobs:
                if first is None:
                    first = rows
                assert (rows == first).all()          # same plan, same ids, every time


# --------------------------------------------------------------------------- factored folds (round 2b)
@pytest.mark.parametrize("fold", [0, 1, 2])
def test_factored_fold_modes(torch_cuda, fold):
    """FACTORED chunk values through the folds: (F, g) pairs composed from the
    families' marked sets in smem (0), the same sets read from global memory
    (1), or canonical SFA ids as before (2) -- same results on cfg3 texts with
    words planted everywhere (single texts and a ragged batch) and cfg4."""
    torch = torch_cuda
    rx = W.cfg3_regex()
    t = W.cfg3_text(48 << 20, plant=False)
    words = W.cfg3_words()
    rng = np.random.default_rng(31 + fold)
    sfa = P.SFA(rx, None)
    sfa.set_tuning(fact_fold=fold)
    d = odfa(rx, None)
    for trial in range(4):
        u = t.copy()
        for _ in range(trial * 3):
            w = np.frombuffer(words[int(rng.integers(0, 32))], np.uint8)
            o = int(rng.integers(0, u.size - w.size))
            u[o:o + w.size] = w
        n = int(rng.integers(5 << 20, u.size))
        buf, v = dev(torch, u[:n], trial)
        assert sfa.match(v) == d.run(u[:n]), (fold, trial)
    assert P.sfa_info(sfa.h)["dfa_window_hot"] > 0                  # MIXED window, factored rows
    texts, off = W.ragged_batch(23, 3000, 50_000, AZ)
    check_batch(torch, sfa, d, texts, off)
    sfa4 = P.SFA(*CFG4)
    sfa4.set_tuning(fact_fold=fold)
    t4 = W.cfg4_text(24 << 20)
    buf, v = dev(torch, t4, 0)
    assert sfa4.match(v) == odfa(*CFG4).run(t4)


def test_factored_two_absorbing_states(torch_cuda):
    """x.*|[ab]* over all bytes: two absorbing states (the accepting sink after
    a leading x, the dead state after any other byte), so a family's marked
    states go to different absorbing images (DevTables::fam_img).  HOT +
    FACTORED forced; texts accepted by either branch, rejected by one byte
    planted anywhere, single and batched."""
    torch = torch_cuda
    rx = "x.*|[ab]*"
    d = odfa(rx, None)
    sfa = P.SFA(rx, None)
    sfa.set_residency(P.RES_HOT_L2)
    rng = np.random.default_rng(77)
    base = rng.integers(0, 2, size=12 << 20).astype(np.uint8) + ord("a")
    cases = []
    cases.append(base.copy())                                    # [ab]*: accepted
    u = base.copy(); u[int(rng.integers(0, u.size))] = ord("c"); cases.append(u)   # one c: dead
    u = base.copy(); u[0] = ord("x"); cases.append(u)            # x...: the accepting sink
    u = base.copy(); u[0] = ord("x"); u[-5] = 0; cases.append(u)  # x... then anything: still accepted
    u = base.copy(); u[7 << 20] = ord("x"); cases.append(u)      # an x later: dead
    for i, u in enumerate(cases):
        for n in (u.size, u.size - 12_345):
            buf, v = dev(torch, u[:n], i % 16)
            assert sfa.match(v) == d.run(u[:n]), (i, n)
    info = P.sfa_info(sfa.h)
    assert info["residency"] == P.RES_HOT_L2 and info["dfa_window_copies"] > 0   # the FACTORED step ran
    texts = np.concatenate([c[: 40_000 + 997 * i] for i, c in enumerate(cases * 6)])
    lens = [40_000 + 997 * i for i in range(len(cases) * 6)]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    check_batch(torch, sfa, d, texts, off)
