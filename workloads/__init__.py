"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is shared by the oracle side and the CUDA side of every test and
of bench.py.  It holds none of the method's arithmetic: no automaton, no
transition table, no SFA.  It only draws bytes (numpy PCG64, DESIGN.md reading
C15) and, for configs 3 and 5, removes accidental occurrences of the word set
by plain substring search (reading C13).

Recipes (BASELINE.json ``configs``):

=====  =======================  ========  ==========================================
cfg    regex                    Sigma     text
=====  =======================  ========  ==========================================
1a     ``(ab|ba)*c``            abc       2^20 bytes i.i.d. U{a,b,c}, seed 0
1b     ``(ab|ba)*c``            abc       524,287 seeded picks of "ab"/"ba", then "c"
2a     ``([0-4]{5}[5-9]{5})*``  digits    26,843,545 blocks: 5 x U('0'..'4'), 5 x U('5'..'9')
2b     same                     digits    2a with one seeded digit moved to the other half
3a/3b  ``.*(w1|...|w32).*``     all 256   2^30 bytes U{a..z}, scrubbed; 3b plants one word
4      ``.*a[ab]{8}``           ab        2^30 bytes i.i.d. U{a,b}
5      cfg 3's regex            all 256   65,536 texts x 65,536 B, scrubbed; 6,554 planted
=====  =======================  ========  ==========================================

Every function takes the size as an argument so tests can draw scaled-down
texts with the same recipe; the defaults are the BASELINE.json sizes.
"""
from __future__ import annotations

import functools

import numpy as np

LOWER = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz", np.uint8)

REGEX = {1: "(ab|ba)*c", 2: "([0-4]{5}[5-9]{5})*", 4: ".*a[ab]{8}"}
ALPHABET = {1: b"abc", 2: b"0123456789", 3: None, 4: b"ab", 5: None}

CFG1_BYTES = 1 << 20
CFG1_PAIRS = 524_287            # 2 * 524,287 + 1 = 2^20 - 1 bytes (reading C11)
CFG2_BLOCKS = 26_843_545        # 268,435,450 bytes (reading C12)
CFG3_BYTES = 1 << 30
CFG4_BYTES = 1 << 30
CFG5_COUNT = 65_536
CFG5_LEN = 65_536
CFG5_PLANTED = 6_554            # a seeded 10% of 65,536 texts


def _streams(cfg: int):
    """cfg k: SeedSequence(k) spawned into words / text / plant / selection."""
    return [np.random.default_rng(s) for s in np.random.SeedSequence(cfg).spawn(4)]


# --------------------------------------------------------------------------- cfg 1
def cfg1_random(n: int = CFG1_BYTES) -> np.ndarray:
    rng = np.random.default_rng(0)
    return rng.integers(97, 100, size=n, dtype=np.uint8)


def cfg1_accepted(pairs: int = CFG1_PAIRS) -> np.ndarray:
    rng = _streams(1)[1]
    pick = rng.integers(0, 2, size=pairs, dtype=np.uint8)       # 0 -> "ab", 1 -> "ba"
    t = np.empty(2 * pairs + 1, np.uint8)
    t[0:2 * pairs:2] = np.where(pick == 0, 97, 98)
    t[1:2 * pairs:2] = np.where(pick == 0, 98, 97)
    t[-1] = 99
    return t


# --------------------------------------------------------------------------- cfg 2
def cfg2_accepted(blocks: int = CFG2_BLOCKS) -> np.ndarray:
    rng = _streams(2)[1]
    t = np.empty((blocks, 10), np.uint8)
    t[:, :5] = rng.integers(48, 53, size=(blocks, 5), dtype=np.uint8)
    t[:, 5:] = rng.integers(53, 58, size=(blocks, 5), dtype=np.uint8)
    return t.reshape(-1)


def cfg2_flip_position(n: int) -> int:
    return int(_streams(2)[2].integers(0, n))


def cfg2_rejected(blocks: int = CFG2_BLOCKS, text: np.ndarray | None = None) -> np.ndarray:
    """2a with one seeded position replaced by a digit from the wrong half."""
    t = cfg2_accepted(blocks).copy() if text is None else text.copy()
    p = cfg2_flip_position(t.size)
    rng = _streams(2)[3]
    if t[p] < 53:
        t[p] = rng.integers(53, 58, dtype=np.uint8)
    else:
        t[p] = rng.integers(48, 53, dtype=np.uint8)
    return t


# --------------------------------------------------------------------------- cfg 3 / 5
@functools.lru_cache(maxsize=None)
def cfg3_words(count: int = 32, seed_cfg: int = 3) -> tuple:
    """32 distinct seeded words, lengths uniform in {4..8}, letters U{a..z} (C14)."""
    rng = _streams(seed_cfg)[0]
    out, seen = [], set()
    while len(out) < count:
        ln = int(rng.integers(4, 9))
        w = bytes(LOWER[rng.integers(0, 26, size=ln)].tolist())
        if w not in seen:
            seen.add(w)
            out.append(w)
    return tuple(out)


def cfg3_regex(words=None) -> str:
    words = cfg3_words() if words is None else words
    return ".*(" + "|".join(w.decode() for w in words) + ").*"


def _prefix_key(w: bytes) -> int:
    return w[0] | (w[1] << 8) | (w[2] << 16) | (w[3] << 24)


def find_occurrences(t: np.ndarray, words, lo: int = 0, hi: int | None = None) -> list:
    """All (pos, word_index) with t[pos:pos+len(w)] == w, pos in [lo, hi).

    Plain substring search: a hashed filter on the 4-byte prefix over four
    uint32 views of the buffer, then an exact comparison.  Words have length
    >= 4."""
    n = t.size
    hi = n if hi is None else min(hi, n)
    if hi - lo < 4:
        return []
    keys = np.array([_prefix_key(w) for w in words], np.uint32)
    mult = np.uint32(0x9E3779B1)
    tbl = np.zeros(1 << 16, bool)
    tbl[(keys * mult) >> np.uint32(16)] = True
    found = []
    block = 1 << 26
    for b0 in range(lo, hi, block):
        b1 = min(hi, b0 + block)
        seg = t[b0:min(n, b1 + 3)]
        for k in range(4):
            m = (seg.size - k) // 4
            if m <= 0:
                continue
            v = np.frombuffer(seg[k:k + 4 * m].tobytes(), dtype="<u4")
            cand = np.nonzero(tbl[(v * mult) >> np.uint32(16)])[0]
            if cand.size == 0:
                continue
            cand = cand[np.isin(v[cand], keys)]
            for j in cand.tolist():
                p = b0 + k + 4 * j
                if p >= b1:
                    continue
                key = int(v[j])
                for wi, w in enumerate(words):
                    if _prefix_key(w) == key and p + len(w) <= n and t[p:p + len(w)].tobytes() == w:
                        found.append((p, wi))
    found.sort()
    return found


def scrub(t: np.ndarray, words) -> int:
    """Remove every occurrence of every word (in place): the last letter of
    an occurrence is replaced by the next letter (cyclic a..z); windows around
    changed bytes are searched again until none is left.  Returns the number
    of bytes changed.  The text stays near-uniform (C13)."""
    changed = 0
    occ = find_occurrences(t, words)
    rounds = 0
    while occ:
        rounds += 1
        if rounds > 64:
            raise RuntimeError("scrub did not converge")
        touched = []
        for p, wi in occ:
            w = words[wi]
            q = p + len(w) - 1
            if t[p:p + len(w)].tobytes() != w:      # already broken by an earlier edit
                continue
            t[q] = 97 + (int(t[q]) - 97 + 1) % 26
            changed += 1
            touched.append(q)
        occ = []
        for q in sorted(set(touched)):
            occ.extend(find_occurrences(t, words, max(0, q - 8), q + 1))
        occ = sorted(set(occ))
    return changed


def letters(rng, n: int) -> np.ndarray:
    return LOWER[rng.integers(0, 26, size=n, dtype=np.uint8)]


def cfg3_text(n: int = CFG3_BYTES, plant: bool = False, words=None) -> np.ndarray:
    """3a (plant=False): scrubbed U{a..z}; 3b: one seeded word at a seeded offset."""
    words = cfg3_words() if words is None else words
    s = _streams(3)
    t = letters(s[1], n)
    scrub(t, words)
    if plant:
        w = words[int(s[3].integers(0, len(words)))]
        off = int(s[2].integers(0, n - len(w) + 1))
        t[off:off + len(w)] = np.frombuffer(w, np.uint8)
    return t


def cfg4_text(n: int = CFG4_BYTES) -> np.ndarray:
    return _streams(4)[1].integers(97, 99, size=n, dtype=np.uint8)


def cfg5_batch(count: int = CFG5_COUNT, length: int = CFG5_LEN, planted: int | None = None, words=None):
    """(texts, offsets, planted_indices): `count` scrubbed texts of `length`
    bytes back to back; a seeded `planted` of them get one word each."""
    words = cfg3_words() if words is None else words
    if planted is None:
        planted = round(count * CFG5_PLANTED / CFG5_COUNT)
    s = _streams(5)
    t = letters(s[1], count * length)
    scrub(t, words)
    idx = np.sort(s[3].choice(count, size=planted, replace=False))
    for i in idx.tolist():
        w = words[int(s[3].integers(0, len(words)))]
        off = i * length + int(s[2].integers(0, length - len(w) + 1))
        t[off:off + len(w)] = np.frombuffer(w, np.uint8)
    offsets = np.arange(count + 1, dtype=np.uint64) * np.uint64(length)
    return t, offsets, idx


def ragged_batch(seed: int, count: int, max_len: int, alphabet: bytes) -> tuple:
    """Texts of seeded lengths in [0, max_len] (empty included) over `alphabet`."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, max_len + 1, size=count)
    if count > 2:
        lens[0] = 0
        lens[1] = max_len
    al = np.frombuffer(alphabet, np.uint8)
    t = al[rng.integers(0, al.size, size=int(lens.sum()))]
    off = np.zeros(count + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    return t, off


# --------------------------------------------------------------------------- r_n family
# r_n = ([0-4]{n}[5-9]{n})*, "1GB string accepted
# by those automata"; r_a = r_n|a* on a repetition of "a".
# Streams: SeedSequence(1000 + n), so every n has its own text.
RN_BYTES = 1 << 30


def rn_regex(n: int) -> str:
    return f"([0-4]{{{n}}}[5-9]{{{n}}})*"


def rn_accepted(n: int, nbytes: int = RN_BYTES) -> np.ndarray:
    """Back-to-back blocks of n digits U('0'..'4') then n digits U('5'..'9'),
    as many whole blocks as fit in nbytes (so the text is accepted)."""
    blocks = max(1, nbytes // (2 * n))
    rng = np.random.default_rng(np.random.SeedSequence(1000 + n))
    t = np.empty((blocks, 2 * n), np.uint8)
    t[:, :n] = rng.integers(48, 53, size=(blocks, n), dtype=np.uint8)
    t[:, n:] = rng.integers(53, 58, size=(blocks, n), dtype=np.uint8)
    return t.reshape(-1)


def ra_regex(n: int) -> str:
    return f"{rn_regex(n)}|a*"


def ra_text(nbytes: int = RN_BYTES) -> np.ndarray:
    return np.full(nbytes, 97, np.uint8)


# --------------------------------------------------------------------------- Ex. 3
# [ap]*[al][alp]{n-2} over {a, l, p}; the minimal DFA has 2^n
# states.  Text: i.i.d. uniform over {a, l, p}, SeedSequence(3000 + n).
def ex3_regex(n: int) -> str:
    return "[ap]*[al][alp]{%d}" % (n - 2)


def ex3_text(n: int, nbytes: int) -> np.ndarray:
    rng = np.random.default_rng(np.random.SeedSequence(3000 + n))
    return np.frombuffer(b"alp", np.uint8)[rng.integers(0, 3, size=nbytes)]
