"""CPU oracle for the SFA matcher -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import this package.  The
product package ``paper_1405_0562_b200`` never imports it, and this package
imports nothing from the product: the two share no code.

It wraps ``oracle/oracle.c`` (plain C, see its header for the PAPER.md
passages it follows) through ctypes:

* ``OracleDFA(regex, alphabet)`` -- regex -> Thompson NFA -> Alg. 1 subset
  construction -> Moore minimisation -> canonical numbering
  (reading C3).
* ``.run(text)`` -- Alg. 2: ``(q_final, accept)``.
* ``brute(regex, alphabet, s)`` -- the regex's meaning evaluated directly on
  the AST (position sets), the independent pin for the automata.
* ``.run_spec(text, bounds)`` -- Alg. 3, the speculative
  DFA baseline, per-chunk mappings and the sequential reduction.
* ``OracleSFA(dfa)`` -- Alg. 4, for SFA-level pins, and
  ``.run_chunked`` -- Alg. 5 with both reductions.
* ``OracleNFA(regex, alphabet)`` / ``OracleNFA.explicit(...)`` -- the
  eps-free view of the Thompson NFA, or an explicit NFA (the paper's Ex. 3);
  ``.run`` is the NFA run by definition.
* ``OracleNSFA(nfa)`` -- Alg. 4 in its general form (set-valued mappings, the
  N-SFA) and Alg. 5 over it, the parallel reduction by
  logical matrix products.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_SO = os.path.join(_HERE, "liboracle.so")

E_NAMES = {1: "syntax", 2: "unsupported", 3: "capacity", 4: "invalid argument"}


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{E_NAMES.get(code, code)}: {msg}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C11, -O2)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        u8p = C.POINTER(C.c_uint8)
        u32p = C.POINTER(C.c_uint32)
        u64p = C.POINTER(C.c_uint64)
        vp = C.c_void_p
        L.oracle_compile.argtypes = [C.c_char_p, u8p, C.c_int, C.POINTER(vp), C.c_char_p, C.c_int]
        L.oracle_compile.restype = C.c_int
        L.oracle_free.argtypes = [vp]
        for f in ("oracle_nfa_states", "oracle_subset_states", "oracle_dfa_states"):
            getattr(L, f).argtypes = [vp]
            getattr(L, f).restype = C.c_uint32
        L.oracle_dfa_dead.argtypes = [vp]
        L.oracle_dfa_dead.restype = C.c_int32
        L.oracle_dfa_export.argtypes = [vp, u32p, u8p]
        L.oracle_run.argtypes = [vp, u8p, C.c_uint64, u32p]
        L.oracle_run.restype = C.c_int
        L.oracle_run_batch.argtypes = [vp, u8p, u64p, C.c_uint64, u32p, u8p]
        L.oracle_run_spec.argtypes = [vp, u8p, u64p, C.c_uint64, u32p, u32p]
        L.oracle_run_spec.restype = C.c_int
        L.oracle_brute.argtypes = [C.c_char_p, u8p, C.c_int, u8p, C.c_int]
        L.oracle_brute.restype = C.c_int
        L.oracle_brute_all.argtypes = [C.c_char_p, u8p, C.c_int, u8p, C.c_int, C.c_int, u8p]
        L.oracle_brute_all.restype = C.c_int64
        L.oracle_sfa_build.argtypes = [vp, C.c_uint32, C.POINTER(vp)]
        L.oracle_sfa_build.restype = C.c_int
        L.oracle_sfa_free.argtypes = [vp]
        L.oracle_sfa_states.argtypes = [vp]
        L.oracle_sfa_states.restype = C.c_uint32
        L.oracle_sfa_export.argtypes = [vp, u32p, u32p, u8p]
        L.oracle_sfa_run_chunked.argtypes = [vp, u8p, u64p, C.c_int, u32p, u32p, u32p]
        L.oracle_sfa_run_chunked.restype = C.c_int
        L.oracle_nfa_compile.argtypes = [C.c_char_p, u8p, C.c_int, C.POINTER(vp), C.c_char_p, C.c_int]
        L.oracle_nfa_compile.restype = C.c_int
        L.oracle_nfa_explicit.argtypes = [C.c_int, u64p, C.c_uint64, C.c_uint64, u8p, C.c_int, C.POINTER(vp)]
        L.oracle_nfa_explicit.restype = C.c_int
        L.oracle_nfa_free.argtypes = [vp]
        L.oracle_nfa_size.argtypes = [vp]
        L.oracle_nfa_size.restype = C.c_uint32
        L.oracle_nfa_run.argtypes = [vp, u8p, C.c_uint64, u64p]
        L.oracle_nfa_run.restype = C.c_int
        L.oracle_nfa_word_map.argtypes = [vp, u8p, C.c_int, u64p]
        L.oracle_nsfa_build.argtypes = [vp, C.c_uint32, C.POINTER(vp)]
        L.oracle_nsfa_build.restype = C.c_int
        L.oracle_nsfa_free.argtypes = [vp]
        L.oracle_nsfa_states.argtypes = [vp]
        L.oracle_nsfa_states.restype = C.c_uint32
        L.oracle_nsfa_run_chunked.argtypes = [vp, u8p, u64p, C.c_int, u32p, u64p, u64p]
        L.oracle_nsfa_run_chunked.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def _sigma(alphabet):
    """alphabet: None (all 256 bytes) or bytes/str listing Sigma."""
    if alphabet is None:
        return None, -1
    if isinstance(alphabet, str):
        alphabet = alphabet.encode("latin-1")
    a = np.frombuffer(bytes(alphabet), dtype=np.uint8).copy()
    if a.size == 0:
        a = np.zeros(1, np.uint8)
        return a, 0
    return a, int(a.size)


def _text(t) -> np.ndarray:
    if isinstance(t, str):
        t = t.encode("latin-1")
    if isinstance(t, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(t), dtype=np.uint8)
    a = np.ascontiguousarray(t, dtype=np.uint8)
    return a


class OracleDFA:
    """Canonical minimal complete DFA of (regex, Sigma) -- DESIGN.md C2/C3."""

    def __init__(self, regex: str, alphabet=None):
        L = lib()
        self._sig, slen = _sigma(alphabet)
        h = C.c_void_p()
        err = C.create_string_buffer(256)
        rc = L.oracle_compile(regex.encode("latin-1"), None if self._sig is None else _ptr(self._sig, C.c_uint8),
                              slen, C.byref(h), err, 256)
        if rc != 0:
            raise OracleError(rc, err.value.decode())
        self._h = h
        self.regex = regex
        self.alphabet = alphabet
        self.n = L.oracle_dfa_states(h)
        self.dead = L.oracle_dfa_dead(h)
        self.nfa_states = L.oracle_nfa_states(h)
        self.subset_states = L.oracle_subset_states(h)
        self.table = np.zeros((self.n, 256), np.uint32)
        self.finals = np.zeros(self.n, np.uint8)
        L.oracle_dfa_export(h, _ptr(self.table, C.c_uint32), _ptr(self.finals, C.c_uint8))

    @property
    def live(self) -> int:
        """|D| without the dead state (the paper's r_n / Ex. 4 convention, C4)."""
        return self.n - (1 if self.dead >= 0 else 0)

    def run(self, text):
        """Alg. 2: returns (q_final, accept)."""
        a = _text(text)
        q = C.c_uint32()
        acc = lib().oracle_run(self._h, _ptr(a, C.c_uint8) if a.size else None, a.size, C.byref(q))
        return int(q.value), bool(acc)

    def run_spec(self, text, bounds):
        """Alg. 3 over chunks [bounds[i], bounds[i+1]):
        returns (q_final, accept, T) with T[i, q] = delta^(q, chunk i)."""
        a = _text(text)
        b = np.ascontiguousarray(bounds, np.uint64)
        p = b.size - 1
        maps = np.zeros((max(p, 1), self.n), np.uint32)
        q = C.c_uint32()
        acc = lib().oracle_run_spec(self._h, _ptr(a, C.c_uint8) if a.size else None, _ptr(b, C.c_uint64), p,
                                    _ptr(maps, C.c_uint32), C.byref(q))
        if acc < 0:
            raise MemoryError("oracle_run_spec")
        return int(q.value), bool(acc), maps[:p]

    def run_batch(self, texts: np.ndarray, offsets: np.ndarray):
        texts = np.ascontiguousarray(texts, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        count = offsets.size - 1
        q = np.zeros(count, np.uint32)
        acc = np.zeros(count, np.uint8)
        lib().oracle_run_batch(self._h, _ptr(texts, C.c_uint8), _ptr(offsets, C.c_uint64), count,
                               _ptr(q, C.c_uint32), _ptr(acc, C.c_uint8))
        return q, acc

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.oracle_free(h)
            self._h = None


def brute(regex: str, alphabet, s) -> bool:
    """The regex's language membership, evaluated on the AST (len(s) <= 62)."""
    sig, slen = _sigma(alphabet)
    a = _text(s)
    r = lib().oracle_brute(regex.encode("latin-1"), None if sig is None else _ptr(sig, C.c_uint8), slen,
                           _ptr(a, C.c_uint8) if a.size else None, int(a.size))
    if r < 0:
        raise OracleError(-r, "brute-force parse failed")
    return bool(r)


def all_strings(chars: bytes, maxlen: int):
    """(texts, offsets) of every string over `chars` of length 0..maxlen in
    shortlex order -- the enumeration order of oracle_brute_all."""
    al = np.frombuffer(chars, np.uint8)
    k = al.size
    parts, lens = [], []
    for ln in range(maxlen + 1):
        cnt = k ** ln
        if ln == 0:
            lens.append(np.zeros(1, np.int64))
            continue
        idx = np.arange(cnt)
        digits = np.empty((cnt, ln), np.uint8)
        for pos in range(ln - 1, -1, -1):
            digits[:, pos] = al[idx % k]
            idx //= k
        parts.append(digits.reshape(-1))
        lens.append(np.full(cnt, ln, np.int64))
    lens = np.concatenate(lens)
    off = np.zeros(lens.size + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    texts = np.concatenate(parts) if parts else np.zeros(0, np.uint8)
    return texts, off


def brute_all(regex: str, alphabet, chars: bytes, maxlen: int) -> np.ndarray:
    """brute() on every string of all_strings(chars, maxlen)."""
    sig, slen = _sigma(alphabet)
    ch = np.frombuffer(chars, np.uint8).copy()
    total = sum(len(chars) ** i for i in range(maxlen + 1))
    out = np.zeros(total, np.uint8)
    r = lib().oracle_brute_all(regex.encode("latin-1"), None if sig is None else _ptr(sig, C.c_uint8), slen,
                               _ptr(ch, C.c_uint8), ch.size, maxlen, _ptr(out, C.c_uint8))
    if r < 0:
        raise OracleError(-r, "brute-force parse failed")
    assert r == total
    return out.astype(bool)


class OracleSFA:
    """D-SFA by Alg. 4 over the oracle DFA; ids canonical (C3)."""

    def __init__(self, dfa: OracleDFA, cap: int = 1 << 22):
        h = C.c_void_p()
        rc = lib().oracle_sfa_build(dfa._h, cap, C.byref(h))
        if rc != 0:
            raise OracleError(rc, "SFA construction")
        self._h = h
        self.dfa = dfa
        self.n = lib().oracle_sfa_states(h)
        self.table = np.zeros((self.n, 256), np.uint32)
        self.maps = np.zeros((self.n, dfa.n), np.uint32)
        self.finals = np.zeros(self.n, np.uint8)
        lib().oracle_sfa_export(h, _ptr(self.table, C.c_uint32), _ptr(self.maps, C.c_uint32),
                                _ptr(self.finals, C.c_uint8))

    def run_chunked(self, text, bounds):
        """Alg. 5 with chunks [bounds[i], bounds[i+1]): (chunk_ids, q_seq, q_par)."""
        a = _text(text)
        b = np.ascontiguousarray(bounds, np.uint64)
        p = b.size - 1
        ids = np.zeros(max(p, 1), np.uint32)
        qs, qp = C.c_uint32(), C.c_uint32()
        buf = a if a.size else np.zeros(1, np.uint8)
        rc = lib().oracle_sfa_run_chunked(self._h, _ptr(buf, C.c_uint8), _ptr(b, C.c_uint64), p,
                                          _ptr(ids, C.c_uint32), C.byref(qs), C.byref(qp))
        if rc != 0:
            raise OracleError(-rc, "run_chunked")
        return ids[:p], int(qs.value), int(qp.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.oracle_sfa_free(h)
            self._h = None


def _bits_to_int(words: np.ndarray) -> int:
    v = 0
    for i, w in enumerate(words.tolist()):
        v |= int(w) << (64 * i)
    return v


class OracleNFA:
    """eps-free NFA (Thompson states; delta(q, b) = closure(move({q}, b)))."""

    def __init__(self, regex=None, alphabet=None, _h=None):
        L = lib()
        if _h is None:
            self._sig, slen = _sigma(alphabet)
            h = C.c_void_p()
            err = C.create_string_buffer(256)
            rc = L.oracle_nfa_compile(regex.encode("latin-1"),
                                      None if self._sig is None else _ptr(self._sig, C.c_uint8), slen, C.byref(h),
                                      err, 256)
            if rc != 0:
                raise OracleError(rc, err.value.decode(errors="replace"))
            _h = h
        self._h = _h
        self.n = L.oracle_nfa_size(_h)
        self.W = (self.n + 63) // 64

    @classmethod
    def explicit(cls, n: int, delta: dict, initial: set, final: set, alphabet=None):
        """delta: {(q, byte): set of successors}; states 0..n-1 (n <= 64)."""
        d = np.zeros(n * 256, np.uint64)
        for (q, b), succ in delta.items():
            for t in succ:
                d[q * 256 + b] |= np.uint64(1 << t)
        sig, slen = _sigma(alphabet)
        h = C.c_void_p()
        rc = lib().oracle_nfa_explicit(n, _ptr(d, C.c_uint64), sum(1 << q for q in initial),
                                       sum(1 << q for q in final), None if sig is None else _ptr(sig, C.c_uint8),
                                       slen, C.byref(h))
        if rc != 0:
            raise OracleError(rc, "explicit NFA")
        obj = cls(_h=h)
        obj._sig = sig
        return obj

    def run(self, text):
        """The NFA run: (accept, final set as an int bitmask over states)."""
        a = _text(text)
        buf = a if a.size else np.zeros(1, np.uint8)
        out = np.zeros(self.W, np.uint64)
        rc = lib().oracle_nfa_run(self._h, _ptr(buf, C.c_uint8), a.size, _ptr(out, C.c_uint64))
        if rc < 0:
            raise OracleError(-rc, "nfa run")
        return bool(rc), _bits_to_int(out)

    def word_map(self, w):
        """f_w by simulation from every state: tuple of n int bitmasks."""
        a = _text(w)
        buf = a if a.size else np.zeros(1, np.uint8)
        out = np.zeros(self.n * self.W, np.uint64)
        lib().oracle_nfa_word_map(self._h, _ptr(buf, C.c_uint8), a.size, _ptr(out, C.c_uint64))
        return tuple(_bits_to_int(out[q * self.W:(q + 1) * self.W]) for q in range(self.n))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.oracle_nfa_free(h)
            self._h = None


class OracleNSFA:
    """N-SFA: Alg. 4 in its general form over an OracleNFA; canonical ids (C3)."""

    def __init__(self, nfa: OracleNFA, cap: int = 1 << 20):
        h = C.c_void_p()
        rc = lib().oracle_nsfa_build(nfa._h, cap, C.byref(h))
        if rc != 0:
            raise OracleError(rc, "N-SFA construction")
        self._h = h
        self.nfa = nfa
        self.n = lib().oracle_nsfa_states(h)

    def run_chunked(self, text, bounds):
        """Alg. 5: (chunk_ids, (acc_seq, set_seq), (acc_par, set_par))."""
        a = _text(text)
        b = np.ascontiguousarray(bounds, np.uint64)
        p = b.size - 1
        ids = np.zeros(max(p, 1), np.uint32)
        ss = np.zeros(self.nfa.W, np.uint64)
        sp = np.zeros(self.nfa.W, np.uint64)
        buf = a if a.size else np.zeros(1, np.uint8)
        rc = lib().oracle_nsfa_run_chunked(self._h, _ptr(buf, C.c_uint8), _ptr(b, C.c_uint64), p,
                                           _ptr(ids, C.c_uint32), _ptr(ss, C.c_uint64), _ptr(sp, C.c_uint64))
        if rc < 0:
            raise OracleError(-rc, "nsfa run_chunked")
        return ids[:p], (bool(rc & 1), _bits_to_int(ss)), (bool(rc & 2), _bits_to_int(sp))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.oracle_nsfa_free(h)
            self._h = None
