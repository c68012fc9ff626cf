"""B200-native SFA matcher (arXiv 1405.0562, "Simultaneous Finite Automata").

Thin ctypes binding over the C-ABI of ``include/sfa.h``
(``paper_1405_0562_b200/_lib/libsfa.so``).  Argument marshalling only: every
step of the hot path (byte -> column, chunk run, composition, finalisation)
runs in the library's sm_100a kernels.  There is no CPU fallback: if the
library is missing or a call fails, an exception is raised.

Device buffers are passed as ``torch`` tensors (``uint8`` / ``int64``
/ ``uint64`` on a CUDA device) or raw integer device pointers; streams as
``torch.cuda.Stream`` or raw ``cudaStream_t`` integers.  PyTorch is used only
for device memory and streams.

Functions keep the C names: ``sfa_compile``, ``sfa_match``,
``sfa_match_async``, ``sfa_match_batch``, ``sfa_match_host``,
``sfa_match_chunked``, ``sfa_match_rows``, ``sfa_set_residency``, ``sfa_set_compose``,
``sfa_set_tuning``, ``sfa_info``, ``sfa_export_dfa``, ``sfa_export_sfa``, ``sfa_free``;
``SFA`` wraps a handle.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFA_LIB") or os.path.join(_HERE, "_lib", "libsfa.so")  # SFA_LIB: A/B builds

SFA_OK, SFA_ERR_SYNTAX, SFA_ERR_UNSUPPORTED, SFA_ERR_CAPACITY, SFA_ERR_INVALID_ARG, SFA_ERR_CUDA, SFA_ERR_OOM = range(7)
RES_AUTO, RES_SMEM_PRIVATE, RES_SMEM_SHARED, RES_HOT_L2, RES_L2 = range(5)
RES_NAMES = {0: "auto", 1: "smem_private", 2: "smem_shared", 3: "hot_l2", 4: "l2"}
COMPOSE_AUTO, COMPOSE_VEC, COMPOSE_TABLE, COMPOSE_REPLAY = range(4)
COMPOSE_NAMES = {0: "auto", 1: "vec", 2: "table", 3: "replay"}
_ERR_NAMES = {1: "syntax", 2: "unsupported", 3: "capacity", 4: "invalid argument", 5: "cuda", 6: "out of memory"}


class SFAError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


class sfa_result(C.Structure):
    _fields_ = [("final_state", C.c_uint32), ("accept", C.c_uint32)]


class sfa_info_t(C.Structure):
    _fields_ = [
        ("nfa_positions", C.c_uint32), ("dfa_subset_states", C.c_uint32), ("dfa_states", C.c_uint32),
        ("dfa_live", C.c_uint32), ("dead_state", C.c_uint32), ("sfa_states", C.c_uint32),
        ("classes", C.c_uint32), ("sfa_depth", C.c_uint32), ("residency", C.c_uint32),
        ("compose_mode", C.c_uint32), ("range_lo", C.c_uint32), ("range_width", C.c_uint32),
        ("device_table_bytes", C.c_uint64), ("dfa_seconds", C.c_double), ("sfa_seconds", C.c_double),
        ("kind", C.c_uint32), ("nfa_states", C.c_uint32), ("has_dfa", C.c_uint32),
        ("lazy_transitions", C.c_uint64), ("lazy_seconds", C.c_double),
        ("dfa_window_copies", C.c_uint32), ("dfa_window_hot", C.c_uint32),
    ]


class sfa_tuning_t(C.Structure):
    _fields_ = [("tma_k", C.c_int32), ("tma_rowb", C.c_int32), ("tma_ring", C.c_int32), ("tma_promo", C.c_int32),
                ("hot_rows", C.c_uint32), ("no_factor", C.c_uint32), ("dfa_copies", C.c_uint32),
                ("private_copies", C.c_uint32), ("row_align", C.c_uint32), ("direct_piece", C.c_uint32),
                ("dfa_u8", C.c_uint32), ("dfa_layout", C.c_uint32), ("dfa_hot", C.c_uint32),
                ("fact_fold", C.c_uint32)]


class sfa_rows_plan(C.Structure):
    _fields_ = [("head", C.c_uint64), ("row_len", C.c_uint64), ("rows", C.c_uint64), ("tail_start", C.c_uint64),
                ("ctas", C.c_uint32), ("rows_hi", C.c_uint32), ("rows_lo", C.c_uint32), ("ctas_hi", C.c_uint32)]


INVALID_STATE = 0xFFFFFFFF

EXPORTS = ("sfa_compile", "sfa_free", "sfa_last_error", "sfa_info", "sfa_match", "sfa_match_async",
           "sfa_match_batch", "sfa_match_host", "sfa_match_chunked", "sfa_set_residency", "sfa_set_compose",
           "sfa_tune_residency", "sfa_match_map", "sfa_combine_maps", "sfa_match_batch_uniform", "sfa_match_speculative",
           "sfa_export_dfa", "sfa_export_sfa", "sfa_set_tuning", "sfa_match_rows", "sfa_match_batch_host", "sfa_compile_nsfa", "sfa_compile_lazy",
           "sfa_match_lazy")

_lib = None


def lib() -> C.CDLL:
    """Loads libsfa.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() or python -m paper_1405_0562_b200._build")
        L = C.CDLL(LIB_PATH)
        vp, u8p, u32p, u64p = C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
        L.sfa_compile.argtypes = [C.c_char_p, u8p, C.c_int, C.c_uint32, C.POINTER(vp)]
        L.sfa_compile_nsfa.argtypes = [C.c_char_p, u8p, C.c_int, C.c_uint32, C.POINTER(vp)]
        L.sfa_compile_lazy.argtypes = [C.c_char_p, u8p, C.c_int, C.c_uint32, C.POINTER(vp)]
        L.sfa_match_lazy.argtypes = [vp, vp, C.c_size_t, vp, u32p, C.POINTER(C.c_int)]
        L.sfa_free.argtypes = [vp]
        L.sfa_free.restype = None
        L.sfa_last_error.restype = C.c_char_p
        L.sfa_info.argtypes = [vp, C.POINTER(sfa_info_t)]
        L.sfa_match.argtypes = [vp, vp, C.c_size_t, vp, u32p, C.POINTER(C.c_int)]
        L.sfa_match_async.argtypes = [vp, vp, C.c_size_t, vp, vp]
        L.sfa_match_batch.argtypes = [vp, vp, vp, C.c_size_t, vp, vp]
        L.sfa_match_host.argtypes = [vp, vp, C.c_size_t, vp, u32p, C.POINTER(C.c_int)]
        L.sfa_match_chunked.argtypes = [vp, vp, C.c_size_t, C.c_uint32, vp, u32p, C.POINTER(C.c_int), u32p]
        L.sfa_set_residency.argtypes = [vp, C.c_int]
        L.sfa_set_compose.argtypes = [vp, C.c_int]
        L.sfa_tune_residency.argtypes = [vp, vp, C.c_size_t, vp]
        L.sfa_match_map.argtypes = [vp, vp, C.c_size_t, vp, vp]
        L.sfa_match_batch_uniform.argtypes = [vp, vp, C.c_size_t, C.c_size_t, vp, vp]
        L.sfa_combine_maps.argtypes = [vp, vp, C.c_size_t, vp, vp]
        L.sfa_match_speculative.argtypes = [vp, vp, C.c_size_t, C.c_uint64, vp, vp, vp]
        L.sfa_set_tuning.argtypes = [vp, C.POINTER(sfa_tuning_t)]
        L.sfa_match_batch_host.argtypes = [vp, vp, vp, C.c_size_t, vp, vp]
        L.sfa_match_rows.argtypes = [vp, vp, C.c_size_t, vp, vp, C.c_size_t, C.POINTER(sfa_rows_plan), vp]
        L.sfa_export_dfa.argtypes = [vp, u32p, u8p]
        L.sfa_export_sfa.argtypes = [vp, u32p, u32p, u8p]
        for f in EXPORTS:
            if f not in ("sfa_free", "sfa_last_error"):
                getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc != SFA_OK:
        raise SFAError(rc, lib().sfa_last_error().decode(errors="replace"))


def _dptr(x) -> int:
    """Device pointer of a CUDA tensor (or an int passed through)."""
    if isinstance(x, int):
        return x
    if not x.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not x.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return x.data_ptr()


def _stream(s) -> int:
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _nbytes(x) -> int:
    return x.numel() * x.element_size()


# --------------------------------------------------------------------------- C names
def sfa_compile(regex, alphabet=None, max_sfa: int = 0, nsfa: bool = False, lazy: bool = False) -> int:
    """regex (str/bytes), alphabet (bytes or None = all 256 bytes) -> handle (int).
    nsfa: the N-SFA of the Glushkov NFA (sfa_compile_nsfa) instead of the D-SFA;
    lazy: the DFA only, the D-SFA built on the fly while matching (sfa_compile_lazy)."""
    rx = regex.encode("latin-1") if isinstance(regex, str) else bytes(regex)
    if b"\0" in rx:
        raise SFAError(SFA_ERR_INVALID_ARG, "regex contains NUL")
    h = C.c_void_p()
    fn = lib().sfa_compile_lazy if lazy else (lib().sfa_compile_nsfa if nsfa else lib().sfa_compile)
    if alphabet is None:
        rc = fn(rx, None, 0, max_sfa, C.byref(h))
    else:
        al = np.frombuffer(bytes(alphabet), np.uint8).copy()
        rc = fn(rx, al.ctypes.data_as(C.POINTER(C.c_uint8)), al.size, max_sfa, C.byref(h))
    _check(rc)
    return h.value


def sfa_free(h: int):
    lib().sfa_free(h)


def sfa_info(h: int) -> dict:
    info = sfa_info_t()
    _check(lib().sfa_info(h, C.byref(info)))
    return {k: getattr(info, k) for k, _ in sfa_info_t._fields_}


def sfa_match(h: int, d_text, n: int | None = None, stream=None):
    """Blocking: -> (final_state, accept)."""
    n = _nbytes(d_text) if n is None else n
    q, a = C.c_uint32(), C.c_int()
    _check(lib().sfa_match(h, _dptr(d_text) if n else None, n, _stream(stream), C.byref(q), C.byref(a)))
    return q.value, bool(a.value)


def sfa_match_lazy(h: int, d_text, n: int | None = None, stream=None):
    """On-the-fly handle (sfa_compile_lazy), blocking: -> (final_state, accept)."""
    n = _nbytes(d_text) if n is None else n
    q, a = C.c_uint32(), C.c_int()
    _check(lib().sfa_match_lazy(h, _dptr(d_text) if n else None, n, _stream(stream), C.byref(q), C.byref(a)))
    return q.value, bool(a.value)


def sfa_match_async(h: int, d_text, d_result, n: int | None = None, stream=None):
    """Stream-ordered: writes (final_state, accept) as 2 x uint32 at d_result (device)."""
    n = _nbytes(d_text) if n is None else n
    _check(lib().sfa_match_async(h, _dptr(d_text) if n else None, n, _stream(stream), _dptr(d_result)))


def sfa_match_batch(h: int, d_texts, d_offsets, count: int, d_results, stream=None):
    """Stream-ordered: d_results (device, count x 2 uint32) per text."""
    if count == 0:
        return
    _check(lib().sfa_match_batch(h, _dptr(d_texts), _dptr(d_offsets), count, _stream(stream), _dptr(d_results)))


def sfa_match_map(h: int, d_text, d_map, n: int | None = None, stream=None):
    """Stream-ordered: d_map (device, |D| x uint32) <- f_text(q) for every DFA state q."""
    n = _nbytes(d_text) if n is None else n
    _check(lib().sfa_match_map(h, _dptr(d_text) if n else None, n, _stream(stream), _dptr(d_map)))


def sfa_combine_maps(h: int, d_maps, count: int, d_result, stream=None):
    """Stream-ordered: d_result (device, 2 x uint32) <- (q, accept) after the shard maps in order."""
    _check(lib().sfa_combine_maps(h, _dptr(d_maps) if count else None, count, _stream(stream), _dptr(d_result)))


def sfa_match_speculative(h: int, d_text, d_result, nchunks: int = 0, d_chunk_maps=None, n: int | None = None,
                          stream=None):
    """The paper's baseline (Alg. 3): the DFA run speculatively from every state per chunk.

    Stream-ordered: d_result (device, 2 x uint32) <- (q_final, accept); d_chunk_maps (device,
    chunks x |D| uint32, optional) <- T_i[q] = delta^(q, chunk i).  nchunks = 0: automatic.
    """
    n = _nbytes(d_text) if n is None else n
    _check(lib().sfa_match_speculative(h, _dptr(d_text) if n else None, n, nchunks, _stream(stream),
                                       _dptr(d_chunk_maps) if d_chunk_maps is not None else None,
                                       _dptr(d_result)))


def sfa_match_batch_uniform(h: int, d_texts, length: int, count: int, d_results, stream=None):
    """Stream-ordered: count back-to-back texts of `length` bytes -> d_results (device, count x 2 uint32)."""
    if count == 0:
        return
    _check(lib().sfa_match_batch_uniform(h, _dptr(d_texts), length, count, _stream(stream), _dptr(d_results)))


def sfa_match_host(h: int, h_text, stream=None):
    """End to end from host memory (numpy array or pinned CPU tensor): -> (final_state, accept)."""
    if isinstance(h_text, np.ndarray):
        ptr, n = h_text.ctypes.data, h_text.nbytes
    else:
        ptr, n = h_text.data_ptr(), _nbytes(h_text)
    q, a = C.c_uint32(), C.c_int()
    _check(lib().sfa_match_host(h, ptr if n else None, n, _stream(stream), C.byref(q), C.byref(a)))
    return q.value, bool(a.value)


def _hptr(x) -> int:
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise ValueError("expected a contiguous array")
        return x.ctypes.data
    if x.is_cuda:
        raise ValueError("expected host memory")
    return x.data_ptr()


def sfa_match_batch_host(h: int, h_texts, h_offsets, count: int | None = None, h_results=None, stream=None):
    """End to end from host memory (numpy arrays or CPU tensors, pinned or not):
    -> (final_states uint32[count], accepts uint32[count]); blocking."""
    off = h_offsets
    count = (off.size if isinstance(off, np.ndarray) else off.numel()) - 1 if count is None else count
    res = np.zeros((max(count, 1), 2), np.uint32) if h_results is None else h_results
    if count:
        _check(lib().sfa_match_batch_host(h, _hptr(h_texts), _hptr(off), count, _stream(stream), _hptr(res)))
    r = res if isinstance(res, np.ndarray) else res.numpy()
    r = r.view(np.uint32).reshape(-1, 2)[:count]
    return r[:, 0], r[:, 1]


def sfa_match_chunked(h: int, d_text, nchunks: int, n: int | None = None, stream=None, want_states: bool = True):
    """Forced SPEC chunking (test knob): -> (final_state, accept, chunk_states or None)."""
    n = _nbytes(d_text) if n is None else n
    q, a = C.c_uint32(), C.c_int()
    cnt = min(nchunks, max(n, 1))
    states = np.zeros(cnt, np.uint32) if want_states else None
    sp = states.ctypes.data_as(C.POINTER(C.c_uint32)) if want_states else None
    _check(lib().sfa_match_chunked(h, _dptr(d_text) if n else None, n, nchunks, _stream(stream),
                                   C.byref(q), C.byref(a), sp))
    return q.value, bool(a.value), states


def sfa_set_residency(h: int, mode: int):
    _check(lib().sfa_set_residency(h, mode))


def sfa_tune_residency(h: int, d_sample=None, n: int | None = None, stream=None):
    """HOT residency: re-rank rows by visit frequency on a device text sample (None: static ranking)."""
    if d_sample is None:
        _check(lib().sfa_tune_residency(h, None, 0, _stream(stream)))
        return
    n = _nbytes(d_sample) if n is None else n
    _check(lib().sfa_tune_residency(h, _dptr(d_sample), n, _stream(stream)))


def sfa_set_tuning(h: int, **knobs):
    """Launch-shape knobs (sfa_tuning_t field names; none changes a result).  No
    arguments: back to automatic.  Blocking; the device tables are rebuilt lazily."""
    if not knobs:
        _check(lib().sfa_set_tuning(h, None))
        return
    t = sfa_tuning_t()
    t.tma_promo = -1
    for k, v in knobs.items():
        if k not in dict(sfa_tuning_t._fields_):
            raise ValueError(f"unknown tuning knob {k}")
        setattr(t, k, int(v))
    _check(lib().sfa_set_tuning(h, C.byref(t)))


def sfa_match_rows(h: int, d_text, d_row_ids, d_result, n: int | None = None, stream=None) -> dict:
    """TMA scan with its per-row SFA ids (diagnostic; n >= 64 KiB): stream-ordered writes of
    d_row_ids (device u32) and d_result; returns the row geometry."""
    n = _nbytes(d_text) if n is None else n
    p = sfa_rows_plan()
    cap = d_row_ids.numel() if not isinstance(d_row_ids, int) else 1 << 40
    _check(lib().sfa_match_rows(h, _dptr(d_text), n, _stream(stream), _dptr(d_row_ids), cap, C.byref(p),
                                _dptr(d_result)))
    return {k: getattr(p, k) for k, _ in sfa_rows_plan._fields_}


def sfa_set_compose(h: int, mode: int):
    _check(lib().sfa_set_compose(h, mode))


def sfa_export_dfa(h: int):
    info = sfa_info(h)
    nd = info["dfa_states"]
    table = np.zeros((nd, 256), np.uint32)
    finals = np.zeros(nd, np.uint8)
    _check(lib().sfa_export_dfa(h, table.ctypes.data_as(C.POINTER(C.c_uint32)),
                                finals.ctypes.data_as(C.POINTER(C.c_uint8))))
    return table, finals


def sfa_export_sfa_table(h: int):
    """D-SFA or N-SFA: (table |S| x 256 ids, None, finals) -- no mapping export."""
    info = sfa_info(h)
    ns = info["sfa_states"]
    table = np.zeros((ns, 256), np.uint32)
    finals = np.zeros(ns, np.uint8)
    _check(lib().sfa_export_sfa(h, table.ctypes.data_as(C.POINTER(C.c_uint32)), None,
                                finals.ctypes.data_as(C.POINTER(C.c_uint8))))
    return table, None, finals


def sfa_export_sfa(h: int):
    info = sfa_info(h)
    ns, nd = info["sfa_states"], info["dfa_states"]
    table = np.zeros((ns, 256), np.uint32)
    maps = np.zeros((ns, nd), np.uint32)
    finals = np.zeros(ns, np.uint8)
    _check(lib().sfa_export_sfa(h, table.ctypes.data_as(C.POINTER(C.c_uint32)),
                                maps.ctypes.data_as(C.POINTER(C.c_uint32)),
                                finals.ctypes.data_as(C.POINTER(C.c_uint8))))
    return table, maps, finals


# --------------------------------------------------------------------------- handle object
class SFA:
    """Owns one compiled handle: ``SFA(regex, alphabet)``."""

    def __init__(self, regex, alphabet=None, max_sfa: int = 0, nsfa: bool = False, lazy: bool = False):
        self.h = sfa_compile(regex, alphabet, max_sfa, nsfa, lazy)
        self._match_async = lib().sfa_match_async

    def close(self):
        if getattr(self, "h", None):
            sfa_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        return sfa_info(self.h)

    def match(self, d_text, stream=None):
        return sfa_match(self.h, d_text, None, stream)

    def match_async(self, d_text, d_result, stream=None):
        # the hot call of serving loops: plain attribute reads, one C call
        n = d_text.numel()
        if n and not (d_text.is_cuda and d_text.dtype.itemsize == 1 and d_text.is_contiguous()):
            raise ValueError("expected a contiguous uint8 CUDA tensor")
        rc = self._match_async(self.h, d_text.data_ptr() if n else None, n,
                               _stream(stream), d_result.data_ptr())
        if rc:
            _check(rc)

    def match_batch(self, d_texts, d_offsets, count, d_results, stream=None):
        return sfa_match_batch(self.h, d_texts, d_offsets, count, d_results, stream)

    def match_batch_uniform(self, d_texts, length, count, d_results, stream=None):
        return sfa_match_batch_uniform(self.h, d_texts, length, count, d_results, stream)

    def match_map(self, d_text, d_map, stream=None):
        return sfa_match_map(self.h, d_text, d_map, None, stream)

    def combine_maps(self, d_maps, count, d_result, stream=None):
        return sfa_combine_maps(self.h, d_maps, count, d_result, stream)

    def match_speculative(self, d_text, d_result, nchunks=0, d_chunk_maps=None, stream=None):
        return sfa_match_speculative(self.h, d_text, d_result, nchunks, d_chunk_maps, None, stream)

    def match_batch_host(self, h_texts, h_offsets, count=None, h_results=None, stream=None):
        return sfa_match_batch_host(self.h, h_texts, h_offsets, count, h_results, stream)

    def match_lazy(self, d_text, stream=None):
        return sfa_match_lazy(self.h, d_text, None, stream)

    def match_host(self, h_text, stream=None):
        return sfa_match_host(self.h, h_text, stream)

    def match_chunked(self, d_text, nchunks, stream=None, want_states=True):
        return sfa_match_chunked(self.h, d_text, nchunks, None, stream, want_states)

    def set_residency(self, mode: int):
        sfa_set_residency(self.h, mode)

    def set_compose(self, mode: int):
        sfa_set_compose(self.h, mode)

    def set_tuning(self, **knobs):
        sfa_set_tuning(self.h, **knobs)

    def match_rows(self, d_text, d_row_ids, d_result, stream=None):
        return sfa_match_rows(self.h, d_text, d_row_ids, d_result, None, stream)

    def tune_residency(self, d_sample=None, stream=None):
        sfa_tune_residency(self.h, d_sample, None, stream)

    def export_dfa(self):
        return sfa_export_dfa(self.h)

    def export_sfa(self):
        return sfa_export_sfa(self.h)
