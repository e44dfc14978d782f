"""ctypes binding of ``libkmerscan_b200.so`` (include/kmerscan_b200.h).

This is the only path to the scan: there is no CPU fallback.  If the library
is missing or no B200 is visible, every scan call raises ``RuntimeError``.
ctypes releases the GIL for the duration of each native call, so scans can be
issued from threads like the reference's nogil kernels (engine.py:219-232).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("KMERSCAN_B200_LIB", _HERE / "_lib" / "libkmerscan_b200.so"))

KS_OK = 0
KS_E_INVALID = -1
KS_E_CUDA = -2
KS_E_CHAIN = -3
KS_E_UNSUPPORTED = -4
KS_E_NOMEM = -5

STRATEGY_LOOKBACK = 1
STRATEGY_MAPSCAN = 2
STRATEGY_SPECULATE = 3
STRATEGY_NAMES = {STRATEGY_LOOKBACK: "lookback", STRATEGY_MAPSCAN: "mapscan",
                  STRATEGY_SPECULATE: "speculate"}


class ReductionChainError(RuntimeError):
    """Internal invariant failure: no chunk result continues the state chain
    (reference engine.py:34-35)."""


class DfaInfo(C.Structure):
    _fields_ = [("n_states", C.c_int32), ("n_expressions", C.c_int32),
                ("n_accepting", C.c_int32), ("strategy", C.c_int32),
                ("sync_depth", C.c_int32), ("stride", C.c_int32),
                ("monoid_size", C.c_int32), ("other_resets", C.c_int32),
                ("table_bytes", C.c_int64), ("tables_in_smem", C.c_int32),
                ("reserved", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("scan_ms", C.c_float), ("total_ms", C.c_float),
                ("kernel_launches", C.c_int32), ("chunks", C.c_int32),
                ("chunk_len", C.c_int64), ("rows", C.c_int64),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64)]


EXPORTED = (
    "ks_open", "ks_close", "ks_set_stream", "ks_set_reserved_sms", "ks_synchronize", "ks_get_stats", "ks_last_error",
    "ks_version", "ks_dfa_upload", "ks_dfa_upload_ex", "ks_dfa_info_get", "ks_dfa_free",
    "ks_seq_upload_codes", "ks_seq_upload_ascii", "ks_seq_encode_device", "ks_seq_length",
    "ks_seq_download_codes", "ks_seq_download_softmask", "ks_seq_free", "ks_count", "ks_locate",
    "ks_count_host_ascii", "ks_count_async", "ks_async_wait", "ks_segment_map_async",
    "ks_count_shard_async", "ks_count_shard_async_signal", "ks_stream_wait_value32", "ks_pack_host_ascii", "ks_pack_host_codes", "ks_count_host_bytes", "ks_pack_host_wire",
    "ks_scan_range", "ks_segment_map", "ks_speculate", "ks_free",
    "ks_open_multi", "ks_close_multi", "ks_multi_info", "ks_mdfa_upload", "ks_mdfa_free",
    "ks_mseq_upload_codes", "ks_mseq_upload_ascii", "ks_mseq_length", "ks_mseq_free", "ks_mcount",
    "ks_mlocate", "ks_reconciliation_sweep",
)

_lib = None
_lib_lock = threading.Lock()

_P = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


def _declare(lib) -> None:
    sig = {
        "ks_open": (C.c_int, [C.c_int, C.POINTER(_P)]),
        "ks_close": (C.c_int, [_P]),
        "ks_set_stream": (C.c_int, [_P, _P]),
        "ks_set_reserved_sms": (C.c_int, [_P, C.c_int32]),
        "ks_synchronize": (C.c_int, [_P]),
        "ks_get_stats": (C.c_int, [_P, C.POINTER(Stats)]),
        "ks_last_error": (C.c_char_p, []),
        "ks_version": (C.c_char_p, []),
        "ks_dfa_upload": (C.c_int, [_P, _i32p, C.c_int32, _i32p, _i32p, C.c_int32, C.POINTER(_P)]),
        "ks_dfa_upload_ex": (C.c_int, [_P, _i32p, C.c_int32, _i32p, _i32p, C.c_int32, C.c_int32,
                                       C.POINTER(_P)]),
        "ks_dfa_info_get": (C.c_int, [_P, C.POINTER(DfaInfo)]),
        "ks_dfa_free": (C.c_int, [_P]),
        "ks_seq_upload_codes": (C.c_int, [_P, _u8p, C.c_int64, C.POINTER(_P)]),
        "ks_seq_upload_ascii": (C.c_int, [_P, _u8p, C.c_int64, C.c_int32, C.POINTER(_P)]),
        "ks_seq_encode_device": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.POINTER(_P)]),
        "ks_seq_length": (C.c_int, [_P, _i64p]),
        "ks_seq_download_codes": (C.c_int, [_P, _P, _u8p]),
        "ks_seq_download_softmask": (C.c_int, [_P, _P, C.POINTER(C.c_uint64), C.c_int64]),
        "ks_seq_free": (C.c_int, [_P]),
        "ks_count": (C.c_int, [_P, _P, _P, _i64p]),
        "ks_locate": (C.c_int, [_P, _P, _P, _i64p, C.POINTER(_i64p), _i64p]),
        "ks_count_host_ascii": (C.c_int, [_P, _P, _u8p, C.c_int64, _i64p]),
        "ks_count_host_bytes": (C.c_int, [_P, _P, _u8p, C.c_int64, C.c_int32, _i64p]),
        "ks_count_async": (C.c_int, [_P, _P, _P, _i64p]),
        "ks_pack_host_ascii": (C.c_int, [_u8p, C.c_int64, C.c_int32, _P, _P, _i32p]),
        "ks_pack_host_wire": (C.c_int, [_u8p, C.c_int64, C.c_int32, _P, _P, _i64p]),
        "ks_pack_host_codes": (C.c_int, [_u8p, C.c_int64, C.c_int32, _P, _P]),
        "ks_segment_map_async": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, _P]),
        "ks_count_shard_async": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, _P, C.c_int32, _P]),
        "ks_count_shard_async_signal": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, _P, C.c_int32, _P, _P,
                                                  C.c_uint32]),
        "ks_stream_wait_value32": (C.c_int, [_P, _P, C.c_uint32]),
        "ks_async_wait": (C.c_int, [_P, C.POINTER(C.c_float), _i32p, _i32p]),
        "ks_scan_range": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, C.c_int32, C.c_int64, _i64p,
                                    _i32p, C.POINTER(_i64p), _i64p]),
        "ks_segment_map": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, _i32p]),
        "ks_speculate": (C.c_int, [_P, _P, _P, C.c_int32, _i64p, _i64p, _i64p, _i32p, C.c_int32,
                                   _i32p, _i64p]),
        "ks_free": (None, [_P]),
        "ks_open_multi": (C.c_int, [C.c_int32, _i32p, C.POINTER(_P)]),
        "ks_close_multi": (C.c_int, [_P]),
        "ks_multi_info": (C.c_int, [_P, _i32p, _i32p]),
        "ks_mdfa_upload": (C.c_int, [_P, _i32p, C.c_int32, _i32p, _i32p, C.c_int32, C.POINTER(_P)]),
        "ks_mdfa_free": (C.c_int, [_P]),
        "ks_mseq_upload_codes": (C.c_int, [_P, _u8p, C.c_int64, C.POINTER(_P)]),
        "ks_mseq_upload_ascii": (C.c_int, [_P, _u8p, C.c_int64, C.c_int32, C.POINTER(_P)]),
        "ks_mseq_length": (C.c_int, [_P, _i64p]),
        "ks_mseq_free": (C.c_int, [_P]),
        "ks_mcount": (C.c_int, [_P, _P, _P, _i64p]),
        "ks_mlocate": (C.c_int, [_P, _P, _P, _i64p, C.POINTER(_i64p), _i64p]),
        "ks_reconciliation_sweep": (C.c_int, [_P, _i32p, C.c_int32, _i32p, _i32p, C.c_int32, _i32p, _i32p,
                                              C.c_int32, C.c_int32, C.c_int32, _i64p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def library():
    """Load (once) and return the native library; raises if it is missing."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"kmerscan_b200 native library not found at {LIB_PATH}; build it with "
                    f"`python -c 'import __graft_entry__ as g; g.build()'` or "
                    f"`make -C paper_1509_01506_b200/csrc`")
            lib = C.CDLL(str(LIB_PATH))
            _declare(lib)
            _lib = lib
        return _lib


def _check(rc: int) -> None:
    if rc == KS_OK:
        return
    msg = library().ks_last_error().decode(errors="replace")
    if rc == KS_E_INVALID:
        raise ValueError(msg)
    if rc == KS_E_CHAIN:
        raise ReductionChainError(msg)
    if rc == KS_E_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"kmerscan_b200: {msg} (status {rc})")


def _ptr(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


class DfaHandle:
    """Device-resident compiled automaton (ks_dfa)."""

    def __init__(self, ctx: "DeviceContext", dfa, strategy: int = 0):
        lib = library()
        trans = np.ascontiguousarray(np.asarray(dfa.transitions, dtype=np.int32))
        if trans.ndim != 2 or trans.shape[1] != 5:
            raise ValueError("transitions must have shape (n_states, 5)")
        off = np.ascontiguousarray(np.asarray(dfa.out_offsets, dtype=np.int32))
        ids = np.ascontiguousarray(np.asarray(dfa.out_ids, dtype=np.int32))
        if off.shape[0] != trans.shape[0] + 1:
            raise ValueError("out_offsets must have n_states + 1 entries")
        h = _P()
        ids_buf = ids if ids.size else np.zeros(1, dtype=np.int32)
        _check(lib.ks_dfa_upload_ex(ctx.handle, _ptr(trans, C.c_int32), int(trans.shape[0]),
                                    _ptr(off, C.c_int32), _ptr(ids_buf, C.c_int32),
                                    int(dfa.n_expressions), int(strategy), C.byref(h)))
        self.ctx = ctx
        self.handle = h
        self.n_states = int(trans.shape[0])
        self.n_expressions = int(dfa.n_expressions)
        info = DfaInfo()
        _check(lib.ks_dfa_info_get(h, C.byref(info)))
        self.info = {name: getattr(info, name) for name, _ in DfaInfo._fields_ if name != "reserved"}
        self.info["strategy_name"] = STRATEGY_NAMES.get(info.strategy, "?")
        self._finalizer = weakref.finalize(self, _free_dfa, lib, h)

    def free(self) -> None:
        self._finalizer()


def _free_dfa(lib, h):
    try:
        lib.ks_dfa_free(h)
    except Exception:  # interpreter shutdown
        pass


def _free_seq(lib, h):
    try:
        lib.ks_seq_free(h)
    except Exception:
        pass


class SeqHandle:
    """Device-resident packed sequence (ks_seq)."""

    def __init__(self, ctx: "DeviceContext", handle):
        self.ctx = ctx
        self.handle = handle
        n = C.c_int64()
        _check(library().ks_seq_length(handle, C.byref(n)))
        self.length = int(n.value)
        self._finalizer = weakref.finalize(self, _free_seq, library(), handle)

    def free(self) -> None:
        self._finalizer()

    def codes(self) -> np.ndarray:
        out = np.empty(max(self.length, 1), dtype=np.uint8)
        _check(library().ks_seq_download_codes(self.ctx.handle, self.handle, _ptr(out, C.c_uint8)))
        return out[: self.length]

    def softmask(self) -> np.ndarray:
        words = max((self.length + 63) // 64, 1)
        out = np.zeros(words, dtype=np.uint64)
        _check(library().ks_seq_download_softmask(self.ctx.handle, self.handle,
                                                  _ptr(out, C.c_uint64), words))
        bits = np.unpackbits(out.view(np.uint8), bitorder="little")
        return bits[: self.length].astype(bool)


class DeviceContext:
    """One CUDA device + stream (ks_ctx).  Calls are serialised per context."""

    def __init__(self, device: int = 0):
        lib = library()
        h = _P()
        _check(lib.ks_open(int(device), C.byref(h)))
        self.device = int(device)
        self.handle = h
        self.lock = threading.RLock()
        self._dfas: dict[int, tuple] = {}
        self._finalizer = weakref.finalize(self, lib.ks_close, h)

    # ---------------------------------------------------------------- uploads
    def dfa(self, dfa, strategy: int = 0) -> DfaHandle:
        """Cached upload of a Dfa (keyed by object identity)."""
        if isinstance(dfa, DfaHandle):
            return dfa
        key = (id(dfa), strategy)
        hit = self._dfas.get(key)
        if hit is not None and hit[0]() is dfa:
            return hit[1]
        handle = DfaHandle(self, dfa, strategy)
        try:
            ref = weakref.ref(dfa, lambda _r, k=key, d=self._dfas: d.pop(k, None))
            self._dfas[key] = (ref, handle)
        except TypeError:
            pass
        return handle

    def upload_codes(self, codes: np.ndarray) -> SeqHandle:
        arr = np.ascontiguousarray(np.asarray(codes, dtype=np.uint8))
        buf = arr if arr.size else np.zeros(1, dtype=np.uint8)
        h = _P()
        with self.lock:
            _check(library().ks_seq_upload_codes(self.handle, _ptr(buf, C.c_uint8), int(arr.size),
                                                 C.byref(h)))
        return SeqHandle(self, h)

    def upload_ascii(self, data, fasta: bool = False) -> SeqHandle:
        """Raw (or FASTA) bytes -> device encode (ks_seq_upload_ascii)."""
        arr = np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray, memoryview)) \
            else np.ascontiguousarray(np.asarray(data, dtype=np.uint8))
        buf = arr if arr.size else np.zeros(1, dtype=np.uint8)
        h = _P()
        with self.lock:
            _check(library().ks_seq_upload_ascii(self.handle, _ptr(buf, C.c_uint8), int(arr.size),
                                                 int(bool(fasta)), C.byref(h)))
        return SeqHandle(self, h)

    def encode_device(self, device_ptr: int, n_bytes: int, fasta: bool = False) -> SeqHandle:
        h = _P()
        with self.lock:
            _check(library().ks_seq_encode_device(self.handle, _P(device_ptr), int(n_bytes), int(bool(fasta)),
                                                  C.byref(h)))
        return SeqHandle(self, h)

    def seq(self, seq) -> SeqHandle:
        """Device form of a Sequence-like object (cached on our Sequence)."""
        if isinstance(seq, SeqHandle):
            return seq
        cache = getattr(seq, "_device", None)
        if isinstance(cache, dict):
            h = cache.get(self.device)
            if h is not None and h.ctx is self:
                return h
        h = self.upload_codes(seq.symbols)
        if isinstance(cache, dict):
            cache[self.device] = h
        return h

    # ------------------------------------------------------------------ scans
    def set_stream(self, stream_ptr: int | None) -> None:
        _check(library().ks_set_stream(self.handle, _P(stream_ptr or 0)))

    def set_reserved_sms(self, n_sms: int) -> None:
        """Leave n_sms SMs free of scan CTAs (for kernels on other streams)."""
        _check(library().ks_set_reserved_sms(self.handle, int(n_sms)))

    def synchronize(self) -> None:
        _check(library().ks_synchronize(self.handle))

    def count(self, dfa: DfaHandle, seq: SeqHandle) -> np.ndarray:
        counts = np.zeros(max(dfa.n_expressions, 1), dtype=np.int64)
        with self.lock:
            _check(library().ks_count(self.handle, dfa.handle, seq.handle, _ptr(counts, C.c_int64)))
        return counts[: dfa.n_expressions]

    def count_async(self, dfa: DfaHandle, seq: SeqHandle, out_pinned: np.ndarray) -> None:
        """Enqueue a count; the int64 counts land in `out_pinned` (a view of
        page-locked memory) once :meth:`async_wait` returns."""
        if out_pinned.dtype != np.int64 or out_pinned.size < max(dfa.n_expressions, 1):
            raise ValueError("out_pinned must be an int64 buffer of n_expressions entries")
        _check(library().ks_count_async(self.handle, dfa.handle, seq.handle, _ptr(out_pinned, C.c_int64)))

    def segment_map_async(self, dfa: DfaHandle, seq: SeqHandle, begin: int, end: int, d_map: int) -> None:
        """Shard boundary map into device memory (int32[n_states]) without syncing."""
        _check(library().ks_segment_map_async(self.handle, dfa.handle, seq.handle, int(begin), int(end),
                                              _P(d_map)))

    def count_shard_async(self, dfa: DfaHandle, seq: SeqHandle, begin: int, end: int, d_maps: int,
                          rank: int, d_counts: int) -> None:
        """Scan a shard from the state composed on the device out of the
        gathered maps of ranks < rank (d_maps = 0 with rank > 0: halo mode,
        the bases before `begin` are the previous shard's tail); counts
        (uint64) into device memory."""
        _check(library().ks_count_shard_async(self.handle, dfa.handle, seq.handle, int(begin), int(end),
                                              _P(d_maps), int(rank), _P(d_counts)))

    def count_shard_async_signal(self, dfa: DfaHandle, seq: SeqHandle, begin: int, end: int, d_maps: int,
                                 rank: int, d_counts: int, d_signal: int, value: int) -> None:
        """count_shard_async, then the device sets *d_signal = value once the
        counts are final (for a collective on another stream)."""
        _check(library().ks_count_shard_async_signal(self.handle, dfa.handle, seq.handle, int(begin), int(end),
                                                     _P(d_maps), int(rank), _P(d_counts), _P(d_signal),
                                                     int(value) & 0xFFFFFFFF))

    @staticmethod
    def stream_wait_value32(stream_ptr: int, d_addr: int, value: int) -> None:
        """The CUDA stream waits until the uint32 at d_addr is >= value."""
        _check(library().ks_stream_wait_value32(_P(stream_ptr), _P(d_addr), int(value) & 0xFFFFFFFF))

    def async_wait(self) -> dict:
        ms, calls, launches = C.c_float(), C.c_int32(), C.c_int32()
        _check(library().ks_async_wait(self.handle, C.byref(ms), C.byref(calls), C.byref(launches)))
        return {"scan_ms_total": ms.value, "calls": calls.value, "kernel_launches": launches.value}

    def count_host_ascii(self, dfa: DfaHandle, data, fasta: bool = False) -> np.ndarray:
        """End-to-end count from a host buffer of raw (or FASTA) bytes:
        pipelined pack/copy/encode + scan (ks_count_host_bytes)."""
        arr = np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray, memoryview)) \
            else np.ascontiguousarray(np.asarray(data, dtype=np.uint8))
        buf = arr if arr.size else np.zeros(1, dtype=np.uint8)
        counts = np.zeros(max(dfa.n_expressions, 1), dtype=np.int64)
        with self.lock:
            _check(library().ks_count_host_bytes(self.handle, dfa.handle, _ptr(buf, C.c_uint8), int(arr.size),
                                                 int(bool(fasta)), _ptr(counts, C.c_int64)))
        return counts[: dfa.n_expressions]

    def locate(self, dfa: DfaHandle, seq: SeqHandle) -> tuple[np.ndarray, np.ndarray]:
        counts = np.zeros(max(dfa.n_expressions, 1), dtype=np.int64)
        rows_p = _i64p()
        n = C.c_int64()
        with self.lock:
            _check(library().ks_locate(self.handle, dfa.handle, seq.handle, _ptr(counts, C.c_int64),
                                       C.byref(rows_p), C.byref(n)))
        return counts[: dfa.n_expressions], _take_rows(rows_p, int(n.value))

    def scan_range(self, dfa: DfaHandle, seq: SeqHandle, begin: int, end: int, entry: int = -1,
                   row_base: int = 0, locate: bool = False):
        """Counts, exit state (original id) and optional rows of [begin, end)."""
        counts = np.zeros(max(dfa.n_expressions, 1), dtype=np.int64)
        exit_state = C.c_int32()
        rows_p = _i64p()
        n = C.c_int64()
        with self.lock:
            _check(library().ks_scan_range(
                self.handle, dfa.handle, seq.handle, int(begin), int(end), int(entry), int(row_base),
                _ptr(counts, C.c_int64), C.byref(exit_state),
                C.byref(rows_p) if locate else None, C.byref(n) if locate else None))
        rows = _take_rows(rows_p, int(n.value)) if locate else None
        return counts[: dfa.n_expressions], int(exit_state.value), rows

    def segment_map(self, dfa: DfaHandle, seq: SeqHandle, begin: int, end: int) -> np.ndarray:
        out = np.zeros(dfa.n_states, dtype=np.int32)
        with self.lock:
            _check(library().ks_segment_map(self.handle, dfa.handle, seq.handle, int(begin), int(end),
                                            _ptr(out, C.c_int32)))
        return out

    def speculate(self, dfa: DfaHandle, seq: SeqHandle, chunk_begin, chunk_end, pss_off, pss,
                  window: int, with_delta: bool = False):
        cb = np.ascontiguousarray(chunk_begin, dtype=np.int64)
        ce = np.ascontiguousarray(chunk_end, dtype=np.int64)
        off = np.ascontiguousarray(pss_off, dtype=np.int64)
        data = np.ascontiguousarray(pss, dtype=np.int32)
        total = int(off[-1]) if off.size else 0
        conv = np.full(max(total, 1), -1, dtype=np.int32)
        delta = np.zeros((max(total, 1), max(dfa.n_expressions, 1)), dtype=np.int64) if with_delta else None
        data_buf = data if data.size else np.zeros(1, dtype=np.int32)
        with self.lock:
            _check(library().ks_speculate(
                self.handle, dfa.handle, seq.handle, int(cb.size), _ptr(cb, C.c_int64),
                _ptr(ce, C.c_int64), _ptr(off, C.c_int64), _ptr(data_buf, C.c_int32), int(window),
                _ptr(conv, C.c_int32), _ptr(delta, C.c_int64) if with_delta else None))
        conv = conv[:total]
        if with_delta:
            delta = delta[:total, : dfa.n_expressions]
        return conv, delta

    def reconciliation_sweep(self, dfa, pss_sets, length: int, window: int) -> np.ndarray:
        """ks_reconciliation_sweep: int64[4] = speculative runs, converged
        runs, count mismatches, final-state mismatches."""
        trans = np.ascontiguousarray(np.asarray(dfa.transitions, dtype=np.int32))
        off = np.ascontiguousarray(np.asarray(dfa.out_offsets, dtype=np.int32))
        ids = np.ascontiguousarray(np.asarray(dfa.out_ids, dtype=np.int32))
        ids = ids if ids.size else np.zeros(1, dtype=np.int32)
        data = np.ascontiguousarray(np.concatenate([np.asarray(p, dtype=np.int32) for p in pss_sets]))
        poff = np.zeros(len(pss_sets) + 1, dtype=np.int32)
        poff[1:] = np.cumsum([len(p) for p in pss_sets])
        out = np.zeros(4, dtype=np.int64)
        with self.lock:
            _check(library().ks_reconciliation_sweep(
                self.handle, _ptr(trans, C.c_int32), int(trans.shape[0]), _ptr(off, C.c_int32),
                _ptr(ids, C.c_int32), int(dfa.n_expressions), _ptr(data, C.c_int32), _ptr(poff, C.c_int32),
                len(pss_sets), int(length), int(window), _ptr(out, C.c_int64)))
        return out

    def stats(self) -> dict:
        st = Stats()
        _check(library().ks_get_stats(self.handle, C.byref(st)))
        return {name: getattr(st, name) for name, _ in Stats._fields_}


def _take_rows(rows_p, n: int) -> np.ndarray:
    """(n, 2) int64 view of library-allocated rows, without a copy: the
    buffer is handed back to ks_free when the array is garbage collected."""
    lib = library()
    if n == 0 or not rows_p:
        if rows_p:
            lib.ks_free(C.cast(rows_p, _P))
        return np.empty((0, 2), dtype=np.int64)
    addr = C.cast(rows_p, C.c_void_p).value
    holder = (C.c_int64 * (2 * n)).from_address(addr)
    weakref.finalize(holder, lib.ks_free, C.c_void_p(addr))
    return np.frombuffer(holder, dtype=np.int64).reshape(n, 2)


_contexts: dict[int, DeviceContext] = {}
_ctx_lock = threading.Lock()


def pack_host_ascii(data, lb: int) -> tuple[np.ndarray, np.ndarray, int]:
    """The streaming count's host packer on its own (no GPU needed): returns
    (bases uint64[2*slots], nmask uint64[slots], flags) in tile-slot order."""
    arr = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8) if isinstance(data, (bytes, bytearray))
                               else np.asarray(data, dtype=np.uint8))
    tile = 32 << lb
    slots = max(-(-((arr.size + 63) // 64) // tile) * tile, 1)
    bases = np.zeros(2 * slots, dtype=np.uint64)
    nmask = np.zeros(slots, dtype=np.uint64)
    flags = C.c_int32()
    buf = arr if arr.size else np.zeros(1, dtype=np.uint8)
    _check(library().ks_pack_host_ascii(_ptr(buf, C.c_uint8), int(arr.size), int(lb), bases.ctypes.data,
                                        nmask.ctypes.data, C.byref(flags)))
    return bases, nmask, int(flags.value)


def pack_host_codes(codes, lb: int) -> tuple[np.ndarray, np.ndarray]:
    """The codes upload's host packer on its own (no GPU needed): symbol codes
    0..4 -> (bases uint64[2*slots], nmask uint64[slots]) in tile-slot order."""
    arr = np.ascontiguousarray(np.asarray(codes, dtype=np.uint8))
    tile = 32 << lb
    slots = max(-(-((arr.size + 63) // 64) // tile) * tile, 1)
    bases = np.zeros(2 * slots, dtype=np.uint64)
    nmask = np.zeros(slots, dtype=np.uint64)
    buf = arr if arr.size else np.zeros(1, dtype=np.uint8)
    _check(library().ks_pack_host_codes(_ptr(buf, C.c_uint8), int(arr.size), int(lb), bases.ctypes.data,
                                        nmask.ctypes.data))
    return bases, nmask


def pack_host_wire(data, fasta: bool) -> tuple[np.ndarray, np.ndarray, int]:
    """Host side of the FASTA/whitespace stream (no GPU needed): (bases
    uint64[2*blocks], special uint64[blocks], retained symbols)."""
    arr = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8))
    nb = max((arr.size + 63) // 64, 1)
    bases = np.zeros(2 * nb, dtype=np.uint64)
    special = np.zeros(nb, dtype=np.uint64)
    kept = C.c_int64()
    buf = arr if arr.size else np.zeros(1, dtype=np.uint8)
    _check(library().ks_pack_host_wire(_ptr(buf, C.c_uint8), int(arr.size), int(bool(fasta)), bases.ctypes.data,
                                       special.ctypes.data, C.byref(kept)))
    return bases, special, int(kept.value)


def _free_with(fn_name: str, h) -> None:
    try:
        getattr(library(), fn_name)(h)
    except Exception:  # interpreter shutdown
        pass


class MultiContext:
    """One sequence over several devices of this process (ks_mctx): slices
    per device, NCCL between distinct devices (peer copies when a device id
    repeats).  Same results as DeviceContext.count/locate on one device."""

    def __init__(self, devices):
        devs = [int(d) for d in devices]
        if not devs or min(devs) < 0:
            raise ValueError("devices must be a non-empty list of device ids")
        arr = np.asarray(devs, dtype=np.int32)
        h = _P()
        _check(library().ks_open_multi(len(devs), _ptr(arr, C.c_int32), C.byref(h)))
        self.devices = tuple(devs)
        self.handle = h
        self.lock = threading.RLock()
        n, nc = C.c_int32(), C.c_int32()
        _check(library().ks_multi_info(h, C.byref(n), C.byref(nc)))
        self.uses_nccl = bool(nc.value)
        self._dfas: dict[int, tuple] = {}
        self._finalizer = weakref.finalize(self, _free_with, "ks_close_multi", h)

    def close(self) -> None:
        self._finalizer()

    def dfa(self, dfa):
        key = id(dfa)
        hit = self._dfas.get(key)
        if hit is not None and hit[0]() is dfa:
            return hit[1]
        trans = np.ascontiguousarray(np.asarray(dfa.transitions, dtype=np.int32))
        off = np.ascontiguousarray(np.asarray(dfa.out_offsets, dtype=np.int32))
        ids = np.ascontiguousarray(np.asarray(dfa.out_ids, dtype=np.int32))
        ids = ids if ids.size else np.zeros(1, dtype=np.int32)
        h = _P()
        with self.lock:
            _check(library().ks_mdfa_upload(self.handle, _ptr(trans, C.c_int32), int(trans.shape[0]),
                                            _ptr(off, C.c_int32), _ptr(ids, C.c_int32), int(dfa.n_expressions),
                                            C.byref(h)))
        handle = _MultiHandle(h, "ks_mdfa_free", n_expressions=int(dfa.n_expressions), owner=self)
        try:
            self._dfas[key] = (weakref.ref(dfa, lambda _r, k=key, d=self._dfas: d.pop(k, None)), handle)
        except TypeError:
            pass
        return handle

    def _seq(self, fn: str, *args):
        h = _P()
        with self.lock:
            _check(getattr(library(), fn)(self.handle, *args, C.byref(h)))
        n = C.c_int64()
        _check(library().ks_mseq_length(h, C.byref(n)))
        return _MultiHandle(h, "ks_mseq_free", length=int(n.value), owner=self)

    def upload_codes(self, codes: np.ndarray):
        arr = np.ascontiguousarray(np.asarray(codes, dtype=np.uint8))
        buf = arr if arr.size else np.zeros(1, dtype=np.uint8)
        return self._seq("ks_mseq_upload_codes", _ptr(buf, C.c_uint8), int(arr.size))

    def upload_ascii(self, data, fasta: bool = False):
        arr = np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray, memoryview)) \
            else np.ascontiguousarray(np.asarray(data, dtype=np.uint8))
        buf = arr if arr.size else np.zeros(1, dtype=np.uint8)
        return self._seq("ks_mseq_upload_ascii", _ptr(buf, C.c_uint8), int(arr.size), int(bool(fasta)))

    def count(self, dfa, seq) -> np.ndarray:
        counts = np.zeros(max(dfa.n_expressions, 1), dtype=np.int64)
        with self.lock:
            _check(library().ks_mcount(self.handle, dfa.handle, seq.handle, _ptr(counts, C.c_int64)))
        return counts[: dfa.n_expressions]

    def locate(self, dfa, seq) -> tuple[np.ndarray, np.ndarray]:
        counts = np.zeros(max(dfa.n_expressions, 1), dtype=np.int64)
        rows_p = _i64p()
        n = C.c_int64()
        with self.lock:
            _check(library().ks_mlocate(self.handle, dfa.handle, seq.handle, _ptr(counts, C.c_int64),
                                        C.byref(rows_p), C.byref(n)))
        return counts[: dfa.n_expressions], _take_rows(rows_p, int(n.value))


class _MultiHandle:
    """ks_mdfa / ks_mseq handle (freed with its context kept alive)."""

    def __init__(self, handle, free_fn: str, owner, **attrs):
        self.handle = handle
        self.owner = owner
        self.__dict__.update(attrs)
        self._finalizer = weakref.finalize(self, _free_with, free_fn, handle)

    def free(self) -> None:
        self._finalizer()


_multi: dict[tuple, MultiContext] = {}


def multi_context(devices) -> MultiContext:
    """Process-wide multi-device context for a tuple of device ids."""
    key = tuple(int(d) for d in devices)
    with _ctx_lock:
        m = _multi.get(key)
        if m is None:
            m = MultiContext(key)
            _multi[key] = m
        return m


def context(device: int = 0) -> DeviceContext:
    """Process-wide context for a device (created on first use)."""
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = DeviceContext(device)
            _contexts[device] = ctx
        return ctx
