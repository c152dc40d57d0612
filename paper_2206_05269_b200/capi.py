"""ctypes binding of libwfcu.so (include/wfcu.h).

The shared library is the product; this module only marshals arguments.  There is
no Python or CPU implementation behind any call: if the library is missing the
import fails loudly, and every compute entry point returns WFCU_ERR_NO_DEVICE when
no sm_100 GPU is present.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libwfcu.so"

OK = 0
ERR_INVALID_ARGUMENT = -1
ERR_CUDA = -2
ERR_NO_DEVICE = -3
ERR_TABLE_FULL = -4
ERR_DEFERRED_FULL = -5
ERR_ARENA_FULL = -6
ERR_BUFFER_TOO_SMALL = -7
ERR_NOT_SORTED = -8
ERR_FRAME_MAGIC, ERR_FRAME_TRUNCATED, ERR_FRAME_TRAILING, ERR_FRAME_ENCODING = -9, -10, -11, -12

MAP_IDENTITY, MAP_SQUARE_ROOT, MAP_ALTERNATING_HARMONIC_TERM, MAP_SQUARE = 0, 1, 2, 3
DTYPE_F32, DTYPE_F64 = 0, 1

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)


class WfcuError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"wfcu error {code}: {message}")
        self.code = code
        self.message = message


class InvalidArgument(WfcuError, ValueError):
    """Maps the reference's std::invalid_argument."""


class CounterConfig(C.Structure):
    _fields_ = [("table_slots", C.c_uint64), ("deferred_slots", C.c_uint64),
                ("arena_bytes", C.c_uint64), ("long_slots", C.c_uint64)]


# name -> (restype, argtypes); every symbol include/wfcu.h declares
SIGNATURES = {
    "wfcu_last_error": (C.c_char_p, []),
    "wfcu_version": (C.c_char_p, []),
    "wfcu_device_count": (C.c_int, []),
    "wfcu_set_device": (C.c_int, [C.c_int]),
    "wfcu_sm_count": (C.c_int, [C.POINTER(C.c_int)]),
    "wfcu_dev_alloc": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint64]),
    "wfcu_dev_free": (None, [C.c_void_p]),
    "wfcu_dev_upload": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "wfcu_dev_download": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "wfcu_map_reduce_dev": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, f64p]),
    "wfcu_map_reduce_dev_async": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]),
    "wfcu_map_reduce_blocked_dev": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_void_p, f64p]),
    "wfcu_map_reduce_host": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_int, f64p]),
    "wfcu_map_reduce_blocked_host": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_int, C.c_uint64, f64p]),
    "wfcu_alternating_harmonic": (C.c_int, [C.c_uint64, C.c_uint64, f64p]),
    "wfcu_counter_create": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(CounterConfig)]),
    "wfcu_counter_destroy": (None, [C.c_void_p]),
    "wfcu_counter_reset": (C.c_int, [C.c_void_p, C.c_void_p]),
    "wfcu_counter_count_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "wfcu_counter_count_host": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), u64p, C.c_uint64]),
    "wfcu_counter_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "wfcu_counter_take_kernel_ms": (C.c_int, [C.c_void_p, f64p, u64p]),
    "wfcu_counter_status": (C.c_int, [C.c_void_p, C.c_void_p]),
    "wfcu_counter_stats": (C.c_int, [C.c_void_p, C.c_void_p, u64p, u64p, u64p]),
    "wfcu_counter_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64]),
    "wfcu_counter_top_k": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_uint64, u64p, u64p]),
    "wfcu_timer_create": (C.c_int, [C.POINTER(C.c_void_p)]),
    "wfcu_timer_start": (C.c_int, [C.c_void_p]),
    "wfcu_timer_stop_ns": (C.c_int, [C.c_void_p, u64p]),
    "wfcu_timer_destroy": (None, [C.c_void_p]),
    "wfcu_wordcount_multi": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "wfcu_tokens_encode_frame": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64, u64p, C.c_void_p]),
    "wfcu_tokens_decode_frame": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p), C.c_void_p]),
    "wfcu_tokens_concat_slices": (C.c_int, [C.c_void_p, u64p, u64p, C.c_uint32, C.POINTER(C.c_void_p)]),
    "wfcu_counter_distinctive": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64,
                                           C.c_void_p, C.c_void_p, C.c_uint64, u64p]),
    "wfcu_counter_merge": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "wfcu_counter_add_words": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64]),
    "wfcu_owner_of": (C.c_uint32, [C.c_void_p, C.c_uint32, C.c_uint32]),
    "wfcu_counter_partition": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "wfcu_counter_max_entries": (C.c_uint64, [C.c_void_p]),
    "wfcu_counter_partition_fixed": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "wfcu_counter_partition_framed": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "wfcu_counter_merge_regions": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p]),
    "wfcu_counter_merge_entries": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "wfcu_counter_long_records": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, u64p, C.c_void_p]),
    "wfcu_counter_merge_long_records": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p]),
    "wfcu_utf8_sanitize_dev": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, u64p, C.c_void_p]),
    "wfcu_utf8_sanitize_host": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, u64p]),
    "wfcu_normalize_words_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p]),
    "wfcu_tokenize_dev": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(C.c_void_p)]),
    "wfcu_tokenize_host": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p)]),
    "wfcu_tokenize_docs_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p)]),
    "wfcu_tokens_destroy": (None, [C.c_void_p]),
    "wfcu_tokens_stats": (C.c_int, [C.c_void_p, u64p, u64p]),
    "wfcu_tokens_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "wfcu_tokens_from_words": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p)]),
    "wfcu_tokens_sort": (C.c_int, [C.c_void_p, C.c_void_p]),
    "wfcu_tokens_reduce_sorted": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "wfcu_counter_count_dev_sorted": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "wfcu_top_k": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, u64p, u64p]),
    "wfcu_distinctive": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, u64p]),
    "wfcu_synth_document": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_double, C.c_uint32, C.c_void_p, C.c_uint64]),
    "wfcu_synth_corpus": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_double, C.c_uint32, C.c_uint64, C.c_void_p, C.c_int]),
    "wfcu_synth_corpus_strided": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_double, C.c_uint32, C.c_uint64, C.c_void_p, C.c_int]),
    "wfcu_synth_uniform": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_void_p]),
    "wfcu_launch_count": (C.c_uint64, []),
}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2206_05269_b200.build` "
            "(there is no fallback implementation)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)   # AttributeError if the library lacks a declared symbol
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = (lib.wfcu_last_error() or b"").decode("utf-8", "replace")
    if rc in (ERR_INVALID_ARGUMENT, ERR_NOT_SORTED):
        raise InvalidArgument(rc, msg)
    raise WfcuError(rc, msg)


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def device_count() -> int:
    return int(lib.wfcu_device_count())


def launch_count() -> int:
    return int(lib.wfcu_launch_count())


def sm_count() -> int:
    out = C.c_int(0)
    check(lib.wfcu_sm_count(C.byref(out)))
    return out.value


# ---- packed word lists <-> python --------------------------------------------------
def pack_words(words: list[bytes]) -> tuple[np.ndarray, np.ndarray]:
    lens = np.fromiter((len(w) for w in words), dtype=np.uint32, count=len(words))
    blob = np.frombuffer(b"".join(words), dtype=np.uint8).copy() if words else np.zeros(0, np.uint8)
    return blob, lens


def unpack_words(blob: np.ndarray, lens: np.ndarray) -> list[bytes]:
    raw = blob.tobytes()
    out, off = [], 0
    for n in lens.tolist():
        out.append(raw[off:off + n])
        off += n
    return out


# ---- map-then-reduce ------------------------------------------------------------------
def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return DTYPE_F32
    if a.dtype == np.float64:
        return DTYPE_F64
    raise InvalidArgument(ERR_INVALID_ARGUMENT, f"unsupported dtype {a.dtype}")


def map_reduce_host(values: np.ndarray, kind: int) -> float:
    values = np.ascontiguousarray(values)
    out = C.c_double(0.0)
    check(lib.wfcu_map_reduce_host(_ptr(values), _dtype_code(values), values.size, kind, C.byref(out)))
    return out.value


def map_reduce_blocked_host(values: np.ndarray, kind: int, block_size: int) -> float:
    values = np.ascontiguousarray(values)
    out = C.c_double(0.0)
    check(lib.wfcu_map_reduce_blocked_host(_ptr(values), _dtype_code(values), values.size, kind, block_size, C.byref(out)))
    return out.value


def alternating_harmonic(n: int, block_size: int = 256) -> float:
    out = C.c_double(0.0)
    check(lib.wfcu_alternating_harmonic(n, block_size, C.byref(out)))
    return out.value


def map_reduce_dev(ptr: int, dtype: int, n: int, kind: int, position_base: int = 0, stream: int = 0) -> float:
    out = C.c_double(0.0)
    check(lib.wfcu_map_reduce_dev(C.c_void_p(ptr), dtype, n, position_base, kind, C.c_void_p(stream), C.byref(out)))
    return out.value


def map_reduce_dev_async(ptr: int, dtype: int, n: int, kind: int, out_ptr: int, position_base: int = 0,
                         stream: int = 0) -> None:
    check(lib.wfcu_map_reduce_dev_async(C.c_void_p(ptr), dtype, n, position_base, kind, C.c_void_p(stream),
                                        C.c_void_p(out_ptr)))


def map_reduce_blocked_dev(ptr: int, dtype: int, n: int, kind: int, block_size: int, position_base: int = 0,
                           stream: int = 0) -> float:
    out = C.c_double(0.0)
    check(lib.wfcu_map_reduce_blocked_dev(C.c_void_p(ptr), dtype, n, position_base, kind, block_size,
                                          C.c_void_p(stream), C.byref(out)))
    return out.value


# ---- counter ----------------------------------------------------------------------------
def utf8_sanitize_host(data) -> bytes:
    """wfc::utf8_sanitize on the device, host buffers in and out."""
    a = np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray, memoryview)) else np.ascontiguousarray(data)
    out = np.zeros(3 * a.size + 16, np.uint8)
    n = C.c_uint64(0)
    check(lib.wfcu_utf8_sanitize_host(_ptr(a), a.size, _ptr(out), out.size, C.byref(n)))
    return out[:n.value].tobytes()


def utf8_sanitize_dev(in_ptr: int, n: int, out_ptr: int, out_cap: int, stream: int = 0) -> int:
    """Device buffers; returns the output length (waits for the stream)."""
    m = C.c_uint64(0)
    check(lib.wfcu_utf8_sanitize_dev(C.c_void_p(in_ptr), n, C.c_void_p(out_ptr), out_cap, C.byref(m), C.c_void_p(stream)))
    return m.value


class HostDocs:
    """The (pointer, length) arrays of wfcu_counter_count_host for a list of host documents.
    Keeps the buffers alive; reusable across calls."""

    def __init__(self, docs):
        self.n = len(docs)
        self._keep = [np.frombuffer(d, dtype=np.uint8) if isinstance(d, (bytes, bytearray, memoryview)) else d for d in docs]
        addr = [a.__array_interface__["data"][0] if a.size else None for a in self._keep]
        self.ptrs = (C.c_void_p * max(self.n, 1))(*addr)
        self.lens = (C.c_uint64 * max(self.n, 1))(*[a.size for a in self._keep])


class StageNs(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("map_ns", "sort_ns", "encode_ns", "exchange_ns", "reduce_ns", "repair_ns", "total_ns")]


class Counter:
    """Device-resident word -> count table (wfcu_counter)."""

    @classmethod
    def _adopt(cls, handle) -> "Counter":
        c = cls.__new__(cls)
        c._h = C.c_void_p(handle)
        return c

    def __init__(self, table_slots: int = 0, deferred_slots: int = 0, arena_bytes: int = 0, long_slots: int = 0):
        self._h = C.c_void_p()
        cfg = CounterConfig(table_slots, deferred_slots, arena_bytes, long_slots)
        check(lib.wfcu_counter_create(C.byref(self._h), C.byref(cfg)))

    def close(self) -> None:
        if getattr(self, "_h", None) and lib is not None:
            lib.wfcu_counter_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def reset(self, stream: int = 0) -> None:
        check(lib.wfcu_counter_reset(self._h, C.c_void_p(stream)))

    def count_dev(self, ptr: int, n: int, stream: int = 0) -> None:
        check(lib.wfcu_counter_count_dev(self._h, C.c_void_p(ptr), n, C.c_void_p(stream)))

    def count_dev_sorted(self, ptr: int, n: int, stream: int = 0) -> None:
        check(lib.wfcu_counter_count_dev_sorted(self._h, C.c_void_p(ptr), n, C.c_void_p(stream)))

    def count_host(self, docs: "list[bytes] | list[np.ndarray] | HostDocs") -> None:
        """docs: host buffers, or a HostDocs made once from them (the pointer/length arrays a C caller
        would hold anyway; building them costs ~1 us per document in Python)."""
        hd = docs if isinstance(docs, HostDocs) else HostDocs(docs)
        check(lib.wfcu_counter_count_host(self._h, hd.ptrs, hd.lens, hd.n))

    def set_timing(self, enabled: bool) -> None:
        check(lib.wfcu_counter_set_timing(self._h, int(enabled)))

    def take_kernel_ms(self) -> tuple[float, int]:
        ms, n = C.c_double(), C.c_uint64()
        check(lib.wfcu_counter_take_kernel_ms(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def status(self, stream: int = 0) -> None:
        check(lib.wfcu_counter_status(self._h, C.c_void_p(stream)))

    def stats(self, stream: int = 0) -> tuple[int, int, int]:
        d, t, b = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib.wfcu_counter_stats(self._h, C.c_void_p(stream), C.byref(d), C.byref(t), C.byref(b)))
        return d.value, t.value, b.value

    def export(self, stream: int = 0, out=None) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(key_bytes, key_lens, counts) in std::map order.
        out: optional (uint8, uint32, uint64) arrays to fill instead of new ones -- e.g. views of page-locked
        memory reused from call to call, which the copy engine fills several times faster than fresh pageable
        arrays; they must be large enough (WfcuError ERR_BUFFER_TOO_SMALL otherwise)."""
        distinct, _, key_bytes = self.stats(stream)
        if out is None:
            blob = np.empty(max(key_bytes, 1), np.uint8)
            lens = np.empty(max(distinct, 1), np.uint32)
            counts = np.empty(max(distinct, 1), np.uint64)
        else:
            blob, lens, counts = out
            if blob.dtype != np.uint8 or lens.dtype != np.uint32 or counts.dtype != np.uint64:
                raise TypeError("export(out=...) wants (uint8, uint32, uint64) arrays")
            if blob.size < key_bytes or lens.size < distinct or counts.size < distinct:
                raise WfcuError(ERR_BUFFER_TOO_SMALL, f"export needs {key_bytes} key bytes and {distinct} rows")
        check(lib.wfcu_counter_export(self._h, C.c_void_p(stream), _ptr(blob), key_bytes, _ptr(lens), _ptr(counts), distinct))
        return blob[:key_bytes], lens[:distinct], counts[:distinct]

    def to_dict(self, stream: int = 0) -> dict[bytes, int]:
        blob, lens, counts = self.export(stream)
        return dict(zip(unpack_words(blob, lens), (int(c) for c in counts)))

    def top_k(self, k: int, stream: int = 0) -> tuple[list[tuple[bytes, int, float]], int]:
        """wfc::top_k straight from the device table: ([(word, count, rel_freq)], total_words)."""
        cap = max(k, 1)
        blob = np.zeros(64 * cap + 4096, np.uint8)
        lens, counts, rel = np.zeros(cap, np.uint32), np.zeros(cap, np.uint64), np.zeros(cap, np.float64)
        rows, total = C.c_uint64(), C.c_uint64()
        while True:
            rc = lib.wfcu_counter_top_k(self._h, k, C.c_void_p(stream), _ptr(blob), blob.size, _ptr(lens), _ptr(counts),
                                        _ptr(rel), cap, C.byref(rows), C.byref(total))
            if rc == ERR_BUFFER_TOO_SMALL and blob.size < (1 << 30):   # very long tokens among the leaders
                blob = np.zeros(blob.size * 8, np.uint8)
                continue
            check(rc)
            break
        n = rows.value
        words = unpack_words(blob, lens[:n])
        return [(words[r], int(counts[r]), float(rel[r])) for r in range(n)], total.value

    def distinctive(self, others: "Counter", k: int, stream: int = 0) -> list[tuple[bytes, float]]:
        """distinctive_words(self, others) on the device tables: [(word, score)], at most k rows."""
        cap = max(k, 1)
        kb = np.zeros(64 * cap + 1024, np.uint8)
        kl = np.zeros(cap, np.uint32)
        sc = np.zeros(cap, np.float64)
        n = C.c_uint64()
        check(lib.wfcu_counter_distinctive(self._h, others._h, k, C.c_void_p(stream), _ptr(kb), kb.size, _ptr(kl),
                                           _ptr(sc), cap, C.byref(n)))
        words = unpack_words(kb, kl[:n.value])
        return [(w, float(sc[i])) for i, w in enumerate(words)]

    def merge(self, other: "Counter", stream: int = 0) -> None:
        check(lib.wfcu_counter_merge(self._h, other._h, C.c_void_p(stream)))

    def add_words(self, words: list[bytes], counts: list[int]) -> None:
        blob, lens = pack_words(words)
        cnt = np.asarray(counts, dtype=np.uint64)
        check(lib.wfcu_counter_add_words(self._h, _ptr(blob), _ptr(lens), _ptr(cnt), len(words)))

    # exchange
    def partition(self, n_parts: int, entries_ptr: int, entries_cap: int, part_counts_ptr: int, stream: int = 0) -> None:
        check(lib.wfcu_counter_partition(self._h, n_parts, C.c_void_p(entries_ptr), entries_cap,
                                         C.c_void_p(part_counts_ptr), C.c_void_p(stream)))

    def partition_fixed(self, n_parts: int, entries_ptr: int, cap_per_part: int, counts_ptr: int, stream: int = 0) -> None:
        check(lib.wfcu_counter_partition_fixed(self._h, n_parts, C.c_void_p(entries_ptr), cap_per_part,
                                               C.c_void_p(counts_ptr), C.c_void_p(stream)))

    def partition_framed(self, n_parts: int, entries_ptr: int, cap_per_part: int, counts_ptr: int, stream: int = 0) -> None:
        check(lib.wfcu_counter_partition_framed(self._h, n_parts, C.c_void_p(entries_ptr), cap_per_part,
                                                C.c_void_p(counts_ptr), C.c_void_p(stream)))

    def merge_regions(self, entries_ptr: int, n_parts: int, cap_per_part: int, counts_ptr: int, stream: int = 0) -> None:
        check(lib.wfcu_counter_merge_regions(self._h, C.c_void_p(entries_ptr), n_parts, cap_per_part,
                                             C.c_void_p(counts_ptr), C.c_void_p(stream)))

    def max_entries(self) -> int:
        return int(lib.wfcu_counter_max_entries(self._h))

    def merge_entries(self, entries_ptr: int, n: int, stream: int = 0) -> None:
        check(lib.wfcu_counter_merge_entries(self._h, C.c_void_p(entries_ptr), n, C.c_void_p(stream)))

    def long_records(self, out_ptr: int = 0, out_cap: int = 0, stream: int = 0) -> int:
        n = C.c_uint64(0)
        check(lib.wfcu_counter_long_records(self._h, C.c_void_p(out_ptr), out_cap, C.byref(n), C.c_void_p(stream)))
        return n.value

    def merge_long_records(self, ptr: int, n_bytes: int, part: int, n_parts: int, stream: int = 0) -> None:
        check(lib.wfcu_counter_merge_long_records(self._h, C.c_void_p(ptr), n_bytes, part, n_parts, C.c_void_p(stream)))


def wordcount_multi(docs, n_workers: int, table_slots: int = 0) -> "tuple[list[Counter], dict[str, int]]":
    """run_wordcount over n_workers workers on this box's GPUs (worker j on device j mod device_count, documents
    d = j mod n): the owner tables, one per worker, and the CUDA-event stage times."""
    hd = docs if isinstance(docs, HostDocs) else HostDocs(docs)
    shards = (C.c_void_p * n_workers)()
    cfg = CounterConfig(table_slots, 0, 0, 0)
    t = StageNs()
    check(lib.wfcu_wordcount_multi(hd.ptrs, hd.lens, hd.n, n_workers, C.byref(cfg), shards, C.byref(t)))
    return [Counter._adopt(h) for h in shards], {k: int(getattr(t, k)) for k, _ in StageNs._fields_}


def owner_of(word: bytes, n_parts: int) -> int:
    buf = np.frombuffer(word, dtype=np.uint8)
    return int(lib.wfcu_owner_of(_ptr(buf), len(word), n_parts))


# ---- tokens -------------------------------------------------------------------------------
class Tokens:
    """Device-resident token list (wfcu_tokens)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    @classmethod
    def tokenize_host(cls, text: bytes) -> "Tokens":
        buf = np.frombuffer(text, dtype=np.uint8)
        h = C.c_void_p()
        check(lib.wfcu_tokenize_host(_ptr(buf) if buf.size else None, buf.size, C.byref(h)))
        return cls(h)

    @classmethod
    def tokenize_docs_host(cls, docs) -> "Tokens":
        """one list for several host documents (a whitespace byte behind each), gathered on the device"""
        hd = docs if isinstance(docs, HostDocs) else HostDocs(docs)
        h = C.c_void_p()
        check(lib.wfcu_tokenize_docs_host(hd.ptrs, hd.lens, hd.n, C.byref(h)))
        return cls(h)

    @classmethod
    def tokenize_dev(cls, ptr: int, n: int, stream: int = 0) -> "Tokens":
        h = C.c_void_p()
        check(lib.wfcu_tokenize_dev(C.c_void_p(ptr), n, C.c_void_p(stream), C.byref(h)))
        return cls(h)

    @classmethod
    def from_words(cls, words: list[bytes]) -> "Tokens":
        blob, lens = pack_words(words)
        h = C.c_void_p()
        check(lib.wfcu_tokens_from_words(_ptr(blob), _ptr(lens), len(words), C.byref(h)))
        return cls(h)

    @classmethod
    def concat_slices(cls, srcs: "list[Tokens]", begins: list[int], ends: list[int]) -> "Tokens":
        """A new device list: the slices [begin, end) of the source lists, in order (device-to-device)."""
        n = len(srcs)
        hs = (C.c_void_p * max(n, 1))(*[t._h for t in srcs])
        b = (C.c_uint64 * max(n, 1))(*begins)
        e = (C.c_uint64 * max(n, 1))(*ends)
        h = C.c_void_p()
        check(lib.wfcu_tokens_concat_slices(hs, b, e, n, C.byref(h)))
        return cls(h)

    def frame_bytes(self, begin: int, end: int, stream: int = 0) -> int:
        """size of the WCX1 frame of tokens [begin, end)"""
        n = C.c_uint64()
        check(lib.wfcu_tokens_encode_frame(self._h, begin, end, None, 0, C.byref(n), C.c_void_p(stream)))
        return n.value

    def encode_frame(self, begin: int, end: int, out_ptr: int, out_cap: int, stream: int = 0) -> int:
        """WCX1 frame of tokens [begin, end) into device memory at out_ptr; returns its size"""
        n = C.c_uint64()
        check(lib.wfcu_tokens_encode_frame(self._h, begin, end, C.c_void_p(out_ptr), out_cap, C.byref(n), C.c_void_p(stream)))
        return n.value

    @classmethod
    def decode_frame(cls, frame_ptr: int, frame_bytes: int, stream: int = 0) -> "Tokens":
        """decode_message of a WCX1 frame in device memory (WfcuError with ERR_FRAME_* codes on a bad frame)"""
        h = C.c_void_p()
        check(lib.wfcu_tokens_decode_frame(C.c_void_p(frame_ptr), frame_bytes, C.byref(h), C.c_void_p(stream)))
        return cls(h)

    def close(self) -> None:
        if getattr(self, "_h", None) and lib is not None:
            lib.wfcu_tokens_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stats(self) -> tuple[int, int]:
        n, b = C.c_uint64(), C.c_uint64()
        check(lib.wfcu_tokens_stats(self._h, C.byref(n), C.byref(b)))
        return n.value, b.value

    def words(self) -> list[bytes]:
        n, b = self.stats()
        blob = np.zeros(max(b, 1), np.uint8)
        lens = np.zeros(max(n, 1), np.uint32)
        check(lib.wfcu_tokens_export(self._h, _ptr(blob), b, _ptr(lens), n))
        return unpack_words(blob[:b], lens[:n])

    def sort(self, stream: int = 0) -> None:
        check(lib.wfcu_tokens_sort(self._h, C.c_void_p(stream)))

    def reduce_sorted(self, into: Counter, stream: int = 0) -> None:
        check(lib.wfcu_tokens_reduce_sorted(self._h, into.handle, C.c_void_p(stream)))


def normalize_words(fragments: list[bytes]) -> list[bytes | None]:
    """wfc::normalize_word over a batch (None = the reference's nullopt)."""
    blob, lens = pack_words(fragments)
    out = np.zeros(3 * blob.size + 16, np.uint8)
    out_lens = np.zeros(max(len(fragments), 1), np.uint32)
    check(lib.wfcu_normalize_words_host(_ptr(blob), _ptr(lens), len(fragments), _ptr(out), out.size, _ptr(out_lens)))
    words = unpack_words(out, out_lens[:len(fragments)])
    return [w if w else None for w in words]


# ---- analysis over exported tables -----------------------------------------------------------
Table = tuple  # (key_bytes, key_lens, counts) as returned by Counter.export()


def top_k(table: Table, k: int) -> tuple[list[tuple[bytes, int, float]], int]:
    """wfc::top_k: ([(word, count, rel_freq)], total_words)."""
    blob, lens, counts = (np.ascontiguousarray(a) for a in table)
    n = len(lens)
    idx = np.zeros(max(min(n, k), 1), np.uint64)
    rel = np.zeros(max(min(n, k), 1), np.float64)
    total, rows = C.c_uint64(), C.c_uint64()
    check(lib.wfcu_top_k(_ptr(blob), _ptr(lens), _ptr(counts), n, k, _ptr(idx), _ptr(rel), C.byref(total), C.byref(rows)))
    words = unpack_words(blob, lens)
    return [(words[int(idx[r])], int(counts[int(idx[r])]), float(rel[r])) for r in range(rows.value)], total.value


def distinctive(target: Table, others: Table, k: int) -> list[tuple[bytes, float]]:
    """wfc::distinctive_words: [(word, score)]."""
    tb, tl, tc = (np.ascontiguousarray(a) for a in target)
    ob, ol, oc = (np.ascontiguousarray(a) for a in others)
    cap = max(min(len(tl) + len(ol), k), 1)
    src, idx, score = np.zeros(cap, np.int32), np.zeros(cap, np.uint64), np.zeros(cap, np.float64)
    rows = C.c_uint64()
    check(lib.wfcu_distinctive(_ptr(tb), _ptr(tl), _ptr(tc), len(tl), _ptr(ob), _ptr(ol), _ptr(oc), len(ol), k,
                               _ptr(src), _ptr(idx), _ptr(score), C.byref(rows)))
    tw, ow = unpack_words(tb, tl), unpack_words(ob, ol)
    return [((ow if src[r] else tw)[int(idx[r])], float(score[r])) for r in range(rows.value)]


# ---- synthetic corpora -----------------------------------------------------------------------
def synth_corpus(seed: int, doc_begin: int, doc_end: int, vocab: int, zipf_s: float = 1.1, speaker: int = 0,
                 doc_bytes: int = 1 << 20, threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    n = (doc_end - doc_begin) * doc_bytes
    if out is None:
        out = np.empty(n, dtype=np.uint8)
    assert out.size >= n and out.dtype == np.uint8
    check(lib.wfcu_synth_corpus(seed, doc_begin, doc_end, vocab, zipf_s, speaker, doc_bytes, _ptr(out), threads))
    return out[:n]


def synth_corpus_strided(seed: int, doc_begin: int, doc_stride: int, n_docs: int, vocab: int, zipf_s: float = 1.1,
                         speaker: int = 0, doc_bytes: int = 1 << 20, threads: int = 0,
                         out: np.ndarray | None = None) -> np.ndarray:
    n = n_docs * doc_bytes
    if out is None:
        out = np.empty(n, dtype=np.uint8)
    assert out.size >= n and out.dtype == np.uint8
    check(lib.wfcu_synth_corpus_strided(seed, doc_begin, doc_stride, n_docs, vocab, zipf_s, speaker, doc_bytes,
                                        _ptr(out), threads))
    return out[:n]


def synth_uniform(seed: int, n: int, dtype=np.float64) -> np.ndarray:
    out = np.empty(n, dtype=dtype)
    check(lib.wfcu_synth_uniform(seed, n, _dtype_code(out), _ptr(out)))
    return out
