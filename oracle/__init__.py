"""Python view of the CPU checkers -- TEST INFRASTRUCTURE ONLY.

`oracle.port()`  loads oracle/liboracle.so   (our plain-C restatement, wfc_oracle.c)
`oracle.ref()`   loads oracle/_ref/libwfc_ref.so (the unmodified reference, compiled
                 by oracle/Makefile from /root/reference/proj/src; prebuilt on the GPU box)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  Both libraries expose the same C shapes (prefix wfo_ /
wfr_), wrapped here by one class.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libwfc_ref.so"

u64p = C.POINTER(C.c_uint64)


class _Decoded(C.Structure):
    _fields_ = [("cp", C.c_uint32), ("len", C.c_uint32), ("valid", C.c_int32)]


def build(quiet: bool = True) -> None:
    """make liboracle.so and, when /root/reference is present, _ref/libwfc_ref.so."""
    subprocess.run(["make", "-C", str(HERE), "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data if a.size else 0)


def _bytes(b) -> np.ndarray:
    if isinstance(b, np.ndarray):
        return np.ascontiguousarray(b, dtype=np.uint8)
    return np.frombuffer(bytes(b), dtype=np.uint8)


def pack_words(words):
    lens = np.fromiter((len(w) for w in words), dtype=np.uint32, count=len(words))
    blob = np.frombuffer(b"".join(words), dtype=np.uint8).copy() if len(words) else np.zeros(0, np.uint8)
    return blob, lens


def unpack_words(blob: np.ndarray, lens: np.ndarray):
    raw = blob.tobytes()
    out, off = [], 0
    for n in lens.tolist():
        out.append(raw[off:off + n])
        off += n
    return out


class CpuLib:
    """One of the two CPU implementations behind a common Python API."""

    def __init__(self, path: Path, prefix: str, kind: str):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.kind = kind            # "port" | "reference"
        self.prefix = prefix
        self.lib = C.CDLL(str(path))
        f = self._fn
        f("utf8_decode", _Decoded, [C.c_void_p, C.c_uint64, C.c_uint64])
        f("is_space", C.c_int, [C.c_uint32])
        f("is_word_char", C.c_int, [C.c_uint32])
        f("simple_lower", C.c_uint32, [C.c_uint32])
        f("utf8_valid", C.c_int, [C.c_void_p, C.c_uint64])
        f("utf8_sanitize", C.c_uint64, [C.c_void_p, C.c_uint64, C.c_void_p])
        f("normalize_word", C.c_uint64, [C.c_void_p, C.c_uint64, C.c_void_p])
        f("tokenize", C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, u64p, u64p])
        f("counts_new", C.c_void_p, [])
        f("counts_free", None, [C.c_void_p])
        f("counts_add_document", None, [C.c_void_p, C.c_void_p, C.c_uint64])
        f("counts_distinct", C.c_uint64, [C.c_void_p])
        f("counts_total", C.c_uint64, [C.c_void_p])
        f("counts_key_bytes", C.c_uint64, [C.c_void_p])
        f("counts_export", None, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p])
        f("counts_merge", None, [C.c_void_p, C.c_void_p])
        f("sort_words", None, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p])
        f("reduce_sorted", C.c_uint64, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p])
        f("plan_partition", C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p])
        f("map_reduce_serial_f64", C.c_double, [C.c_void_p, C.c_uint64, C.c_int])
        f("top_k", C.c_uint64, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, u64p])
        f("distinctive", C.c_uint64, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                      C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p])
        if kind == "port":
            f("map_reduce_serial_f32", C.c_double, [C.c_void_p, C.c_uint64, C.c_int])
            f("map_reduce_blocked_f64", C.c_double, [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.POINTER(C.c_int)])
            f("map_reduce_blocked_f32", C.c_double, [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.POINTER(C.c_int)])
            f("alternating_harmonic", C.c_double, [C.c_uint64, C.c_uint64, C.POINTER(C.c_int)])
            f("counts_add", None, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64])
        else:
            f("map_reduce_blocked_f64", C.c_double, [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_uint, C.POINTER(C.c_int)])
            f("alternating_harmonic", C.c_double, [C.c_uint64, C.c_uint64, C.c_uint, C.POINTER(C.c_int)])
            f("serial_wordcount", C.c_void_p, [C.c_void_p, C.c_void_p, C.c_uint64])
            f("fill_uniform", None, [C.c_uint64, C.c_void_p, C.c_uint64])
            f("run_wordcount", C.c_void_p, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_char_p, C.c_uint64])

    def _fn(self, name, res, args):
        fn = getattr(self.lib, self.prefix + name)
        fn.restype = res
        fn.argtypes = args
        setattr(self, "_" + name, fn)

    # ---- unicode / text ----
    def utf8_decode(self, data: bytes, pos: int):
        a = _bytes(data)
        d = self._utf8_decode(_ptr(a), a.size, pos)
        return d.cp, d.len, bool(d.valid)

    def is_space(self, cp): return bool(self._is_space(cp))
    def is_word_char(self, cp): return bool(self._is_word_char(cp))
    def simple_lower(self, cp): return int(self._simple_lower(cp))

    def utf8_valid(self, data: bytes) -> bool:
        a = _bytes(data)
        return bool(self._utf8_valid(_ptr(a), a.size))

    def utf8_sanitize(self, data: bytes) -> bytes:
        a = _bytes(data)
        out = np.zeros(3 * a.size + 4, np.uint8)
        n = self._utf8_sanitize(_ptr(a), a.size, _ptr(out))
        return out[:n].tobytes()

    def normalize_word(self, frag: bytes):
        a = _bytes(frag)
        out = np.zeros(3 * a.size + 4, np.uint8)
        n = self._normalize_word(_ptr(a), a.size, _ptr(out))
        return out[:n].tobytes() if n else None

    def tokenize_packed(self, text) -> tuple[np.ndarray, np.ndarray]:
        a = _bytes(text)
        nt, nb = C.c_uint64(), C.c_uint64()
        blob = np.zeros(a.size + 16, np.uint8)
        lens = np.zeros(a.size // 2 + 2, np.uint32)
        rc = self._tokenize(_ptr(a), a.size, _ptr(blob), blob.size, _ptr(lens), lens.size, C.byref(nt), C.byref(nb))
        if rc:   # invalid bytes expand 1 -> 3
            blob = np.zeros(nb.value + 16, np.uint8)
            lens = np.zeros(nt.value + 2, np.uint32)
            rc = self._tokenize(_ptr(a), a.size, _ptr(blob), blob.size, _ptr(lens), lens.size, C.byref(nt), C.byref(nb))
            assert rc == 0
        return blob[:nb.value], lens[:nt.value]

    def tokenize(self, text) -> list[bytes]:
        return unpack_words(*self.tokenize_packed(text))

    # ---- counting map ----
    def wordcount_packed(self, docs) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """serial_wordcount over documents -> (key_bytes, key_lens, counts) in std::map order."""
        h = self._counts_new()
        try:
            for d in docs:
                a = _bytes(d)
                self._counts_add_document(h, _ptr(a), a.size)
            return self._export(h)
        finally:
            self._counts_free(h)

    def _export(self, h):
        n = self._counts_distinct(h)
        nb = self._counts_key_bytes(h)
        blob = np.zeros(max(nb, 1), np.uint8)
        lens = np.zeros(max(n, 1), np.uint32)
        counts = np.zeros(max(n, 1), np.uint64)
        self._counts_export(h, _ptr(blob), _ptr(lens), _ptr(counts))
        return blob[:nb], lens[:n], counts[:n]

    def wordcount(self, docs) -> dict[bytes, int]:
        blob, lens, counts = self.wordcount_packed(docs)
        return dict(zip(unpack_words(blob, lens), (int(c) for c in counts)))

    def run_wordcount(self, docs, n_workers: int):
        """reference only: wfc::run_wordcount -> (dict, timings_ns[7])."""
        assert self.kind == "reference"
        arrs = [_bytes(d) for d in docs]
        ptrs = (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])
        lens = (C.c_uint64 * max(len(arrs), 1))(*[a.size for a in arrs])
        tim = (C.c_uint64 * 7)()
        err = C.create_string_buffer(512)
        h = self._run_wordcount(ptrs, lens, len(arrs), n_workers, tim, err, 512)
        if not h:
            raise RuntimeError(err.value.decode())
        try:
            blob, kl, counts = self._export(h)
        finally:
            self._counts_free(h)
        return dict(zip(unpack_words(blob, kl), (int(c) for c in counts))), list(tim)

    # ---- sort + RLE ----
    def sort_words(self, words):
        blob, lens = pack_words(words)
        ob, ol = np.zeros_like(blob), np.zeros_like(lens)
        self._sort_words(_ptr(blob), _ptr(lens), len(words), _ptr(ob), _ptr(ol))
        return unpack_words(ob, ol)

    def reduce_sorted(self, words):
        """-> list of (word, count) or None when the list is not sorted."""
        blob, lens = pack_words(words)
        first = np.zeros(max(len(words), 1), np.uint64)
        cnt = np.zeros(max(len(words), 1), np.uint64)
        r = self._reduce_sorted(_ptr(blob), _ptr(lens), len(words), _ptr(first), _ptr(cnt))
        if r == 2**64 - 1:
            return None
        return [(words[int(first[i])], int(cnt[i])) for i in range(r)]

    def plan_partition(self, k, worker_id, n_workers):
        b = np.zeros(n_workers + 1, np.uint64)
        rc = self._plan_partition(k, worker_id, n_workers, _ptr(b))
        return None if rc else [int(x) for x in b]

    # ---- engine ----
    def map_reduce_serial(self, values: np.ndarray, kind: int) -> float:
        values = np.ascontiguousarray(values)
        if values.dtype == np.float32:
            if self.kind == "port":
                return float(self._map_reduce_serial_f32(_ptr(values), values.size, kind))
            values = values.astype(np.float64)
        return float(self._map_reduce_serial_f64(_ptr(values), values.size, kind))

    def map_reduce_blocked(self, values: np.ndarray, kind: int, block: int, workers: int = 1):
        """-> value, or None when the configuration is rejected."""
        values = np.ascontiguousarray(values)
        err = C.c_int(0)
        if self.kind == "port":
            fn = self._map_reduce_blocked_f32 if values.dtype == np.float32 else self._map_reduce_blocked_f64
            v = fn(_ptr(values), values.size, kind, block, C.byref(err))
        else:
            values = values.astype(np.float64)
            v = self._map_reduce_blocked_f64(_ptr(values), values.size, kind, block, workers, C.byref(err))
        return None if err.value else float(v)

    def alternating_harmonic(self, n: int, block: int = 256, workers: int = 1):
        err = C.c_int(0)
        if self.kind == "port":
            v = self._alternating_harmonic(n, block, C.byref(err))
        else:
            v = self._alternating_harmonic(n, block, workers, C.byref(err))
        return None if err.value else float(v)

    def fill_uniform(self, seed: int, n: int) -> np.ndarray:
        assert self.kind == "reference"
        out = np.empty(n, np.float64)
        self._fill_uniform(seed, _ptr(out), n)
        return out

    # ---- analysis ----
    def top_k(self, table: dict[bytes, int], k: int):
        words = sorted(table)
        blob, lens = pack_words(words)
        counts = np.array([table[w] for w in words], dtype=np.uint64)
        idx = np.zeros(max(len(words), 1), np.uint64)
        rel = np.zeros(max(len(words), 1), np.float64)
        total = C.c_uint64()
        m = self._top_k(_ptr(blob), _ptr(lens), _ptr(counts), len(words), k, _ptr(idx), _ptr(rel), C.byref(total))
        return [(words[int(idx[i])], int(counts[int(idx[i])]), float(rel[i])) for i in range(m)], total.value

    def distinctive(self, target: dict[bytes, int], others: dict[bytes, int], k: int):
        tw, ow = sorted(target), sorted(others)
        tb, tl = pack_words(tw)
        ob, ol = pack_words(ow)
        tc = np.array([target[w] for w in tw], dtype=np.uint64)
        oc = np.array([others[w] for w in ow], dtype=np.uint64)
        cap = max(len(tw) + len(ow), 1)
        src = np.zeros(cap, np.int32)
        idx = np.zeros(cap, np.uint64)
        score = np.zeros(cap, np.float64)
        m = self._distinctive(_ptr(tb), _ptr(tl), _ptr(tc), len(tw), _ptr(ob), _ptr(ol), _ptr(oc), len(ow),
                              k, _ptr(src), _ptr(idx), _ptr(score))
        return [((ow if src[i] else tw)[int(idx[i])], float(score[i])) for i in range(m)]


_cache: dict[str, CpuLib] = {}
SYNTH_LIB = HERE / "libwfsynth.so"


def _synth():
    if "synth" not in _cache:
        if not SYNTH_LIB.exists():
            build()
        lib = C.CDLL(str(SYNTH_LIB))
        lib.wfs_corpus_strided.restype = C.c_int
        lib.wfs_corpus_strided.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_double,
                                           C.c_uint32, C.c_uint64, C.c_void_p, C.c_int]
        lib.wfs_uniform.restype = C.c_int
        lib.wfs_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_void_p]
        _cache["synth"] = lib
    return _cache["synth"]


def synth_corpus(seed: int, doc_begin: int, n_docs: int, vocab: int, zipf_s: float = 1.1, speaker: int = 0,
                 doc_bytes: int = 1 << 20, doc_stride: int = 1) -> np.ndarray:
    """The bench corpus (documents doc_begin, doc_begin + stride, ...) without the CUDA library in the process."""
    out = np.empty(n_docs * doc_bytes, np.uint8)
    rc = _synth().wfs_corpus_strided(seed, doc_begin, doc_stride, n_docs, vocab, zipf_s, speaker, doc_bytes, _ptr(out), 0)
    assert rc == 0
    return out


def synth_uniform(seed: int, n: int, dtype=np.float64) -> np.ndarray:
    """mt19937_64(seed) + uniform(0,1), the reference bench's input recipe (proj/src/cli.cpp:120-125)."""
    out = np.empty(n, dtype)
    rc = _synth().wfs_uniform(seed, n, 1 if out.dtype == np.float64 else 0, _ptr(out))
    assert rc == 0
    return out


def port() -> CpuLib:
    if "port" not in _cache:
        if not PORT_LIB.exists():
            build()
        _cache["port"] = CpuLib(PORT_LIB, "wfo_", "port")
    return _cache["port"]


def ref_available() -> bool:
    return REF_LIB.exists()


def ref() -> CpuLib:
    if "ref" not in _cache:
        _cache["ref"] = CpuLib(REF_LIB, "wfr_", "reference")
    return _cache["ref"]
