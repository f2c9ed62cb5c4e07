"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU oracle libraries.

* ``Oracle``    — my restatement (``oracle/liboracle.so``, built from
  ``oracle/tsidx_oracle.cpp``).
* ``Reference`` — the unmodified reference core compiled in place
  (``oracle/_ref/libtsidx_ref.so``, built by ``oracle/Makefile``).

Only ``tests/``, ``bench.py`` (cpu_baseline / ``--impl reference``) and
``__graft_entry__.smoke()`` import this module, and only as the checker or
the timed CPU baseline. The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtsidx_ref.so")
REF_CORE = "/root/reference/proj/core"

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u64, u32, i32, f64 = C.c_uint64, C.c_uint32, C.c_int, C.c_double


def build(ref: bool | None = None) -> None:
    """Compile the oracle (and, when /root/reference is present, oracle/_ref)."""
    targets = ["liboracle.so"]
    if ref or (ref is None and os.path.isdir(REF_CORE)):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _sig(lib, name, res, *args):
    fn = getattr(lib, name)
    fn.restype = res
    fn.argtypes = list(args)
    return fn


class Oracle:
    """My restatement of the reference hot path (see tsidx_oracle.cpp)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        lib = C.CDLL(path)
        self.lib = lib
        _sig(lib, "orc_breakpoints", i32, i32, _f64p)
        _sig(lib, "orc_inverse_normal_cdf", f64, f64)
        _sig(lib, "orc_normal_cdf", f64, f64)
        _sig(lib, "orc_mix_seed", u64, u64, u64)
        _sig(lib, "orc_random_walk_series", None, u64, u64, u64, _f32p)
        _sig(lib, "orc_znormalize", i32, _f32p, u64)
        _sig(lib, "orc_generate_rows", None, u64, u64, u64, u64, i32, C.c_uint, _f32p)
        _sig(lib, "orc_generate_kind", None, i32, u64, u64, u64, u64, C.c_uint, _f32p)
        _sig(lib, "orc_c5_query", None, u64, u64, f64, u64, u64, u64, _f32p, C.POINTER(u64))
        _sig(lib, "orc_paa", None, _f32p, u64, i32, _f64p)
        _sig(lib, "orc_summarise", None, _f32p, u64, u64, i32, i32, C.c_uint, _u8p)
        _sig(lib, "orc_root_key", u64, _u8p, i32)
        _sig(lib, "orc_symbol", C.c_uint, _f64p, C.c_uint, f64)
        _sig(lib, "orc_mindist_paa_isax", f64, _f64p, _u8p, _u8p, i32, u64)
        _sig(lib, "orc_euclidean", f64, _f32p, _f32p, u64, f64)
        _sig(lib, "orc_squared_l2", f64, _f32p, _f32p, u64, f64)
        _sig(lib, "orc_scan_nn", None, _f32p, u64, u64, _f32p, C.c_uint, C.POINTER(f64), C.POINTER(u32))
        _sig(lib, "orc_cmin", u64, _u8p, u64, i32, i32, u64, _f64p, f64)
        _sig(lib, "orc_keogh_envelope", None, _f32p, u64, i32, i32, _f32p, _f32p, _f64p, _f64p)
        _sig(lib, "orc_lb_keogh", f64, _f32p, _f32p, _f32p, u64)
        _sig(lib, "orc_mindist_envelope_isax", f64, _f64p, _f64p, _u8p, _u8p, i32, u64)
        _sig(lib, "orc_dtw", f64, _f32p, _f32p, u64, i32, f64)
        _sig(lib, "orc_scan_nn_dtw", None, _f32p, u64, u64, _f32p, i32, C.c_uint, C.POINTER(f64), C.POINTER(u32))

    def breakpoints(self, bits: int) -> np.ndarray:
        out = np.empty((1 << bits) - 1, np.float64)
        assert self.lib.orc_breakpoints(bits, out) == 0
        return out

    def generate(self, count, length, seed, znorm=True, begin=0, threads=0) -> np.ndarray:
        out = np.empty((count, length), np.float32)
        self.lib.orc_generate_rows(seed, begin, begin + count, length, 1 if znorm else 0, threads, out)
        return out

    def generate_c3(self, count, length, seed, begin=0, threads=0) -> np.ndarray:
        """BASELINE config 3: AR(1) + random-phase sinusoid, z-normalised."""
        out = np.empty((count, length), np.float32)
        self.lib.orc_generate_kind(3, seed, begin, count, length, threads, out)
        return out

    def generate_c4(self, count, length, seed, begin=0, threads=0) -> np.ndarray:
        """BASELINE config 4: 1024-component Gaussian mixture, z-normalised."""
        out = np.empty((count, length), np.float32)
        self.lib.orc_generate_kind(4, seed, begin, count, length, threads, out)
        return out

    def c5_queries(self, nq, sigma, query_seed, data_seed, count, length, begin=0):
        """BASELINE config 5: dataset rows (regenerated) + N(0, sigma^2), re-z-normalised."""
        out = np.empty((nq, length), np.float32)
        rows = np.empty(nq, np.uint64)
        for j in range(nq):
            r = u64()
            self.lib.orc_c5_query(query_seed, begin + j, sigma, data_seed, count, length, out[j], C.byref(r))
            rows[j] = r.value
        return out, rows

    def znormalize(self, s: np.ndarray) -> bool:
        return bool(self.lib.orc_znormalize(s, s.size))

    def paa(self, s: np.ndarray, w: int) -> np.ndarray:
        s = np.ascontiguousarray(s, np.float32)
        out = np.empty(w, np.float64)
        self.lib.orc_paa(s, s.size, w, out)
        return out

    def summarise(self, rows: np.ndarray, w: int, bits: int = 8, threads: int = 0) -> np.ndarray:
        rows = np.ascontiguousarray(rows, np.float32)
        count, n = rows.shape
        out = np.empty((count, w), np.uint8)
        self.lib.orc_summarise(rows, count, n, w, bits, threads, out)
        return out

    def symbol(self, bits: int, v: float) -> int:
        thr = self.breakpoints(bits)
        return int(self.lib.orc_symbol(thr, 1 << bits, v))

    def root_key(self, sym: np.ndarray) -> int:
        sym = np.ascontiguousarray(sym, np.uint8)
        return int(self.lib.orc_root_key(sym, sym.size))

    def mindist(self, qpaa, sym, card_bits, n) -> float:
        sym = np.ascontiguousarray(sym, np.uint8)
        cb = np.ascontiguousarray(card_bits, np.uint8)
        return self.lib.orc_mindist_paa_isax(np.ascontiguousarray(qpaa, np.float64), sym, cb, sym.size, n)

    def euclidean(self, a, b, cutoff=-1.0) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.orc_euclidean(a, b, a.size, cutoff)

    def squared_l2(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.orc_squared_l2(a, b, a.size, -1.0)

    def scan_nn(self, rows: np.ndarray, q: np.ndarray, threads: int = 0):
        rows = np.ascontiguousarray(rows, np.float32)
        q = np.ascontiguousarray(q, np.float32)
        d, p = f64(), u32()
        self.lib.orc_scan_nn(rows, rows.shape[0], rows.shape[1], q, threads, C.byref(d), C.byref(p))
        return d.value, p.value

    # ---- DTW ----
    def keogh_envelope(self, q, window: int, w: int):
        q = np.ascontiguousarray(q, np.float32)
        n = q.size
        up, lo = np.empty(n, np.float32), np.empty(n, np.float32)
        upaa, lpaa = np.empty(w, np.float64), np.empty(w, np.float64)
        self.lib.orc_keogh_envelope(q, n, window, w, up, lo, upaa, lpaa)
        return up, lo, upaa, lpaa

    def lb_keogh(self, q, window: int, c) -> float:
        up, lo, _, _ = self.keogh_envelope(q, window, 1)
        return self.lib.orc_lb_keogh(up, lo, np.ascontiguousarray(c, np.float32), up.size)

    def mindist_envelope(self, q, window: int, w: int, sym, bits: int = 8) -> float:
        _, _, upaa, lpaa = self.keogh_envelope(q, window, w)
        sym = np.ascontiguousarray(sym, np.uint8)
        cb = np.full(w, bits, np.uint8)
        return self.lib.orc_mindist_envelope_isax(lpaa, upaa, sym, cb, w, np.asarray(q).size)

    def dtw(self, a, b, window: int, cutoff: float = -1.0) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.lib.orc_dtw(a, b, a.size, window, cutoff)

    def scan_nn_dtw(self, rows, q, window: int, threads: int = 0):
        rows = np.ascontiguousarray(rows, np.float32)
        q = np.ascontiguousarray(q, np.float32)
        d, p = f64(), u32()
        self.lib.orc_scan_nn_dtw(rows, rows.shape[0], rows.shape[1], q, window, threads, C.byref(d), C.byref(p))
        return d.value, p.value

    def cmin(self, words: np.ndarray, qpaa: np.ndarray, n: int, d_nn: float, bits: int = 8) -> int:
        words = np.ascontiguousarray(words, np.uint8)
        return int(self.lib.orc_cmin(words, words.shape[0], words.shape[1], bits, n,
                                     np.ascontiguousarray(qpaa, np.float64), d_nn))


class RefError(Exception):
    pass


class Reference:
    """The unmodified reference core (oracle/_ref), driven through ref_capi.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            if os.path.isdir(REF_CORE):
                build(ref=True)
            else:
                raise FileNotFoundError(f"{path} missing and no reference sources to build it")
        lib = C.CDLL(path)
        self.lib = lib
        _sig(lib, "ref_last_error", C.c_char_p)
        _sig(lib, "ref_hardware_concurrency", C.c_uint)
        _sig(lib, "ref_generate_random_walk", i32, u64, u64, u64, _f32p)
        _sig(lib, "ref_znormalize", i32, _f32p, u64)
        _sig(lib, "ref_znormalize_rows", i32, _f32p, u64, u64, C.c_uint, C.POINTER(u64))
        _sig(lib, "ref_breakpoints", i32, C.c_uint, _f64p)
        _sig(lib, "ref_inverse_normal_cdf", f64, f64)
        _sig(lib, "ref_normal_cdf", f64, f64)
        _sig(lib, "ref_paa", i32, _f32p, u64, i32, _f64p)
        _sig(lib, "ref_symbol_for_value", C.c_uint, f64, C.c_uint)
        _sig(lib, "ref_summarise", i32, _f32p, u64, u64, i32, i32, C.c_uint, _u8p)
        _sig(lib, "ref_root_key", u64, _u8p, i32)
        _sig(lib, "ref_mindist_paa_isax", i32, _f64p, _u8p, _u8p, i32, u64, C.POINTER(f64))
        _sig(lib, "ref_euclidean", i32, _f32p, _f32p, u64, f64, C.POINTER(f64))
        _sig(lib, "ref_dataset_new", C.c_void_p, _f32p, u64, u64)
        _sig(lib, "ref_dataset_free", None, C.c_void_p)
        _sig(lib, "ref_scan_nn", i32, C.c_void_p, _f32p, C.c_uint, C.POINTER(f64), C.POINTER(u32))
        _sig(lib, "ref_build_index", i32, _f32p, u64, u64, i32, i32, u64, u64, C.c_uint,
             C.POINTER(C.c_void_p), _u64p)
        _sig(lib, "ref_index_free", None, C.c_void_p)
        _sig(lib, "ref_exact_search", i32, C.c_void_p, _f32p, C.c_uint, C.c_uint, i32,
             C.POINTER(f64), C.POINTER(u32), _u64p, C.POINTER(u64))
        _sig(lib, "ref_approximate_search", i32, C.c_void_p, _f32p, C.POINTER(f64), C.POINTER(u32))
        _sig(lib, "ref_build_generated", i32, u64, u64, u64, i32, i32, i32, u64, u64, C.c_uint,
             C.POINTER(C.c_void_p), _u64p, C.POINTER(u64))
        _sig(lib, "ref_series_window", i32, u64, u64, u64, u64, i32, _f32p)
        _sig(lib, "ref_dtw", i32, _f32p, _f32p, u64, i32, f64, C.POINTER(f64))
        _sig(lib, "ref_keogh_envelope", i32, _f32p, u64, i32, i32, _f32p, _f32p, _f64p, _f64p)
        _sig(lib, "ref_lb_keogh", i32, _f32p, u64, i32, i32, _f32p, C.POINTER(f64))
        _sig(lib, "ref_mindist_envelope_isax", i32, _f32p, u64, i32, i32, _u8p, i32, C.POINTER(f64))
        _sig(lib, "ref_scan_nn_dtw", i32, C.c_void_p, _f32p, i32, C.c_uint, C.POINTER(f64), C.POINTER(u32))
        _sig(lib, "ref_exact_search_dtw", i32, C.c_void_p, _f32p, i32, C.POINTER(f64), C.POINTER(u32))

    def build_generated(self, count, n, seed, znorm=True, w=16, bits=8, leaf_capacity=2000, chunk=20000,
                        workers=0):
        """generate_random_walk + z-norm + build_index inside the reference, no host copy."""
        h = C.c_void_p()
        st = np.zeros(8, np.uint64)
        gen_ns = u64()
        self._check(self.lib.ref_build_generated(count, n, seed, 1 if znorm else 0, w, bits, leaf_capacity, chunk,
                                                 workers, C.byref(h), st, C.byref(gen_ns)))
        return RefIndex.adopt(self, h, n, st), gen_ns.value

    def series_window(self, begin, count, n, seed, znorm=True) -> np.ndarray:
        out = np.empty((count, n), np.float32)
        self._check(self.lib.ref_series_window(begin, count, n, seed, 1 if znorm else 0, out))
        return out

    def _check(self, rc):
        if rc != 0:
            raise RefError(f"reference rc={rc}: {self.lib.ref_last_error().decode()}")

    def hardware_concurrency(self) -> int:
        return int(self.lib.ref_hardware_concurrency())

    def generate_random_walk(self, count, length, seed) -> np.ndarray:
        out = np.empty((count, length), np.float32)
        self._check(self.lib.ref_generate_random_walk(count, length, seed, out))
        return out

    def znormalize_rows(self, rows: np.ndarray, threads: int = 0) -> int:
        deg = u64()
        self._check(self.lib.ref_znormalize_rows(rows, rows.shape[0], rows.shape[1], threads, C.byref(deg)))
        return deg.value

    def breakpoints(self, card: int) -> np.ndarray:
        out = np.empty(card - 1, np.float64)
        self._check(self.lib.ref_breakpoints(card, out))
        return out

    def paa(self, s, w) -> np.ndarray:
        s = np.ascontiguousarray(s, np.float32)
        out = np.empty(w, np.float64)
        self._check(self.lib.ref_paa(s, s.size, w, out))
        return out

    def summarise(self, rows, w, bits=8, threads=0) -> np.ndarray:
        rows = np.ascontiguousarray(rows, np.float32)
        out = np.empty((rows.shape[0], w), np.uint8)
        self._check(self.lib.ref_summarise(rows, rows.shape[0], rows.shape[1], w, bits, threads, out))
        return out

    def mindist(self, qpaa, sym, card_bits, n) -> float:
        sym = np.ascontiguousarray(sym, np.uint8)
        out = f64()
        self._check(self.lib.ref_mindist_paa_isax(np.ascontiguousarray(qpaa, np.float64), sym,
                                                  np.ascontiguousarray(card_bits, np.uint8),
                                                  sym.size, n, C.byref(out)))
        return out.value

    def euclidean(self, a, b, cutoff=-1.0) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = f64()
        self._check(self.lib.ref_euclidean(a, b, a.size, cutoff, C.byref(out)))
        return out.value

    def scan_nn(self, rows, q, threads=0):
        rows = np.ascontiguousarray(rows, np.float32)
        h = self.lib.ref_dataset_new(rows, rows.shape[0], rows.shape[1])
        try:
            d, p = f64(), u32()
            self._check(self.lib.ref_scan_nn(h, np.ascontiguousarray(q, np.float32), threads,
                                             C.byref(d), C.byref(p)))
            return d.value, p.value
        finally:
            self.lib.ref_dataset_free(h)

    # ---- DTW ----
    def dtw(self, a, b, window: int, cutoff: float = -1.0) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = f64()
        self._check(self.lib.ref_dtw(a, b, a.size, window, cutoff, C.byref(out)))
        return out.value

    def keogh_envelope(self, q, window: int, w: int):
        q = np.ascontiguousarray(q, np.float32)
        n = q.size
        up, lo = np.empty(n, np.float32), np.empty(n, np.float32)
        upaa, lpaa = np.empty(w, np.float64), np.empty(w, np.float64)
        self._check(self.lib.ref_keogh_envelope(q, n, window, w, up, lo, upaa, lpaa))
        return up, lo, upaa, lpaa

    def lb_keogh(self, q, window: int, c) -> float:
        q = np.ascontiguousarray(q, np.float32)
        out = f64()
        self._check(self.lib.ref_lb_keogh(q, q.size, window, 1, np.ascontiguousarray(c, np.float32), C.byref(out)))
        return out.value

    def mindist_envelope(self, q, window: int, w: int, sym, bits: int = 8) -> float:
        q = np.ascontiguousarray(q, np.float32)
        out = f64()
        self._check(self.lib.ref_mindist_envelope_isax(q, q.size, window, w, np.ascontiguousarray(sym, np.uint8),
                                                       bits, C.byref(out)))
        return out.value

    def scan_nn_dtw(self, rows, q, window: int, threads: int = 0):
        rows = np.ascontiguousarray(rows, np.float32)
        h = self.lib.ref_dataset_new(rows, rows.shape[0], rows.shape[1])
        try:
            d, p = f64(), u32()
            self._check(self.lib.ref_scan_nn_dtw(h, np.ascontiguousarray(q, np.float32), window, threads,
                                                 C.byref(d), C.byref(p)))
            return d.value, p.value
        finally:
            self.lib.ref_dataset_free(h)

    def dataset(self, rows):
        return RefDataset(self, rows)

    def build_index(self, rows, w=16, bits=8, leaf_capacity=2000, chunk=20000, workers=0):
        return RefIndex(self, rows, w, bits, leaf_capacity, chunk, workers)


class RefDataset:
    def __init__(self, ref: Reference, rows):
        rows = np.ascontiguousarray(rows, np.float32)
        self.ref, self.n = ref, rows.shape[1]
        self.h = ref.lib.ref_dataset_new(rows, rows.shape[0], rows.shape[1])

    def scan_nn(self, q, threads=0):
        d, p = f64(), u32()
        self.ref._check(self.ref.lib.ref_scan_nn(self.h, np.ascontiguousarray(q, np.float32), threads,
                                                 C.byref(d), C.byref(p)))
        return d.value, p.value

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_dataset_free(self.h)
            self.h = None


BUILD_STAT_FIELDS = ("build_ns", "series", "nodes", "inner_nodes", "leaves", "empty_leaves",
                     "overflow_leaves", "max_depth")
SEARCH_STAT_FIELDS = ("lb_node_calcs", "lb_entry_calcs", "real_dist_calcs", "bsf_updates",
                      "pruned_subtrees", "queue_insertions")


class RefIndex:
    def __init__(self, ref: Reference, rows, w, bits, leaf_capacity, chunk, workers):
        rows = np.ascontiguousarray(rows, np.float32)
        self.ref, self.n = ref, rows.shape[1]
        h = C.c_void_p()
        st = np.zeros(8, np.uint64)
        ref._check(ref.lib.ref_build_index(rows, rows.shape[0], rows.shape[1], w, bits,
                                           leaf_capacity, chunk, workers, C.byref(h), st))
        self.h = h
        self.build_stats = dict(zip(BUILD_STAT_FIELDS, map(int, st)))

    @classmethod
    def adopt(cls, ref: Reference, h, n, st):
        self = cls.__new__(cls)
        self.ref, self.n, self.h = ref, n, h
        self.build_stats = dict(zip(BUILD_STAT_FIELDS, map(int, st)))
        return self

    def exact_search(self, q, workers=0, queues=0, mode=-1):
        d, p, ns = f64(), u32(), u64()
        st = np.zeros(6, np.uint64)
        self.ref._check(self.ref.lib.ref_exact_search(self.h, np.ascontiguousarray(q, np.float32),
                                                      workers, queues, mode, C.byref(d), C.byref(p),
                                                      st, C.byref(ns)))
        return d.value, p.value, dict(zip(SEARCH_STAT_FIELDS, map(int, st))), ns.value

    def exact_search_dtw(self, q, window: int):
        d, p = f64(), u32()
        self.ref._check(self.ref.lib.ref_exact_search_dtw(self.h, np.ascontiguousarray(q, np.float32), window,
                                                          C.byref(d), C.byref(p)))
        return d.value, p.value

    def approximate_search(self, q):
        d, p = f64(), u32()
        self.ref._check(self.ref.lib.ref_approximate_search(self.h, np.ascontiguousarray(q, np.float32),
                                                            C.byref(d), C.byref(p)))
        return d.value, p.value

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_index_free(self.h)
            self.h = None
