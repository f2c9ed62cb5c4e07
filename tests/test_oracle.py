"""Pins the CPU oracle (oracle/tsidx_oracle.cpp) before it is trusted:
against the reference's golden vectors (tests/golden, produced by the
unmodified reference) and, when oracle/_ref is built, against the reference
itself. The known-answer tests restate the reference's own unit tests
(paths relative to /root/reference/proj/tests)."""
import math

import numpy as np
import pytest


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64 if a.dtype == np.float64 else np.uint32)


# ---- breakpoints: test_breakpoints.cpp ---------------------------------------

def test_breakpoints_match_golden_bitwise(oracle, golden):
    g = golden["load"]("breakpoints.npz")
    for b in range(1, 9):
        assert np.array_equal(bits(oracle.breakpoints(b)), bits(g[f"bits{b}"])), b


def test_quartiles_and_card8_outer(oracle):
    thr = oracle.breakpoints(2)  # test_breakpoints.cpp:23-29
    assert thr[0] == pytest.approx(-0.6745, rel=1e-4) and thr[2] == pytest.approx(0.6745, rel=1e-4)
    assert abs(thr[1]) < 1e-12
    thr8 = oracle.breakpoints(3)  # :31-37
    assert thr8[0] == pytest.approx(-1.1503, rel=1e-4) and thr8[6] == pytest.approx(1.1503, rel=1e-4)


def test_quantile_property_sorted_symmetric(oracle):
    for b in range(1, 9):  # :39-52
        c = 1 << b
        thr = oracle.breakpoints(b)
        cdf = np.array([oracle.lib.orc_normal_cdf(t) for t in thr])
        assert np.allclose(cdf, np.arange(1, c) / c, rtol=1e-6)
        assert np.all(np.diff(thr) > 0)
        assert np.array_equal(thr, -thr[::-1])


# ---- summarisation: test_sax.cpp ----------------------------------------------

def test_paa_example(oracle):
    assert np.allclose(oracle.paa(np.array([0, 2, 4, 6], np.float32), 2), [1.0, 5.0])  # :33-45


def test_symbol_boundary_convention(oracle):
    for b in (1, 2, 4, 8):  # :47-63: a value on a threshold takes the upper region
        thr = oracle.breakpoints(b)
        for i, t in enumerate(thr):
            assert oracle.symbol(b, t) == i + 1
    assert oracle.symbol(2, 0.0) == 2 and oracle.symbol(2, -1.0) == 0 and oracle.symbol(2, 0.1) == 2


def test_zeros_map_to_middle_and_left_alignment(oracle):
    w = oracle.summarise(np.zeros((1, 256), np.float32), 16, 8)  # :65-73
    assert np.all(w == 128)
    w4 = oracle.summarise(np.zeros((1, 16), np.float32), 4, 4)  # :75-81
    assert np.all(w4 == 0x80)


def test_root_key_msb_first(oracle):
    assert oracle.root_key(np.array([0x80, 0x00, 0xFF, 0x00], np.uint8)) == 0b1010  # :83-94
    assert oracle.root_key(np.array([0xFF] * 4, np.uint8)) == 15
    assert oracle.root_key(np.zeros(4, np.uint8)) == 0


def test_words_match_golden(oracle, golden):
    g = golden["load"]("rw600x64.npz")
    assert np.array_equal(oracle.summarise(g["data"], 16, 8), g["words16"])
    assert np.array_equal(oracle.summarise(g["data"], 8, 4), g["words8b4"])
    assert np.array_equal(oracle.summarise(g["data"], 4, 8), g["words4"])
    for n in (96, 128):
        h = golden["load"](f"rw400x{n}.npz")
        assert np.array_equal(oracle.summarise(h["data"], 16, 8), h["words16"])


# ---- generator: test_data.cpp + Appendix B ---------------------------------------

def test_generator_matches_golden_and_prefix_property(oracle, golden):
    import hashlib

    raw = oracle.generate(600, 64, 11, znorm=False)
    assert hashlib.sha256(raw.tobytes()).hexdigest() == golden["rw600x64"]["raw_sha256"]
    g = golden["load"]("rw600x64.npz")
    assert np.array_equal(bits(oracle.generate(600, 64, 11)), bits(g["data"]))
    assert np.array_equal(bits(oracle.generate(12, 64, 12)), bits(g["queries"]))
    # series i depends only on (seed, i): a window regenerates identically
    assert np.array_equal(bits(oracle.generate(100, 64, 11, begin=250)), bits(g["data"][250:350]))
    c1p = oracle.generate(1000, 256, 1)
    assert hashlib.sha256(c1p.tobytes()).hexdigest() == golden["c1_prefix1000_sha256"]
    assert hashlib.sha256(oracle.summarise(c1p, 16).tobytes()).hexdigest() == golden["c1_prefix1000_sax_sha256"]


def test_znormalize_flags_constant_series(oracle):
    flat = np.full(16, 3.25, np.float32)  # test_data.cpp znormalize cases
    assert not oracle.znormalize(flat) and np.all(flat == 3.25)
    v = np.array([0.0, 2.0], np.float32)
    assert oracle.znormalize(v) and np.allclose(v, [-1, 1])


# ---- metrics: test_metrics.cpp ---------------------------------------------------

def test_euclidean_basics_and_abandonment(oracle):
    a, b = np.zeros(4, np.float32), np.ones(4, np.float32)
    assert oracle.euclidean(a, b) == pytest.approx(2.0)  # :43-50
    assert oracle.euclidean(a, b, 1.5) == math.inf  # :52-57
    assert oracle.euclidean(a, b, 2.0) == pytest.approx(2.0)  # equal sum survives


def test_abandoning_equals_plain_bitwise(oracle):
    rng = np.random.default_rng(3)  # :59-70
    for _ in range(200):
        a = np.cumsum(rng.standard_normal(96)).astype(np.float32)
        b = np.cumsum(rng.standard_normal(96)).astype(np.float32)
        full = oracle.euclidean(a, b)
        assert oracle.euclidean(a, b, full + 1.0) == full
        assert oracle.euclidean(a, b, full * 0.5) == math.inf
        plain = math.sqrt(float(np.sum((a.astype(np.float64) - b.astype(np.float64)) ** 2)))
        assert full == pytest.approx(plain, rel=1e-12)


def test_mindist_example_and_soundness(oracle):
    # n=4, w=2, query means -1 vs upper-half words -> 2 (:72-79)
    assert oracle.mindist(np.array([-1.0, -1.0]), np.array([0x80, 0x80], np.uint8),
                          np.array([1, 1], np.uint8), 4) == pytest.approx(2.0)
    rng = np.random.default_rng(17)  # :88-104, LB <= ED + 1e-9
    for _ in range(500):
        q = np.cumsum(rng.standard_normal(64)).astype(np.float32)
        s = np.cumsum(rng.standard_normal(64)).astype(np.float32)
        word = oracle.summarise(s[None], 8)[0]
        cb = np.full(8, 8, np.uint8)
        assert oracle.mindist(oracle.paa(q, 8), word, cb, 64) <= oracle.euclidean(q, s) + 1e-9


# ---- scan: test_scan.cpp -----------------------------------------------------------

def test_scan_matches_golden_and_is_thread_invariant(oracle, golden):
    g = golden["load"]("rw600x64.npz")
    for k, q in enumerate(g["queries"]):
        d, p = oracle.scan_nn(g["data"], q, 1)
        assert p == int(g["scan"][k, 1]) and d == g["scan"][k, 0]
        for t in (2, 5):
            assert oracle.scan_nn(g["data"], q, t) == (d, p)


def test_scan_ties_lowest_position(oracle, golden):
    g = golden["load"]("ties50x32.npz")
    for t in (1, 4):
        d, p = oracle.scan_nn(g["data"], g["query"], t)
        assert d == 0.0 and p == 7


# ---- live comparison against the reference (oracle/_ref) ---------------------------

def test_oracle_equals_reference_random(oracle, reference):
    rng = np.random.default_rng(5)
    for n, w, b in ((64, 16, 8), (96, 16, 8), (60, 5, 3), (30, 3, 8)):
        rows = rng.standard_normal((300, n)).astype(np.float32) * rng.uniform(0.1, 3)
        assert np.array_equal(oracle.summarise(rows, w, b), reference.summarise(rows, w, b))
        q = rows[17] + rng.standard_normal(n).astype(np.float32) * 0.1
        assert oracle.scan_nn(rows, q, 3) == reference.scan_nn(rows, q, 3)
        assert oracle.euclidean(rows[0], rows[1]) == reference.euclidean(rows[0], rows[1])
        qp = oracle.paa(q, w)
        assert np.array_equal(qp, reference.paa(q, w))
        cb = np.full(w, b, np.uint8)
        word = oracle.summarise(rows[3:4], w, b)[0]
        assert oracle.mindist(qp, word, cb, n) == reference.mindist(qp, word, cb, n)


# ---- DTW: the restatement against the compiled reference ----

def test_dtw_matches_reference(oracle, reference):
    rng = np.random.default_rng(11)
    for n, r in ((8, 0), (8, 1), (16, 3), (64, 6), (96, 95), (128, 12), (33, 5)):
        for trial in range(6):
            a = np.cumsum(rng.standard_normal(n)).astype(np.float32)
            b = np.cumsum(rng.standard_normal(n)).astype(np.float32)
            want = reference.dtw(a, b, r)
            assert oracle.dtw(a, b, r) == want
            assert oracle.dtw(b, a, r) == want  # symmetric, bit for bit
            assert reference.dtw(b, a, r) == want
            cut = want * (0.7 + 0.6 * (trial % 2))
            assert oracle.dtw(a, b, r, cut) == reference.dtw(a, b, r, cut)
    a = rng.standard_normal(40).astype(np.float32)
    assert oracle.dtw(a, a, 4) == 0.0
    # window 0 is the Euclidean distance summed sequentially
    b = rng.standard_normal(40).astype(np.float32)
    assert oracle.dtw(a, b, 0) == pytest.approx(np.sqrt(((a.astype(np.float64) - b) ** 2).sum()), rel=1e-15)


def test_envelope_bounds_match_reference(oracle, reference):
    rng = np.random.default_rng(12)
    for n, r, w in ((64, 6, 16), (96, 10, 16), (128, 0, 8), (256, 25, 16), (60, 59, 5)):
        q = np.cumsum(rng.standard_normal(n)).astype(np.float32)
        mine, theirs = oracle.keogh_envelope(q, r, w), reference.keogh_envelope(q, r, w)
        for x, y in zip(mine, theirs):
            assert np.array_equal(x, y)
        c = np.cumsum(rng.standard_normal(n)).astype(np.float32)
        assert oracle.lb_keogh(q, r, c) == reference.lb_keogh(q, r, c)
        sym = oracle.summarise(c[None, :], w)[0]
        assert oracle.mindist_envelope(q, r, w, sym) == reference.mindist_envelope(q, r, w, sym)
        # soundness: both bounds are below the DTW distance
        d = oracle.dtw(q, c, r)
        assert oracle.lb_keogh(q, r, c) <= d + 1e-9 and oracle.mindist_envelope(q, r, w, sym) <= d + 1e-9


def test_scan_nn_dtw_matches_reference(oracle, reference):
    rows = oracle.generate(400, 64, 31)
    qs = oracle.generate(4, 64, 32)
    for r in (0, 3, 12):
        for q in qs:
            assert oracle.scan_nn_dtw(rows, q, r, threads=3) == reference.scan_nn_dtw(rows, q, r, threads=5)
    # the reference index agrees on the answer
    idx = reference.build_index(rows, w=16, leaf_capacity=20)
    for q in qs:
        d, p = idx.exact_search_dtw(q, 6)
        dd, pp = oracle.scan_nn_dtw(rows, q, 6)
        assert p == pp and d == pytest.approx(dd, rel=1e-12)
