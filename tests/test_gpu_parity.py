"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and
the reference's golden vectors. Bar: words bit-exact; 1-NN position
identical with ties to the lowest position; distance bit-identical to the
reference's blocked FP64 sum (the north_star tolerance is 1e-5 relative, the
tests hold the stricter bitwise bar and report any miss)."""
import hashlib
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2009_00786_b200 as tg  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def device_words(rows, w, bits=8):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(rows, np.float32)).cuda()
    words, keys = tg.summarise(t, w, bits)
    torch.cuda.synchronize()
    return words.cpu().numpy()[:, :w], keys.cpu().numpy().astype(np.uint32)


def assert_words_equal(got, want):
    mism = int(np.count_nonzero(got != want))
    assert mism == 0, f"{mism} symbol mismatches of {want.size}"


# ---- K1 summarise ----------------------------------------------------------------

def test_summarise_matches_golden(golden, oracle):
    g = golden["load"]("rw600x64.npz")
    for w, b, key in ((16, 8, "words16"), (8, 4, "words8b4"), (4, 8, "words4")):
        words, keys = device_words(g["data"], w, b)
        assert_words_equal(words, g[key])
        assert all(int(keys[i]) == oracle.root_key(g[key][i]) for i in range(0, 600, 37))
    for n in (96, 128):
        h = golden["load"](f"rw400x{n}.npz")
        assert_words_equal(device_words(h["data"], 16)[0], h["words16"])


@pytest.mark.parametrize("count,n,w,bits", [
    (1, 256, 16, 8), (31, 256, 16, 8), (33, 256, 16, 8), (5000, 256, 16, 8), (4099, 128, 16, 8),
    (3001, 96, 16, 8), (2000, 64, 8, 8), (2000, 64, 32, 8), (1500, 64, 16, 3), (1200, 30, 3, 8),
    (1000, 60, 5, 5), (777, 512, 16, 8), (999, 192, 24, 8),
])
def test_summarise_random_shapes(oracle, count, n, w, bits):
    rng = np.random.default_rng(count + n + w)
    rows = np.cumsum(rng.standard_normal((count, n)), axis=1).astype(np.float32)
    rows = (rows - rows.mean(1, keepdims=True)) / (rows.std(1, keepdims=True) + 1e-9)
    rows = rows.astype(np.float32)
    words, keys = device_words(rows, w, bits)
    want = oracle.summarise(rows, w, bits)
    assert_words_equal(words, want)
    for i in range(0, count, max(1, count // 17)):
        assert int(keys[i]) == oracle.root_key(want[i])


def test_summarise_threshold_values_go_up(oracle):
    # every segment mean exactly on a breakpoint (test_sax.cpp:47-63 at the word level)
    thr = oracle.breakpoints(8).astype(np.float32).astype(np.float64)
    rows = np.repeat(thr.astype(np.float32)[:, None], 64, axis=1)  # constant rows -> mean == value
    words, _ = device_words(rows, 16)
    assert_words_equal(words, oracle.summarise(rows, 16))


def test_summarise_config1_sha(oracle, golden):
    """All 16M config-1 symbols vs the reference's c1_sax.u8 digest."""
    data = oracle.generate(1_000_000, 256, 1)
    assert sha(data) == golden["c1"]["data_sha256"]
    words, _ = device_words(data, 16)
    assert sha(words) == golden["c1"]["sax_sha256"]


def test_device_generator_matches_reference(oracle):
    import torch

    for seed, begin, count, n, znorm in ((1, 0, 4000, 256, True), (7, 123456, 2000, 128, True),
                                         (3, 0, 2000, 96, False)):
        dev = tg.generate_random_walk_device(count, n, seed, znorm=znorm, begin=begin).cpu().numpy()
        host = oracle.generate(count, n, seed, znorm=znorm, begin=begin)
        bad_rows = int(np.count_nonzero(np.any(dev.view(np.uint32) != host.view(np.uint32), axis=1)))
        assert bad_rows == 0, f"{bad_rows} of {count} series differ from the reference generator"
        torch.cuda.synchronize()


# ---- build + exact search ----------------------------------------------------------

def check_against_scan(oracle, rows, queries, cfg, expect_bitwise=True, index=None):
    index = index or tg.build_index(rows, cfg)
    res = tg.exact_search_batch(index, queries)
    for k, q in enumerate(queries):
        d, p = oracle.scan_nn(rows, q, 0)
        assert res[k].position == p, (k, res[k].position, p, res[k].distance, d)
        if expect_bitwise:
            assert res[k].distance == d, (k, res[k].distance, d)
        assert res[k].distance == pytest.approx(d, rel=1e-12)
        st = res[k].stats
        assert st.real_dist_calcs <= st.queue_insertions + st.lb_entry_calcs
        assert st.lb_entry_calcs <= len(rows)
        assert st.bsf_updates >= 1
    return index, res


def test_exact_search_matches_golden(golden, oracle):
    g = golden["load"]("rw600x64.npz")
    cfg = tg.IndexConfig(n=64, w=16, leaf_capacity=20, chunk_size=100)
    index = tg.build_index(g["data"], cfg)
    for k, q in enumerate(g["queries"]):
        r = tg.exact_search(index, q)
        assert r.position == int(g["scan"][k, 1]) and r.distance == g["scan"][k, 0]
        # the reference's own exact_search agrees too
        assert r.position == int(g["exact"][k, 1]) and r.distance == pytest.approx(g["exact"][k, 0], rel=1e-9)
        a = tg.approximate_search(index, q)
        assert a.distance >= r.distance


@pytest.mark.parametrize("count,n,w,bits,leaf", [
    (3000, 64, 16, 8, 20), (3000, 64, 16, 8, 2), (3000, 64, 16, 8, 2000), (2500, 64, 8, 4, 7),
    (2000, 96, 16, 8, 50), (2000, 128, 16, 8, 100), (4000, 256, 16, 8, 2000), (1500, 30, 3, 8, 10),
    (1500, 64, 32, 8, 16), (1000, 60, 5, 2, 4), (1200, 512, 16, 8, 40), (800, 1024, 32, 8, 25),
    (900, 200, 8, 8, 30),
])
def test_exact_matches_scan(oracle, count, n, w, bits, leaf):
    rng = np.random.default_rng(count * 7 + n)
    rows = oracle.generate(count, n, 700 + n)
    queries = np.concatenate([oracle.generate(6, n, 900 + n),
                              rows[rng.integers(0, count, 4)] + 0.05 * rng.standard_normal((4, n)).astype(np.float32)])
    cfg = tg.IndexConfig(n=n, w=w, max_card_bits=bits, leaf_capacity=leaf)
    check_against_scan(oracle, rows, queries.astype(np.float32), cfg)


def test_member_queries_return_themselves(oracle):
    rows = oracle.generate(2000, 64, 1001, znorm=False)
    index = tg.build_index(rows, tg.IndexConfig(n=64, w=16, leaf_capacity=20))
    for m in (17, 655, 1999):
        r = tg.exact_search(index, rows[m])
        assert r.distance == 0.0 and r.position == m
        assert tg.approximate_search(index, rows[m]).distance == 0.0


def test_ties_resolve_to_lowest_position(golden):
    g = golden["load"]("ties50x32.npz")
    index = tg.build_index(g["data"], tg.IndexConfig(n=32, w=16, leaf_capacity=4))
    r = tg.exact_search(index, g["query"])
    assert r.distance == 0.0 and r.position == 7


def test_duplicates_overflow_leaves(oracle):
    protos = oracle.generate(10, 256, 20230505, znorm=False)
    rows = np.tile(protos, (1000, 1))  # acceptance.cpp:375-418: 1000 copies of 10 series
    index = tg.build_index(rows, tg.IndexConfig(leaf_capacity=100))
    assert index.build_stats().overflow_leaves > 0
    for p in range(10):
        r = tg.exact_search(index, protos[p])
        assert r.distance == 0.0 and r.position == p


def test_many_exact_ties(oracle):
    """7500 exact duplicates of three series, shuffled: every batch slot's
    finalize must still return the lowest position among thousands of ties."""
    protos = oracle.generate(3, 64, 4242, znorm=False)
    rows = np.concatenate([oracle.generate(1000, 64, 4243, znorm=False), np.tile(protos, (2500, 1))])
    rng = np.random.default_rng(5)
    perm = np.concatenate([np.arange(1000), 1000 + rng.permutation(7500)])
    rows = np.ascontiguousarray(rows[perm])
    index = tg.build_index(rows, tg.IndexConfig(n=64, w=16, leaf_capacity=50))
    for p in range(3):
        want = int(np.flatnonzero((rows == protos[p]).all(axis=1))[0])
        res = tg.exact_search_batch(index, np.stack([protos[p]] * 3))  # several lanes
        for r in res:
            assert r.distance == 0.0 and r.position == want
    # near-ties (one ulp apart in the data) resolve by distance, then position
    check_against_scan(oracle, rows, np.concatenate([protos, protos + np.float32(1e-3)]).astype(np.float32),
                       tg.IndexConfig(n=64, w=16, leaf_capacity=50))


def test_single_series_dataset(oracle):
    rows = oracle.generate(1, 256, 20230506, znorm=False)
    index = tg.build_index(rows, tg.IndexConfig())
    r = tg.exact_search(index, rows[0])
    assert r.distance == 0.0 and r.position == 0


def test_device_rows_build_equals_host_build(oracle):
    import torch

    rows = oracle.generate(5000, 256, 99)
    q = oracle.generate(8, 256, 98)
    a = tg.exact_search_batch(tg.build_index(rows), q)
    t = torch.from_numpy(rows).cuda()
    b = tg.exact_search_batch(tg.build_index(t), torch.from_numpy(q).cuda())
    assert [(x.distance, x.position) for x in a] == [(x.distance, x.position) for x in b]


def test_index_layout_invariants(oracle):
    rows = oracle.generate(20000, 64, 4242)
    cfg = tg.IndexConfig(n=64, w=16, leaf_capacity=50)
    index = tg.build_index(rows, cfg)
    words, pos, off, poff, lo, hi = index.export()
    ref_words = oracle.summarise(rows, 16)
    assert sorted(pos.tolist()) == list(range(20000))
    assert np.array_equal(words[:, :16], ref_words[pos])
    L, P = index.build_stats().leaves, index.build_stats().pages
    assert off[0] == 0 and off[-1] == 20000 and np.all(np.diff(off.astype(np.int64)) > 0) and len(off) == L + 1
    assert poff[0] == 0 and poff[-1] == 20000 and np.all(np.diff(poff.astype(np.int64)) > 0) and len(poff) == P + 1
    assert set(off.tolist()) <= set(poff.tolist())  # pages never straddle leaves
    assert np.all(np.diff(poff.astype(np.int64)) <= 128)
    roots = np.array([oracle.root_key(w) for w in words[:, :16]])
    # plane-major order of the first 48 key bits (root key first; the sorted key width, build.cu kSortBits)
    planes = np.unpackbits(words[:, :16], axis=1).reshape(-1, 16, 8).transpose(0, 2, 1).reshape(-1, 128)[:, :64]
    keys = np.packbits(planes, axis=1).view(">u8").ravel() & np.uint64(0xFFFFFFFFFFFF0000)
    assert np.all(keys[1:] >= keys[:-1])
    for l in range(L):
        a, b = off[l], off[l + 1]
        assert len(set(roots[a:b].tolist())) == 1  # a leaf never straddles root subtrees
        if b - a > 50:
            assert np.all(keys[a:b] == keys[a])  # only identical-key ranges may overflow
    for p in range(P):
        a, b = poff[p], poff[p + 1]
        assert np.array_equal(lo[p, :16], words[a:b, :16].min(0)) and np.array_equal(hi[p, :16], words[a:b, :16].max(0))
        # equal keys keep position order (stable sort), like drain_in_position_order
        same = keys[a:b][1:] == keys[a:b][:-1]
        assert np.all(pos[a:b][1:][same] > pos[a:b][:-1][same])
    assert index.build_stats().root_children == len(set(roots.tolist()))


def test_query_validation():
    rows = np.random.default_rng(0).standard_normal((100, 64)).astype(np.float32)
    index = tg.build_index(rows, tg.IndexConfig(n=64))
    with pytest.raises(tg.InvalidArgument):
        tg.exact_search(index, np.zeros(63, np.float32))
    with pytest.raises(tg.InvalidArgument):
        tg.exact_search(index, np.zeros(64, np.float32), tg.Measure.dtw(64))
    with pytest.raises(tg.InvalidArgument):
        tg.exact_search(index, np.zeros(64, np.float32), tg.Measure.dtw(-1))


def test_build_rejects_bad_inputs():
    cfg = tg.IndexConfig(n=64, w=16, leaf_capacity=20)
    with pytest.raises(tg.InvalidArgument, match="empty dataset"):
        tg.build_index(np.zeros((0, 64), np.float32), cfg)
    with pytest.raises(tg.InvalidArgument, match="does not match config.n"):
        tg.build_index(np.zeros((10, 32), np.float32), cfg)
    bad = tg.IndexConfig(n=64, w=0)
    with pytest.raises(tg.InvalidArgument):
        tg.build_index(np.zeros((10, 64), np.float32), bad)


def test_config1_answers_sha(oracle, golden):
    """100 config-1 queries: answers formatted like the survey's scan oracle
    ("%zu %u %.17g") hash to the reference's c1_answers.txt digest."""
    data = oracle.generate(1_000_000, 256, 1)
    queries = oracle.generate(100, 256, 2)
    assert sha(queries) == golden["c1"]["queries_sha256"]
    index = tg.build_index(data, tg.IndexConfig())
    res = tg.exact_search_batch(index, queries)
    text = "".join("%d %d %.17g\n" % (k, r.position, r.distance) for k, r in enumerate(res))
    assert hashlib.sha256(text.encode()).hexdigest() == golden["c1"]["answers_sha256"], text[:300]
    assert res[0].position == 842660 and res[0].distance == 6.0047035858932869


def test_launch_counter_moves():
    before = tg.launch_count()
    rows = np.random.default_rng(1).standard_normal((500, 64)).astype(np.float32)
    tg.exact_search(tg.build_index(rows, tg.IndexConfig(n=64)), rows[3])
    assert tg.launch_count() > before


# ---- BASELINE configs 3-5: generators and exact search on their distributions ------

def _row_mismatch(a, b):
    return int(np.count_nonzero(np.any(a.view(np.uint32) != b.view(np.uint32), axis=1)))


def test_device_generators_c3_c4_c5_match_oracle(oracle):
    import torch

    c4d = tg.generate_device("c4", 3000, 96, 41, begin=5000).cpu().numpy()
    assert _row_mismatch(c4d, oracle.generate_c4(3000, 96, 41, begin=5000)) == 0
    c5d = tg.generate_device("c5", 200, 256, 77, noise=0.1, data_count=100_000_000, data_seed=1).cpu().numpy()
    c5h, _ = oracle.c5_queries(200, 0.1, 77, 1, 100_000_000, 256)
    assert _row_mismatch(c5d, c5h) == 0
    # c3 evaluates sin(): libdevice vs glibc may differ in the last bit of a few values
    c3d = tg.generate_device("c3", 3000, 128, 31, begin=123).cpu().numpy()
    c3h = oracle.generate_c3(3000, 128, 31, begin=123)
    assert float(np.abs(c3d - c3h).max()) < 1e-4
    assert _row_mismatch(c3d, c3h) <= 30, _row_mismatch(c3d, c3h)
    torch.cuda.synchronize()


@pytest.mark.parametrize("kind,n,leaf", [("c3", 128, 2000), ("c3", 128, 50), ("c4", 96, 2000), ("c4", 96, 64)])
def test_exact_matches_scan_c3_c4(oracle, kind, n, leaf):
    gen = oracle.generate_c3 if kind == "c3" else oracle.generate_c4
    rows = gen(20000, n, 900)
    queries = gen(12, n, 900, begin=10_000_000)  # same process, unseen series
    check_against_scan(oracle, rows, queries, tg.IndexConfig(n=n, leaf_capacity=leaf))


@pytest.mark.parametrize("sigma", [0.01, 0.1, 0.5, 1.0])
def test_exact_matches_scan_c5_noisy_queries(oracle, sigma):
    rows = oracle.generate(30000, 256, 1)  # the first 30000 rows of configs 1/2
    queries, src = oracle.c5_queries(10, sigma, 5, 1, 30000, 256)
    _, res = check_against_scan(oracle, rows, queries, tg.IndexConfig())
    if sigma <= 0.01:  # near-duplicates find their source row
        assert sum(int(r.position) == int(s) for r, s in zip(res, src)) >= 8


@pytest.mark.parametrize("slot_cap,batched", [(64, True), (200, True), (200, False), (600, True)])
def test_slot_overflow_reruns_full_size(oracle, monkeypatch, slot_cap, batched):
    """Queries whose candidates outgrow a batch slot are rerun: together in the batch slots
    re-sliced into fewer, larger slots when those hold the shard at least twice (slot caps 200 and
    600: 128 slots x cap >= 2 x 6000 rows, in chunks when more queries overflow than fit), else
    (cap 64, or TSG_NO_BATCHED_RERUN) alone in a full-size slot."""
    monkeypatch.setenv("TSG_SLOT_CAP", str(slot_cap))  # read when the index is built
    if not batched:
        monkeypatch.setenv("TSG_NO_BATCHED_RERUN", "1")
    rows = oracle.generate(6000, 64, 515)
    cfg = tg.IndexConfig(n=64, w=8, max_card_bits=2, leaf_capacity=20)  # coarse words: many candidates
    index = tg.build_index(rows, cfg)
    queries = np.concatenate([oracle.generate(9, 64, 516), rows[[3, 4000, 5999]] + np.float32(0.3)]).astype(np.float32)
    check_against_scan(oracle, rows, queries, cfg, index=index)


def test_many_batches_one_call(oracle):
    """More queries than batch slots in one call: consecutive batches reuse the slots."""
    rows = oracle.generate(4000, 96, 517)
    rng = np.random.default_rng(3)
    queries = np.concatenate([oracle.generate(150, 96, 518),
                              rows[rng.integers(0, 4000, 150)] + 0.05 * rng.standard_normal((150, 96)).astype(np.float32)])
    cfg = tg.IndexConfig(n=96, w=16, leaf_capacity=50)
    check_against_scan(oracle, rows, queries.astype(np.float32), cfg)


@pytest.mark.parametrize("slots", [1, 3, 320])
def test_batch_widths_stay_exact(oracle, monkeypatch, slots):
    """Query slots from 1 to more than a block has threads (TSG_BATCH): the persistent kernels'
    block-wide query selection strides over the batch, the weighted refinement start falls back
    to the uniform one above 256 queries, and launches with less work than blocks retire their
    surplus blocks (easy member queries next to hard ones)."""
    monkeypatch.setenv("TSG_BATCH", str(slots))
    rows = oracle.generate(6000, 64, 531)
    rng = np.random.default_rng(7)
    queries = np.concatenate([oracle.generate(200, 64, 532), rows[rng.integers(0, 6000, 130)],
                              rows[rng.integers(0, 6000, 20)] + 0.5 * rng.standard_normal((20, 64)).astype(np.float32)])
    cfg = tg.IndexConfig(n=64, w=16, leaf_capacity=40)
    check_against_scan(oracle, rows, queries.astype(np.float32), cfg)


def test_approximate_batch_matches_single(oracle):
    rows = oracle.generate(3000, 128, 519)
    index = tg.build_index(rows, tg.IndexConfig(n=128, w=16, leaf_capacity=30))
    qs = oracle.generate(8, 128, 520)
    for q in qs:
        a = tg.approximate_search(index, q)
        e = tg.exact_search(index, q)
        assert a.distance >= e.distance
        d, p = oracle.scan_nn(rows, q, 0)
        assert e.position == p and e.distance == d


def test_build_from_file_equals_build_from_memory(oracle, tmp_path):
    """load_dataset + build_index streamed from a file (chunks overlapped with K1)
    gives the same index and answers as the in-memory build; several chunks."""
    rows = oracle.generate(600_000, 128, 521)  # ~307 MB: three 128 MB chunks
    path = tmp_path / "c.f32"
    tg.save_dataset(path, rows)
    cfg = tg.IndexConfig(n=128, w=16, leaf_capacity=500)
    a = tg.build_index_from_file(path, cfg)
    b = tg.build_index(rows, cfg)
    ea, eb = a.export(), b.export()
    for x, y in zip(ea, eb):
        assert np.array_equal(x, y)
    assert a.build_stats().leaves == b.build_stats().leaves
    qs = np.concatenate([oracle.generate(6, 128, 522), rows[[5, 599_999]] + np.float32(0.01)]).astype(np.float32)
    ra, rb = tg.exact_search_batch(a, qs), tg.exact_search_batch(b, qs)
    for x, y in zip(ra, rb):
        assert x.position == y.position and x.distance == y.distance
    assert np.array_equal(a.data()[599_999], rows[599_999])


def test_build_from_file_errors(tmp_path):
    bad = tmp_path / "bad.f32"
    bad.write_bytes(b"0123456789")
    with pytest.raises(tg.TsgError, match="10 bytes"):
        tg.build_index_from_file(bad, tg.IndexConfig(n=32, w=16))
    with pytest.raises(tg.TsgError, match="cannot stat"):
        tg.build_index_from_file(tmp_path / "missing.f32", tg.IndexConfig(n=32, w=16))


# ---- DTW: exact search under Measure::dtw(window) ----------------

@pytest.mark.parametrize("count,n,w,leaf,window", [
    (3000, 64, 16, 20, 0), (3000, 64, 16, 20, 6), (2500, 64, 16, 200, 31), (2000, 96, 16, 50, 40),
    (1500, 128, 16, 30, 100), (1200, 60, 5, 10, 12), (1000, 256, 16, 64, 25), (800, 32, 8, 2000, 31),
])
def test_dtw_exact_matches_scan(oracle, count, n, w, leaf, window):
    rng = np.random.default_rng(count + n + window)
    rows = oracle.generate(count, n, 800 + n)
    queries = np.concatenate([oracle.generate(4, n, 900 + n + window),
                              rows[rng.integers(0, count, 3)] + 0.1 * rng.standard_normal((3, n)).astype(np.float32)])
    index = tg.build_index(rows, tg.IndexConfig(n=n, w=w, leaf_capacity=leaf))
    res = tg.exact_search_batch(index, queries.astype(np.float32), tg.Measure.dtw(window))
    for k, q in enumerate(queries.astype(np.float32)):
        d, p = oracle.scan_nn_dtw(rows, q, window)
        assert res[k].position == p, (k, res[k].position, p, res[k].distance, d)
        assert res[k].distance == d, (k, res[k].distance, d)
        one = tg.exact_search(index, q, tg.Measure.dtw(window))
        assert one.position == p and one.distance == d
        a = tg.approximate_search(index, q, tg.Measure.dtw(window))
        assert a.distance >= d


def test_dtw_members_and_limits(oracle):
    rows = oracle.generate(1500, 64, 1301, znorm=False)
    index = tg.build_index(rows, tg.IndexConfig(n=64, w=16, leaf_capacity=20))
    for m in (3, 777, 1499):
        r = tg.exact_search(index, rows[m], tg.Measure.dtw(5))
        assert r.distance == 0.0 and r.position == m
    big = tg.build_index(oracle.generate(300, 512, 1302), tg.IndexConfig(n=512, w=16))
    with pytest.raises(tg.InvalidArgument):
        tg.exact_search(big, np.zeros(512, np.float32), tg.Measure.dtw(256))  # above the device band limit


# ---- fine summary (second lower bound in front of refinement) ------------------

def fine_symbols_reference(rows, fw):
    """Uniform quantisation of the half-segment means (sequential FP64 sums) over [-2.5, 2.5)."""
    count, n = rows.shape
    h = n // fw
    x = rows.astype(np.float64).reshape(count, fw, h)
    s = np.zeros((count, fw))
    for j in range(h):
        s = s + x[:, :, j]
    m = s / h
    return np.clip(np.floor((m + 2.5) * 51.2), 0, 255).astype(np.int32), m


@pytest.mark.parametrize("count,n,w,bits", [(3000, 256, 16, 8), (2000, 128, 16, 8), (2000, 96, 16, 8),
                                            (1500, 64, 8, 4), (1200, 60, 5, 8), (1000, 128, 32, 8)])
def test_fine_summary_quantises_half_segment_means(oracle, count, n, w, bits):
    """Fine summary = the 2w half-segment means quantised in 5/256 steps (boundary cases counted)."""
    rows = oracle.generate(count, n, 31 * n + w)
    index = tg.build_index(rows, tg.IndexConfig(n=n, w=w, max_card_bits=bits, leaf_capacity=50))
    fine = index.export_fine()
    if n % (2 * w) or 2 * w > 64:
        assert fine is None
        return
    want, m = fine_symbols_reference(rows, 2 * w)
    assert fine.shape == want.shape
    diff = fine.astype(np.int32) - want
    bad = diff != 0
    # only float rounding at a region boundary may move a symbol, by one
    assert np.all(np.abs(diff) <= 1)
    edge = np.abs((m + 2.5) * 51.2 - np.round((m + 2.5) * 51.2)) < 1e-3
    assert np.all(edge[bad]), int(np.count_nonzero(bad & ~edge))


def test_fine_summary_prunes_refinement_without_changing_answers(oracle, monkeypatch):
    rows = oracle.generate(40000, 256, 1)
    rng = np.random.default_rng(11)
    queries = np.concatenate([oracle.generate(12, 256, 2),
                              rows[rng.integers(0, 40000, 4)] + 0.2 * rng.standard_normal((4, 256)).astype(np.float32),
                              rows[[5, 17]]]).astype(np.float32)
    cfg = tg.IndexConfig(n=256, w=16, leaf_capacity=200)
    _, with_fine = check_against_scan(oracle, rows, queries, cfg)
    monkeypatch.setenv("TSG_NO_FINE", "1")  # read when the index is built
    index = tg.build_index(rows, cfg)
    assert index.export_fine() is None
    _, without = check_against_scan(oracle, rows, queries, cfg, index=index)
    for a, b in zip(with_fine, without):
        assert (a.position, a.distance) == (b.position, b.distance)
        assert b.fine_calcs == 0
    assert sum(r.fine_calcs for r in with_fine) > 0
    assert sum(r.stats.real_dist_calcs for r in with_fine) < sum(r.stats.real_dist_calcs for r in without)


def test_fine_summary_saturating_values_stay_exact(oracle):
    """Rows far outside the fine quantiser's [-2.5, 2.5) range (scaled, shifted, constant) keep exact answers."""
    rng = np.random.default_rng(77)
    base = oracle.generate(6000, 256, 91)
    rows = np.concatenate([base[:2000] * np.float32(1000.0),          # saturating both ends
                           base[2000:4000] + np.float32(40.0),        # all in the top open region
                           np.repeat(rng.standard_normal((40, 1)).astype(np.float32), 256, axis=1),  # constant rows
                           base[4040:]]).astype(np.float32)
    queries = np.concatenate([rows[[5, 2500, 4010, 5000]] + np.float32(0.01),
                              oracle.generate(4, 256, 92) * np.float32(1000.0),
                              oracle.generate(4, 256, 93)]).astype(np.float32)
    _, res = check_against_scan(oracle, rows, queries, tg.IndexConfig(n=256, w=16, leaf_capacity=100))
    assert sum(r.fine_calcs for r in res) > 0


def test_batch_records_equal_batch_results(oracle):
    """exact_search_batch_records (record array over the C ABI results) == exact_search_batch."""
    import torch

    rows = oracle.generate(5000, 128, 61)
    queries = oracle.generate(20, 128, 62)
    index = tg.build_index(rows, tg.IndexConfig(n=128, leaf_capacity=100))
    want = tg.exact_search_batch(index, queries)
    for q in (queries, torch.from_numpy(queries).cuda()):
        got = tg.exact_search_batch_records(index, q)
        assert got.dtype == tg.RESULT_DTYPE and len(got) == len(want)
        for g, w in zip(got, want):
            assert (float(g["distance"]), int(g["position"])) == (w.distance, w.position)
            assert int(g["stats"][2]) == w.stats.real_dist_calcs and int(g["fine_calcs"]) == w.fine_calcs


def _torch_bruteforce_nn(rows, q, chunk=1 << 20):
    """Independent exhaustive 1-NN in torch (FP64 squared distances, chunked): (distance, lowest position)."""
    import torch

    qd = q.double()
    best_d, best_p = float("inf"), -1
    for a in range(0, rows.shape[0], chunk):
        d = ((rows[a:a + chunk].double() - qd) ** 2).sum(dim=1)
        v, i = torch.min(d, dim=0)
        v = float(v)
        if v < best_d:  # strict: an earlier chunk keeps equal distances (lowest position)
            best_d, best_p = v, a + int(i)
    return math.sqrt(best_d), best_p


def test_exact_at_scale_matches_bruteforce():
    """25M-series prefix of config 2 (25.6 GB in HBM): answers equal an independent exhaustive scan."""
    import torch

    N, n = 25_000_000, 256
    rows = tg.generate_device("rw", N, n, 1)
    queries = torch.cat([tg.generate_device("rw", 6, n, 2, begin=N), rows[[123_456, N - 7]] + 0.001])
    index = tg.build_index(rows, tg.IndexConfig(n=n))
    res = tg.exact_search_batch(index, queries)
    for k in range(queries.shape[0]):
        d, p = _torch_bruteforce_nn(rows, queries[k])
        assert res[k].position == p, (k, res[k].position, p)
        assert res[k].distance == pytest.approx(d, rel=1e-12)
    assert sum(r.stats.real_dist_calcs for r in res) < 0.001 * N * len(res)  # the index pruned >99.9%
    del index, rows
    torch.cuda.empty_cache()


@pytest.mark.gpu
def test_graph_replays_with_new_query_buffers(oracle):
    """The batch pipeline runs as a cached CUDA graph keyed by batch shape, not by the query
    pointer: replays with other device query buffers (same batch size, and a batch-size
    change in between) must still answer each buffer's own queries exactly."""
    import torch

    rows = oracle.generate(5000, 128, 611)
    index = tg.build_index(rows, tg.IndexConfig(n=128, w=16, leaf_capacity=40))
    rng = np.random.default_rng(612)
    for it, nq in enumerate([7, 7, 3, 7, 1, 7]):
        qs = oracle.generate(nq, 128, 700 + it)
        if it % 2:  # member-derived queries in every other buffer
            qs = (rows[rng.integers(0, 5000, nq)] + 0.02 * rng.standard_normal((nq, 128))).astype(np.float32)
        dq = torch.from_numpy(np.ascontiguousarray(qs)).cuda()
        res = tg.exact_search_batch(index, dq)
        del dq  # the next buffer may land elsewhere (or at the same address with other contents)
        for k, q in enumerate(qs):
            d, p = oracle.scan_nn(rows, q, 0)
            assert res[k].position == p and res[k].distance == d, (it, k, res[k], d, p)


def test_headline_config_answers_equal_reference_golden():
    """north_star's target on the headline config (BASELINE configs[1]): exact 1-NN answers of the 100
    BASELINE queries over 100M x 256 z-normalised random walks equal the reference's exhaustive
    answers (tests/golden/c2_answers.txt: the unmodified reference's scan_nn over all 100M series,
    oracle/make_c2_golden.py) - identical positions, bit-identical distances, same digest."""
    import json
    import os

    import torch

    gdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    meta = json.load(open(os.path.join(gdir, "c2_golden.json")))
    golden = open(os.path.join(gdir, "c2_answers.txt")).read()
    N, n = meta["count"], meta["n"]
    free, _ = torch.cuda.mem_get_info()
    if free < 150e9:
        pytest.skip("needs ~150 GB of free HBM")
    rows = tg.generate_device("rw", N, n, 1)  # device generator = the reference's bytes (tested above)
    queries = tg.generate_device("rw", 100, n, 2)
    index = tg.build_index(rows, tg.IndexConfig(n=n))
    for host in (False, True):
        res = tg.exact_search_batch_records(index, queries.cpu().numpy() if host else queries)
        text = "".join("%d %d %.17g\n" % (k, int(r["position"]), float(r["distance"])) for k, r in enumerate(res))
        assert hashlib.sha256(text.encode()).hexdigest() == meta["answers_sha256"]
        assert text == golden
    # and the 100M-series index passes the full audit (chunked re-derivation of every word)
    r = tg.validate_index(index)
    assert r.ok(), r.violations
    assert r.total_entries == N
    index.free()
    del rows
    torch.cuda.empty_cache()


def test_uploaded_thresholds_equal_reference_bitwise(golden, oracle):
    """the threshold table in HBM that K1 and the query kernels read is the
    reference's breakpoints_for(2^bits) bit for bit (tests/golden/breakpoints.npz), for every
    cardinality."""
    g = golden["load"]("breakpoints.npz")
    rows = oracle.generate(500, 64, 5)
    for bits in range(1, 9):
        index = tg.build_index(rows, tg.IndexConfig(n=64, w=8, max_card_bits=bits, leaf_capacity=20))
        got = index.thresholds()
        k = (1 << bits) - 1
        assert np.array_equal(got[:k].view(np.uint64), g[f"bits{bits}"].view(np.uint64)), bits
        assert np.all(np.isposinf(got[k:])), bits
        index.free()


def test_file_built_index_answers_equal_scan(oracle, tmp_path):
    """Ingestion parity (load_dataset + build_index, src/dataset.cpp:87-117, src/index.cpp:258-318):
    an index streamed from a headerless float32 file answers exactly like scan_nn over the file's
    rows, across several streaming chunks."""
    n = 256
    rows = oracle.generate(200_000, n, 91)  # 205 MB: two ~128 MB chunks
    rows[150_000] = rows[10]  # a duplicate: the lower position wins
    path = tmp_path / "rows.f32"
    tg.save_dataset(path, rows)
    queries = np.concatenate([oracle.generate(6, n, 92), rows[[10, 199_999, 130_000]]])
    index = tg.build_index_from_file(path, tg.IndexConfig(n=n))
    assert index.build_stats().series == rows.shape[0]
    for k, r in enumerate(tg.exact_search_batch(index, queries)):
        d, p = oracle.scan_nn(rows, queries[k], 0)
        assert (r.position, r.distance) == (p, d), k
    index.free()


def test_device_inputs_are_checked(oracle):
    """CUDA-tensor inputs must be float32, 2-D and on the index's device (read by the library on its
    own stream after torch's current stream is synchronised): anything else fails loudly instead of
    being reinterpreted."""
    import torch

    rows = oracle.generate(2000, 64, 3)
    index = tg.build_index(rows, tg.IndexConfig(n=64, leaf_capacity=50))
    q = torch.from_numpy(oracle.generate(3, 64, 4)).cuda()
    with pytest.raises(tg.InvalidArgument, match="float32"):
        tg.exact_search_batch(index, q.double())
    with pytest.raises(tg.InvalidArgument, match="float32"):
        tg.exact_search_batch_records(index, q.half())
    with pytest.raises(tg.InvalidArgument, match="float32"):
        tg.build_index(torch.from_numpy(rows).cuda().double(), tg.IndexConfig(n=64))
    # a non-contiguous view (every other row) is copied on torch's stream and still answers exactly
    view = torch.cat([q, q], dim=0)[::2]
    assert not view.is_contiguous()
    res = tg.exact_search_batch(index, view)
    for k, r in enumerate(res):
        d, p = oracle.scan_nn(rows, view[k].cpu().numpy(), 0)
        assert (r.position, r.distance) == (p, d)
    index.free()
