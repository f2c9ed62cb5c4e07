"""validate_index on the device (reference src/index.cpp:332-484,
include/tsidx/index.hpp:180-202): the audit passes on every index the library
builds, its counts agree with the build, and each kind of corruption of the
flat index (injected through the tsg_index_debug_poke test hook) is caught
with the reference's style of message."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2009_00786_b200 as tg  # noqa: E402


def build(oracle, count=6000, n=64, w=16, bits=8, leaf=64, seed=11, rows=None):
    rows = oracle.generate(count, n, seed) if rows is None else rows
    return tg.build_index(rows, tg.IndexConfig(n=n, w=w, max_card_bits=bits, leaf_capacity=leaf)), rows


@pytest.mark.parametrize("count,n,w,bits,leaf", [(6000, 64, 16, 8, 64), (20000, 256, 16, 8, 2000), (3000, 96, 8, 4, 16),
                                                 (5000, 128, 32, 8, 40), (700, 30, 3, 5, 2)])
def test_audit_passes_and_matches_build(oracle, count, n, w, bits, leaf):
    index, _ = build(oracle, count, n, w, bits, leaf)
    r = tg.validate_index(index)
    bs = index.build_stats()
    assert r.ok(), r.violations
    assert r.total_entries == count
    assert (r.leaves, r.inner_nodes, r.nodes, r.overflow_leaves, r.max_depth) == \
        (bs.leaves, bs.inner_nodes, bs.nodes, bs.overflow_leaves, bs.max_depth)
    assert sum(r.leaf_fill_histogram) == r.leaves
    assert r.leaf_fill_histogram[10] == r.overflow_leaves
    assert r.pages == bs.pages and r.checked_boxes > r.pages
    assert "violations=0" in r.summary()


def test_audit_overflow_leaves_are_legal(oracle):
    rows = oracle.generate(400, 64, 3)
    rows = np.concatenate([rows, np.repeat(rows[:1], 300, axis=0)])  # 301 identical series: unsplittable
    index, _ = build(oracle, rows=rows, leaf=20)
    r = tg.validate_index(index)
    assert r.ok(), r.violations
    assert r.overflow_leaves >= 1


def test_audit_local_shards(oracle):
    rows = oracle.generate(9000, 64, 5)
    ctx = tg.Context((0, 0, 0))
    index = tg.build_index(rows, tg.IndexConfig(n=64, leaf_capacity=50), context=ctx)
    r = tg.validate_index(index)
    assert r.ok(), r.violations
    assert r.total_entries == 9000 and r.leaves == index.build_stats().leaves
    index.free()
    ctx.close()


def _corrupt(oracle, array, offset, data):
    index, _ = build(oracle)
    index.debug_poke(array, offset, data)
    r = tg.validate_index(index)
    assert not r.ok()
    return r


def test_audit_catches_a_changed_word(oracle):
    r = _corrupt(oracle, 0, 16 * 5 + 3, bytes([0x55]))
    assert any("stored word differs from the recomputed word" in v for v in r.violations), r.violations


def test_audit_catches_a_duplicated_position(oracle):
    index, _ = build(oracle)
    _, pos, _, _, _, _ = index.export()
    index.debug_poke(1, 4 * 3, np.uint32(pos[4]).tobytes())  # entry 3 now claims entry 4's series
    r = tg.validate_index(index)
    assert any(f"position {pos[4]} stored twice" in v for v in r.violations), r.violations
    assert any(f"position {pos[3]} missing from every leaf" in v for v in r.violations), r.violations


def test_audit_catches_a_broken_leaf(oracle):
    index, _ = build(oracle)
    _, _, leaf_off, _, _, _ = index.export()
    index.debug_poke(2, 4 * 1, np.uint32(leaf_off[2]).tobytes())  # leaf 0 swallows leaf 1, leaf 1 is empty
    r = tg.validate_index(index)
    assert any("offsets do not tile" in v for v in r.violations), r.violations


def test_audit_catches_box_corruption(oracle):
    r = _corrupt(oracle, 3, 16 * 2 + 1, bytes([0xFF]))  # a page min above its words
    assert any("page 2: box is not the min / max" in v for v in r.violations), r.violations
    r = _corrupt(oracle, 4, 32 * 7 + 0, bytes([0xFF]))  # quad boxes are (min, max) pairs
    assert any("quad 7: box is not the min / max" in v for v in r.violations), r.violations
    r = _corrupt(oracle, 6, 32 * 1 + 9, bytes([0x00]))
    assert any("run 1: box is not the min / max" in v for v in r.violations), r.violations
    r = _corrupt(oracle, 7, 16 * 0 + 4, bytes([0xFF]))
    assert any("not contained in its parent" in v for v in r.violations), r.violations


def test_audit_catches_fine_summary_corruption(oracle):
    index, _ = build(oracle)
    fine = index.export_fine()
    assert fine is not None
    index.debug_poke(5, 32 * 10 + 7, bytes([(int(fine[0, 0]) + 1) % 256]))
    r = tg.validate_index(index)
    assert any("fine summary differs" in v for v in r.violations), r.violations


def test_debug_poke_bounds(oracle):
    index, _ = build(oracle)
    with pytest.raises(tg.InvalidArgument, match="out of range"):
        index.debug_poke(0, 16 * 6000, b"\0")
    with pytest.raises(tg.InvalidArgument, match="unknown array"):
        index.debug_poke(42, 0, b"\0")
