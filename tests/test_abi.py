"""CPU-side checks of the C ABI boundary: the library loads, exports every
symbol include/tsgpu.h declares, validates IndexConfig exactly like the
reference (src/config.cpp:22-35), and fails loudly (no CPU fallback) when
there is no GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2009_00786_b200 import _lib
from paper_2009_00786_b200.tsidx import IndexConfig, InvalidArgument

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tsgpu.h")).read()
    return sorted(set(re.findall(r"\b(tsg_[a-z_]+)\s*\(", src)))


def test_header_declarations_match_binding_table():
    assert sorted(_lib.EXPORTS) == declared_symbols()


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_defaults_mirror_index_config():
    c = _lib.tsg_config()
    _lib.lib().tsg_config_default(C.byref(c))
    d = IndexConfig()
    assert (c.n, c.w, c.max_card_bits, c.leaf_capacity, c.chunk_size, c.n_queues, c.queue_mode,
            c.initial_buffer_part_size) == (d.n, d.w, d.max_card_bits, d.leaf_capacity, d.chunk_size, d.n_queues,
                                            int(d.queue_mode), d.initial_buffer_part_size)


@pytest.mark.parametrize("field,value,msg", [
    ("w", 0, "w must be at least 1"),
    ("w", 65, "w must be at most 64"),
    ("max_card_bits", 0, "max_card_bits must be in [1, 8]"),
    ("max_card_bits", 9, "max_card_bits must be in [1, 8]"),
    ("n", 8, "n must be at least w"),
    ("n", 250, "must be a multiple of w"),
    ("leaf_capacity", 1, "leaf_capacity must be at least 2"),
    ("chunk_size", 0, "chunk_size must be at least 1"),
    ("n_queues", 0, "n_queues must be at least 1"),
    ("initial_buffer_part_size", 0, "initial_buffer_part_size must be at least 1"),
])
def test_config_validation_messages(field, value, msg):
    cfg = IndexConfig()
    setattr(cfg, field, value)
    with pytest.raises(InvalidArgument, match=re.escape(msg)):
        cfg.validate()


def test_valid_config_passes():
    IndexConfig().validate()
    IndexConfig(n=64, w=8, max_card_bits=4, leaf_capacity=2).validate()


def test_device_path_limit_on_w():
    with pytest.raises(InvalidArgument, match="at most 32 on the device path"):
        IndexConfig(n=40 * 4, w=40).validate()


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") is None and os.path.exists("/dev/nvidia0"),
                    reason="a GPU is present")
def test_no_gpu_fails_loudly():
    h = C.c_void_p()
    st = _lib.lib().tsg_open(1, None, C.byref(h))
    if st == _lib.TSG_OK:
        pytest.skip("a GPU is visible")
    assert st == _lib.TSG_CUDA
    assert "no CUDA device" in _lib.lib().tsg_last_error().decode()


def test_dataset_file_roundtrip_and_errors(tmp_path):
    """load_dataset / save_dataset with the reference's checks (test_data.cpp:94-113)."""
    import paper_2009_00786_b200 as tg

    rows = np.random.default_rng(0).standard_normal((7, 33)).astype(np.float32)
    path = tmp_path / "ds.f32"
    tg.save_dataset(path, rows)
    back = tg.load_dataset(path, 33)
    assert back.shape == (7, 33) and np.array_equal(back.view(np.uint32), rows.view(np.uint32))
    bad = tmp_path / "bad.f32"
    bad.write_bytes(b"0123456789")
    with pytest.raises(tg.TsgError, match="10 bytes"):
        tg.load_dataset(bad, 33)
    with pytest.raises(tg.TsgError):
        tg.load_dataset(tmp_path / "missing.f32", 8)
    with pytest.raises(tg.InvalidArgument, match="length must be positive"):
        tg.load_dataset(path, 0)


def test_ctypes_structs_match_the_c_header(tmp_path):
    """The Python binding's struct layouts equal the C compiler's (sizes and field offsets)."""
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no C compiler")
    structs = {"tsg_config": _lib.tsg_config, "tsg_build_stats": _lib.tsg_build_stats,
               "tsg_search_stats": _lib.tsg_search_stats, "tsg_result": _lib.tsg_result,
               "tsg_comm_id": _lib.tsg_comm_id}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "tsgpu.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([gcc, "-std=c99", "-I", os.path.join(root, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == C.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)


def test_result_record_dtype_matches_the_c_struct():
    """The record-array view of batch results (exact_search_batch_records) has tsg_result's layout."""
    from paper_2009_00786_b200.tsidx import RESULT_DTYPE

    assert RESULT_DTYPE.itemsize == C.sizeof(_lib.tsg_result)
    for name in ("distance", "position", "box_calcs", "stats", "fine_calcs"):
        assert RESULT_DTYPE.fields[name][1] == getattr(_lib.tsg_result, name).offset, name
    rec = np.zeros(2, RESULT_DTYPE)
    raw = (_lib.tsg_result * 2)()
    raw[1].distance, raw[1].position, raw[1].fine_calcs = 2.5, 7, 9
    raw[1].stats.real_dist_calcs = 3
    C.memmove(rec.ctypes.data, raw, C.sizeof(raw))
    assert (rec[1]["distance"], rec[1]["position"], rec[1]["fine_calcs"], rec[1]["stats"][2]) == (2.5, 7, 9, 3)


def test_nccl_unique_id_without_a_gpu():
    """The multi-process communicator id comes from NCCL, loaded at run time (no GPU needed)."""
    import torch  # noqa: F401  (the process's NCCL: torch's bundled libnccl.so.2)

    a, b = _lib.tsg_comm_id(), _lib.tsg_comm_id()
    _lib.check(_lib.lib().tsg_comm_unique_id(C.byref(a)))
    _lib.check(_lib.lib().tsg_comm_unique_id(C.byref(b)))
    assert bytes(a.internal) != bytes(b.internal)
    assert any(bytes(a.internal))


def test_comm_init_needs_a_context():
    cid = _lib.tsg_comm_id()
    st = _lib.lib().tsg_comm_init(None, 2, 0, C.byref(cid))
    assert st == _lib.TSG_INVALID_ARGUMENT
    assert "null argument" in _lib.lib().tsg_last_error().decode()


def test_library_breakpoints_equal_reference_bitwise(golden):
    """The thresholds libtsgpu uploads (host_breakpoints) equal the reference's
    breakpoints_for(2^bits) bit for bit, sign of zero included, for every
    cardinality (src/breakpoints.cpp:65-114; tests/golden/breakpoints.npz is
    the reference's output), padded with +inf."""
    import paper_2009_00786_b200 as tg

    g = golden["load"]("breakpoints.npz")
    for bits in range(1, 9):
        got = tg.breakpoints(bits)
        want = g[f"bits{bits}"]
        k = (1 << bits) - 1
        assert np.array_equal(got[:k].view(np.uint64), want.view(np.uint64)), bits
        assert np.all(np.isposinf(got[k:])), bits
    with pytest.raises(tg.InvalidArgument, match="bits must be in"):
        tg.breakpoints(9)
