"""Host-side mirror of the reference ``tsidx`` API over the C ABI.

Same names, argument meaning and error behaviour as the reference's public
interface (paths relative to /root/reference/proj/core):

* ``IndexConfig``            include/tsidx/config.hpp:12-32 (validate: src/config.cpp:22-35)
* ``build_index``            include/tsidx/index.hpp:158, src/index.cpp:258-318
* ``exact_search``           include/tsidx/query.hpp:150-151, src/query.cpp:258-298
* ``approximate_search``     include/tsidx/query.hpp:133-134
* ``Measure``                include/tsidx/metrics.hpp:19-27
* ``SearchOptions`` / ``SearchResult`` / ``SearchStats`` / ``BuildStats``
                             include/tsidx/query.hpp:17-27,136-148; index.hpp:121-132

``std::invalid_argument`` surfaces as :class:`InvalidArgument` (a ValueError),
``std::logic_error`` as :class:`LogicError`. Every compute call goes through
``libtsgpu.so`` on the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import InvalidArgument, LogicError, TsgError, check, lib  # noqa: F401


class QueueMode(enum.IntEnum):
    single = 0
    multi = 1


@dataclasses.dataclass
class IndexConfig:
    n: int = 256
    w: int = 16
    max_card_bits: int = 8
    leaf_capacity: int = 2000
    chunk_size: int = 20000
    n_index_workers: int = 0
    n_search_workers: int = 0
    n_queues: int = 24
    queue_mode: QueueMode = QueueMode.multi
    initial_buffer_part_size: int = 5

    def segment_length(self) -> int:
        return self.n // self.w

    def to_c(self) -> _lib.tsg_config:
        for f in ("n", "leaf_capacity", "chunk_size", "n_index_workers", "n_search_workers", "n_queues",
                  "initial_buffer_part_size"):
            if getattr(self, f) < 0:
                raise InvalidArgument(f"IndexConfig: {f} must be non-negative")
        c = _lib.tsg_config()
        c.n, c.w, c.max_card_bits = self.n, self.w, self.max_card_bits
        c.leaf_capacity, c.chunk_size = self.leaf_capacity, self.chunk_size
        c.n_index_workers, c.n_search_workers = self.n_index_workers, self.n_search_workers
        c.n_queues, c.queue_mode = self.n_queues, int(self.queue_mode)
        c.initial_buffer_part_size = self.initial_buffer_part_size
        return c

    def validate(self) -> None:
        """Raises InvalidArgument naming the offending field (src/config.cpp:22-35)."""
        if self.w < -(2 ** 31) or self.w >= 2 ** 31:
            raise InvalidArgument("IndexConfig: w out of range")
        c = self.to_c()
        check(lib().tsg_config_validate(C.byref(c)))


class MeasureKind(enum.IntEnum):
    euclidean = 0
    dtw = 1


@dataclasses.dataclass(frozen=True)
class Measure:
    kind: MeasureKind = MeasureKind.euclidean
    window: int = 0

    @staticmethod
    def ed() -> "Measure":
        return Measure(MeasureKind.euclidean, 0)

    @staticmethod
    def dtw(window: int) -> "Measure":
        return Measure(MeasureKind.dtw, window)


@dataclasses.dataclass
class SearchOptions:
    workers: int = 0
    queues: int = 0
    mode: Optional[QueueMode] = None


@dataclasses.dataclass
class SearchStats:
    lb_node_calcs: int = 0
    lb_entry_calcs: int = 0
    real_dist_calcs: int = 0
    bsf_updates: int = 0
    pruned_subtrees: int = 0
    queue_insertions: int = 0

    def kv_line(self) -> str:
        return (f"lb_node={self.lb_node_calcs} lb_entry={self.lb_entry_calcs} real_dist={self.real_dist_calcs} "
                f"bsf_updates={self.bsf_updates} pruned_subtrees={self.pruned_subtrees} "
                f"queue_insertions={self.queue_insertions}")


@dataclasses.dataclass
class SearchResult:
    distance: float
    position: int
    stats: SearchStats
    box_calcs: int = 0  # quad box bounds evaluated (device extension of SearchStats)
    fine_calcs: int = 0  # fine-summary lower bounds evaluated before refinement (device extension)


@dataclasses.dataclass
class BuildStats:
    build_ns: int = 0
    series: int = 0
    nodes: int = 0
    inner_nodes: int = 0
    leaves: int = 0
    empty_leaves: int = 0
    overflow_leaves: int = 0
    max_depth: int = 0
    root_children: int = 0
    pages: int = 0
    h2d_ns: int = 0
    summarise_ms: float = 0.0
    organise_ms: float = 0.0
    leaves_ms: float = 0.0

    def kv_line(self) -> str:
        return (f"build series={self.series} time_ns={self.build_ns} nodes={self.nodes} inner={self.inner_nodes} "
                f"leaves={self.leaves} empty_leaves={self.empty_leaves} overflow_leaves={self.overflow_leaves} "
                f"max_depth={self.max_depth}")


@dataclasses.dataclass
class ValidationReport:
    """tsidx::ValidationReport (include/tsidx/index.hpp:180-196) of the device index."""
    nodes: int = 0
    inner_nodes: int = 0
    leaves: int = 0
    empty_leaves: int = 0
    overflow_leaves: int = 0
    max_depth: int = 0
    total_entries: int = 0
    leaf_fill_histogram: tuple = ()
    violations: list = dataclasses.field(default_factory=list)
    violation_count: int = 0
    pages: int = 0
    checked_boxes: int = 0

    def ok(self) -> bool:
        return self.violation_count == 0

    def summary(self) -> str:
        return (f"validate nodes={self.nodes} inner={self.inner_nodes} leaves={self.leaves} "
                f"empty_leaves={self.empty_leaves} overflow_leaves={self.overflow_leaves} max_depth={self.max_depth} "
                f"entries={self.total_entries} violations={self.violation_count}")


def validate_index(index: "Index") -> ValidationReport:
    """tsidx::validate_index (src/index.cpp:332-484): a full audit of the device index (tsg_index_validate)."""
    r = _lib.tsg_validation_report()
    check(lib().tsg_index_validate(index.handle, C.byref(r)))
    return ValidationReport(r.nodes, r.inner_nodes, r.leaves, r.empty_leaves, r.overflow_leaves, r.max_depth,
                            r.total_entries, tuple(r.leaf_fill_histogram),
                            [r.violations[i].value.decode() for i in range(r.n_violations)], r.violation_count,
                            r.pages, r.checked_boxes)


def _stats_from_c(s: _lib.tsg_build_stats) -> BuildStats:
    return BuildStats(**{f: getattr(s, f) for f, _ in _lib.tsg_build_stats._fields_})


def _result_from_c(r: _lib.tsg_result) -> SearchResult:
    st = SearchStats(**{f: getattr(r.stats, f) for f, _ in _lib.tsg_search_stats._fields_})
    return SearchResult(float(r.distance), int(r.position), st, int(r.box_calcs), int(r.fine_calcs))


class Context:
    """A set of devices an index is sharded over (tsg_open)."""

    def __init__(self, devices: Sequence[int] = (0,)):
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        self._lib = lib()  # held so teardown at interpreter exit needs no module globals
        check(self._lib.tsg_open(len(devices), devs, C.byref(h)))
        self._h = h
        self.devices = tuple(devices)

    @property
    def handle(self):
        return self._h

    def comm_init(self, nranks: int, rank: int, comm_id: bytes) -> None:
        """Join this one-device context to a communicator of `nranks` processes (one GPU each,
        SURVEY 8(e)). Searches on an index built on the context are then collective: every rank
        calls them with the same queries and receives the global answers."""
        cid = _lib.tsg_comm_id()
        if len(comm_id) != 128:
            raise InvalidArgument("comm_init: the id is 128 bytes (comm_unique_id)")
        C.memmove(cid.internal, bytes(comm_id), 128)
        check(self._lib.tsg_comm_init(self._h, nranks, rank, C.byref(cid)))

    def comm_info(self) -> tuple:
        """(transport, nranks, rank); transport 0 none, 1 local shards, 2 NCCL."""
        t, n, r = C.c_int(), C.c_int(), C.c_int()
        check(self._lib.tsg_comm_info(self._h, C.byref(t), C.byref(n), C.byref(r)))
        return t.value, n.value, r.value

    def close(self):
        if getattr(self, "_h", None):
            self._lib.tsg_close(self._h)
            self._h = None

    def __del__(self):
        self.close()


def comm_unique_id() -> bytes:
    """A fresh 128-byte communicator id (rank 0 creates it; the caller distributes it)."""
    cid = _lib.tsg_comm_id()
    check(lib().tsg_comm_unique_id(C.byref(cid)))
    return bytes(cid.internal)


_default_ctx: dict = {}


def _context(devices) -> Context:
    key = tuple(devices)
    if key not in _default_ctx:
        _default_ctx[key] = Context(key)
    return _default_ctx[key]


class Index:
    """The device index. Owns (a host view of) its dataset like the reference's
    Index owns its Dataset (src/index.cpp:255-256)."""

    def __init__(self, handle, data, config: IndexConfig, stats: BuildStats, ctx: Context, keepalive=None):
        self._lib = lib()
        self._h = handle
        self._data = data
        self._config = config
        self._stats = stats
        self._ctx = ctx
        self._keepalive = keepalive

    def config(self) -> IndexConfig:
        return self._config

    def device(self) -> int:
        """The (first) device of the index's context: where device queries must live."""
        return self._ctx.devices[0]

    def data(self):
        return self._data

    def series(self, position: int):
        return self._data[position]

    def build_stats(self) -> BuildStats:
        return self._stats

    @property
    def handle(self):
        return self._h

    def export(self):
        """(words[count][stride], positions[count], leaf_offsets[L+1], page_offsets[P+1],
        page_lo[P][stride], page_hi[P][stride]) in index order."""
        count = len(self._data)
        ws = lib().tsg_word_stride(self._config.w)
        L, P = self._stats.leaves, self._stats.pages
        words = np.empty((count, ws), np.uint8)
        pos = np.empty(count, np.uint32)
        off = np.empty(L + 1, np.uint32)
        poff = np.empty(P + 1, np.uint32)
        lo = np.empty((P, ws), np.uint8)
        hi = np.empty((P, ws), np.uint8)
        check(lib().tsg_index_export(self._h, words.ctypes.data, pos.ctypes.data, off.ctypes.data,
                                     poff.ctypes.data, lo.ctypes.data, hi.ctypes.data))
        return words, pos, off, poff, lo, hi

    def debug_poke(self, array: int, offset: int, data: bytes) -> None:
        """Test hook (tsg_index_debug_poke): overwrite bytes of one device array of the index."""
        buf = C.create_string_buffer(bytes(data), len(data))
        check(lib().tsg_index_debug_poke(self._h, array, offset, buf, len(data)))

    def thresholds(self) -> np.ndarray:
        """The 256-entry threshold table in HBM the index's kernels read (breakpoints, then +inf)."""
        out = np.empty(256, np.float64)
        check(lib().tsg_index_thresholds(self._h, out.ctypes.data))
        return out

    def export_fine(self):
        """Fine summary rows [count][fine_width] in dataset order (None when the index has none)."""
        fw = C.c_uint32(0)
        check(lib().tsg_index_export_fine(self._h, C.byref(fw), None))
        if fw.value == 0:
            return None
        stride = (fw.value + 15) // 16 * 16
        out = np.empty((len(self._data), stride), np.uint8)
        check(lib().tsg_index_export_fine(self._h, None, out.ctypes.data))
        return out[:, :fw.value]

    def free(self):
        if getattr(self, "_h", None):
            self._lib.tsg_index_free(self._h)
            self._h = None
        if self._keepalive is not None:  # a borrowed device dataset can be released by the caller now
            self._keepalive = None
            self._data = None

    def __del__(self):
        self.free()


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


def _device_tensor(t, what: str, device: int, dims: int = 2):
    """A CUDA tensor argument checked (float32, `dims`-D, on the index's device) and made
    contiguous, with torch's current stream of that device synchronised: the library reads it on
    its own non-blocking stream, so pending writes (t.contiguous(), generators, user kernels) on
    torch's stream must have finished first."""
    import torch

    if t.dtype != torch.float32 or t.dim() != dims:
        raise InvalidArgument(f"{what} must be a {dims}-D float32 tensor")
    if t.device.index != device:
        raise InvalidArgument(f"{what} is on cuda:{t.device.index}, the index on cuda:{device}")
    t = t.contiguous()
    torch.cuda.current_stream(t.device).synchronize()
    return t


def build_index(dataset, config: IndexConfig = None, devices: Sequence[int] = (0,), position_offset: int = 0,
                context: "Context" = None) -> Index:
    """tsidx::build_index. ``dataset``: a (count, n) float32 array on the host
    (copied into HBM), or a CUDA tensor already resident on the device
    (borrowed, zero-copy; single-device only). ``context`` (instead of
    ``devices``): a Context, e.g. one joined to a multi-process communicator."""
    config = config or IndexConfig()
    cfg = config.to_c()
    st = _lib.tsg_build_stats()
    h = C.c_void_p()
    ctx = context if context is not None else _context(devices)
    if _is_cuda_tensor(dataset):
        if len(ctx.devices) != 1:
            raise InvalidArgument("tsg_index_build_device: device rows need a single-device context")
        t = _device_tensor(dataset, "build_index: device dataset", ctx.devices[0])
        count, length = (t.shape[0], t.shape[1]) if t.numel() else (0, config.n)
        check(lib().tsg_index_build_device(ctx.handle, C.c_void_p(t.data_ptr()), count, length, C.byref(cfg),
                                           position_offset, C.byref(h), C.byref(st)))
        return Index(h, t, config, _stats_from_c(st), ctx, keepalive=t)
    arr = np.asarray(dataset, dtype=np.float32)
    if arr.ndim == 1 and arr.size == 0:
        arr = arr.reshape(0, config.n)
    if arr.ndim != 2:
        raise InvalidArgument("build_index: dataset must be 2-D (count, length)")
    arr = np.ascontiguousarray(arr)
    check(lib().tsg_index_build(ctx.handle, arr.ctypes.data, arr.shape[0], arr.shape[1], C.byref(cfg),
                                position_offset, C.byref(h), C.byref(st)))
    return Index(h, arr, config, _stats_from_c(st), ctx)


def build_index_from_file(path, config: IndexConfig = None, devices: Sequence[int] = (0,),
                          position_offset: int = 0, context: "Context" = None) -> Index:
    """tsidx::load_dataset(path, config.n) + tsidx::build_index, streamed: each
    device reads its range of the headerless float32 file in chunks while K1
    summarises the chunks already in HBM (no host copy of the dataset). The
    index's ``data()`` is a read-only memory map of the file."""
    config = config or IndexConfig()
    cfg = config.to_c()
    st = _lib.tsg_build_stats()
    h = C.c_void_p()
    ctx = context if context is not None else _context(devices)
    check(lib().tsg_index_build_file(ctx.handle, os.fsencode(os.fspath(path)), config.n, C.byref(cfg),
                                     position_offset, C.byref(h), C.byref(st)))
    data = np.memmap(path, dtype=np.float32, mode="r").reshape(-1, config.n)
    return Index(h, data, config, _stats_from_c(st), ctx)


def load_dataset(path, length: int) -> np.ndarray:
    """tsidx::load_dataset (src/dataset.cpp:87-110): a headerless float32 file
    of count x length values, with the reference's checks and messages."""
    if length <= 0:
        raise InvalidArgument("load_dataset: length must be positive")
    path = os.fspath(path)
    try:
        size = os.stat(path).st_size
    except OSError as e:
        raise TsgError(f"load_dataset: cannot stat {path}: {e.strerror}") from None
    series_bytes = length * 4
    if size == 0 or size % series_bytes != 0:
        raise TsgError(f"load_dataset: {path} holds {size} bytes, not a positive multiple of "
                       f"{series_bytes} (length {length} * 4)")
    return np.fromfile(path, dtype=np.float32).reshape(-1, length)


def save_dataset(path, rows) -> None:
    """tsidx::save_dataset (src/dataset.cpp:112-117): the values, row-major, no header."""
    np.ascontiguousarray(np.asarray(rows, dtype=np.float32)).tofile(os.fspath(path))


def _check_measure(measure: Measure, n: int) -> None:
    if measure.kind == MeasureKind.dtw and (measure.window < 0 or measure.window >= n):
        raise InvalidArgument("dtw window must be in [0, n)")


def _measure_c(measure: Measure) -> "_lib.tsg_measure":
    return _lib.tsg_measure(_lib.TSG_MEASURE_DTW if measure.kind == MeasureKind.dtw else _lib.TSG_MEASURE_ED,
                            measure.window)


def _query_array(index: Index, query) -> np.ndarray:
    q = np.ascontiguousarray(np.asarray(query, dtype=np.float32))
    n = index.config().n
    if q.ndim != 1 or q.size != n:
        raise InvalidArgument(f"query length {q.size if q.ndim == 1 else q.shape} does not match the index "
                              f"series length {n}")
    return q


def exact_search(index: Index, query, measure: Measure = Measure.ed(), options: SearchOptions = None) -> SearchResult:
    """tsidx::exact_search: Euclidean or DTW (Measure.dtw(window)). options.workers/queues/mode are
    accepted and ignored."""
    _check_measure(measure, index.config().n)
    q = _query_array(index, query)
    out = (_lib.tsg_result * 1)()
    if measure.kind == MeasureKind.euclidean:
        check(lib().tsg_search(index.handle, q.ctypes.data, 1, out))
    else:
        m = _measure_c(measure)
        check(lib().tsg_search_measure(index.handle, q.ctypes.data, 0, 1, C.byref(m), 0, out))
    return _result_from_c(out[0])


def exact_search_batch(index: Index, queries, measure: Measure = Measure.ed()) -> list:
    """Exact 1-NN for a (nq, n) block of queries in one call (queries answered in order)."""
    _check_measure(measure, index.config().n)
    n = index.config().n
    m = _measure_c(measure)
    if _is_cuda_tensor(queries):
        t = _device_tensor(queries, "queries", index.device())
        if t.shape[1] != n:
            raise InvalidArgument(f"query length {tuple(t.shape)} does not match the index series length {n}")
        out = (_lib.tsg_result * t.shape[0])()
        if measure.kind == MeasureKind.euclidean:
            check(lib().tsg_search_device(index.handle, C.c_void_p(t.data_ptr()), t.shape[0], out))
        else:
            check(lib().tsg_search_measure(index.handle, C.c_void_p(t.data_ptr()), 1, t.shape[0], C.byref(m), 0, out))
        return [_result_from_c(r) for r in out]
    q = np.ascontiguousarray(np.asarray(queries, dtype=np.float32))
    if q.ndim != 2 or q.shape[1] != n:
        raise InvalidArgument(f"query length {q.shape} does not match the index series length {n}")
    out = (_lib.tsg_result * q.shape[0])()
    if measure.kind == MeasureKind.euclidean:
        check(lib().tsg_search(index.handle, q.ctypes.data, q.shape[0], out))
    else:
        check(lib().tsg_search_measure(index.handle, q.ctypes.data, 0, q.shape[0], C.byref(m), 0, out))
    return [_result_from_c(r) for r in out]


# numpy view of tsg_result (include/tsgpu.h): one record per query
RESULT_DTYPE = np.dtype({"names": ["distance", "position", "box_calcs", "stats", "fine_calcs"],
                         "formats": [np.float64, np.uint32, np.uint32, (np.uint64, 6), np.uint64],
                         "offsets": [_lib.tsg_result.distance.offset, _lib.tsg_result.position.offset,
                                     _lib.tsg_result.box_calcs.offset, _lib.tsg_result.stats.offset,
                                     _lib.tsg_result.fine_calcs.offset],
                         "itemsize": C.sizeof(_lib.tsg_result)})


def _res_ptr(arr: np.ndarray):
    return C.cast(arr.ctypes.data, C.POINTER(_lib.tsg_result))


def exact_search_batch_records(index: Index, queries, measure: Measure = Measure.ed()) -> np.ndarray:
    """exact_search_batch without per-query Python objects: a structured array (RESULT_DTYPE) over
    the C ABI's result records (distance, position, box_calcs, stats[6] in SearchStats order,
    fine_calcs). For batch pipelines where building SearchResult objects would cost host time."""
    _check_measure(measure, index.config().n)
    n = index.config().n
    m = _measure_c(measure)
    if _is_cuda_tensor(queries):
        t = _device_tensor(queries, "queries", index.device())
        if t.shape[1] != n:
            raise InvalidArgument(f"query length {tuple(t.shape)} does not match the index series length {n}")
        out = np.empty(t.shape[0], RESULT_DTYPE)
        if measure.kind == MeasureKind.euclidean:
            check(lib().tsg_search_device(index.handle, C.c_void_p(t.data_ptr()), t.shape[0], _res_ptr(out)))
        else:
            check(lib().tsg_search_measure(index.handle, C.c_void_p(t.data_ptr()), 1, t.shape[0], C.byref(m), 0,
                                           _res_ptr(out)))
        return out
    q = np.ascontiguousarray(np.asarray(queries, dtype=np.float32))
    if q.ndim != 2 or q.shape[1] != n:
        raise InvalidArgument(f"query length {q.shape} does not match the index series length {n}")
    out = np.empty(q.shape[0], RESULT_DTYPE)
    if measure.kind == MeasureKind.euclidean:
        check(lib().tsg_search(index.handle, q.ctypes.data, q.shape[0], _res_ptr(out)))
    else:
        check(lib().tsg_search_measure(index.handle, q.ctypes.data, 0, q.shape[0], C.byref(m), 0, _res_ptr(out)))
    return out


def approximate_search(index: Index, query, measure: Measure = Measure.ed()) -> SearchResult:
    """tsidx::approximate_search: the best series in the query's closest leaf."""
    _check_measure(measure, index.config().n)
    q = _query_array(index, query)
    out = (_lib.tsg_result * 1)()
    m = _measure_c(measure)
    check(lib().tsg_search_measure(index.handle, q.ctypes.data, 0, 1, C.byref(m), 1, out))
    return _result_from_c(out[0])


def summarise(rows_cuda, w: int = 16, bits: int = 8):
    """K1 alone on a CUDA tensor of rows: returns (words uint8 [count, stride], root_keys int32 [count])."""
    import torch

    t = rows_cuda.contiguous()
    count, n = t.shape
    ws = lib().tsg_word_stride(w)
    words = torch.empty((count, ws), dtype=torch.uint8, device=t.device)
    keys = torch.empty((count,), dtype=torch.int32, device=t.device)
    stream = torch.cuda.current_stream(t.device).cuda_stream
    check(lib().tsg_summarise(C.c_void_p(t.data_ptr()), count, n, w, bits, C.c_void_p(words.data_ptr()),
                              C.c_void_p(keys.data_ptr()), C.c_void_p(stream)))
    return words, keys


def generate_random_walk_device(count: int, length: int, seed: int, znorm: bool = True, begin: int = 0,
                                device: int = 0):
    """Rows [begin, begin+count) of the reference generator, created in HBM (input setup)."""
    import torch

    out = torch.empty((count, length), dtype=torch.float32, device=f"cuda:{device}")
    stream = torch.cuda.current_stream(out.device).cuda_stream
    check(lib().tsg_generate_random_walk(C.c_void_p(out.data_ptr()), begin, count, length, seed,
                                         1 if znorm else 0, C.c_void_p(stream)))
    return out


def generate_device(kind: str, count: int, length: int, seed: int, begin: int = 0, device: int = 0,
                    noise: float = 0.0, data_count: int = 0, data_seed: int = 1, znorm: bool = True):
    """BASELINE workloads generated in HBM: kind 'rw' (configs 1-2), 'c3', 'c4', or 'c5'
    (noisy queries over a `data_count`-series random-walk dataset of `data_seed`)."""
    import torch

    kinds = {"rw": 0, "c3": 3, "c4": 4, "c5": 5}
    out = torch.empty((count, length), dtype=torch.float32, device=f"cuda:{device}")
    stream = torch.cuda.current_stream(out.device).cuda_stream
    check(lib().tsg_generate_series(kinds[kind], C.c_void_p(out.data_ptr()), begin, count, length, seed,
                                    1 if znorm else 0, float(noise), data_count, data_seed, C.c_void_p(stream)))
    return out


def breakpoints(bits: int) -> np.ndarray:
    """tsidx::breakpoints_for(2**bits) as the library computes it for upload: 256 doubles (the
    2**bits - 1 breakpoints, then +inf)."""
    out = np.empty(256, np.float64)
    check(lib().tsg_breakpoints(bits, out.ctypes.data))
    return out


def launch_count() -> int:
    return int(lib().tsg_launch_count())
