"""Python mirror of the reference's operator / query API (namespace ``tq``).

Same names, argument meaning and error behaviour as /root/reference/proj:

* ``TileConfig`` / ``PredicateSpec`` / ``ScheduleMode``   include/tq/tile.hpp, kernel.hpp
* ``run_query`` / ``QueryResult`` / ``QueryStats`` / ``diff_results``
                                                         include/tq/ssb_queries.hpp
* ``select_*_into`` / ``select_*``                       include/tq/select.hpp
* ``project_{linear,sigmoid}[_into]``                    include/tq/project.hpp
* ``HashTable.build`` / ``join_probe_*``                 include/tq/hash_table.hpp, join.hpp
* ``lsb_radix_sort`` / ``msb_radix_sort``                include/tq/radix.hpp
* ``ConfigError`` / ``ContractError`` / ``BuildError`` / ``IoError``
                                                         include/tq/common.hpp:16-34

Every call goes through the C ABI (libcrystal_b200.so) to sm_100a kernels.
"Spans" are torch CUDA tensors (device-resident columns, the fast path) or
numpy arrays (host spans: staged H2D/D2H inside the call).  ``workers`` keeps
its reference meaning of a parallelism degree and is validated (>= 1); on one
GPU the grid is sized by the hardware, so it does not change the result.
"""
from __future__ import annotations

import ctypes as C
import enum
import json
import os
import threading
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import LIB

# ----------------------------------------------------------------- errors


class ConfigError(ValueError):
    """tq::ConfigError (std::invalid_argument)."""


class ContractError(RuntimeError):
    """tq::ContractError (std::logic_error)."""


class BuildError(RuntimeError):
    """tq::BuildError (std::runtime_error)."""


class IoError(RuntimeError):
    """tq::IoError (std::runtime_error)."""


class CudaError(RuntimeError):
    """CUDA runtime failure (no reference analogue)."""


class NotBuiltError(RuntimeError):
    """The requested kernel shape is not compiled for sm_100a."""


class NcclError(RuntimeError):
    """NCCL missing or failed (device groups; no reference analogue)."""


_ERRORS = {_lib.CRYS_ECONFIG: ConfigError, _lib.CRYS_ECONTRACT: ContractError,
           _lib.CRYS_EBUILD: BuildError, _lib.CRYS_EIO: IoError, _lib.CRYS_ECUDA: CudaError,
           _lib.CRYS_ENOTBUILT: NotBuiltError, _lib.CRYS_ENCCL: NcclError}


def check(status: int) -> None:
    if status != _lib.CRYS_OK:
        msg = LIB.crys_last_error().decode()
        raise _ERRORS.get(status, RuntimeError)(msg)


# ----------------------------------------------------------------- tile model

@dataclass(frozen=True)
class TileConfig:
    """tile.hpp:24-36 (default 128 x 4; any positive shape is valid)."""
    block_threads: int = 128
    items_per_thread: int = 4

    def tile_size(self) -> int:
        return self.block_threads * self.items_per_thread

    def validate(self) -> None:
        if self.block_threads <= 0:
            raise ConfigError("TileConfig: block_threads must be positive")
        if self.items_per_thread <= 0:
            raise ConfigError("TileConfig: items_per_thread must be positive")


kSweepBlockThreads = (32, 64, 128, 256, 512, 1024)
kSweepItemsPerThread = (1, 2, 4, 8)


class ScheduleMode(enum.Enum):
    kDeterministic = 0
    kArrivalOrder = 1


class PredOp(enum.IntEnum):
    LT = _lib.CRYS_LT
    LE = _lib.CRYS_LE
    GT = _lib.CRYS_GT
    GE = _lib.CRYS_GE
    EQ = _lib.CRYS_EQ
    BETWEEN = _lib.CRYS_BETWEEN


class PredCombine(enum.Enum):
    INIT = 0
    AND = 1


@dataclass(frozen=True)
class PredicateSpec:
    """tile.hpp:99-133."""
    op: PredOp = PredOp.LT
    lo: int = 0
    hi: int = 0
    combine: PredCombine = PredCombine.INIT

    @staticmethod
    def lt(v): return PredicateSpec(PredOp.LT, v, v)

    @staticmethod
    def le(v): return PredicateSpec(PredOp.LE, v, v)

    @staticmethod
    def gt(v): return PredicateSpec(PredOp.GT, v, v)

    @staticmethod
    def ge(v): return PredicateSpec(PredOp.GE, v, v)

    @staticmethod
    def eq(v): return PredicateSpec(PredOp.EQ, v, v)

    @staticmethod
    def between(lo, hi):
        if hi < lo:
            raise ConfigError("PredicateSpec: BETWEEN requires lo <= hi")
        return PredicateSpec(PredOp.BETWEEN, lo, hi)

    def then_and(self):
        return PredicateSpec(self.op, self.lo, self.hi, PredCombine.AND)

    def eval(self, y) -> bool:
        return {PredOp.LT: y < self.lo, PredOp.LE: y <= self.lo, PredOp.GT: y > self.lo,
                PredOp.GE: y >= self.lo, PredOp.EQ: y == self.lo,
                PredOp.BETWEEN: self.lo <= y <= self.hi}[self.op]

    def _c(self) -> _lib.crys_pred:
        return _lib.crys_pred(int(self.op), int(self.lo), int(self.hi))


# ----------------------------------------------------------------- context

class Context:
    """One CUDA device + stream + scratch (replaces the per-call thread pool of
    parallel_for_blocks, kernel.cpp:60-103).  A context is not thread-safe:
    ``Context.default`` hands every host thread its own context per device.

    ``Context.group(devices)`` is a DEVICE GROUP (crys_init_group): one
    lineorder shard per entry of ``devices`` (an ordinal may repeat: several
    shards on one GPU), dimensions replicated per device, and each query merged
    by ONE NCCL reduce inside the library -- the reference's ``workers``
    fan-out driven from one host thread."""

    _default = threading.local()

    def __init__(self, device: int = 0, _handle=None):
        self.device = device
        if _handle is None:
            h = C.c_void_p()
            check(LIB.crys_init(device, C.byref(h)))
            _handle = h
        self.h = _handle

    @classmethod
    def default(cls, device: Optional[int] = None) -> "Context":
        if device is None:
            import torch
            device = torch.cuda.current_device()
        per_thread = getattr(cls._default, "ctxs", None)
        if per_thread is None:
            per_thread = cls._default.ctxs = {}
        if device not in per_thread:
            per_thread[device] = Context(device)
        return per_thread[device]

    @classmethod
    def group(cls, devices: Sequence[int]) -> "Context":
        devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        check(LIB.crys_init_group(len(devices), devs, C.byref(h)))
        return cls(int(devices[0]), h)

    def shards(self) -> int:
        return LIB.crys_group_shards(self.h)

    def devices(self) -> int:
        return LIB.crys_group_devices(self.h)

    def uses_nccl(self) -> bool:
        return bool(LIB.crys_group_uses_nccl(self.h))

    def bind_torch_stream(self) -> None:
        """Run subsequent calls on torch's current stream (ordering with torch ops)."""
        import torch
        s = torch.cuda.current_stream(self.device)
        # torch's default stream is the legacy stream (handle 0): bind it as
        # cudaStreamLegacy, not NULL (NULL selects the ctx's own non-blocking
        # stream, which would race with torch and NCCL ops on the default stream)
        check(LIB.crys_set_stream(self.h, C.c_void_p(s.cuda_stream or _lib.CRYS_STREAM_LEGACY)))

    def launches(self) -> int:
        return LIB.crys_kernel_launches(self.h)

    def enable_timing(self, on: bool = True) -> None:
        check(LIB.crys_enable_timing(self.h, 1 if on else 0))

    def last_timing(self) -> Tuple[float, float]:
        k, t = C.c_double(), C.c_double()
        check(LIB.crys_last_timing(self.h, C.byref(k), C.byref(t)))
        return k.value, t.value

    def synchronize(self) -> None:
        check(LIB.crys_synchronize(self.h))

    def close(self) -> None:
        if self.h:
            LIB.crys_destroy(self.h)
            self.h = None


# ----------------------------------------------------------------- SSB

class QueryId(enum.IntEnum):
    """ssb_plans.hpp:19-24; values follow all_query_ids() order."""
    kQ11 = 0
    kQ12 = 1
    kQ13 = 2
    kQ21 = 3
    kQ22 = 4
    kQ23 = 5
    kQ31 = 6
    kQ32 = 7
    kQ33 = 8
    kQ34 = 9
    kQ41 = 10
    kQ42 = 11
    kQ43 = 12


_QNAMES = ["q11", "q12", "q13", "q21", "q22", "q23", "q31", "q32", "q33", "q34", "q41", "q42", "q43"]
# GroupPart labels per plan (ssb_plans.cpp:110-275)
_GROUP_LABELS = {
    0: [], 1: [], 2: [],
    3: ["d_year", "p_brand1"], 4: ["d_year", "p_brand1"], 5: ["d_year", "p_brand1"],
    6: ["c_nation", "s_nation", "d_year"], 7: ["c_city", "s_city", "d_year"],
    8: ["c_city", "s_city", "d_year"], 9: ["c_city", "s_city", "d_year"],
    10: ["d_year", "c_nation"], 11: ["d_year", "s_nation", "p_category"],
    12: ["d_year", "s_city", "p_brand1"],
}


def query_name(qid) -> str:
    return _QNAMES[int(qid)]


def query_id_from_name(name: str) -> QueryId:
    if name not in _QNAMES:
        raise ConfigError(f"unknown query id: {name}")
    return QueryId(_QNAMES.index(name))


def all_query_ids() -> List[QueryId]:
    return list(QueryId)


def query_shape(qid) -> Tuple[int, int, int]:
    """(cells, group arity, joins) of the plan (AggregateTable::cells)."""
    cells, ng, nj = C.c_int64(), C.c_int32(), C.c_int32()
    check(LIB.crys_query_shape(int(qid), C.byref(cells), C.byref(ng), C.byref(nj)))
    return cells.value, ng.value, nj.value


def query_plan(qid) -> dict:
    """plan_for(id) (ssb_plans.cpp:21-322) as a dict: fact filters, ordered
    joins with their inclusive-range filters and payloads, group parts, agg."""
    n = C.c_size_t()
    check(LIB.crys_query_plan_json(int(qid), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(LIB.crys_query_plan_json(int(qid), buf, n.value + 1, C.byref(n)))
    return json.loads(buf.value.decode())


@dataclass
class ResultRow:
    group: Tuple[int, ...]
    sum: int


class QueryResult:
    """ssb_queries.hpp:52-62: rows sorted by group (lexicographic).

    Backed by two arrays straight from the C ABI (``groups`` int32[n, arity],
    ``sums`` int64[n]); ``rows`` materialises ResultRow objects on first use."""

    def __init__(self, group_labels=None, rows=None, groups=None, sums=None):
        self.group_labels = list(group_labels or [])
        if rows is not None:
            self._rows = list(rows)
            self.groups = np.array([r.group for r in self._rows], np.int32).reshape(len(self._rows), -1)
            self.sums = np.array([r.sum for r in self._rows], np.int64)
        else:
            self._rows = None
            self.groups = groups if groups is not None else np.zeros((0, len(self.group_labels)), np.int32)
            self.sums = sums if sums is not None else np.zeros(0, np.int64)

    def __len__(self) -> int:
        return len(self.sums)

    @property
    def rows(self) -> List[ResultRow]:
        if self._rows is None:
            self._rows = [ResultRow(tuple(int(x) for x in g), int(v)) for g, v in
                          zip(self.groups.tolist(), self.sums.tolist())]
        return self._rows

    @rows.setter
    def rows(self, value) -> None:
        self._rows = list(value)

    def as_tuples(self) -> List[Tuple[Tuple[int, ...], int]]:
        if self._rows is not None:
            return [(tuple(r.group), int(r.sum)) for r in self._rows]
        return [(tuple(g), v) for g, v in zip(self.groups.tolist(), self.sums.tolist())]


@dataclass
class QueryStats:
    """ssb_queries.hpp:70-74."""
    survivors: List[int] = field(default_factory=list)


def sort_result(result: QueryResult) -> None:
    result.rows.sort(key=lambda r: tuple(r.group))


def diff_results(got: QueryResult, expected: QueryResult) -> str:
    """ssb_queries.cpp:67-88: empty string when equal, else a short diff."""
    out = []
    if len(got.rows) != len(expected.rows):
        out.append(f"row count {len(got.rows)} vs {len(expected.rows)}; ")
    reported = 0
    for i, (g, e) in enumerate(zip(got.rows, expected.rows)):
        if reported >= 5:
            break
        if tuple(g.group) == tuple(e.group) and g.sum == e.sum:
            continue
        reported += 1
        out.append(f"row {i}: ({','.join(map(str, g.group))})={g.sum} vs "
                   f"({','.join(map(str, e.group))})={e.sum}; ")
    return "".join(out)


LO_COLS = ["lo_orderdate", "lo_custkey", "lo_suppkey", "lo_partkey", "lo_quantity",
           "lo_discount", "lo_extendedprice", "lo_revenue", "lo_supplycost"]
DIM_COLS = {
    "date": ["d_datekey", "d_year", "d_yearmonthnum", "d_yearmonth", "d_weeknuminyear"],
    "supplier": ["s_suppkey", "s_city", "s_nation", "s_region"],
    "customer": ["c_custkey", "c_city", "c_nation", "c_region"],
    "part": ["p_partkey", "p_brand1", "p_category", "p_mfgr"],
}


class DeviceDatabase:
    """HBM-resident columnar SSB database (the B200 `SsbDatabase`).  Lineorder
    may be a row-range shard [lo_begin, lo_end); dimensions are whole."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.h = handle

    @classmethod
    def generate(cls, sf: int, seed: int = 42, lo_begin: int = 0, lo_end: int = -1,
                 ctx: Optional[Context] = None) -> "DeviceDatabase":
        """generate_ssb(sf, seed) (ssb_gen.cpp:243-270), computed in HBM."""
        ctx = ctx or Context.default()
        h = C.c_void_p()
        check(LIB.crys_db_generate(ctx.h, int(sf), int(seed), int(lo_begin), int(lo_end), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_host(cls, tables: Dict[str, Dict[str, np.ndarray]], ctx: Optional[Context] = None,
                  sf: int = 1, seed: int = 0) -> "DeviceDatabase":
        ctx = ctx or Context.default()
        h = C.c_void_p()
        check(LIB.crys_db_create(ctx.h, sf, seed, C.byref(h)))
        db = cls(ctx, h)
        for t, cols in tables.items():
            for c, a in cols.items():
                db.upload(t, c, a)
        return db

    def upload_host(self, tables, order=None) -> None:
        """Asynchronous bulk H2D of host columns (crys_db_upload_host): copies
        are issued in ``order`` (a list of (table, column); default: mapping
        order) on the copy stream and each query waits only for the columns it
        reads.  The arrays must stay alive (and, for a true DMA, be pinned)
        until the queries that read them have completed; they are kept
        referenced by this object until the next upload_host."""
        if order is None:
            order = [(t, c) for t, cs in tables.items() for c in cs]
        keep, cols = [], []
        for t, c in order:
            a = tables[t][c]
            if not (isinstance(a, np.ndarray) and a.dtype == np.int32 and a.flags.c_contiguous):
                a = np.ascontiguousarray(a, dtype=np.int32)
            keep.append(a)
            cols.append(_lib.crys_host_column(t.encode(), c.encode(), a.ctypes.data, len(a)))
        arr = (_lib.crys_host_column * len(cols))(*cols)
        check(LIB.crys_db_upload_host(self.h, arr, len(cols)))
        self._host_keep = keep

    def load_column_file(self, table: str, column: str, path: str) -> None:
        """load_column (column_io.cpp:65-100) of a CRYS file straight into HBM."""
        check(LIB.crys_db_load_column_file(self.h, table.encode(), column.encode(), os.fsencode(path)))

    def save_column_file(self, table: str, column: str, path: str) -> None:
        """save_column (column_io.cpp:50-63) of an HBM column."""
        check(LIB.crys_db_save_column_file(self.h, table.encode(), column.encode(), os.fsencode(path)))

    def has_column(self, table: str, column: str) -> bool:
        p, n = C.c_void_p(), C.c_int64()
        return LIB.crys_db_column(self.h, table.encode(), column.encode(), C.byref(p), C.byref(n)) == 0

    def upload(self, table: str, column: str, data) -> None:
        a = np.ascontiguousarray(data, dtype=np.int32)
        check(LIB.crys_db_upload_column(self.h, table.encode(), column.encode(),
                                        a.ctypes.data_as(C.c_void_p), len(a)))

    def column_ptr(self, table: str, column: str) -> Tuple[int, int]:
        p, n = C.c_void_p(), C.c_int64()
        check(LIB.crys_db_column(self.h, table.encode(), column.encode(), C.byref(p), C.byref(n)))
        return p.value or 0, n.value

    def rows(self, table: str, column: str) -> int:
        n = C.c_int64()
        check(LIB.crys_db_column_rows(self.h, table.encode(), column.encode(), C.byref(n)))
        return n.value

    def download(self, table: str, column: str) -> np.ndarray:
        n = self.rows(table, column)
        out = np.empty(n, np.int32)
        check(LIB.crys_db_download_column(self.h, table.encode(), column.encode(),
                                          out.ctypes.data_as(C.c_void_p), n))
        return out

    def free(self) -> None:
        if self.h:
            LIB.crys_db_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


SSB_TABLES = ["lineorder", "date", "supplier", "customer", "part"]


def load_database(directory: str, ctx: Optional[Context] = None) -> DeviceDatabase:
    """load_database (column_io.cpp:142-190): manifest.json + one CRYS file per
    column, every column streamed into HBM (IoError on a malformed manifest,
    file or a length that disagrees with the manifest)."""
    mpath = os.path.join(directory, "manifest.json")
    try:
        with open(mpath) as f:
            manifest = json.load(f)
    except OSError:
        raise IoError(f"cannot open manifest in {directory}")
    except ValueError as e:
        raise IoError(f"manifest parse error in {directory}: {e}")
    try:
        if manifest["format"] != "crys-manifest":
            raise IoError(f"not a database manifest: {directory}")
        db = DeviceDatabase.from_host({}, ctx=ctx, sf=int(manifest["scale_factor"]), seed=int(manifest["seed"]))
        for t in SSB_TABLES:
            for jc in manifest["tables"][t]["columns"]:
                if jc["kind"] != "int32":
                    raise IoError(f"element kind mismatch: {jc['file']} holds {jc['kind']}, expected int32")
                db.load_column_file(t, jc["name"], os.path.join(directory, jc["file"]))
                _, n = db.column_ptr(t, jc["name"])
                if n != int(jc["length"]):
                    raise IoError(f"column length disagrees with manifest: {jc['name']}")
    except (KeyError, TypeError) as e:
        raise IoError(f"manifest field error in {directory}: {e}")
    return db


def save_database(db: DeviceDatabase, directory: str, scale_factor: int, seed: int,
                  dictionaries: Optional[Dict[str, List[str]]] = None) -> None:
    """save_database (column_io.cpp:104-140): one CRYS file per HBM column of the
    SSB tables + manifest.json in the reference's layout."""
    os.makedirs(directory, exist_ok=True)
    tables = {}
    for t in SSB_TABLES:
        names = LO_COLS if t == "lineorder" else DIM_COLS[t]
        cols, rows = [], 0
        for c in names:
            if not db.has_column(t, c):
                continue
            file = f"{t}.{c}.col"
            db.save_column_file(t, c, os.path.join(directory, file))
            _, n = db.column_ptr(t, c)
            rows = n
            cols.append({"name": c, "file": file, "kind": "int32", "length": n})
        tables[t] = {"rows": rows, "columns": cols}
    manifest = {"format": "crys-manifest", "version": 1, "scale_factor": int(scale_factor), "seed": int(seed),
                "tables": tables, "dictionaries": dictionaries or {}}
    with open(os.path.join(directory, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=2)
        f.write("\n")


def random_i32(out, seed: int, stream: int, lo: int, hi: int, index0: int = 0) -> None:
    """Fill a CUDA int32 tensor with the reference CLI's random_i32 stream
    (tools/tq_main.cpp:147-152): out[i] = Rng(seed, stream).uniform_i32(index0+i, lo, hi)."""
    p, n = _dev(out, "int32")
    ctx = _ctx_for(out)
    check(LIB.crys_fill_uniform_i32(ctx.h, C.c_void_p(p), n, int(seed), int(stream), int(index0),
                                    int(lo), int(hi)))


def project_inputs(x1, x2, seed: int, stream: int = 2, lo: float = -4.0, hi: float = 4.0) -> None:
    """The project microbenchmark inputs (tools/tq_main.cpp:335-340), in HBM."""
    p1, n1 = _dev(x1, "float32")
    p2, n2 = _dev(x2, "float32")
    if n1 != n2:
        raise ConfigError("project inputs: length mismatch")
    ctx = _ctx_for(x1)
    check(LIB.crys_fill_float_pairs(ctx.h, C.c_void_p(p1), C.c_void_p(p2), n1, int(seed), int(stream),
                                    float(lo), float(hi)))


def generate_ssb(sf: int, seed: int = 42, ctx: Optional[Context] = None) -> DeviceDatabase:
    return DeviceDatabase.generate(sf, seed, ctx=ctx)


_OUT = threading.local()


def _out_buffers(qid: int, maxr: int):
    """Per-thread, per-query output buffers of the C ABI, allocated once: a
    fresh np.empty of q4.3's 1.75 M-row bound costs an mmap/munmap pair on
    every call.  Results are copied out (_rows_from_buffers)."""
    cache = getattr(_OUT, "bufs", None)
    if cache is None:
        cache = _OUT.bufs = {}
    b = cache.get(qid)
    if b is None:
        groups = np.empty(3 * maxr, np.int32)
        sums = np.empty(maxr, np.int64)
        surv = np.zeros(4, np.int64)
        b = cache[qid] = (groups, sums, surv, C.c_void_p(groups.ctypes.data), C.c_void_p(sums.ctypes.data),
                         C.c_void_p(surv.ctypes.data))
    return b


def _rows_from_buffers(qid, groups, sums, n) -> QueryResult:
    labels = _GROUP_LABELS[int(qid)]
    ng = len(labels)
    g = groups[:3 * n].reshape(n, 3)[:, :ng].copy() if n else np.zeros((0, ng), np.int32)
    return QueryResult(list(labels), groups=g, sums=np.array(sums[:n], np.int64))


_SHAPES: Dict[int, Tuple[int, int, int]] = {}


def _shape(qid: int) -> Tuple[int, int, int]:
    sh = _SHAPES.get(qid)
    if sh is None:
        sh = _SHAPES[qid] = query_shape(qid)
    return sh


def run_query(db, qid, config: TileConfig = TileConfig(), workers: int = 1,
              stats: Optional[QueryStats] = None, ctx: Optional[Context] = None) -> QueryResult:
    """tq::run_query (ssb_queries.hpp:76-78) on one B200.

    ``db`` is a DeviceDatabase (HBM-resident columns) or a host mapping
    {table: {column: ndarray}} -- the latter copies the query's columns H2D in
    the call, like handing the reference a host `const SsbDatabase&`."""
    config.validate()
    if workers < 1:
        raise ConfigError("run_query: workers must be >= 1")
    qid = int(qid)
    cells, ng, nj = _shape(qid)
    maxr = max(cells, 1)
    groups, sums, surv, gp, sp, vp = _out_buffers(qid, maxr)  # reused; rows are copied out below
    surv[:] = 0
    n = C.c_int64()
    if isinstance(db, DeviceDatabase):
        ctx = db.ctx
        check(LIB.crys_run_query(ctx.h, db.h, qid, config.block_threads, config.items_per_thread,
                                 gp, sp, maxr, C.byref(n), vp))
    else:
        ctx = ctx or Context.default()
        cols, keep = [], []
        for t, cs in db.items():
            for c, a in cs.items():
                a = np.ascontiguousarray(a, dtype=np.int32)
                keep.append(a)
                cols.append(_lib.crys_host_column(t.encode(), c.encode(), a.ctypes.data, len(a)))
        arr = (_lib.crys_host_column * len(cols))(*cols)
        check(LIB.crys_run_query_host(ctx.h, arr, len(cols), qid, config.block_threads,
                                      config.items_per_thread, groups.ctypes.data_as(C.c_void_p),
                                      sums.ctypes.data_as(C.c_void_p), maxr, C.byref(n),
                                      surv.ctypes.data_as(C.c_void_p)))
    if stats is not None:
        stats.survivors = [int(x) for x in surv[:max(nj, 1)]]
    return _rows_from_buffers(qid, groups, sums, n.value)


def finalize_host(qid, agg: np.ndarray, header: Optional[np.ndarray] = None) -> QueryResult:
    """Dense [sums | counts] int64 aggregate -> QueryResult, on the host.
    ``header`` (int64[CRYS_PARTIAL_HEADER], a reduced partial header) supplies
    the survivors and raises the build / group-domain errors it carries."""
    qid = int(qid)
    cells, _, nj = query_shape(qid)
    agg = np.ascontiguousarray(agg, dtype=np.int64)
    if agg.size != 2 * cells:
        raise ContractError("aggregate buffer has the wrong shape")
    hp = None
    if header is not None:
        header = np.ascontiguousarray(header, dtype=np.int64)
        if header.size != _lib.CRYS_PARTIAL_HEADER:
            raise ContractError("partial header has the wrong shape")
        hp = header.ctypes.data_as(C.c_void_p)
    maxr = max(cells, 1)
    groups = np.zeros(3 * maxr, np.int32)
    sums = np.zeros(maxr, np.int64)
    surv = np.zeros(4, np.int64)
    n = C.c_int64()
    check(LIB.crys_query_finalize_host(qid, agg.ctypes.data_as(C.c_void_p), hp,
                                       groups.ctypes.data_as(C.c_void_p),
                                       sums.ctypes.data_as(C.c_void_p), maxr, C.byref(n),
                                       surv.ctypes.data_as(C.c_void_p)))
    res = _rows_from_buffers(qid, groups, sums, n.value)
    res.survivors = [int(x) for x in surv[:max(nj, 1)]]
    return res


# ----------------------------------------------------------------- spans

def _dev(t, dtype_name: str):
    """Torch CUDA tensor -> (ptr, n).  Raises for anything else."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ContractError("expected a CUDA tensor (device span)")
    want = {"int32": torch.int32, "float32": torch.float32}[dtype_name]
    if t.dtype != want or not t.is_contiguous():
        raise ContractError(f"expected a contiguous {dtype_name} CUDA tensor")
    return t.data_ptr(), t.numel()


def _ctx_for(t) -> Context:
    ctx = Context.default(t.device.index)
    ctx.bind_torch_stream()
    return ctx


def _is_host(x) -> bool:
    return isinstance(x, np.ndarray)


def _to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _select(inp, pred: PredicateSpec, out, order: int, config: TileConfig) -> int:
    if _is_host(inp):
        d_in = _to_dev(np.asarray(inp, np.int32))
        import torch
        d_out = torch.empty_like(d_in)
        n = _select(d_in, pred, d_out, order, config)
        out[:n] = d_out[:n].cpu().numpy()
        return n
    pi, n = _dev(inp, "int32")
    po, no = _dev(out, "int32")
    if no < n:
        raise ContractError("select: output capacity too small")
    ctx = _ctx_for(inp)
    cnt = C.c_int64()
    check(LIB.crys_select_i32(ctx.h, C.c_void_p(pi), n, pred._c(), C.c_void_p(po), C.byref(cnt),
                              order, config.block_threads, config.items_per_thread))
    return cnt.value


def select_branching_into(inp, pred: PredicateSpec, out, workers: int = 1) -> int:
    """select.hpp:56-73; output in input order (the workers=1 order)."""
    if workers < 1:
        raise ConfigError("select: workers must be >= 1")
    return _select(inp, pred, out, _lib.CRYS_ORDER_INPUT, TileConfig())


def select_predicated_into(inp, pred: PredicateSpec, out, workers: int = 1) -> int:
    """select.hpp:75-91 (same output as branching)."""
    return select_branching_into(inp, pred, out, workers)


def select_per_element_into(inp, pred: PredicateSpec, out, workers: int = 1) -> int:
    """select.hpp:93-105 (input order on the GPU)."""
    return select_branching_into(inp, pred, out, workers)


def select_tile_into(inp, pred: PredicateSpec, out, config: TileConfig = TileConfig(),
                     mode: ScheduleMode = ScheduleMode.kDeterministic, workers: int = 1) -> int:
    """select.hpp:107-135.  kDeterministic: the exact Crystal order for
    `config`; kArrivalOrder only promises a permutation, so it is served by the
    same deterministic kernel."""
    config.validate()
    if workers < 1:
        raise ConfigError("run_kernel: workers must be >= 1")
    return _select(inp, pred, out, _lib.CRYS_ORDER_CRYSTAL, config)


def block_ops_run(column, pred: PredicateSpec, config: TileConfig) -> Dict[str, np.ndarray]:
    """The Crystal device primitives over `column` (a CUDA int32 tensor), one
    logical tile per CTA (crys_block_ops_run): per tile the compacted tile
    (BlockLoad -> BlockPred -> BlockScan -> BlockShuffle -> BlockStore), the
    per-logical-thread counts and exclusive prefixes, the match total and
    BlockAggregate SUM/COUNT/MIN/MAX over the matches and over all valid
    slots.  Returned as host arrays (test / inspection API)."""
    import torch
    config.validate()
    pi, n = _dev(column, "int32")
    bt, ipt = config.block_threads, config.items_per_thread
    tiles = (n + bt * ipt - 1) // (bt * ipt)
    dev = column.device
    out = torch.zeros(tiles * bt * ipt, dtype=torch.int32, device=dev)
    counts = torch.zeros(tiles * bt, dtype=torch.int64, device=dev)
    prefix = torch.zeros(tiles * bt, dtype=torch.int64, device=dev)
    totals = torch.zeros(tiles, dtype=torch.int64, device=dev)
    aggs = torch.zeros(tiles * 8, dtype=torch.int64, device=dev)
    ctx = _ctx_for(column)
    check(LIB.crys_block_ops_run(ctx.h, C.c_void_p(pi), n, bt, ipt, pred._c(), C.c_void_p(out.data_ptr()),
                                 C.c_void_p(counts.data_ptr()), C.c_void_p(prefix.data_ptr()),
                                 C.c_void_p(totals.data_ptr()), C.c_void_p(aggs.data_ptr())))
    return {"out": out.cpu().numpy().reshape(tiles, bt * ipt), "counts": counts.cpu().numpy().reshape(tiles, bt),
            "prefix": prefix.cpu().numpy().reshape(tiles, bt), "totals": totals.cpu().numpy(),
            "aggs": aggs.cpu().numpy().reshape(tiles, 8)}


def stream_read_gbs(buf, reps: int = 5) -> float:
    """Measured read-only HBM bandwidth over a CUDA tensor (crys_stream_read_gbs)."""
    ctx = _ctx_for(buf)
    g = C.c_double()
    check(LIB.crys_stream_read_gbs(ctx.h, C.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size(),
                                   int(reps), C.byref(g)))
    return g.value


def _project(x1, x2, a, b, out, sigmoid, config):
    config.validate()
    if _is_host(x1):
        d1, d2 = _to_dev(np.asarray(x1, np.float32)), _to_dev(np.asarray(x2, np.float32))
        import torch
        do = torch.empty_like(d1)
        _project(d1, d2, a, b, do, sigmoid, config)
        out[:len(x1)] = do.cpu().numpy()
        return
    p1, n1 = _dev(x1, "float32")
    p2, n2 = _dev(x2, "float32")
    po, no = _dev(out, "float32")
    if n1 != n2:
        raise ConfigError("project: input length mismatch")
    if no < n1:
        raise ContractError("project: output capacity too small")
    ctx = _ctx_for(x1)
    check(LIB.crys_project_f32(ctx.h, C.c_void_p(p1), C.c_void_p(p2), n1, float(a), float(b),
                               C.c_void_p(po), 1 if sigmoid else 0, config.block_threads,
                               config.items_per_thread))


def project_linear_into(x1, x2, a, b, out, config: TileConfig = TileConfig(), workers: int = 1):
    """project.hpp:49-54."""
    _project(x1, x2, a, b, out, False, config)


def project_sigmoid_into(x1, x2, a, b, out, config: TileConfig = TileConfig(), workers: int = 1):
    """project.hpp:56-64."""
    _project(x1, x2, a, b, out, True, config)


class HashTable:
    """hash_table.hpp:21-63 -- device-resident, interleaved {key,payload} slots."""
    kEmptyKey = -(2 ** 31)
    kFibonacci = 2654435769

    def __init__(self, ctx: Context, handle, size: int):
        self.ctx = ctx
        self.h = handle
        self._size = size

    @classmethod
    def build(cls, keys, payloads, capacity: int, workers: int = 1) -> "HashTable":
        if _is_host(keys):
            return cls.build(_to_dev(np.asarray(keys, np.int32)), _to_dev(np.asarray(payloads, np.int32)),
                             capacity, workers)
        pk, nk = _dev(keys, "int32")
        pp, npay = _dev(payloads, "int32")
        if nk != npay:
            raise ConfigError("HashTable: key/payload length mismatch")
        ctx = _ctx_for(keys)
        h = C.c_void_p()
        check(LIB.crys_ht_build(ctx.h, C.c_void_p(pk), C.c_void_p(pp), nk, int(capacity), C.byref(h)))
        return cls(ctx, h, nk)

    def capacity(self) -> int:
        return LIB.crys_ht_capacity(self.h)

    def size(self) -> int:
        return self._size

    def slots(self) -> Tuple[np.ndarray, np.ndarray]:
        cap = self.capacity()
        k = np.empty(cap, np.int32)
        p = np.empty(cap, np.int32)
        check(LIB.crys_ht_download(self.h, k.ctypes.data_as(C.c_void_p), p.ctypes.data_as(C.c_void_p)))
        return k, p

    def free(self) -> None:
        if self.h:
            LIB.crys_ht_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def join_probe_tile(probe_keys, probe_payloads, table: HashTable, config: TileConfig = TileConfig(),
                    workers: int = 1) -> int:
    """join.cpp:69-96: sum over hits of (build payload + probe payload)."""
    config.validate()
    if _is_host(probe_keys):
        return join_probe_tile(_to_dev(np.asarray(probe_keys, np.int32)),
                               _to_dev(np.asarray(probe_payloads, np.int32)), table, config, workers)
    pk, nk = _dev(probe_keys, "int32")
    pp, npay = _dev(probe_payloads, "int32")
    if nk != npay:
        raise ConfigError("join probe: key/payload length mismatch")
    if workers < 1:
        raise ConfigError("join probe: workers must be >= 1")
    ctx = _ctx_for(probe_keys)
    out = C.c_int64()
    check(LIB.crys_join_probe_sum(ctx.h, C.c_void_p(pk), C.c_void_p(pp), nk, table.h,
                                  config.block_threads, config.items_per_thread, C.byref(out)))
    return out.value


def join_probe_scalar(probe_keys, probe_payloads, table: HashTable, workers: int = 1) -> int:
    return join_probe_tile(probe_keys, probe_payloads, table, TileConfig(), workers)


def join_probe_prefetch(probe_keys, probe_payloads, table: HashTable, workers: int = 1,
                        distance: int = 16) -> int:
    if distance < 1:
        raise ConfigError("join probe: prefetch distance must be >= 1")
    return join_probe_tile(probe_keys, probe_payloads, table, TileConfig(), workers)


def _sort(keys, payloads, algo, bits):
    if _is_host(keys):
        dk, dp = _to_dev(np.asarray(keys, np.int32)), _to_dev(np.asarray(payloads, np.int32))
        _sort(dk, dp, algo, bits)
        keys[:] = dk.cpu().numpy()
        payloads[:] = dp.cpu().numpy()
        return
    pk, nk = _dev(keys, "int32")
    pp, npay = _dev(payloads, "int32")
    if nk != npay:
        raise ContractError("radix sort: key/payload length mismatch")
    ctx = _ctx_for(keys)
    check(LIB.crys_sort_pairs(ctx.h, C.c_void_p(pk), C.c_void_p(pp), nk, algo, bits))


def lsb_radix_sort(keys, payloads, workers: int = 1, bits_per_pass: int = 8) -> None:
    """radix.cpp:138-163: stable, == std::stable_sort by key (in place)."""
    if not 1 <= bits_per_pass <= 8:
        raise ConfigError("lsb_radix_sort: bits_per_pass must be in [1,8]")
    _sort(keys, payloads, _lib.CRYS_SORT_LSB, bits_per_pass)


def msb_radix_sort(keys, payloads, workers: int = 1) -> None:
    """radix.cpp:210-216: keys ascending, (key, payload) pairs preserved."""
    _sort(keys, payloads, _lib.CRYS_SORT_MSB, 8)


def radix_histogram(keys, start_bit: int, num_bits: int, num_owners: int = 1) -> np.ndarray:
    """radix_histogram (radix.cpp:33-53) on the device: counts[owner][digit],
    owner = contiguous chunk of ceil(n / num_owners) keys."""
    pk, n = _dev(keys, "int32")
    if not (1 <= num_bits <= 8 and start_bit >= 0 and start_bit + num_bits <= 32):
        raise ConfigError("RadixPass: bit range exceeds 32-bit keys")
    out = np.zeros((int(num_owners), 1 << int(num_bits)), np.int64)
    ctx = _ctx_for(keys)
    check(LIB.crys_radix_histogram(ctx.h, C.c_void_p(pk), n, int(start_bit), int(num_bits), int(num_owners),
                                   out.ctypes.data_as(C.c_void_p)))
    return out


def radix_partition(keys, payloads, out_keys, out_payloads, start_bit: int, num_bits: int) -> None:
    """radix_shuffle with a stable pass (radix.cpp:75-136): the pairs stably
    partitioned by digit, out of place, on the device."""
    pk, n = _dev(keys, "int32")
    pp, n2 = _dev(payloads, "int32")
    ok, n3 = _dev(out_keys, "int32")
    op, n4 = _dev(out_payloads, "int32")
    if not n == n2 == n3 == n4:
        raise ContractError("radix partition: length mismatch")
    ctx = _ctx_for(keys)
    check(LIB.crys_radix_partition(ctx.h, C.c_void_p(pk), C.c_void_p(pp), n, int(start_bit), int(num_bits),
                                   C.c_void_p(ok), C.c_void_p(op)))
