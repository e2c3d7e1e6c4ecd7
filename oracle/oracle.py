"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the parity checkers.

* ``Oracle``  -> ``oracle/liboracle.so``: my plain-C restatement (oracle.c).
* ``RefImpl`` -> ``oracle/_ref/libtqref.so``: the reference's own C++ hot path
  compiled from /root/reference/proj (oracle/Makefile), used to pin goldens
  and as the CPU arm of bench.py.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(``paper_2003_01178_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
I64P = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")

QUERY_NAMES = ["q11", "q12", "q13", "q21", "q22", "q23", "q31", "q32", "q33", "q34",
               "q41", "q42", "q43"]
LO_COLS = ["lo_orderdate", "lo_custkey", "lo_suppkey", "lo_partkey", "lo_quantity",
           "lo_discount", "lo_extendedprice", "lo_revenue", "lo_supplycost"]
DIM_COLS = {
    "date": ["d_datekey", "d_year", "d_yearmonthnum", "d_yearmonth", "d_weeknuminyear"],
    "supplier": ["s_suppkey", "s_city", "s_nation", "s_region"],
    "customer": ["c_custkey", "c_city", "c_nation", "c_region"],
    "part": ["p_partkey", "p_brand1", "p_category", "p_mfgr"],
}
OPS = {"lt": 0, "le": 1, "gt": 2, "ge": 3, "eq": 4, "between": 5}


class OrcDB(C.Structure):
    _fields_ = [("lo_rows", C.c_int64), ("date_rows", C.c_int64), ("supp_rows", C.c_int64),
                ("cust_rows", C.c_int64), ("part_rows", C.c_int64),
                ("lo", C.c_void_p * 9), ("date", C.c_void_p * 5), ("supp", C.c_void_p * 4),
                ("cust", C.c_void_p * 4), ("part", C.c_void_p * 4)]


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise RuntimeError(f"checker library {path} not built (run __graft_entry__.build())")
    return C.CDLL(path)


class Oracle:
    """The plain-C restatement (oracle/oracle.c)."""

    def __init__(self):
        L = self.L = _load(os.path.join(HERE, "liboracle.so"))
        L.orc_rng_base.restype = C.c_uint64
        L.orc_rng_base.argtypes = [C.c_uint64] * 4
        L.orc_random_i32.argtypes = [I32P, C.c_int64, C.c_uint64, C.c_uint64, C.c_int32, C.c_int32]
        L.orc_project_inputs.argtypes = [F32P, F32P, C.c_int64, C.c_uint64]
        for f in ("orc_lineorder_rows", "orc_supplier_rows", "orc_customer_rows", "orc_part_rows"):
            getattr(L, f).restype = C.c_int64
            getattr(L, f).argtypes = [C.c_int64]
        L.orc_gen_date.argtypes = [I32P]
        L.orc_gen_geo.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_int64, I32P]
        L.orc_gen_part.argtypes = [C.c_int64, C.c_uint64, C.c_int64, I32P]
        L.orc_gen_lineorder_col.argtypes = [C.c_int64, C.c_uint64, C.c_int, C.c_int64,
                                            C.c_int64, I32P, C.c_int]
        L.orc_query_cells.restype = C.c_int64
        L.orc_query_cells.argtypes = [C.c_int]
        L.orc_query_ngroup.argtypes = [C.c_int]
        L.orc_query_partial.argtypes = [C.POINTER(OrcDB), C.c_int, C.c_int64, C.c_int64,
                                        I64P, I64P, I64P]
        L.orc_query.restype = C.c_int64
        L.orc_query.argtypes = [C.POINTER(OrcDB), C.c_int, I32P, I64P, C.c_int64, I64P]
        L.orc_cell_key.argtypes = [C.c_int, C.c_int64, I32P]
        L.orc_ht_build.argtypes = [I32P, I32P, C.c_int64, C.c_int64, I32P, I32P]
        L.orc_join_checksum.restype = C.c_int64
        L.orc_join_checksum.argtypes = [I32P, I32P, C.c_int64, I32P, I32P, C.c_int64]
        for f in ("orc_select_input_order",):
            getattr(L, f).restype = C.c_int64
            getattr(L, f).argtypes = [I32P, C.c_int64, C.c_int, C.c_int32, C.c_int32, I32P]
        L.orc_select_crystal_order.restype = C.c_int64
        L.orc_select_crystal_order.argtypes = [I32P, C.c_int64, C.c_int, C.c_int32, C.c_int32,
                                               C.c_int, C.c_int, I32P]
        for f in ("orc_project_linear", "orc_project_sigmoid"):
            getattr(L, f).argtypes = [F32P, F32P, C.c_int64, C.c_float, C.c_float, F32P]
        L.orc_radix_digit.restype = C.c_uint32
        L.orc_radix_digit.argtypes = [C.c_int32, C.c_int, C.c_int]
        L.orc_lsb_sort.argtypes = [I32P, I32P, C.c_int64, C.c_int]

    # -- generators -------------------------------------------------------
    def random_i32(self, n, seed, stream, lo, hi):
        out = np.empty(n, np.int32)
        self.L.orc_random_i32(out, n, seed, stream, lo, hi)
        return out

    def project_inputs(self, n, seed=42):
        x1 = np.empty(n, np.float32)
        x2 = np.empty(n, np.float32)
        self.L.orc_project_inputs(x1, x2, n, seed)
        return x1, x2

    def generate(self, sf, seed=42, lo_begin=0, lo_end=None, nthreads=None):
        """Host SSB database as {table: {column: ndarray}} (ssb_gen.cpp:243-270)."""
        L = self.L
        nthreads = nthreads or os.cpu_count() or 1
        db = {}
        d = np.empty(5 * 2556, np.int32)
        L.orc_gen_date(d)
        db["date"] = {c: d[i * 2556:(i + 1) * 2556].copy() for i, c in enumerate(DIM_COLS["date"])}
        for name, tid, rows in (("supplier", 3, L.orc_supplier_rows(sf)),
                                ("customer", 4, L.orc_customer_rows(sf))):
            buf = np.empty(4 * rows, np.int32)
            L.orc_gen_geo(tid, sf, seed, rows, buf)
            db[name] = {c: buf[i * rows:(i + 1) * rows].copy() for i, c in enumerate(DIM_COLS[name])}
        rows = L.orc_part_rows(sf)
        buf = np.empty(4 * rows, np.int32)
        L.orc_gen_part(sf, seed, rows, buf)
        db["part"] = {c: buf[i * rows:(i + 1) * rows].copy() for i, c in enumerate(DIM_COLS["part"])}
        n = L.orc_lineorder_rows(sf)
        lo_end = n if lo_end is None else lo_end
        db["lineorder"] = {}
        for cid, c in enumerate(LO_COLS):
            out = np.empty(lo_end - lo_begin, np.int32)
            L.orc_gen_lineorder_col(sf, seed, cid, lo_begin, lo_end, out, nthreads)
            db["lineorder"][c] = out
        return db

    # -- SSB ----------------------------------------------------------------
    @staticmethod
    def make_orcdb(db):
        s = OrcDB()
        keep = []

        def ptr(a):
            a = np.ascontiguousarray(a, dtype=np.int32)
            keep.append(a)
            return a.ctypes.data

        s.lo_rows = len(db["lineorder"]["lo_orderdate"])
        s.date_rows = len(db["date"]["d_datekey"])
        s.supp_rows = len(db["supplier"]["s_suppkey"])
        s.cust_rows = len(db["customer"]["c_custkey"])
        s.part_rows = len(db["part"]["p_partkey"])
        for i, c in enumerate(LO_COLS):
            s.lo[i] = ptr(db["lineorder"][c])
        for fld, t in (("date", "date"), ("supp", "supplier"), ("cust", "customer"), ("part", "part")):
            arr = getattr(s, fld)
            for i, c in enumerate(DIM_COLS[t]):
                arr[i] = ptr(db[t][c])
        s._keep = keep
        return s

    def cells(self, qid):
        return self.L.orc_query_cells(qid)

    def ngroup(self, qid):
        return self.L.orc_query_ngroup(qid)

    def partial(self, db, qid, begin, end, sums=None, counts=None):
        cells = self.cells(qid)
        sums = np.zeros(cells, np.int64) if sums is None else sums
        counts = np.zeros(cells, np.int64) if counts is None else counts
        surv = np.zeros(4, np.int64)
        s = self.make_orcdb(db)
        rc = self.L.orc_query_partial(C.byref(s), qid, begin, end, sums, counts, surv)
        if rc:
            raise RuntimeError(f"oracle partial failed rc={rc}")
        return sums, counts, surv

    def query(self, db, qid):
        """-> (rows [(group tuple, sum)], survivors list)"""
        cells = self.cells(qid)
        maxr = max(cells, 1)
        groups = np.zeros(3 * maxr, np.int32)
        sums = np.zeros(maxr, np.int64)
        surv = np.zeros(4, np.int64)
        s = self.make_orcdb(db)
        n = self.L.orc_query(C.byref(s), qid, groups, sums, maxr, surv)
        if n < 0:
            raise RuntimeError(f"oracle query failed rc={n}")
        ng = self.ngroup(qid)
        rows = [(tuple(int(x) for x in groups[3 * i:3 * i + ng]), int(sums[i])) for i in range(n)]
        njoins = 1 if qid < 3 else (3 if qid < 10 else 4)
        return rows, [int(x) for x in surv[:njoins]]

    def cell_key(self, qid, cell):
        v = np.zeros(3, np.int32)
        self.L.orc_cell_key(qid, cell, v)
        return tuple(int(x) for x in v[:self.ngroup(qid)])

    # -- operators ----------------------------------------------------------
    def ht_build(self, keys, payloads, capacity):
        sk = np.empty(capacity, np.int32)
        sp = np.empty(capacity, np.int32)
        rc = self.L.orc_ht_build(np.ascontiguousarray(keys, np.int32),
                                 np.ascontiguousarray(payloads, np.int32), len(keys), capacity, sk, sp)
        return rc, sk, sp

    def join_checksum(self, pk, pp, sk, sp):
        return self.L.orc_join_checksum(pk, pp, len(pk), sk, sp, len(sk))

    def select(self, x, op, lo, hi=0, order="input", bt=128, ipt=4):
        out = np.empty(max(len(x), 1), np.int32)
        if order == "input":
            n = self.L.orc_select_input_order(x, len(x), OPS[op], lo, hi, out)
        else:
            n = self.L.orc_select_crystal_order(x, len(x), OPS[op], lo, hi, bt, ipt, out)
        return out[:n]

    def project(self, x1, x2, a, b, sigmoid=False):
        out = np.empty(len(x1), np.float32)
        f = self.L.orc_project_sigmoid if sigmoid else self.L.orc_project_linear
        f(x1, x2, len(x1), a, b, out)
        return out

    def lsb_sort(self, keys, payloads, bits=8):
        k = np.array(keys, np.int32)
        p = np.array(payloads, np.int32)
        self.L.orc_lsb_sort(k, p, len(k), bits)
        return k, p


class RefImpl:
    """The reference's own hot path (oracle/_ref/libtqref.so)."""

    def __init__(self):
        L = self.L = _load(os.path.join(HERE, "_ref", "libtqref.so"))
        L.tqref_last_error.restype = C.c_char_p
        L.tqref_generate.restype = C.c_void_p
        L.tqref_generate.argtypes = [C.c_int64, C.c_uint64]
        L.tqref_db_empty.restype = C.c_void_p
        L.tqref_db_set_column.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, I32P, C.c_int64]
        L.tqref_db_free.argtypes = [C.c_void_p]
        L.tqref_db_column.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p,
                                      C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.c_int64)]
        L.tqref_query.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  I32P, I64P, C.c_int64, C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int32), I64P, C.POINTER(C.c_int32),
                                  C.POINTER(C.c_double)]
        L.tqref_select.restype = C.c_int64
        L.tqref_select.argtypes = [C.c_int, I32P, C.c_int64, C.c_int, C.c_int32, C.c_int32,
                                   I32P, C.c_int, C.c_int, C.c_int, C.c_int]
        L.tqref_project.argtypes = [C.c_int, F32P, F32P, C.c_int64, C.c_float, C.c_float, F32P,
                                    C.c_int, C.c_int, C.c_int]
        L.tqref_ht_build.restype = C.c_void_p
        L.tqref_ht_build.argtypes = [I32P, I32P, C.c_int64, C.c_int64, C.c_int,
                                     C.POINTER(C.c_int)]
        L.tqref_ht_slots.argtypes = [C.c_void_p, C.POINTER(C.POINTER(C.c_int32)),
                                     C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.c_int64)]
        L.tqref_ht_free.argtypes = [C.c_void_p]
        L.tqref_join_probe.argtypes = [C.c_int, I32P, I32P, C.c_int64, C.c_void_p, C.c_int,
                                       C.c_int, C.c_int, C.POINTER(C.c_int64)]
        L.tqref_sort.argtypes = [C.c_int, I32P, I32P, C.c_int64, C.c_int, C.c_int]

    def error(self):
        return self.L.tqref_last_error().decode()

    def generate(self, sf, seed=42):
        h = self.L.tqref_generate(sf, seed)
        if not h:
            raise RuntimeError(self.error())
        return h

    def db_from_tables(self, db):
        h = self.L.tqref_db_empty()
        for t, cols in db.items():
            for c, a in cols.items():
                a = np.ascontiguousarray(a, np.int32)
                self.L.tqref_db_set_column(h, t.encode(), c.encode(), a, len(a))
        return h

    def free(self, h):
        self.L.tqref_db_free(h)

    def column(self, h, table, col):
        p = C.POINTER(C.c_int32)()
        n = C.c_int64()
        rc = self.L.tqref_db_column(h, table.encode(), col.encode(), C.byref(p), C.byref(n))
        if rc:
            raise RuntimeError(self.error())
        return np.ctypeslib.as_array(p, shape=(n.value,)).copy() if n.value else np.zeros(0, np.int32)

    def tables(self, h):
        out = {"lineorder": {c: self.column(h, "lineorder", c) for c in LO_COLS}}
        for t, cols in DIM_COLS.items():
            out[t] = {c: self.column(h, t, c) for c in cols}
        return out

    def query(self, h, qid, reference=True, bt=128, ipt=4, workers=1, max_rows=2_000_000):
        groups = np.zeros(3 * max_rows, np.int32)
        sums = np.zeros(max_rows, np.int64)
        surv = np.zeros(4, np.int64)
        nrows = C.c_int64()
        ng = C.c_int32()
        ns = C.c_int32()
        ms = C.c_double()
        rc = self.L.tqref_query(h, qid, 1 if reference else 0, bt, ipt, workers, groups, sums,
                                max_rows, C.byref(nrows), C.byref(ng), surv, C.byref(ns),
                                C.byref(ms))
        if rc:
            raise RuntimeError(f"rc={rc}: {self.error()}")
        g = ng.value
        rows = [(tuple(int(x) for x in groups[3 * i:3 * i + g]), int(sums[i]))
                for i in range(nrows.value)]
        return rows, [int(x) for x in surv[:ns.value]], ms.value

    def select(self, variant, x, op, lo, hi=0, bt=128, ipt=4, mode=0, workers=1):
        out = np.empty(max(len(x), 1), np.int32)
        n = self.L.tqref_select(variant, x, len(x), OPS[op], lo, hi, out, bt, ipt, mode, workers)
        if n < 0:
            raise RuntimeError(self.error())
        return out[:n]

    def project(self, x1, x2, a, b, sigmoid=False, bt=128, ipt=4, workers=1):
        out = np.empty(len(x1), np.float32)
        rc = self.L.tqref_project(1 if sigmoid else 0, x1, x2, len(x1), a, b, out, bt, ipt, workers)
        if rc:
            raise RuntimeError(self.error())
        return out

    def ht_build(self, keys, payloads, capacity, workers=1):
        st = C.c_int()
        h = self.L.tqref_ht_build(np.ascontiguousarray(keys, np.int32),
                                  np.ascontiguousarray(payloads, np.int32), len(keys), capacity,
                                  workers, C.byref(st))
        return st.value, h

    def ht_slots(self, h):
        k = C.POINTER(C.c_int32)()
        p = C.POINTER(C.c_int32)()
        cap = C.c_int64()
        self.L.tqref_ht_slots(h, C.byref(k), C.byref(p), C.byref(cap))
        return (np.ctypeslib.as_array(k, shape=(cap.value,)).copy(),
                np.ctypeslib.as_array(p, shape=(cap.value,)).copy())

    def ht_free(self, h):
        self.L.tqref_ht_free(h)

    def join_probe(self, h, pk, pp, variant=0, bt=128, ipt=4, workers=1):
        out = C.c_int64()
        rc = self.L.tqref_join_probe(variant, pk, pp, len(pk), h, bt, ipt, workers, C.byref(out))
        if rc:
            raise RuntimeError(self.error())
        return out.value

    def sort(self, keys, payloads, msb=False, workers=1, bits=8):
        rc = self.L.tqref_sort(1 if msb else 0, keys, payloads, len(keys), workers, bits)
        if rc:
            raise RuntimeError(self.error())


def block_ops(column, bt, ipt, lo, hi):
    """Restatement of the reference's block primitives for every tile of
    `column` (P:include/tq/block_ops.hpp): block_load (:23-32), block_pred
    with an inclusive [lo, hi] predicate (:54-69), block_thread_counts +
    block_scan (:73-96), block_shuffle (:101-122) and block_aggregate
    SUM/COUNT/MIN/MAX (:141-173; i64 accumulation, identities 0/0/INT32_MAX/
    INT32_MIN), masked by the flags and over all valid slots.  Same layout as
    tq.block_ops_run.  Pure Python loops: small inputs only."""
    x = np.asarray(column, np.int64)
    n = len(x)
    S = bt * ipt
    tiles = (n + S - 1) // S
    out = np.zeros((tiles, S), np.int32)
    counts = np.zeros((tiles, bt), np.int64)
    prefix = np.zeros((tiles, bt), np.int64)
    totals = np.zeros(tiles, np.int64)
    aggs = np.zeros((tiles, 8), np.int64)
    imax, imin = 2 ** 31 - 1, -2 ** 31
    for b in range(tiles):
        tile = x[b * S:min(n, (b + 1) * S)]
        valid = len(tile)
        flags = (tile >= lo) & (tile <= hi)
        for t in range(bt):
            counts[b, t] = int(flags[t:valid:bt].sum())
        prefix[b] = np.concatenate([[0], np.cumsum(counts[b])[:-1]])
        totals[b] = counts[b].sum()
        pos = 0
        for t in range(bt):
            for i in range(t, valid, bt):
                if flags[i]:
                    out[b, pos] = tile[i]
                    pos += 1
        for j, m in enumerate((flags, np.ones(valid, bool))):
            v = tile[m]
            aggs[b, 4 * j:4 * j + 4] = [int(v.sum()), len(v), int(v.min()) if len(v) else imax,
                                        int(v.max()) if len(v) else imin]
    return {"out": out, "counts": counts, "prefix": prefix, "totals": totals, "aggs": aggs}


def fnv_rows(rows):
    """FNV-1a-64 over result rows (SURVEY.md Appendix A definition)."""
    h = 1469598103934665603
    P = 1099511628211
    M = (1 << 64) - 1

    def feed(h, v):
        for b in int(v & M).to_bytes(8, "little"):
            h ^= b
            h = (h * P) & M
        return h

    for group, s in rows:
        for v in group:
            h = feed(h, v & 0xFFFFFFFF)
        h = feed(h, s)
    return f"{h:016x}"


def sort_digest(keys, payloads, stride=4097):
    """SURVEY.md A.4 LSB-sort sample digest (word-wise FNV over every 4097th pair)."""
    h = 1469598103934665603
    P = 1099511628211
    M = (1 << 64) - 1
    k = np.asarray(keys)[::stride].astype(np.int64) & 0xFFFFFFFF
    p = np.asarray(payloads)[::stride].astype(np.int64) & 0xFFFFFFFF
    for a, b in zip(k.tolist(), p.tolist()):
        h ^= a
        h = (h * P) & M
        h ^= b
        h = (h * P) & M
    return f"{h:016x}"
