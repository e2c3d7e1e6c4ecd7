"""CPU-side checks of the product library: the C ABI loads and exports every
declared symbol, and the host logic (plans, result compaction, error mapping,
API validation) behaves like the reference.  No kernel runs here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from helpers import QUERY_NAMES, golden, golden_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "crystal_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(crys_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2003_01178_b200 import _lib
    names = declared_symbols()
    assert len(names) >= 25
    lib = C.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_library_is_sm100a():
    import subprocess
    from paper_2003_01178_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_query_shapes_match_reference_domains():
    from paper_2003_01178_b200 import tq
    # Appendix A.2 / ssb_plans.cpp group parts
    cells = [tq.query_shape(q)[0] for q in range(13)]
    assert cells == [1, 1, 1, 7000, 7000, 7000, 4375, 437500, 437500, 437500, 175, 4375, 1750000]
    assert [tq.query_shape(q)[2] for q in range(13)] == [0, 0, 0, 3, 3, 3, 3, 3, 3, 3, 4, 4, 4]
    with pytest.raises(tq.ConfigError):
        tq.query_shape(13)


def test_query_names_round_trip():
    # test_ssb.cpp "query names round-trip"
    from paper_2003_01178_b200 import tq
    ids = tq.all_query_ids()
    assert len(ids) == 13
    for i in ids:
        assert tq.query_id_from_name(tq.query_name(i)) == i
    assert tq.query_id_from_name("q21") == tq.QueryId.kQ21
    with pytest.raises(tq.ConfigError):
        tq.query_id_from_name("q99")


@pytest.mark.parametrize("q", range(13))
def test_finalize_host_matches_oracle(q):
    """Dense partial (oracle) -> product compaction -> reference rows (SF=1)."""
    from oracle.oracle import Oracle
    from paper_2003_01178_b200 import tq
    orc = Oracle()
    db = _sf1(orc)
    s, c, _ = orc.partial(db, q, 0, len(db["lineorder"]["lo_orderdate"]))
    res = tq.finalize_host(q, np.concatenate([s, c]))
    assert res.as_tuples() == golden_rows(golden("sf1")["queries"][QUERY_NAMES[q]])


_SF1 = {}


def _sf1(orc):
    if "db" not in _SF1:
        _SF1["db"] = orc.generate(1, 42)
    return _SF1["db"]


def test_finalize_host_occupancy_not_sum():
    """A group whose sum is 0 but which had rows is emitted (ssb_queries.cpp:32-35);
    flight 1 always emits its single row (ssb_queries.cpp:207-209)."""
    from paper_2003_01178_b200 import tq
    cells = tq.query_shape(10)[0]
    agg = np.zeros(2 * cells, np.int64)
    agg[cells + 3] = 2          # occupied, sum 0
    agg[7] = -200
    agg[cells + 7] = 1
    res = tq.finalize_host(10, agg)
    assert res.as_tuples() == [((1992, 3), 0), ((1992, 7), -200)]
    assert res.group_labels == ["d_year", "c_nation"]
    res1 = tq.finalize_host(0, np.zeros(2, np.int64))
    assert res1.as_tuples() == [((), 0)]
    res2 = tq.finalize_host(3, np.zeros(2 * 7000, np.int64))
    assert res2.rows == []


def test_api_validation_errors():
    from paper_2003_01178_b200 import tq
    with pytest.raises(tq.ConfigError):
        tq.TileConfig(0, 4).validate()
    with pytest.raises(tq.ConfigError):
        tq.TileConfig(128, 0).validate()
    tq.TileConfig(257, 8).validate()
    assert tq.TileConfig(257, 8).tile_size() == 2056
    with pytest.raises(tq.ConfigError):
        tq.PredicateSpec.between(5, 4)
    with pytest.raises(tq.ConfigError):
        tq.run_query({}, 0, tq.TileConfig(), 0)
    with pytest.raises(tq.ConfigError):
        tq.run_query({}, 0, tq.TileConfig(0, 4))
    with pytest.raises(tq.ConfigError):
        tq.lsb_radix_sort(np.zeros(4, np.int32), np.zeros(4, np.int32), bits_per_pass=9)


def test_predicate_eval():
    from paper_2003_01178_b200 import tq
    P = tq.PredicateSpec
    assert P.lt(5).eval(4) and not P.lt(5).eval(5)
    assert P.le(5).eval(5) and P.ge(5).eval(5) and P.gt(5).eval(6) and P.eq(5).eval(5)
    assert P.between(2, 4).eval(2) and P.between(2, 4).eval(4) and not P.between(2, 4).eval(5)
    assert P.lt(5).then_and().combine == tq.PredCombine.AND


def test_shard_ranges_cover():
    from paper_2003_01178_b200.dist import shard_range
    for total in (0, 1, 7, 600_000_000):
        for world in (1, 2, 3, 4, 8):
            r = [shard_range(total, k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == total
            for (a, b), (c, d) in zip(r, r[1:]):
                assert b == c and b >= a
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1


def test_nccl_loads_without_breaking_torch():
    """Device groups dlopen NCCL lazily; the package points the library at the
    libnccl torch ships, so loading it first must not break `import torch`
    (a second, older libnccl.so.2 in the process would)."""
    import subprocess
    import sys
    code = ("from paper_2003_01178_b200._lib import LIB; v = LIB.crys_nccl_version().decode(); "
            "import torch; print(v)")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().startswith("libnccl "), r.stdout
