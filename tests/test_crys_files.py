"""CRYS column files (the reference's column_io format, column_io.hpp:3-13).

tests/golden/crys_fixture/ and crys_*.col were written by the reference's OWN
save_database / save_column (tests/golden/make_crys_golden.sh).  CPU tests pin
the format against fixture.json; GPU tests load them through
crys_db_load_column_file and run the queries, round-trip SF=1 through
save/load, and check the IoError paths."""
import json
import os

import numpy as np
import pytest

from helpers import GOLDEN, QUERY_NAMES, fixture_tables, golden, golden_rows

FIX = os.path.join(GOLDEN, "crys_fixture")


def read_crys(path):
    """Format restatement (column_io.cpp:65-100) -- test infrastructure."""
    raw = open(path, "rb").read()
    assert raw[:4] == b"CRYS" and int.from_bytes(raw[4:6], "little") == 1
    kind = raw[6]
    n = int.from_bytes(raw[8:16], "little")
    assert len(raw) == 16 + 4 * n
    return kind, np.frombuffer(raw[16:], np.int32 if kind == 0 else np.float32)


def test_reference_files_match_fixture():
    man = json.load(open(os.path.join(FIX, "manifest.json")))
    assert man["format"] == "crys-manifest" and man["version"] == 1
    tabs = fixture_tables()
    for t, cols in tabs.items():
        listed = {c["name"]: c for c in man["tables"][t]["columns"]}
        assert set(listed) == set(cols)
        for c, v in cols.items():
            kind, got = read_crys(os.path.join(FIX, listed[c]["file"]))
            assert kind == 0 and listed[c]["length"] == len(v)
            assert np.array_equal(got, v)
    kind, f = read_crys(os.path.join(GOLDEN, "crys_float.col"))
    assert kind == 1 and f.tolist() == [1.5, -2.25, 3.0]


@pytest.fixture(scope="module")
def tq():
    from paper_2003_01178_b200 import tq as _tq
    return _tq


@pytest.mark.gpu
def test_load_reference_database_and_query(tq):
    db = tq.load_database(FIX)
    for q in range(13):
        rec = golden("fixture")["queries"][QUERY_NAMES[q]]
        stats = tq.QueryStats()
        assert tq.run_query(db, q, tq.TileConfig(), 1, stats).as_tuples() == golden_rows(rec), QUERY_NAMES[q]
        assert stats.survivors == rec["survivors"]
    db.free()


@pytest.mark.gpu
def test_load_errors(tq):
    db = tq.DeviceDatabase.from_host({})
    for name, msg in (("crys_badmagic.col", "bad magic"), ("crys_truncated.col", "truncated payload"),
                      ("crys_float.col", "kind mismatch"), ("no_such_file.col", "cannot open")):
        with pytest.raises(tq.IoError, match=msg):
            db.load_column_file("part", "p_mfgr", os.path.join(GOLDEN, name))
    db.free()
    with pytest.raises(tq.IoError):
        tq.load_database(os.path.join(GOLDEN, "no_such_dir"))


@pytest.mark.gpu
def test_sf1_save_load_round_trip(tq, tmp_path):
    src = tq.DeviceDatabase.generate(1, 42)
    tq.save_database(src, str(tmp_path), 1, 42)
    # a file we wrote reads back through the format restatement
    kind, v = read_crys(str(tmp_path / "supplier.s_region.col"))
    assert kind == 0 and np.array_equal(v, src.download("supplier", "s_region"))
    db = tq.load_database(str(tmp_path))
    for q in (0, 3, 6, 12):
        rec = golden("sf1")["queries"][QUERY_NAMES[q]]
        assert tq.run_query(db, q).as_tuples() == golden_rows(rec), QUERY_NAMES[q]
    src.free()
    db.free()
