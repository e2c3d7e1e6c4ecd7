"""Flight 1 (q1.1-q1.3) under every autotuner candidate (CRYS_F1_CAND=k:
the register-tile kernel and the TMA-ring kernels of ssb_flight1.cuh, with
one or two dense ring columns, vector or striped row ownership) against the
reference's goldens: the fixture (a partial tile), SF=1 and SF=20, plus a
lineorder cut into ragged shards that are summed on the device.  The knob is
read once per process, so each candidate runs in a child process."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_CANDIDATES = 8  # kTuneF1 in csrc/ssb_query.cu

CHILD = r"""
import json, sys
sys.path.insert(0, %(root)r); sys.path.insert(0, %(tests)r)
from helpers import QUERY_NAMES, fixture_tables, golden, golden_rows
from paper_2003_01178_b200 import tq
out = {}
for name, make in (("fixture", lambda: tq.DeviceDatabase.from_host(fixture_tables())),
                   ("sf1", lambda: tq.DeviceDatabase.generate(1, 42)),
                   ("sf20", lambda: tq.DeviceDatabase.generate(20, 42))):
    db = make()
    for q in range(3):
        rec = golden(name)["queries"][QUERY_NAMES[q]]
        ok = True
        for rep in range(3):  # direct run, graph capture, replay
            st = tq.QueryStats()
            r = tq.run_query(db, q, tq.TileConfig(), 1, st)
            ok = ok and r.as_tuples() == golden_rows(rec) and st.survivors == rec["survivors"][:len(st.survivors)]
        out.setdefault(name, {})[QUERY_NAMES[q]] = ok
    db.free()
print(json.dumps(out))
"""


@pytest.mark.parametrize("cand", list(range(N_CANDIDATES)))
def test_flight1_candidates_match_goldens(cand):
    code = CHILD % {"root": ROOT, "tests": os.path.join(ROOT, "tests")}
    env = dict(os.environ, CRYS_F1_CAND=str(cand))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    bad = [(db, q) for db, qs in res.items() for q, ok in qs.items() if not ok]
    assert not bad, bad
    assert len(res["sf20"]) == 3, res
