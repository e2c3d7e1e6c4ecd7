"""Split SSB plans (csrc/ssb_scan.cuh or, with CRYS_BM=1, ssb_scanbm.cuh +
ssb_gather.cuh: the first D joins streamed densely into a survivor list, the
rest of the plan gathered at the listed rows) forced for every join query
with CRYS_SPLIT=D, D in {1, 2, 3},
against the reference's goldens (fixture, SF=1, SF=20).  The knob is read
once per process, so each D runs in a child process; the autotuner picks
split plans by itself in the default configuration."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

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
    for q in range(3, 13):
        if %(split)d >= tq.query_shape(q)[2]:
            continue
        rec = golden(name)["queries"][QUERY_NAMES[q]]
        for rep in range(2):  # direct run, then graph capture
            st = tq.QueryStats()
            r = tq.run_query(db, q, tq.TileConfig(), 1, st)
            ok = r.as_tuples() == golden_rows(rec) and st.survivors == rec["survivors"][:len(st.survivors)]
            out.setdefault(name, {})[QUERY_NAMES[q]] = out.get(name, {}).get(QUERY_NAMES[q], True) and ok
    db.free()
print(json.dumps(out))
"""


@pytest.mark.parametrize("bm", [0, 1])
@pytest.mark.parametrize("split", [1, 2, 3])
def test_split_plans_match_goldens(split, bm):
    """bm=1: the late-materialising head (membership bitmaps, ssb_scanbm.cuh)
    with the uint4 survivor list and the digit joins resolved in the gather."""
    code = CHILD % {"root": ROOT, "tests": os.path.join(ROOT, "tests"), "split": split}
    env = dict(os.environ, CRYS_SPLIT=str(split), CRYS_BM=str(bm))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    bad = [(db, q) for db, qs in res.items() for q, ok in qs.items() if not ok]
    assert not bad, bad
    assert res["sf20"], res
