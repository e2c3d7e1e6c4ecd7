"""The cost-model restatement (paper_2003_01178_b200/cost_models.py) against
the reference's own cost_models.cpp outputs (tests/golden/cost_models.json,
produced by tests/golden/make_cost_golden.sh)."""
import math

import pytest

from helpers import golden
from paper_2003_01178_b200 import cost_models as cm

B200_GOLDEN = cm.HardwareProfile("b200", 6539.9e9, 6539.9e9, 32, [cm.CacheLevel(126e6, 12e12)])
PROFILES = {"table2-cpu": cm.HardwareProfile.table2_cpu(), "table2-gpu": cm.HardwareProfile.table2_gpu(),
            "b200": B200_GOLDEN}


def _run(rec):
    a = rec["args"]
    p = PROFILES[a["profile"]]
    m = rec["model"]
    if m == "project":
        return cm.model_project(a["n"], p)
    if m == "select":
        return cm.model_select(a["n"], a["sigma"], p)
    if m == "sort":
        return cm.model_sort(a["n"], a["passes"], p)
    if m == "join_probe":
        return cm.model_join_probe(a["p"], a["ht_bytes"], p)
    if m == "q21":
        return cm.model_q21(cm.Q21Params.ssb_sf20(), p, a["target"])
    raise AssertionError(m)


@pytest.mark.parametrize("i", range(len(golden("cost_models"))))
def test_models_match_reference(i):
    rec = golden("cost_models")[i]
    est = _run(rec)
    assert math.isclose(est.total_seconds, rec["total_seconds"], rel_tol=1e-12, abs_tol=1e-30), rec
    assert [t for t, _ in est.terms] == [t for t, _ in rec["terms"]]
    for (_, a), (_, b) in zip(est.terms, rec["terms"]):
        assert math.isclose(a, b, rel_tol=1e-12, abs_tol=1e-30)


def test_validation_errors():
    with pytest.raises(cm.ConfigError):
        cm.model_select(10, 1.5, B200_GOLDEN)
    with pytest.raises(cm.ConfigError):
        cm.model_sort(10, 0, B200_GOLDEN)
    with pytest.raises(cm.ConfigError):
        cm.model_join_probe(10, 8192, cm.HardwareProfile("x", 1e9, 1e9, 64, []))
    with pytest.raises(cm.ConfigError):
        cm.HardwareProfile("x", 0, 1e9).validate()


def test_ssb_bound_is_16L_and_24L():
    p = cm.b200_profile()
    rows = 120_000_000
    assert math.isclose(cm.model_ssb_query(0, rows, p).total_seconds, 16 * rows / p.read_bw)
    assert math.isclose(cm.model_ssb_query(12, rows, p).total_seconds, 24 * rows / p.read_bw)
