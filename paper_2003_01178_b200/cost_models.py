"""Bandwidth-saturation cost models of the paper, with a B200 profile.

Restates the reference's cost models (P = /root/reference/proj):
``model_project`` / ``model_select`` / ``model_join_probe`` / ``model_sort`` /
``model_q21`` (src/cost_models.cpp:131-269, include/tq/cost_models.hpp) term by
term, so a measured time can be reported as a fraction of the model, as the
reference's ``--model`` / ``--compare-model`` do (tools/tq_main.cpp:226-243,
:323-326).  Pinned against the reference's own implementation by
tests/golden/cost_models.json (tests/golden/make_cost_golden.sh).

``b200_profile()`` fills the profile from MEASURED_PEAKS.json (read = write =
the measured HBM copy bandwidth), 32 B DRAM sectors, and the 126 MB L2 as the
last cache level.  ``model_ssb_query`` is the SSB bound the paper uses: the
fact columns a plan references streamed once (16 B/row for q1-q3, 24 B/row
for q4; PAPER section 3.1's 16L bound), with q2.1 alternatively given by
``model_q21`` (gpu_like).
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class ConfigError(ValueError):
    pass


def _check(cond: bool, msg: str) -> None:
    if not cond:
        raise ConfigError(msg)


@dataclass
class CacheLevel:
    size_bytes: float
    bandwidth_bytes_per_sec: Optional[float] = None  # None: never binds (cost_models.hpp:18-23)


@dataclass
class HardwareProfile:
    label: str
    read_bw: float
    write_bw: float
    cache_line_bytes: float = 64
    cache_levels: List[CacheLevel] = field(default_factory=list)
    interconnect_bw: Optional[float] = None

    def validate(self) -> None:  # cost_models.cpp:28-42
        _check(self.read_bw > 0, "profile read_bw must be > 0")
        _check(self.write_bw > 0, "profile write_bw must be > 0")
        _check(self.cache_line_bytes > 0, "profile cache_line_bytes must be > 0")
        prev = 0.0
        for lv in self.cache_levels:
            _check(lv.size_bytes > prev, "cache level sizes must be positive and strictly increasing")
            if lv.bandwidth_bytes_per_sec is not None:
                _check(lv.bandwidth_bytes_per_sec > 0, "cache level bandwidth must be > 0 when given")
            prev = lv.size_bytes
        if self.interconnect_bw is not None:
            _check(self.interconnect_bw > 0, "interconnect_bw must be > 0")

    @staticmethod
    def table2_cpu() -> "HardwareProfile":  # cost_models.cpp:44-53
        return HardwareProfile("table2-cpu", 53e9, 55e9, 64, [CacheLevel(256e3), CacheLevel(20e6, 157e9)], 12.8e9)

    @staticmethod
    def table2_gpu() -> "HardwareProfile":  # cost_models.cpp:55-64
        return HardwareProfile("table2-gpu", 880e9, 880e9, 128, [CacheLevel(6e6)], 12.8e9)


@dataclass
class CostEstimate:
    terms: List[Tuple[str, float]]
    total_seconds: float

    @property
    def total_ms(self) -> float:
        return self.total_seconds * 1e3


def _finish(terms) -> CostEstimate:  # cost_models.cpp:15-20
    return CostEstimate(list(terms), float(sum(t for _, t in terms)))


def _clamp01(x: float) -> float:
    return min(1.0, max(0.0, x))


# L2 bandwidth used for the B200 profile's last cache level: the LTS
# throughput cap (~6300 B/cycle at ~1.9 GHz, /opt/skills/guides/B300_MICROARCH.md
# L2 section), i.e. where L2-resident hash probes bind.
B200_L2_BYTES = 126e6
B200_L2_BW = 12e12


def b200_profile(cache_line_bytes: float = 32) -> HardwareProfile:
    hbm, _ = hbm_peak()
    return HardwareProfile("b200", hbm * 1e9, hbm * 1e9, cache_line_bytes,
                           [CacheLevel(B200_L2_BYTES, B200_L2_BW)], None)


def hbm_peak() -> Tuple[float, str]:
    """(GB/s, 'measured' | 'fallback') -- MEASURED_PEAKS.json, else the
    B200_PROFILING.md fallback."""
    try:
        with open(os.path.join(_ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ models

def model_project(n: int, p: HardwareProfile) -> CostEstimate:  # cost_models.cpp:131-137
    p.validate()
    _check(n >= 0, "element count must be >= 0")
    dn = float(n)
    return _finish([("read two columns", 8 * dn / p.read_bw), ("write result column", 4 * dn / p.write_bw)])


def model_select(n: int, sigma: float, p: HardwareProfile) -> CostEstimate:  # :139-146
    p.validate()
    _check(n >= 0, "element count must be >= 0")
    _check(0 <= sigma <= 1, "sigma must lie in [0,1]")
    dn = float(n)
    return _finish([("read input column", 4 * dn / p.read_bw), ("write matches", 4 * sigma * dn / p.write_bw)])


def model_join_probe(probe_count: int, ht_bytes: float, p: HardwareProfile) -> CostEstimate:  # :148-187
    p.validate()
    _check(probe_count >= 0, "probe count must be >= 0")
    _check(ht_bytes > 0, "hash table size must be > 0")
    _check(len(p.cache_levels) > 0, "join probe model needs cache levels in the profile")
    pc = float(probe_count)
    c = p.cache_line_bytes
    scan = 8 * pc / p.read_bw
    levels = p.cache_levels
    fit = len(levels)
    for k, lv in enumerate(levels):
        if ht_bytes <= lv.size_bytes:
            fit = k
            break
    if fit < len(levels):
        hit_below = 0.0 if fit == 0 else _clamp01(levels[fit - 1].size_bytes / ht_bytes)
        probe = 0.0
        if levels[fit].bandwidth_bytes_per_sec is not None:
            probe = (1 - hit_below) * pc * c / levels[fit].bandwidth_bytes_per_sec
        if probe > scan:
            return _finish([("cache line fetches", probe)])
        return _finish([("probe column scan", scan)])
    hit = _clamp01(levels[-1].size_bytes / ht_bytes)
    return _finish([("probe column scan", scan), ("memory line fetches", (1 - hit) * pc * c / p.read_bw)])


def model_sort(n: int, passes: int, p: HardwareProfile) -> CostEstimate:  # :189-198
    p.validate()
    _check(n >= 0, "element count must be >= 0")
    _check(passes >= 1, "pass count must be >= 1")
    dn, k = float(n), float(passes)
    return _finish([("histogram reads", k * 4 * dn / p.read_bw), ("shuffle reads", k * 8 * dn / p.read_bw),
                    ("shuffle writes", k * 8 * dn / p.write_bw)])


@dataclass
class Q21Params:  # cost_models.hpp:85-95
    l: float = 0
    s: float = 0
    p: float = 0
    d: float = 0
    sigma1: float = 0
    sigma2: float = 0
    part_ht_bytes: float = 0

    @staticmethod
    def ssb_sf20() -> "Q21Params":  # cost_models.cpp:212-222
        return Q21Params(120e6, 40e3, 1e6, 2500, 1.0 / 5.0, 1.0 / 25.0, 8e6)


def model_q21(q: Q21Params, p: HardwareProfile, target: str = "gpu_like") -> CostEstimate:  # :224-269
    p.validate()
    _check(q.l > 0 and q.s > 0 and q.p > 0 and q.d > 0, "q21 cardinalities must be > 0")
    _check(0 <= q.sigma1 <= 1 and 0 <= q.sigma2 <= 1, "q21 selectivities must lie in [0,1]")
    _check(q.part_ht_bytes > 0, "part hash table size must be > 0")
    c, br, bw = p.cache_line_bytes, p.read_bw, p.write_bw
    survivors1 = q.l * q.sigma1
    survivors2 = survivors1 * q.sigma2
    full_scan_lines = 4 * q.l / c
    r1 = (full_scan_lines + min(full_scan_lines, survivors1) + 2 * min(full_scan_lines, survivors2)) * c / br
    if target == "cpu_like":
        r2 = (2 * q.s + 2 * q.d + 2 * q.p) * c / br
    else:
        _check(len(p.cache_levels) > 0, "gpu_like q21 needs cache levels in the profile")
        resident = 8 * (q.s + q.d)
        available = p.cache_levels[-1].size_bytes - resident
        pi = _clamp01(available / q.part_ht_bytes)
        r2 = (2 * q.s + 2 * q.d + (1 - pi) * survivors1) * c / br
    r3 = survivors2 * c / br + survivors2 * c / bw
    return _finish([("fact column reads", r1), ("hash table probes", r2), ("result table traffic", r3)])


# Fact columns each SSB plan streams (ssb_queries.cpp:184-199, :237-251).
SSB_FACT_COLS = [4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 6, 6, 6]


def model_ssb_query(qid: int, lineorder_rows: int, p: HardwareProfile) -> CostEstimate:
    """The paper's bandwidth-saturation bound for one SSB query: every fact
    column the plan references read once (PAPER 3.1, 16L for q1.x)."""
    p.validate()
    cols = SSB_FACT_COLS[int(qid)]
    return _finish([(f"{cols} fact columns", 4.0 * cols * lineorder_rows / p.read_bw)])
