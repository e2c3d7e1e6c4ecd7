"""Every input-order select instantiation (CRYS_SEL_RR round-robin variants,
the segmented launches CRYS_SEL_CFG=2, count/scan/write CFG=3) gives the
input-order result, and both Crystal-order paths (round-robin, and
count/scan/write with CRYS_SEL_RRC=0) give the Crystal order: the knobs are read once per process, so each runs in a
subprocess.  Reference = the boolean-mask gather x[pred(x)], which keeps
input order (select.hpp:56-73, workers=1)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, torch
sys.path.insert(0, %r)
from paper_2003_01178_b200 import tq
g = torch.Generator(device="cuda").manual_seed(5)
for n in (1, 3, 4096, 4099, 4096 * 148 * 5 + 13, (1 << 24) + 7):
    x = torch.randint(-1000, 1000, (n,), dtype=torch.int32, device="cuda", generator=g)
    out = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    for lo in (-1001, 0, 999):
        k = tq.select_branching_into(x, tq.PredicateSpec.lt(lo), out)
        ref = x[x < lo]
        assert k == ref.numel() and torch.equal(out[:k], ref), (n, lo)
    k = tq.select_branching_into(x[1:], tq.PredicateSpec.between(-5, 400), out)  # misaligned span
    ref = x[1:][(x[1:] >= -5) & (x[1:] <= 400)]
    assert k == ref.numel() and torch.equal(out[:k], ref), n
    # Crystal order (select.hpp:107-135): slot j*S + t + k*bt, output thread-major per logical tile
    for bt, ipt in ((128, 4), (32, 1), (256, 8), (64, 16), (96, 2), (3, 5)):
        S = bt * ipt
        tiles = (n + S - 1) // S
        pad = torch.full((tiles * S,), 5000, dtype=torch.int32, device="cuda")  # never selected
        pad[:n] = x
        v = pad.view(tiles, ipt, bt).transpose(1, 2).reshape(-1)
        for lo in (-1001, 0, 999):
            k = tq.select_tile_into(x, tq.PredicateSpec.lt(lo), out, tq.TileConfig(bt, ipt))
            ref = v[v < lo]
            assert k == ref.numel() and torch.equal(out[:k], ref), (n, bt, ipt, lo)
print("ok")
""" % ROOT


@pytest.mark.parametrize("env", [{"CRYS_SEL_RR": "0"}, {"CRYS_SEL_RR": "1"}, {"CRYS_SEL_RR": "2"}, {"CRYS_SEL_RR": "3"},
                                 {"CRYS_SEL_RR": "4"}, {"CRYS_SEL_RR": "5"}, {"CRYS_SEL_RR": "6"},
                                 {"CRYS_SEL_RR": "7"}, {"CRYS_SEL_RR": "8"}, {"CRYS_SEL_RR": "9"}, {"CRYS_SEL_RR": "10"},
                                 {"CRYS_SEL_RR": "11"}, {"CRYS_SEL_RR": "12"}, {"CRYS_SEL_RR": "13"}, {"CRYS_SEL_RRC_WS": "0"}, {"CRYS_SEL_CFG": "2"}, {"CRYS_SEL_CFG": "3"},
                                 {"CRYS_SEL_RRC": "0"}])
def test_input_order_variants(env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
