"""The reference's OWN unit-test suites (P:tests/test_*.cpp, unmodified,
compiled by dropin/Makefile into oracle/_ref/dropin/) run against the B200
drop-in: src/{ssb_queries,hash_table,join,radix}.cpp and include/tq/{select,
project}.hpp replaced by dropin/, which calls libcrystal_b200.so.

The binaries are built in the container that has /root/reference (build())
and ship to the GPU box with the snapshot; each must report 0 failed cases."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin")
SUITES = ["test_ssb", "test_hash_join", "test_radix", "test_select", "test_project", "test_tile_engine"]
# the drop-in's own suite (dropin/tests/): workers -> device groups, upload cache
OWN_SUITES = ["test_dropin_group"]


def _binary(suite):
    p = os.path.join(BIN, suite)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (needs /root/reference at build time: make -C dropin)")
    return p


def _run(suite, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([_binary(suite)], capture_output=True, text=True, timeout=900, env=e)
    summary = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert summary, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.returncode == 0 and summary.group(3) == "0", r.stdout[-4000:] + r.stderr[-4000:]


@pytest.mark.gpu
def test_reference_ssb_suite_sharded_workers():
    """The reference's test_ssb with every `workers` value (1, 2, 3, 4) run as
    that many lineorder shards (device group; emulated on one GPU)."""
    _run("test_ssb", {"CRYS_GROUP_EMULATE": "1"})


@pytest.mark.gpu
@pytest.mark.parametrize("suite", OWN_SUITES)
def test_dropin_own_suite_passes_on_b200(suite):
    _run(suite)


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_b200(suite):
    r = subprocess.run([_binary(suite)], capture_output=True, text=True, timeout=900)
    summary = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert summary, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.returncode == 0 and summary.group(3) == "0", r.stderr[-4000:]


@pytest.mark.parametrize("suite", SUITES + OWN_SUITES)
def test_dropin_binaries_bind_the_b200_library(suite):
    """The replaced symbols come from dropin/ and the compute from
    libcrystal_b200.so (no reference implementation of them is linked)."""
    p = _binary(suite)
    ldd = subprocess.run(["ldd", p], capture_output=True, text=True).stdout
    assert "libcrystal_b200.so" in ldd and "not found" not in ldd
    syms = subprocess.run(["nm", "-C", p], capture_output=True, text=True).stdout
    assert "crys_init" in syms  # bound through the C ABI
