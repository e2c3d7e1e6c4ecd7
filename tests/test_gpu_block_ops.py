"""The Crystal device primitives themselves (csrc/crystal.cuh: BlockLoad,
BlockPred, BlockScan, BlockShuffle, BlockStore, BlockAggregate) through
crys_block_ops_run, one logical tile per CTA, against the restatement of
block_ops.hpp (oracle.block_ops, pinned to the reference's worked examples in
tests/test_oracle.py): the Figure-5 tile, every sweep shape of
test_tile_engine.cpp, odd shapes and random partial tiles."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tq():
    from paper_2003_01178_b200 import tq as _tq
    return _tq


def _check(tq, col, bt, ipt, pred, lo, hi):
    import torch
    from oracle.oracle import block_ops
    got = tq.block_ops_run(torch.from_numpy(np.asarray(col, np.int32)).cuda(), pred, tq.TileConfig(bt, ipt))
    exp = block_ops(col, bt, ipt, lo, hi)
    for k in ("counts", "prefix", "totals", "aggs"):
        assert np.array_equal(got[k], exp[k]), (k, bt, ipt)
    for b, tot in enumerate(exp["totals"]):
        assert np.array_equal(got["out"][b][:tot], exp["out"][b][:tot]), (b, bt, ipt)


def test_figure5_tile(tq):
    fig5 = [9, 4, 7, 6, 4, 1, 6, 1, 3, 8, 9, 7, 6, 2, 8, 8]
    import torch
    r = tq.block_ops_run(torch.tensor(fig5, dtype=torch.int32).cuda(), tq.PredicateSpec.gt(5), tq.TileConfig(4, 4))
    assert r["counts"][0].tolist() == [2, 1, 4, 3]
    assert r["prefix"][0].tolist() == [0, 2, 3, 7]
    assert r["totals"][0] == 10
    assert r["out"][0][:10].tolist() == [9, 6, 8, 7, 6, 9, 8, 6, 7, 8]
    assert r["aggs"][0][:4].tolist() == [9 + 6 + 8 + 7 + 6 + 9 + 8 + 6 + 7 + 8, 10, 6, 9]


def test_aggregate_identities_and_wide_sums(tq):
    import torch
    vals = torch.tensor([3, -7, 12, 0, 5, 5, -2, 9], dtype=torch.int32).cuda()
    r = tq.block_ops_run(vals, tq.PredicateSpec.ge(-2 ** 31), tq.TileConfig(4, 2))
    assert r["aggs"][0][4:].tolist() == [25, 8, -7, 12]
    r = tq.block_ops_run(vals, tq.PredicateSpec.gt(100), tq.TileConfig(4, 2))
    assert r["aggs"][0][:4].tolist() == [0, 0, 2 ** 31 - 1, -2 ** 31]
    big = torch.full((8,), 2 ** 31 - 1, dtype=torch.int32).cuda()
    r = tq.block_ops_run(big, tq.PredicateSpec.ge(0), tq.TileConfig(4, 2))
    assert r["aggs"][0][0] == 8 * (2 ** 31 - 1)


@pytest.mark.parametrize("bt", [32, 64, 128, 256, 512, 1024])
@pytest.mark.parametrize("ipt", [1, 2, 4, 8])
def test_sweep_shapes_random_partial_tiles(tq, bt, ipt):
    from oracle.oracle import Oracle
    n = 3 * bt * ipt + 17  # the last tile is partial
    col = Oracle().random_i32(n, 42, 7, 0, 999)
    _check(tq, col, bt, ipt, tq.PredicateSpec.lt(400), -2 ** 31, 399)


@pytest.mark.parametrize("bt,ipt", [(3, 5), (257, 8), (1, 1), (7, 16), (100, 3)])
def test_odd_shapes(tq, bt, ipt):
    from oracle.oracle import Oracle
    n = 2 * bt * ipt + bt // 2 + 1
    col = Oracle().random_i32(n, 42, 9, -50, 50)
    _check(tq, col, bt, ipt, tq.PredicateSpec.between(-10, 20), -10, 20)
