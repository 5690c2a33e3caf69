"""GPU: the reference's full count-table range. Entries whose joint
configuration space exceeds K1's dense shared-memory counter (the reference
switches CountTable to an ordered map above 2^22 cells, scoring.cpp:13, 53-80)
are scored by K1W (precompute_wide.cuh); tables and count tables are
bit-exact with the unmodified reference (oracle/_ref)."""
import numpy as np
import pytest

import paper_1210_5128_b200 as P
from paper_1210_5128_b200 import _lib
from oracle import ref

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def instance(seed, cards, m, skew=0.0):
    rng = np.random.default_rng(seed)
    cards = np.asarray(cards, np.int32)
    n = cards.size
    cells = np.empty((m, n), np.uint8)
    for j, c in enumerate(cards):
        if skew > 0:  # few active configurations: most rows share low states
            p = np.exp(-skew * np.arange(c))
            cells[:, j] = rng.choice(c, size=m, p=p / p.sum())
        else:
            cells[:, j] = rng.integers(0, c, m)
    # correlated columns so joint configurations repeat
    for j in range(1, n):
        mask = rng.random(m) < 0.4
        cells[mask, j] = cells[mask, j - 1] % cards[j]
    return cells, cards


CASES = {
    "3state_s7": ([3] * 10, 7, 400, 0.0),
    "3state_s8": ([3] * 10, 8, 300, 0.0),
    "6state_s4": ([6] * 8, 4, 500, 0.0),
    "10state_s4": ([10] * 7, 4, 600, 0.5),
    "col256": ([3, 3, 256, 3, 2, 4, 3], 3, 700, 0.0),
    "mixed_s5": ([2, 9, 4, 7, 3, 10, 5, 2, 6], 5, 500, 0.3),
    "256_all": ([256] * 5, 4, 64, 0.0),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_wide_tables_bit_exact_vs_reference(name):
    cards, s, m, skew = CASES[name]
    cells, cards = instance(sum(map(ord, name)), cards, m, skew)
    for mode, gamma, ess in ((P.AlphaMode.BDEU, 0.1, 1.0), (P.AlphaMode.K2, 0.4, 1.0)):
        cfg = P.RunConfig(max_parents=s, gamma=gamma, ess=ess, alpha_mode=mode,
                          memory_cap_bytes=(1 << 64) - 1)
        cache = P.ScoreCache.build(P.Dataset(cards, cells), cfg)
        t = cache.table()
        k1, wide = P.api.C.c_float(), P.api.C.c_uint64()
        _lib.check(_lib.lib().bnmc_gpu_table_k1_stats(cache.handle, P.api.C.byref(k1),
                                                       P.api.C.byref(wide), None, None))
        assert wide.value > 0, "instance should exercise the wide path"
        r = ref.Cache.build(cells, cards, s, gamma, ess, k2=mode == P.AlphaMode.K2).table()
        np.testing.assert_array_equal(t.view(np.uint64), r.view(np.uint64))


def test_wide_path_with_zero_rows():
    cards = np.array([3] * 9, np.int32)
    cfg = P.RunConfig(max_parents=8, memory_cap_bytes=(1 << 64) - 1)
    t = P.ScoreCache.build(P.Dataset(cards, np.zeros((0, 9), np.uint8)), cfg).table()
    r = ref.Cache.build(np.zeros((0, 9), np.uint8), cards, 8).table()
    np.testing.assert_array_equal(t.view(np.uint64), r.view(np.uint64))


def test_configuration_overflow_is_a_capacity_error():
    cards = np.array([256] * 9, np.int32)  # 8 parents of 256 states: 2^64 configurations
    cells = np.zeros((3, 9), np.uint8)
    with pytest.raises(P.CapacityError, match="overflows 64 bits"):
        P.ScoreCache.build(P.Dataset(cards, cells),
                           P.RunConfig(max_parents=8, memory_cap_bytes=(1 << 64) - 1))
    with pytest.raises(P.CapacityError):
        P.count_statistics(P.Dataset(cards, cells), 0, 0x1FE)


@pytest.mark.parametrize("cards,node,pset,m", [
    ([3] * 12, 0, 0b111111111110, 500),       # 3^11 x 3 cells: sparse
    ([10] * 8, 3, 0b11110111, 800),           # 10^7 x 10: sparse
    ([3, 256, 256, 256, 4], 4, 0b1110, 300),  # 2^24 x 4: sparse
    ([3, 3, 3, 3], 2, 0b1011, 200),           # dense
    ([256] * 4, 0, 0b1110, 0),                # no rows
])
def test_count_statistics_dense_and_sparse_match_reference(cards, node, pset, m):
    cells, cards = instance(5, cards, m)
    d = P.Dataset(cards, cells)
    t = P.count_statistics(d, node, pset)
    cfg, cnt = ref.count_statistics_active(cells, cards, node, pset)
    got = list(t.for_each_active())
    assert [k for k, _ in got] == [int(x) for x in cfg]
    for (k, row), want in zip(got, cnt):
        np.testing.assert_array_equal(np.asarray(row), want)
    assert t.samples() == m
    r = int(np.prod([int(cards[p]) for p in range(len(cards)) if pset >> p & 1], dtype=object))
    assert t.configs() == r
    assert t.is_dense() == (r * int(cards[node]) <= 1 << 22)
