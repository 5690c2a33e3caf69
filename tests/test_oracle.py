"""CPU: pin the plain-C oracle (oracle/bnmc_oracle.c) against the reference.

* golden vectors produced by the unmodified reference (tests/golden, made by
  tests/golden/make_golden.py through oracle/_ref);
* the reference's own known-answer tests (proj/tests/test_*.cpp), re-expressed;
* randomized cross-checks against oracle/_ref when it is built here.
"""
import hashlib
import itertools
import math

import numpy as np
import pytest

from oracle import port, ref

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------ golden vectors
@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_port_table_matches_reference_golden(name, golden, golden_meta):
    g = golden(name)
    meta = golden_meta[name]
    assert sha(g["cells"]) == meta["cells_sha256"]
    t = port.cache_build(g["cells"], g["cards"], meta["k"])
    assert sha(t) == meta["table_sha256"]
    np.testing.assert_array_equal(t.view(np.uint64), g["table"].view(np.uint64))


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_port_order_scores_match_golden(name, golden, golden_meta):
    g = golden(name)
    pri = g.get("priors")
    for perm, mk, tot in zip(g["orders"], g["order_masks"], g["order_totals"]):
        m, b, t = port.score_order(g["table"], golden_meta[name]["k"], perm, pri)
        np.testing.assert_array_equal(m, mk)
        assert t == tot
        assert math.fsum(b) == pytest.approx(t, rel=1e-12)


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_port_chain_matches_golden_trace(name, golden, golden_meta):
    g = golden(name)
    meta = golden_meta[name]
    r = port.run_mcmc(g["table"], meta["k"], meta["iterations"], meta["seed"], g.get("priors"))
    np.testing.assert_array_equal(r["trace_proposed"], g["trace_proposed"])
    np.testing.assert_array_equal(r["trace_accepted"], g["trace_accepted"])
    np.testing.assert_array_equal(r["trace_best"], g["trace_best"])
    np.testing.assert_array_equal(r["final_order"], g["final_order"])
    np.testing.assert_array_equal(r["tracker_masks"], g["tracker_masks"])
    np.testing.assert_array_equal(r["tracker_totals"], g["tracker_totals"])
    assert r["accepted"] == meta["accepted"] and r["final_score"] == meta["final_score"]


def test_tie_fixture_golden(golden_meta):
    tf = golden_meta["tie_fixture"]
    n, s = tf["n"], tf["s"]
    t = port.cache_build(np.zeros((0, n), np.uint8), [3] * n, s, gamma=1.0)
    assert not t.any()
    m, b, tot = port.score_order(t, s, tf["perm"])
    assert [int(x) for x in m] == tf["masks"] and tot == tf["total"]


# ------------------------------------------- reference known-answer tests
def test_binomial_and_counts():  # test_combinatorics.cpp:10-17, 59-68
    assert port.binomial(6, 4) == 15 and port.binomial(59, 4) == 455126
    assert port.binomial(5, 0) == 1 and port.binomial(3, 7) == 0
    for n_ in range(0, 65):
        for k in range(0, n_ + 1):
            assert port.binomial(n_, k) == math.comb(n_, k)
    assert port.bounded_subset_count(6, 4) == 57


def test_global_index_worked_values():  # test_combinatorics.cpp:59-68
    bit = lambda *xs: sum(1 << x for x in xs)
    assert port.global_index(bit(0, 1, 2, 3), 6, 4) == 0
    assert port.global_index(bit(0, 1, 2, 4), 6, 4) == 1
    assert port.global_index(bit(0, 1, 2, 5), 6, 4) == 2
    assert port.global_index(bit(0, 1, 3, 4), 6, 4) == 3
    assert port.global_index(bit(5), 6, 4) == 55
    assert port.global_index(0, 6, 4) == 56


@pytest.mark.parametrize("c", range(0, 13))
def test_global_index_bijection(c):  # test_combinatorics.cpp:70-88
    pst = port.build_pst(c, 4)
    assert len(pst) == port.bounded_subset_count(c, 4)
    for g, m in enumerate(pst):
        assert port.global_index(int(m), c, 4) == g
        assert port.subset_at(g, c, 4) == int(m)
    # lexicographic within sizes, sizes descending
    expect = [sum(1 << x for x in comb) for k in range(min(4, c), 0, -1)
              for comb in itertools.combinations(range(c), k)] + [0]
    assert [int(x) for x in pst] == expect


def test_pst_rows():  # test_combinatorics.cpp:126-142
    t = port.build_pst(6, 4)
    assert len(t) == 57 and t[0] == 0b1111 and t[1] == 0b10111 and t[55] == 1 << 5 and t[56] == 0
    tiny = port.build_pst(1, 4)
    assert list(tiny) == [1, 0]


def test_count_statistics_kats():  # test_scoring.cpp:31-67
    d = np.zeros((0, 2), np.uint8)
    t = port.count_statistics(d, [2, 2], 0, 1 << 1)
    assert t.shape == (2, 2) and not t.any()
    d = np.array([[0], [1], [1]], np.uint8)
    t = port.count_statistics(d, [2], 0, 0)
    assert t.tolist() == [[1, 2]]
    d = np.array([[0, 0, 0], [0, 1, 1], [1, 0, 1], [1, 1, 0]], np.uint8)
    t = port.count_statistics(d, [2, 2, 2], 2, 0b11)
    for k in range(4):
        v0, v1 = k & 1, k >> 1
        assert t[k, v0 ^ v1] == 1 and t[k, 1 - (v0 ^ v1)] == 0
    with pytest.raises(port.OracleError):
        port.count_statistics(np.zeros((1, 2), np.uint8), [2, 2], 0, 0b1)


def test_local_score_closed_forms():  # test_scoring.cpp:69-118
    d3 = np.zeros((0, 3), np.uint8)
    assert port.local_score(d3, [2, 2, 2], 0, 0, 0.1, 1.0) == 0.0
    assert port.local_score(d3, [2, 2, 2], 0, 0b110, 0.1, 1.0) == pytest.approx(
        2 * math.log10(0.1), rel=1e-14)
    assert port.local_score(np.array([[0], [1]], np.uint8), [2], 0, 0, 1.0, 1.0) == pytest.approx(
        math.log10(1 / 8), rel=1e-12)
    d = np.array([[0], [1], [1]], np.uint8)
    assert port.local_score(d, [2], 0, 0, 1.0, 1.0) == pytest.approx(math.log10(1 / 16), rel=1e-12)
    assert port.local_score(d, [2], 0, 0, 1.0, 1.0, k2=True) == pytest.approx(
        math.log10(1 / 12), rel=1e-12)


def test_ppf_values():  # test_scoring.cpp:120-129, acceptance.cpp:483-519
    assert port.ppf(0.5) == 0.0 and port.ppf(1.0) == 12.5 and port.ppf(0.0) == -12.5
    assert port.ppf(0.2) == pytest.approx(-2.7, rel=1e-12)


def test_exhaustive_n4_orders_dominate_graphs():  # test_scoring.cpp:310-338, criterion 1
    rng = np.random.default_rng(1234)
    cells = rng.integers(0, 2, (60, 4)).astype(np.uint8)
    t = port.cache_build(cells, [2] * 4, 3)
    pri = np.full((4, 4), 0.5)
    pri[1, 0], pri[3, 2] = 0.75, 0.2
    w = np.where(np.eye(4, dtype=bool), 0.0, 100.0 * (pri - 0.5) ** 3)

    def eff(v, ps):  # effective_local_score, ascending parents from the lookup
        tot = t[v, port.index_of(4, 3, v, ps)]
        for p in range(4):
            if ps >> p & 1:
                tot += w[v, p]
        return tot
    best_order = max(port.score_order(t, 3, perm, pri)[2]
                     for perm in itertools.permutations(range(4)))
    best_graph = -np.inf
    for parents in itertools.product(range(16), repeat=4):  # all DAGs on 4 nodes
        if any(parents[v] >> v & 1 for v in range(4)):
            continue
        # acyclic check via repeated removal of parentless nodes
        left, ok = set(range(4)), True
        while left and ok:
            free = [v for v in left if not any(parents[v] >> p & 1 for p in left)]
            ok = bool(free)
            left -= set(free)
        if not ok:
            continue
        tot = 0.0
        for v in range(4):
            tot += eff(v, parents[v])
        best_graph = max(best_graph, tot)
    assert best_order == pytest.approx(best_graph, rel=1e-12)


# ---------------------------------------------- cross-checks vs reference
@needs_ref
def test_rng_streams_match_reference():
    o = port.lib()
    for seed, tag in [(0, -1), (7, 2), (12345, 3), (2**63 + 5, 101)]:
        u = ref.rng_stream(seed, tag, 0, 64)
        # restate with the port: split then next_u64
        import ctypes as C
        class R(C.Structure):
            _fields_ = [("state", C.c_uint64)]
        o.orc_rng_make.restype = R
        o.orc_rng_make.argtypes = [C.c_uint64]
        o.orc_rng_split.restype = R
        o.orc_rng_split.argtypes = [C.POINTER(R), C.c_uint64]
        o.orc_next_u64.restype = C.c_uint64
        o.orc_next_u64.argtypes = [C.POINTER(R)]
        r = o.orc_rng_make(seed)
        if tag >= 0:
            r = o.orc_rng_split(C.byref(r), tag)
        mine = [o.orc_next_u64(C.byref(r)) for _ in range(64)]
        assert mine == [int(x) for x in u]


@needs_ref
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_counts_and_scores_vs_reference(seed):
    rng = np.random.default_rng(seed)
    n = 7
    cards = rng.integers(2, 5, n).astype(np.int32)
    cells = (rng.integers(0, 1 << 30, (300, n)) % cards).astype(np.uint8)
    for _ in range(40):
        node = int(rng.integers(n))
        ps = int(rng.integers(1 << n)) & ~(1 << node) & ((1 << n) - 1)
        np.testing.assert_array_equal(port.count_statistics(cells, cards, node, ps),
                                      ref.count_statistics(cells, cards, node, ps))
        for k2 in (False, True):
            a = port.local_score(cells, cards, node, ps, 0.3, 2.5, k2)
            b = ref.local_score(cells, cards, node, ps, 0.3, 2.5, k2)
            assert a == b


@needs_ref
def test_sparse_count_path_vs_reference():
    """r*card above 2^22 takes the reference's std::map path (scoring.cpp:13)."""
    n = 6
    cards = np.array([256, 256, 200, 3, 2, 2], np.int32)
    rng = np.random.default_rng(5)
    cells = (rng.integers(0, 1 << 30, (500, n)) % cards).astype(np.uint8)
    ps = 0b111
    assert port.local_score(cells, cards, 3, ps) == ref.local_score(cells, cards, 3, ps)


@needs_ref
@pytest.mark.parametrize("strict", [False, True])
def test_chain_vs_reference_small(strict):
    cards = [2] * 6
    cells, truth = ref.generate(6, 3, 120, cards, seed=33, edge_prob=0.4, concentration=0.5,
                                tags=(1, 2, 3))
    cache = ref.Cache.build(cells, cards, 4)
    pri = np.full((6, 6), 0.5)
    pri[3, 1], pri[4, 2] = 0.85, 0.15
    r = ref.run_mcmc(cells, cards, 4, 300, 1234, priors=pri, strict=strict, prebuilt=cache,
                     debug_recheck=True)
    o = port.run_mcmc(cache.table(), 4, 300, 1234, pri, strict=strict)
    np.testing.assert_array_equal(o["trace_proposed"], r.trace_proposed)
    np.testing.assert_array_equal(o["trace_best"], r.trace_best)
    np.testing.assert_array_equal(o["tracker_masks"], r.tracker_masks)
    assert o["accepted"] == r.accepted


@needs_ref
def test_parallel_engine_equals_serial_reference():
    """The reference's own invariance (test_engine.cpp:153-185) holds for the port."""
    cells, truth = ref.generate(9, 3, 150, [2] * 9, seed=42, tags=(1, 2, 3))
    cache = ref.Cache.build(cells, [2] * 9, 4)
    pri = np.full((9, 9), 0.5)
    pri[3, 1], pri[7, 2] = 0.85, 0.15
    rng = np.random.default_rng(77)
    for _ in range(10):
        perm = rng.permutation(9).astype(np.int32)
        m_ref, t_ref = cache.score_order(perm, pri)
        for workers, tasks, pst in [(1, 0, True), (3, 7, False), (8, 1, True)]:
            m, t = ref.Scorer(cache, pri, workers, tasks, pst).score(perm)
            np.testing.assert_array_equal(m, m_ref)
            assert t == t_ref
        m, b, t = port.score_order(cache.table(), 4, perm, pri)
        np.testing.assert_array_equal(m, m_ref)
        assert t == t_ref
