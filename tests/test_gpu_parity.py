"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bars (BASELINE.json north_star): bit-exact cut points, bin indices, sampled row sets and their
fixed-point gradients, histograms, partitions and chosen splits; gains and leaf weights are
in fact bit-exact too (same IEEE operation order, R14) and are checked with == and, as the
stated bar, rel. error <= 1e-6; AUC after training within 1e-3 relative.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

ob = pytest.importorskip("paper_2005_09148_b200")


def _oracle_cuts_bins(X, max_bin, seed=2):
    cv, cp = oracle.cuts(X, max_bin, seed=seed)
    return cv, cp, oracle.bins(X, cv, cp)


SHAPES = [
    (1, 1, 256), (7, 3, 2), (100, 17, 16), (1000, 33, 256), (2049, 20, 256), (5000, 64, 64),
    (10000, 20, 256),  # config 1 shape
]


@pytest.mark.parametrize("n,m,max_bin", SHAPES)
@pytest.mark.parametrize("stress", [False, True])
def test_cuts_and_bins_bit_exact(ctx, n, m, max_bin, stress):
    if m < 4 and stress:
        pytest.skip("stress needs >= 4 features")
    if n >= 50 and m >= 2:
        X, _ = synth.make_classification(n, m, seed=n + m, stress=stress)
    else:
        X = np.random.default_rng(0).normal(size=(n, m)).astype(np.float32)
    cv, cp, B = _oracle_cuts_bins(X, max_bin)
    d = ctx.quantise(X, max_bin)
    gv, gp = d.get_cuts()
    np.testing.assert_array_equal(gp, cp)
    assert gv.tobytes() == cv.tobytes()
    np.testing.assert_array_equal(d.get_bins(), B)
    d.close()


def test_cuts_negative_zero_and_ties(ctx):
    X = np.array([[-0.0, 1.0], [0.0, 1.0], [2.0, 1.0], [-1.0, 1.0]] * 10, np.float32)
    cv, cp, B = _oracle_cuts_bins(X, 256)
    d = ctx.quantise(X, 256)
    gv, gp = d.get_cuts()
    assert gv.tobytes() == cv.tobytes()
    np.testing.assert_array_equal(d.get_bins(), B)
    d.close()


@pytest.mark.parametrize("n,max_bin,tie_frac", [(1003, 16, 0.5), (40001, 256, 0.5), (5000, 7, 0.7), (4099, 256, 0.6)])
def test_cuts_heavy_ties_more_than_B_distinct(ctx, n, max_bin, tie_frac):
    """R1 step 4 (ceil rank, repeats dropped) on the GPU: more than B distinct values, a large
    share of them tied on a few values, n not a multiple of B; cuts and bins bit-exact."""
    rng = np.random.default_rng(n)
    X = rng.normal(size=(n, 5)).astype(np.float32) * 4
    for j in range(5):
        k = int(n * tie_frac)
        idx = rng.choice(n, size=k, replace=False)
        X[idx, j] = rng.choice(np.array([-1.5, 0.25, 3.0, 7.75], np.float32) + j, size=k)
        assert len(np.unique(X[:, j])) > max_bin
    cv, cp, B = _oracle_cuts_bins(X, max_bin)
    assert any(cp[j + 1] - cp[j] < max_bin for j in range(5))  # some repeats were dropped
    d = ctx.quantise(X, max_bin)
    gv, gp = d.get_cuts()
    np.testing.assert_array_equal(gp, cp)
    assert gv.tobytes() == cv.tobytes()
    np.testing.assert_array_equal(d.get_bins(), B)
    d.close()


def test_nonfinite_rejected(ctx):
    """R4: +-inf is rejected; a NaN is a missing value (R27), accepted whenever the feature's bins
    leave symbol 255 free (here every feature has one bin)."""
    X = np.ones((10, 3), np.float32)
    X[4, 1] = np.inf
    with pytest.raises(ob.OocgbError) as e:
        ctx.quantise(X, 256)
    assert e.value.status == ob.ERR_ARG
    X[4, 1] = np.nan
    d = ctx.quantise(X, 256)
    assert d.info()["has_missing"] == 1 and d.get_bins()[4, 1] == 255
    d.close()


def test_sketch_sample_large_n(ctx):
    """n_global > 2^20: the sketch is the Philox row sample (R2), independent of pushing order."""
    n, m = (1 << 20) + 4096, 4
    rng = np.random.default_rng(5)
    X = rng.normal(size=(n, m)).astype(np.float32)
    X[:, 3] = np.round(X[:, 3] * 3)  # few distinct values
    cv, cp = oracle.cuts(X, 256, seed=9)
    d = ctx.sketch_begin(m, 256, n, seed=9)
    half = n // 2
    d.sketch_push(X[half:], half)  # reverse order on purpose
    d.sketch_push(X[:half], 0)
    d.cuts_finalize()
    d.pages_push(X[:half], 0)
    d.pages_push(X[half:], half)
    gv, gp = d.get_cuts()
    np.testing.assert_array_equal(gp, cp)
    assert gv.tobytes() == cv.tobytes()
    idx = rng.integers(0, n, size=5000)
    np.testing.assert_array_equal(d.get_bins()[idx], oracle.bins(X[idx], cv, cp))
    d.close()


# ------------------------------------------------------------------------------------------ sampling
@pytest.mark.parametrize("mode,ratio", [(0, 1.0), (1, 0.5), (1, 0.1), (2, 0.1), (2, 0.3), (2, 0.5), (2, 1.0)])
@pytest.mark.parametrize("kind", ["logistic", "wide", "ties"])
@pytest.mark.parametrize("n", [1, 777, 20000])
def test_sample_bit_exact(ctx, mode, ratio, kind, n):
    X = np.zeros((n, 2), np.float32)
    X[:, 0] = np.arange(n)
    g, h = synth.gradient_pairs(n, seed=n + mode, kind=kind)
    d = ctx.quantise(X, 16)
    d.set_gradients(g, h)
    info = d.sample(mode, ratio, mvs_lambda=1.0, seed=11, round=3, quant_bits=16)
    s = oracle.sample(g, h, mode, ratio, 1.0, 11, 3)
    sel = s["selected"].astype(bool)
    qg, e_g = oracle.quantise(s["gs"][sel], 16)
    qh, e_h = oracle.quantise(s["hs"][sel], 16)
    assert info["n_selected_local"] == s["n_selected"]
    gid, gq, hq = d.get_sample(info["n_selected_local"])
    np.testing.assert_array_equal(gid, np.nonzero(sel)[0])
    assert (info["e_g"], info["e_h"]) == (e_g, e_h)
    np.testing.assert_array_equal(gq, qg)
    np.testing.assert_array_equal(hq, qh)
    if mode == 2 and not info["fallback_uniform"]:
        assert info["k_star"] == s["k_star"]
        assert info["mu"] == s["mu"]
    d.close()


@pytest.mark.parametrize("a,b", [(0.1, 0.1), (0.2, 0.25), (0.0, 0.5), (0.3, 0.7)])
@pytest.mark.parametrize("kind", ["logistic", "wide", "ties"])
@pytest.mark.parametrize("n", [5, 3001, 40000])
def test_goss_bit_exact(ctx, a, b, kind, n):
    X = np.zeros((n, 2), np.float32)
    g, h = synth.gradient_pairs(n, seed=n + 7, kind=kind)
    d = ctx.quantise(X, 16)
    d.set_gradients(g, h)
    info = d.sample_goss(a, b, seed=13, round=4, quant_bits=16)
    s = oracle.sample_goss(g, h, a, b, 13, 4)
    sel = s["selected"].astype(bool)
    assert info["n_selected_local"] == s["n_selected"]
    assert info["k_star"] == s["k_a"]
    gid, gq, hq = d.get_sample(info["n_selected_local"])
    np.testing.assert_array_equal(gid, np.nonzero(sel)[0])
    qg, e_g = oracle.quantise(s["gs"][sel], 16)
    qh, e_h = oracle.quantise(s["hs"][sel], 16)
    assert (info["e_g"], info["e_h"]) == (e_g, e_h)
    np.testing.assert_array_equal(gq, qg)
    np.testing.assert_array_equal(hq, qh)
    d.close()


# ------------------------------------------------------------------------------------------ trees
def _oracle_tree(B, m, cv, cp, g, h, mode, ratio, depth, quant_bits=16, lam=1.0, gamma=0.0, mcw=1.0,
                 eta=0.1, seed=1, round_=0):
    s = oracle.sample(g, h, mode, ratio, 1.0, seed, round_)
    sel = s["selected"].astype(bool)
    qg, e_g = oracle.quantise(s["gs"][sel], quant_bits)
    qh, e_h = oracle.quantise(s["hs"][sel], quant_bits)
    nodes, lor, hist = oracle.build_tree(B[sel], m, cv, cp, qg, qh, e_g, e_h, depth, lam, gamma, mcw, eta,
                                         want_hist=True)
    return nodes, lor, hist, sel


def _compare_trees(gn, on):
    assert gn.shape == on.shape
    for f in ("feature", "split_bin", "n_rows"):
        np.testing.assert_array_equal(gn[f], on[f], err_msg=f)
    pres = on["feature"] != -2
    sp = on["feature"] >= 0
    np.testing.assert_array_equal(gn["split_value"][sp], on["split_value"][sp])
    np.testing.assert_array_equal(gn["leaf_value"][pres], on["leaf_value"][pres])
    # bars: rel <= 1e-6 (north_star); in fact bit-exact by construction (R14)
    np.testing.assert_allclose(gn["gain"][sp], on["gain"][sp], rtol=1e-6)
    np.testing.assert_array_equal(gn["gain"][sp], on["gain"][sp])
    np.testing.assert_array_equal(gn["sum_g"][pres], on["sum_g"][pres])
    np.testing.assert_array_equal(gn["sum_h"][pres], on["sum_h"][pres])


TREE_CASES = [
    # n, m, max_bin, depth, mode, ratio, stress
    (1, 1, 256, 3, 0, 1.0, False),
    (50, 3, 8, 4, 0, 1.0, False),
    (3000, 20, 256, 6, 0, 1.0, False),
    (10000, 20, 256, 6, 0, 1.0, False),   # config 1
    (10000, 20, 256, 6, 0, 1.0, True),
    (12345, 45, 64, 7, 2, 0.3, False),
    (20000, 33, 256, 8, 1, 0.5, True),
    (20000, 70, 256, 5, 2, 0.1, False),
    (4096, 8, 256, 0, 0, 1.0, False),
    (5000, 10, 256, 10, 0, 1.0, False),
    # > 256 segments at the deepest levels (the block-strided plan) with int64 (> kmax rows) nodes
    # at the top and int32 ones below: both evaluation lists and the general plan path
    (60000, 12, 256, 10, 0, 1.0, False),
    (40000, 16, 256, 11, 2, 0.5, True),
    (70000, 8, 256, 11, 0, 1.0, "noise"),   # > 256 segments: the block-strided plan
]


@pytest.mark.parametrize("n,m,max_bin,depth,mode,ratio,stress", TREE_CASES)
def test_tree_bit_exact(ctx, n, m, max_bin, depth, mode, ratio, stress):
    if n >= 50:
        X, y = synth.make_classification(n, max(m, 2), seed=7 + n, stress=stress is True and m >= 4)
        X = np.ascontiguousarray(X[:, :m])
    else:
        rng = np.random.default_rng(n)
        X = rng.normal(size=(n, m)).astype(np.float32)
        y = (rng.random(n) < 0.5).astype(np.float32)
    cv, cp, B = _oracle_cuts_bins(X, max_bin)
    margin = np.random.default_rng(n).normal(scale=0.5, size=n).astype(np.float32)
    g, h = oracle.logistic_grad(margin, y)
    if stress == "noise":  # random gradient pairs: noise splits everywhere, hundreds of segments
        rng = np.random.default_rng(n + 1)
        g = rng.uniform(-1.0, 1.0, n).astype(np.float32)
        h = rng.uniform(0.05, 1.0, n).astype(np.float32)
    _check_tree(ctx, X, max_bin, cv, cp, B, g, h, mode, ratio, depth, 16)


def leaf_dfs_rank(nodes):
    """Leaves of a tree in left-first depth-first order (the order RepartitionInstances, Alg. 1
    L172-173, lays the children of every split out: left segment, then right)."""
    rank = {}

    def dfs(v):
        if v >= len(nodes) or nodes["feature"][v] == -2:
            return
        if nodes["feature"][v] >= 0:
            dfs(2 * v + 1)
            dfs(2 * v + 2)
        else:
            rank[v] = len(rank)

    dfs(0)
    return rank


def check_row_order(order, nodes, leaf_of_row):
    """The device's final partition (R26): a permutation of the selected rows in which every
    leaf's rows form one contiguous block, blocks in left-first depth-first leaf order; the order
    of rows inside a block is not part of the result (set semantics: every exported value is an
    exact integer sum or a per-row value)."""
    n = len(leaf_of_row)
    assert np.array_equal(np.sort(order), np.arange(n)), "row order is not a permutation"
    rank = leaf_dfs_rank(nodes)
    key = np.array([rank[int(v)] for v in leaf_of_row], np.int64)
    assert np.all(np.diff(key[order]) >= 0), "leaf blocks are not contiguous in depth-first order"


def _check_tree(ctx, X, max_bin, cv, cp, B, g, h, mode, ratio, depth, quant_bits):
    n, m = X.shape
    on, olor, ohist, sel = _oracle_tree(B, m, cv, cp, g, h, mode, ratio, depth, quant_bits=quant_bits)
    d = ctx.quantise(X, max_bin)
    d.set_gradients(g, h)
    info = d.sample(mode, ratio, 1.0, 1, 0, quant_bits)
    t = d.build_tree(depth, 1.0, 0.0, 1.0, 0.1, keep_debug=True)
    gn = t.export()
    _compare_trees(gn, on)
    # histograms of every present node with depth < D: bit-exact
    for v in range((1 << depth) - 1):
        if on["feature"][v] == -2:
            continue
        np.testing.assert_array_equal(t.get_histogram(v), ohist[v], err_msg=f"node {v}")
    # partition: final node of every selected row, bit-exact
    np.testing.assert_array_equal(t.get_partition(info["n_selected_local"]), olor)
    # partition layout (R26): contiguous leaf blocks in depth-first order
    check_row_order(t.get_row_order(info["n_selected_local"]), on, olor)
    # predict (binned traversal) == oracle predict, bit-exact float32
    m0 = np.random.default_rng(1).normal(size=n).astype(np.float32)
    gm = d.predict([t], m0.copy())
    om = oracle.predict(B, on, m0)
    np.testing.assert_array_equal(gm, om)
    if mode == 0:
        um = d.update_margin(t, m0.copy())
        np.testing.assert_array_equal(um, om)
    t.close()
    d.close()
    return on


# quant_bits decides kmax = (2^31 - 1) >> P, i.e. the histogram chunking, which nodes go to the
# int64 (general) or int32 (narrow) evaluation list and which parents are kept as compact s32
# pairs: each case has nodes above and below kmax and multi-chunk pairs (R12)
QB_CASES = [
    # n, m, depth, mode, ratio, quant_bits
    (20000, 24, 6, 0, 1.0, 20),      # kmax 2047: every node of the top levels is multi-chunk int64
    (30000, 16, 7, 2, 0.5, 20),
    (20000, 24, 6, 0, 1.0, 8),       # kmax 8.4M: everything narrow
    (600000, 8, 5, 0, 1.0, 12),      # kmax 524287: root int64, children int32
    (9000000, 3, 3, 0, 1.0, 8),      # kmax 8388607: root int64 at P = 8
]


@pytest.mark.parametrize("n,m,depth,mode,ratio,quant_bits", QB_CASES)
def test_tree_bit_exact_quant_bits(ctx, n, m, depth, mode, ratio, quant_bits):
    X, y = synth.fast_classification(n, m, seed=31 + n) if n > 100000 else synth.make_classification(n, m, seed=31 + n)
    cv, cp, B = _oracle_cuts_bins(X, 256)
    margin = np.random.default_rng(n).normal(scale=0.5, size=n).astype(np.float32)
    g, h = oracle.logistic_grad(margin, y)
    kmax = (2**31 - 1) >> quant_bits
    on = _check_tree(ctx, X, 256, cv, cp, B, g, h, mode, ratio, depth, quant_bits)
    rows = on["n_rows"][on["feature"] != -2]
    if quant_bits != 8 or n > kmax:
        assert rows.max() > kmax and rows.min() <= kmax  # both evaluation lists are exercised


def test_logistic_gradients_close(ctx):
    n = 5000
    rng = np.random.default_rng(3)
    margin = rng.normal(scale=3, size=n).astype(np.float32)
    y = (rng.random(n) < 0.5).astype(np.float32)
    X = rng.normal(size=(n, 2)).astype(np.float32)
    d = ctx.quantise(X, 16)
    d.set_logistic_gradients(margin, y)
    d.sample(0, 1.0)
    _, qg, qh = d.get_sample(n)
    g, h = oracle.logistic_grad(margin, y)
    og, _ = oracle.quantise(g.astype(np.float64), 16)
    oh, _ = oracle.quantise(h.astype(np.float64), 16)
    assert np.max(np.abs(qg - og)) <= 1 and np.max(np.abs(qh - oh)) <= 1
    d.close()


def test_out_of_core_equals_in_core(ctx):
    """without sampling the out-of-core algorithm equals the in-core one (bit-exact)."""
    n, m = 30000, 40
    X, y = synth.make_classification(n, m, seed=3)
    g, h = oracle.logistic_grad(np.zeros(n, np.float32), y)
    trees = []
    for placement, page in [(ob.PLACE_DEVICE, 0), (ob.PLACE_PINNED_HOST, 4096 * 64)]:
        d = ctx.quantise(X, 256, page_bytes=page, placement=placement)
        st = d.info()["row_stride"]
        assert st == 64
        assert d.info()["n_pages"] == (1 if page == 0 else -(-n // (page // st)))
        d.set_gradients(g, h)
        d.sample(0, 1.0)
        t = d.build_tree(6)
        trees.append((d, t, t.export()))
    _compare_trees(trees[0][2], trees[1][2])
    m0 = np.zeros(n, np.float32)
    p0 = trees[0][0].predict([trees[0][1]], m0.copy())
    p1 = trees[1][0].predict([trees[1][1]], m0.copy())
    np.testing.assert_array_equal(p0, p1)
    for d, t, _ in trees:
        t.close()
        d.close()


@pytest.mark.parametrize("n,m,depth,page_rows", [(30000, 40, 6, 4096), (5000, 70, 5, 700), (1, 3, 3, 1)])
def test_streamed_build_alg6_equals_in_core_and_oracle(ctx, n, m, depth, page_rows):
    """Alg. 6 (NEXT #1): f = 1 trees built by streaming the pinned pages once per level equal the
    in-core tree and the oracle (fields, histograms, final partition)."""
    X, y = synth.make_classification(n, m, seed=9) if n >= 50 else (
        np.random.default_rng(1).normal(size=(n, m)).astype(np.float32), np.ones(n, np.float32))
    cv, cp, B = _oracle_cuts_bins(X, 256)
    g, h = oracle.logistic_grad(np.random.default_rng(3).normal(size=n).astype(np.float32), y)
    on, olor, ohist, _ = _oracle_tree(B, m, cv, cp, g, h, 0, 1.0, depth)
    stride = (m + 31) // 32 * 32
    d = ctx.quantise(X, 256, page_bytes=page_rows * stride, placement=ob.PLACE_PINNED_HOST)
    d.set_streaming(True)
    d.set_gradients(g, h)
    d.sample(0, 1.0)
    t = d.build_tree(depth, keep_debug=True)
    _compare_trees(t.export(), on)
    for v in range((1 << depth) - 1):
        if on["feature"][v] == -2:
            continue
        np.testing.assert_array_equal(t.get_histogram(v), ohist[v], err_msg=f"node {v}")
    np.testing.assert_array_equal(t.get_partition(n), olor)
    m0 = np.random.default_rng(4).normal(size=n).astype(np.float32)
    np.testing.assert_array_equal(d.update_margin(t, m0.copy()), oracle.predict(B, on, m0))
    np.testing.assert_array_equal(d.predict([t], m0.copy()), oracle.predict(B, on, m0))
    t.close()
    d.close()


@pytest.mark.parametrize("mode,ratio", [(2, 0.1), (1, 0.3)])
def test_out_of_core_sampled_matches_oracle(ctx, mode, ratio):
    """Alg. 7: sample, compact the pinned pages into one device page, build in-core."""
    n, m = 25000, 24
    X, y = synth.make_classification(n, m, seed=4)
    cv, cp, B = _oracle_cuts_bins(X, 256)
    g, h = oracle.logistic_grad(np.random.default_rng(2).normal(size=n).astype(np.float32), y)
    on, olor, _, sel = _oracle_tree(B, m, cv, cp, g, h, mode, ratio, 6, seed=5, round_=9)
    d = ctx.quantise(X, 256, page_bytes=3000 * 32, placement=ob.PLACE_PINNED_HOST)
    d.set_gradients(g, h)
    info = d.sample(mode, ratio, 1.0, 5, 9, 16)
    t = d.build_tree(6, keep_debug=True)
    _compare_trees(t.export(), on)
    np.testing.assert_array_equal(t.get_partition(info["n_selected_local"]), olor)
    t.close()
    d.close()


def test_training_auc_config1(ctx):
    """Config 1 (10k x 20, 256 bins, depth 6, 10 rounds, binary:logistic): AUC vs oracle <= 1e-3 rel."""
    from sklearn.metrics import roc_auc_score
    n, m = 10000, 20
    X, y = synth.make_classification(n, m, seed=0)
    cv, cp, B = _oracle_cuts_bins(X, 256)
    d = ctx.quantise(X, 256)
    gm = np.zeros(n, np.float32)
    om = np.zeros(n, np.float32)
    prev_o = None
    for r in range(10):
        d.set_logistic_gradients(gm, y)
        d.sample(0, 1.0, round=r)
        t = d.build_tree(6)
        d.predict([t], gm)
        t.close()
        on, om, _ = oracle.boosting_round(B, m, cv, cp, om, y, max_depth=6, prev_tree=prev_o, round_=r)
        prev_o = on
    om = oracle.predict(B, prev_o, om)
    a_gpu, a_orc = roc_auc_score(y, gm), roc_auc_score(y, om)
    assert abs(a_gpu - a_orc) / a_orc <= 1e-3
    assert a_gpu > 0.8
    d.close()


@pytest.mark.parametrize("mode,ratio", [(0, 1.0), (2, 0.5)])
def test_run_to_run_determinism(ctx, mode, ratio):
    """R26: the partition's row order inside a node follows the tiles' atomic reservations, so it
    may differ between runs; every exported result may not.  Three builds of the same round:
    identical tree fields, histograms of every node, leaf of every row and predictions."""
    n, m, depth = 200000, 64, 8
    X, y = synth.fast_classification(n, m, seed=17)
    g, h = oracle.logistic_grad(np.random.default_rng(2).normal(scale=0.5, size=n).astype(np.float32), y)
    d = ctx.quantise(X, 256)
    ref = None
    for rep in range(3):
        d.set_gradients(g, h)
        info = d.sample(mode, ratio, 1.0, 3, 5, 16)
        t = d.build_tree(depth, keep_debug=True)
        got = (t.export(), [t.get_histogram(v) for v in range((1 << depth) - 1)],
               t.get_partition(info["n_selected_local"]), d.predict([t], np.zeros(n, np.float32)))
        t.close()
        if ref is None:
            ref = got
            assert int((got[0]["feature"] >= 0).sum()) > 50
            continue
        for f in ref[0].dtype.names:
            np.testing.assert_array_equal(got[0][f], ref[0][f], err_msg=f"rep {rep}: {f}")
        for v, (a, b) in enumerate(zip(got[1], ref[1])):
            np.testing.assert_array_equal(a, b, err_msg=f"rep {rep}: histogram of node {v}")
        np.testing.assert_array_equal(got[2], ref[2])
        np.testing.assert_array_equal(got[3], ref[3])
    d.close()


def test_streaming_after_in_core_build(ctx):
    """an in-core build of PINNED_HOST f = 1 data, then set_streaming(1) on the same
    data: the streamed build needs its int64 node buffers (allocated on demand) and gives the
    same tree."""
    n, m = 20000, 24
    X, y = synth.make_classification(n, m, seed=12)
    g, h = oracle.logistic_grad(np.zeros(n, np.float32), y)
    d = ctx.quantise(X, 256, page_bytes=4096 * 32, placement=ob.PLACE_PINNED_HOST)
    d.set_gradients(g, h)
    d.sample(0, 1.0)
    t0 = d.build_tree(6)
    d.set_streaming(True)
    d.sample(0, 1.0)
    t1 = d.build_tree(6)
    _compare_trees(t1.export(), t0.export())
    t0.close()
    t1.close()
    d.close()


def test_update_margin_refuses_tree_of_older_sample(ctx):
    """MVS sample -> tree -> sample(NONE) -> update_margin(tree) must be ERR_STATE
    (the tree's partition covers another sample), not out-of-bounds work."""
    n, m = 5000, 8
    X, y = synth.make_classification(n, m, seed=13)
    g, h = oracle.logistic_grad(np.zeros(n, np.float32), y)
    d = ctx.quantise(X, 256)
    d.set_gradients(g, h)
    d.sample(2, 0.3)
    t = d.build_tree(4)
    d.sample(0, 1.0)
    with pytest.raises(ob.OocgbError) as e:
        d.update_margin(t, np.zeros(n, np.float32))
    assert e.value.status == ob.ERR_STATE
    t2 = d.build_tree(4)
    with pytest.raises(ob.OocgbError) as e:  # not the latest tree either
        d.update_margin(t, np.zeros(n, np.float32))
    assert e.value.status == ob.ERR_STATE
    d.update_margin(t2, np.zeros(n, np.float32))
    t.close()
    t2.close()
    d.close()


def test_ctx_destroy_with_live_tree_is_state_error():
    c = ob.Context(0)
    n, m = 500, 4
    X, y = synth.make_classification(n, m, seed=14)
    d = c.quantise(X, 256)
    d.set_gradients(*oracle.logistic_grad(np.zeros(n, np.float32), y))
    d.sample(0, 1.0)
    t = d.build_tree(3)
    d.close()
    with pytest.raises(ob.OocgbError) as e:
        c.close()
    assert e.value.status == ob.ERR_STATE
    t.close()
    c.close()


def test_state_errors(ctx):
    X = np.random.default_rng(0).normal(size=(100, 3)).astype(np.float32)
    d = ctx.quantise(X, 16)
    with pytest.raises(ob.OocgbError) as e:
        d.build_tree(3)
    assert e.value.status == ob.ERR_STATE
    with pytest.raises(ob.OocgbError) as e:
        d.sample(0, 1.0)
    assert e.value.status == ob.ERR_STATE
    d.set_gradients(np.zeros(100, np.float32), np.ones(100, np.float32))
    with pytest.raises(ob.OocgbError) as e:
        d.sample(1, 0.0)
    assert e.value.status == ob.ERR_ARG
    with pytest.raises(ob.OocgbError) as e:
        d.set_gradients(np.zeros(99, np.float32), np.ones(99, np.float32))
    assert e.value.status == ob.ERR_ARG
    d.close()


# ------------------------------------------------------------------------------ R27 missing values
def _missing_data(n, m, seed, rates=None):
    """make_classification rows with missing values (NaN): per-feature missing rates, one feature
    entirely missing when m >= 4, and in feature 1 the missingness depends on the label (so the
    default direction carries signal)."""
    X, y = synth.make_classification(n, m, seed=seed)
    rng = np.random.default_rng(seed)
    rates = rates if rates is not None else rng.uniform(0.0, 0.5, size=m)
    for j in range(m):
        X[rng.random(n) < rates[j], j] = np.nan
    if m >= 2:
        X[(y > 0.5) & (rng.random(n) < 0.6), 1] = np.nan
    if m >= 4:
        X[:, 3] = np.nan
    return X, y


MISS_CASES = [
    # n, m, depth, mode, ratio
    (3000, 6, 5, 0, 1.0),
    (20000, 24, 7, 0, 1.0),
    (20000, 33, 6, 2, 0.3),
    (60000, 12, 9, 0, 1.0),
]


@pytest.mark.parametrize("n,m,depth,mode,ratio", MISS_CASES)
def test_tree_with_missing_bit_exact(ctx, n, m, depth, mode, ratio):
    """R27 on the GPU: cuts skip missing values, symbol 255, both default directions evaluated,
    missing rows partitioned / predicted by the learned direction -- every tree field (with
    default_left), node histogram, leaf of every row and prediction bit-exact vs the oracle."""
    X, y = _missing_data(n, m, seed=40 + n + m)
    cv, cp = oracle.cuts(X, 255, seed=2)
    B = oracle.bins(X, cv, cp)
    d = ctx.quantise(X, 255)
    assert d.info()["has_missing"] == 1
    gv, gp = d.get_cuts()
    np.testing.assert_array_equal(gp, cp)
    assert gv.tobytes() == cv.tobytes()
    np.testing.assert_array_equal(d.get_bins(), B)
    margin = np.random.default_rng(n).normal(scale=0.5, size=n).astype(np.float32)
    g, h = oracle.logistic_grad(margin, y)
    s = oracle.sample(g, h, mode, ratio, 1.0, 1, 0)
    sel = s["selected"].astype(bool)
    qg, e_g = oracle.quantise(s["gs"][sel], 16)
    qh, e_h = oracle.quantise(s["hs"][sel], 16)
    on, olor, ohist = oracle.build_tree(B[sel], m, cv, cp, qg, qh, e_g, e_h, depth, 1.0, 0.0, 1.0, 0.1,
                                        want_hist=True, has_missing=True)
    assert (on["default_left"][on["feature"] >= 0] == 1).any(), "fixture should learn a default-left split"
    d.set_gradients(g, h)
    info = d.sample(mode, ratio, 1.0, 1, 0, 16)
    t = d.build_tree(depth, 1.0, 0.0, 1.0, 0.1, keep_debug=True)
    gn = t.export()
    for f in on.dtype.names:
        np.testing.assert_array_equal(gn[f], on[f], err_msg=f)
    for v in range((1 << depth) - 1):
        if on["feature"][v] != -2:
            np.testing.assert_array_equal(t.get_histogram(v), ohist[v], err_msg=f"node {v}")
    np.testing.assert_array_equal(t.get_partition(info["n_selected_local"]), olor)
    check_row_order(t.get_row_order(info["n_selected_local"]), on, olor)
    m0 = np.random.default_rng(1).normal(size=n).astype(np.float32)
    om = oracle.predict(B, on, m0, has_missing=True)
    np.testing.assert_array_equal(d.predict([t], m0.copy()), om)
    if mode == 0:
        np.testing.assert_array_equal(d.update_margin(t, m0.copy()), om)
    t.close()
    d.close()


def test_csr_input_equals_dense_with_missing(ctx):
    """oocgb_quantise_csr (the pages come from CSR): absent entries are missing; cuts,
    bins and the tree equal oocgb_quantise on the dense matrix with NaN there, and the oracle.
    The CSR arrays are passed from the host and from the device, with a non-zero indptr[0]."""
    import scipy.sparse as sp
    import torch
    n, m, depth = 15000, 20, 6
    X, y = _missing_data(n, m, seed=77)
    # CSR of the present values (an explicit 0.0 stays a present value)
    mask = ~np.isnan(X)
    rows, cols = np.nonzero(mask)
    csr = sp.csr_matrix((X[mask], (rows, cols)), shape=(n, m))
    csr.sort_indices()
    indptr = csr.indptr.astype(np.int64) + 5          # a non-zero base offset
    indices = np.concatenate([np.zeros(5, np.int32), csr.indices.astype(np.int32)])
    values = np.concatenate([np.zeros(5, np.float32), csr.data.astype(np.float32)])
    dense = ctx.quantise(X, 255)
    for src in ("host", "device"):
        if src == "host":
            dc = ctx.quantise_csr(indptr, indices, values, m, 255)
        else:
            dc = ctx.quantise_csr(torch.from_numpy(indptr).cuda(), torch.from_numpy(indices).cuda(),
                                  torch.from_numpy(values).cuda(), m, 255)
        assert dc.info()["has_missing"] == 1
        a, b = dense.get_cuts(), dc.get_cuts()
        assert a[0].tobytes() == b[0].tobytes() and np.array_equal(a[1], b[1])
        np.testing.assert_array_equal(dc.get_bins(), dense.get_bins())
        g, h = oracle.logistic_grad(np.zeros(n, np.float32), y)
        trees = []
        for dd in (dense, dc):
            dd.set_gradients(g, h)
            dd.sample(0, 1.0)
            tt = dd.build_tree(depth)
            trees.append(tt.export())
            tt.close()
        for f in trees[0].dtype.names:
            np.testing.assert_array_equal(trees[0][f], trees[1][f], err_msg=f)
        dc.close()
    dense.close()


def test_missing_values_with_max_bin_256_rejected(ctx):
    rng = np.random.default_rng(5)
    X = rng.normal(size=(5000, 3)).astype(np.float32)
    X[7, 1] = np.nan
    with pytest.raises(ob.OocgbError) as e:
        ctx.quantise(X, 256)
    assert e.value.status == ob.ERR_ARG
    X[8, 2] = np.inf
    with pytest.raises(ob.OocgbError) as e:
        ctx.quantise(X, 255)
    assert e.value.status == ob.ERR_ARG


def test_missing_out_of_core_and_streamed(ctx):
    """Missing values through the pinned-page paths: Alg. 7 compaction (MVS) and the Alg. 6
    streamed build (f = 1) give the oracle's trees."""
    n, m = 20000, 16
    X, y = _missing_data(n, m, seed=91)
    cv, cp = oracle.cuts(X, 255, seed=2)
    B = oracle.bins(X, cv, cp)
    g, h = oracle.logistic_grad(np.random.default_rng(3).normal(size=n).astype(np.float32), y)
    for mode, ratio, streamed in [(2, 0.3, False), (0, 1.0, True)]:
        d = ctx.quantise(X, 255, page_bytes=3000 * 32, placement=ob.PLACE_PINNED_HOST)
        if streamed:
            d.set_streaming(True)
        s = oracle.sample(g, h, mode, ratio, 1.0, 5, 2)
        sel = s["selected"].astype(bool)
        qg, e_g = oracle.quantise(s["gs"][sel], 16)
        qh, e_h = oracle.quantise(s["hs"][sel], 16)
        on, olor, _ = oracle.build_tree(B[sel], m, cv, cp, qg, qh, e_g, e_h, 6, has_missing=True)
        d.set_gradients(g, h)
        info = d.sample(mode, ratio, 1.0, 5, 2, 16)
        t = d.build_tree(6, keep_debug=True)
        gn = t.export()
        for f in on.dtype.names:
            np.testing.assert_array_equal(gn[f], on[f], err_msg=f"streamed={streamed}: {f}")
        np.testing.assert_array_equal(t.get_partition(info["n_selected_local"]), olor)
        m0 = np.zeros(n, np.float32)
        np.testing.assert_array_equal(d.predict([t], m0.copy()), oracle.predict(B, on, m0, has_missing=True))
        t.close()
        d.close()
