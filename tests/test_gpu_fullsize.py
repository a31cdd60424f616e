"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times, on outputs
the oracle can compute: config 2 (1M x 500) cuts of sampled features, bins of sampled rows, the
complete root histogram, the root split and the level-1 partition; config 3 scale (20M rows)
complete MVS sample set.  Plus degenerate inputs (0 rows, 1 row, max_bin = 2, depth 16)."""
import numpy as np
import pytest

import oracle
import synth
from test_gpu_parity import check_row_order

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ob = pytest.importorskip("paper_2005_09148_b200")


@pytest.fixture(scope="module")
def config2():
    X, y = synth.fast_classification(1_000_000, 500, seed=1000)  # bench.py's rank-0 data
    return X, y


@pytest.fixture(scope="module")
def config2_oracle(config2):
    """Oracle cuts (500 sorts of 1M values, ~1 min single thread) and bins of config 2."""
    X, _ = config2
    cv, cp = oracle.cuts(X, 256)
    return cv, cp, oracle.bins(X, cv, cp)


def test_config2_cuts_bins_root_histogram_split(ctx, config2, config2_oracle):
    X, y = config2
    n, m = X.shape
    d = ctx.quantise(X, 256)
    gv, gp = d.get_cuts()
    rng = np.random.default_rng(0)
    feats = np.sort(rng.choice(m, size=8, replace=False))
    # cuts of sampled features (oracle sorts the full 1M-value column, R1)
    cv, cp = oracle.cuts(np.ascontiguousarray(X[:, feats]), 256)
    for k, j in enumerate(feats):
        np.testing.assert_array_equal(gv[gp[j]:gp[j + 1]], cv[cp[k]:cp[k + 1]], err_msg=f"feature {j}")
    cv_all, cp_all, B = config2_oracle
    assert gv.tobytes() == cv_all.tobytes() and np.array_equal(gp, cp_all)
    rows = np.sort(rng.choice(n, size=10_000, replace=False))
    B_s = oracle.bins(X[rows], cv_all, cp_all)
    np.testing.assert_array_equal(d.get_bins()[rows], B_s)
    # one round at f = 1 with bench.py's parameters; root histogram + depth-1 tree
    margin = np.zeros(n, np.float32)
    g, h = oracle.logistic_grad(margin, y)
    d.set_gradients(g, h)
    d.sample(ob.SAMPLE_NONE, 1.0, quant_bits=16)
    t = d.build_tree(1, 1.0, 0.0, 1.0, 0.1, keep_debug=True)
    qg, e_g = oracle.quantise(g.astype(np.float64), 16)
    qh, e_h = oracle.quantise(h.astype(np.float64), 16)
    on, lor, hist = oracle.build_tree(B, m, cv_all, cp_all, qg, qh, e_g, e_h, 1, want_hist=True)
    np.testing.assert_array_equal(t.get_histogram(0), hist[0])
    gn = t.export()
    for f in on.dtype.names:
        np.testing.assert_array_equal(gn[f], on[f], err_msg=f)
    np.testing.assert_array_equal(t.get_partition(n), lor)
    t.close()
    # the bench's depth-8 tree: conservation and sibling consistency of the GPU tree itself
    t8 = d.build_tree(8)
    n8 = t8.export()
    for v in range(255):
        if n8["feature"][v] >= 0:
            assert n8["n_rows"][2 * v + 1] + n8["n_rows"][2 * v + 2] == n8["n_rows"][v]
            assert n8["gain"][v] > 0
    assert n8["n_rows"][0] == n
    t8.close()
    d.close()


@pytest.mark.parametrize("quant_bits,mode,ratio", [(16, 0, 1.0), (16, 2, 0.1)])
def test_config2_depth8_two_rounds_vs_oracle(ctx, config2, config2_oracle, quant_bits, mode, ratio):
    """The benchmarked configuration itself (bench.py: 1M x 500, 256 bins, depth 8, f = 1,
    lambda 1, gamma 0, mcw 1, eta 0.1, the same CUDA graph and kernels), two consecutive boosting
    rounds with the margin updated in between (Eq. 1 via the partition, update_margin): every
    tree field, the histogram of every node of depth < 8 (built and derived), the leaf of every
    row and the updated margins are bit-exact against the oracle (Alg. 1; Eq. 8
    P:L144-151; Eq. 6).  Also with MVS f = 0.1 at full size (the in-core sampled path:
    the selected-row list, Eq. 9 sampling R9, the build graph reused across rounds whose sample
    sizes differ, predict by traversal)."""
    X, y = config2
    cv, cp, B = config2_oracle
    n, m = X.shape
    d = ctx.quantise(X, 256)
    gm = np.zeros(n, np.float32)
    om = np.zeros(n, np.float32)
    for r in range(2):
        np.testing.assert_array_equal(gm, om, err_msg=f"margins before round {r}")
        g, h = oracle.logistic_grad(om, y)  # identical gradients on both sides
        d.set_gradients(g, h)
        info = d.sample(mode, ratio, 1.0, seed=3, round=r, quant_bits=quant_bits)
        t = d.build_tree(8, 1.0, 0.0, 1.0, 0.1, keep_debug=True)
        s_ = oracle.sample(g, h, mode, ratio, 1.0, 3, r)
        sel = s_["selected"].astype(bool)
        assert info["n_selected_local"] == int(sel.sum())
        qg, e_g = oracle.quantise(s_["gs"][sel], quant_bits)
        qh, e_h = oracle.quantise(s_["hs"][sel], quant_bits)
        on, lor, hist = oracle.build_tree(B[sel], m, cv, cp, qg, qh, e_g, e_h, 8, 1.0, 0.0, 1.0, 0.1,
                                          want_hist=True)
        gn = t.export()
        for f in on.dtype.names:
            np.testing.assert_array_equal(gn[f], on[f], err_msg=f"round {r}: {f}")
        assert int((on["feature"] >= 0).sum()) > 100, "the tree should be deep and bushy"
        for v in range(255):
            if on["feature"][v] == -2:
                continue
            np.testing.assert_array_equal(t.get_histogram(v), hist[v], err_msg=f"round {r}: node {v}")
        ns = int(sel.sum())
        np.testing.assert_array_equal(t.get_partition(ns), lor, err_msg=f"round {r}: leaf of row")
        check_row_order(t.get_row_order(ns), on, lor)
        # every row gets the new tree (R18): from the partition at f = 1, by traversal otherwise
        gm = d.update_margin(t, gm) if mode == 0 else d.predict([t], gm)
        om = oracle.predict(B, on, om)
        np.testing.assert_array_equal(gm, om, err_msg=f"round {r}: margins after the update")
        t.close()
        del hist
    d.close()


def test_config3_scale_mvs_sample_set(ctx):
    """20M rows (config 3's row count), MVS f = 0.1: the complete selected set, k*, mu and the
    fixed-point pairs are bit-exact against the oracle's sort-based threshold (R9)."""
    n = 20_000_000
    g, h = synth.gradient_pairs(n, seed=21, kind="logistic")
    X = np.zeros((n, 1), np.float32)
    d = ctx.quantise(X, 2)
    d.set_gradients(g, h)
    info = d.sample(ob.SAMPLE_MVS, 0.1, 1.0, seed=4, round=11, quant_bits=16)
    s = oracle.sample(g, h, oracle.SAMPLE_MVS, 0.1, 1.0, 4, 11)
    sel = s["selected"].astype(bool)
    assert info["n_selected_local"] == s["n_selected"]
    assert (info["k_star"], info["mu"]) == (s["k_star"], s["mu"])
    gid, qg, qh = d.get_sample(info["n_selected_local"])
    np.testing.assert_array_equal(gid, np.nonzero(sel)[0])
    og, e_g = oracle.quantise(s["gs"][sel], 16)
    oh, e_h = oracle.quantise(s["hs"][sel], 16)
    assert (info["e_g"], info["e_h"]) == (e_g, e_h)
    np.testing.assert_array_equal(qg, og)
    np.testing.assert_array_equal(qh, oh)
    d.close()


def test_zero_rows(ctx):
    X = np.zeros((0, 7), np.float32)
    d = ctx.quantise(X, 256)
    cv, cp = d.get_cuts()
    assert list(cp) == list(range(8)) and np.all(cv == 0)  # R1: empty column -> one cut 0.0
    d.set_gradients(np.zeros(0, np.float32), np.zeros(0, np.float32))
    info = d.sample(ob.SAMPLE_MVS, 0.5)
    assert info["n_selected_global"] == 0
    t = d.build_tree(4)
    nd = t.export()
    assert nd["feature"][0] == -1 and nd["n_rows"][0] == 0 and nd["leaf_value"][0] == 0.0
    assert np.all(nd["feature"][1:] == -2)
    assert d.predict([t], np.zeros(0, np.float32)).shape == (0,)
    t.close()
    d.close()


# depth 16 (the ABI maximum) with tiny m: keep_debug stores (2^D - 1) node histograms
@pytest.mark.parametrize("n,m,max_bin,depth", [(1, 5, 256, 3), (300, 3, 2, 16), (64, 40, 4, 10)])
def test_degenerate_shapes_match_oracle(ctx, n, m, max_bin, depth):
    rng = np.random.default_rng(n + m)
    X = rng.normal(size=(n, m)).astype(np.float32)
    y = (rng.random(n) < 0.5).astype(np.float32)
    cv, cp = oracle.cuts(X, max_bin)
    B = oracle.bins(X, cv, cp)
    g, h = oracle.logistic_grad(rng.normal(size=n).astype(np.float32), y)
    qg, e_g = oracle.quantise(g.astype(np.float64), 16)
    qh, e_h = oracle.quantise(h.astype(np.float64), 16)
    on, lor, _ = oracle.build_tree(B, m, cv, cp, qg, qh, e_g, e_h, depth, 1.0, 0.0, 0.0, 0.1)
    d = ctx.quantise(X, max_bin)
    np.testing.assert_array_equal(d.get_bins(), B)
    d.set_gradients(g, h)
    d.sample(ob.SAMPLE_NONE, 1.0)
    t = d.build_tree(depth, 1.0, 0.0, 0.0, 0.1, keep_debug=True)
    gn = t.export()
    for f in on.dtype.names:
        np.testing.assert_array_equal(gn[f], on[f], err_msg=f)
    np.testing.assert_array_equal(t.get_partition(n), lor)
    t.close()
    d.close()
