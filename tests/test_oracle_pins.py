"""Pins of the CPU oracle against what the paper and mathematics fix — NOT against itself.

Each test names the pin kind: a worked example (tests/golden/, cited), a closed form, an
invariant, a library routine that computes the same definition (numpy / sklearn / fractions),
or brute force on tiny inputs.  Chosen so a dropped term, a wrong sign or index, or a transposed
operand in oracle/oocgb_oracle.c fails at least one of them.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


# ------------------------------------------------------------------------------ O3 Philox RNG
def test_philox_known_answer():
    """Random123 known-answer vector (golden, cited)."""
    k = GOLD["philox_kat"]
    out = oracle.philox4x64_10(k["ctr"], k["key"])
    assert [f"{int(x):016x}" for x in out] == k["out"]


@pytest.mark.parametrize("seed", [0, 1, 7, 2**63 + 5])
def test_philox_matches_numpy(seed):
    """numpy.random.Philox (an independent implementation) emits block ctr+1."""
    rng = np.random.default_rng(seed % 1000)
    for _ in range(20):
        key = rng.integers(0, 2**63, size=2, dtype=np.uint64)
        ctr = rng.integers(0, 2**63, size=4, dtype=np.uint64)
        bg = np.random.Philox(key=key, counter=ctr)
        ref = bg.random_raw(4)
        nxt = ctr.copy()
        nxt[0] += np.uint64(1)  # no carry for these ranges
        np.testing.assert_array_equal(oracle.philox4x64_10(nxt, key), ref)


def test_uniform_definition_range():
    us = [oracle.uniform(3, 4, r, 0) for r in range(2000)]
    assert min(us) >= 0.0 and max(us) < 1.0
    assert abs(np.mean(us) - 0.5) < 0.03
    # u = (x >> 11) 2^-53 with x the first Philox word
    x = int(oracle.philox4x64_10([17, 0, 0, 0], [3, 4])[0])
    assert oracle.uniform(3, 4, 17, 0) == (x >> 11) * 2.0**-53


# ------------------------------------------------------------------------------ O1 cuts
@pytest.mark.parametrize("ex", GOLD["cuts"], ids=lambda e: e["cite"][:12])
def test_cuts_worked_examples(ex):
    X = np.array(ex["values"], np.float32)[:, None]
    cv, cp = oracle.cuts(X, ex["max_bin"])
    assert list(cp) == [0, len(ex["cuts"])]
    assert list(cv) == ex["cuts"]


def test_cuts_distinct_values_equal_unique():
    """D_j <= B: the cuts are the distinct values (np.unique, library routine)."""
    rng = np.random.default_rng(1)
    X = rng.integers(-5, 6, size=(500, 6)).astype(np.float32) * 0.5
    cv, cp = oracle.cuts(X, 256)
    for j in range(6):
        np.testing.assert_array_equal(cv[cp[j]:cp[j + 1]], np.unique(X[:, j]))


@pytest.mark.parametrize("B", [4, 16, 256])
def test_cuts_rank_accuracy(B):
    """S:L140 rank accuracy: fraction of values <= c_b is within (b+1)/B +- 1/B (continuous data,
    where no cut is dropped), and the last cut is the column max."""
    rng = np.random.default_rng(B)
    X = rng.normal(size=(20000, 3)).astype(np.float32)
    cv, cp = oracle.cuts(X, B)
    for j in range(3):
        c = cv[cp[j]:cp[j + 1]]
        assert len(c) == B
        assert np.all(np.diff(c) > 0)
        col = np.sort(X[:, j])
        frac = np.searchsorted(col, c, side="right") / len(col)
        assert np.all(np.abs(frac - (np.arange(B) + 1) / B) <= 1.0 / B + 1e-12)
        assert c[-1] == col[-1]


@pytest.mark.parametrize("N,B,tie_frac", [(1003, 16, 0.5), (777, 256, 0.5), (5000, 7, 0.7), (4099, 256, 0.6)])
def test_cuts_ceil_rank_with_ties_equals_np_sort(N, B, tie_frac):
    """O1 step 4 / R1 exactly, from np.sort: with more than B distinct values the cuts are
    v[ceil(b N / B)] (1-based, b = 1..B) of the sorted column with repeats dropped, and the last
    cut is the column max.  N is not a multiple of B and a large share of the values are tied, so a
    floor-rank, an off-by-one index or kept repeats all change the result (checked below)."""
    rng = np.random.default_rng(N + B)
    n_tie = int(N * tie_frac)
    ties = rng.choice(np.array([-1.5, 0.25, 3.0, 7.75], np.float32), size=n_tie)
    cont = rng.normal(size=N - n_tie).astype(np.float32) * 4 + 1.0
    col = np.concatenate([ties, cont])
    rng.shuffle(col)
    X = col[:, None]
    assert len(np.unique(col)) > B
    cv, cp = oracle.cuts(X, B)
    v = np.sort(col)
    b = np.arange(1, B + 1)
    ceil_idx = (b * N + B - 1) // B          # 1-based ceil(b N / B)
    expect = np.unique(v[ceil_idx - 1])      # sorted -> unique = drop repeats, keep increasing
    np.testing.assert_array_equal(cv[cp[0]:cp[1]], expect)
    assert cv[cp[1] - 1] == v[-1]
    # the fixture discriminates the plausible mistakes
    floor_idx = np.maximum(1, (b * N) // B)
    assert not np.array_equal(np.unique(v[floor_idx - 1]), expect) or not np.array_equal(v[ceil_idx - 1], expect)
    assert len(v[ceil_idx - 1]) != len(expect)  # repeats really were dropped


def test_cuts_negative_zero_canonical():
    X = np.array([[-0.0], [0.0], [1.0]], np.float32)
    cv, cp = oracle.cuts(X, 256)
    assert list(cv) == [0.0, 1.0] and not np.signbit(cv[0])


def test_cuts_sketch_sample_keyed_by_global_row():
    """R2: for n_global > 2^20 the sample depends only on (seed, global row): the same cuts
    whichever rank holds the row (checked via the selection predicate)."""
    n_global = (1 << 20) * 4
    sel = [oracle.lib().orc_sketch_row_selected(n_global, 9, r) for r in range(40000)]
    assert abs(np.mean(sel) - 0.25) < 0.01
    u = np.array([oracle.uniform(9, 2**64 - 1, r, 1) for r in range(200)])
    np.testing.assert_array_equal(np.array(sel[:200], bool), u < 0.25)


def test_cuts_reject_nonfinite():
    with pytest.raises(oracle.OracleError):
        oracle.cuts(np.array([[1.0], [np.inf]], np.float32), 4)


# ------------------------------------------------------------------------------ O2 bins
@pytest.mark.parametrize("ex", GOLD["lookup_bin"], ids=lambda e: e["cite"][:12])
def test_lookup_worked_examples(ex):
    cuts = np.array(ex["cuts"], np.float32)
    b = oracle.bins(np.array([[ex["value"]]], np.float32), cuts, np.array([0, len(cuts)], np.int32))
    assert b[0, 0] == ex["bin"]


def test_bins_equal_searchsorted():
    """lower_bound == numpy.searchsorted(side='left') clipped to B_j - 1; stride padding is 0."""
    X, _ = synth.make_classification(3000, 21, seed=2, stress=True)
    cv, cp = oracle.cuts(X, 32)
    B = oracle.bins(X, cv, cp)
    assert B.shape == (3000, 32)
    assert np.all(B[:, 21:] == 0)
    for j in range(21):
        c = cv[cp[j]:cp[j + 1]]
        ref = np.minimum(np.searchsorted(c, X[:, j], side="left"), len(c) - 1)
        np.testing.assert_array_equal(B[:, j], ref)
    # out-of-range values clamp (prediction time)
    Y = np.full((1, 21), 1e30, np.float32)
    np.testing.assert_array_equal(oracle.bins(Y, cv, cp)[0, :21], np.diff(cp) - 1)


def test_bins_decode_roundtrip():
    """decode(encode(x)) brackets x: c_{b-1} < x <= c_b for in-range values."""
    X, _ = synth.make_classification(2000, 8, seed=5)
    cv, cp = oracle.cuts(X, 64)
    B = oracle.bins(X, cv, cp)
    for j in range(8):
        c = cv[cp[j]:cp[j + 1]].astype(np.float64)
        b = B[:, j].astype(int)
        assert np.all(X[:, j] <= c[b])
        lo = np.where(b > 0, c[np.maximum(b - 1, 0)], -np.inf)
        assert np.all(X[:, j] > lo)


# ------------------------------------------------------------------------------ O4 sampling
def _p_fraction_bruteforce(ghat_int, s: Fraction):
    """Solve sum_i min(1, a_i / mu) = s exactly with rationals by trying every number k of
    capped rows (the definition of capped PPS), independent of the D(k) recursion."""
    a = sorted(ghat_int, reverse=True)
    n = len(a)
    nz = sum(1 for x in a if x > 0)
    if s >= nz:
        return None  # every non-zero row has p = 1
    for k in range(0, n):
        if s - k <= 0:
            break
        R = sum(a[k:])
        if R == 0:
            break
        mu = Fraction(R) / (s - k)
        if (k == 0 or a[k - 1] >= mu) and a[k] < mu:
            return mu
    return None


def test_mvs_ghat_closed_form():
    """Eq. 9 with g=3, h=4, lambda=1 -> g_hat = 5 (golden S:L322), observed through p: with 8
    rows g_hat = [5, 1 x 7] (h = 0 for the others) and f = 1/4 (s = 2): sum g_hat = 12, no row
    is capped (5 < 12/2), mu = 6 and p = [5/6, 1/6 x 7] (exact); a wrong g_hat breaks p[0]."""
    ex = GOLD["mvs_ghat"]
    g = np.array([ex["g"]] + [1.0] * 7, np.float32)
    h = np.array([ex["h"]] + [0.0] * 7, np.float32)
    s = oracle.sample(g, h, oracle.SAMPLE_MVS, 0.25, ex["lambda"], seed=1)
    assert s["k_star"] == 0
    assert s["p"][0] == 5.0 / 6.0
    np.testing.assert_array_equal(s["p"][1:], np.full(7, 1.0 / 6.0))


def test_mvs_worked_example_probabilities():
    """Golden S:L323: g_hat = [10,1,1,1,1], f n = 2 -> mu = 4, p = [1, 1/4 x 4] (padded with
    zero-gradient rows to n = 8, f = 1/4 so that f n lies on the 2^-32 grid)."""
    ex = GOLD["mvs_probabilities"]
    g = np.array(ex["ghat"] + [0, 0, 0], np.float32)
    h = np.zeros(8, np.float32)
    s = oracle.sample(g, h, oracle.SAMPLE_MVS, ex["f_times_n"] / 8, 0.0, seed=3)
    np.testing.assert_array_equal(s["p"], np.array(ex["p"] + [0, 0, 0], np.float64))
    assert s["k_star"] == 1
    scale = 2.0 ** s["e_prime"]
    assert s["mu"] == ex["mu"] * scale


@pytest.mark.parametrize("trial", range(60))
def test_mvs_threshold_fraction_bruteforce(trial):
    """Exact rational solution on tiny integer inputs: same mu (as double) and same capped set."""
    rng = np.random.default_rng(trial)
    n = int(rng.integers(1, 12))
    vals = rng.integers(0, 6, size=n) * (1 + (trial % 3 == 0) * 7)
    f = [0.125, 0.25, 0.5, 0.75][trial % 4]
    g = vals.astype(np.float32)
    h = np.zeros(n, np.float32)
    s = oracle.sample(g, h, oracle.SAMPLE_MVS, f, 0.0, seed=trial)
    if g.max() == 0:
        return
    scale = 2 ** s["e_prime"]
    a_int = [int(v) * scale for v in vals]  # exact: g_hat integers times a power of two
    F = Fraction(int(round(f * 2**32)) * n, 2**32)
    mu = _p_fraction_bruteforce(a_int, F)
    if mu is None:
        np.testing.assert_array_equal(s["p"], (vals > 0).astype(float))
    else:
        p_ref = np.array([min(Fraction(1), Fraction(a) / mu) for a in a_int], dtype=object)
        np.testing.assert_allclose(s["p"], p_ref.astype(float), rtol=1e-14, atol=0)
        assert sum(p_ref) == F


@pytest.mark.parametrize("f", [0.1, 0.3, 0.5])
@pytest.mark.parametrize("kind", ["logistic", "wide", "ties"])
def test_mvs_expected_size_and_monotone(f, kind):
    """S:L337 sum p = f n (within 1e-9 n) and S:L339 monotone inclusion."""
    n = 3000
    g, h = synth.gradient_pairs(n, seed=int(f * 10), kind=kind)
    s = oracle.sample(g, h, oracle.SAMPLE_MVS, f, 1.0, seed=5)
    p = s["p"]
    assert abs(p.sum() - f * n) <= 1e-9 * n
    ghat = np.sqrt(g.astype(np.float64) ** 2 + h.astype(np.float64) ** 2)
    o = np.argsort(ghat, kind="stable")
    assert np.all(np.diff(p[o]) >= -1e-15)
    assert np.all((p >= 0) & (p <= 1))


def test_mvs_f1_identity():
    """f = 1 -> every row with g_hat > 0 has p = 1, scale 1."""
    g, h = synth.gradient_pairs(500, seed=2)
    s = oracle.sample(g, h, oracle.SAMPLE_MVS, 1.0, 1.0, seed=1)
    assert np.all(s["p"] == 1.0) and s["n_selected"] == 500
    np.testing.assert_array_equal(s["gs"], g.astype(np.float64))


def test_mvs_unbiased_monte_carlo():
    """S:L336 / north_star: over 1000 seeds the mean of sum selected g' (and h') is within 2%."""
    n = 1000
    g, h = synth.gradient_pairs(n, seed=11, kind="wide")
    G, H = float(np.sum(g, dtype=np.float64)), float(np.sum(h, dtype=np.float64))
    sg, sh = [], []
    for seed in range(1000):
        s = oracle.sample(g, h, oracle.SAMPLE_MVS, 0.2, 1.0, seed=seed, round_=3)
        sg.append(s["gs"].sum())
        sh.append(s["hs"].sum())
    assert abs(np.mean(sg) - G) <= 0.02 * np.sum(np.abs(g))
    assert abs(np.mean(sh) - H) <= 0.02 * abs(H)


def test_uniform_sampling_frequency_and_scale():
    """SGB: selection frequency ~ f per row, scale 1."""
    n = 200
    g, h = synth.gradient_pairs(n, seed=1)
    cnt = np.zeros(n)
    for seed in range(2000):
        s = oracle.sample(g, h, oracle.SAMPLE_UNIFORM, 0.5, seed=seed)
        cnt += s["selected"]
        sel = s["selected"].astype(bool)
        np.testing.assert_array_equal(s["gs"][sel], g[sel].astype(np.float64))
    assert np.all(np.abs(cnt / 2000 - 0.5) < 0.06)
    assert abs(cnt.mean() / 2000 - 0.5) < 0.01


def test_all_zero_ghat_falls_back_to_uniform():
    """all g_hat = 0 -> uniform sampling."""
    n = 4000
    s = oracle.sample(np.zeros(n, np.float32), np.zeros(n, np.float32), oracle.SAMPLE_MVS, 0.25, 1.0, seed=2)
    assert abs(s["n_selected"] / n - 0.25) < 0.03


def test_goss_worked_example():
    """Golden S:L313: |g| = [5,4,3,2,1], a = 0.2, b = 0.25 -> the |g| = 5 row always (scale 1),
    the others with p = b / (1 - a) and scale (1 - a) / b = 3.2."""
    ex = GOLD["goss"]
    g = np.array(ex["abs_g"], np.float32) * np.array([1, -1, 1, -1, 1], np.float32)
    h = np.ones(5, np.float32)
    hits = np.zeros(5)
    for seed in range(400):
        s = oracle.sample_goss(g, h, ex["a"], ex["b"], seed=seed)
        assert s["selected"][0] == 1 and s["p"][0] == 1.0 and s["gs"][0] == g[0]
        assert s["k_a"] == 1
        rest = s["selected"][1:].astype(bool)
        np.testing.assert_allclose(s["gs"][1:][rest] / g[1:][rest], ex["rest_scale"], rtol=1e-9)
        hits += s["selected"]
    assert abs(hits[1:].mean() / 400 - ex["b"] / (1 - ex["a"])) < 0.05


def test_goss_top_set_is_argsort_definition():
    """The top set = the k_a largest |g| (np.argsort, library routine), ties to the same side."""
    g, h = synth.gradient_pairs(5000, seed=3, kind="wide")
    s = oracle.sample_goss(g, h, 0.1, 0.2, seed=1)
    k = s["k_a"]
    assert k == int((round(0.1 * 2**32) * 5000 + 2**31) >> 32) == 500
    order = np.argsort(-np.abs(g.astype(np.float64)), kind="stable")
    thr = np.abs(g[order[k - 1]])
    top = np.abs(g) >= thr
    np.testing.assert_array_equal(s["p"] == 1.0, top)
    assert top.sum() >= k


def test_goss_unbiased_monte_carlo():
    """P:L228 'scaled by (1-a)/b to make the gradient statistics unbiased': mean over 1000 seeds of
    sum selected g' within 2% (and h')."""
    g, h = synth.gradient_pairs(1000, seed=12, kind="logistic")
    G, H = float(np.sum(g, dtype=np.float64)), float(np.sum(h, dtype=np.float64))
    sg, sh = [], []
    for seed in range(1000):
        s = oracle.sample_goss(g, h, 0.1, 0.2, seed=seed, round_=5)
        sg.append(s["gs"].sum())
        sh.append(s["hs"].sum())
    assert abs(np.mean(sg) - G) <= 0.02 * np.sum(np.abs(g))
    assert abs(np.mean(sh) - H) <= 0.02 * abs(H)


# ------------------------------------------------------------------------------ O5 fixed point
def test_quantise_properties():
    rng = np.random.default_rng(0)
    x = rng.normal(scale=3.0, size=5000)
    for P in (8, 16, 20):
        q, e = oracle.quantise(x, P)
        M = np.max(np.abs(x))
        assert 2.0 ** (P - 1) <= np.max(np.abs(q)) <= 2.0 ** P
        assert np.all(np.abs(q.astype(np.float64) * 2.0 ** -e - x) <= 2.0 ** -(e + 1))
        assert 2.0 ** (P - e - 1) <= M < 2.0 ** (P - e)


def test_quantise_round_half_even():
    """rint ties to even: x 2^e = 0.5 -> 0, 1.5 -> 2, 2.5 -> 2 (P = 16, max 1.0 -> e = 15)."""
    x = np.array([1.0, 0.5 * 2**-15, 1.5 * 2**-15, 2.5 * 2**-15, -0.5 * 2**-15])
    q, e = oracle.quantise(x, 16)
    assert e == 15
    assert list(q) == [2**15, 0, 2, 2, 0]


def test_quantise_zero():
    q, e = oracle.quantise(np.zeros(4), 16)
    assert e == 0 and np.all(q == 0)


# ------------------------------------------------------------------------------ O6 histogram
def _hist_addat(B, m, rows, qg, qh):
    H = np.zeros((m, 256, 2), np.int64)
    for j in range(m):
        np.add.at(H[j, :, 0], B[rows, j], qg[rows])
        np.add.at(H[j, :, 1], B[rows, j], qh[rows])
    return H


def test_histogram_bruteforce_conservation_additivity():
    X, _ = synth.make_classification(4000, 13, seed=3, stress=True)
    cv, cp = oracle.cuts(X, 256)
    B = oracle.bins(X, cv, cp)
    rng = np.random.default_rng(0)
    qg = rng.integers(-2**16, 2**16 + 1, size=4000)
    qh = rng.integers(0, 2**16 + 1, size=4000)
    rows = np.sort(rng.choice(4000, size=1500, replace=False))
    Hh = oracle.histogram(B, 13, rows, qg, qh)
    np.testing.assert_array_equal(Hh, _hist_addat(B, 13, rows, qg, qh))   # numpy add.at
    assert np.all(Hh[:, :, 0].sum(axis=1) == qg[rows].sum())               # conservation
    assert np.all(Hh[:, :, 1].sum(axis=1) == qh[rows].sum())
    A, C = rows[:700], rows[700:]
    np.testing.assert_array_equal(oracle.histogram(B, 13, A, qg, qh) + oracle.histogram(B, 13, C, qg, qh), Hh)


# ------------------------------------------------------------------------------ O7-O10 trees
def _gain(GL, HL, GR, HR, lam, gamma):
    """Eq. 8 written independently in rationals."""
    f = lambda G, H: Fraction(G) ** 2 / (Fraction(H) + Fraction(lam))
    return Fraction(1, 2) * (f(GL, HL) + f(GR, HR) - f(GL + GR, HL + HR)) - Fraction(gamma)


def _two_bin_tree(gvals, hvals, binsv, lam=1.0, gamma=0.0, mcw=0.0, eta=1.0, depth=1):
    n = len(gvals)
    B = np.zeros((n, 16), np.uint8)
    B[:, 0] = binsv
    cv = np.array([0.0, 1.0], np.float32)
    cp = np.array([0, 2], np.int32)
    qg, e_g = oracle.quantise(np.array(gvals, np.float64), 16)
    qh, e_h = oracle.quantise(np.array(hvals, np.float64), 16)
    return oracle.build_tree(B, 1, cv, cp, qg, qh, e_g, e_h, depth, lam, gamma, mcw, eta)


def test_split_gain_worked_example():
    """Golden S:L399: G_L=-4, H_L=2, G_R=0, H_R=2, lambda=1, gamma=0 -> gain 1.0667 (= 16/15)."""
    ex = GOLD["split_gain"]
    nodes, lor, _ = _two_bin_tree([-2, -2, 0, 0], [1, 1, 1, 1], [0, 0, 1, 1])
    assert nodes["feature"][0] == 0 and nodes["split_bin"][0] == 0
    assert abs(nodes["gain"][0] - ex["gain_approx"]) < 1e-4
    assert abs(nodes["gain"][0] - float(_gain(-4, 2, 0, 2, 1, 0))) <= 4e-16
    np.testing.assert_array_equal(lor, [1, 1, 2, 2])


def test_symmetric_halves_no_split():
    """Golden S:L400: symmetric halves, lambda = 0 -> gain 0 -> leaf (gain > 0 strictly, R13)."""
    nodes, lor, _ = _two_bin_tree([-1, -1, -1, -1], [1, 1, 1, 1], [0, 0, 1, 1], lam=0.0)
    assert nodes["feature"][0] == -1
    assert np.all(lor == 0)


def test_leaf_weight_worked_example():
    """Golden S:L408: G=-4, H=2, lambda=1 -> w = 4/3 (eta = 1, depth 0)."""
    ex = GOLD["leaf_weight"]
    nodes, _, _ = _two_bin_tree([-2, -2], [1, 1], [0, 1], depth=0)
    assert nodes["leaf_value"][0] == np.float32(ex["w"])
    assert nodes["sum_g"][0] == -4.0 and nodes["sum_h"][0] == 2.0


@pytest.mark.parametrize("seed", [4, 5, 6])
def test_objective_identity(seed):
    """Eq. 7 -> Eq. 8: Eq. 7 of the one-leaf tree minus Eq. 7 of the split
    tree (gamma T included) equals the chosen split's gain.  The fixture
    always splits: bin 0 carries g ~ -2, bin 1 carries g ~ +1.5, so the only candidate has a gain
    far above gamma (a skipped draw would pin nothing)."""
    rng = np.random.default_rng(seed)
    bins_ = np.arange(64) % 2
    g = np.where(bins_ == 0, -2.0, 1.5) + rng.normal(scale=0.1, size=64)
    h = rng.uniform(0.1, 1, size=64)
    nodes, _, _ = _two_bin_tree(g, h, bins_, lam=1.0, gamma=0.3, mcw=0.0)
    assert nodes["feature"][0] == 0 and nodes["split_bin"][0] == 0
    # Eq. 7 of a whole tree: -1/2 sum_leaves G^2 / (H + lambda) + gamma T
    eq7 = lambda leaves: sum(-0.5 * G * G / (H + 1.0) for G, H in leaves) + 0.3 * len(leaves)
    before = eq7([(nodes["sum_g"][0], nodes["sum_h"][0])])
    after = eq7([(nodes["sum_g"][1], nodes["sum_h"][1]), (nodes["sum_g"][2], nodes["sum_h"][2])])
    assert nodes["gain"][0] > 1.0
    # the loss reduction of the split is Eq. 8's gain (gamma included once, for the extra leaf)
    assert abs((before - after) - nodes["gain"][0]) < 1e-12 * max(1.0, abs(nodes["gain"][0]))


def _greedy_raw(X, qg, qh, e_g, e_h, rows, depth, D, lam, gamma, mcw, out, v):
    """Exact-greedy tree straight from raw values (no histograms, no bins): for every feature
    and every distinct value t, left = {x <= t}.  Python ints for sums (exact), Python floats
    for Eq. 8 — an independent enumeration of the definition."""
    G, H = int(qg[rows].sum()), int(qh[rows].sum())
    out[v] = dict(G=G, H=H, n=len(rows), feature=-1)
    if depth == D or len(rows) == 0:
        return
    sc_g, sc_h = 2.0 ** -e_g, 2.0 ** -e_h
    gP, hP = G * sc_g, H * sc_h
    tP = (gP * gP) / (hP + lam)
    best = None
    for j in range(X.shape[1]):
        vals = np.unique(X[rows, j])
        for t in vals[:-1]:
            L = rows[X[rows, j] <= t]
            GL, HL = int(qg[L].sum()), int(qh[L].sum())
            gl, hl, gr, hr = GL * sc_g, HL * sc_h, (G - GL) * sc_g, (H - HL) * sc_h
            if not (hl >= mcw and hr >= mcw):
                continue
            gain = 0.5 * (((gl * gl) / (hl + lam) + (gr * gr) / (hr + lam)) - tP) - gamma
            if best is None or gain > best[0]:
                best = (gain, j, float(t), L)
    if best is None or best[0] <= 0:
        return
    gain, j, t, L = best
    out[v].update(feature=j, value=t, gain=gain)
    R = np.setdiff1d(rows, L)
    _greedy_raw(X, qg, qh, e_g, e_h, L, depth + 1, D, lam, gamma, mcw, out, 2 * v + 1)
    _greedy_raw(X, qg, qh, e_g, e_h, R, depth + 1, D, lam, gamma, mcw, out, 2 * v + 2)


@pytest.mark.parametrize("trial", range(12))
def test_tree_equals_exhaustive_greedy(trial):
    rng = np.random.default_rng(100 + trial)
    n = int(rng.integers(2, 200))
    m = int(rng.integers(1, 5))
    X = np.round(rng.normal(size=(n, m)) * (2 + trial % 3)).astype(np.float32)
    y = (rng.random(n) < 0.5).astype(np.float32)
    g, h = oracle.logistic_grad(rng.normal(size=n).astype(np.float32), y)
    qg, e_g = oracle.quantise(g.astype(np.float64), 16)
    qh, e_h = oracle.quantise(h.astype(np.float64), 16)
    cv, cp = oracle.cuts(X, 256)   # max_bin >= distinct values -> bins are value ranks
    B = oracle.bins(X, cv, cp)
    D = 4
    lam, gamma, mcw = [(1.0, 0.0, 1e-3), (0.5, 0.01, 0.0), (1.0, 0.0, 0.2)][trial % 3]
    nodes, lor, _ = oracle.build_tree(B, m, cv, cp, qg, qh, e_g, e_h, D, lam, gamma, mcw, 1.0)
    ref = {}
    _greedy_raw(X, qg, qh, e_g, e_h, np.arange(n), 0, D, lam, gamma, mcw, ref, 0)
    for v, r in ref.items():
        assert nodes["n_rows"][v] == r["n"]
        assert nodes["sum_g"][v] == r["G"] * 2.0 ** -e_g
        assert nodes["feature"][v] == r["feature"], f"node {v}"
        if r["feature"] >= 0:
            assert nodes["split_value"][v] == np.float32(r["value"])
            assert abs(nodes["gain"][v] - r["gain"]) <= 1e-9 * max(1.0, abs(r["gain"]))
    present = set(ref)
    for v in range(len(nodes)):
        if v not in present:
            assert nodes["feature"][v] == -2
    # partition: every row satisfies its path predicates on raw values
    for i in range(n):
        v = lor[i]
        while v > 0:
            p = (v - 1) // 2
            left = v == 2 * p + 1
            assert (X[i, nodes["feature"][p]] <= nodes["split_value"][p]) == left
            v = p


def test_depth0_single_leaf():
    """max_depth = 0 -> one leaf with weight -G/(H+lambda)."""
    nodes, lor, _ = _two_bin_tree([0.5, -1.0, 2.0], [0.25, 0.5, 1.0], [0, 1, 1], depth=0, eta=1.0)
    assert len(nodes) == 1 and nodes["feature"][0] == -1
    assert nodes["leaf_value"][0] == np.float32(-1.5 / (1.75 + 1.0))


def test_separable_feature_depth1():
    """one feature perfectly separates the labels -> the root splits on it (n <= 256 so
    every distinct value is a cut and the separating threshold is a candidate)."""
    rng = np.random.default_rng(0)
    n = 250
    y = (rng.random(n) < 0.5).astype(np.float32)
    X = rng.normal(size=(n, 5)).astype(np.float32)
    X[:, 3] = y * 10 + rng.normal(scale=0.1, size=n).astype(np.float32)
    cv, cp = oracle.cuts(X, 256)
    B = oracle.bins(X, cv, cp)
    g, h = oracle.logistic_grad(np.zeros(n, np.float32), y)
    qg, e_g = oracle.quantise(g.astype(np.float64), 16)
    qh, e_h = oracle.quantise(h.astype(np.float64), 16)
    nodes, lor, _ = oracle.build_tree(B, 5, cv, cp, qg, qh, e_g, e_h, 1)
    assert nodes["feature"][0] == 3
    assert np.all((lor == 2) == (y == 1))


def test_tree_histograms_conserve_and_add():
    """Every internal node's histogram = left child's + right child's (additivity), and each
    feature's bins sum to the node totals (conservation)."""
    X, y = synth.make_classification(3000, 9, seed=8)
    cv, cp = oracle.cuts(X, 64)
    B = oracle.bins(X, cv, cp)
    g, h = oracle.logistic_grad(np.zeros(3000, np.float32), y)
    qg, e_g = oracle.quantise(g.astype(np.float64), 16)
    qh, e_h = oracle.quantise(h.astype(np.float64), 16)
    nodes, lor, H = oracle.build_tree(B, 9, cv, cp, qg, qh, e_g, e_h, 4, want_hist=True)
    for v in range(7):
        if nodes["feature"][v] < 0:
            continue
        assert np.all(H[v][:, :, 0].sum(axis=1) * 2.0 ** -e_g == nodes["sum_g"][v])
        if 2 * v + 2 < 15:
            np.testing.assert_array_equal(H[v], H[2 * v + 1] + H[2 * v + 2])


# ------------------------------------------------------------------------------ O11-O12
def test_predict_binned_equals_raw_traversal():
    """R3: right-inclusive cuts make the binned traversal equal the raw-value one."""
    X, y = synth.make_classification(2000, 7, seed=6)
    cv, cp = oracle.cuts(X, 32)
    B = oracle.bins(X, cv, cp)
    g, h = oracle.logistic_grad(np.zeros(2000, np.float32), y)
    qg, e_g = oracle.quantise(g.astype(np.float64), 16)
    qh, e_h = oracle.quantise(h.astype(np.float64), 16)
    nodes, lor, _ = oracle.build_tree(B, 7, cv, cp, qg, qh, e_g, e_h, 5)
    m0 = np.zeros(2000, np.float32)
    pm = oracle.predict(B, nodes, m0)
    ref = np.zeros(2000, np.float32)
    for i in range(2000):
        v = 0
        while nodes["feature"][v] >= 0:
            v = 2 * v + 1 if X[i, nodes["feature"][v]] <= nodes["split_value"][v] else 2 * v + 2
        ref[i] = nodes["leaf_value"][v]
        assert v == lor[i]
    np.testing.assert_array_equal(pm, ref)


def test_logistic_gradient_pins():
    """Golden S:L486 and finite differences of the logistic loss."""
    ex = GOLD["logistic_grad"]
    g, h = oracle.logistic_grad(np.array([ex["margin"]], np.float32), np.array([ex["y"]], np.float32))
    assert g[0] == ex["g"] and h[0] == ex["h"]
    m = np.linspace(-4, 4, 33).astype(np.float32)
    for yv in (0.0, 1.0):
        g, h = oracle.logistic_grad(m, np.full_like(m, yv))
        loss = lambda z: np.log1p(np.exp(-z)) if yv == 1 else np.log1p(np.exp(z))
        eps = 1e-4
        md = m.astype(np.float64)
        fd_g = (loss(md + eps) - loss(md - eps)) / (2 * eps)
        fd_h = (loss(md + eps) - 2 * loss(md) + loss(md - eps)) / eps**2
        np.testing.assert_allclose(g, fd_g, atol=1e-5)
        np.testing.assert_allclose(h, fd_h, atol=1e-3)


def test_auc_bruteforce_matches_sklearn():
    from sklearn.metrics import roc_auc_score
    rng = np.random.default_rng(0)
    s = np.round(rng.normal(size=300), 1).astype(np.float32)  # ties
    y = (rng.random(300) < 0.4).astype(np.float32)
    assert abs(oracle.auc_bruteforce(s, y) - roc_auc_score(y, s)) < 1e-12


def test_boosting_round_reduces_loss():
    """Config-1-shaped training through the oracle: the logistic loss decreases every round."""
    X, y = synth.make_classification(3000, 20, seed=0)
    cv, cp = oracle.cuts(X, 256)
    B = oracle.bins(X, cv, cp)
    margin = np.zeros(3000, np.float32)
    prev = None
    losses = []
    for r in range(4):
        prev, margin, _ = oracle.boosting_round(B, 20, cv, cp, margin, y, max_depth=6, prev_tree=prev, round_=r)
        mm = margin.astype(np.float64)
        losses.append(np.mean(np.log1p(np.exp(-np.where(y > 0, mm, -mm)))))
    assert all(b < a for a, b in zip(losses, losses[1:]))


# ------------------------------------------------------------------------------ R27 missing values
def _greedy_raw_missing(X, qg, qh, e_g, e_h, rows, depth, D, lam, gamma, mcw, out, v):
    """Exact greedy with missing values (NaN) straight from the raw rows: for every feature, every
    threshold t among the feature's present distinct values over ALL rows but the largest (its
    cut points) and both default directions (missing rows right, then left), left = {x <= t}
    (+ the missing rows for 'left'); so a node can also split present-vs-missing.  Python ints for
    the sums, Python floats for Eq. 8, (feature, t, direction) order with strict > (R13, R27)."""
    G, H = int(qg[rows].sum()), int(qh[rows].sum())
    out[v] = dict(G=G, H=H, n=len(rows), feature=-1)
    if depth == D or len(rows) == 0:
        return
    sc_g, sc_h = 2.0 ** -e_g, 2.0 ** -e_h
    gP, hP = G * sc_g, H * sc_h
    tP = (gP * gP) / (hP + lam)
    best = None
    for j in range(X.shape[1]):
        col = X[rows, j]
        miss = np.isnan(col)
        allv = X[:, j]
        vals = np.unique(allv[~np.isnan(allv)])  # the feature's cut points (max_bin >= distinct)
        for t in vals[:-1]:
            for dleft in (0, 1):
                L = rows[(col <= t) | (miss & bool(dleft))]
                GL, HL = int(qg[L].sum()), int(qh[L].sum())
                gl, hl, gr, hr = GL * sc_g, HL * sc_h, (G - GL) * sc_g, (H - HL) * sc_h
                if not (hl >= mcw and hr >= mcw):
                    continue
                gain = 0.5 * (((gl * gl) / (hl + lam) + (gr * gr) / (hr + lam)) - tP) - gamma
                if best is None or gain > best[0]:
                    best = (gain, j, float(t), dleft, L)
    if best is None or best[0] <= 0:
        return
    gain, j, t, dleft, L = best
    out[v].update(feature=j, value=t, gain=gain, default_left=dleft)
    R = np.setdiff1d(rows, L)
    _greedy_raw_missing(X, qg, qh, e_g, e_h, L, depth + 1, D, lam, gamma, mcw, out, 2 * v + 1)
    _greedy_raw_missing(X, qg, qh, e_g, e_h, R, depth + 1, D, lam, gamma, mcw, out, 2 * v + 2)


def _with_missing(rng, X, rates):
    X = X.copy()
    for j, r in enumerate(rates):
        X[rng.random(X.shape[0]) < r, j] = np.nan
    return X


def test_cuts_bins_skip_missing_values():
    """R27: the cuts of a feature are the R1 cuts of its present values (np.unique / the ceil rank
    of np.sort on the non-NaN values); a missing value's symbol is 255; an all-missing feature
    gets the single cut 0.0 (R1 step 5)."""
    rng = np.random.default_rng(31)
    X = rng.normal(size=(3000, 4)).astype(np.float32)
    X[:, 1] = np.round(X[:, 1] * 2)  # few distinct values
    X = _with_missing(rng, X, [0.2, 0.5, 0.0, 1.0])
    B = 64
    cv, cp = oracle.cuts(X, B)
    for j in range(4):
        pres = np.sort(X[~np.isnan(X[:, j]), j])
        c = cv[cp[j]:cp[j + 1]]
        if len(pres) == 0:
            assert list(c) == [0.0]
        elif len(np.unique(pres)) <= B:
            np.testing.assert_array_equal(c, np.unique(pres))
        else:
            N = len(pres)
            idx = (np.arange(1, B + 1) * N + B - 1) // B
            np.testing.assert_array_equal(c, np.unique(pres[idx - 1]))
    bins = oracle.bins(X, cv, cp)
    for j in range(4):
        miss = np.isnan(X[:, j])
        assert np.all(bins[miss, j] == 255)
        c = cv[cp[j]:cp[j + 1]]
        exp = np.minimum(np.searchsorted(c, X[~miss, j], side="left"), len(c) - 1)
        np.testing.assert_array_equal(bins[~miss, j], exp)


def test_missing_values_need_max_bin_255():
    """Symbol 255 marks a missing value, so a feature with 256 bins cannot hold one (ERR_ARG)."""
    rng = np.random.default_rng(32)
    X = rng.normal(size=(2000, 1)).astype(np.float32)
    cv, cp = oracle.cuts(X, 256)
    assert cp[1] == 256
    X[5, 0] = np.nan
    with pytest.raises(oracle.OracleError):
        oracle.bins(X, cv, cp)
    cv, cp = oracle.cuts(X, 255)
    assert oracle.bins(X, cv, cp)[5, 0] == 255


@pytest.mark.parametrize("trial", range(10))
def test_tree_with_missing_equals_exhaustive_greedy(trial):
    """R27: the binned oracle with missing values (symbol 255, both default directions) equals the
    exact greedy tree computed from the raw values with NaN, node by node (feature, value,
    default direction, gain, sums); every row satisfies its path predicates with missing values
    following the default directions."""
    rng = np.random.default_rng(300 + trial)
    n = int(rng.integers(10, 200))
    m = int(rng.integers(1, 5))
    X = np.round(rng.normal(size=(n, m)) * (2 + trial % 3)).astype(np.float32)
    X = _with_missing(rng, X, rng.uniform(0.0, 0.6, size=m))
    y = (rng.random(n) < 0.5).astype(np.float32)
    g, h = oracle.logistic_grad(rng.normal(size=n).astype(np.float32), y)
    qg, e_g = oracle.quantise(g.astype(np.float64), 16)
    qh, e_h = oracle.quantise(h.astype(np.float64), 16)
    cv, cp = oracle.cuts(X, 255)
    B = oracle.bins(X, cv, cp)
    D = 4
    lam, gamma, mcw = [(1.0, 0.0, 1e-3), (0.5, 0.01, 0.0), (1.0, 0.0, 0.2)][trial % 3]
    nodes, lor, _ = oracle.build_tree(B, m, cv, cp, qg, qh, e_g, e_h, D, lam, gamma, mcw, 1.0, has_missing=True)
    ref = {}
    _greedy_raw_missing(X, qg, qh, e_g, e_h, np.arange(n), 0, D, lam, gamma, mcw, ref, 0)
    for v, r in ref.items():
        assert nodes["n_rows"][v] == r["n"]
        assert nodes["sum_g"][v] == r["G"] * 2.0 ** -e_g
        assert nodes["feature"][v] == r["feature"], f"node {v}"
        if r["feature"] >= 0:
            assert nodes["split_value"][v] == np.float32(r["value"])
            assert nodes["default_left"][v] == r["default_left"], f"node {v}"
            assert abs(nodes["gain"][v] - r["gain"]) <= 1e-9 * max(1.0, abs(r["gain"]))
    for i in range(n):
        v = lor[i]
        while v > 0:
            p = (v - 1) // 2
            x = X[i, nodes["feature"][p]]
            goes_left = bool(nodes["default_left"][p]) if np.isnan(x) else x <= nodes["split_value"][p]
            assert goes_left == (v == 2 * p + 1)
            v = p


def test_missing_rows_pick_their_side():
    """A fixture where only the default direction differs between the candidates: feature 0 is 0
    on rows 0-29 (g = +1), 1 on rows 30-59 (g = +0.9) and missing on rows 60-89 (g = -1); its one
    threshold (bin 0) is tried with the missing rows on either side, and the partition follows the
    default direction the split records (R27)."""
    n = 90
    X = np.zeros((n, 1), np.float32)
    X[30:60, 0] = 1.0
    X[60:, 0] = np.nan
    g = np.where(np.arange(n) < 60, 1.0, -1.0)
    g[30:60] = 0.9
    h = np.full(n, 0.25)
    qg, e_g = oracle.quantise(g, 16)
    qh, e_h = oracle.quantise(h, 16)
    cv, cp = oracle.cuts(X, 255)
    B = oracle.bins(X, cv, cp)
    nodes, lor, _ = oracle.build_tree(B, 1, cv, cp, qg, qh, e_g, e_h, 1, 1.0, 0.0, 0.0, 1.0, has_missing=True)
    assert nodes["feature"][0] == 0 and nodes["split_bin"][0] == 0
    exp_left = set(range(30)) if nodes["default_left"][0] == 0 else set(range(30)) | set(range(60, 90))
    assert set(np.nonzero(lor == 1)[0]) == exp_left
    assert nodes["gain"][0] > 0


def test_predict_with_missing_follows_default_direction():
    """Binned predict (symbol 255 -> the node's default direction) equals a raw traversal of the
    tree on the values with NaN."""
    rng = np.random.default_rng(33)
    n, m = 400, 3
    X = _with_missing(rng, np.round(rng.normal(size=(n, m)) * 3).astype(np.float32), [0.3, 0.1, 0.5])
    y = (rng.random(n) < 0.5).astype(np.float32)
    g, h = oracle.logistic_grad(rng.normal(size=n).astype(np.float32), y)
    qg, e_g = oracle.quantise(g.astype(np.float64), 16)
    qh, e_h = oracle.quantise(h.astype(np.float64), 16)
    cv, cp = oracle.cuts(X, 255)
    B = oracle.bins(X, cv, cp)
    nodes, _, _ = oracle.build_tree(B, m, cv, cp, qg, qh, e_g, e_h, 5, 1.0, 0.0, 0.1, 1.0, has_missing=True)
    assert (nodes["default_left"][nodes["feature"] >= 0] == 1).any()
    m0 = rng.normal(size=n).astype(np.float32)
    got = oracle.predict(B, nodes, m0, has_missing=True)
    exp = m0.copy()
    for i in range(n):
        v = 0
        while nodes["feature"][v] >= 0:
            x = X[i, nodes["feature"][v]]
            left = bool(nodes["default_left"][v]) if np.isnan(x) else x <= nodes["split_value"][v]
            v = 2 * v + 1 if left else 2 * v + 2
        exp[i] = exp[i] + nodes["leaf_value"][v]
    np.testing.assert_array_equal(got, exp)
