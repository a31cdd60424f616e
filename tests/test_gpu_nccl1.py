"""The NCCL transport of the sharded path on ONE GPU: a context created with an NCCL
id and world = 1 runs the multi-GPU code path on a 1-rank communicator -- the sketch all-gather,
the fixed-point maxima and MVS radix statistics all-reduces, the per-level int64 histogram
all-reduce (k_reduce_partials + ncclAllReduce, captured in the build's CUDA graph), the node
row-count all-reduce and the separate plan kernel.  Every result must be bit-identical to the
plain 1-GPU context (and hence to the oracle, which the plain context is pinned to elsewhere).
The multi-rank exchange itself is covered by test_gpu_multirank.py (host transport, 2 ranks)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _round(ctx, X, y, margin, mode, ratio, depth, rounds=2):
    d = ctx.quantise(X, 256)
    out = []
    prev = None
    m = margin.copy()
    for r in range(rounds):
        if prev is not None:
            m = d.predict([prev], m)
            prev.close()
        d.set_logistic_gradients(m, y)
        info = d.sample(mode, ratio, 1.0, seed=7, round=r, quant_bits=16)
        gid, qg, qh = d.get_sample(info["n_selected_local"])
        t = d.build_tree(depth)
        out.append((info, gid, qg, qh, t.export()))
        prev = t
    cv, cp = d.get_cuts()
    bins = d.get_bins()
    pm = d.predict([prev], np.zeros(len(y), np.float32))
    prev.close()
    d.close()
    return out, cv, cp, bins, pm


@pytest.mark.parametrize("n,m,mode,ratio,depth", [
    (30000, 40, 0, 1.0, 6),        # SAMPLE_NONE: every level's histogram through ncclAllReduce
    (50000, 70, 2, 0.3, 7),        # MVS: radix statistics all-reduces, compaction of the sample
    (20000, 33, 1, 0.5, 5),        # UNIFORM
])
def test_nccl_one_rank_matches_plain_context(n, m, mode, ratio, depth):
    import paper_2005_09148_b200 as ob
    X, y = synth.make_classification(n, m, seed=11)
    margin = np.random.default_rng(5).normal(scale=0.3, size=n).astype(np.float32)
    c_plain = ob.Context(0)
    ref = _round(c_plain, X, y, margin, mode, ratio, depth)
    c_plain.close()
    c_nccl = ob.Context(0, 0, 1, nccl_id=ob.nccl_unique_id())
    got = _round(c_nccl, X, y, margin, mode, ratio, depth)
    c_nccl.close()
    (r_rounds, r_cv, r_cp, r_bins, r_pm), (g_rounds, g_cv, g_cp, g_bins, g_pm) = ref, got
    assert r_cv.tobytes() == g_cv.tobytes() and np.array_equal(r_cp, g_cp), "cuts differ"
    assert np.array_equal(r_bins, g_bins), "bins differ"
    for (ri, rg, rqg, rqh, rn), (gi, gg, gqg, gqh, gn) in zip(r_rounds, g_rounds):
        for k in ("n_selected_global", "e_g", "e_h", "k_star", "mu"):
            if k in ri:
                assert ri[k] == gi[k], k
        assert np.array_equal(rg, gg) and np.array_equal(rqg, gqg) and np.array_equal(rqh, gqh), "sample differs"
        for f in rn.dtype.names:
            assert np.array_equal(rn[f], gn[f]), f"tree field {f} differs (NCCL 1-rank vs plain)"
        assert int((rn["feature"] >= 0).sum()) > 0, "degenerate tree"
    assert np.array_equal(r_pm, g_pm), "predictions differ"
