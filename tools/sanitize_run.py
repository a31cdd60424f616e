"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): the library's
whole hot path on small seeded inputs through the public API -- quantise (sketch, cuts, bins),
logistic gradients, sample (NONE, UNIFORM, MVS, GOSS), build_tree (multi-chunk root, int64 and
int32 evaluation lists, the partition's inline plan, > 256 segments at depth 10), update_margin,
predict, and the out-of-core path (pinned pages, compaction, Alg. 6 streamed build).
usage: compute-sanitizer --tool <tool> python tools/sanitize_run.py [small]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_09148_b200 as ob  # noqa: E402
import synth  # noqa: E402


def main(small):
    ctx = ob.Context(0)
    cases = [(5000, 40, 6), (40000, 24, 10)] if small else [(5000, 40, 6), (120000, 64, 8), (70000, 8, 11)]
    for n, m, depth in cases:
        X, y = synth.make_classification(n, m, seed=n)
        d = ctx.quantise(X, 256)
        margin = np.zeros(n, np.float32)
        prev = None
        for r, (mode, ratio) in enumerate([(0, 1.0), (2, 0.3), (1, 0.5)]):
            if prev is not None:
                margin = d.predict([prev], margin)
                prev.close()
            d.set_logistic_gradients(margin, y)
            d.sample(mode, ratio, 1.0, seed=1, round=r, quant_bits=16)
            prev = d.build_tree(depth, keep_debug=(r == 0))
            if mode == 0:
                margin = d.update_margin(prev, margin)
        d.sample_goss(0.1, 0.2, seed=1, round=9, quant_bits=16)
        t = d.build_tree(depth)
        t.close()
        prev.close()
        d.close()
        print("in-core ok", n, m, depth, flush=True)
    n, m = 20000, 40
    X, y = synth.make_classification(n, m, seed=3)
    d = ctx.quantise(X, 256, page_bytes=3000 * 64, placement=ob.PLACE_PINNED_HOST)
    d.set_logistic_gradients(np.zeros(n, np.float32), y)
    d.sample(2, 0.2, 1.0, seed=1, round=0, quant_bits=16)
    t = d.build_tree(6)
    mg = d.predict([t], np.zeros(n, np.float32))
    t.close()
    d.set_streaming(True)
    d.set_logistic_gradients(mg, y)
    d.sample(0, 1.0, round=1)
    t = d.build_tree(6)
    d.update_margin(t, mg)
    t.close()
    d.close()
    ctx.close()
    print("out-of-core ok")


if __name__ == "__main__":
    main("small" in sys.argv)
