"""Precision study for DESIGN.md reading R12 (fixed-point gradient pairs, quant_bits = P).

Not collected by pytest (long-running evidence script; lives under tests/ because it calls the
oracle, which only tests may).  It answers VERDICT r1 item 2: does the library's P = 16 lose
anything against the P = 24 SURVEY O5 proposed and against (effectively) float64 gradients?

Everything here is the CPU oracle (oracle/), which implements R12 for any P (int64 sums):
  * P = 40 stands in for float64 gradients: |q| <= 2^40, the quantisation step of the largest
    row is 2^-40 relative (float64 arithmetic on the sums is 2^-53), n <= 2^23 keeps the int64
    sums exact.
  * trajectories: 100 boosting rounds (binary:logistic, lambda 1, gamma 0, mcw 1, eta 0.1, f = 1)
    at P = 16, 24 and 40 from margin 0; held-out AUC (sklearn) after rounds 10, 50 and 100.
  * per-tree agreement on the SAME gradients: every 5th round of the P = 40 trajectory, trees
    at P = 16 and P = 24 are built from that round's gradients and compared node by node with
    the P = 40 tree: same split (feature, bin) at every node, relative error of the gain at
    nodes with the same split, max |leaf difference|.

usage: python tests/study_precision.py {config1|config2} P_traj [--out file]
       (one trajectory per process; run P = 16, 24, 40 in parallel; the P = 40 run also does the
       per-tree comparison)
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402


def workload(name):
    if name == "config1":
        X, y = synth.make_classification(12000, 20, seed=0)
        return X[:10000], y[:10000], X[10000:], y[10000:], 6
    X, y = synth.fast_classification(1_050_000, 500, seed=1000)
    return X[:1_000_000], y[:1_000_000], X[1_000_000:], y[1_000_000:], 8


def build(B, m, cv, cp, g, h, P, depth):
    qg, e_g = oracle.quantise(g.astype(np.float64), P)
    qh, e_h = oracle.quantise(h.astype(np.float64), P)
    nodes, lor, _ = oracle.build_tree(B, m, cv, cp, qg, qh, e_g, e_h, depth, 1.0, 0.0, 1.0, 0.1)
    return nodes


def compare(ref, other):
    sp = ref["feature"] >= 0
    same = (ref["feature"] == other["feature"]) & (ref["split_bin"] == other["split_bin"])
    both = sp & same
    rel = np.abs(other["gain"][both] - ref["gain"][both]) / np.abs(ref["gain"][both])
    pres = (ref["feature"] != -2) & (other["feature"] != -2)
    return {"split_nodes": int(sp.sum()), "same_split": int((sp & same).sum()),
            "first_diff_node": int(np.nonzero(sp & ~same)[0][0]) if (sp & ~same).any() else -1,
            "gain_rel_err_max": float(rel.max()) if rel.size else 0.0,
            "gain_rel_err_median": float(np.median(rel)) if rel.size else 0.0,
            "leaf_abs_diff_max": float(np.max(np.abs(other["leaf_value"][pres] - ref["leaf_value"][pres])))
            if pres.any() else 0.0}


def main():
    from sklearn.metrics import roc_auc_score
    name, P = sys.argv[1], int(sys.argv[2])
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    rounds = 100
    X, y, Xe, ye, depth = workload(name)
    m = X.shape[1]
    t0 = time.time()
    cv, cp = oracle.cuts(X, 256)
    B = oracle.bins(X, cv, cp)
    Be = oracle.bins(Xe, cv, cp)
    del X, Xe
    margin = np.zeros(len(y), np.float32)
    em = np.zeros(len(ye), np.float32)
    auc, cmp16, cmp24 = {}, [], []
    for r in range(rounds):
        g, h = oracle.logistic_grad(margin, y)
        nodes = build(B, m, cv, cp, g, h, P, depth)
        if P == 40 and r % 5 == 0:
            cmp16.append(dict(round=r, **compare(nodes, build(B, m, cv, cp, g, h, 16, depth))))
            cmp24.append(dict(round=r, **compare(nodes, build(B, m, cv, cp, g, h, 24, depth))))
            print(r, cmp16[-1], cmp24[-1], flush=True)
        margin = oracle.predict(B, nodes, margin)
        em = oracle.predict(Be, nodes, em)
        if r + 1 in (10, 50, 100):
            auc[r + 1] = float(roc_auc_score(ye, em))
            print(name, "P", P, "round", r + 1, "auc", auc[r + 1], f"{time.time() - t0:.0f}s", flush=True)
    res = {"workload": name, "quant_bits": P, "rounds": rounds, "depth": depth, "held_out_rows": int(len(ye)),
           "auc": auc, "seconds": time.time() - t0}
    if cmp16:
        res["per_tree_vs_P40"] = {"P16": cmp16, "P24": cmp24}
    text = json.dumps(res)
    print(text)
    if out:
        with open(out, "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    main()
