"""Multi-rank parity on ONE GPU: two processes (ranks) share cuda:0 and exchange through the
host-callback transport (gloo), exercising every exchange step of the sharded algorithm
(P:L188-190): the sketch all-gather, fixed-point maxima, MVS radix statistics, per-level
histogram all-reduce and node row counts.  The 2-rank trees, cuts and sample sets must be
bit-identical to the 1-rank run on the full data (integer sums are order independent, every
random draw is keyed by the global row)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys, json
sys.path.insert(0, os.environ["OOCGB_ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2005_09148_b200 as ob, synth, oracle
from paper_2005_09148_b200.dist import shard_rows, gloo_collective
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
n, m, mode, ratio, depth = int(os.environ["N"]), int(os.environ["M"]), int(os.environ["MODE"]), float(os.environ["RATIO"]), 6
X, y = synth.make_classification(n, m, seed=5) if n < 200000 else synth.fast_classification(n, m, seed=5)
rng = np.random.default_rng(3)
margin = rng.normal(scale=0.5, size=n).astype(np.float32)
row0, nl = shard_rows(n, rank, world)
ctx = ob.Context(0, rank, world, host_collective=gloo_collective())
d = ctx.quantise(X[row0:row0 + nl], 256, row0_global=row0, n_rows_global=n)
g_all, h_all = oracle.logistic_grad(margin, y)  # host gradients: identical inputs for the oracle
d.set_gradients(g_all[row0:row0 + nl], h_all[row0:row0 + nl])
info = d.sample(mode, ratio, 1.0, seed=7, round=2, quant_bits=16)
gid, qg, qh = d.get_sample(info["n_selected_local"])
t = d.build_tree(depth, keep_debug=True)
nodes = t.export()
hist0 = t.get_histogram(0)   # complete over all features (each rank evaluated a feature slice)
hist1 = t.get_histogram(1) if nodes["feature"][0] >= 0 else None
cv, cp = d.get_cuts()
pm = d.predict([t], np.zeros(nl, np.float32))
res = dict(rank=rank, cuts=cv.tobytes().hex()[:4000], ncuts=int(cp[-1]), cuts_hash=hash(cv.tobytes()),
           gid=gid.tolist()[:50], nsel=info["n_selected_local"], nsel_g=info["n_selected_global"],
           k_star=info["k_star"], mu=info["mu"], e=(info["e_g"], info["e_h"]),
           nodes=[list(map(float, r)) for r in nodes.tolist()], pm_hash=hash(pm.tobytes()))
# single-rank reference on the full data (rank 0 only)
if rank == 0:
    c1 = ob.Context(0)
    d1 = c1.quantise(X, 256)
    d1.set_gradients(g_all, h_all)
    i1 = d1.sample(mode, ratio, 1.0, seed=7, round=2, quant_bits=16)
    g1, _, _ = d1.get_sample(i1["n_selected_local"])
    t1 = d1.build_tree(depth)
    n1 = t1.export()
    cv1, cp1 = d1.get_cuts()
    assert cv1.tobytes() == cv.tobytes() and np.array_equal(cp1, cp), "cuts differ"
    assert i1["n_selected_global"] == info["n_selected_global"], "sample size differs"
    assert (i1["k_star"], i1["mu"], i1["e_g"], i1["e_h"]) == (info["k_star"], info["mu"], info["e_g"], info["e_h"])
    assert np.array_equal(g1[: len(gid)], gid) or rank != 0, "rank-0 selected rows differ"
    for f in n1.dtype.names:
        assert np.array_equal(n1[f], nodes[f]), f"tree field {f} differs (2 ranks vs 1)"
    p1 = d1.predict([t1], np.zeros(n, np.float32))
    assert np.array_equal(p1[row0:row0 + nl], pm), "predict differs"
    # the oracle on the full data (Alg. 1 + Eq. 8, R9 sampling, R12 fixed point): the 2-rank tree
    # is compared with it directly, field by field
    ocv, ocp = oracle.cuts(X, 256, seed=2)
    assert ocv.tobytes() == cv.tobytes() and np.array_equal(ocp, cp), "cuts differ from the oracle"
    OB = oracle.bins(X, ocv, ocp)
    s_ = oracle.sample(g_all, h_all, mode, ratio, 1.0, 7, 2)
    sel_ = s_["selected"].astype(bool)
    assert int(sel_.sum()) == info["n_selected_global"], "sample size differs from the oracle"
    oqg, oe_g = oracle.quantise(s_["gs"][sel_], 16)
    oqh, oe_h = oracle.quantise(s_["hs"][sel_], 16)
    assert (oe_g, oe_h) == (info["e_g"], info["e_h"]), "fixed-point exponents differ from the oracle"
    on_, _, ohist_ = oracle.build_tree(OB[sel_], m, ocv, ocp, oqg, oqh, oe_g, oe_h, depth, want_hist=True)
    for f in on_.dtype.names:
        assert np.array_equal(on_[f], nodes[f]), f"tree field {f} differs (2 ranks vs oracle)"
    assert np.array_equal(hist0, ohist_[0]), "root histogram differs from the oracle"
    if hist1 is not None:
        assert np.array_equal(hist1, ohist_[1]), "node-1 histogram differs from the oracle"
    op = oracle.predict(OB, on_, np.zeros(n, np.float32))
    assert np.array_equal(op[row0:row0 + nl], pm), "predict differs from the oracle"
    print("RANK0-REFERENCE-OK", info["n_selected_global"], int((n1["feature"] >= 0).sum()))
all_g = [None] * world
dist.all_gather_object(all_g, gid.tolist())
if rank == 0 and ratio < 1.0:
    cat = np.concatenate([np.array(a, np.int64) for a in all_g])
    assert np.array_equal(cat, g1), "union of the ranks' selections != 1-rank selection"
    print("UNION-OK", len(cat))
dist.barrier()
print("worker ok", rank)
'''


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,m,mode,ratio,world", [(30000, 40, 0, 1.0, 2), (25000, 33, 2, 0.3, 2),
                                                  (20000, 24, 1, 0.5, 2), ((1 << 20) + 5000, 8, 2, 0.1, 2),
                                                  (20000, 8, 0, 1.0, 3)])
def test_two_ranks_one_gpu_bit_exact(ctx, tmp_path, n, m, mode, ratio, world):
    """World 2 (and 3: feature slices of 3, 3 and 2 features) on one GPU through the host transport:
    sharded rows, reduce-scattered histograms with a feature-sharded evaluation, all-gathered
    candidates -- bit-identical to 1 rank and to the oracle."""
    script = tmp_path / "w.py"
    script.write_text(WORKER)
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), OOCGB_ROOT=ROOT, N=str(n), M=str(m), MODE=str(mode), RATIO=str(ratio))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-4000:]
    assert "RANK0-REFERENCE-OK" in outs[0], outs[0][-3000:]
