import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle, synth, paper_2005_09148_b200 as ob
from test_gpu_parity import _oracle_cuts_bins, _oracle_tree
n, m, max_bin, depth = 3000, 20, 256, 6
X, y = synth.make_classification(n, m, seed=7 + n, stress=False)
X = np.ascontiguousarray(X[:, :m])
cv, cp, B = _oracle_cuts_bins(X, max_bin)
margin = np.random.default_rng(n).normal(scale=0.5, size=n).astype(np.float32)
g, h = oracle.logistic_grad(margin, y)
on, olor, ohist, sel = _oracle_tree(B, m, cv, cp, g, h, 0, 1.0, depth, quant_bits=16)
ctx = ob.Context(0)
d = ctx.quantise(X, max_bin); d.set_gradients(g, h)
info = d.sample(0, 1.0, 1.0, 1, 0, 16)
t = d.build_tree(depth, 1.0, 0.0, 1.0, 0.1, keep_debug=True)
gn = t.export()
for f in ('feature','split_bin','n_rows'):
    bad = np.nonzero(gn[f] != on[f])[0]
    print(f, 'mismatch nodes', bad[:20], gn[f][bad[:5]], on[f][bad[:5]])
lor = t.get_partition(n)
bad = np.nonzero(lor != olor)[0]
print('partition mismatches', len(bad))
import collections
print(collections.Counter(zip(lor[bad].tolist(), olor[bad].tolist())).most_common(10))
