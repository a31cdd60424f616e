"""CPU-only checks of the boundary and the host logic (no GPU compute):
 - liboocgb.so builds for sm_100a, loads, and exports every symbol include/oocgb.h declares;
 - the Python binding declares exactly that ABI;
 - the product package never imports the oracle (no CPU fallback);
 - multi-process (gloo, world_size 2): row sharding, NCCL-id bootstrap, and the exactness of the
   data path's only exchange (an int64 sum of per-rank histograms) against the oracle.
"""
import os
import re
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "oocgb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(oocgb_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2005_09148_b200 import build
    path = build.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", path], text=True)
    exported = set(re.findall(r"\bT (oocgb_\w+)", out))
    missing = [s for s in _header_symbols() if s not in exported]
    assert not missing, f"declared but not exported: {missing}"
    import paper_2005_09148_b200 as ob
    assert sorted(ob.ABI_SYMBOLS) == _header_symbols()
    L = ob.load_library()
    assert L.oocgb_abi_version() == 2  # 2: default_left, has_missing, CSR input (R27)


def test_library_is_sm100a():
    from paper_2005_09148_b200 import build
    path = build.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], text=True)
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2005_09148_b200 as ob
    with pytest.raises(ob.OocgbError) as e:
        ob.Context(0)
    assert e.value.status in (ob.ERR_ARG, ob.ERR_DEVICE)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2005_09148_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "orc_" not in txt, f


def test_shard_rows_partition():
    from paper_2005_09148_b200.dist import shard_rows
    for n in (0, 1, 7, 1000, 10**8 + 3):
        for w in (1, 2, 3, 8):
            spans = [shard_rows(n, r, w) for r in range(w)]
            assert spans[0][0] == 0
            for (a, na), (b, _) in zip(spans, spans[1:]):
                assert a + na == b
            assert sum(s[1] for s in spans) == n
            assert max(s[1] for s in spans) - min(s[1] for s in spans) <= 1


_WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["OOCGB_ROOT"])
import numpy as np, torch, torch.distributed as dist
import oracle, synth
from paper_2005_09148_b200.dist import shard_rows, bootstrap_nccl_id
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
nid = bootstrap_nccl_id(rank, lambda: bytes(range(128)))
assert nid == bytes(range(128))
# same global data on every rank (seeded); each rank owns a contiguous row shard
n, m = 3001, 11
X, y = synth.make_classification(n, m, seed=4)
cv, cp = oracle.cuts(X, 64)
B = oracle.bins(X, cv, cp)
rng = np.random.default_rng(1)
qg = rng.integers(-2**16, 2**16 + 1, size=n); qh = rng.integers(0, 2**16 + 1, size=n)
row0, nl = shard_rows(n, rank, world)
rows = np.arange(row0, row0 + nl)
h = torch.from_numpy(oracle.histogram(B, m, rows, qg, qh).copy())
dist.all_reduce(h)            # the exchange step of P:L188-190 (int64 sum)
full = oracle.histogram(B, m, np.arange(n), qg, qh)
assert np.array_equal(h.numpy(), full), "sharded int64 histogram sum != full histogram"
# sampling is keyed by global row: a rank's selection of its rows equals the global one
g, hh = synth.gradient_pairs(n, seed=2)
s_full = oracle.sample(g, hh, oracle.SAMPLE_UNIFORM, 0.3, seed=5, round_=2)
u = np.array([oracle.uniform(5, 2, r, 0) for r in rows])
assert np.array_equal(s_full["selected"][rows].astype(bool), u < (round(0.3 * 2**32) * 2.0**-32))
dist.barrier()
print("worker ok", rank)
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_world2_exchange_is_exact(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), OOCGB_ROOT=ROOT)
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=240)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
        assert "worker ok" in o


def test_bench_reference_arm_under_torchrun_rank1_exits_clean():
    """bench.py --impl reference: rank != 0 exits 0 without work (contract for N > 1)."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""


PLANNER_CHECK = r'''
#include "paper_2005_09148_b200/csrc/internal.cuh"
#include <cstdio>
#include <random>
#include <vector>
// hist_chunk_rows (the histogram chunk planner of the root level and the streamed batches):
// chunks never exceed kmax rows (the s32 exactness bound), hold every pair, and fill at most
// the fewest whole waves of the k_hist grid that hold the level with >= 2 n_pairs - 1 chunks.
int main() {
  std::mt19937_64 g(5);
  int bad = 0;
  for (int it = 0; it < 20000; ++it) {
    const int n_fg = 1 + (int)(g() % 32), grid = 148 * (1 + (int)(g() % 3));
    const long long kmax = 0x7fffffffLL >> (10 + (int)(g() % 12));
    const int n_pairs = 1 + (int)(g() % 300);
    std::vector<long long> c(n_pairs);
    long long tot = 0;
    for (auto &x : c) { x = (long long)(g() % (1 + (g() % 2 ? 4000 : 400000))); tot += x; }
    const long long cr = oocgb::hist_chunk_rows(tot, n_pairs, n_fg, grid, kmax);
    long long chunks = 0;
    for (auto x : c) chunks += (x + cr - 1) / cr;
    const long long lo = kmax < 1024 ? kmax : 1024;
    // the wave count the planner picked: the smallest w whose budget C admits cr
    long long C = 0;
    for (long long w = 1;; ++w) {
      C = w * grid / n_fg;
      if (C < 2LL * n_pairs - 1 || C < 1) continue;
      const long long t = (tot + (C - n_pairs + 1) - 1) / (C - n_pairs + 1);
      if (t <= kmax) break;
    }
    if (cr > kmax || cr < lo || chunks > C) {
      if (bad++ < 5) printf("bad: tot %lld pairs %d n_fg %d grid %d kmax %lld -> cr %lld chunks %lld C %lld\n", tot,
                            n_pairs, n_fg, grid, kmax, cr, chunks, C);
    }
  }
  printf("%s\n", bad ? "FAIL" : "OK");
  return bad ? 1 : 0;
}
'''


def test_hist_chunk_planner_invariants(tmp_path):
    """The chunk planner (internal.cuh hist_chunk_rows, DESIGN.md §5 item scheduling), compiled for
    the host: chunk rows within [min(1024, kmax), kmax] (s32 exactness of the partials, R12) and the
    chunk count within the chosen number of whole waves, over random levels."""
    import shutil
    import subprocess
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    src = tmp_path / "planner.cu"
    src.write_text(PLANNER_CHECK)
    exe = tmp_path / "planner"
    subprocess.check_call([nvcc, "-std=c++17", "-O1", "-I", ROOT, "-o", str(exe), str(src)],
                          stdout=subprocess.DEVNULL, stderr=subprocess.STDOUT)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip().endswith("OK"), out.stdout


_SHARD_WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["OOCGB_ROOT"])
import torch, torch.distributed as dist
import bench, synth
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
n_global, m, chunk = 4501, 6, 1000
row0, n, pieces = bench.shard_chunks(n_global, rank, world, chunk=chunk)
Xs, ys = [], []
for c0, cn, b, e in pieces:
    assert c0 % chunk == 0 and 0 <= b < e <= cn
    X, y = synth.torch_classification_chunk(c0, cn, m, seed=5, device="cpu")
    Xs.append(X[b:e]); ys.append(y[b:e])
X = torch.cat(Xs); y = torch.cat(ys)
assert X.shape == (n, m) and y.shape == (n,)
meta = [None] * world
dist.all_gather_object(meta, (row0, n, X.numpy().tobytes(), y.numpy().tobytes()))
if rank == 0:
    # the ranks' rows tile [0, n_global) and equal the 1-rank generation of the same global grid
    r = 0
    for (r0, nn, _, _) in meta:
        assert r0 == r
        r += nn
    assert r == n_global
    _, _, pieces1 = bench.shard_chunks(n_global, 0, 1, chunk=chunk)
    X1 = torch.cat([synth.torch_classification_chunk(c0, cn, m, seed=5, device="cpu")[0][b:e] for c0, cn, b, e in pieces1])
    got = b"".join(mm[2] for mm in meta)
    assert got == X1.numpy().tobytes(), "sharded generation differs from the 1-rank data set"
dist.barrier()
print("worker ok", rank)
'''


@pytest.mark.parametrize("world", [2, 3])
def test_bench_multirank_data_path_gloo(tmp_path, world):
    """bench.py's multi-GPU data path on CPU with gloo: every rank generates its
    rows of the global chunk grid (synth.torch_classification_chunk, here on the CPU), the shards
    tile the global rows, and their union is exactly the 1-rank data set, for any world size."""
    script = tmp_path / "shard.py"
    script.write_text(_SHARD_WORKER)
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), OOCGB_ROOT=ROOT)
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=240)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
        assert "worker ok" in o
