"""Root-histogram rate vs input size (L2-resident vs HBM-streamed): depth-1 trees, k_hist phase
time from the library's CUDA-event timings.  usage: python tools/hist_rate.py [rows ...]"""
import sys

import numpy as np
import torch

import paper_2005_09148_b200 as ob
import synth


def main(sizes):
    ctx = ob.Context(0)
    ctx.set_profiling(True)
    for n in sizes:
        X, y = synth.fast_classification(n, 500, seed=7)
        d = ctx.quantise(X, 256)
        rng = np.random.default_rng(1)
        g = rng.uniform(-1, 1, n).astype(np.float32)
        h = rng.uniform(0.01, 0.25, n).astype(np.float32)
        d.set_gradients(g, h)
        d.sample(ob.SAMPLE_NONE, 1.0)
        for _ in range(3):
            d.build_tree(1).close()
        torch.cuda.synchronize()
        t0 = ctx.get_timings()
        reps = 20
        for _ in range(reps):
            d.build_tree(1).close()
        t1 = ctx.get_timings()
        ms = (t1["hist_ms"] - t0["hist_ms"]) / reps
        sym = n * 500
        print(f"rows {n:>9d}: root k_hist {ms * 1e3:8.1f} us  {sym / (ms * 1e-3) / 1e12:6.3f} T symbols/s  "
              f"{sym * 2 / 32 / (ms * 1e-3) / 148 / 1.9e9:5.3f} warp-atomics/clk/SM", flush=True)
        d.close()


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [50_000, 100_000, 200_000, 1_000_000])
