"""Sampling-only timing at config-4 size (100M rows): sample(mode, f) per mode with CUDA events, the
gradients resident on the device (logistic-shaped, generated on the GPU), X a single constant
feature (quantise is not what is timed).  usage: python tools/sample_bench.py [rows] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_09148_b200 as ob  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx = ob.Context(0, stream=st.cuda_stream)
    d = ctx.quantise(torch.zeros((n, 1), dtype=torch.float32, device="cuda"), 2)
    gen = torch.Generator(device="cuda").manual_seed(1)
    p = torch.rand(n, generator=gen, device="cuda") * 0.96 + 0.02
    y = (torch.rand(n, generator=gen, device="cuda") < 0.5).float()
    g = (p - y).contiguous()
    h = (p * (1 - p)).contiguous()
    d.set_gradients(g, h)
    for name, call in [("none", lambda r: d.sample(0, 1.0, round=r)),
                       ("uniform 0.1", lambda r: d.sample(1, 0.1, seed=1, round=r)),
                       ("mvs 0.1", lambda r: d.sample(2, 0.1, 1.0, seed=1, round=r)),
                       ("goss 0.05+0.05", lambda r: d.sample_goss(0.05, 0.05, seed=1, round=r))]:
        call(0)
        ts = []
        for r in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            info = call(r + 1)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"{name:16s} median {sorted(ts)[len(ts) // 2]:.3f} ms  (selected {info['n_selected_global']})", flush=True)
    d.close()
    ctx.close()


if __name__ == "__main__":
    main()
