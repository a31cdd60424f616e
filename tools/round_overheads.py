"""Config-2 round time under three host/graph regimes (diagnostic): (a) profiling event nodes in
the graph + per-round tree export, (b) no event nodes + per-round export, (c) no event nodes,
exports after the loop.  usage: PYTHONPATH=. python tools/round_overheads.py"""
import torch

import paper_2005_09148_b200 as ob
import synth


def main(rows=1_000_000, steps=20):
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = ob.Context(0, stream=stream.cuda_stream)
    X, y = synth.fast_classification(rows, 500, seed=1000)
    d = ctx.quantise(torch.from_numpy(X).cuda(), 256)
    yd = torch.from_numpy(y).cuda()
    margin = torch.zeros(rows, dtype=torch.float32, device="cuda")
    state = {"tree": None, "r": 0}

    def rnd():
        if state["tree"] is not None:
            d.update_margin(state["tree"], margin)
        d.set_logistic_gradients(margin, yd)
        d.sample(ob.SAMPLE_NONE, 1.0, round=state["r"], quant_bits=16, want_info=False)
        t = d.build_tree(8, 1.0, 0.0, 1.0, 0.1)
        state["r"] += 1
        return t

    for name, prof, export_each in (("a: events+export", True, True), ("b: export each", False, True),
                                    ("c: export after", False, False)):
        ctx.set_profiling(prof)
        for _ in range(3):
            t = rnd()
            if state["tree"] is not None:
                state["tree"].close()
            state["tree"] = t
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        trees = []
        e0.record(stream)
        for _ in range(steps):
            t = rnd()
            if export_each:
                t.export()
            trees.append(t)
            state["tree"] = t
        for t in trees if not export_each else []:
            t.export()
        e1.record(stream)
        torch.cuda.synchronize()
        for t in trees[:-1]:
            t.close()
        print(f"{name:20s} {e0.elapsed_time(e1) / steps:.4f} ms/round", flush=True)
    ctx.get_timings()


if __name__ == "__main__":
    main()
