"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel launch count,
total and per-launch microseconds (cold-cache, serialised: compare shares, not absolutes).
One-time setup kernels (quantisation: sketch, CUB sorts, cuts, binning; torch fills) are listed
separately, not per round.  usage: python tools/launch_summary.py launches.csv [rounds]"""
import collections
import csv
import sys


SETUP = ("cub::", "k_bin_rows", "k_sketch_append", "k_transpose_keys", "k_extract_cuts", "at::")


def main(path, rounds=3):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("oocgb::", "")
        v = float(d["Metric Value"])
        unit = d.get("Metric Unit", "nsecond")
        us = v / 1000.0 if unit.startswith("n") else (v if unit.startswith("u") else v * 1000.0)
        per.setdefault(name, []).append(us)
    setup = {k: v for k, v in per.items() if any(k.startswith(p) or p in k for p in SETUP)}
    per = collections.OrderedDict((k, v) for k, v in per.items() if k not in setup)
    total = sum(sum(v) for v in per.values()) / rounds
    print(f"{'kernel':28s} {'launches/round':>14s} {'us/round':>9s} {'share':>6s}")
    for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        t = sum(v) / rounds
        print(f"{name:28s} {len(v) / rounds:14.1f} {t:9.1f} {100 * t / total:5.1f}%")
    print(f"{'total':28s} {'':14s} {total:9.1f}")
    print(f"one-time setup (quantisation, not per round): {sum(sum(v) for v in setup.values()):.1f} us in "
          f"{sum(len(v) for v in setup.values())} launches")
    for name, v in per.items():
        k = len(v) // rounds
        if k > 1:
            print(f"{name} per launch (last round): {[round(x, 1) for x in v[-k:]]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3)
