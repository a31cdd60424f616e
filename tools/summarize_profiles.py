"""Derive the committed profile summaries from raw ncu outputs of tools/gpu_round.sh:
  profiles/<tag>_launches_summary.txt  (per-kernel shares of one round, from the launch list)
  profiles/<tag>_k_hist_ncu_full.txt   (per-level k_hist metrics from the --set full capture)
  profiles/k_hist_traffic.json         (dram read + write per k_hist launch -> bench.py `traffic`)
usage: python tools/summarize_profiles.py gpurun_out/launches.csv gpurun_out/prof_hist.ncu-rep r01"""
import contextlib
import csv
import io
import json
import subprocess
import sys

sys.path.insert(0, "tools")
import launch_summary  # noqa: E402

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def main(launches_csv, rep, tag):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        launch_summary.main(launches_csv, 3)
    with open(f"profiles/{tag}_launches_summary.txt", "w") as f:
        f.write(f"# {tag} launch list: ncu --metrics gpu__time_duration.sum --clock-control none over\n"
                "# bench.py --profile-only --steps 2 --warmup 1 (config 2: 1M x 500, depth 8, f=1): 3 rounds, per round;\n"
                "# cold-cache serialised per-launch times: compare SHARES with the bench's live phases\n")
        f.write(buf.getvalue())
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = [hdr.index(m) for m in METRICS]
    rd = wr = 0.0
    lines = [f"# {tag} ncu --set full --clock-control none, k_hist, the {len(data)} level launches of one config-2 round",
             "# columns: " + ", ".join(f"{m} [{units[i]}]" for m, i in zip(METRICS, idx))]
    for r in data:
        lines.append(" | ".join(r[i] for i in idx))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd += float(r[idx[1]].replace(",", "")) * scale[units[idx[1]]]
        wr += float(r[idx[2]].replace(",", "")) * scale[units[idx[2]]]
    with open(f"profiles/{tag}_k_hist_ncu_full.txt", "w") as f:
        f.write("\n".join(lines) + "\n")
    n = len(data)
    with open("profiles/k_hist_traffic.json", "w") as f:
        json.dump({"kernel": "k_hist", "source": f"profiles/{tag}_k_hist_ncu_full.txt (ncu --set full, {n} launches = "
                   "one config-2 round)", "dram_read_MB_total": rd / 1e6, "dram_write_MB_total": wr / 1e6,
                   "launches": n, "traffic_bytes_per_launch": (rd + wr) / max(1, n)}, f, indent=1)
    print(open(f"profiles/{tag}_launches_summary.txt").read())
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
