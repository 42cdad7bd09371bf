"""Summarise a round's ncu artefacts into profiles/ (run here, after gpurun).

  python tools/summarize_ncu.py --tag r01b
reads gpurun_out/{prof_round.ncu-rep, launches.csv, bench.log} and writes
profiles/<tag>_round_kernel_ncu.txt, <tag>_launch_list.txt, <tag>_bench_line.json
and profiles/superkernel_traffic.json (the bench's roofline 'traffic' source).
"""
import argparse
import collections
import csv
import io
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--cmd", default="python tools/ncu_target.py --round --rounds 2 (-k regex:superkernel -s 1 -c 1)")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", "gpurun_out/prof_round.ncu-rep", "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    m = {n: (uu, vv) for n, uu, vv in zip(h, u, v)}
    name = m.get("Kernel Name", ("", "?"))[1]
    with open(f"profiles/{a.tag}_round_kernel_ncu.txt", "w") as f:
        f.write(f"# ncu --set full --clock-control none --import-source on, kernel {name}\n")
        f.write(f"# round program: 4 tenants x ResNet-50@224 b8, one launch per round; command: {a.cmd}\n")
        for k in KEYS:
            if k in m:
                f.write(f"{k:90s} {m[k][0]:10s} {m[k][1]}\n")
    rd = float(m["dram__bytes_read.sum"][1]) * (1e6 if m["dram__bytes_read.sum"][0] == "Mbyte" else 1e9)
    wr = float(m["dram__bytes_write.sum"][1]) * (1e6 if m["dram__bytes_write.sum"][0] == "Mbyte" else 1e9)
    json.dump({"kernel": "gmb::dev::superkernel<256> round program", "dram__bytes_read.sum_MB": rd / 1e6,
               "dram__bytes_write.sum_MB": wr / 1e6, "dram_bytes_per_launch": rd + wr,
               "gpu__time_duration_us": float(m["gpu__time_duration.sum"][1]),
               "source": f"gpurun_out/prof_round.ncu-rep (ncu --set full, 1 launch), summarised in "
                         f"profiles/{a.tag}_round_kernel_ncu.txt"},
              open("profiles/superkernel_traffic.json", "w"), indent=1)
    # launch list
    lines = [ln for ln in open("gpurun_out/launches.csv") if ln.startswith('"')]
    rdr = csv.DictReader(io.StringIO("".join(lines)))
    tot = collections.defaultdict(lambda: [0, 0.0])
    ours = []
    for r in rdr:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", "")) * (1e3 if r["Metric Unit"] == "usecond" else 1)
        k = r["Kernel Name"]
        tot[k][0] += 1
        tot[k][1] += ns
        if "gmb::" in k:
            ours.append((r["ID"], k, ns))
    allns = sum(t[1] for t in tot.values())
    with open(f"profiles/{a.tag}_launch_list.txt", "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
        f.write("# command: python bench.py --steps 2 --warmup 1 --table1 '' --cpu-seconds 0.1 --serve-seconds 0 "
                "--extra '' (all modes + setup)\n# per-kernel totals over the whole command:\n")
        for k, (n, ns) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:12]:
            f.write(f"{n:6d} launches {ns / 1e3:11.1f} us {100 * ns / allns:5.1f}%  {k[:120]}\n")
        f.write("\n# our kernels, launch by launch (ID, kernel, ns):\n")
        for i, k, ns in ours:
            f.write(f"{i}\t{k[:60]}\t{ns:.0f}\n")
    line = [x for x in open("gpurun_out/bench.log") if x.startswith("{")][-1]
    open(f"profiles/{a.tag}_bench_line.json", "w").write(line)
    print("wrote profiles for", a.tag)


if __name__ == "__main__":
    main()
