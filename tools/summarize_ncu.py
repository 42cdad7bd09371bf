"""Summarise ncu artefacts of a profiling pass into profiles/ (run here, after gpurun).

  python tools/summarize_ncu.py --tag r02a [--configs headline,bert4,mix4,table1]

reads gpurun_out/prof_<config>.ncu-rep (ncu --set full, one round-program
launch each, tools/profile_r02.sh), gpurun_out/launches.csv (the bench
command's launch list) and gpurun_out/bench.log, and writes
  profiles/<tag>_<config>_ncu.txt     key counters + algorithmic work per launch
  profiles/<tag>_launch_list.txt      per-kernel totals and our launches
  profiles/<tag>_bench_line.json      the bench line
  profiles/superkernel_traffic.json   the headline kernel's DRAM bytes (bench 'traffic')
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]

DESC = {
    "headline": "4 tenants x ResNet-50@224 b8 (BASELINE configs[1], bench headline)",
    "bert4": "16 tenants x BERT-base 12-layer GEMM chains, seq 128, b4 (configs[3])",
    "mix4": "2 x {ResNet-50, VGG-16, MobileNet-v2}@224 b4 (configs[2] round)",
    "table1": "120 tenants x conv2_2 (256,128,1152) b1 (Table 1, R=120)",
}


def algorithmic(config):
    """(FLOPs, compulsory bf16 bytes) of one round launch."""
    from paper_1901_00041_b200 import workload as W
    if config == "headline":
        models, batch = [W.resnet50(224)] * 4, [8] * 4
    elif config == "bert4":
        models, batch = [W.bert_base_gemms(128, layers=12)] * 16, [4] * 16
    elif config == "mix4":
        models, batch = [W.resnet50(224), W.vgg16(224), W.mobilenet_v2(224)] * 2, [4] * 6
    else:
        models, batch = [W.table1_layers("resnet18-conv2_2")] * 120, [1] * 120
    f = sum(L.flops(b) for m, b in zip(models, batch) for L in m)
    by = sum(L.compulsory_bytes(b) for m, b in zip(models, batch) for L in m)
    return f, by


def to_bytes(unit, value):
    return float(value) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]


def summarize(tag, config, peaks):
    rep = f"gpurun_out/prof_{config}.ncu-rep"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    m = {n: (uu, vv) for n, uu, vv in zip(h, u, v)}
    name = m.get("Kernel Name", ("", "?"))[1]
    us = float(m["gpu__time_duration.sum"][1]) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                                                   "msecond": 1e3}[m["gpu__time_duration.sum"][0]]
    rd = to_bytes(*m["dram__bytes_read.sum"])
    wr = to_bytes(*m["dram__bytes_write.sum"])
    flops, algo = algorithmic(config)
    with open(f"profiles/{tag}_{config}_ncu.txt", "w") as f:
        f.write(f"# ncu --set full --clock-control none --import-source on, kernel {name}\n")
        f.write(f"# {DESC[config]}; one round-program launch; command: python tools/ncu_target.py "
                f"--config {config} --round --rounds 2 (-k regex:superkernel -s 1 -c 1)\n")
        for k in KEYS:
            hit = [n for n in m if n == k or n.endswith("." + k)]
            for n in hit:
                f.write(f"{n:90s} {m[n][0]:10s} {m[n][1]}\n")
        f.write("\n# derived (this launch, cold-cache serialised ncu replay)\n")
        f.write(f"algorithmic FLOPs                 {flops / 1e9:12.2f} GFLOP\n")
        f.write(f"algorithmic compulsory bytes      {algo / 1e6:12.1f} MB (bf16 in + weights + out per op)\n")
        f.write(f"DRAM bytes (read + write)         {(rd + wr) / 1e6:12.1f} MB = {(rd + wr) / algo:.2f} x algorithmic\n")
        f.write(f"achieved tensor rate              {flops / us / 1e6:12.1f} TFLOP/s = "
                f"{flops / us / 1e6 / peaks['bf16_tflops']:.3f} of burst {peaks['bf16_tflops']}\n")
        f.write(f"achieved algorithmic bytes rate   {algo / us / 1e3:12.1f} GB/s = "
                f"{algo / us / 1e3 / peaks['hbm_gbs']:.3f} of HBM {peaks['hbm_gbs']}\n")
        f.write(f"achieved DRAM rate                {(rd + wr) / us / 1e3:12.1f} GB/s\n")
    return {"us": us, "dram": rd + wr, "name": name}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--configs", default="headline,bert4,mix4,table1")
    a = ap.parse_args()
    peaks = json.load(open("MEASURED_PEAKS.json"))
    got = {}
    for c in a.configs.split(","):
        if os.path.exists(f"gpurun_out/prof_{c}.ncu-rep"):
            got[c] = summarize(a.tag, c, peaks)
    if "headline" in got:
        g = got["headline"]
        json.dump({"kernel": "gmb::dev::superkernel<256> round program", "dram_bytes_per_launch": g["dram"],
                   "gpu__time_duration_us": g["us"],
                   "source": f"gpurun_out/prof_headline.ncu-rep (ncu --set full, 1 launch), summarised in "
                             f"profiles/{a.tag}_headline_ncu.txt"},
                  open("profiles/superkernel_traffic.json", "w"), indent=1)
    if os.path.exists("gpurun_out/launches.csv"):
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
    if os.path.exists("gpurun_out/bench.log"):
        line = [x for x in open("gpurun_out/bench.log") if x.startswith("{")][-1]
        open(f"profiles/{a.tag}_bench_line.json", "w").write(line)
    print("wrote profiles for", a.tag, sorted(got))


if __name__ == "__main__":
    main()
