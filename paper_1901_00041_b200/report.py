"""CSV v1 rows of measured B200 runs in the reference's reporting schema
(SURVEY §8(f) rank 3), so a real-hardware Table 1 diffs directly against the
simulator's sweep output.

Schema and formatting follow ``proj/include/gpumux/csv.hpp:13-16`` (column
order is part of the contract) and ``proj/src/csv.cpp:10-41`` (locale-free
``%.9g``, latencies in ms, empty metric columns unless status is ``ok``).
Policy names are the reference's wire names (``policies.cpp:8-26``): the
packed round program is ``space-time``, serial per-tenant launches
``time-mux``, one stream per tenant ``space-implicit``.
"""
from __future__ import annotations

from typing import Dict, Iterable, List, Optional

CSV_SCHEMA_VERSION = 1
CSV_HEADER = ("schema_version,workload,policy,replicas,batch,seed,status,"
              "throughput_gflops,utilization,mean_ms,p50_ms,p99_ms,fairness_gap,"
              "slo_attainment,launches,peak_mem_bytes,cancelled")

MODE_POLICY = {"packed": "space-time", "time_only": "time-mux", "space_only": "space-implicit"}


def format_double(v: float) -> str:
    """csv.cpp:10-14 (``%.9g``)."""
    return "%.9g" % v


def csv_line(workload: str, policy: str, replicas: int, batch: int, seed: int, status: str = "ok",
             metrics: Optional[Dict[str, float]] = None) -> str:
    """csv.cpp:16-41.  ``metrics`` keys: throughput_gflops, utilization,
    mean_ms, p50_ms, p99_ms, fairness_gap, slo_attainment, launches,
    peak_mem_bytes, cancelled (latencies already in ms)."""
    out = [str(CSV_SCHEMA_VERSION), workload, policy, str(int(replicas)), str(int(batch)), str(int(seed)), status]
    if status == "ok":
        m = metrics or {}
        out += [format_double(m.get("throughput_gflops", 0.0)), format_double(m.get("utilization", 0.0)),
                format_double(m.get("mean_ms", 0.0)), format_double(m.get("p50_ms", 0.0)),
                format_double(m.get("p99_ms", 0.0)), format_double(m.get("fairness_gap", 0.0)),
                format_double(m.get("slo_attainment", 1.0)), str(int(m.get("launches", 0))),
                format_double(m.get("peak_mem_bytes", 0.0)), str(int(m.get("cancelled", 0)))]
    else:
        out += [""] * 10
    return ",".join(out)


def bench_rows(line: dict, peak_tflops: Optional[float] = None, seed: int = 42) -> List[str]:
    """CSV v1 rows of one bench.py JSON line: the headline modes and, when
    present, every Table-1 point (R tenants x conv2_2), one row per policy.
    ``utilization`` is achieved / dense bf16 peak (the reference's is
    achieved / modelled peak, metrics.cpp:61)."""
    peak = peak_tflops or line.get("roofline", {}).get("tensor_view", {}).get("peak_tflops") or 1.0
    rows = []
    cfg = line.get("config", {})
    tenants = int(cfg.get("tenants_per_gpu", 1)) * int(line.get("n_gpus", 1))
    batch = int(cfg.get("batch", 1))
    for mode, policy in MODE_POLICY.items():
        r = line.get("modes", {}).get(mode)
        if r is None:
            continue
        rows.append(csv_line("resnet50@224", policy, tenants, batch, seed, "ok", {
            "throughput_gflops": r["tflops"] * 1e3, "utilization": r["tflops"] / peak,
            "mean_ms": r["ms_per_step"], "p50_ms": r["ms_per_step"], "p99_ms": r["p99_ms"],
            "launches": r["launches_per_step"]}))
    t1 = line.get("table1", {})
    suites = [("resnet18-conv2_2", t1)] + list(t1.get("other_presets", {}).items())
    for name, suite in suites:
        for row in suite.get("rows", []):
            for mode, policy in MODE_POLICY.items():
                tf = row[mode + "_tflops"]
                rows.append(csv_line(name, policy, row["R"], 1, seed, "ok", {
                    "throughput_gflops": tf * 1e3, "utilization": tf / peak}))
    return rows


def write_csv(path: str, rows: Iterable[str]) -> None:
    """csv.hpp write_csv: header line then rows."""
    with open(path, "w") as f:
        f.write(CSV_HEADER + "\n")
        for r in rows:
            f.write(r + "\n")
