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


# ---------------------------------------------------------------- report --kind table1

# PolicyKind order (policies.hpp:16-22): ties in the next-best count go to the
# earlier kind, as std::map iteration does in speedup_table.
_COMPETITORS = ("time-mux", "space-implicit", "space-explicit")


def read_csv(path: str) -> List[Dict[str, str]]:
    """csv.cpp:75-87: header must match, blank lines skipped."""
    with open(path) as f:
        lines = f.read().splitlines()
    if not lines:
        raise ValueError(f"csv: empty file {path}")
    if lines[0] != CSV_HEADER:
        raise ValueError(f"csv: unexpected header in {path}")
    cols = CSV_HEADER.split(",")
    out = []
    for ln in lines[1:]:
        if ln:
            vals = ln.split(",")
            if len(vals) != len(cols):
                raise ValueError(f"csv: bad row in {path}: {ln}")
            out.append(dict(zip(cols, vals)))
    return out


def speedup_table(rows: Iterable[Dict[str, str]], workload: str,
                  r_range: Optional[Iterable[int]] = None) -> Dict[str, object]:
    """metrics.cpp:90-138 over the ok rows of one workload: per R, space-time
    throughput / the best competitor's, the geomean of those ratios, and the
    most frequent best competitor.  Competitors absent from every row are
    skipped (this path measures time-mux and space-implicit); a missing cell
    of a present policy raises like the reference."""
    from .scheduler import geomean
    cells = {(r["policy"], int(r["replicas"])): float(r["throughput_gflops"])
             for r in rows if r["workload"] == workload and r["status"] == "ok"}
    present = [p for p in _COMPETITORS if any(k[0] == p for k in cells)]
    if not present:
        raise ValueError(f"speedup_table: no competitor rows for workload={workload}")
    rs = sorted({k[1] for k in cells}) if r_range is None else list(r_range)
    out_rows, wins = [], {p: 0 for p in present}
    for r in rs:
        if ("space-time", r) not in cells:
            raise ValueError(f"speedup_table: missing cell workload={workload} R={r} policy=space-time")
        best, best_p = 0.0, present[0]
        for p in present:
            if (p, r) not in cells:
                raise ValueError(f"speedup_table: missing cell workload={workload} R={r} policy={p}")
            if cells[(p, r)] > best:
                best, best_p = cells[(p, r)], p
        out_rows.append({"R": r, "speedup": cells[("space-time", r)] / best, "next_best": best_p})
        wins[best_p] += 1
    top = max(wins.values())
    return {"workload": workload, "rows": out_rows, "geomean_speedup": geomean([x["speedup"] for x in out_rows]),
            "next_best": next(p for p in present if wins[p] == top)}


def table1_report(rows: List[Dict[str, str]], workloads: Optional[Iterable[str]] = None) -> str:
    """`gpumux report --kind table1` (gpumux.cpp:195-235): R = 10 / R = 20
    speedups, geomean and next best per workload, aligned like print_table
    (gpumux.cpp:153-171).  Default workloads: the Table-1 presets present."""
    names = sorted({r["workload"] for r in rows}) if workloads is None else list(workloads)
    if workloads is None:
        names = [w for w in names if w in ("resnet18-conv2_2", "rnn-matvec", "square-256")]
    tables = [speedup_table(rows, w) for w in names]
    table = [["row"] + names]
    present = {x["R"] for t in tables for x in t["rows"]}
    for spot in (10, 20):
        if spot not in present:
            continue
        row = ["R = %d" % spot]
        for t in tables:
            cell = "-"
            for x in t["rows"]:
                if x["R"] == spot:
                    cell = "%.2fx" % x["speedup"]
            row.append(cell)
        table.append(row)
    table.append(["geomean"] + ["%.2fx" % t["geomean_speedup"] for t in tables])
    table.append(["next best"] + [t["next_best"] for t in tables])
    widths = [max(len(r[i]) for r in table) for i in range(len(table[0]))]
    lines = []
    for r in table:
        lines.append("".join(c + (" " * (widths[i] - len(c) + 2) if i + 1 < len(r) else "") for i, c in enumerate(r)))
    return "\n".join(lines) + "\n"


def trace_ndjson_lines(dispatches: Iterable[Dict[str, float]]) -> List[str]:
    """The reference's NDJSON trace (gpumux.cpp:64-79: one JSON object per
    dispatch event, keys start_ns, end_ns, policy, launches, flops, members)
    for real-clock serving dispatches (ServeResult.dispatches).  ``members``
    is the number of queries served; device_ms, tenants and tiles are
    measured extras; the modelled occupancy / context_switches are not
    emitted."""
    import json
    out = []
    for d in dispatches:
        out.append(json.dumps({"start_ns": int(d["start_ns"]), "end_ns": int(d["end_ns"]), "policy": "space-time",
                               "launches": int(d["launches"]), "flops": float(d["flops"]),
                               "members": int(d["queries"]), "tenants": int(d["tenants"]),
                               "device_ms": float(d["device_ms"]), "tiles": int(d["tiles"])},
                              separators=(",", ":")))
    return out


def write_trace_ndjson(path: str, dispatches: Iterable[Dict[str, float]]) -> None:
    with open(path, "w") as f:
        for ln in trace_ndjson_lines(dispatches):
            f.write(ln + "\n")


if __name__ == "__main__":  # python -m paper_1901_00041_b200.report table1 <runs.csv>
    import sys
    if len(sys.argv) != 3 or sys.argv[1] != "table1":
        raise SystemExit("usage: python -m paper_1901_00041_b200.report table1 <runs.csv>")
    sys.stdout.write(table1_report(read_csv(sys.argv[2])))
