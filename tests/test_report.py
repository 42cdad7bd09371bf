"""CSV v1 emitter of measured runs against the
reference's schema (proj/include/gpumux/csv.hpp:13-16, csv.cpp:10-41)."""
import json
import os
import re

import pytest

from refshim import ROOT

from paper_1901_00041_b200 import report


def test_header_is_the_reference_contract():
    ref = "/root/reference/proj/include/gpumux/csv.hpp"
    if os.path.exists(ref):
        text = open(ref).read()
        parts = re.findall(r'"([^"]*)"', text[text.index("kCsvHeader"):text.index(";", text.index("kCsvHeader"))])
        assert report.CSV_HEADER == "".join(parts)
    assert report.CSV_HEADER.count(",") == 16


def test_line_format_matches_csv_cpp():
    ok = report.csv_line("w", "space-time", 4, 8, 42, "ok", {"throughput_gflops": 349248.45937, "p99_ms": 0.7493,
                                                            "launches": 1})
    f = ok.split(",")
    assert len(f) == 17 and f[:7] == ["1", "w", "space-time", "4", "8", "42", "ok"]
    assert f[7] == "349248.459" and f[11] == "0.7493" and f[14] == "1"
    bad = report.csv_line("w", "time-mux", 4, 8, 42, "oom")
    assert bad.endswith(",oom" + "," * 10) and len(bad.split(",")) == 17


def test_bench_line_rows():
    line = json.loads(open(os.path.join(ROOT, "profiles", "r01c_bench_line.json")).read())
    rows = report.bench_rows(line)
    assert len(rows) == 3 + 3 * len(line["table1"]["rows"])
    assert {r.split(",")[2] for r in rows} == {"space-time", "time-mux", "space-implicit"}


def test_bench_rows_cover_every_table1_preset():
    row = {"R": 2, "packed_tflops": 1.0, "time_only_tflops": 0.5, "space_only_tflops": 0.8}
    line = {"modes": {}, "table1": {"rows": [row], "other_presets": {"rnn-matvec": {"rows": [row, row]},
                                                                     "square-256": {"rows": [row]}}}}
    rows = report.bench_rows(line, peak_tflops=1000.0)
    assert len(rows) == 3 * 4
    assert {r.split(",")[1] for r in rows} == {"resnet18-conv2_2", "rnn-matvec", "square-256"}



def test_table1_report_matches_bench_geomeans():
    """report --kind table1 (gpumux.cpp:195-235) over a committed CSV of a
    real run: the speedup_table geomeans equal the bench line's."""
    csv = os.path.join(ROOT, "profiles", "r01i_runs.csv")
    line = json.loads(open(os.path.join(ROOT, "profiles", "r01i_bench_line.json")).read())
    rows = report.read_csv(csv)
    t = report.speedup_table(rows, "resnet18-conv2_2")
    assert t["geomean_speedup"] == pytest.approx(line["table1"]["geomean_over_space_only"], rel=1e-6)
    assert [x["R"] for x in t["rows"]] == [r["R"] for r in line["table1"]["rows"]]
    for name, suite in line["table1"]["other_presets"].items():
        assert report.speedup_table(rows, name)["geomean_speedup"] == pytest.approx(
            suite["geomean_over_space_only"], rel=1e-6)
    text = report.table1_report(rows)
    lines = text.splitlines()
    assert lines[0].split() == ["row", "resnet18-conv2_2", "rnn-matvec", "square-256"]
    assert lines[1].startswith("R = 10") and lines[3].startswith("geomean") and lines[4].startswith("next best")


def test_speedup_table_semantics():
    def row(w, p, r, g):
        return {"workload": w, "policy": p, "replicas": str(r), "status": "ok", "throughput_gflops": str(g)}
    rows = [row("w", "space-time", 2, 10), row("w", "time-mux", 2, 5), row("w", "space-implicit", 2, 4),
            row("w", "space-time", 4, 12), row("w", "time-mux", 4, 3), row("w", "space-implicit", 4, 6)]
    t = report.speedup_table(rows, "w")
    assert [x["speedup"] for x in t["rows"]] == [2.0, 2.0]
    assert t["next_best"] == "time-mux"  # one win each: the earlier PolicyKind
    with pytest.raises(ValueError, match="missing cell"):
        report.speedup_table(rows[:5], "w")


def test_trace_ndjson_lines():
    d = {"start_ns": 10, "end_ns": 700010, "device_ms": 0.66, "flops": 2.6e11, "queries": 32, "tenants": 4,
         "launches": 1, "tiles": 14224}
    (ln,) = report.trace_ndjson_lines([d])
    obj = json.loads(ln)
    assert obj["policy"] == "space-time" and obj["members"] == 32 and obj["start_ns"] == 10
    assert set(obj) >= {"start_ns", "end_ns", "policy", "launches", "flops", "members"}
