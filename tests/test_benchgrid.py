"""Bench CSV compatibility: the latency grid is written with the
reference report tool's BENCH column set (reports/src/mpcreports/schemas.py:9, restated
here), readable by its validating reader semantics (header must match exactly)."""

import csv

import pytest

from paper_2605_29155_b200 import benchgrid

REPORT_BENCH_SCHEMA = ["mode", "B", "T", "K", "forward_ms", "backward_ms", "dispatches"]


def _read(path):
    with open(path, newline="") as f:
        r = csv.DictReader(f)
        assert list(r.fieldnames) == REPORT_BENCH_SCHEMA
        return list(r)


def test_header_matches_report_schema(tmp_path):
    assert benchgrid.LATENCY_CSV_HEADER == REPORT_BENCH_SCHEMA
    p = tmp_path / "bench.csv"
    benchgrid.write_latency_csv([{"mode": "b200", "B": 1, "T": 10, "K": 10, "forward_ms": 0.2,
                                  "backward_ms": 0.1, "dispatches": 2}], p)
    rows = _read(p)
    assert rows[0]["mode"] == "b200" and rows[0]["dispatches"] == "2"


@pytest.mark.gpu
def test_latency_grid_on_gpu(tmp_path):
    rows = benchgrid.latency_probe([1, 64], [5], reps=2, K=3)
    p = tmp_path / "bench.csv"
    benchgrid.write_latency_csv(rows, p)
    got = _read(p)
    assert [int(r["B"]) for r in got] == [1, 64]
    assert all(int(r["dispatches"]) == 2 and float(r["forward_ms"]) > 0 for r in got)
