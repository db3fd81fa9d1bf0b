"""Measured-trace export: host-side formatting.

The GPU side (device clock stamps) is exercised by tests/test_gpu_parity.py;
here the trace reconstruction and the CSV formats are checked against the
reference's golden trace and Gantt layout."""
import csv
import io
from types import SimpleNamespace

import numpy as np

from conftest import GOLDEN
from paper_2601_08800_b200.measured import (GANTT_CSV_HEADER, gantt_csv, gantt_rows,
                                            layer_trace, stamp_trace)
from paper_2601_08800_b200.trace import TRACE_CSV_HEADER, trace_to_csv


def _fake_layer_2x2():
    # reference golden 2x2: token t -> expert t%2 -> host t%2 (T/test_golden.py)
    cnt = np.array([[1, 1], [1, 1]])
    send = np.array([[1, 1], [1, 1]])
    return SimpleNamespace(E=2, n=2, m=2, T=2, h=8,
                           routing_counts=lambda: (cnt, send))


def _phases(off):
    names = ["route", "barrier_counts", "layout", "dispatch", "barrier_dispatch",
             "gemm1_swiglu", "gemm2", "barrier_partials", "combine", "barrier_out"]
    return {nm: (off + i * 1e-6, off + (i + 1) * 1e-6) for i, nm in enumerate(names)}


def test_layer_trace_is_the_reference_trace():
    events, stages = layer_trace(_fake_layer_2x2())
    assert trace_to_csv(events) == (GOLDEN / "trace_2x2.csv").read_text()
    assert [stages[e.event_id] for e in events if e.op == "route"] == ["route"] * 4
    assert all(stages[e.event_id] == "expert" for e in events if e.op == "expert_compute")
    assert all(stages[e.event_id] == "combine" for e in events
               if e.op in ("reduce_scatter", "local_reduce"))
    # dispatch sends precede every expert event, combine sends follow
    first_exp = min(e.event_id for e in events if e.op == "expert_compute")
    for e in events:
        if e.op == "isend":
            assert stages[e.event_id] == ("dispatch" if e.event_id < first_exp else "combine")


def test_stamp_trace_columns_and_spans():
    events, stages = layer_trace(_fake_layer_2x2())
    per_rank = [_phases(r * 1e-7) for r in range(4)]
    text = stamp_trace(events, stages, per_rank, wire="slot")
    rows = list(csv.reader(io.StringIO(text)))
    assert rows[0] == TRACE_CSV_HEADER + ["start_s", "end_s", "phase"]
    assert len(rows) == len(events) + 1
    for row in rows[1:]:
        rank, phase = int(row[1]), row[12]
        a, b = float(row[10]), float(row[11])
        ph = per_rank[rank]
        if phase == "dispatch":
            assert (a, b) == ph["dispatch"]
        elif phase == "expert":
            assert (a, b) == (ph["gemm1_swiglu"][0], ph["gemm2"][1])
        elif phase == "combine":
            assert (a, b) == ph["combine"]
        else:
            assert (a, b) == (ph["route"][0], ph["layout"][1])


def test_gantt_layout_matches_reference_format():
    per_rank = [_phases(0.0), _phases(5e-7)]
    rows = gantt_rows(per_rank, {"dispatch": 4096, "combine": 8192})
    text = gantt_csv(rows)
    lines = text.splitlines()
    assert lines[0] == GANTT_CSV_HEADER == "rank,lane,op,start_s,end_s,bytes"
    assert len(lines) == 1 + 2 * 10
    starts = [float(line.split(",")[3]) for line in lines[1:]]
    assert starts == sorted(starts)
    lanes = {line.split(",")[2]: line.split(",")[1] for line in lines[1:]}
    assert lanes["dispatch"] == "inter" and lanes["combine"] == "inter"
    assert lanes["gemm1_swiglu"] == "compute" and lanes["barrier_out"] == "intra"
    assert any(line.endswith(",4096") for line in lines if ",dispatch," in line)
