"""Measured traces in the reference's formats.

The reference models a layer as a trace of per-rank events (``TraceEvent``,
simcluster.py:70-136) list-scheduled onto three lanes per rank (intra link,
inter link, compute) by ``timeline.schedule`` (timeline.py:97-154), exported
as a Gantt CSV ``rank,lane,op,start_s,end_s,bytes`` (timeline.py:216-233).
This module produces the MEASURED counterpart from a B200 run:

* :func:`measure_phases` runs the fused forward phase by phase with a
  device clock stamp (``mx_stamp``: ``%globaltimer`` after every earlier
  launch) after each phase; t = 0 is the stamp right after an aligning
  device barrier, so ranks share an origin to within the barrier's skew;
* :func:`gantt_rows` / :func:`gantt_csv` -- one row per (rank, phase) on the
  reference's lanes (dispatch/combine ride NVLink between groups: "inter";
  device barriers: "intra"; kernels: "compute") with the phase's
  algorithmic bytes;
* :func:`stamp_trace` -- the reference trace of the same routing (built by
  :class:`TraceBuilder` from the GPU's counts, byte-identical to the
  reference's) with every event's measured ``start_s``/``end_s``: a fused
  kernel executes all rounds of its phase at once, so each event spans the
  phase that carries it (dispatch rounds -> dispatch kernel, expert_compute
  -> the grouped GEMMs, RS/pairwise/local_reduce/AG -> combine).

``tools/measured_trace.py`` writes both for a configuration;
``tools/model_vs_measured.py`` (build container only) schedules the same
trace with the reference's own ``timeline.schedule`` on the calibrated B200
links and compares modelled and measured makespans.
"""
from __future__ import annotations

import csv
import io

import numpy as np
import torch

from .trace import TRACE_CSV_HEADER, TraceBuilder

GANTT_CSV_HEADER = "rank,lane,op,start_s,end_s,bytes"
LANE = {"route": "compute", "layout": "compute", "dispatch": "inter", "expand": "compute",
        "gemm1_swiglu": "compute", "gemm2": "compute", "pair_reduce": "compute",
        "combine": "inter", "barrier_counts": "intra", "barrier_dispatch": "intra",
        "barrier_partials": "intra", "barrier_out": "intra"}


def measure_phases(layer, x, logits, iters=10, stream=None):
    """Per-phase (start_s, end_s) of this rank, median over ``iters`` runs.

    Returns ``{phase: (start_s, end_s)}`` relative to the aligning stamp."""
    s = stream or torch.cuda.current_stream()
    p, r = layer.plan, layer.rank
    names = layer.phase_names()
    if len(names) + 1 > 64:
        raise ValueError("too many phases for the stamp buffer")
    runs = []
    view = p.stamps_view(r)
    for _ in range(iters):
        p.barrier(stream=s)
        slot = [0]

        def mark(name):
            p.stamp(slot[0], rank=r, stream=s)
            slot[0] += 1

        layer.run_phases(x, logits, mark, s)
        s.synchronize()
        runs.append(view[:len(names)].cpu().numpy().astype(np.int64))
    st = np.median(np.stack([v - v[0] for v in runs]), axis=0) / 1e9
    return {names[i]: (float(st[i - 1]), float(st[i])) for i in range(1, len(names))}


def gather_phases(phases):
    """All ranks' phase dicts (list indexed by rank); identity without a
    process group."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [phases]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, phases)
    return out


def gantt_rows(per_rank, phase_bytes=None):
    """Rows ``(rank, lane, op, start_s, end_s, bytes)`` sorted like the
    reference's ``_gantt_rows`` (timeline.py:206-210)."""
    rows = []
    for rank, phases in enumerate(per_rank):
        pb = (phase_bytes[rank] if isinstance(phase_bytes, list) else phase_bytes) or {}
        for op, (a, b) in phases.items():
            rows.append((rank, LANE.get(op, "compute"), op, a, b, int(pb.get(op, 0))))
    rows.sort(key=lambda row: (row[3], row[0], row[1], row[2]))
    return rows


def gantt_csv(rows) -> str:
    lines = [GANTT_CSV_HEADER]
    for rank, lane, op, a, b, nbytes in rows:
        lines.append(f"{rank},{lane},{op},{a!r},{b!r},{nbytes}")
    return "\n".join(lines) + "\n"


def _span(phases, name, wire):
    tok = wire == "token"
    if name == "expert":
        a = phases["expand" if tok else "gemm1_swiglu"][0]
        return a, phases["gemm2"][1]
    if name == "combine":
        a = phases["pair_reduce" if tok else "combine"][0]
        return a, phases["combine"][1]
    if name == "dispatch":
        return phases["dispatch"][0], phases["dispatch"][1]
    return phases["route"][0], phases["layout"][1]


def stamp_trace(events, stages, per_rank, wire="slot") -> str:
    """Reference trace CSV plus measured ``start_s,end_s,phase`` columns;
    ``stages`` maps event id -> route / dispatch / expert / combine (from
    :func:`layer_trace`)."""
    which = stages
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(TRACE_CSV_HEADER + ["start_s", "end_s", "phase"])
    for ev in events:
        a, b = _span(per_rank[ev.rank], which[ev.event_id], wire)
        w.writerow([ev.event_id, ev.rank, ev.op, ev.peer_or_group, ev.bytes, ev.round,
                    ";".join(map(str, ev.dep_ids)), ev.scope, ev.group_size, repr(ev.work),
                    repr(a), repr(b), which[ev.event_id]])
    return buf.getvalue()


def layer_trace(layer):
    """The reference's fused-layer trace for the layer's last routing, built
    from the GPU counts (same bytes as run_moe_block's trace), and the
    builder stage of every event (route / dispatch / expert / combine)."""
    cnt, send = layer.routing_counts()
    E, n = layer.E, layer.n
    host_of = (np.arange(E) * n) // E
    tot = cnt.astype(np.int64).sum(axis=0)
    expert_rows = [[(int(e), int(tot[e])) for e in range(E) if host_of[e] == d and tot[e] > 0]
                   for d in range(n)]
    tb = TraceBuilder(n, layer.m, layer.T, layer.h, send.astype(np.int64))
    tb.dispatch()
    n_disp = len(tb.trace.events)
    comp = tb.expert(expert_rows, tb.expert_deps())
    n_exp = len(tb.trace.events)
    tb.combine(comp)
    stages = {}
    for ev in tb.trace.events:
        i = ev.event_id
        stages[i] = ("route" if ev.op == "route" else "dispatch" if i < n_disp
                     else "expert" if i < n_exp else "combine")
    return tb.trace.events, stages
