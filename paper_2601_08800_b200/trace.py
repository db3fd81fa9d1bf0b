"""Logical communication trace in the reference's format.

The reference emits one ``TraceEvent`` per (rank, op, round) while it walks
its routing table (sim:70-136 types/CSV, sim:353-393 dispatch,
sim:443-504 combine, sim:546-561 expert compute, sim:609-666 baseline).
Here the same event stream is generated from the routing *counts* the GPU
router produced -- ``S[j][d]`` (slots of group j hosted on d) and the
per-host ``[(expert, rows)]`` -- so a B200 run yields a byte-identical
``trace.csv`` (golden: tests/golden/trace_2x2.csv).  Byte counts keep the
reference's float64 accounting (8 B per element) and its per-shard RS/AG
convention; the physical NVLink bytes of the B200 kernels
are reported separately by the bench.
"""
from __future__ import annotations

import csv
import io
from dataclasses import dataclass
from pathlib import Path

FLOAT_BYTES = 8
TRACE_CSV_HEADER = ["event_id", "rank", "op", "peer_or_group", "bytes",
                    "round", "dep_ids", "scope", "group_size", "work"]


@dataclass(frozen=True)
class TraceEvent:
    event_id: int
    rank: int
    op: str
    peer_or_group: str
    bytes: int
    round: int
    dep_ids: tuple[int, ...]
    scope: str
    group_size: int = 1
    work: float = 0.0


class Trace:
    """Append-only event log with sequential ids (sim:84-96)."""

    def __init__(self) -> None:
        self.events: list[TraceEvent] = []

    def add(self, rank, op, peer_or_group, nbytes, round_, deps, scope,
            group_size=1, work=0.0) -> int:
        eid = len(self.events)
        self.events.append(TraceEvent(eid, rank, op, peer_or_group, int(nbytes),
                                      round_, tuple(deps), scope, group_size,
                                      work))
        return eid


def trace_to_csv(events) -> str:
    out = io.StringIO()
    w = csv.writer(out, lineterminator="\n")
    w.writerow(TRACE_CSV_HEADER)
    for ev in events:
        w.writerow([ev.event_id, ev.rank, ev.op, ev.peer_or_group, ev.bytes,
                    ev.round, ";".join(map(str, ev.dep_ids)), ev.scope,
                    ev.group_size, repr(ev.work)])
    return out.getvalue()


def trace_from_csv(text: str) -> list[TraceEvent]:
    rows = csv.reader(io.StringIO(text))
    header = next(rows, None)
    if header != TRACE_CSV_HEADER:
        raise ValueError(f"unexpected trace header: {header}")
    events = []
    for lineno, row in enumerate(rows, start=2):
        if not row:
            continue
        try:
            events.append(TraceEvent(
                int(row[0]), int(row[1]), row[2], row[3], int(row[4]),
                int(row[5]), tuple(int(d) for d in row[6].split(";") if d),
                row[7], int(row[8]), float(row[9])))
        except (IndexError, ValueError) as exc:
            raise ValueError(f"malformed trace row at line {lineno}: {row}") from exc
    return events


def save_trace(events, path) -> None:
    Path(path).write_text(trace_to_csv(events))


def _widths(h, m):
    return [h // m + (1 if t < h % m else 0) for t in range(m)]


def _shard(nbytes, m):
    return nbytes // m if m > 1 else 0


class TraceBuilder:
    """Emits the reference's event stream for one cluster and table."""

    def __init__(self, n, m, T, h, send, trace=None):
        self.n, self.m, self.W, self.T, self.h = n, m, n * m, T, h
        self.S = [[int(send[j][d]) for d in range(n)] for j in range(n)]
        self.trace = trace if trace is not None else Trace()
        self.width = _widths(h, m)

    # rows of host `host` whose tokens belong to group `owner`
    def rows(self, host, owner):
        return self.S[owner][host]

    def dispatch(self):
        """sim:353-393"""
        tr, n, m, W = self.trace, self.n, self.m, self.W
        route = [tr.add(r, "route", "local", 0, 0, (), "compute",
                        work=float(self.T)) for r in range(W)]
        sends, recvs = {}, {}
        for i in range(1, n):
            for r in range(W):
                g, t = divmod(r, m)
                nb = self.rows((g + i) % n, g) * self.width[t] * FLOAT_BYTES
                sends[r, i] = tr.add(r, "isend", f"rank:{(r + i * m) % W}", nb,
                                     i, (route[r],), "inter")
            for r in range(W):
                g, t = divmod(r, m)
                peer = (r - i * m) % W
                nb = self.rows(g, (g - i) % n) * self.width[t] * FLOAT_BYTES
                recvs[r, i] = tr.add(r, "irecv", f"rank:{peer}", nb, i,
                                     (sends[peer, i],), "inter")
        for i in range(1, n):
            for r in range(W):
                g = r // m
                nb = self.rows(g, (g - i) % n) * self.h * FLOAT_BYTES
                tr.add(r, "all_gather", f"tp:node{g}", _shard(nb, m), i,
                       tuple(recvs[g * m + q, i] for q in range(m)), "intra",
                       group_size=m)
        return tr

    def expert_deps(self):
        """all_gather + route ids per rank (sim:584-587)."""
        deps = {r: [] for r in range(self.W)}
        for ev in self.trace.events:
            if ev.op in ("all_gather", "route"):
                deps[ev.rank].append(ev.event_id)
        return {r: tuple(v) for r, v in deps.items()}

    def expert(self, expert_rows, deps, full_width=False):
        """sim:546-561 (fused, work rows*h/m) / sim:642-650 (baseline)."""
        ids = {}
        for d in range(self.n):
            for t in range(self.m):
                r = d * self.m + t
                ids[r] = tuple(
                    self.trace.add(r, "expert_compute", f"expert:{e}", 0, 0,
                                   deps.get(r, ()), "compute",
                                   work=float(rows * self.h if full_width
                                              else rows * self.h / self.m))
                    for e, rows in expert_rows[d])
        return ids

    def combine(self, compute_deps=None):
        """sim:443-504"""
        tr, n, m, W, h = self.trace, self.n, self.m, self.W, self.h
        compute_deps = compute_deps or {}
        reduces = {r: [] for r in range(W)}
        for i in range(1, n):
            rs, sends, recvs = {}, {}, {}
            for r in range(W):
                g = r // m
                nb = self.rows(g, (g + i) % n) * h * FLOAT_BYTES
                rs[r] = tr.add(r, "reduce_scatter", f"tp:node{g}", _shard(nb, m),
                               i, compute_deps.get(r, ()), "intra", group_size=m)
            for r in range(W):
                g, t = divmod(r, m)
                nb = self.rows(g, (g + i) % n) * self.width[t] * FLOAT_BYTES
                sends[r] = tr.add(r, "isend", f"rank:{(r + i * m) % W}", nb, i,
                                  (rs[r],), "inter")
            for r in range(W):
                g, t = divmod(r, m)
                peer = (r - i * m) % W
                nb = self.rows((g - i) % n, g) * self.width[t] * FLOAT_BYTES
                recvs[r] = tr.add(r, "irecv", f"rank:{peer}", nb, i,
                                  (sends[peer],), "inter")
            for r in range(W):
                g = r // m
                work = float(self.rows((g - i) % n, g) * h / m)
                reduces[r].append(tr.add(r, "local_reduce", "local", 0, i,
                                         (recvs[r],), "compute", work=work))
        last = {}
        for r in range(W):
            g = r // m
            nb = self.rows(g, g) * h * FLOAT_BYTES
            last[r] = tr.add(r, "reduce_scatter", f"tp:node{g}", _shard(nb, m), n,
                             compute_deps.get(r, ()), "intra", group_size=m)
        for r in range(W):
            g = r // m
            reduces[r].append(tr.add(r, "local_reduce", "local", 0, n, (last[r],),
                                     "compute", work=float(self.rows(g, g) * h / m)))
        for r in range(W):
            g = r // m
            tr.add(r, "all_gather", f"tp:node{g}",
                   _shard(self.T * h * FLOAT_BYTES, m), n, tuple(reduces[r]),
                   "intra", group_size=m)
        return tr

    def baseline(self, expert_rows):
        """_run_baseline's stream (sim:609-666): full-width A2A both ways,
        full compute per TP rank, then RS + AG over the TP group."""
        tr, n, m, W, h = self.trace, self.n, self.m, self.W, self.h
        route = {r: tr.add(r, "route", "local", 0, 0, (), "compute",
                           work=float(self.T)) for r in range(W)}

        def a2a(nbytes_of, deps_of):
            ids = {}
            for i in range(1, n):
                for r in range(W):
                    g = r // m
                    ids[r, i, "s"] = tr.add(r, "isend", f"rank:{(r + i * m) % W}",
                                            nbytes_of(g, (g + i) % n), i,
                                            deps_of(r), "inter")
                for r in range(W):
                    g = r // m
                    peer = (r - i * m) % W
                    ids[r, i, "r"] = tr.add(r, "irecv", f"rank:{peer}",
                                            nbytes_of((g - i) % n, g), i,
                                            (ids[peer, i, "s"],), "inter")
            return {r: tuple(v for key, v in ids.items()
                             if key[0] == r and key[2] == "r") for r in range(W)}

        disp = a2a(lambda src, dst: self.rows(dst, src) * h * FLOAT_BYTES,
                   lambda r: (route[r],))
        comp = self.expert(expert_rows, disp, full_width=True)
        back = a2a(lambda src, dst: self.rows(src, dst) * h * FLOAT_BYTES,
                   lambda r: comp[r])
        for r in range(W):
            g = r // m
            nb = _shard(self.T * h * FLOAT_BYTES, m)
            rs = tr.add(r, "reduce_scatter", f"tp:node{g}", nb, 0, back[r],
                        "intra", group_size=m)
            tr.add(r, "all_gather", f"tp:node{g}", nb, 0, (rs,), "intra",
                   group_size=m)
        return tr
