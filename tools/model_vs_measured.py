"""Modelled vs measured: schedule a measured trace with the reference's own
timeline model (build container only -- imports /root/reference).

    PYTHONPATH=/root/reference/pkg/src python tools/model_vs_measured.py \
        --trace profiles/r01_mt_n4_trace.csv --links profiles/b200_links_n4.csv \
        --n 2 --m 2 --out profiles/r01_model_vs_measured_n4.json

Reads the stamped trace written by tools/measured_trace.py (reference trace
columns + measured start_s/end_s/phase), re-creates the reference
``TraceEvent`` list, calibrates links with the reference's ``calibrate`` on
the NCCL rows measured on the box and the compute coefficient on the
measured expert spans (seconds per unit of the trace's ``work``), then runs
the reference's ``schedule`` on the fused trace and on ``make_sync_trace``
and reports both modelled makespans beside the measured one.  Analysis only:
nothing here runs on the GPU box or in the product path.
"""
import argparse
import csv
import json
from pathlib import Path

from moeplan.analyzer import calibrate, load_observations
from moeplan.config import CalibrationCoefficients, ClusterConfig
from moeplan.simcluster import TraceEvent
from moeplan.timeline import make_sync_trace, overlap_metrics, schedule


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trace", required=True)
    ap.add_argument("--links", required=True)
    ap.add_argument("--n", type=int, required=True)
    ap.add_argument("--m", type=int, required=True)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = list(csv.DictReader(open(a.trace)))
    events = [TraceEvent(int(r["event_id"]), int(r["rank"]), r["op"], r["peer_or_group"],
                         int(r["bytes"]), int(r["round"]),
                         tuple(int(d) for d in r["dep_ids"].split(";") if d), r["scope"],
                         int(r["group_size"]), float(r["work"])) for r in rows]
    measured = max(float(r["end_s"]) for r in rows)
    # compute coefficient: measured expert span / trace work, per rank (max)
    span, work = {}, {}
    for r in rows:
        if r["phase"] == "expert":
            k = int(r["rank"])
            span[k] = float(r["end_s"]) - float(r["start_s"])
            work[k] = work.get(k, 0.0) + float(r["work"])
    coeff = max(span[k] / work[k] for k in span if work[k] > 0)
    links = calibrate(load_observations(a.links), ar_literal=False)
    cal = CalibrationCoefficients(compute_coeff=coeff, intra_alpha=links.intra_alpha,
                                  intra_beta=links.intra_beta, inter_alpha=links.inter_alpha,
                                  inter_beta=links.inter_beta, ar_literal=False)
    cluster = ClusterConfig(a.n, a.m, links.intra_alpha, links.intra_beta, links.inter_alpha,
                            links.inter_beta, 180e9, 1.0 / coeff)
    fused = schedule(events, cluster, cal)
    sync = schedule(make_sync_trace(events), cluster, cal)
    ov = overlap_metrics(fused, sync)
    res = {"measured_makespan_s": measured, "modelled_fused_makespan_s": fused.makespan,
           "modelled_sync_makespan_s": sync.makespan, "overlap": ov.to_dict(),
           "model_over_measured": fused.makespan / measured,
           "calibration": {"compute_coeff_s_per_work": coeff,
                           "link_alpha_s": links.intra_alpha,
                           "link_beta_GBps": links.intra_beta / 1e9},
           "note": "measured = device-clock stamps of the fused B200 layer (one kernel per "
                   "phase, all rounds concurrent); modelled = reference timeline.schedule "
                   "of the same trace with NCCL-calibrated links"}
    print(json.dumps(res, indent=1))
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
