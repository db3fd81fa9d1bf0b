"""Summarise an ncu launch list and ``--set full`` captures for profiles/.

    python tools/ncu_summary.py --launches gpurun_out/X_launches.csv \
        --full gpurun_out/X_gemm.ncu-rep gpurun_out/X_misc.ncu-rep \
        --title "..." --out profiles/X_ncu_summary.txt [--traffic-key n1]

The launch list is the ``--metrics gpu__time_duration.sum --clock-control
none`` pass (cold-cache, serialised: compare SHARES, not absolutes); the
full captures give DRAM bytes (the bench's ``roofline.traffic``), tensor-pipe
activity, occupancy and clocks per kernel.  ``--traffic-key`` also writes the
per-launch DRAM bytes into profiles/traffic.json under that key.
"""
import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
]
# kernel name -> bench phase (traffic.json keys)
PHASE = {"k_grouped_gemm<256, 1": "gemm1_swiglu", "k_grouped_gemm<256, 0": "gemm2",
         "k_combine": "combine", "k_dispatch": "dispatch", "k_gate": "route_gate",
         "k_route<": "route", "k_layout": "layout", "k_expand": "expand",
         "k_pair_reduce": "pair_reduce"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name):
    name = name.replace("(anonymous namespace)::", "")
    return name.split("(")[0].replace("void ", "")[:60]


def launch_table(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        us = float(d["Metric Value"].replace(",", "")) / (1e3 if d["Metric Unit"] in ("ns", "nsecond") else 1)
        agg.setdefault(short(d["Kernel Name"]), []).append(us)
    mine = {k: v for k, v in agg.items() if k.startswith(("mx::", "gemm::"))}
    steps = max(len(v) for v in mine.values())
    per_step = {k: sum(v) / len(v) for k, v in mine.items() if len(v) == steps}
    total = sum(per_step.values())
    out = [f"{'kernel':60s} {'launches':>8s} {'avg us':>9s} {'share':>7s}"]
    for k, v in per_step.items():
        out.append(f"{k:60s} {len(mine[k]):8d} {v:9.1f} {100 * v / total:6.1f}%")
    out.append(f"{'sum of one step':60s} {'':8s} {total:9.1f}")
    other = [k for k, v in mine.items() if len(v) != steps]
    if other:
        out.append("setup-only kernels (not per step): " + ", ".join(other))
    return out, per_step


def full_table(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--metrics",
                          ",".join(FULL_METRICS)], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rec = {"kernel": short(d["Kernel Name"])}
        for m in FULL_METRICS:
            if m not in d:
                continue
            if m.startswith("dram__bytes"):
                rec[m] = float(d[m].replace(",", "")) * SCALE.get(u[m], 1)
            else:
                rec[m] = d[m] + (" " + u[m] if u[m] else "")
        out.append(rec)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", required=True)
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--title", default="")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic-key", default=None)
    a = ap.parse_args()
    lines = [f"# {a.title}",
             "# launch list: ncu --metrics gpu__time_duration.sum --clock-control none "
             "(cold-cache, serialised; compare shares)", ""]
    tab, _ = launch_table(a.launches)
    lines += tab
    traffic = {}
    for rep in a.full:
        lines += ["", f"# ncu --set full --clock-control none --import-source on: {Path(rep).name}"]
        for rec in full_table(rep):
            lines.append(json.dumps(rec, indent=1))
            tot = rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
            for key, ph in PHASE.items():
                if key in rec["kernel"] and ph not in traffic:
                    traffic[ph] = tot
    Path(a.out).write_text("\n".join(lines) + "\n")
    if a.traffic_key and traffic:
        tf = ROOT / "profiles" / "traffic.json"
        data = json.loads(tf.read_text()) if tf.exists() else {}
        data[a.traffic_key] = traffic
        data["source"] = ("ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per "
                          f"launch; {Path(a.out).name}")
        tf.write_text(json.dumps(data, indent=1) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()
