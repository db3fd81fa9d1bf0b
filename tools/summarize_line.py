"""One-line summary of a bench.py JSON line (for gpurun logs)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "no line:", e)
        continue
    nccl = d.get("nccl_baseline") or {}
    comm = d.get("comm_us") or {}
    out = {"file": path, "Mtok_s": round(d["value"] / 1e6, 3), "ms": round(d["ms_per_step"], 4),
           "layout": d["config"].get("parallelism"), "e2e_Mtok_s": round(d["e2e"]["value"] / 1e6, 3),
           "roof": {k: round(v, 3) if isinstance(v, float) else v
                    for k, v in (d.get("roofline") or {}).items() if k in ("kernel", "frac", "achieved")},
           "nccl_ms": nccl.get("ms_per_step"), "nccl_captured": nccl.get("captured"),
           "comm_us": {k: round(v, 1) for k, v in comm.items() if k in ("fused", "nccl")},
           "overlap_ms": (d.get("overlapped_schedule") or {}).get("ms_per_step"),
           "ep_only_ms": (d.get("layout_ep_only") or {}).get("ms_per_step"),
           "slot_ms": (d.get("wire_slot") or {}).get("ms_per_step"),
           "probe_gbs": (d.get("nvlink_probe") or {}).get("gbs_per_gpu"),
           "gemm_mhz": d.get("gemm_sm_mhz"), "clocks": d.get("clocks", {}).get("reasons"),
           "phases": {k: round(v, 1) for k, v in d.get("phases_us", {}).items()}}
    print(json.dumps(out))
