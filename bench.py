#!/usr/bin/env python
"""MoE-layer tokens/s of the B200 TP-EP layer (BASELINE.json metric).

Workload: BASELINE.json configs[1], the Qwen3-30B-A3B-shaped MoE layer
(h=2048, moe_intermediate=768, 128 experts, top-8, bf16 SwiGLU experts,
fp32 gate logits) on a prefill batch of 8192 tokens; one step = one full
layer forward (gate top-k -> dispatch -> grouped GEMM -> combine) over the
8192 tokens.  Total work is fixed as N grows ("scaling": "strong"); the
cluster is TP2 x EP(N/2) (config B's TP2xEP4 at N=8), pure 1x1 at N=1.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Timing: CUDA events on the launching stream around every step, L2 flushed
(256 MiB write) between steps outside the events, max over ranks.  Per-
phase events inside the same timed steps give the roofline of the dominant
kernel.  ``e2e`` repeats the step through the public API with pinned host
inputs and the output copied back.  The CPU baseline is the oracle port
(oracle/, numpy + BLAS, all host threads) on a bounded token sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

H, INTER, E, K_TOP, T_GLOBAL = 2048, 768, 128, 8, 8192
NVLINK_PEER_GBS = 770.0      # measured peer copy, B200_PROFILING.md
# what SM-issued 16 B peer stores of 4 KB rows reach on 4 B200s (every GPU
# pushing at once; tools/nvlink_bench.py -> profiles/r01_nvlink_ceiling_n4.jsonl)
NVLINK_SM_STORE_GBS = 680.0
HBM_REF_GBS = 6539.5         # MEASURED_PEAKS.json copy bandwidth (bound selection only)
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


OUT = sys.stdout  # the JSON line's stream (see json_stdout)


def json_stdout():
    """Keep the process's stdout to the one JSON line: file descriptor 1 is
    routed to stderr (NCCL / c10d / library banners included) and the
    returned file writes to the original stdout."""
    sys.stdout.flush()
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    return out


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return FALLBACK, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def wait_first(self, timeout=5.0):
        t0 = time.monotonic()
        while self.proc and not self.lines and time.monotonic() - t0 < timeout:
            time.sleep(0.02)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0=None, t1=None, margin=0.25):
        """Median SM clock and active throttle reasons of the samples taken
        inside [t0 - margin, t1 + margin] (the timed region)."""
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = [ln for ts, ln in self.lines
                 if t0 is None or (t0 - margin <= ts <= t1 + margin)]
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "window": "timed region +-0.25 s"}


# ------------------------------------------------------------------ CPU
REF_DIR = ROOT / "oracle" / "_ref"   # the unmodified reference (oracle/install_ref.sh)


def _import_reference():
    """moeplan from oracle/_ref (pip-installed from /root/reference by
    oracle/install_ref.sh; git-ignored, travels to the GPU box), or None."""
    if not (REF_DIR / "moeplan" / "simcluster.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import moeplan.simcluster as sim
    if not str(Path(sim.__file__).resolve()).startswith(str(REF_DIR.resolve())):
        return None
    return sim


def reference_layer_step(sim, n, m, x, router, experts):
    """One bounded sample of the layer through the reference's own stock
    path: ``run_moe_block(mode="fused")`` (sim:565-595), f64, affine experts
    (``ExpertSpec.default``), the whole n x m cluster simulated on the host."""
    y, _trace = sim.run_moe_block(sim.build_cluster(n, m), x, router, experts, mode="fused")
    return y


def reference_inputs(sim, n, m, sample, seed=1):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((sample, H))
    router = sim.RouterSpec.random(sample, E, K_TOP, seed=seed + 1)
    return x, router, sim.ExpertSpec.default(E)


def time_reference(n, m, sample, reps=None, target_s=10.0, warmup=1):
    """Mean seconds per ``run_moe_block`` over a ``sample``-token batch of
    the workload's shape (h, E, k, cluster n x m), on this host."""
    sim = _import_reference()
    if sim is None:
        return None
    x, router, ex = reference_inputs(sim, n, m, sample)
    for _ in range(max(1, warmup)):
        reference_layer_step(sim, n, m, x, router, ex)
    if reps is None:
        t0 = time.perf_counter()
        reference_layer_step(sim, n, m, x, router, ex)
        reps = max(3, int(np.ceil(target_s / max(time.perf_counter() - t0, 1e-3))))
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        reference_layer_step(sim, n, m, x, router, ex)
        times.append(time.perf_counter() - t0)
    return float(np.mean(times)), reps


def swiglu_port_experts(seed=0):
    """SwiGLU expert weights for the CPU port, N(0, 1/fan_in) rounded to
    bf16 (numpy only: the reference arm never imports the product)."""
    from oracle import mixserve_oracle as orc
    rng = np.random.default_rng(seed)
    mk = lambda *s, fan: orc.bf16_round((rng.standard_normal(s, dtype=np.float32)
                                         / np.float32(fan ** 0.5)))
    return orc.SwiGLUOracle(mk(E, INTER, H, fan=H), mk(E, INTER, H, fan=H),
                            mk(E, H, INTER, fan=INTER))


def cpu_oracle_step(x, logits, experts_np):
    """One bounded sample of the SwiGLU layer on the host (the oracle port):
    oracle gate + batched SwiGLU experts (numpy/BLAS), expert-ascending
    accumulation."""
    from oracle import mixserve_oracle as orc
    ids, w = orc.router_topk(logits, K_TOP, renormalize=True)
    return orc.moe_layer_swiglu(x, ids, w, experts_np)


def time_swiglu_port(sample_tokens=512, target_s=10.0, seed=0):
    from oracle import mixserve_oracle as orc
    onp = swiglu_port_experts(seed)
    rng = np.random.default_rng(seed)
    x = orc.bf16_round(rng.standard_normal((sample_tokens, H)).astype(np.float32))
    logits = rng.standard_normal((sample_tokens, E)).astype(np.float32)
    cpu_oracle_step(x[:64], logits[:64], onp)   # warm BLAS
    t0 = time.perf_counter()
    cpu_oracle_step(x, logits, onp)
    one = time.perf_counter() - t0
    reps = max(3, int(np.ceil(target_s / max(one, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(reps):
        cpu_oracle_step(x, logits, onp)
    return (time.perf_counter() - t0) / reps, reps


def cpu_threads():
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def cpu_baseline(n, m, ref_sample=1024, port_sample=512, target_s=10.0):
    """The reference's own CPU path (kind "reference": oracle/_ref's
    run_moe_block, one core -- pure Python + elementwise numpy) on a bounded
    sample of the workload, plus the SwiGLU port (numpy/BLAS, all host
    threads) as a second, labelled line."""
    port_dt, port_reps = time_swiglu_port(port_sample, target_s)
    port = {"value": port_sample / port_dt, "unit": "tokens/s", "cores": cpu_threads(),
            "kind": "port",
            "sample": f"{port_sample} tokens of the {T_GLOBAL}-token batch: oracle gate + "
                      f"SwiGLU experts (f32 numpy/BLAS), mean of {port_reps} repetitions"}
    ref = time_reference(n, m, ref_sample, target_s=target_s)
    if ref is None:
        port["note"] = "oracle/_ref missing (run oracle/install_ref.sh): the port is the baseline"
        return port
    dt, reps = ref
    return {"value": ref_sample / dt, "unit": "tokens/s", "cores": 1, "kind": "reference",
            "sample": f"{ref_sample} tokens through the unmodified reference "
                      f"run_moe_block(mode='fused') on a simulated {n}x{m} cluster (f64, "
                      f"affine ExpertSpec.default({E}), RouterSpec.random top-{K_TOP}, "
                      f"h={H}), mean of {reps} repetitions",
            "seconds_per_sample": dt, "swiglu_port": port}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref: the unmodified moeplan, pip-installed from /root/reference
    by oracle/install_ref.sh) through its public API, run_moe_block
    (mode="fused"), f64 with its stock affine experts, on a bounded token
    sample of this arm's workload (same h, E, k and n x m cluster layout).
    Rank 0 only; the reference is single-threaded Python + numpy."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n, m = reference_layout(args)
    sim = _import_reference()
    sample = args.ref_sample
    if sim is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref missing: run oracle/install_ref.sh "
                                         "(pip install --target oracle/_ref /root/reference)"}),
              file=OUT, flush=True)
        return
    x, router, ex = reference_inputs(sim, n, m, sample)
    for _ in range(max(1, min(args.warmup, 2))):
        reference_layer_step(sim, n, m, x, router, ex)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        reference_layer_step(sim, n, m, x, router, ex)
        times.append(time.perf_counter() - t0)
    dt = float(np.mean(times))
    value = sample / dt
    line = {
        "impl": "reference", "metric": "MoE-layer tokens/s", "value": value,
        "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{WORKLOAD} (bounded sample of {sample} tokens per step)",
                   "hidden": H, "moe_intermediate": INTER, "experts": E, "top_k": K_TOP,
                   "groups_n": n, "tp_m": m, "parallelism": f"TP{m}xEP{n}",
                   "experts_kind": "reference ExpertSpec.default (affine, f64)"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": 1, "kind": "reference",
                         "sample": f"{sample} tokens per step through the unmodified "
                                   f"reference run_moe_block(mode='fused'), f64"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), file=OUT, flush=True)


# ------------------------------------------------------------------ ours
def phase_model(S, cnt, n, m, group, tp, T, U=None, wire="slot"):
    """Algorithmic bytes / flops per launch of every phase on this rank
    (SURVEY.md §8(d)); S[j][d] = slots of group j hosted on group d,
    U[j][d] = tokens of group j hitting host d (wire TOKEN)."""
    It = INTER // m
    S_d = int(S[:, group].sum())             # rows this rank's GEMMs process
    remote_in = int(S[:, group].sum() - S[group, group])   # rows received over NVLink
    local_rows = int(S[group, group])
    hb = H * 2
    slots = T * K_TOP
    model = {}
    model["route"] = {"bound": "hbm", "bytes": T * E * 4 + slots * 16 + E * 4}
    if n * m == 1:
        # x read once (slot rows re-read from L2), expert-major rows written
        model["dispatch"] = {"bound": "hbm", "bytes": T * hb + S_d * hb}
        model["combine"] = {"bound": "hbm", "bytes": slots * hb + T * hb}
    else:
        if remote_in > 0:
            model["dispatch"] = {"bound": "nvlink", "bytes": remote_in * hb,
                                 "local_hbm_bytes": 2 * local_rows * hb}
        else:   # one group (pure TP): every row is a local gather
            model["dispatch"] = {"bound": "hbm", "bytes": T * hb + S_d * hb}
        # pulls: every slot's column shard from the m TP ranks of its host,
        # minus the one local read; plus the (m-1)/m of y pushed by TP peers
        own_host_slots = int(S[group, group])
        remote_pull = (slots * m - own_host_slots) * (H // m) * 2
        model["combine"] = {"bound": "nvlink",
                            "bytes": remote_pull + T * H * (m - 1) // m * 2}
    if wire == "token" and U is not None:
        U = np.asarray(U, dtype=np.int64)
        remote_pairs = int(U[:, group].sum() - U[group, group])
        if remote_pairs > 0:
            # pair rows arriving over NVLink (own-group rows are written
            # straight into RECV by the same kernel, local HBM)
            model["dispatch"] = {"bound": "nvlink", "bytes": remote_pairs * hb,
                                 "local_hbm_bytes": T * hb + local_rows * hb}
        else:   # one group: the dispatch is a local expert-major copy
            model["dispatch"] = {"bound": "hbm", "bytes": T * hb + local_rows * hb}
        # expand moves only the remote pairs: XBUF row read once, written to
        # each of the pair's slot rows
        model["expand"] = {"bound": "hbm", "bytes": remote_pairs * hb + remote_in * hb}
        pairs_host = int(U[:, group].sum())
        # the pre-reduction pushes each pair's row (as m column shards) into
        # the owners' ZIN: all of it crosses NVLink for other groups' tokens,
        # (m-1)/m of it for the own group's; it reads S_d partial rows locally
        own = int(U[group, group])
        push = (pairs_host - own) * hb + own * hb * (m - 1) // m
        if push > 0:
            model["pair_reduce"] = {"bound": "nvlink", "bytes": push,
                                    "local_hbm_bytes": S_d * hb}
        else:
            model["pair_reduce"] = {"bound": "hbm", "bytes": S_d * hb + pairs_host * hb}
        # the owner sums its local ZIN planes and pushes its y shard to the
        # group's other TP ranks (final all-gather)
        zin_read = int(U[group].sum()) * hb
        y_push = T * H * (m - 1) // m * 2
        if y_push > 0:
            model["combine"] = {"bound": "nvlink", "bytes": y_push, "local_hbm_bytes": zin_read}
        else:
            model["combine"] = {"bound": "hbm", "bytes": zin_read + T * hb}
    # a phase that moves both NVLink and local HBM bytes is judged against
    # whichever of the two takes longer at its peak
    for spec in model.values():
        loc = spec.pop("local_hbm_bytes", None)
        if loc is not None and spec["bound"] == "nvlink" and \
                loc / HBM_REF_GBS > spec["bytes"] / NVLINK_PEER_GBS:
            spec["nvlink_bytes"] = spec["bytes"]
            spec["bound"], spec["bytes"] = "hbm", loc
        elif loc is not None:
            spec["local_hbm_bytes"] = loc
    model["gemm1_swiglu"] = {"bound": "tensor", "flops": 2 * S_d * H * 2 * It}
    model["gemm2"] = {"bound": "tensor", "flops": 2 * S_d * It * H}
    return model


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2601_08800_b200 import SwiGLUExperts
    from paper_2601_08800_b200.layer import MoELayer, layout_for

    n, m = layout_for(world, args.tp)
    group, tp = divmod(rank, m)
    T = T_GLOBAL // n
    ex = SwiGLUExperts.random(E, H, INTER, seed=0)
    w13, w2 = ex.rank_shard(n, m, rank)
    del ex
    torch.cuda.empty_cache()
    # TOKEN wire whenever there is a peer: dedup dispatch + pair pre-reduction
    # (for n == 1 the TP reduction then moves T rows instead of T*k slots)
    wire = args.wire if args.wire != "auto" else ("token" if world > 1 else "slot")
    layer = MoELayer(n, m, T, H, E, K_TOP, INTER, w13=w13, w2=w2, rank=rank, wire=wire)
    g = torch.Generator(device="cuda").manual_seed(1000 + group)
    x = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=g)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        layer.forward(x, logits)
    sync_all()
    S = layer.routing_counts()[1].astype(np.int64)
    cnt = layer.routing_counts()[0]
    U = layer.pair_counts()

    # ---- timed region: K replays of the captured layer forward (one CUDA
    #      graph: every launch and device barrier), CUDA events around each
    #      replay on the launching stream, L2 flushed between steps
    runner = layer.capture(x, logits)
    step_ev = []
    with ClockSampler(local) as clk:
        clk.wait_first()
        sync_all()
        t_region0 = time.monotonic()
        for _ in range(args.steps):
            flush.fill_(1)
            layer.plan.barrier()   # align ranks before the start event (launch skew)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            runner()
            b.record(stream)
            step_ev.append((a, b))
        torch.cuda.synchronize()
        t_region1 = time.monotonic()
    total_ms = float(sum(a.elapsed_time(b) for a, b in step_ev))
    t = torch.tensor([total_ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = T_GLOBAL / (ms_per_step / 1e3)

    # ---- per-kernel times: the same forward captured with an external
    #      event after every phase (each event node adds ~3 us, so this loop
    #      is reported apart from the headline), K replays, L2 flushed
    phased = layer.capture(x, logits, with_events=True)
    phase_times = {}
    for _ in range(args.steps):
        flush.fill_(1)
        layer.plan.barrier()
        phased()
        torch.cuda.synchronize()
        for name, ms in phased.phase_ms():
            phase_times.setdefault(name, []).append(ms)

    # ---- e2e through the public API, streamed the way a server feeds
    #      batches: every step copies its tokens/logits in from pinned host
    #      memory and its output back out; the H2D of step i+1 and the D2H of
    #      step i run on their own streams under the forward of step i
    #      (double-buffered inputs, two captured graphs).  One timed region
    #      over the K steps, max over ranks.
    x_h = x.cpu().pin_memory()
    l_h = logits.cpu().pin_memory()
    y_hs = [torch.empty(T, H, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    copy_out = tp == 0
    xs, ls = [x, torch.empty_like(x)], [logits, torch.empty_like(logits)]
    runners = [runner, layer.capture(xs[1], ls[1])]
    y_stage = [torch.empty(T, H, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    ev_d2h = [torch.cuda.Event() for _ in range(2)]

    def h2d_step(i):
        b = i % 2
        if i >= 2:
            h2d_s.wait_event(ev_free[b])          # step i-2 has read this buffer
        with torch.cuda.stream(h2d_s):
            xs[b].copy_(x_h, non_blocking=True)   # public API: host tokens in
            ls[b].copy_(l_h, non_blocking=True)
        ev_in[b].record(h2d_s)

    sync_all()
    flush.fill_(1)
    layer.plan.barrier()
    e_a = torch.cuda.Event(enable_timing=True)
    e_b = torch.cuda.Event(enable_timing=True)
    e_a.record(stream)
    h2d_s.wait_event(e_a)
    d2h_s.wait_event(e_a)
    h2d_step(0)
    for i in range(args.steps):
        b = i % 2
        if i + 1 < args.steps:
            h2d_step(i + 1)
        stream.wait_event(ev_in[b])
        y = runners[b]()                           # the captured forward
        ev_free[b].record(stream)
        if copy_out:
            if i >= 2:
                stream.wait_event(ev_d2h[b])       # y_stage[b] drained to host
            y_stage[b].copy_(y, non_blocking=True)
            ev_out[b].record(stream)
            d2h_s.wait_event(ev_out[b])
            with torch.cuda.stream(d2h_s):
                y_hs[b].copy_(y_stage[b], non_blocking=True)   # host result out
            ev_d2h[b].record(d2h_s)
    stream.wait_stream(h2d_s)
    stream.wait_stream(d2h_s)
    e_b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e_a.elapsed_time(e_b)], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_step = float(t.item()) / args.steps
    x_h_bytes = x_h.numel() * 2
    del runners
    h2d = (x_h_bytes + l_h.numel() * 4) * world
    d2h = T * H * 2 * n

    # ---- the reference's per-slot wire on the same config (N > 1)
    slot_wire = None
    if world > 1 and wire == "token" and not args.no_nccl:
        alt = MoELayer(n, m, T, H, E, K_TOP, INTER, w13=w13, w2=w2, rank=rank, wire="slot")
        alt_run = alt.capture(x, logits)
        ev = []
        for _ in range(args.steps):
            flush.fill_(1)
            alt.plan.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            alt_run()
            b.record(stream)
            ev.append((a, b))
        torch.cuda.synchronize()
        st = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / args.steps], device="cuda")
        dist.all_reduce(st, op=dist.ReduceOp.MAX)
        slot_wire = {"ms_per_step": float(st.item()),
                     "tokens_per_s": T_GLOBAL / (float(st.item()) / 1e3),
                     "wire": "slot (the reference's one-row-per-slot A2A layout)"}
        del alt_run
        alt.close()

    # ---- the other layout of the same GPUs: EP only (TP1 x EP N) -- the
    #      layout the strategy question is about (config E / SURVEY §8 a15)
    ep_only = None
    if world > 1 and m > 1 and not args.no_nccl:
        xe_g = torch.Generator(device="cuda").manual_seed(1000 + rank)
        Te = T_GLOBAL // world
        xe = torch.randn(Te, H, device="cuda", generator=xe_g).to(torch.bfloat16)
        le = torch.randn(Te, E, device="cuda", generator=xe_g)
        ex2 = SwiGLUExperts.random(E, H, INTER, seed=0)
        w13e, w2e = ex2.rank_shard(world, 1, rank)
        del ex2
        alt = MoELayer(world, 1, Te, H, E, K_TOP, INTER, w13=w13e, w2=w2e, rank=rank, wire="token")
        alt_run = alt.capture(xe, le)
        ev = []
        for _ in range(args.steps):
            flush.fill_(1)
            alt.plan.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            alt_run()
            b.record(stream)
            ev.append((a, b))
        torch.cuda.synchronize()
        st = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / args.steps], device="cuda")
        dist.all_reduce(st, op=dist.ReduceOp.MAX)
        ep_only = {"parallelism": f"TP1xEP{world}", "wire": "token",
                   "ms_per_step": float(st.item()),
                   "tokens_per_s": T_GLOBAL / (float(st.item()) / 1e3)}
        del alt_run
        alt.close()
        del w13e, w2e, xe, le
        torch.cuda.empty_cache()

    # ---- NCCL AR + A2A baseline on the same config (N > 1)
    nccl = None
    if world > 1 and not args.no_nccl:
        for _ in range(2):
            layer.forward_baseline(x, logits)
        sync_all()
        bl = []
        for _ in range(max(3, args.steps // 2)):
            flush.fill_(1)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            layer.forward_baseline(x, logits)
            b.record(stream)
            bl.append((a, b))
        torch.cuda.synchronize()
        blt = torch.tensor([float(np.mean([a.elapsed_time(b) for a, b in bl]))], device="cuda")
        dist.all_reduce(blt, op=dist.ReduceOp.MAX)
        nccl = {"ms_per_step": float(blt.item()),
                "tokens_per_s": T_GLOBAL / (float(blt.item()) / 1e3),
                "layout": "NCCL all_to_all_single x2 (full width, every TP rank) + TP all_reduce",
                "fused_speedup": float(blt.item()) / ms_per_step}

    # ---- roofline of the dominant kernel (this rank; rank 0 reports)
    pk, pk_kind = peaks()
    model = phase_model(S, cnt, n, m, group, tp, T, U, wire)
    avg = {k: float(np.mean(v)) for k, v in phase_times.items()}
    rooflines = {}
    for ph, spec in model.items():
        if ph not in avg or avg[ph] <= 0 or spec.get("bytes", 1) == 0:
            continue
        sec = avg[ph] / 1e3
        if spec["bound"] == "tensor":
            ach = spec["flops"] / sec / 1e12
            peak, unit = pk["bf16_tflops_sustained"], "TFLOP/s"
            peak_src = f"{pk_kind} bf16 sustained"
        elif spec["bound"] == "hbm":
            ach = spec["bytes"] / sec / 1e9
            peak, unit = pk["hbm_gbs"], "GB/s"
            peak_src = f"{pk_kind} HBM copy"
        else:
            ach = spec["bytes"] / sec / 1e9
            peak, unit = NVLINK_PEER_GBS, "GB/s"
            peak_src = "NVLink peer copy 770 GB/s/direction (B200_PROFILING.md)"
        rooflines[ph] = {"bound": spec["bound"], "achieved": ach, "peak": peak, "unit": unit,
                         "frac": ach / peak, "us": avg[ph] * 1e3, "peak_source": peak_src}
        if spec["bound"] == "nvlink":
            rooflines[ph]["frac_sm_store_ceiling"] = ach / NVLINK_SM_STORE_GBS
            rooflines[ph]["sm_store_ceiling_source"] = (
                f"{NVLINK_SM_STORE_GBS:.0f} GB/s, profiles/r01_nvlink_ceiling_n4.jsonl")
    kernels = {k: v for k, v in rooflines.items()}
    dom = max(kernels, key=lambda k: kernels[k]["us"]) if kernels else None
    traffic = None
    tp_file = ROOT / "profiles" / "traffic.json"
    if dom and tp_file.exists():
        traffic = json.loads(tp_file.read_text()).get(f"n{world}", {}).get(dom)
    roof = dict(kernels[dom]) if dom else None
    if roof is not None:
        roof["kernel"] = dom
        roof["traffic"] = traffic

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(sample_tokens=args.cpu_sample)

    # gate, route, scan, layout, dispatch, gemm1, gemm2, combine (+3 barriers,
    # +1 TP-group barrier when m > 1; +expand, +pair_reduce for wire TOKEN)
    # -- profiles/r01_n1_launches.csv
    launches_per_step = (8 + ((4 if m > 1 else 3) if world > 1 else 0)
                         + (2 if wire == "token" else 0))
    if rank == 0:
        line = {
            "metric": "MoE-layer tokens/s", "value": value, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "Qwen3-30B-A3B-shaped MoE layer (BASELINE configs[1]), "
                                   "8192-token prefill, bf16 SwiGLU experts, fp32 gate logits",
                       "hidden": H, "moe_intermediate": INTER, "experts": E, "top_k": K_TOP,
                       "global_tokens": T_GLOBAL, "groups_n": n, "tp_m": m,
                       "parallelism": f"TP{m}xEP{n}", "l2": "flushed (256 MiB write) between steps",
                       "wire": wire,
                       "weights": "random init, seed 0"},
            "clocks": clk.summary(t_region0, t_region1),
            "e2e": {"value": T_GLOBAL / (e2e_step / 1e3), "unit": "tokens/s",
                    "ms_per_step": e2e_step, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "note": "every step: pinned host x/logits copied in (H2D stream), the "
                            "captured MoELayer forward, y copied back to pinned host (D2H "
                            "stream); copies of neighbouring steps overlap the forward "
                            "(double-buffered); one timed region over all steps"},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roof,
            "rooflines": rooflines,
            "phases_us": {k: v * 1e3 for k, v in avg.items()},
            "phases_note": "per-phase CUDA events inside a second captured graph, same K, "
                           "L2 flushed; each event node adds ~3 us",
            "cpu_baseline": cpu,
        }
        if nccl is not None:
            line["nccl_baseline"] = nccl
        if slot_wire is not None:
            line["wire_slot"] = slot_wire
        if ep_only is not None:
            line["layout_ep_only"] = ep_only
        print(json.dumps(line), file=OUT, flush=True)
    layer.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tp", type=int, default=None)
    ap.add_argument("--tokens", type=int, default=None,
                    help="override the global token count (default 8192, BASELINE configs[1])")
    ap.add_argument("--wire", default="auto", choices=["auto", "slot", "token"],
                    help="auto: token (dedup dispatch, pre-reduced combine) when n > 1")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=512)
    ap.add_argument("--ref-sample", type=int, default=512)
    args = ap.parse_args()
    if args.tokens:
        global T_GLOBAL
        T_GLOBAL = args.tokens
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    global OUT
    OUT = json_stdout()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    OUT.flush()


if __name__ == "__main__":
    main()
