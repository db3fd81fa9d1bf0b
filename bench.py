#!/usr/bin/env python
"""MoE-layer tokens/s of the B200 TP-EP layer (BASELINE.json metric).

Workload (``--config``):
  B (default) BASELINE.json configs[1], the Qwen3-30B-A3B-shaped MoE layer
    (h=2048, moe_intermediate=768, 128 experts, top-8, bf16 SwiGLU experts,
    fp32 gate logits), TP2 x EP(N/2) -- config B's TP2xEP4 at N=8;
  C BASELINE.json configs[2], the DeepSeek-R1-shaped layer (h=7168,
    I=2048, 256 routed experts top-8 + a 2048-wide shared expert, fp8 e4m3
    experts, DeepSeek-V3 gate), TP(N/2) x EP2 -- TP4xEP2 at N=8.
One step = one full layer forward (gate top-k -> dispatch -> grouped GEMM
-> combine) over a prefill batch of 8192 tokens; total work is fixed as N
grows ("scaling": "strong"); pure 1x1 at N=1.  ``--tp auto`` takes the
fused-layer model's layout pick for the run's own routing.

    python bench.py [--gpus N --steps K --warmup W] [--config B|C] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Timing: CUDA events on the launching stream around every step, L2 flushed
(256 MiB write) between steps outside the events, max over ranks.  Per-
phase events inside a second captured graph give each kernel's roofline
(tensor phases against the burst bf16 peak -- they run inside a region of a
few ms -- with the sustained figure beside it; NVLink phases against the
same run's mx_nvlink_probe, 900 GB/s nominal beside it).  ``e2e`` streams
pinned host inputs through the public API with the output copied back.  At
N>1 the NCCL AR+A2A baseline is graph-captured the same way (static split
sizes of this routing) and ``comm_us`` compares the two communicators.
``cpu_baseline`` / ``--impl reference`` time the unmodified reference
(oracle/_ref, run_moe_block) on a bounded token sample.
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


def cpu_baseline(n, m, ref_sample=1024, port_sample=512, target_s=10.0, with_port=True):
    """The reference's own CPU path (kind "reference": oracle/_ref's
    run_moe_block, one core -- pure Python + elementwise numpy) on a bounded
    sample of the workload, plus the SwiGLU port (numpy/BLAS, all host
    threads) as a second, labelled line."""
    port = None
    if with_port:
        port_dt, port_reps = time_swiglu_port(port_sample, target_s)
        port = {"value": port_sample / port_dt, "unit": "tokens/s", "cores": cpu_threads(),
                "kind": "port",
                "sample": f"{port_sample} tokens of the {T_GLOBAL}-token batch: oracle gate + "
                          f"SwiGLU experts (f32 numpy/BLAS), mean of {port_reps} repetitions"}
    ref = time_reference(n, m, ref_sample, target_s=target_s)
    if ref is None and port is None:
        return None
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
def phase_model(S, n, m, group, T, U=None, wire="slot"):
    """Algorithmic bytes / flops per launch of every phase on this rank
    (SURVEY.md §8(d)); S[j][d] = slots of group j hosted on group d,
    U[j][d] = tokens of group j hitting host d (wire TOKEN).  Wire rows are
    WROW bytes (bf16: 2h; fp8: h e4m3 + 16 B scale tail), partials / ZIN /
    y rows 2h bytes (bf16)."""
    It = INTER // m
    Ist = SHARED // m
    S_d = int(S[:, group].sum())             # rows this rank's GEMMs process
    remote_in = int(S[:, group].sum() - S[group, group])   # rows received over NVLink
    local_rows = int(S[group, group])
    hb = WROW                                # a token row on the wire
    ob = H * 2                               # a partial / output row
    slots = T * K_TOP
    model = {}
    model["route"] = {"bound": "hbm", "bytes": T * E * 4 + slots * 16 + E * 4}
    if n * m == 1:
        # x read once (slot rows re-read from L2), expert-major rows written
        model["dispatch"] = {"bound": "hbm", "bytes": T * H * 2 + S_d * hb}
        model["combine"] = {"bound": "hbm", "bytes": slots * ob + T * ob}
    else:
        if remote_in > 0:
            model["dispatch"] = {"bound": "nvlink", "bytes": remote_in * hb,
                                 "local_hbm_bytes": 2 * local_rows * hb}
        else:   # one group (pure TP): every row is a local gather
            model["dispatch"] = {"bound": "hbm", "bytes": T * hb + S_d * hb}
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
        push = (pairs_host - own) * ob + own * ob * (m - 1) // m
        if push > 0:
            model["pair_reduce"] = {"bound": "nvlink", "bytes": push,
                                    "local_hbm_bytes": S_d * ob}
        else:
            model["pair_reduce"] = {"bound": "hbm", "bytes": S_d * ob + pairs_host * ob}
        # the owner sums its local ZIN planes and pushes its y shard to the
        # group's other TP ranks (final all-gather)
        zin_read = int(U[group].sum()) * ob
        y_push = T * H * (m - 1) // m * 2
        if y_push > 0:
            model["combine"] = {"bound": "nvlink", "bytes": y_push, "local_hbm_bytes": zin_read}
        else:
            model["combine"] = {"bound": "hbm", "bytes": zin_read + T * ob}
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
    # stage 1 = routed GEMM1 (+ the shared expert's GEMM1), stage 2 = GEMM2s
    model["gemm1_swiglu"] = {"bound": "tensor",
                             "flops": 2 * S_d * H * 2 * It + 2 * T * H * 2 * Ist}
    model["gemm2"] = {"bound": "tensor", "flops": 2 * S_d * It * H + 2 * T * Ist * H}
    return model


def measure_fp8_peak(dev):
    """Dense e4m3 matmul peak on this GPU, the MEASURED_PEAKS method for
    bf16 applied to fp8: torch._scaled_mm 8192^3 (cuBLASLt), best of 10,
    CUDA events (TFLOP/s)."""
    import torch
    n = 8192
    a = torch.randn(n, n, device=dev).to(torch.float8_e4m3fn)
    b = torch.randn(n, n, device=dev).to(torch.float8_e4m3fn).t()
    one = torch.ones((), device=dev)
    for _ in range(3):
        torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2.0 * n ** 3 / (best / 1e3) / 1e12


def nvlink_probe(layer, world, reps=5, mb_per_peer=32):
    """Same-run NVLink denominator: every rank copies ``mb_per_peer`` MB
    to every peer at once through the layer's own IPC heaps (16 B loads +
    16 B stores, mx_nvlink_probe); per-GPU egress GB/s, the slowest rank of
    the best of ``reps`` timed launches."""
    import torch
    import torch.distributed as dist
    from paper_2601_08800_b200 import _native as N
    from paper_2601_08800_b200.plan import stream_ptr
    p = layer.plan
    recv_room = p.buffer_bytes(layer.rank, N.MX_BUF_RECV) // world
    part_room = p.buffer_bytes(layer.rank, N.MX_BUF_PARTIAL)
    per_peer = min(mb_per_peer << 20, recv_room, part_room) & ~4095
    s = torch.cuda.current_stream()
    best = None
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        dist.barrier()
        p.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        N.check(N.load().mx_nvlink_probe(p._plan, per_peer, stream_ptr(s)), "probe")
        b.record(s)
        torch.cuda.synchronize()
        ms = torch.tensor([a.elapsed_time(b)], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        t = float(ms.item())
        best = t if best is None else min(best, t)
    gbs = per_peer * (world - 1) / (best / 1e3) / 1e9
    return {"gbs_per_gpu": gbs, "bytes_per_peer": per_peer, "ms": best,
            "how": "mx_nvlink_probe: every rank copies bytes_per_peer of local HBM to every "
                   "peer's heap at once (16 B loads, 16 B NVLink stores), best of "
                   f"{reps}, slowest rank"}


def gemm_clocks(layer):
    """Effective SM clock of the last GEMM launches: CTA 0 of each grouped
    GEMM records its SM cycles and %globaltimer ns (stamp slots 56-63).
    Sustained tensor-core load is power-capped; nvidia-smi's 50 ms samples
    cannot see a 0.2-0.4 ms kernel's clock, this can."""
    st = layer.plan.stamps_view(layer.rank)[56:64].cpu().numpy().astype(np.float64)
    out = {}
    for name, i in (("gemm1", 0), ("gemm2", 2), ("gemm1_fp8", 4), ("gemm2_fp8", 6)):
        cyc, ns = st[i], st[i + 1]
        if ns > 0 and cyc > 0:
            out[name] = round(cyc / ns * 1e3, 1)
    return out


def timed_replays(run, steps, flush, plan_barrier, stream, world):
    """Sum of per-step CUDA-event times of ``run()`` over ``steps`` replays
    (L2 flushed and ranks aligned before each), max over ranks (ms)."""
    import torch
    import torch.distributed as dist
    ev = []
    for _ in range(steps):
        flush.fill_(1)
        plan_barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run()
        b.record(stream)
        ev.append((a, b))
    torch.cuda.synchronize()
    t = torch.tensor([float(sum(a.elapsed_time(b) for a, b in ev))], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def phase_avgs(runner, steps, flush, plan_barrier):
    import torch
    times = {}
    for _ in range(steps):
        flush.fill_(1)
        plan_barrier()
        runner()
        torch.cuda.synchronize()
        for name, ms in runner.phase_ms():
            times.setdefault(name, []).append(ms)
    return {k: float(np.mean(v)) for k, v in times.items()}


FUSED_COMM = ("barrier_counts", "dispatch", "barrier_dispatch", "expand", "pair_reduce",
              "barrier_partials", "combine", "barrier_out")
NCCL_COMM = ("a2a_dispatch", "a2a_combine", "allreduce")


def build_layer(args, world, rank, n, m, wire, T):
    """The MoE layer of the selected config with random-init weights."""
    import torch
    from paper_2601_08800_b200 import FP8SwiGLUExperts, SwiGLUExperts
    from paper_2601_08800_b200.layer import MoELayer
    from paper_2601_08800_b200.plan import GateSpec
    if CONFIG == "C":
        ex = FP8SwiGLUExperts.random(E, H, INTER, shared_inter=SHARED, seed=0)
        ex.rank_shard(n, m, rank)                     # cached e4m3 shard of this rank
        ex.src = ex.shared = None                     # free the bf16 sources
        torch.cuda.empty_cache()
        bias = (0.05 * torch.randn(E, generator=torch.Generator().manual_seed(3))).float()
        gate = GateSpec.deepseek_v3(bias, groups=8, topk_groups=4, scaling=2.5)
        layer = MoELayer(n, m, T, H, E, K_TOP, INTER, experts=ex, rank=rank, wire=wire,
                         gate=gate)
        return layer, None
    ex = SwiGLUExperts.random(E, H, INTER, seed=0)
    w13, w2 = ex.rank_shard(n, m, rank)
    del ex
    torch.cuda.empty_cache()
    layer = MoELayer(n, m, T, H, E, K_TOP, INTER, w13=w13, w2=w2, rank=rank, wire=wire)
    return layer, (w13, w2)


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
    from paper_2601_08800_b200.layer import MoELayer, layout_for

    n, m = choose_layout(args, world)
    group, tp = divmod(rank, m)
    T = T_GLOBAL // n
    # TOKEN wire whenever there is a peer: dedup dispatch + pair pre-reduction
    wire = args.wire if args.wire != "auto" else ("token" if world > 1 else "slot")
    layer, weights = build_layer(args, world, rank, n, m, wire, T)
    g = torch.Generator(device="cuda").manual_seed(1000 + group)
    x = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=g)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    barrier = layer.plan.barrier

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        layer.forward(x, logits)                  # eager, error-checked
    sync_all()
    S = layer.routing_counts()[1].astype(np.int64)
    U = layer.pair_counts()

    # ---- timed region: K replays of the captured layer forward (one CUDA
    #      graph: every launch and device barrier), CUDA events around each
    #      replay on the launching stream, L2 flushed between steps
    runner = layer.capture(x, logits)
    with ClockSampler(local) as clk:
        clk.wait_first()
        sync_all()
        t_region0 = time.monotonic()
        total_ms = timed_replays(runner, args.steps, flush, barrier, stream, world)
        t_region1 = time.monotonic()
    runner.check()                                # errors flagged during the replays
    ms_per_step = total_ms / args.steps
    value = T_GLOBAL / (ms_per_step / 1e3)

    # ---- per-kernel times: the same forward captured with an external
    #      event after every phase (each event node adds ~3 us, so this loop
    #      is reported apart from the headline), K replays, L2 flushed
    phased = layer.capture(x, logits, with_events=True)
    avg = phase_avgs(phased, args.steps, flush, barrier)
    del phased
    gemm_clk = gemm_clocks(layer)

    # ---- the opt-in overlapped schedule (MX_OVERLAP=1: dispatch, expand and
    #      the other groups' pair pushes on a side stream under source-group
    #      halves of the grouped GEMMs), for its measured effect
    extras_pre = {}
    if world > 1 and wire == "token" and n > 1 and CONFIG == "B" and not args.no_nccl:
        os.environ["MX_OVERLAP"] = "1"
        ovl = layer.capture(x, logits)
        del os.environ["MX_OVERLAP"]
        ovl_ms = timed_replays(ovl, args.steps, flush, barrier, stream, world) / args.steps
        del ovl
        extras_pre["overlapped_schedule"] = {
            "ms_per_step": ovl_ms, "vs_headline": ovl_ms / ms_per_step,
            "note": "MX_OVERLAP=1 (opt-in): NVLink phases on a side stream under the "
                    "source-group halves of the grouped GEMMs; the headline runs every "
                    "phase in order (the split re-streams the expert weights)"}

    # ---- e2e through the public API (see run_e2e)
    e2e = run_e2e(layer, runner, x, logits, args, world, tp, n, T, stream, flush, sync_all)
    del runner

    extras = dict(extras_pre)
    nvl = None
    if world > 1:
        nvl = nvlink_probe(layer, world)
        extras["nvlink_probe"] = nvl
    nvl_peak = nvl["gbs_per_gpu"] if nvl else NVLINK_PEER_GBS

    # ---- NCCL AR + A2A baseline, graph-captured with this routing's split
    #      sizes fixed (no host sync inside), same timing loop; per-phase
    #      events give the communicator-only comparison
    if world > 1 and not args.no_nccl:
        bl = layer.capture_baseline(x, logits)
        bl_ms = timed_replays(bl, args.steps, flush, barrier, stream, world) / args.steps
        blp = layer.capture_baseline(x, logits, with_events=True)
        bl_avg = phase_avgs(blp, args.steps, flush, barrier)
        del blp
        nccl = {"ms_per_step": bl_ms, "tokens_per_s": T_GLOBAL / (bl_ms / 1e3),
                "layout": "NCCL all_to_all_single x2 (full width, every TP rank) + TP all_reduce",
                "captured": bl.graph is not None,
                "split_sizes": "this routing's send matrix, read once before capture (static)",
                "fused_speedup": bl_ms / ms_per_step, "phases_us": {k: v * 1e3 for k, v in bl_avg.items()}}
        if bl.error:
            nccl["capture_error"] = bl.error
        del bl
        extras["nccl_baseline"] = nccl
        fused_comm = sum(avg.get(k, 0.0) for k in FUSED_COMM) * 1e3
        nccl_comm = sum(bl_avg.get(k, 0.0) for k in NCCL_COMM) * 1e3
        extras["comm_us"] = {
            "fused": fused_comm, "nccl": nccl_comm,
            "fused_phases": [k for k in FUSED_COMM if k in avg],
            "nccl_phases": list(NCCL_COMM),
            "speedup": nccl_comm / fused_comm if fused_comm else None,
            "overlap_with_expert_gemms": "none: fused phases are serialized with the GEMMs",
            "note": "fused: dispatch/expand/pair pre-reduction (RS fused)/combine (AG fused) + "
                    "device barriers; NCCL: pack + all_to_all (dispatch), pack + all_to_all "
                    "(combine), unpack + TP all_reduce; per-phase events, L2 flushed"}

    # ---- the reference's per-slot wire, and EP-only, on the same GPUs
    if world > 1 and wire == "token" and not args.no_nccl and CONFIG == "B":
        alt = MoELayer(n, m, T, H, E, K_TOP, INTER, w13=weights[0], w2=weights[1], rank=rank,
                       wire="slot")
        ms = timed_replays(alt.capture(x, logits), args.steps, flush, alt.plan.barrier,
                           stream, world) / args.steps
        extras["wire_slot"] = {"ms_per_step": ms, "tokens_per_s": T_GLOBAL / (ms / 1e3),
                               "wire": "slot (the reference's one-row-per-slot A2A layout)"}
        alt.close()
    if world > 1 and m > 1 and not args.no_nccl and CONFIG == "B":
        from paper_2601_08800_b200 import SwiGLUExperts
        xe_g = torch.Generator(device="cuda").manual_seed(1000 + rank)
        Te = T_GLOBAL // world
        xe = torch.randn(Te, H, device="cuda", generator=xe_g).to(torch.bfloat16)
        le = torch.randn(Te, E, device="cuda", generator=xe_g)
        ex2 = SwiGLUExperts.random(E, H, INTER, seed=0)
        w13e, w2e = ex2.rank_shard(world, 1, rank)
        del ex2
        alt = MoELayer(world, 1, Te, H, E, K_TOP, INTER, w13=w13e, w2=w2e, rank=rank,
                       wire="token")
        ms = timed_replays(alt.capture(xe, le), args.steps, flush, alt.plan.barrier,
                           stream, world) / args.steps
        extras["layout_ep_only"] = {"parallelism": f"TP1xEP{world}", "wire": "token",
                                    "ms_per_step": ms, "tokens_per_s": T_GLOBAL / (ms / 1e3)}
        alt.close()
        del w13e, w2e, xe, le
        torch.cuda.empty_cache()

    # ---- roofline of every phase (this rank; rank 0 reports) and of the
    #      dominant kernel
    pk, pk_kind = peaks()
    if CONFIG == "C":
        tensor_peak = measure_fp8_peak("cuda")
        tensor_peak_src = ("measured in-run: torch._scaled_mm e4m3 8192^3, best of 10 "
                           "(cuBLASLt, the MEASURED_PEAKS bf16 method)")
        tensor_sus, tensor_sus_src = None, None
    else:
        tensor_peak = pk["bf16_tflops"]
        tensor_peak_src = (f"{pk_kind} bf16 burst (best-of-10 8192^3 matmul): the kernels "
                           f"are timed inside a {total_ms:.0f} ms region")
        tensor_sus = pk.get("bf16_tflops_sustained")
        tensor_sus_src = f"{pk_kind} bf16 sustained (4 s back-to-back)"
    model = phase_model(S, n, m, group, T, U, wire)
    rooflines = {}
    for ph, spec in model.items():
        if ph not in avg or avg[ph] <= 0 or spec.get("bytes", 1) == 0:
            continue
        sec = avg[ph] / 1e3
        r = {"bound": spec["bound"], "us": avg[ph] * 1e3}
        if spec["bound"] == "tensor":
            r.update(achieved=spec["flops"] / sec / 1e12, peak=tensor_peak, unit="TFLOP/s",
                     peak_source=tensor_peak_src)
            if tensor_sus:
                r.update(peak_sustained=tensor_sus, frac_sustained=r["achieved"] / tensor_sus)
        elif spec["bound"] == "hbm":
            r.update(achieved=spec["bytes"] / sec / 1e9, peak=pk["hbm_gbs"], unit="GB/s",
                     peak_source=f"{pk_kind} HBM copy")
        else:
            r.update(achieved=spec["bytes"] / sec / 1e9, peak=nvl_peak, unit="GB/s",
                     peak_source=("same-run mx_nvlink_probe (SM-issued peer copies, all "
                                  "peers at once)") if nvl else "NVLink peer copy 770 GB/s",
                     nominal=900.0, frac_nominal=spec["bytes"] / sec / 1e9 / 900.0)
        r["frac"] = r["achieved"] / r["peak"]
        rooflines[ph] = r
    # the tensor phases' peak at the clock they actually ran at (gemm_sm_mhz,
    # power capped): context for the burst fraction, not a replacement
    for ph, key in (("gemm1_swiglu", "gemm1"), ("gemm2", "gemm2")):
        if CONFIG == "C":
            key += "_fp8"
        r = rooflines.get(ph)
        mhz = gemm_clk.get(key)
        if r and mhz:
            r["peak_at_gemm_clock"] = r["peak"] * mhz / 1965.0
            r["frac_at_gemm_clock"] = r["achieved"] / r["peak_at_gemm_clock"]
            r["gemm_sm_mhz"] = mhz
    dom = max(rooflines, key=lambda k: rooflines[k]["us"]) if rooflines else None
    roof = dict(rooflines[dom]) if dom else None
    if roof is not None:
        roof["kernel"] = dom
        traffic = None
        tp_file = ROOT / "profiles" / "traffic.json"
        if tp_file.exists():
            traffic = json.loads(tp_file.read_text()).get(f"{CONFIG}{world}", {}).get(dom)
        roof["traffic"] = traffic
        roof["traffic_source"] = ("ncu --set full capture of this kernel at this config "
                                  "(profiles/traffic.json), not measured in this run"
                                  if traffic is not None else None)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(n, m, ref_sample=args.ref_sample if CONFIG == "B" else 256,
                           port_sample=args.cpu_sample, with_port=CONFIG == "B")

    if rank == 0:
        line = {
            "metric": "MoE-layer tokens/s", "value": value, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp8" if CONFIG == "C" else "bf16",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "config": CONFIG,
                       "hidden": H, "moe_intermediate": INTER, "experts": E, "top_k": K_TOP,
                       "shared_intermediate": SHARED, "global_tokens": T_GLOBAL,
                       "groups_n": n, "tp_m": m, "parallelism": f"TP{m}xEP{n}",
                       "layout_choice": LAYOUT_NOTE,
                       "l2": "flushed (256 MiB write) between steps", "wire": wire,
                       "weights": "random init, seed 0"},
            "clocks": clk.summary(t_region0, t_region1),
            "e2e": e2e,
            "gpu_launches": launches_per_step(world, m, wire) * args.steps,
            "roofline": roof,
            "rooflines": rooflines,
            "phases_us": {k: v * 1e3 for k, v in avg.items()},
            "gemm_sm_mhz": gemm_clk,
            "gemm_sm_mhz_note": "SM clock inside the grouped GEMMs (cycles / globaltimer of "
                                "CTA 0, last replay): the tensor phases run power-capped "
                                "below the sampled clock",
            "phases_note": "per-phase CUDA events inside a second captured graph, same K, "
                           "L2 flushed; each event node adds ~3 us",
            "cpu_baseline": cpu,
        }
        line.update(extras)
        print(json.dumps(line), file=OUT, flush=True)
    layer.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def launches_per_step(world, m, wire):
    """Kernels of one captured forward (profiles/r01_n1_launches.csv):
    gate, route, scan, layout, dispatch, gemm1, gemm2, combine; + barriers
    (3, +1 TP-group barrier when m > 1) with peers; + expand, pair_reduce on
    the token wire; config C adds the token quantisation, the activation
    re-quantisation and the shared expert's two GEMMs + quantisation."""
    k = 8 + ((4 if m > 1 else 3) if world > 1 else 0) + (2 if wire == "token" else 0)
    if CONFIG == "C":
        k += 5
    return k


def run_e2e(layer, runner, x, logits, args, world, tp, n, T, stream, flush, sync_all):
    """e2e through the public API, streamed the way a server feeds batches:
    every step copies its tokens/logits in from pinned host memory and its
    output back out; the H2D of step i+1 and the D2H of step i run on their
    own streams under the forward of step i (double-buffered inputs, two
    captured graphs).  One timed region over the K steps, max over ranks."""
    import torch
    import torch.distributed as dist
    x_h = x.cpu().pin_memory()
    l_h = logits.cpu().pin_memory()
    y_hs = [torch.empty(T, H, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    copy_out = tp == 0
    xs, ls = [x, x.clone()], [logits, logits.clone()]   # second graph's buffers (valid tokens)
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

    def pipeline(steps):
        """``steps`` streamed steps; returns the device time of all of them
        (ms, max over ranks)."""
        sync_all()
        layer.plan.barrier()
        e_a = torch.cuda.Event(enable_timing=True)
        e_b = torch.cuda.Event(enable_timing=True)
        e_a.record(stream)
        h2d_s.wait_event(e_a)
        d2h_s.wait_event(e_a)
        h2d_step(0)
        for i in range(steps):
            b = i % 2
            if i + 1 < steps:
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
        return float(t.item())

    pipeline(max(3, args.warmup))        # untimed: first DMA from the pinned buffers, streams
    t_ms = pipeline(args.steps)
    runners[1].check()
    e2e_step = t_ms / args.steps
    h2d = (x_h.numel() * 2 + l_h.numel() * 4) * world
    d2h = T * H * 2 * n
    return {"value": T_GLOBAL / (e2e_step / 1e3), "unit": "tokens/s",
            "ms_per_step": e2e_step, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h),
            "note": "every step: pinned host x/logits copied in (H2D stream), the captured "
                    "MoELayer forward, y copied back to pinned host (D2H stream); copies of "
                    "neighbouring steps overlap the forward (double-buffered); W untimed "
                    "warm-up steps of the same pipeline, then one timed region over all K "
                    "steps"}


LAYOUT_NOTE = ""


def named_tp(world):
    """TP degree of the config's named layout family: config B TP2 x EP(N/2)
    (TP2xEP4 at 8 GPUs), config C TP(N/2) x EP2 (TP4xEP2 at 8 GPUs; at 4
    GPUs TP2xEP2 measured 1.76 vs 1.97 ms for TP4, profiles/r02_configC_n4_layouts.jsonl)."""
    if world == 1:
        return 1
    return max(1, world // 2) if CONFIG == "C" else min(world, 2)


def auto_default(world):
    """Config B at 2 and 4 GPUs, where BASELINE.json names no layout: the
    fused-layer model's pick (the strategy selection the layer is built
    around) instead of extrapolating the 8-GPU TP2 x EP4."""
    return CONFIG == "B" and world in (2, 4)


def choose_layout(args, world):
    """(n, m) of the run: an explicit --tp; --tp auto (and, by default, config
    B at 2 and 4 GPUs): the fused-layer model's first pick
    (layer_model.select_layout) for this run's own routing (every rank
    computes it from the same seeded logits); otherwise the config's named
    layout family (B: TP2 x EP(N/2) -- TP2xEP4 at 8 GPUs; C: TP(N/2) x EP2 --
    TP4xEP2 at 8 GPUs; pure TP/EP below that)."""
    global LAYOUT_NOTE
    from paper_2601_08800_b200.layer import layout_for
    if (args.tp == "auto" or (args.tp is None and auto_default(world))) and world > 1:
        import torch
        logits = torch.cat([torch.randn(T_GLOBAL // world, E, device="cuda",
                                        generator=torch.Generator(device="cuda").manual_seed(
                                            2000 + r)) for r in range(world)])
        ids = torch.topk(logits, K_TOP, dim=-1).indices.cpu().numpy()
        n, m = layout_for(world, "auto", routing=ids, num_experts=E, hidden=H, inter=INTER)
        LAYOUT_NOTE = ("auto: layer_model.select_layout on a routing sample of this workload"
                       + ("" if args.tp == "auto" else
                          " (default where BASELINE names no layout; TP2xEP4 at 8 GPUs)"))
        return n, m
    if args.tp not in (None, "auto"):
        LAYOUT_NOTE = "--tp"
        return layout_for(world, int(args.tp))
    tp = named_tp(world)
    LAYOUT_NOTE = f"config {CONFIG}'s named layout family (TP{tp} x EP{world // tp})"
    return layout_for(world, tp)


CONFIGS = {
    "B": dict(H=2048, INTER=768, E=128, K=8, SHARED=0, T=8192,
              workload="Qwen3-30B-A3B-shaped MoE layer (BASELINE configs[1]), 8192-token "
                       "prefill, bf16 SwiGLU experts, fp32 gate logits"),
    "C": dict(H=7168, INTER=2048, E=256, K=8, SHARED=2048, T=8192,
              workload="DeepSeek-R1-shaped MoE layer (BASELINE configs[2]): 256 routed experts "
                       "top-8 + a 2048-wide shared expert, fp8 e4m3 experts (per-row activation "
                       "and per-channel weight scales), DeepSeek-V3 group-limited gate, "
                       "8192-token prefill"),
}
CONFIG = "B"
SHARED = 0
WROW = H * 2
WORKLOAD = CONFIGS["B"]["workload"]


def set_config(name, tokens=None):
    global CONFIG, H, INTER, E, K_TOP, SHARED, T_GLOBAL, WROW, WORKLOAD
    c = CONFIGS[name]
    CONFIG, H, INTER, E, K_TOP, SHARED = name, c["H"], c["INTER"], c["E"], c["K"], c["SHARED"]
    T_GLOBAL = tokens or c["T"]
    WROW = H + 16 if name == "C" else H * 2
    WORKLOAD = c["workload"]


def reference_layout(args):
    """(n, m) the reference arm simulates: this arm's explicit --tp, else the
    config's named layout; where our arm defaults to the model's pick
    (config B at 2 / 4 GPUs) the EP-only layout it takes on the uniform
    router (the reference arm never imports the product package to ask)."""
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if world == 1:
        return 1, 1
    if args.tp is None and auto_default(world):
        return world, 1
    tp = int(args.tp) if args.tp not in (None, "auto") else named_tp(world)
    return world // tp, tp


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="B", choices=sorted(CONFIGS),
                    help="B: Qwen3-30B-A3B shape, bf16 (BASELINE configs[1], default); "
                         "C: DeepSeek-R1 shape, fp8 + shared expert (configs[2])")
    ap.add_argument("--tp", default=None,
                    help="TP degree, or 'auto' (fused-layer model pick); default: the "
                         "config's named layout")
    ap.add_argument("--tokens", type=int, default=None,
                    help="override the global token count (default 8192)")
    ap.add_argument("--wire", default="auto", choices=["auto", "slot", "token"],
                    help="auto: token (dedup dispatch, pre-reduced combine) when n > 1")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=512)
    ap.add_argument("--ref-sample", type=int, default=1024)
    args = ap.parse_args()
    set_config(args.config, args.tokens)
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
