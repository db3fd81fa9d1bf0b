"""SPMD TP-EP MoE layer: one process per GPU, NVLink peer heaps.

This is the serving-side entry of the same hot path as ``run_moe_block``
(sim:565-595): rank ``r = group*m + tp`` (node-major, sim:63-67) owns the
tokens of its group (replicated across the group's TP ranks, sim:383-384),
the experts of its group (contiguous, sim:210-212) with the TP shard ``tp``
of their intermediate dimension, and after ``forward`` the combined output
of its group's tokens.

``forward`` runs the fused path (K1 route -> K2 dispatch -> K3 grouped GEMM
-> K4 combine, device flag barriers between phases).  ``forward_baseline``
runs the NCCL AR + A2A layout of ``_run_baseline`` (sim:598-680) on the
same buffers, for the fused-vs-NCCL comparison of BASELINE.json.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .plan import LayerPlan, stream_ptr
from .simcluster import FP8SwiGLUExperts, SwiGLUExperts


def layout_for(world: int, tp: int | str | None = None, *, routing=None, num_experts=None,
               hidden=None, inter=None, calib=None):
    """(n_group, tp) for a world size; default keeps TP=2 (config B,
    TP2 x EP4 at 8 GPUs) and falls back to pure TP/EP for 1 GPU.

    ``tp="auto"``: the layout :func:`.layer_model.select_layout` ranks first
    for a routing sample -- ``routing`` the [T_global, k] expert ids of a
    representative batch, identical on every rank (e.g. all-gathered), and
    the expert shapes.  On one NVSwitch box that is EP-only for a uniform
    router and TP2 x EP for a skewed one (config E)."""
    if tp == "auto":
        if routing is None or None in (num_experts, hidden, inter):
            raise ValueError("tp='auto' needs routing, num_experts, hidden and inter")
        from .layer_model import select_layout
        ranked = select_layout(routing, world, num_experts, hidden, inter, calib)
        if not ranked:
            raise ValueError(f"no layout of {world} GPUs fits these expert shapes")
        return ranked[0]["n"], ranked[0]["m"]
    if tp is None:
        tp = 1 if world == 1 else 2
    if world % tp:
        raise ValueError(f"world {world} not divisible by tp {tp}")
    return world // tp, tp


def tp_ep_groups(n: int, m: int, rank: int):
    """(EP group, TP group) of ``rank`` in the n x m layout, rank ``d*m + t``
    node-major (sim:63-67): the EP group is the n ranks with the same TP
    index t (the all-to-all peers of ``_run_baseline``, sim:598-680), the TP
    group the m ranks of node d (its all-reduce).  Collective: every rank
    must call it, in the same order, since ``new_group`` is."""
    if not dist.is_initialized():
        raise RuntimeError("tp_ep_groups needs an initialised process group")
    if dist.get_world_size() < n * m:
        raise ValueError(f"layout {n}x{m} needs {n * m} ranks, world has {dist.get_world_size()}")
    ep = [dist.new_group([d * m + t for d in range(n)]) for t in range(m)]
    tp = [dist.new_group([j * m + t for t in range(m)]) for j in range(n)]
    group, t = divmod(rank, m)
    return ep[t], tp[group]


def baseline_splits(S, group: int):
    """Row split sizes of node ``group``'s two all-to-alls (sim:617-640):
    ``send[d]`` = its slots hosted on node d (row ``S[group]``), ``recv[j]``
    = node j's slots it hosts (column ``S[:, group]``).  The dispatch sends
    ``send`` and receives ``recv``; the combine swaps them."""
    S = np.asarray(S)
    if S.ndim != 2 or S.shape[0] != S.shape[1] or not 0 <= group < S.shape[0]:
        raise ValueError(f"send matrix {S.shape} has no node {group}")
    return [int(v) for v in S[group]], [int(v) for v in S[:, group]]


class MoELayer:
    def __init__(self, n, m, tokens_per_group, hidden, num_experts, top_k,
                 inter, experts: SwiGLUExperts | None = None, *, rank=None,
                 w13=None, w2=None, dtype=torch.bfloat16, renormalize=True,
                 capacity=None, expert_kind="swiglu", scales=None, biases=None,
                 process_group=None, wire="slot", gate=None):
        self.n, self.m, self.W = n, m, n * m
        if rank is None:
            rank = dist.get_rank() if dist.is_initialized() else 0
        self.rank = rank
        self.group, self.tp_rank = divmod(rank, m)
        self.T, self.h, self.E, self.k, self.I = (tokens_per_group, hidden,
                                                  num_experts, top_k, inter)
        self.dtype = dtype
        if isinstance(experts, FP8SwiGLUExperts):
            expert_kind = "swiglu_fp8"
        shared_inter = experts.Is if expert_kind == "swiglu_fp8" else 0
        self.plan = LayerPlan(n, m, tokens_per_group, hidden, num_experts,
                              top_k, dtype=dtype, expert_kind=expert_kind,
                              inter=inter, renormalize=renormalize,
                              capacity=capacity, emulate=False, rank=rank,
                              process_group=process_group, wire=wire,
                              shared_inter=shared_inter, gate=gate)
        self.wire = wire
        if expert_kind == "swiglu_fp8":
            self.shards = experts.rank_shard(n, m, rank)
            self.params = experts.params(self.shards)
        elif expert_kind == "swiglu":
            if w13 is None:
                w13, w2 = experts.rank_shard(n, m, rank)
            self.w13, self.w2 = w13, w2
            self.params = N.ExpertParams(None, None, w13.data_ptr(), w2.data_ptr())
        else:
            acc = torch.float64 if dtype is torch.float64 else torch.float32
            self.scales = torch.as_tensor(np.asarray(scales), device="cuda").to(acc)
            self.biases = torch.as_tensor(np.asarray(biases), device="cuda").to(acc)
            self.params = N.ExpertParams(self.scales.data_ptr(),
                                         self.biases.data_ptr(), None, None)
        self.y = self.plan.y_view(rank)
        self._ep_group = self._tp_group = None

    # ------------------------------------------------------------ fused path
    def forward(self, x, logits=None, ids=None, weights=None, out=None,
                stream=None, check=True):
        """Fused layer forward.  ``x``: [T, h] tokens of this rank's group
        (device, or host -> copied in on ``stream``); ``logits`` [T, E] f32
        or ``ids``/``weights`` [T, k].  Returns the [T, h] output (a view of
        the layer's buffer, valid until the next call), or ``out`` when given
        -- a host ``out`` is filled by a device-to-host copy on ``stream``
        that has completed when this returns.

        ``check`` (eager calls only; skipped while a CUDA graph captures)
        synchronizes the stream and raises what the kernels flagged:
        CapacityError when a host's routed slots exceed ``capacity``
        (sim:346-351 -- the kernels never write past it), StrategyError for
        an expert id out of range, NativeLibraryError when a peer barrier's
        watchdog expired."""
        dev = self.plan.device
        s = stream or torch.cuda.current_stream(dev)
        with torch.cuda.stream(s):
            if not x.is_cuda:
                x = x.to(dev, non_blocking=True)
            if logits is not None and not logits.is_cuda:
                logits = logits.to(dev, non_blocking=True)
            self.plan.forward(x, self.params, logits=logits, ids=ids,
                              weights=weights, rank=self.rank, stream=s)
            capturing = torch.cuda.is_current_stream_capturing()
            if check and not capturing:
                self.plan.check(rank=self.rank, stream=s)
            if out is None:
                return self.y
            out.copy_(self.y, non_blocking=True)
            if not out.is_cuda and not capturing:
                s.synchronize()
        return out

    def forward_stepped(self, x, logits=None, ids=None, weights=None, host_barrier=None):
        """The fused forward's phases with every device barrier replaced by
        arrive -> host synchronization (``host_barrier()``, e.g. a gloo
        ``dist.barrier``) -> verify: for ranks that share ONE GPU as separate
        processes, where a kernel spinning on a peer's flag has no guarantee
        of ever running beside the peer's kernel.  Exercises the IPC heaps,
        peer stores/loads and the epoch-flag protocol of the SPMD layer;
        raises through :meth:`LayerPlan.check` like :meth:`forward`."""
        p, r = self.plan, self.rank
        lib = N.load()
        sp = stream_ptr(None)
        host_barrier = host_barrier or (lambda: dist.barrier())

        def bar(group=False):
            p.barrier_split(1, group)
            torch.cuda.synchronize()
            host_barrier()
            p.barrier_split(2, group)

        p.route(logits=logits, ids=ids, weights=weights, rank=r)
        bar()
        p.layout(rank=r)
        p.dispatch(x, rank=r)
        bar()
        tok = self.wire == "token"
        stages = ([3] if tok else []) + [1, 2] + ([4] if tok else [])
        for st in stages:
            N.check(lib.mx_expert_stage(p._plan, r, C.byref(self.params), st, sp), "expert")
        bar()
        p.combine(rank=r)
        if self.m > 1:
            bar(group=True)
        torch.cuda.synchronize()
        host_barrier()
        p.check(rank=r)
        return self.y

    def forward_phases(self, x, logits, events, stream=None, event_factory=None):
        """Same launches as :meth:`forward`, phase by phase, recording a CUDA
        event after each phase (for per-kernel timing in bench.py)."""
        s = stream or torch.cuda.current_stream()
        make = event_factory or (lambda: torch.cuda.Event(enable_timing=True))

        def mark(name):
            ev = make()
            ev.record(s)
            events.append((name, ev))

        return self.run_phases(x, logits, mark, s)

    def phase_names(self):
        tok = self.wire == "token"
        return (["start", "route", "barrier_counts", "layout", "dispatch", "barrier_dispatch"]
                + (["expand"] if tok else []) + ["gemm1_swiglu", "gemm2"]
                + (["pair_reduce"] if tok else [])
                + ["barrier_partials", "combine", "barrier_out"])

    def run_phases(self, x, logits, mark, stream):
        """The fused forward's launches in order, calling ``mark(phase)``
        after each phase (and ``mark("start")`` first)."""
        p, r, s = self.plan, self.rank, stream
        lib = N.load()
        sp = stream_ptr(s)
        mark("start")
        p.route(logits=logits, rank=r, stream=s); mark("route")
        p.barrier(stream=s); mark("barrier_counts")
        p.layout(rank=r, stream=s); mark("layout")
        p.dispatch(x, rank=r, stream=s); mark("dispatch")
        p.barrier(stream=s); mark("barrier_dispatch")
        tok = self.wire == "token"
        if tok:
            N.check(lib.mx_expert_stage(p._plan, r, C.byref(self.params), 3, sp), "expand")
            mark("expand")
        N.check(lib.mx_expert_stage(p._plan, r, C.byref(self.params), 1, sp), "gemm1")
        mark("gemm1_swiglu")
        N.check(lib.mx_expert_stage(p._plan, r, C.byref(self.params), 2, sp), "gemm2")
        mark("gemm2")
        if tok:
            N.check(lib.mx_expert_stage(p._plan, r, C.byref(self.params), 4, sp), "pair_reduce")
            mark("pair_reduce")
        p.barrier(stream=s); mark("barrier_partials")
        p.combine(rank=r, stream=s); mark("combine")
        p.barrier(stream=s); mark("barrier_out")
        return self.y

    def capture(self, x, logits=None, ids=None, weights=None, with_events=False):
        """Capture one forward (all launches and device barriers) in a CUDA
        graph bound to these input buffers; see :class:`CapturedForward`."""
        return CapturedForward(self, x, logits, ids, weights, with_events)

    def routing_counts(self):
        """(cnt_all [n,E], send [n,n]) of the last forward, on the host."""
        v = self.plan.rank_views(self.rank)
        return v["cnt_all"].cpu().numpy(), v["send"].cpu().numpy()

    def pair_counts(self):
        """U[j][d]: tokens of group j hitting host d (last forward), host."""
        import numpy as _np
        upos = self.plan.buffer(self.rank, N.MX_BUF_UPOS, torch.int32, (self.T, self.n))
        mine = (upos >= 0).sum(0).to(torch.int64)
        if dist.is_initialized() and self.W > 1:
            allv = [torch.empty_like(mine) for _ in range(self.W)]
            dist.all_gather(allv, mine)
            return _np.stack([allv[j * self.m].cpu().numpy() for j in range(self.n)])
        return mine.cpu().numpy()[None, :]

    # ------------------------------------------------------------ NCCL baseline
    def _groups(self):
        if self._ep_group is None:
            self._ep_group, self._tp_group = tp_ep_groups(self.n, self.m, self.rank)
        return self._ep_group, self._tp_group

    def forward_baseline(self, x, logits, stream=None, events=None, splits=None, mark=None):
        """NCCL AR + A2A layout (sim:598-680): full-width all_to_all dispatch
        from every TP rank, the same expert kernels, full-width all_to_all
        combine of TP partials, TP all_reduce.

        NCCL's all_to_all_single needs the split sizes on the host: without
        ``splits`` (the [n, n] send matrix S of this routing) they are read
        back with one D2H sync, as any dynamic NCCL MoE layer does; with
        ``splits`` nothing syncs and the call can be captured in a CUDA
        graph (:meth:`capture_baseline`).  ``mark(name)`` / ``events`` record
        a point after each phase: route, a2a_dispatch, expert, a2a_combine,
        allreduce."""
        p, r, lib = self.plan, self.rank, N.load()
        s = stream or torch.cuda.current_stream()
        sp = stream_ptr(s)
        ep_g, tp_g = self._groups()

        def _mark(name):
            if mark is not None:
                mark(name)
            elif events is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(s)
                events.append((name, ev))

        _mark("start")
        p.route(logits=logits, rank=r, stream=s)
        p.barrier(stream=s)          # count rows published (our K1 exchange)
        p.layout(rank=r, stream=s)
        S = np.asarray(splits) if splits is not None else \
            p.rank_views(r)["send"].cpu().numpy()   # host sync for the split sizes
        _mark("route")
        j, n, h = self.group, self.n, self.h
        in_split, out_split = baseline_splits(S, j)
        send_rows, recv_rows = sum(in_split), sum(out_split)
        key = (send_rows, recv_rows)
        if getattr(self, "_bl_key", None) != key:
            dev = x.device
            self._bl_bufs = dict(
                send=torch.empty(max(1, send_rows), h, dtype=self.dtype, device=dev),
                recv=torch.empty(max(1, recv_rows), h, dtype=self.dtype, device=dev),
                back=torch.empty(max(1, recv_rows), h, dtype=self.dtype, device=dev),
                ret=torch.empty(max(1, send_rows), h, dtype=self.dtype, device=dev),
                y=torch.empty(self.T, h, dtype=self.dtype, device=dev),
                cnt=torch.empty(n, dtype=torch.int32, device=dev))
            self._bl_key = key
        b = self._bl_bufs
        N.check(lib.mx_baseline_dispatch_pack(p._plan, r, C.c_void_p(x.data_ptr()),
                                              C.c_void_p(b["send"].data_ptr()),
                                              C.c_void_p(b["cnt"].data_ptr()), sp), "pack")
        dist.all_to_all_single(b["recv"][:recv_rows], b["send"][:send_rows],
                               output_split_sizes=out_split, input_split_sizes=in_split,
                               group=ep_g)
        _mark("a2a_dispatch")
        N.check(lib.mx_baseline_dispatch_unpack(p._plan, r, C.c_void_p(b["recv"].data_ptr()),
                                                sp), "unpack")
        for stage in (1, 2):  # the GEMMs only (no wire-TOKEN expand/pre-reduce)
            N.check(lib.mx_expert_stage(p._plan, r, C.byref(self.params), stage, sp), "expert")
        _mark("expert")
        N.check(lib.mx_baseline_combine_pack(p._plan, r, C.c_void_p(b["back"].data_ptr()),
                                             C.c_void_p(b["cnt"].data_ptr()), sp), "pack back")
        dist.all_to_all_single(b["ret"][:send_rows], b["back"][:recv_rows],
                               output_split_sizes=in_split, input_split_sizes=out_split,
                               group=ep_g)
        _mark("a2a_combine")
        N.check(lib.mx_baseline_combine_unpack(p._plan, r, C.c_void_p(b["ret"].data_ptr()),
                                               C.c_void_p(b["y"].data_ptr()), sp), "unpack back")
        if self.m > 1:
            dist.all_reduce(b["y"], group=tp_g)
        _mark("allreduce")
        return b["y"]

    def capture_baseline(self, x, logits, with_events=False):
        """The NCCL baseline with this routing's split sizes fixed on the
        host (read once, outside), captured as one CUDA graph like the fused
        forward: no host sync and no per-launch CPU overhead inside, so the
        comparison with :meth:`capture` is communicator against
        communicator.  Falls back to eager replays of the static-split call
        when NCCL collectives cannot be captured (``.graph`` is False)."""
        return CapturedBaseline(self, x, logits, with_events)

    def close(self):
        self.plan.close()


class CapturedForward:
    """A layer forward captured once and replayed as one CUDA graph.

    Barrier epochs live on the device, so replays stay in lockstep across
    ranks; inputs are read from the captured buffers (copy new tokens into
    ``x``/``logits`` before calling).  ``with_events`` records an external
    CUDA event after every phase inside the graph (per-kernel timing)."""

    def __init__(self, layer, x, logits=None, ids=None, weights=None, with_events=False):
        self.layer, self.x, self.logits = layer, x, logits
        self.events = []
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):            # warm-up outside the graph
            layer.forward(x, logits, ids=ids, weights=weights)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            if with_events:
                evs = []
                layer.forward_phases(x, logits, evs, event_factory=_external_event)
                self.events = evs
            else:
                layer.forward(x, logits, ids=ids, weights=weights)
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier()

    def __call__(self):
        self.graph.replay()
        return self.layer.y

    def check(self, stream=None):
        """Synchronize and raise the errors the replays flagged (capacity,
        expert ids, barrier watchdog); see :meth:`MoELayer.forward`."""
        self.layer.plan.check(rank=self.layer.rank, stream=stream)

    def phase_ms(self):
        """(name, ms) per phase of the last replay (call after a sync)."""
        return [(b, ea.elapsed_time(eb))
                for (a, ea), (b, eb) in zip(self.events[:-1], self.events[1:])]


class CapturedBaseline:
    """See :meth:`MoELayer.capture_baseline`."""

    def __init__(self, layer, x, logits, with_events=False):
        self.layer, self.x, self.logits = layer, x, logits
        self.events = []
        self.with_events = with_events
        layer.forward_baseline(x, logits)            # eager: split sizes, NCCL warm-up
        p = layer.plan
        self.splits = p.rank_views(layer.rank)["send"].cpu().numpy().copy()
        layer.forward_baseline(x, logits, splits=self.splits)
        torch.cuda.synchronize()
        dist.barrier()
        self.graph = None
        self.error = None
        try:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                layer.forward_baseline(x, logits, splits=self.splits)
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            dist.barrier()
            with torch.cuda.graph(g):
                if with_events:
                    evs = []

                    def mark(name):
                        ev = _external_event()
                        ev.record()
                        evs.append((name, ev))
                    layer.forward_baseline(x, logits, splits=self.splits, mark=mark)
                    self.events = evs
                else:
                    layer.forward_baseline(x, logits, splits=self.splits)
            torch.cuda.synchronize()
            dist.barrier()
            self.graph = g
        except Exception as e:  # NCCL capture unsupported: eager static-split replays
            self.error = f"{type(e).__name__}: {e}"[:300]
            torch.cuda.synchronize()
            dist.barrier()

    def __call__(self):
        if self.graph is not None:
            self.graph.replay()
            return self.layer._bl_bufs["y"]
        evs = [] if self.with_events else None
        y = self.layer.forward_baseline(self.x, self.logits, splits=self.splits, events=evs)
        if evs is not None:
            self.events = evs
        return y

    def phase_ms(self):
        return [(b, ea.elapsed_time(eb))
                for (a, ea), (b, eb) in zip(self.events[:-1], self.events[1:])]


def _external_event():
    return torch.cuda.Event(enable_timing=True, external=True)
