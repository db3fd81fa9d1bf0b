"""Reference-compatible API of the TP-EP MoE layer, executed on the B200.

Drop-in for ``moeplan.simcluster`` (``/root/reference/pkg/src/moeplan/
simcluster.py``, "sim"): the same names, signatures, return shapes and
exceptions, but every data-path step runs in the CUDA extension through the
C-ABI (``include/mixserve_b200.h``):

=============================  ==========================================
reference (sim)                B200 implementation
=============================  ==========================================
build_routing_table  236-251   K1 ``mx_route`` + ``mx_layout``
fused_ag_dispatch    330-407   K2 ``mx_dispatch`` (one-hop NVLink stores)
_partial_expert_outputs 535    K3 ``mx_expert`` (affine / tcgen05 SwiGLU)
fused_rs_combine     410-521   K4 ``mx_combine`` (pull-reduce + push-AG)
run_moe_block        565-595   all of the above (``mx_forward``)
_run_baseline        598-680   baseline pack/unpack kernels (+NCCL in SPMD)
moe_oracle           302-310   independent dense GPU kernel ``mx_dense_moe``
=============================  ==========================================

The whole-cluster functions emulate every rank of an ``n x m`` cluster on
the current GPU (kernel boundaries are the barriers); the SPMD layer
(:mod:`paper_2601_08800_b200.layer`) runs one rank per GPU over NVLink.
numpy float64 inputs run the f64 path, which reproduces the reference's
association order and is bit-identical to it; torch inputs keep their dtype
(f64 / f32 / bf16).
"""
from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import CapacityError, StrategyError, VerificationError
from .plan import DTYPES, LayerPlan
from .trace import (FLOAT_BYTES, TRACE_CSV_HEADER, Trace, TraceBuilder,
                    TraceEvent, save_trace, trace_from_csv, trace_to_csv)

__all__ = [
    "FLOAT_BYTES", "SimRank", "SimCluster", "build_cluster", "TraceEvent",
    "Trace", "TRACE_CSV_HEADER", "trace_to_csv", "trace_from_csv",
    "save_trace", "RouterSpec", "ExpertSpec", "SwiGLUExperts", "FP8SwiGLUExperts",
    "expert_home_node", "Slot", "RoutingTable", "build_routing_table",
    "ref_reduce_scatter", "ref_all_gather", "ref_all_reduce",
    "ref_all_to_all_pairwise", "moe_oracle", "fused_ag_dispatch",
    "fused_rs_combine", "run_moe_block", "verify_against_oracle",
]


# ---------------------------------------------------------------- cluster
@dataclass
class SimRank:
    global_rank: int
    node: int
    tp_rank: int
    inbox: dict = field(default_factory=dict)  # kept for API parity (unused)


@dataclass
class SimCluster:
    """``n_node`` groups of ``n_proc`` TP ranks, node-major (sim:49-67)."""

    n_node: int
    n_proc: int
    ranks: list

    @property
    def world_size(self) -> int:
        return self.n_node * self.n_proc

    def rank(self, r: int) -> SimRank:
        return self.ranks[r]


def build_cluster(n_node: int, n_proc: int) -> SimCluster:
    if n_node < 1 or n_proc < 1:
        raise StrategyError("cluster needs at least one node and one device")
    return SimCluster(n_node, n_proc,
                      [SimRank(r, r // n_proc, r % n_proc)
                       for r in range(n_node * n_proc)])


# ---------------------------------------------------------------- routing
@dataclass(frozen=True)
class RouterSpec:
    """Per-token ordered expert ids and weights (sim:143-186)."""

    num_experts: int
    expert_ids: tuple
    weights: tuple

    def __post_init__(self) -> None:
        if len(self.expert_ids) != len(self.weights):
            raise ValueError("expert_ids and weights must align per token")
        for t, (ids, ws) in enumerate(zip(self.expert_ids, self.weights)):
            if len(ids) != len(ws):
                raise ValueError(f"token {t}: ids and weights length mismatch")
            if len(set(ids)) != len(ids):
                raise ValueError(f"token {t}: duplicate expert id")
            if any(e < 0 or e >= self.num_experts for e in ids):
                raise ValueError(f"token {t}: expert id out of range")

    @property
    def num_tokens(self) -> int:
        return len(self.expert_ids)

    @classmethod
    def round_robin(cls, num_tokens, num_experts, k):
        return cls(num_experts,
                   tuple(tuple((t + i) % num_experts for i in range(k))
                         for t in range(num_tokens)),
                   tuple(tuple(1.0 / k for _ in range(k))
                         for _ in range(num_tokens)))

    @classmethod
    def random(cls, num_tokens, num_experts, k, seed):
        # same generator calls in the same order as sim:175-186, so a seed
        # reproduces the reference's routing under the same numpy
        rng = np.random.default_rng(seed)
        ids, ws = [], []
        for _ in range(num_tokens):
            chosen = sorted(int(e) for e in rng.choice(num_experts, size=k,
                                                       replace=False))
            raw = rng.uniform(0.1, 1.0, size=k)
            raw = raw / raw.sum()
            ids.append(tuple(chosen))
            ws.append(tuple(float(w) for w in raw))
        return cls(num_experts, tuple(ids), tuple(ws))

    @classmethod
    def from_arrays(cls, num_experts, ids, weights):
        ids = np.asarray(ids)
        weights = np.asarray(weights, dtype=np.float64)
        return cls(num_experts, tuple(tuple(int(e) for e in r) for r in ids),
                   tuple(tuple(float(w) for w in r) for r in weights))

    def arrays(self):
        """(ids [T,k] int32, weights [T,k] f64); k must be uniform."""
        ks = {len(r) for r in self.expert_ids}
        if len(ks) > 1:
            raise StrategyError("the B200 router needs the same top-k for every token")
        k = ks.pop() if ks else 0
        if not self.expert_ids:  # empty batch
            return np.zeros((0, 0), dtype=np.int32), np.zeros((0, 0), dtype=np.float64)
        ids = np.asarray(self.expert_ids, dtype=np.int32).reshape(-1, k)
        w = np.asarray(self.weights, dtype=np.float64).reshape(-1, k)
        return ids, w


@dataclass(frozen=True)
class ExpertSpec:
    """Affine expert stand-in ``scale*x + bias`` (sim:189-207)."""

    scales: tuple
    biases: tuple

    @classmethod
    def default(cls, num_experts):
        return cls(tuple(float(e + 1) for e in range(num_experts)),
                   tuple(float(e) for e in range(num_experts)))

    @property
    def num_experts(self) -> int:
        return len(self.scales)

    def apply(self, e, x):
        return self.scales[e] * x + self.biases[e]


class SwiGLUExperts:
    """Real expert FFNs ``down(silu(x Wg^T) * (x Wu^T))``, bf16 weights on
    the GPU: ``w_gate``/``w_up`` ``[E, I, h]``, ``w_down`` ``[E, h, I]``.

    Sharded for the TP-EP layout by :meth:`rank_shard`: rank (d, t) holds
    the experts of group d (contiguous, sim:210-212) with intermediate
    columns ``[t*I/m, (t+1)*I/m)`` -- a column-parallel up-projection and a
    row-parallel down-projection whose TP partials sum to the expert
    output (the real counterpart of the stand-in at sim:535-562)."""

    def __init__(self, w_gate, w_up, w_down):
        self.w_gate = w_gate.to(torch.bfloat16).contiguous()
        self.w_up = w_up.to(torch.bfloat16).contiguous()
        self.w_down = w_down.to(torch.bfloat16).contiguous()
        self.E, self.I, self.h = self.w_gate.shape
        self._cache = {}

    @classmethod
    def random(cls, num_experts, hidden, inter, seed=0, device="cuda"):
        g = torch.Generator(device=device).manual_seed(seed)
        mk = lambda *s, fan: (torch.randn(*s, generator=g, device=device) /
                              fan ** 0.5).to(torch.bfloat16)
        return cls(mk(num_experts, inter, hidden, fan=hidden),
                   mk(num_experts, inter, hidden, fan=hidden),
                   mk(num_experts, hidden, inter, fan=inter))

    @property
    def num_experts(self) -> int:
        return self.E

    def apply(self, e, x):
        """Duck-typed ``ExpertSpec.apply`` (numpy in/out) so the reference's
        own ``moe_oracle``/baseline can consume these experts."""
        xt = torch.as_tensor(np.atleast_2d(x), dtype=torch.float32,
                             device=self.w_gate.device)
        g = xt @ self.w_gate[e].float().T
        u = xt @ self.w_up[e].float().T
        a = (g * torch.sigmoid(g) * u).to(torch.bfloat16).float()
        out = (a @ self.w_down[e].float().T).double().cpu().numpy()
        return out[0] if np.ndim(x) == 1 else out

    def rank_shard(self, n, m, rank):
        """Packed (w13, w2) bf16 shards of one rank (see mx_swiglu_pack_w13)."""
        key = (n, m, rank)
        if key in self._cache:
            return self._cache[key]
        d, t = divmod(rank, m)
        if self.I % m or (self.I // m) % 128:
            raise StrategyError("intermediate/tp must be a multiple of 128")
        It = self.I // m
        e0 = -(-d * self.E // n)
        e1 = -(-(d + 1) * self.E // n)
        gate = self.w_gate[e0:e1, t * It:(t + 1) * It].contiguous()
        up = self.w_up[e0:e1, t * It:(t + 1) * It].contiguous()
        w13 = torch.empty(e1 - e0, 2 * It, self.h, dtype=torch.bfloat16,
                          device=self.w_gate.device)
        if e1 > e0:
            N.call("mx_swiglu_pack_w13", gate.data_ptr(), up.data_ptr(),
                   w13.data_ptr(), e1 - e0, It, self.h,
                   torch.cuda.current_stream().cuda_stream)
        w2 = self.w_down[e0:e1, :, t * It:(t + 1) * It].contiguous()
        self._cache[key] = (w13, w2)
        return w13, w2

    def stacked_shards(self, n, m):
        """Rank-major stack of every rank's shard (emulated cluster)."""
        key = ("stack", n, m)
        if key in self._cache:
            return self._cache[key]
        per = [self.rank_shard(n, m, r) for r in range(n * m)]
        el = max(w.shape[0] for w, _ in per)
        It = self.I // m
        w13 = torch.zeros(n * m, el, 2 * It, self.h, dtype=torch.bfloat16,
                          device=self.w_gate.device)
        w2 = torch.zeros(n * m, el, self.h, It, dtype=torch.bfloat16,
                         device=self.w_gate.device)
        for r, (a, b) in enumerate(per):
            w13[r, :a.shape[0]] = a
            w2[r, :b.shape[0]] = b
        self._cache[key] = (w13, w2)
        return w13, w2


def _quant_rows_torch(w):
    """Per-row e4m3 weights: scale = amax/448 (fp32), values (w/scale) rounded
    to e4m3 (RNE; |w/scale| <= 448 by construction)."""
    w = w.float()
    s = (w.abs().amax(-1) / 448.0).clamp_min(1e-30)
    return (w / s[..., None]).to(torch.float8_e4m3fn), s.contiguous()


class FP8SwiGLUExperts:
    """fp8 (e4m3) SwiGLU experts + optional shared expert (BASELINE config C,
    DeepSeek-R1 shape: 256 routed + 1 shared, fp8 experts).

    Each rank's TP shard is quantised per output channel (row) after
    sharding; tokens are quantised per row by the layer before dispatch and
    the activation is re-quantised per row of each TP shard between the two
    GEMMs.  ``shared`` is a one-expert :class:`SwiGLUExperts` applied to
    every token with weight 1, TP-sharded inside each group."""

    def __init__(self, experts: SwiGLUExperts, shared: SwiGLUExperts | None = None):
        self.src, self.shared = experts, shared
        self.E, self.I, self.h = experts.E, experts.I, experts.h
        self.Is = shared.I if shared is not None else 0
        self._cache = {}

    @classmethod
    def random(cls, num_experts, hidden, inter, shared_inter=0, seed=0, device="cuda"):
        ex = SwiGLUExperts.random(num_experts, hidden, inter, seed=seed, device=device)
        sh = (SwiGLUExperts.random(1, hidden, shared_inter, seed=seed + 7919, device=device)
              if shared_inter else None)
        return cls(ex, sh)

    @property
    def num_experts(self) -> int:
        return self.E

    def rank_shard(self, n, m, rank):
        """dict of this rank's e4m3 shards (uint8 views) and fp32 scales."""
        key = (n, m, rank)
        if key in self._cache:
            return self._cache[key]
        w13, w2 = self.src.rank_shard(n, m, rank)
        out = {}
        out["w13"], out["w13_scale"] = _quant_rows_torch(w13)
        out["w2"], out["w2_scale"] = _quant_rows_torch(w2)
        if self.shared is not None:
            s13, s2 = self.shared.rank_shard(1, m, rank % m)
            out["w13_shared"], out["w13_shared_scale"] = _quant_rows_torch(s13[0])
            out["w2_shared"], out["w2_shared_scale"] = _quant_rows_torch(s2[0])
        self._cache[key] = out
        return out

    def stacked_shards(self, n, m):
        key = ("stack", n, m)
        if key in self._cache:
            return self._cache[key]
        per = [self.rank_shard(n, m, r) for r in range(n * m)]
        el = max(p["w13"].shape[0] for p in per)
        out = {}
        for name, t in per[0].items():
            full = torch.zeros((n * m, el) + tuple(t.shape[1:]) if name in ("w13", "w2", "w13_scale", "w2_scale")
                               else (n * m,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            for r, p in enumerate(per):
                if name in ("w13", "w2", "w13_scale", "w2_scale"):
                    full[r, :p[name].shape[0]] = p[name]
                else:
                    full[r] = p[name]
            out[name] = full
        self._cache[key] = out
        return out

    def params(self, shards):
        ptr = lambda name: shards[name].data_ptr() if name in shards else None
        return N.ExpertParams(None, None, ptr("w13"), ptr("w2"), ptr("w13_scale"),
                              ptr("w2_scale"), ptr("w13_shared"), ptr("w2_shared"),
                              ptr("w13_shared_scale"), ptr("w2_shared_scale"))

    def oracle_arrays(self, n, m):
        """Dequantised per-(rank shard) weights for the CPU replica:
        gate/up [E, m, It, h], down [E, m, h, It] (+ shared [m, ...])."""
        It = self.I // m
        gate = np.zeros((self.E, m, It, self.h), np.float32)
        up = np.zeros_like(gate)
        down = np.zeros((self.E, m, self.h, It), np.float32)
        sh = None
        for r in range(n * m):
            d, t = divmod(r, m)
            e0 = -(-d * self.E // n)
            p = self.rank_shard(n, m, r)
            w13 = (p["w13"].float() * p["w13_scale"][..., None]).cpu().numpy()
            w2 = (p["w2"].float() * p["w2_scale"][..., None]).cpu().numpy()
            for i in range(w13.shape[0]):
                blocks = w13[i].reshape(-1, 2, 64, self.h)
                gate[e0 + i, t] = blocks[:, 0].reshape(It, self.h)
                up[e0 + i, t] = blocks[:, 1].reshape(It, self.h)
                down[e0 + i, t] = w2[i]
            if self.shared is not None and d == 0:
                if sh is None:
                    Ist = self.Is // m
                    sh = [np.zeros((m, Ist, self.h), np.float32),
                          np.zeros((m, Ist, self.h), np.float32),
                          np.zeros((m, self.h, Ist), np.float32)]
                s13 = (p["w13_shared"].float() * p["w13_shared_scale"][..., None]).cpu().numpy()
                blocks = s13.reshape(-1, 2, 64, self.h)
                sh[0][t] = blocks[:, 0].reshape(-1, self.h)
                sh[1][t] = blocks[:, 1].reshape(-1, self.h)
                sh[2][t] = (p["w2_shared"].float() * p["w2_shared_scale"][..., None]).cpu().numpy()
        return gate, up, down, sh


def expert_home_node(expert, n_node, num_experts):
    """Contiguous block placement (sim:210-212)."""
    return expert * n_node // num_experts


@dataclass(frozen=True)
class Slot:
    token: int
    expert: int
    weight: float
    src_node: int
    host_node: int


class RoutingTable:
    """Routing table produced on the GPU (sim:226-251).

    Holds per-host arrays in token-major table order; ``slots_by_host``
    materialises the reference's ``Slot`` tuples on first use."""

    def __init__(self, n_node, tokens_per_node, token, expert, weight, src,
                 send, expert_rows, num_experts=None):
        self.n_node = n_node
        self.num_experts = num_experts
        self.tokens_per_node = tokens_per_node
        self.token, self.expert, self.weight, self.src = token, expert, weight, src
        self.send = send                # S[j][d]
        self.expert_rows = expert_rows  # per host [(expert, rows)]
        self._slots = None

    @property
    def slots_by_host(self):
        if self._slots is None:
            self._slots = tuple(
                tuple(Slot(int(t), int(e), float(w), int(s), d)
                      for t, e, w, s in zip(self.token[d], self.expert[d],
                                            self.weight[d], self.src[d]))
                for d in range(self.n_node))
        return self._slots

    def total_slots(self) -> int:
        return int(sum(len(t) for t in self.token))


# ---------------------------------------------------------------- plans
_PLANS: "OrderedDict[tuple, LayerPlan]" = OrderedDict()


def _plan(n, m, T, h, E, k, dtype, kind="affine", inter=0, capacity=None, shared_inter=0):
    key = (n, m, T, h, E, k, dtype, kind, inter, capacity, shared_inter,
           torch.cuda.current_device())
    p = _PLANS.get(key)
    if p is None:
        p = LayerPlan(n, m, T, h, E, k, dtype=dtype, expert_kind=kind,
                      inter=inter, capacity=capacity, emulate=True,
                      shared_inter=shared_inter)
        _PLANS[key] = p
        while len(_PLANS) > 4:
            _PLANS.popitem(last=False)[1].close()
    else:
        _PLANS.move_to_end(key)
    return p


def _device():
    if not torch.cuda.is_available():
        raise N.NativeLibraryError("the B200 MoE layer needs a CUDA device "
                                   "(there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(x, dtype=None):
    if isinstance(x, torch.Tensor):
        t = x.to(_device())
        return t.to(dtype) if dtype is not None else t
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=_device(),
                           dtype=dtype or torch.float64)


def _router_tensors(router, wdtype):
    ids, w = router.arrays()
    dev = _device()
    return (torch.as_tensor(ids, device=dev).contiguous(),
            torch.as_tensor(w, device=dev).to(wdtype).contiguous())


def _expert_params(plan, experts, dtype):
    """ExpertParams struct + the tensors it points to (kept alive)."""
    if isinstance(experts, FP8SwiGLUExperts):
        sh = experts.stacked_shards(plan.n, plan.m)
        return experts.params(sh), sh
    if isinstance(experts, SwiGLUExperts):
        w13, w2 = experts.stacked_shards(plan.n, plan.m)
        return N.ExpertParams(None, None, w13.data_ptr(), w2.data_ptr()), (w13, w2)
    acc = torch.float64 if dtype is torch.float64 else torch.float32
    sc = torch.as_tensor(np.asarray(experts.scales, dtype=np.float64),
                         device=_device()).to(acc)
    bi = torch.as_tensor(np.asarray(experts.biases, dtype=np.float64),
                         device=_device()).to(acc)
    return N.ExpertParams(sc.data_ptr(), bi.data_ptr(), None, None), (sc, bi)


def _kind(experts):
    if isinstance(experts, FP8SwiGLUExperts):
        return "swiglu_fp8"
    return "swiglu" if isinstance(experts, SwiGLUExperts) else "affine"


def _route(plan, router, check_capacity=True):
    ids, w = _router_tensors(router, plan.wdtype)
    plan.route(ids=ids, weights=w)
    plan.layout(check_capacity=check_capacity)
    return ids, w


def _export_table(plan, n, T):
    """Host RoutingTable from the layout of every group (rank g*m)."""
    tok, exp, wts, src = ([[] for _ in range(n)] for _ in range(4))
    per_group = []
    for g in range(n):
        v = plan.rank_views(g * plan.m)
        per_group.append({k: t.cpu().numpy() for k, t in v.items()})
    cnt = per_group[0]["cnt_all"].astype(np.int64)
    send = per_group[0]["send"].astype(np.int64)
    E = plan.num_experts
    host_of = (np.arange(E) * n) // E
    tot = cnt.sum(axis=0)
    expert_rows = [[(int(e), int(tot[e])) for e in range(E)
                    if host_of[e] == d and tot[e] > 0] for d in range(n)]
    for d in range(n):
        S_d = int(send[:, d].sum())
        t_d = np.empty(S_d, np.int64)
        e_d = np.empty(S_d, np.int64)
        w_d = np.empty(S_d, np.float64)
        s_d = np.empty(S_d, np.int64)
        filled = np.zeros(S_d, bool)
        for g in range(n):
            pg = per_group[g]
            ids = pg["ids"].astype(np.int64)
            sel = host_of[ids] == d
            tm = pg["slot_tm"][sel]
            t_d[tm] = (np.nonzero(sel)[0] + g * T)
            e_d[tm] = ids[sel]
            w_d[tm] = pg["weights"][sel]
            s_d[tm] = g
            filled[tm] = True
        if not filled.all():
            raise RuntimeError("GPU layout is not a permutation of the table")
        tok[d], exp[d], wts[d], src[d] = t_d, e_d, w_d, s_d
    return RoutingTable(n, T, tok, exp, wts, src, send, expert_rows, E)


def build_routing_table(router: RouterSpec, n_node: int,
                        tokens_per_node: int) -> RoutingTable:
    """GPU routing (K1) exported as the reference's table (sim:236-251)."""
    if router.num_tokens != n_node * tokens_per_node:
        raise StrategyError(
            f"router covers {router.num_tokens} tokens, cluster carries "
            f"{n_node * tokens_per_node}")
    ids, _ = router.arrays()
    k = ids.shape[1]
    plan = _plan(n_node, 1, tokens_per_node, 8, router.num_experts, k,
                 torch.float64)
    _route(plan, router, check_capacity=False)
    return _export_table(plan, n_node, tokens_per_node)


# ---------------------------------------------------------------- collectives
def _same_shapes(tensors):
    shapes = {t.shape for t in tensors}
    if len(shapes) != 1:
        raise StrategyError(f"group members supplied mismatched shapes: {sorted(shapes)}")


def ref_reduce_scatter(tensors, axis=-1):
    """Collective semantics spec (sim:264-270): rank-ascending sum, shard i
    to rank i.  Host helper for tests and docs; not on the layer path."""
    _same_shapes(tensors)
    total = tensors[0].copy()
    for t in tensors[1:]:
        total = total + t
    return [s.copy() for s in np.array_split(total, len(tensors), axis=axis)]


def ref_all_gather(shards, axis=-1):
    full = np.concatenate(shards, axis=axis)
    return [full.copy() for _ in shards]


def ref_all_reduce(tensors, axis=-1):
    return ref_all_gather(ref_reduce_scatter(tensors, axis), axis)


def ref_all_to_all_pairwise(buffers):
    size = len(buffers)
    if any(len(row) != size for row in buffers):
        raise StrategyError("each rank must supply one buffer per peer")
    out = [[None] * size for _ in range(size)]
    for r in range(size):
        out[r][r] = buffers[r][r].copy()
    for i in range(1, size):
        for r in range(size):
            out[(r + i) % size][r] = buffers[r][(r + i) % size].copy()
    return out


# ---------------------------------------------------------------- oracle
def moe_oracle(x, router: RouterSpec, experts):
    """Dense single-device MoE (sim:302-310) on the GPU, independent of the
    fused path: y[t] = sum over ascending expert ids of w * expert(x[t])."""
    numpy_in = not isinstance(x, torch.Tensor)
    kind = _kind(experts)
    dtype = torch.bfloat16 if kind == "swiglu" else (
        torch.float64 if numpy_in else x.dtype)
    xd = _to_dev(x, dtype).contiguous()
    T, h = xd.shape
    ids, w = _router_tensors(router, torch.float64 if dtype is torch.float64
                             else torch.float32)
    k = ids.shape[1] if ids.numel() else 0
    s = torch.cuda.current_stream().cuda_stream
    if kind == "swiglu":
        y = torch.zeros(T, h, dtype=torch.float32, device=xd.device)
        N.call("mx_dense_moe", T, h, experts.E, k, N.MX_BF16, N.MX_EXPERT_SWIGLU,
               experts.I, xd.data_ptr(), ids.data_ptr(), w.data_ptr(), None, None,
               experts.w_gate.data_ptr(), experts.w_up.data_ptr(),
               experts.w_down.data_ptr(), y.data_ptr(), s)
    else:
        acc = torch.float64 if dtype is torch.float64 else torch.float32
        sc = torch.as_tensor(np.asarray(experts.scales), device=xd.device).to(acc)
        bi = torch.as_tensor(np.asarray(experts.biases), device=xd.device).to(acc)
        y = torch.empty_like(xd)
        N.call("mx_dense_moe", T, h, len(experts.scales), k, DTYPES[dtype],
               N.MX_EXPERT_AFFINE, 0, xd.data_ptr(), ids.data_ptr(), w.data_ptr(),
               sc.data_ptr(), bi.data_ptr(), None, None, None, y.data_ptr(), s)
    if numpy_in:
        return y.double().cpu().numpy()
    return y


def verify_against_oracle(y, x_global, router, experts, rtol=1e-9) -> float:
    """``max|y-e| / max(|e|,1)`` against :func:`moe_oracle` (sim:683-694)."""
    expected = moe_oracle(x_global, router, experts)
    if isinstance(expected, torch.Tensor):
        expected = expected.double().cpu().numpy()
    y = y.double().cpu().numpy() if isinstance(y, torch.Tensor) else np.asarray(y, np.float64)
    scale = np.maximum(np.abs(expected), 1.0)
    max_rel = float(np.max(np.abs(y - expected) / scale)) if expected.size else 0.0
    if max_rel > rtol:
        raise VerificationError(
            f"simulated output deviates from oracle: max relative error "
            f"{max_rel:.3e} > {rtol:g}")
    return max_rel


# ---------------------------------------------------------------- fused path
def _stack_groups(x_per_node, dtype=None):
    if isinstance(x_per_node[0], torch.Tensor):
        return torch.cat([_to_dev(x, dtype) for x in x_per_node], 0).contiguous()
    return _to_dev(np.concatenate([np.asarray(x, np.float64) for x in x_per_node], 0),
                   dtype).contiguous()


def fused_ag_dispatch(cluster: SimCluster, x_per_node, router: RouterSpec,
                      capacity=None, trace=None):
    """Fused AG-dispatch (sim:330-407) via K1 + K2.  Returns
    ``(received, table, trace)``; ``received[d]`` holds full rows of host
    d's slots in table order (a view of the expert-major GPU buffer)."""
    m, n = cluster.n_proc, cluster.n_node
    T, h = x_per_node[0].shape[0], x_per_node[0].shape[1]
    for j, x in enumerate(x_per_node):
        if tuple(x.shape) != (T, h):
            raise StrategyError(f"node {j}: input shape {tuple(x.shape)} mismatches {(T, h)}")
    if router.num_tokens != n * T:
        raise StrategyError(f"router covers {router.num_tokens} tokens, cluster "
                            f"carries {n * T}")
    numpy_in = not isinstance(x_per_node[0], torch.Tensor)
    xg = _stack_groups(x_per_node)
    ids, _ = router.arrays()
    plan = _plan(n, m, T, h, router.num_experts, ids.shape[1], xg.dtype,
                 capacity=capacity)
    _route(plan, router, check_capacity=True)
    plan.dispatch(xg)
    table = _export_table(plan, n, T)
    received = []
    for d in range(n):
        v = plan.rank_views(d * m)
        recv = plan.recv_view(d * m)
        S_d = len(table.token[d])
        out = torch.empty(S_d, h, dtype=xg.dtype, device=xg.device)
        # table order <- expert-major rows (glue for the reference layout)
        for g in range(n):
            pg = plan.rank_views(g * m)
            host = (pg["ids"].long() * n) // plan.num_experts
            sel = host == d
            out[pg["slot_tm"][sel].long()] = recv[pg["slot_pos"][sel].long()]
        received.append(out.double().cpu().numpy() if numpy_in else out)
    tb = TraceBuilder(n, m, T, h, table.send, trace)
    tb.dispatch()
    return received, table, tb.trace


def fused_rs_combine(cluster: SimCluster, partials, table: RoutingTable,
                     trace=None, compute_deps=None):
    """Fused RS-combine (sim:410-521) via K4.  ``partials[d][t]`` is TP rank
    t's partial on host d in table order.  Returns ``(y_per_node, trace)``."""
    m, n = cluster.n_proc, cluster.n_node
    h = partials[0][0].shape[1]
    for d in range(n):
        if len(partials[d]) != m:
            raise StrategyError(f"node {d}: expected {m} TP partials")
        for t in range(m):
            expect = (len(table.token[d]), h)
            if tuple(partials[d][t].shape) != expect:
                raise StrategyError(f"node {d} rank {t}: partial shape "
                                    f"{tuple(partials[d][t].shape)} mismatches {expect}")
    numpy_in = not isinstance(partials[0][0], torch.Tensor)
    dtype = torch.float64 if numpy_in else partials[0][0].dtype
    T = table.tokens_per_node
    k = max(1, table.total_slots() // max(1, n * T))
    E = int(max([int(e.max()) for e in table.expert if len(e)] + [0])) + 1
    # rebuild the router from the table so the device layout matches it
    ids = np.zeros((n * T, k), np.int64)
    w = np.zeros((n * T, k), np.float64)
    fill = np.zeros(n * T, np.int64)
    for d in range(n):
        for t_, e_, w_ in zip(table.token[d], table.expert[d], table.weight[d]):
            ids[t_, fill[t_]] = e_
            w[t_, fill[t_]] = w_
            fill[t_] += 1
    num_experts = table.num_experts or E
    router = RouterSpec.from_arrays(num_experts, ids, w)
    plan = _plan(n, m, T, h, num_experts, k, dtype)
    _route(plan, router, check_capacity=True)
    for d in range(n):
        for t in range(m):
            r = d * m + t
            part = _to_dev(partials[d][t], dtype)
            pv = plan.partial_view(r)
            for g in range(n):
                pg = plan.rank_views(g * m)
                sel = ((pg["ids"].long() * n) // num_experts) == d
                pv[pg["slot_pos"][sel].long()] = part[pg["slot_tm"][sel].long()]
    y = torch.empty(n * T, h, dtype=dtype, device=_device())
    plan.combine(y_out=y)
    tb = TraceBuilder(n, m, T, h, table.send, trace)
    tb.combine(compute_deps)
    ys = [y[j * T:(j + 1) * T] for j in range(n)]
    if numpy_in:
        ys = [t.cpu().numpy() for t in ys]
    return ys, tb.trace


def run_moe_block(cluster: SimCluster, x_global, router: RouterSpec, experts,
                  mode: str = "fused", capacity=None):
    """Dispatch, expert compute and combine over the cluster (sim:565-595).

    Returns ``(y_global, trace)``.  numpy input -> numpy f64 output (the f64
    path, bit-identical to the reference for affine experts); torch input
    keeps its dtype and device.  ``SwiGLUExperts`` run the bf16 tcgen05
    grouped GEMM."""
    n, m = cluster.n_node, cluster.n_proc
    if x_global.shape[0] % n != 0:
        raise StrategyError(f"{x_global.shape[0]} tokens do not split evenly over {n} nodes")
    if mode not in ("fused", "baseline"):
        raise ValueError(f"unknown mode {mode!r}")
    T = x_global.shape[0] // n
    h = x_global.shape[1]
    if router.num_tokens != x_global.shape[0]:
        raise StrategyError(f"router covers {router.num_tokens} tokens, cluster "
                            f"carries {x_global.shape[0]}")
    numpy_in = not isinstance(x_global, torch.Tensor)
    kind = _kind(experts)
    if kind in ("swiglu", "swiglu_fp8"):
        dtype = torch.bfloat16
    else:
        dtype = torch.float64 if numpy_in else x_global.dtype
    xg = _to_dev(x_global, dtype).contiguous()
    ids, _ = router.arrays()
    if T == 0:
        # empty batch: nothing to route or move; the reference still emits
        # its zero-byte event schedule (sim:353-520), and so does the builder
        tb = TraceBuilder(n, m, 0, h, np.zeros((n, n), dtype=np.int64))
        if mode == "fused":
            tb.dispatch()
            tb.combine(tb.expert([[] for _ in range(n)], tb.expert_deps()))
        else:
            tb.baseline([[] for _ in range(n)])
        y = torch.empty(0, h, dtype=dtype, device=xg.device)
        return (y.double().cpu().numpy() if numpy_in else y), tb.trace
    plan = _plan(n, m, T, h, router.num_experts, ids.shape[1], dtype, kind,
                 experts.I if kind != "affine" else 0, capacity,
                 experts.Is if kind == "swiglu_fp8" else 0)
    params, keep = _expert_params(plan, experts, dtype)
    _route(plan, router, check_capacity=True)
    cnt = plan.rank_views(0)["cnt_all"].cpu().numpy().astype(np.int64)
    send = plan.rank_views(0)["send"].cpu().numpy().astype(np.int64)
    E = plan.num_experts
    host_of = (np.arange(E) * n) // E
    tot = cnt.sum(axis=0)
    expert_rows = [[(int(e), int(tot[e])) for e in range(E)
                    if host_of[e] == d and tot[e] > 0] for d in range(n)]
    y = torch.empty(n * T, h, dtype=dtype, device=xg.device)
    tb = TraceBuilder(n, m, T, h, send)
    if mode == "fused":
        plan.dispatch(xg)
        plan.expert(params)
        plan.combine(y_out=y)
        tb.dispatch()
        comp = tb.expert(expert_rows, tb.expert_deps())
        tb.combine(comp)
    else:
        _baseline_emulated(plan, xg, params, y, send)
        tb.baseline(expert_rows)
    del keep
    out = y.double().cpu().numpy() if numpy_in else y
    return out, tb.trace


def _baseline_emulated(plan, xg, params, y, send):
    """Unfused AR + A2A (sim:598-680) on the emulated cluster: full-width
    pack -> (device copies standing in for NCCL all_to_all) -> unpack ->
    expert -> pack -> all_to_all back -> weighted unpack -> TP all-reduce."""
    n, m, T, h = plan.n, plan.m, plan.tokens, plan.hidden
    dev, dt = xg.device, xg.dtype
    s = torch.cuda.current_stream().cuda_stream
    lib = N.load()
    sends, counts = {}, {}
    for r in range(n * m):
        g = r // m
        buf = torch.empty(T * plan.top_k, h, dtype=dt, device=dev)
        cnt = torch.empty(n, dtype=torch.int32, device=dev)
        N.check(lib.mx_baseline_dispatch_pack(plan._plan, r,
                                              xg.data_ptr(), buf.data_ptr(),
                                              cnt.data_ptr(), s), "baseline pack")
        sends[r], counts[r] = buf, cnt
    S = np.asarray(send, dtype=np.int64)
    for r in range(n * m):
        d, t = divmod(r, m)
        blocks = []
        for j in range(n):
            off = int(S[j, :d].sum())
            blocks.append(sends[j * m + t][off:off + int(S[j, d])])
        recv = torch.cat(blocks, 0).contiguous() if blocks else sends[r][:0]
        N.check(lib.mx_baseline_dispatch_unpack(plan._plan, r, recv.data_ptr(), s),
                "baseline unpack")
        plan.expert(params, rank=r)
    backs = {}
    for r in range(n * m):
        d = r // m
        buf = torch.empty(max(1, int(S[:, d].sum())), h, dtype=dt, device=dev)
        cnt = torch.empty(n, dtype=torch.int32, device=dev)
        N.check(lib.mx_baseline_combine_pack(plan._plan, r, buf.data_ptr(),
                                             cnt.data_ptr(), s), "baseline pack back")
        backs[r] = buf
    for j in range(n):
        acc = None
        for t in range(m):
            r = j * m + t
            blocks = []
            for d in range(n):
                off = int(S[:j, d].sum())
                blocks.append(backs[d * m + t][off:off + int(S[j, d])])
            back = torch.cat(blocks, 0).contiguous()
            yt = torch.empty(T, h, dtype=dt, device=dev)
            N.check(lib.mx_baseline_combine_unpack(plan._plan, r, back.data_ptr(),
                                                   yt.data_ptr(), s), "baseline unpack back")
            acc = yt if acc is None else acc + yt  # TP all-reduce, rank order
        y[j * T:(j + 1) * T] = acc
