"""Host wrapper of the communicator + layer plan (C-ABI objects).

A :class:`LayerPlan` owns one ``mx_comm`` (the symmetric heaps) and one
``mx_plan`` (buffer layout of one TP-EP MoE layer shape).  Two modes:

* **emulated** -- one process holds every rank of an ``n x m`` cluster on one
  device; each phase is launched for all ranks in turn, kernel boundaries
  being the barriers.  This backs the whole-cluster reference API
  (``run_moe_block(cluster, x_global, ...)``, sim:565) on a single GPU.
* **SPMD** -- one process per GPU (``torchrun``); heaps are exchanged as CUDA
  IPC handles over ``torch.distributed`` and the kernels store to / load from
  peer heaps over NVLink, with device-side flag barriers between phases.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _native as N
from .errors import StrategyError

DTYPES = {torch.float64: N.MX_F64, torch.float32: N.MX_F32,
          torch.bfloat16: N.MX_BF16}
_TYPESTR = {torch.float64: "<f8", torch.float32: "<f4", torch.int32: "<i4", torch.int64: "<i8",
            torch.bfloat16: "<i2"}


class _DevArray:
    """Minimal ``__cuda_array_interface__`` holder (zero-copy views)."""

    def __init__(self, ptr, shape, typestr, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape), "typestr": typestr,
            "data": (int(ptr), False), "version": 3, "strides": None,
            "stream": None}


def device_view(ptr, shape, dtype, owner, device):
    """Wrap raw device memory as a torch tensor without copying."""
    raw = torch.as_tensor(_DevArray(ptr, shape, _TYPESTR[dtype], owner),
                          device=device)
    return raw.view(torch.bfloat16) if dtype is torch.bfloat16 else raw


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@dataclass(frozen=True)
class GateSpec:
    """The gate ``route`` applies to logits (``mx_router`` in the C ABI).

    ``softmax``: Qwen3-MoE -- softmax over E, top-k by logit (the plan's
    ``renormalize`` renormalises over the k).  ``group_limited``:
    DeepSeek-V3 -- sigmoid scores, correction ``bias`` [E] fp32, top-2-sum
    group scores, ``topk_groups`` of ``groups`` kept, weights scaled by
    ``scaling`` (transformers modeling_deepseek_v3.py
    ``DeepseekV3MoE.route_tokens_to_experts``)."""

    kind: str = "softmax"
    groups: int = 0
    topk_groups: int = 0
    scaling: float = 1.0
    bias: object = None

    @classmethod
    def deepseek_v3(cls, bias=None, groups=8, topk_groups=4, scaling=2.5):
        return cls("group_limited", groups, topk_groups, scaling, bias)


class LayerPlan:
    def __init__(self, n, m, tokens, hidden, num_experts, top_k, *,
                 dtype=torch.float64, expert_kind="affine", inter=0,
                 renormalize=True, capacity=None, emulate=True, rank=None,
                 process_group=None, device=None, wire="slot", shared_inter=0,
                 gate=None):
        lib = N.load()
        if not torch.cuda.is_available():
            raise N.NativeLibraryError("no CUDA device: the MoE layer runs "
                                       "only on the GPU (no CPU fallback)")
        if dtype not in DTYPES:
            raise StrategyError(f"unsupported hidden dtype {dtype}")
        self.n, self.m, self.W = n, m, n * m
        self.tokens, self.hidden = tokens, hidden
        self.num_experts, self.top_k = num_experts, top_k
        self.dtype = dtype
        self.wdtype = torch.float64 if dtype is torch.float64 else torch.float32
        self.expert_kind = expert_kind
        self.inter = inter
        self.emulate = emulate
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.desc = N.PlanDesc(
            n, m, tokens, hidden, num_experts, top_k, inter, DTYPES[dtype],
            {"swiglu": N.MX_EXPERT_SWIGLU, "swiglu_fp8": N.MX_EXPERT_SWIGLU_FP8}.get(
                expert_kind, N.MX_EXPERT_AFFINE),
            1 if renormalize else 0,
            N.MX_WIRE_TOKEN if wire == "token" else N.MX_WIRE_SLOT, int(shared_inter),
            int(capacity or 0))
        self.gate = gate or GateSpec()
        if self.gate.kind == "group_limited":
            self._gate_bias = None
            if self.gate.bias is not None:
                self._gate_bias = torch.as_tensor(self.gate.bias).to(
                    self.device, torch.float32).contiguous()
                if self._gate_bias.numel() != num_experts:
                    raise StrategyError("gate bias needs one entry per expert")
            self.desc.router = N.MX_ROUTER_GROUP_LIMITED
            self.desc.router_groups = int(self.gate.groups)
            self.desc.router_topk_groups = int(self.gate.topk_groups)
            self.desc.routed_scaling = float(self.gate.scaling)
            self.desc.router_bias = (self._gate_bias.data_ptr()
                                     if self._gate_bias is not None else None)
        elif self.gate.kind != "softmax":
            raise StrategyError(f"unknown gate {self.gate.kind!r}")
        self.wire = wire
        heap = C.c_size_t()
        N.check(lib.mx_plan_heap_bytes(C.byref(self.desc), C.byref(heap)),
                "plan")
        self.heap_bytes = heap.value
        self.rank = -1 if emulate else int(rank)
        comm = C.c_void_p()
        with torch.cuda.device(self.device):
            N.check(lib.mx_comm_create(n, m, self.rank, 1 if emulate else 0,
                                       self.heap_bytes, C.byref(comm)), "comm")
        self._comm = comm
        if not emulate and self.W > 1:
            self._open_peers(process_group)
        plan = C.c_void_p()
        N.check(lib.mx_plan_create(comm, C.byref(self.desc), C.byref(plan)),
                "plan")
        self._plan = plan
        self.capacity = int(self.buffer_bytes(self._any_rank(), N.MX_BUF_RECV)
                            // max(1, hidden * torch.tensor([], dtype=dtype).element_size()))

    # ------------------------------------------------------------ plumbing
    def _any_rank(self):
        return 0 if self.emulate else self.rank

    def _open_peers(self, group):
        import torch.distributed as dist
        handle = (C.c_char * 64)()
        N.check(N.load().mx_comm_ipc_handle(self._comm, handle), "ipc")
        mine = bytes(handle)
        allh = [None] * self.W
        dist.all_gather_object(allh, mine, group=group)
        buf = (C.c_char * (64 * self.W)).from_buffer_copy(b"".join(allh))
        N.check(N.load().mx_comm_open_peers(self._comm, buf), "open peers")

    def buffer_bytes(self, rank, which):
        ptr, nbytes = C.c_void_p(), C.c_size_t()
        N.check(N.load().mx_plan_buffer(self._plan, rank, which, C.byref(ptr),
                                        C.byref(nbytes)), "buffer")
        return nbytes.value

    def buffer(self, rank, which, dtype, shape):
        ptr, nbytes = C.c_void_p(), C.c_size_t()
        N.check(N.load().mx_plan_buffer(self._plan, rank, which, C.byref(ptr),
                                        C.byref(nbytes)), "buffer")
        return device_view(ptr.value, shape, dtype, self, self.device)

    def close(self):
        lib = N.load()
        if getattr(self, "_plan", None):
            lib.mx_plan_destroy(self._plan)
            self._plan = None
        if getattr(self, "_comm", None):
            lib.mx_comm_destroy(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ phases
    def _r(self, rank):
        return -1 if rank is None else int(rank)

    def _rows(self):
        # emulated plans take every group's tokens stacked [n*T, ...]
        return self.n * self.tokens if self.emulate else self.tokens

    def _on_device(self, t, name, dtype, cols, convert):
        """``t`` as a contiguous [rows, cols] ``dtype`` tensor on the plan's
        device.  Routing tensors are converted (ids straight from
        ``torch.topk`` are int64); the hidden states must already be the
        plan's dtype.  Raises StrategyError like the reference's shape checks
        (sim:341-344)."""
        if not isinstance(t, torch.Tensor):
            raise StrategyError(f"{name} must be a torch tensor, got {type(t).__name__}")
        shape = (self._rows(), cols)
        if tuple(t.shape) != shape:
            raise StrategyError(f"{name} shape {tuple(t.shape)} mismatches {shape}")
        if t.dtype != dtype:
            if not convert:
                raise StrategyError(f"{name} dtype {t.dtype} mismatches the plan's {dtype}")
            t = t.to(dtype)
        if t.device != self.device:
            if t.is_cuda:
                raise StrategyError(f"{name} lives on {t.device}, the plan on {self.device}")
            t = t.to(self.device, non_blocking=True)
        return t.contiguous()

    def _routing_inputs(self, logits, ids, weights):
        if (logits is None) == (ids is None):
            raise StrategyError("pass exactly one of logits or ids")
        if logits is not None:
            return self._on_device(logits, "logits", torch.float32, self.num_experts, True), None, None
        if weights is None:
            raise StrategyError("ids need weights")
        return (None, self._on_device(ids, "ids", torch.int32, self.top_k, True),
                self._on_device(weights, "weights", self.wdtype, self.top_k, True))

    def route(self, logits=None, ids=None, weights=None, rank=None, stream=None):
        lib = N.load()
        logits, ids, weights = self._routing_inputs(logits, ids, weights)
        N.check(lib.mx_route(self._plan, self._r(rank),
                             C.c_void_p(logits.data_ptr()) if logits is not None else None,
                             C.c_void_p(ids.data_ptr()) if ids is not None else None,
                             C.c_void_p(weights.data_ptr()) if weights is not None else None,
                             stream_ptr(stream)), "route")

    def layout(self, rank=None, check_capacity=False, stream=None):
        N.check(N.load().mx_layout(self._plan, self._r(rank), int(check_capacity),
                                   stream_ptr(stream)), "layout")

    def barrier(self, stream=None):
        N.check(N.load().mx_comm_barrier(self._comm, stream_ptr(stream)), "barrier")

    def barrier_split(self, half, group_only=False, stream=None):
        """Non-spinning barrier halves (1 arrive, 2 verify) for ranks sharing
        one GPU; the caller synchronizes the processes in between."""
        N.check(N.load().mx_comm_barrier_split(self._comm, int(half), int(group_only),
                                               stream_ptr(stream)), "barrier")

    def stamp(self, slot, rank=None, stream=None):
        """Device clock (ns) into stamp ``slot`` after all earlier launches."""
        N.check(N.load().mx_stamp(self._plan, self._r(rank), int(slot), stream_ptr(stream)),
                "stamp")

    def stamps_view(self, rank):
        return self.buffer(rank, N.MX_BUF_STAMPS, torch.int64, (64,))

    def dispatch(self, x, rank=None, stream=None):
        x = self._on_device(x, "x", self.dtype, self.hidden, False)
        N.check(N.load().mx_dispatch(self._plan, self._r(rank),
                                     C.c_void_p(x.data_ptr()), stream_ptr(stream)),
                "dispatch")

    def expert(self, params, rank=None, stream=None):
        N.check(N.load().mx_expert(self._plan, self._r(rank), C.byref(params),
                                   stream_ptr(stream)), "expert")

    def combine(self, y_out=None, rank=None, stream=None):
        N.check(N.load().mx_combine(self._plan, self._r(rank),
                                    C.c_void_p(y_out.data_ptr()) if y_out is not None else None,
                                    stream_ptr(stream)), "combine")

    def forward(self, x, params, logits=None, ids=None, weights=None,
                y_out=None, rank=None, stream=None):
        x = self._on_device(x, "x", self.dtype, self.hidden, False)
        logits, ids, weights = self._routing_inputs(logits, ids, weights)
        N.check(N.load().mx_forward(
            self._plan, self._r(rank), C.c_void_p(x.data_ptr()),
            C.c_void_p(logits.data_ptr()) if logits is not None else None,
            C.c_void_p(ids.data_ptr()) if ids is not None else None,
            C.c_void_p(weights.data_ptr()) if weights is not None else None,
            C.byref(params),
            C.c_void_p(y_out.data_ptr()) if y_out is not None else None,
            stream_ptr(stream)), "forward")

    def check(self, rank=None, stream=None):
        """Synchronize ``stream`` and raise the errors the device flagged
        since the last check: CapacityError (a host's routed slots exceed
        the capacity, sim:346-351), StrategyError (expert id out of range),
        NativeLibraryError (peer barrier watchdog)."""
        N.check(N.load().mx_plan_check(self._plan, self._r(rank), stream_ptr(stream)),
                "forward")

    # ------------------------------------------------------------ views
    def rank_views(self, rank):
        """Device views of one rank's routing/layout buffers."""
        T, k, E, n = self.tokens, self.top_k, self.num_experts, self.n
        return dict(
            ids=self.buffer(rank, N.MX_BUF_IDS, torch.int32, (T, k)),
            weights=self.buffer(rank, N.MX_BUF_WEIGHTS, self.wdtype, (T, k)),
            slot_pos=self.buffer(rank, N.MX_BUF_SLOT_POS, torch.int32, (T, k)),
            slot_tm=self.buffer(rank, N.MX_BUF_SLOT_TM, torch.int32, (T, k)),
            cnt_all=self.buffer(rank, N.MX_BUF_CNT_ALL, torch.int32, (n, E)),
            exp_off=self.buffer(rank, N.MX_BUF_EXP_OFF, torch.int32, (E,)),
            exp_cnt=self.buffer(rank, N.MX_BUF_EXP_CNT, torch.int32, (E,)),
            send=self.buffer(rank, N.MX_BUF_SEND, torch.int32, (n, n)),
        )

    def recv_view(self, rank):
        return self.buffer(rank, N.MX_BUF_RECV, self.dtype, (self.capacity, self.hidden))

    def partial_view(self, rank):
        return self.buffer(rank, N.MX_BUF_PARTIAL, self.dtype, (self.capacity, self.hidden))

    def y_view(self, rank):
        return self.buffer(rank, N.MX_BUF_Y, self.dtype, (self.tokens, self.hidden))
