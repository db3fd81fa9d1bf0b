"""The benched configurations at full size against the CPU oracle, and the
serving layer's error surfacing.  Runs on a B200 (``-m gpu``).

* config B exactly as ``bench.py`` runs it at N=1 (n=m=1, 8192 tokens,
  h=2048, I=768, 128 experts top-8, bf16): every output row of a token
  sample against ``orc.moe_layer_swiglu`` -- a token's output depends only on
  its own row and routing, so sampled rows compare one for one;
* config C's expert set (256 routed experts top-8 + the 2048-wide shared
  expert, h=7168, I=2048, fp8 e4m3, DeepSeek-V3 gate) against
  ``orc.moe_layer_fp8`` on a token sample, the replica's dequantised
  weights built per routed expert;
* a caller-set capacity below the routed rows raises CapacityError with the
  reference's message (sim:346-351) on both wires instead of returning y
  with dropped rows; routing tensors straight from ``torch.topk`` (int64)
  are accepted, a hidden state of the wrong dtype raises StrategyError.
"""
import numpy as np
import pytest
import torch

from oracle import mixserve_oracle as orc

pytestmark = pytest.mark.gpu

FP8_FRO, FP8_MAX = 1e-2, 5e-2   # as tests/test_gpu_parity.py (same replica)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    torch.cuda.set_device(0)


@pytest.mark.parametrize("wire", ["slot", "token"])
def test_config_b_bench_shape_vs_cpu_oracle(wire):
    from paper_2601_08800_b200 import SwiGLUExperts
    from paper_2601_08800_b200.layer import MoELayer
    T, h, E, k, I = 8192, 2048, 128, 8, 768
    ex = SwiGLUExperts.random(E, h, I, seed=0)
    w13, w2 = ex.rank_shard(1, 1, 0)
    layer = MoELayer(1, 1, T, h, E, k, I, w13=w13, w2=w2, rank=0, wire=wire)
    g = torch.Generator(device="cuda").manual_seed(1000)
    x = torch.randn(T, h, device="cuda", generator=g).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=g)
    y = layer.forward(x, logits).float().cpu().numpy()
    ids_all, _ = orc.router_topk(logits.cpu().numpy(), k)
    v = layer.plan.rank_views(0)
    assert np.array_equal(v["ids"].cpu().numpy(), ids_all)
    assert np.array_equal(v["exp_cnt"].cpu().numpy(),
                          np.bincount(ids_all.reshape(-1), minlength=E))
    sample = np.random.default_rng(5).choice(T, 1024, replace=False)
    sample.sort()
    oex = orc.SwiGLUOracle(ex.w_gate.float().cpu().numpy(), ex.w_up.float().cpu().numpy(),
                           ex.w_down.float().cpu().numpy())
    ids, w = orc.router_topk(logits.cpu().numpy()[sample], k)
    y_o = orc.moe_layer_swiglu(x.float().cpu().numpy()[sample], ids, w, oex)
    err = orc.verify_metric(y[sample], y_o)
    assert err <= 2e-2, err
    layer.close()


class _LazyShard:
    """[E, m=1, ...] dequantised expert weights for the fp8 replica, built
    on demand per routed expert (256 full-size experts dequantised at once
    would be 45 GB of host f32)."""

    def __init__(self, shards, which, It, h):
        self.shards, self.which, self.It, self.h = shards, which, It, h
        self.cache = {}
        E = shards["w13"].shape[0]
        self.shape = (E, 1, h, It) if which == "down" else (E, 1, It, h)

    def __getitem__(self, e):
        e = int(e)
        if e not in self.cache:
            p = self.shards
            if self.which == "down":
                a = (p["w2"][e].float() * p["w2_scale"][e][:, None]).cpu().numpy()
            else:
                w13 = (p["w13"][e].float() * p["w13_scale"][e][:, None]).cpu().numpy()
                blocks = w13.reshape(-1, 2, 64, self.h)   # 64-row gate/up interleave
                a = blocks[:, 0 if self.which == "gate" else 1].reshape(self.It, self.h)
            self.cache[e] = a[None]
        return self.cache[e]


def test_config_c_full_expert_set_vs_cpu_oracle():
    from paper_2601_08800_b200 import FP8SwiGLUExperts
    from paper_2601_08800_b200.layer import MoELayer
    from paper_2601_08800_b200.plan import GateSpec
    T, h, E, k, I, Is = 1024, 7168, 256, 8, 2048, 2048
    ex = FP8SwiGLUExperts.random(E, h, I, shared_inter=Is, seed=51)
    shards = ex.rank_shard(1, 1, 0)
    ex.src = None                          # bf16 sources no longer needed
    torch.cuda.empty_cache()
    gen = torch.Generator(device="cuda").manual_seed(52)
    x = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=gen)
    bias = (0.05 * torch.randn(E, generator=torch.Generator().manual_seed(53))).float()
    gate = GateSpec.deepseek_v3(bias, groups=8, topk_groups=4, scaling=2.5)
    layer = MoELayer(1, 1, T, h, E, k, I, experts=ex, rank=0, gate=gate)
    y = layer.forward(x, logits).double().cpu().numpy()
    ids, w = orc.router_group_limited(logits.cpu().numpy(), bias.numpy(), k, 8, 4, True, 2.5)
    assert np.array_equal(layer.plan.rank_views(0)["ids"].cpu().numpy(), ids)
    sample = np.arange(0, T, 64)           # 16 tokens, ~120 distinct experts
    shared = [(shards[nm].float() * shards[nm + "_scale"][:, None]).cpu().numpy()
              for nm in ("w13_shared", "w2_shared")]
    blocks = shared[0].reshape(-1, 2, 64, h)
    sh = [blocks[:, 0].reshape(-1, h)[None], blocks[:, 1].reshape(-1, h)[None], shared[1][None]]
    y_o = orc.moe_layer_fp8(x.float().cpu().numpy()[sample], ids[sample], w[sample],
                            _LazyShard(shards, "gate", I, h), _LazyShard(shards, "up", I, h),
                            _LazyShard(shards, "down", I, h), sh)
    got = y[sample]
    mx = orc.verify_metric(got, y_o)
    fro = float(np.linalg.norm(got - y_o) / np.linalg.norm(y_o))
    assert fro <= FP8_FRO and mx <= FP8_MAX, (fro, mx)
    layer.close()


@pytest.mark.parametrize("wire", ["slot", "token"])
def test_capacity_overflow_raises_in_serving_forward(wire):
    from paper_2601_08800_b200 import CapacityError, SwiGLUExperts
    from paper_2601_08800_b200.layer import MoELayer
    T, h, E, k, I = 256, 256, 16, 4, 256
    ex = SwiGLUExperts.random(E, h, I, seed=2)
    gen = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=gen)
    layer = MoELayer(1, 1, T, h, E, k, I, experts=ex, rank=0, wire=wire, capacity=T * k - 1)
    with pytest.raises(CapacityError, match=f"node 0 receives {T * k} routed slots, "
                                            f"capacity {T * k - 1}"):
        layer.forward(x, logits)
    layer.close()
    # exactly at capacity: fine, and the output matches an unconstrained layer
    ok = MoELayer(1, 1, T, h, E, k, I, experts=ex, rank=0, wire=wire, capacity=T * k)
    ref = MoELayer(1, 1, T, h, E, k, I, experts=ex, rank=0, wire=wire)
    assert torch.equal(ok.forward(x, logits).clone(), ref.forward(x, logits).clone())
    ok.close()
    ref.close()


def test_captured_forward_reports_capacity():
    from paper_2601_08800_b200 import CapacityError, SwiGLUExperts
    from paper_2601_08800_b200.layer import MoELayer
    T, h, E, k, I = 256, 256, 16, 4, 256
    ex = SwiGLUExperts.random(E, h, I, seed=2)
    x = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    logits = torch.zeros(T, E, device="cuda")
    layer = MoELayer(1, 1, T, h, E, k, I, experts=ex, rank=0, capacity=T * k)
    run = layer.capture(x, logits)
    run()
    run.check()                             # within capacity: no error
    layer.close()
    # capturing over capacity raises on the capture's eager warm-up forward
    layer = MoELayer(1, 1, T, h, E, k, I, experts=ex, rank=0, capacity=T * k - 8)
    with pytest.raises(CapacityError, match="capacity"):
        layer.capture(x, logits)
    layer.close()
    # a host of an emulated 2-group cluster over capacity (all tokens of both
    # groups routed to group 0's experts) -- the whole-cluster API raises too
    from paper_2601_08800_b200 import RouterSpec, build_cluster, fused_ag_dispatch
    xr = np.random.default_rng(0).standard_normal((2 * T, 64))
    skew = RouterSpec(E, tuple((0, 1) for _ in range(2 * T)),
                      tuple((0.5, 0.5) for _ in range(2 * T)))
    with pytest.raises(CapacityError, match="node 0 receives"):
        fused_ag_dispatch(build_cluster(2, 1), [xr[:T], xr[T:]], skew, capacity=T)


def test_routing_tensor_validation():
    from paper_2601_08800_b200 import StrategyError, SwiGLUExperts
    from paper_2601_08800_b200.layer import MoELayer
    T, h, E, k, I = 128, 256, 16, 4, 256
    ex = SwiGLUExperts.random(E, h, I, seed=7)
    gen = torch.Generator(device="cuda").manual_seed(8)
    x = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=gen)
    layer = MoELayer(1, 1, T, h, E, k, I, experts=ex, rank=0)
    y_gate = layer.forward(x, logits).clone()
    # ids from torch.topk are int64 and weights may come from the host
    w, ids = torch.softmax(logits, -1).topk(k, dim=-1)
    w = w / w.sum(-1, keepdim=True)
    y_ids = layer.forward(x, ids=ids, weights=w.cpu()).clone()
    assert orc.verify_metric(y_ids.float().cpu().numpy(), y_gate.float().cpu().numpy()) <= 2e-2
    with pytest.raises(StrategyError, match="dtype"):
        layer.forward(x.float(), logits)
    with pytest.raises(StrategyError, match="shape"):
        layer.forward(x[:-1], logits[:-1])
    with pytest.raises(StrategyError, match="exactly one"):
        layer.forward(x)
    # host output: the copy has landed when forward returns
    out = torch.empty(T, h, dtype=torch.bfloat16).pin_memory()
    layer.forward(x, logits, out=out)
    assert torch.equal(out, y_gate.cpu())
    layer.close()
