"""Parity of the CUDA path (through the C-ABI) against the CPU oracle and the
reference's frozen outputs.  Runs on a B200 (``-m gpu``)."""
import json

import numpy as np
import pytest
import torch

from conftest import golden_names, load_golden
from oracle import mixserve_oracle as orc

pytestmark = pytest.mark.gpu


def _meta(g):
    return json.loads(str(g["meta"]))


def _router(g):
    from paper_2601_08800_b200 import RouterSpec
    return RouterSpec.from_arrays(_meta(g)["E"], g["ids"], g["weights"])


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    torch.cuda.set_device(0)
    from paper_2601_08800_b200 import _native
    _native.load()


# ----------------------------------------------------------------- routing
@pytest.mark.parametrize("name", golden_names())
def test_routing_table_bit_exact(name):
    from paper_2601_08800_b200 import build_routing_table
    g = load_golden(name)
    mt = _meta(g)
    n = mt["n"]
    tab = build_routing_table(_router(g), n, mt["tokens"] // n)
    for d in range(n):
        assert np.array_equal(tab.token[d], g[f"tok_{d}"])
        assert np.array_equal(tab.expert[d], g[f"exp_{d}"])
        assert np.array_equal(tab.src[d], g[f"src_{d}"])
        assert np.array_equal(tab.weight[d], g[f"w_{d}"])
    ref = orc.Table(g["ids"], g["weights"], n, mt["tokens"] // n, mt["E"])
    assert np.array_equal(np.asarray(tab.send), ref.send_counts())
    assert tab.total_slots() == mt["tokens"] * g["ids"].shape[1]
    # reference Slot objects materialise identically
    s0 = tab.slots_by_host[0][:3]
    for i, s in enumerate(s0):
        assert (s.token, s.expert, s.src_node, s.host_node) == (
            int(g["tok_0"][i]), int(g["exp_0"][i]), int(g["src_0"][i]), 0)


@pytest.mark.parametrize("name", golden_names())
def test_expert_major_layout_bit_exact(name):
    """slot_pos reproduces concat(_expert_rows) (sim:528-532) exactly."""
    from paper_2601_08800_b200.simcluster import _plan, _route
    g = load_golden(name)
    mt = _meta(g)
    n, m, T = mt["n"], mt["m"], mt["tokens"] // mt["n"]
    router = _router(g)
    plan = _plan(n, m, T, mt["h"], mt["E"], g["ids"].shape[1], torch.float64)
    _route(plan, router)
    ref = orc.Table(g["ids"], g["weights"], n, T, mt["E"])
    for d in range(n):
        # table index of the slot stored at every expert-major row of host d
        S_d = ref.slots(d)
        at_row = np.full(S_d, -1)
        for grp in range(n):
            v = {k: t.cpu().numpy() for k, t in plan.rank_views(grp * m).items()}
            sel = (v["ids"].astype(np.int64) * n) // mt["E"] == d
            at_row[v["slot_pos"][sel]] = v["slot_tm"][sel]
        assert np.array_equal(at_row, g[f"emajor_{d}"])


# ----------------------------------------------------------------- layer
@pytest.mark.parametrize("name", golden_names())
def test_fused_layer_f64_bit_exact(name):
    from paper_2601_08800_b200 import (ExpertSpec, build_cluster, run_moe_block,
                                       verify_against_oracle)
    from paper_2601_08800_b200.trace import trace_to_csv
    g = load_golden(name)
    mt = _meta(g)
    cluster = build_cluster(mt["n"], mt["m"])
    router, experts = _router(g), ExpertSpec.default(mt["E"])
    y, trace = run_moe_block(cluster, g["x"], router, experts, mode="fused")
    assert np.array_equal(y, g["y_fused"])          # same association, f64
    assert trace_to_csv(trace.events) == str(g["trace_csv"])
    assert verify_against_oracle(y, g["x"], router, experts) <= 1e-9


@pytest.mark.parametrize("name", golden_names())
def test_baseline_layer_matches_reference(name):
    from paper_2601_08800_b200 import ExpertSpec, build_cluster, run_moe_block
    from paper_2601_08800_b200.trace import trace_to_csv
    g = load_golden(name)
    mt = _meta(g)
    y, trace = run_moe_block(build_cluster(mt["n"], mt["m"]), g["x"], _router(g),
                             ExpertSpec.default(mt["E"]), mode="baseline")
    assert np.allclose(y, g["y_baseline"], rtol=1e-9, atol=1e-12)
    assert trace_to_csv(trace.events) == str(g["trace_baseline_csv"])


@pytest.mark.parametrize("name", golden_names())
def test_dense_gpu_oracle_bit_exact(name):
    from paper_2601_08800_b200 import ExpertSpec, moe_oracle
    g = load_golden(name)
    y = moe_oracle(g["x"], _router(g), ExpertSpec.default(_meta(g)["E"]))
    assert np.array_equal(y, g["y_oracle"])


def test_dispatch_received_rows_bit_exact():
    from paper_2601_08800_b200 import build_cluster, fused_ag_dispatch
    g = load_golden("ref_grid_07")
    mt = _meta(g)
    n, m, T = mt["n"], mt["m"], mt["tokens"] // mt["n"]
    xs = [g["x"][j * T:(j + 1) * T] for j in range(n)]
    received, table, trace = fused_ag_dispatch(build_cluster(n, m), xs, _router(g))
    ref = orc.Table(g["ids"], g["weights"], n, T, mt["E"])
    want = orc.dispatch_received(xs, ref)
    for d in range(n):
        assert np.array_equal(received[d], want[d])


def test_rs_combine_from_oracle_partials():
    from paper_2601_08800_b200 import build_cluster, fused_rs_combine
    from paper_2601_08800_b200.simcluster import build_routing_table
    g = load_golden("ref_grid_05")
    mt = _meta(g)
    n, m, T, h, E = mt["n"], mt["m"], mt["tokens"] // mt["n"], mt["h"], mt["E"]
    ref = orc.Table(g["ids"], g["weights"], n, T, E)
    xs = [g["x"][j * T:(j + 1) * T] for j in range(n)]
    parts = orc.partial_affine(orc.dispatch_received(xs, ref), ref,
                               [e + 1.0 for e in range(E)], [float(e) for e in range(E)],
                               m, h)
    table = build_routing_table(_router(g), n, T)
    ys, _ = fused_rs_combine(build_cluster(n, m), parts, table)
    assert np.array_equal(np.concatenate(ys), g["y_fused"])


@pytest.mark.parametrize("mode", ["fused", "baseline"])
def test_empty_batch_matches_reference(mode):
    """Zero tokens: the reference returns an empty output and its zero-byte
    event schedule; same shape, byte-identical trace (frozen by
    tests/golden/make_golden.py)."""
    from conftest import GOLDEN
    from paper_2601_08800_b200 import ExpertSpec, RouterSpec, build_cluster, run_moe_block
    from paper_2601_08800_b200.trace import trace_to_csv
    x = np.zeros((0, 8))
    y, tr = run_moe_block(build_cluster(2, 2), x, RouterSpec(4, (), ()), ExpertSpec.default(4),
                          mode=mode)
    assert y.shape == (0, 8)
    assert trace_to_csv(tr.events) == (GOLDEN / f"trace_empty_2x2_{mode}.csv").read_text()


def test_verify_detects_corrupted_output():
    """verify_against_oracle raises VerificationError on a perturbed output
    (T/test_simcluster.py: corrupted output detected)."""
    from paper_2601_08800_b200 import (ExpertSpec, RouterSpec, VerificationError,
                                       build_cluster, run_moe_block, verify_against_oracle)
    x = np.arange(32.0).reshape(4, 8)
    router = RouterSpec.round_robin(4, 2, 1)
    y, _ = run_moe_block(build_cluster(2, 2), x, router, ExpertSpec.default(2))
    assert verify_against_oracle(y, x, router, ExpertSpec.default(2)) == 0.0
    y2 = y.copy()
    y2[0, 0] += 1.0
    with pytest.raises(VerificationError):
        verify_against_oracle(y2, x, router, ExpertSpec.default(2))


def test_expert_permutation_safety_and_determinism():
    """Relabelling the experts consistently in router and experts leaves the
    layer output unchanged (T/test_simcluster.py:232-251, rtol 1e-9); two
    runs are byte-identical, trace included (:225-229)."""
    from paper_2601_08800_b200 import ExpertSpec, RouterSpec, build_cluster, run_moe_block
    from paper_2601_08800_b200.trace import trace_to_csv
    rng = np.random.default_rng(17)
    n, m, T, k, E = 2, 2, 8, 2, 4
    x = rng.standard_normal((n * T, 16))
    router = RouterSpec.random(n * T, E, k, seed=17)
    experts = ExpertSpec(tuple(rng.standard_normal(E).tolist()), tuple(rng.standard_normal(E).tolist()))
    perm = [2, 0, 3, 1]
    prouter = RouterSpec(
        E, tuple(tuple(sorted(perm[e] for e in ids)) for ids in router.expert_ids),
        tuple(tuple(w for _, w in sorted((perm[e], w) for e, w in zip(ids, ws)))
              for ids, ws in zip(router.expert_ids, router.weights)))
    inv = [perm.index(e) for e in range(E)]
    pexperts = ExpertSpec(tuple(experts.scales[inv[e]] for e in range(E)),
                          tuple(experts.biases[inv[e]] for e in range(E)))
    cl = build_cluster(n, m)
    y1, t1 = run_moe_block(cl, x, router, experts)
    y1b, t1b = run_moe_block(cl, x, router, experts)
    y2, _ = run_moe_block(cl, x, prouter, pexperts)
    assert np.array_equal(y1, y1b)
    assert trace_to_csv(t1.events) == trace_to_csv(t1b.events)
    assert np.allclose(y1, y2, rtol=1e-9, atol=1e-12)


def test_randomized_shapes_f64_bit_exact():
    """Seeded random clusters and shapes (the reference's hypothesis
    equivalence test, T/test_simcluster.py:216-252): the fused f64 layer is
    bit-identical to the oracle's restatement of the reference value path."""
    from paper_2601_08800_b200 import ExpertSpec, RouterSpec, build_cluster, run_moe_block
    rng = np.random.default_rng(2026)
    for _ in range(12):
        n, m = int(rng.integers(1, 5)), int(rng.integers(1, 4))
        E = int(rng.integers(n, 3 * n + 6))
        k = int(rng.integers(1, min(E, 6) + 1))
        T = int(rng.integers(1, 40))
        h = int(rng.integers(m, 48))
        x = rng.standard_normal((n * T, h))
        router = RouterSpec.random(n * T, E, k, seed=int(rng.integers(1 << 30)))
        experts = ExpertSpec(tuple(rng.standard_normal(E).tolist()),
                             tuple(rng.standard_normal(E).tolist()))
        y, _ = run_moe_block(build_cluster(n, m), x, router, experts)
        ids, w = router.arrays()
        y_ref, _ = orc.run_fused_affine(n, m, x, ids, w, E, experts.scales, experts.biases)
        assert np.array_equal(y, y_ref), (n, m, E, k, T, h)


def test_partial_shape_mismatch_raises():
    """fused_rs_combine rejects partials of the wrong shape (sim:421-429;
    T/test_simcluster.py:200-206)."""
    from paper_2601_08800_b200 import (RouterSpec, StrategyError, build_cluster,
                                       build_routing_table, fused_rs_combine)
    cluster = build_cluster(2, 2)
    table = build_routing_table(RouterSpec.round_robin(4, 4, 1), 2, 2)
    bad = [[np.zeros((1, 8)), np.zeros((1, 8))] for _ in range(2)]
    with pytest.raises(StrategyError, match="mismatch"):
        fused_rs_combine(cluster, bad, table)


def test_capacity_error():
    from paper_2601_08800_b200 import (CapacityError, RouterSpec, build_cluster,
                                       fused_ag_dispatch)
    x = np.random.default_rng(0).standard_normal((8, 8))
    skew = RouterSpec(4, tuple((0,) for _ in range(8)), tuple((1.0,) for _ in range(8)))
    with pytest.raises(CapacityError, match="capacity"):
        fused_ag_dispatch(build_cluster(2, 2), [x[:4], x[4:]], skew, capacity=4)


def test_uneven_tokens_raise_strategy_error():
    from paper_2601_08800_b200 import (ExpertSpec, RouterSpec, StrategyError,
                                       build_cluster, run_moe_block)
    x = np.zeros((3, 8))
    with pytest.raises(StrategyError, match="split evenly"):
        run_moe_block(build_cluster(2, 1), x, RouterSpec.round_robin(3, 2, 1),
                      ExpertSpec.default(2))


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
@pytest.mark.parametrize("shape", [(1, 1), (2, 2), (4, 2), (2, 4)])
def test_fused_layer_low_precision(dtype, tol, shape):
    from paper_2601_08800_b200 import ExpertSpec, build_cluster, run_moe_block
    n, m = shape
    g = load_golden("ref_config_a") if shape == (2, 2) else None
    rng = np.random.default_rng(11)
    T_g, h, E, k = 64 * n, 128, 16, 4
    x = rng.standard_normal((T_g, h)) if g is None else g["x"]
    from paper_2601_08800_b200 import RouterSpec
    router = RouterSpec.random(x.shape[0], E, k, seed=3) if g is None else _router(g)
    E = router.num_experts
    experts = ExpertSpec.default(E)
    xt = torch.as_tensor(x).to(dtype).cuda()
    y, _ = run_moe_block(build_cluster(n, m), xt, router, experts)
    ids, w = router.arrays()
    xr = xt.double().cpu().numpy()
    y_ref = orc.dense_oracle(xr, ids, w, orc.affine_apply(experts.scales, experts.biases))
    y = y.double().cpu().numpy()
    if dtype is torch.bfloat16:
        # bf16 stores the TP partials scale_e*x + bias_e/m (|.| up to ~4E):
        # tolerance is relative to the output scale, max|y-e| / max|e|
        assert np.max(np.abs(y - y_ref)) / max(np.max(np.abs(y_ref)), 1.0) <= tol
    else:
        assert orc.verify_metric(y, y_ref) <= tol


# ----------------------------------------------------------------- router
@pytest.mark.parametrize("T,E,k,renorm", [(64, 16, 4, True), (300, 128, 8, True),
                                          (257, 256, 8, False), (128, 60, 6, True),
                                          (1000, 1024, 8, True), (5, 8, 8, True)])
def test_router_topk_bit_exact(T, E, k, renorm):
    from paper_2601_08800_b200.plan import LayerPlan
    rng = np.random.default_rng(T + E)
    logits = rng.standard_normal((T, E)).astype(np.float32)
    logits[0, :] = 0.5                       # all-equal row: ids 0..k-1
    if T > 3:
        logits[3, 1] = logits[3, E - 1] = 9.0  # exact tie -> lowest id first
    ids_ref, w_ref = orc.router_topk(logits, k, renormalize=renorm)
    plan = LayerPlan(1, 1, T, 8, E, k, dtype=torch.float32, renormalize=renorm)
    plan.route(logits=torch.as_tensor(logits).cuda())
    plan.layout(check_capacity=True)
    v = plan.rank_views(0)
    assert np.array_equal(v["ids"].cpu().numpy(), ids_ref)
    np.testing.assert_allclose(v["weights"].cpu().numpy(), w_ref, rtol=2e-6, atol=1e-7)
    counts = np.bincount(ids_ref.reshape(-1), minlength=E)
    assert np.array_equal(v["cnt_all"].cpu().numpy()[0], counts)
    assert np.array_equal(v["exp_cnt"].cpu().numpy(), counts)
    plan.close()


@pytest.mark.parametrize("name", ["r1", "small", "negbias"])
def test_group_limited_router_bit_exact(name):
    """DeepSeek-V3 gate kernel vs the oracle restatement (itself pinned to
    transformers): ids bit-exact, weights bit-exact (same fp32 op order)."""
    from paper_2601_08800_b200.plan import GateSpec, LayerPlan
    z = np.load(__import__("conftest").GOLDEN / "deepseek_router.npz")
    T, E, k, ng, tg, norm = (int(x) for x in z[f"{name}_cfg"])
    sc = float(z[f"{name}_scaling"][0])
    logits, bias = z[f"{name}_logits"], z[f"{name}_bias"]
    ids_ref, w_ref = orc.router_group_limited(logits, bias, k, ng, tg, bool(norm), sc)
    gate = GateSpec("group_limited", ng, tg, sc, torch.as_tensor(bias))
    plan = LayerPlan(1, 1, T, 8, E, k, dtype=torch.float32, renormalize=bool(norm), gate=gate)
    plan.route(logits=torch.as_tensor(logits).cuda())
    plan.layout(check_capacity=True)
    v = plan.rank_views(0)
    assert np.array_equal(v["ids"].cpu().numpy(), ids_ref)
    assert np.array_equal(v["weights"].cpu().numpy(), w_ref)
    counts = np.bincount(ids_ref.reshape(-1), minlength=E)
    assert np.array_equal(v["exp_cnt"].cpu().numpy(), counts)
    plan.close()


def test_group_limited_router_deepseek_shape_random():
    """R1 shape (256 experts, 8 groups keep 4, top-8, scaling 2.5) on 4096
    tokens with a tie row and an all-equal row."""
    from paper_2601_08800_b200.plan import GateSpec, LayerPlan
    rng = np.random.default_rng(5)
    T, E, k = 4096, 256, 8
    logits = rng.standard_normal((T, E)).astype(np.float32)
    logits[0, :] = 0.25
    logits[1, 7] = logits[1, 200] = 6.0
    bias = (0.02 * rng.standard_normal(E)).astype(np.float32)
    ids_ref, w_ref = orc.router_group_limited(logits, bias, k, 8, 4, True, 2.5)
    plan = LayerPlan(1, 1, T, 8, E, k, dtype=torch.float32,
                     gate=GateSpec.deepseek_v3(torch.as_tensor(bias)))
    plan.route(logits=torch.as_tensor(logits).cuda())
    v = plan.rank_views(0)
    assert np.array_equal(v["ids"].cpu().numpy(), ids_ref)
    assert np.array_equal(v["weights"].cpu().numpy(), w_ref)
    plan.close()


def test_router_topk_feeds_layer_2x2():
    """Gate -> table on a 2x2 cluster equals the reference fed by our gate."""
    from paper_2601_08800_b200 import build_routing_table
    z = np.load(__import__("conftest").GOLDEN / "router_topk_logits.npz")
    g = load_golden("ref_router_topk")
    tab = build_routing_table(_router(g), 2, 32)
    for d in range(2):
        assert np.array_equal(tab.token[d], g[f"tok_{d}"])
        assert np.array_equal(tab.expert[d], g[f"exp_{d}"])
    assert np.array_equal(g["ids"], z["ids"].astype(np.int64))


# ----------------------------------------------------------------- GEMM
@pytest.mark.parametrize("G,N,K,out", [(4, 256, 128, "bf16"), (3, 128, 192, "f32"),
                                       (8, 512, 2048, "bf16"), (5, 768, 384, "f32")])
def test_grouped_gemm_vs_torch_fp32(G, N, K, out):
    from paper_2601_08800_b200 import _native
    gen = torch.Generator(device="cuda").manual_seed(G * N + K)
    cnts = torch.tensor([0, 1, 127, 128, 129, 300, 5, 256][:G], dtype=torch.int32)
    offs = torch.zeros(G, dtype=torch.int32)
    offs[1:] = torch.cumsum(cnts, 0)[:-1]
    M = int(cnts.sum())
    A = torch.randn(M + 64, K, device="cuda", generator=gen).to(torch.bfloat16)
    B = (torch.randn(G, N, K, device="cuda", generator=gen) / K ** 0.5).to(torch.bfloat16)
    dt = torch.bfloat16 if out == "bf16" else torch.float32
    D = torch.full((M + 64, N), 7.0, device="cuda", dtype=dt)
    offs_d, cnts_d = offs.cuda(), cnts.cuda()   # keep alive across the launch
    _native.call("mx_grouped_gemm", A.data_ptr(), B.data_ptr(), D.data_ptr(),
                 _native.MX_BF16 if out == "bf16" else _native.MX_F32,
                 offs_d.data_ptr(), cnts_d.data_ptr(), G, M, N, K, 0,
                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for g in range(G):
        o, c = int(offs[g]), int(cnts[g])
        ref = A[o:o + c].float() @ B[g].float().T
        got = D[o:o + c].float()
        tol = 2e-2 if out == "bf16" else 1e-3
        assert torch.allclose(got, ref, rtol=tol, atol=tol), (g, (got - ref).abs().max())
    assert torch.all(D[M:].float() == 7.0)   # rows past the groups untouched


@pytest.mark.parametrize("counts", [(130, 0, 64), (5, 0, 9)])  # 256- and 128-wide tiles
def test_grouped_gemm_swiglu_epilogue(counts):
    from paper_2601_08800_b200 import _native
    G, I, K = 3, 256, 256
    gen = torch.Generator(device="cuda").manual_seed(1)
    cnts = torch.tensor(counts, dtype=torch.int32)
    offs = torch.zeros(G, dtype=torch.int32)
    offs[1:] = torch.cumsum(cnts, 0)[:-1]
    M = int(cnts.sum())
    A = torch.randn(M, K, device="cuda", generator=gen).to(torch.bfloat16)
    wg = (torch.randn(G, I, K, device="cuda", generator=gen) / 16).to(torch.bfloat16)
    wu = (torch.randn(G, I, K, device="cuda", generator=gen) / 16).to(torch.bfloat16)
    w13 = torch.empty(G, 2 * I, K, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    _native.call("mx_swiglu_pack_w13", wg.data_ptr(), wu.data_ptr(), w13.data_ptr(), G, I, K, s)
    D = torch.zeros(M, I, device="cuda", dtype=torch.bfloat16)
    offs_d, cnts_d = offs.cuda(), cnts.cuda()
    _native.call("mx_grouped_gemm", A.data_ptr(), w13.data_ptr(), D.data_ptr(), _native.MX_BF16,
                 offs_d.data_ptr(), cnts_d.data_ptr(), G, M, 2 * I, K, 1, s)
    torch.cuda.synchronize()
    for g in range(G):
        o, c = int(offs[g]), int(cnts[g])
        gate = A[o:o + c].float() @ wg[g].float().T
        up = A[o:o + c].float() @ wu[g].float().T
        ref = torch.nn.functional.silu(gate) * up
        assert torch.allclose(D[o:o + c].float(), ref, rtol=2e-2, atol=2e-2)


# ----------------------------------------------------------------- SwiGLU layer
@pytest.mark.parametrize("shape", [(1, 1), (2, 2), (4, 2), (2, 4), (1, 2)])
def test_swiglu_layer_vs_oracle(shape):
    from paper_2601_08800_b200 import (RouterSpec, SwiGLUExperts, build_cluster,
                                       moe_oracle, run_moe_block)
    n, m = shape
    E, h, I, T_g, k = 16, 256, 512, 96 * n, 4
    ex = SwiGLUExperts.random(E, h, I, seed=n * 10 + m)
    x = torch.randn(T_g, h, device="cuda").to(torch.bfloat16)
    router = RouterSpec.random(T_g, E, k, seed=5)
    y, _ = run_moe_block(build_cluster(n, m), x, router, ex)
    oex = orc.SwiGLUOracle(ex.w_gate.float().cpu().numpy(), ex.w_up.float().cpu().numpy(),
                           ex.w_down.float().cpu().numpy())
    ids, w = router.arrays()
    y_o = orc.moe_layer_swiglu(x.float().cpu().numpy(), ids, w, oex)
    assert orc.verify_metric(y.float().cpu().numpy(), y_o) <= 2e-2
    # the package's own dense GPU oracle agrees with the CPU one
    y_d = moe_oracle(x, router, ex)
    assert orc.verify_metric(y_d.double().cpu().numpy(), y_o) <= 1e-3


# ----------------------------------------------------------------- SPMD layer, 1 GPU
def test_layer_graph_replay_matches_eager_and_oracle():
    from paper_2601_08800_b200 import SwiGLUExperts
    from paper_2601_08800_b200.layer import MoELayer
    T, h, E, k, I = 512, 256, 32, 4, 256
    ex = SwiGLUExperts.random(E, h, I, seed=9)
    layer = MoELayer(1, 1, T, h, E, k, I, experts=ex, rank=0)
    gen = torch.Generator(device="cuda").manual_seed(2)
    x = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=gen)
    y_eager = layer.forward(x, logits).clone()
    run = layer.capture(x, logits, with_events=True)
    for _ in range(3):
        y_g = run().clone()
    torch.cuda.synchronize()
    assert torch.equal(y_g, y_eager)
    assert [n for n, _ in run.phase_ms()][0] == "route"
    # new tokens copied into the captured buffers
    x.copy_(torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16))
    y2 = run().clone()
    oex = orc.SwiGLUOracle(ex.w_gate.float().cpu().numpy(), ex.w_up.float().cpu().numpy(),
                           ex.w_down.float().cpu().numpy())
    ids, w = orc.router_topk(logits.cpu().numpy(), k)
    y_o = orc.moe_layer_swiglu(x.float().cpu().numpy(), ids, w, oex)
    assert orc.verify_metric(y2.float().cpu().numpy(), y_o) <= 2e-2
    layer.close()


@pytest.mark.parametrize("wire", ["slot", "token"])
def test_gathered_gemm1_equals_copied_rows(wire, monkeypatch):
    """GEMM1 gathering A rows through the row table (LDGSTS producer) gives
    the same bits as the materialised expert-major copy (MX_GATHER=0, the
    default)."""
    from paper_2601_08800_b200 import SwiGLUExperts
    from paper_2601_08800_b200.layer import MoELayer
    T, h, E, k, I = 1000, 512, 16, 4, 256
    ex = SwiGLUExperts.random(E, h, I, seed=4)
    gen = torch.Generator(device="cuda").manual_seed(6)
    x = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=gen)
    outs = {}
    for g in ("0", "1", "4"):  # copy, LDGSTS gather, TMA tile::gather4
        monkeypatch.setenv("MX_GATHER", "0" if g == "0" else "1")
        monkeypatch.setenv("MX_GATHER4", "1" if g == "4" else "0")
        layer = MoELayer(1, 1, T, h, E, k, I, experts=ex, rank=0, wire=wire)
        outs[g] = layer.forward(x, logits).clone()
        layer.close()
    assert torch.equal(outs["0"], outs["1"])
    assert torch.equal(outs["0"], outs["4"])
    oex = orc.SwiGLUOracle(ex.w_gate.float().cpu().numpy(), ex.w_up.float().cpu().numpy(),
                           ex.w_down.float().cpu().numpy())
    ids, w = orc.router_topk(logits.cpu().numpy(), k)
    y_o = orc.moe_layer_swiglu(x.float().cpu().numpy(), ids, w, oex)
    assert orc.verify_metric(outs["1"].float().cpu().numpy(), y_o) <= 2e-2


def test_measured_phases_and_stamped_trace():
    """Device-clock stamps bracket every phase in order; the stamped trace
    carries the reference's events with spans inside the measured run."""
    from paper_2601_08800_b200 import SwiGLUExperts
    from paper_2601_08800_b200.layer import MoELayer
    from paper_2601_08800_b200.measured import layer_trace, measure_phases, stamp_trace
    T, h, E, k, I = 512, 256, 32, 4, 256
    ex = SwiGLUExperts.random(E, h, I, seed=9)
    for wire in ("slot", "token"):
        layer = MoELayer(1, 1, T, h, E, k, I, experts=ex, rank=0, wire=wire)
        gen = torch.Generator(device="cuda").manual_seed(2)
        x = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
        logits = torch.randn(T, E, device="cuda", generator=gen)
        layer.forward(x, logits)
        ph = measure_phases(layer, x, logits, iters=3)
        names = layer.phase_names()[1:]
        assert list(ph) == names
        prev = 0.0
        for nm in names:
            a, b = ph[nm]
            assert prev <= a + 1e-12 and a <= b
            prev = b
        assert ph["gemm1_swiglu"][1] - ph["gemm1_swiglu"][0] > 0
        events, stages = layer_trace(layer)
        text = stamp_trace(events, stages, [ph], wire)
        assert text.count("expert_compute") == sum(1 for e in events if e.op == "expert_compute")
        layer.close()


# ----------------------------------------------------------------- wire TOKEN
@pytest.mark.parametrize("shape", [(1, 1), (2, 1), (2, 2), (4, 2), (2, 4), (8, 1), (4, 4)])
def test_wire_token_f64_affine_emulated(shape):
    """Dedup dispatch + pre-reduced combine: same outputs as the reference
    layer up to f64 association (weights folded before the TP sum)."""
    from paper_2601_08800_b200 import RouterSpec, _native as N
    from paper_2601_08800_b200.plan import LayerPlan
    n, m = shape
    T, h, E, k = 40, 64, 16, 4
    rng = np.random.default_rng(n * 7 + m)
    x = rng.standard_normal((n * T, h))
    router = RouterSpec.random(n * T, E, k, seed=n + m)
    ids, w = router.arrays()
    sc, bi = np.arange(1, E + 1, dtype=np.float64), np.arange(E, dtype=np.float64)
    plan = LayerPlan(n, m, T, h, E, k, dtype=torch.float64, wire="token")
    sct, bit = torch.as_tensor(sc).cuda(), torch.as_tensor(bi).cuda()
    params = N.ExpertParams(sct.data_ptr(), bit.data_ptr(), None, None)
    y = torch.empty(n * T, h, dtype=torch.float64, device="cuda")
    xt = torch.as_tensor(x).cuda()
    plan.forward(xt, params, ids=torch.as_tensor(ids).cuda(), weights=torch.as_tensor(w).cuda(),
                 y_out=y)
    y_ref, _ = orc.run_fused_affine(n, m, x, ids, w, E, sc, bi)
    assert orc.verify_metric(y.cpu().numpy(), y_ref) <= 1e-12
    plan.close()


@pytest.mark.parametrize("shape", [(2, 2), (4, 2), (2, 4)])
def test_wire_token_swiglu_emulated(shape):
    from paper_2601_08800_b200 import SwiGLUExperts, _native as N
    from paper_2601_08800_b200.plan import LayerPlan
    n, m = shape
    T, h, E, k, I = 64, 256, 16, 4, 512
    ex = SwiGLUExperts.random(E, h, I, seed=4)
    w13, w2 = ex.stacked_shards(n, m)
    gen = torch.Generator(device="cuda").manual_seed(8)
    x = torch.randn(n * T, h, device="cuda", generator=gen).to(torch.bfloat16)
    logits = torch.randn(n * T, E, device="cuda", generator=gen)
    plan = LayerPlan(n, m, T, h, E, k, dtype=torch.bfloat16, expert_kind="swiglu", inter=I,
                     wire="token")
    y = torch.empty(n * T, h, dtype=torch.bfloat16, device="cuda")
    plan.forward(x, N.ExpertParams(None, None, w13.data_ptr(), w2.data_ptr()), logits=logits,
                 y_out=y)
    oex = orc.SwiGLUOracle(ex.w_gate.float().cpu().numpy(), ex.w_up.float().cpu().numpy(),
                           ex.w_down.float().cpu().numpy())
    ids, w = orc.router_topk(logits.cpu().numpy(), k)
    y_o = orc.moe_layer_swiglu(x.float().cpu().numpy(), ids, w, oex)
    assert orc.verify_metric(y.float().cpu().numpy(), y_o) <= 2e-2
    plan.close()


@pytest.mark.parametrize("shape,k,E,hot,T", [((2, 2), 4, 16, False, 2560),
                                             ((4, 1), 12, 48, True, 1280),
                                             ((2, 2), 12, 16, False, 2560),
                                             ((1, 2), 12, 16, False, 96)])
def test_wire_token_pair_reduce_slot_counts(shape, k, E, hot, T):
    """Both pre-reductions: the bulk-copy ring for many short pairs (k <= 4n
    and T*n >= 148*32; it stages pairs of at most 8 slots and reads longer
    ones straight from HBM -- ``hot`` routes half the tokens to all 12
    experts of host 0) and the register kernel for long pairs (k > 4n) or
    small batches."""
    from paper_2601_08800_b200 import SwiGLUExperts, _native as N
    from paper_2601_08800_b200.plan import LayerPlan
    n, m = shape
    h, I = 256, 256
    ex = SwiGLUExperts.random(E, h, I, seed=5)
    w13, w2 = ex.stacked_shards(n, m)
    gen = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(n * T, h, device="cuda", generator=gen).to(torch.bfloat16)
    logits = torch.randn(n * T, E, device="cuda", generator=gen)
    if hot:
        logits[: n * T // 2, : E // n] += 8.0
    plan = LayerPlan(n, m, T, h, E, k, dtype=torch.bfloat16, expert_kind="swiglu", inter=I,
                     wire="token")
    y = torch.empty(n * T, h, dtype=torch.bfloat16, device="cuda")
    plan.forward(x, N.ExpertParams(None, None, w13.data_ptr(), w2.data_ptr()), logits=logits,
                 y_out=y)
    oex = orc.SwiGLUOracle(ex.w_gate.float().cpu().numpy(), ex.w_up.float().cpu().numpy(),
                           ex.w_down.float().cpu().numpy())
    ids, w = orc.router_topk(logits.cpu().numpy(), k)
    if hot:
        on0 = ((ids * n) // E == 0).sum(axis=1)
        assert on0.max() > 8  # some pairs exceed the staged 8 slots
    y_o = orc.moe_layer_swiglu(x.float().cpu().numpy(), ids, w, oex)
    assert orc.verify_metric(y.float().cpu().numpy(), y_o) <= 2e-2
    plan.close()


@pytest.mark.parametrize("shape,T", [((2, 2), 48), ((4, 1), 1280)])
def test_wire_token_f32_affine_emulated(shape, T):
    """f32 rows through both pre-reductions (affine experts; the bulk-copy
    ring at 4 x 1280 tokens): within f32 association of the reference."""
    from paper_2601_08800_b200 import RouterSpec, _native as N
    from paper_2601_08800_b200.plan import LayerPlan
    n, m = shape
    h, E, k = 64, 16, 4
    rng = np.random.default_rng(n * 5 + m)
    x = rng.standard_normal((n * T, h)).astype(np.float32)
    router = RouterSpec.random(n * T, E, k, seed=n * 3 + m)
    ids, w = router.arrays()
    sc = np.linspace(0.5, 1.5, E).astype(np.float32)
    bi = np.linspace(-0.1, 0.1, E).astype(np.float32)
    plan = LayerPlan(n, m, T, h, E, k, dtype=torch.float32, wire="token")
    sct, bit = torch.as_tensor(sc).cuda(), torch.as_tensor(bi).cuda()
    params = N.ExpertParams(sct.data_ptr(), bit.data_ptr(), None, None)
    y = torch.empty(n * T, h, dtype=torch.float32, device="cuda")
    plan.forward(torch.as_tensor(x).cuda(), params, ids=torch.as_tensor(ids).cuda(),
                 weights=torch.as_tensor(w.astype(np.float32)).cuda(), y_out=y)
    y_ref, _ = orc.run_fused_affine(n, m, x.astype(np.float64), ids, w, E,
                                    sc.astype(np.float64), bi.astype(np.float64))
    assert orc.verify_metric(y.cpu().numpy().astype(np.float64), y_ref) <= 1e-5
    plan.close()


@pytest.mark.parametrize("s_zipf,wire", [(1.2, "token"), (1.2, "slot"), (0.8, "token")])
def test_zipf_skew_layer_emulated(s_zipf, wire):
    """Config E on the emulated 4x2 cluster: Zipf-skewed gate logits, the
    hot host receives far more than its share; routing counts bit-exact and
    the layer within the bf16 tolerance of the oracle."""
    from paper_2601_08800_b200 import SwiGLUExperts, _native as N
    from paper_2601_08800_b200.plan import LayerPlan
    from paper_2601_08800_b200.skew import host_skew, zipf_logits
    n, m = 4, 2
    T, h, E, k, I = 128, 256, 32, 4, 256
    ex = SwiGLUExperts.random(E, h, I, seed=12)
    w13, w2 = ex.stacked_shards(n, m)
    gen = torch.Generator(device="cuda").manual_seed(21)
    x = torch.randn(n * T, h, device="cuda", generator=gen).to(torch.bfloat16)
    logits = zipf_logits(n * T, E, s_zipf, seed=3, device="cuda", generator=gen)
    plan = LayerPlan(n, m, T, h, E, k, dtype=torch.bfloat16, expert_kind="swiglu", inter=I,
                     wire=wire)
    y = torch.empty(n * T, h, dtype=torch.bfloat16, device="cuda")
    plan.forward(x, N.ExpertParams(None, None, w13.data_ptr(), w2.data_ptr()), logits=logits,
                 y_out=y)
    ids, w = orc.router_topk(logits.cpu().numpy(), k)
    counts = np.bincount(ids.reshape(-1), minlength=E)
    assert host_skew(counts, n) > 1.2
    v = plan.rank_views(0)
    assert np.array_equal(v["exp_cnt"].cpu().numpy(), counts)
    oex = orc.SwiGLUOracle(ex.w_gate.float().cpu().numpy(), ex.w_up.float().cpu().numpy(),
                           ex.w_down.float().cpu().numpy())
    y_o = orc.moe_layer_swiglu(x.float().cpu().numpy(), ids, w, oex)
    assert orc.verify_metric(y.float().cpu().numpy(), y_o) <= 2e-2
    plan.close()


# ----------------------------------------------------------------- fp8 (config C)
def test_quant_rows_e4m3_bit_exact():
    from paper_2601_08800_b200 import _native
    R, Cc = 300, 1792
    gen = torch.Generator(device="cuda").manual_seed(3)
    x = (torch.randn(R, Cc, device="cuda", generator=gen) * 3).to(torch.bfloat16)
    x[5] = 0
    x[7, 11] = 1e4
    ld = Cc + 16
    q = torch.zeros(R, ld, dtype=torch.uint8, device="cuda")
    _native.call("mx_quant_rows_e4m3", x.data_ptr(), Cc, q.data_ptr(), ld, R, Cc,
                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    vals = q[:, :Cc].contiguous().view(torch.float8_e4m3fn).float().cpu().numpy()
    scales = q[:, Cc:Cc + 4].contiguous().view(torch.float32)[:, 0].cpu().numpy()
    q_ref, s_ref = orc.quant_rows_e4m3(x.float().cpu().numpy())
    assert np.array_equal(scales, s_ref)
    assert np.array_equal(vals, q_ref)


@pytest.mark.parametrize("swiglu", [False, True])
def test_grouped_gemm_fp8_vs_dequantized_torch(swiglu):
    from paper_2601_08800_b200 import _native
    G, N, K = 3, 512, 1024
    gen = torch.Generator(device="cuda").manual_seed(5)
    cnts = torch.tensor([200, 0, 77], dtype=torch.int32)
    offs = torch.tensor([0, 200, 200], dtype=torch.int32)
    M = 277
    a32 = torch.randn(M, K, device="cuda", generator=gen)
    lda = K + 16
    A = torch.zeros(M, lda, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    a16 = a32.to(torch.bfloat16)
    _native.call("mx_quant_rows_e4m3", a16.data_ptr(), K, A.data_ptr(), lda, M, K, s)
    w = torch.randn(G, N, K, device="cuda", generator=gen) / K ** 0.5
    ws = (w.abs().amax(-1) / 448).clamp_min(1e-12)
    Bq = (w / ws[..., None]).to(torch.float8_e4m3fn)
    D = torch.zeros(M, N // 2 if swiglu else N, dtype=torch.bfloat16, device="cuda")
    od, cd = offs.cuda(), cnts.cuda()
    _native.call("mx_grouped_gemm_fp8", A.data_ptr(), lda, Bq.view(torch.uint8).data_ptr(),
                 ws.contiguous().data_ptr(), D.data_ptr(), od.data_ptr(), cd.data_ptr(), G, M, N,
                 K, int(swiglu), s)
    torch.cuda.synchronize()
    aq = A[:, :K].contiguous().view(torch.float8_e4m3fn).float()
    asc = A[:, K:K + 4].contiguous().view(torch.float32)[:, 0]
    for g in range(G):
        o, c = int(offs[g]), int(cnts[g])
        if c == 0:
            continue
        ref = (aq[o:o + c] * asc[o:o + c, None]) @ (Bq[g].float() * ws[g][:, None]).T
        if swiglu:
            # w13 interleave: per 128-row block, 64 gate rows then 64 up rows
            blocks = ref.view(c, N // 128, 2, 64)
            ref = (torch.nn.functional.silu(blocks[:, :, 0]) * blocks[:, :, 1]).reshape(c, N // 2)
        got = D[o:o + c].float()
        assert torch.allclose(got, ref, rtol=2e-2, atol=2e-2), (g, (got - ref).abs().max())


def _fp8_case(n, m, T, h, E, k, I, Is, wire="slot", seed=1):
    from paper_2601_08800_b200 import FP8SwiGLUExperts, RouterSpec, build_cluster, run_moe_block
    from paper_2601_08800_b200 import _native as N
    from paper_2601_08800_b200.plan import LayerPlan
    ex = FP8SwiGLUExperts.random(E, h, I, shared_inter=Is, seed=seed)
    gen = torch.Generator(device="cuda").manual_seed(seed + 1)
    x = torch.randn(n * T, h, device="cuda", generator=gen).to(torch.bfloat16)
    router = RouterSpec.random(n * T, E, k, seed=seed + 2)
    if wire == "slot":
        y, _ = run_moe_block(build_cluster(n, m), x, router, ex)
    else:
        plan = LayerPlan(n, m, T, h, E, k, dtype=torch.bfloat16, expert_kind="swiglu_fp8",
                         inter=I, shared_inter=Is, wire=wire)
        sh = ex.stacked_shards(n, m)
        ids, w = router.arrays()
        y = torch.empty(n * T, h, dtype=torch.bfloat16, device="cuda")
        plan.forward(x, ex.params(sh), ids=torch.as_tensor(ids).cuda(),
                     weights=torch.as_tensor(w, dtype=torch.float32).cuda(), y_out=y)
        plan.close()
    gate, up, down, shared = ex.oracle_arrays(n, m)
    ids, w = router.arrays()
    y_o = orc.moe_layer_fp8(x.float().cpu().numpy(), ids, w, gate, up, down, shared)
    yg = y.double().cpu().numpy()
    return orc.verify_metric(yg, y_o), float(np.linalg.norm(yg - y_o) / np.linalg.norm(y_o))


# fp8 tolerance (unspecified by the north star): the replica applies identical
# quantisation, so the residual is e4m3 rounding-boundary flips after fp32-vs-
# f64 accumulation differences -- bounded as relative Frobenius error <= 1e-2
# and max |y-e|/max(|e|,1) <= 5e-2.
FP8_FRO, FP8_MAX = 1e-2, 5e-2


@pytest.mark.parametrize("n,m,Is,wire", [(1, 1, 0, "slot"), (2, 2, 256, "slot"), (2, 4, 512, "slot"),
                                         (4, 2, 256, "token"), (2, 4, 512, "token")])
def test_fp8_layer_vs_oracle(n, m, Is, wire):
    mx, fro = _fp8_case(n, m, 48, 512, 16, 4, 512, Is, wire)
    assert fro <= FP8_FRO and mx <= FP8_MAX, (fro, mx)


@pytest.mark.parametrize("n,m,wire,Is", [(2, 2, "token", 256), (2, 4, "slot", 512)])
def test_fp8_layer_deepseek_gate(n, m, wire, Is):
    """Config C end to end: DeepSeek-V3 group-limited gate (sigmoid, bias,
    8 groups keep 4, routed scaling 2.5) feeding fp8 experts + shared expert;
    ids bit-exact with the oracle router, layer within the fp8 tolerance."""
    from paper_2601_08800_b200 import FP8SwiGLUExperts, _native as N
    from paper_2601_08800_b200.plan import GateSpec, LayerPlan
    T, h, E, k, I = 64, 512, 32, 4, 512
    ex = FP8SwiGLUExperts.random(E, h, I, shared_inter=Is, seed=41)
    gen = torch.Generator(device="cuda").manual_seed(42)
    x = torch.randn(n * T, h, device="cuda", generator=gen).to(torch.bfloat16)
    logits = torch.randn(n * T, E, device="cuda", generator=gen)
    bias = (0.05 * torch.randn(E, generator=torch.Generator().manual_seed(43))).float()
    gate = GateSpec.deepseek_v3(bias, groups=8, topk_groups=4, scaling=2.5)
    plan = LayerPlan(n, m, T, h, E, k, dtype=torch.bfloat16, expert_kind="swiglu_fp8",
                     inter=I, shared_inter=Is, wire=wire, gate=gate)
    sh = ex.stacked_shards(n, m)
    y = torch.empty(n * T, h, dtype=torch.bfloat16, device="cuda")
    plan.forward(x, ex.params(sh), logits=logits, y_out=y)
    ids, w = orc.router_group_limited(logits.cpu().numpy(), bias.numpy(), k, 8, 4, True, 2.5)
    for r in range(n * m):
        g = r // m
        got = plan.rank_views(r)["ids"].cpu().numpy()
        assert np.array_equal(got, ids[g * T:(g + 1) * T])
    gate_w, up, down, shared = ex.oracle_arrays(n, m)
    y_o = orc.moe_layer_fp8(x.float().cpu().numpy(), ids, w, gate_w, up, down, shared)
    yg = y.double().cpu().numpy()
    mx = orc.verify_metric(yg, y_o)
    fro = float(np.linalg.norm(yg - y_o) / np.linalg.norm(y_o))
    assert fro <= FP8_FRO and mx <= FP8_MAX, (fro, mx)
    plan.close()


@pytest.mark.parametrize("wire", ["token", "slot"])
def test_config_b_full_size_8_ranks_emulated(wire):
    """Config B at full size in the 8-GPU layout (TP2 x EP4, 8192 tokens,
    128 experts top-8, h=2048, I=768), all 8 ranks emulated on one GPU:
    the layer within the bf16 tolerance of the dense GPU oracle."""
    from paper_2601_08800_b200 import SwiGLUExperts, moe_oracle, RouterSpec, _native as N
    from paper_2601_08800_b200.plan import LayerPlan
    n, m, Tg, h, E, k, I = 4, 2, 8192, 2048, 128, 8, 768
    ex = SwiGLUExperts.random(E, h, I, seed=31)
    w13, w2 = ex.stacked_shards(n, m)
    gen = torch.Generator(device="cuda").manual_seed(32)
    x = torch.randn(Tg, h, device="cuda", generator=gen).to(torch.bfloat16)
    logits = torch.randn(Tg, E, device="cuda", generator=gen)
    plan = LayerPlan(n, m, Tg // n, h, E, k, dtype=torch.bfloat16, expert_kind="swiglu",
                     inter=I, wire=wire)
    y = torch.empty(Tg, h, dtype=torch.bfloat16, device="cuda")
    plan.forward(x, N.ExpertParams(None, None, w13.data_ptr(), w2.data_ptr()), logits=logits,
                 y_out=y)
    ids, w = orc.router_topk(logits.cpu().numpy(), k)
    v = plan.rank_views(0)
    assert np.array_equal(v["exp_cnt"].cpu().numpy(), np.bincount(ids.reshape(-1), minlength=E))
    router = RouterSpec(E, tuple(map(tuple, ids.tolist())),
                        tuple(map(tuple, w.astype(np.float64).tolist())))
    y_d = moe_oracle(x, router, ex)
    err = orc.verify_metric(y.float().cpu().numpy(), y_d.float().cpu().numpy())
    assert err <= 2e-2, err
    plan.close()


def test_fp8_deepseek_shape_layer():
    """BASELINE configs[2] shape: h=7168, moe_intermediate=2048, top-8 with a
    2048-wide shared expert, TP4 x EP2 (emulated 8 ranks on one GPU); expert
    count reduced to 16 to keep the fp8 weights in the test's budget."""
    mx, fro = _fp8_case(2, 4, 16, 7168, 16, 8, 2048, 2048, "slot", seed=11)
    assert fro <= FP8_FRO and mx <= FP8_MAX, (fro, mx)
