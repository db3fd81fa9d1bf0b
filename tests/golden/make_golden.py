"""Freeze reference outputs as golden fixtures (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the UNMODIFIED reference ``moeplan`` read-only and records, for a
grid of cluster shapes and seeded inputs, everything the B200 path must
reproduce: routing tables (sim:236-251), expert-major orders (sim:528-532),
send counts, fused/baseline/oracle outputs (sim:565-694) and the trace CSV
(sim:99-136).  ``/root/reference`` does not exist on the GPU box, so the
fixtures are committed; tests never import the reference at run time.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

from moeplan.simcluster import (ExpertSpec, RouterSpec, _expert_rows,
                                build_cluster, build_routing_table,
                                moe_oracle, run_moe_block, trace_to_csv)

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
from oracle.mixserve_oracle import SwiGLUOracle, bf16_round, router_topk  # noqa: E402


def table_arrays(table):
    out = {}
    for d, slots in enumerate(table.slots_by_host):
        out[f"tok_{d}"] = np.array([s.token for s in slots], dtype=np.int64)
        out[f"exp_{d}"] = np.array([s.expert for s in slots], dtype=np.int64)
        out[f"src_{d}"] = np.array([s.src_node for s in slots], dtype=np.int64)
        out[f"w_{d}"] = np.array([s.weight for s in slots], dtype=np.float64)
        em = [i for _, rows in _expert_rows(slots) for i in rows]
        out[f"emajor_{d}"] = np.array(em, dtype=np.int64)
    return out


def routed_case(name, n, m, tokens, k, E, h, seed, router=None, x=None):
    cluster = build_cluster(n, m)
    if x is None:
        rng = np.random.default_rng(seed)
        x = rng.standard_normal((tokens, h))
    if router is None:
        router = RouterSpec.random(tokens, E, k, seed=seed + 1)
    experts = ExpertSpec.default(E)
    y_f, trace = run_moe_block(cluster, x, router, experts, mode="fused")
    y_b, trace_b = run_moe_block(cluster, x, router, experts, mode="baseline")
    y_o = moe_oracle(x, router, experts)
    table = build_routing_table(router, n, tokens // n)
    arrays = dict(
        x=x, ids=np.array(router.expert_ids, dtype=np.int64).reshape(tokens, -1),
        weights=np.array(router.weights, dtype=np.float64).reshape(tokens, -1),
        y_fused=y_f, y_baseline=y_b, y_oracle=y_o,
        trace_csv=np.array(trace_to_csv(trace.events)),
        trace_baseline_csv=np.array(trace_to_csv(trace_b.events)),
        meta=np.array(json.dumps(dict(n=n, m=m, tokens=tokens, k=k, E=E, h=h,
                                      seed=seed))),
    )
    arrays.update(table_arrays(table))
    np.savez_compressed(HERE / f"{name}.npz", **arrays)


def main():
    # the reference's own 2x2 golden fixture (pkg/tests/test_golden.py:18-22)
    routed_case("ref_2x2_golden", 2, 2, 4, 1, 2, 8, 0,
                router=RouterSpec.round_robin(4, 2, 1),
                x=np.arange(32.0).reshape(4, 8))
    (HERE / "trace_2x2.csv").write_text(
        str(np.load(HERE / "ref_2x2_golden.npz")["trace_csv"]))
    # empty batch: the reference still emits its zero-byte event schedule
    for mode in ("fused", "baseline"):
        _, tr = run_moe_block(build_cluster(2, 2), np.zeros((0, 8)), RouterSpec(4, (), ()),
                              ExpertSpec.default(4), mode=mode)
        (HERE / f"trace_empty_2x2_{mode}.csv").write_text(trace_to_csv(tr.events))
    # BASELINE.json configs[0]: n=2, m=2, 256 tokens, h=512, 8 experts top-2
    routed_case("ref_config_a", 2, 2, 256, 2, 8, 512, 1)
    # shape grid after pkg/tests/test_simcluster.py:216-224 and
    # test_acceptance.py:29-46
    grid = [(1, 1, 8, 2, 8, 8), (1, 2, 8, 2, 8, 8), (2, 1, 16, 2, 8, 8),
            (2, 2, 16, 4, 8, 24), (2, 4, 32, 2, 8, 16), (4, 2, 32, 4, 16, 16),
            (4, 4, 64, 8, 32, 32), (4, 2, 64, 8, 128, 64),
            (2, 4, 64, 8, 256, 64), (8, 1, 64, 2, 16, 8), (1, 8, 16, 4, 8, 16),
            (2, 2, 12, 3, 5, 10), (4, 2, 16, 2, 6, 8)]
    for i, (n, m, tokens, k, E, h) in enumerate(grid):
        routed_case(f"ref_grid_{i:02d}", n, m, tokens, k, E, h, 100 + i)
    # skew: every token on expert 0 (pkg/tests/test_simcluster.py:190-198)
    skew = RouterSpec(8, tuple((0,) for _ in range(16)),
                      tuple((1.0,) for _ in range(16)))
    routed_case("ref_skew", 2, 4, 16, 1, 8, 8, 7, router=skew)

    # gate extension: our router restatement feeding the reference
    rng = np.random.default_rng(42)
    logits = rng.standard_normal((64, 16)).astype(np.float32)
    logits[3, 5] = logits[3, 9] = logits[3].max() + 1.0  # exact tie
    ids, w = router_topk(logits, 4)
    router = RouterSpec(16, tuple(tuple(int(e) for e in r) for r in ids),
                        tuple(tuple(float(v) for v in r) for r in w))
    routed_case("ref_router_topk", 2, 2, 64, 4, 16, 16, 3, router=router)
    np.savez_compressed(HERE / "router_topk_logits.npz", logits=logits,
                        ids=ids, weights=w)

    # SwiGLU expert through the reference's moe_oracle and baseline mode
    # (duck-typed .apply)
    rng = np.random.default_rng(5)
    E, h, I, tokens, k = 8, 64, 32, 16, 2
    wg = bf16_round(rng.standard_normal((E, I, h)) / np.sqrt(h))
    wu = bf16_round(rng.standard_normal((E, I, h)) / np.sqrt(h))
    wd = bf16_round(rng.standard_normal((E, h, I)) / np.sqrt(I))
    x = bf16_round(rng.standard_normal((tokens, h))).astype(np.float64)
    router = RouterSpec.random(tokens, E, k, seed=6)
    experts = SwiGLUOracle(wg, wu, wd)
    y_o = moe_oracle(x, router, experts)
    y_b, _ = run_moe_block(build_cluster(2, 2), x, router, experts,
                           mode="baseline")
    np.savez_compressed(
        HERE / "ref_swiglu.npz", x=x, wg=wg, wu=wu, wd=wd,
        ids=np.array(router.expert_ids), weights=np.array(router.weights),
        y_oracle=y_o, y_baseline=y_b)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
