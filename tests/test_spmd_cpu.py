"""The multi-rank host logic on CPU: gloo process groups of 2-8 ranks.

Each rank is a separate process holding only its own node's tokens, its
experts' TP shard and its slice of the exchange -- the SPMD layout of
``MoELayer`` (rank ``d*m + t``, sim:63-67).  The exchanges run through real
``torch.distributed`` collectives over gloo with the package's own host
logic -- ``layout_for``, ``tp_ep_groups`` (the EP / TP groups of the NCCL
arm), ``baseline_splits`` (its all-to-all split sizes), ``routing_stats``
(the send matrix S) and ``expert_home_node`` -- and the per-rank values are
checked against the single-process CPU oracle:

* the fused path (sim:565-592): the column-shard dispatch into every TP rank
  of the host (AG fused into the A2A, sim:395-406), the TP pre-reduction and
  the weighted combine in the reference's arrival order (sim:506-520) --
  bit-exact in f64 against ``orc.run_fused_affine``;
* the NCCL arm's layout (``_run_baseline``, sim:598-680): full-width
  all-to-all dispatch and combine over the EP group, TP all-reduce -- within
  1e-12 (the all-reduce associates differently).

The device kernels of the same path are covered by ``test_spmd_gpu.py``
(2-8 processes on one GPU) and the 2/4-GPU runs in ``profiles/``; this file
needs no GPU and runs in the CPU suite.  The oracle is the checker only.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mixserve_oracle as orc
from paper_2601_08800_b200.layer import baseline_splits, layout_for, tp_ep_groups
from paper_2601_08800_b200.layer_model import routing_stats
from paper_2601_08800_b200.simcluster import expert_home_node

T, H, E, K = 24, 10, 12, 3     # h=10 splits unevenly over 4 TP ranks (3,3,2,2)


def _inputs(n, seed, empty_host=False):
    """The same seeded global batch on every rank (distinct experts/token);
    ``empty_host``: no token routes to the last node's experts, so it
    receives nothing and sends nothing back (zero splits both ways)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n * T, H))
    pool = E if not empty_host else -(-(n - 1) * E // n)   # experts homed on nodes < n-1
    ids = np.stack([rng.permutation(pool)[:K] for _ in range(n * T)]).astype(np.int64)
    w = rng.random((n * T, K))
    scales = rng.uniform(0.5, 1.5, E)
    biases = rng.standard_normal(E)
    return x, ids, w, scales, biases


def _partial(recv, experts, scales, biases, cols, m):
    """TP rank's affine partial (sim:535-562) of its host's received rows."""
    part = np.zeros_like(recv)
    part[:, cols] = scales[experts][:, None] * recv[:, cols]
    part += (biases[experts] / m)[:, None]
    return part


def _a2a(chunks, group=None):
    """Variable-size all-to-all of flat f64 chunks (one per group rank)."""
    send = torch.from_numpy(np.concatenate([c.ravel() for c in chunks]) if chunks
                            else np.zeros(0))
    in_sizes = [c.size for c in chunks]
    sizes = torch.tensor(in_sizes, dtype=torch.int64)
    out_sizes = torch.empty_like(sizes)
    dist.all_to_all_single(out_sizes, sizes, group=group)
    recv = torch.empty(int(out_sizes.sum()), dtype=torch.float64)
    dist.all_to_all_single(recv, send, output_split_sizes=out_sizes.tolist(),
                           input_split_sizes=in_sizes, group=group)
    return np.split(recv.numpy(), np.cumsum(out_sizes.tolist())[:-1])


def _worker(rank, world, tp, port, seed, empty_host):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _check_rank(rank, world, tp, seed, empty_host)
    finally:
        dist.destroy_process_group()


def _check_rank(rank, world, tp, seed, empty_host):
    n, m = layout_for(world, tp)
    node, t = divmod(rank, m)
    ep_g, tp_g = tp_ep_groups(n, m, rank)
    assert dist.get_world_size(ep_g) == n and dist.get_world_size(tp_g) == m
    assert dist.get_rank(ep_g) == node and dist.get_rank(tp_g) == t

    x, ids, w, scales, biases = _inputs(n, seed, empty_host)
    table = orc.Table(ids, w, n, T, E)
    if empty_host:
        assert table.slots(n - 1) == 0 and table.slots(0) > 0
    S, _ = routing_stats(ids, n, E)
    assert np.array_equal(S, table.send_counts())
    assert all(int(expert_home_node(e, n, E)) == int(orc.home(e, n, E)) for e in range(E))
    cols = orc.col_slices(H, m)
    x_mine = x[node * T:(node + 1) * T]           # replicated over the node's TP ranks

    # expected values from the single-process oracle
    x_nodes = [x[j * T:(j + 1) * T] for j in range(n)]
    recv_ref = orc.dispatch_received(x_nodes, table)[node]
    part_ref = orc.partial_affine(orc.dispatch_received(x_nodes, table), table,
                                  scales, biases, m, H)[node][t]
    y_ref, _ = orc.run_fused_affine(n, m, x, ids, w, E, scales, biases)
    y_ref = y_ref[node * T:(node + 1) * T]

    # ---- fused: column-shard dispatch into every TP rank of each host
    chunks = []
    for dst in range(world):
        d = dst // m
        rows = table.rows_from(d, node)
        chunks.append(x_mine[table.token[d][rows] - node * T][:, cols[t]])
    got = _a2a(chunks)
    recv = np.full((table.slots(node), H), np.nan)
    for src in range(world):
        j, ts = divmod(src, m)
        rows = table.rows_from(node, j)
        recv[np.ix_(rows, np.arange(H)[cols[ts]])] = got[src].reshape(len(rows), cols[ts].stop - cols[ts].start)
    assert np.array_equal(recv, recv_ref)                  # bit-exact rows

    part = _partial(recv, table.expert[node], scales, biases, cols[t], m)
    assert np.array_equal(part, part_ref)

    # TP pre-reduction of the node's partials, rank-ascending (sim:433-441)
    allp = [torch.empty(part.shape, dtype=torch.float64) for _ in range(m)]
    dist.all_gather(allp, torch.from_numpy(part), group=tp_g)
    reduced = allp[0].numpy().copy()
    for q in range(1, m):
        reduced = reduced + allp[q].numpy()
    red_mine = reduced[:, cols[t]]

    # combine: column shard back to each source node's TP rank t (EP group)
    back = _a2a([red_mine[table.rows_from(node, j)] for j in range(n)], group=ep_g)
    width = red_mine.shape[1]
    y_cols = np.zeros((T, width))
    for d in [(node - i) % n for i in range(1, n)] + [node]:    # arrival order
        rows = table.rows_from(d, node)
        vals = back[d].reshape(len(rows), width)
        np.add.at(y_cols, table.token[d][rows] - node * T, table.weight[d][rows][:, None] * vals)
    assert np.array_equal(y_cols, y_ref[:, cols[t]])      # bit-exact column shard
    pad = T * max(c.stop - c.start for c in cols)
    gathered = [torch.empty(pad, dtype=torch.float64) for _ in range(m)]
    mine = torch.zeros(pad, dtype=torch.float64)
    mine[:y_cols.size] = torch.from_numpy(y_cols.ravel())
    dist.all_gather(gathered, mine, group=tp_g)
    y = np.concatenate([gathered[q][:T * (c.stop - c.start)].numpy().reshape(T, -1)
                        for q, c in enumerate(cols)], axis=1)
    assert np.array_equal(y, y_ref)

    # ---- NCCL arm's layout: full-width A2A over the EP group, TP all-reduce
    send_split, recv_split = baseline_splits(S, node)
    assert sum(send_split) == sum(len(table.rows_from(d, node)) for d in range(n))
    send_rows = np.concatenate([x_mine[table.token[d][table.rows_from(d, node)] - node * T]
                                for d in range(n)])
    rx = torch.empty(sum(recv_split), H, dtype=torch.float64)
    dist.all_to_all_single(rx, torch.from_numpy(np.ascontiguousarray(send_rows)),
                           output_split_sizes=recv_split, input_split_sizes=send_split,
                           group=ep_g)
    recv_b = np.empty((table.slots(node), H))
    for j, blk in enumerate(torch.split(rx, recv_split)):
        recv_b[table.rows_from(node, j)] = blk.numpy()
    assert np.array_equal(recv_b, recv_ref)
    part_b = _partial(recv_b, table.expert[node], scales, biases, cols[t], m)
    out = np.concatenate([part_b[table.rows_from(node, j)] for j in range(n)])
    ret = torch.empty(sum(send_split), H, dtype=torch.float64)
    dist.all_to_all_single(ret, torch.from_numpy(np.ascontiguousarray(out)),
                           output_split_sizes=send_split, input_split_sizes=recv_split,
                           group=ep_g)
    y_b = np.zeros((T, H))
    for d, blk in enumerate(torch.split(ret, send_split)):
        rows = table.rows_from(d, node)
        np.add.at(y_b, table.token[d][rows] - node * T, table.weight[d][rows][:, None] * blk.numpy())
    y_bt = torch.from_numpy(y_b)
    dist.all_reduce(y_bt, group=tp_g)
    np.testing.assert_allclose(y_bt.numpy(), y_ref, rtol=0, atol=1e-12)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,tp,empty_host", [(2, 1, False), (2, 2, False), (4, 2, False),
                                                 (4, 4, False), (8, 2, False), (4, 1, True),
                                                 (4, 2, True)])
def test_spmd_exchange_gloo(world, tp, empty_host):
    mp.spawn(_worker, args=(world, tp, _free_port(), 1000 + 10 * world + tp, empty_host),
             nprocs=world, join=True)


def test_layout_and_splits_host_logic():
    assert layout_for(1) == (1, 1)
    assert layout_for(8) == (4, 2)          # config B's named TP2 x EP4
    assert layout_for(8, 4) == (2, 4)       # config C's TP4 x EP2
    with pytest.raises(ValueError):
        layout_for(6, 4)
    S = np.array([[3, 1, 0], [2, 5, 4], [0, 0, 7]])
    assert baseline_splits(S, 1) == ([2, 5, 4], [1, 5, 0])
    with pytest.raises(ValueError):
        baseline_splits(S, 3)
    if not dist.is_initialized():
        with pytest.raises(RuntimeError):
            tp_ep_groups(2, 1, 0)
