"""World-size-2 gloo test of the head-group sharding plan.

Each rank runs the oracle restricted to its head groups and the partial
layer outputs are summed with torch.distributed (gloo, 127.0.0.1); the result
must equal the single-process oracle step.  CPU only.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import palu_oracle as po


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _partial_step(L, wo_f, store_rows, x, shard, n, dh, base, T):
    """Oracle step for the heads of one shard -> partial output (attention.py:392-448)."""
    from paper_2407_21118_b200.parallel_plan import shard_layer_arrays

    o_off = po.head_offsets(L.value_ranks, L.s_v, n)
    sl = shard_layer_arrays(L.wq, wo_f, o_off, L.ak, L.bk, L.av, L.bv, dh, shard)
    scale = 1.0 / np.sqrt(dh)
    out = np.zeros(n * dh)
    hk = {g: np.vstack([store_rows["k"][g], x @ L.ak[g]]) for g in shard.k_groups}
    hv = {g: np.vstack([store_rows["v"][g], x @ L.av[g]]) for g in shard.v_groups}
    positions = np.arange(T + 1, dtype=np.float64)
    row = 0
    for j, h in enumerate(shard.heads):
        q = x @ sl["wq"][:, j * dh:(j + 1) * dh]
        q = po.rope_rows(q[None], np.array([float(T)]), base)[0]
        g, p = divmod(h, L.s_k)
        k = hk[g] @ L.bk[g][:, p * dh:(p + 1) * dh]
        k = po.rope_rows(k, positions, base)
        probs = po.softmax(k @ q * scale)
        ctx = probs @ hv[h // L.s_v]
        r = o_off[h + 1] - o_off[h]
        out += ctx @ sl["wo_fused"][row:row + r]
        row += r
    return out


def _worker(rank, world, port, result_q):
    import torch
    import torch.distributed as dist

    from paper_2407_21118_b200.parallel_plan import allreduce_sum, plan_groups

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, dh, T, base = 8, 16, 40, 10000.0
    L = po.synth_layer(n * dh, n, dh, 2, [5, 7, 6, 4], 4, [9, 6], seed=77)
    wo_f = po.build_wo_fused(L, n, dh)
    X = po.random_matrix(T, n * dh, 78)
    rows = {"k": [X @ a for a in L.ak], "v": [X @ a for a in L.av]}
    x = po.random_matrix(1, n * dh, 79)[0]
    shard = plan_groups(n, L.s_k, L.s_v, world, rank)
    part = torch.from_numpy(_partial_step(L, wo_f, rows, x, shard, n, dh, base, T))
    full = allreduce_sum(part).numpy()
    if rank == 0:
        cache = po.OracleCache([L])
        cache.fill_direct(0, X)
        cache.t = T
        want = po.decode_step_rope([L], [wo_f], cache, x, n, dh, base)
        result_q.put(float(np.linalg.norm(full - want) / np.linalg.norm(want)))
    dist.barrier()
    dist.destroy_process_group()


def test_head_group_sharding_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=5) < 1e-12


def test_plan_groups_partitions_heads():
    from paper_2407_21118_b200.errors import ValidationError
    from paper_2407_21118_b200.parallel_plan import plan_groups

    for world in (1, 2, 4, 8):
        seen = []
        for r in range(world):
            sh = plan_groups(32, 4, 4, world, r)
            seen.extend(sh.heads)
            assert all(h // 4 in sh.k_groups for h in sh.heads)
        assert sorted(seen) == list(range(32))
    sh = plan_groups(8, 1, 4, 2, 1)  # mixed granularity: K per head, V joint per 4
    assert sh.heads == (4, 5, 6, 7) and sh.k_groups == (4, 5, 6, 7) and sh.v_groups == (1,)
    with pytest.raises(ValidationError):
        plan_groups(32, 4, 4, 3, 0)
