"""Multi-process execution of the GPU engine with head-group shards
(SURVEY 8(e)): two processes on cuda:0, each holding its shard of a
synthetic Llama-2-7B-shaped layer stack, with the per-layer partial-output
sum installed through ``sharding.attach_allreduce`` over a gloo group.
gloo cannot be captured in a CUDA graph, so this also exercises the step's
eager fallback; NCCL (the bench path) needs one GPU per rank, which gpurun
does not offer.  The summed output must equal the unsharded step on the
same cache, over several steps (cache growth included, which rebuilds the
session: the reduction hook must survive it).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2407_21118_b200 as P
        from paper_2407_21118_b200.harness import synthetic_engine
        from paper_2407_21118_b200.sharding import attach_allreduce, shard_engine

        torch.cuda.set_device(0)
        T = 3000
        w, fused, cache = synthetic_engine(layers=2, batch=1, context=T, extra=0, seed=21)
        xs = np.random.default_rng(5).standard_normal((4, 4096)) * 0.5
        fs, cs = shard_engine(fused, cache, rank, world)

        def allreduce(t):
            host = t.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.SUM)
            t.copy_(host)

        attach_allreduce(cs, allreduce)
        ys = []
        for i in range(4):
            if i == 2:
                cs.reserve(cs.capacity + 1)  # growth rebuilds the session
            ys.append(P.palu_decode_step_rope(w, fs, cs, xs[i]))
        assert cs._session.allreduce is allreduce
        assert not cs._session.use_graph  # gloo is not capturable: eager fallback
        if rank == 0:
            want = [P.palu_decode_step_rope(w, fused, cache, xs[i]) for i in range(4)]
            errs = [float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(ys, want)]
            q.put(("ok", errs))
        dist.barrier()
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put(("error", f"rank {rank}: {type(exc).__name__}: {exc}"))
        raise
    finally:
        dist.destroy_process_group()


def test_two_process_head_shards_match_full_step():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert all(p.exitcode == 0 for p in procs), msgs
    ok = [m for m in msgs if m[0] == "ok"]
    assert ok, msgs
    assert max(ok[0][1]) < 1e-4, ok
