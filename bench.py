"""Bench: Palu RoPE latent-KV decode on B200 (BASELINE.json metric/config).

Workload (configs[1]): Llama-2-7B-shaped model, all 32 layers (d 4096, 32
heads, d_h 128), G-LRD group 4, 50% rank (r_k = r_v = 256 per group), bf16,
batch 1 per GPU, 64K cached tokens; one "step" = one decode step through
all 32 layers (append latents, RoPE score with online key reconstruction,
softmax, fused value path, output projection).  Synthetic random-init
weights; latent caches (17.2 GB) far exceed L2, so no flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl palu|reference]

Multi-GPU (torchrun): head-group sharding by default (rank k owns G/N key and
value groups, its W_q columns, A/B factors and wo_fused rows; one NCCL
all-reduce of the [B x d] layer output per layer inside the step graph;
"scaling": "strong"); --shard batch runs independent replicas ("weak").
Timing = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D, NH, DH, GS, RANK, LAYERS = 4096, 32, 128, 4, 256, 32


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="palu", choices=["palu", "reference"])
    ap.add_argument("--context", type=int, default=65536)
    ap.add_argument("--batch", type=int, default=1, help="sequences per GPU")
    ap.add_argument("--layers", type=int, default=LAYERS)
    ap.add_argument("--bits", default="16", help="latent bits: 16 | 2/3/4/8 | k_bits,v_bits (e.g. 16,4)")
    ap.add_argument("--rank-k", type=int, default=RANK, help="kept key rank per group (256 = uniform 50%%)")
    ap.add_argument("--rank-v", type=int, default=RANK, help="kept value rank per group (paper preset: 128/384)")
    ap.add_argument("--dtype", default="bfloat16")
    ap.add_argument("--shard", default="auto", choices=["auto", "batch", "heads"],
                    help="multi-GPU: head-group shards with one NCCL all-reduce of the layer "
                         "output per layer (strong scaling; the default for N > 1, SURVEY 8(e)) "
                         "or batch replicas (weak scaling)")
    ap.add_argument("--rope-base", type=float, default=None,
                    help="RoPE base (default 1e4; 1e6 with --kv-heads, Mistral-7B v0.2)")
    ap.add_argument("--rank-plan", default="", choices=["", "kv25-75"],
                    help="SURVEY 8(f)4: per-layer, per-group (r_k, r_v) from rank_plan.allocate "
                         "(ranks.py:131-219) on synthetic Fisher scores, K budget 25%%, V 75%%")
    ap.add_argument("--kv-heads", type=int, default=0,
                    help="GQA (BASELINE configs[3], Mistral-7B: 8): one G-LRD group per KV head, "
                         "replicated B (MHA-equivalent); ranks default to 64 = 50%% of a KV head")
    ap.add_argument("--rope", default="on", choices=["on", "off"],
                    help="off: palu_decode_step_norope path (attention.py:365-389)")
    ap.add_argument("--score-kernel", default="auto")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-baseline", action="store_true", help="skip the uncompressed comparators")
    a = ap.parse_args()
    if a.rope_base is None:
        a.rope_base = 1e6 if a.kv_heads else 10000.0
    if a.kv_heads and a.rank_k == RANK and a.rank_v == RANK:
        a.rank_k = a.rank_v = DH // 2
    a.plan = None
    if a.rank_plan:
        from paper_2407_21118_b200 import rank_plan as RP
        rk, rv, _, _ = RP.kv_plan(a.layers, NH // GS, GS * DH, D, 0.25, 0.75, min_rank=8)
        a.plan = (rk, rv)
        # accounting (bytes, FLOPs) uses the mean group rank
        a.rank_k = round(sum(map(sum, rk)) / (a.layers * (NH // GS)))
        a.rank_v = round(sum(map(sum, rv)) / (a.layers * (NH // GS)))
    b = [int(x) for x in str(a.bits).split(",")]
    a.bits = b[0] if len(b) == 1 else (b[0], b[1])
    return a


METRIC = "RoPE-attn decode us/step & HBM GB/s vs roofline, Llama-2-7B layer, 4K-64K ctx"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port of palu_decode_step_rope (reference algorithm)
# ---------------------------------------------------------------------------
def cpu_layer_steps(T: int, warmup: int, steps: int, seed: int = 11, rank_k: int = RANK,
                    rank_v: int = RANK, rope: bool = True):
    """Seconds of `steps` timed one-layer decode steps at T cached tokens
    (after `warmup` untimed ones), numpy oracle, cache rolled back between."""
    import numpy as np

    from oracle import palu_oracle as po

    rng = np.random.default_rng(seed)
    L = po.synth_layer(D, NH, DH, GS, rank_k, GS, rank_v, seed=seed)
    cache = po.OracleCache([L], bits=16)
    for st in cache.k_stores[0]:
        st.extend(rng.standard_normal((T, rank_k)) / 3.0)
    for st in cache.v_stores[0]:
        st.extend(rng.standard_normal((T, rank_v)) / 3.0)
    cache.t = T
    wo_f = [po.build_wo_fused(L, NH, DH)]
    wq_f = [po.build_wq_fused(L, NH, DH)] if not rope else None
    x = po.random_matrix(1, D, seed + 1)[0]
    out = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        if rope:
            po.decode_step_rope([L], wo_f, cache, x, NH, DH, 10000.0)
        else:
            po.decode_step_norope([L], wq_f, wo_f, cache, x, NH, DH)
        if i >= warmup:
            out.append(time.perf_counter() - t0)
        for st in cache.k_stores[0] + cache.v_stores[0]:
            st.truncate(T)
        cache.t = T
    return out


def cpu_layer_step_seconds(T: int, reps: int = 2, seed: int = 11, rank_k: int = RANK,
                           rank_v: int = RANK, rope: bool = True):
    """Best-of-reps seconds for one Llama-2-7B-layer decode step at T cached
    tokens, run by the numpy oracle (attention.py:392-448, or :365-389 with
    rope off, restated), with all host threads available to BLAS."""
    import numpy as np

    from oracle import palu_oracle as po

    rng = np.random.default_rng(seed)
    L = po.synth_layer(D, NH, DH, GS, rank_k, GS, rank_v, seed=seed)
    cache = po.OracleCache([L], bits=16)
    for st in cache.k_stores[0]:
        st.extend(rng.standard_normal((T, rank_k)) / 3.0)
    for st in cache.v_stores[0]:
        st.extend(rng.standard_normal((T, rank_v)) / 3.0)
    cache.t = T
    wo_f = [po.build_wo_fused(L, NH, DH)]
    wq_f = [po.build_wq_fused(L, NH, DH)] if not rope else None
    x = po.random_matrix(1, D, seed + 1)[0]
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        if rope:
            po.decode_step_rope([L], wo_f, cache, x, NH, DH, 10000.0)
        else:
            po.decode_step_norope([L], wq_f, wo_f, cache, x, NH, DH)
        best = min(best, time.perf_counter() - t0)
        for st in cache.k_stores[0] + cache.v_stores[0]:
            st.truncate(T)
        cache.t = T
    return best


def host_info() -> dict:
    """CPU model, threads and numpy/BLAS build of the host that ran the CPU leg."""
    import numpy as np
    info = {"threads": os.cpu_count(), "numpy": np.__version__,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS", "unset (all cores)")}
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        cfg = np.show_config(mode="dicts")
        blas = cfg.get("Build Dependencies", {}).get("blas", {})
        info["blas"] = f"{blas.get('name', '?')} {blas.get('version', '')}".strip()
    except Exception:
        pass
    return info


def cpu_baseline(args):
    """One Llama-2-7B layer decode step at the headline context, timed
    directly (no extrapolation in T), scaled by layers x batch."""
    kw = dict(rank_k=args.rank_k, rank_v=args.rank_v, rope=args.rope == "on")
    s1 = cpu_layer_step_seconds(args.context, reps=1, **kw)
    us = s1 * args.layers * args.batch * 1e6
    step = "palu_decode_step_rope" if args.rope == "on" else "palu_decode_step_norope"
    return {
        "value": us, "unit": "us/step", "cores": os.cpu_count(), "kind": "port",
        "sample": (f"oracle {step}, one Llama-2-7B layer (gs4 r_k {args.rank_k} r_v {args.rank_v} "
                   f"fp64) at T={args.context} timed directly ({s1:.2f} s), x {args.layers} layers "
                   f"x batch {args.batch}"),
        "host": host_info(),
    }


def workload_config(args, world: int, heads: bool) -> dict:
    """The `config` of the bench line (shared by both arms)."""
    model = (f"mistral-7b-gqa{args.kv_heads}-32L-palu50-kvgroup" if args.kv_heads
             else "llama2-7b-32L-palu50-gs4" + ("-plan" if args.plan else ""))
    return {"workload": (f"{model}-rk{args.rank_k}-rv{args.rank_v}-"
                         + ("rope" if args.rope == "on" else "norope")),
            "context": args.context, "rank_k": args.rank_k, "rank_v": args.rank_v,
            "batch_per_gpu": args.batch,
            "global_batch": args.batch if heads else args.batch * world,
            "layers": args.layers, "bits": args.bits, "rope_base": args.rope_base,
            "parallelism": (f"heads{world}" if heads else f"replicas{world}"),
            "l2": "inputs larger than L2 (latent cache 17 GB/step)"}


# ---------------------------------------------------------------------------
def clocks_start(gpu_index: int):
    try:
        f = open(os.path.join("/tmp", f"clocks_{os.getpid()}.csv"), "w")
        p = subprocess.Popen(
            ["nvidia-smi", "-i", str(gpu_index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
             "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
            stdout=f, stderr=subprocess.DEVNULL)
        return p, f
    except Exception:
        return None, None


def clocks_stop(handle):
    p, f = handle
    if p is None:
        return None
    p.terminate()
    p.wait()
    f.close()
    rows = []
    for line in open(f.name):
        parts = [x.strip() for x in line.split(",")]
        if len(parts) >= 8:
            rows.append(parts)
    os.unlink(f.name)
    if not rows:
        return None
    sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
    smax = max(float(r[1]) for r in rows)
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
    loaded = [v for v in sm if v > 0.5 * smax] or sm
    return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": reasons,
            "samples": len(rows)}


# ---------------------------------------------------------------------------
def uncompressed_baseline(args, palu_ms):
    """Uncompressed bf16 MHA decode step on the same GPU and shape (the paper's
    speedup claim), timed exactly like the Palu step (CUDA
    graph of all layers, replayed K times between CUDA events):
      * flashinfer: per layer the fused q|k|v GEMV, RoPE + append of row t into
        an HND paged cache (palu_dense_append_paged), flashinfer's trtllm-gen
        decode kernel, bf16->fp32 cast, W_o GEMV -- the comparator the north
        star names ("uncompressed fused attention on the same GPU");
      * own K0 (palu_dense_decode): the repo's simple CUDA-core uncompressed
        kernel, reported for reference only (not a speed-up basis)."""
    import statistics as st

    import torch

    from paper_2407_21118_b200 import _lib
    from paper_2407_21118_b200.attention import _ptr, _stream
    from paper_2407_21118_b200.dense import DenseModel
    from paper_2407_21118_b200.model import AttentionConfig

    out = {}
    T, B, Lyr = args.context, args.batch, args.layers
    d, n, dh = D, NH, DH
    nkv = args.kv_heads or n  # GQA: the uncompressed cache holds the KV heads only
    cfg = AttentionConfig(D, NH, DH, layers=Lyr, rope=True, rope_base=args.rope_base)
    cap = T + 64
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    sc = 1.0 / math.sqrt(D)
    wqkv = [((torch.rand(D + 2 * nkv * DH, D, device="cuda", generator=g) * 2 - 1) * sc).bfloat16()
            for _ in range(Lyr)]
    wo = [((torch.rand(D, D, device="cuda", generator=g) * 2 - 1) * sc).bfloat16() for _ in range(Lyr)]
    K = max(5, args.steps // 2)

    def time_graph(launch, warm=3):
        import gc

        launch()
        torch.cuda.synchronize()
        gc.collect()
        gr = torch.cuda.CUDAGraph()
        s_ = torch.cuda.Stream()
        s_.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_):
            with torch.cuda.graph(gr, stream=s_):
                launch()
        torch.cuda.current_stream().wait_stream(s_)
        for _ in range(warm):
            gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        del gr
        return e0.elapsed_time(e1) / K

    kv_bytes = 2 * (T + 1) * nkv * dh * 2 * B
    # ---- flashinfer trtllm-gen step (graph) ----------------------------
    try:
        import flashinfer

        page = 64
        pps = (cap + page - 1) // page
        kv = [torch.empty(pps * B, 2, nkv, page, dh, device="cuda", dtype=torch.bfloat16)
              for _ in range(Lyr)]
        for t_ in kv:
            t_.normal_(0.0, 0.3)
        bt = torch.arange(pps * B, device="cuda", dtype=torch.int32).view(B, pps)
        t_dev = torch.full((1,), T, device="cuda", dtype=torch.int32)
        seq = torch.full((B,), T + 1, device="cuda", dtype=torch.int32)
        theta = torch.from_numpy(__import__("numpy").array(
            [args.rope_base ** (-2.0 * i / dh) for i in range(dh // 2)])).cuda()
        x = torch.randn(B, d, device="cuda") * 0.5
        nqkv = d + 2 * nkv * dh
        qkv = torch.zeros(B, nqkv, device="cuda")
        qb = torch.zeros(B, n, dh, device="cuda", dtype=torch.bfloat16)
        ob = torch.zeros(B, n, dh, device="cuda", dtype=torch.bfloat16)
        attn = torch.zeros(B, d, device="cuda")
        ws = torch.zeros(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
        code = _lib.DTYPE_BF16

        def fi_step():
            st_ = _stream()
            torch.add(t_dev, 1, out=seq)  # every sequence holds t + 1 rows after the append
            for li in range(Lyr):
                _lib.call("palu_gemv", code, _ptr(wqkv[li]), nqkv, d, _ptr(x), B, d, _ptr(qkv), nqkv, 0, st_)
                _lib.call("palu_dense_append_paged", _ptr(qkv), B, n, nkv, dh, _ptr(kv[li]), page, pps,
                          _ptr(theta), _ptr(t_dev), _ptr(qb), st_)
                flashinfer.decode.trtllm_batch_decode_with_kv_cache(
                    qb, kv[li], ws, bt, seq, cap, bmm1_scale=1.0 / math.sqrt(dh), bmm2_scale=1.0,
                    out=ob, kv_layout="HND")
                _lib.call("palu_cast_bf16_f32", _ptr(ob), _ptr(attn), B * d, st_)
                _lib.call("palu_gemv", code, _ptr(wo[li]), d, d, _ptr(attn), B, d, _ptr(x), d, 0, st_)
            # position fixed at T: the comparator re-decodes the same row each replay

        fi_ms = st.median(time_graph(fi_step) for _ in range(2))
        out["flashinfer_step_us"] = fi_ms * 1e3
        # attention kernel alone, one layer, back to back (HBM efficiency)
        R = 20
        fn = lambda: flashinfer.decode.trtllm_batch_decode_with_kv_cache(
            qb, kv[0], ws, bt, seq, cap, bmm1_scale=1.0 / math.sqrt(dh), bmm2_scale=1.0, out=ob,
            kv_layout="HND")
        fn()
        torch.cuda.synchronize()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(R):
            fn()
        b_.record()
        torch.cuda.synchronize()
        fa = a.elapsed_time(b_) / R
        out["flashinfer_attn_us_per_layer"] = fa * 1e3
        out["flashinfer_attn_hbm_gbs"] = kv_bytes / (fa * 1e-3) / 1e9
        out["speedup_vs_flashinfer_step"] = fi_ms / palu_ms
        del kv, ws
    except Exception as exc:  # comparator only; never the product path
        out["flashinfer_error"] = f"{type(exc).__name__}: {str(exc)[:200]}"
    torch.cuda.empty_cache()
    # ---- own simple K0 (reference only; MHA) --------------------------------
    try:
        if nkv != n:
            raise RuntimeError("own K0 implements MHA only")
        m = DenseModel(cfg, [w.float() for w in wqkv], [w.float() for w in wo], dtype="bfloat16",
                       batch=B, capacity=cap)
        m.kc.normal_(0.0, 0.3)
        m.vc.normal_(0.0, 0.3)
        m.t = T
        m.t_dev.fill_(T)
        m.x.normal_(0.0, 0.5)
        out["own_k0_us_per_step"] = time_graph(m.launch_step) * 1e3
        del m
    except (torch.OutOfMemoryError, RuntimeError) as exc:
        out["own_k0_error"] = f"{type(exc).__name__}: {str(exc)[:120]}"
    del wqkv, wo
    torch.cuda.empty_cache()
    return out


def run_reference(args):
    """--impl reference: the reference algorithm (oracle port of
    palu_decode_step_rope, numpy fp64, all host threads) on the box's CPU.
    Each step = one full Llama-2-7B layer at the headline context (the
    per-layer work of the workload, timed directly); value = median x layers
    x batch (the reference has no cross-layer state beyond x)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    kw = dict(rank_k=args.rank_k, rank_v=args.rank_v, rope=args.rope == "on")
    per = cpu_layer_steps(args.context, W, K, **kw)
    med = statistics.median(per)
    us = med * args.layers * args.batch * 1e6
    step = "palu_decode_step_rope" if args.rope == "on" else "palu_decode_step_norope"
    sample = (f"oracle port of {step} (numpy fp64, {os.cpu_count()} host threads): each step = one "
              f"Llama-2-7B layer at T={args.context} (median {med:.2f} s over {K} steps after {W} "
              f"warm-up), x {args.layers} layers x batch {args.batch}")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    line = {"metric": METRIC, "value": us, "unit": "us/step", "impl": "reference", "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": us / 1e3, "higher_is_better": False,
            "scaling": "strong" if args.shard == "heads" else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world, args.shard == "heads"),
            "cpu_baseline": {"value": us, "unit": "us/step", "cores": os.cpu_count(), "kind": "port",
                             "sample": sample, "host": host_info(),
                             "per_layer_s": [round(v, 3) for v in per]},
            "e2e": {"value": us, "unit": "us/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        if args.shard == "auto":
            args.shard = "heads" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "batch"
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2407_21118_b200 as P
    from paper_2407_21118_b200 import _lib
    from paper_2407_21118_b200.attention import _session
    from paper_2407_21118_b200.harness import synthetic_engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.shard == "auto":
        args.shard = "heads" if world > 1 else "batch"
    if args.shard == "heads" and (NH // GS) % world:
        raise SystemExit(f"--shard heads needs the {NH // GS} head groups to split over {world} GPUs")
    _lib.load()
    _lib.call("palu_device_check", local)

    K, W = args.steps, args.warmup
    extra = 2 * (K + W) + 16
    heads = args.shard == "heads"
    weights, fused, cache = synthetic_engine(layers=args.layers, batch=args.batch,
                                             context=args.context, extra=extra, bits=args.bits,
                                             dtype=args.dtype, seed=1234 + (0 if heads else rank),
                                             rank_k=args.plan[0] if args.plan else args.rank_k,
                                             rank_v=args.plan[1] if args.plan else args.rank_v,
                                             rope=args.rope == "on", rope_base=args.rope_base,
                                             kv_heads=args.kv_heads)
    if heads:
        # this rank keeps its head groups; one all-reduce per layer
        from paper_2407_21118_b200.sharding import attach_allreduce, shard_engine

        fused, cache = shard_engine(fused, cache, rank, world)
        torch.cuda.empty_cache()
    sess = _session(fused, cache, score_kernel=args.score_kernel)
    if heads and world > 1:
        attach_allreduce(sess, lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM))
    sess.x.copy_(torch.randn(args.batch, D, device="cuda") * 0.5)
    torch.cuda.synchronize()

    # --- device-resident timed region (graph replay of the whole step) ----
    for _ in range(W):
        sess.step_device()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks_start(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(K):
        sess.step_device()
    ev1.record()
    torch.cuda.synchronize()
    clocks = clocks_stop(clk)
    ms = ev0.elapsed_time(ev1) / K
    cache.t += W + K
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()

    # --- live per-kernel timing for the roofline (same warm state) ------
    prof = sess.profile_step()
    rep_used = "palu_rope_score_tc_rep" in prof  # K reconstructed once per KV head (GQA)
    for alias in ("palu_rope_score_tc_pf", "palu_rope_score_tc_rep"):  # other rope score entries
        if alias in prof:
            prof["palu_rope_score_tc"] = prof.pop(alias)
    cache.t += 1
    torch.cuda.synchronize()

    # --- e2e through the public API with host buffers --------------------
    e2e = None
    if not args.no_e2e:
        step_fn = P.palu_decode_step_rope if args.rope == "on" else P.palu_decode_step_norope
        xh = np.random.default_rng(rank).standard_normal((args.batch, D)) * 0.5
        x_in = xh[0] if args.batch == 1 else xh
        for _ in range(2):
            step_fn(weights, fused, cache, x_in)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(K):
            step_fn(weights, fused, cache, x_in)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / K
        if world > 1:
            t = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": e2e_ms * 1e3, "unit": "us/step",
               "h2d_bytes_per_step": 4 * D * args.batch, "d2h_bytes_per_step": 4 * D * args.batch,
               "path": "paper_2407_21118_b200.palu_decode_step_rope (numpy in/out, pinned staging)"}

    # --- roofline of the dominant kernel --------------------------------
    # peaks: MEASURED_PEAKS.json; the kernels are timed alone over ~0.1 ms
    # launches, so the tensor-bound score kernel is held against the BURST
    # bf16 figure (the sustained one is reported beside it)
    hbm, tf_burst, tf_sus, src = _peaks()
    T1 = args.context + W + K + 1  # rows scored in the profiled step (approx.)
    shards = world if heads else 1  # head-group shards: this rank's share of groups/heads
    n_groups = NH // GS // shards
    kb, vb = (args.bits, args.bits) if isinstance(args.bits, int) else args.bits
    meta = lambda b: 0 if b == 16 else 8  # fp32 scale + fp32 zero point per token and group
    k_tok = n_groups * (args.rank_k * kb / 8 + meta(kb))  # latent bytes per token
    v_tok = n_groups * (args.rank_v * vb / 8 + meta(vb))
    for score_name in ("palu_rope_attend_tc", "palu_rope_score_tc", "palu_rope_score",
                       "palu_latent_score_tc", "palu_latent_score"):
        if score_name in prof:
            break
    score_ms = statistics.mean(prof[score_name])
    rec_heads = (args.kv_heads if rep_used else NH) // shards  # heads whose K is reconstructed
    flops = 2.0 * T1 * rec_heads * args.rank_k * DH * args.batch  # reconstruction
    k_bytes = T1 * k_tok * args.batch
    v_bytes = T1 * v_tok * args.batch
    achieved_tf = flops / (score_ms * 1e-3) / 1e12
    total_kernel_ms = sum(sum(v) for v in prof.values())
    sv_name = next((k for k in ("palu_value_tc", "palu_softmax_value") if k in prof), None)
    sv_ms = statistics.mean(prof[sv_name]) if sv_name else 0.0
    latent_total = k_bytes + v_bytes
    # rope off: no reconstruction, the score kernel streams H_k (HBM-bound);
    # GQA with K rebuilt once per KV head: the key stream outlasts the MMAs
    if args.rope == "off" or k_bytes / (hbm * 1e9) > flops / (tf_burst * 1e12):
        achieved_gbs = k_bytes / (score_ms * 1e-3) / 1e9
        roofline_head = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": achieved_gbs / hbm, "traffic": None,
                         "peak_source": f"{src} HBM copy (MEASURED_PEAKS.json hbm_gbs)"}
    else:
        roofline_head = {"bound": "tensor", "achieved": achieved_tf, "peak": tf_burst, "unit": "TFLOP/s",
                         "frac": achieved_tf / tf_burst, "traffic": None,
                         "peak_source": f"{src} burst bf16 (MEASURED_PEAKS.json bf16_tflops)",
                         "frac_of_sustained": achieved_tf / tf_sus}
    # measured DRAM traffic of the dominant kernel, from a committed ncu capture
    # of the same workload (profiles/*_traffic.json), else null
    workload = workload_config(args, 1, False)["workload"]
    bits_key = list(args.bits) if isinstance(args.bits, tuple) else args.bits
    for tf_name in ("r02_traffic.json", "r01_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", tf_name)) as fh:
                entries = json.load(fh).get(score_name) or []
            entries = entries if isinstance(entries, list) else [entries]
            tr = next((e for e in entries if e["workload"] == workload and e["context"] == args.context
                       and e["batch"] == args.batch and e.get("bits", 16) == bits_key), None)
            if tr:
                roofline_head["traffic"] = tr["bytes"]
                roofline_head["traffic_source"] = "profiles/" + tr["capture"]
                break
        except (OSError, ValueError, KeyError):
            pass
    stream_ms = score_ms + sv_ms
    roofline = {**roofline_head,
                "kernel": score_name, "kernel_ms": score_ms,
                "algorithmic_flops_per_launch": flops,
                "share_of_step": sum(prof[score_name]) / total_kernel_ms,
                "score_hbm_gbs": (latent_total if sv_ms == 0.0 else k_bytes) / (score_ms * 1e-3) / 1e9,
                "value_kernel": sv_name, "value_ms": sv_ms,
                "value_hbm_gbs": v_bytes / (sv_ms * 1e-3) / 1e9 if sv_ms else None,
                "latent_bytes_per_layer": latent_total,
                "hbm_peak_gbs": hbm,
                "per_kernel_ms": {k: statistics.mean(v) for k, v in prof.items()}}
    # north star: HBM fraction of the latent-cache stream (K and V latents of
    # a layer over the time of the kernels that stream them)
    latent_stream = {"gbs": latent_total / (stream_ms * 1e-3) / 1e9,
                     "aggregate_gbs_all_ranks": latent_total * shards / (stream_ms * 1e-3) / 1e9,
                     "frac": latent_total / (stream_ms * 1e-3) / 1e9 / hbm,
                     "kernels": [score_name] + ([sv_name] if sv_name else []),
                     "bytes_per_layer": latent_total, "ms_per_layer": stream_ms}

    uncompressed = None
    if not args.no_baseline:
        # free the Palu engine first: the uncompressed caches are 2x the latent ones
        del sess
        cache._session = None
        del weights, fused, cache
        import gc

        gc.collect()
        torch.cuda.empty_cache()
        try:
            uncompressed = uncompressed_baseline(args, ms)
        except torch.OutOfMemoryError as exc:  # comparator only: keep the Palu line
            uncompressed = {"error": f"OutOfMemoryError: {str(exc)[:120]}"}
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args)

    if rank == 0:
        launches_per_step = sum(len(v) for v in prof.values())
        line = {
            "metric": METRIC, "value": ms * 1e3, "unit": "us/step", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong" if heads else "weak",
            "vs_baseline": None, "dtype": "bf16" if args.dtype == "bfloat16" else "f32",
            "data": "synthetic (random-init weights, N(0,1/9) latent cache rows)",
            "config": workload_config(args, world, heads),
            "tokens_per_s": (args.batch if heads else args.batch * world) / (ms * 1e-3),
            "gpu_launches": launches_per_step * K,
            "clocks": clocks, "roofline": roofline,
            "latent_stream_hbm_frac": latent_stream["frac"], "latent_stream": latent_stream,
            "speedup_vs_flashinfer_step": (uncompressed or {}).get("speedup_vs_flashinfer_step"),
            "cpu_baseline": cpu, "e2e": e2e,
            "uncompressed": uncompressed,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
