"""Benchmark of the AnTKV decode path on B200 (contract: see DESIGN.md §6).

Workload (BASELINE.json metric, configs[2]/north star shape on one GPU):
LLaMA-3-8B attention shapes (32 Q / 8 KV heads, d=128), 128K-token context
per GPU, 1-bit VQ KV (d8m256), 1 % anchors, 32-token window, batch 1.  One
step = one decode token through the attention of all 32 layers (each layer
has its own cache: ~1.2 GB of state per step, far above the 126 MB L2, so no
L2 flush is needed).  Per layer the step appends the token, runs split-KV
decode attention over codes + anchors + window with RoPE after
reconstruction, merges the splits and evicts/encodes the oldest window row.

value = decode-attention tok/s as BASELINE.md defines it
        (batch / time of one layer's decode-attention call, all heads);
        at N > 1 the context is N x 128K tokens sharded by sequence and the
        partials are merged over peer memory (or NCCL with --exchange nccl);
        the rate is not multiplied by N (one token per step).
--impl reference times the reference package's own
QuantizedKVCache.decode_step (cache.py:149-194, staged into oracle/_ref by
oracle/Makefile) on the host cores, one single-head cache per core, on a
bounded sample of the same workload.
"""

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HQ, HKV, D = 32, 8, 128
METRIC = "decode attn tok/s & HBM GB/s at 128K ctx, 1-bit VQ KV; encode tok/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--ctx", type=int, default=131072, help="context tokens per GPU")
    p.add_argument("--layers", type=int, default=32)
    p.add_argument("--batch", type=int, default=1)
    p.add_argument("--notation", default="d8m256")
    p.add_argument("--kernel", default="fast", choices=["fast", "generic"])
    p.add_argument("--splits", type=int, default=0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="eager launches instead of CUDA graphs")
    p.add_argument("--shared-stream", action="store_true",
                   help="do not declare the captured decode chains exclusive (all reads after the PDL wait)")
    p.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                   help="N > 1: shard partials over peer memory (default) or NCCL all-gather")
    p.add_argument("--no-prefill", action="store_true", help="skip the prefill timing")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    return p.parse_args()


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        j = json.loads(f.read_text())
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every 50 ms through
    NVML during the timed region (same counters as `nvidia-smi
    --query-gpu=clocks.sm,clocks_event_reasons.*`)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index):
        self.index = index
        self.sm = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() else self.index
            self._h = N.nvmlDeviceGetHandleByIndex(phys)
            self._N = N
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM)
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        except Exception as exc:  # NVML missing: record why
            self.error = repr(exc)
        return self

    def _run(self):
        N = self._N
        while not self._stop.is_set():
            try:
                self.sm.append(N.nvmlDeviceGetClockInfo(self._h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, const in self.REASONS:
                    if r & getattr(N, const, 0):
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.01)

    def __exit__(self, *a):
        self._stop.set()
        if self._thread:
            self._thread.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz,
                    "reasons": ["unsampled: " + getattr(self, "error", "no samples")]}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


# ------------------------------------------------------------------ ours
def build_layers(args, rank, world, torch):
    from paper_2506_19505_b200 import CacheConfig, Codebook, QuantizedKVCache, VqConfig
    from paper_2506_19505_b200.anchors import select_anchors_device
    vq = VqConfig.from_notation(args.notation)
    # only the tail shard holds the full-precision window (and appends)
    cfg = CacheConfig(vq=vq, anchor_fraction=0.01, window_size=32 if rank == world - 1 else 0,
                      theta_base=500000.0)
    n = args.ctx
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    rng = np.random.default_rng(1000 + rank)
    caches = []
    global_n = n * world
    offset = rank * n
    for layer in range(args.layers):
        ck = rng.standard_normal((HKV, vq.m, vq.d_sub)).astype(np.float32)
        cv = rng.standard_normal((HKV, vq.m, vq.d_sub)).astype(np.float32)
        cache = QuantizedKVCache(cfg, Codebook(vq, ck), Codebook(vq, cv), batch=args.batch,
                                 q_heads=HQ, fast=(args.kernel == "fast"), splits=args.splits,
                                 capacity=n + args.steps + args.warmup + 96, token_offset=offset)
        K = torch.randn((args.batch, HKV, n, D), device="cuda", generator=g).to(torch.bfloat16)
        V = torch.randn((args.batch, HKV, n, D), device="cuda", generator=g).to(torch.bfloat16)
        # anchors: the real top-k kernel on synthetic anchor scores; this
        # shard holds 1 % of its tokens (its share of the global budget)
        budget = cfg.budget_for(n)
        sc_k = torch.rand((args.batch * HKV, n), device="cuda", generator=g)
        sc_v = torch.rand((args.batch * HKV, n), device="cuda", generator=g)
        anchors = select_anchors_device(sc_k, sc_v, budget).view(args.batch, HKV, budget)
        pos = (torch.arange(n, device="cuda", dtype=torch.int64) + offset)[None].repeat(args.batch, 1)
        cache.build_from(K, V, pos, anchors)
        if world > 1 and rank == world - 1:
            # the tail shard promotes window rows against the global budget:
            # it counts every shard's anchors (each shard holds `budget`)
            cache.tensors["hstate"][:, :, 0] = budget * world
        del K, V, sc_k, sc_v
        caches.append(cache)
    torch.cuda.synchronize()
    return caches, cfg


def measured_traffic(args):
    """DRAM bytes per decode launch from the committed ncu --set full capture
    (profiles/decode_fast_traffic.json) when it was taken on this workload."""
    f = ROOT / "profiles" / "decode_fast_traffic.json"
    try:
        t = json.loads(f.read_text())
    except (OSError, ValueError):
        return None
    if (t.get("ctx"), t.get("notation"), t.get("batch")) == (args.ctx, args.notation, args.batch) \
            and args.kernel == "fast":
        return t["dram_bytes_per_launch"]
    return None


def verify_exchange(exchange, cache, rank, world, torch):
    """One attention-only step of layer 0 merged both ways (peer-memory
    stores + antkv_lse_merge_wait vs NCCL all-gather + LSE combine): every
    rank must agree before the timed run uses the peer path."""
    import torch.distributed as dist
    from paper_2506_19505_b200.parallel import gather_partials, lse_merge
    B = cache.B
    g = torch.Generator(device="cuda").manual_seed(91)
    q = torch.randn((B, HQ, D), device="cuda", generator=g).to(torch.bfloat16)
    qpos = torch.full((B,), cache.token_count * world, dtype=torch.int64, device="cuda")
    out = torch.empty((B, HQ, D), dtype=torch.float32, device="cuda")
    lse = torch.empty((B, HQ), dtype=torch.float32, device="cuda")
    p2p = torch.empty((B * HQ, D), dtype=torch.float32, device="cuda")
    exchange.advance()
    cache.step_publish(q, None, None, qpos, out, lse, exchange)
    exchange.merge(p2p)
    cache.attend_device(q, qpos, out, lse)
    o_all, l_all = gather_partials(out, lse)
    ref = lse_merge(o_all, l_all, torch.empty((B, HQ, D), dtype=torch.float32, device="cuda"))
    ok = torch.tensor([float(torch.isfinite(p2p).all() and
                             (p2p.view_as(ref) - ref).abs().max() <= 1e-5 * ref.abs().max())], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    return bool(ok.item() > 0)


def launches_per_layer_step(cache, args, world):
    """Our kernel launches per layer-step on rank 0: the fused d8m256 step is
    one launch (N=1) or attention + merge (N>1); the staged / generic paths
    run append, attention (+ split merge in the staged kernel, a separate
    combine launch in the generic one) and the two eviction launches."""
    vq = cache.config.vq
    fused = (args.kernel == "fast" and vq.d_sub == 8 and vq.m <= 256 and HQ == 4 * HKV)
    staged = args.kernel == "fast" and not fused
    if world == 1:
        return 1 if fused else (4 if staged else 5)
    return 2 if fused else (2 if staged else 3)


def smem_roofline(args, launch_ms, sm_mhz):
    """The bound the fused kernel actually runs against: shared-memory
    wavefronts (one 128-byte wavefront per SM per clock) of its codebook
    gathers, from the committed ncu count per launch (decode_fast_traffic.json)
    over the live launch time.  None off that workload."""
    f = ROOT / "profiles" / "decode_fast_traffic.json"
    try:
        t = json.loads(f.read_text())
    except (OSError, ValueError):
        return None
    if (t.get("ctx"), t.get("notation"), t.get("batch")) != (args.ctx, args.notation, args.batch) \
            or args.kernel != "fast" or "smem_wavefronts_per_launch" not in t:
        return None
    w = t["smem_wavefronts_per_launch"]
    per_clk = w / (launch_ms * 1e-3 * sm_mhz * 1e6 * 148)
    return {"bound": "smem", "unit": "wavefronts/clk/SM", "achieved": per_clk, "peak": 1.0,
            "frac": per_clk, "wavefronts_per_launch": w, "sm_mhz": sm_mhz,
            "note": "whole launch incl. prologue/combine; ~4 wavefronts (512 B of fp16 centroids) "
                    "per token-head are the floor of any exact fp16 reconstruction"}


def algorithmic_bytes(cache, torch):
    """Bytes one decode-attention call must move (SURVEY.md §8d formula):
    H_kv*[n_q*(code bytes/token) + n_fp*2*d*2] + 2*H_q*d*2 + codebooks."""
    t = cache.tensors
    n = cache.token_count
    vq = cache.config.vq
    code_b = 2 * (D // vq.d_sub) * vq.index_bits / 8.0
    total = 0.0
    hs = t["hstate"].cpu().numpy()
    for b in range(cache.B):
        for h in range(cache.Hkv):
            n_fp = int((t["pool_kind"][b, h] >= 0).sum())
            total += (n - n_fp) * code_b + n_fp * 2 * D * 2
    total += cache.B * (2 * HQ * D * 2)
    total += cache.Hkv * 2 * vq.m * vq.d_sub * 4
    return total


def encode_throughput(torch, n=131072, reps=5, vq_m=256, d_sub=8):
    """tokens/s through K+V encoding of all 8 KV heads of one layer."""
    from paper_2506_19505_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(7)
    X = torch.randn((2 * HKV, n, D), device="cuda", generator=g).to(torch.bfloat16)
    C = torch.randn((2 * HKV, vq_m, d_sub), device="cuda", generator=g)
    cbytes = 1 if vq_m <= 256 else 2
    codes = torch.empty((2 * HKV, n, D // d_sub * cbytes), dtype=torch.uint8, device="cuda")
    st = _lib.stream()

    def run():
        for i in range(2 * HKV):
            _lib.call("antkv_vq_encode", _lib.ptr(X[i]), _lib.BF16, n, D, _lib.ptr(C[i]), vq_m,
                      d_sub, _lib.ptr(codes[i]), cbytes, st)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = n * 2 * HKV * (D // d_sub) * vq_m * d_sub * 2
    return {"value": n / (ms / 1e3), "unit": "tok/s", "ms_per_layer": ms, "tokens": n,
            "config": f"d{d_sub}m{vq_m}, K+V, 8 KV heads, d=128, float32 distances",
            "tflops": flops / (ms / 1e3) / 1e12}


def prefill_throughput(torch, n=131072):
    """One layer's prefill (FA + aux, AnS, anchor selection, encode, layout)
    at LLaMA-3-8B attention shapes, bf16 inputs."""
    from paper_2506_19505_b200 import CacheConfig, Codebook, QuantizedKVCache, VqConfig
    vq = VqConfig.from_notation("d8m256")
    cfg = CacheConfig(vq=vq, anchor_fraction=0.01, window_size=32, theta_base=500000.0)
    rng = np.random.default_rng(3)
    cbk = rng.standard_normal((HKV, vq.m, vq.d_sub)).astype(np.float32)
    cbv = rng.standard_normal((HKV, vq.m, vq.d_sub)).astype(np.float32)
    g = torch.Generator(device="cuda").manual_seed(9)
    Q = torch.randn((1, HQ, n, D), device="cuda", generator=g).to(torch.bfloat16)
    K = torch.randn((1, HKV, n, D), device="cuda", generator=g).to(torch.bfloat16)
    V = torch.randn((1, HKV, n, D), device="cuda", generator=g).to(torch.bfloat16)
    pos = np.arange(n)
    times = []
    for _ in range(2):   # the first run warms up
        cache = QuantizedKVCache(cfg, Codebook(vq, cbk), Codebook(vq, cbv), batch=1, q_heads=HQ)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cache.prefill(Q, K, V, pos)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = times[-1]
    flops = 6 * HQ * D * n * n / 2      # FA (4 HQ d n^2 / 2) + AnS (2 HQ d n^2 / 2), causal
    del Q, K, V, cache
    return {"ctx": n, "ms_per_layer": ms, "tok_s": n / (ms / 1e3), "tflops_attention": flops / (ms / 1e3) / 1e12,
            "config": "one layer, 32 Q / 8 KV heads, d=128, d8m256, 1% anchors; includes host-side "
                      "checks and the anchor-count readback"}


def run_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_SINGLE_DEVICE_CHECK=1: functional check of the N>1 path with every
    # rank on device 0 and gloo collectives (no timing value)
    single = os.environ.get("BENCH_SINGLE_DEVICE_CHECK") == "1"
    if single:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if single:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2506_19505_b200 import _lib
    from paper_2506_19505_b200.parallel import PeerExchange, gather_partials, lse_merge
    _lib.load()
    caches, cfg = build_layers(args, rank, world, torch)
    # N > 1: partials travel over peer memory (the decode launch stores them
    # into every rank's receive slots, antkv_lse_merge_wait merges); NCCL
    # all-gather if the buffers cannot be mapped (--exchange nccl forces it)
    exchange, exchange_kind = None, "none"
    if world > 1:
        exchange_kind = "nccl"
        # (the one-device functional check keeps NCCL/gloo: ranks sharing a GPU
        # must not spin on each other's flags)
        if args.exchange == "p2p" and not single:
            try:
                exchange = PeerExchange(args.batch * HQ, D)
                exchange_kind = "p2p"
            except Exception as exc:  # noqa: BLE001 (reported in the JSON line)
                print(f"peer exchange unavailable ({exc}); NCCL all-gather", file=sys.stderr)
            if exchange is not None and not verify_exchange(exchange, caches[0], rank, world, torch):
                print("peer exchange disagrees with the NCCL all-gather merge; using NCCL", file=sys.stderr)
                exchange.close()
                exchange, exchange_kind = None, "nccl"
    L, B = args.layers, args.batch
    n0 = caches[0].token_count
    is_tail = rank == world - 1
    g = torch.Generator(device="cuda").manual_seed(77)
    total_steps = args.warmup + args.steps
    qs = torch.randn((total_steps, L, B, HQ, D), device="cuda", generator=g).to(torch.bfloat16)
    ks = torch.randn((total_steps, L, B, HKV, D), device="cuda", generator=g).to(torch.bfloat16)
    vs = torch.randn((total_steps, L, B, HKV, D), device="cuda", generator=g).to(torch.bfloat16)
    gpos0 = n0 * world
    qpos = [torch.full((B,), gpos0 + s, dtype=torch.int64, device="cuda") for s in range(total_steps)]
    out = torch.empty((B, HQ, D), dtype=torch.float32, device="cuda")
    lse = torch.empty((B, HQ), dtype=torch.float32, device="cuda")
    merged = torch.empty((B, HQ, D), dtype=torch.float32, device="cuda")

    def layer_step(s, l, cache):
        if world == 1:
            cache.step_device(qs[s, l], ks[s, l], vs[s, l], qpos[s], out)
            return out
        # sequence shards: the tail appends / attends / evicts in one fused
        # launch, the other shards attend; (o, lse) exchanged and merged
        if exchange is not None:
            exchange.advance()
            cache.step_publish(qs[s, l], ks[s, l] if is_tail else None, vs[s, l] if is_tail else None,
                               qpos[s], out, lse, exchange)
            exchange.merge(merged.view(-1, D))
            return merged
        if is_tail:
            cache.step_device(qs[s, l], ks[s, l], vs[s, l], qpos[s], out, lse)
        else:
            cache.attend_device(qs[s, l], qpos[s], out, lse)
        o_all, l_all = gather_partials(out, lse)
        return lse_merge(o_all, l_all, merged)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    use_graph = world == 1 and not args.no_graph

    def chain_ctx():
        # the captured chains hold only this library's kernels (plus memcpy
        # nodes): the stream is declared exclusive so the fused decode launch
        # may read its inputs before griddepcontrol.wait (antkv_stream_exclusive)
        import contextlib
        return contextlib.nullcontext() if args.shared_stream else _lib.exclusive_stream()
    if use_graph:
        # CUDA graphs: one step = the 32 per-layer decode kernels, replayed so
        # host launch overhead is outside the measurement
        q_st, k_st, v_st = qs[0].clone(), ks[0].clone(), vs[0].clone()
        qpos_st = qpos[0].clone()
        out_st = torch.empty((L, B, HQ, D), dtype=torch.float32, device="cuda")

        def body():
            for l in range(L):
                caches[l].step_device(q_st[l], k_st[l], v_st[l], qpos_st, out_st[l])
            qpos_st.add_(1)

        body()                       # eager warm-up (lazy init), advances the caches by 1
        torch.cuda.synchronize()
        step_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(step_graph), chain_ctx():
            body()
        run_step = step_graph.replay
        advanced = 1
    else:
        def run_step_s(s):
            for l in range(L):
                layer_step(s, l, caches[l])
        advanced = 0

    for s in range(args.warmup):
        run_step() if use_graph else run_step_s(s)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record()
        for s in range(args.warmup, total_steps):
            run_step() if use_graph else run_step_s(s)
        e1.record()
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    for c in caches:
        c._n += (args.warmup + args.steps + advanced) if is_tail else 0

    # attention-kernel-only timing on the same caches (no append/evict),
    # graph-captured: per-launch device time of the decode-attention kernel
    reps = max(3, min(args.steps, 10))
    qlast = (qpos_st if use_graph else qpos[-1]).clone()
    for l in range(L):
        caches[l].attend_device(qs[0, l], qlast, out)
    torch.cuda.synchronize()
    if use_graph:
        att_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(att_graph), chain_ctx():
            for l in range(L):
                caches[l].attend_device(qs[0, l], qlast, out)
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for r in range(reps):
        if use_graph:
            att_graph.replay()
        else:
            for l in range(L):
                caches[l].attend_device(qs[r % total_steps, l], qlast, out)
    a1.record()
    torch.cuda.synchronize()
    attn_ms = a0.elapsed_time(a1) / (reps * L)
    clk_mhz = clk.summary().get("sm_mhz") or clk.max_mhz or 1965.0
    alg_bytes = algorithmic_bytes(caches[0], torch)

    # e2e through the public step API with pinned host buffers: every step
    # copies q/k/v of every layer host->device and the outputs device->host
    qh = qs[0].cpu().pin_memory()
    kh = ks[0].cpu().pin_memory()
    vh = vs[0].cpu().pin_memory()
    outh = torch.empty((L, B, HQ, D), dtype=torch.float32).pin_memory()
    e2e_steps = max(3, min(args.steps, 8))
    cap_left = min(c.capacity for c in caches) - caches[0].token_count - 4
    e2e_steps = min(e2e_steps, max(1, cap_left - 1))
    if use_graph:
        dq, dk, dv, p_dev, o_dev = q_st, k_st, v_st, qpos_st, out_st
    else:
        dq, dk, dv = torch.empty_like(qs[0]), torch.empty_like(ks[0]), torch.empty_like(vs[0])
        p_dev = qpos[-1] + 1
        o_dev = torch.empty((L, B, HQ, D), dtype=torch.float32, device="cuda")

    def e2e_body():
        dq.copy_(qh, non_blocking=True)
        dk.copy_(kh, non_blocking=True)
        dv.copy_(vh, non_blocking=True)
        for l in range(L):
            if world == 1:
                caches[l].step_device(dq[l], dk[l], dv[l], p_dev, o_dev[l])
            elif exchange is not None:
                exchange.advance()
                caches[l].step_publish(dq[l], dk[l] if is_tail else None, dv[l] if is_tail else None,
                                       p_dev, out, lse, exchange)
                exchange.merge(o_dev[l].view(-1, D))
            else:
                if is_tail:
                    caches[l].step_device(dq[l], dk[l], dv[l], p_dev, out, lse)
                else:
                    caches[l].attend_device(dq[l], p_dev, out, lse)
                o_all, l_all = gather_partials(out, lse)
                o_dev[l].copy_(lse_merge(o_all, l_all, merged))
        outh.copy_(o_dev, non_blocking=True)
        p_dev.add_(1)

    if use_graph:
        e2e_body()
        torch.cuda.synchronize()
        e2e_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(e2e_graph), chain_ctx():
            e2e_body()
        for c in caches:
            c._n += 1
    barrier()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record()
    for s in range(e2e_steps):
        e2e_graph.replay() if use_graph else e2e_body()
    x1.record()
    torch.cuda.synchronize()
    for c in caches:
        c._n += e2e_steps if (world == 1) else 0
    e2e_ms = x0.elapsed_time(x1) / e2e_steps
    t = torch.tensor([e2e_ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    enc = encode_throughput(torch) if rank == 0 else None
    # config #3's 0.375-bit code (m = 4096): the tensor-core encoder of encode_tc.cu
    enc3 = encode_throughput(torch, n=32768, vq_m=4096, d_sub=32) if rank == 0 else None
    pre = prefill_throughput(torch) if rank == 0 and not args.no_prefill else None
    peak, peak_kind = peaks()
    achieved = alg_bytes / (attn_ms / 1e3) / 1e9
    # one token per sequence per layer-step, whatever the number of sequence
    # shards: N GPUs serve an N-times longer context at (ideally) the same rate
    value = B * L / (ms / 1e3)
    result = None
    if rank == 0:
        result = {
            "metric": METRIC,
            "value": value,
            "unit": "tok/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f16-mma/f32-accum" if args.kernel == "fast" else "f32",
            "data": "synthetic (seeded randn bf16 K/V, random N(0,1) codebooks)",
            "config": {
                "workload": f"decode attention, {args.ctx // 1024}K ctx per GPU x {world} GPU(s), "
                            f"{args.notation} ({caches[0].config.vq.index_bits / caches[0].config.vq.d_sub:.3g}-bit), 1% anchors, window 32, {HQ} Q / {HKV} KV heads, "
                            f"d={D}, batch {B}, {L} layers per step",
                "ctx_per_gpu": args.ctx, "layers_per_step": L, "batch": B, "kernel": args.kernel,
                "l2": f"no flush: per-step working set {alg_bytes * L / 1e9:.2f} GB > 126 MB L2",
                "tok_s_definition": "batch * layers / step time (BASELINE.md: batch / one layer's "
                                    "decode-attention call); at N > 1 the context is N x ctx_per_gpu "
                                    "(sequence shards) and the rate is NOT multiplied by N",
                "context_tokens": args.ctx * world,
                "model_tok_s": B / (ms / 1e3),
                "launch": "CUDA graph per step" if use_graph else "eager",
                "exchange": exchange_kind,
            },
            "hbm_gbs": achieved,
            "roofline": {"bound": "hbm", "kernel": "decode attention (split-KV + combine)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "aggregate_gbs": achieved * world, "aggregate_peak": peak * world,
                         "traffic": measured_traffic(args), "algorithmic_bytes_per_launch": alg_bytes,
                         "launch_ms": attn_ms,
                         "secondary": smem_roofline(args, attn_ms, clk_mhz)},
            "e2e": {"value": B * L / (e2e_ms / 1e3), "unit": "tok/s",
                    "h2d_bytes_per_step": (qh.numel() + kh.numel() + vh.numel()) * 2,
                    "d2h_bytes_per_step": outh.numel() * 4, "ms_per_step": e2e_ms,
                    "path": ("QuantizedKVCache.step_device per layer (antkv_decode_step)" if world == 1
                             else "per layer: fused step on the tail shard / attention on the others, "
                                  + ("partials stored into every rank's slots by the same launch over "
                                     "peer memory, antkv_lse_merge_wait" if exchange is not None
                                     else "NCCL all-gather of (o, lse), antkv_lse_combine"))
                            + " with pinned-host q/k/v H2D and output D2H inside the timed region"
                            + (", CUDA-graph replay" if use_graph else "")},
            # our kernels per layer-step on rank 0: the fused step (N=1) or attention +
            # LSE combine (N>1, rank 0 is not the tail); generic path: append, attention,
            # combine, evict
            "gpu_launches": args.steps * L * launches_per_layer_step(caches[0], args, world),
            "clocks": clk.summary(),
            "encode": enc,
            "encode_d32m4096": enc3,
            "prefill": pre,
        }
    if exchange is not None:
        barrier()
        exchange.close()
    return result, caches


# ------------------------------------------------------------- reference
# The reference arm runs the reference package's OWN decode step,
# QuantizedKVCache.decode_step (cache.py:149-194: append, dequantize, RoPE of
# every cached key, softmax, A.V, window eviction with promotion or encode),
# with its compiled _ckernels, staged by oracle/Makefile into
# oracle/_ref/pkg/antkv (git-ignored; built from /root/reference in the build
# container, travels to the GPU box).  Nothing of this repo's package or
# native library is imported on this path.  The reference is single-head, so
# the 32 query heads of a layer are 32 independent single-head caches (the
# GQA group's KV rows replicated per query head, "MHA-expanded"); a layer-step
# is 32 head decode steps.  One worker process per host core (one BLAS
# thread each) owns one head cache; a timed step is one round of those
# workers' decode steps -- a bounded sample of min(cores, 32)/32 of a
# layer-step at the full context.  Without the staged package (no
# /root/reference at build time) the oracle restatement stands in ("port").

def _reference_module():
    pkg = ROOT / "oracle" / "_ref" / "pkg"
    if (pkg / "antkv" / "cache.py").exists():
        sys.path.insert(0, str(pkg))
        import antkv
        return antkv, "reference"
    sys.path.insert(0, str(ROOT / "oracle"))
    import antkv_oracle
    return antkv_oracle, "port"


def round_bf16(x):
    """Round to the nearest bfloat16 (even on ties), returned as float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(np.shape(x))


def _ref_head_state(n, m, d_sub, head, window=32, frac=0.01):
    """Synthetic single-head cache contents at n tokens (seeded per head):
    1 % anchors outside the window, the last `window` other tokens windowed,
    the rest random code indices; bf16-exact float32 rows; N(0,1) codebooks."""
    rng = np.random.default_rng(5000 + head)
    G = D // d_sub
    anchors = np.sort(rng.choice(n - window, size=math.ceil(frac * n), replace=False))
    is_fp = np.zeros(n, dtype=bool)
    is_fp[anchors] = True
    win = np.flatnonzero(~is_fp)[-window:]
    is_fp[win] = True
    fp = np.flatnonzero(is_fp)
    rows_k = round_bf16(rng.standard_normal((len(fp), D)))
    rows_v = round_bf16(rng.standard_normal((len(fp), D)))
    codes = rng.integers(0, m, size=(n, 2, G))
    ck = rng.standard_normal((m, d_sub)).astype(np.float32)
    cv = rng.standard_normal((m, d_sub)).astype(np.float32)
    return anchors, win, fp, rows_k, rows_v, codes, ck, cv


def _ref_build_cache(mod, kind, n, notation, head, theta):
    """One single-head reference cache holding the synthetic state, installed
    field by field as the reference's own load() does (cache.py:286-342)."""
    vq = mod.VqConfig.from_notation(notation) if kind == "reference" else None
    m = vq.m if vq else int(notation.split("m")[1])
    d_sub = vq.d_sub if vq else int(notation[1:].split("m")[0])
    anchors, win, fp, rows_k, rows_v, codes, ck, cv = _ref_head_state(n, m, d_sub, head)
    if kind == "port":
        c = mod.OracleCache([ck], [cv], anchor_fraction=0.01, window_size=32, theta_base=theta)
        K = np.zeros((1, n, D))
        V = np.zeros((1, n, D))
        K[0, fp], V[0, fp] = rows_k, rows_v
        c.prefill(None, K, V, np.arange(n), anchors=[anchors], codes=[(codes[:, 0], codes[:, 1])])
        return c
    cfg = mod.CacheConfig(vq=vq, anchor_fraction=0.01, window_size=32, theta_base=theta)
    c = mod.QuantizedKVCache(cfg, mod.Codebook(config=vq, centroids=ck), mod.Codebook(config=vq, centroids=cv))
    c.d = D
    c.positions = list(range(n))
    kinds = [mod.cache.KIND_QUANTIZED] * n
    for j in anchors:
        kinds[j] = mod.cache.KIND_ANCHOR
    for j in win:
        kinds[j] = mod.cache.KIND_WINDOWED
    c.kinds = kinds
    fp_set = set(int(j) for j in fp)
    c.k_rows = {int(j): rows_k[i] for i, j in enumerate(fp)}
    c.v_rows = {int(j): rows_v[i] for i, j in enumerate(fp)}
    c.k_codes = {j: codes[j, 0] for j in range(n) if j not in fp_set}
    c.v_codes = {j: codes[j, 1] for j in range(n) if j not in fp_set}
    c.anchor_indices = anchors.astype(np.int64)
    return c


def _ref_worker(conn, head, n, notation, theta):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    mod, kind = _reference_module()
    t0 = time.perf_counter()
    cache = _ref_build_cache(mod, kind, n, notation, head, theta)
    conn.send(time.perf_counter() - t0)
    rng = np.random.default_rng(9000 + head)
    while True:
        s = conn.recv()
        if s is None:
            break
        q, k, v = rng.standard_normal((3, D))
        t0 = time.perf_counter()
        if kind == "port":
            cache.decode_step(q[None], k[None], v[None], n + s)
        else:
            cache.decode_step(q, k, v, n + s)
        conn.send(time.perf_counter() - t0)
    conn.close()


class RefPool:
    """One process per host core (at most HQ), each owning one single-head
    reference cache at the workload's context; step(s) runs one decode step
    on every worker and returns the round's wall time."""

    def __init__(self, n, notation, theta=500000.0, workers=None):
        import multiprocessing as mp
        self.kind = _reference_module()[1]
        self.P = max(1, min(HQ, workers or os.cpu_count() or 1))
        ctx = mp.get_context("fork")
        self.conns, self.procs = [], []
        for h in range(self.P):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_ref_worker, args=(b, h, n, notation, theta), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        self.build_s = max(c.recv() for c in self.conns)

    def step(self, s):
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(s)
        head_s = [c.recv() for c in self.conns]
        return time.perf_counter() - t0, head_s

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.procs:
            p.join(timeout=30)


def ref_config1_timing(theta=500000.0):
    """BASELINE config #1 on the reference itself, one core: a 2048-token
    single-head prefill (cache.py:100-140) and 128 decode steps
    (cache.py:149-194), d8m256, 1 % anchors, window 32.  Returns ms per head."""
    mod, kind = _reference_module()
    if kind != "reference":
        return None
    from threadpoolctl import threadpool_limits
    rng = np.random.default_rng(101)
    n, steps = 2048, 128
    Q, K, V = (round_bf16(rng.standard_normal((n + steps, D))).astype(np.float64) for _ in range(3))
    vq = mod.VqConfig.from_notation("d8m256")
    cb = [mod.Codebook(config=vq, centroids=rng.standard_normal((256, 8)).astype(np.float32)) for _ in range(2)]
    cache = mod.QuantizedKVCache(mod.CacheConfig(vq=vq, anchor_fraction=0.01, window_size=32, theta_base=theta),
                                 cb[0], cb[1])
    with threadpool_limits(1):
        t0 = time.perf_counter()
        cache.prefill(Q[:n], K[:n], V[:n], np.arange(n))
        t1 = time.perf_counter()
        for t in range(n, n + steps):
            cache.decode_step(Q[t], K[t], V[t], t)
        t2 = time.perf_counter()
    dec = (t2 - t1) / steps
    return {"prefill_ms_per_head": (t1 - t0) * 1e3, "decode_step_ms_per_head": dec * 1e3,
            "layer_step_s_one_core": dec * HQ, "cores": 1,
            "what": "reference QuantizedKVCache (its compiled _ckernels), one head, 2048-token prefill + "
                    "128 decode steps; a layer-step is 32 such head steps"}


def run_reference(args):
    """--impl reference: the reference package's own decode step on the host
    cores, on the same workload config as the GPU arm (rank 0 only)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    c1 = ref_config1_timing()
    pool = RefPool(args.ctx, args.notation)
    try:
        for s in range(args.warmup):
            pool.step(s)
        walls, heads = [], []
        for s in range(args.warmup, args.warmup + args.steps):
            w, h = pool.step(s)
            walls.append(w)
            heads += h
    finally:
        pool.close()
    t = float(np.mean(walls))
    value = args.batch * (pool.P / HQ) / t      # layer-steps per second
    sample = (f"each step: {pool.P} single-head reference caches at {args.ctx} tokens, one decode step "
              f"each, in parallel ({pool.P} of the {HQ} head steps of a layer-step; {t:.2f} s wall, "
              f"{np.mean(heads):.2f} s per head step)")
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "tok/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded random codes, 1% anchors, bf16-exact rows, N(0,1) codebooks)",
        "config": {"workload": f"decode step, {args.ctx // 1024}K ctx, {args.notation}, 1% anchors, window 32, "
                               f"{HQ} Q / {HKV} KV heads (MHA-expanded: the reference is single-head), d={D}, "
                               f"batch {args.batch}; value = layer-steps/s (= batch x layers / s)",
                   "ctx_per_gpu": args.ctx, "path": f"{pool.kind}: QuantizedKVCache.decode_step "
                                                    "(cache.py:149-194) incl. append and evict/encode",
                   "head_cache_build_s": pool.build_s},
        "cpu_baseline": {"value": value, "unit": "tok/s", "cores": pool.P, "kind": pool.kind,
                         "sample": sample},
        "config1_reference": c1,
        "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_so_loaded": repo_libraries_mapped(),
    }


def repo_libraries_mapped():
    """Shared objects of this repository's product package mapped into this
    process (the reference arm must map none)."""
    try:
        maps = Path("/proc/self/maps").read_text()
    except OSError:
        return None
    pkg = str(ROOT / "paper_2506_19505_b200")
    return sorted({ln.split()[-1] for ln in maps.splitlines() if ln.split() and ln.split()[-1].startswith(pkg)
                   and ".so" in ln.split()[-1]})


def main():
    args = parse()
    if args.impl == "reference":
        res = run_reference(args)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    res, caches = run_ours(args)
    rank = int(os.environ.get("RANK", "0"))
    if rank == 0:
        if not args.no_cpu_baseline and int(os.environ.get("WORLD_SIZE", "1")) == 1:
            pool = RefPool(args.ctx, args.notation)
            try:
                t, heads = pool.step(0)
            finally:
                pool.close()
            res["cpu_baseline"] = {"value": args.batch * (pool.P / HQ) / t, "unit": "tok/s", "cores": pool.P,
                                   "kind": pool.kind,
                                   "sample": f"one round of {pool.P} single-head reference decode steps "
                                             f"(QuantizedKVCache.decode_step at {args.ctx} tokens, one per "
                                             f"core) = {pool.P}/{HQ} of a layer-step, {t:.2f} s wall"}
        print(json.dumps(res), flush=True)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
