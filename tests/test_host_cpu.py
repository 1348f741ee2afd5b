"""CPU-only tests: the C-ABI library loads and exports every declared symbol,
the ctypes descriptor matches the C struct layout, host-side logic mirrors the
reference, and the sequence-sharded merge works over a 2-rank gloo group."""

import ctypes
import os
import re
import subprocess
import sys
import tempfile
import json
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import antkv_oracle as O

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "antkv_b200.h"


def _lib():
    from paper_2506_19505_b200 import _lib
    return _lib


def test_library_exports_every_header_symbol():
    lib = _lib()
    if not lib.LIB_PATH.exists():
        pytest.fail("libantkv_b200.so missing: run __graft_entry__.build()")
    declared = set(re.findall(r"ANTKV_API[^;(]*?\b(antkv_\w+)\s*\(", HEADER.read_text()))
    assert len(declared) >= 20
    handle = ctypes.CDLL(str(lib.LIB_PATH))
    for name in declared:
        assert hasattr(handle, name), name
    assert declared == set(lib.EXPORTED)
    lib.load(check_device=False)            # argtypes bind without a GPU


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib().LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_cache_desc_layout_matches_c_header(tmp_path):
    lib = _lib()
    fields = [f for f, _ in lib.CacheDesc._fields_]
    src = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"', "int main(void){",
           'printf("%zu\\n", sizeof(antkv_cache_desc));']
    src += [f'printf("%zu\\n", offsetof(antkv_cache_desc, {f}));' for f in fields]
    src += ["return 0;}"]
    (tmp_path / "l.c").write_text("\n".join(src))
    subprocess.run(["gcc", "-o", str(tmp_path / "l"), str(tmp_path / "l.c")], check=True)
    vals = [int(x) for x in subprocess.run([str(tmp_path / "l")], capture_output=True, text=True,
                                           check=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(lib.CacheDesc)
    for f, off in zip(fields, vals[1:]):
        assert getattr(lib.CacheDesc, f).offset == off, f


def test_no_cpu_path_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2506_19505_b200 import Codebook, VqConfig, encode_rows
    cb = Codebook(VqConfig(4, 16), np.zeros((16, 4), np.float32))
    with pytest.raises((RuntimeError, AssertionError)):
        encode_rows(np.zeros((2, 8)), cb)


def test_vq_config_and_bits_table():
    from paper_2506_19505_b200 import VqConfig, bits_per_element
    for notation, expected in [("d2m256", 4.0), ("d4m256", 2.0), ("d8m256", 1.0),
                               ("d16m4096", 0.75), ("d32m4096", 0.375)]:
        assert float(bits_per_element(VqConfig.from_notation(notation))) == expected
    with pytest.warns(UserWarning):
        assert bits_per_element(VqConfig(4, 100)) == pytest.approx(7 / 4)
    with pytest.raises(ValueError):
        VqConfig.from_notation("x8m2")
    with pytest.raises(ValueError):
        VqConfig(0, 4)


def test_cache_config_budget_kats():
    from paper_2506_19505_b200 import CacheConfig, VqConfig
    vq = VqConfig(4, 16)
    assert CacheConfig(vq=vq, anchor_fraction=0.01).budget_for(200) == 2
    assert CacheConfig(vq=vq, anchor_fraction=0.01).budget_for(50) == 1
    assert CacheConfig(vq=vq, anchor_count=7).budget_for(50) == 7
    assert CacheConfig(vq=vq, anchor_count=99).budget_for(50) == 50
    for bad in (dict(anchor_fraction=1.5), dict(window_size=-1), dict(policy="nope")):
        with pytest.raises(ValueError):
            CacheConfig(vq=vq, **bad)
    for n in (1, 7, 100, 2048, 131072, 840000):
        assert CacheConfig(vq=vq).budget_for(n) == O.budget_for(n, 0.01)


def test_pack_indices_matches_reference_format(rng):
    from paper_2506_19505_b200.util import pack_indices, unpack_indices
    for bits in (1, 3, 8, 12, 16):
        vals = rng.integers(2 ** bits, size=37)
        packed = pack_indices(vals, bits)
        assert packed == O.pack_indices(vals, bits)
        assert list(unpack_indices(packed, bits, 37)) == list(vals)
    with pytest.raises(ValueError):
        pack_indices([4], 2)


def test_codebook_roundtrip(tmp_path, rng):
    from paper_2506_19505_b200 import Codebook, VqConfig, load_codebook, save_codebook
    cb = Codebook(VqConfig(4, 16), rng.standard_normal((16, 4)).astype(np.float32), groups=3)
    save_codebook(cb, tmp_path / "cb.json")
    back = load_codebook(tmp_path / "cb.json")
    assert np.array_equal(back.centroids, cb.centroids) and back.groups == 3
    cb3 = Codebook(VqConfig(8, 256), rng.standard_normal((8, 256, 8)).astype(np.float32))
    save_codebook(cb3, tmp_path / "cb3.json")
    assert np.array_equal(load_codebook(tmp_path / "cb3.json").centroids, cb3.centroids)


def test_shard_ranges():
    from paper_2506_19505_b200.parallel import shard_ranges
    assert shard_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert shard_ranges(840000, 8)[-1] == (735000, 840000)


def _oracle_merge(o_all, l_all):
    o = o_all.double().numpy()
    lse = l_all.double().numpy()
    M = lse.max(axis=0)
    w = np.exp(lse - M[None])
    return torch.from_numpy((w[..., None] * o).sum(axis=0) / w.sum(axis=0)[..., None])


def _shard_worker(rank, world, port, q, K, V, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_19505_b200.parallel import gather_partials, shard_ranges
    s, e = shard_ranges(K.shape[0], world)[rank]
    logits = (K[s:e] @ q) / np.sqrt(q.shape[0])
    m = logits.max()
    p = np.exp(logits - m)
    o_r = torch.from_numpy((p @ V[s:e]) / p.sum()).float()[None]
    lse_r = torch.tensor([m + np.log(p.sum())], dtype=torch.float32)
    o_all, l_all = gather_partials(o_r, lse_r)
    merged = _oracle_merge(o_all, l_all)
    if rank == 0:
        ret.put(merged.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sequence_sharded_merge_gloo_world2():
    rng = np.random.default_rng(3)
    q = rng.standard_normal(16)
    K = rng.standard_normal((101, 16))
    V = rng.standard_normal((101, 16))
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q, K, V, ret)) for r in range(2)]
    for p in procs:
        p.start()
    merged = ret.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A = O.softmax_rows((q[None] @ K.T) / np.sqrt(16))
    assert np.abs(merged[0] - (A @ V)[0]).max() < 1e-5


def test_package_never_imports_the_oracle():
    """The product path has no CPU fallback: nothing in the package (Python or
    CUDA sources) refers to oracle/ or numpy re-implementations of the path."""
    import re
    from pathlib import Path
    pkg = Path(__file__).resolve().parent.parent / "paper_2506_19505_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        src = f.read_text()
        assert not re.search(r"^\s*(import|from)\s+\S*oracle", src, re.M), f
        assert "antkv_oracle" not in src, f
        assert "/root/reference" not in src, f


class _OraclePrefillOps:
    """Block ops restated with the oracle (fp64, per head), so the ring
    schedule, the partial merge and the candidate selection of the sharded
    prefill can run on CPU ranks over gloo."""

    def __init__(self, block=16):
        self.block = block

    def attention_block(self, Q, K, V, qpos, kpos, causal, theta):
        B, Hq, nq, d = Q.shape
        g = Hq // K.shape[1]
        O_, M_, L_, N_ = (np.zeros((B, Hq, nq, d)), np.zeros((B, Hq, nq)), np.zeros((B, Hq, nq)),
                          np.zeros((B, Hq, nq)))
        for b in range(B):
            for h in range(Hq):
                q = Q[b, h].double().numpy()
                Qs = O.apply_rope(q, qpos[b].numpy(), theta) / np.sqrt(d)
                Kr = O.apply_rope(K[b, h // g].double().numpy(), kpos[b].numpy(), theta)
                O_[b, h], L_[b, h], M_[b, h] = O.flash_aux(Qs, Kr, V[b, h // g].double().numpy(),
                                                           self.block, self.block, causal)
                N_[b, h] = np.sqrt((q ** 2).sum(axis=1))
        return tuple(torch.from_numpy(x) for x in (O_, M_, L_, N_))

    def score_block(self, Q, K, qpos, kpos, M, L, qn, causal, theta):
        B, Hq, nq, d = Q.shape
        Hkv, nk = K.shape[1], K.shape[2]
        g = Hq // Hkv
        ak, av = np.zeros((B, Hkv, nk)), np.zeros((B, Hkv, nk))
        for b in range(B):
            for h in range(Hq):
                Qs = O.apply_rope(Q[b, h].double().numpy(), qpos[b].numpy(), theta) / np.sqrt(d)
                Kr = O.apply_rope(K[b, h // g].double().numpy(), kpos[b].numpy(), theta)
                k_, v_ = O.ans_blocked(Qs, Kr, M[b, h].numpy(), L[b, h].numpy(), qn[b, h].numpy(),
                                       self.block, self.block, causal)
                ak[b, h // g] += k_
                av[b, h // g] += v_
        return torch.from_numpy(ak), torch.from_numpy(av)

    def select(self, sk, sv, budget, policy):
        rows = [O.select_anchors(sk[r].double().numpy(), sv[r].double().numpy(), budget, policy)
                for r in range(sk.shape[0])]
        return torch.from_numpy(np.stack(rows)).to(torch.int32)


def _prefill_shard_worker(rank, world, port, Q, K, V, budget, policy, theta, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_19505_b200.parallel import (RingTransport, choose_anchors, shard_candidates,
                                                shard_ranges, sharded_anchor_scores,
                                                sharded_attention)
    ops = _OraclePrefillOps()
    tr = RingTransport()
    B, Hq, n, d = Q.shape
    Hkv = K.shape[1]
    ranges = shard_ranges(n, world)
    s, e = ranges[rank]
    pos = torch.arange(n, dtype=torch.int64)[None].repeat(B, 1)
    Qr, Kr, Vr, pr = Q[:, :, s:e], K[:, :, s:e], V[:, :, s:e], pos[:, s:e].contiguous()

    def like_kv(o):
        m = ranges[o][1] - ranges[o][0]
        return (torch.empty((B, Hkv, m, d), dtype=K.dtype), torch.empty((B, Hkv, m, d), dtype=V.dtype),
                torch.empty((B, m), dtype=torch.int64))

    def like_q(o):
        m = ranges[o][1] - ranges[o][0]
        return (torch.empty((B, Hq, m, d), dtype=Q.dtype), torch.empty((B, m), dtype=torch.int64),
                *[torch.empty((B, Hq, m), dtype=torch.float64) for _ in range(3)])

    Ob, Mb, Lb, qn = sharded_attention(Qr, Kr, Vr, pr, tr.ring((Kr, Vr, pr), like_kv), rank, ops,
                                       theta)
    ak, av = sharded_anchor_scores(Kr, pr, tr.ring((Qr, pr, Mb, Lb, qn), like_q), rank, ops, theta)
    sk, sv, g = shard_candidates(ak.view(B * Hkv, -1), av.view(B * Hkv, -1), budget, s, ops)
    local, glob = choose_anchors(tr.all_gather(sk), tr.all_gather(sv), tr.all_gather(g), budget,
                                 policy, s, e, ops)
    ret.put((rank, Ob.numpy(), Mb.numpy(), Lb.numpy(), ak.numpy(), av.numpy(), local.numpy(),
             glob.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("policy", ["by_sum", "by_k", "by_v"])
def test_sequence_sharded_prefill_gloo_world3(policy):
    """Context-parallel prefill over 3 gloo ranks (FA ring, AnS ring,
    candidate all-gather + global selection) reproduces the unsharded
    reference pipeline: O/M/L/AnS to fp64 rounding, anchors exactly."""
    rng = np.random.default_rng(11)
    B, Hq, Hkv, n, d, theta, budget = 1, 4, 2, 70, 8, 10000.0, 9
    Q = torch.from_numpy(rng.standard_normal((B, Hq, n, d)))
    K = torch.from_numpy(rng.standard_normal((B, Hkv, n, d)))
    V = torch.from_numpy(rng.standard_normal((B, Hkv, n, d)))
    K[0, :, [5, 33, 61]] *= 4.0          # heavy hitters on every shard
    world = 3
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = 29500 + ((os.getpid() + 7 + len(policy)) % 1000)
    procs = [ctx.Process(target=_prefill_shard_worker,
                         args=(r, world, port, Q, K, V, budget, policy, theta, ret))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([ret.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = Hq // Hkv
    pos = np.arange(n)
    from paper_2506_19505_b200.parallel import shard_ranges
    ranges = shard_ranges(n, world)
    ans_k = np.zeros((Hkv, n))
    ans_v = np.zeros((Hkv, n))
    for h in range(Hq):
        q, k, v = Q[0, h].numpy(), K[0, h // g].numpy(), V[0, h // g].numpy()
        Or, Lr, Mr, qn = O.flash_attention_aux(q, k, v, 16, 16, pos, theta, causal=True)
        ak, av = O.anchor_scores_blocked(q, k, Mr, Lr, qn, 16, 16, pos, theta, causal=True)
        ans_k[h // g] += ak
        ans_v[h // g] += av
        for r, (s, e) in enumerate(ranges):
            assert np.abs(res[r][1][0, h] - Or[s:e]).max() < 1e-10
            assert np.abs(res[r][2][0, h] - Mr[s:e]).max() < 1e-10
            assert np.abs(res[r][3][0, h] / Lr[s:e] - 1).max() < 1e-10
    for h in range(Hkv):
        want = O.select_anchors(ans_k[h], ans_v[h], budget, policy)
        for r, (s, e) in enumerate(ranges):
            assert np.abs(res[r][4][0, h] - ans_k[h, s:e]).max() < 1e-9
            assert np.abs(res[r][5][0, h] - ans_v[h, s:e]).max() < 1e-9
            assert res[r][7][h].tolist() == want.tolist()
            loc = res[r][6][h]
            assert [int(j) + s for j in loc if j >= 0] == [int(j) for j in want if s <= j < e]


def test_generate_qkv_matches_reference_streams():
    """The evaluation data generator draws the reference's streams
    (harness.py:35-72): the golden records carry sum(Q) per case."""
    import json
    from fixtures_gen import EVAL_CASES
    from paper_2506_19505_b200.harness import generate_qkv
    g = json.loads((ROOT / "tests" / "golden" / "eval.json").read_text())
    for name, spec in EVAL_CASES.items():
        data = generate_qkv(spec[0], spec[1], spec[2], spec[3])
        assert float(np.asarray(data["Q"], np.float64).sum()) == g[name]["data_Q_sum"]
    hh = generate_qkv(1, 300, 8, "heavy_hitter")
    assert hh["planted"] == [1, 3, 5]


def test_packed_code_units_roundtrip(rng):
    """12-bit packed cache codes (code_bytes = 3): the host pack/unpack pair is
    exact and follows the device layout (unit u at bits [12u, 12u + 12),
    little-endian: common.cuh code_get / code_put_row)."""
    from paper_2506_19505_b200.cache import pack_units, unpack_units
    u = rng.integers(0, 4096, size=4 * 1000).astype(np.uint16)
    raw = pack_units(u, 3)
    assert raw.size == u.size * 3 // 2
    assert np.array_equal(unpack_units(raw, 3), u)
    bits = np.unpackbits(raw, bitorder="little")
    for k in (0, 1, 2, 3, 777, 3999):
        assert int(sum(int(bits[12 * k + i]) << i for i in range(12))) == int(u[k])
    for kind, dt in ((1, np.uint8), (2, np.uint16)):
        v = rng.integers(0, 256 if kind == 1 else 65536, size=64).astype(dt)
        assert np.array_equal(unpack_units(pack_units(v, kind), kind), v)


def test_bench_reference_arm_installs_a_faithful_reference_cache():
    """bench.py's reference arm installs its synthetic state into the
    reference's own QuantizedKVCache (oracle/_ref/pkg, staged from
    /root/reference by oracle/Makefile); its decode steps -- append,
    dequantize, attention, eviction -- equal the oracle restatement holding
    the same state (the port fallback) to 1e-12."""
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    import bench
    mod, kind = bench._reference_module()
    if kind != "reference":
        pytest.skip("oracle/_ref/pkg not built (no /root/reference)")
    import antkv_oracle
    n = 300
    ref = bench._ref_build_cache(mod, "reference", n, "d8m256", 3, 5e5)
    port = bench._ref_build_cache(antkv_oracle, "port", n, "d8m256", 3, 5e5)
    rng = np.random.default_rng(0)
    for s in range(40):                       # past the window: promotions and encodes
        q, k, v = rng.standard_normal((3, bench.D))
        a = ref.decode_step(q, k, v, n + s)
        b = port.decode_step(q[None], k[None], v[None], n + s)[0]
        assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()
    assert list(ref.anchor_indices) == list(port.heads[0].anchor_indices)
    assert ref.kinds == port.heads[0].kinds


def test_bench_reference_arm_runs_without_the_native_library():
    """`bench.py --impl reference` (tiny context) prints one JSON line with
    the same steps / warm-up as requested, kind "reference", and never maps
    this repo's libantkv_b200.so."""
    import subprocess
    if not (ROOT / "oracle" / "_ref" / "pkg" / "antkv" / "cache.py").exists():
        pytest.skip("oracle/_ref/pkg not built (no /root/reference)")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--ctx", "2048",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                         env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["native_so_loaded"] == []
    assert line["value"] > 0


def test_fp64_anchor_score_restatement_matches_oracle():
    """tests/fp64_ans.py (the float64 torch restatement used to check the
    128K prefill anchors on the GPU) against the numpy oracle's GQA prefill
    scores, causal, positions with an offset, several query blocks."""
    import antkv_oracle as O
    from fp64_ans import group_anchor_scores
    rng = np.random.default_rng(3)
    Hq, Hkv, n, d = 4, 2, 300, 32
    Q = rng.standard_normal((Hq, n, d))
    K = rng.standard_normal((Hkv, n, d))
    V = rng.standard_normal((Hkv, n, d))
    pos = np.arange(n) + 17
    ck = rng.standard_normal((Hkv, 16, 8))
    ref = O.OracleCache(ck, ck, anchor_fraction=0.05, window_size=4)
    ref.prefill(Q, K, V, pos)
    sk_ref, sv_ref = ref.last_scores
    g = Hq // Hkv
    for hk in range(Hkv):
        sk, sv = group_anchor_scores(torch.from_numpy(Q[hk * g:(hk + 1) * g]), torch.from_numpy(K[hk]),
                                     torch.from_numpy(pos), block=128)
        assert np.abs(sk.numpy() - sk_ref[hk]).max() <= 1e-12 * np.abs(sk_ref[hk]).max()
        assert np.abs(sv.numpy() - sv_ref[hk]).max() <= 1e-12 * np.abs(sv_ref[hk]).max()
