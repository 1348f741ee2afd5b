"""CPU-only tests: the C-ABI library loads and exports every declared symbol,
the ctypes descriptor matches the C struct layout, host-side logic mirrors the
reference, and the sequence-sharded merge works over a 2-rank gloo group."""

import ctypes
import os
import re
import subprocess
import sys
import tempfile
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
