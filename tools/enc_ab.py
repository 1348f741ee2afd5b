"""A/B the encoders of two library builds on the same random bf16 rows:
python tools/enc_ab.py LIB_A LIB_B (codes must be identical)."""
import ctypes, os, subprocess, sys, json
import numpy as np
if len(sys.argv) == 4:    # child: encode with one library, print codes checksum + codes
    lib_path, notation, out = sys.argv[1:]
    os.environ["ANTKV_LIB"] = lib_path
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    from paper_2506_19505_b200 import VqConfig, _lib
    vq = VqConfig.from_notation(notation)
    g = torch.Generator(device="cuda").manual_seed(11)
    n = 65536
    X = torch.randn((n, 128), device="cuda", generator=g).to(torch.bfloat16)
    C = torch.randn((vq.m, vq.d_sub), device="cuda", generator=g)
    cb = 1 if vq.m <= 256 else 2
    codes = torch.empty((n, (128 // vq.d_sub) * cb), dtype=torch.uint8, device="cuda")
    _lib.call("antkv_vq_encode", _lib.ptr(X), _lib.BF16, n, 128, _lib.ptr(C), vq.m, vq.d_sub, _lib.ptr(codes),
              cb, _lib.stream())
    np.save(out, codes.cpu().numpy())
    sys.exit(0)
a, b = sys.argv[1:3]
for nt in ["d8m256", "d4m256", "d32m4096", "d16m256"]:
    outs = []
    for i, lib in enumerate((a, b)):
        f = f"/tmp/enc_ab_{i}.npy"
        subprocess.run([sys.executable, __file__, lib, nt, f], check=True)
        outs.append(np.load(f))
    print(nt, "identical" if np.array_equal(*outs) else f"DIFFER in {(outs[0] != outs[1]).any(1).sum()} rows")
