"""Golden fixture for BASELINE config #1 at its real shape: one LLaMA-3-8B
attention layer (32 Q / 8 KV heads, d = 128), a 2048-token prefill and 128
decode steps, d8m256 (1-bit) K/V codes, 1 % anchors (by_sum), window 32.

Produced by the CPU oracle (oracle/antkv_oracle.py), whose single-head path
is pinned bit-for-bit to the reference package (tests/test_oracle.py against
tests/golden/*.npz written by make_golden.py) and whose GQA rule (one anchor
set per KV head from the group-summed scores) is SURVEY.md §7 hard part 7.
The reference itself is single-head, so this is the GQA restatement run at
the reference's algorithm: cache.py:100-194 per KV head.

    python tests/golden/make_config1_golden.py      # ~35 s, writes config1.npz

Inputs are regenerated from CONFIG1 (tests/fixtures_gen.py); only outputs
are stored: per-head anchor sets and kinds before / after decode, every
token's K/V code indices after decode (prefill codes are unchanged by
decode, so the evicted tokens' codes are the rows whose kind changed), the
float64 anchor scores (for the float32-margin rule), a strided sample of the
prefill output rows and all 128 decode outputs (float32).
"""

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent / "oracle"))

import antkv_oracle as O  # noqa: E402
from fixtures_gen import CONFIG1, codebooks, qkv  # noqa: E402

KIND = {"anchor": 0, "quantized": 1, "windowed": 2}


def main():
    t0 = time.time()
    c = CONFIG1
    Q, K, V = qkv(c["seed"], c["Hq"], c["Hkv"], c["n"] + c["steps"], c["d"], heavy=c["heavy"])
    ck, cv = codebooks(c["seed"], c["Hkv"], 256, 8)
    ref = O.OracleCache(ck, cv, anchor_fraction=c["frac"], window_size=c["window"],
                        policy=c["policy"], theta_base=c["theta"])
    n = c["n"]
    Op = ref.prefill(Q[:, :n], K[:, :n], V[:, :n], np.arange(n))
    sk, sv = ref.last_scores
    anchors0 = np.stack([h.anchor_indices for h in ref.heads])
    kinds0 = np.array([[KIND[k] for k in h.kinds] for h in ref.heads], dtype=np.uint8)
    print(f"prefill {time.time() - t0:.1f} s", flush=True)
    outs = []
    for t in range(n, n + c["steps"]):
        outs.append(ref.decode_step(Q[:, t], K[:, t], V[:, t], t))
    print(f"decode {time.time() - t0:.1f} s", flush=True)
    N = ref.token_count
    G = c["d"] // 8
    codes1 = np.zeros((c["Hkv"], N, 2, G), dtype=np.uint8)
    for hk, h in enumerate(ref.heads):
        for j, code in h.k_codes.items():
            codes1[hk, j, 0] = code
            codes1[hk, j, 1] = h.v_codes[j]
    kinds1 = np.array([[KIND[k] for k in h.kinds] for h in ref.heads], dtype=np.uint8)
    amax = max(len(h.anchor_indices) for h in ref.heads)
    anchors1 = np.full((c["Hkv"], amax), -1, dtype=np.int64)
    for hk, h in enumerate(ref.heads):
        anchors1[hk, :len(h.anchor_indices)] = h.anchor_indices
    rows = np.unique(np.concatenate([np.arange(0, n, c["o_stride"]), [n - 1]]))
    np.savez_compressed(
        HERE / "config1.npz",
        scores_k=sk, scores_v=sv, anchors0=anchors0, kinds0=kinds0, kinds1=kinds1,
        anchors1=anchors1, codes1=codes1, prefill_rows=rows,
        prefill_O=Op[:, rows].astype(np.float32), decode_out=np.array(outs, dtype=np.float32),
        mem=np.array([ref.memory_report(h)[0] for h in range(c["Hkv"])], dtype=np.int64))
    print(f"wrote {HERE / 'config1.npz'} in {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
