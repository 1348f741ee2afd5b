"""CPU oracle for the AnTKV anchor-token sub-bit KV-cache path.

TEST INFRASTRUCTURE ONLY.  This module is a plain-numpy restatement of the
reference algorithm (``/root/reference/pkg/src/antkv``, arXiv 2506.19505).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (and ``bench.py --impl reference``) may import it, and only as the
checker / the timed CPU arm.  The product package ``paper_2506_19505_b200``
never imports it and has no CPU fallback.

Parity pinning: every function below is checked against golden vectors that
were produced by running the reference package itself in the build container
(``tests/golden/make_golden.py``) and, where available, against the
reference's compiled Cython kernels built from the reference sources by
``oracle/Makefile`` into ``oracle/_ref`` (``tests/test_oracle.py``).

Extension beyond the single-head reference (GQA): the reference is
single-head.  ``OracleCache`` keeps one cache state per KV head
and selects that head's anchors from the anchor scores summed over the Q heads
of its group.  AnS is a sum over query rows (anchors.py:61-62), so for a
group size of 1 this is exactly the reference; the tests check that
bit-for-bit against ``QuantizedKVCache``.
"""

import math

import numpy as np

__all__ = [
    "rope_trig", "apply_rope", "softmax_rows", "flash_aux", "ans_blocked",
    "assign_nearest", "encode_rows", "decode_rows", "ranked", "select_anchors",
    "budget_for", "index_bits", "pack_indices", "unpack_indices",
    "attention_exact", "OracleCache", "KIND_ANCHOR", "KIND_QUANTIZED",
    "KIND_WINDOWED", "POLICIES", "weighted_kmeans",
]

POLICIES = ("by_k", "by_v", "by_sum")          # anchors.py:29
KIND_ANCHOR = "anchor"                         # cache.py:24-26
KIND_QUANTIZED = "quantized"
KIND_WINDOWED = "windowed"


# --------------------------------------------------------------------- RoPE
def rope_trig(positions, d, theta_base):
    """cos/sin of positions * theta_base**(-2i/d) in float64.
    Follows attention.py:82-86 (_rope_trig)."""
    half = d // 2
    freqs = theta_base ** (-2.0 * np.arange(half) / d)
    angles = np.asarray(positions, dtype=np.int64)[:, None].astype(np.float64) * freqs[None, :]
    return np.cos(angles), np.sin(angles)


def apply_rope(X, positions, theta_base=10000.0, sign=1.0):
    """Interleaved-pair rotation (2i, 2i+1).  attention.py:89-106."""
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    cos, sin = rope_trig(np.asarray(positions)[:n], d, theta_base)
    sin = sign * sin
    x0 = X[:, 0::2]
    x1 = X[:, 1::2]
    out = np.empty_like(X)
    out[:, 0::2] = x0 * cos - x1 * sin
    out[:, 1::2] = x0 * sin + x1 * cos
    return out


def softmax_rows(M, causal=False):
    """Row softmax with max subtraction.  attention.py:70-79."""
    M = np.asarray(M, dtype=np.float64)
    if causal:
        n_q, n_k = M.shape
        mask = np.arange(n_k)[None, :] > np.arange(n_q)[:, None]
        M = np.where(mask, -np.inf, M)
    m = M.max(axis=1, keepdims=True)
    P = np.exp(M - m)
    return P / P.sum(axis=1, keepdims=True)


def attention_exact(Q, K, V, positions=None, theta_base=10000.0, causal=False):
    """Unblocked attention (attention.py:121-143)."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    if positions is not None:
        Q = apply_rope(Q, positions, theta_base)
        K = apply_rope(K, positions, theta_base)
    logits = (Q @ K.T) / np.sqrt(Q.shape[1])
    return softmax_rows(logits, causal=causal) @ np.asarray(V, dtype=np.float64)


# ------------------------------------------------------- blocked attention
def flash_aux(Qs, Kr, V, block_q, block_k, causal):
    """Blocked online-softmax attention returning (O, L, M).
    Same block order as kernels/pure.py:13-52 and _ckernels.pyx:10-88:
    query blocks outer, key blocks inner; M is the max scaled logit and L the
    normaliser at M."""
    Qs = np.ascontiguousarray(Qs, dtype=np.float64)
    Kr = np.ascontiguousarray(Kr, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    n_q, d = Qs.shape
    n_k = Kr.shape[0]
    O = np.zeros((n_q, V.shape[1]))
    L = np.zeros(n_q)
    M = np.full(n_q, -np.inf)
    for q0 in range(0, n_q, block_q):
        q1 = min(q0 + block_q, n_q)
        m_run = np.full(q1 - q0, -np.inf)
        l_run = np.zeros(q1 - q0)
        acc = np.zeros((q1 - q0, V.shape[1]))
        for k0 in range(0, n_k, block_k):
            if causal and k0 > q1 - 1:
                break
            k1 = min(k0 + block_k, n_k)
            S = Qs[q0:q1] @ Kr[k0:k1].T
            if causal:
                S = np.where(np.arange(k0, k1)[None, :] <= np.arange(q0, q1)[:, None], S, -np.inf)
            m_new = np.maximum(m_run, S.max(axis=1))
            with np.errstate(invalid="ignore"):
                alpha = np.where(m_run == -np.inf, 0.0, np.exp(m_run - m_new))
            P = np.exp(S - m_new[:, None])
            l_run = l_run * alpha + P.sum(axis=1)
            acc = acc * alpha[:, None] + P @ V[k0:k1]
            m_run = m_new
        O[q0:q1] = acc / l_run[:, None]
        L[q0:q1] = l_run
        M[q0:q1] = m_run
    return O, L, M


def ans_blocked(Qs, Kr, M, L, q_norms, block_q, block_k, causal):
    """Alg. 1 second pass: A = exp(S - M_i)/L_i rebuilt blockwise, key blocks
    outer; ans_v = sum_i A_ij, ans_k = sum_i A_ij (1 - A_ij) ||Q_i||.
    kernels/pure.py:55-81, _ckernels.pyx:91-131."""
    Qs = np.ascontiguousarray(Qs, dtype=np.float64)
    Kr = np.ascontiguousarray(Kr, dtype=np.float64)
    M = np.asarray(M, dtype=np.float64)
    L = np.asarray(L, dtype=np.float64)
    q_norms = np.asarray(q_norms, dtype=np.float64)
    n_q = Qs.shape[0]
    n_k = Kr.shape[0]
    ans_k = np.zeros(n_k)
    ans_v = np.zeros(n_k)
    for k0 in range(0, n_k, block_k):
        k1 = min(k0 + block_k, n_k)
        for q0 in range(0, n_q, block_q):
            q1 = min(q0 + block_q, n_q)
            if causal and k0 > q1 - 1:
                continue
            S = Qs[q0:q1] @ Kr[k0:k1].T
            if causal:
                S = np.where(np.arange(k0, k1)[None, :] <= np.arange(q0, q1)[:, None], S, -np.inf)
            A = np.exp(S - M[q0:q1, None]) / L[q0:q1, None]
            ans_v[k0:k1] += A.sum(axis=0)
            ans_k[k0:k1] += (A * (1.0 - A) * q_norms[q0:q1, None]).sum(axis=0)
    return ans_k, ans_v


def flash_attention_aux(Q, K, V, block_q, block_k, positions=None, theta_base=10000.0,
                        causal=False):
    """attention.py:146-169: rotate, scale Q by 1/sqrt(d), blocked pass, and
    q_norms from the PRE-RoPE queries (attention.py:167)."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    if positions is not None:
        Qr, Kr = apply_rope(Q, positions, theta_base), apply_rope(K, positions, theta_base)
    else:
        Qr, Kr = Q, K
    Qs = Qr / np.sqrt(Q.shape[1])
    O, L, M = flash_aux(Qs, Kr, V, block_q, block_k, causal)
    q_norms = np.sqrt((Q ** 2).sum(axis=1))
    return O, L, M, q_norms


def anchor_scores_blocked(Q, K, M, L, q_norms, block_q, block_k, positions=None,
                          theta_base=10000.0, causal=False):
    """anchors.py:66-87."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    if positions is not None:
        Qr, Kr = apply_rope(Q, positions, theta_base), apply_rope(K, positions, theta_base)
    else:
        Qr, Kr = Q, K
    Qs = Qr / np.sqrt(Q.shape[1])
    return ans_blocked(Qs, Kr, M, L, q_norms, block_q, block_k, causal)


# ---------------------------------------------------------------------- VQ
def index_bits(m):
    """vq.py:49-51."""
    return max(1, math.ceil(math.log2(m))) if m > 1 else 1


def assign_nearest(X, C):
    """Exact float64 sum_t (x_t - c_t)^2, accumulated over t in order (as
    _ckernels.pyx:150-162 does), strict-< argmin so ties go to the lowest
    index.  Vectorised over points in chunks."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    C = np.ascontiguousarray(C, dtype=np.float64)
    n, d = X.shape
    m = C.shape[0]
    idx = np.empty(n, dtype=np.int64)
    d2 = np.empty(n, dtype=np.float64)
    chunk = max(1, int(2 ** 22 // max(1, m)))
    for s in range(0, n, chunk):
        e = min(s + chunk, n)
        acc = np.zeros((e - s, m))
        for t in range(d):
            diff = X[s:e, t][:, None] - C[None, :, t]
            acc += diff * diff
        best = np.argmin(acc, axis=1)          # first minimum == lowest index
        idx[s:e] = best
        d2[s:e] = acc[np.arange(e - s), best]
    return idx, d2


def encode_rows(X, centroids):
    """vq.py:218-232: split each row into d/d_sub sub-vectors and assign."""
    X = np.asarray(X, dtype=np.float64)
    m, d_sub = centroids.shape
    n, d = X.shape
    if d % d_sub:
        raise ValueError(f"d={d} not divisible by d_sub={d_sub}")
    idx, _ = assign_nearest(X.reshape(n * (d // d_sub), d_sub),
                            np.asarray(centroids, dtype=np.float32).astype(np.float64))
    return idx.reshape(n, -1)


def decode_rows(codes, centroids):
    """vq.py:243-248 (float32 gather)."""
    codes = np.asarray(codes)
    C = np.asarray(centroids, dtype=np.float32)
    if np.any(codes < 0) or np.any(codes >= C.shape[0]):
        raise ValueError("code index out of range")
    n = codes.shape[0]
    return C[codes.reshape(-1)].reshape(n, -1)


def _pp_seed(X, w, m, rng):
    """Weighted k-means++ (vq.py:120-138): the first centre drawn with
    probability w/sum(w), each later one with probability w*D^2/sum(w*D^2)
    (uniform index when that sum is zero); D^2 = squared distance to the
    nearest centre chosen so far."""
    C = np.empty((m, X.shape[1]))
    C[0] = X[rng.choice(len(X), p=w / w.sum())]
    D2 = ((X - C[0]) ** 2).sum(axis=1)
    for k in range(1, m):
        s = w * D2
        tot = s.sum()
        j = int(rng.integers(len(X))) if tot <= 0 else rng.choice(len(X), p=s / tot)
        C[k] = X[j]
        D2 = np.minimum(D2, ((X - C[k]) ** 2).sum(axis=1))
    return C


def weighted_kmeans(X, w, m, seed, max_iter=100, tol=1e-10, init_centroids=None):
    """vq.py:141-214 with this module's assign_nearest (the compiled
    backend's operation order).  Returns (centroids float32 [m, d],
    objective trace, iterations, padded_init)."""
    X = np.asarray(X, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    n, d = X.shape
    rng = np.random.default_rng(seed)
    padded = False
    if init_centroids is not None:                       # vq.py:164-167
        C = np.array(init_centroids, dtype=np.float64)
    elif m > n:                                          # vq.py:168-174
        padded = True
        scale = max(np.abs(X).max(), 1.0)
        reps = np.tile(X, (m // n + 1, 1))[: m - n]
        C = np.concatenate([X, reps + rng.normal(scale=1e-6 * scale, size=(m - n, d))])
    else:
        C = _pp_seed(X, w, m, rng)
    trace, prev, it = [], None, 0
    for it in range(1, max_iter + 1):                    # vq.py:178-197
        idx, d2 = assign_nearest(X, C)
        trace.append(float((w * d2).sum()))
        wsum = np.zeros(m)
        csum = np.zeros((m, d))
        wx = w[:, None] * X
        for j in range(n):                               # point order, as add.at
            wsum[idx[j]] += w[j]
            csum[idx[j]] += wx[j]
        Cn = C.copy()
        live = wsum > 0
        Cn[live] = csum[live] / wsum[live, None]
        wd2 = w * d2
        for e in np.flatnonzero(~live):                  # empty-cluster repair
            far = int(np.argmax(wd2))
            Cn[e] = X[far]
            wd2[far] = -1.0
        stop = (prev is not None and np.array_equal(idx, prev)) or \
            (len(trace) >= 2 and trace[-2] - trace[-1] < tol)
        C, prev = Cn, idx
        if stop:
            break
    return C.astype(np.float32), trace, it, padded


def pack_indices(indices, bits):
    """Big-endian bitstream padded to a byte (util.py:19-36)."""
    acc = 0
    nbits = 0
    out = bytearray()
    for v in indices:
        v = int(v)
        if v < 0 or v >= (1 << bits):
            raise ValueError(f"index {v} does not fit in {bits} bits")
        acc = (acc << bits) | v
        nbits += bits
        while nbits >= 8:
            nbits -= 8
            out.append((acc >> nbits) & 0xFF)
    if nbits:
        out.append((acc << (8 - nbits)) & 0xFF)
    return bytes(out)


def unpack_indices(data, bits, count):
    """util.py:39-53."""
    out = np.empty(count, dtype=np.int64)
    acc = 0
    nbits = 0
    pos = 0
    for i in range(count):
        while nbits < bits:
            acc = (acc << 8) | data[pos]
            pos += 1
            nbits += 8
        nbits -= bits
        out[i] = (acc >> nbits) & ((1 << bits) - 1)
        acc &= (1 << nbits) - 1
    return out


# ---------------------------------------------------------------- anchors
def ranked(scores):
    """Descending score, ties to the lower index (anchors.py:90-93)."""
    n = len(scores)
    return np.lexsort((np.arange(n), -np.asarray(scores, dtype=np.float64)))


def select_anchors(ans_k, ans_v, budget, policy="by_sum"):
    """anchors.py:96-132.  Returns sorted int64 indices."""
    if policy not in POLICIES:
        raise ValueError(f"unknown policy {policy!r}")
    n = len(ans_v)
    budget = int(np.clip(budget, 0, n))
    if policy == "by_k":
        chosen = ranked(ans_k)[:budget]
    elif policy == "by_v":
        chosen = ranked(ans_v)[:budget]
    else:
        by_k = ranked(ans_k)
        by_v = ranked(ans_v)
        picked = list(by_k[: budget // 2])
        seen = set(int(j) for j in picked)
        for j in by_v:
            if len(picked) >= budget:
                break
            if int(j) not in seen:
                picked.append(j)
                seen.add(int(j))
        for j in by_k:
            if len(picked) >= budget:
                break
            if int(j) not in seen:
                picked.append(j)
                seen.add(int(j))
        chosen = np.asarray(picked, dtype=np.int64)
    return np.sort(np.asarray(chosen, dtype=np.int64))


def budget_for(n, anchor_fraction=0.01, anchor_count=None):
    """cache.py:54-57."""
    if anchor_count is not None:
        return int(np.clip(anchor_count, 0, n))
    return int(np.clip(math.ceil(anchor_fraction * n), 0, n))


# ------------------------------------------------------------------ cache
class _HeadState:
    """One KV head of one sequence: the reference QuantizedKVCache state
    (cache.py:83-90) with dense dequantised rows kept incrementally."""

    def __init__(self):
        self.kinds = []
        self.k_rows = {}
        self.v_rows = {}
        self.k_codes = {}
        self.v_codes = {}
        self.anchor_indices = np.empty(0, dtype=np.int64)
        # dense dequantised rows (what dequantize() reassembles every call,
        # cache.py:196-211), kept up to date as tokens change kind
        self.Khat = np.zeros((0, 0), dtype=np.float32)
        self.Vhat = np.zeros((0, 0), dtype=np.float32)

    def set_row(self, j, k, v):
        if j >= self.Khat.shape[0]:
            grow = max(j + 1, 2 * self.Khat.shape[0], 64)
            d = len(k)
            K2 = np.zeros((grow, d), dtype=np.float32)
            V2 = np.zeros((grow, d), dtype=np.float32)
            if self.Khat.size:
                K2[:self.Khat.shape[0]] = self.Khat
                V2[:self.Vhat.shape[0]] = self.Vhat
            self.Khat, self.Vhat = K2, V2
        self.Khat[j] = k
        self.Vhat[j] = v


class OracleCache:
    """GQA restatement of QuantizedKVCache (cache.py:68-243).

    Q has H_q heads, K/V have H_kv heads, H_q % H_kv == 0; Q head h attends
    KV head h // (H_q // H_kv).  Codebooks are per KV head:
    ``codebooks_k[h]`` is a float32 [m, d_sub] array."""

    def __init__(self, codebooks_k, codebooks_v, anchor_fraction=0.01,
                 anchor_count=None, window_size=32, policy="by_sum",
                 theta_base=10000.0, block_q=64, block_k=64):
        self.cb_k = [np.asarray(c, dtype=np.float32) for c in codebooks_k]
        self.cb_v = [np.asarray(c, dtype=np.float32) for c in codebooks_v]
        self.h_kv = len(self.cb_k)
        self.m, self.d_sub = self.cb_k[0].shape
        self.anchor_fraction = anchor_fraction
        self.anchor_count = anchor_count
        self.window_size = window_size
        self.policy = policy
        self.theta_base = theta_base
        self.block_q = block_q
        self.block_k = block_k
        self.positions = []
        self.heads = [_HeadState() for _ in range(self.h_kv)]
        self.d = None
        self.last_scores = None

    @property
    def token_count(self):
        return len(self.positions)

    def budget_for(self, n):
        return budget_for(n, self.anchor_fraction, self.anchor_count)

    # cache.py:100-140
    def prefill(self, Q, K, V, positions, anchors=None, codes=None):
        """``anchors`` (test hook, not in the reference): per-KV-head index
        arrays that replace the selection -- the FA + AnS passes are then
        skipped and None is returned.  Used to replay the reference's layout,
        decode and eviction from another implementation's anchor set when
        the two sets legitimately differ at the float32 margin.  ``codes``
        (test hook): per-KV-head (k_codes, v_codes) int arrays [n, groups]
        used instead of encoding the rows (for long contexts whose codes
        are checked separately, on a sample, by the margin rule)."""
        K = np.asarray(K, dtype=np.float64)
        V = np.asarray(V, dtype=np.float64)
        h_kv, n, d = K.shape
        self.d = d
        positions = np.asarray(positions, dtype=np.int64)
        O = None
        if anchors is None:
            Q = np.asarray(Q, dtype=np.float64)
            h_q = Q.shape[0]
            group = h_q // self.h_kv
            O = np.empty((h_q, n, d))
            ans_k = np.zeros((self.h_kv, n))
            ans_v = np.zeros((self.h_kv, n))
            for hq in range(h_q):
                hk = hq // group
                O[hq], L, M, qn = flash_attention_aux(
                    Q[hq], K[hk], V[hk], self.block_q, self.block_k,
                    positions=positions, theta_base=self.theta_base, causal=True)
                sk, sv = anchor_scores_blocked(
                    Q[hq], K[hk], M, L, qn, self.block_q, self.block_k,
                    positions=positions, theta_base=self.theta_base, causal=True)
                ans_k[hk] += sk
                ans_v[hk] += sv
            self.last_scores = (ans_k, ans_v)
            budget = self.budget_for(n)
        K32 = K.astype(np.float32)
        V32 = V.astype(np.float32)
        self.positions = [int(p) for p in positions]
        for hk in range(self.h_kv):
            st = self.heads[hk]
            if anchors is None:
                st.anchor_indices = select_anchors(ans_k[hk], ans_v[hk], budget, self.policy)
            else:
                st.anchor_indices = np.sort(np.asarray(anchors[hk], dtype=np.int64))
            anchor_set = set(int(j) for j in st.anchor_indices)
            if codes is None:
                kc = encode_rows(K[hk], self.cb_k[hk])
                vc = encode_rows(V[hk], self.cb_v[hk])
            else:
                kc, vc = (np.asarray(x, dtype=np.int64) for x in codes[hk])
            Kd = decode_rows(kc, self.cb_k[hk])
            Vd = decode_rows(vc, self.cb_v[hk])
            for j in range(n):
                if j in anchor_set:
                    st.kinds.append(KIND_ANCHOR)
                    st.k_rows[j] = K32[hk, j].copy()
                    st.v_rows[j] = V32[hk, j].copy()
                    st.set_row(j, K32[hk, j], V32[hk, j])
                elif j >= n - self.window_size:
                    st.kinds.append(KIND_WINDOWED)
                    st.k_rows[j] = K32[hk, j].copy()
                    st.v_rows[j] = V32[hk, j].copy()
                    st.set_row(j, K32[hk, j], V32[hk, j])
                else:
                    st.kinds.append(KIND_QUANTIZED)
                    st.k_codes[j] = kc[j]
                    st.v_codes[j] = vc[j]
                    st.set_row(j, Kd[j], Vd[j])
        return O

    def dequantize(self, hk):
        """cache.py:196-211 for KV head hk: anchors and window exact, the
        rest decoded from their codes (decode_rows).  The rows are kept
        assembled as tokens change kind (_HeadState.set_row) instead of
        being re-gathered token by token on every call."""
        st = self.heads[hk]
        n = self.token_count
        return st.Khat[:n].copy(), st.Vhat[:n].copy()

    # cache.py:149-194
    def decode_step(self, q, k, v, position):
        if self.positions and position <= max(self.positions):
            raise ValueError("position must exceed all existing positions")
        q = np.asarray(q, dtype=np.float64)
        h_q = q.shape[0]
        group = h_q // self.h_kv
        if self.d is None:
            self.d = q.shape[1]
        j = self.token_count
        self.positions.append(int(position))
        for hk in range(self.h_kv):
            st = self.heads[hk]
            st.kinds.append(KIND_WINDOWED)
            st.k_rows[j] = np.asarray(k[hk], dtype=np.float32).copy()
            st.v_rows[j] = np.asarray(v[hk], dtype=np.float32).copy()
            st.set_row(j, st.k_rows[j], st.v_rows[j])
        out = np.empty((h_q, self.d))
        pos = np.asarray(self.positions, dtype=np.int64)
        for hk in range(self.h_kv):
            Khat, Vhat = self.dequantize(hk)
            Kr = apply_rope(Khat.astype(np.float64), pos, self.theta_base)
            for hq in range(hk * group, (hk + 1) * group):
                qr = apply_rope(q[hq][None, :], np.asarray([position]), self.theta_base)
                logits = (qr @ Kr.T) / np.sqrt(self.d)
                A = softmax_rows(logits)
                out[hq] = (A @ Vhat.astype(np.float64))[0]
        for hk in range(self.h_kv):
            self._evict(hk)
        return out

    def _evict(self, hk):
        st = self.heads[hk]
        windowed = [t for t, kind in enumerate(st.kinds) if kind == KIND_WINDOWED]
        while len(windowed) > self.window_size:
            evicted = windowed.pop(0)
            if len(st.anchor_indices) < self.budget_for(self.token_count):
                st.kinds[evicted] = KIND_ANCHOR
                st.anchor_indices = np.sort(np.append(st.anchor_indices, evicted))
            else:
                st.k_codes[evicted] = encode_rows(
                    st.k_rows.pop(evicted).astype(np.float64)[None, :], self.cb_k[hk])[0]
                st.v_codes[evicted] = encode_rows(
                    st.v_rows.pop(evicted).astype(np.float64)[None, :], self.cb_v[hk])[0]
                st.kinds[evicted] = KIND_QUANTIZED
                st.set_row(evicted, decode_rows(st.k_codes[evicted][None, :], self.cb_k[hk])[0],
                           decode_rows(st.v_codes[evicted][None, :], self.cb_v[hk])[0])

    def attention_from_cache(self, Q):
        """cache.py:213-223 per Q head (materialised causal softmax)."""
        Q = np.asarray(Q, dtype=np.float64)
        h_q = Q.shape[0]
        group = h_q // self.h_kv
        pos = np.asarray(self.positions, dtype=np.int64)
        out = np.empty((h_q, Q.shape[1], self.d))
        for hq in range(h_q):
            Khat, Vhat = self.dequantize(hq // group)
            Kr = apply_rope(Khat.astype(np.float64), pos, self.theta_base)
            Qr = apply_rope(Q[hq], pos, self.theta_base)
            A = softmax_rows((Qr @ Kr.T) / np.sqrt(self.d), causal=True)
            out[hq] = A @ Vhat.astype(np.float64)
        return out

    def memory_report(self, hk=0):
        """cache.py:225-243 for one KV head: (payload, codebook, eff, fp)."""
        st = self.heads[hk]
        bits = index_bits(self.m)
        groups = self.d // self.d_sub
        payload = sum(2 * groups * bits if k == KIND_QUANTIZED else 2 * self.d * 32
                      for k in st.kinds)
        denom = 2 * self.token_count * self.d
        return payload, 2 * self.m * self.d_sub * 32, payload / denom, denom * 32
