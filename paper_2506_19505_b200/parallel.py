"""Sequence (context) sharding of the quantised cache across GPUs.

Rank r owns a contiguous token range of every sequence: its codes, anchors
and (on the last rank) the full-precision window that receives appended
tokens.  A decode step runs the local split-KV kernel on every rank, producing
a normalised partial output and its log-sum-exp, all-gathers the partials
(NCCL over NVLink; ~Hq*(d+1)*4 bytes per rank per layer-step) and merges them
with the LSE combine kernel.  This is the only exchange on the decode path
(SURVEY.md §5, §8e).

Prefill shards the same way (context parallelism, SURVEY.md §8e "prefill
partitioning"): the FA pass rings the key/value blocks past every rank and
folds the block partials (O, M, L) online; the AnS pass rings the query
blocks (with their final M, L and ‖q‖) past every rank, each rank summing the
column scores of its own keys; selection all-gathers each shard's candidate
set (its local top-B by each score, with both scores and global indices)
and every rank runs the same selection on the union, which contains every
token the global by_k / by_v / by_sum selection can reach.  Ties keep the
lower global index because the union is laid out in global order.
"""

import numpy as np
import torch
import torch.distributed as dist

from . import _lib

__all__ = ["shard_ranges", "gather_partials", "lse_merge", "ShardedDecoder", "PeerExchange",
           "RingTransport",
           "CudaPrefillOps", "merge_partial", "sharded_attention", "sharded_anchor_scores",
           "shard_candidates", "choose_anchors", "sharded_prefill"]


def shard_ranges(n, world):
    """Contiguous [start, stop) token ranges, sizes differing by at most one."""
    base, extra = divmod(n, world)
    out, s = [], 0
    for r in range(world):
        e = s + base + (1 if r < extra else 0)
        out.append((s, e))
        s = e
    return out


def gather_partials(o, lse, group=None):
    """All-gather (o [rows, d], lse [rows]) -> ([P, rows, d], [P, rows])."""
    world = dist.get_world_size(group)
    o = o.contiguous()
    lse = lse.contiguous()
    # concatenated along dim 0 (the form every backend accepts), then viewed
    o_all = torch.empty((world * o.shape[0],) + tuple(o.shape[1:]), dtype=o.dtype, device=o.device)
    l_all = torch.empty((world * lse.shape[0],) + tuple(lse.shape[1:]), dtype=lse.dtype,
                        device=lse.device)
    dist.all_gather_into_tensor(o_all, o, group=group)
    dist.all_gather_into_tensor(l_all, lse, group=group)
    return o_all.view((world,) + tuple(o.shape)), l_all.view((world,) + tuple(lse.shape))


def lse_merge(o_all, lse_all, out=None, lse_out=None):
    """Merge P normalised partials: out = sum_p w_p o_p, w_p ∝ exp(lse_p)
    (antkv_lse_combine).  GPU only."""
    P, rows, d = o_all.shape[0], int(np.prod(o_all.shape[1:-1])), o_all.shape[-1]
    if out is None:
        out = torch.empty(o_all.shape[1:], dtype=torch.float32, device=o_all.device)
    o_all, lse_all = o_all.contiguous(), lse_all.contiguous()
    _lib.call("antkv_lse_combine", _lib.ptr(o_all), _lib.ptr(lse_all),
              P, rows, d, _lib.ptr(out), _lib.ptr(lse_out), _lib.stream())
    return out


class PeerExchange:
    """Peer-memory exchange of the sequence-shard partials (the NCCL
    all-gather replaced by NVLink stores from the decode kernel itself).

    Every rank allocates receive buffers for all P slots in two halves used
    by alternate steps (o [2][P][rows][d], lse [2][P][rows], flags [2][P]:
    a rank one step ahead never overwrites a slot a slower peer still
    merges); the CUDA IPC handles are all-gathered once and
    each rank maps its peers' buffers.  A step: each rank's decode launch
    stores its partial into its slot of every rank's buffers and releases the
    slot flags with the step's sequence number (antkv_decode_step_publish);
    each rank then merges locally once all flags reached it
    (antkv_lse_merge_wait).  `local_slots` (no process group) emulates P
    ranks inside one process on one buffer set, for tests."""

    def __init__(self, rows, d, group=None, local_slots=None):
        import ctypes
        self.rows, self.d = int(rows), int(d)
        if local_slots is not None:
            self.P, self.rank, distributed = int(local_slots), 0, False
        else:
            self.P, self.rank, distributed = dist.get_world_size(group), dist.get_rank(group), True
        P = self.P
        self._sizes = (2 * P * self.rows * self.d * 4, 2 * P * self.rows * 4, 2 * P * 4)
        nbytes = sum(self._sizes)
        lib = _lib.load()
        base = ctypes.c_void_p()
        _lib.check(lib.antkv_p2p_alloc(nbytes, ctypes.byref(base)))
        self._own = base.value
        self._mapped = []
        bases = [self._own] * P   # local emulation: every "peer" is this buffer (n_dst == P)
        if distributed and P > 1:
            h = (ctypes.c_ubyte * 64)()
            _lib.check(lib.antkv_ipc_get_handle(ctypes.c_void_p(self._own), h))
            handles = [None] * P
            dist.all_gather_object(handles, bytes(h), group=group)
            bases = []
            for r in range(P):
                if r == self.rank:
                    bases.append(self._own)
                    continue
                ptr = ctypes.c_void_p()
                hb = (ctypes.c_ubyte * 64).from_buffer_copy(handles[r])
                _lib.check(lib.antkv_ipc_open_handle(hb, ctypes.byref(ptr)))
                self._mapped.append(ptr.value)
                bases.append(ptr.value)
        dev = torch.device("cuda", torch.cuda.current_device())
        o_off, l_off = 0, self._sizes[0]
        f_off = l_off + self._sizes[1]
        self.dst_o = torch.tensor([b + o_off for b in bases], dtype=torch.int64, device=dev)
        self.dst_lse = torch.tensor([b + l_off for b in bases], dtype=torch.int64, device=dev)
        self.dst_flags = torch.tensor([b + f_off for b in bases], dtype=torch.int64, device=dev)
        self.n_dst = len(bases)
        self._recv = (self._own + o_off, self._own + l_off, self._own + f_off)
        self.seq = 0

    def advance(self):
        """Start the next step (its flags carry the new sequence number)."""
        self.seq = (self.seq + 1) & 0xFFFFFFFF or 1   # 0 is the flags' initial value
        return self.seq

    def merge(self, out, lse_out=None):
        """Wait for every slot of this step, merge into out [rows, d] float32."""
        o, l, f = self._recv
        lib = _lib.load(check_device=False)
        _lib.check(lib.antkv_lse_merge_wait(o, l, f, self.P, self.seq, self.rows, self.d, _lib.ptr(out),
                                            _lib.ptr(lse_out), _lib.stream()))
        return out

    def close(self):
        lib = _lib.load(check_device=False)
        torch.cuda.synchronize()
        for p in self._mapped:
            lib.antkv_ipc_close_handle(p)
        self._mapped = []
        if self._own:
            lib.antkv_p2p_free(self._own)
            self._own = None


class ShardedDecoder:
    """Decode driver for one rank's shard.

    ``cache`` holds this rank's token range (its ``desc.token_offset`` is the
    global index of its first slot).  Only the tail rank (``is_tail``) appends
    and evicts; every rank attends.  ``combine`` defaults to the GPU LSE merge;
    tests may pass another merge to exercise the collective on CPU/gloo."""

    def __init__(self, cache, is_tail, group=None, combine=None, exchange=None):
        self.cache = cache
        self.is_tail = is_tail
        self.group = group
        self.combine = combine or lse_merge
        self.exchange = exchange

    def step(self, q, k, v, qpos, out_local, lse_local):
        """q [B, Hq, d], k/v [B, Hkv, d] (only used on the tail), qpos [B].
        The tail shard appends, attends and evicts in one fused launch
        (antkv_decode_step with the log-sum-exp output); the others attend.
        With a PeerExchange the same launch publishes the partial to every
        rank over peer memory and the merge waits on the slot flags; without
        one the partials are all-gathered with NCCL."""
        c = self.cache
        if self.exchange is not None:
            ex = self.exchange
            ex.advance()
            c.step_publish(q, k if self.is_tail else None, v if self.is_tail else None, qpos,
                           out_local, lse_local, ex)
            if self.is_tail:
                c._n += 1
            return ex.merge(torch.empty_like(out_local).view(-1, out_local.shape[-1])).view_as(out_local)
        if self.is_tail:
            c.step_device(q, k, v, qpos, out_local, lse_local)
            c._n += 1
        else:
            c.attend_device(q, qpos, out_local, lse_local)
        o_all, l_all = gather_partials(out_local, lse_local, self.group)
        return self.combine(o_all, l_all)


# ------------------------------------------------------------------ prefill
class RingTransport:
    """Blocks travel rank r -> r+1 over the process group; while the caller
    computes on the block it was handed, the next one is already in flight
    (one batched isend/irecv per step).  NCCL moves device tensors directly;
    other backends (gloo, CPU tests) stage through host memory."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._device_ok = dist.get_backend(group) == "nccl"

    def _peer(self, r):
        return r if self.group is None else dist.get_global_rank(self.group, r)

    def _exchange(self, send, recv):
        dst = self._peer((self.rank + 1) % self.world)
        src = self._peer((self.rank - 1) % self.world)
        if self._device_ok:
            stage_s, stage_r = [t.contiguous() for t in send], list(recv)
        else:
            stage_s = [t.detach().cpu().contiguous() for t in send]
            stage_r = [torch.empty(t.shape, dtype=t.dtype) for t in recv]
        ops = [dist.P2POp(dist.isend, t, dst, self.group) for t in stage_s]
        ops += [dist.P2POp(dist.irecv, t, src, self.group) for t in stage_r]
        return dist.batch_isend_irecv(ops), stage_r

    def ring(self, local, like):
        """Yield (origin, block) for origin = r, r-1, ..., r-P+1 (mod P).
        `local` is this rank's block (a tuple of tensors), `like(origin)`
        returns empty tensors shaped as that origin's block."""
        cur = tuple(local)
        for s in range(self.world):
            pending = None
            if s < self.world - 1:
                nxt = like((self.rank - s - 1) % self.world)
                pending = (nxt,) + self._exchange(cur, nxt)
            yield (self.rank - s) % self.world, cur
            if pending is not None:
                nxt, works, staged = pending
                for w in works:
                    w.wait()
                if not self._device_ok:
                    for dst_t, src_t in zip(nxt, staged):
                        dst_t.copy_(src_t)
                cur = nxt

    def all_gather(self, t):
        """[*shape] -> [P, *shape]."""
        t = t.contiguous()
        src = t if self._device_ok else t.cpu()
        out = torch.empty((self.world * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype,
                          device=src.device)
        dist.all_gather_into_tensor(out, src, group=self.group)
        return out.view((self.world,) + tuple(src.shape)).to(t.device)


class CudaPrefillOps:
    """Per-block prefill kernels (antkv_prefill_attention_block,
    antkv_prefill_anchor_scores_block, antkv_select_anchors)."""

    @staticmethod
    def _tag(*ts):
        tag = _lib.dtype_tag(ts[0])
        if any(_lib.dtype_tag(t) != tag for t in ts[1:]):
            raise ValueError("Q, K and V must share one dtype")
        return tag

    def attention_block(self, Q, K, V, qpos, kpos, causal, theta):
        B, Hq, nq, d = Q.shape
        Hkv, nk = K.shape[1], K.shape[2]
        O = torch.empty((B, Hq, nq, d), dtype=torch.float32, device=Q.device)
        M = torch.empty((B, Hq, nq), dtype=torch.float32, device=Q.device)
        L = torch.empty_like(M)
        qn = torch.empty_like(M)
        _lib.call("antkv_prefill_attention_block", _lib.ptr(Q), _lib.ptr(K), _lib.ptr(V),
                  self._tag(Q, K, V), _lib.ptr(qpos), _lib.ptr(kpos), B, Hq, Hkv, nq, nk, d,
                  float(theta), int(bool(causal)), _lib.ptr(O), _lib.ptr(M), _lib.ptr(L),
                  _lib.ptr(qn), _lib.stream())
        return O, M, L, qn

    def score_block(self, Q, K, qpos, kpos, M, L, qn, causal, theta):
        M, L, qn = M.contiguous(), L.contiguous(), qn.contiguous()
        B, Hq, nq, d = Q.shape
        Hkv, nk = K.shape[1], K.shape[2]
        ak = torch.empty((B, Hkv, nk), dtype=torch.float32, device=K.device)
        av = torch.empty_like(ak)
        _lib.call("antkv_prefill_anchor_scores_block", _lib.ptr(Q), _lib.ptr(K), self._tag(Q, K),
                  _lib.ptr(qpos), _lib.ptr(kpos), _lib.ptr(M), _lib.ptr(L), _lib.ptr(qn),
                  B, Hq, Hkv, nq, nk, d,
                  float(theta), int(bool(causal)), _lib.ptr(ak), _lib.ptr(av), _lib.stream())
        return ak, av

    def select(self, sk, sv, budget, policy):
        from .anchors import select_anchors_device
        return select_anchors_device(sk.contiguous(), sv.contiguous(), int(budget), policy)


def merge_partial(acc, part):
    """Fold a block partial (O, M, L) into the running one: the softmax over
    the union of the two key sets (normalised O, M = max scaled logit, L =
    sum of exp(s - M))."""
    if acc is None:
        return part
    O1, M1, L1 = acc
    O2, M2, L2 = part
    M = torch.maximum(M1, M2)
    a1 = L1 * torch.exp(M1 - M)
    a2 = L2 * torch.exp(M2 - M)
    L = a1 + a2
    O = (O1 * a1[..., None] + O2 * a2[..., None]) / L[..., None]
    return O, M, L


def sharded_attention(Q, K, V, pos, ring, rank, ops, theta):
    """FA pass on rank `rank`: Q [B, Hq, n_r, d] against every key block
    of ranks <= rank (causal on the diagonal).  `ring` yields (origin,
    (K_o, V_o, pos_o)).  Returns (O, M, L, q_norms) of the local queries."""
    acc, qn = None, None
    for o, (Ko, Vo, po) in ring:
        if o > rank:
            continue
        O, M, L, qn_b = ops.attention_block(Q, Ko, Vo, pos, po, o == rank, theta)
        acc = merge_partial(acc, (O, M, L))
        if o == rank:
            qn = qn_b
    return acc[0], acc[1], acc[2], qn


def sharded_anchor_scores(K, pos, ring, rank, ops, theta):
    """AnS pass on rank `rank`: the column scores of the local keys
    [B, Hkv, n_r] summed over every query block of ranks >= rank.  `ring`
    yields (origin, (Q_o, pos_o, M_o, L_o, qn_o))."""
    ak = av = None
    for o, (Qo, po, Mo, Lo, qno) in ring:
        if o < rank:
            continue
        bk, bv = ops.score_block(Qo, K, po, pos, Mo, Lo, qno, o == rank, theta)
        ak = bk if ak is None else ak + bk
        av = bv if av is None else av + bv
    return ak, av


def shard_candidates(ak, av, budget, start, ops):
    """One shard's selection candidates: the union of its local top-budget by
    ans_k and by ans_v, in ascending index order, padded to 2*budget with
    score -1 / index -1.  ak/av [R, n_r] -> (sk, sv float32, gidx int64)
    [R, 2*budget].  (Scores are nonnegative, so padding never wins.)"""
    R, n = ak.shape
    c = min(int(budget), n)
    width = 2 * int(budget)
    sk = torch.full((R, width), -1.0, dtype=torch.float32, device=ak.device)
    sv = torch.full_like(sk, -1.0)
    gidx = torch.full((R, width), -1, dtype=torch.int64, device=ak.device)
    if c == 0:
        return sk, sv, gidx
    ik = ops.select(ak, ak, c, "by_k").long()
    iv = ops.select(av, av, c, "by_v").long()
    cand, _ = torch.cat([ik, iv], 1).sort(1)
    dup = torch.zeros_like(cand, dtype=torch.bool)
    dup[:, 1:] = cand[:, 1:] == cand[:, :-1]
    cand, _ = torch.where(dup, n, cand).sort(1)
    valid = cand < n
    safe = cand.clamp(max=n - 1)
    w = cand.shape[1]
    sk[:, :w] = torch.where(valid, ak.float().gather(1, safe), -1.0)
    sv[:, :w] = torch.where(valid, av.float().gather(1, safe), -1.0)
    gidx[:, :w] = torch.where(valid, cand + int(start), -1)
    return sk, sv, gidx


def choose_anchors(sk_all, sv_all, g_all, budget, policy, start, stop, ops):
    """Global selection from every shard's candidates ([P, R, C] each, rank
    order): the policy runs on the union laid out in global index order, so
    ties resolve to the lower global index as in anchors.py:90-93.  Returns
    (local int32 [R, A] sorted, -1 padded; global int64 [R, budget])."""
    P, R, C = sk_all.shape
    SK = sk_all.permute(1, 0, 2).reshape(R, P * C).contiguous()
    SV = sv_all.permute(1, 0, 2).reshape(R, P * C).contiguous()
    G = g_all.permute(1, 0, 2).reshape(R, P * C)
    sel = ops.select(SK, SV, int(budget), policy).long()
    glob = G.gather(1, sel)
    mine = (glob >= start) & (glob < stop)
    big = torch.iinfo(torch.int64).max
    local, _ = torch.where(mine, glob - start, big).sort(1)
    width = max(int(mine.sum(1).max()) if R else 0, 1)
    local = local[:, :width]
    local = torch.where(local == big, -1, local).to(torch.int32)
    return local, glob


def sharded_prefill(cache, Q, K, V, positions, start, n_total, transport, is_tail, ops=None):
    """Context-parallel prefill of one rank's shard [start, start + n_r) of
    every sequence: FA ring, AnS ring, global anchor selection, and the
    shard's cache layout (cache.py:100-140 over the whole sequence).  The
    cache must be empty and created with token_offset=start (window 0 on
    non-tail ranks).  Returns the shard's full-precision output
    O [B, Hq, n_r, d] float32."""
    ops = ops or CudaPrefillOps()
    B, Hq, n, d = Q.shape
    Hkv = K.shape[1]
    theta = float(cache.config.theta_base)
    pos = positions.contiguous()
    ranges = shard_ranges(n_total, transport.world)
    if ranges[transport.rank] != (start, start + n):
        raise ValueError("shard does not match shard_ranges(n_total, world)")
    dev = Q.device

    def like_kv(o):
        m = ranges[o][1] - ranges[o][0]
        return (torch.empty((B, Hkv, m, d), dtype=K.dtype, device=dev),
                torch.empty((B, Hkv, m, d), dtype=V.dtype, device=dev),
                torch.empty((B, m), dtype=torch.int64, device=dev))

    O, M, L, qn = sharded_attention(Q, K, V, pos, transport.ring((K, V, pos), like_kv),
                                    transport.rank, ops, theta)

    def like_q(o):
        m = ranges[o][1] - ranges[o][0]
        return (torch.empty((B, Hq, m, d), dtype=Q.dtype, device=dev),
                torch.empty((B, m), dtype=torch.int64, device=dev),
                torch.empty((B, Hq, m), dtype=torch.float32, device=dev),
                torch.empty((B, Hq, m), dtype=torch.float32, device=dev),
                torch.empty((B, Hq, m), dtype=torch.float32, device=dev))

    ak, av = sharded_anchor_scores(K, pos, transport.ring((Q, pos, M, L, qn), like_q),
                                   transport.rank, ops, theta)
    budget = int(cache.config.budget_for(n_total))
    sk, sv, g = shard_candidates(ak.view(B * Hkv, n), av.view(B * Hkv, n), budget, start,
                                ops)
    local, _ = choose_anchors(transport.all_gather(sk), transport.all_gather(sv),
                              transport.all_gather(g), budget, cache.config.policy, start,
                              start + n, ops)
    cache.Hq, cache.Hkv = Hq, Hkv
    cache.build_from(K, V, pos, local.view(B, Hkv, -1))
    if is_tail:
        # promotions on the tail follow the global anchor count
        cache.tensors["hstate"][:, :, _lib.HS_ANCHORS] = budget
    cache.last_scores = (ak, av)
    return O
