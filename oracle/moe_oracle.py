"""TEST INFRASTRUCTURE ONLY - CPU oracle for the HarMoEny MoE block.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module, and
only as the checker / timed CPU baseline.  The product package
``paper_2506_12417_b200`` never imports it, and has no CPU fallback.

Two halves:

* Integer scheduling path -> ``liborc_sched.so`` (``sched_oracle.c``), a C
  restatement of ``moesim.policies`` (policies.py:91-171) pinned against the
  reference by the golden fixtures in ``tests/golden`` (made by
  ``tests/golden/make_golden.py`` importing ``/root/reference/pkg/src``).
* Numeric stages that the reference does not implement (it is count-only,
  pkg/README.md:10-12).  Restated here from the paper: Alg. 1 steps 1-6
  (PAPER.md:584-620), expert = x W1 W2, weighted top-k
  combine.  These are *parity unpinned* by any reference
  test; the rounding points mirror the CUDA path (bf16 inputs/weights, fp32
  accumulation, H rounded to bf16, expert output rounded to bf16, fp32 combine
  in fixed slot order, bf16 output).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc_sched.so")
_lib = None


def build() -> str:
    """Compile sched_oracle.c with gcc (seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "sched_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        p64 = ctypes.POINTER(ctypes.c_int64)
        p32 = ctypes.POINTER(ctypes.c_int32)
        L.orc_initial_assign.argtypes = [p64, p64, ctypes.c_int, ctypes.c_int, p64]
        L.orc_rebalance.argtypes = [p64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, p64]
        L.orc_schedule.argtypes = [p64, p64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int, p64, p64]
        L.orc_histogram.argtypes = [p32, ctypes.c_int64, ctypes.c_int, p64]
        L.orc_histogram.restype = None
        L.orc_dispatch_ranks.argtypes = [p32, ctypes.c_int64, p64, ctypes.c_int, ctypes.c_int, ctypes.c_int, p32, p32]
        L.orc_plan_order.argtypes = [p64, p32, ctypes.c_int, p32]
        L.orc_even_split.argtypes = [p64, ctypes.c_int, ctypes.c_int, p64]
        L.orc_even_split.restype = None
        L.orc_affinity.argtypes = [p64, ctypes.c_int, ctypes.c_int, ctypes.c_int, p64]
        L.orc_round_robin.argtypes = [ctypes.c_int, ctypes.c_int, p64]
        L.orc_round_robin.restype = None
        L.orc_blocked.argtypes = [ctypes.c_int, ctypes.c_int, p64]
        L.orc_blocked.restype = None
        _lib = L
    return _lib


def _p64(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _p32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


# --------------------------------------------------------------------------------------------
# integer scheduling path (C)
# --------------------------------------------------------------------------------------------
def round_robin_home(E: int, G: int) -> np.ndarray:
    h = np.empty(E, np.int64)
    lib().orc_round_robin(E, G, _p64(h))
    return h


def blocked_home(E: int, G: int) -> np.ndarray:
    h = np.empty(E, np.int64)
    lib().orc_blocked(E, G, _p64(h))
    return h


def initial_assign(m_all, home) -> np.ndarray:
    m = np.ascontiguousarray(m_all, dtype=np.int64)
    h = np.ascontiguousarray(home, dtype=np.int64)
    G, E = m.shape
    S = np.empty((G, E, G), np.int64)
    if lib().orc_initial_assign(_p64(m), _p64(h), G, E, _p64(S)):
        raise ValueError("placement dimensions do not match routing matrix")
    return S


def rebalance_with_stats(S0, q: int):
    S = np.array(S0, dtype=np.int64, copy=True, order="C")
    G, E, _ = S.shape
    it = np.zeros(1, np.int64)
    if lib().orc_rebalance(_p64(S), G, E, int(q), _p64(it)):
        raise ValueError("token threshold q must be >= 1")
    return S, int(it[0])


def even_split(m_all) -> np.ndarray:
    """even_split_assign (policies.py:174-203)."""
    m = np.ascontiguousarray(m_all, dtype=np.int64)
    G, E = m.shape
    S = np.empty((G, E, G), np.int64)
    lib().orc_even_split(_p64(m), G, E, _p64(S))
    return S


def affinity_home(counts, G: int, slots: int) -> np.ndarray:
    """affinity_placement (policies.py:206-229) -> home[E]."""
    c = np.ascontiguousarray(counts, dtype=np.int64)
    h = np.empty(c.shape[0], np.int64)
    if lib().orc_affinity(_p64(c), c.shape[0], int(G), int(slots), _p64(h)):
        raise ValueError(f"infeasible placement: {c.shape[0]} experts > {G} GPUs x {slots} slots")
    return h


def schedule(m_all, home, q: int, rebalance: bool = True):
    m = np.ascontiguousarray(m_all, dtype=np.int64)
    h = np.ascontiguousarray(home, dtype=np.int64)
    G, E = m.shape
    S = np.empty((G, E, G), np.int64)
    it = np.zeros(1, np.int64)
    rc = lib().orc_schedule(_p64(m), _p64(h), G, E, int(q), int(bool(rebalance)), _p64(S), _p64(it))
    if rc:
        raise ValueError("invalid schedule arguments")
    return S, int(it[0])


def histogram(idx, E: int) -> np.ndarray:
    i = np.ascontiguousarray(idx, dtype=np.int32).reshape(-1)
    h = np.empty(E, np.int64)
    lib().orc_histogram(_p32(i), i.size, E, _p64(h))
    return h


def dispatch_ranks(idx, S, g: int):
    """(dest, rank) per assignment of source g (SURVEY §8(a) A13 contract)."""
    i = np.ascontiguousarray(idx, dtype=np.int32).reshape(-1)
    S = np.ascontiguousarray(S, dtype=np.int64)
    G, E, _ = S.shape
    dest = np.empty(i.size, np.int32)
    rank = np.empty(i.size, np.int32)
    if lib().orc_dispatch_ranks(_p32(i), i.size, _p64(S), g, G, E, _p32(dest), _p32(rank)):
        raise ValueError("schedule does not cover the routed assignments")
    return dest, rank


def plan_order(work, resident) -> np.ndarray:
    w = np.ascontiguousarray(work, dtype=np.int64)
    r = np.ascontiguousarray(resident, dtype=np.int32)
    out = np.empty(w.size, np.int32)
    n = lib().orc_plan_order(_p64(w), _p32(r), w.size, _p32(out))
    return out[:n]


# --------------------------------------------------------------------------------------------
# buffer layouts of the scatter (restatement of the contract the device layout kernel follows)
# --------------------------------------------------------------------------------------------
def _excl_cumsum(a, axis):
    c = np.cumsum(a, axis=axis)
    return c - a


def local_positions(idx_all, S, tokens_per_rank: int):
    """LOCAL layout (all G ranks on one device): buffer [dest][expert][source][rank].
    Returns pos[T, k] (buffer row of every assignment) and segments in plan order."""
    S = np.asarray(S, dtype=np.int64)
    G, E, _ = S.shape
    n = S.sum(axis=0).T  # [d, e]
    base = np.concatenate([[0], np.cumsum(n.sum(axis=1))[:-1]])  # [d]
    off = _excl_cumsum(n, axis=1)  # [d, e]
    src_pre = _excl_cumsum(S, axis=0)  # [g, e, d]: sum_{g'<g} S[g', e, d]
    cum_d = _excl_cumsum(S, axis=2)  # [g, e, d]: sum_{d'<d} S[g, e, d']
    T, k = idx_all.shape
    pos = np.empty((T, k), np.int64)
    for g in range(G):
        sl = slice(g * tokens_per_rank, (g + 1) * tokens_per_rank)
        e = idx_all[sl].astype(np.int64)
        dest, rank = dispatch_ranks(idx_all[sl], S, g)
        dest = dest.reshape(e.shape).astype(np.int64)
        rank = rank.reshape(e.shape).astype(np.int64)
        pos[sl] = base[dest] + off[dest, e] + src_pre[g, e, dest] + rank - cum_d[g, e, dest]
    return pos


def local_segments(S, home):
    S = np.asarray(S, dtype=np.int64)
    G, E, _ = S.shape
    n = S.sum(axis=0).T
    base = np.concatenate([[0], np.cumsum(n.sum(axis=1))[:-1]])
    off = _excl_cumsum(n, axis=1)
    segs = []
    for d in range(G):
        for e in plan_order(n[d], (np.asarray(home) == d).astype(np.int32)):
            segs.append((int(base[d] + off[d, e]), int(n[d, e]), int(e), int(e)))
    return segs


def ep_send_positions(idx_local, S, me: int):
    """EP send buffer of rank `me`: [dest][expert][rank] (NCCL all_to_all chunks)."""
    S = np.asarray(S, dtype=np.int64)
    flows_me = S[me].sum(axis=0)  # [d]
    send_off = np.concatenate([[0], np.cumsum(flows_me)[:-1]])
    pre_e = _excl_cumsum(S[me], axis=0)  # [e, d]
    cum_d = _excl_cumsum(S[me], axis=1)  # [e, d]
    e = idx_local.astype(np.int64)
    dest, rank = dispatch_ranks(idx_local, S, me)
    dest = dest.reshape(e.shape).astype(np.int64)
    rank = rank.reshape(e.shape).astype(np.int64)
    return send_off[dest] + pre_e[e, dest] + rank - cum_d[e, dest]


def ep_recv_segments(S, home, me: int):
    """EP receive buffer of rank `me`: chunks per source g, experts ascending inside a chunk.
    Segments (row_start, nrows, wslot, expert) in plan order of experts, then source."""
    S = np.asarray(S, dtype=np.int64)
    G, E, _ = S.shape
    home = np.asarray(home)
    flows_to_me = S[:, :, me].sum(axis=1)
    chunk_off = np.concatenate([[0], np.cumsum(flows_to_me)[:-1]])
    pre = _excl_cumsum(S[:, :, me], axis=1)  # [g, e]
    n_e = S[:, :, me].sum(axis=0)
    resident = (home == me).astype(np.int32)
    order = plan_order(n_e, resident)
    n_home = int(resident.sum())
    hslot = np.cumsum(resident) - resident
    n_res_work = int(sum(1 for e in order if resident[e]))
    segs = []
    for o, e in enumerate(order):
        wslot = int(hslot[e]) if resident[e] else n_home + (o - n_res_work)
        for g in range(G):
            if S[g, e, me] > 0:
                segs.append((int(chunk_off[g] + pre[g, e]), int(S[g, e, me]), wslot, int(e)))
    return segs


def ep_expert_layout(S, home, me: int, cache_slots: int = 0):
    """HM_LAYOUT_EP_EXPERT (one-sided p2p dispatch): every rank d's receive buffer is
    [expert (ascending)][source][rank].  Returns slot_base [G,E,G] (row of bucket (g,e,d) in d's
    buffer) and rank me's segments (row_start, nrows, wslot, expert), one per expert in plan
    order (residents first, then fetched experts; engine.py:233-234)."""
    S = np.asarray(S, dtype=np.int64)
    G, E, _ = S.shape
    home = np.asarray(home)
    n = S.sum(axis=0).T  # [d, e]
    off = _excl_cumsum(n, axis=1)  # [d, e]
    slot_base = off.T[None, :, :] + _excl_cumsum(S, axis=0)  # [g, e, d]
    resident = (home == me).astype(np.int32)
    order = plan_order(n[me], resident)
    n_home = int(resident.sum())
    hslot = np.cumsum(resident) - resident
    n_res_work = int(sum(1 for e in order if resident[e]))
    segs = []
    for o, e in enumerate(order):
        fi = o - n_res_work
        wslot = int(hslot[e]) if resident[e] else n_home + (fi % cache_slots if cache_slots > 0 else fi)
        segs.append((int(off[me, e]), int(n[me, e]), wslot, int(e)))
    return slot_base, segs


# --------------------------------------------------------------------------------------------
# bf16 helpers (numpy has no bf16): values carried as uint16 bit patterns
# --------------------------------------------------------------------------------------------
def bf16_to_f32(bits) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bits (NaN kept quiet)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32)
    rounding = ((u >> 16) & 1) + np.uint32(0x7FFF)
    out = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_ulp(x) -> np.ndarray:
    """Spacing of bf16 values at |x| (8 significant bits): 2^(floor(log2|x|) - 7); 0 at 0."""
    a = np.abs(np.asarray(x, np.float32))
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    return np.where(a > 0, np.exp2(e - 7), 0.0).astype(np.float32)


def round_bf16(x) -> np.ndarray:
    return bf16_to_f32(f32_to_bf16(x))


# --------------------------------------------------------------------------------------------
# numeric stages (restatement; rounding points mirror the CUDA kernels)
# --------------------------------------------------------------------------------------------
def router(x_bits, wg_bits, bias, k: int, renormalize: bool, idx=None):
    """Step 1.  logits = x Wg^T (+bias) in fp32; top-k over the
    fp32 logits with lowest-index ties; weights = softmax probabilities of the
    selected experts (renormalised over the k when ``renormalize``).  ``idx`` [T, k]
    overrides the selection (the weights are still the oracle's softmax at those experts):
    used to check the rest of the block on tokens whose top-k is an oracle near-tie."""
    x = bf16_to_f32(x_bits)
    wg = bf16_to_f32(wg_bits)
    logits = (x.astype(np.float64) @ wg.T.astype(np.float64)).astype(np.float32)
    if bias is not None:
        logits = (logits + np.asarray(bias, np.float32)[None, :]).astype(np.float32)
    idx = topk_lowest_index(logits, k) if idx is None else np.asarray(idx, np.int64)
    mx = logits.max(axis=1, keepdims=True)
    ex = np.exp((logits - mx).astype(np.float32))
    p = ex / ex.sum(axis=1, keepdims=True, dtype=np.float32)
    w = np.take_along_axis(p, idx, axis=1).astype(np.float32)
    if renormalize:
        w = w / w.sum(axis=1, keepdims=True, dtype=np.float32)
    return logits, idx.astype(np.int32), w.astype(np.float32)


def topk_lowest_index(logits, k: int) -> np.ndarray:
    order = np.argsort(-logits, axis=1, kind="stable")
    return order[:, :k]


def topk_min_gap(logits, k: int) -> np.ndarray:
    """Smallest gap between consecutive sorted logits among the top k+1 per row: the top-k
    SET and ORDER are decided by gaps at least this large (inf when k == E == 1)."""
    s = -np.sort(-np.asarray(logits, np.float64), axis=1)
    kk = min(k + 1, logits.shape[1])
    if kk < 2:
        return np.full(logits.shape[0], np.inf)
    return np.min(s[:, : kk - 1] - s[:, 1:kk], axis=1)


NEAR_TIE_REL = 1e-4  # a top-k decided by a logit gap below this * max(1, max|logit|) is a near tie


def routing_parity(idx_gpu, logits, idx_ref, k: int):
    """Strict routing check (SURVEY.md §7 "Hard parts"): the GPU's top-k must equal the
    oracle's on every token, except tokens whose oracle top-k is decided by a near tie
    (gap < NEAR_TIE_REL * max(1, max|logit|) of the row).  Returns (agree mask, number of
    near-tie tokens, number of disagreeing tokens); raises AssertionError on any
    disagreement outside the near ties."""
    idx_gpu = np.asarray(idx_gpu)
    agree = np.all(idx_gpu == np.asarray(idx_ref), axis=1)
    gap = topk_min_gap(logits, k)
    near = gap < NEAR_TIE_REL * np.maximum(1.0, np.abs(np.asarray(logits, np.float64)).max(axis=1))
    bad = ~agree & ~near
    if bad.any():
        t = int(np.nonzero(bad)[0][0])
        raise AssertionError(f"router: {int(bad.sum())} tokens disagree with the oracle outside near ties "
                             f"(first t={t}: gpu {idx_gpu[t].tolist()} oracle {np.asarray(idx_ref)[t].tolist()}, "
                             f"gap {gap[t]:.3e})")
    return agree, int(near.sum()), int((~agree).sum())


def topk_margin(logits, k: int) -> np.ndarray:
    """Gap between the k-th and (k+1)-th largest logit (inf when k == E)."""
    s = -np.sort(-logits, axis=1)
    if k >= logits.shape[1]:
        return np.full(logits.shape[0], np.inf, np.float32)
    return (s[:, k - 1] - s[:, k]).astype(np.float32)


def expert_ffn(xe_f32, w1_bits, w2_bits, act: str, w3_bits=None):
    """Expert e: act(x W1^T) W2^T (Switch: relu, 2 matrices) or SwiGLU
    (silu(x Wg^T) * (x Wu^T)) Wd^T with W1=gate, W3=up.  H and the output are
    rounded to bf16 like the kernel epilogues."""
    a = xe_f32 @ bf16_to_f32(w1_bits).T
    if act == "swiglu":
        u = xe_f32 @ bf16_to_f32(w3_bits).T
        h = (a / (1.0 + np.exp(-a))) * u
    elif act == "relu":
        h = np.maximum(a, 0.0)
    else:
        raise ValueError(act)
    h = round_bf16(h.astype(np.float32))
    y = h @ bf16_to_f32(w2_bits).T
    return round_bf16(y.astype(np.float32))


def moe_block(x_bits, wg_bits, bias, w1_bits, w2_bits, k, act, renormalize, w3_bits=None, return_scale=False,
              idx=None):
    """Full single-rank block: router -> per-expert FFN -> weighted combine.
    The schedule never changes the math (each token row is computed by its
    expert's weights wherever it runs), so the oracle output is G-independent.
    ``idx`` overrides the routing (see ``router``)."""
    logits, idx, w = router(x_bits, wg_bits, bias, k, renormalize, idx=idx)
    x = bf16_to_f32(x_bits)
    T = x.shape[0]
    E = wg_bits.shape[0]
    d = x.shape[1]
    yk = np.zeros((T, k, d), np.float32)
    for e in range(E):
        sel = np.nonzero(idx == e)
        if sel[0].size == 0:
            continue
        xe = x[sel[0]]
        ye = expert_ffn(xe, w1_bits[e], w2_bits[e], act, None if w3_bits is None else w3_bits[e])
        yk[sel[0], sel[1]] = ye
    acc = np.zeros((T, d), np.float32)
    for j in range(k):
        acc = (acc + w[:, j : j + 1] * yk[:, j, :]).astype(np.float32)
    if return_scale:
        # sum_j |w_j| ulp_bf16(Y_j): one bf16 unit in the last place of every combined expert
        # output.  Each Y_j is an fp32 accumulation rounded to bf16; where the exact value sits
        # within the accumulation-order error of a rounding boundary, kernel and oracle may round
        # it different ways - a one-ulp, order-dependent difference neither side can remove.
        scale = np.einsum("tk,tkd->td", np.abs(w), bf16_ulp(yk)).astype(np.float32)
        return f32_to_bf16(acc), idx, w, logits, scale
    return f32_to_bf16(acc), idx, w, logits
