"""Torch-tensor wrappers over the C ABI (device memory + streams are torch's;
the compute is libharmoe.so).  Every function is stream-ordered on the current
torch CUDA stream unless ``stream`` is given, allocates only its outputs, and
never synchronises the host.
"""

from __future__ import annotations

import torch

from . import _lib
from ._lib import (  # noqa: F401
    HM_EPI_RELU,
    HM_EPI_STORE,
    HM_EPI_SWIGLU,
    HM_LAYOUT_EP,
    HM_LAYOUT_EP_EXPERT,
    HM_LAYOUT_LOCAL,
    HM_POLICY_EVEN_SPLIT,
    HM_POLICY_NONE,
    HM_POLICY_REBALANCE,
)

TILE_M = 128


def _require_cuda(*tensors):
    for t in tensors:
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError("harmoe ops need CUDA tensors (no CPU fallback)")
        if not t.is_contiguous():
            raise ValueError("harmoe ops need contiguous tensors")


def _require_dtype(dtype, *tensors, what: str = "tensor"):
    for t in tensors:
        if t is not None and t.dtype != dtype:
            raise ValueError(f"{what} must be {dtype}, got {t.dtype}")


def _policy(rebalance) -> int:
    """bool (rebalance on/off) or an HM_POLICY_* code -> the C ABI's policy argument."""
    if isinstance(rebalance, bool):
        return HM_POLICY_REBALANCE if rebalance else HM_POLICY_NONE
    code = int(rebalance)
    if code not in (HM_POLICY_NONE, HM_POLICY_REBALANCE, HM_POLICY_EVEN_SPLIT):
        raise ValueError(f"unknown scheduling policy code {code}")
    return code


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def e_pad(E: int) -> int:
    return (E + 15) // 16 * 16


def router_topk(x, wg, bias, n_ranks: int, tokens_per_rank: int, k: int, renormalize: bool, E: int | None = None,
                stream=None):
    """K1+K2.  x [n_ranks*T_g, d] bf16, wg [E_pad, d] bf16 (rows >= E are zero padding), bias [E] fp32|None.
    Returns topk_idx [T,k] i32, topk_w [T,k] f32, tile_hist [tiles, E] i32, lrank [T,k] i32."""
    _require_cuda(x, wg, bias)
    if x.dtype != torch.bfloat16 or wg.dtype != torch.bfloat16:
        raise ValueError("router expects bf16 x and wg")
    T, d = x.shape
    if T != n_ranks * tokens_per_rank:
        raise ValueError("x rows must equal n_ranks * tokens_per_rank")
    if E is None:
        E = bias.numel() if bias is not None else wg.shape[0]
    if bias is not None and bias.numel() != E:
        raise ValueError("bias must have E entries")
    if wg.shape[0] != e_pad(E) or wg.shape[1] != d:
        raise ValueError(f"wg must be [E_pad={e_pad(E)}, d]")
    tiles = n_ranks * ((tokens_per_rank + TILE_M - 1) // TILE_M)
    dev = x.device
    idx = torch.empty((T, k), dtype=torch.int32, device=dev)
    w = torch.empty((T, k), dtype=torch.float32, device=dev)
    tile_hist = torch.empty((tiles, E), dtype=torch.int32, device=dev)
    lrank = torch.empty((T, k), dtype=torch.int32, device=dev)
    _lib.call("hm_router_topk", _ptr(x), _ptr(wg), _ptr(bias), n_ranks, tokens_per_rank, d, E, k,
              int(bool(renormalize)), _ptr(idx), _ptr(w), _ptr(tile_hist), _ptr(lrank), _stream(stream))
    return idx, w, tile_hist, lrank


def hist_scan(tile_hist, n_ranks: int, tiles_per_rank: int, stream=None):
    """Per-rank histogram m_expert [n_ranks, E] + per-tile exclusive offsets."""
    _require_cuda(tile_hist)
    E = tile_hist.shape[1]
    hist = torch.empty((n_ranks, E), dtype=torch.int32, device=tile_hist.device)
    tile_off = torch.empty_like(tile_hist)
    _lib.call("hm_hist_scan", _ptr(tile_hist), n_ranks, tiles_per_rank, E, _ptr(hist), _ptr(tile_off),
              _stream(stream))
    return hist, tile_off


def schedule(m_all, home, q: int, rebalance: bool = True, stream=None):
    """K3: S [G,E,G] i32, iters [1] i32, loads [G] i32 — all on device."""
    _require_cuda(m_all, home)
    if m_all.dtype != torch.int32 or home.dtype != torch.int32:
        raise ValueError("schedule expects int32 m_all and home")
    G, E = m_all.shape
    dev = m_all.device
    S = torch.empty((G, E, G), dtype=torch.int32, device=dev)
    iters = torch.empty(1, dtype=torch.int32, device=dev)
    loads = torch.empty(G, dtype=torch.int32, device=dev)
    _lib.call("hm_schedule", _ptr(m_all), _ptr(home), G, E, int(q), _policy(rebalance), _ptr(S), _ptr(iters),
              _ptr(loads), _stream(stream))
    return S, iters, loads


def schedule_batched(m_all, home, q: int, rebalance: bool = True, stream=None):
    """K3 over B instances in one launch: m_all [B,G,E] i32 -> S [B,G,E,G], iters [B], loads [B,G]."""
    _require_cuda(m_all, home)
    if m_all.dtype != torch.int32 or home.dtype != torch.int32:
        raise ValueError("schedule expects int32 m_all and home")
    B, G, E = m_all.shape
    dev = m_all.device
    S = torch.empty((B, G, E, G), dtype=torch.int32, device=dev)
    iters = torch.empty(B, dtype=torch.int32, device=dev)
    loads = torch.empty((B, G), dtype=torch.int32, device=dev)
    _lib.call("hm_schedule_batched", _ptr(m_all), _ptr(home), B, G, E, int(q), _policy(rebalance), _ptr(S),
              _ptr(iters), _ptr(loads), _stream(stream))
    return S, iters, loads


def rebalance_(S, q: int, stream=None):
    """In-place rebalance of S [G,E,G] i32; returns (iters, loads) device tensors."""
    _require_cuda(S)
    if S.dtype != torch.int32:
        raise ValueError("rebalance expects int32 S")
    G, E, _ = S.shape
    iters = torch.empty(1, dtype=torch.int32, device=S.device)
    loads = torch.empty(G, dtype=torch.int32, device=S.device)
    _lib.call("hm_rebalance", _ptr(S), G, E, int(q), _ptr(iters), _ptr(loads), _stream(stream))
    return iters, loads


class Layout:
    """Device-side result of hm_dispatch_layout."""

    __slots__ = ("slot_base", "segs", "n_seg", "mtile_prefix", "fetch", "n_fetch")

    def __init__(self, slot_base, segs, n_seg, mtile_prefix, fetch, n_fetch):
        self.slot_base, self.segs, self.n_seg = slot_base, segs, n_seg
        self.mtile_prefix, self.fetch, self.n_fetch = mtile_prefix, fetch, n_fetch


def dispatch_layout(S, home, mode: int, me: int = 0, cache_slots: int = 0, stream=None) -> Layout:
    _require_cuda(S, home)
    G, E, _ = S.shape
    dev = S.device
    cap = G * E
    slot_base = torch.zeros((G, E, G), dtype=torch.int32, device=dev)
    segs = torch.empty((cap, 4), dtype=torch.int32, device=dev)
    n_seg = torch.empty(1, dtype=torch.int32, device=dev)
    mprefix = torch.empty(cap + 1, dtype=torch.int32, device=dev)
    fetch = torch.empty(E, dtype=torch.int32, device=dev)
    n_fetch = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.call("hm_dispatch_layout", _ptr(S), _ptr(home), G, E, int(mode), int(me), _ptr(slot_base), _ptr(segs),
              _ptr(n_seg), _ptr(mprefix), _ptr(fetch), _ptr(n_fetch), int(cache_slots), _stream(stream))
    return Layout(slot_base, segs, n_seg, mprefix, fetch, n_fetch)


class Plan:
    """Device-side result of hm_plan (m_all, tile offsets, schedule, layout)."""

    __slots__ = ("m_all", "tile_off", "S", "iters", "loads", "layout")

    def __init__(self, m_all, tile_off, S, iters, loads, layout):
        self.m_all, self.tile_off, self.S, self.iters, self.loads, self.layout = m_all, tile_off, S, iters, loads, layout


def plan(home, G: int, E: int, q: int, rebalance: bool, mode: int, me: int = 0, tile_hist=None,
         tiles_per_rank: int = 0, m_all=None, cache_slots: int = 0, stream=None) -> Plan:
    """Fused planner: (hist reduce) + schedule + layout in one launch."""
    _require_cuda(home, tile_hist, m_all)
    dev = home.device
    i32 = dict(dtype=torch.int32, device=dev)
    m_out = torch.empty((G, E), **i32) if tile_hist is not None else m_all
    tile_off = torch.empty_like(tile_hist) if tile_hist is not None else None
    S = torch.empty((G, E, G), **i32)
    iters = torch.empty(1, **i32)
    loads = torch.empty(G, **i32)
    cap = G * E
    # slot_base rows the permute reads (every source in LOCAL, row `me` in EP) are all written
    lay = Layout(torch.empty((G, E, G), **i32), torch.empty((cap, 4), **i32), torch.empty(1, **i32),
                 torch.empty(cap + 1, **i32), torch.empty(E, **i32), torch.empty(1, **i32))
    _lib.call("hm_plan", _ptr(tile_hist), int(tiles_per_rank), _ptr(m_all), _ptr(home), G, E, int(q),
              _policy(rebalance), int(mode), int(me), _ptr(m_out) if tile_hist is not None else None,
              _ptr(tile_off), _ptr(S), _ptr(iters), _ptr(loads), _ptr(lay.slot_base), _ptr(lay.segs),
              _ptr(lay.n_seg), _ptr(lay.mtile_prefix), _ptr(lay.fetch), _ptr(lay.n_fetch), int(cache_slots),
              _stream(stream))
    return Plan(m_out, tile_off, S, iters, loads, lay)


class PushList:
    """Device-side push work list of hm_plan_dispatch (expert-ordered dispatch)."""

    __slots__ = ("items", "cprefix", "ebase")

    def __init__(self, items, cprefix, ebase):
        self.items, self.cprefix, self.ebase = items, cprefix, ebase


def plan_dispatch(home, G: int, E: int, q: int, rebalance, me: int, m_all, cache_slots: int = 0,
                  stream=None) -> tuple[Plan, PushList]:
    """hm_plan (EP_EXPERT layout of rank ``me`` from the all-gathered m_all) plus this rank's push
    work list in every destination's plan order (hm_dispatch_push_ordered)."""
    _require_cuda(home, m_all)
    dev = home.device
    i32 = dict(dtype=torch.int32, device=dev)
    S = torch.empty((G, E, G), **i32)
    iters = torch.empty(1, **i32)
    loads = torch.empty(G, **i32)
    cap = G * E
    lay = Layout(torch.empty((G, E, G), **i32), torch.empty((cap, 4), **i32), torch.empty(1, **i32),
                 torch.empty(cap + 1, **i32), torch.empty(E, **i32), torch.empty(1, **i32))
    pl = PushList(torch.empty((cap, 4), **i32), torch.empty(cap + 1, **i32), torch.empty(E + 1, **i32))
    _lib.call("hm_plan_dispatch", _ptr(m_all), _ptr(home), G, E, int(q), _policy(rebalance), int(me), _ptr(S),
              _ptr(iters), _ptr(loads), _ptr(lay.slot_base), _ptr(lay.segs), _ptr(lay.n_seg), _ptr(lay.mtile_prefix),
              _ptr(lay.fetch), _ptr(lay.n_fetch), int(cache_slots), _ptr(pl.items), _ptr(pl.cprefix), _ptr(pl.ebase),
              _stream(stream))
    return Plan(m_all, None, S, iters, loads, lay), pl


def dispatch_push_ordered(x, topk_idx, lrank, tile_off, S, slot_base, push: PushList, me: int, dst_rows, dst_tok,
                          dst_arrive, order, sync, pos=None, stream=None):
    """Expert-ordered fused scatter + dispatch: the rows of hm_dispatch_push (EP_EXPERT layout)
    in every destination's plan order, 8-row units (one warp each), each followed by a system-scope add of its
    row count to the destination's arrival counter dst_arrive[d][expert]."""
    _require_cuda(x, topk_idx, lrank, tile_off, S, slot_base, dst_rows, dst_tok, dst_arrive, order, sync, pos)
    T, d = x.shape
    k = topk_idx.shape[1]
    G, E, _ = S.shape
    _lib.call("hm_dispatch_push_ordered", _ptr(x), _ptr(topk_idx), _ptr(lrank), _ptr(tile_off), _ptr(S),
              _ptr(slot_base), _ptr(push.items), _ptr(push.cprefix), _ptr(push.ebase), T, int(me), G, E, k, d,
              _ptr(dst_rows), _ptr(dst_tok), _ptr(dst_arrive), _ptr(order), _ptr(pos), _ptr(sync), _stream(stream))


def grouped_gemm_arrive(A, W, N: int, layout: "Layout", epilogue: int, a_arrive, out=None, slot_ready=None,
                        ready_from_slot: int = 0, epoch: int = 0, slot_done=None, fetch=None, pdl: bool = True,
                        stream=None):
    """K5 over an expert-major receive buffer whose rows are still arriving: each segment's
    producer waits until a_arrive[expert] >= its rows; pdl launches it behind the push kernel."""
    _require_cuda(A, W, a_arrive, slot_ready, slot_done)
    _require_dtype(torch.int32, a_arrive, what="arrival counters")
    rows, K = A.shape
    ncols = N // 2 if epilogue == HM_EPI_SWIGLU else N
    if out is None:
        out = torch.empty((max(rows, 1), ncols), dtype=torch.bfloat16, device=A.device)
    _lib.call("hm_grouped_gemm_arrive", _ptr(A), rows, _ptr(W), W.shape[0], N, K, _ptr(layout.segs),
              _ptr(layout.n_seg), _ptr(layout.mtile_prefix), int(epilogue), _ptr(out), _ptr(slot_ready),
              int(ready_from_slot), int(epoch), _ptr(slot_done), _fetch_ref(fetch), _ptr(a_arrive), int(bool(pdl)),
              _stream(stream))
    return out


def permute(x, topk_idx, lrank, tile_off, S, slot_base, n_ranks: int, tokens_per_rank: int, src_rank_base: int,
            out_rows: int, out=None, with_inverse: bool = False, index_only: bool = False, stream=None):
    """K4.  Returns (out [out_rows, d] bf16 | None, pos [T,k] i32, inv [out_rows] i32 | None).
    index_only: no row copies (the FFN1 GEMM gathers rows through inv)."""
    _require_cuda(x, topk_idx, lrank, tile_off, S, slot_base)
    _require_dtype(torch.bfloat16, x, out, what="permute rows")
    _require_dtype(torch.int32, topk_idx, lrank, tile_off, S, slot_base, what="permute index tensors")
    T, d = x.shape
    k = topk_idx.shape[1]
    G, E, _ = S.shape
    if index_only:
        out = None
        with_inverse = True
    elif out is None:
        out = torch.empty((max(out_rows, 1), d), dtype=x.dtype, device=x.device)
    pos = torch.empty((T, k), dtype=torch.int32, device=x.device)
    inv = torch.empty(max(out_rows, 1), dtype=torch.int32, device=x.device) if with_inverse else None
    _lib.call("hm_permute", _ptr(x), _ptr(topk_idx), _ptr(lrank), _ptr(tile_off), _ptr(S), _ptr(slot_base),
              n_ranks, tokens_per_rank, src_rank_base, G, E, k, d, _ptr(out), _ptr(pos), _ptr(inv), _stream(stream))
    return out, pos, inv


def grouped_gemm(A, W, N: int, layout_or_segs, epilogue: int, out=None, row_map=None, slot_ready=None,
                 ready_from_slot: int = 0, epoch: int = 0, a_gather=None, a_gather_div: int = 1, out_rows=None,
                 slot_done=None, fetch=None, stream=None):
    """K5.  A [rows, K] bf16, W [slots*N, K] bf16 -> out [rows, N or N/2] bf16
    (row r written to row_map[r] when a row map is given).  With a_gather, buffer row r
    reads A[a_gather[r] // a_gather_div] (cp.async loader warps in the 2-CTA kernel, TMA
    gather4 in the 1-CTA one) and out has ``out_rows`` rows."""
    if isinstance(layout_or_segs, Layout):
        segs, n_seg, mprefix = layout_or_segs.segs, layout_or_segs.n_seg, layout_or_segs.mtile_prefix
    else:
        segs, n_seg, mprefix = layout_or_segs
    _require_cuda(A, W, segs, n_seg, mprefix, slot_ready, row_map, a_gather, slot_done)
    _require_dtype(torch.bfloat16, A, W, out, what="grouped_gemm operands")
    _require_dtype(torch.int32, segs, n_seg, mprefix, row_map, a_gather, slot_ready, slot_done,
                   what="grouped_gemm index tensors")
    rows, K = A.shape
    if a_gather is not None:
        rows_out = out_rows if out_rows is not None else a_gather.numel()
    else:
        rows_out = rows
    ncols = N // 2 if epilogue == HM_EPI_SWIGLU else N
    if out is None:
        out = torch.empty((max(rows_out, 1), ncols), dtype=torch.bfloat16, device=A.device)
    _lib.call("hm_grouped_gemm", _ptr(A), rows, _ptr(W), W.shape[0], N, K, _ptr(segs), _ptr(n_seg), _ptr(mprefix),
              int(epilogue), _ptr(out), _ptr(row_map), _ptr(a_gather), int(a_gather_div), _ptr(slot_ready),
              int(ready_from_slot), int(epoch), _ptr(slot_done), _fetch_ref(fetch), _stream(stream))
    return out


def grouped_gemm_swap(A, W, N: int, layout: "Layout", epilogue: int, out=None, row_map=None, topk_w=None,
                      residual=None, y=None, stream=None):
    """K5 with swap-AB tiles (weights on the MMA's M, 64 token rows on N) for weight-streaming
    shapes.  With topk_w (top-1, STORE): returns y = (residual +) w * row at row_map (combine
    fused, bit-identical); else returns out [rows, N]."""
    segs, n_seg = (layout.segs, layout.n_seg) if isinstance(layout, Layout) else (layout[0], layout[1])
    _require_cuda(A, W, row_map, topk_w, residual, y, out, segs, n_seg)
    _require_dtype(torch.bfloat16, A, W, out, y, residual, what="grouped_gemm_swap operands")
    rows, K = A.shape
    if topk_w is not None:
        _require_dtype(torch.float32, topk_w, what="combine weights")
        if topk_w.dim() > 1 and topk_w.shape[-1] != 1:
            raise ValueError("grouped_gemm_swap: the fused combine is the top-1 one")
        if y is None:
            y = torch.empty((topk_w.shape[0], N), dtype=torch.bfloat16, device=A.device)
    elif out is None:
        out = torch.empty((max(rows, 1), N), dtype=torch.bfloat16, device=A.device)
    _lib.call("hm_grouped_gemm_swap", _ptr(A), rows, _ptr(W), W.shape[0], N, K, _ptr(segs), _ptr(n_seg),
              int(epilogue), _ptr(out), _ptr(row_map), _ptr(topk_w), _ptr(residual), _ptr(y), _stream(stream))
    return y if topk_w is not None else out


def grouped_gemm_combine(H, W, N: int, layout: "Layout", row_map, topk_w, counters, Y=None, y=None, residual=None,
                         stream=None):
    """K5 (FFN2, STORE epilogue, token-major scatter through row_map) with K7 fused into the
    epilogue: returns (Y [T*k, N], y [T, N]) where y = (residual +) sum_j w[t,j] Y[t*k+j] is
    bit-identical to combine(Y, None, topk_w, residual=residual).  counters: int32 [T * N/64],
    zero before the first call (every call leaves them zero).  Top-1 (k == 1): the epilogue writes
    y directly (no counters, Y not written: returned as None)."""
    _require_cuda(H, W, row_map, topk_w, counters, residual, Y, y)
    _require_dtype(torch.bfloat16, H, W, Y, y, residual, what="grouped_gemm_combine operands")
    _require_dtype(torch.float32, topk_w, what="combine weights")
    _require_dtype(torch.int32, row_map, counters, what="grouped_gemm_combine index tensors")
    T, k = topk_w.shape
    if k != 1 and (counters is None or counters.numel() < T * (N // 64)):
        raise ValueError("grouped_gemm_combine: counters must hold T * N/64 entries")
    if Y is None and k != 1:
        Y = torch.empty((max(T * k, 1), N), dtype=torch.bfloat16, device=H.device)
    if y is None:
        y = torch.empty((T, N), dtype=torch.bfloat16, device=H.device)
    _lib.call("hm_grouped_gemm_combine", _ptr(H), H.shape[0], _ptr(W), W.shape[0], N, H.shape[1], _ptr(layout.segs),
              _ptr(layout.n_seg), _ptr(layout.mtile_prefix), _ptr(Y), _ptr(row_map), _ptr(topk_w), k,
              _ptr(residual), _ptr(y), _ptr(counters), _stream(stream))
    return Y, y


def fetch_plan(fetch, n_fetch, src_in, src_out, dst_in, dst_out, in_bytes: int, out_bytes: int, first_slot: int,
               n_slots: int, ready_in, ready_out, counters, value: int, phase: int, pairs: int = 2):
    """hm_fetch_plan for the K6 fetch pairs of a grouped-GEMM launch (bounded expert cache):
    phase 1 = the FFN1 launch, 2 = the FFN2 launch.  Keep the returned object alive until the
    launch call returns (the struct is copied into the kernel parameters)."""
    _require_cuda(fetch, n_fetch, src_in, src_out, dst_in, dst_out, ready_in, ready_out, counters)
    _require_dtype(torch.int32, fetch, n_fetch, ready_in, ready_out, counters, what="fetch plan index tensors")
    return _lib.FetchPlan(_ptr(fetch), _ptr(n_fetch), _ptr(src_in), _ptr(src_out), _ptr(dst_in), _ptr(dst_out),
                          int(in_bytes), int(out_bytes), int(first_slot), int(n_slots), _ptr(ready_in),
                          _ptr(ready_out), _ptr(counters), counters.numel(), int(value), int(pairs), int(phase))


def _fetch_ref(fp):
    import ctypes

    return None if fp is None else ctypes.addressof(fp)


def fetch_expert(dst, src, ready_flag=None, epoch: int = 0, stream=None):
    """K6 primitive: async copy src -> dst (peer HBM / pinned host) + flag publish."""
    if dst.numel() * dst.element_size() != src.numel() * src.element_size():
        raise ValueError("fetch_expert: size mismatch")
    _lib.call("hm_fetch_expert", _ptr(dst), _ptr(src), dst.numel() * dst.element_size(),
              None if ready_flag is None else ready_flag.data_ptr(), int(epoch), _stream(stream))


def combine(Y, pos, topk_w, out=None, residual=None, stream=None):
    """K7.  y [T, d] bf16 = (residual +) sum_j w[t,j] * Y[pos[t,j]]; pos=None: Y is token-major [T*k, d]."""
    _require_cuda(Y, pos, topk_w, residual)
    _require_dtype(torch.bfloat16, Y, residual, out, what="combine rows")
    _require_dtype(torch.float32, topk_w, what="combine weights")
    _require_dtype(torch.int32, pos, what="combine positions")
    T, k = topk_w.shape
    d = Y.shape[1]
    if out is None:
        out = torch.empty((T, d), dtype=torch.bfloat16, device=Y.device)
    _lib.call("hm_combine", _ptr(Y), _ptr(pos), _ptr(topk_w), T, k, d, _ptr(residual), _ptr(out), _stream(stream))
    return out


# ------------------------------------------------------------------------------------------
# expert parallelism over peer memory (ep.py transport "p2p")
# ------------------------------------------------------------------------------------------
def ep_offsets(S, me: int, dst_delta=None, recv_split=None, stream=None):
    """dst_delta [G] (send-layout row -> receive row of destination d), recv_split [G+1]."""
    _require_cuda(S)
    G, E, _ = S.shape
    if dst_delta is None:
        dst_delta = torch.empty(G, dtype=torch.int32, device=S.device)
    if recv_split is None:
        recv_split = torch.empty(G + 1, dtype=torch.int32, device=S.device)
    _lib.call("hm_ep_offsets", _ptr(S), G, E, int(me), _ptr(dst_delta), _ptr(recv_split), _stream(stream))
    return dst_delta, recv_split


def dispatch_push(x, topk_idx, lrank, tile_off, S, slot_base, dst_delta, me: int, dst_rows, dst_tok, pos=None,
                  stream=None):
    """Fused scatter + dispatch: rows land in the destination ranks' receive buffers.
    dst_rows / dst_tok: uint64 (int64) device tensors of G peer pointers.  dst_delta=None:
    slot_base is an HM_LAYOUT_EP_EXPERT layout and the stored token index is tagged with the
    source rank ((me << 24) | t*k + j)."""
    _require_cuda(x, topk_idx, lrank, tile_off, S, slot_base, dst_delta, dst_rows, dst_tok, pos)
    T, d = x.shape
    k = topk_idx.shape[1]
    G, E, _ = S.shape
    _lib.call("hm_dispatch_push", _ptr(x), _ptr(topk_idx), _ptr(lrank), _ptr(tile_off), _ptr(S), _ptr(slot_base),
              _ptr(dst_delta), T, int(me), G, E, k, d, _ptr(dst_rows), _ptr(dst_tok), _ptr(pos), _stream(stream))


def grouped_gemm_remote(A, W, N: int, layout: "Layout", epilogue: int, out_ptrs, out_split, row_map, slot_ready=None,
                        ready_from_slot: int = 0, epoch: int = 0, a_rows: int | None = None, slot_done=None,
                        fetch=None, stream=None):
    """K5 with the rows of each segment stored into the owning source rank's buffer (peer pointer):
    per segment via out_split, or (out_split=None) per row via the source tag in row_map."""
    _require_cuda(A, W, out_ptrs, out_split, row_map, slot_ready, slot_done)
    rows = A.shape[0] if a_rows is None else int(a_rows)
    K = A.shape[1]
    _lib.call("hm_grouped_gemm_remote", _ptr(A), rows, _ptr(W), W.shape[0], N, K, _ptr(layout.segs),
              _ptr(layout.n_seg), _ptr(layout.mtile_prefix), int(epilogue), _ptr(out_ptrs), _ptr(out_split),
              out_ptrs.numel(), _ptr(row_map), _ptr(slot_ready), int(ready_from_slot), int(epoch), _ptr(slot_done),
              _fetch_ref(fetch), _stream(stream))


def fetch_experts(fetch, n_fetch, src_in, src_out, in_bytes: int, out_bytes: int, dst_in, dst_out, first_slot: int,
                  n_slots: int, ready_in, ready_out, counters, value: int = 1, ctas: int = 0, stream=None):
    """Device-driven K6 over the layout's fetch list (no host round trip); ready flags per expert."""
    _require_cuda(fetch, n_fetch, src_in, src_out, dst_in, dst_out, ready_in, ready_out, counters)
    _lib.call("hm_fetch_experts", _ptr(fetch), _ptr(n_fetch), _ptr(src_in), _ptr(src_out), int(in_bytes),
              int(out_bytes), _ptr(dst_in), _ptr(dst_out), int(first_slot), int(n_slots), _ptr(ready_in),
              _ptr(ready_out), _ptr(counters), counters.numel(), int(value), int(ctas), _stream(stream))


def stream_signal(addresses, value: int, stream=None):
    """Write `value` to each device address (ints: peer flag words) after prior stream work."""
    import ctypes

    arr = (ctypes.c_void_p * len(addresses))(*[int(a) for a in addresses])
    _lib.call("hm_stream_signal", arr, len(addresses), int(value) & 0xFFFFFFFF, _stream(stream))


def stream_wait(flags, value: int, stream=None):
    """Block the stream until every int32 of `flags` (device tensor) is >= value."""
    _require_cuda(flags)
    _lib.call("hm_stream_wait", _ptr(flags), flags.numel(), int(value) & 0xFFFFFFFF, _stream(stream))
