"""Expert-parallel HarMoEny block: one process per GPU, G = world size.

Alg. 1 across ranks, every step a kernel or a collective:

  1 router + histogram          hm_router_topk / hm_hist_scan on the local tokens
  2 metadata exchange           all_gather of hist[E] int32 -> m_all[G,E] (4 KB at G=8)
  3 schedule                    hm_schedule, replicated bit-identically on every rank
  4 scatter                     hm_permute into a dest-major send buffer + all_to_all_single
  5 experts + async fetch       hm_grouped_gemm x2 over the receive buffer's (expert, source)
                                segments in plan order; experts this rank does not host are
                                fetched (hm_fetch_expert) from the home GPU's HBM over NVLink
                                (CUDA IPC) or from pinned host memory, on a dedicated stream,
                                one transfer channel in plan order (engine.py:253-265); the
                                GEMM's producer waits on a per-slot ready flag
  6 gather                      all_to_all_single back + hm_combine

That is transport "nccl".  The split sizes of the all_to_all are host arguments in NCCL, so S is
copied to the host once per layer (32 KB at G=8, E=128).  Host-side plumbing lives in plain
functions (``ep_counts``, ``exchange_*``) that are exercised with the gloo backend on CPU by
tests/test_ep_gloo.py.

Transport "p2p" (the default of bench.py) has no collective and no host round trip: every rank
maps every peer's arena through CUDA IPC once; step 2 pushes the histogram row into every peer's
m_all and raises a stream flag; step 4 is hm_dispatch_push writing each token row straight into
its destination's EXPERT-MAJOR receive buffer (HM_LAYOUT_EP_EXPERT: rows placed from the
replicated S, one GEMM segment per expert); step 6 is FFN2's epilogue storing every row into its
source rank's token-major output (the source rides in the pushed token index), then the combine.
A bounded expert cache (expert_cache_size below the fetchable experts) runs K6 as fetch pairs
inside the GEMM launches (hm_fetch_plan).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, ops
from .block import BlockStats, MoEConfig, pack_w13, placement_home


# ------------------------------------------------------------------------------------------
# host-side plumbing (device agnostic; gloo-testable)
# ------------------------------------------------------------------------------------------
def ep_counts(S: np.ndarray, me: int):
    """Rows this rank sends to / receives from every rank: the flows matrix of
    engine._exchange_byte_vectors (engine.py:278-284), flows[g_from, g_to] = sum_e S."""
    flows = np.asarray(S, dtype=np.int64).sum(axis=1)
    return flows[me, :].tolist(), flows[:, me].tolist()


def _host_staged(t: torch.Tensor, group) -> bool:
    """gloo has no device collectives: stage CUDA tensors through host memory.  Only the
    test harness runs EP ranks over gloo (several ranks sharing one GPU); production
    runs one rank per GPU over NCCL."""
    return t.is_cuda and dist.get_backend(group) != "nccl"


def exchange_metadata(hist_local: torch.Tensor, group=None) -> torch.Tensor:
    """Step 2: all_gather of the local histogram [1, E] -> m_all [G, E]."""
    G = dist.get_world_size(group)
    src = hist_local.reshape(1, -1).contiguous()
    if _host_staged(src, group):
        parts = [torch.empty_like(src, device="cpu") for _ in range(G)]
        dist.all_gather(parts, src.cpu(), group=group)
        return torch.cat(parts).to(hist_local.device)
    out = torch.empty((G, hist_local.shape[-1]), dtype=hist_local.dtype, device=hist_local.device)
    dist.all_gather_into_tensor(out, src, group=group)
    return out


def exchange_tokens(send_buf: torch.Tensor, send_counts, recv_counts, group=None, out=None) -> torch.Tensor:
    """Step 4 scatter: all_to_all_single with per-destination row counts."""
    rows = int(sum(recv_counts))
    if out is None:
        out = torch.empty((max(rows, 1), send_buf.shape[1]), dtype=send_buf.dtype, device=send_buf.device)
    src = send_buf[: int(sum(send_counts))]
    if _host_staged(src, group):  # raw bytes (gloo has no bf16 / int16 kernels)
        h_out = torch.empty((rows, send_buf.shape[1] * send_buf.element_size()), dtype=torch.uint8)
        dist.all_to_all_single(h_out, src.cpu().view(torch.uint8), output_split_sizes=list(recv_counts),
                               input_split_sizes=list(send_counts), group=group)
        out[:rows].copy_(h_out.view(send_buf.dtype))
        return out
    dist.all_to_all_single(out[:rows], src, output_split_sizes=list(recv_counts), input_split_sizes=list(send_counts),
                           group=group)
    return out


def return_tokens(y_recv: torch.Tensor, send_counts, recv_counts, group=None, out=None) -> torch.Tensor:
    """Step 6 gather: the mirror all_to_all (engine.py:368-371) - every row goes home."""
    return exchange_tokens(y_recv, recv_counts, send_counts, group=group, out=out)


# ------------------------------------------------------------------------------------------
# the block
# ------------------------------------------------------------------------------------------
class PeerAccessError(RuntimeError):
    """CUDA IPC / peer mapping failed on at least one rank.  Raised on EVERY rank at the same
    point (after a collective agreement), so the caller can rebuild the block with the NCCL
    transport and host-memory expert fetches without desynchronising the process group."""


def _agree_all_ok(ok: bool, group, device) -> bool:
    """True iff every rank's `ok` is True (one small all_reduce)."""
    dev = device if dist.get_backend(group) == "nccl" else "cpu"
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return bool(flag.item())


class EPHarMoEnyBlock:
    """One MoE layer sharded by expert over the ranks of `group` (NCCL)."""

    KERNELS_PER_FORWARD = 8

    def __init__(self, cfg: MoEConfig, wg, w1, w2, w3=None, bias=None, device=None, group=None):
        if not dist.is_initialized():
            raise RuntimeError("EPHarMoEnyBlock needs torch.distributed (one process per GPU)")
        self.group = group
        self.G = dist.get_world_size(group)
        self.me = dist.get_rank(group)
        if cfg.world_size != self.G or cfg.rank != self.me:
            raise ValueError("MoEConfig rank/world_size must match the process group")
        self.cfg = cfg
        device = torch.device(device if device is not None else "cuda")
        self.device = device
        E, d, f = cfg.num_experts, cfg.d_model, cfg.d_ff
        bf = torch.bfloat16
        wgp = torch.zeros((ops.e_pad(E), d), dtype=bf, device=device)
        wgp[:E] = wg.to(device=device, dtype=bf)
        self.wg = wgp
        self.bias = None if bias is None else bias.to(device=device, dtype=torch.float32).contiguous()
        self.home_np = placement_home(cfg)
        self.home = torch.from_numpy(self.home_np).to(device)
        self.home_experts = [e for e in range(E) if self.home_np[e] == self.me]
        self.n_home = len(self.home_experts)
        # K6 cache slots beside the home experts.  expert_cache_size = 0: one per expert this rank
        # could ever fetch.  A smaller cache is the reference's bounded expert cache
        # (engine.py:204-275): fetch i overwrites the slot of fetch i - n_cache once the GEMMs have
        # finished that expert (the earliest slot to free up, fetched experts running in plan
        # order).  Home slots are never overwritten: they are the master copies the other ranks
        # fetch from over NVLink (the reference's overwritable residents assume a host master).
        n_fetchable = E - self.n_home
        self.n_cache = cfg.expert_cache_size if cfg.expert_cache_size > 0 else n_fetchable
        self.bounded = 0 < self.n_cache < n_fetchable
        # bounded cache: the channel must wait on the GEMMs' progress (a slot frees when its
        # occupant's tiles are done) while the GEMMs wait on the channel, so the copy runs as
        # FETCH_PAIRS CTA pairs inside each GEMM launch (hm_fetch_plan): co-resident by
        # construction.  A separate copy kernel or copy-engine stream cannot guarantee that
        # (measured: a stream aliasing the GEMM's hardware queue serialises behind it and
        # deadlocks)
        if cfg.activation == "swiglu":
            if w3 is None:
                raise ValueError("SwiGLU experts need w3")
            w_in_all = pack_w13(w1.to(device=device, dtype=bf), w3.to(device=device, dtype=bf)).view(E, 2 * f, d)
            self.n_in, self.epi_in = 2 * f, ops.HM_EPI_SWIGLU
        else:
            w_in_all = w1.to(device=device, dtype=bf).reshape(E, f, d)
            self.n_in, self.epi_in = f, ops.HM_EPI_RELU
        w_out_all = w2.to(device=device, dtype=bf).reshape(E, d, f)
        slots = self.n_home + self.n_cache
        self.w_in = torch.empty((slots, self.n_in, d), dtype=bf, device=device)
        self.w_out = torch.empty((slots, d, f), dtype=bf, device=device)
        if self.n_home:
            idx = torch.tensor(self.home_experts, device=device)
            self.w_in[: self.n_home] = w_in_all[idx]
            self.w_out[: self.n_home] = w_out_all[idx]
        # fetch sources
        self.fetch_source = cfg.fetch_source
        self._hslot = {}
        for g in range(self.G):
            for i, e in enumerate([e for e in range(E) if self.home_np[e] == g]):
                self._hslot[e] = i
        if self.fetch_source == "host":
            self.w_in_host = w_in_all.cpu().pin_memory()
            self.w_out_host = w_out_all.cpu().pin_memory()
        elif self.fetch_source == "peer":
            self._open_peers()
        else:
            raise ValueError("fetch_source must be 'peer' or 'host'")
        del w_in_all, w_out_all
        # per-EXPERT ready flags (a bounded cache reuses slots within one forward) and the GEMMs'
        # per-expert tile completion counters (slot reuse)
        self.ready_in = torch.zeros(E, dtype=torch.int32, device=device)
        self.ready_out = torch.zeros(E, dtype=torch.int32, device=device)
        self.done_in = torch.zeros(E, dtype=torch.int32, device=device)
        self.done_out = torch.zeros(E, dtype=torch.int32, device=device)
        self._fetch_sources()
        self.epoch = 0
        self.fetch_stream = torch.cuda.Stream(device=device)
        self._last_gemm = None
        self.S_host = torch.empty((self.G, E, self.G), dtype=torch.int32, pin_memory=True)
        self.fetch_host = torch.empty(E + 1, dtype=torch.int32, pin_memory=True)
        self.stats = BlockStats()
        # expert-ordered dispatch overlapped with FFN1 (MoEConfig.overlap_dispatch)
        env = os.environ.get("HM_OVERLAP_DISPATCH", "")
        want = (env == "1") if env in ("0", "1") else cfg.overlap_dispatch
        supported = (cfg.transport == "p2p" and self.G & (self.G - 1) == 0 and
                     cfg.policy_code != ops.HM_POLICY_EVEN_SPLIT)
        if want and not supported:
            raise ValueError("overlap_dispatch needs the p2p transport, a power-of-two world size and the "
                             "harmony / static policy")
        self.overlap = bool(want)
        if cfg.transport == "p2p":
            self._setup_p2p()
            # ours: router, hist_scan, plan, dispatch_push, fetch, gemm1, gemm2, combine
            self.KERNELS_PER_FORWARD = 8

    # CTA pairs of each GEMM launch that run the bounded-cache K6 channel: TMA bulk copies reach
    # ~90 GB/s per pair HBM->HBM on B200 (tools/fetch_pairs_bw.py: 1 / 2 / 4 pairs = 94 / 177 / 317 GB/s)
    FETCH_PAIRS = 4

    def _fetch_sources(self):
        """Device tables of every expert's weight blocks at its home rank (NVLink, CUDA IPC) or
        in pinned host memory: the sources of the device-driven K6 (fetch kernel or the fetch
        pairs inside the GEMM launches)."""
        cfg, E, d = self.cfg, self.cfg.num_experts, self.cfg.d_model
        in_bytes, out_bytes = self.n_in * d * 2, d * cfg.d_ff * 2
        src_in, src_out = [], []
        for e in range(E):
            h, hs = int(self.home_np[e]), self._hslot[e]
            if self.fetch_source == "host":
                src_in.append(self.w_in_host[e].data_ptr())
                src_out.append(self.w_out_host[e].data_ptr())
            else:
                src_in.append(self.peer_in[h] + hs * in_bytes)
                src_out.append(self.peer_out[h] + hs * out_bytes)
        i64 = dict(dtype=torch.int64, device=self.device)
        self._src_host = (src_in, src_out)
        self.fetch_src_in = torch.tensor(src_in, **i64)
        self.fetch_src_out = torch.tensor(src_out, **i64)
        self.fetch_counters = torch.zeros(2 * E, dtype=torch.int32, device=self.device)

    def _fetch_plan(self, lay, phase: int, value: int):
        """hm_fetch_plan of a bounded cache: fetch i -> slot n_home + i % n_cache once expert
        fetch[i - n_cache]'s tiles are done (engine.py:239-257 overwrite order)."""
        d, f = self.cfg.d_model, self.cfg.d_ff
        return ops.fetch_plan(lay.fetch, lay.n_fetch, self.fetch_src_in, self.fetch_src_out, self.w_in, self.w_out,
                              self.n_in * d * 2, d * f * 2, self.n_home, self.n_cache, self.ready_in, self.ready_out,
                              self.fetch_counters, value, phase, pairs=self.FETCH_PAIRS)

    @classmethod
    def random(cls, cfg: MoEConfig, seed: int = 0, device="cuda", zipf_s=None, std: float = 0.02, group=None):
        """Identical random weights on every rank (same seed), calibrated Zipf router bias."""
        from .block import random_weights

        return cls(cfg, *random_weights(cfg, seed, device, zipf_s, std), device=device, group=group)

    def _open_peers(self):
        """Exchange CUDA IPC handles of every rank's home-expert weights (once)."""
        L = _lib.load()
        hs, err = [], None
        try:  # a failed export must not leave the other ranks waiting in the gather below
            for t in (self.w_in, self.w_out):
                hs.append(self._export_handle(L, t))
        except Exception as e:  # noqa: BLE001 - reported on every rank below
            hs, err = None, e
        allh = [None] * self.G
        dist.all_gather_object(allh, hs, group=self.group)
        self.peer_in, self.peer_out = [], []
        self._ipc_bases = []
        if any(h is None for h in allh):
            bad = [g for g, h in enumerate(allh) if h is None]
            raise PeerAccessError(f"CUDA IPC export failed on rank(s) {bad}: {err}") from err
        try:
            for g in range(self.G):
                if g == self.me:
                    self.peer_in.append(self.w_in.data_ptr())
                    self.peer_out.append(self.w_out.data_ptr())
                    continue
                ptrs = []
                for h, off in allh[g]:
                    p = ctypes.c_void_p()
                    _lib.check(L.hm_ipc_open(h, ctypes.byref(p)), "hm_ipc_open")
                    self._ipc_bases.append(p.value)
                    ptrs.append(p.value + off)  # the handle maps the allocation base
                self.peer_in.append(ptrs[0])
                self.peer_out.append(ptrs[1])
        except Exception as e:  # noqa: BLE001 - re-raised on every rank below
            err = e
        if not _agree_all_ok(err is None, self.group, self.device):
            self._close_peers()
            raise PeerAccessError(f"peer weight mapping failed on some rank: {err}") from err

    # ---------------------------------------------------------------------------------------
    # transport "p2p": one-sided pushes into peer-mapped buffers (NVLink / NVSwitch)
    # ---------------------------------------------------------------------------------------
    @staticmethod
    def _export_handle(L, t: torch.Tensor):
        """(IPC handle bytes, offset of t inside the allocation the handle names)."""
        buf = ctypes.create_string_buffer(64)
        off = ctypes.c_size_t(0)
        _lib.check(L.hm_ipc_get_handle(t.data_ptr(), buf, ctypes.byref(off)), "hm_ipc_get_handle")
        return bytes(buf.raw), int(off.value)

    def _ipc_export_open(self, t: torch.Tensor):
        """Exchange one IPC handle per rank for tensor `t`; returns every rank's device address.
        Export or mapping failures on any rank raise PeerAccessError on every rank."""
        L = _lib.load()
        try:  # e.g. cudaIpcGetMemHandle refusing expandable-segment allocations
            mine, err = self._export_handle(L, t), None
        except Exception as e:  # noqa: BLE001 - reported on every rank below
            mine, err = None, e
        allh = [None] * self.G
        dist.all_gather_object(allh, mine, group=self.group)
        if any(h is None for h in allh):
            bad = [g for g, h in enumerate(allh) if h is None]
            self._close_peers()
            raise PeerAccessError(f"CUDA IPC export failed on rank(s) {bad}: {err}") from err
        addrs = []
        err = None
        try:
            for g in range(self.G):
                if g == self.me:
                    addrs.append(t.data_ptr())
                    continue
                p = ctypes.c_void_p()
                _lib.check(L.hm_ipc_open(allh[g][0], ctypes.byref(p)), "hm_ipc_open")
                self._ipc_bases.append(p.value)
                addrs.append(p.value + allh[g][1])
        except Exception as e:  # noqa: BLE001 - re-raised on every rank below
            err = e
        if not _agree_all_ok(err is None, self.group, self.device):
            self._close_peers()
            raise PeerAccessError(f"peer buffer mapping failed on some rank: {err}") from err
        return addrs

    def _close_peers(self):
        L = _lib.load()
        for b in getattr(self, "_ipc_bases", []):
            L.hm_ipc_close(ctypes.c_void_p(b))
        self._ipc_bases = []

    def _setup_p2p(self):
        """Allocate this rank's peer-visible arena (flags, m_all rows, receive buffer + token
        indices, token-major output) and map every rank's arena (one IPC handle each)."""
        cfg, G, E, d = self.cfg, self.G, self.cfg.num_experts, self.cfg.d_model
        k, Tmax = cfg.top_k, cfg.max_tokens_per_rank
        if not hasattr(self, "_ipc_bases"):
            self._ipc_bases = []
        self.cap_send = Tmax * k
        self.cap_recv = G * Tmax * k

        def al(n):
            return (n + 255) // 256 * 256

        lay = {}
        off = 0
        for name, nbytes in (("flags", 3 * G * 4), ("m_all", G * E * 4), ("arrive", E * 4),
                             ("recv_tok", self.cap_recv * 4), ("x_recv", self.cap_recv * d * 2),
                             ("y_ret", self.cap_send * d * 2)):
            lay[name] = off
            off += al(nbytes)
        self.arena = torch.zeros(off, dtype=torch.uint8, device=self.device)
        a = self.arena
        self.flags = a[lay["flags"]: lay["flags"] + 3 * G * 4].view(torch.int32).view(3, G)
        self.m_all_buf = a[lay["m_all"]: lay["m_all"] + G * E * 4].view(torch.int32).view(G, E)
        self.arrive = a[lay["arrive"]: lay["arrive"] + E * 4].view(torch.int32)  # rows of each expert landed
        self.recv_tok = a[lay["recv_tok"]: lay["recv_tok"] + self.cap_recv * 4].view(torch.int32)
        self.x_recv = a[lay["x_recv"]: lay["x_recv"] + self.cap_recv * d * 2].view(torch.bfloat16).view(-1, d)
        self.y_ret = a[lay["y_ret"]: lay["y_ret"] + self.cap_send * d * 2].view(torch.bfloat16).view(-1, d)
        self.h_buf = torch.empty((self.cap_recv, cfg.d_ff), dtype=torch.bfloat16, device=self.device)
        torch.cuda.synchronize(self.device)
        bases = self._ipc_export_open(self.arena)
        i64 = dict(dtype=torch.int64, device=self.device)
        self.p2p_rows = torch.tensor([b + lay["x_recv"] for b in bases], **i64)
        self.p2p_tok = torch.tensor([b + lay["recv_tok"] for b in bases], **i64)
        self.p2p_out = torch.tensor([b + lay["y_ret"] for b in bases], **i64)
        self.p2p_arrive = torch.tensor([b + lay["arrive"] for b in bases], **i64)
        self.push_order = torch.empty(self.cap_send, dtype=torch.int32, device=self.device)
        self.push_sync = torch.zeros(2, dtype=torch.int32, device=self.device)
        me = self.me
        self.meta_addrs = [b + lay["flags"] + (0 * G + me) * 4 for b in bases]
        self.tok_addrs = [b + lay["flags"] + (1 * G + me) * 4 for b in bases]
        self.y_addrs = [b + lay["flags"] + (2 * G + me) * 4 for b in bases]
        self.mall_row_addrs = [b + lay["m_all"] + me * E * 4 for b in bases]
        base0 = self.arena.data_ptr() + lay["flags"]
        self.local_flag_addrs = [[base0 + (c * G + g) * 4 for g in range(G)] for c in range(3)]
        dist.barrier(group=self.group)  # every arena zeroed and mapped before anyone signals

    def _p2p_stages(self, st, s):
        """The p2p forward as stream-ordered stages over the state dict ``st`` (input st["x"]):
        "dispatch" (router, metadata push, plan, fused scatter + dispatch push), "gemm1"
        (device-driven fetch forked onto the fetch stream + FFN1, joined; bounded cache: fetch
        pairs inside FFN1), "combine" (FFN2 storing into the source ranks - bounded cache: with
        its fetch pairs - + combine).  Each stage is graph-capturable."""
        cfg, G, E, me = self.cfg, self.G, self.cfg.num_experts, self.me
        k, d = cfg.top_k, cfg.d_model
        L = _lib.load()

        def dispatch():
            x = st["x"]
            Tg = x.shape[0]
            if Tg > cfg.max_tokens_per_rank:
                raise ValueError(f"{Tg} tokens exceed max_tokens_per_rank={cfg.max_tokens_per_rank}")
            idx, w, tile_hist, lrank = ops.router_topk(x, self.wg, self.bias, 1, Tg, k, cfg.renormalize, E=E,
                                                       stream=s)
            hist, tile_off = ops.hist_scan(tile_hist, 1, (Tg + ops.TILE_M - 1) // ops.TILE_M, stream=s)
            # step 2: my histogram row into every rank's m_all (peer stores), then flags
            for addr in self.mall_row_addrs:
                _lib.check(L.hm_fetch_expert(addr, hist.data_ptr(), E * 4, None, 0, s.cuda_stream), "m_all push")
            ops.stream_signal(self.meta_addrs, 1, s)
            ops.stream_wait(self.flags[0], 1, s)
            ops.stream_signal(self.local_flag_addrs[0], 0, s)
            # expert-major receive buffers: every sender places its rows from the replicated S, and
            # this rank's GEMMs see one segment per expert (all sources' rows contiguous)
            cache = self.n_cache if self.bounded else 0
            pos = torch.empty((Tg, k), dtype=torch.int32, device=self.device)
            if self.overlap:
                # rows pushed in every destination's plan order, counted per expert on arrival;
                # FFN1 (next kernel on this stream, PDL) waits per segment instead of on a flag
                p, pl = ops.plan_dispatch(self.home, G, E, cfg.eq_tokens, cfg.policy_code, me, self.m_all_buf,
                                          cache_slots=cache, stream=s)
                m_all = self.m_all_buf.clone()
                ops.dispatch_push_ordered(x, idx, lrank, tile_off, p.S, p.layout.slot_base, pl, me, self.p2p_rows,
                                          self.p2p_tok, self.p2p_arrive, self.push_order, self.push_sync, pos=pos,
                                          stream=s)
            else:
                p = ops.plan(self.home, G, E, cfg.eq_tokens, cfg.policy_code, ops.HM_LAYOUT_EP_EXPERT, me,
                             m_all=self.m_all_buf, cache_slots=cache, stream=s)
                m_all = self.m_all_buf.clone()  # peers may push the next forward's rows before the host reads stats
                ops.dispatch_push(x, idx, lrank, tile_off, p.S, p.layout.slot_base, None, me, self.p2p_rows,
                                  self.p2p_tok, pos=pos, stream=s)
                ops.stream_signal(self.tok_addrs, 1, s)
                ops.stream_wait(self.flags[1], 1, s)
                ops.stream_signal(self.local_flag_addrs[1], 0, s)
            st.update(idx=idx, w=w, plan=p, m_all=m_all, pos=pos, Tg=Tg)
            self.stats = BlockStats(m_all=m_all, schedule=p.S, iters=p.iters, loads=p.loads,
                                    extras=dict(topk_idx=idx, topk_w=w, pos=pos, layout=p.layout))

        # K6 from the device-side fetch list on the fetch stream, overlapping FFN1 (async), or in
        # stream order ahead of it (sync ablation: the GEMM's ready-flag waits pass at once); a
        # bounded cache runs it inside the GEMM launches instead (fetch pairs, see __init__)
        fs = self.fetch_stream if cfg.async_fetch else s

        def gemm1():
            lay = st["plan"].layout
            kw = {}
            if self.bounded:
                kw = dict(slot_done=self.done_in, fetch=self._fetch_plan(lay, 1, 1))
            elif self.n_cache > 0:
                if fs is not s:
                    fs.wait_stream(s)
                ops.fetch_experts(lay.fetch, lay.n_fetch, self.fetch_src_in, self.fetch_src_out, self.n_in * d * 2,
                                  d * cfg.d_ff * 2, self.w_in, self.w_out, self.n_home, self.n_cache, self.ready_in,
                                  self.ready_out, self.fetch_counters, value=1, stream=fs)
            if self.overlap:
                ops.grouped_gemm_arrive(self.x_recv, self.w_in.view(-1, d), self.n_in, lay, self.epi_in, self.arrive,
                                        out=self.h_buf, slot_ready=self.ready_in, ready_from_slot=self.n_home,
                                        epoch=1, pdl=True, stream=s, **kw)
            else:
                ops.grouped_gemm(self.x_recv, self.w_in.view(-1, d), self.n_in, lay, self.epi_in, out=self.h_buf,
                                 slot_ready=self.ready_in, ready_from_slot=self.n_home, epoch=1, stream=s, **kw)
            if self.n_cache > 0 and fs is not s and not self.bounded:
                s.wait_stream(fs)

        def combine():
            lay = st["plan"].layout
            kw = dict(slot_done=self.done_out, fetch=self._fetch_plan(lay, 2, 1)) if self.bounded else {}
            ops.grouped_gemm_remote(self.h_buf, self.w_out.view(-1, cfg.d_ff), d, lay, ops.HM_EPI_STORE,
                                    self.p2p_out, None, self.recv_tok, slot_ready=self.ready_out,
                                    ready_from_slot=self.n_home, epoch=1, stream=s, **kw)
            if self.n_cache > 0:
                self.ready_in.zero_()
                self.ready_out.zero_()
                if self.bounded:
                    self.done_in.zero_()
                    self.done_out.zero_()
            if self.overlap:  # every row of this forward has landed (FFN1 waited for all of them)
                self.arrive.zero_()
            ops.stream_signal(self.y_addrs, 1, s)
            ops.stream_wait(self.flags[2], 1, s)
            ops.stream_signal(self.local_flag_addrs[2], 0, s)
            x = st["x"]
            st["y"] = ops.combine(self.y_ret[: st["Tg"] * k], None, st["w"], residual=x if cfg.residual else None,
                                  stream=s)

        return [("dispatch", dispatch), ("gemm1", gemm1), ("combine", combine)]

    def _forward_p2p(self, x, s, mark):
        st = {"x": x}
        for name, fn in self._p2p_stages(st, s):
            fn()
            mark(name)
        return st["y"]

    def capture(self, num_tokens: int, pool=None):
        """CUDA-graph the p2p forward (every rank must call it, same token count): the
        forward never synchronises the host and its cross-rank waits are stream flags, so
        all of it is captured, one graph per stage."""
        from .block import CapturedForward

        if self.cfg.transport != "p2p":
            raise ValueError("only the p2p transport is graph-capturable (NCCL split sizes are host arguments)")
        x = torch.zeros((num_tokens, self.cfg.d_model), dtype=torch.bfloat16, device=self.device)
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                self.forward(x, stream=side)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize(self.device)
        st = {"x": x}
        pool = pool if pool is not None else torch.cuda.graph_pool_handle()
        graphs = []
        for name, fn in self._p2p_stages(st, side):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=pool, stream=side):
                fn()
            graphs.append((name, g))
        torch.cuda.synchronize(self.device)
        return CapturedForward(graphs, x, st["y"], self.stats)

    def _fetch(self, experts):
        """K6 on the copy engines (no SM taken from the GEMMs): one transfer channel (the fetch
        stream), plan order, fetched experts in cache slots n_home + i, a ready flag per expert.
        (A bounded cache is fetched by the pairs inside the GEMM launches instead.)"""
        if self.bounded:
            return
        if len(experts) > self.n_cache:
            raise RuntimeError(f"{len(experts)} experts to fetch exceed the {self.n_cache} cache slots")
        d, f = self.cfg.d_model, self.cfg.d_ff
        # async: one transfer channel beside the compute stream; sync ablation: the compute
        # stream itself (FFN1 starts only after every fetch landed)
        s = self.fetch_stream if self.cfg.async_fetch else torch.cuda.current_stream()
        if self._last_gemm is not None and s is self.fetch_stream:
            s.wait_event(self._last_gemm)  # previous layer's GEMMs are done with the slots
        in_bytes = self.n_in * d * 2
        out_bytes = d * f * 2
        L = _lib.load()
        for i, e in enumerate(experts):
            slot = self.n_home + i
            src_in, src_out = self._src_host[0][e], self._src_host[1][e]
            _lib.check(L.hm_fetch_expert(self.w_in[slot].data_ptr(), src_in, in_bytes,
                                         self.ready_in[e:].data_ptr(), self.epoch, s.cuda_stream),
                       "hm_fetch_expert")
            _lib.check(L.hm_fetch_expert(self.w_out[slot].data_ptr(), src_out, out_bytes,
                                         self.ready_out[e:].data_ptr(), self.epoch, s.cuda_stream),
                       "hm_fetch_expert")

    def forward(self, x: torch.Tensor, stream=None, marks=None) -> torch.Tensor:
        cfg = self.cfg
        if x.dim() != 2 or x.shape[1] != cfg.d_model or x.dtype != torch.bfloat16:
            raise ValueError(f"x must be bf16 [T, {cfg.d_model}]")
        s = stream if stream is not None else torch.cuda.current_stream()
        Tg, k, E, G, me = x.shape[0], cfg.top_k, cfg.num_experts, self.G, self.me
        tiles = (Tg + ops.TILE_M - 1) // ops.TILE_M
        self.epoch += 1

        def mark(name):
            if marks is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(s)
                marks.append((name, ev))

        with torch.cuda.stream(s):
            mark("start")
            x = x.contiguous()
            if cfg.transport == "p2p":
                return self._forward_p2p(x, s, mark)
            idx, w, tile_hist, lrank = ops.router_topk(x, self.wg, self.bias, 1, Tg, k, cfg.renormalize, E=E,
                                                       stream=s)
            hist, tile_off = ops.hist_scan(tile_hist, 1, tiles, stream=s)
            mark("router")
            m_all = exchange_metadata(hist, self.group)
            p = ops.plan(self.home, G, E, cfg.eq_tokens, cfg.policy_code, ops.HM_LAYOUT_EP, me, m_all=m_all,
                         cache_slots=self.n_cache if self.bounded else 0, stream=s)
            S, iters, loads, lay = p.S, p.iters, p.loads, p.layout
            self.S_host.copy_(S, non_blocking=True)
            self.fetch_host[:E].copy_(lay.fetch, non_blocking=True)
            self.fetch_host[E:].copy_(lay.n_fetch, non_blocking=True)
            s.synchronize()  # NCCL split sizes are host arguments
            mark("schedule")
            S_np = self.S_host.numpy()
            n_fetch = int(self.fetch_host[E])
            self._fetch(self.fetch_host[:n_fetch].tolist())
            send_counts, recv_counts = ep_counts(S_np, me)
            send, pos, _ = ops.permute(x, idx, lrank, tile_off, S, lay.slot_base, 1, Tg, me, Tg * k, stream=s)
            mark("permute")
            recv = exchange_tokens(send, send_counts, recv_counts, self.group)
            mark("dispatch_a2a")
            dn_in = dict(slot_done=self.done_in, fetch=self._fetch_plan(lay, 1, self.epoch)) if self.bounded else {}
            dn_out = dict(slot_done=self.done_out, fetch=self._fetch_plan(lay, 2, self.epoch)) if self.bounded else {}
            h = ops.grouped_gemm(recv, self.w_in.view(-1, cfg.d_model), self.n_in, lay, self.epi_in,
                                 slot_ready=self.ready_in, ready_from_slot=self.n_home, epoch=self.epoch, stream=s,
                                 **dn_in)
            mark("gemm1")
            yr = ops.grouped_gemm(h, self.w_out.view(-1, cfg.d_ff), cfg.d_model, lay, ops.HM_EPI_STORE,
                                  slot_ready=self.ready_out, ready_from_slot=self.n_home, epoch=self.epoch,
                                  stream=s, **dn_out)
            if self.bounded:  # the next forward's fetch pairs wait on fresh counts
                self.done_in.zero_()
                self.done_out.zero_()
            self._last_gemm = torch.cuda.Event()
            self._last_gemm.record(s)
            mark("gemm2")
            ys = return_tokens(yr, send_counts, recv_counts, self.group)
            mark("combine_a2a")
            y = ops.combine(ys, pos, w, residual=x if cfg.residual else None, stream=s)
            mark("combine")
        self.stats = BlockStats(m_all=m_all, schedule=S, iters=iters, loads=loads,
                                extras=dict(topk_idx=idx, topk_w=w, pos=pos, layout=lay, n_fetch=n_fetch,
                                            send_counts=send_counts, recv_counts=recv_counts))
        return y

    __call__ = forward

    def forward_host(self, x_host, y_host=None, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            x = x_host.to(self.device, non_blocking=True)
            y = self.forward(x, stream=s)
            if y_host is None:
                y_host = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
            y_host.copy_(y, non_blocking=True)
        return y_host
