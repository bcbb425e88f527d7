"""The HarMoEny MoE block on B200: Alg. 1 as a chain of
hand-written sm_100a kernels behind the C ABI.

    forward(x) (LOCAL, this module):              kernels (csrc/)
      1 router: logits, top-k, weights            hm_router_topk      (K1, tcgen05)
        per-tile histogram + (token,slot) ranks   (fused K2)
      2+3 metadata, schedule S, layout            hm_plan: histogram reduce + K3 (bit-exact) + layout
      4 scatter tokens                            hm_permute (K4): index-only when FFN1 gathers rows
                                                  itself (top_k >= 4, >= 256 rows/expert), else copies
      5 experts                                   hm_grouped_gemm x2  (K5, tcgen05 cta_group::2)
      6 gather + reconstruct                      FFN2 rows land token-major; hm_combine (K7)
    EP (ep.py) adds the metadata exchange, the dispatch / return over NVLink (or NCCL) and the
    async expert fetch (K6).

Two placements of the G ranks:

* LOCAL ("logical ranks"): one process owns the whole batch and simulates G
  GPUs on one device (BASELINE config 1 "simulated 4 GPUs").  The schedule is
  the real HarMoEny schedule of the G token shards; buffer rows are laid out
  [dest][expert][source], every expert's weights are local, no collectives.
* EP (expert parallel): one process per GPU, G = world size; see ep.py.

The paper's integration API (MoEConfig + replace_moe_layer)
is kept: ``MoEConfig(rank, world_size, scheduling_policy, expert_cache_size,
eq_tokens, d_model, num_experts, ...)``; eq_tokens is the threshold q
(SPEC.md:529).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .policies import PlacementKind, SchedulingPolicy, blocked_placement, round_robin_placement


_POLICY_CODES = {
    "harmony": ops.HM_POLICY_REBALANCE, "harmoeny": ops.HM_POLICY_REBALANCE, "rebalance": ops.HM_POLICY_REBALANCE,
    "round_robin": ops.HM_POLICY_NONE, "static": ops.HM_POLICY_NONE, "none": ops.HM_POLICY_NONE,
    "even_split": ops.HM_POLICY_EVEN_SPLIT,
}


@dataclass
class MoEConfig:
    rank: int = 0
    world_size: int = 1
    # "harmony"/"rebalance" (Alg. 2), "round_robin" (static placement, no rebalancing) or
    # "even_split" (the paper's even-split baseline, policies.py:174-203)
    scheduling_policy: str = "harmony"
    expert_cache_size: int = 0  # fetch slots per GPU (0 = one per fetched expert)
    eq_tokens: int = 32  # token threshold q (Eq. 4)
    d_model: int = 2048
    num_experts: int = 128
    d_ff: int = 768
    top_k: int = 8
    activation: str = "swiglu"  # "swiglu" (Qwen/Mixtral) or "relu" (Switch)
    renormalize: bool | None = None  # default: True for k > 1, False for top-1
    placement: str = "round_robin"
    logical_ranks: int = 1  # LOCAL mode: number of simulated GPUs (world_size must be 1)
    fetch_source: str = "peer"  # EP mode: "peer" (NVLink) or "host" (pinned host memory)
    # EP mode: fetch rebalanced experts' weights on a side stream overlapped with FFN1 of the
    # resident experts (True, SimFlags.async_loading_enabled) or on the compute stream ahead
    # of it (False: the synchronous-loading ablation, engine.py:266-269)
    async_fetch: bool = True
    residual: bool = False  # decoder-layer residual y = x + MoE(x), fused into the combine kernel
    # LOCAL mode: run the weighted combine inside the FFN2 epilogue (hm_grouped_gemm_combine:
    # the k-th arriving row of each token chunk combines it; bit-identical output) instead of
    # a separate combine kernel.  Off by default: measured 820 us for the fused FFN2 vs 351 + 98 us
    # separately at Qwen-128 (the epilogue waits on its arrival atomics, fences and the other
    # rows' DRAM reads every tile, which stalls the MMA pipeline; profiles/r2_experiments.txt).
    # HM_FUSED_COMBINE=0/1 overrides.
    fused_combine: bool = False
    # EP mode: "nccl" (all_to_all_single; split sizes need S on the host once per layer) or "p2p"
    # (one-sided pushes into peers' buffers over NVLink/NVSwitch, no host round trip)
    transport: str = "nccl"
    max_tokens_per_rank: int = 16384  # p2p: capacity of the peer-mapped buffers
    # EP p2p: push the rows expert by expert in every destination's plan order with per-expert
    # arrival counters, and start FFN1 right behind the push (programmatic dependent launch) so
    # each expert's tiles run as soon as its rows have landed (hm_dispatch_push_ordered; needs a
    # power-of-two world size and the harmony / static policy).  Off by default: measured slower
    # than the unordered push + token flags + FFN1 (profiles/r2_experiments.txt).
    # HM_OVERLAP_DISPATCH=0/1 overrides.
    overlap_dispatch: bool = False

    def __post_init__(self):
        if self.eq_tokens < 1:
            raise ValueError("token_threshold_q must be >= 1")
        if str(getattr(self.scheduling_policy, "value", self.scheduling_policy)).lower() not in _POLICY_CODES:
            raise ValueError(f"unknown scheduling_policy {self.scheduling_policy!r}")
        if self.transport not in ("nccl", "p2p"):
            raise ValueError("transport must be 'nccl' or 'p2p'")
        if self.max_tokens_per_rank < 1:
            raise ValueError("max_tokens_per_rank must be >= 1")
        if self.activation not in ("swiglu", "relu"):
            raise ValueError("activation must be 'swiglu' or 'relu'")
        # grouped-GEMM tiling (256-wide n-blocks, 64-deep k-blocks): FFN1 N = d_ff (ReLU) or
        # 2*d_ff (SwiGLU), FFN2 N = d_model; K = d_model / d_ff.  Every BASELINE shape fits.
        n_in = self.d_ff if self.activation == "relu" else 2 * self.d_ff
        if self.d_model % 256 or n_in % 256 or self.d_ff % 64:
            raise ValueError("d_model must be a multiple of 256 and d_ff a multiple of "
                             f"{256 if self.activation == 'relu' else 128} (grouped-GEMM tiles)")
        if not 1 <= self.top_k <= self.num_experts:
            raise ValueError("top_k must be in [1, num_experts]")
        if self.renormalize is None:
            self.renormalize = self.top_k > 1
        if self.world_size > 1 and self.logical_ranks not in (1, self.world_size):
            raise ValueError("logical ranks are a single-process mode (world_size == 1)")
        if self.expert_cache_size < 0:
            raise ValueError("expert_cache_size must be >= 0 (0 = one slot per fetchable expert)")
        if self.world_size > 1 and self.expert_cache_size > 0 and not self.async_fetch:
            n_home = int((placement_home(self) == self.rank).sum())
            if self.expert_cache_size < self.num_experts - n_home:
                raise ValueError("a bounded expert cache (expert_cache_size below the experts this rank may fetch) "
                                 "needs async_fetch=True: synchronous loading would stall the stream on slots that "
                                 "only a later kernel frees")

    @property
    def policy_code(self) -> int:
        """HM_POLICY_* code the planner kernel runs."""
        return _POLICY_CODES[str(getattr(self.scheduling_policy, "value", self.scheduling_policy)).lower()]

    @property
    def rebalance(self) -> bool:
        return self.policy_code == ops.HM_POLICY_REBALANCE

    @property
    def num_ranks(self) -> int:
        return self.world_size if self.world_size > 1 else self.logical_ranks


def pack_w13(w_gate: torch.Tensor, w_up: torch.Tensor) -> torch.Tensor:
    """[E,f,d] gate + [E,f,d] up -> [E*2f, d], block-interleaved by 128 rows (the
    SwiGLU epilogue of hm_grouped_gemm reads gate rows [0,128) and up rows
    [128,256) of each 256-row block)."""
    E, f, d = w_gate.shape
    if f % 128 != 0:
        raise ValueError("SwiGLU path needs d_ff % 128 == 0")
    g = w_gate.reshape(E, f // 128, 128, d)
    u = w_up.reshape(E, f // 128, 128, d)
    return torch.stack([g, u], dim=2).reshape(E * 2 * f, d).contiguous()


def random_weights(cfg: MoEConfig, seed: int = 0, device="cuda", zipf_s: float | None = None, std: float = 0.02):
    """(wg, w1, w2, w3, bias) for a block of this architecture, identical for a given seed."""
    from .workload import calibrated_router_bias

    g = torch.Generator(device=device).manual_seed(seed)
    E, d, f = cfg.num_experts, cfg.d_model, cfg.d_ff
    kw = dict(device=device, dtype=torch.float32, generator=g)
    wg = (torch.randn((E, d), **kw) * (1.0 / d) ** 0.5).to(torch.bfloat16)
    w1 = (torch.randn((E, f, d), **kw) * std).to(torch.bfloat16)
    w2 = (torch.randn((E, d, f), **kw) * std).to(torch.bfloat16)
    w3 = (torch.randn((E, f, d), **kw) * std).to(torch.bfloat16) if cfg.activation == "swiglu" else None
    bias = None
    if zipf_s is not None:
        bias = torch.from_numpy(calibrated_router_bias(E, zipf_s, cfg.top_k)).to(device)
    return wg, w1, w2, w3, bias


def placement_home(cfg: MoEConfig):
    G = cfg.num_ranks
    kind = PlacementKind(cfg.placement)
    p = blocked_placement(cfg.num_experts, G) if kind is PlacementKind.BLOCKED else round_robin_placement(
        cfg.num_experts, G)
    return np.asarray(p.home, dtype=np.int32)


class CapturedForward:
    """A graph-captured block forward over static buffers (see HarMoEnyBlock.capture)."""

    def __init__(self, graphs, x, y, stats):
        self.graphs, self.x, self.y, self.stats = graphs, x, y, stats

    def replay(self, marks: list | None = None, stream=None, only=None):
        """Replay on the current stream; ``marks`` receives (group name, event) after every group
        and ("start", event) before the first.  ``only`` (a set of group names) brackets just those
        groups - a ("pre", event) before each unless the previous group was bracketed too - since
        every event recorded between graph launches costs the stream a short bubble (Switch-128:
        ~13 us per step for the five marks of a full breakdown)."""
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            prev = False  # the previous group ended with a mark
            if marks is not None and only is None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(s)
                marks.append(("start", ev))
                prev = True
            for name, g in self.graphs:
                want = marks is not None and (only is None or name in only)
                if want and not prev:
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record(s)
                    marks.append(("pre", ev))
                g.replay()
                if want:
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record(s)
                    marks.append((name, ev))
                prev = want
        return self.y

    def __call__(self, x=None, marks=None, only=None):
        if x is not None:
            self.x.copy_(x)
        return self.replay(marks, only=only)

    def forward_host(self, x_host, y_host, stream=None):
        """End-to-end call with pinned host buffers: H2D -> graphs -> D2H (stream-ordered)."""
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self.x.copy_(x_host, non_blocking=True)
            self.replay(stream=s)
            y_host.copy_(self.y, non_blocking=True)
        return y_host


class HostPipeline:
    """End-to-end forward from pinned host memory: the batch is cut into ``n_chunks``
    token chunks whose H2D copy, block forward (a captured graph per chunk) and D2H copy
    run on three streams, so PCIe traffic in both directions overlaps the kernels.
    Tokens are independent in the MoE block, so the output equals the unchunked forward
    (each chunk is routed, scheduled and combined on its own)."""

    def __init__(self, block: "HarMoEnyBlock", num_tokens: int, n_chunks: int = 4, n_sets: int = 2):
        if num_tokens % n_chunks or (num_tokens // n_chunks) % block.cfg.num_ranks:
            raise ValueError("chunk size must divide evenly (and over the logical ranks)")
        self.n, self.chunk = n_chunks, num_tokens // n_chunks
        # one graph per chunk (all stages): minimal host work per launch.  ``n_sets`` buffer
        # sets ping-pong between successive runs, so run i+1's H2D / forward never wait for
        # run i's forward / D2H of the same chunk.
        all_stages = (("router", "schedule", "permute", "gemm1", "gemm2", "combine"),)
        self.sets = [[block.capture(self.chunk, groups=all_stages) for _ in range(n_chunks)] for _ in range(n_sets)]
        dev = block.device
        self.h2d, self.comp, self.d2h = (torch.cuda.Stream(device=dev) for _ in range(3))
        ev = lambda: [[torch.cuda.Event() for _ in range(n_chunks)] for _ in range(n_sets)]  # noqa: E731
        self.ev_in, self.ev_out, self.ev_back = ev(), ev(), ev()
        self.used = [False] * n_sets
        self.run_i = 0
        self.started = False

    def run(self, x_host: torch.Tensor, y_host: torch.Tensor) -> torch.Tensor:
        """Enqueue one forward; the caller's stream waits for the last D2H.  Successive runs
        are chained only through the per-chunk buffer events, so the H2D of run i+1 overlaps
        the tail of run i (host buffers follow the usual async rule: do not overwrite x_host
        or read y_host before synchronising)."""
        cur = torch.cuda.current_stream()
        if not self.started:
            for s in (self.h2d, self.comp, self.d2h):
                s.wait_stream(cur)
        b = self.run_i % len(self.sets)
        ev_in, ev_out, ev_back = self.ev_in[b], self.ev_out[b], self.ev_back[b]
        for c, cap in enumerate(self.sets[b]):
            rows = slice(c * self.chunk, (c + 1) * self.chunk)
            with torch.cuda.stream(self.h2d):
                if self.used[b]:
                    self.h2d.wait_event(ev_out[c])  # the last forward on this buffer set read x
                cap.x.copy_(x_host[rows], non_blocking=True)
                ev_in[c].record(self.h2d)
            self.comp.wait_event(ev_in[c])
            if self.used[b]:
                self.comp.wait_event(ev_back[c])  # the last D2H from this buffer set read y
            cap.replay(stream=self.comp)
            ev_out[c].record(self.comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(ev_out[c])
                y_host[rows].copy_(cap.y, non_blocking=True)
                ev_back[c].record(self.d2h)
        self.used[b] = True
        self.run_i += 1
        self.started = True
        cur.wait_stream(self.d2h)
        cur.wait_stream(self.comp)
        return y_host


@dataclass
class BlockStats:
    """Device tensors describing the last forward (read them after a sync)."""

    m_all: torch.Tensor | None = None
    schedule: torch.Tensor | None = None
    iters: torch.Tensor | None = None
    loads: torch.Tensor | None = None
    extras: dict = field(default_factory=dict)

    def load_imbalance(self) -> float:
        loads = self.loads.double()
        return float(loads.max() / loads.mean()) if float(loads.mean()) > 0 else 1.0


class HarMoEnyBlock:
    """One MoE layer: router + experts, weights resident in HBM (bf16).

    LOCAL mode only here (world_size == 1); multi-process expert parallelism
    lives in :class:`paper_2506_12417_b200.ep.EPHarMoEnyBlock`.
    """

    def __init__(self, cfg: MoEConfig, wg: torch.Tensor, w1: torch.Tensor, w2: torch.Tensor,
                 w3: torch.Tensor | None = None, bias: torch.Tensor | None = None, device=None):
        if cfg.world_size != 1:
            raise ValueError("HarMoEnyBlock is the single-process block; use ep.EPHarMoEnyBlock for world_size > 1")
        device = torch.device(device if device is not None else "cuda")
        if device.type != "cuda":
            raise ValueError("HarMoEnyBlock runs on CUDA only (no CPU fallback)")
        self.cfg = cfg
        E, d, f = cfg.num_experts, cfg.d_model, cfg.d_ff
        bf = torch.bfloat16
        wgp = torch.zeros((ops.e_pad(E), d), dtype=bf, device=device)
        wgp[:E] = wg.to(device=device, dtype=bf)
        self.wg = wgp
        self.bias = None if bias is None else bias.to(device=device, dtype=torch.float32).contiguous()
        if cfg.activation == "swiglu":
            if w3 is None:
                raise ValueError("SwiGLU experts need w3 (up projection)")
            self.w_in = pack_w13(w1.to(device=device, dtype=bf), w3.to(device=device, dtype=bf))
            self.n_in = 2 * f
            self.epi_in = ops.HM_EPI_SWIGLU
        else:
            self.w_in = w1.to(device=device, dtype=bf).reshape(E * f, d).contiguous()
            self.n_in = f
            self.epi_in = ops.HM_EPI_RELU
        self.w_out = w2.to(device=device, dtype=bf).reshape(E * d, f).contiguous()
        self.home_np = placement_home(cfg)
        self.home = torch.from_numpy(self.home_np).to(device)
        self.device = device
        self.stats = BlockStats()
        # fused scatter: FFN1 gathers token rows itself with cp.async loader warps, so the
        # k-fold replicated token buffer (T*k*d*2 bytes written, then read) never exists.  With
        # the m-major pair-tile walk the NB pairs sharing an A tile gather the same rows side by
        # side (L2 hits).  Measured on B200: Qwen-128 16k tokens (top-8, ~1000 rows per expert)
        # +4.5% short / +3.7% power-capped, 4k tokens even; but where FFN1 streams weights for
        # small segments the gather latency throttles the weight pipeline: Qwen-128 at 256 /
        # 1024 tokens -17% / -13%, Switch-128 (top-1) -31%, Mixtral (top-2) -2%.  Auto (None):
        # on for top_k >= 4 with >= 256 rows per expert on average.  HM_FUSED_SCATTER=0/1 or
        # assigning True/False overrides.
        env = os.environ.get("HM_FUSED_SCATTER", "")
        self.fused_scatter = (env == "1") if env in ("0", "1") else None

    def uses_fused_scatter(self, num_tokens: int) -> bool:
        if self.fused_scatter is not None:
            return bool(self.fused_scatter)
        cfg = self.cfg
        return cfg.top_k >= 4 and num_tokens * cfg.top_k >= 256 * cfg.num_experts

    @classmethod
    def random(cls, cfg: MoEConfig, seed: int = 0, device="cuda", zipf_s: float | None = None, std: float = 0.02):
        """Random-init weights of the named architecture (no checkpoints offline):
        experts ~ N(0, std), Wg ~ N(0, 1/d) (logits ~ N(0,1) for x ~ N(0,1)), and, with
        zipf_s, a router bias calibrated so the realised top-k routing has the Zipf(s)
        Gumbel-top-k expert shares (workload.calibrated_router_bias)."""
        return cls(cfg, *random_weights(cfg, seed, device, zipf_s, std), device=device)

    # ------------------------------------------------------------------------------------
    def forward(self, x: torch.Tensor, stream=None, marks: list | None = None) -> torch.Tensor:
        """y = MoE(x) for x [T, d] bf16 on this device.  ``marks``, if given, receives
        (stage, cuda.Event) pairs recorded after each stage (bench instrumentation)."""
        cfg = self.cfg
        if x.dim() != 2 or x.shape[1] != cfg.d_model:
            raise ValueError(f"x must be [T, {cfg.d_model}]")
        if x.dtype != torch.bfloat16:
            raise ValueError("x must be bf16")
        G = cfg.num_ranks
        T = x.shape[0]
        if T % G != 0:
            raise ValueError("token count must divide evenly over the logical ranks")
        if T == 0:  # empty batch: empty output, all-zero routing matrix / schedule (no kernels)
            i32 = dict(dtype=torch.int32, device=x.device)
            E = cfg.num_experts
            self.stats = BlockStats(m_all=torch.zeros((G, E), **i32), schedule=torch.zeros((G, E, G), **i32),
                                    iters=torch.zeros(1, **i32), loads=torch.zeros(G, **i32),
                                    extras=dict(topk_idx=torch.zeros((0, cfg.top_k), **i32)))
            return torch.empty((0, cfg.d_model), dtype=torch.bfloat16, device=x.device)
        s = stream if stream is not None else torch.cuda.current_stream()
        st = {"x": x.contiguous()}

        def mark(name):
            if marks is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(s)
                marks.append((name, ev))

        mark("start")
        for name, fn in self._stages(st, G, T // G, s):
            fn()
            mark(name)
        return st["y"]

    def _stages(self, st: dict, G: int, Tg: int, s):
        """The forward as named, stream-ordered stages over a state dict (so the bench
        and the graph capture can group them); every stage is one kernel launch."""
        cfg = self.cfg
        k, E = cfg.top_k, cfg.num_experts
        T = G * Tg
        tiles_per_rank = (Tg + ops.TILE_M - 1) // ops.TILE_M

        def router():
            st["idx"], st["w"], st["tile_hist"], st["lrank"] = ops.router_topk(
                st["x"], self.wg, self.bias, G, Tg, k, cfg.renormalize, E=E, stream=s)

        def plan():
            # steps 2+3 fused: per-rank histograms (m_all), schedule S, layout + GEMM work list
            p = ops.plan(self.home, G, E, cfg.eq_tokens, cfg.policy_code, ops.HM_LAYOUT_LOCAL,
                         tile_hist=st["tile_hist"], tiles_per_rank=tiles_per_rank, stream=s)
            st["plan"] = p
            self.stats = BlockStats(m_all=p.m_all, schedule=p.S, iters=p.iters, loads=p.loads,
                                    extras=dict(topk_idx=st["idx"], topk_w=st["w"], layout=p.layout,
                                                lrank=st["lrank"], tile_off=p.tile_off))

        fused = self.uses_fused_scatter(G * Tg)

        def permute():
            # fused: index-only scatter (buffer positions + inverse map); the FFN1 GEMM then
            # gathers each buffer row straight from x with cp.async loader warps, so the
            # permuted copy of x (T*k rows, 2x512 MB of HBM traffic at Qwen-128) is never
            # written.  Otherwise: 128-bit row copies into the segment-contiguous buffer.
            p = st["plan"]
            st["xs"], st["pos"], st["inv"] = ops.permute(st["x"], st["idx"], st["lrank"], p.tile_off, p.S,
                                                         p.layout.slot_base, G, Tg, 0, T * k, with_inverse=True,
                                                         index_only=fused, stream=s)
            self.stats.extras["pos"] = st["pos"]

        # swap-AB tiles (hm_grouped_gemm_swap: the weights on the MMA's M, 64 token rows on N, 9
        # stages of 16 KB weights + 4 KB tokens) for weight-streaming shapes, <= 64 rows per expert
        # on average: FFN2 by default (Switch-128 C1: 125 -> 119 us, step 284 -> 281 us); FFN1 only
        # on request - its short K = 768 tiles make the transposing epilogue cost more than the
        # padding rows it saves (120 -> 122 us).  Bit-identical either way.
        # HM_GEMM_SWAP=0 (never) / 1 (FFN1 and FFN2) / ffn2 overrides.
        env_sw = os.environ.get("HM_GEMM_SWAP", "")
        small = T * k <= 64 * E
        fits = G * E <= 512  # the swap kernel stages the segment table (<= G*E segments) in smem
        swap2 = fits and ((env_sw in ("1", "ffn2")) or (env_sw == "" and small))
        swap = fits and env_sw == "1" and not fused and cfg.activation == "relu"

        def gemm1():
            if swap:
                st["h"] = ops.grouped_gemm_swap(st["xs"], self.w_in, self.n_in, st["plan"].layout, self.epi_in,
                                                stream=s)
                return
            if fused:
                st["h"] = ops.grouped_gemm(st["x"], self.w_in, self.n_in, st["plan"].layout, self.epi_in,
                                           a_gather=st["inv"], a_gather_div=k, out_rows=T * k, stream=s)
            else:
                st["h"] = ops.grouped_gemm(st["xs"], self.w_in, self.n_in, st["plan"].layout, self.epi_in,
                                           stream=s)

        fuse_comb = self.uses_fused_combine()
        # top-1: the FFN2 epilogue writes y = (x +) w * Y itself (no counters, bit-identical)
        direct_comb = fuse_comb and k == 1

        def gemm2():
            # FFN2 scatters its rows token-major (row_map = inverse permutation) so the
            # combine reads each token's k expert outputs as one contiguous block
            if swap2 and (not fuse_comb or direct_comb):
                if direct_comb:
                    st["ys"] = None
                    st["y"] = ops.grouped_gemm_swap(st["h"], self.w_out, cfg.d_model, st["plan"].layout,
                                                    ops.HM_EPI_STORE, row_map=st["inv"], topk_w=st["w"],
                                                    residual=st["x"] if cfg.residual else None, stream=s)
                else:
                    st["ys"] = ops.grouped_gemm_swap(st["h"], self.w_out, cfg.d_model, st["plan"].layout,
                                                     ops.HM_EPI_STORE, row_map=st["inv"], stream=s)
                return
            if fuse_comb:
                st["ys"], st["y"] = ops.grouped_gemm_combine(
                    st["h"], self.w_out, cfg.d_model, st["plan"].layout, st["inv"], st["w"],
                    None if direct_comb else self._combine_counters(T), residual=st["x"] if cfg.residual else None,
                    stream=s)
            else:
                st["ys"] = ops.grouped_gemm(st["h"], self.w_out, cfg.d_model, st["plan"].layout, ops.HM_EPI_STORE,
                                            row_map=st["inv"], stream=s)

        def combine():
            if not fuse_comb:  # (fused: the FFN2 epilogue already wrote y)
                st["y"] = ops.combine(st["ys"], None, st["w"], residual=st["x"] if cfg.residual else None, stream=s)

        return [("router", router), ("schedule", plan), ("permute", permute), ("gemm1", gemm1),
                ("gemm2", gemm2), ("combine", combine)]

    @property
    def KERNELS_PER_FORWARD(self) -> int:  # router, plan, permute, gemm1, gemm2 (+ combine unless fused)
        return 5 if self.uses_fused_combine() else 6

    def uses_fused_combine(self) -> bool:
        """FFN2 with the combine in its epilogue (bit-identical either way): always for top-1 (the
        epilogue scales its row into y directly - no arrival counters; Switch-128 C1 287.7 ->
        283.9 us), else MoEConfig.fused_combine (top-8 Qwen: 820 vs 450 us; top-2 Mixtral: within
        run-to-run noise of the power-capped GEMMs, 3,091-3,240 vs 3,110-3,261 us for FFN2 + combine).
        HM_FUSED_COMBINE=0/1 overrides."""
        env = os.environ.get("HM_FUSED_COMBINE")
        return (env == "1") if env is not None else (self.cfg.fused_combine or self.cfg.top_k == 1)

    def _combine_counters(self, T: int) -> torch.Tensor:
        """Arrival counters of the fused combine, [T * d/64] int32; they return to zero after every
        forward, so one zeroed allocation (grown with the largest batch) serves every call."""
        n = T * (self.cfg.d_model // 64)
        if getattr(self, "_comb_ctr", None) is None or self._comb_ctr.numel() < n:
            self._comb_ctr = torch.zeros(n, dtype=torch.int32, device=self.device)
        return self._comb_ctr

    def capture(self, num_tokens: int, groups=(("router", "schedule", "permute"), ("gemm1",), ("gemm2",),
                                               ("combine",)), x_static: torch.Tensor | None = None,
                pool=None) -> "CapturedForward":
        """CUDA-graph the forward for a fixed token count.  The LOCAL forward never
        synchronises the host, so every kernel is captured; replay removes the launch gaps.
        Stages are captured in ``groups`` (one graph per group) so a caller can time
        groups with stream events between replays.  Write inputs into ``.x`` (or pass
        ``x_static``, e.g. the previous layer's static output)."""
        cfg = self.cfg
        G = cfg.num_ranks
        if num_tokens % G:
            raise ValueError("token count must divide evenly over the logical ranks")
        x = x_static if x_static is not None else torch.zeros((num_tokens, cfg.d_model), dtype=torch.bfloat16,
                                                              device=self.device)
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
        with torch.cuda.stream(side):
            stages = dict(self._stages(st, G, num_tokens // G, side))
        for grp in groups:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=pool, stream=side):
                for name in grp:
                    stages[name]()
            graphs.append(("+".join(grp), g))
        torch.cuda.synchronize(self.device)
        return CapturedForward(graphs, x, st["y"], self.stats)

    def host_pipeline(self, num_tokens: int, n_chunks: int = 4) -> HostPipeline:
        """Pinned-host end-to-end forward with H2D / compute / D2H overlapped by chunks."""
        return HostPipeline(self, num_tokens, n_chunks)

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Public end-to-end call with host buffers: H2D of x (pinned -> HBM), the block,
        D2H of y into pinned host memory.  Stream-ordered; sync before reading y_host."""
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            x = x_host.to(self.device, non_blocking=True)
            y = self.forward(x, stream=s)
            if y_host is None:
                y_host = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
            y_host.copy_(y, non_blocking=True)
        return y_host

    __call__ = forward
