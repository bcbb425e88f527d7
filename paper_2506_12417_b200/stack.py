"""BASELINE config 4: a multi-layer MoE decoder stack, h_{l+1} = h_l + MoE_l(h_l).

The reference replays a trace layer by layer: batch latency is the sum over layers
of the layer latency (+ a fixed non-MoE constant), every layer schedules its own
routing matrix, and fetched experts never outlive their layer (engine.py:13-15,
393-477).  Here each layer is a full B200 block with its own router, experts and
HarMoEny schedule (per-layer rebalancing; in EP mode per-layer async fetches into
that layer's cache slots), and the decoder residual is fused into each layer's
combine kernel.  The attention / dense parts of a real decoder are not part of this
hot path; the reference models them as a constant
(``non_moe_layer_time``, core.py:75).
"""

from __future__ import annotations

from dataclasses import replace

import torch

from .block import BlockStats, CapturedForward, HarMoEnyBlock, MoEConfig, random_weights


class MoEStack:
    def __init__(self, layers: list):
        if not layers:
            raise ValueError("a stack needs at least one layer")
        self.layers = layers
        self.cfg = layers[0].cfg

    @classmethod
    def random(cls, cfg: MoEConfig, num_layers: int, seed: int = 0, device="cuda", zipf_s: float | None = None,
               std: float = 0.02, group=None):
        cfg = replace(cfg, residual=True)
        layers = []
        for i in range(num_layers):
            w = random_weights(cfg, seed + 1000 * i, device, zipf_s, std)
            if cfg.world_size > 1:
                from .ep import EPHarMoEnyBlock

                layers.append(EPHarMoEnyBlock(cfg, *w, device=device, group=group))
            else:
                layers.append(HarMoEnyBlock(cfg, *w, device=device))
        return cls(layers)

    @property
    def stats(self) -> list[BlockStats]:
        return [blk.stats for blk in self.layers]

    @property
    def device(self):
        return self.layers[0].device

    @property
    def KERNELS_PER_FORWARD(self) -> int:
        return sum(blk.KERNELS_PER_FORWARD for blk in self.layers)

    def forward(self, x: torch.Tensor, stream=None, marks: list | None = None) -> torch.Tensor:
        h = x
        for blk in self.layers:
            lm = [] if marks is not None else None
            h = blk.forward(h, stream=stream, marks=lm)
            if marks is not None:
                marks.extend(lm if not marks else lm[1:])
        return h

    __call__ = forward

    def forward_host(self, x_host, y_host=None, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            x = x_host.to(self.layers[0].device, non_blocking=True)
            y = self.forward(x, stream=s)
            if y_host is None:
                y_host = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
            y_host.copy_(y, non_blocking=True)
        return y_host

    def capture(self, num_tokens: int, groups=(("router", "schedule", "permute"), ("gemm1",), ("gemm2",),
                                               ("combine",))) -> CapturedForward:
        """Graph every layer (LOCAL mode), chaining each layer's static input to the previous
        layer's static output; replay runs all layers' groups in order."""
        pool = torch.cuda.graph_pool_handle()
        caps = []
        x_static = None
        for blk in self.layers:
            cap = blk.capture(num_tokens, groups=groups, x_static=x_static, pool=pool)
            caps.append(cap)
            x_static = cap.y
        graphs = [g for cap in caps for g in cap.graphs]
        return CapturedForward(graphs, caps[0].x, caps[-1].y, [c.stats for c in caps])

    def host_pipeline(self, num_tokens: int, n_chunks: int = 2):
        from .block import HostPipeline

        return HostPipeline(self, num_tokens, n_chunks)
