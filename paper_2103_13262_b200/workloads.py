"""Synthetic workloads of BASELINE.json beyond the single layer.

* ``zipf_routing`` -- cfg5, the skewed-gate stress.  The reference gate cannot
  produce a Zipf distribution, so the routing is injected: a seeded sampler
  with P(e) ~ 1/(e+1)^s over expert ids in natural order, scores ~ U[0.5, 1].
  The same IndexMatrix is fed to the reference's build_plan
  (dispatch.hpp:28) and to ``MoELayer.forward_routed`` here.
* ``MoEStack`` -- cfg4, the GPT-style MoE FFN stack: ``n_layers`` independent
  MoE layers chained y_{l+1} = MoE_l(y_l) with no residual or norm (the
  reference has none), forward through all layers then backward through all.
  Layer l is initialised with init_state(seed + l) (moe_layer.cpp:28-45).
  All layers share one context (one stream and, under expert parallelism, one
  transport), so a stack costs one communicator, not one per layer.

Host-side generators only; every step runs through the C-ABI.
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np
import torch

from .api import Context, MoEConfig, MoELayer, ShapeError, World


def zipf_probabilities(num_experts: int, s: float = 1.0) -> np.ndarray:
    p = 1.0 / np.power(np.arange(1, num_experts + 1, dtype=np.float64), s)
    return p / p.sum()


def zipf_routing(n: int, num_experts: int, k: int = 1, s: float = 1.0, seed: int = 0):
    """(topk_idx [n, k] int32, topk_scores [n, k] float32) with expert e drawn
    with probability ~ 1/(e+1)^s; the k experts of a row are distinct
    (sampled without replacement, Gumbel top-k), scores ~ U[0.5, 1]."""
    if not 1 <= k <= num_experts:
        raise ShapeError("zipf_routing: k must lie in [1, num_experts]")
    rng = np.random.default_rng(seed)
    p = zipf_probabilities(num_experts, s)
    if k == 1:
        idx = rng.choice(num_experts, size=(n, 1), p=p).astype(np.int32)
    else:
        g = np.log(p)[None, :] - np.log(-np.log(rng.random((n, num_experts))))
        idx = np.argsort(-g, axis=1, kind="stable")[:, :k].astype(np.int32)
    scores = rng.uniform(0.5, 1.0, size=(n, k)).astype(np.float32)
    return idx, scores


class MoEStack:
    """``n_layers`` MoE layers chained without residual."""

    def __init__(self, config: MoEConfig, n_layers: int, rank: int = 0, dtype: torch.dtype = torch.bfloat16,
                 device=None):
        if n_layers < 1:
            raise ShapeError("MoEStack: n_layers must be at least 1")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.ctx = Context(dev.index if dev.index is not None else torch.cuda.current_device())
        self.config = config
        self.layers: List[MoELayer] = []
        for i in range(n_layers):
            c = MoEConfig(config.n_b, config.d_m, config.d_h, config.k, config.n_e_local, config.world_size,
                          config.seed + i)
            self.layers.append(MoELayer(c, rank=rank, dtype=dtype, device=dev, ctx=self.ctx))
        shape = (config.n_b, config.d_m)
        # activations between layers: each layer keeps its input alive until backward
        self.acts = [torch.empty(shape, dtype=dtype, device=dev) for _ in range(n_layers)]
        self.grads = [torch.empty(shape, dtype=dtype, device=dev) for _ in range(2)]

    def connect(self, dist):
        """Expert parallelism over NCCL: one communicator for the whole stack."""
        self.ctx.init_nccl(dist, self.config.world_size, self.layers[0].rank)

    def connect_peers(self, dist):
        """Fused peer-memory exchange for every layer, buffers swapped through
        torch.distributed (any backend); no device transport afterwards."""
        for layer in self.layers:
            layer.connect_peers(dist)

    def join(self, world: World):
        self.ctx.join_world(world, self.layers[0].rank)

    def forward(self, x: torch.Tensor, y: Optional[torch.Tensor] = None) -> torch.Tensor:
        """y = MoE_{L-1}(... MoE_0(x)); x must stay alive until backward()."""
        cur = x
        for i, layer in enumerate(self.layers):
            last = i == len(self.layers) - 1
            out = (y if y is not None else self.acts[i]) if last else self.acts[i]
            cur = layer.forward(cur, out)
        return cur

    def backward(self, dy: torch.Tensor, dx: Optional[torch.Tensor] = None) -> torch.Tensor:
        cur = dy
        for j, layer in enumerate(reversed(self.layers)):
            first_layer = j == len(self.layers) - 1
            out = dx if (first_layer and dx is not None) else self.grads[j & 1]
            cur = layer.backward(cur, out)
        return cur
