"""Graph Transformer attention layer on the fused 3S pass (second half;
PAPER.md:683-694: the GT model's attention layer, whose 3S kernel the paper swaps for Fused3S).

  h -> QKV = h W_qkv            one library GEMM (cuBLAS, fp16/bf16 in, fp32 accumulate), output
                                [n, 3, H, d] used in place: f3s_attention_strided reads Q, K, V
                                through their row strides (no split copies)
     O   = softmax_row(scale (Q K^T) ⊙ A) V     the fused 3S pass (libf3s, tcgen05)
     out = O W_o                one library GEMM on O cast to the input dtype

Weights are random-initialised (no trained weights exist offline); no bias, residual or
normalisation (those belong to the surrounding block).  forward() is the inference layer;
forward_train() the same layer under autograd, its 3S backward on the tensor cores (f3).
"""
from __future__ import annotations

import math

from . import f3s


class GTAttention:
    """Multi-head graph attention layer of the Graph Transformer over one plan (A fixed)."""

    def __init__(self, heads: int, d: int, *, dtype=None, device=None, seed: int = 0):
        import torch
        self.H, self.d = heads, d
        self.dtype = dtype or torch.float16
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        D = heads * d
        g = torch.Generator(device="cpu").manual_seed(seed)
        std = 1.0 / math.sqrt(D)  # keeps projections O(1) for O(1) inputs
        self.W_qkv = (torch.randn((D, 3 * D), generator=g) * std).to(self.dtype).to(self.device)
        self.W_o = (torch.randn((D, D), generator=g) * std).to(self.dtype).to(self.device)
        self.scale = 1.0 / math.sqrt(d)

    def project(self, h):
        """QKV = h W_qkv as [n, 3, H, d] (library GEMM)."""
        return (h @ self.W_qkv).view(h.shape[0], 3, self.H, self.d)

    def forward(self, plan: "f3s.Plan", h, *, stream=None):
        """h [n, H*d] (dtype) -> out [n, H*d] (dtype); A is the plan's graph (square)."""
        qkv = self.project(h)
        O = f3s.attention_qkv(plan, qkv, scale=self.scale, stream=stream)
        return O.view(h.shape[0], self.H * self.d).to(self.dtype) @ self.W_o

    __call__ = forward

    def parameters(self):
        return [self.W_qkv, self.W_o]

    def project_split(self, h):
        """Q, K, V = h W_q, h W_k, h W_v as three contiguous [n, H, d] GEMM outputs (the column blocks
        of W_qkv): the training pair needs contiguous operands, and three GEMMs write them directly
        instead of one packed output plus three copies."""
        D = self.H * self.d
        return tuple((h @ self.W_qkv[:, i * D:(i + 1) * D]).view(h.shape[0], self.H, self.d) for i in range(3))

    def forward_train(self, plan: "f3s.Plan", h):
        """The same layer with autograd (a training step): Q, K, V from project_split, the 3S pass
        runs f3s_attention_fwd and its backward f3s_attention_backward_saved_lp (attention_autograd,
        the attention output cast to the input dtype so that its gradient arrives in it); set
        requires_grad on the weights and/or h."""
        Q, K, V = self.project_split(h)
        O = f3s.attention_autograd(plan, Q, K, V, scale=self.scale, out_dtype=self.dtype)
        return O.view(h.shape[0], self.H * self.d) @ self.W_o
