"""Graph Transformer attention layer on config 5's shape
(batched molecule-like graphs, 8 heads, d = 64).  Two checks:
  * the fused pass reading Q, K, V in place from the projection output [n, 3, H, d]
    (f3s_attention_strided) against the fp64 oracle on exactly those fp16 values;
  * the whole layer against an fp64 chain (h W_qkv rounded to fp16 -> oracle attention -> O
    rounded to fp16 -> O W_o): GEMM accumulation order changes the fp16 rounding of a few
    projection values by one unit, so the layer is compared within BASELINE's tolerances relative
    to the output's scale."""
import numpy as np
import pytest

import f3s_inputs as fi
from helpers import assert_close

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_gt_layer(oracle_mod, dtype):
    import torch

    from paper_2505_08098_b200 import f3s
    from paper_2505_08098_b200.gt import GTAttention
    tdt = torch.float16 if dtype == "fp16" else torch.bfloat16
    g = fi.molecules(800, seed=23)
    n, H, d = g.n_rows, 8, 64
    plan = f3s.plan(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda(), n)
    layer = GTAttention(H, d, dtype=tdt, seed=5)
    gen = torch.Generator(device="cpu").manual_seed(9)
    h = (torch.rand((n, H * d), generator=gen) * 2 - 1).to(tdt).cuda()
    out = layer(plan, h)
    qkv = layer.project(h)
    O = f3s.attention_qkv(plan, qkv, scale=layer.scale)
    torch.cuda.synchronize()
    # (1) the strided fused pass on the GEMM's own fp16 output, against the oracle
    bits = qkv.view(torch.int16).cpu().numpy().view(np.uint16)
    Qb, Kb, Vb = (np.ascontiguousarray(bits[:, i]) for i in range(3))
    ref_O = oracle_mod.attention(g.row_ptr, g.col_idx, Qb, Kb, Vb, scale=layer.scale, dtype=dtype)
    assert_close(O.cpu().numpy(), ref_O)
    # (2) the layer against the fp64 chain
    h64 = h.double().cpu()
    q64 = (h64 @ layer.W_qkv.double().cpu()).to(tdt).view(n, 3, H, d)
    b64 = q64.view(torch.int16).numpy().view(np.uint16)
    O64 = oracle_mod.attention(g.row_ptr, g.col_idx, *(np.ascontiguousarray(b64[:, i]) for i in range(3)),
                               scale=layer.scale, dtype=dtype)
    out64 = torch.from_numpy(O64).view(n, H * d).to(tdt).double() @ layer.W_o.double().cpu()
    scale = float(out64.abs().max())
    assert_close(out.double().cpu().numpy() / scale, out64.numpy() / scale)
