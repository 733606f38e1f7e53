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


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_gt_layer_training_step(oracle_mod, dtype):
    """One training step of the layer (loss = <out, G>): autograd through the library GEMMs and
    attention_autograd (f3s_attention_fwd + f3s_attention_backward_saved) against the fp64 chain
    written out by hand -- dO = G W_o^T, the oracle backward for dQ, dK, dV, then dW_qkv = h^T
    [dQ | dK | dV] and dW_o = O^T G -- on the same fp16/bf16 projection values."""
    import torch

    from paper_2505_08098_b200 import f3s
    from paper_2505_08098_b200.gt import GTAttention
    tdt = torch.float16 if dtype == "fp16" else torch.bfloat16
    g = fi.molecules(400, seed=29)
    n, H, d = g.n_rows, 8, 64
    plan = f3s.plan(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda(), n)
    layer = GTAttention(H, d, dtype=tdt, seed=6)
    for w in layer.parameters():
        w.requires_grad_(True)
    gen = torch.Generator(device="cpu").manual_seed(10)
    h = (torch.rand((n, H * d), generator=gen) * 2 - 1).to(tdt).cuda()
    G = (torch.rand((n, H * d), generator=gen) * 2 - 1).cuda()
    out = layer.forward_train(plan, h)
    (out.float() * G).sum().backward()
    torch.cuda.synchronize()
    # fp64 chain on the layer's own rounded projection values
    Qb, Kb, Vb = (x.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
                  for x in layer.project_split(h))
    from conftest import decode
    Q64, K64, V64 = (decode(x, dtype) for x in (Qb, Kb, Vb))
    O64 = oracle_mod.attention_f64(g.row_ptr, g.col_idx, Q64, K64, V64, scale=layer.scale)
    # the chain rounds where the layer's tensors are stored in the input dtype: dout (the gradient
    # of the dtype output), dO (a dtype GEMM output), O (cast before W_o) and dQ, dK, dV (cast back)
    rnd = lambda x: torch.from_numpy(np.asarray(x, np.float64)).to(tdt).double().numpy()
    Wo = layer.W_o.detach().double().cpu().numpy()
    G64 = rnd(G.double().cpu().numpy())
    dO64 = rnd(G64 @ Wo.T).reshape(n, H, d)
    dQ, dK, dV = oracle_mod.attention_backward(g.row_ptr, g.col_idx, Q64, K64, V64, dO64, scale=layer.scale)
    dqkv = rnd(np.concatenate([x.reshape(n, H * d) for x in (dQ, dK, dV)], axis=1))
    dWqkv64 = h.double().cpu().numpy().T @ dqkv
    dWo64 = rnd(O64.reshape(n, H * d)).T @ G64
    for got, ref in ((layer.W_qkv.grad, dWqkv64), (layer.W_o.grad, dWo64)):
        got = got.double().cpu().numpy()
        scale = float(np.abs(ref).max())
        # the backward's inputs enter the tensor cores in the input dtype and the weight gradients
        # are rounded to it: BASELINE's tolerances relative to the gradient's scale
        assert_close(got / scale, ref / scale)


def test_autograd_packed_equals_split():
    """attention_autograd_qkv (packed [n, 3, H, d] operand and gradient) and attention_autograd on
    the three slices give the same O and the same gradients bit for bit (same kernels)."""
    import torch

    from paper_2505_08098_b200 import f3s
    g = fi.molecules(200, seed=31)
    n, H, d = g.n_rows, 8, 64
    plan = f3s.plan(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda(), n)
    gen = torch.Generator(device="cpu").manual_seed(12)
    qkv = (torch.rand((n, 3, H, d), generator=gen) * 2 - 1).half().cuda().requires_grad_(True)
    G = (torch.rand((n, H, d), generator=gen) * 2 - 1).half().cuda()
    O1 = f3s.attention_autograd_qkv(plan, qkv, scale=0.125, out_dtype=torch.float16)
    O1.backward(G)
    parts = [qkv.detach()[:, i].contiguous().requires_grad_(True) for i in range(3)]
    O2 = f3s.attention_autograd(plan, *parts, scale=0.125, out_dtype=torch.float16)
    O2.backward(G)
    torch.cuda.synchronize()
    assert torch.equal(O1, O2)
    for i in range(3):
        assert torch.equal(qkv.grad[:, i], parts[i].grad)
