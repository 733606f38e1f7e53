"""Graph Transformer attention layer on config 5 (batched molecules, 8 heads, d = 64): device time of
the projection GEMM, the fused 3S pass (strided, in place), the cast and the output GEMM, and of one
training step (forward_train + autograd backward: f3s_attention_fwd / f3s_attention_backward_saved_lp
between the GEMMs), as one JSON line (CUDA events, warm-up 3, median of 20)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from f3s_inputs import configs
    from paper_2505_08098_b200 import f3s
    from paper_2505_08098_b200.gt import GTAttention
    w = configs.get("batched")
    csr = w.graph()
    H, d = w.H, w.d
    plan = f3s.plan(torch.from_numpy(csr.row_ptr).cuda(), torch.from_numpy(csr.col_idx).cuda(), csr.n_rows)
    layer = GTAttention(H, d, dtype=torch.float16, seed=1)
    h = (torch.rand((csr.n_rows, H * d), device="cuda") * 2 - 1).half()
    stages = {}
    for _ in range(3):
        layer(plan, h)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ts = {k: [] for k in ("qkv_gemm", "fused_3s", "cast", "out_gemm", "layer")}
    for _ in range(20):
        ev[0].record()
        qkv = layer.project(h)
        ev[1].record()
        O = f3s.attention_qkv(plan, qkv, scale=layer.scale)
        ev[2].record()
        Oh = O.view(csr.n_rows, H * d).half()
        ev[3].record()
        Oh @ layer.W_o
        ev[4].record()
        torch.cuda.synchronize()
        for i, k in enumerate(("qkv_gemm", "fused_3s", "cast", "out_gemm")):
            ts[k].append(ev[i].elapsed_time(ev[i + 1]))
        ts["layer"].append(ev[0].elapsed_time(ev[4]))
    # one training step of the layer: forward_train (QKV GEMM, f3s_attention_fwd, output GEMM) and
    # the backward through autograd (output GEMM grads, f3s_attention_backward_saved_lp, QKV GEMM grads)
    for wgt in layer.parameters():
        wgt.requires_grad_(True)
    G = torch.rand((csr.n_rows, H * d), device="cuda").half()
    for _ in range(3):
        layer.forward_train(plan, h).backward(G)
    tr = {"train_forward": [], "train_backward": [], "train_step": []}
    for _ in range(20):
        for wgt in layer.parameters():
            wgt.grad = None
        ev[0].record()
        out = layer.forward_train(plan, h)
        ev[1].record()
        out.backward(G)
        ev[2].record()
        torch.cuda.synchronize()
        tr["train_forward"].append(ev[0].elapsed_time(ev[1]))
        tr["train_backward"].append(ev[1].elapsed_time(ev[2]))
        tr["train_step"].append(ev[0].elapsed_time(ev[2]))
    ts.update(tr)
    med = {k: round(float(np.median(v)), 4) for k, v in ts.items()}
    D = H * d
    gemm_flops = 2.0 * csr.n_rows * D * (3 * D + D)
    print(json.dumps({"layer": "GT attention (h W_qkv -> fused 3S -> O W_o)", "workload": w.description,
                      "n": csr.n_rows, "nnz": int(csr.nnz), "heads": H, "d": d, "dtype": "f16", "ms": med,
                      "gemm_tflops": round(gemm_flops / ((med["qkv_gemm"] + med["out_gemm"]) * 1e-3) / 1e12, 1),
                      "edge_gflops_3s": round(4.0 * csr.nnz * d * H / (med["fused_3s"] * 1e-3) / 1e9, 1)}))


if __name__ == "__main__":
    main()
