"""Time f3s_attention_backward on a bench workload and print one JSON line.

  python tools/bench_backward.py [--config arxiv] [--steps 20 --warmup 5] [--variant tc|simt]

useful FLOPs per call: 8 * nnz * d * H (dP = dO V^T, dQ, dK, dV; the recomputed scores are not
counted).  Algorithmic bytes per call (HBM bound, no reuse across rows or columns):
  row pass     nnz*H*d*(2+2)   K and V rows per edge (fp16/bf16)      + N*H*d*(2+4+4)  Q, dO in, dQ out
  column pass  nnz*H*d*(2+4)   Q and dO rows per edge                 + Nc*H*d*(2+2+4+4) K, V in, dK, dV out
  + 8*N*H (LSE, D written) + 8*nnz*H (read back per edge).
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="arxiv")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--variant", default="tc", choices=["tc", "simt", "saved", "saved_lp"],
                    help="saved: f3s_attention_backward_saved on the outputs of f3s_attention_fwd (no recomputed forward)")
    a = ap.parse_args()
    import torch
    from f3s_inputs import configs
    from paper_2505_08098_b200 import f3s
    w = configs.get(a.config)
    csr = w.graph()
    Qb, Kb, Vb = w.qkv(csr)
    tdt = torch.float16 if w.dtype == "fp16" else torch.bfloat16
    dev = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(tdt)
    p = f3s.plan(torch.from_numpy(csr.row_ptr).cuda(), torch.from_numpy(csr.col_idx).cuda(), csr.n_rows)
    Q, K, V = dev(Qb), dev(Kb), dev(Vb)
    H, d = Q.shape[1], Q.shape[2]
    g = torch.Generator(device="cuda").manual_seed(1)
    dO = torch.randn(Q.shape, generator=g, device="cuda", dtype=torch.float32)
    if a.variant in ("saved", "saved_lp"):
        O, ml = f3s.attention_fwd(p, Q, K, V, scale=w.scale)
        dOs = dO.to(tdt) if a.variant == "saved_lp" else dO  # saved_lp: dO in the input dtype
        step = lambda: f3s.attention_backward_saved(p, Q, K, V, O, ml, dOs, scale=w.scale)
    else:
        step = lambda: f3s.attention_backward(p, Q, K, V, dO, scale=w.scale, variant=a.variant)
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.steps):
        step()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.steps
    fwd_ms = None
    if a.variant in ("saved", "saved_lp"):  # the training forward alone, for the fwd + bwd step time
        O2, ml2 = torch.empty_like(O), torch.empty_like(ml)
        for _ in range(3):
            f3s.attention_fwd(p, Q, K, V, O2, ml2, scale=w.scale)
        s.record()
        for _ in range(a.steps):
            f3s.attention_fwd(p, Q, K, V, O2, ml2, scale=w.scale)
        e.record()
        torch.cuda.synchronize()
        fwd_ms = s.elapsed_time(e) / a.steps
    info = p.info()
    nnz, N, Nc = info["nnz"], csr.n_rows, csr.n_cols
    flops = 8.0 * nnz * d * H
    alg = (nnz * H * d * (2 + 2) + N * H * d * (2 + 4 + 4) + nnz * H * d * (2 + 4) + Nc * H * d * (2 + 2 + 4 + 4)
           + 8 * N * H + 8 * nnz * H)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    gbs = alg / (ms * 1e-3) / 1e9
    print(json.dumps({"metric": "backward edge-GFLOP/s (8*nnz*d*heads / time)", "value": round(flops / (ms * 1e-3) / 1e9, 3),
                      "unit": "GFLOP/s", "ms_per_step": round(ms, 4), "steps": a.steps, "warmup": a.warmup,
                      "config": {"workload": a.config, "n": N, "nnz": nnz, "heads": H, "d": d, "dtype": w.dtype},
                      "roofline": {"bound": "hbm", "achieved": round(gbs, 2), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                   "frac": round(gbs / peaks["hbm_gbs"], 4), "alg_bytes_per_call": int(alg)},
                      "variant": a.variant,
                      "training_forward_ms": None if fwd_ms is None else round(fwd_ms, 4),
                      "kernels": {"tc": "forward (partial) + k_bwd_prep + k_bwd_sm100 rows + k_bwd_sm100 columns (tcgen05)",
                                  "saved": "k_bwd_prep + k_bwd_sm100 rows + k_bwd_sm100 columns (tcgen05); O, (m, l) saved "
                                           "by f3s_attention_fwd",
                                  "saved_lp": "k_bwd_prep (dO in the input dtype, read in place) + k_bwd_sm100 rows + "
                                              "k_bwd_sm100 columns (tcgen05); O, (m, l) saved by f3s_attention_fwd",
                                  "simt": "k_bwd_rows + k_bwd_cols (CUDA cores)"}[a.variant]}))


if __name__ == "__main__":
    main()
