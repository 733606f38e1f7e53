"""Time f3s_attention_backward on a bench workload and print one JSON line.

  python tools/bench_backward.py [--config arxiv] [--steps 20 --warmup 5] [--variant tc|simt|saved|saved_lp]

useful FLOPs per call: 8 * nnz * d * H (dP = dO V^T, dQ, dK, dV; the recomputed scores are not
counted).  Algorithmic HBM bytes per call (no reuse across rows or columns; e = H*d elements per row):
  prep         saved: O fp32 + dO fp32 read, dO16 written      N*e*(4+4+2)   + 8*N*H (LSE, D)
               saved_lp: O fp32 + dO (input dtype) read        N*e*(4+2)     + 8*N*H
  row pass     K and V rows per edge; Q, dO per row; dQ out    nnz*e*(2+2) + N*e*(2+2) + N*e*g
  column pass  Q and dO rows per edge (+ LSE, D); K, V per key row; dK, dV out
                                                               nnz*e*(2+2) + 8*nnz*H + Nc*e*(2+2) + 2*Nc*e*g
  with g = 4 (fp32 gradients) or 2 (saved_lp: gradients in the input dtype); tc (recomputing) adds the
  forward in partial mode: nnz*e*(2+2) + N*e*(2+4) + 8*N*H.
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
    e = H * d
    g = 2 if a.variant == "saved_lp" else 4
    prep = N * e * ((4 + 2) if a.variant == "saved_lp" else (4 + 4 + 2)) + 8 * N * H
    rows = nnz * e * 4 + N * e * 4 + N * e * g
    cols = nnz * e * 4 + 8 * nnz * H + Nc * e * 4 + 2 * Nc * e * g
    fwd = nnz * e * 4 + N * e * 6 + 8 * N * H if a.variant == "tc" else 0
    alg = prep + rows + cols + fwd
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
