"""F3S_TRACE profile mode: per-CTA SM cycles spent per pipeline phase, summed per role (printed as us at
the measured SM clock)."""
import argparse, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
NAMES = {0: "index: wait slot", 1: "index: queue fetch", 2: "index: issue",
         8: "prod: wait ids", 9: "prod: wait Q slot", 10: "prod: wait ring", 11: "prod: issue",
         24: "smax: wait idx", 25: "smax: wait S", 26: "smax: S->max", 27: "smax: bar+combine", 28: "smax: wait pempty",
         29: "smax: fence+arrive", 30: "smax: exp+rowsum", 31: "smax: P/m/l stores",
         32: "corr: wait P", 33: "corr: wait O", 34: "corr: merge", 35: "corr: store"}

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="arxiv")
    ap.add_argument("--out", default=None)
    ap.add_argument("--dtype", default="fp16", choices=["fp16", "e4m3"])
    a = ap.parse_args()
    import torch
    from f3s_inputs import configs
    from paper_2505_08098_b200 import f3s
    w = configs.get(a.config)
    csr = w.graph()
    Qb, Kb, Vb = w.qkv(csr)
    dev = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(torch.float16)
    if a.dtype == "e4m3":
        dev = lambda b: torch.from_numpy(b.view(np.float16).astype(np.float32)).to(torch.float8_e4m3fn).cuda()
    p = f3s.plan(torch.from_numpy(csr.row_ptr).cuda(), torch.from_numpy(csr.col_idx).cuda(), csr.n_rows)
    Q, K, V = dev(Qb), dev(Kb), dev(Vb)
    O = torch.empty(Q.shape, dtype=torch.float32, device="cuda")
    for _ in range(3):
        f3s.attention(p, Q, K, V, O, scale=w.scale)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tr = f3s.attention_trace(p, Q, K, V, O, scale=w.scale, trace_chunks=0)
    s.record(); tr = f3s.attention_trace(p, Q, K, V, O, scale=w.scale, trace_chunks=0); e.record(); torch.cuda.synchronize()
    print(f"{a.config}: profile-mode kernel {s.elapsed_time(e):.3f} ms")
    s.record(); f3s.attention(p, Q, K, V, O, scale=w.scale); e.record(); torch.cuda.synchronize()
    tr = tr.view(-1)[: tr.shape[0] * 64].view(tr.shape[0], 64).cpu().numpy()
    tr = tr[tr.any(1)]
    print(f"{a.config}: kernel {s.elapsed_time(e):.3f} ms (no diag)")
    ghz = float(os.environ.get("F3S_SM_GHZ", "1.92"))
    tot = tr.astype(np.float64).mean(0) / 1e3 / ghz
    for k, nm in NAMES.items():
        print(f"  {nm:24s} {tot[k]:9.1f} us/CTA")
    if a.out:
        np.save(a.out, tr)
    for ex, nm in [(1, "no softmax exp"), (2, "no MMA2"), (4, "no MMA1"), (6, "no MMAs"), (8, "no gathers"), (9, "no gathers+exp"), (14, "no gathers, no MMAs"), (16, "consumer proxy fence"), (32, "no S ld/max"), (33, "no S ld/max/exp"), (64, "no O stores"), (46, "skeleton: 2+4+8+32"), (110, "skeleton+no O stores"),
                   (128, "no correction work"), (128 + 33, "no corr, no S ld/exp"), (128 + 46, "skeleton, no corr")]:
        f3s.attention_trace(p, Q, K, V, O, scale=w.scale, trace_chunks=-ex)
        s.record(); f3s.attention_trace(p, Q, K, V, O, scale=w.scale, trace_chunks=-ex); e.record(); torch.cuda.synchronize()
        print(f"  experiment {ex:2d} ({nm:22s}): {s.elapsed_time(e):.3f} ms")

if __name__ == "__main__":
    main()
