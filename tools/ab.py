"""Same-process A/B of experiment builds (libf3s_<variant>.so): the workload is generated once,
each library builds its own plan, and the variants are timed round-robin (CUDA events, L2 flushed
before every call) so that box-to-box drift cancels.  Outputs are compared with the first variant's.

  python tools/ab.py --configs products reddit --variants base w1 w2 [--reps 10] [--rounds 3]
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def load(variant):
    name = "libf3s.so" if variant == "base" else f"libf3s_{variant}.so"
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2505_08098_b200", name), mode=ctypes.RTLD_LOCAL)
    vp, i32, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_float
    lib.f3s_plan.argtypes = [vp, vp, i32, vp, ctypes.POINTER(vp)]
    lib.f3s_attention.argtypes = [vp, vp, vp, vp, vp, f32, i32, i32, i32, vp]
    lib.f3s_last_error.restype = ctypes.c_char_p
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["products", "reddit", "arxiv", "batched"])
    ap.add_argument("--variants", nargs="+", required=True)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--dtype", default="fp16")
    a = ap.parse_args()
    import torch
    from f3s_inputs import configs
    libs = {v: load(v) for v in a.variants}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for cfg in a.configs:
        w = configs.get(cfg)
        csr = w.graph()
        Qb, Kb, Vb = w.qkv(csr, dtype=a.dtype)
        tdt = torch.float16 if a.dtype == "fp16" else torch.bfloat16
        dev = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(tdt)
        Q, K, V = dev(Qb), dev(Kb), dev(Vb)
        rp = torch.from_numpy(csr.row_ptr).cuda()
        ci = torch.from_numpy(csr.col_idx).cuda()
        plans, outs = {}, {}
        for v, lib in libs.items():
            p = ctypes.c_void_p()
            st = lib.f3s_plan(rp.data_ptr(), ci.data_ptr(), csr.n_rows, stream, ctypes.byref(p))
            assert st == 0, (v, st, lib.f3s_last_error())
            plans[v] = p
            outs[v] = torch.empty(Q.shape, dtype=torch.float32, device="cuda")
        dt = 0 if a.dtype == "fp16" else 1

        def call(v):
            st = libs[v].f3s_attention(plans[v], Q.data_ptr(), K.data_ptr(), V.data_ptr(), outs[v].data_ptr(),
                                       w.scale, w.H, w.d, dt, stream)
            assert st == 0, (v, st, libs[v].f3s_last_error())

        for v in libs:
            for _ in range(3):
                call(v)
        torch.cuda.synchronize()
        times = {v: [] for v in libs}
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for _ in range(a.rounds):
            for v in libs:
                for _ in range(a.reps):
                    flush.fill_(1)
                    ev[0].record()
                    call(v)
                    ev[1].record()
                    torch.cuda.synchronize()
                    times[v].append(ev[0].elapsed_time(ev[1]))
        ref = outs[a.variants[0]]
        for v in libs:
            t = np.array(times[v])
            diff = (outs[v] - ref).abs().max().item()
            print(f"{cfg:9s} {v:8s} median {np.median(t):8.4f} ms  p10 {np.percentile(t, 10):8.4f}  "
                  f"p90 {np.percentile(t, 90):8.4f}  max|O-O_{a.variants[0]}| {diff:.2e}", flush=True)
        del plans, outs, Q, K, V
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
