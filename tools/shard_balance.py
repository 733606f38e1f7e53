"""Per-shard kernel times of an N-GPU row-sharded run, measured on one GPU (each shard's plan and
Q rows alone, full K/V, cold L2): the kernel part of the strong-scaling curve.  The N-GPU kernel
makespan is the slowest shard; the [K||V] all-gather (one NCCL call, not measurable on one GPU) is
reported as bytes per rank.  Batched: graph-aligned shards with local K/V (weak sharding, no
collective).  Default split bound = the global one (shards bitwise equal to the 1-GPU result).

  python tools/shard_balance.py [--configs products arxiv reddit batched] [--worlds 1 2 4 8] [--reps 5]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["products", "arxiv", "reddit", "batched"])
    ap.add_argument("--worlds", nargs="+", type=int, default=[1, 2, 4, 8])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch
    from f3s_inputs import configs
    from paper_2505_08098_b200 import dist, f3s
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def timed(plan, Ql, K, V, O, scale):
        for _ in range(2):
            f3s.attention(plan, Ql, K, V, O, scale=scale)
        t = []
        for _ in range(a.reps):
            flush.fill_(1)
            ev[0].record()
            f3s.attention(plan, Ql, K, V, O, scale=scale)
            ev[1].record()
            torch.cuda.synchronize()
            t.append(ev[0].elapsed_time(ev[1]))
        return float(np.median(t))

    for cfg in a.configs:
        w = configs.get(cfg)
        csr = w.graph()
        Qb, Kb, Vb = w.qkv(csr)
        dev = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(torch.float16)
        Q, K, V = dev(Qb), dev(Kb), dev(Vb)
        batched = cfg == "batched"
        gptr = csr.graph_ptr if batched else None
        full = f3s.plan(torch.from_numpy(csr.row_ptr).cuda(), torch.from_numpy(csr.col_idx).cuda(), csr.n_rows)
        gbound = f3s.default_split_chunks(full.info()["total_chunks"], sms)
        del full
        t1 = None
        for world in a.worlds:
            bounds = dist.partition(csr.row_ptr, world, gptr)
            per = []
            for r in range(world):
                spec = dist.shard_spec(csr.row_ptr, csr.col_idx, r, world, gptr, bounds=bounds)
                p = f3s.plan_rows(torch.from_numpy(spec.row_ptr).cuda(), torch.from_numpy(spec.col_idx).cuda(),
                                  spec.row_end - spec.row_begin, spec.n_cols)
                p.set_split(gbound)
                Ql = Q[spec.row_begin:spec.row_end].contiguous()
                if batched:  # the rank's own graphs: local K/V rows
                    Kl, Vl = K[spec.row_begin:spec.row_end].contiguous(), V[spec.row_begin:spec.row_end].contiguous()
                else:
                    Kl, Vl = K, V
                Ol = torch.empty(Ql.shape, dtype=torch.float32, device="cuda")
                per.append(timed(p, Ql, Kl, Vl, Ol, w.scale))
                del p, Ql, Ol
            mk = max(per)
            t1 = mk if world == 1 else t1
            kv_bytes = 0 if batched or world == 1 else 2 * (-(-csr.n_rows // world)) * w.H * w.d * 2 * world
            print(f"{cfg:9s} N={world}: kernel makespan {mk:8.3f} ms (mean {np.mean(per):.3f}, "
                  f"imbalance {mk / np.mean(per):.3f}), kernel speedup vs 1 GPU {t1 / mk:5.2f} "
                  f"(ideal {world}), all-gather per rank {kv_bytes / 1e9:.3f} GB"
                  + ("  [weak: graph-aligned, no collective]" if batched else ""), flush=True)
        del Q, K, V
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
