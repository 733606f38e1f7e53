"""Achievable K/V row-gather bandwidth on this GPU for a workload's plan (diagnostics)."""
import ctypes, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def main():
    import torch
    from f3s_inputs import configs
    from paper_2505_08098_b200 import f3s
    so = os.path.join(ROOT, "tools", "libgather_bench.so")
    lib = ctypes.CDLL(so)
    lib.gather_bench.restype = ctypes.c_float
    lib.gather_bench.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    for name in sys.argv[1:] or ["arxiv"]:
        w = configs.get(name)
        csr = w.graph()
        p = f3s.plan(torch.from_numpy(csr.row_ptr).cuda(), torch.from_numpy(csr.col_idx).cuda(), csr.n_rows)
        rw_ptr, cols, masks, order = p.export()
        W = len(cols)
        dcols = torch.from_numpy(cols).cuda()
        K = torch.randn((csr.n_cols, w.H, w.d), device="cuda").half()
        V = torch.randn((csr.n_cols, w.H, w.d), device="cuda").half()
        gb = W * w.H * w.d * 2 * 2 / 1e9
        print(f"{name}: W={W} H={w.H} d={w.d} gathered K+V = {gb:.2f} GB")
        for mode, grids, blocks in [(0, [148 * 8, 148 * 16], [256, 512]), (1, [148 * 4, 148 * 8], [256, 512]), (2, [148 * 4, 148 * 8], [128])]:
            for g in grids:
                for b in blocks:
                    ms = lib.gather_bench(mode, dcols.data_ptr(), W, w.H, w.d, K.data_ptr(), V.data_ptr(), csr.n_cols, g, b, 4)
                    print(f"  mode {['ldg','cp.async','tma.gather4'][mode]:12s} grid {g:5d} block {b:4d}: {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s")

if __name__ == "__main__":
    main()
