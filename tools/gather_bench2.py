"""Loader-design gather throughput in the fused kernel's shape (tools/gather_bench2.cu; diagnostics)."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from f3s_inputs import configs
    import oracle
    lib = ctypes.CDLL(os.path.join(ROOT, "tools", "libgather_bench2.so"))
    lib.gather_bench2.restype = ctypes.c_float
    lib.gather_bench2.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64]
    for name in sys.argv[1:] or ["products"]:
        w = configs.get(name)
        csr = w.graph()
        # the compacted columns of every row window, in window order (what the kernel gathers)
        rows16 = np.repeat(np.arange(csr.n_rows, dtype=np.int64) // 16, np.diff(csr.row_ptr))
        keys = np.unique(rows16 << 32 | csr.col_idx.astype(np.int64))
        cols = (keys & 0xFFFFFFFF).astype(np.int32)
        W = len(cols) // 128 * 128
        dcols = torch.from_numpy(cols[:W].copy()).cuda()
        H = w.H if w.d == 64 else 1
        K = torch.randn((csr.n_cols, H, 64), device="cuda").half()
        V = torch.randn((csr.n_cols, H, 64), device="cuda").half()
        n_chunks = W // 128 * H
        gb = n_chunks * 128 * 256 / 1e9
        print(f"{name}: {n_chunks} chunks of 128 rows x (K+V) 128 B, H={H}: {gb:.2f} GB", flush=True)
        for mode, nl, ntiles, pf in [(0, 8, 6, 0), (7, 8, 6, 0), (7, 16, 6, 0), (7, 24, 6, 0), (7, 24, 4, 0)]:
            ms = lib.gather_bench2(mode, nl, dcols.data_ptr(), n_chunks, H, K.data_ptr(), V.data_ptr(), ntiles, pf, 4, csr.n_cols)
            print(f"  {['cp.async','ldg+sts','tma.g4','K:tma,V:cpa','cp.async.ca','hyb 3/4','hyb 1/2','ldg pipe3'][mode]:9s} loaders {nl:2d} tiles {ntiles} prefetch {pf:2d}: "
                  f"{ms:8.3f} ms  {gb / ms * 1e3:6.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
