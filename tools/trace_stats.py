"""Summarise an F3S_TRACE dump: per-stage latencies and per-CTA throughput."""
import sys

import numpy as np

names = ["ids", "gather", "mma1", "S", "P", "mma2", "O", "store"]


def main(path):
    tr = np.load(path)["trace"].astype(np.int64)
    tr = tr[(tr[:, :, 1] > 0).any(1)]  # CTAs that ran
    G, C, E = tr.shape
    valid = tr[:, :, 1] > 0
    t0 = tr[tr > 0].min()
    t1 = tr.max()
    print(f"{path}: grid={G} chunks/CTA max={valid.sum(1).max()} mean={valid.sum(1).mean():.1f} span={(t1 - t0) / 1e3:.1f} us")
    v = tr[valid]
    for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6)]:
        d = (v[:, b] - v[:, a]) / 1e3
        print(f"  {names[a]:>6s} -> {names[b]:<6s} median {np.median(d):7.2f} us  p90 {np.percentile(d, 90):7.2f}")
    st = v[v[:, 7] > 0]
    d = (st[:, 7] - st[:, 6]) / 1e3
    print(f"  {'O':>6s} -> {'store':<6s} median {np.median(d):7.2f} us")
    # per-CTA inter-chunk interval at each stage (throughput of each role)
    for e in [1, 2, 3, 6]:
        iv = []
        for g in range(G):
            x = tr[g, valid[g], e]
            if len(x) > 2:
                iv.append(np.median(np.diff(x)))
        print(f"  per-CTA median interval between consecutive '{names[e]}' events: {np.median(iv) / 1e3:.2f} us")
    end = np.array([tr[g][valid[g]].max() if valid[g].any() else t0 for g in range(G)])
    start = np.array([tr[g][valid[g]][:, 0].min() if valid[g].any() else t0 for g in range(G)])
    print(f"  CTA start spread {(start.max() - start.min()) / 1e3:.1f} us, end spread {(end.max() - end.min()) / 1e3:.1f} us")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
