"""Summarise an ncu report (one kernel) into the numbers profiles/ keeps:
duration, DRAM bytes, throughputs, L2 hit rate, tensor/TMA pipe activity, occupancy, top stalls.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json] [--alg-bytes B]
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum": "l2_to_sm_read",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_elapsed": "tma_pipe_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "instructions",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9,
         "second": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--json")
    ap.add_argument("--alg-bytes", type=float, default=None)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")][:120]}
    stalls = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            out[KEYS[h]] = x * SCALE.get(u, 1) if u in SCALE else x
            if u in SCALE:
                out[KEYS[h] + "_unit"] = "bytes" if "byte" in u else "s"
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v.replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1
    out["stall_share_top"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
    if "dram_read" in out and "dram_write" in out:
        out["dram_traffic_bytes"] = out["dram_read"] + out["dram_write"]
        if "duration" in out:
            out["dram_GBps"] = out["dram_traffic_bytes"] / out["duration"] / 1e9
    if a.alg_bytes and "duration" in out:
        out["alg_bytes"] = a.alg_bytes
        out["alg_GBps"] = a.alg_bytes / out["duration"] / 1e9
    for k, v in out.items():
        print(f"{k:28s} {v}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
