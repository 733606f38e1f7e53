"""profiles/traffic.json[config] = dram__bytes_read.sum + dram__bytes_write.sum of the fused kernel
(one `ncu --set full` capture per config): python tools/update_traffic.py TAG config [config ...]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
path = os.path.join(ROOT, "profiles", "traffic.json")
traffic = json.load(open(path)) if os.path.exists(path) else {}
for c in sys.argv[2:]:
    rep = os.path.join(ROOT, "gpurun_out", f"{tag}_prof_{c}.ncu-rep")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "--json", "/tmp/_t.json"],
                         capture_output=True, text=True)
    j = json.load(open("/tmp/_t.json"))
    traffic[c] = int(j["dram_read"] + j["dram_write"])
    print(c, traffic[c])
json.dump(traffic, open(path, "w"), indent=1, sort_keys=True)
