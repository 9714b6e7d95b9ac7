"""profiles/ncu_traffic.json from an ncu summary (tools/ncu_summary.py output):
per kernel, dram__bytes_read.sum + dram__bytes_write.sum of its one captured
launch (an `ncu --set full` capture of the bench command), which bench.py
reports as the roofline's `traffic`.
    python tools/ncu_traffic.py profiles/r01_ncu_full_vN.json [workload]
(workload = the bench config the capture ran, default av2: bench.py uses the
figures only for that workload)"""
import json
import re
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def nbytes(s: str) -> float:
    v, u = s.split()
    return float(v.replace(",", "")) * UNITS[u]


src = sys.argv[1]
workload = sys.argv[2] if len(sys.argv) > 2 else "av2"
d = json.load(open(src))
# kernels this capture does not cover keep their entry from an earlier capture
try:
    out = json.load(open("profiles/ncu_traffic.json"))
except FileNotFoundError:
    out = {}
for rep, ks in d.items():
    for k in ks:
        name = k["kernel"]
        m = re.search(r"::(k_\w+)(<[^>]*>)?", name)
        if not m or "dram__bytes_read.sum" not in k:
            continue
        key = m.group(1) + (m.group(2) or "").replace(" ", "")
        out[key] = {"dram_bytes_per_launch": nbytes(k["dram__bytes_read.sum"]) +
                    nbytes(k["dram__bytes_write.sum"]),
                    "duration": k.get("gpu__time_duration.sum"), "source": src, "report": rep,
                    "workload": workload}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1, sort_keys=True)
print(json.dumps(out, indent=1, sort_keys=True))
