"""Turn gpurun_out/prof/* (tools/profile_round.sh) into the committed
summaries under profiles/ (round tag argv[1], e.g. r01)."""
import json, os, subprocess, sys
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = "gpurun_out/prof"
def run(*a):
    return subprocess.run([sys.executable, *a], capture_output=True, text=True).stdout
os.makedirs("profiles", exist_ok=True)
open(f"profiles/{tag}_launches_bench_summary.txt", "w").write(run("tools/launch_profile.py", f"{src}/launches_bench.csv"))
subprocess.run(["cp", f"{src}/launches_bench.csv", f"profiles/{tag}_launches_bench.csv"])
for name in ("dgemm", "batched", "fft_rows", "gen", "panel", "ola_rows"):
    rep = f"{src}/{name}.ncu-rep"
    if os.path.exists(rep):
        txt = run("tools/ncu_summary.py", rep) + "\n-- top source lines by stall samples --\n" + run("tools/ncu_lines.py", rep, "25")
        open(f"profiles/{tag}_{name}_full_summary.txt", "w").write(txt)
# per-launch DRAM traffic of the A*G GEMM for bench.py's roofline.traffic
import csv, io
raw = subprocess.run(["ncu", "-i", f"{src}/dgemm.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6,
         "second": 1e9}
def num(k):  # value in base units (bytes, ns)
    return float(d[k].replace(",", "")) * SCALE.get(rows[1][h.index(k)], 1)
traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
json.dump({"kernel": d.get("Kernel Name", "")[:120], "dram_bytes_per_launch": traffic,
           "gpu_time_ns": num("gpu__time_duration.sum"),
           "source": f"ncu --set full capture ({src}/dgemm.ncu-rep)"},
          open(f"profiles/{tag}_dgemm_traffic.json", "w"), indent=1)
# the batched kernel's per-launch DRAM traffic (bench.py's secondary roofline.traffic)
if os.path.exists(f"{src}/batched.ncu-rep"):
    raw = subprocess.run(["ncu", "-i", f"{src}/batched.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, v = rows[0], rows[2]
    d = dict(zip(h, v))
    traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    json.dump({"kernel": d.get("Kernel Name", "")[:120], "dram_bytes_per_launch": traffic,
               "gpu_time_ns": num("gpu__time_duration.sum"), "systems": 65536,
               "source": f"ncu --set full capture ({src}/batched.ncu-rep)"},
              open(f"profiles/{tag}_batched_traffic.json", "w"), indent=1)
print("ok")
