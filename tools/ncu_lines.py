"""Top CUDA source lines of a kernel by warp-stall samples (needs -lineinfo and
ncu --import-source on). usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
data, fname = [], ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 5 and r[0].isdigit():
        try:
            data.append((int(r[4] or 0), int(r[7] or 0), f"{fname}:{r[0]}", r[1].strip()[:100]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
for v, ex, ln, src in sorted(data, reverse=True)[:N]:
    print(f"{100*v/tot:5.1f}%  exec {ex:>10}  {ln:>22}  {src}")
