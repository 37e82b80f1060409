"""Aggregate ncu warp-stall samples by CUDA source line for one profiled kernel.

    python tools/ncu_lines.py report.ncu-rep <kernel regex or -> [launch index] [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
idx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
       "--launch-skip", str(idx), "--launch-count", "1"]
if kre != "-":
    cmd += ["--kernel-name", "regex:" + kre]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
res, f, hdr = [], None, None
for x in csv.reader(io.StringIO(out)):
    if x and x[0] == "File Path":
        f = x[1].split("/")[-1]
        continue
    if x and x[0] == "Function Name":
        continue
    if x and x[0] == "Line No":
        hdr = x
        continue
    if hdr and x and x[0] != "":
        try:
            res.append((float(x[4] or 0), f, x[0], x[1].strip()[:100]))
        except ValueError:
            pass
tot = sum(a for a, *_ in res) or 1.0
res.sort(key=lambda t: -t[0])
print(f"total samples {tot:.0f}")
for a, fn, ln, src in res[:top]:
    print(f"{100 * a / tot:5.1f}% {fn}:{ln}  {src}")
