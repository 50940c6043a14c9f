"""Per-source-line instruction / stall-sample shares of one kernel in an ncu report.

    python scripts/ncu_lines.py gpurun_out/prof.ncu-rep [kernel_regex] [min_share]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else ".*"
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.012
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      f"regex:{kre}"], capture_output=True, text=True).stdout


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


cur, data = None, []
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r and r[0].isdigit():
        data.append((cur, r))
ts = sum(f(r[4]) for _, r in data) or 1
te = sum(f(r[7]) for _, r in data) or 1
print(f"stall samples {ts:.0f}, warp instructions {te:.0f}")
for fn, r in data:
    s, e = f(r[4]), f(r[7])
    if s / ts > thr or e / te > thr:
        print(f"{fn[:16]:>16}:{r[0]:>4} {100 * s / ts:5.1f}% {100 * e / te:5.1f}%  {r[1][:90]}")
