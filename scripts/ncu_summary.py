"""Summarise an ncu --set full report into profiles/ (run here, no GPU needed).

    python scripts/ncu_summary.py gpurun_out/prof_c2.ncu-rep c2 r01 [sum]

writes profiles/<round>_<workload>_ncu.json (per-launch key metrics) and merges
the per-launch DRAM traffic into profiles/ncu_traffic.json (read by bench.py
for roofline.traffic): the mean over the captured launches, or with ``sum`` the
sum of the captured launches (one step made of several kernels, e.g. the C4
fresh query = K3 + K4).  The warp-stall sample counts of every launch are kept.
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1}
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
       "launch__block_size", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "l1tex__t_bytes.sum", "lts__t_bytes.sum"]


def summarise(rep: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, m in enumerate(hdr):
            if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("_not_issued"):
                try:
                    v = float(r[k].replace(",", ""))
                except ValueError:
                    continue
                if v:
                    d.setdefault("stall_samples", {})[m[len("smsp__pcsamp_warps_issue_stalled_"):]] = v
        for m in RAW:
            if m in hdr:
                k = hdr.index(m)
                try:
                    v = float(r[k].replace(",", ""))
                except ValueError:
                    continue
                u = units[k]
                d[m] = v * SCALE.get(u, 1) if u in SCALE else v
                if u and u not in SCALE:
                    d[m + ".unit"] = u
        out.append(d)
    return out


def main():
    rep, workload, rnd = sys.argv[1], sys.argv[2], sys.argv[3]
    mode = sys.argv[4] if len(sys.argv) > 4 else "mean"
    launches = summarise(rep)
    prof = os.path.join(ROOT, "profiles")
    with open(os.path.join(prof, f"{rnd}_{workload}_ncu.json"), "w") as fp:
        json.dump({"source": f"ncu --set full --clock-control none ({os.path.basename(rep)})",
                   "launches": launches}, fp, indent=1)
    traffic = [d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in launches
               if "dram__bytes_read.sum" in d]
    tpath = os.path.join(prof, "ncu_traffic.json")
    t = json.load(open(tpath)) if os.path.exists(tpath) else {}
    if traffic and mode == "sum":
        t[workload] = round(sum(traffic))
        t[workload + "_source"] = (f"profiles/{rnd}_{workload}_ncu.json: sum over the step's {len(traffic)} "
                                   "kernels of dram__bytes_read.sum + dram__bytes_write.sum")
    elif traffic:
        t[workload] = round(sum(traffic) / len(traffic))
        t[workload + "_source"] = (f"profiles/{rnd}_{workload}_ncu.json: mean over {len(traffic)} launch(es) of "
                                   "dram__bytes_read.sum + dram__bytes_write.sum")
    with open(tpath, "w") as fp:
        json.dump(t, fp, indent=1)
    for d in launches:
        print(workload, d["kernel"][:50], {k: d[k] for k in ("gpu__time_duration.sum", "dram__bytes_read.sum",
                                                             "dram__bytes_write.sum") if k in d})


if __name__ == "__main__":
    main()
