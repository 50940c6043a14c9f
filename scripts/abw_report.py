"""Fresh-query times of the gpu_abw.sh logs."""
import glob, json
for f in sorted(glob.glob("gpurun_out/abw_*.log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            fq = d["fresh_query_ms"]
            print(f"{f[15:-4]:28s} k3 {fq['k3_directory']:.4f}  k4 {fq['k4_first_eval']:.4f}  total {fq['total']:.4f}  popcount {d['popcount']}")
