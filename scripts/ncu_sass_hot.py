"""Per-region instruction / stall-sample breakdown of an ncu source page (sass view).

    ncu -i rep --page source --csv --print-source sass > x.csv
    python scripts/ncu_sass_hot.py x.csv [region_size_bytes]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, isamp, iexec = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
data = [r for r in rows[2:] if len(r) > iexec and r[ia].startswith("0x")]
base = int(data[0][ia], 16)
tot_s = sum(float(r[isamp] or 0) for r in data)
tot_e = sum(float(r[iexec] or 0) for r in data)
reg = int(sys.argv[2]) if len(sys.argv) > 2 else 0x100
agg = {}
for r in data:
    off = int(r[ia], 16) - base
    k = off // reg
    s, e = agg.get(k, (0.0, 0.0))
    agg[k] = (s + float(r[isamp] or 0), e + float(r[iexec] or 0))
print(f"total samples {tot_s:.0f}, warp-instr {tot_e:.0f}")
for k, (s, e) in sorted(agg.items()):
    if s / tot_s > 0.01 or e / tot_e > 0.01:
        print(f"0x{k*reg:05x}-0x{(k+1)*reg:05x}  samples {100*s/tot_s:5.1f}%  instr {100*e/tot_e:5.1f}%")
