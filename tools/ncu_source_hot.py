"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`,
plus the sample share of labelled regions (by address range)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iss, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ia], 16) if r[ia].startswith("0x") else int(r[ia]), r[isrc], float(r[iss] or 0), float(r[iex] or 0)))
    except (ValueError, IndexError):
        pass
tot = sum(d[2] for d in data) or 1
print(f"total samples {tot:.0f}, instructions {sum(d[3] for d in data):.0f}")
for a, s, n, e in sorted(data, key=lambda d: -d[2])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{a:6x} {100*n/tot:5.1f}% exec={e:9.0f}  {s[:90]}")
