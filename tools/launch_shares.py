"""Per-kernel share of one step from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X`).  ncu serialises
kernels, so compare SHARES, not the sum, with the overlapped step time.

  python tools/launch_shares.py gpurun_out/launches_v3.csv [label]
"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot, n = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    name = re.sub(r"^void ", "", r[ik]).split("(")[0].split("<")[0]
    tot[name] += float(r[iv]) / 1e3
    n[name] += 1
s = sum(tot.values())
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{k:30s} n={n[k]:4d} total={tot[k]:10.1f} us  share={100 * tot[k] / s:5.1f}%  avg={tot[k] / n[k]:8.2f} us")
print(f"sum of kernel time (serialised by ncu) = {s:.1f} us for {sys.argv[2] if len(sys.argv) > 2 else 'the listed launches'}")
