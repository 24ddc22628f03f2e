"""Attribute warp-stall samples of a GEMM ncu report to the mbarrier each spin
loop waits on (TRYWAIT + BRA pairs), plus the top non-spin instructions."""
import csv, re, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
names = {}  # offset base -> name, caller passes e.g. 0x30000=full,0x30040=empty
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    names[int(k, 16)] = v
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr, rows = r[1], r[2:]
i = hdr.index("Warp Stall Sampling (All Samples)")
j = hdr.index("Source")
tot = sum(float(x[i] or 0) for x in rows)
agg = defaultdict(float)
other = []
last = None
for x in rows:
    s = float(x[i] or 0)
    src = x[j].strip()
    m = re.search(r"TRYWAIT.*\+0x([0-9a-f]+)\]", src)
    if m:
        off = int(m.group(1), 16)
        base = max([b for b in names if b <= off], default=None)
        last = f"{names.get(base, '?')}+{off - (base or 0):#x}" if base is not None else hex(off)
        agg[last.split('+')[0]] += s
        continue
    if "BRA" in src and last is not None and s > 0:
        agg[last.split('+')[0]] += s
        continue
    last = None if "BRA" not in src else last
    other.append((s, src))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"spin on {k:10s} {100 * v / tot:5.1f}%")
for s, src in sorted(other, key=lambda t: -t[0])[:12]:
    print(f"{100 * s / tot:5.1f}%  {src[:100]}")
