"""Top SASS lines by warp-stall samples from an ncu source-page CSV export."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[iss]), r[ia], r[isrc]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for s, a, src in sorted(data, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% {a} {src[:110]}")
