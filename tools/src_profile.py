"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export per source line and
per region: warp instructions executed per tile-step (divide by the tile count x warps)."""
import csv, collections, sys

path = sys.argv[1]
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
rows = list(csv.reader(open(path)))
cur = None; ie = None; sc = None
agg = collections.Counter(); samp = collections.Counter(); src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split('/')[-1]; continue
    if r[0] == "Line No":
        ie = r.index("Instructions Executed"); sc = r.index("Warp Stall Sampling (All Samples)"); continue
    if r[0] == "Function Name" or ie is None:
        continue
    if r[0] != "":
        cur = (f, int(r[0])); src[cur] = r[1]; continue
    if r[ie].isdigit():
        agg[cur] += int(r[ie])
    if r[sc].isdigit():
        samp[cur] += int(r[sc])
tot = sum(agg.values()); ts = sum(samp.values())
print(f"total warp instructions {tot} ({tot / norm:.1f} per unit), stall samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v / norm:7.1f} {100 * samp[k] / max(ts, 1):5.1f}%s  {k[0]}:{k[1]:<5d} {src[k][:90]}")
