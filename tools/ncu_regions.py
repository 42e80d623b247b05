"""Instructions and stall samples of one kernel aggregated over source-line ranges:
python tools/ncu_regions.py rep kernel_regex name:file:lo-hi [name:file:lo-hi ...]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
regions = []
for spec in sys.argv[3:]:
    name, f, rng = spec.split(":")
    lo, hi = (int(x) for x in rng.split("-"))
    regions.append((name, f, lo, hi))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--launch-count", "1", "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, hdr, stats = None, None, {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        ws = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        ie = int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    stats[(cur_file, int(r[0]))] = (ie, ws)
ti = sum(v[0] for v in stats.values()) or 1
ts = sum(v[1] for v in stats.values()) or 1
acc = {}
for (f, l), (ie, ws) in stats.items():
    name = "other"
    for n, rf, lo, hi in regions:
        if f == rf and lo <= l <= hi:
            name = n
            break
    a = acc.setdefault(name, [0, 0])
    a[0] += ie
    a[1] += ws
for n, (ie, ws) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:28s} instr {100 * ie / ti:5.1f}%  stall samples {100 * ws / ts:5.1f}%")
