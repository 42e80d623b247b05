"""Per-CUDA-source-line instruction counts and stall samples from an ncu report."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--launch-count", "1", "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file = None
stats = {}
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] != "":
        try:
            ws = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            ie = int(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        stats[(cur_file, int(r[0]))] = (ie, ws, r[1].strip()[:100])
tot = sum(v[0] for v in stats.values()) or 1
tws = sum(v[1] for v in stats.values()) or 1
print(f"total warp-inst {tot}, stall samples {tws}")
print("by stall:")
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"  {100*v[1]/tws:5.1f}% st {100*v[0]/tot:5.1f}% in  {k[0]}:{k[1]}  {v[2]}")
print("by instructions:")
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"  {100*v[0]/tot:5.1f}% in {100*v[1]/tws:5.1f}% st  {k[0]}:{k[1]}  {v[2]}")
