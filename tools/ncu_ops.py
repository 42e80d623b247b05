"""Per-opcode dynamic instruction counts (lane-ops per code) and stall reasons of one kernel in
an ncu report: python tools/ncu_ops.py rep.ncu-rep kernel_regex [codes]"""
import collections, csv, io, re, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
codes = float(sys.argv[3]) if len(sys.argv) > 3 else 134217728.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if "Instructions Executed" in r)
start = rows.index(h) + 1
si, ie, ws = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
cnt, st = collections.Counter(), collections.Counter()
tot = tws = 0
for r in rows[start:]:
    try:
        n, w = int(r[ie] or 0), int(r[ws] or 0)
    except (ValueError, IndexError):
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_.]+)", r[si])
    op = m.group(2) if m else r[si]
    cnt[op] += n
    st[op] += w
    tot += n
    tws += w
W = codes / 32
print(f"{tot} warp-instr = {tot / W:.2f} lane-ops/code, {tws} stall samples")
for o, n in cnt.most_common(30):
    print(f"  {o:24s} {n:>11} {n / W:6.2f}/code  stall {100 * st[o] / max(tws, 1):5.1f}%")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
row = next(r for r in rr[2:] if re.search(kern, r[hh.index("Kernel Name")]))
print("stall reasons (samples):")
for i, k in enumerate(hh):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            v = float(row[i])
        except ValueError:
            continue
        if v > 0.02 * max(tws, 1):
            print(f"  {k[33:]:30s} {v:8.0f} {100 * v / max(tws, 1):5.1f}%")
