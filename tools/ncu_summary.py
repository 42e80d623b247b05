"""Summarise an ncu report: key metrics per kernel + SASS opcode / stall breakdown."""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second"]
for r in rows[2:]:
    if kern and kern not in r[hdr.index("Kernel Name")]:
        continue
    print("----")
    for w in want:
        if w in hdr:
            print(f"  {w:60s} {r[hdr.index(w)]} {rows[1][hdr.index(w)]}")
if kern:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    si, ie, ws = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((r[si].strip(), int(r[ie] or 0), int(r[ws] or 0)))
        except Exception:
            pass
    tot = sum(d[1] for d in data) or 1
    tws = sum(d[2] for d in data) or 1
    op, ops = collections.Counter(), collections.Counter()
    for s, n, w in data:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", s)
        o = m.group(2) if m else s
        op[o] += n
        ops[o] += w
    print(f"SASS: {len(data)} instr, {tot} warp-inst executed, {tws} stall samples")
    for o, n in op.most_common(25):
        print(f"  {o:12s} {n:>12} {100 * n / tot:5.1f}%  stall {100 * ops[o] / tws:5.1f}%")
    print("top stall instructions:")
    for s, n, w in sorted(data, key=lambda d: -d[2])[:25]:
        print(f"  {100 * w / tws:5.1f}%  {n:>10}  {s[:90]}")
