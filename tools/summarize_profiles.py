"""Summarise gpurun_out/{launches.csv, full.ncu-rep} into profiles/<round>_*.{md,json}."""
import collections, csv, io, json, os, subprocess, sys

rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out")
prof = os.path.join(root, "profiles")
os.makedirs(prof, exist_ok=True)

# ---- launch list: per-kernel count and total time (cold-cache, serialised) ----
rows = []
with open(os.path.join(go, "launches.csv")) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(io.StringIO("".join(lines))):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        rows.append((r["Kernel Name"].split("(")[0].replace("void ", ""), float(r["Metric Value"]), r["Metric Unit"]))
agg = collections.OrderedDict()
for name, v, unit in rows:
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v * scale
ours = {k: v for k, v in agg.items() if k.startswith("fz::") or k.startswith("k_")}
tot = sum(v[1] for v in ours.values()) or 1.0
with open(os.path.join(prof, f"{rnd}_launches.md"), "w") as f:
    f.write(f"# {rnd} launch list (ncu --metrics gpu__time_duration.sum --clock-control none)\n\n")
    f.write("Command: `python bench.py --steps 2 --warmup 1 --no-cpu-baseline` (c4 512^3 REL 1e-3).\n")
    f.write("Per-launch times are cold-cache and serialised: compare shares, not absolutes.\n\n")
    f.write("| kernel | launches | total us | us/launch | share of libfz time |\n|---|---|---|---|---|\n")
    for k, (c, t) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
        f.write(f"| {k} | {c} | {t:.1f} | {t / c:.1f} | {100 * t / tot:.1f}% |\n")
    other = {k: v for k, v in agg.items() if k not in ours}
    f.write(f"\nOther (torch) kernels in the run: {sum(v[0] for v in other.values())} launches "
            f"({', '.join(sorted(set(k[:40] for k in other)))})\n")

# ---- ncu --set full: key metrics per kernel ----
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def summarize(rep, md, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    res = collections.OrderedDict()
    for r in rr[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        d = {}
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                d[w] = (r[i], units[i])
        res.setdefault(name, []).append(d)
    traffic = {}
    with open(md, "w") as f:
        f.write(title)
        for name, lst in res.items():
            d = lst[-1]
            f.write(f"## {name} ({len(lst)} captured launch(es), last shown)\n\n")
            for k, (v, u) in d.items():
                f.write(f"- {k}: {v} {u}\n")
            rd = to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else 0
            wr = to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else 0
            short = name.split("::")[-1].split("<")[0]
            traffic[short] = int(rd + wr)
            f.write(f"- dram traffic per launch: {(rd + wr) / 1e6:.1f} MB\n\n")
    return traffic


out = {"c4": summarize(os.path.join(go, "full.ncu-rep"), os.path.join(prof, f"{rnd}_ncu_full.md"),
                       f"# {rnd} ncu --set full (clock-control none), c4 512^3 REL 1e-3 via tools/prof_step.py\n\n")}
cl = os.path.join(go, "full_cl.ncu-rep")
if os.path.exists(cl):
    out["c4_chunk_local"] = summarize(cl, os.path.join(prof, f"{rnd}_ncu_full_cl.md"),
                                      f"# {rnd} ncu --set full, c4 512^3 REL 1e-3, chunk-local mode (f1), "
                                      f"tools/prof_step.py (launches after the field-global steps)\n\n")
out["_source"] = f"profiles/{rnd}_ncu_full*.md (dram__bytes_read.sum + dram__bytes_write.sum)"
with open(os.path.join(prof, "ncu_traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
