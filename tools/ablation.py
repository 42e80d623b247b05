"""Ablations of the fused design (analogous to the paper's Fig. 8).

Runs bench.py (c4 512^3 REL 1e-3, 1 GPU) once per variant, selected by FZ_EXP bits (bench.py
passes them to fz_debug_set_variant; libfz reads no environment), and writes profiles/<round>_ablation.md with the step, compress and decompress
throughput and the per-kernel times:
  base          row-walking compressor with the fused range phase (k_compress_zr + k_compact),
                row-walking decoder (k_dzr_*), programmatic dependent launch
  range_unfused FZ_EXP=2097152 separate k_range launch before the row walker
  no_pdl        FZ_EXP=67108864 kernels launched without programmatic dependent launch
  dec_chunk16   FZ_EXP=33554432 decoder units of 16 planes instead of the balanced depth
  zr_3stage     FZ_EXP=16384 row walker with three TMA stages (two CTAs per SM)
  zband_comp    FZ_EXP=8192 z-band compressor (k_compress_zb, round 1's)
  ws_comp       FZ_EXP=9216 warp-specialized single-pass compressor (TMA + scanner warp look-back)
  plane_dec     FZ_EXP=32768 plane decoder (x+y fused, int32 field) + z walk (round 1's)
  unfused_dec   FZ_EXP=32896 tile decoder (x only) + separate y and z walks
Usage (GPU box): python tools/ablation.py [round] [steps]
"""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
steps = sys.argv[2] if len(sys.argv) > 2 else "10"
variants = [("base", "0"), ("range_unfused", "2097152"), ("no_pdl", "67108864"), ("dec_chunk16", "33554432"),
            ("zr_3stage", "16384"), ("zband_comp", "8192"), ("ws_comp", "9216"),
            ("plane_dec", "32768"), ("unfused_dec", "32896")]
rows = []
for name, e in variants:
    env = dict(os.environ, FZ_EXP=e)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", steps, "--warmup", "3",
                          "--no-cpu-baseline"], env=env, capture_output=True, text=True, cwd=ROOT)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    k = {n: round(v["ms_per_launch"] * 1e3, 1) for n, v in line["kernels"].items() if v["ms_per_launch"] > 0.02}
    rows.append((name, e, line["value"], line["ms_per_step"], line["compress_gbs"], line["decompress_gbs"],
                 line.get("parity_vs_oracle"), k))
    if name == "base" and "chunk_local" in line:
        c = line["chunk_local"]
        rows.append(("chunk_local (f1)", "mode flag", c["value"], c["ms_per_step"], c["compress_gbs"],
                     c["decompress_gbs"], None, {n: round(t * 1e3, 1) for n, t in c["kernels_ms"].items()}))
    print(name, line["value"], line["ms_per_step"], k, flush=True)
md = [f"# {rnd} ablations (c4 512^3 REL 1e-3, 1 B200, `python tools/ablation.py`)", "",
      "Each variant is `bench.py --steps %s --warmup 3` with the FZ_EXP bits shown (read by libfz)." % steps,
      "Kernel times are CUDA-event means per launch (us).", "",
      "| variant | FZ_EXP | step GB/s | ms/step | compress GB/s | decompress GB/s | kernels (us/launch) |",
      "|---|---|---|---|---|---|---|"]
for name, e, v, ms, c, d, par, k in rows:
    ks = ", ".join(f"{n} {t}" for n, t in sorted(k.items(), key=lambda kv: -kv[1]))
    md.append(f"| {name} | {e} | {v} | {ms} | {c} | {d} | {ks} |")
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", f"{rnd}_ablation.md"), "w") as f:
    f.write("\n".join(md) + "\n")
print("\n".join(md))
