"""Aggregate an ncu source page (cuda,sass) per CUDA source line:
instructions executed and warp-stall samples (top N)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = None
recs = []
for r in rows:
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        d = dict(zip(hdr[2:], r[2:]))
        try:
            recs.append((int(r[0]), r[1][:90], int(d["Warp Stall Sampling (All Samples)"]),
                         int(d["Instructions Executed"]),
                         {k: int(v) for k, v in d.items() if k.startswith("stall_") and
                          "Not Issued" not in k and v.isdigit() and int(v) > 0}))
        except (ValueError, KeyError):
            pass
tot_s = sum(r[2] for r in recs) or 1
tot_i = sum(r[3] for r in recs) or 1
print(f"total samples {tot_s}, total warp-instructions {tot_i}")
print("--- by stall samples")
for ln, src, s, i, st in sorted(recs, key=lambda r: -r[2])[:top]:
    top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{ln:5d} {100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins  {src:90s} {top3}")
