"""Per-source-line warp-stall samples of an ncu --set full report (needs -lineinfo):
top lines of a given file with their dominant stall reasons.
  python scripts/ncu_source_stalls.py gpurun_out/prof.ncu-rep bwd2.cuh [top=40] >> profiles/x.txt
"""
import csv
import subprocess
import sys

rep, wanted = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
cur = hdr = None
agg = []
for r in csv.reader(raw.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            s = float(r[4])
        except ValueError:
            s = 0.0
        st = {k[6:]: float(v) for k, v in d.items()
              if k.startswith("stall_") and "(Not" not in k and v not in ("", "0", "-")}
        agg.append((s, cur, int(r[0]), r[1].strip()[:90], st))
tot = sum(a[0] for a in agg) or 1.0
print(f"# warp-stall samples per source line ({rep}); all files: {tot:.0f} samples")
for s, f, l, src, st in sorted(agg, key=lambda a: -a[0])[:top]:
    if wanted != "*" and f != wanted and f != "ptx.cuh":
        continue
    reasons = ", ".join(f"{k} {v / s:.0%}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{100 * s / tot:5.1f}%  {f}:{l:<5d} {src:90s} [{reasons}]")
