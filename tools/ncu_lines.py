"""Per-CUDA-source-line warp-stall share from an ncu report (cuda,sass view).
usage: python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, src, fname = {}, {}, None
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        continue
    if hdr is None or row[0] in ("Function Name",):
        continue
    if row[0]:  # source line row (aggregated)
        key = (fname, int(row[0]))
        try:
            agg[key] = (float(row[si] or 0), float(row[ii] or 0))
        except ValueError:
            continue
        src[key] = row[1]
tot = sum(v[0] for v in agg.values()) or 1.0
toti = sum(v[1] for v in agg.values()) or 1.0
print(f"total stall samples {tot:.0f}, warp instructions {toti:.3g}")
for key, (s, i) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * s / tot:5.1f}% stall {100 * i / toti:5.1f}% inst  {key[0]}:{key[1]:<5} {src[key].strip()[:90]}")
