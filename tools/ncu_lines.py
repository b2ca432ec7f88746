"""Per-CUDA-source-line stall samples and instructions of one ncu report.
    python tools/ncu_lines.py gpurun_out/prof_X.ncu-rep [n] [units_for_per_unit]"""
import collections
import csv
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                      "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, agg, src = None, collections.defaultdict(lambda: [0.0, 0.0]), {}
for r in rows[3:]:
    if len(r) < 8:
        continue
    if r[0] and r[0].isdigit():  # a source line row (aggregate): take its name only
        cur = int(r[0])
        src[cur] = r[1]
        continue
    try:
        s, i = float(r[4] or 0), float(r[7] or 0)
    except ValueError:
        continue
    if cur is not None:
        agg[cur][0] += s
        agg[cur][1] += i
tot = sum(v[0] for v in agg.values()) or 1.0
toti = sum(v[1] for v in agg.values())
print(f"samples {tot:.0f} instructions {toti:.4g} ({toti / units:.1f} per unit)")
for line, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{line:5d} {100 * s / tot:5.1f}%  {i / units:7.1f}/unit  {src.get(line, '')[:95]}")
