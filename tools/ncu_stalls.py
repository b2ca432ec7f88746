"""Top stall reasons and hottest SASS lines of one ncu report.
    python tools/ncu_stalls.py gpurun_out/prof_X.ncu-rep [n]"""
import csv
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def f(r, k):
    try:
        return float(r[ix[k]] or 0)
    except (KeyError, ValueError):
        return 0.0


tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print(f"samples {tot:.0f}  instructions {sum(f(r, 'Instructions Executed') for r in data):.4g}")
for s, v in sorted(((s, sum(f(r, s) for r in data)) for s in stalls), key=lambda kv: -kv[1])[:8]:
    print(f"  {s:24s} {100 * v / tot:5.1f}%")
top = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:n]
for r in top:
    print(f"{f(r, 'Warp Stall Sampling (All Samples)'):8.0f} {r[ix['Address']][-5:]} "
          f"{r[ix['Source']][:64]:64s} ex={f(r, 'Instructions Executed'):.3g} "
          f"wf={r[ix['L1 Wavefronts Shared']]}/{r[ix['L1 Wavefronts Shared Ideal']]}")
