"""Top stalled SASS instructions of a captured kernel (ncu --page source --print-source sass)
-> markdown.  Usage: python scripts/ncu_hot.py gpurun_out/prof_TAG.ncu-rep [N] > profiles/ncu_TAG_hot.md"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kern = rows[0][1] if rows and len(rows[0]) > 1 else "?"
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]


def f(r, k):
    try:
        return float(r[idx[k]])
    except (KeyError, ValueError):
        return 0.0


tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {c: sum(f(r, c) for r in data) for c in stall_cols}
print(f"# Hot SASS of `{kern}`\n\nsource: `{rep}`; {int(tot)} warp-state samples, "
      f"{int(sum(f(r, 'Instructions Executed') for r in data))} warp instructions executed.\n")
print("## stall reasons (all samples)\n\n| reason | samples | share |\n|---|---|---|")
for c, v in sorted(agg.items(), key=lambda x: -x[1])[:12]:
    print(f"| {c[6:]} | {int(v)} | {100 * v / max(tot, 1):.1f}% |")
print(f"\n## top {top} instructions by not-issued samples\n\n| address | SASS | samples | not issued | top reason |\n|---|---|---|---|---|")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (Not-issued Samples)"))[:top]:
    best = max(stall_cols, key=lambda c: f(r, c))
    print(f"| {r[idx['Address']][-5:]} | `{r[idx['Source']].strip()[:70]}` | {int(f(r, 'Warp Stall Sampling (All Samples)'))} | "
          f"{int(f(r, 'Warp Stall Sampling (Not-issued Samples)'))} | {best[6:]} |")
