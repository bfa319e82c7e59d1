"""Per-opcode shared-memory wavefronts and instruction mix of one ncu capture (source page)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]].replace(',', ''))
    except Exception: return 0.0
agg = {}; ops = {}; tot_wf = 0; tot_inst = 0
for r in data:
    src = r[ix['Source']].strip()
    toks = src.split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    ex = f(r, 'Instructions Executed'); wf = f(r, 'L1 Wavefronts Shared')
    tot_inst += ex; tot_wf += wf
    base = op.split('.')[0]
    ops[base] = ops.get(base, 0) + ex
    if wf > 0:
        a = agg.setdefault(op, [0, 0, 0]); a[0] += ex; a[1] += wf; a[2] += f(r, 'L1 Wavefronts Shared Ideal')
print(f"warp instructions {tot_inst:.0f}, smem wavefronts {tot_wf:.0f}")
for k, (ex, wf, ideal) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:22s} inst {ex:11.0f} wf {wf:11.0f} wf/inst {wf / max(ex, 1):5.2f} ideal {ideal / max(ex, 1):5.2f}")
print("opcode mix (top 20):")
for k, v in sorted(ops.items(), key=lambda x: -x[1])[:20]:
    print(f"  {k:10s} {v:11.0f} {100 * v / tot_inst:5.1f}%")
