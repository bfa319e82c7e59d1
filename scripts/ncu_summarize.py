"""Summarise the ncu captures of scripts/ncu_profile.sh into profiles/ (tracked).

  python scripts/ncu_summarize.py --tag r01 [--layer L8B.GateUp --m 32]

Reads gpurun_out/prof_<tag>.ncu-rep (zipgemm_kernel, --set full), gpurun_out/
prof_decomp_<tag>.ncu-rep (decompress_kernel) and gpurun_out/launches_<tag>.csv (the
gpu__time_duration launch list of the bench command) and writes
  profiles/ncu_summary.json         machine-readable (bench.py reads roofline.traffic here)
  profiles/ncu_<tag>.md             human-readable summary
  profiles/launches_<tag>.csv       copy of the launch list
Runs on the dev container (ncu -i only needs the report files).
"""
import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / cycle"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {}
        for name, _ in METRICS:
            if name in hdr:
                i = hdr.index(name)
                d[name] = (vals[i], units[i])
        kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        kernels.append((kname, d))
    return kernels


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    return float(v.replace(",", "")) * scale


def to_us(v, u):
    return float(v.replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[u]


def launches(path):
    agg = collections.defaultdict(list)
    with open(path) as f:
        for r in csv.reader(f):
            if len(r) < 15 or r[0] == "ID" or r[12] != "gpu__time_duration.sum":
                continue
            agg[r[4]].append(to_us(r[14], r[13]))
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--layer", default="L8B.GateUp")
    ap.add_argument("--m", type=int, default=32)
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--decomp-layer", default="L8B.GateUp", help="layer of the captured decompress launch")
    ap.add_argument("--alg-bytes", type=float, default=None, help="algorithmic bytes per zipgemm launch")
    a = ap.parse_args()
    src = os.path.join(ROOT, "gpurun_out")
    dst = os.path.join(ROOT, "profiles")
    os.makedirs(dst, exist_ok=True)
    summ_path = os.path.join(dst, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    md = [f"# ncu summary, round {a.tag}", ""]
    md.append("Captured with `scripts/ncu_profile.sh` on one B200 (`--set full --clock-control none`, cold caches, "
              "serialised replays: absolute times are slower than the bench's; shares and counters are what count).")
    md.append("")
    for kind, rep in (("zipgemm", f"prof_{a.tag}.ncu-rep"), ("decompress", f"prof_decomp_{a.tag}.ncu-rep")):
        p = os.path.join(src, rep)
        if not os.path.exists(p):
            continue
        for kname, d in raw(p)[:1]:
            rd = to_bytes(*d["dram__bytes_read.sum"])
            wr = to_bytes(*d["dram__bytes_write.sum"])
            us = to_us(*d["gpu__time_duration.sum"])
            key = f"{a.layer}.M{a.m}.w{a.world}" if kind == "zipgemm" else a.decomp_layer
            entry = {"kernel": kname, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                     "duration_us_under_ncu": us, "report": f"gpurun_out/{rep} (round {a.tag})"}
            for name, label in METRICS:
                if name in d:
                    entry[name] = d[name][0]
            summ.setdefault(kind, {})[key] = entry
            md.append(f"## {kind}: `{kname}` ({key})")
            md.append("")
            md.append("| metric | value | unit |")
            md.append("|---|---|---|")
            for name, label in METRICS:
                if name in d:
                    md.append(f"| {label} (`{name}`) | {d[name][0]} | {d[name][1]} |")
            md.append(f"| DRAM bytes per launch (read + write) | {rd + wr:.4g} | byte |")
            if kind == "zipgemm" and a.alg_bytes:
                md.append(f"| algorithmic bytes per launch (bench) | {a.alg_bytes:.4g} | byte |")
                md.append(f"| DRAM / algorithmic | {(rd + wr) / a.alg_bytes:.3f} | |")
            md.append("")
    lp = os.path.join(src, f"launches_{a.tag}.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(dst, f"launches_{a.tag}.csv"))
        agg = launches(lp)
        tot = sum(sum(v) for v in agg.values())
        md.append(f"## launch list of `bench.py` ({os.path.basename(lp)})")
        md.append("")
        md.append("| kernel | launches | mean us | share of GPU time |")
        md.append("|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| `{k[:70]}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v) / tot:.1%} |")
        md.append("")
    json.dump(summ, open(summ_path, "w"), indent=1, sort_keys=True)
    open(os.path.join(dst, f"ncu_{a.tag}.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
