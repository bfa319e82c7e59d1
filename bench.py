#!/usr/bin/env python
"""ZipGEMM benchmark (driver contract).  One JSON line on rank 0.

Workload (BASELINE.json configs[1]): LLaMA-3.1-8B GateUp_proj, K=4096, N=28672, synthetic
sigma=0.02 Gaussian BF16 weights compressed with TCA-TBE, X ~ N(0,1) BF16, M=32 tokens.
One step = one ZipGEMM Y[M][N] = X W^T (the whole hot path: TMA stream of the compressed
tiles, decode, tcgen05 MMA, split-K fixup, BF16 epilogue).  With --gpus N the weight is
column-sharded over N ranks (N/w output features each) and the Y slices are all-gathered
over NCCL every step (strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--m M] [--layer NAME] [--impl reference]

L2 hygiene: every step reads a different copy of the compressed weight (R copies, R x bytes
> 3 x L2), so HBM, not L2, is measured.  Timing: CUDA events on the launching stream,
barrier + synchronize on both sides, max over ranks.  Clocks are sampled with NVML during
the warm-up + timed region.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import zs_inputs as G  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--m", type=int, default=32)
    ap.add_argument("--layer", default="L8B.GateUp")
    ap.add_argument("--impl", default="zipgemm", choices=["zipgemm", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the cuBLAS / per-M context timings")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--plumbing-check", action="store_true",
                    help="CPU-only check of the N-rank harness (spawn, gloo process group, max-over-ranks timing, "
                         "rank-0 line) with a numpy stand-in step; prints a line marked as not a measurement")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="N>1 output exchange: NCCL all-gather + permute, or the fused zs_gemm_peer epilogue "
                         "(stores into every rank's Y over NVLink, CUDA IPC) + zs_peer_wait")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks (NVML)
class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(device_index).uuid)
            try:
                self.h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid) if not uuid.startswith("GPU-") else uuid)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = repr(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU oracle legs
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def oracle_sample(layer, M, seconds_budget):
    """Time the CPU oracle (decode + fp64 GEMM, as it stands) on a bounded row sample: once on
    one core, then with one worker thread per host core on disjoint row blocks (the oracle is
    plain C called through ctypes, which releases the GIL, so the threads run in parallel)."""
    import concurrent.futures as cf

    import oracle as O
    K, N = G.LAYERS[layer]
    w = G.gaussian_bf16(N, K, 0.02, G.seed_of(layer))[:8192]   # same seeded weights, first rows
    x = G.activations_bf16(M, K, seed=G.seed_of(layer + ".X") + M)
    eb = O.encode(w[:64]).base_exp
    encs = {}

    def enc(r0, r1):                                            # offline, untimed
        if (r0, r1) not in encs:
            encs[(r0, r1)] = O.encode(w[r0:r1], base_exp=eb)
        return encs[(r0, r1)]

    def work(r0, r1):
        wd = O.decode_sequential(enc(r0, r1))
        O.gemm_f64(x, wd)

    def timed_single(rows):
        enc(0, rows)
        t0 = time.perf_counter()
        work(0, rows)
        return time.perf_counter() - t0

    rows = 64
    t = timed_single(rows)
    if t < seconds_budget:
        rows = int(min(4096, max(64, (seconds_budget / t) * rows)) // 64 * 64)
        t = timed_single(rows)
    single = 2.0 * M * rows * K / t / 1e12
    # all cores: `cores` threads, each on its own 64-row-aligned block, sized like the single run
    cores = host_cores()
    per = max(64, min(8192 // cores // 64 * 64, rows)) if cores > 1 else rows
    blocks = [(i * per, (i + 1) * per) for i in range(cores) if (i + 1) * per <= 8192]
    for b in blocks:
        enc(*b)
    with cf.ThreadPoolExecutor(len(blocks)) as ex:
        t0 = time.perf_counter()
        list(ex.map(lambda b: work(*b), blocks))
        tall = time.perf_counter() - t0
    allv = 2.0 * M * per * len(blocks) * K / tall / 1e12
    return {"value": allv, "unit": "TFLOP/s", "cores": len(blocks), "kind": "oracle",
            "sample": f"{layer} rows [0,{per * len(blocks)}) of N={N}, K={K}, M={M}: oracle decode_sequential + "
                      f"fp64 gemm, {len(blocks)} threads x {per} rows in {tall:.2f} s",
            "single_core": {"value": single, "cores": 1,
                            "sample": f"rows [0,{rows}) in {t:.2f} s on one thread"},
            "cpu": cpu_model()}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:  # pragma: no cover
        pass
    return None


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    layer, M = args.layer, args.m
    K, N = G.LAYERS[layer]
    w = G.gaussian_bf16(N, K, 0.02, G.seed_of(layer))[:64]
    x = G.activations_bf16(M, K, seed=G.seed_of(layer + ".X") + M)
    enc = O.encode(w)  # offline (the paper's compressor), not timed
    budget = 150.0 / max(1, args.steps + args.warmup)

    def step(r):
        wd = O.decode_sequential(enc)
        O.gemm_f64(x, wd[:r])

    t0 = time.perf_counter()
    step(64)
    t64 = time.perf_counter() - t0
    r = int(max(1, min(64, 64 * budget / max(t64, 1e-9))))
    for _ in range(args.warmup):
        step(r)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(r)
    el = time.perf_counter() - t0
    flops = 2.0 * M * r * K * args.steps
    val = flops / el / 1e12
    print(json.dumps({
        "impl": "reference", "metric": metric_name(), "value": val, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{layer} ZipGEMM M={M} (K={K}, N={N})", "layer": layer, "M": M, "K": K, "N": N},
        "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": 1, "kind": "oracle", "cpu": cpu_model(),
                         "sample": f"per step: oracle decode of one 64x{K} BlockTile row band + fp64 gemm of {r} "
                                   f"rows at M={M}"},
        "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def metric_name():
    return "ZipGEMM TFLOP/s, HBM GB/s vs cuBLAS BF16 (LLaMA-3 8B/70B layers, M=1–8192)"


# ------------------------------------------------------------------ GPU arm
def spawn_ranks(args):
    """`bench.py --gpus N` without a launcher: start N copies of this script as ranks
    0..N-1 (one process per GPU, rendezvous on 127.0.0.1) and wait for them; rank 0 prints
    the line.  Under torchrun (WORLD_SIZE set) this is skipped."""
    import socket
    import subprocess
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], env=env))
    rcs = [p.wait() for p in procs]
    sys.exit(max(rcs))


def init_ranks(args, need_gpu=True):
    """(world, rank, local, device, backend) of this process; joins the process group."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    # ZS_BENCH_ONE_GPU=1: every rank on cuda:0 over gloo -- a plumbing check of the N > 1
    # paths on a one-GPU box (the ranks time-slice one GPU; the numbers mean nothing)
    one_gpu = os.environ.get("ZS_BENCH_ONE_GPU") == "1" or not need_gpu
    if one_gpu:
        local = 0
    dev = None
    if need_gpu:
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
    backend = None
    if world > 1:
        backend = "gloo" if one_gpu else "nccl"
        if backend == "nccl":
            # communicator init is logged (to stderr, so stdout keeps its one JSON line)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    return world, rank, local, dev, backend


def reduce_max(v, world, dev):
    """max over ranks of a host float (the contract's max-over-ranks timing)."""
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], device=dev if dev is not None and dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def plumbing_check(args):
    """The N-rank harness on CPU (gloo): same spawn / process group / barrier / max-over-ranks
    / rank-0 line as the GPU arm, with a numpy stand-in for the step.  Not a measurement."""
    import torch
    import torch.distributed as dist
    world, rank, _, _, backend = init_ranks(args, need_gpu=False)
    a = np.ones((64, 64)) * (rank + 1)
    for _ in range(args.warmup):
        a @ a
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        y = torch.from_numpy((a @ a)[:1].copy())
        if world > 1:
            buf = [torch.empty_like(y) for _ in range(world)]
            dist.all_gather(buf, y)
            y = torch.cat(buf, 1)
    if world > 1:
        dist.barrier()
    ms = reduce_max((time.perf_counter() - t0) * 1e3, world, None)
    ok = y.shape[1] == 64 * world and all(float(y[0, 64 * r]) == 64.0 * (r + 1) ** 2 for r in range(world))
    if rank == 0:
        print(json.dumps({"metric": metric_name(), "value": None, "unit": "TFLOP/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                          "data": "plumbing-check (CPU numpy stand-in, not a measurement)",
                          "config": {"workload": "plumbing-check", "parallelism": f"cols{world}",
                                     "backend": backend, "gathered_ok": bool(ok)}}))
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
        return
    if args.plumbing_check:
        plumbing_check(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2603_17435_b200 as Z
    from paper_2603_17435_b200 import dist as D

    world, rank, local, dev, backend = init_ranks(args)
    one_gpu = backend == "gloo"

    def barrier():
        if world > 1:
            dist.barrier()

    peaks, peak_src = load_peaks()
    layer, M = args.layer, args.m
    K, N = G.LAYERS[layer]
    w = G.gaussian_bf16(N, K, 0.02, G.seed_of(layer))
    zh_full = Z.encode(w)
    r0, r1 = D.shard_bounds(N, world, rank)
    zh = D.shard_rows(zh_full, r0, r1) if world > 1 else zh_full
    nloc = r1 - r0
    wbytes = zh.nbytes()
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    R = max(2, math.ceil(3 * l2 / wbytes))
    wdev = [zh.to(dev) for _ in range(R)]
    x_host = G.activations_bf16(M, K, seed=G.seed_of(layer + ".X") + M)
    x = torch.from_numpy(x_host.view(np.int16)).view(torch.bfloat16).to(dev)
    y = torch.empty((M, nloc), dtype=torch.bfloat16, device=dev)
    ws = Z.workspace(M, nloc, K, dev)
    stream = torch.cuda.current_stream(dev)

    peer = None
    if world > 1 and args.exchange == "peer":
        # 3 output buffers: a rank's GEMM of step i+2 (whose signal lets the peers start
        # step i+3, i.e. overwrite buffer i % 3) is ordered after its own reads of step i
        peer = D.PeerOutputs(M, N, rank, world, dev, nbuf=3)
        pws = Z.peer_workspace(M, nloc, K, dev)
    epoch = [0]

    def exchange_step(i, xin):
        epoch[0] += 1
        b = epoch[0] % 3
        Z.gemm_peer(xin, wdev[i % R], peer.y_tables[b], peer.flag_table, rank, r0, epoch[0], ldy=N, ws=pws)
        n = Z.last_launch_count()
        Z.peer_wait(peer.flags, world, epoch[0])
        return peer.y[b], n + 1

    def step(i, out_full=None):
        if peer is not None:
            return exchange_step(i, x)[0]
        Z.gemm(x, wdev[i % R], out=y, ws=ws)
        if world > 1:
            return D.gather_columns(y, world)
        return y

    # correctness gate on this very launch configuration: sampled output columns against a
    # dense fp32 torch matmul of the uncompressed weight rows (north-star error metric C15)
    if peer is not None:
        yg, launches_per_step = exchange_step(0, x)
    else:
        yg = step(0)
        launches_per_step = Z.last_launch_count()
    torch.cuda.synchronize()
    cols = np.unique(np.linspace(0, N - 1, 97).astype(np.int64))
    wc = torch.from_numpy(w[cols].view(np.int16)).view(torch.bfloat16).to(dev).float()
    yref = x.float() @ wc.t()
    scale = x.float().abs() @ wc.abs().t()
    gate_err = float(((yg[:, torch.from_numpy(cols).to(dev)].float() - yref).abs() / scale.clamp_min(1e-30)).max())
    assert gate_err <= 1e-2, f"bench correctness gate failed: err {gate_err}"

    # CUDA graphs of S consecutive steps each (rotating through the weight copies): launch
    # overhead off the critical path, and consecutive ZipGEMMs in one graph overlap their
    # prologue with the previous kernel's tail (programmatic dependent launch, csrc/zs_gemm.cu)
    S = next(s for s in (10, 5, 4, 2, 1) if args.steps % s == 0)
    graphs = None
    if world == 1:
        try:
            graphs = []
            s = torch.cuda.Stream(dev)
            s.wait_stream(stream)
            with torch.cuda.stream(s):
                for _ in range(3):
                    step(0)
            stream.wait_stream(s)
            for r in range(R):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for j in range(S):
                        step(r + j)
                graphs.append(g)
        except Exception as e:  # pragma: no cover
            print(f"[bench] graph capture failed ({e!r}); timing eager launches", file=sys.stderr)
            graphs = None
    if graphs is None:
        S = 1

    def run_step(i):
        # i counts graph replays (S steps each) when graphs are used, else single steps
        if graphs is not None:
            graphs[i % R].replay()
        else:
            step(i)

    clocks = ClockSampler(local)
    nrep = args.steps // S
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nrep)]
    with clocks:
        for i in range(max(1, -(-args.warmup // S))):   # >= W warm-up steps
            run_step(i)
        barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(nrep):
            ev[i][0].record(stream)
            run_step(i)
            ev[i][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = t0.elapsed_time(t1)
    kern_ms = statistics.mean(a.elapsed_time(b) for a, b in ev) / S   # per launch (one ZipGEMM per step)
    ms = reduce_max(ms, world, dev)
    multi = multi_gpu_breakdown(args, Z, D, x, y, ws, wdev, R, world, rank, dev, stream, zh_full, M, K, N, ms / args.steps,
                                exchange=peer is not None) if world > 1 else None
    sec = ms / 1e3
    flops_step = 2.0 * M * N * K
    bytes_step_alg = zh_full.nbytes() + 2.0 * M * K * world + 2.0 * M * N
    value = flops_step * args.steps / sec / 1e12
    hbm_gbs = bytes_step_alg * args.steps / sec / 1e9

    # roofline of the dominant kernel (zipgemm_kernel): algorithmic bytes per launch / duration
    bytes_launch = wbytes + 2.0 * M * K + 2.0 * M * nloc
    achieved = bytes_launch / (kern_ms / 1e3) / 1e9
    peak = float(peaks["hbm_gbs"])
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            key = f"{layer}.M{M}.w{world}"
            if key in pj.get("zipgemm", {}):
                traffic = pj["zipgemm"][key].get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # e2e: host buffers through the public API (H2D of X, ZipGEMM, D2H of Y every step).
    # The D2H of Y runs on a second stream with double-buffered device Y, so it overlaps the
    # next step's ZipGEMM (events order each buffer's reuse); the timed region still contains
    # every step's copies.
    xh = torch.from_numpy(x_host.view(np.int16)).view(torch.bfloat16).pin_memory()
    yh = [torch.empty((M, N), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
    xd = [torch.empty_like(x) for _ in range(2)]
    yd = [torch.empty_like(y) for _ in range(2)]
    cstream = torch.cuda.Stream(dev)
    ev_y = [torch.cuda.Event() for _ in range(2)]        # Y[b] (gathered) written
    ev_yfree = [torch.cuda.Event() for _ in range(2)]    # D2H of Y[b] done
    for e in ev_yfree:
        e.record(stream)

    ev_y3 = [torch.cuda.Event() for _ in range(3)]        # exchange: D2H of buffer b done
    for e in ev_y3:
        e.record(stream)

    def e2e_step(i):
        bsel = i & 1
        xd[bsel].copy_(xh, non_blocking=True)             # 256 KB at M = 32: same stream
        stream.wait_event(ev_yfree[bsel])
        if peer is not None:
            # this step's signal lets the peers overwrite buffer (epoch + 1) % 3, which the
            # D2H of two steps ago reads: wait for that copy first
            stream.wait_event(ev_y3[(epoch[0] + 2) % 3])
            yy = exchange_step(i, xd[bsel])[0]
        else:
            Z.gemm(xd[bsel], wdev[i % R], out=yd[bsel], ws=ws)
            yy = D.gather_columns(yd[bsel], world) if world > 1 else yd[bsel]
        ev_y[bsel].record(stream)
        with torch.cuda.stream(cstream):
            cstream.wait_event(ev_y[bsel])
            yh[bsel].copy_(yy, non_blocking=True)
            ev_yfree[bsel].record(cstream)
            ev_y3[epoch[0] % 3].record(cstream)          # D2H of buffer epoch % 3 done

    e2e_api = "eager zs.gemm + torch copies"
    if world == 1:
        # the serving executor (runtime.GraphedZipLinear): S steps per CUDA graph, each with
        # its own pinned-host H2D of X and D2H of Y, pipelined on a compute and a copy stream
        from paper_2603_17435_b200.runtime import GraphedZipLinear
        # 20 steps per graph where the step count allows: the graph boundary (first H2D, last
        # D2H not overlapped) is paid once per graph
        SE = next(v for v in (20, 10, 5, 4, 2, 1) if args.steps % v == 0)
        runners = [GraphedZipLinear(wdev[r], M, steps=SE) for r in range(R)]   # one per rotated W copy
        for rn in runners:
            for j in range(SE):
                rn.x_host[j].copy_(xh)
        e2e_api = f"runtime.GraphedZipLinear ({SE} steps per graph, {R} rotated W copies)"

        def e2e_rep():
            e2e_rep.i += 1
            runners[e2e_rep.i % R].run()
        e2e_rep.i = 0
        nrep_e2e, per_rep = args.steps // SE, SE
    else:
        def e2e_rep():
            e2e_rep.i += 1
            e2e_step(e2e_rep.i)
        e2e_rep.i = 0
        nrep_e2e, per_rep = args.steps, 1
    for i in range(max(1, min(args.warmup, 20) // per_rep)):
        e2e_rep()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(nrep_e2e):
        e2e_rep()
    for e in ev_yfree:
        stream.wait_event(e)                              # the last D2H copies are inside
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = reduce_max(e0.elapsed_time(e1), world, dev)
    e2e_val = flops_step * args.steps / (e2e_ms / 1e3) / 1e12

    extras = {}
    if not args.no_extras and world == 1:
        extras = context_timings(Z, zh, w, layer, K, N, dev, R, l2)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(layer, M, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": metric_name(), "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{layer} ZipGEMM M={M} (K={K}, N={N})", "layer": layer, "M": M, "K": K,
                       "N": N, "weights": "N(0,0.02^2) fp32 -> bf16 RNE, TCA-TBE", "parallelism": f"cols{world}",
                       "exchange": (args.exchange if world > 1 else None),
                       "l2_hygiene": f"{R} rotated weight copies ({R * wbytes / 1e6:.0f} MB > 3x L2 {l2 / 1e6:.0f} MB)",
                       "bits_per_element": zh_full.bits_per_element(), "base_exp": zh_full.base_exp,
                       "coverage": zh_full.covered / (N * K), "graphs": graphs is not None,
                       "steps_per_graph": S, "pdl": True},
            "hbm_gbs": hbm_gbs,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})",
                         "kernel": "zipgemm_kernel", "bytes_per_launch": bytes_launch,
                         "kernel_us": kern_ms * 1e3},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": 2 * M * K,
                    "d2h_bytes_per_step": 2 * M * N, "api": e2e_api},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(),
        }
        line["config"]["gate_err"] = gate_err
        if multi:
            line["multi_gpu"] = multi
        if extras:
            line["context"] = extras
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def multi_gpu_breakdown(args, Z, D, x, y, ws, wdev, R, world, rank, dev, stream, zh_full, M, K, N, step_ms,
                        exchange):
    """Per-rank split of the N-GPU step (max over ranks of each part): the shard's ZipGEMM
    alone, the NCCL all-gather + permute alone, the whole step, and T_1 / (w T_w) with T_1 the
    unsharded ZipGEMM timed on this GPU (6.5)."""
    import torch

    def timed(fn, n):
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(n):
            fn(i)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    n = max(10, min(args.steps, 200))
    gemm_ms = timed(lambda i: Z.gemm(x, wdev[i % R], out=y, ws=ws), n)
    gather_ms = timed(lambda i: D.gather_columns(y, world), n) if not exchange else None
    out = {"gemm_us": reduce_max(gemm_ms, world, dev) * 1e3,
           "allgather_us": (reduce_max(gather_ms, world, dev) * 1e3) if gather_ms is not None else None,
           "step_us": step_ms * 1e3, "backend": "nccl" if not os.environ.get("ZS_BENCH_ONE_GPU") else "gloo"}
    try:
        out["nccl_version"] = ".".join(str(v) for v in torch.cuda.nccl.version())
    except Exception:  # pragma: no cover
        pass
    if rank == 0:
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size
        nf = max(2, math.ceil(3 * l2 / zh_full.nbytes()))
        full = [zh_full.to(dev) for _ in range(nf)]
        yf = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        wsf = Z.workspace(M, N, K, dev)
        t1 = timed(lambda i: Z.gemm(x, full[i % nf], out=yf, ws=wsf), n)
        out["t1_us"] = t1 * 1e3
        out["t1_over_w_tw"] = t1 / (world * step_ms)
        del full
    return out


def context_timings(Z, zh, w, layer, K, N, dev, R, l2):
    """cuBLAS BF16 (torch F.linear on the uncompressed W) vs ZipGEMM at M = 1, 8, 32 (context)."""
    import torch
    wd_dense = torch.from_numpy(w.view(np.int16)).view(torch.bfloat16).to(dev)
    Rd = max(2, math.ceil(3 * l2 / (w.size * 2)))
    dense = [wd_dense.clone() for _ in range(Rd)]
    comp = [zh.to(dev) for _ in range(R)]
    out = {}
    for M in (1, 8, 32):
        x = torch.randn((M, K), device=dev).to(torch.bfloat16)
        ws = Z.workspace(M, N, K, dev)
        y = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        res = {}
        for name, fn, n in (("zipgemm", lambda i: Z.gemm(x, comp[i % R], out=y, ws=ws), R),
                            ("cublas", lambda i: torch.mm(x, dense[i % Rd].t(), out=y), Rd)):
            for i in range(10):
                fn(i)
            gs = []
            s = torch.cuda.Stream(dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s):
                fn(0)
            torch.cuda.current_stream(dev).wait_stream(s)
            for i in range(n):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    fn(i)
                gs.append(g)
            iters = 300
            for i in range(20):
                gs[i % n].replay()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            for i in range(iters):
                gs[i % n].replay()
            b.record()
            torch.cuda.synchronize()
            res[name + "_us"] = a.elapsed_time(b) * 1e3 / iters
        res["speedup_vs_cublas"] = res["cublas_us"] / res["zipgemm_us"]
        res["zipgemm_tflops"] = 2 * M * N * K / (res["zipgemm_us"] * 1e-6) / 1e12
        res["zipgemm_gbs"] = (zh.nbytes() + 2 * M * K + 2 * M * N) / (res["zipgemm_us"] * 1e-6) / 1e9
        out[f"M{M}"] = res
    return out


if __name__ == "__main__":
    main()
