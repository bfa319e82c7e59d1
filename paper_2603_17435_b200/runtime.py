"""Serving executor for ZipGEMM: host batches in, host results out, one CUDA graph per S steps.

`GraphedZipLinear(w, M, S)` owns S pinned host input slots X[j] [M][K] and S pinned host output
slots Y[j] [M][N].  `run()` replays one CUDA graph that, for j = 0..S-1, copies X[j] to the
device, runs zs_gemm (the fused ZipGEMM kernel, or the decoupled path at large M) and copies
the result back to Y[j].  Three streams inside the graph: all S host-to-device copies are
queued first on an H2D stream (each step has its own device buffer, so nothing waits for
reuse), the ZipGEMMs run back to back on the compute stream (each waits only for its own
input; consecutive launches keep their programmatic-dependent-launch overlap), and each
step's device-to-host copy runs on a D2H stream as soon as its GEMM is done, overlapping the
next GEMMs.  The H2D copies are issued before any D2H so the copy engine never queues an
input behind an output.  Every step's H2D and D2H run inside run().

The compute is libzs.so's (zs_gemm through the ctypes binding); torch provides pinned memory,
device buffers, streams, events and the graph capture -- no compute of its own.
"""
from __future__ import annotations

from .zs import ZsDevice, gemm, last_launch_count, lib


class GraphedZipLinear:
    def __init__(self, w: ZsDevice, M: int, steps: int = 10):
        import torch
        dev = w.device
        self.w, self.M, self.S = w, M, steps
        K, N = w.cols, w.rows
        bf16 = torch.bfloat16
        self.x_host = torch.zeros((steps, M, K), dtype=bf16).pin_memory()
        self.y_host = torch.zeros((steps, M, N), dtype=bf16).pin_memory()
        self._xd = [torch.zeros((M, K), dtype=bf16, device=dev) for _ in range(steps)]
        self._yd = [torch.zeros((M, N), dtype=bf16, device=dev) for _ in range(steps)]
        # a private, zero-initialised workspace: the graph captures its address, and another
        # executor's graph (or an eager zs.gemm) may run concurrently on another stream
        self._ws = torch.zeros(max(int(lib().zs_gemm_workspace_bytes(M, N, K)), 16), dtype=torch.uint8, device=dev)
        main, h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_x = [torch.cuda.Event() for _ in range(steps)]
        ev_y = [torch.cuda.Event() for _ in range(steps)]
        ev_start = torch.cuda.Event()

        def body():
            ev_start.record(main)
            h2d.wait_event(ev_start)                        # fork the copy streams off main
            d2h.wait_event(ev_start)
            with torch.cuda.stream(h2d):
                for j in range(steps):
                    self._xd[j].copy_(self.x_host[j], non_blocking=True)
                    ev_x[j].record(h2d)
            for j in range(steps):
                main.wait_event(ev_x[j])
                gemm(self._xd[j], w, out=self._yd[j], ws=self._ws, stream=main)
                ev_y[j].record(main)
                d2h.wait_event(ev_y[j])
                with torch.cuda.stream(d2h):
                    self.y_host[j].copy_(self._yd[j], non_blocking=True)
            ev_end = torch.cuda.Event()
            ev_end.record(d2h)
            main.wait_event(ev_end)                         # join
            main.wait_stream(h2d)

        cur = torch.cuda.current_stream(dev)
        main.wait_stream(cur)
        with torch.cuda.stream(main):                       # warm-up (cuBLAS handle, tensor map)
            body()
        self.launches_per_step = last_launch_count()
        cur.wait_stream(main)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=main):
            body()
        torch.cuda.synchronize(dev)

    @property
    def h2d_bytes_per_step(self) -> int:
        return self.x_host[0].numel() * 2

    @property
    def d2h_bytes_per_step(self) -> int:
        return self.y_host[0].numel() * 2

    def run(self):
        """Replay the S steps (asynchronous on the current stream; synchronize before reading
        y_host)."""
        self.graph.replay()
