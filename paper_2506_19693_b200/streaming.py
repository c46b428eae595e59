"""Host-resident batches through the device with copies overlapped (the
end-to-end path of bench.py's `e2e` and of any caller whose ciphertexts live in
host memory, e.g. serialised RBCT payloads).

A batch is split into chunks along dim 0.  Chunk i's host->device copy runs on
an upload stream, its compute on the compute stream (the caller's kernels go on
the then-current stream), and its device->host copy on a download stream, so
with pinned host buffers PCIe traffic in both directions overlaps the kernels
of neighbouring chunks.  Ordering is enforced with CUDA events only; the call
returns after the last download is enqueued (synchronise before reading the
host outputs).
"""

from __future__ import annotations

import torch


class Pipeline:
    def __init__(self, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.up = torch.cuda.Stream(self.device)
        self.comp = torch.cuda.Stream(self.device)
        self.down = torch.cuda.Stream(self.device)

    def run(self, fn, host_in: list, host_out: list, chunk: int) -> None:
        """fn(device_inputs: list[Tensor], lo, hi) -> list[Tensor] (device outputs
        for rows lo:hi, shaped like host_out[k][lo:hi])."""
        n = host_in[0].shape[0]
        caller = torch.cuda.current_stream(self.device)
        self.up.wait_stream(caller)
        self.comp.wait_stream(caller)
        self.down.wait_stream(caller)
        for lo in range(0, n, chunk):
            hi = min(n, lo + chunk)
            with torch.cuda.stream(self.up):
                dev_in = [h[lo:hi].to(self.device, non_blocking=True) for h in host_in]
                ready = torch.cuda.Event()
                ready.record(self.up)
            with torch.cuda.stream(self.comp):
                self.comp.wait_event(ready)
                for t in dev_in:
                    t.record_stream(self.comp)
                outs = fn(dev_in, lo, hi)
                done = torch.cuda.Event()
                done.record(self.comp)
            with torch.cuda.stream(self.down):
                self.down.wait_event(done)
                for h, o in zip(host_out, outs):
                    o.record_stream(self.down)
                    h[lo:hi].copy_(o, non_blocking=True)
        caller.wait_stream(self.down)
