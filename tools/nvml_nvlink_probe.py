"""Calibrates bench.py's NVML NVLink counters (NvlCounters): copies 1 GiB
GPU0 -> GPU1 with cudaMemcpyPeer (torch) and prints every rank's counter deltas,
so the field units / directions are checked against a known transfer."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

G = torch.cuda.device_count()
cs = [bench.NvlCounters(i) for i in range(G)]
x = torch.empty(1 << 28, dtype=torch.float32, device="cuda:0")      # 1 GiB
x.fill_(1.0)
torch.cuda.synchronize()
r0 = [c.read() for c in cs]
t = time.time()
for _ in range(4):
    y = x.to("cuda:1")
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
dt = time.time() - t
r1 = [c.read() for c in cs]
import pynvml as N
diag = {}
for i, c in enumerate(cs):
    if c.h is None:
        diag[i] = c.err
        continue
    vals = N.nvmlDeviceGetFieldValues(c.h, [138, 139, 140, 141] + [(202, l) for l in range(18)] +
                                      [(204, l) for l in range(18)])
    diag[i] = [(v.fieldId, v.scopeId, v.nvmlReturn, int(v.value.ullVal)) for v in vals]
print(json.dumps({"bytes_copied": 4 * (1 << 30), "seconds": dt, "schemes": [c.scheme for c in cs],
                  "errors": [c.err for c in cs],
                  "deltas": [bench.NvlCounters.delta(a, b) for a, b in zip(r0, r1)], "raw_after": diag}, indent=1))
