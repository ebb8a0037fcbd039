"""Probe HBM read-only / write-only / copy bandwidth with plain torch kernels
(calibration for the asymmetric codec kernels; L2 flushed between trials)."""
import json
import torch

def t(fn, reps=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]

out = {}
for mib in (64, 512):
    n = mib << 20
    x = torch.randn(n // 4, device="cuda")
    y = torch.empty_like(x)
    r = t(lambda: x.sum())
    w = t(lambda: y.fill_(1.0))
    c = t(lambda: y.copy_(x))
    out[f"{mib}MiB"] = {"read_GBps": round(n / r / 1e6, 1), "write_GBps": round(n / w / 1e6, 1),
                        "copy_GBps(rd+wr)": round(2 * n / c / 1e6, 1)}
print(json.dumps(out))
