"""A/B timing of the bf16 encoder (dev tool): CUDA events on the launching
stream, L2 flushed before every launch, median of R launches, for several
sizes / bit widths.  Also checks that the payload bytes equal those of the
one-tile-per-warp kernel (FC2_ENC=grp in a child process would be cleaner;
here both libraries are loaded through FC2_LIB by the caller).

    python tools/enc_ab.py [--reps 30] [--sizes 16,64,256]
"""
import argparse
import hashlib
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2508_03760_b200 as fc  # noqa: E402
from bench import flush_l2, spiky_bf16  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--sizes", default="16,64,256")
ap.add_argument("--cells", default="4sr,4rtn,3sr,2sr,8sr")
ap.add_argument("--tag", default=os.environ.get("FC2_ENC", "default"))
a = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
for mib in [int(v) for v in a.sizes.split(",")]:
    n = mib * (1 << 20) // 2
    x = spiky_bf16(n, 0, dev)
    for cell in a.cells.split(","):
        bits, sch = int(cell[0]), cell[1:]
        cfg = fc.QuantConfig(bits, group_size=128, chunk_size=128,
                             scheme=fc.Scheme.SPIKE_RESERVING if sch == "sr" else fc.Scheme.RTN)
        F = fc.footprint_bytes(cfg, n)
        pay = torch.empty(F, dtype=torch.uint8, device=dev)
        ts = []
        for i in range(a.reps + 3):
            flush_l2(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fc.encode_payload(x, cfg, n, out=pay, err=err, check=False)
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
        med = statistics.median(ts)
        h = hashlib.sha256(pay.cpu().numpy().tobytes()).hexdigest()[:12]
        print(f"{a.tag} {mib}MiB b{bits}{sch}: median {med:.2f} us  min {min(ts):.2f}  "
              f"{(2 * n + F) / med / 1e3:.0f} GB/s  sha {h}", flush=True)
print("err", int(err.item()))
