"""Event-timing floor on this GPU (dev tool): an almost empty kernel timed with CUDA
events, (a) from an idle GPU (includes host launch latency) and (b) queued behind an
L2 flush (the bench's situation: the GPU is busy when the events are recorded)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import flush_l2  # noqa: E402

x = torch.zeros(1, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(10):
    x.add_(1)
for busy in (False, True):
    for nk in (1, 2):
        ev = []
        for i in range(50):
            if busy:
                flush_l2(flush)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(nk):
                x.add_(1)
            e.record()
            ev.append((s, e))
            if not busy:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        ts = [s.elapsed_time(e) * 1e3 for s, e in ev[5:]]
        print(f"{'busy' if busy else 'idle'} {nk} kernel(s): median {statistics.median(ts):.2f} us  min {min(ts):.2f}")
