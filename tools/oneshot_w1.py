"""World-1 latency of the small-message AllReduce algorithms (dev tool): with one
rank there is no peer traffic, so this isolates each algorithm's kernel chain."""
import os
import socket
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2508_03760_b200 as fc  # noqa: E402
from paper_2508_03760_b200.dist import QComm  # noqa: E402
from bench import spiky_bf16  # noqa: E402

s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
dist.init_process_group("gloo", rank=0, world_size=1)
torch.cuda.set_device(0)
cfg = fc.QuantConfig(4, group_size=128, chunk_size=128, scheme=fc.Scheme.SPIKE_RESERVING)
comm = QComm(max_elems=1 << 20, config=cfg, timeout_s=30.0, oneshot_max_elems=1 << 19)
for nb in (1 << 16, 1 << 18, 1 << 20):
    n = nb // 2
    xs = [spiky_bf16(n, k, torch.device("cuda")) for k in range(3)]
    y = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    row = {}
    for algo in ("one_shot", "fused", "two_step"):
        for i in range(5):
            comm.all_reduce(xs[i % 3], out=y, algo=algo)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000)
        a.record()
        for i in range(50):
            comm.all_reduce(xs[i % 3], out=y, algo=algo)
        b.record()
        torch.cuda.synchronize()
        row[algo] = round(a.elapsed_time(b) / 50 * 1e3, 2)
    comm.check()
    print(f"{nb >> 10} KiB world-1 us:", row, flush=True)
comm.close()
dist.destroy_process_group()
