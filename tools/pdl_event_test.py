"""Does a PDL-launched kernel respect a cross-stream event wait that sits between
it and its (early-triggering) predecessor in the stream?  (dev tool)

Stream S: decode (PDL, releases dependents at its start) ; wait(E) ; encode(X)
Stream T: spin 2 ms ; X <- second tensor ; record E
If the encode started after the decode's early trigger without honouring E, it
would read the old X and its payload would differ from encode(second tensor)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_03760_b200 as fc  # noqa: E402
from bench import spiky_bf16  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
n = 1 << 24
cfg = fc.QuantConfig(4, group_size=128, chunk_size=128, scheme=fc.Scheme.SPIKE_RESERVING)
a, b = spiky_bf16(n, 1, dev), spiky_bf16(n, 2, dev)
want = fc.encode_payload(b, cfg, n).clone()
pay0 = fc.encode_payload(a, cfg, n)
y = torch.empty(n, dtype=torch.bfloat16, device=dev)
S, T = torch.cuda.Stream(), torch.cuda.Stream()
bad = 0
for trial in range(20):
    X = a.clone()
    out = torch.empty_like(want)
    torch.cuda.synchronize()
    E = torch.cuda.Event()
    with torch.cuda.stream(T):
        torch.cuda._sleep(4_000_000)  # ~2 ms
        X.copy_(b)
        E.record(T)
    with torch.cuda.stream(S):
        fc.decode_payload(pay0, cfg, n, out=y, check=False)
        S.wait_event(E)
        fc.encode_payload(X, cfg, n, out=out, check=False)
    torch.cuda.synchronize()
    bad += int(not torch.equal(out, want))
print("mismatches", bad, "of 20")
