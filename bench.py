"""Benchmark contract for the FlashCommunication-V2 hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N == 1 (default): BASELINE configs[1] -- codec round trip (encode -> packed
payload -> decode) of a 64 MiB bf16 tensor (33,554,432 elements), 4-bit,
group 128, spike reserving; the full bit-width sweep rides along in "sweep".
value = algbw = tensor bytes / round-trip latency (GB/s, nccl-tests style).

N > 1 (torchrun, one rank per GPU): BASELINE configs[2] -- two-step quantized
AllReduce of 8192 x 4096 bf16 per rank (4-bit SR g128) over CUDA-IPC peer
memory, with the bf16 NCCL AllReduce timed on the same box; value = aggregate
algbw over all ranks, latency = max over ranks.

--impl reference: the reference's CPU algorithm (oracle/ numpy port; the
reference is pure Python+numpy) on the same workload, bounded
sample per step, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "quantized AllReduce/All2All algbw GB/s & latency at 2/4/8 B200 vs bf16 NCCL"
N_ELEMS = 8192 * 4096  # 64 MiB of bf16


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_traffic(kernel_key: str):
    """DRAM bytes per launch from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(kernel_key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:  # first sample before timing starts
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm, N == 1: codec round trip
# ---------------------------------------------------------------------------


def flush_l2(buf):
    """Evict L2 between timed steps: write a buffer twice the size of the
    126 MB L2, then read it back so the lines left behind are clean (a
    write-only flush leaves ~126 MB of dirty lines whose write-back would be
    billed to the next timed kernel).  FC2_FLUSH_READ=0: write only."""
    buf.zero_()
    if os.environ.get("FC2_FLUSH_READ", "1") != "0":
        buf.view(-1, 4096).amax(dim=1)


def spiky_bf16(n, seed, device):
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    x = torch.randn(n, device=device, generator=g)
    spike = torch.rand(n, device=device, generator=g) < 1 / 64
    return torch.where(spike, torch.sign(x) * 50, x).to(torch.bfloat16)


def time_roundtrip(fc, x, cfg, steps, warmup, flush):
    """Per-step CUDA-event time of encode + decode (and each kernel alone)."""
    import torch

    n = x.numel()
    F = fc.footprint_bytes(cfg, n)
    pay = torch.empty(F, dtype=torch.uint8, device=x.device)
    y = torch.empty(n, dtype=torch.bfloat16, device=x.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for _ in range(warmup):
        flush_l2(flush)
        fc.encode_payload(x, cfg, n, out=pay, err=err, check=False)
        fc.decode_payload(pay, cfg, n, out=y, err=err, check=False)
    torch.cuda.synchronize()
    lib = fc._lib.lib()
    l0 = lib.fc2_launch_count()
    for i in range(steps):
        flush_l2(flush)  # evict L2 between steps (outside the timed region)
        ev[i][0].record()
        fc.encode_payload(x, cfg, n, out=pay, err=err, check=False)
        ev[i][1].record()
        fc.decode_payload(pay, cfg, n, out=y, err=err, check=False)
        ev[i][2].record()
    torch.cuda.synchronize()
    launches = lib.fc2_launch_count() - l0
    enc = [ev[i][0].elapsed_time(ev[i][1]) for i in range(steps)]
    dec = [ev[i][1].elapsed_time(ev[i][2]) for i in range(steps)]
    if int(err.item()):
        raise RuntimeError(f"device error word {int(err.item())} during bench")
    return enc, dec, F, launches, (pay, y)


def two_step_stage_times(fc, x, cfg, flush, steps, N=8):
    import torch

    from paper_2508_03760_b200.collectives import reduce_requant

    n = x.numel()
    S = n // N
    F = fc.footprint_bytes(cfg, S)
    slot = (F + 15) // 16 * 16
    land = torch.empty(N * slot, dtype=torch.uint8, device=x.device)
    for s in range(N):  # 8 different packed sources (the shards of this rank's tensor)
        fc.encode_payload(x[s * S:(s + 1) * S], cfg, S, out=land[s * slot:s * slot + F])
    gath = torch.empty(N * slot, dtype=torch.uint8, device=x.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    y = torch.empty(n, dtype=torch.bfloat16, device=x.device)
    import ctypes

    c = cfg.c_struct()
    lib = fc._lib.lib()

    def red():
        reduce_requant(cfg, [land.data_ptr() + s * slot for s in range(N)], S, [gath.data_ptr()], err)

    def gat():
        fc._lib.check(lib.fc2_gather_decode(ctypes.byref(c), N, fc._lib.ptr_array(
            [land.data_ptr() + o * slot for o in range(N)]), S, y.data_ptr(), 0, n, err.data_ptr(),
            torch.cuda.current_stream().cuda_stream))

    out = {}
    from paper_2508_03760_b200.collectives import _encode_jobs

    def enc():  # stage 1: this rank's 8 shards into 8 landing slots, one launch
        _encode_jobs(cfg, 0, [(x.data_ptr() + s * S * 2, S, S, land.data_ptr() + s * slot) for s in range(N)], err)

    for name, fn, nbytes in (("encode_8shards", enc, 2 * n + N * F), ("reduce_requant_8src", red, N * F + F),
                             ("gather_decode_8shards", gat, N * F + 2 * n)):
        for _ in range(2):
            fn()
        ts = []
        for _ in range(steps):
            flush_l2(flush)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = statistics.mean(ts)
        out[name] = {"us": round(t * 1e3, 2), "bytes": nbytes, "GBps": round(nbytes / (t * 1e-3) / 1e9, 1)}
    return out


def time_e2e(fc, x_host, cfg, steps, warmup, serial=False):
    """Host-buffer round trip through the public API: pinned bf16 chunk in ->
    packed payload bytes and decoded bf16 values back in pinned host memory.
    Default: one roundtrip_host call (fc2_roundtrip_host: the chunk is sliced
    and H2D / kernels / D2H of different slices overlap on internal streams).
    serial=True: the unpipelined sequence H2D -> encode -> D2H payload ->
    decode -> D2H values on one stream, for comparison."""
    import torch

    n = x_host.numel()
    F = fc.footprint_bytes(cfg, n)
    dev = torch.device("cuda")
    pay_h = torch.empty(F, dtype=torch.uint8).pin_memory()
    y_h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    if serial:
        xd = torch.empty(n, dtype=torch.bfloat16, device=dev)
        pay = torch.empty(F, dtype=torch.uint8, device=dev)
        yd = torch.empty(n, dtype=torch.bfloat16, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)

        def step():
            xd.copy_(x_host, non_blocking=True)
            fc.encode_payload(xd, cfg, n, out=pay, err=err, check=False)
            pay_h.copy_(pay, non_blocking=True)
            fc.decode_payload(pay, cfg, n, out=yd, err=err, check=False)
            y_h.copy_(yd, non_blocking=True)
    else:
        def step():
            fc.roundtrip_host(x_host, cfg, payload=pay_h, out=y_h, check=False)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        step()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    if not serial:  # the bytes that came back are the device path's bytes
        want = fc.encode_payload(x_host.cuda(), cfg, n).cpu()
        if not torch.equal(pay_h, want):
            raise RuntimeError("roundtrip_host payload differs from the device path")
    return ms, 2 * n, F + 2 * n


def cpu_baseline_codec(n_sample, reps, bits, g, sr):
    """The oracle (numpy port of the reference algorithm) timed on host cores."""
    import numpy as np

    from oracle import fc2_oracle as O

    if reps <= 0:
        return None, None
    x = O.bf16_snap(O.spiky(n_sample, 0)).astype(np.float32)
    t0 = time.perf_counter()
    for _ in range(reps):
        planes, meta = O.encode(x, bits, g, sr)
        O.decode(planes, meta, n_sample, bits, g, sr)
    dt = (time.perf_counter() - t0) / reps
    return 2 * n_sample / dt / 1e9, dt


def run_codec(args):
    import torch

    import paper_2508_03760_b200 as fc

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n = args.n
    sr = args.scheme == "sr"
    cfg = fc.QuantConfig(args.bits, group_size=args.group,
                         scheme=fc.Scheme.SPIKE_RESERVING if sr else fc.Scheme.RTN, chunk_size=args.group)
    x = spiky_bf16(n, 0, dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    with ClockSampler(dev.index) as clk:
        enc, dec, F, launches, _ = time_roundtrip(fc, x, cfg, args.steps, args.warmup, flush)
        # keep the timed loop running long enough for the sampler to see it
        t_end = time.time() + 1.0
        while time.time() < t_end:
            time_roundtrip(fc, x, cfg, args.steps, 0, flush)
    t_enc, t_dec = statistics.mean(enc), statistics.mean(dec)
    ms = t_enc + t_dec
    value = 2 * n / (ms * 1e-3) / 1e9
    peak, peak_kind = _peaks()
    enc_bytes, dec_bytes = 2 * n + F, F + 2 * n
    kernels = {
        "encode": {"ms": t_enc, "bytes": enc_bytes, "GBps": enc_bytes / (t_enc * 1e-3) / 1e9},
        "decode": {"ms": t_dec, "bytes": dec_bytes, "GBps": dec_bytes / (t_dec * 1e-3) / 1e9},
    }
    dom = "encode" if t_enc >= t_dec else "decode"
    # size-matched context: a plain device copy of the same 64 MiB (read + write
    # bytes / time), same L2 flush, same event timing
    yc = torch.empty_like(x)
    tc = []
    for i in range(args.steps + 3):
        flush_l2(flush)
        a, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        yc.copy_(x)
        b2.record()
        torch.cuda.synchronize()
        if i >= 3:
            tc.append(a.elapsed_time(b2))
    copy_gbps = 2 * x.numel() * 2 / (statistics.mean(tc) * 1e-3) / 1e9
    del yc
    roof = {
        "kernel": "k_encode_grp" if dom == "encode" else "k_decode_fast",
        "bound": "hbm",
        "achieved": kernels[dom]["GBps"],
        "peak": peak,
        "peak_kind": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json, burst copy)",
        "unit": "GB/s",
        "frac": kernels[dom]["GBps"] / peak,
        "traffic": _ncu_traffic(f"{dom}_b{args.bits}_{args.scheme}_g{args.group}"),
        "algorithmic_bytes_per_launch": kernels[dom]["bytes"],
        "copy_same_size_GBps": round(copy_gbps, 1),
        "frac_of_copy_same_size": round(kernels[dom]["GBps"] / copy_gbps, 4),
    }
    # bit-width sweep (configs[1]): RTN and SR for 2/3/4/5/6/8 bits
    sweep = {}
    if not args.no_sweep:
        for b in (2, 3, 4, 5, 6, 8):
            for sch in ("rtn", "sr"):
                c = fc.QuantConfig(b, group_size=args.group, chunk_size=args.group,
                                   scheme=fc.Scheme.SPIKE_RESERVING if sch == "sr" else fc.Scheme.RTN)
                e, d, Fb, _, _ = time_roundtrip(fc, x, c, max(3, args.steps // 2), 2, flush)
                te, td = statistics.mean(e), statistics.mean(d)
                sweep[f"b{b}_{sch}"] = {"roundtrip_GBps": round(2 * n / ((te + td) * 1e-3) / 1e9, 1),
                                        "encode_GBps": round((2 * n + Fb) / (te * 1e-3) / 1e9, 1),
                                        "decode_GBps": round((Fb + 2 * n) / (td * 1e-3) / 1e9, 1),
                                        "payload_bytes": Fb}
    # per-rank kernels of the N=8 two-step AllReduce (BASELINE configs[2]) timed
    # on one GPU: stage-2 reduce+requant of one 4 Mi-element shard from 8
    # packed sources, and the final gather-decode of 8 shards to bf16
    stages = two_step_stage_times(fc, x, cfg, flush, max(3, args.steps // 2))
    # message-size sweep of the codec round trip (BASELINE configs[4] sizes,
    # 64 KB .. 1 GB of bf16 per call), same cfg, L2 flushed before each step
    size_sweep = {}
    if not args.no_sweep:
        for nb in (1 << 16, 1 << 20, 1 << 24, 1 << 26, 1 << 28, 1 << 30):
            m = nb // 2
            xs = x[:m] if m <= n else spiky_bf16(m, 7, dev)
            e, d, Fm, _, _ = time_roundtrip(fc, xs, cfg, max(3, args.steps // 2), 2, flush)
            te, td = statistics.mean(e), statistics.mean(d)
            size_sweep[f"{nb >> 10}KiB" if nb < (1 << 20) else f"{nb >> 20}MiB"] = {
                "encode_us": round(te * 1e3, 2), "decode_us": round(td * 1e3, 2),
                "roundtrip_GBps": round(2 * m / ((te + td) * 1e-3) / 1e9, 1),
                "encode_hbm_GBps": round((2 * m + Fm) / (te * 1e-3) / 1e9, 1),
                "decode_hbm_GBps": round((Fm + 2 * m) / (td * 1e-3) / 1e9, 1)}
            del xs
    # end to end through host buffers
    x_host = x.cpu().pin_memory()
    e2e_ms, h2d, d2h = time_e2e(fc, x_host, cfg, max(3, args.steps), 2)
    e2e_serial_ms, _, _ = time_e2e(fc, x_host, cfg, max(3, args.steps // 2), 1, serial=True)
    cpu_val, cpu_dt = cpu_baseline_codec(n, args.cpu_reps, args.bits, args.group, sr)
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 5),
        "latency_us": round(ms * 1e3, 2),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16 in/out, fp32 math (f64 on near-ties), packed u8 planes",
        "data": "synthetic: N(0,1) with 1/64 of entries at +-50 (reference default_spiky_spec), bf16",
        "config": {"workload": "codec round trip, 64 MiB bf16 tensor (BASELINE configs[1])",
                   "n": n, "bits": args.bits, "group": args.group, "scheme": args.scheme,
                   "payload_bytes": F, "l2": "flushed before every step (256 MiB write, then read back)"},
        "kernels": kernels,
        "roofline": roof,
        "e2e": {"value": round(2 * n / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "roundtrip_host -> fc2_roundtrip_host (C ABI): pinned host chunk in, payload bytes + "
                        "decoded bf16 back in pinned host memory; 4 Mi-element slices, PCIe both ways "
                        "overlapped with the kernels",
                "serial_value": round(2 * n / (e2e_serial_ms * 1e-3) / 1e9, 2),
                "serial_path": "H2D -> encode_payload -> D2H payload -> decode_payload -> D2H values, one stream"},
        "cpu_baseline": None if cpu_val is None else {
            "value": round(cpu_val, 4), "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"full workload ({n} elements) x {args.cpu_reps}, oracle/fc2_oracle.py "
                      f"(numpy restatement of codec.py), {cpu_dt:.2f} s per round trip"},
        "sweep": sweep,
        "two_step_n8_per_rank_kernels": stages,
        "size_sweep": size_sweep,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm, N > 1: SPMD two-step AllReduce over NVLink
# ---------------------------------------------------------------------------


def run_allreduce(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2508_03760_b200 as fc
    from paper_2508_03760_b200 import dist as fcd

    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local_rank % ndev)
    torch.cuda.set_device(dev)
    # one process per GPU over NCCL; --backend gloo lets several ranks share one
    # GPU (CUDA IPC works between processes on a device) to validate the path
    backend = args.backend
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    sr = args.scheme == "sr"
    cfg = fc.QuantConfig(args.bits, group_size=args.group, chunk_size=args.group,
                         scheme=fc.Scheme.SPIKE_RESERVING if sr else fc.Scheme.RTN)
    n = args.n
    x = spiky_bf16(n, 1000 + rank, dev)
    # MoE All2All (BASELINE configs[3]): 4096 tokens x 7168, top-8 of 256
    # experts, EP = world; one copy per distinct destination rank
    hidden, tokens, topk, experts = 7168, args.moe_tokens, 8, 256
    g = torch.Generator().manual_seed(4242)
    mats = []
    for r in range(world):
        sel = torch.rand(tokens, experts, generator=g).topk(topk, dim=1).indices // (experts // world)
        hit = torch.zeros(tokens, world, dtype=torch.bool)
        hit.scatter_(1, sel, True)
        mats.append(hit.sum(0))
    tok_mat = torch.stack(mats).numpy()                    # tokens src -> dst
    a2a_mat = tok_mat * hidden                               # elements
    cap = 0
    for d in range(world):
        for s2 in range(world):
            m = int(a2a_mat[s2, d])
            if s2 != d and m:
                cap += (fc.footprint_bytes(cfg, -(-m // args.group) * args.group) + 15) // 16 * 16
    comm = fcd.QComm(dist.group.WORLD, max_elems=n, config=cfg, a2a_bytes=cap + 4096,
                     oneshot_max_elems=min(n, 1 << 19))
    y = torch.empty_like(x)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            flush_l2(flush)
            fn()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(steps):
            flush_l2(flush)
            dist.barrier()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            tot += s.elapsed_time(e)
        t = torch.tensor([tot / steps], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    lib = fc._lib.lib()
    l0 = lib.fc2_launch_count()
    with ClockSampler(local_rank) as clk:
        ms = timed(lambda: comm.all_reduce(x, out=y), args.steps, args.warmup)
    launches = lib.fc2_launch_count() - l0
    xb = x.clone()
    ms_nccl = timed(lambda: dist.all_reduce(xb), args.steps, args.warmup) if backend == "nccl" else None
    # the same NCCL AllReduce with NVLS (NVSwitch in-switch reduction) forced off, on a
    # second communicator created after the env change (hard part 6)
    ms_nccl_nonvls = None
    if backend == "nccl" and os.environ.get("NCCL_NVLS_ENABLE") != "0":
        prev = os.environ.get("NCCL_NVLS_ENABLE")
        os.environ["NCCL_NVLS_ENABLE"] = "0"
        try:
            g2 = dist.new_group(backend="nccl")
            ms_nccl_nonvls = timed(lambda: dist.all_reduce(xb, group=g2), args.steps, args.warmup)
        except Exception:
            ms_nccl_nonvls = None
        finally:
            if prev is None:
                os.environ.pop("NCCL_NVLS_ENABLE", None)
            else:
                os.environ["NCCL_NVLS_ENABLE"] = prev
    # e2e: pinned host in -> allreduce -> host out
    xh = x.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    xd = torch.empty_like(x)

    def e2e():
        xd.copy_(xh, non_blocking=True)
        comm.all_reduce(xd, out=y)
        yh.copy_(y, non_blocking=True)

    ms_e2e = timed(e2e, max(3, args.steps), 2)
    # All2All dispatch and combine: quantized (ours) vs bf16 NCCL all_to_all
    send = spiky_bf16(int(a2a_mat[rank].sum()), 7000 + rank, dev)
    ms_disp = timed(lambda: comm.all2all(send, a2a_mat, out_dtype=torch.bfloat16), args.steps, args.warmup)
    back = spiky_bf16(int(a2a_mat[:, rank].sum()), 8000 + rank, dev)
    ms_comb = timed(lambda: comm.all2all(back, a2a_mat.T.copy(), out_dtype=torch.bfloat16), args.steps, args.warmup)
    # small messages (BASELINE configs[4], latency end): two-step vs one-shot vs NCCL bf16
    small = {}
    for m in (1 << 15, 1 << 17, 1 << 19):
        if m > n:
            continue
        xs, ys = x[:m], y[:m]
        row = {"two_step_us": round(1e3 * timed(lambda: comm.all_reduce(xs, out=ys, algo="two_step"),
                                                args.steps, args.warmup), 2),
               "one_shot_us": round(1e3 * timed(lambda: comm.all_reduce(xs, out=ys, algo="one_shot"),
                                                args.steps, args.warmup), 2)}
        if backend == "nccl":
            xbs = x[:m].clone()
            row["nccl_bf16_us"] = round(1e3 * timed(lambda: dist.all_reduce(xbs), args.steps, args.warmup), 2)
        small[f"{2 * m >> 10}KiB"] = row
    ms_disp_nccl = None
    if backend == "nccl":
        recv = torch.empty(int(a2a_mat[:, rank].sum()), dtype=torch.bfloat16, device=dev)
        ins = [int(v) for v in a2a_mat[rank]]
        outs = [int(v) for v in a2a_mat[:, rank]]
        ms_disp_nccl = timed(lambda: dist.all_to_all_single(recv, send, outs, ins), args.steps, args.warmup)
    sent_bytes = 2 * int(a2a_mat[rank].sum() - a2a_mat[rank, rank])
    if rank == 0:
        algbw = 2 * n / (ms * 1e-3) / 1e9
        F = fc.footprint_bytes(cfg, comm.shard_len)
        line = {
            "metric": METRIC,
            "value": round(algbw * world, 2),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 5),
            "latency_us": round(ms * 1e3, 2),
            "per_rank_algbw_GBps": round(algbw, 2),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16 in/out, fp32 reduce, packed u8 planes",
            "data": "synthetic spiky bf16 per rank",
            "config": {"workload": "two-step quantized AllReduce, 8192x4096 bf16 per rank (BASELINE configs[2])",
                       "n": n, "bits": args.bits, "group": args.group, "scheme": args.scheme,
                       "l2": "flushed before every step (256 MiB write, then read back)", "parallelism": f"tp{world}"},
            "nccl_bf16": None if ms_nccl is None else {
                "ms": round(ms_nccl, 5), "algbw_GBps": round(2 * n / (ms_nccl * 1e-3) / 1e9, 2),
                "speedup": round(ms_nccl / ms, 3), "nvls_env": os.environ.get("NCCL_NVLS_ENABLE", "default"),
                "nvls_off_ms": None if ms_nccl_nonvls is None else round(ms_nccl_nonvls, 5),
                "speedup_vs_nvls_off": None if ms_nccl_nonvls is None else round(ms_nccl_nonvls / ms, 3)},
            "backend": backend,
            "roofline": {"bound": "nvlink", "unit": "GB/s",
                         "achieved": round(2 * (world - 1) / world * F * world / (ms * 1e-3) / 1e9 / world, 2),
                         "peak": 770.0, "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
                         "frac": round(2 * (world - 1) / world * F * world / (ms * 1e-3) / 1e9 / world / 770.0, 4),
                         "traffic": None},
            "all2all_moe": {
                "shape": f"{tokens} tok x {hidden}, top-{topk} of {experts}, EP={world}",
                "dispatch_ms": round(ms_disp, 4), "combine_ms": round(ms_comb, 4),
                "dispatch_algbw_GBps": round(sent_bytes / (ms_disp * 1e-3) / 1e9, 2),
                "nccl_bf16_dispatch_ms": None if ms_disp_nccl is None else round(ms_disp_nccl, 4),
                "speedup_vs_nccl": None if ms_disp_nccl is None else round(ms_disp_nccl / ms_disp, 3)},
            "e2e": {"value": round(2 * n * world / (ms_e2e * 1e-3) / 1e9, 2), "unit": "GB/s",
                    "ms_per_step": round(ms_e2e, 4), "h2d_bytes_per_step": 2 * n, "d2h_bytes_per_step": 2 * n},
            "small_message_allreduce": small,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------


_REF_X = None  # the reference arm's input, shared with forked pool workers


def _ref_slice(bounds):
    """One pool worker's share of the reference round trip: encode + decode
    of a group-aligned slice (groups are independent, codec.py:485)."""
    from oracle import fc2_oracle as O

    a, b, bits, g, sr = bounds
    planes, meta = O.encode(_REF_X[a:b], bits, g, sr)
    O.decode(planes, meta, b - a, bits, g, sr)
    return b - a


_REF_RANKS = None  # padded float32 payloads of the simulated ranks (forked workers)


def _ref_shard(job):
    """One shard of the reference two-step (collectives.py:278-311) in a pool
    worker: every source's QDQ of the shard summed in fp32 in rank order from
    +0, then the owner's QDQ of the sum -- the same arithmetic as
    oracle.two_step, one shard per process."""
    import numpy as np

    from oracle import fc2_oracle as O

    shard, S, bits, g, sr = job
    acc = np.zeros(S, dtype=np.float32)
    for src in range(len(_REF_RANKS)):
        acc += O.qdq_f32(_REF_RANKS[src][shard * S:(shard + 1) * S], bits, g, sr)[0]
    return O.qdq_f32(acc, bits, g, sr)[0]


def run_reference(args, rank, world):
    if rank != 0:
        return
    sr = args.scheme == "sr"
    n_sample = args.ref_sample
    times = []
    from oracle import fc2_oracle as O
    import numpy as np

    cores = 1
    if world > 1:
        # two-step AllReduce of the oracle on a bounded per-rank sample, one
        # shard per pool process (shards are independent, collectives.py:276)
        import multiprocessing as mproc

        global _REF_RANKS
        payloads = [O.bf16_snap(O.spiky(n_sample, s)).astype(np.float32) for s in O.child_seeds(0, world)]
        mult = world * args.group
        padded = -(-n_sample // mult) * mult
        _REF_RANKS = [np.pad(p, (0, padded - n_sample)) for p in payloads]
        S = padded // world
        cores = max(1, min(os.cpu_count() or 1, world))
        with mproc.get_context("fork").Pool(cores) as pool:
            for i in range(args.warmup + args.steps):
                t0 = time.perf_counter()
                shards = pool.map(_ref_shard, [(j, S, args.bits, args.group, sr) for j in range(world)])
                out = O.bf16_snap(np.concatenate(shards)[:n_sample])
                if i >= args.warmup:
                    times.append(time.perf_counter() - t0)
        want, _ = O.two_step(payloads, args.bits, args.group, sr)
        assert np.array_equal(out, want[0]), "pooled reference differs from oracle.two_step"
        dt = statistics.mean(times)
        value = 2 * n_sample * world / dt / 1e9
        what = (f"oracle two-step over {world} simulated ranks x {n_sample} elements, one shard per "
                f"process ({cores} processes)")
    else:
        # the full 64 MiB workload, split into group-aligned slices over a pool
        # of forked processes (all host cores; the reference is single-threaded
        # numpy per process, SPEC.md:312 allows a process pool)
        import multiprocessing as mproc

        global _REF_X
        n_sample = args.n
        cores = max(1, min(os.cpu_count() or 1, 64))
        _REF_X = O.bf16_snap(O.spiky(n_sample, 0)).astype(np.float32)
        step = -(-n_sample // (cores * 4) // args.group) * args.group
        parts = [(a, min(a + step, n_sample), args.bits, args.group, sr) for a in range(0, n_sample, step)]
        with mproc.get_context("fork").Pool(cores) as pool:
            for i in range(args.warmup + args.steps):
                t0 = time.perf_counter()
                done = sum(pool.map(_ref_slice, parts))
                if i >= args.warmup:
                    times.append(time.perf_counter() - t0)
        assert done == n_sample
        dt = statistics.mean(times)
        value = 2 * n_sample / dt / 1e9
        what = (f"oracle encode+decode of the full {n_sample}-element bf16 workload in {len(parts)} "
                f"group-aligned slices over a pool of {cores} processes")
    cb = {"value": round(value, 5), "unit": "GB/s", "cores": cores, "kind": "port",
          "sample": what + " (numpy restatement of the pure-Python reference; numpy elementwise is single-threaded)"}
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": cb["value"],
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64 codec math (numpy), fp32 reduce",
        "data": "synthetic spiky bf16",
        "config": {"workload": ("two-step quantized AllReduce" if world > 1 else "codec round trip"),
                   "n": n_sample, "bits": args.bits, "group": args.group, "scheme": args.scheme},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--group", type=int, default=128)
    ap.add_argument("--scheme", choices=["sr", "rtn"], default="sr")
    ap.add_argument("--elems", dest="n", type=int, default=N_ELEMS)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--cpu-reps", type=int, default=2)
    ap.add_argument("--ref-sample", type=int, default=1 << 22)
    ap.add_argument("--moe-tokens", type=int, default=4096)
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="process-group backend for N>1 (gloo: several ranks may share one GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        run_allreduce(args, rank, world, local_rank)
    else:
        run_codec(args)


if __name__ == "__main__":
    main()
