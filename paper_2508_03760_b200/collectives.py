"""Drop-in quantized collectives (reference: collectives.py) on one B200.

The reference simulates N ranks in one process.  These functions keep its
signatures -- a list of N per-rank payloads plus a topology -- and run every
rank's work on the current CUDA device with the same kernels the SPMD
multi-GPU path (``paper_2508_03760_b200.dist``) uses over NVLink:

* stage 1: one batched encode launch quantizes every (src, shard) block
  straight into the per-shard landing slots (what ``dist`` stores into peer
  memory);
* stage 2: one fused decode + fp32 rank-order reduce + re-encode launch per
  shard (``k_reduce_fast``), writing the packed reduced shard to the gather
  slot(s);
* stage 3: one decode launch writes the bf16 output, padding stripped.

Traffic bookkeeping (ledger, trace) is analytic host data with exactly the
reference's event order.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .config import QuantConfig, footprint_bytes
from .errors import ConfigError, DataError, NotApplicableError
from .topology import Topology, cross_numa_partition

RAW_BYTES_PER_ELEMENT = 2  # bf16 wire baseline (collectives.py:26)
_SLOT_ALIGN = 16


# ---------------------------------------------------------------------------
# result / trace types (collectives.py:29-144)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class TransferEvent:
    stage: str
    wave: int
    src: int
    dst: int
    elements: int
    actual_bytes: int

    @property
    def raw_bytes(self) -> int:
        return self.elements * RAW_BYTES_PER_ELEMENT


@dataclass(frozen=True)
class ComputeEvent:
    stage: str
    wave: int
    device: int
    kind: str  # "quantize" | "dequantize" | "reduce"
    elements: int


@dataclass
class Stage:
    name: str
    transfers: list = field(default_factory=list)
    computes: list = field(default_factory=list)


@dataclass
class StageTrace:
    stages: list = field(default_factory=list)

    def stage(self, name: str) -> Stage:
        st = Stage(name)
        self.stages.append(st)
        return st


@dataclass
class RankState:
    rank: int
    payload: object


class TrafficLedger:
    """Per-link, per-direction raw (2 B/elem) and actual byte counters + event log."""

    def __init__(self, topo: Topology):
        self.topo = topo
        self.events: list[TransferEvent] = []
        self.raw_by_linkdir: dict = {}
        self.actual_by_linkdir: dict = {}

    def record(self, ev: TransferEvent) -> None:
        self.events.append(ev)
        for link, direction in self.topo.route(ev.src, ev.dst):
            k = (link.name, direction)
            self.raw_by_linkdir[k] = self.raw_by_linkdir.get(k, 0) + ev.raw_bytes
            self.actual_by_linkdir[k] = self.actual_by_linkdir.get(k, 0) + ev.actual_bytes

    @property
    def total_raw(self) -> int:
        return sum(e.raw_bytes for e in self.events)

    @property
    def total_actual(self) -> int:
        return sum(e.actual_bytes for e in self.events)

    def bridge_per_direction(self) -> dict:
        br = self.topo.bridge()
        if br is None:
            return {}
        return {d: {"raw": self.raw_by_linkdir.get((br.name, d), 0),
                    "actual": self.actual_by_linkdir.get((br.name, d), 0)} for d in ("ab", "ba")}


@dataclass
class CollectiveResult:
    outputs: list
    ledger: TrafficLedger
    trace: StageTrace


def volume_report(ledger: TrafficLedger, topo: Topology | None = None) -> dict:
    """Raw/actual totals, cross-NUMA max, per-link breakdown (collectives.py:126-144)."""
    per_dir = ledger.bridge_per_direction()
    return {
        "total_raw": ledger.total_raw,
        "total_actual": ledger.total_actual,
        "cross_numa_raw": max((d["raw"] for d in per_dir.values()), default=0),
        "cross_numa_actual": max((d["actual"] for d in per_dir.values()), default=0),
        "per_link": {f"{n}:{d}": {"raw": ledger.raw_by_linkdir[(n, d)],
                                  "actual": ledger.actual_by_linkdir[(n, d)]}
                     for (n, d) in sorted(ledger.raw_by_linkdir)},
    }


# ---------------------------------------------------------------------------
# staging helpers
# ---------------------------------------------------------------------------


def _round_up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


def _stage_payloads(payloads, n_ranks: int, equal_sizes: bool = True):
    """Validate + move payloads to the device as float32 (or bf16, which is
    exact in float32): the reference's ``_check_payloads`` cast
    (collectives.py:152-164).  Non-finite values surface as DataError from
    the encoder's device flag."""
    if len(payloads) != n_ranks:
        raise ConfigError(f"expected {n_ranks} payloads, got {len(payloads)}")
    dev = _device.require_cuda()
    device_in = all(_device.is_cuda_tensor(p) for p in payloads) and n_ranks > 0
    ts = []
    for p in payloads:
        if isinstance(p, torch.Tensor):
            t = p.detach().reshape(-1)
            if not t.is_cuda:
                t = t.to(dev)
        else:
            a = np.asarray(p).reshape(-1)
            if a.dtype != np.float32:
                a = np.asarray(p, dtype=np.float64).reshape(-1)
            t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        ts.append(t)
    if equal_sizes and len({t.numel() for t in ts}) > 1:
        raise DataError(f"payload lengths differ: {sorted({t.numel() for t in ts})}")
    if ts and all(t.dtype == torch.bfloat16 for t in ts):
        ts = [t.contiguous() for t in ts]
    else:
        ts = [t.to(torch.float32).contiguous() for t in ts]  # RNE cast, == numpy astype
    return ts, device_in, dev


def _encode_jobs(cfg: QuantConfig, dtype_code: int, jobs, err: torch.Tensor) -> None:
    """jobs: (x_ptr, n_valid, n, out_ptr); issued in launches of <= FC2_MAX_JOBS."""
    c = cfg.c_struct()
    lib = _lib.lib()
    for i in range(0, len(jobs), 256):
        part = jobs[i:i + 256]
        _lib.check(lib.fc2_encode_batch(
            ctypes.byref(c), dtype_code, len(part), _lib.ptr_array([j[0] for j in part]),
            _lib.i64_array([j[1] for j in part]), _lib.i64_array([j[2] for j in part]),
            _lib.ptr_array([j[3] for j in part]), err.data_ptr(), _device.stream_handle()))


def _decode_jobs(cfg: QuantConfig, y_code: int, jobs, err: torch.Tensor) -> None:
    """jobs: (payload_ptr, n, y_ptr, n_out)."""
    c = cfg.c_struct()
    lib = _lib.lib()
    for i in range(0, len(jobs), 256):
        part = jobs[i:i + 256]
        _lib.check(lib.fc2_decode_batch(
            ctypes.byref(c), y_code, len(part), _lib.ptr_array([j[0] for j in part]),
            _lib.i64_array([j[1] for j in part]), _lib.ptr_array([j[2] for j in part]),
            _lib.i64_array([j[3] for j in part]), err.data_ptr(), _device.stream_handle()))


def reduce_requant(cfg: QuantConfig, src_ptrs, n: int, dst_ptrs, err: torch.Tensor) -> None:
    c = cfg.c_struct()
    _lib.check(_lib.lib().fc2_reduce_requant(
        ctypes.byref(c), len(src_ptrs), _lib.ptr_array(src_ptrs), n, len(dst_ptrs),
        _lib.ptr_array(dst_ptrs), err.data_ptr(), _device.stream_handle()))


# ---------------------------------------------------------------------------
# two-step AllReduce (collectives.py:263-315)
# ---------------------------------------------------------------------------


class TwoStepPlan:
    """Reusable device workspace for the simulated N-rank two-step AllReduce."""

    def __init__(self, cfg: QuantConfig, n_ranks: int, n: int, device):
        self.cfg, self.N, self.n = cfg, n_ranks, n
        mult = n_ranks * cfg.group_size
        self.padded = _round_up(n, mult) if n else 0
        self.S = self.padded // n_ranks if n_ranks else 0
        self.F = footprint_bytes(cfg, self.S)
        self.slot = _round_up(max(self.F, 1), _SLOT_ALIGN)
        self.land = torch.empty(n_ranks * n_ranks * self.slot, dtype=torch.uint8, device=device)
        self.gath = torch.empty(n_ranks * self.slot, dtype=torch.uint8, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)

    def land_ptr(self, shard: int, src: int) -> int:
        return self.land.data_ptr() + (shard * self.N + src) * self.slot

    def gath_ptr(self, shard: int) -> int:
        return self.gath.data_ptr() + shard * self.slot

    def run(self, xs: list[torch.Tensor], y: torch.Tensor) -> None:
        """xs: N device vectors (bf16 or f32) of n elements; y: bf16/f32 output of n."""
        N, S, n, cfg = self.N, self.S, self.n, self.cfg
        if cfg.int_log:
            _device.ensure_intlog(cfg.theta, y.device)
        esz = xs[0].element_size()
        jobs = []
        for src in range(N):
            base = xs[src].data_ptr()
            for shard in range(N):
                nv = max(0, min(S, n - shard * S))
                ptr = base + shard * S * esz if nv else base
                jobs.append((ptr, nv, S, self.land_ptr(shard, src)))
        _encode_jobs(cfg, _device.dtype_code(xs[0]), jobs, self.err)
        for shard in range(N):
            reduce_requant(cfg, [self.land_ptr(shard, s) for s in range(N)], S,
                           [self.gath_ptr(shard)], self.err)
        c = cfg.c_struct()
        _lib.check(_lib.lib().fc2_gather_decode(
            ctypes.byref(c), N, _lib.ptr_array([self.gath_ptr(j) for j in range(N)]), S,
            y.data_ptr(), _device.dtype_code(y), n, self.err.data_ptr(), _device.stream_handle()))


def _two_step_ledger(topo: Topology, N: int, S: int, F: int):
    trace, ledger = StageTrace(), TrafficLedger(topo)
    st = trace.stage("scatter")
    for src in range(N):
        for shard in range(N):
            st.computes.append(ComputeEvent(st.name, 0, src, "quantize", S))
            if src != shard:
                ev = TransferEvent(st.name, 1, src, shard, S, F)
                st.transfers.append(ev)
                ledger.record(ev)
            st.computes.append(ComputeEvent(st.name, 2, shard, "dequantize", S))
    for shard in range(N):
        st.computes.append(ComputeEvent(st.name, 3, shard, "reduce", N * S))
    st = trace.stage("gather")
    for owner in range(N):
        st.computes.append(ComputeEvent(st.name, 0, owner, "quantize", S))
        for dst in range(N):
            if dst == owner:
                continue
            ev = TransferEvent(st.name, 1, owner, dst, S, F)
            st.transfers.append(ev)
            ledger.record(ev)
            st.computes.append(ComputeEvent(st.name, 2, dst, "dequantize", S))
    return ledger, trace


def two_step_allreduce_q(payloads, topo: Topology, config: QuantConfig) -> CollectiveResult:
    """Quantized AllReduce = quantized scatter-reduce + quantized all-gather.

    Same contract as collectives.py:263-315 (rule R14 of SURVEY 8.0): every
    rank quantizes every shard (its own included), shards are reduced in fp32
    in rank order, the owner requantizes, everyone decodes, outputs are
    bf16-rounded with padding stripped, and all outputs are bit-identical.
    Host payloads give float32 numpy outputs; CUDA payloads give CUDA tensors.
    """
    N = topo.n_devices
    xs, device_in, dev = _stage_payloads(payloads, N)
    n = xs[0].numel() if xs else 0
    plan = TwoStepPlan(config, N, n, dev)
    y = torch.empty(n, dtype=torch.bfloat16, device=dev)
    if n:
        plan.run(xs, y)
    _device.check_err(plan.err)
    ledger, trace = _two_step_ledger(topo, N, plan.S, plan.F)
    out = y.to(torch.float32)
    if device_in:
        outputs = [out] + [out.clone() for _ in range(N - 1)]
    else:
        host = out.cpu().numpy()
        outputs = [host.copy() for _ in range(N)]
    return CollectiveResult(outputs, ledger, trace)


def hierarchical_two_step_q(payloads, topo: Topology, config: QuantConfig) -> CollectiveResult:
    """Quantized AllReduce over two NUMA islands joined by a bridge
    (collectives.py:318-425): scatter-reduce inside each island, a half-segment
    swap between paired ranks across the bridge, all-gather inside each island.

    Every quantize-dequantize runs on the GPU codec (batched encode + decode
    launches per stage, the encode of stage s+1 fed by the fp32 sums of stage
    s); the fp32 sums keep the reference's order (member order from +0.0, then
    ``mine + peer``).  Raises NotApplicableError without a bridge -- a B200
    NVSwitch box has none, where ``two_step_allreduce_q`` is the algorithm.
    """
    groups, _bridge = cross_numa_partition(topo)
    if len(groups) != 2 or len(groups[0]) != len(groups[1]):
        raise ConfigError("hierarchical all-reduce needs two equal NUMA groups")
    N = topo.n_devices
    gsz = len(groups[0])
    xs, device_in, dev = _stage_payloads(payloads, N)
    n = xs[0].numel()
    padded = _round_up(n, N * config.group_size)
    seg = padded // gsz
    half = seg // 2
    f_seg, f_half = footprint_bytes(config, seg), footprint_bytes(config, half)
    xp = []
    for x in xs:  # zero padding (collectives.py:167-172), float32 like _check_payloads
        t = torch.zeros(padded, dtype=torch.float32, device=dev)
        t[:n] = x
        xp.append(t)

    def qdq(blocks):
        return _quantized_blocks(config, [(0, 0, b) for b in blocks], dev)[0] if blocks else []

    trace, ledger = StageTrace(), TrafficLedger(topo)

    # ---- stage rs: scatter-reduce inside each island
    st = trace.stage("rs")
    reduced = {}
    for members in groups:
        dq = qdq([xp[src][li * seg:(li + 1) * seg] for src in members for li in range(gsz)])
        for a, src in enumerate(members):
            for li, owner in enumerate(members):
                st.computes.append(ComputeEvent(st.name, 0, src, "quantize", seg))
                if src != owner:
                    ev = TransferEvent(st.name, 1, src, owner, seg, f_seg)
                    st.transfers.append(ev)
                    ledger.record(ev)
                st.computes.append(ComputeEvent(st.name, 2, owner, "dequantize", seg))
        for li, owner in enumerate(members):
            acc = torch.zeros(seg, dtype=torch.float32, device=dev)
            for a in range(gsz):
                acc += dq[a * gsz + li]
            reduced[owner] = acc
            st.computes.append(ComputeEvent(st.name, 3, owner, "reduce", gsz * seg))

    # ---- stage xn: paired ranks swap opposite halves across the bridge
    st = trace.stage("xn")
    pairs = list(zip(groups[0], groups[1]))
    first = qdq([b for i, j in pairs for b in (reduced[i][half:], reduced[j][:half])])
    totals = []
    for k, (i, j) in enumerate(pairs):
        dq_high_i, dq_low_j = first[2 * k], first[2 * k + 1]
        totals += [reduced[i][:half] + dq_low_j, reduced[j][half:] + dq_high_i]
    second = qdq(totals)
    final = {}
    for k, (i, j) in enumerate(pairs):
        st.computes.append(ComputeEvent(st.name, 0, i, "quantize", half))
        for ev in (TransferEvent(st.name, 1, i, j, half, f_half),):
            st.transfers.append(ev)
            ledger.record(ev)
        st.computes.append(ComputeEvent(st.name, 0, j, "quantize", half))
        ev = TransferEvent(st.name, 1, j, i, half, f_half)
        st.transfers.append(ev)
        ledger.record(ev)
        st.computes += [ComputeEvent(st.name, 2, i, "dequantize", half), ComputeEvent(st.name, 2, j, "dequantize", half),
                        ComputeEvent(st.name, 3, i, "reduce", 2 * half), ComputeEvent(st.name, 3, j, "reduce", 2 * half),
                        ComputeEvent(st.name, 4, i, "quantize", half)]
        ev = TransferEvent(st.name, 5, i, j, half, f_half)
        st.transfers.append(ev)
        ledger.record(ev)
        st.computes.append(ComputeEvent(st.name, 4, j, "quantize", half))
        ev = TransferEvent(st.name, 5, j, i, half, f_half)
        st.transfers.append(ev)
        ledger.record(ev)
        st.computes += [ComputeEvent(st.name, 6, i, "dequantize", half), ComputeEvent(st.name, 6, j, "dequantize", half)]
        final[i] = final[j] = torch.cat([second[2 * k], second[2 * k + 1]])

    # ---- stage ag: all-gather inside each island
    st = trace.stage("ag")
    outs = {}
    for members in groups:
        dq = qdq([final[o] for o in members])
        merged = torch.cat(dq)
        for li, owner in enumerate(members):
            st.computes.append(ComputeEvent(st.name, 0, owner, "quantize", seg))
            for dst in members:
                if dst != owner:
                    ev = TransferEvent(st.name, 1, owner, dst, seg, f_seg)
                    st.transfers.append(ev)
                    ledger.record(ev)
                st.computes.append(ComputeEvent(st.name, 2, dst, "dequantize", seg))
        y = torch.empty(n, dtype=torch.bfloat16, device=dev)
        if n:
            _lib.check(_lib.lib().fc2_f32_to_bf16_bits(merged.data_ptr(), n, y.data_ptr(), _device.stream_handle()))
        out = y.to(torch.float32)
        for dst in members:
            outs[dst] = out
    outputs = [outs[r].clone() if device_in else outs[r].cpu().numpy() for r in range(N)]
    return CollectiveResult(outputs, ledger, trace)


# ---------------------------------------------------------------------------
# All2All dispatch / combine (collectives.py:428-482)
# ---------------------------------------------------------------------------


def _dispatch_matrix(ranks, N, dispatch_matrix):
    if dispatch_matrix is None:
        per = ranks[0].numel() // N if N else 0
        if per * N != (ranks[0].numel() if N else 0):
            raise ConfigError(f"payload size {ranks[0].numel()} not divisible by {N} ranks")
        return np.full((N, N), per, dtype=np.int64)
    m = np.asarray(dispatch_matrix, dtype=np.int64)
    if m.shape != (N, N):
        raise ConfigError(f"dispatch matrix must be {N}x{N}, got {m.shape}")
    if np.any(m < 0):
        raise ConfigError("dispatch matrix entries must be non-negative")
    for i in range(N):
        if int(m[i].sum()) != ranks[i].numel():
            raise ConfigError(f"rank {i}: dispatch row sums to {int(m[i].sum())}, "
                              f"payload has {ranks[i].numel()} elements")
    return m


def _quantized_blocks(config: QuantConfig, blocks, dev):
    """blocks: list of (src, dst, tensor_view) of remote blocks.  Returns the
    decoded float32 tensors (QDQ of each zero-padded block) and per-block
    payload bytes."""
    gs = config.group_size
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    if config.int_log:
        _device.ensure_intlog(config.theta, dev)
    metas = []
    total = 0
    for (_, _, t) in blocks:
        plen = _round_up(t.numel(), gs)
        F = footprint_bytes(config, plen)
        metas.append((plen, F, total))
        total += _round_up(max(F, 1), _SLOT_ALIGN)
    pay = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
    outs = [torch.empty(t.numel(), dtype=torch.float32, device=dev) for (_, _, t) in blocks]
    by_dtype: dict[int, list] = {}
    for (_, _, t), (plen, F, off) in zip(blocks, metas):
        by_dtype.setdefault(_device.dtype_code(t), []).append((t.data_ptr(), t.numel(), plen, pay.data_ptr() + off))
    for code, jobs in by_dtype.items():
        _encode_jobs(config, code, jobs, err)
    _decode_jobs(config, _lib.F32,
                 [(pay.data_ptr() + off, plen, o.data_ptr(), o.numel())
                  for (plen, F, off), o in zip(metas, outs)], err)
    _device.check_err(err)
    return outs, [F for (_, F, _) in metas]


def _exact_block(v: torch.Tensor, err: torch.Tensor) -> torch.Tensor:
    """A block that never crosses a wire (diagonal, collectives.py:466-468):
    exact float32 copy; non-finite values set the DataError bit
    (collectives.py:152-164 checks every payload before dispatch)."""
    out = torch.empty(v.numel(), dtype=torch.float32, device=v.device)
    if v.numel():
        _lib.check(_lib.lib().fc2_copy_check(v.data_ptr(), _device.dtype_code(v), out.data_ptr(), _lib.F32,
                                              v.numel(), err.data_ptr(), _device.stream_handle()))
    return out


def all2all_dispatch_q(payloads, topo: Topology, config: QuantConfig, dispatch_matrix=None) -> CollectiveResult:
    """Quantized All2All dispatch (collectives.py:428-482, rule R15).

    ``outputs[dst][src]``: exact float32 copy on the diagonal, empty for empty
    blocks, else the block zero-padded to a group multiple, quantized as one
    chunk, dequantized to float32 and sliced back."""
    N = topo.n_devices
    ranks, device_in, dev = _stage_payloads(payloads, N, equal_sizes=dispatch_matrix is None)
    matrix = _dispatch_matrix(ranks, N, dispatch_matrix)
    views = {}
    for src in range(N):
        edges = np.concatenate([[0], np.cumsum(matrix[src])])
        for dst in range(N):
            views[(src, dst)] = ranks[src][int(edges[dst]):int(edges[dst + 1])]
    remote = [(s, d, views[(s, d)]) for s in range(N) for d in range(N)
              if s != d and views[(s, d)].numel() > 0]
    decoded, nbytes = _quantized_blocks(config, remote, dev) if remote else ([], [])
    got = {(s, d): (o, f) for (s, d, _), o, f in zip(remote, decoded, nbytes)}

    trace, ledger = StageTrace(), TrafficLedger(topo)
    st = trace.stage("dispatch")
    out = [[None] * N for _ in range(N)]
    err = _device.new_err(dev)
    for src in range(N):
        for dst in range(N):
            v = views[(src, dst)]
            if src == dst or v.numel() == 0:
                out[dst][src] = _exact_block(v, err)
                continue
            o, f = got[(src, dst)]
            st.computes.append(ComputeEvent(st.name, 0, src, "quantize", v.numel()))
            ev = TransferEvent(st.name, 1, src, dst, int(v.numel()), f)
            st.transfers.append(ev)
            ledger.record(ev)
            st.computes.append(ComputeEvent(st.name, 2, dst, "dequantize", v.numel()))
            out[dst][src] = o
    _device.check_err(err)
    if not device_in:
        out = [[t.cpu().numpy() for t in row] for row in out]
    return CollectiveResult(out, ledger, trace)


def all2all_combine_q(blocks, topo: Topology, config: QuantConfig) -> CollectiveResult:
    """Quantized All2All combine -- the reverse of dispatch (north-star
    addition; the reference ships dispatch only).

    ``blocks[src][dst]`` is what expert-rank ``src`` returns to token-owner
    ``dst``; it travels with the same codec as dispatch.  Returns
    ``outputs[dst][src]`` with the dispatch conventions."""
    N = topo.n_devices
    if len(blocks) != N or any(len(r) != N for r in blocks):
        raise ConfigError(f"combine needs an {N}x{N} list of blocks")
    flat, device_in, dev = _stage_payloads([b for row in blocks for b in row], N * N, equal_sizes=False)
    views = {(s, d): flat[s * N + d] for s in range(N) for d in range(N)}
    remote = [(s, d, views[(s, d)]) for s in range(N) for d in range(N)
              if s != d and views[(s, d)].numel() > 0]
    decoded, nbytes = _quantized_blocks(config, remote, dev) if remote else ([], [])
    got = {(s, d): (o, f) for (s, d, _), o, f in zip(remote, decoded, nbytes)}
    trace, ledger = StageTrace(), TrafficLedger(topo)
    st = trace.stage("combine")
    out = [[None] * N for _ in range(N)]
    err = _device.new_err(dev)
    for src in range(N):
        for dst in range(N):
            v = views[(src, dst)]
            if src == dst or v.numel() == 0:
                out[dst][src] = _exact_block(v, err)
                continue
            o, f = got[(src, dst)]
            st.computes.append(ComputeEvent(st.name, 0, src, "quantize", v.numel()))
            ev = TransferEvent(st.name, 1, src, dst, int(v.numel()), f)
            st.transfers.append(ev)
            ledger.record(ev)
            st.computes.append(ComputeEvent(st.name, 2, dst, "dequantize", v.numel()))
            out[dst][src] = o
    _device.check_err(err)
    if not device_in:
        out = [[t.cpu().numpy() for t in row] for row in out]
    return CollectiveResult(out, ledger, trace)
