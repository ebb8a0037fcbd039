"""MoE token dispatch / combine with the quantized All2All (BASELINE configs[3],
north_star item 3: "the same codec fused into the All2All MoE token dispatch
and combine").

The reference ships only the block All2All (collectives.py:428-482): block
(src, dst) of a flat payload is quantized as one zero-padded chunk, the
diagonal stays exact.  MoE dispatch is that exchange where block (src, dst)
is the rows of rank src's tokens routed to at least one expert on rank dst
(one copy per distinct destination rank, token order); combine returns every
block to its source rank with the same codec and the source sums, per token,
the returned rows in rank order in fp32.  The routing (``fc2_moe_route``),
the row gather (fused into the encoders: ``fc2_encode_batch_rows``) and the
combine reduction (``fc2_moe_combine_sum``) run on the GPU; this module is
host orchestration only.

``moe_dispatch_q`` / ``moe_combine_q`` simulate N ranks on one device with
the reference's calling convention (a list of per-rank payloads + topology);
``dist.QComm.moe_dispatch`` / ``moe_combine`` are the one-process-per-GPU
form over NVLink peer memory.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .collectives import (
    CollectiveResult,
    ComputeEvent,
    StageTrace,
    TrafficLedger,
    TransferEvent,
    _encode_jobs,
    _decode_jobs,
    _round_up,
)
from .config import QuantConfig, footprint_bytes
from .errors import ConfigError
from .topology import Topology

_ALIGN = 16


@dataclass
class MoeLayout:
    """Routing of one dispatch: ``counts[s][d]`` = rows rank s sends to rank d;
    per source rank the device lists ``rows[s]`` (int32, dst d at
    ``[d * T_s, d * T_s + counts[s][d])``) and ``pos[s]`` (int32 [T_s, N]:
    index of token t in dst d's list, or -1)."""

    counts: np.ndarray
    rows: list
    pos: list
    tokens: list
    hidden: int
    n_experts: int

    def recv_offsets(self, dst: int) -> list[int]:
        """Row offset of each source's block inside rank dst's receive buffer."""
        return [int(v) for v in np.concatenate([[0], np.cumsum(self.counts[:, dst])])[:-1]]


def route(topk_ids: torch.Tensor, world: int, n_experts: int, err: torch.Tensor):
    """Device routing of one rank's tokens: (counts [world] int32, rows
    [world * T] int32, pos [T, world] int32), stream-ordered."""
    ids = topk_ids
    if ids.dim() != 2:
        raise ConfigError(f"topk ids must be [tokens, k], got shape {tuple(ids.shape)}")
    if ids.dtype not in (torch.int32, torch.int64):
        ids = ids.to(torch.int64)
    ids = ids.contiguous()
    T, K = ids.shape
    dev = ids.device
    counts = torch.empty(world, dtype=torch.int32, device=dev)
    rows = torch.empty(max(1, world * T), dtype=torch.int32, device=dev)
    pos = torch.empty((T, world), dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().fc2_moe_route(ids.data_ptr(), int(ids.dtype == torch.int64), T, K, int(n_experts),
                                        int(world), counts.data_ptr(), rows.data_ptr(), pos.data_ptr(),
                                        err.data_ptr(), _device.stream_handle()))
    return counts, rows, pos


def _stage_tokens(tokens, N: int, dev):
    if len(tokens) != N:
        raise ConfigError(f"expected {N} token tensors, got {len(tokens)}")
    out = []
    for t in tokens:
        if not isinstance(t, torch.Tensor):
            t = torch.from_numpy(np.ascontiguousarray(np.asarray(t, dtype=np.float32)))
        if t.dim() != 2:
            raise ConfigError(f"tokens must be [tokens, hidden], got shape {tuple(t.shape)}")
        t = t.to(dev)
        if t.dtype not in (torch.bfloat16, torch.float32):
            t = t.to(torch.float32)
        out.append(t.contiguous())
    H = out[0].shape[1]
    if any(t.shape[1] != H for t in out):
        raise ConfigError("every rank's tokens must have the same hidden size")
    if H % 8:
        raise ConfigError(f"hidden size {H} must be a multiple of 8")
    return out, H


def _ledger_events(st, ledger, counts, H, cfg, name_rank_pairs):
    for (src, dst) in name_rank_pairs:
        k = int(counts[src, dst]) * H
        f = footprint_bytes(cfg, _round_up(k, cfg.group_size))
        st.computes.append(ComputeEvent(st.name, 0, src, "quantize", k))
        ev = TransferEvent(st.name, 1, src, dst, k, f)
        st.transfers.append(ev)
        ledger.record(ev)
        st.computes.append(ComputeEvent(st.name, 2, dst, "dequantize", k))


@dataclass
class MoeResult(CollectiveResult):
    layout: MoeLayout | None = None


def moe_dispatch_q(tokens, topk_ids, topo: Topology, config: QuantConfig, n_experts: int = 256) -> MoeResult:
    """Quantized MoE token dispatch over ``topo.n_devices`` simulated ranks.

    ``tokens[s]``: [T_s, H] bf16/f32 of rank s; ``topk_ids[s]``: [T_s, K]
    expert ids (experts split contiguously over the ranks).  ``outputs[d]``:
    float32 [sum_s counts[s][d], H], the rows from source ranks in order --
    QDQ'd with the block All2All codec (collectives.py:462-480), exact for the
    rank's own tokens.  ``layout`` feeds :func:`moe_combine_q`."""
    N = topo.n_devices
    dev = _device.require_cuda()
    xs, H = _stage_tokens(tokens, N, dev)
    if len(topk_ids) != N:
        raise ConfigError(f"expected {N} routing tensors, got {len(topk_ids)}")
    if config.int_log:
        _device.ensure_intlog(config.theta, dev)
    err = _device.new_err(dev)
    ids = [torch.as_tensor(np.asarray(t) if not isinstance(t, torch.Tensor) else t).to(dev) for t in topk_ids]
    routes = []
    for s in range(N):
        if ids[s].shape[0] != xs[s].shape[0]:
            raise ConfigError(f"rank {s}: {ids[s].shape[0]} routing rows for {xs[s].shape[0]} tokens")
        routes.append(route(ids[s], N, n_experts, err))
    counts = torch.stack([r[0] for r in routes]).cpu().numpy().astype(np.int64)
    _device.check_err(err)
    G = config.group_size
    outs = [torch.empty((int(counts[:, d].sum()), H), dtype=torch.float32, device=dev) for d in range(N)]
    # packed blocks (s -> d), one slot each
    slots = {}
    total = 0
    for s in range(N):
        for d in range(N):
            k = int(counts[s, d]) * H
            if s != d and k:
                slots[(s, d)] = total
                total += _round_up(footprint_bytes(config, _round_up(k, G)), _ALIGN)
    pay = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
    c = config.c_struct()
    lib = _lib.lib()
    dec = []
    for s in range(N):
        T = xs[s].shape[0]
        dsts = [d for d in range(N) if (s, d) in slots]
        if dsts:  # one gather-encode launch per source rank
            rows = [routes[s][1].data_ptr() + 4 * d * T for d in dsts]
            nv = [int(counts[s, d]) * H for d in dsts]
            _lib.check(lib.fc2_encode_batch_rows(
                ctypes.byref(c), _device.dtype_code(xs[s]), len(dsts), xs[s].data_ptr(), _lib.ptr_array(rows), H,
                _lib.i64_array(nv), _lib.i64_array([_round_up(v, G) for v in nv]),
                _lib.ptr_array([pay.data_ptr() + slots[(s, d)] for d in dsts]), err.data_ptr(),
                _device.stream_handle()))
        for d in range(N):
            k = int(counts[s, d])
            if not k:
                continue
            off = int(counts[:s, d].sum())
            dst = outs[d][off:off + k]
            if s == d:  # the rank's own tokens never cross a wire: exact rows (collectives.py:466-468)
                _lib.check(lib.fc2_gather_rows_check(
                    xs[s].data_ptr(), _device.dtype_code(xs[s]), routes[s][1].data_ptr() + 4 * d * T, k, H,
                    dst.data_ptr(), _lib.F32, err.data_ptr(), _device.stream_handle()))
            else:
                dec.append((pay.data_ptr() + slots[(s, d)], _round_up(k * H, G), dst.data_ptr(), k * H))
    if dec:
        _decode_jobs(config, _lib.F32, dec, err)
    _device.check_err(err)
    trace, ledger = StageTrace(), TrafficLedger(topo)
    _ledger_events(trace.stage("dispatch"), ledger, counts, H, config, sorted(slots))
    layout = MoeLayout(counts, [r[1] for r in routes], [r[2] for r in routes], [x.shape[0] for x in xs], H,
                       int(n_experts))
    return MoeResult(outs, ledger, trace, layout)


def moe_combine_q(expert_out, layout: MoeLayout, topo: Topology, config: QuantConfig) -> CollectiveResult:
    """Quantized MoE combine: ``expert_out[e]`` = [rows, H] bf16/f32 outputs of
    rank e in its dispatch order.  Block (e -> s) returns to source rank s
    with the dispatch codec; ``outputs[s]`` = float32 [T_s, H], the per-token
    fp32 sum over e = 0..N-1 of the returned rows (exact for e == s)."""
    N = topo.n_devices
    dev = _device.require_cuda()
    ys, H = _stage_tokens(expert_out, N, dev)
    if H != layout.hidden:
        raise ConfigError(f"hidden size {H} differs from the dispatch's {layout.hidden}")
    counts = layout.counts
    for e in range(N):
        if ys[e].shape[0] != int(counts[:, e].sum()):
            raise ConfigError(f"rank {e}: {ys[e].shape[0]} expert rows, dispatch delivered {int(counts[:, e].sum())}")
    if config.int_log:
        _device.ensure_intlog(config.theta, dev)
    err = _device.new_err(dev)
    G = config.group_size
    # blocks (e -> s): rows [off, off + counts[s][e]) of ys[e]
    enc, dec, slots = {}, [], {}
    total = 0
    for e in range(N):
        for s in range(N):
            k = int(counts[s, e]) * H
            if s != e and k:
                slots[(e, s)] = total
                total += _round_up(footprint_bytes(config, _round_up(k, G)), _ALIGN)
    pay = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
    # fused combine (fc2_moe_combine_q) reads the packed blocks directly; other
    # shapes decode every block to float32 first (fc2_moe_combine_sum)
    fused = G % 32 == 0 and H % 32 == 0
    scratch = [] if fused else [torch.empty((int(counts[s].sum()), H), dtype=torch.float32, device=dev)
                                for s in range(N)]
    for (e, s), off in slots.items():
        k = int(counts[s, e])
        r0 = int(counts[:s, e].sum())
        enc.setdefault(_device.dtype_code(ys[e]), []).append(
            (ys[e][r0:r0 + k].data_ptr(), k * H, _round_up(k * H, G), pay.data_ptr() + off))
        if not fused:
            so = int(counts[s, :e].sum())
            dec.append((pay.data_ptr() + off, _round_up(k * H, G), scratch[s][so:so + k].data_ptr(), k * H))
    for code, jobs in enc.items():
        _encode_jobs(config, code, jobs, err)
    if dec:
        _decode_jobs(config, _lib.F32, dec, err)
    outs = []
    c = config.c_struct()
    for s in range(N):
        T = layout.tokens[s]
        out = torch.empty((T, H), dtype=torch.float32, device=dev)
        if fused:
            r0 = int(counts[:s, s].sum())
            pays = [pay.data_ptr() + slots[(e, s)] if (e, s) in slots else pay.data_ptr() for e in range(N)]
            ns = [_round_up(int(counts[s, e]) * H, G) for e in range(N)]
            if T:
                _lib.check(_lib.lib().fc2_moe_combine_q(
                    ctypes.byref(c), N, s, _lib.ptr_array(pays), _lib.i64_array(ns),
                    ys[s].data_ptr() + r0 * H * ys[s].element_size(), _device.dtype_code(ys[s]),
                    layout.pos[s].data_ptr(), T, H, out.data_ptr(), _lib.F32, err.data_ptr(),
                    _device.stream_handle()))
            outs.append(out)
            continue
        srcs, dts, chk = [], [], []
        for e in range(N):
            if e == s:
                r0 = int(counts[:s, s].sum())
                srcs.append(ys[s].data_ptr() + r0 * H * ys[s].element_size())
                dts.append(_device.dtype_code(ys[s]))
                chk.append(1)
            else:
                srcs.append(scratch[s][int(counts[s, :e].sum()):].data_ptr() if counts[s, e] else scratch[s].data_ptr())
                dts.append(_lib.F32)
                chk.append(0)
        dt = np.asarray(dts, dtype=np.int32)
        ck = np.asarray(chk, dtype=np.int32)
        if T:
            _lib.check(_lib.lib().fc2_moe_combine_sum(
                N, _lib.ptr_array(srcs), dt.ctypes.data, ck.ctypes.data, layout.pos[s].data_ptr(), T, H,
                out.data_ptr(), _lib.F32, err.data_ptr(), _device.stream_handle()))
        outs.append(out)
    _device.check_err(err)
    trace, ledger = StageTrace(), TrafficLedger(topo)
    _ledger_events(trace.stage("combine"), ledger, counts.T, H, config, sorted(slots))
    return CollectiveResult(outs, ledger, trace)
