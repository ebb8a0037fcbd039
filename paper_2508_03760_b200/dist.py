"""SPMD quantized collectives: one process per GPU (the multi-GPU form of
``two_step_allreduce_q`` / ``all2all_dispatch_q``, collectives.py:263-315,
428-482).

Two transports, same arithmetic and bit-identical results:

* ``"ipc"`` (default): every rank maps every peer's symmetric buffer through
  CUDA IPC (handles exchanged over the ``torch.distributed`` group); the
  codec kernels store packed shards straight into peer memory over NVLink
  and stream-ordered device barriers separate the stages
  (``fc2_allreduce_2step`` / ``fc2_a2a_q`` in the C ABI).  No NCCL on the
  data path.
* ``"nccl"``: encode into a local send buffer, ``all_to_all_single`` /
  ``all_gather_into_tensor`` of the packed bytes, reduce + requantize and
  decode locally -- the "NCCL send/recv of packed bytes" alternative.

The orchestration of the ``"nccl"`` transport is written against a small
codec interface (:class:`CudaCodec`), which is what the CPU tests drive with
gloo and a test-only codec double; the product codec is the CUDA library.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _lib
from .config import QuantConfig, footprint_bytes
from .errors import ConfigError, DataError

_SLOT_ALIGN = 16


def _round_up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


@dataclass(frozen=True)
class TwoStepLayout:
    """Shard geometry of the two-step AllReduce for n elements on N ranks
    (collectives.py:275-276: zero-pad to a multiple of N*g, contiguous shards)."""

    n: int
    world: int
    group_size: int
    bitwidth: int
    shard_bytes: int  # footprint of one packed shard
    slot_bytes: int   # shard_bytes rounded up to 16

    @staticmethod
    def make(n: int, world: int, config: QuantConfig) -> "TwoStepLayout":
        if world < 1:
            raise ConfigError("world must be >= 1")
        mult = world * config.group_size
        padded = _round_up(max(n, 0), mult)
        S = padded // world
        F = footprint_bytes(config, S)
        return TwoStepLayout(n, world, config.group_size, config.bitwidth, F,
                             _round_up(max(F, 1), _SLOT_ALIGN))

    @property
    def padded(self) -> int:
        return _round_up(self.n, self.world * self.group_size)

    @property
    def shard_len(self) -> int:
        return self.padded // self.world

    def valid(self, shard: int) -> int:
        """Real (unpadded) elements of shard j."""
        return max(0, min(self.shard_len, self.n - shard * self.shard_len))


def pipe_chunk_len(shard_len: int, chunks: int, group_size: int) -> int:
    """Microchunk length of the pipelined two-step (fc2_allreduce_2step_pipe):
    ceil(S / chunks) rounded up to whole groups and a multiple of 1024."""
    q = 1024
    while q % group_size:
        q += 1024
    return _round_up(-(-shard_len // max(1, chunks)), q)


def a2a_slot_offsets(matrix: np.ndarray, config: QuantConfig, dst: int) -> list[int]:
    """Byte offset of each source's packed block inside rank dst's receive
    region (same rule as fc2_a2a_q)."""
    N = matrix.shape[0]
    g = config.group_size
    offs, off = [], 0
    for s in range(N):
        offs.append(off)
        m = int(matrix[s, dst])
        if s != dst and m > 0:
            off += _round_up(footprint_bytes(config, _round_up(m, g)), _SLOT_ALIGN)
    offs.append(off)
    return offs


class CudaCodec:
    """The CUDA library behind the transport-agnostic orchestration."""

    def __init__(self, config: QuantConfig, device):
        self.cfg = config
        self.device = device
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        if config.int_log:
            _device.ensure_intlog(config.theta, device)

    def empty(self, nbytes: int) -> torch.Tensor:
        return torch.empty(nbytes, dtype=torch.uint8, device=self.device)

    def encode_shards(self, x: torch.Tensor, lay: TwoStepLayout, send: torch.Tensor) -> None:
        """Shard j of x -> send[j*slot : ...] (all shards in one launch)."""
        esz = x.element_size()
        jobs = [((x.data_ptr() + j * lay.shard_len * esz) if lay.valid(j) else x.data_ptr(),
                 lay.valid(j), lay.shard_len, send.data_ptr() + j * lay.slot_bytes) for j in range(lay.world)]
        from .collectives import _encode_jobs
        _encode_jobs(self.cfg, _device.dtype_code(x), jobs, self.err)

    def reduce(self, recv: torch.Tensor, lay: TwoStepLayout, out: torch.Tensor) -> None:
        """Decode the N packed copies of my shard, fp32 rank-order sum, re-encode."""
        from .collectives import reduce_requant
        reduce_requant(self.cfg, [recv.data_ptr() + s * lay.slot_bytes for s in range(lay.world)],
                       lay.shard_len, [out.data_ptr()], self.err)

    def decode_gathered(self, gath: torch.Tensor, lay: TwoStepLayout, y: torch.Tensor) -> None:
        c = self.cfg.c_struct()
        _lib.check(_lib.lib().fc2_gather_decode(
            ctypes.byref(c), lay.world, _lib.ptr_array([gath.data_ptr() + o * lay.slot_bytes
                                                        for o in range(lay.world)]),
            lay.shard_len, y.data_ptr(), _device.dtype_code(y), lay.n, self.err.data_ptr(),
            _device.stream_handle()))

    def check(self) -> None:
        bits = int(self.err.item())
        if bits:
            self.err.zero_()  # later calls start from a clean word
            _lib.raise_dev_err(bits)


def two_step_via_collectives(x: torch.Tensor, codec, lay: TwoStepLayout, group=None,
                             out: torch.Tensor | None = None) -> torch.Tensor:
    """Two-step AllReduce with torch.distributed collectives moving the packed
    bytes (collectives.py:278-314):
      encode N shards -> all_to_all (packed) -> reduce + requantize my shard ->
      all_gather (packed) -> decode all shards."""
    N, slot = lay.world, lay.slot_bytes
    send = codec.empty(N * slot)
    recv = codec.empty(N * slot)
    codec.encode_shards(x, lay, send)
    dist.all_to_all_single(recv, send, group=group)
    mine = codec.empty(slot)
    codec.reduce(recv, lay, mine)
    gath = codec.empty(N * slot)
    dist.all_gather_into_tensor(gath, mine, group=group)
    y = out if out is not None else torch.empty(lay.n, dtype=x.dtype, device=x.device)
    codec.decode_gathered(gath, lay, y)
    return y


class QComm:
    """Quantized collectives over one process group (one process per GPU).

    ``max_elems`` sizes the symmetric buffers for AllReduce payloads;
    ``a2a_bytes`` reserves the All2All receive region.
    """

    def __init__(self, group=None, max_elems: int = 1 << 25, config: QuantConfig | None = None,
                 transport: str = "ipc", a2a_bytes: int = 0, timeout_s: float = 60.0,
                 oneshot_max_elems: int = 1 << 18, pipe_chunks: int = 4):
        self.device = _device.require_cuda()
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.cfg = config or QuantConfig(4, group_size=128, chunk_size=128)
        self.transport = transport
        self.timeout_s = float(timeout_s)
        self.max_lay = TwoStepLayout.make(max_elems, self.world, self.cfg)
        self.a2a_off = 2 * self.world * self.max_lay.slot_bytes
        # one-shot region (small messages): 2 N^2 landing slots + N result slots
        self.os_lay = TwoStepLayout.make(min(int(oneshot_max_elems), max_elems), self.world, self.cfg)
        self.a2a_bytes = _round_up(int(a2a_bytes), _SLOT_ALIGN)
        self.os_off = self.a2a_off + self.a2a_bytes
        # pipelined two-step region: 2 parity sets x (land + gath) x N x chunks slots
        self.pipe_chunks = max(1, min(16, int(pipe_chunks)))
        # algo="auto" above the one-shot size: two-step or pipelined, whichever
        # the first call of a (size, codec) measured faster on this box (max
        # over ranks, so every rank picks the same one)
        self.autotune = True
        self._tuned: dict = {}
        sk = pipe_chunk_len(self.max_lay.shard_len, self.pipe_chunks, self.cfg.group_size)
        self.pipe_chunk_bytes = _round_up(max(footprint_bytes(self.cfg, sk), 1), _SLOT_ALIGN)
        self.pipe_bytes = 4 * self.world * self.pipe_chunks * self.pipe_chunk_bytes
        self.pipe_off = self.os_off + (2 * self.world * self.world + self.world) * self.os_lay.slot_bytes
        self.codec = CudaCodec(self.cfg, self.device)
        self.err = self.codec.err
        self._c = None
        self._nbytes = 0
        if transport not in ("ipc", "nccl"):
            raise ConfigError(f"unknown transport {transport!r}")
        if transport == "ipc":
            lib = _lib.lib()
            hb = lib.fc2_comm_handle_bytes()
            handle = (ctypes.c_uint8 * hb)()
            ptr = ctypes.c_void_p()
            nbytes = self.pipe_off + self.pipe_bytes
            self._nbytes = nbytes
            _lib.check(lib.fc2_comm_create(self.rank, self.world, nbytes, ctypes.byref(ptr),
                                           ctypes.cast(handle, ctypes.c_void_p)))
            self._c = ptr
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(handle), group=group)
            allh = (ctypes.c_uint8 * (hb * self.world)).from_buffer_copy(b"".join(handles))
            _lib.check(lib.fc2_comm_open_peers(self._c, ctypes.cast(allh, ctypes.c_void_p)))
            dist.barrier(group=group)

    def buffer_ptr(self, peer: int) -> int:
        """Device address of ``peer``'s symmetric buffer as mapped in this
        process (own rank: local memory; others: NVLink via CUDA IPC)."""
        if self._c is None:
            raise ConfigError("buffer_ptr needs the ipc transport")
        return int(_lib.lib().fc2_comm_buffer(self._c, int(peer)) or 0)

    @property
    def buffer_bytes(self) -> int:
        return self._nbytes

    @property
    def shard_len(self) -> int:
        return self.max_lay.shard_len

    def all_reduce(self, x: torch.Tensor, out: torch.Tensor | None = None, check: bool = False,
                   algo: str = "auto", config: QuantConfig | None = None) -> torch.Tensor:
        """Two-step quantized AllReduce of a 1-D bf16/f32 CUDA tensor; every
        rank gets the identical bf16-grid result (collectives.py:313-314).

        ``algo``: ``"two_step"`` (two packed exchanges), ``"one_shot"`` (one
        all-gather of packed shards, every rank reduces every shard: fewer
        barriers for latency-bound sizes, same bits), ``"fused"`` (the
        one-shot as one cooperative kernel with in-kernel flags),
        ``"pipelined"`` (microchunked two-step on three streams), or
        ``"auto"`` (on the ipc transport: up to ``oneshot_max_elems`` the
        one-shot or its fused form, above it the two-step or the pipelined
        two-step -- whichever the first call of that size measured faster,
        agreed over the ranks).  ``config``
        overrides the communicator's codec for this call when its packed
        shards fit the communicator's slots (e.g. fewer bits)."""
        cfg = self.cfg if config is None else config
        if cfg.int_log:
            _device.ensure_intlog(cfg.theta, self.device)
        x = x.reshape(-1)
        if not x.is_contiguous():
            x = x.contiguous()
        n = x.numel()
        if n > self.max_lay.n:
            raise DataError(f"payload of {n} elements exceeds the communicator's {self.max_lay.n}")
        if x.device != self.device:
            raise ConfigError(f"input on {x.device}, communicator on {self.device}")
        if out is not None and (out.device != self.device or not out.is_contiguous() or out.numel() != n):
            raise ConfigError(f"out must be a contiguous {n}-element tensor on {self.device}")
        y = out.reshape(-1) if out is not None else torch.empty(n, dtype=x.dtype, device=x.device)
        lay = TwoStepLayout.make(n, self.world, cfg)
        if algo not in ("auto", "two_step", "one_shot", "pipelined", "fused"):
            raise ConfigError(f"unknown allreduce algorithm {algo!r}")
        if algo == "fused":
            # the one-shot's result from one cooperative kernel (row f1)
            if self.transport != "ipc" or n > self.os_lay.n:
                raise ConfigError("fused needs the ipc transport and n <= oneshot_max_elems")
            if x.dtype not in (torch.bfloat16, torch.float32) or y.dtype not in (torch.bfloat16, torch.float32):
                raise ConfigError("fused takes bf16 / float32 tensors")
            c = cfg.c_struct()
            _lib.check(_lib.lib().fc2_allreduce_fused(
                self._c, ctypes.byref(c), x.data_ptr(), _device.dtype_code(x), y.data_ptr(),
                _device.dtype_code(y), n, self.os_lay.slot_bytes, self.os_off, self.err.data_ptr(),
                self.timeout_s, _device.stream_handle()))
            if check:
                self.check()
            return y
        if algo == "pipelined":
            if self.transport != "ipc":
                raise ConfigError("the pipelined two-step needs the ipc transport")
            c = cfg.c_struct()
            _lib.check(_lib.lib().fc2_allreduce_2step_pipe(
                self._c, ctypes.byref(c), x.data_ptr(), _device.dtype_code(x), y.data_ptr(),
                _device.dtype_code(y), n, self.pipe_chunks, self.pipe_chunk_bytes, self.pipe_off, self.pipe_bytes,
                self.err.data_ptr(), self.timeout_s, _device.stream_handle()))
            if check:
                self.check()
            return y
        if algo == "auto" and self.autotune and self.transport == "ipc" and self.world > 1:
            small = n <= self.os_lay.n
            cands = (("one_shot", "fused") if x.dtype in (torch.bfloat16, torch.float32)
                     and y.dtype in (torch.bfloat16, torch.float32) and cfg.group_size <= 256
                     else ("one_shot",)) if small else ("two_step", "pipelined")
            if len(cands) > 1:
                key = (n, cfg.bitwidth, cfg.group_size, cfg.scheme, cfg.scale_encoding, cfg.theta, x.dtype, y.dtype)
                if key not in self._tuned:
                    self._tuned[key] = self._tune(x, y, cfg, cands)
                algo = self._tuned[key]
                if algo in ("pipelined", "fused"):
                    return self.all_reduce(x, out=y, check=check, algo=algo, config=config)
        one = self.transport == "ipc" and n <= self.os_lay.n and algo != "two_step"
        if algo == "one_shot" and not one:
            raise ConfigError("one_shot needs the ipc transport and n <= oneshot_max_elems")
        if one:
            c = cfg.c_struct()
            _lib.check(_lib.lib().fc2_allreduce_oneshot(
                self._c, ctypes.byref(c), x.data_ptr(), _device.dtype_code(x), y.data_ptr(),
                _device.dtype_code(y), n, self.os_lay.slot_bytes, self.os_off, self.err.data_ptr(),
                self.timeout_s, _device.stream_handle()))
        elif self.transport == "ipc":
            c = cfg.c_struct()
            _lib.check(_lib.lib().fc2_allreduce_2step(
                self._c, ctypes.byref(c), x.data_ptr(), _device.dtype_code(x), y.data_ptr(),
                _device.dtype_code(y), n, self.max_lay.slot_bytes, self.err.data_ptr(), self.timeout_s,
                _device.stream_handle()))
        else:
            codec = self.codec if cfg == self.cfg else CudaCodec(cfg, self.device)
            two_step_via_collectives(x, codec, lay, self.group, y)
        if check:
            self.check()
        return y

    def _tune(self, x: torch.Tensor, y: torch.Tensor, cfg: QuantConfig, algos) -> str:
        """Time the candidate algorithms on this call's own buffers (each result
        is the same bits, so the caller's output is valid whichever ran last)
        and agree on the fastest across ranks."""
        ts = []
        # in-place calls (out aliases x): the timed runs write a private output,
        # so the caller's input is intact for the call that follows
        xs, xe = x.data_ptr(), x.data_ptr() + x.numel() * x.element_size()
        ys, ye = y.data_ptr(), y.data_ptr() + y.numel() * y.element_size()
        if xs < ye and ys < xe:
            y = torch.empty_like(y)
        for a in algos:
            self.all_reduce(x, out=y, algo=a, config=cfg)  # warm
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            self.all_reduce(x, out=y, algo=a, config=cfg)
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        dev = self.device if dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        t = torch.tensor(ts, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        t = t.cpu().tolist()
        return algos[min(range(len(algos)), key=lambda i: t[i])]

    def all2all(self, x: torch.Tensor, matrix, out: torch.Tensor | None = None,
                out_dtype: torch.dtype = torch.float32, check: bool = False) -> torch.Tensor:
        """Quantized All2All (dispatch; combine = transposed matrix).

        ``matrix[src][dst]`` = elements src sends to dst (known on all ranks).
        ``x`` holds this rank's blocks for dst 0..N-1 back to back; the result
        holds the blocks from src 0..N-1 back to back: exact copy on the
        diagonal, QDQ'd (zero-padded to a group multiple) elsewhere."""
        if self.transport != "ipc":
            raise ConfigError("all2all is implemented on the ipc transport")
        m = np.ascontiguousarray(np.asarray(matrix, dtype=np.int64))
        N, r = self.world, self.rank
        if m.shape != (N, N) or np.any(m < 0):
            raise ConfigError(f"dispatch matrix must be a non-negative {N}x{N} array")
        if int(m[r].sum()) != x.numel():
            raise ConfigError("dispatch row does not match the payload size")
        n_out = int(m[:, r].sum())
        if out is not None and (out.device != self.device or not out.is_contiguous() or out.numel() != n_out):
            raise ConfigError(f"out must be a contiguous {n_out}-element tensor on {self.device}")
        y = out if out is not None else torch.empty(n_out, dtype=out_dtype, device=x.device)
        x = x.reshape(-1).contiguous()
        c = self.cfg.c_struct()
        mp = m.reshape(-1)
        # remote blocks into the receivers' All2All regions, the diagonal block
        # copied exactly (non-finite values flagged, collectives.py:152-164)
        _lib.check(_lib.lib().fc2_a2a_q(
            self._c, ctypes.byref(c), x.data_ptr(), _device.dtype_code(x),
            mp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), y.data_ptr(), _device.dtype_code(y),
            self.a2a_off, self.a2a_bytes, self.err.data_ptr(), self.timeout_s, _device.stream_handle()))
        if check:
            self.check()
        return y

    def moe_dispatch(self, x: torch.Tensor, topk_ids: torch.Tensor, n_experts: int = 256,
                     out_dtype: torch.dtype = torch.bfloat16, check: bool = False):
        """Quantized MoE token dispatch (BASELINE configs[3]; moe.moe_dispatch_q
        is the simulated form).  ``x``: [T, H] bf16/f32 tokens of this rank,
        ``topk_ids``: [T, K] expert ids (experts split contiguously over the
        ranks).  Routing runs on the device (``fc2_moe_route``), the counts are
        all-gathered through the communicator (one host read), and every
        remote block is gather-encoded straight from the token rows into the
        receiver's All2All region.  Returns ``(recv, handle)``: recv [R, H]
        holds the rows from source ranks in order; ``handle`` feeds
        :meth:`moe_combine`."""
        from .moe import route

        if self.transport != "ipc":
            raise ConfigError("moe_dispatch is implemented on the ipc transport")
        if x.dim() != 2:
            raise ConfigError(f"tokens must be [tokens, hidden], got shape {tuple(x.shape)}")
        x = x.contiguous()
        T, H = x.shape
        N, r = self.world, self.rank
        counts, rows, pos = route(topk_ids.to(self.device), N, n_experts, self.err)
        allc = torch.empty(N * N, dtype=torch.int32, device=self.device)
        _lib.check(_lib.lib().fc2_comm_allgather_i32(self._c, counts.data_ptr(), N, allc.data_ptr(),
                                                     self.err.data_ptr(), self.timeout_s, _device.stream_handle()))
        tm = np.ascontiguousarray(allc.cpu().numpy().astype(np.int64).reshape(N, N))
        if int(self.err.item()):
            self.check()
        y = torch.empty((int(tm[:, r].sum()), H), dtype=out_dtype, device=self.device)
        c = self.cfg.c_struct()
        _lib.check(_lib.lib().fc2_moe_dispatch(
            self._c, ctypes.byref(c), x.data_ptr(), _device.dtype_code(x), T, H, rows.data_ptr(),
            tm.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), y.data_ptr(), _device.dtype_code(y),
            self.a2a_off, self.a2a_bytes, self.err.data_ptr(), self.timeout_s, _device.stream_handle()))
        if check:
            self.check()
        return y, {"matrix": tm, "rows": rows, "pos": pos, "tokens": T, "hidden": H}

    def moe_combine(self, y: torch.Tensor, handle: dict, out: torch.Tensor | None = None,
                    out_dtype: torch.dtype = torch.bfloat16, check: bool = False) -> torch.Tensor:
        """Quantized MoE combine: ``y`` = the expert outputs [R, H] in the
        order :meth:`moe_dispatch` delivered the rows.  Each block returns to
        its source rank with the same codec; the result [T, H] is, per token,
        the fp32 sum of its returned rows in rank order (exact for this rank's
        own experts)."""
        if self.transport != "ipc":
            raise ConfigError("moe_combine is implemented on the ipc transport")
        tm, T, H = handle["matrix"], handle["tokens"], handle["hidden"]
        N, r = self.world, self.rank
        y = y.contiguous()
        if y.dim() != 2 or y.shape[1] != H or y.shape[0] != int(tm[:, r].sum()):
            raise ConfigError(f"expert outputs must be [{int(tm[:, r].sum())}, {H}], got {tuple(y.shape)}")
        if out is not None and (out.device != self.device or not out.is_contiguous() or out.numel() != T * H):
            raise ConfigError(f"out must be a contiguous [{T}, {H}] tensor on {self.device}")
        res = out if out is not None else torch.empty((T, H), dtype=out_dtype, device=self.device)
        scratch = _device.workspace("moe_scratch", max(16, 4 * int(tm[r].sum()) * H), self.device)
        c = self.cfg.c_struct()
        _lib.check(_lib.lib().fc2_moe_combine(
            self._c, ctypes.byref(c), y.data_ptr(), _device.dtype_code(y), T, H,
            tm.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), handle["pos"].data_ptr(), scratch.data_ptr(),
            res.data_ptr(), _device.dtype_code(res), self.a2a_off, self.a2a_bytes, self.err.data_ptr(),
            self.timeout_s, _device.stream_handle()))
        if check:
            self.check()
        return res

    def check(self) -> None:
        """Raise for any error bit the device set since the last check (the
        reference's DataError / DecodeFormatError, or a cross-rank timeout), then
        clear the word so later calls start clean.  Synchronizes the stream."""
        bits = int(self.err.item())
        if bits:
            self.err.zero_()
            _lib.raise_dev_err(bits)

    def close(self) -> None:
        if self._c is not None:
            _lib.lib().fc2_comm_destroy(self._c)
            self._c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# MoE All2All helpers (BASELINE configs[3]) used by bench.py
# ---------------------------------------------------------------------------


def moe_token_matrix(routing, world: int, experts: int) -> np.ndarray:
    """tokens[src][dst]: how many of rank src's tokens route to at least one
    expert on rank dst (one copy per distinct destination rank, SURVEY 8 d).
    routing: int64 [world, tokens, topk] expert ids, experts contiguous per rank."""
    per = experts // world
    mat = np.zeros((world, world), dtype=np.int64)
    r = np.asarray(routing)
    for s in range(world):
        hit = np.zeros((r.shape[1], world), dtype=bool)
        np.put_along_axis(hit, r[s] // per, True, axis=1)
        mat[s] = hit.sum(0)
    return mat


def moe_region_bytes(config: QuantConfig, world: int, tokens: int, hidden: int, routing,
                     experts: int = 256) -> int:
    """All2All receive-region bytes for the MoE dispatch/combine of ``routing``."""
    mat = moe_token_matrix(routing, world, experts) * hidden
    need = 0
    for d in range(world):
        tot = sum(_round_up(footprint_bytes(config, _round_up(int(mat[s, d]), config.group_size)), _SLOT_ALIGN)
                  for s in range(world) if s != d and mat[s, d])
        tot_c = sum(_round_up(footprint_bytes(config, _round_up(int(mat[d, s]), config.group_size)), _SLOT_ALIGN)
                    for s in range(world) if s != d and mat[d, s])
        need = max(need, tot, tot_c)
    return need + 4096


def bench_moe(comm: "QComm", config: QuantConfig, routing, tokens: int, hidden: int, timed, steps: int,
              warmup: int, with_nccl: bool, experts: int = 256) -> dict:
    """MoE dispatch + combine driven by real top-k routing (moe_dispatch /
    moe_combine: device routing, row gather fused into the encoder, combine
    reduction), vs the bf16 NCCL all_to_all of the same token rows."""
    import statistics

    world, rank = comm.world, comm.rank
    g = torch.Generator(device=comm.device).manual_seed(7000 + rank)
    x = torch.randn((tokens, hidden), device=comm.device, generator=g).to(torch.bfloat16)
    ids = torch.as_tensor(np.asarray(routing[rank])).to(comm.device)
    recv, h = comm.moe_dispatch(x, ids, n_experts=experts, check=True)
    yexp = recv.clone()
    t_d = statistics.mean(timed(lambda: comm.moe_dispatch(x, ids, n_experts=experts), steps, warmup))
    t_c = statistics.mean(timed(lambda: comm.moe_combine(yexp, h), steps, warmup))
    tm = h["matrix"]
    sent = int(tm[rank].sum() - tm[rank, rank]) * hidden
    out = {"shape": f"{tokens} tok x {hidden}, top-8 of {experts}, EP={world}",
           "form": "token routing (fc2_moe_route) + gather-encode + combine sum",
           "copies_per_token": round(float(tm[rank].sum()) / tokens, 3),
           "dispatch_ms": round(t_d, 4), "combine_ms": round(t_c, 4),
           "dispatch_algbw_GBps": round(2 * sent / (t_d * 1e-3) / 1e9, 2)}
    if with_nccl:
        import torch.distributed as dist

        rows = [h["rows"][d * tokens:d * tokens + int(tm[rank, d])].long() for d in range(world)]
        send = torch.cat([x[r] for r in rows]).reshape(-1)
        rbuf = torch.empty(int(tm[:, rank].sum()) * hidden, dtype=torch.bfloat16, device=comm.device)
        ins = [int(v) * hidden for v in tm[rank]]
        outs = [int(v) * hidden for v in tm[:, rank]]
        t_n = statistics.mean(timed(lambda: dist.all_to_all_single(rbuf, send, outs, ins, group=comm.group),
                                    steps, warmup))
        out["nccl_bf16_dispatch_ms"] = round(t_n, 4)
        out["nccl_note"] = "bf16 all_to_all_single of the already-gathered rows (routing/gather not timed)"
        out["speedup_vs_nccl"] = round(t_n / t_d, 3)
    return out
