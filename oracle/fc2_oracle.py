"""CPU oracle for the FlashCommunication-V2 hot path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The shipped package
(``paper_2508_03760_b200``) never imports anything under ``oracle/``; its
compute path is the CUDA library and it fails loudly when that is missing.

What it is
----------
A numpy restatement of the reference ``qcomm`` algorithm for the hot path
(reference = ``/root/reference/pkg/src/qcomm``, pure Python + numpy, float64
codec arithmetic).  Each function cites the reference file:line it restates.
The arithmetic contract it implements is SURVEY.md section 8.0, rules R1-R15.

Parity pinning
--------------
``tests/golden/make_golden.py`` imports the real reference in the build
container and writes ``tests/golden/*.npz`` (inputs + the reference's own
payload bytes / outputs).  ``tests/test_oracle_golden.py`` checks this oracle
byte-for-byte against those fixtures and against the reference's own
known-answer tests (5-bit plane golden, constant-chunk golden bytes, Table-5
footprints, RTN tie cases).  The oracle is therefore *pinned*.

Known unpinned corner (documented in DESIGN.md): the sign bit of a ``zero``
metadata field whose value is +-0.0 depends on numpy's SIMD min order in the
reference; codes, scales and decoded values are unaffected.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# configuration constants
# ---------------------------------------------------------------------------

# bit-split units, low bits first (codec.py:143-151, 154-162)
UNITS = {2: (2,), 3: (2, 1), 4: (4,), 5: (4, 1), 6: (4, 2), 7: (4, 2, 1), 8: (8,)}

INT8_SENTINEL = -128  # codec.py:37


class OracleError(ValueError):
    """Raised where the reference raises ConfigError/DataError/DecodeFormatError."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


def levels(bits: int) -> int:
    # codec.py:88-90
    return (1 << bits) - 1


def record_nbytes(sr: bool, intlog: bool) -> int:
    # codec.py:400-425: BF16 4 (+8 SR) bytes; INT_LOG 2 (+6 SR) bytes
    if intlog:
        return 8 if sr else 2
    return 12 if sr else 4


def footprint(bits: int, g: int, sr: bool, intlog: bool, n: int) -> int:
    # codec.py:428-432
    if n < 0 or n % g:
        raise OracleError("config", f"{n} not a multiple of {g}")
    return n * bits // 8 + (n // g) * record_nbytes(sr, intlog)


# ---------------------------------------------------------------------------
# bfloat16 (bfloat16.py:16-36)
# ---------------------------------------------------------------------------


def bf16_bits(x) -> np.ndarray:
    """float32 -> bf16 bit pattern, round-to-nearest-even via the +0x7FFF bias
    (bfloat16.py:16-25).  NaN maps to 0x7FC0."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    out = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return np.where(np.isnan(f), np.uint16(0x7FC0), out)


def bf16_value(bits) -> np.ndarray:
    """bf16 bit pattern -> float32, exact (bfloat16.py:28-31)."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32)
    return (b << 16).view(np.float32)


def bf16_snap(x) -> np.ndarray:
    """Snap to the bf16 grid, returned as float32 (bfloat16.py:34-36)."""
    return bf16_value(bf16_bits(x))


# ---------------------------------------------------------------------------
# bit planes (codec.py:165-238)
# ---------------------------------------------------------------------------


def pack(codes, bits: int) -> list[bytes]:
    """Codes -> one byte plane per unit.  Unit u carries code bits
    [off_u, off_u + w_u); inside a byte element i sits at bits [i*w, (i+1)*w)
    (codec.py:165-175, 204-225; 1-bit plane == packbits little)."""
    c = np.asarray(codes).astype(np.int64).reshape(-1)
    if c.size % 8:
        raise OracleError("data", "code count must be a multiple of 8")
    if c.size and (c.min() < 0 or c.max() >= (1 << bits)):
        raise OracleError("coderange", "code out of range")
    c = c.astype(np.uint32)
    planes, off = [], 0
    for w in UNITS[bits]:
        per = 8 // w
        part = ((c >> off) & ((1 << w) - 1)).reshape(-1, per)
        shifts = (np.arange(per, dtype=np.uint32) * w)[None, :]
        planes.append((part << shifts).sum(axis=1).astype(np.uint8).tobytes())
        off += w
    return planes


def unpack(planes, bits: int, n: int) -> np.ndarray:
    """Inverse of :func:`pack` (codec.py:178-201, 228-238)."""
    units = UNITS[bits]
    if len(planes) != len(units):
        raise OracleError("format", "plane count")
    out = np.zeros(n, dtype=np.uint32)
    off = 0
    for plane, w in zip(planes, units):
        raw = np.frombuffer(bytes(plane), dtype=np.uint8).astype(np.uint32)
        if raw.size != n * w // 8:
            raise OracleError("format", "plane length")
        per = 8 // w
        shifts = (np.arange(per, dtype=np.uint32) * w)[None, :]
        part = (raw[:, None] >> shifts) & ((1 << w) - 1)
        out |= part.reshape(-1)[:n] << off
        off += w
    return out.astype(np.uint8)


# ---------------------------------------------------------------------------
# encode / decode (codec.py:246-275, 454-563)
# ---------------------------------------------------------------------------


def _round_half_away(x):
    # codec.py:246-248: copysign(floor(|x| + 0.5), x) -- NOT np.round
    return np.copysign(np.floor(np.abs(x) + 0.5), x)


def _codes(rows, scale, offset, L):
    # codec.py:251-256
    pos = scale > 0
    denom = np.where(pos, scale, 1.0)[:, None]
    q = _round_half_away((rows - offset[:, None]) / denom)
    q = np.where(pos[:, None], q, 0.0)
    return np.clip(q, 0, L).astype(np.uint8)


def _intlog_params(scale, zero, theta):
    # codec.py:463-474 (R13)
    pos = scale > 0
    with np.errstate(divide="ignore"):
        lg = _round_half_away(np.log2(np.where(pos, scale, 1.0)) * theta)
    si = np.where(pos, np.clip(lg, -128, 127), INT8_SENTINEL).astype(np.int8)
    s_eff = np.where(si == INT8_SENTINEL, 0.0, np.exp2(si.astype(np.float64) / theta))
    denom = np.where(s_eff > 0, s_eff, 1.0)
    z = np.where(s_eff > 0, np.clip(_round_half_away(-zero / denom), -128, 127), 0.0)
    z = z.astype(np.int8)
    return si, z, s_eff, -z.astype(np.float64) * s_eff


def encode(values, bits: int, g: int, sr: bool = False, intlog: bool = False,
           theta: int = 10) -> tuple[list[bytes], bytes]:
    """One chunk -> (planes, meta) exactly as ``encode_chunk`` (codec.py:477-519).

    R1 widen to float64; R2 non-finite -> error; R3 contiguous groups;
    R4/R5 range or spike-reserved shrunk range; R6 scale in f64; R7 bf16
    metadata from the unrounded f64 scale/zero; R8 codes; R9 planes; R10 meta.
    """
    v = np.asarray(values, dtype=np.float64).reshape(-1)
    if v.size % g:
        raise OracleError("data", "length not a multiple of group size")
    if not np.all(np.isfinite(v)):
        raise OracleError("data", "non-finite input")
    L = levels(bits)
    rows = v.reshape(-1, g)
    G = rows.shape[0]
    gi = np.arange(G)
    if sr:
        # first-occurrence argmin/argmax; all-equal rows use (0, 1)  (codec.py:259-266)
        lo_i = np.argmin(rows, axis=1)
        hi_i = np.argmax(rows, axis=1)
        same = lo_i == hi_i
        lo_i = np.where(same, 0, lo_i)
        hi_i = np.where(same, 1, hi_i)
        smin = bf16_bits(rows[gi, lo_i].astype(np.float32))
        smax = bf16_bits(rows[gi, hi_i].astype(np.float32))
        # shrunk range over the other g-2 slots  (codec.py:269-275)
        masked = rows.copy()
        masked[gi, lo_i] = np.nan
        masked[gi, hi_i] = np.nan
        zero = np.nanmin(masked, axis=1)
        vmax = np.nanmax(masked, axis=1)
        # reserved slots are quantized as 0.0  (codec.py:494-496)
        qrows = rows.copy()
        qrows[gi, lo_i] = 0.0
        qrows[gi, hi_i] = 0.0
    else:
        zero = rows.min(axis=1)
        vmax = rows.max(axis=1)
        qrows = rows
    scale = (vmax - zero) / L  # codec.py:512
    if intlog:
        si, zi, s_eff, offset = _intlog_params(scale, zero, theta)
        codes = _codes(qrows, s_eff, offset, L)
        if sr:
            rec = np.zeros(G, dtype=[("s", "i1"), ("z", "i1"), ("a", "<u2"), ("b", "<u2"),
                                     ("ia", "u1"), ("ib", "u1")])
            rec["a"], rec["b"] = smin, smax
            rec["ia"], rec["ib"] = lo_i.astype(np.uint8), hi_i.astype(np.uint8)
        else:
            rec = np.zeros(G, dtype=[("s", "i1"), ("z", "i1")])
        rec["s"], rec["z"] = si, zi
    else:
        codes = _codes(qrows, scale, zero, L)
        cols = [bf16_bits(scale.astype(np.float32)), bf16_bits(zero.astype(np.float32))]
        if sr:
            cols += [smin, smax, bf16_bits(lo_i.astype(np.float32)),
                     bf16_bits(hi_i.astype(np.float32))]
        rec = np.stack(cols, axis=1).astype("<u2")
    return pack(codes.reshape(-1), bits), rec.tobytes()


def decode(planes, meta: bytes, n: int, bits: int, g: int, sr: bool = False,
           intlog: bool = False, theta: int = 10) -> np.ndarray:
    """(planes, meta) -> float64 values exactly as ``decode_chunk`` (codec.py:522-563)."""
    codes = unpack(planes, bits, n).astype(np.float64).reshape(-1, g)
    G = codes.shape[0]
    rb = record_nbytes(sr, intlog)
    if len(meta) != G * rb:
        raise OracleError("format", "metadata length")
    raw = np.frombuffer(bytes(meta), dtype=np.uint8).reshape(G, rb)
    if intlog:
        si = raw[:, 0].view(np.int8).astype(np.float64)
        zi = raw[:, 1].view(np.int8).astype(np.float64)
        scale = np.where(si == INT8_SENTINEL, 0.0, np.exp2(si / theta))
        offset = -zi * scale
        if sr:
            smin = raw[:, 2:4].copy().view("<u2")[:, 0]
            smax = raw[:, 4:6].copy().view("<u2")[:, 0]
            lo_i = raw[:, 6].astype(np.int64)
            hi_i = raw[:, 7].astype(np.int64)
    else:
        cols = raw.copy().view("<u2")
        scale = bf16_value(cols[:, 0]).astype(np.float64)
        offset = bf16_value(cols[:, 1]).astype(np.float64)
        if sr:
            smin, smax = cols[:, 2], cols[:, 3]
            with np.errstate(invalid="ignore"):
                lo_i = bf16_value(cols[:, 4]).astype(np.int64)
                hi_i = bf16_value(cols[:, 5]).astype(np.int64)
    out = codes * scale[:, None] + offset[:, None]
    if sr:
        bad = (lo_i < 0) | (lo_i >= g) | (hi_i < 0) | (hi_i >= g)
        if np.any(bad):
            raise OracleError("format", "spike index out of range")
        gi = np.arange(G)
        out[gi, lo_i] = bf16_value(smin).astype(np.float64)
        out[gi, hi_i] = bf16_value(smax).astype(np.float64)
    return out.reshape(-1)


def qdq_f32(vec_f32: np.ndarray, bits, g, sr, intlog=False, theta=10):
    """Quantize-dequantize one buffer; (decoded float32, wire bytes)
    (collectives.py:179-182)."""
    planes, meta = encode(vec_f32.astype(np.float64), bits, g, sr, intlog, theta)
    dq = decode(planes, meta, vec_f32.size, bits, g, sr, intlog, theta).astype(np.float32)
    return dq, sum(len(p) for p in planes) + len(meta)


# ---------------------------------------------------------------------------
# collectives (collectives.py:152-186, 263-315, 428-482)
# ---------------------------------------------------------------------------


def _as_f32_payloads(payloads, equal=True):
    # collectives.py:152-164
    out = [np.asarray(p, dtype=np.float32).reshape(-1) for p in payloads]
    if equal and len({p.size for p in out}) > 1:
        raise OracleError("data", "payload lengths differ")
    for p in out:
        if not np.all(np.isfinite(p)):
            raise OracleError("data", "non-finite payload")
    return out


def two_step(payloads, bits, g, sr, intlog=False, theta=10):
    """Two-step quantized AllReduce (collectives.py:263-315, rule R14).

    Returns (outputs, wire_bytes_per_shard_payload).  Every rank QDQs every
    shard including its own; receivers reduce in fp32 in rank order from +0;
    the owner QDQs the reduced shard and every rank (owner included) uses the
    decoded values; outputs are bf16-rounded and padding is stripped.
    """
    ranks = _as_f32_payloads(payloads)
    N = len(ranks)
    n = ranks[0].size
    mult = N * g
    padded = -(-n // mult) * mult
    ranks = [np.pad(p, (0, padded - n)) for p in ranks]
    S = padded // N
    reduced = []
    nbytes = 0
    for shard in range(N):
        acc = np.zeros(S, dtype=np.float32)
        for src in range(N):
            dq, nbytes = qdq_f32(ranks[src][shard * S:(shard + 1) * S], bits, g, sr, intlog, theta)
            acc += dq
        reduced.append(acc)
    merged = np.concatenate([qdq_f32(r, bits, g, sr, intlog, theta)[0] for r in reduced]) \
        if N else np.zeros(0, np.float32)
    out = bf16_snap(merged[:n])
    return [out.copy() for _ in range(N)], nbytes


def hierarchical(payloads, groups, bits, g, sr, intlog=False, theta=10):
    """Hierarchical quantized AllReduce over two NUMA islands joined by a
    bridge (collectives.py:318-425).  ``groups``: the two equal-size lists of
    device ids (cross_numa_partition order).  Stage rs: scatter-reduce inside
    each island (every member QDQs every segment, fp32 sum in member order from
    +0).  Stage xn: paired ranks i (island 0) / j (island 1) swap opposite
    halves -- total_low = low_i + QDQ(low_j), total_high = high_j + QDQ(high_i)
    -- and both keep QDQ(total_low) ++ QDQ(total_high).  Stage ag: every owner
    QDQs its segment once more and its island decodes it.  bf16 out, padding
    stripped."""
    ranks = _as_f32_payloads(payloads)
    N = len(ranks)
    gsz = len(groups[0])
    n = ranks[0].size
    mult = N * g
    padded = -(-n // mult) * mult
    ranks = [np.pad(p, (0, padded - n)) for p in ranks]
    seg = padded // gsz
    half = seg // 2
    q = lambda v: qdq_f32(v, bits, g, sr, intlog, theta)[0]
    reduced = {}
    for members in groups:
        for li, owner in enumerate(members):
            acc = np.zeros(seg, dtype=np.float32)
            for src in members:
                acc += q(ranks[src][li * seg:(li + 1) * seg])
            reduced[owner] = acc
    final = {}
    for i, j in zip(groups[0], groups[1]):
        total_low = reduced[i][:half] + q(reduced[j][:half])
        total_high = reduced[j][half:] + q(reduced[i][half:])
        final[i] = final[j] = np.concatenate([q(total_low), q(total_high)])
    outs = []
    for r in range(N):
        members = groups[0] if r in groups[0] else groups[1]
        outs.append(bf16_snap(np.concatenate([q(final[o]) for o in members])[:n]))
    return outs


def a2a_dispatch(payloads, bits, g, sr, matrix=None, intlog=False, theta=10):
    """Quantized All2All dispatch (collectives.py:428-482, rule R15).

    out[dst][src] is block (src -> dst): exact float32 copy on the diagonal,
    empty when the block is empty, otherwise the block zero-padded to a group
    multiple, QDQ'd as one chunk and sliced back (float32, no bf16 rounding).
    """
    N = len(payloads)
    ranks = _as_f32_payloads(payloads, equal=matrix is None)
    if matrix is None:
        per = ranks[0].size // N
        if per * N != ranks[0].size:
            raise OracleError("config", "payload not divisible by ranks")
        matrix = np.full((N, N), per, dtype=np.int64)
    matrix = np.asarray(matrix, dtype=np.int64)
    out = [[None] * N for _ in range(N)]
    for src in range(N):
        edges = np.concatenate([[0], np.cumsum(matrix[src])])
        for dst in range(N):
            blk = ranks[src][edges[dst]:edges[dst + 1]]
            if src == dst or blk.size == 0:
                out[dst][src] = blk.copy()
                continue
            plen = -(-blk.size // g) * g
            dq, _ = qdq_f32(np.pad(blk, (0, plen - blk.size)), bits, g, sr, intlog, theta)
            out[dst][src] = dq[:blk.size]
    return out


def a2a_combine(blocks, bits, g, sr, intlog=False, theta=10):
    """Quantized All2All combine -- the north-star addition with no reference
    function.  ``blocks[src][dst]`` is the float32 block expert-rank ``src``
    returns to token-owner ``dst``; it travels with the same codec as dispatch
    (pad to a group multiple, QDQ as one chunk, slice), the diagonal stays
    exact.  Returns out[dst][src] (same convention as :func:`a2a_dispatch`)."""
    N = len(blocks)
    out = [[None] * N for _ in range(N)]
    for src in range(N):
        for dst in range(N):
            blk = np.asarray(blocks[src][dst], dtype=np.float32).reshape(-1)
            if src == dst or blk.size == 0:
                out[dst][src] = blk.copy()
                continue
            plen = -(-blk.size // g) * g
            dq, _ = qdq_f32(np.pad(blk, (0, plen - blk.size)), bits, g, sr, intlog, theta)
            out[dst][src] = dq[:blk.size]
    return out


# ---------------------------------------------------------------------------
# MoE token dispatch / combine (BASELINE configs[3]) -- the reference's block
# All2All (collectives.py:428-482) applied to routed token rows
# ---------------------------------------------------------------------------


def moe_route(topk_ids, world: int, n_experts: int):
    """Per destination rank, the ascending token indices that route to at
    least one of its experts (experts split contiguously, n_experts // world
    per rank), and pos[t, d] = the token's index in that list or -1."""
    ids = np.asarray(topk_ids, dtype=np.int64)
    per = n_experts // world
    hit = np.zeros((ids.shape[0], world), dtype=bool)
    if ids.size:
        np.put_along_axis(hit, ids // per, True, axis=1)
    rows = [np.flatnonzero(hit[:, d]) for d in range(world)]
    pos = np.full((ids.shape[0], world), -1, dtype=np.int64)
    for d in range(world):
        pos[rows[d], d] = np.arange(rows[d].size)
    return rows, pos


def moe_dispatch(tokens, topk_ids, bits, g, sr, n_experts, intlog=False, theta=10):
    """tokens[s]: [T_s, H] float32 of rank s; topk_ids[s]: [T_s, K].
    Block (s -> d) = rows routes[s][d] of tokens[s], flattened, through
    :func:`a2a_dispatch` (QDQ'd as one zero-padded chunk, the diagonal exact).
    Returns recv[d] ([sum_s rows, H] float32, sources in rank order) and the
    per-source routing (rows, pos)."""
    N = len(tokens)
    H = np.asarray(tokens[0]).shape[1]
    routes = [moe_route(topk_ids[s], N, n_experts) for s in range(N)]
    matrix = np.array([[routes[s][0][d].size * H for d in range(N)] for s in range(N)], dtype=np.int64)
    flat = [np.concatenate([np.asarray(tokens[s], dtype=np.float32)[routes[s][0][d]].reshape(-1)
                            for d in range(N)]) for s in range(N)]
    out = a2a_dispatch(flat, bits, g, sr, matrix, intlog, theta)
    recv = [np.concatenate([out[d][s] for s in range(N)]).reshape(-1, H) for d in range(N)]
    return recv, routes


def moe_combine(expert_out, routes, bits, g, sr, intlog=False, theta=10):
    """expert_out[e]: [rows, H] float32 in rank e's dispatch order (the rows
    it received, sources in rank order).  Block (e -> s) = the rows that came
    from s, QDQ'd like dispatch (:func:`a2a_combine`, diagonal exact); rank s
    sums per token the returned rows over e = 0..N-1 in fp32 from +0.0."""
    N = len(expert_out)
    H = np.asarray(expert_out[0]).shape[1]
    counts = np.array([[routes[s][0][e].size for e in range(N)] for s in range(N)], dtype=np.int64)
    blocks = [[None] * N for _ in range(N)]
    for e in range(N):
        off = 0
        y = np.asarray(expert_out[e], dtype=np.float32)
        for s in range(N):
            k = int(counts[s, e])
            blocks[e][s] = y[off:off + k].reshape(-1)
            off += k
    back = a2a_combine(blocks, bits, g, sr, intlog, theta)
    outs = []
    for s in range(N):
        T = routes[s][1].shape[0]
        acc = np.zeros((T, H), dtype=np.float32)
        for e in range(N):
            rows = back[s][e].reshape(-1, H)
            sel = routes[s][0][e]
            acc[sel] = acc[sel] + rows  # float32 + float32, rank order
        outs.append(acc)
    return outs


# ---------------------------------------------------------------------------
# synthetic inputs (synthetic.py:25-49) -- used to regenerate benchmark data
# ---------------------------------------------------------------------------


def spiky(n: int, seed: int, rate: float = 1.0 / 64.0, mag: float = 50.0) -> np.ndarray:
    """N(0,1) with a ``rate`` fraction replaced by +-mag (synthetic.py:30-43)."""
    rng = np.random.default_rng(seed)
    vals = rng.normal(0.0, 1.0, n)
    hit = rng.random(n) < rate
    sign = rng.integers(0, 2, n) * 2 - 1
    vals[hit] = sign[hit] * mag
    return vals


def child_seeds(seed: int, n: int) -> list[int]:
    # synthetic.py:46-49
    return [int(c.generate_state(1)[0]) for c in np.random.SeedSequence(seed).spawn(n)]


# ---------------------------------------------------------------------------
# per-group scalar API (codec.py:278-343) and int-log helpers (codec.py:366-392)
# ---------------------------------------------------------------------------


def rtn_group(values, bits):
    """(codes, scale, zero) of one group (codec.py:278-290)."""
    v = np.asarray(values, dtype=np.float64)
    L = levels(bits)
    zero = v.min()
    scale = (v.max() - zero) / L
    codes = _codes(v[None, :], np.array([scale]), np.array([zero]), L)[0]
    return codes, float(scale), float(zero)


def spike_group(values, bits):
    """(codes, scale, zero, smin, smax, imin, imax) of one group (codec.py:298-329)."""
    v = np.asarray(values, dtype=np.float64)
    L = levels(bits)
    lo, hi = int(np.argmin(v)), int(np.argmax(v))
    if lo == hi:
        lo, hi = 0, 1
    smin = float(bf16_value(bf16_bits(np.float32(v[lo]))))
    smax = float(bf16_value(bf16_bits(np.float32(v[hi]))))
    rest = np.delete(v, [lo, hi])
    zero, vmax = rest.min(), rest.max()
    scale = (vmax - zero) / L
    work = v.copy()
    work[[lo, hi]] = 0.0
    codes = _codes(work[None, :], np.array([scale]), np.array([zero]), L)[0]
    return codes, float(scale), float(zero), smin, smax, lo, hi


def group_decode(codes, scale, zero):
    # codec.py:293-295
    return np.asarray(codes, dtype=np.float64) * scale + zero


def scale_to_int(scale, theta=10):
    # codec.py:366-381
    s = np.asarray(scale, dtype=np.float64)
    pos = s > 0
    with np.errstate(divide="ignore"):
        raw = _round_half_away(np.log2(np.where(pos, s, 1.0)) * theta)
    return np.where(pos, np.clip(raw, -128, 127), INT8_SENTINEL).astype(np.int8)


def int_to_scale(si, theta=10):
    # codec.py:384-392
    v = np.asarray(si, dtype=np.float64)
    return np.where(v == INT8_SENTINEL, 0.0, np.exp2(v / theta))
