// fc2_decode.cuh -- dequantizer cores (decode_chunk, codec.py:522-563; R12).
//
// BF16 metadata: value = fma(code, scale_bf16, zero_bf16).  The product is
// exact (<= 16 significant bits), so a float32 FMA equals the reference's
// float64 `codes*scale + offset` followed by .astype(float32), and a float64
// FMA equals its float64 result.  INT_LOG metadata: float64 mul then add
// (two roundings, as numpy does), scale from the host-computed exp2 table.
// Reserved spikes overwrite imin, then imax (codec.py:559-561).
#pragma once

#include "fc2_common.cuh"

namespace fc2 {

struct DecCtx {
  int64_t n;         // chunk elements
  int64_t meta_off;  // byte offset of metadata
  int B, G;
  bool sr, intlog;
  int theta;
  const double* lut;
  int32_t* err;
};

// decoded metadata of one group
struct GroupMeta {
  float s32, z32;       // BF16 mode
  double s64, o64;      // INT_LOG mode (scale, offset)
  float smin, smax;     // reserved values
  int imin, imax;       // reserved indices (validated, else -1)
};

// the group's metadata from its raw record words (load_record)
__device__ __forceinline__ GroupMeta meta_from_record(const uint32_t (&r)[3], const DecCtx& c) {
  GroupMeta m;
  m.imin = m.imax = -1;
  m.smin = m.smax = 0.f;
  if (!c.intlog) {
    m.s32 = bf16_val(r[0] & 0xFFFFu);
    m.z32 = bf16_val(r[0] >> 16);
    m.s64 = 0.0; m.o64 = 0.0;
    if (c.sr) {
      m.smin = bf16_val(r[1] & 0xFFFFu);
      m.smax = bf16_val(r[1] >> 16);
      // indices ride in bf16 float slots; astype(int64) truncates (codec.py:550-551)
      float fi = bf16_val(r[2] & 0xFFFFu), fa = bf16_val(r[2] >> 16);
      bool ok = (fi > -1.0f) && (fi < (float)c.G) && (fa > -1.0f) && (fa < (float)c.G);
      if (ok) { m.imin = (int)fi; m.imax = (int)fa; }
      else if (c.err) atomicOr(c.err, FC2_ERR_SPIKE_INDEX);
    }
  } else {
    int si = (int)(int8_t)(r[0] & 0xFFu), zi = (int)(int8_t)((r[0] >> 8) & 0xFFu);
    m.s64 = si == -128 ? 0.0 : c.lut[si + 128];
    m.o64 = __dmul_rn(-(double)zi, m.s64);  // codec.py:544
    m.s32 = 0.f; m.z32 = 0.f;
    if (c.sr) {
      m.smin = bf16_val(r[0] >> 16);
      m.smax = bf16_val(r[1] & 0xFFFFu);
      int ii = (int)((r[1] >> 16) & 0xFFu), ia = (int)(r[1] >> 24);
      if (ii < c.G && ia < c.G) { m.imin = ii; m.imax = ia; }
      else if (c.err) atomicOr(c.err, FC2_ERR_SPIKE_INDEX);
    }
  }
  return m;
}

__device__ __forceinline__ GroupMeta read_meta(const uint8_t* payload, int64_t grp, const DecCtx& c) {
  uint32_t r[3] = {0, 0, 0};
  load_record(payload + c.meta_off + grp * rec_bytes(c.sr, c.intlog), r, rec_bytes(c.sr, c.intlog));
  return meta_from_record(r, c);
}

__device__ __forceinline__ float code_f32(uint32_t c) {  // exact int -> float
  return __fsub_rn(__uint_as_float(0x4B000000u | c), 8388608.0f);
}

// one element's value in float32 / float64 from its code
__device__ __forceinline__ float dq32(uint32_t code, const GroupMeta& m, bool intlog) {
  if (!intlog) return __fmaf_rn(code_f32(code), m.s32, m.z32);
  return __double2float_rn(__dadd_rn(__dmul_rn((double)code, m.s64), m.o64));
}
__device__ __forceinline__ double dq64(uint32_t code, const GroupMeta& m, bool intlog) {
  if (!intlog) return fma((double)code, (double)m.s32, (double)m.z32);
  return __dadd_rn(__dmul_rn((double)code, m.s64), m.o64);
}

// Codes of the RUN=32 consecutive elements starting at e0 (e0 % 32 == 0):
// returns them unpacked into c[32].
template <int B>
__device__ __forceinline__ void load_codes32(const uint8_t* payload, int64_t n, int64_t e0, uint32_t* c) {
#pragma unroll
  for (int k = 0; k < 32; ++k) c[k] = 0;
#pragma unroll
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u), O = unit_off(B, u);
    const uint8_t* p = payload + (n * O) / 8 + (e0 * W) / 8;  // 4W bytes, 4-byte aligned
    uint32_t w[8];
    uintptr_t a = reinterpret_cast<uintptr_t>(p);
    if (W >= 4 && (a & 15u) == 0) {
#pragma unroll
      for (int i = 0; i < W; i += 4) {
        uint4 q = *reinterpret_cast<const uint4*>(p + 4 * i);
        w[i] = q.x; w[i + 1] = q.y; w[i + 2] = q.z; w[i + 3] = q.w;
      }
    } else if (W >= 2 && (a & 7u) == 0) {
#pragma unroll
      for (int i = 0; i < W; i += 2) {
        uint2 q = *reinterpret_cast<const uint2*>(p + 4 * i);
        w[i] = q.x; w[i + 1] = q.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < W; ++i) w[i] = reinterpret_cast<const uint32_t*>(p)[i];
    }
    const uint32_t m = (1u << W) - 1u;
#pragma unroll
    for (int k = 0; k < 32; ++k) c[k] |= ((w[(k * W) >> 5] >> ((k * W) & 31)) & m) << O;
  }
}

// 32 decoded float32 values of one run (BF16 metadata: code*s + z as one
// FMA; codes become floats exactly via the 2^23 magic), packed f32x2 math.
template <int B>
__device__ __forceinline__ void dq_run32(const uint8_t* payload, int64_t n, int64_t e0, const GroupMeta& m,
                                         bool intlog, float* v) {
  uint32_t c[32];
  load_codes32<B>(payload, n, e0, c);
  if (!intlog) {
#pragma unroll
    for (int k = 0; k < 32; k += 2) {
      float a, b;
      add2(a, b, __uint_as_float(0x4B000000u | c[k]), __uint_as_float(0x4B000000u | c[k + 1]), -8388608.0f,
           -8388608.0f);
      fma2(v[k], v[k + 1], a, b, m.s32, m.s32, m.z32, m.z32);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = __double2float_rn(__dadd_rn(__dmul_rn((double)c[k], m.s64), m.o64));
  }
}

// Codes of elements 8q .. 8q+7 of a 32-element run, from its bit-split plane
// words (unit-major, unit u at w[O .. O + W)), as bytes: byte i of E = code of
// element 8q + 2i, byte i of Od = code of element 8q + 2i + 1.
//   W = 4: the nibble word q, even / odd nibbles masked out;
//   W = 2: the 16 bits of the 8 elements spread to one 2-bit field per nibble
//          (PRMT, then two shift-or-mask steps), even / odd nibbles masked out;
//   W = 1: byte q of the word; its even (odd) bits land on bit 0 (1) of bytes
//          0..3 with one multiply by 1 + 2^6 + 2^12 + 2^18 (the partial
//          products collide only on positions no target bit reads).
// Unit u's bits are then added at bit offset O (no overlap, so + is |).
template <int B>
__device__ __forceinline__ void split_codes8(const uint32_t* w, int q, uint32_t& E, uint32_t& Od) {
  E = 0u;
  Od = 0u;
#pragma unroll
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u), O = unit_off(B, u);
    uint32_t ev, od;
    if (W == 4) {
      const uint32_t x = w[O + q];
      ev = x & 0x0F0F0F0Fu;
      od = (x >> 4) & 0x0F0F0F0Fu;
    } else if (W == 2) {
      uint32_t x = __byte_perm(w[O + (q >> 1)], 0u, (q & 1) ? 0x4342 : 0x4140);  // [0, t_hi, 0, t_lo]
      x = (x | (x << 4)) & 0x0F0F0F0Fu;  // two elements per byte
      x = (x | (x << 2)) & 0x33333333u;  // one element per nibble
      ev = x & 0x03030303u;
      od = (x >> 4) & 0x03030303u;
    } else {  // W == 1
      const uint32_t t = __byte_perm(w[O], 0u, 0x4440 | q);
      ev = ((t & 0x55u) * 0x41041u) & 0x01010101u;
      od = (((t & 0xAAu) * 0x41041u) & 0x02020202u) >> 1;
    }
    E += ev << O;
    Od += od << O;
  }
}

// 32 code values (as 2^23 + code float bits) of one 32-element run from its plane words
// (unit-major: w[O .. O + W) are unit u's words)
template <int B>
__device__ __forceinline__ void run_code_floats(const uint32_t* w, uint32_t* cf) {
  if constexpr (B == 4) {
#pragma unroll
    for (int wd = 0; wd < 4; ++wd) {
      const uint32_t ev = w[wd] & 0x0F0F0F0Fu, od = (w[wd] >> 4) & 0x0F0F0F0Fu;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        cf[8 * wd + 2 * k] = __byte_perm(ev, 0x4B000000u, 0x7650 + k);
        cf[8 * wd + 2 * k + 1] = __byte_perm(od, 0x4B000000u, 0x7650 + k);
      }
    }
  } else if constexpr (B == 8) {
#pragma unroll
    for (int wd = 0; wd < 8; ++wd)
#pragma unroll
      for (int k = 0; k < 4; ++k) cf[4 * wd + k] = __byte_perm(w[wd], 0x4B000000u, 0x7650 + k);
  } else {
    // bit-split widths: per 8 elements, rebuild the even and odd elements'
    // codes as bytes (SWAR, no per-element bit extraction), then one PRMT per
    // element as for B = 4
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t E, Od;
      split_codes8<B>(w, q, E, Od);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        cf[8 * q + 2 * k] = __byte_perm(E, 0x4B000000u, 0x7650 + k);
        cf[8 * q + 2 * k + 1] = __byte_perm(Od, 0x4B000000u, 0x7650 + k);
      }
    }
  }
}

// Substitute the reserved values (imin first, then imax: codec.py:559-561) into
// a lane's 32 decoded run values.  ha / hz: the slot lies in this run (ka, kz
// run-relative).  Registers cannot be indexed by a data-dependent position, so
// the run round-trips through the lane's 16-byte-aligned smem spill row (32
// floats).  QUAD: only the float4 quads holding a slot make the trip, each
// predicated on its own, so a hit lane moves 32 B each way instead of 128 B.
template <bool QUAD>
__device__ __forceinline__ void subst_reserved(float (&v)[32], float* spill, bool ha, int ka, float smin, bool hz,
                                               int kz, float smax) {
  const int qa = ha ? ka >> 2 : -1, qz = hz ? kz >> 2 : -1;
#pragma unroll
  for (int k = 0; k < 32; k += 4)
    if (!QUAD || qa == k / 4 || qz == k / 4)
      *reinterpret_cast<float4*>(spill + k) = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
  if (ha) spill[ka] = smin;
  if (hz) spill[kz] = smax;
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    if (!QUAD || qa == k / 4 || qz == k / 4) {
      const float4 q = *reinterpret_cast<const float4*>(spill + k);
      v[k] = q.x; v[k + 1] = q.y; v[k + 2] = q.z; v[k + 3] = q.w;
    }
  }
}

// Code of one element (generic path, any alignment).
__device__ __forceinline__ uint32_t load_code1(const uint8_t* payload, int64_t n, int64_t e, int B) {
  uint32_t c = 0;
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u), O = unit_off(B, u);
    const uint8_t* p = payload + (n * O) / 8;
    const int64_t bit = e * W;
    uint32_t byte = p[bit >> 3];
    c |= ((byte >> (bit & 7)) & ((1u << W) - 1u)) << O;
  }
  return c;
}

// Element e of a chunk as float32 (generic path).
__device__ __forceinline__ float decode_elem32(const uint8_t* payload, int64_t e, const DecCtx& c) {
  const int64_t grp = e / c.G;
  GroupMeta m = read_meta(payload, grp, c);
  const int idx = (int)(e - grp * c.G);
  if (c.sr) {
    if (idx == m.imax) return m.smax;  // imax written last (codec.py:561)
    if (idx == m.imin) return m.smin;
  }
  return dq32(load_code1(payload, c.n, e, c.B), m, c.intlog);
}
__device__ __forceinline__ double decode_elem64(const uint8_t* payload, int64_t e, const DecCtx& c) {
  const int64_t grp = e / c.G;
  GroupMeta m = read_meta(payload, grp, c);
  const int idx = (int)(e - grp * c.G);
  if (c.sr) {
    if (idx == m.imax) return (double)m.smax;
    if (idx == m.imin) return (double)m.smin;
  }
  return dq64(load_code1(payload, c.n, e, c.B), m, c.intlog);
}

}  // namespace fc2
