// fc2_common.cuh -- device helpers shared by the FlashCommunication-V2 kernels.
//
// Arithmetic contract: SURVEY.md section 8.0 (R1-R15), which restates
// /root/reference/pkg/src/qcomm/codec.py and bfloat16.py.  Every helper
// here cites the reference line it must reproduce bit-for-bit.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/fc2.h"

namespace fc2 {

// ---------------------------------------------------------------------------
// bit-split units, low bits first (codec.py:143-151, 154-162)
// ---------------------------------------------------------------------------

__host__ __device__ constexpr int n_units(int b) {
  return b == 2 ? 1 : b == 3 ? 2 : b == 4 ? 1 : b == 5 ? 2 : b == 6 ? 2 : b == 7 ? 3 : 1;
}
__host__ __device__ constexpr int unit_w(int b, int u) {
  // 2:(2) 3:(2,1) 4:(4) 5:(4,1) 6:(4,2) 7:(4,2,1) 8:(8)
  return b == 2 ? (u == 0 ? 2 : 0)
       : b == 3 ? (u == 0 ? 2 : u == 1 ? 1 : 0)
       : b == 4 ? (u == 0 ? 4 : 0)
       : b == 5 ? (u == 0 ? 4 : u == 1 ? 1 : 0)
       : b == 6 ? (u == 0 ? 4 : u == 1 ? 2 : 0)
       : b == 7 ? (u == 0 ? 4 : u == 1 ? 2 : u == 2 ? 1 : 0)
       : (u == 0 ? 8 : 0);
}
// bit offset of unit u inside a code == cumulative width of earlier units
__host__ __device__ constexpr int unit_off(int b, int u) {
  return u == 0 ? 0 : unit_off(b, u - 1) + unit_w(b, u - 1);
}

// metadata record bytes (codec.py:400-425)
__host__ __device__ constexpr int rec_bytes(bool sr, bool intlog) {
  return intlog ? (sr ? 8 : 2) : (sr ? 12 : 4);
}

// ---------------------------------------------------------------------------
// bfloat16 (bfloat16.py:16-31)
// ---------------------------------------------------------------------------

// float32 -> bf16 bits, RNE via the 0x7FFF bias (bfloat16.py:16-25).  Inputs
// on this path are finite or +-inf; inf maps to 0x7F80 exactly like numpy.
__device__ __forceinline__ uint32_t bf16_bits(float f) {
  uint32_t u = __float_as_uint(f);
  if (f != f) return 0x7FC0u;
  return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}
__device__ __forceinline__ float bf16_val(uint32_t bits) {
  return __uint_as_float(bits << 16);
}

// NaN-propagating min/max (a NaN anywhere poisons the group statistics, which
// is how the encoder detects non-finite input, codec.py:482-483).
__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// ---------------------------------------------------------------------------
// exact per-element code (codec.py:246-256, R8), float64, no contraction
// ---------------------------------------------------------------------------

__device__ __forceinline__ int exact_code(double v, double off, double div, int L) {
  if (!(div > 0.0)) return 0;                       // np.where(scale > 0, q, 0)
  double q = __ddiv_rn(__dsub_rn(v, off), div);      // (rows - offset) / safe
  if (!(q > 0.0)) return 0;                          // copysign(...) <= 0 -> clip 0
  double r = floor(__dadd_rn(q, 0.5));               // floor(|q| + 0.5)
  return r >= (double)L ? L : (int)r;                // clip(., 0, L)
}

// round half away from zero (codec.py:246-248)
__device__ __forceinline__ double rha(double x) {
  double r = floor(__dadd_rn(fabs(x), 0.5));
  return copysign(r, x);
}

// Programmatic dependent launch for the library's kernels: launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, a kernel's CTAs may be
// scheduled while its stream predecessor is still draining its last wave;
// each CTA first lets its own dependents go (launch_dependents) and then waits
// for the predecessor's completion and memory flush (griddepcontrol.wait)
// before touching global memory, so stream semantics are unchanged and only
// the launch latency / ramp overlaps the predecessor's tail.
#ifndef FC2_PDL
#define FC2_PDL 1
#endif
// spin-wait kernels: may start early (one CTA parks behind the predecessor)
// but never release their own dependents early
__device__ __forceinline__ void pdl_wait_only() {
#if FC2_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_enter() {
#if FC2_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
// Host paths that schedule kernels on several streams with event waits (the
// host-resident pipeline, the pipelined two-step) hold a NoPdl guard: their
// launches are plain, so no kernel can start ahead of an event it waits on.
inline int& pdl_off_depth() {
  static thread_local int d = 0;
  return d;
}
struct NoPdl {
  NoPdl() { ++pdl_off_depth(); }
  ~NoPdl() { --pdl_off_depth(); }
};
template <typename K, typename... Args>
inline void launch_pdl(K kern, unsigned grid, unsigned block, int smem, cudaStream_t st, Args... args) {
#if FC2_PDL
  if (pdl_off_depth() > 0) {
    kern<<<grid, block, smem, st>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
#else
  kern<<<grid, block, smem, st>>>(args...);
#endif
}

// (every kernel launched through launch_pdl must begin with pdl_enter or
// pdl_wait_only).  The communicator's spin-wait kernels (k_barrier,
// k_flag_wait / k_flag_signal) use pdl_wait_only: they never release their
// dependents early: a
// dependent grid launched early parks its CTAs in griddepcontrol.wait, and
// behind a kernel that waits for another stream or a peer those parked CTAs
// can take the SM slots that stream / peer needs (a deadlock observed with
// back-to-back pipelined AllReduce calls).

// ---------------------------------------------------------------------------
// fp32 code estimate with a 14-bit fixed-point fraction:
//   y = (v - off) * inv + (0.5 + 8*2^-14) + 512
// lands in [512, 1024) where the float32 ulp is 2^-14, so bits(y) holds
// floor(q + 0.5 + 8u) in bits [14, 22) and the fraction in bits [0, 14).
// When bits [4, 14) are all zero the element is within 8u of a rounding tie
// and is recomputed exactly in float64; the estimate error is < 2.2e-4 < 7.5u,
// so every other element provably gets the reference's float64 code.
// ---------------------------------------------------------------------------

constexpr int kFixBits = 14;
constexpr float kFixC = 0.5f + 8.0f / 16384.0f;
constexpr float kFixMagic = 512.0f;
constexpr float kFixCM = 512.5f + 8.0f / 16384.0f;  // exactly representable
constexpr uint32_t kTieMask = 0x3FF0u;
constexpr float kFoldLimit = 1024.0f;               // |off * inv| bound for the folded form

__device__ __forceinline__ uint32_t fix_est_clamped(float v, float off32, float inv32, float Lh) {
  float d = __fsub_rn(v, off32);
  float f = __fmaf_rn(d, inv32, kFixC);
  f = fminf(fmaxf(f, kFixC), Lh);  // codes may legitimately clip at both ends
  return __float_as_uint(__fadd_rn(f, kFixMagic));
}
__device__ __forceinline__ bool fix_is_tie(uint32_t X) { return (X & kTieMask) == 0u; }

// Fixed-point parameters by fraction width: 16 bits when codes fit 7 bits
// (y in [128, 256), code = byte 2 of bits(y)), 14 bits for 8-bit codes.
template <int FB>
struct Fix;
template <>
struct Fix<14> {
  static constexpr int kBits = 14;
  static constexpr float kC = 0.5f + 8.0f / 16384.0f;
  static constexpr float kM = 512.0f;
  static constexpr float kCM = 512.5f + 8.0f / 16384.0f;
  static constexpr uint32_t kTie = 0x3FF0u;
  static constexpr float kFold = 1024.0f;
};
// 15-bit fraction: y in [256, 512), code in bits [15, 23), fraction bits
// [0, 15); the tie test (bits [4, 15) zero) never touches bit 15, so packed
// f16 zero tests on fraction pairs are exact.
template <>
struct Fix<15> {
  static constexpr int kBits = 15;
  static constexpr float kC = 0.5f + 8.0f / 32768.0f;
  static constexpr float kM = 256.0f;
  static constexpr float kCM = 256.5f + 8.0f / 32768.0f;
  static constexpr uint32_t kTie = 0x7FF0u;
  static constexpr float kFold = 512.0f;
};
// 16-bit fraction (B <= 7): y in [128, 256), code in bits [16, 24) -- a whole
// byte, so plane words are gathered with byte permutes; fraction = low half.
// kFold bounds |nz| for the single-FFMA form y = fma(v, inv, nz + kCM):
// |error| <= 2^-24 (127.5 + 128) + 2^-16 (nz + kCM rounding) + 2^-17 (fma)
// ~ 2.5 ulp of 2^-16, inside the 8-ulp tie window.
template <>
struct Fix<16> {
  static constexpr int kBits = 16;
  static constexpr float kC = 0.5f + 8.0f / 65536.0f;
  static constexpr float kM = 128.0f;
  static constexpr float kCM = 128.5f + 8.0f / 65536.0f;
  static constexpr uint32_t kTie = 0xFFF0u;
  static constexpr float kFold = 128.0f;
};
template <int B>
struct FixFor {
  static constexpr int FB = B <= 7 ? 16 : 15;
};

template <int FB>
__device__ __forceinline__ uint32_t fixq_clamped(float v, float off32, float inv32, float Lh) {
  float d = __fsub_rn(v, off32);
  float f = __fmaf_rn(d, inv32, Fix<FB>::kC);
  f = fminf(fmaxf(f, Fix<FB>::kC), Lh);
  return __float_as_uint(__fadd_rn(f, Fix<FB>::kM));
}

// tie mask bits for a pair of fixed-point words: bit `pp` for X0 and bit
// `16 + pp` for X1 when the fraction is within 8 ulps of a rounding tie
// (FB = 16: the masked fraction can be 0x8000 == -0.0 as f16, so it is
// XOR-ed onto 1.0 first: equal to 1.0 exactly when the masked bits are zero)
template <int FB>
__device__ __forceinline__ uint32_t pair_tie_bits(uint32_t X0, uint32_t X1, int pp) {
  constexpr uint32_t M = Fix<FB>::kTie | (Fix<FB>::kTie << 16);
  if constexpr (FB == 16) {
    // (x & M) ^ 1.0: equal to 1.0 exactly when the masked fraction is zero
    // (the raw masked fraction can be 0x8000 == -0.0, which a zero test would
    // also accept; an |.| < tiny test would flag exact-integer q, which bf16
    // data hits often)
    uint32_t one;  // 1.0 as f16x2, in a register so (x & M) ^ one is one LOP3
    asm("mov.b32 %0, 0x3C003C00;" : "=r"(one));
    uint32_t fr = (__byte_perm(X0, X1, 0x5410) & M) ^ one;
    __half2 h = *reinterpret_cast<const __half2*>(&fr);
    return __heq2_mask(h, __float2half2_rn(1.0f)) & (0x00010001u << pp);
  } else {
    uint32_t fr = __byte_perm(X0, X1, 0x5410) & M;
    __half2 h = *reinterpret_cast<const __half2*>(&fr);
    return __heq2_mask(h, __float2half2_rn(0.0f)) & (0x00010001u << pp);
  }
}

// FB = 16 tie flags with the work on the FMA pipe (the ALU pipe is the
// encoder's bottleneck).  y + kTieShift moves the tie window frac(y) in
// [0, 16] ulp to [0x7BF0, 0x7C00], which is exactly the set of 16-bit
// patterns an ordered f16 compare h >= 65024 (0x7BF0) accepts (0x7C00 = +inf, NaNs and
// negatives compare false) -- so one PRMT + one HFMA2.SAT (tie_ge) test a pair, with no
// masking; exact-integer codes (frac = 0x8008) land on negative f16 and are
// not flagged.  The 1.0 / 0.0 results are summed as r * 2^k into an f16 pair
// that starts at 1024 (HFMA2): pair k of 8 sets bit k of the low byte of each
// half (1024 + v, v < 256, is exact).  tie_bits16 merges the two
// accumulators of a run into the split layout of pair_tie_bits.
constexpr float kTieShift = 31728.0f / 65536.0f;  // 0x7BF0 ulp of 2^-16
// 1.0 where h >= 65024 (0x7BF0) as an ordered f16 compare, else 0.0, on the
// FMA pipe: sat(h - 64992).  Every f16 at or above 65024 is at least 32 above
// 64992 (the ulp there is 32; the difference is exact) and saturates to 1,
// +inf gives 1, NaN flushes to +0, and everything below 65024 gives a result
// <= 0 that saturates to 0 (checked over all 65536 patterns).  Against an
// HSET2 on the ALU pipe: 64 MiB b4 SR encode 20.45 -> 19.92 us, b3 SR
// 22.6 -> 22.1 us.
__device__ __forceinline__ __half2 tie_ge(__half2 h) {
  return __hfma2_sat(h, __half2(__ushort_as_half(0x3C00), __ushort_as_half(0x3C00)),
                     __half2(__ushort_as_half(0xFBEF), __ushort_as_half(0xFBEF)));  // 1.0, -64992
}
__device__ __forceinline__ void add2(float& r0, float& r1, float a0, float a1, float b0, float b1);
__device__ __forceinline__ void tie_acc16(__half2& acc, float y0, float y1, int k) {
  float z0, z1;  // exact: y in [128, 256) on the 2^-16 grid, y + shift < 256
  add2(z0, z1, y0, y1, kTieShift, kTieShift);
  const uint32_t h = __byte_perm(__float_as_uint(z0), __float_as_uint(z1), 0x5410);
  acc = __hfma2(tie_ge(*reinterpret_cast<const __half2*>(&h)), __float2half2_rn((float)(1 << k)), acc);
}
// FB = 15 (B = 8): bit 15 of the low half is the code's LSB, so the same
// window is tested on |h| (the f16 abs ignores bit 15); y + shift carries into
// the code bits harmlessly (y < 511.5 + 8u, the sum stays below 512, exact).
constexpr float kTieShift15 = 31728.0f / 32768.0f;  // 0x7BF0 ulp of 2^-15
__device__ __forceinline__ void tie_acc15(__half2& acc, float y0, float y1, int k) {
  float z0, z1;
  add2(z0, z1, y0, y1, kTieShift15, kTieShift15);
  const uint32_t h = __byte_perm(__float_as_uint(z0), __float_as_uint(z1), 0x5410);
  acc = __hfma2(tie_ge(__habs2(*reinterpret_cast<const __half2*>(&h))), __float2half2_rn((float)(1 << k)), acc);
}
__device__ __forceinline__ uint32_t tie_bits16(const __half2 (&acc)[2]) {
  return __byte_perm(*reinterpret_cast<const uint32_t*>(&acc[0]), *reinterpret_cast<const uint32_t*>(&acc[1]),
                     0x6240);
}

// packed float32x2 arithmetic (sm_100: FFMA2 / FADD2)
__device__ __forceinline__ void fma2(float& r0, float& r1, float a0, float a1, float b0, float b1, float c0,
                                     float c1) {
  asm("{\n\t.reg .b64 a, b, c, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
      "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r0), "=f"(r1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void add2(float& r0, float& r1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r0), "=f"(r1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// ---------------------------------------------------------------------------
// per-group parameters (codec.py:454-474, 512; R6, R7, R13)
// ---------------------------------------------------------------------------

struct GroupParams {
  double off;        // code offset: zero (BF16) or -z*s_eff (INT_LOG)
  double div;        // code divisor: scale (BF16) or s_eff (INT_LOG); 0 => codes 0
  float off32;       // fast-path float copies
  float inv32;
  float nz;          // -off32 * inv32 (folded form: q ~ fma(v, inv32, nz))
  bool fold;         // |nz| small enough for the folded form
  bool exact;        // range too small/large for the fp32 estimate: exact f64 for all
  uint32_t sz;       // BF16: scale_bits | zero_bits << 16 ; INT_LOG: (u8)si | (u8)zi << 8
};

__device__ __forceinline__ GroupParams group_params(double zero, double vmax, int L, bool intlog,
                                                    int theta, const double* __restrict__ lut,
                                                    int32_t* err) {
  GroupParams p;
  double scale = __ddiv_rn(__dsub_rn(vmax, zero), (double)L);  // codec.py:512
  if (!intlog) {
    p.off = zero;
    p.div = scale;
    p.sz = bf16_bits(__double2float_rn(scale)) | (bf16_bits(__double2float_rn(zero)) << 16);
  } else {
    int si = -128;
    if (scale > 0.0) {
      double t = __dmul_rn(log2(scale), (double)theta);
      double ft = fabs(t) - floor(fabs(t));
      if (fabs(ft - 0.5) < 1e-9 && err) atomicOr(err, FC2_ERR_LOG2_TIE);
      double r = rha(t);
      r = r < -128.0 ? -128.0 : (r > 127.0 ? 127.0 : r);
      si = (int)r;
    }
    double s_eff = si == -128 ? 0.0 : lut[si + 128];               // codec.py:468
    int zi = 0;
    if (s_eff > 0.0) {
      double r = rha(__ddiv_rn(-zero, s_eff));                      // codec.py:471
      r = r < -128.0 ? -128.0 : (r > 127.0 ? 127.0 : r);
      zi = (int)r;
    }
    p.off = __dmul_rn(-(double)zi, s_eff);                          // codec.py:473
    p.div = s_eff;
    p.sz = (uint32_t)(uint8_t)(int8_t)si | ((uint32_t)(uint8_t)(int8_t)zi << 8);
  }
  if (p.div > 0.0) {
    p.exact = !(p.div >= 1e-32 && p.div <= 1e28);
    p.off32 = __double2float_rn(p.off);
    p.inv32 = __frcp_rn(__double2float_rn(p.div));
    if (p.exact) { p.off32 = 0.f; p.inv32 = 0.f; }
  } else {
    p.exact = false;
    p.off32 = 0.f;
    p.inv32 = 0.f;
  }
  p.nz = -__fmul_rn(p.off32, p.inv32);
  p.fold = !p.exact && fabsf(p.nz) <= kFoldLimit;
  return p;
}

// ---------------------------------------------------------------------------
// misc
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// lanes per group of the lane-per-group encoder: each lane owns at most
// FC2_ENC_EPL consecutive elements of its group (host and device agree)
#ifndef FC2_ENC_EPL
#define FC2_ENC_EPL 128
#endif
__host__ __device__ constexpr int enc_lpg(int G) { return G > FC2_ENC_EPL ? G / FC2_ENC_EPL : 1; }
// small chunks (less than one resident wave of bandwidth tiles): one 32-element
// run per lane, so each warp's serial work (and the launch's latency) shrinks
// by G / 32 at the cost of a few shuffles per group
__host__ __device__ constexpr int enc_lpg_small(int G) { return G / 32 > 0 ? G / 32 : 1; }
#ifndef FC2_ENC_SMALL_TILES
#define FC2_ENC_SMALL_TILES 592  // bandwidth tiles below which the small-chunk shape is used (148 SMs x 4;
                                 // measured crossover ~2.5 Mi elements at g = 128)
#endif

// store nbytes (<= 12) from words[]; widest stores the alignment allows
__device__ __forceinline__ void store_record(uint8_t* p, const uint32_t* w, int nbytes) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if ((a & 3u) == 0 && (nbytes & 3) == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (i < nbytes / 4) reinterpret_cast<uint32_t*>(p)[i] = w[i];
  } else if ((a & 1u) == 0 && (nbytes & 1) == 0) {
#pragma unroll
    for (int i = 0; i < 6; ++i)
      if (i < nbytes / 2) reinterpret_cast<uint16_t*>(p)[i] = (uint16_t)(w[i >> 1] >> ((i & 1) * 16));
  } else {
#pragma unroll
    for (int i = 0; i < 12; ++i)
      if (i < nbytes) p[i] = (uint8_t)(w[i >> 2] >> ((i & 3) * 8));
  }
}

__device__ __forceinline__ void load_record(const uint8_t* p, uint32_t* w, int nbytes) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p);
  w[0] = w[1] = w[2] = 0;
  if ((a & 3u) == 0 && (nbytes & 3) == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (i < nbytes / 4) w[i] = reinterpret_cast<const uint32_t*>(p)[i];
  } else if ((a & 1u) == 0 && (nbytes & 1) == 0) {
#pragma unroll
    for (int i = 0; i < 6; ++i)
      if (i < nbytes / 2) w[i >> 1] |= (uint32_t)reinterpret_cast<const uint16_t*>(p)[i] << ((i & 1) * 16);
  } else {
#pragma unroll
    for (int i = 0; i < 12; ++i)
      if (i < nbytes) w[i >> 2] |= (uint32_t)p[i] << ((i & 3) * 8);
  }
}

}  // namespace fc2
