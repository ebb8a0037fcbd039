// fc2_encode.cuh -- group quantizer cores (encode_chunk, codec.py:477-519).
//
// Two implementations of the same contract:
//  * encode_lane<>: the fast path.  One lane owns 32 consecutive elements in
//    registers; a group of G in {32,64,128,256} spans G/32 adjacent lanes
//    (shuffle reductions).  Statistics use packed bf16x2 min/max when the
//    values are bf16, codes use the fp32 fixed-point estimate with an exact
//    float64 recompute of near-tie elements.  Packed plane words are built in
//    registers and stored with 4/8/16-byte stores.
//  * generic_encode_group(): warp-per-group, every element in exact float64;
//    any group size that is a multiple of 8, any input type (bf16/f32/f64).
#pragma once

#include "fc2_common.cuh"

namespace fc2 {

// ------------------------------------------------------------------------
// value containers for one lane's 32 elements
// ------------------------------------------------------------------------

// XOR swizzle of 16-byte chunks in a warp's staging tile: conflict-free for
// the coalesced fill (chunk c = lane + 32 j) and for the per-lane read-back
// (chunks CPL*lane .. CPL*lane + CPL - 1); CPL = chunks per lane.
template <int CPL>
__device__ __forceinline__ int swz(int c) { return c ^ ((c >> 3) & (CPL - 1)); }

struct Bf16Vals {  // w[k] = elements (2k, 2k+1) as packed bf16x2
  uint32_t w[16];
  const uint8_t* st;  // the warp's staging tile (for rare dynamic reads)
  __device__ __forceinline__ float get(int k) const {
    return (k & 1) ? __uint_as_float(w[k >> 1] & 0xFFFF0000u) : __uint_as_float(w[k >> 1] << 16);
  }
  __device__ __forceinline__ float get_dyn(int k) const {  // rare path: re-read smem
    const int c = 4 * (int)lane_id() + (k >> 3);
    uint32_t b = *reinterpret_cast<const uint16_t*>(st + swz<4>(c) * 16 + (k & 7) * 2);
    return __uint_as_float(b << 16);
  }
  // min/max (RTN) with NaN propagation
  __device__ __forceinline__ void minmax(float& mn, float& mx) const {
    __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&w[0]), b = a;
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(&w[k]);
      a = __hmin2_nan(a, x);
      b = __hmax2_nan(b, x);
    }
    mn = fmin_nan(__low2float(a), __high2float(a));
    mx = fmax_nan(__low2float(b), __high2float(b));
  }
  // two smallest / two largest (multiset order statistics) with NaN propagation
  __device__ __forceinline__ void top2(float& mn1, float& mn2, float& mx1, float& mx2) const {
    const __nv_bfloat162 pinf = __floats2bfloat162_rn(__int_as_float(0x7f800000), __int_as_float(0x7f800000));
    const __nv_bfloat162 ninf = __floats2bfloat162_rn(__int_as_float(0xff800000), __int_as_float(0xff800000));
    __nv_bfloat162 a1 = *reinterpret_cast<const __nv_bfloat162*>(&w[0]), a2 = pinf;
    __nv_bfloat162 b1 = a1, b2 = ninf;
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(&w[k]);
      a2 = __hmin2_nan(a2, __hmax2_nan(a1, x));
      a1 = __hmin2_nan(a1, x);
      b2 = __hmax2_nan(b2, __hmin2_nan(b1, x));
      b1 = __hmax2_nan(b1, x);
    }
    float l1 = __low2float(a1), h1 = __high2float(a1), l2 = __low2float(a2), h2 = __high2float(a2);
    mn1 = fmin_nan(l1, h1);
    mn2 = fmin_nan(fmax_nan(l1, h1), fmin_nan(l2, h2));
    l1 = __low2float(b1); h1 = __high2float(b1); l2 = __low2float(b2); h2 = __high2float(b2);
    mx1 = fmax_nan(l1, h1);
    mx2 = fmax_nan(fmin_nan(l1, h1), fmax_nan(l2, h2));
  }
  // first k with element k == m (float equality: -0 == +0, codec.py:261-262), 64 if none
  __device__ __forceinline__ int first_eq(float m) const {
    __nv_bfloat162 mm = __float2bfloat162_rn(m);  // m is a bf16 value: exact
    uint32_t msk = 0;  // bit k: element 2k matches; bit 16+k: element 2k+1 matches
#pragma unroll
    for (int k = 0; k < 16; ++k)
      msk |= __heq2_mask(*reinterpret_cast<const __nv_bfloat162*>(&w[k]), mm) & (0x00010001u << k);
    const uint32_t lo = msk & 0xFFFFu, hi = msk >> 16;
    const int fl = lo ? 2 * (__ffs(lo) - 1) : 64;
    const int fh = hi ? 2 * (__ffs(hi) - 1) + 1 : 64;
    return min(fl, fh);
  }
  __device__ __forceinline__ void pair(int k, float& a, float& b) const {
    a = __uint_as_float(w[k] << 16);
    b = __uint_as_float(w[k] & 0xFFFF0000u);
  }
};

struct F32Vals {
  float f[32];
  const uint8_t* st;  // staging tile (cp.async fill) or nullptr
  const float* spill; // per-lane copy of f[] in smem when st == nullptr
  __device__ __forceinline__ float get(int k) const { return f[k]; }
  __device__ __forceinline__ float get_dyn(int k) const {  // rare path: re-read smem
    if (st) {
      const int c = 8 * (int)lane_id() + (k >> 2);
      return *reinterpret_cast<const float*>(st + swz<8>(c) * 16 + (k & 3) * 4);
    }
    return spill[k];
  }
  __device__ __forceinline__ void minmax(float& mn, float& mx) const {
    mn = f[0]; mx = f[0];
#pragma unroll
    for (int k = 1; k < 32; ++k) { mn = fmin_nan(mn, f[k]); mx = fmax_nan(mx, f[k]); }
  }
  __device__ __forceinline__ void top2(float& mn1, float& mn2, float& mx1, float& mx2) const {
    mn1 = f[0]; mx1 = f[0];
    mn2 = __int_as_float(0x7f800000); mx2 = __int_as_float(0xff800000);
#pragma unroll
    for (int k = 1; k < 32; ++k) {
      float x = f[k];
      mn2 = fmin_nan(mn2, fmax_nan(mn1, x));
      mn1 = fmin_nan(mn1, x);
      mx2 = fmax_nan(mx2, fmin_nan(mx1, x));
      mx1 = fmax_nan(mx1, x);
    }
  }
  __device__ __forceinline__ int first_eq(float m) const {
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k) r |= (f[k] == m ? 1u : 0u) << k;
    return r ? __ffs(r) - 1 : 64;
  }
  __device__ __forceinline__ void pair(int k, float& a, float& b) const {
    a = f[2 * k];
    b = f[2 * k + 1];
  }
};

// ------------------------------------------------------------------------
// packed plane words for one lane (32 codes): unit u has unit_w(B,u) words
// ------------------------------------------------------------------------

template <int B>
struct LaneWords {
  static constexpr int NU = n_units(B);
  uint32_t w[B];  // words of unit 0, then unit 1, ... (sum of widths == B words)
  static constexpr __host__ __device__ int base(int u) { return unit_off(B, u); }
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int i = 0; i < B; ++i) w[i] = 0;
  }
  // insert code bits from the fixed-point word X (code in bits [kFixBits, kFixBits+8))
  __device__ __forceinline__ void put_fix(int k, uint32_t X) {
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int W = unit_w(B, u), O = unit_off(B, u);
      const int wi = (k * W) >> 5, pos = (k * W) & 31;
      const uint32_t m = (1u << W) - 1u;
      const int sh = pos - (kFixBits + O);
      uint32_t t = sh >= 0 ? (X << sh) : (X >> (-sh));
      w[base(u) + wi] |= t & (m << pos);
    }
  }
  // same with an explicit fraction width FB (code in bits [FB, FB+8))
  template <int FB>
  __device__ __forceinline__ void put_fixb(int k, uint32_t X, int u0 = 0) {
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      if (u < u0) continue;
      const int W = unit_w(B, u), O = unit_off(B, u);
      const int wi = (k * W) >> 5, pos = (k * W) & 31;
      const uint32_t m = (1u << W) - 1u;
      const int sh = pos - (FB + O);
      uint32_t t = sh >= 0 ? (X << sh) : (X >> (-sh));
      w[base(u) + wi] |= t & (m << pos);
    }
  }
  // overwrite element k (dynamic) with code c
  __device__ __forceinline__ void patch(int k, int c) {
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int W = unit_w(B, u), O = unit_off(B, u);
      const uint32_t m = (1u << W) - 1u;
      const int wi = (k * W) >> 5, pos = (k * W) & 31;
      const uint32_t bits = ((uint32_t)c >> O) & m;
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (j == wi) w[base(u) + j] = (w[base(u) + j] & ~(m << pos)) | (bits << pos);
    }
  }
};

// store W words at p (p is 4-byte aligned); vectorize when aligned
template <int W>
__device__ __forceinline__ void store_words(uint8_t* p, const uint32_t* w) {
  uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if constexpr (W % 4 == 0) {
    if ((a & 15u) == 0) {
#pragma unroll
      for (int i = 0; i < W; i += 4)
        *reinterpret_cast<uint4*>(p + 4 * i) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
      return;
    }
  }
  if constexpr (W % 2 == 0) {
    if ((a & 7u) == 0) {
#pragma unroll
      for (int i = 0; i < W; i += 2) *reinterpret_cast<uint2*>(p + 4 * i) = make_uint2(w[i], w[i + 1]);
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < W; ++i) reinterpret_cast<uint32_t*>(p)[i] = w[i];
}

struct EncCtx {
  int64_t n;          // chunk length (elements)
  int64_t meta_off;   // byte offset of the metadata section (n*B/8)
  int intlog, theta;
  const double* lut;
  int32_t* err;
};

// ------------------------------------------------------------------------
// fast path: one lane = 32 consecutive elements of one chunk
// ------------------------------------------------------------------------

template <int B, bool SR, int G, class V, class StoreFn>
__device__ __forceinline__ void encode_lane(const V& v, bool active, int64_t e0, const EncCtx& cx,
                                            StoreFn&& store) {
  static_assert(G == 32 || G == 64 || G == 128 || G == 256, "fast path group sizes");
  constexpr int TPG = G / 32;   // lanes per group
  constexpr int L = (1 << B) - 1;
  const int lig = (int)(lane_id() % TPG);  // lane index inside the group

  // ---- group statistics (R4 / R5) --------------------------------------
  float mn1, mn2 = 0.f, mx1, mx2 = 0.f;
  if constexpr (SR) {
    v.top2(mn1, mn2, mx1, mx2);
  } else {
    v.minmax(mn1, mx1);
  }
#pragma unroll
  for (int o = 1; o < TPG; o <<= 1) {
    float a1 = __shfl_xor_sync(0xffffffffu, mn1, o);
    float b1 = __shfl_xor_sync(0xffffffffu, mx1, o);
    if constexpr (SR) {
      float a2 = __shfl_xor_sync(0xffffffffu, mn2, o);
      float b2 = __shfl_xor_sync(0xffffffffu, mx2, o);
      mn2 = fmin_nan(fmax_nan(mn1, a1), fmin_nan(mn2, a2));
      mx2 = fmax_nan(fmin_nan(mx1, b1), fmax_nan(mx2, b2));
    }
    mn1 = fmin_nan(mn1, a1);
    mx1 = fmax_nan(mx1, b1);
  }
  const bool finite = isfinite(mn1) && isfinite(mx1);
  if (active && !finite && lig == 0) atomicOr(cx.err, FC2_ERR_NONFINITE);

  // ---- spike positions: first argmin / argmax, all-equal -> (0,1) -------
  int imin = 0, imax = 1;
  uint32_t smin_bits = 0, smax_bits = 0;
  if constexpr (SR) {
    const int li = v.first_eq(mn1), la = v.first_eq(mx1);
    int fi = li < 32 ? lig * 32 + li : 1 << 20;
    int fa = la < 32 ? lig * 32 + la : 1 << 20;
#pragma unroll
    for (int o = 1; o < TPG; o <<= 1) {
      fi = min(fi, __shfl_xor_sync(0xffffffffu, fi, o));
      fa = min(fa, __shfl_xor_sync(0xffffffffu, fa, o));
    }
    if (fi >= G) fi = 0;  // only with NaN input (already flagged)
    if (fa >= G) fa = 1;
    if (fi == fa) { fi = 0; fa = 1; }
    imin = fi; imax = fa;
    // reserved values: bf16 of the element itself (codec.py:492-493).  Equal
    // to bf16(mn1) unless the extreme is a signed zero; then fetch the element.
    float sv_min = mn1, sv_max = mx1;
    const bool zero_case = (mn1 == 0.f) || (mx1 == 0.f) || (mn1 == mx1);
    if (__any_sync(0xffffffffu, zero_case)) {
      const int base_lane = (int)lane_id() - lig;
      float cmin = (lig == (imin >> 5)) ? v.get_dyn(imin & 31) : 0.f;
      float cmax = (lig == (imax >> 5)) ? v.get_dyn(imax & 31) : 0.f;
      float gmin = __shfl_sync(0xffffffffu, cmin, base_lane + (imin >> 5));
      float gmax = __shfl_sync(0xffffffffu, cmax, base_lane + (imax >> 5));
      if (zero_case) { sv_min = gmin; sv_max = gmax; }
    }
    smin_bits = bf16_bits(sv_min);
    smax_bits = bf16_bits(sv_max);
  }
  const float zf = SR ? mn2 : mn1, vf = SR ? mx2 : mx1;

  // ---- per-group parameters (R6, R7, R13) -------------------------------
  GroupParams p = group_params((double)zf, (double)vf, L, cx.intlog != 0, cx.theta, cx.lut,
                               active && lig == 0 ? cx.err : nullptr);

  // ---- codes --------------------------------------------------------------
  LaneWords<B> lw;
  lw.clear();
  uint32_t tie = 0;
  if (!cx.intlog) {
    // warp-uniform choice between the folded form q ~ fma(v, inv, -off*inv)
    // (2 packed ops per pair) and the explicit v - off form (3 packed ops)
    if (__all_sync(0xffffffffu, p.fold || p.exact || !active)) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        float a, b, t0, t1, y0, y1;
        v.pair(k, a, b);
        fma2(t0, t1, a, b, p.inv32, p.inv32, p.nz, p.nz);
        add2(y0, y1, t0, t1, kFixCM, kFixCM);
        const uint32_t X0 = __float_as_uint(y0), X1 = __float_as_uint(y1);
        tie |= (fix_is_tie(X0) ? 1u : 0u) << (2 * k);
        tie |= (fix_is_tie(X1) ? 1u : 0u) << (2 * k + 1);
        lw.put_fix(2 * k, X0);
        lw.put_fix(2 * k + 1, X1);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        float a, b, d0, d1, t0, t1, y0, y1;
        v.pair(k, a, b);
        add2(d0, d1, a, b, -p.off32, -p.off32);
        fma2(t0, t1, d0, d1, p.inv32, p.inv32, kFixC, kFixC);
        add2(y0, y1, t0, t1, kFixMagic, kFixMagic);
        const uint32_t X0 = __float_as_uint(y0), X1 = __float_as_uint(y1);
        tie |= (fix_is_tie(X0) ? 1u : 0u) << (2 * k);
        tie |= (fix_is_tie(X1) ? 1u : 0u) << (2 * k + 1);
        lw.put_fix(2 * k, X0);
        lw.put_fix(2 * k + 1, X1);
      }
    }
  } else {
    const float Lh = (float)L + 0.5f;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      uint32_t X = fix_est_clamped(v.get(k), p.off32, p.inv32, Lh);
      tie |= (fix_is_tie(X) ? 1u : 0u) << k;
      lw.put_fix(k, X);
    }
  }
  if (p.exact) tie = 0xffffffffu;
  if (!active) tie = 0;
  while (tie) {  // exact float64 recompute of near-tie elements (rare)
    const int k = __ffs(tie) - 1;
    tie &= tie - 1;
    lw.patch(k, exact_code((double)v.get_dyn(k), p.off, p.div, L));
  }
  if constexpr (SR) {  // reserved slots are quantized as 0.0 (codec.py:494-496)
    int sc;
    const uint32_t Xs = fix_est_clamped(0.0f, p.off32, p.inv32, (float)L + 0.5f);
    if (p.exact || fix_is_tie(Xs)) sc = exact_code(0.0, p.off, p.div, L);
    else sc = (int)((Xs >> kFixBits) & (uint32_t)L);
    if (lig == (imin >> 5)) lw.patch(imin & 31, sc);
    if (lig == (imax >> 5)) lw.patch(imax & 31, sc);
  }

  // ---- metadata record (R10) --------------------------------------------
  uint32_t rec[3];
  int rb;
  if (!cx.intlog) {
    rec[0] = p.sz;
    if constexpr (SR) {
      rec[1] = smin_bits | (smax_bits << 16);
      rec[2] = (__float_as_uint((float)imin) >> 16) | (__float_as_uint((float)imax) & 0xFFFF0000u);
      rb = 12;
    } else {
      rb = 4;
    }
  } else {
    if constexpr (SR) {
      rec[0] = (p.sz & 0xFFFFu) | (smin_bits << 16);
      rec[1] = smax_bits | ((uint32_t)imin << 16) | ((uint32_t)imax << 24);
      rb = 8;
    } else {
      rec[0] = p.sz & 0xFFFFu;
      rb = 2;
    }
  }
  if (active) store(lw.w, e0, lig == 0, (e0 / G) * rb, rec, rb);
}

// ------------------------------------------------------------------------
// generic path: one warp = one group, exact float64 throughout
// ------------------------------------------------------------------------

template <typename T>
__device__ __forceinline__ double load_elem(const T* x, int64_t i, int64_t n_valid);
template <>
__device__ __forceinline__ double load_elem<__nv_bfloat16>(const __nv_bfloat16* x, int64_t i, int64_t nv) {
  return i < nv ? (double)__bfloat162float(x[i]) : 0.0;
}
template <>
__device__ __forceinline__ double load_elem<float>(const float* x, int64_t i, int64_t nv) {
  return i < nv ? (double)x[i] : 0.0;
}
template <>
__device__ __forceinline__ double load_elem<double>(const double* x, int64_t i, int64_t nv) {
  return i < nv ? x[i] : 0.0;
}

// merge (value, index, second) triples: first occurrence wins ties
__device__ __forceinline__ void merge_min(double& v1, int& i1, double& v2, double o1, int oi, double o2) {
  if (o1 < v1 || (o1 == v1 && oi < i1)) {
    v2 = fmin(v1, o2);
    v1 = o1;
    i1 = oi;
  } else {
    v2 = fmin(v2, o1);
  }
}
__device__ __forceinline__ void merge_max(double& v1, int& i1, double& v2, double o1, int oi, double o2) {
  if (o1 > v1 || (o1 == v1 && oi < i1)) {
    v2 = fmax(v1, o2);
    v1 = o1;
    i1 = oi;
  } else {
    v2 = fmax(v2, o1);
  }
}

// Destination list: the same payload bytes go to every pointer (one for a
// plain encode, N for the stage-2 gather push of the two-step AllReduce).
struct OutList {
  uint8_t* p[8];
  int nd;
};

__device__ __forceinline__ void out_record(const OutList& o, int64_t off, const uint32_t* w, int nb) {
  for (int d = 0; d < o.nd; ++d) store_record(o.p[d] + off, w, nb);
}

// Encode group `gi` of a chunk with one full warp.  `ld(i)` returns element i
// of the chunk as a double (zero padding included).
// est: codes from the fp32 fixed-point estimate with the exact float64
// recompute only for near ties (the fast kernels' contract, same bits); off:
// every code in float64.
template <class Loader>
__device__ void generic_encode_group(const Loader& ld, const OutList& out, int64_t n, int64_t gi,
                                     int B, int G, bool sr, const EncCtx& cx, bool est);
template <class Loader>
__device__ void generic_encode_group(const Loader& ld, const OutList& out, int64_t n, int64_t gi,
                                     int B, int G, bool sr, const EncCtx& cx) {
  generic_encode_group(ld, out, n, gi, B, G, sr, cx, false);
}
template <class Loader>
__device__ void generic_encode_group(const Loader& ld, const OutList& out, int64_t n, int64_t gi,
                                     int B, int G, bool sr, const EncCtx& cx, bool est) {
  const int lane = (int)lane_id();
  const int L = (1 << B) - 1;
  const int64_t g0 = gi * (int64_t)G;
  double mn1 = INFINITY, mn2 = INFINITY, mx1 = -INFINITY, mx2 = -INFINITY;
  int i1 = 1 << 30, j1 = 1 << 30;
  bool bad = false;
  for (int e = lane; e < G; e += 32) {
    double v = ld(g0 + e);
    if (!isfinite(v)) bad = true;
    merge_min(mn1, i1, mn2, v, e, INFINITY);
    merge_max(mx1, j1, mx2, v, e, -INFINITY);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    double a1 = __shfl_xor_sync(0xffffffffu, mn1, o), a2 = __shfl_xor_sync(0xffffffffu, mn2, o);
    int ai = __shfl_xor_sync(0xffffffffu, i1, o);
    double b1 = __shfl_xor_sync(0xffffffffu, mx1, o), b2 = __shfl_xor_sync(0xffffffffu, mx2, o);
    int bi = __shfl_xor_sync(0xffffffffu, j1, o);
    merge_min(mn1, i1, mn2, a1, ai, a2);
    merge_max(mx1, j1, mx2, b1, bi, b2);
  }
  bad = __any_sync(0xffffffffu, bad);
  if (bad) {
    if (lane == 0) atomicOr(cx.err, FC2_ERR_NONFINITE);
    return;
  }
  double zero, vmax;
  int imin = 0, imax = 1;
  uint32_t smin_bits = 0, smax_bits = 0;
  if (sr) {
    imin = i1; imax = j1;
    if (imin == imax) { imin = 0; imax = 1; }
    // spike values are the elements themselves (codec.py:492-493)
    smin_bits = bf16_bits(__double2float_rn(ld(g0 + imin)));
    smax_bits = bf16_bits(__double2float_rn(ld(g0 + imax)));
    zero = mn2; vmax = mx2;  // shrunk range == 2nd order statistics (codec.py:269-275)
  } else {
    zero = mn1; vmax = mx1;
  }
  GroupParams p = group_params(zero, vmax, L, cx.intlog != 0, cx.theta, cx.lut, lane == 0 ? cx.err : nullptr);
  const int sc = sr ? exact_code(0.0, p.off, p.div, L) : 0;
  const bool fast = est && !p.exact;
  const float Lh = (float)L + 0.5f;
  // codes: lane handles runs of 8 consecutive elements -> W bytes per unit
  const int nu = n_units(B);
  for (int e = lane * 8; e < G; e += 256) {
    int c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int idx = e + j;
      if (sr && (idx == imin || idx == imax)) {
        c[j] = sc;
      } else {
        const double v = ld(g0 + idx);
        if (fast) {  // estimate within 2.5 ulp of 2^-14; near ties go float64
          const uint32_t X = fix_est_clamped((float)v, p.off32, p.inv32, Lh);
          c[j] = fix_is_tie(X) ? exact_code(v, p.off, p.div, L) : (int)((X >> kFixBits) & 0xFFu);
        } else {
          c[j] = exact_code(v, p.off, p.div, L);
        }
      }
    }
    for (int u = 0; u < nu; ++u) {
      const int W = unit_w(B, u), O = unit_off(B, u);
      uint64_t bits = 0;  // 8 codes * W bits = W bytes
#pragma unroll
      for (int j = 0; j < 8; ++j) bits |= (uint64_t)(((uint32_t)c[j] >> O) & ((1u << W) - 1u)) << (j * W);
      uint32_t w2[2] = {(uint32_t)bits, (uint32_t)(bits >> 32)};
      out_record(out, (n * O) / 8 + ((g0 + e) * W) / 8, w2, W);
    }
  }
  if (lane == 0) {
    uint32_t rec[3];
    int rb;
    if (!cx.intlog) {
      rec[0] = p.sz;
      rb = 4;
      if (sr) {
        rec[1] = smin_bits | (smax_bits << 16);
        rec[2] = (__float_as_uint((float)imin) >> 16) | (__float_as_uint((float)imax) & 0xFFFF0000u);
        rb = 12;
      }
    } else {
      if (sr) {
        rec[0] = (p.sz & 0xFFFFu) | (smin_bits << 16);
        rec[1] = smax_bits | ((uint32_t)imin << 16) | ((uint32_t)imax << 24);
        rb = 8;
      } else {
        rec[0] = p.sz & 0xFFFFu;
        rb = 2;
      }
    }
    out_record(out, cx.meta_off + gi * rb, rec, rb);
  }
}

}  // namespace fc2
