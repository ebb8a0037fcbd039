// fc2_reduce_group.cuh -- two-step middle stage, lane-per-group
// (collectives.py:291-311): decode the N packed copies of one shard, sum in
// float32 in source order from +0.0, re-encode the sum, push the packed shard
// to every destination.
//
// Warp tile = 32 groups of the shard; lane l owns group l.  Per 32-element run
// the lane loads the codes of all sources at once (memory-level parallelism),
// decodes them in packed fp32x2 and accumulates in registers; reserved spike
// slots are patched through the lane's own region of the f32 tile (which then
// receives the finished sums).  The f32 tile feeds the same lane-per-group
// encoder structure as the bf16 path (statistics, spike search, fixed-point
// codes with exact near-tie recompute, smem output stage), and the copy-out
// writes the packed shard to all destinations (NVLink peer stores in the SPMD
// path).
#pragma once

#include "fc2_decode.cuh"
#include "fc2_encode_group.cuh"

namespace fc2 {

constexpr int kRedMaxSrc = 8;

struct TopF {
  float a1, a2, b1, b2;
};

template <bool SR>
__device__ __forceinline__ void topf_add(TopF& s, float x) {
  if constexpr (SR) {
    s.a2 = fmin_nan(s.a2, fmax_nan(s.a1, x));
    s.b2 = fmax_nan(s.b2, fmin_nan(s.b1, x));
  }
  s.a1 = fmin_nan(s.a1, x);
  s.b1 = fmax_nan(s.b1, x);
}

template <bool SR>
__device__ __forceinline__ void topf_merge(TopF& s, const TopF& o) {
  if constexpr (SR) {
    s.a2 = fmin_nan(fmax_nan(s.a1, o.a1), fmin_nan(s.a2, o.a2));
    s.b2 = fmax_nan(fmin_nan(s.b1, o.b1), fmax_nan(s.b2, o.b2));
  }
  s.a1 = fmin_nan(s.a1, o.a1);
  s.b1 = fmax_nan(s.b1, o.b1);
}

// pass 3 for the f32 tile (pairs come straight from the chunk, no unpack)
template <int B, int G, int MODE>
__device__ __forceinline__ void quant_runs_f32(const uint8_t* ist, uint8_t* ost, const GroupParams& p, float Lh,
                                               bool active) {
  using IT = GTile<float, G>;
  constexpr int RUNS = G / 32;
  constexpr int FB = FixFor<B>::FB;
  using FX = Fix<FB>;
  const int lane = (int)lane_id();
  constexpr int L = (1 << B) - 1;
#pragma unroll 1
  for (int r = 0; r < RUNS; ++r) {
    LaneWords<B> lw;
    lw.clear();
    uint32_t tmj[2] = {0u, 0u};
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // 8 chunks of 4 floats = 32 elements
      uint32_t& tm = tmj[j & 1];
      const float4 q = *reinterpret_cast<const float4*>(ist + IT::in_pos(lane, 8 * r + j) * 16);
      const float vv[4] = {q.x, q.y, q.z, q.w};
      uint32_t X[4];
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const float a = vv[2 * pp], b = vv[2 * pp + 1];
        float y0, y1;
        if constexpr (MODE == 0) {
          float t0, t1;
          fma2(t0, t1, a, b, p.inv32, p.inv32, p.nz, p.nz);
          add2(y0, y1, t0, t1, FX::kCM, FX::kCM);
        } else if constexpr (MODE == 1) {
          float d0, d1, t0, t1;
          add2(d0, d1, a, b, -p.off32, -p.off32);
          fma2(t0, t1, d0, d1, p.inv32, p.inv32, FX::kC, FX::kC);
          add2(y0, y1, t0, t1, FX::kM, FX::kM);
        } else {
          y0 = __uint_as_float(fixq_clamped<FB>(a, p.off32, p.inv32, Lh));
          y1 = __uint_as_float(fixq_clamped<FB>(b, p.off32, p.inv32, Lh));
        }
        X[2 * pp] = __float_as_uint(y0);
        X[2 * pp + 1] = __float_as_uint(y1);
        tm |= pair_tie_bits<FB>(X[2 * pp], X[2 * pp + 1], 2 * j + pp);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) lw.template put_fixb<FB>(4 * j + e, X[e], 0);
    }
#pragma unroll
    for (int u = 0; u < n_units(B); ++u) {
      const int W = unit_w(B, u);
      uint8_t* base = ost + OutStage<B, G>::off(u);
      const uint32_t* w = lw.w + LaneWords<B>::base(u);
      if (W == 1) stage_words<G, 1>(base, lane, r, w);
      else if (W == 2) stage_words<G, 2>(base, lane, r, w);
      else if (W == 4) stage_words<G, 4>(base, lane, r, w);
      else stage_words<G, 8>(base, lane, r, w);
    }
    // split layout: bit i < 16 -> element 2i, bit 16 + i -> element 2i + 1
    uint32_t tm = (p.exact ? 0xffffffffu : (tmj[0] | tmj[1])) & (active ? 0xffffffffu : 0u);
    while (tm) {
      const int k = __ffs(tm) - 1;
      tm &= tm - 1;
      const int e = 32 * r + (k < 16 ? 2 * k : 2 * (k - 16) + 1);
      const float v = *reinterpret_cast<const float*>(ist + IT::in_pos(lane, e >> 2) * 16 + (e & 3) * 4);
      stage_patch<B, G>(ost, lane, e, exact_code((double)v, p.off, p.div, L));
    }
  }
}

// encode the lane's group from the f32 tile; packed bytes go to every
// destination in `outs` (same layout at each)
template <int B, bool SR, int G>
__device__ __forceinline__ void encode_tile_f32(const uint8_t* ist, uint8_t* ost, bool active, int64_t g_abs,
                                                const EncCtx& cx, uint8_t* const* outs, int nout, int64_t tile_g0,
                                                int ng) {
  using IT = GTile<float, G>;
  constexpr int L = (1 << B) - 1;
  constexpr int RUNS = G / 32;
  constexpr int FB = FixFor<B>::FB;
  using FX = Fix<FB>;
  const int lane = (int)lane_id();
  auto chunk = [&](int c) -> float4 { return *reinterpret_cast<const float4*>(ist + IT::in_pos(lane, c) * 16); };

  // ---- pass 1: statistics, two accumulator sets, running extremes per run
  TopF ts, tt;
  int ra = 0, rz = 0;
  float rmin = 0.f, rmax = 0.f;
  {
    const float4 q = chunk(0);
    ts.a1 = ts.b1 = q.x;
    tt.a1 = tt.b1 = q.y;
    ts.a2 = tt.a2 = __int_as_float(0x7f800000);
    ts.b2 = tt.b2 = __int_as_float(0xff800000);
    topf_add<SR>(ts, q.z);
    topf_add<SR>(tt, q.w);
  }
#pragma unroll 1
  for (int r = 0; r < RUNS; ++r) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (r == 0 && j == 0) continue;
      const float4 q = chunk(8 * r + j);
      topf_add<SR>(ts, q.x); topf_add<SR>(tt, q.y); topf_add<SR>(ts, q.z); topf_add<SR>(tt, q.w);
    }
    if constexpr (SR) {
      const float nmin = fmin_nan(ts.a1, tt.a1), nmax = fmax_nan(ts.b1, tt.b1);
      if (r == 0 || nmin < rmin) ra = r;
      if (r == 0 || nmax > rmax) rz = r;
      rmin = nmin;
      rmax = nmax;
    }
  }
  topf_merge<SR>(ts, tt);
  const float mn1 = ts.a1, mx1 = ts.b1;
  const float mn2 = SR ? ts.a2 : mn1, mx2 = SR ? ts.b2 : mx1;
  if (active && !(isfinite(mn1) && isfinite(mx1))) atomicOr(cx.err, FC2_ERR_NONFINITE);

  int imin = 0, imax = 1;
  uint32_t smin_bits = 0, smax_bits = 0;
  if constexpr (SR) {
    auto first_in_run = [&](int r, float m) -> int {
      uint32_t em = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 q = chunk(8 * r + j);
        em |= (q.x == m ? 1u : 0u) << (4 * j);
        em |= (q.y == m ? 1u : 0u) << (4 * j + 1);
        em |= (q.z == m ? 1u : 0u) << (4 * j + 2);
        em |= (q.w == m ? 1u : 0u) << (4 * j + 3);
      }
      return em ? 32 * r + __ffs(em) - 1 : 1 << 20;
    };
    int fi = first_in_run(ra, mn1), fa = first_in_run(rz, mx1);
    if (fi >= G) fi = 0;
    if (fa >= G) fa = 1;
    if (fi == fa) { fi = 0; fa = 1; }
    imin = fi; imax = fa;
    auto elem = [&](int e) -> float {
      return *reinterpret_cast<const float*>(ist + IT::in_pos(lane, e >> 2) * 16 + (e & 3) * 4);
    };
    smin_bits = bf16_bits(elem(imin));
    smax_bits = bf16_bits(elem(imax));
  }
  const float zf = SR ? mn2 : mn1, vf = SR ? mx2 : mx1;
  GroupParams p = group_params((double)zf, (double)vf, L, cx.intlog != 0, cx.theta, cx.lut,
                               active ? cx.err : nullptr);
  const bool fold_ok = !p.exact && fabsf(p.nz) <= FX::kFold;
  const float Lh = (float)L + 0.5f;
  if (cx.intlog) {
    quant_runs_f32<B, G, 2>(ist, ost, p, Lh, active);
  } else if (__all_sync(0xffffffffu, fold_ok || p.exact || !active)) {
    quant_runs_f32<B, G, 0>(ist, ost, p, Lh, active);
  } else {
    quant_runs_f32<B, G, 1>(ist, ost, p, Lh, active);
  }
  if constexpr (SR) {
    int sc;
    const uint32_t Xs = fixq_clamped<FB>(0.0f, p.off32, p.inv32, Lh);
    if (p.exact || (Xs & FX::kTie) == 0u) sc = exact_code(0.0, p.off, p.div, L);
    else sc = (int)((Xs >> FB) & (uint32_t)L);
    if (active) {
      stage_patch<B, G>(ost, lane, imin, sc);
      stage_patch<B, G>(ost, lane, imax, sc);
    }
  }
  if (active) {
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
    for (int d = 0; d < nout; ++d) store_record(outs[d] + cx.meta_off + g_abs * rb, rec, rb);
  }
  __syncwarp();
  for (int d = 0; d < nout; ++d) {
#pragma unroll
    for (int u = 0; u < n_units(B); ++u) {
      const int W = unit_w(B, u), O = unit_off(B, u);
      const uint8_t* base = ost + OutStage<B, G>::off(u);
      uint8_t* dst = outs[d] + (cx.n * O) / 8 + tile_g0 * (G * W / 8);
      if (W == 1) copy_out<G, 1>(base, dst, ng);
      else if (W == 2) copy_out<G, 2>(base, dst, ng);
      else if (W == 4) copy_out<G, 4>(base, dst, ng);
      else copy_out<G, 8>(base, dst, ng);
    }
  }
  __syncwarp();
}



// ===========================================================================
// CTA-parallel variant: one CTA (G/32 warps) per 32 groups.  Accumulation:
// warp w owns run w (elements [32w, 32w+32)) of all 32 groups, lane = group.
// Encode: G/32 lanes per group, one run per lane.  The f32 tile swizzle keeps
// both access patterns bank-conflict free.
// ===========================================================================

template <int G>
struct RTile {
  static constexpr int LPG = G / 32;        // lanes per group in the encode phase
  static constexpr int CPG = G / 4;         // float4 chunks per group
  static constexpr int BYTES = 32 * G * 4;
  __device__ static __forceinline__ int pos(int g, int c) {
    const int run = c >> 3;
    return g * CPG + (c ^ ((g ^ (run * (8 / (LPG < 8 ? LPG : 8)))) & 7));
  }
};

// encode one 32-element run of group gl (part li) from the f32 tile
template <int B, bool SR, int G>
__device__ __forceinline__ void encode_run_f32(const uint8_t* tile, uint8_t* ost, int gl, int li, bool active,
                                               int64_t g_abs, const EncCtx& cx, uint8_t* const* outs, int nout,
                                               int64_t out_off = 0) {
  constexpr int LPG = G / 32;
  constexpr int L = (1 << B) - 1;
  constexpr int FB = FixFor<B>::FB;
  using FX = Fix<FB>;
  auto chunk = [&](int c) -> float4 { return *reinterpret_cast<const float4*>(tile + RTile<G>::pos(gl, c) * 16); };
  auto elem = [&](int e) -> float {
    return *reinterpret_cast<const float*>(tile + RTile<G>::pos(gl, e >> 2) * 16 + (e & 3) * 4);
  };
  // ---- statistics of this lane's run, merged over the group's lanes
  TopF ts, tt;
  {
    const float4 q = chunk(8 * li);
    ts.a1 = ts.b1 = q.x;
    tt.a1 = tt.b1 = q.y;
    ts.a2 = tt.a2 = __int_as_float(0x7f800000);
    ts.b2 = tt.b2 = __int_as_float(0xff800000);
    topf_add<SR>(ts, q.z);
    topf_add<SR>(tt, q.w);
  }
#pragma unroll
  for (int j = 1; j < 8; ++j) {
    const float4 q = chunk(8 * li + j);
    topf_add<SR>(ts, q.x); topf_add<SR>(tt, q.y); topf_add<SR>(ts, q.z); topf_add<SR>(tt, q.w);
  }
  topf_merge<SR>(ts, tt);
  float mn1 = ts.a1, mx1 = ts.b1, mn2 = SR ? ts.a2 : ts.a1, mx2 = SR ? ts.b2 : ts.b1;
  const float lmin = mn1, lmax = mx1;
#pragma unroll
  for (int o = 1; o < LPG; o <<= 1) {
    const float a1 = __shfl_xor_sync(0xffffffffu, mn1, o), b1 = __shfl_xor_sync(0xffffffffu, mx1, o);
    if constexpr (SR) {
      const float a2 = __shfl_xor_sync(0xffffffffu, mn2, o), b2 = __shfl_xor_sync(0xffffffffu, mx2, o);
      mn2 = fmin_nan(fmax_nan(mn1, a1), fmin_nan(mn2, a2));
      mx2 = fmax_nan(fmin_nan(mx1, b1), fmax_nan(mx2, b2));
    }
    mn1 = fmin_nan(mn1, a1);
    mx1 = fmax_nan(mx1, b1);
  }
  if (!SR) { mn2 = mn1; mx2 = mx1; }
  if (active && li == 0 && !(isfinite(mn1) && isfinite(mx1))) atomicOr(cx.err, FC2_ERR_NONFINITE);
  // ---- spikes: first argmin / argmax (codec.py:259-266)
  int imin = 0, imax = 1;
  uint32_t smin_bits = 0, smax_bits = 0;
  if constexpr (SR) {
    auto first = [&](float m) -> int {
      uint32_t em = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 q = chunk(8 * li + j);
        em |= (q.x == m ? 1u : 0u) << (4 * j);
        em |= (q.y == m ? 1u : 0u) << (4 * j + 1);
        em |= (q.z == m ? 1u : 0u) << (4 * j + 2);
        em |= (q.w == m ? 1u : 0u) << (4 * j + 3);
      }
      return em ? 32 * li + __ffs(em) - 1 : 1 << 20;
    };
    int fi = lmin == mn1 ? first(mn1) : 1 << 20;
    int fa = lmax == mx1 ? first(mx1) : 1 << 20;
#pragma unroll
    for (int o = 1; o < LPG; o <<= 1) {
      fi = min(fi, __shfl_xor_sync(0xffffffffu, fi, o));
      fa = min(fa, __shfl_xor_sync(0xffffffffu, fa, o));
    }
    if (fi >= G) fi = 0;
    if (fa >= G) fa = 1;
    if (fi == fa) { fi = 0; fa = 1; }
    imin = fi; imax = fa;
    smin_bits = bf16_bits(elem(imin));
    smax_bits = bf16_bits(elem(imax));
  }
  const float zf = SR ? mn2 : mn1, vf = SR ? mx2 : mx1;
  GroupParams p = group_params((double)zf, (double)vf, L, cx.intlog != 0, cx.theta, cx.lut,
                               active && li == 0 ? cx.err : nullptr);
  const bool fold_ok = !p.exact && fabsf(p.nz) <= FX::kFold;
  const float Lh = (float)L + 0.5f;
  const int mode = cx.intlog ? 2 : (__all_sync(0xffffffffu, fold_ok || p.exact || !active) ? 0 : 1);
  // ---- codes of this run
  LaneWords<B> lw;
  lw.clear();
  uint32_t tmj[2] = {0u, 0u};
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t& tm = tmj[j & 1];
    const float4 q = chunk(8 * li + j);
    const float vv[4] = {q.x, q.y, q.z, q.w};
    uint32_t X[4];
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const float a = vv[2 * pp], b = vv[2 * pp + 1];
      float y0, y1;
      if (mode == 0) {
        float t0, t1;
        fma2(t0, t1, a, b, p.inv32, p.inv32, p.nz, p.nz);
        add2(y0, y1, t0, t1, FX::kCM, FX::kCM);
      } else if (mode == 1) {
        float d0, d1, t0, t1;
        add2(d0, d1, a, b, -p.off32, -p.off32);
        fma2(t0, t1, d0, d1, p.inv32, p.inv32, FX::kC, FX::kC);
        add2(y0, y1, t0, t1, FX::kM, FX::kM);
      } else {
        y0 = __uint_as_float(fixq_clamped<FB>(a, p.off32, p.inv32, Lh));
        y1 = __uint_as_float(fixq_clamped<FB>(b, p.off32, p.inv32, Lh));
      }
      X[2 * pp] = __float_as_uint(y0);
      X[2 * pp + 1] = __float_as_uint(y1);
      tm |= pair_tie_bits<FB>(X[2 * pp], X[2 * pp + 1], 2 * j + pp);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) lw.template put_fixb<FB>(4 * j + e, X[e], 0);
  }
#pragma unroll
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u);
    uint8_t* base = ost + OutStage<B, G>::off(u);
    const uint32_t* w = lw.w + LaneWords<B>::base(u);
    if (W == 1) stage_words<G, 1>(base, gl, li, w);
    else if (W == 2) stage_words<G, 2>(base, gl, li, w);
    else if (W == 4) stage_words<G, 4>(base, gl, li, w);
    else stage_words<G, 8>(base, gl, li, w);
  }
  uint32_t tm = (p.exact ? 0xffffffffu : (tmj[0] | tmj[1])) & (active ? 0xffffffffu : 0u);
  while (tm) {
    const int k = __ffs(tm) - 1;
    tm &= tm - 1;
    const int e = 32 * li + (k < 16 ? 2 * k : 2 * (k - 16) + 1);
    stage_patch<B, G>(ost, gl, e, exact_code((double)elem(e), p.off, p.div, L));
  }
  if constexpr (SR) {
    int sc;
    const uint32_t Xs = fixq_clamped<FB>(0.0f, p.off32, p.inv32, Lh);
    if (p.exact || (Xs & FX::kTie) == 0u) sc = exact_code(0.0, p.off, p.div, L);
    else sc = (int)((Xs >> FB) & (uint32_t)L);
    if (active) {
      if ((imin >> 5) == li) stage_patch<B, G>(ost, gl, imin, sc);
      if ((imax >> 5) == li) stage_patch<B, G>(ost, gl, imax, sc);
    }
  }
  if (active && li == 0) {
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
    for (int d = 0; d < nout; ++d) store_record(outs[d] + out_off + cx.meta_off + g_abs * rb, rec, rb);
  }
}

// copy groups [g_first, g_first + count) of a unit's output stage to dst
template <int G, int W>
__device__ __forceinline__ void copy_out_groups(const uint8_t* base, uint8_t* dst, int g_first, int count) {
  const int lane = (int)lane_id();
  constexpr int GB = OTile<G, W>::GB;
  const int bytes = count * GB;
  if (bytes <= 0) return;
  const int b0 = g_first * GB;  // byte offset of the first group inside the tile segment
  if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && (bytes & 15) == 0 && (b0 & 15) == 0) {
    for (int t = lane; t < bytes / 16; t += 32)
      *reinterpret_cast<uint4*>(dst + 16 * t) = *reinterpret_cast<const uint4*>(base + OTile<G, W>::lin_pos(b0 / 16 + t));
  } else {
    for (int t = lane; t < bytes / 4; t += 32) {
      const int bb = b0 + 4 * t;
      const int lp = OTile<G, W>::lin_pos(bb >> 4) + (bb & 15);
      *reinterpret_cast<uint32_t*>(dst + 4 * t) = *reinterpret_cast<const uint32_t*>(base + lp);
    }
  }
}

}  // namespace fc2
