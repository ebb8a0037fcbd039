// fc2_encode_group.cuh -- lane-per-group encoder (the production fast path).
//
// A warp tile is 32 consecutive groups (32 / LPG at g = 256); lane l owns
// group l of the tile, so every per-group step (statistics, spike search,
// scale/zero, metadata) runs once per G elements with no shuffles.
//
//   global --cp.async--> input stage (swizzled 16-byte chunks, one per warp)
//   pass 1  stats       packed bf16x2 min/max per 32-element run
//   pass 2  spikes      first argmin / argmax via packed equality masks (only
//                       the run holding each extreme is searched); in-range
//                       stand-ins written over the two reserved slots
//   pass 3  codes       fp32x2 fixed-point estimate -> byte-gathered plane
//                       words -> 256-bit stores straight to the payload, one
//                       per run pair; near-tie masks left in smem
//   ties                the warp compacts all near-tie elements into one list,
//                       recomputes them in float64 (32 per round) and patches
//                       the payload words with red.and / red.or
//   metadata            one record per group from the owning lane
//
// Contract: SURVEY 8.0 R1-R11/R13 (codec.py:477-519).
#pragma once

#include "fc2_encode.cuh"

namespace fc2 {

template <typename T, int G, int LPG = 1>
struct GTile {
  static constexpr int CPG = G * (int)sizeof(T) / 16;   // input chunks per group
  static constexpr int IN_BYTES = 32 * G * (int)sizeof(T);
  // input swizzle: chunk c of group g -> slot g*CPG + (c ^ s).  With LPG lanes
  // per group, s mixes in the reading lane (g*LPG + part) so that 8 lanes
  // reading "their" chunk hit 8 different 16-byte bank groups.
  static constexpr int IM = CPG >= 8 ? 7 : CPG - 1;
  __device__ static __forceinline__ int in_pos(int g, int c) {
    if constexpr (CPG >= 8) {
      return g * CPG + (c ^ ((g * LPG + c / (CPG / LPG)) & 7));
    } else {
      return g * CPG + (c ^ ((g >> (CPG == 4 ? 1 : (CPG == 2 ? 2 : 3))) & IM));
    }
  }
  // The chunks a lane reads are 4 r + j (run r of its group, j < 4) and the
  // XOR key of in_pos is constant per lane (the part index c / (CPG / LPG) is
  // the lane's own), so in_pos(g, 4 r + j) = g CPG + (4 r ^ (s & 4)) + (j ^ (s & 3)):
  // one base per run plus four per-lane offsets.
  struct Lane {
    const uint8_t* A;  // group base
    int s4;            // key bit 2 (flips the run's chunk block)
    int s3;            // key bits 0-1, pre-scaled: byte offset of chunk j = (16 j) ^ s3
    __device__ __forceinline__ Lane(const uint8_t* ist, int g, int li) {
      int sk;
      if constexpr (CPG >= 8) sk = (g * LPG + li) & 7;
      else sk = (g >> (CPG == 4 ? 1 : (CPG == 2 ? 2 : 3))) & IM;
      A = ist + 16 * g * CPG;
      s4 = sk & 4;
      s3 = 16 * (sk & 3);
    }
    __device__ __forceinline__ int jx(int j) const { return (16 * j) ^ s3; }
    __device__ __forceinline__ const uint8_t* run(int r) const { return A + 16 * ((4 * r) ^ s4); }
    __device__ __forceinline__ const uint8_t* chunk(int c) const { return run(c >> 2) + jx(c & 3); }
    // element e (group-relative, inside this lane's runs)
    __device__ __forceinline__ const uint8_t* elem(int e) const { return chunk(e >> 3) + 2 * (e & 7); }
  };
};

// output staging for one unit of width W: the tile's plane segment
// (32 * G * W / 8 bytes) in 16-byte chunks, swizzled when a group owns >= 1 chunk
template <int G, int W>
struct OTile {
  static constexpr int GB = G * W / 8;                 // bytes per group
  static constexpr int CPG = GB >= 16 ? GB / 16 : 0;   // chunks per group (0: linear)
  static constexpr int BYTES = 32 * GB;
  __device__ static __forceinline__ int chunk_pos(int g, int c) {
    if constexpr (CPG == 0) {
      return 0;
    } else if constexpr (CPG >= 8) {
      return g * CPG + (c ^ (g & 7));
    } else {
      constexpr int sh = CPG == 4 ? 1 : (CPG == 2 ? 2 : 3);
      return g * CPG + (c ^ ((g >> sh) & (CPG - 1)));
    }
  }
  // byte address of byte `b` of group g's segment
  __device__ static __forceinline__ int byte_pos(int g, int b) {
    if constexpr (CPG == 0) return g * GB + b;
    else return chunk_pos(g, b >> 4) * 16 + (b & 15);
  }
  // linear chunk t of the tile segment -> its slot
  __device__ static __forceinline__ int lin_pos(int t) {
    if constexpr (CPG == 0) return t * 16;
    else return chunk_pos(t / CPG, t % CPG) * 16;
  }
};

template <int B, int G, int GPT = 32>
struct OutStage {  // GPT groups per tile
  static constexpr int NU = n_units(B);
  __host__ __device__ static constexpr int off(int u) {
    return u == 0 ? 0 : off(u - 1) + GPT * G * unit_w(B, u - 1) / 8;
  }
  static constexpr int BYTES = GPT * G * B / 8;
};

// patch element e (group-relative) of group g with code c in the output stage
template <int B, int G, int GPT = 32>
__device__ __forceinline__ void stage_patch(uint8_t* ost, int g, int e, int c) {
#pragma unroll
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u), O = unit_off(B, u);
    const int bit = e * W;
    uint8_t* p;
    if (W == 1) p = ost + OutStage<B, G, GPT>::off(u) + OTile<G, 1>::byte_pos(g, bit >> 3);
    else if (W == 2) p = ost + OutStage<B, G, GPT>::off(u) + OTile<G, 2>::byte_pos(g, bit >> 3);
    else if (W == 4) p = ost + OutStage<B, G, GPT>::off(u) + OTile<G, 4>::byte_pos(g, bit >> 3);
    else p = ost + OutStage<B, G, GPT>::off(u) + OTile<G, 8>::byte_pos(g, bit >> 3);
    const uint32_t m = ((1u << W) - 1u) << (bit & 7);
    const uint32_t v = (((uint32_t)c >> O) << (bit & 7)) & m;
    *p = (uint8_t)((*p & ~m) | v);
  }
}

// write one 32-element run's words (unit u) of group g into the output stage
template <int G, int W>
__device__ __forceinline__ void stage_words(uint8_t* base, int g, int run, const uint32_t* w) {
  // run r covers bytes [r*4W, r*4W + 4W) of the group segment
  const int b0 = run * 4 * W;
  if constexpr (OTile<G, W>::CPG == 0 || W < 4) {
#pragma unroll
    for (int i = 0; i < W; ++i)
      *reinterpret_cast<uint32_t*>(base + OTile<G, W>::byte_pos(g, b0 + 4 * i)) = w[i];
  } else {
#pragma unroll
    for (int i = 0; i < W; i += 4)
      *reinterpret_cast<uint4*>(base + OTile<G, W>::byte_pos(g, b0 + 4 * i)) =
          make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
  }
}

// copy the tile's unit segment (ng groups) from the stage to global, coalesced
template <int G, int W, int GPT = 32>
__device__ __forceinline__ void copy_out(const uint8_t* base, uint8_t* dst, int ng) {
  const int lane = (int)lane_id();
  const int bytes = ng * OTile<G, W>::GB;
  constexpr int FULL = GPT * OTile<G, W>::GB;  // bytes of a full tile segment
  if (ng == GPT && FULL % 512 == 0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
#pragma unroll
    for (int i = 0; i < FULL / 512; ++i) {
      const int t = lane + 32 * i;
      *reinterpret_cast<uint4*>(dst + 16 * t) = *reinterpret_cast<const uint4*>(base + OTile<G, W>::lin_pos(t));
    }
  } else if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && (bytes & 15) == 0) {
    for (int t = lane; t < bytes / 16; t += 32)
      *reinterpret_cast<uint4*>(dst + 16 * t) = *reinterpret_cast<const uint4*>(base + OTile<G, W>::lin_pos(t));
  } else {
    for (int t = lane; t < bytes / 4; t += 32) {
      const int lp = OTile<G, W>::lin_pos(t >> 2) + 4 * (t & 3);
      *reinterpret_cast<uint32_t*>(dst + 4 * t) = *reinterpret_cast<const uint32_t*>(base + lp);
    }
  }
}

// ---- direct output: plane words straight from registers ----------------------

// NW consecutive 32-bit words to global with the widest stores the (warp-
// uniform) alignment allows; a lane's pair of runs of a 4- or 8-bit plane is a
// whole number of 32-byte sectors
template <int NW>
__device__ __forceinline__ void store_words_g(uint8_t* p, const uint32_t* w) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if constexpr (NW % 8 == 0) {
    if ((a & 31u) == 0) {
#pragma unroll
      for (int i = 0; i < NW; i += 8)
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p + 4 * i), "r"(w[i]),
                     "r"(w[i + 1]), "r"(w[i + 2]), "r"(w[i + 3]), "r"(w[i + 4]), "r"(w[i + 5]), "r"(w[i + 6]),
                     "r"(w[i + 7])
                     : "memory");
      return;
    }
  }
  if constexpr (NW % 4 == 0) {
    if ((a & 15u) == 0) {
#pragma unroll
      for (int i = 0; i < NW; i += 4)
        *reinterpret_cast<uint4*>(p + 4 * i) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
      return;
    }
  }
  if constexpr (NW % 2 == 0) {
    if ((a & 7u) == 0) {
#pragma unroll
      for (int i = 0; i < NW; i += 2) *reinterpret_cast<uint2*>(p + 4 * i) = make_uint2(w[i], w[i + 1]);
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < NW; ++i) *reinterpret_cast<uint32_t*>(p + 4 * i) = w[i];
}

// patch element e of absolute group ga in the payload (global) with code c
// (other lanes patch other elements of the same 32-bit word concurrently)
template <int B, int G>
__device__ __forceinline__ void payload_patch_xor(uint8_t* out, int64_t n, int64_t ga, int e, int c) {
#pragma unroll
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u), O = unit_off(B, u);
    const int bit = e * W;
    const int64_t byte = n * O / 8 + ga * (G * W / 8) + (bit >> 3);
    unsigned int* wp = reinterpret_cast<unsigned int*>(out + (byte & ~(int64_t)3));
    const int sh = (int)(byte & 3) * 8 + (bit & 7);
    const uint32_t m = (1u << W) - 1u, want = ((uint32_t)c >> O) & m;
    // clear then set this element's bits: two fire-and-forget reductions
    // (same thread, same address: ordered), commuting with other lanes' patches
    asm volatile("red.global.and.b32 [%0], %1;" ::"l"(wp), "r"(~(m << sh)) : "memory");
    asm volatile("red.global.or.b32 [%0], %1;" ::"l"(wp), "r"(want << sh) : "memory");
  }
}

// ---- per-chunk helpers on 16-byte chunks -----------------------------------

// Pack the 32 codes of a run into plane words (LaneWords layout: unit-major,
// word t of a W-bit unit holds codes [32t/W, 32(t+1)/W) LSB-first).  FB = 16
// puts each code in byte 2 of its fixed-point word, so four codes are
// gathered into one word with three byte permutes; slice s of a word holds
// codes k0 + s, k0 + s + S, ... (S = 8 / W) and is merged with one shift-or.
// MASK: codes may be out of range (unclamped spike slots, patched later).
template <int B, bool MASK>
__device__ __forceinline__ void pack_run_fb16(const uint32_t (&X)[32], uint32_t (&w)[B]) {
#pragma unroll
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u), O = unit_off(B, u);
    const int S = 8 / W;
    const uint32_t mrep = ((1u << W) - 1u) * 0x01010101u;
#pragma unroll
    for (int t = 0; t < W; ++t) {
      uint32_t word = 0;
#pragma unroll
      for (int sl = 0; sl < S; ++sl) {
        const int k0 = t * (32 / W) + sl;
        const uint32_t lo = __byte_perm(X[k0], X[k0 + S], 0x0062);
        const uint32_t hi = __byte_perm(X[k0 + 2 * S], X[k0 + 3 * S], 0x0062);
        const uint32_t A = __byte_perm(lo, hi, 0x5410);  // codes as bytes
        uint32_t v;
        if (W == B && !MASK) {
          v = A << (W * sl);
        } else {
          const int sh = W * sl - O;
          v = sh >= 0 ? ((A & (mrep << O)) << sh) : ((A >> (-sh)) & (mrep << (W * sl)));
        }
        word += v;  // disjoint fields: the add is the or, and folds with the shift into one IMAD (FMA pipe)
      }
      w[LaneWords<B>::base(u) + t] = word;
    }
  }
}

// pass 3 for all runs of the lane's group with the code form fixed at compile
// time (MODE 0: folded fma, 1: explicit v - off, 2: INT_LOG clamped).
// Writes packed words into the output stage; near-tie elements (split-layout
// tie masks: bit i < 16 element 2i, bit 16 + i element 2i + 1) are recomputed
// exactly and patched in the stage.
template <int B, bool SR, int G, int MODE, int LPG>
__device__ __forceinline__ void quant_runs(const uint8_t* ist, uint32_t* tms, const GroupParams& p, float Lh,
                                           bool active, uint8_t* out, int64_t n, int64_t g_abs) {
  using IT = GTile<__nv_bfloat16, G, LPG>;
  constexpr int RUNS = G / 32 / LPG;  // runs of this lane
  constexpr int PAIR = RUNS >= 2 ? 2 : 1;
  const int gl = (int)lane_id() / LPG, r0 = ((int)lane_id() % LPG) * RUNS;
  constexpr int FB = FixFor<B>::FB;
  using FX = Fix<FB>;
  // FB = 16 folded form: one FFMA, y = fma(v, inv, nz + kCM) (bound: Fix<16>)
  const float c16 = __fadd_rn(p.nz, FX::kCM);
  const typename IT::Lane la(ist, gl, (int)lane_id() % LPG);
#pragma unroll 1
  for (int rp = 0; rp < RUNS; rp += PAIR) {
  uint32_t pw[PAIR][B];  // plane words of the pair's runs (LaneWords layout)
#pragma unroll
  for (int q = 0; q < PAIR; ++q) {
    const int rr = rp + q;
    const int r = r0 + rr;  // run index inside the group
    const uint8_t* rb = la.run(r);
    LaneWords<B> lw;
    lw.clear();
    // tie flags gathered as f16 sums on the FMA pipe (tie_acc16 / tie_acc15)
    __half2 tacc[2] = {__float2half2_rn(1024.f), __float2half2_rn(1024.f)};
    uint32_t XR[32];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 q = *reinterpret_cast<const uint4*>(rb + la.jx(j));
      const uint32_t ww[4] = {q.x, q.y, q.z, q.w};
      uint32_t X[8];
#pragma unroll
      for (int pp = 0; pp < 4; ++pp) {
        const float a = __uint_as_float(ww[pp] << 16), b = __uint_as_float(ww[pp] & 0xFFFF0000u);
        float y0, y1;
        if constexpr (MODE == 0) {
          if constexpr (FB == 16) {
            fma2(y0, y1, a, b, p.inv32, p.inv32, c16, c16);
          } else {
            float t0, t1;
            fma2(t0, t1, a, b, p.inv32, p.inv32, p.nz, p.nz);
            add2(y0, y1, t0, t1, FX::kCM, FX::kCM);
          }
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
        if constexpr (FB == 16) tie_acc16(tacc[j >> 1], y0, y1, 4 * (j & 1) + pp);
        else tie_acc15(tacc[j >> 1], y0, y1, 4 * (j & 1) + pp);
      }
      // FB = 15 (8-bit codes in bits [15, 23)): one shift (IMAD on the FMA
      // pipe) puts the code in byte 2 as for FB = 16, so the same byte-permute
      // packing applies
#pragma unroll
      for (int e = 0; e < 8; ++e) XR[8 * j + e] = FB == 16 ? X[e] : X[e] << 1;
    }
    // spike slots hold an in-range stand-in (encode_tile_bf16), so every code
    // fits its width and no masking is needed when the unit is the whole code
    pack_run_fb16<B, false>(XR, lw.w);
#pragma unroll
    for (int i = 0; i < B; ++i) pw[q][i] = lw.w[i];
    // near-tie masks of this run, resolved after all runs (one divergent
    // pass per tile instead of one per run)
    tms[32 * rr + (int)lane_id()] = tie_bits16(tacc);
  }
  if (active) {  // the pair's bytes of every unit: [4W (r0 + rp), +4W PAIR) of the group
#pragma unroll
    for (int u = 0; u < n_units(B); ++u) {
      const int W = unit_w(B, u), O = unit_off(B, u);
      uint32_t w[PAIR * 8];
#pragma unroll
      for (int q = 0; q < PAIR; ++q)
#pragma unroll
        for (int i = 0; i < W; ++i) w[q * W + i] = pw[q][O + i];
      uint8_t* dst = out + n * O / 8 + g_abs * (G * W / 8) + (r0 + rp) * 4 * W;
      if (W == 1) store_words_g<PAIR * 1>(dst, w);
      else if (W == 2) store_words_g<PAIR * 2>(dst, w);
      else if (W == 4) store_words_g<PAIR * 4>(dst, w);
      else store_words_g<PAIR * 8>(dst, w);
    }
  }
  }
}

// Exact float64 recompute of the near-tie elements of the tile, done by the
// whole warp: every lane's tie masks (one per run, left in smem by pass 3:
// bit i < 16 -> element 2i, bit 16 + i -> element 2i + 1) are compacted into
// one list (lane << 16 | element), and the 32 lanes resolve 32 entries per
// round, each fetching its group's offset/divisor from the owning lane by
// shuffle.  Ties are ~0.1-0.3% of elements, so one round usually covers the
// tile instead of one divergent pass per run.  Groups that need float64 for
// every element (p.exact) loop on their own.
template <int B, int G, int LPG>
__device__ __forceinline__ void resolve_ties_coop(const uint8_t* ist, uint32_t* tms, const GroupParams& p,
                                                  bool active, uint8_t* out, int64_t n, int64_t tile_g0) {
  using IT = GTile<__nv_bfloat16, G, LPG>;
  constexpr int RUNS = G / 32 / LPG;
  constexpr int L = (1 << B) - 1;
  constexpr int CAP = RUNS * 32;  // list entries that fit in the mask area
  const int lane = (int)lane_id();
  const int gl = lane / LPG, r0 = (lane % LPG) * RUNS;
  auto value = [&](int g, int e) -> double {
    return (double)__uint_as_float(
        (uint32_t)*reinterpret_cast<const uint16_t*>(ist + IT::in_pos(g, e >> 3) * 16 + (e & 7) * 2) << 16);
  };
  __syncwarp();
  uint32_t m[RUNS];
  int cnt = 0;
  const bool listed = active && !p.exact;
#pragma unroll
  for (int rr = 0; rr < RUNS; ++rr) {
    m[rr] = listed ? tms[32 * rr + lane] : 0u;
    cnt += __popc(m[rr]);
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (total > 0) {  // warp-uniform
    if (total <= CAP) {
      __syncwarp();  // every lane has read its masks before the list overwrites them
      int pos = incl - cnt;
#pragma unroll
      for (int rr = 0; rr < RUNS; ++rr) {
        uint32_t t = m[rr];
        while (t) {
          const int k = __ffs(t) - 1;
          t &= t - 1;
          tms[pos++] = ((uint32_t)lane << 16) | (uint32_t)(32 * (r0 + rr) + (k < 16 ? 2 * k : 2 * (k - 16) + 1));
        }
      }
      __syncwarp();
      for (int base = 0; base < total; base += 32) {  // warp-uniform rounds
        const int i = base + lane;
        const uint32_t ent = i < total ? tms[i] : 0u;
        const int src = (int)(ent >> 16), e = (int)(ent & 0xFFFFu);
        const double off = __shfl_sync(0xffffffffu, p.off, src), div = __shfl_sync(0xffffffffu, p.div, src);
        if (i < total) {
          const int c = exact_code(value(src / LPG, e), off, div, L);
          payload_patch_xor<B, G>(out, n, tile_g0 + src / LPG, e, c);
        }
      }
    } else {  // many ties in one tile (rare): each lane resolves its own
#pragma unroll 1
      for (int rr = 0; rr < RUNS; ++rr) {
        uint32_t t = m[0];
#pragma unroll
        for (int q = 1; q < RUNS; ++q) t = rr == q ? m[q] : t;
        while (t) {
          const int k = __ffs(t) - 1;
          t &= t - 1;
          const int e = 32 * (r0 + rr) + (k < 16 ? 2 * k : 2 * (k - 16) + 1);
          const int c = exact_code(value(gl, e), p.off, p.div, L);
          payload_patch_xor<B, G>(out, n, tile_g0 + gl, e, c);
        }
      }
    }
  }
  if (active && p.exact) {  // every element of the group in float64
#pragma unroll 1
    for (int e = r0 * 32; e < (r0 + RUNS) * 32; ++e) {
      const int c = exact_code(value(gl, e), p.off, p.div, L);
      payload_patch_xor<B, G>(out, n, tile_g0 + gl, e, c);
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// the kernel body for one warp tile (bf16 input)
// ---------------------------------------------------------------------------

template <int B, bool SR, int G, int LPG>
__device__ __forceinline__ void encode_tile_bf16(uint8_t* ist, uint32_t* tms, bool active,
                                                 int64_t g_abs, const EncCtx& cx, uint8_t* out, int64_t tile_g0,
                                                 int ng) {
  using IT = GTile<__nv_bfloat16, G, LPG>;
  constexpr int L = (1 << B) - 1;
  const int lane = (int)lane_id();
  const int gl = lane / LPG, li = lane % LPG;   // group of the tile, part of the group
  constexpr int RUNS = G / 32 / LPG;            // 32-element runs of this lane
  const int r0 = li * RUNS;                     // first run (group-relative)
  const typename IT::Lane la(ist, gl, li);
  auto chunk = [&](int c) -> uint4 { return *reinterpret_cast<const uint4*>(la.chunk(c)); };

  constexpr int FB = FixFor<B>::FB;
  using FX = Fix<FB>;

  // ---- pass 1: packed bf16x2 min / max of every run of this lane ----------
  __nv_bfloat162 rmn[RUNS], rmx[RUNS];
#pragma unroll
  for (int rr = 0; rr < RUNS; ++rr) {
    const int r = r0 + rr;
    const uint4 q0 = chunk(4 * r), q1 = chunk(4 * r + 1), q2 = chunk(4 * r + 2), q3 = chunk(4 * r + 3);
    auto h = [](uint32_t w) { return *reinterpret_cast<const __nv_bfloat162*>(&w); };
    const __nv_bfloat162 a0 = __hmin2_nan(__hmin2_nan(h(q0.x), h(q0.y)), __hmin2_nan(h(q0.z), h(q0.w)));
    const __nv_bfloat162 a1 = __hmin2_nan(__hmin2_nan(h(q1.x), h(q1.y)), __hmin2_nan(h(q1.z), h(q1.w)));
    const __nv_bfloat162 a2 = __hmin2_nan(__hmin2_nan(h(q2.x), h(q2.y)), __hmin2_nan(h(q2.z), h(q2.w)));
    const __nv_bfloat162 a3 = __hmin2_nan(__hmin2_nan(h(q3.x), h(q3.y)), __hmin2_nan(h(q3.z), h(q3.w)));
    rmn[rr] = __hmin2_nan(__hmin2_nan(a0, a1), __hmin2_nan(a2, a3));
    const __nv_bfloat162 b0 = __hmax2_nan(__hmax2_nan(h(q0.x), h(q0.y)), __hmax2_nan(h(q0.z), h(q0.w)));
    const __nv_bfloat162 b1 = __hmax2_nan(__hmax2_nan(h(q1.x), h(q1.y)), __hmax2_nan(h(q1.z), h(q1.w)));
    const __nv_bfloat162 b2 = __hmax2_nan(__hmax2_nan(h(q2.x), h(q2.y)), __hmax2_nan(h(q2.z), h(q2.w)));
    const __nv_bfloat162 b3 = __hmax2_nan(__hmax2_nan(h(q3.x), h(q3.y)), __hmax2_nan(h(q3.z), h(q3.w)));
    rmx[rr] = __hmax2_nan(__hmax2_nan(b0, b1), __hmax2_nan(b2, b3));
  }
  __nv_bfloat162 tmn = rmn[0], tmx = rmx[0];
#pragma unroll
  for (int rr = 1; rr < RUNS; ++rr) {
    tmn = __hmin2_nan(tmn, rmn[rr]);
    tmx = __hmax2_nan(tmx, rmx[rr]);
  }
  float mn1 = fmin_nan(__low2float(tmn), __high2float(tmn));
  float mx1 = fmax_nan(__low2float(tmx), __high2float(tmx));
#pragma unroll
  for (int o = 1; o < LPG; o <<= 1) {  // merge the LPG parts of the group
    mn1 = fmin_nan(mn1, __shfl_xor_sync(0xffffffffu, mn1, o));
    mx1 = fmax_nan(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
  }
  float mn2 = mn1, mx2 = mx1;
  const bool finite = isfinite(mn1) && isfinite(mx1);
  if (active && !finite && li == 0) atomicOr(cx.err, FC2_ERR_NONFINITE);

  // ---- spikes (codec.py:259-275): first argmin / argmax, and the extremes of
  // the rest.  Only the first run holding the extreme is searched; it also
  // yields that run's extreme with the extreme's occurrences removed.  With
  // one occurrence in the group the shrunk extreme is min(other runs, that);
  // with several it is the extreme itself.
  int imin = 0, imax = 1;
  uint32_t smin_bits = 0, smax_bits = 0;
  if constexpr (SR) {
    // search run `r` for value m: first index, occurrences, extreme of the rest
    auto search = [&](int r, float m, bool is_min, int& first, int& occ, float& rest) {
      const __nv_bfloat162 mm = __float2bfloat162_rn(m);
      const uint32_t sent = is_min ? 0x7F807F80u : 0xFF80FF80u;  // +inf / -inf
      uint32_t em = 0;
      __nv_bfloat162 acc = *reinterpret_cast<const __nv_bfloat162*>(&sent);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 q = chunk(4 * r + j);
        const uint32_t ww[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
          const uint32_t eq = __heq2_mask(*reinterpret_cast<const __nv_bfloat162*>(&ww[pp]), mm);
          em |= eq & (0x00010001u << (4 * j + pp));
          const uint32_t xr = (ww[pp] & ~eq) | (sent & eq);
          const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(&xr);
          acc = is_min ? __hmin2_nan(acc, x) : __hmax2_nan(acc, x);
        }
      }
      const uint32_t lo = em & 0xFFFFu, hi = em >> 16;
      const int f = min(lo ? 2 * (__ffs(lo) - 1) : 64, hi ? 2 * (__ffs(hi) - 1) + 1 : 64);
      first = f < 32 ? 32 * r + f : 1 << 20;
      occ = __popc(em);
      rest = is_min ? fmin_nan(__low2float(acc), __high2float(acc)) : fmax_nan(__low2float(acc), __high2float(acc));
    };
    const __nv_bfloat162 mm = __float2bfloat162_rn(mn1), MM = __float2bfloat162_rn(mx1);
    int ra = -1, rz = -1, omin = 0, omax = 0;
#pragma unroll
    for (int rr = RUNS - 1; rr >= 0; --rr) {  // first run holding each extreme
      if (__heq2_mask(rmn[rr], mm)) { if (ra >= 0) omin += 1; ra = rr; }
      if (__heq2_mask(rmx[rr], MM)) { if (rz >= 0) omax += 1; rz = rr; }
    }
    // runs of this lane other than ra / rz
    float omn = __int_as_float(0x7f800000), omx = __int_as_float(0xff800000);
#pragma unroll
    for (int rr = 0; rr < RUNS; ++rr) {
      const uint32_t pinf = 0x7F807F80u, ninf = 0xFF80FF80u;
      const __nv_bfloat162 a = rr == ra ? *reinterpret_cast<const __nv_bfloat162*>(&pinf) : rmn[rr];
      const __nv_bfloat162 z = rr == rz ? *reinterpret_cast<const __nv_bfloat162*>(&ninf) : rmx[rr];
      omn = fmin_nan(omn, fmin_nan(__low2float(a), __high2float(a)));
      omx = fmax_nan(omx, fmax_nan(__low2float(z), __high2float(z)));
    }
    int fi = 1 << 20, fa = 1 << 20;
    if (ra >= 0) {
      int occ;
      float rest;
      search(r0 + ra, mn1, true, fi, occ, rest);
      omin += occ;
      omn = fmin_nan(omn, rest);
    }
    if (rz >= 0) {
      int occ;
      float rest;
      search(r0 + rz, mx1, false, fa, occ, rest);
      omax += occ;
      omx = fmax_nan(omx, rest);
    }
#pragma unroll
    for (int o = 1; o < LPG; o <<= 1) {
      fi = min(fi, __shfl_xor_sync(0xffffffffu, fi, o));
      fa = min(fa, __shfl_xor_sync(0xffffffffu, fa, o));
      omin += __shfl_xor_sync(0xffffffffu, omin, o);
      omax += __shfl_xor_sync(0xffffffffu, omax, o);
      omn = fmin_nan(omn, __shfl_xor_sync(0xffffffffu, omn, o));
      omx = fmax_nan(omx, __shfl_xor_sync(0xffffffffu, omx, o));
    }
    mn2 = omin >= 2 ? mn1 : omn;
    mx2 = omax >= 2 ? mx1 : omx;
    if (fi >= G) fi = 0;  // only with NaN input (already flagged)
    if (fa >= G) fa = 1;
    if (fi == fa) { fi = 0; fa = 1; }
    imin = fi; imax = fa;
    // reserved values are the elements themselves (codec.py:492-493)
    auto elem = [&](int e) -> uint32_t {
      // (any lane of the group reads them: the element may sit in another
      // lane's part, so the swizzle key is the chunk's, not this lane's)
      return *reinterpret_cast<const uint16_t*>(ist + IT::in_pos(gl, e >> 3) * 16 + (e & 7) * 2);
    };
    smin_bits = elem(imin);
    smax_bits = elem(imax);
  }
  const float zf = SR ? mn2 : mn1, vf = SR ? mx2 : mx1;
  GroupParams p = group_params((double)zf, (double)vf, L, cx.intlog != 0, cx.theta, cx.lut,
                               active ? cx.err : nullptr);

  // ---- pass 3: codes -> output stage (+ exact recompute of near ties) --------
  // 0: folded fma form, 1: explicit (v - off) form, 2: INT_LOG (clamped)
  const bool fold_ok = !p.exact && fabsf(p.nz) <= FX::kFold;
  const float Lh = (float)L + 0.5f;
  if constexpr (SR) {
    // Reserved slots are quantized as 0.0 (codec.py:494-496).  0.0 may lie
    // outside [zero, vmax] and then clips to code 0 (below) or L (above);
    // the in-range bf16 stand-in with the same code is written over both
    // slots, so pass 3 yields their codes directly and no code word ever
    // needs masking.  (Reserved values were read out above.)
    // (INT_LOG codes are clamped in pass 3 and 0.0 stays as is.)
    const uint32_t sv = cx.intlog ? 0u
                                  : (zf > 0.f ? __float_as_uint(zf) >> 16 : (vf < 0.f ? __float_as_uint(vf) >> 16 : 0u));
    if (active) {
      if (imin / (G / LPG) == li)
        *reinterpret_cast<uint16_t*>(const_cast<uint8_t*>(la.elem(imin))) = (uint16_t)sv;
      if (imax / (G / LPG) == li)
        *reinterpret_cast<uint16_t*>(const_cast<uint8_t*>(la.elem(imax))) = (uint16_t)sv;
    }
    if constexpr (LPG > 1) __syncwarp();
  }
  if (cx.intlog) {
    quant_runs<B, SR, G, 2, LPG>(ist, tms, p, Lh, active, out, cx.n, g_abs);
  } else if (__all_sync(0xffffffffu, fold_ok || p.exact || !active)) {
    quant_runs<B, SR, G, 0, LPG>(ist, tms, p, Lh, active, out, cx.n, g_abs);
  } else {
    quant_runs<B, SR, G, 1, LPG>(ist, tms, p, Lh, active, out, cx.n, g_abs);
  }
  __syncwarp();  // plane stores of all lanes before the tie fix-ups modify them
  resolve_ties_coop<B, G, LPG>(ist, tms, p, active, out, cx.n, tile_g0);

  // ---- metadata record (R10), straight from the group's first lane ---------
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
    store_record(out + cx.meta_off + g_abs * rb, rec, rb);
  }
  __syncwarp();
  __syncwarp();
}

}  // namespace fc2
