// fc2_reduce_run.cuh -- two-step middle stage (collectives.py:291-311) with a
// bulk-copy (TMA) staged source tile and the sums kept in registers.
//
// One warp = one tile of 1024 shard elements; lane l owns run l (32
// consecutive elements; a group of G spans G/32 lanes).
//
//   1. lane 0 arms the warp's mbarrier and issues one cp.async.bulk per
//      bit-split plane and one for the metadata records of every source
//      (8 sources x 2 copies at b4): the whole tile's operands (~4.9 KB) are
//      in flight at once, with ~20 one-warp CTAs resident per SM;
//   2. per source, in rank order: the lane reads its run's code words and its
//      group's record from shared memory (the next source's are read while
//      this one is decoded), decodes 32 values in packed fp32x2 (code -> float
//      via the 2^23 magic, one FFMA2 per pair), substitutes the reserved spike
//      values (imin, then imax, codec.py:559-561) through the lane's smem
//      spill row -- only lanes whose run holds a spike -- and adds into 32
//      fp32 accumulators from +0.0 (collectives.py:293-297);
//   3. the sums never leave registers: encode_lane (statistics, spikes,
//      fixed-point codes with exact float64 near-tie recompute) packs them and
//      stores the plane words straight to every destination (the owner's
//      gather slot and, in the SPMD path, every peer's over NVLink).
//
// Measured (B200, 8 sources x 4 Mi elements, b4 SR g128): 22.8 us (23.9 before the
// per-quad spike substitution), ~10.6 M
// warp instructions at ~1.9 IPC -- instruction-bound (profiles/r2_reduce_run_ncu_full.md).
#pragma once

#include "fc2_decode.cuh"
#include "fc2_encode.cuh"
#include "fc2_tma.cuh"

#ifndef FC2_RUN_MINB
#define FC2_RUN_MINB 18  // min resident one-warp CTAs per SM (register cap 112; 96 used, no spills)
#endif
#ifndef FC2_RUN_STAGES
#define FC2_RUN_STAGES 1  // 2: persistent warps prefetch their next tile
#endif

namespace fc2 {

constexpr int kRunStageSrc = 8;  // sources staged per tile (N <= 8 ranks of one node)

template <int B, bool SR, int G>
struct RunTile {
  static constexpr int ELEMS = 1024;
  static constexpr int GROUPS = ELEMS / G;
  static constexpr int CODE_BYTES = ELEMS * B / 8;                     // all planes of the tile
  static constexpr int REC_MAX = GROUPS * (SR ? 12 : 4);              // BF16 records are the larger
  static constexpr int SRC_BYTES = (CODE_BYTES + REC_MAX + 15) / 16 * 16;
  static constexpr int STAGE_BYTES = kRunStageSrc * SRC_BYTES;
  static constexpr int SPILL_FLOATS = 36;                             // per lane (16-B rows, conflict-free)
  static constexpr int WARP_BYTES = 16 + FC2_RUN_STAGES * STAGE_BYTES + 32 * SPILL_FLOATS * 4;
  __host__ __device__ static constexpr int uoff(int u) {  // plane u inside a source's stage
    return u == 0 ? 0 : uoff(u - 1) + ELEMS * unit_w(B, u - 1) / 8;
  }
};

template <int B, bool SR, int G>
__global__ void __launch_bounds__(32, FC2_RUN_MINB) k_reduce_run(const __grid_constant__ ReduceArgs a) {
  pdl_enter();
  using RT = RunTile<B, SR, G>;
  constexpr int LPG = G / 32;  // lanes per group
  constexpr int NST = FC2_RUN_STAGES;
  extern __shared__ __align__(16) uint8_t rsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(rsm);  // one mbarrier per stage
  uint8_t* stages = rsm + 16;
  float* spill = reinterpret_cast<float*>(stages + NST * RT::STAGE_BYTES) + lane_id() * RT::SPILL_FLOATS;
  const int lane = (int)lane_id();
  const int lig = lane % LPG;
  const bool intlog = a.intlog != 0;
  const int rb = rec_bytes(SR, intlog);
  const int64_t n = a.n;
  const int64_t meta_off = n * B / 8;
  const int64_t tps = (n + RT::ELEMS - 1) / RT::ELEMS;  // tiles per shard
  const int ns = a.nsrc;
  EncCtx cx;
  cx.n = n; cx.meta_off = meta_off; cx.intlog = a.intlog; cx.theta = a.theta; cx.lut = a.lut; cx.err = a.err;

  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NST; ++i) mbar_init(bar + i, 1);
    fence_proxy_async_smem();
  }
  __syncwarp();
  uint32_t phase = 0;  // bit i: parity of stage i

  // bulk copies of every source's planes + records of a full tile (lane 0)
  auto issue = [&](int64_t t, int si) {
    const int64_t sh = t / tps;
    const int64_t e0 = (t - sh * tps) * RT::ELEMS;
    if (e0 + RT::ELEMS > n) return;  // partial tile: plain loads at consume time
    if (lane == 0) {
      const int64_t soff = sh * a.sstride;
      const int recb = RT::GROUPS * rb;
      uint8_t* stage = stages + si * RT::STAGE_BYTES;
      mbar_arrive_expect_tx(bar + si, (uint32_t)(ns * (RT::CODE_BYTES + recb)));
      for (int i = 0; i < ns; ++i) {
        const uint8_t* src = a.src[i] + soff;
        uint8_t* st = stage + i * RT::SRC_BYTES;
#pragma unroll
        for (int u = 0; u < n_units(B); ++u) {
          const int W = unit_w(B, u), O = unit_off(B, u);
          bulk_g2s(st + RT::uoff(u), src + n * O / 8 + e0 * W / 8, RT::ELEMS * W / 8, bar + si);
        }
        bulk_g2s(st + RT::CODE_BYTES, src + meta_off + (e0 / G) * rb, (uint32_t)recb, bar + si);
      }
    }
  };

  int si = 0;
  if (NST == 2 && (int64_t)blockIdx.x < a.total) issue(blockIdx.x, 0);
  for (int64_t t = blockIdx.x; t < a.total; t += gridDim.x, si = (si + 1) % NST) {
    fence_proxy_async_smem();  // generic reads of the stage being refilled came first (__syncwarp below)
    if (NST == 2) {
      if (t + gridDim.x < a.total) issue(t + gridDim.x, si ^ 1);  // next tile, other stage
    } else {
      issue(t, si);
    }
    const int64_t sh = t / tps;
    const int64_t e0 = (t - sh * tps) * RT::ELEMS;
    const int64_t soff = sh * a.sstride, doff = sh * a.dstride;
    const int64_t er = e0 + 32 * lane;  // this lane's run
    const bool active = er < n;
    const int ngv = (int)min((int64_t)RT::GROUPS, (n - e0) / G);  // valid groups of the tile
    uint8_t* stage = stages + si * RT::STAGE_BYTES;
    if (e0 + RT::ELEMS <= n) {
      mbar_wait(bar + si, (phase >> si) & 1u);
      phase ^= 1u << si;
    } else {  // partial last tile of the shard: plain loads of the valid bytes
      const int64_t ev = n - e0;  // valid elements (a multiple of G)
      for (int i = 0; i < ns; ++i) {
        const uint8_t* src = a.src[i] + soff;
        uint8_t* st = stage + i * RT::SRC_BYTES;
#pragma unroll
        for (int u = 0; u < n_units(B); ++u) {
          const int W = unit_w(B, u), O = unit_off(B, u);
          const int nb = (int)(ev * W / 8);  // a multiple of 4 (ev % 32 == 0)
          const uint8_t* p = src + n * O / 8 + e0 * W / 8;
          for (int b = 4 * lane; b < nb; b += 128)
            *reinterpret_cast<uint32_t*>(st + RT::uoff(u) + b) = *reinterpret_cast<const uint32_t*>(p + b);
        }
        const uint8_t* mp = src + meta_off + (e0 / G) * rb;
        for (int b = lane; b < ngv * rb; b += 32) st[RT::CODE_BYTES + b] = mp[b];
      }
      __syncwarp();
    }
    float acc[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) acc[k] = 0.0f;  // acc = zeros(float32) (collectives.py:293)

    // ---- accumulate the staged sources in rank order; source i + 1's code
    // words and record are read from the stage while source i is decoded
    auto load_words = [&](int i, uint32_t* wv) {
      const uint8_t* st = stage + i * RT::SRC_BYTES;
#pragma unroll
      for (int u = 0; u < n_units(B); ++u) {
        const int W = unit_w(B, u), O = unit_off(B, u);
        const uint8_t* p = st + RT::uoff(u) + lane * 4 * W;
        if (W == 8) {
          const uint4 q0 = *reinterpret_cast<const uint4*>(p), q1 = *reinterpret_cast<const uint4*>(p + 16);
          wv[O] = q0.x; wv[O + 1] = q0.y; wv[O + 2] = q0.z; wv[O + 3] = q0.w;
          wv[O + 4] = q1.x; wv[O + 5] = q1.y; wv[O + 6] = q1.z; wv[O + 7] = q1.w;
        } else if (W == 4) {
          const uint4 q0 = *reinterpret_cast<const uint4*>(p);
          wv[O] = q0.x; wv[O + 1] = q0.y; wv[O + 2] = q0.z; wv[O + 3] = q0.w;
        } else if (W == 2) {
          const uint2 q0 = *reinterpret_cast<const uint2*>(p);
          wv[O] = q0.x; wv[O + 1] = q0.y;
        } else {
          wv[O] = *reinterpret_cast<const uint32_t*>(p);
        }
      }
    };
    auto load_rec = [&](int i, uint32_t* rv) {  // BF16 records (R10): 4 or 12 bytes
      const uint8_t* rp = stage + i * RT::SRC_BYTES + RT::CODE_BYTES + (lane / LPG) * rb;
      rv[0] = *reinterpret_cast<const uint32_t*>(rp);
      if constexpr (SR) {
        rv[1] = *reinterpret_cast<const uint32_t*>(rp + 4);
        rv[2] = *reinterpret_cast<const uint32_t*>(rp + 8);
      }
    };
    uint32_t wn[B], rn[3] = {0u, 0u, 0u};
    load_words(0, wn);
    if (!intlog) load_rec(0, rn);
#pragma unroll 1
    for (int i = 0; i < ns; ++i) {
      const uint8_t* st = stage + i * RT::SRC_BYTES;
      uint32_t w[B], rc[3];
#pragma unroll
      for (int k = 0; k < B; ++k) w[k] = wn[k];
      rc[0] = rn[0]; rc[1] = rn[1]; rc[2] = rn[2];
      if (i + 1 < ns) {
        load_words(i + 1, wn);
        if (!intlog) load_rec(i + 1, rn);
      }
      // the group's record (R10 layouts)
      const uint8_t* rp = st + RT::CODE_BYTES + (lane / LPG) * rb;
      uint32_t cf[32];
      run_code_floats<B>(w, cf);
      float d[32];
      float smin = 0.f, smax = 0.f;
      int ka = -1, kz = -1;  // spike positions inside this lane's run
      bool hit = false;
      if (!intlog) {
        const uint32_t r0 = rc[0];
        const float s32 = bf16_val(r0 & 0xFFFFu), z32 = bf16_val(r0 >> 16);
        if constexpr (SR) {
          const uint32_t r1 = rc[1];
          const uint32_t r2 = rc[2];
          smin = bf16_val(r1 & 0xFFFFu);
          smax = bf16_val(r1 >> 16);
          // indices ride in bf16 float slots; astype(int64) truncates (codec.py:550-551)
          const float fi = bf16_val(r2 & 0xFFFFu), fa = bf16_val(r2 >> 16);
          if ((fi > -1.0f) && (fi < (float)G) && (fa > -1.0f) && (fa < (float)G)) {
            ka = (int)fi - 32 * lig;
            kz = (int)fa - 32 * lig;
            hit = (unsigned)ka < 32u || (unsigned)kz < 32u;
          } else if (active && lig == 0) {
            atomicOr(a.err, FC2_ERR_SPIKE_INDEX);
          }
        }
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          float c0, c1;
          add2(c0, c1, __uint_as_float(cf[k]), __uint_as_float(cf[k + 1]), -8388608.0f, -8388608.0f);
          fma2(d[k], d[k + 1], c0, c1, s32, s32, z32, z32);
        }
      } else {
        uint32_t r0 = 0, r1 = 0;
        if (rb == 8) {
          const uint2 q = *reinterpret_cast<const uint2*>(rp);
          r0 = q.x; r1 = q.y;
        } else {
          r0 = *reinterpret_cast<const uint16_t*>(rp);
        }
        const int si8 = (int)(int8_t)(r0 & 0xFFu), zi = (int)(int8_t)((r0 >> 8) & 0xFFu);
        const double s64 = si8 == -128 ? 0.0 : a.lut[si8 + 128];
        const double o64 = __dmul_rn(-(double)zi, s64);
        if constexpr (SR) {
          smin = bf16_val(r0 >> 16);
          smax = bf16_val(r1 & 0xFFFFu);
          const int ii = (int)((r1 >> 16) & 0xFFu), ia = (int)(r1 >> 24);
          if (ii < G && ia < G) {
            ka = ii - 32 * lig;
            kz = ia - 32 * lig;
            hit = (unsigned)ka < 32u || (unsigned)kz < 32u;
          } else if (active && lig == 0) {
            atomicOr(a.err, FC2_ERR_SPIKE_INDEX);
          }
        }
#pragma unroll
        for (int k = 0; k < 32; ++k)
          d[k] = __double2float_rn(__dadd_rn(__dmul_rn((double)(cf[k] & 0xFFu), s64), o64));
      }
      if constexpr (SR) {  // reserved values, imin then imax; only lanes whose run holds one
        // b4 / b8: per-quad round trip (8 sources x 4 Mi elements: b4 23.9 ->
        // 22.8 us, b8 28.3 -> 27.0 us); b3 / b2 were slower that way (25.2 ->
        // 26.7, 24.6 -> 24.9 us) and keep the whole-run round trip
        if (hit)
          subst_reserved<B == 4 || B == 8>(d, spill, (unsigned)ka < 32u, ka, smin, (unsigned)kz < 32u, kz, smax);
      }
#pragma unroll
      for (int k = 0; k < 32; k += 2) add2(acc[k], acc[k + 1], acc[k], acc[k + 1], d[k], d[k + 1]);
    }
    __syncwarp();  // every lane is done with this stage before it is refilled

    // ---- requantize the sums (registers) and store to every destination
    F32Vals v;
    v.st = nullptr;
    v.spill = spill;
#pragma unroll
    for (int k = 0; k < 32; ++k) v.f[k] = acc[k];
#pragma unroll
    for (int k = 0; k < 32; k += 4)  // rare exact paths read values back by index
      *reinterpret_cast<float4*>(spill + k) = make_float4(acc[k], acc[k + 1], acc[k + 2], acc[k + 3]);
    auto store = [&](const uint32_t* wv, int64_t e_, bool meta, int64_t moff, const uint32_t* rec, int rbb) {
      for (int dd = 0; dd < a.ndst; ++dd) {
        uint8_t* out = a.dst[dd] + doff;
#pragma unroll
        for (int u = 0; u < n_units(B); ++u) {
          const int W = unit_w(B, u), O = unit_off(B, u);
          uint8_t* p = out + (n * O) / 8 + (e_ * W) / 8;
          if (W == 1) store_words<1>(p, wv + LaneWords<B>::base(u));
          else if (W == 2) store_words<2>(p, wv + LaneWords<B>::base(u));
          else if (W == 4) store_words<4>(p, wv + LaneWords<B>::base(u));
          else store_words<8>(p, wv + LaneWords<B>::base(u));
        }
        if (meta) store_record(out + meta_off + moff, rec, rbb);
      }
    };
    encode_lane<B, SR, G>(v, active, active ? er : 0, cx, store);
    __syncwarp();
  }
}

template <int B, bool SR, int G>
struct RedRun {
  static constexpr int SMEM = RunTile<B, SR, G>::WARP_BYTES;
  // the tile's bulk copies need 16-byte aligned segments everywhere
  static bool ok(const ReduceArgs& a) {
    using RT = RunTile<B, SR, G>;
    if (a.nsrc > kRunStageSrc) return false;
    for (int s = 0; s < a.nsrc; ++s)
      if (reinterpret_cast<uintptr_t>(a.src[s]) & 15u) return false;
    if (a.nshard > 1 && (a.sstride & 15)) return false;
    for (int u = 1; u < n_units(B); ++u)
      if ((a.n * unit_off(B, u) / 8) & 15) return false;
    if ((a.n * B / 8) & 15) return false;
    const int rb = rec_bytes(SR, a.intlog != 0);
    if ((RT::GROUPS * rb) & 15) return false;
    return true;
  }
  static int go(const ReduceArgs& a0, cudaStream_t st) {
    ReduceArgs a = a0;
    const int64_t tps = (a.n + 1023) / 1024;
    a.total = tps * a.nshard;
    constexpr auto kern = k_reduce_run<B, SR, G>;
    smem_attr<kern>(SMEM);
    int64_t blocks = a.total;  // one tile per one-warp CTA: the block scheduler balances the tail
    if (FC2_RUN_STAGES == 2) {  // persistent warps, equal tile counts
      static int resident = 0;
      if (!resident) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, 32, SMEM);
        if (resident < 1) resident = 1;
      }
      const int64_t cap = (int64_t)num_sms() * resident;
      const int64_t per = (a.total + cap - 1) / cap;
      blocks = (a.total + per - 1) / per;
    }
    if (blocks < 1) blocks = 1;
    launch_pdl(kern, (unsigned)blocks, 32, SMEM, st, a);
    return cuda_check("k_reduce_run");
  }
};

}  // namespace fc2
