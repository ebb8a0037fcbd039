// fc2_kernels.cuh -- kernel templates + per-bitwidth launchers (instantiated in
// fc2_inst_b<B>.cu so the 8 bitwidths compile in parallel).
#pragma once
#include <atomic>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <utility>

#include "fc2_decode.cuh"
#include "fc2_encode.cuh"
#include "fc2_encode_group.cuh"
#include "fc2_reduce_group.cuh"

namespace fc2 {

// library state lives in fc2_codec.cu
int set_err(int code, const char* fmt, ...);
int cuda_check(const char* what);
int num_sms();

// Opt a kernel into `bytes` of dynamic shared memory, once per device (the
// attribute is per device; several GPUs may be driven from one process).
template <auto KERN>
inline void smem_attr(int bytes) {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.fetch_or(bit, std::memory_order_release);
  }
}

// ---------------------------------------------------------------------------
// job tables (passed by value as __grid_constant__ kernel parameters)
// ---------------------------------------------------------------------------

// Jobs per launch: the job table travels as a __grid_constant__ kernel
// parameter, so it is kept small (larger batches become several launches;
// the public limit per call is FC2_MAX_JOBS).
#ifndef FC2_KERNEL_JOBS
#define FC2_KERNEL_JOBS 64
#endif

struct EncJob {
  const void* x;
  uint8_t* out;
  // row gather (MoE token dispatch): element e of the chunk is x[rows[e / row_len] * row_len + e % row_len]
  // (nullptr: x is the chunk itself)
  const int32_t* rows;
  int64_t n_valid, n, t0;  // t0: first global tile (fast) / group (generic)
};
struct EncBatch {
  int nj, B, G, sr, intlog, theta;
  int lpg;  // lanes per group of the bf16 lane-per-group encoder (enc_lpg / enc_lpg_small)
  int row_len;  // elements per gathered row (jobs with rows != nullptr; a multiple of 8)
  int64_t total;
  const double* lut;
  int32_t* err;
  EncJob j[FC2_KERNEL_JOBS];
};

struct DecJob {
  const uint8_t* pay;
  void* y;
  int64_t n, n_out, t0;
};
struct DecBatch {
  int nj, B, G, sr, intlog, theta;
  int round_bf16;  // snap float32 outputs to the bf16 grid (collectives.py:185-186)
  int64_t total;
  const double* lut;
  int32_t* err;
  DecJob j[FC2_KERNEL_JOBS];
};

#define FC2_MAX_PEERS 16
struct ReduceArgs {
  int nsrc, ndst, B, G, sr, intlog, theta;
  int64_t n, total;
  int64_t nshard, sstride, dstride;  // independent shards: shard k at src[s] + k sstride, dst[d] + k dstride
  const double* lut;
  int32_t* err;
  const uint8_t* src[FC2_MAX_PEERS];
  uint8_t* dst[FC2_MAX_PEERS];
};

template <class Batch>
__device__ __forceinline__ int find_job(const Batch& b, int64_t t) {
  if (b.nj == 1) return 0;  // the common single-chunk launch: no search
  int lo = 0, hi = b.nj - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (b.j[mid].t0 <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// fast encoder
// ---------------------------------------------------------------------------

constexpr int kEncWarps = 4;   // warps per CTA
constexpr int kStages = 3;     // cp.async pipeline depth per warp

template <typename T>
struct Stage {
  static constexpr int EPC = 16 / sizeof(T);   // elements per 16-byte chunk
  static constexpr int CPL = 32 / EPC;         // chunks per lane (32 elements)
  static constexpr int CHUNKS = 32 * CPL;      // chunks per warp tile
  static constexpr int BYTES = CHUNKS * 16;    // bytes per warp tile stage
  // XOR swizzle: conflict-free for both the coalesced fill (chunk c = l + 32j)
  // and the per-lane read-back (chunks CPL*l .. CPL*l + CPL - 1)
  __device__ static __forceinline__ int pos(int c) { return swz<CPL>(c); }
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <typename T>
__device__ __forceinline__ void issue_tile(const EncBatch& b, int64_t t, uint8_t* stage) {
  using S = Stage<T>;
  const int ji = find_job(b, t);
  const EncJob& jb = b.j[ji];
  const int64_t e_base = (t - jb.t0) * 1024;
  const int lane = (int)lane_id();
  const T* x = reinterpret_cast<const T*>(jb.x);
#pragma unroll
  for (int j = 0; j < S::CPL; ++j) {
    const int c = lane + 32 * j;
    const int64_t e = e_base + (int64_t)c * S::EPC;
    int64_t valid = jb.n_valid - e;
    valid = valid < 0 ? 0 : (valid > S::EPC ? S::EPC : valid);
    const T* p = x + e;
    if (jb.rows && valid > 0) {  // gathered rows (row_len % 8 == 0: a chunk never straddles rows)
      const uint32_t q = (uint32_t)e / (uint32_t)b.row_len;
      p = x + (int64_t)__ldg(jb.rows + q) * b.row_len + ((uint32_t)e - q * (uint32_t)b.row_len);
    }
    const void* src = valid > 0 ? (const void*)p : (const void*)x;
    cp_async16(stage + S::pos(c) * 16, src, (int)(valid * sizeof(T)));
  }
}

template <typename T, int B, bool SR, int G>
__global__ void __launch_bounds__(kEncWarps * 32) k_encode_fast(const __grid_constant__ EncBatch b) {
  using S = Stage<T>;
  extern __shared__ __align__(16) uint8_t smem[];
  const int warp = (int)(threadIdx.x >> 5), lane = (int)lane_id();
  uint8_t* my = smem + warp * kStages * S::BYTES;
  const int64_t nw = (int64_t)gridDim.x * kEncWarps;
  int64_t t = (int64_t)blockIdx.x * kEncWarps + warp;

  // prologue: put kStages-1 tiles in flight
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    const int64_t tt = t + s * nw;
    if (tt < b.total) issue_tile<T>(b, tt, my + s * S::BYTES);
    cp_async_commit();
  }
  int stage = 0;
  for (; t < b.total; t += nw) {
    {  // refill the slot consumed in the previous iteration
      const int64_t tt = t + (kStages - 1) * nw;
      const int s = (stage + kStages - 1) % kStages;
      if (tt < b.total) issue_tile<T>(b, tt, my + s * S::BYTES);
      cp_async_commit();
    }
    cp_async_wait<kStages - 1>();
    __syncwarp();
    const uint8_t* st = my + stage * S::BYTES;

    const int ji = find_job(b, t);
    const EncJob& jb = b.j[ji];
    const int64_t e0 = (t - jb.t0) * 1024 + lane * 32;
    const bool active = e0 < jb.n;
    EncCtx cx;
    cx.n = jb.n;
    cx.meta_off = jb.n * B / 8;
    cx.intlog = b.intlog;
    cx.theta = b.theta;
    cx.lut = b.lut;
    cx.err = b.err;
    uint8_t* out = jb.out;
    auto store = [&](const uint32_t* w, int64_t e0_, bool meta, int64_t moff, const uint32_t* rec, int rb) {
#pragma unroll
      for (int u = 0; u < n_units(B); ++u) {
        const int W = unit_w(B, u), O = unit_off(B, u);
        uint8_t* p = out + (cx.n * O) / 8 + (e0_ * W) / 8;
        if (W == 1) store_words<1>(p, w + LaneWords<B>::base(u));
        else if (W == 2) store_words<2>(p, w + LaneWords<B>::base(u));
        else if (W == 4) store_words<4>(p, w + LaneWords<B>::base(u));
        else store_words<8>(p, w + LaneWords<B>::base(u));
      }
      if (meta) store_record(out + cx.meta_off + moff, rec, rb);
    };
    if constexpr (sizeof(T) == 2) {
      Bf16Vals v;
      v.st = st;
#pragma unroll
      for (int j = 0; j < S::CPL; ++j) {
        uint4 q = *reinterpret_cast<const uint4*>(st + S::pos(S::CPL * lane + j) * 16);
        v.w[4 * j] = q.x; v.w[4 * j + 1] = q.y; v.w[4 * j + 2] = q.z; v.w[4 * j + 3] = q.w;
      }
      __syncwarp();
      encode_lane<B, SR, G>(v, active, e0, cx, store);
    } else {
      F32Vals v;
      v.st = st;
      v.spill = nullptr;
#pragma unroll
      for (int j = 0; j < S::CPL; ++j) {
        float4 q = *reinterpret_cast<const float4*>(st + S::pos(S::CPL * lane + j) * 16);
        v.f[4 * j] = q.x; v.f[4 * j + 1] = q.y; v.f[4 * j + 2] = q.z; v.f[4 * j + 3] = q.w;
      }
      __syncwarp();
      encode_lane<B, SR, G>(v, active, e0, cx, store);
    }
    __syncwarp();  // every lane is done with this slot before it is refilled
    stage = (stage + 1) % kStages;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// lane-per-group encoder (bf16 input, G in {32,64,128,256})
// ---------------------------------------------------------------------------

template <int G, int LPG>
__device__ __forceinline__ void issue_grp_tile(const EncJob& jb, int64_t t, uint8_t* stage, int row_len) {
  using IT = GTile<__nv_bfloat16, G, LPG>;
  constexpr int GPT = 32 / LPG;  // groups per warp tile
  const int64_t e0 = (t - jb.t0) * GPT * G;
  const int lane = (int)lane_id();
  const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(jb.x);
  constexpr int NJ = IT::CPG / LPG;  // 16-byte chunks per lane
  if (jb.rows) {  // MoE dispatch: gathered token rows (a 16-byte chunk never straddles rows)
    const uint32_t H = (uint32_t)row_len;
    uint32_t e = (uint32_t)(e0 + 8 * lane);  // chunk lane + 32 j starts at element e + 256 j
    uint32_t q = e / H, r = e - q * H;
#pragma unroll 4
    for (int j = 0; j < NJ; ++j) {
      const int tc = lane + 32 * j;
      const int64_t v = jb.n_valid - (int64_t)e;
      const int valid = v <= 0 ? 0 : (v >= 8 ? 8 : (int)v);
      const void* src = valid > 0 ? (const void*)(x + (int64_t)__ldg(jb.rows + q) * H + r) : (const void*)x;
      cp_async16(stage + IT::in_pos(tc / IT::CPG, tc % IT::CPG) * 16, src, valid * 2);
      e += 256;
      r += 256;
      while (r >= H) { r -= H; ++q; }
    }
  } else if (e0 + GPT * G <= jb.n_valid) {  // whole tile present: plain 16-byte copies
    const uint8_t* src = reinterpret_cast<const uint8_t*>(x + e0);
    if constexpr (IT::CPG <= 32 && 32 % IT::CPG == 0 && NJ > 8) {
      // chunk lane + 32 j: group g0 + K j, column c; the swizzle only sees
      // (group & 7), so slots repeat every 8 j with a 256-chunk stride
      constexpr int K = 32 / IT::CPG;
      const int g0 = lane / IT::CPG, c = lane % IT::CPG;
      int sb[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) sb[j] = IT::in_pos(g0 + K * j, c) * 16;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        cp_async16(stage + sb[j % 8] + (j / 8) * (8 * K * IT::CPG * 16), src + 16 * (lane + 32 * j), 16);
    } else {
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int tc = lane + 32 * j;
        cp_async16(stage + IT::in_pos(tc / IT::CPG, tc % IT::CPG) * 16, src + 16 * tc, 16);
      }
    }
  } else {  // tail tile: zero-fill past n_valid (the padding of collectives.py:167-172)
    const int64_t rem = jb.n_valid - e0;  // may be <= 0
#pragma unroll 4
    for (int j = 0; j < IT::CPG / LPG; ++j) {
      const int tc = lane + 32 * j;
      const int64_t v = rem - (int64_t)tc * 8;
      const int valid = v <= 0 ? 0 : (v >= 8 ? 8 : (int)v);
      const void* src = valid > 0 ? (const void*)(x + e0 + (int64_t)tc * 8) : (const void*)x;
      cp_async16(stage + IT::in_pos(tc / IT::CPG, tc % IT::CPG) * 16, src, valid * 2);
    }
  }
}

// Register budget per thread of the lane-per-group encoder: 85 lets 24 warps
// (8.5 KB of smem each with direct output) share an SM; B = 8 (16 plane words
// per run pair) and B = 7 (three planes) need more to stay spill-free.
#ifndef FC2_ENC_REGS
#define FC2_ENC_REGS 85
#endif
__host__ __device__ constexpr int enc_min_ctas(int B, int warps) {
  return 65536 / (warps * 32 * (B == 7 ? 128 : (B == 8 ? 102 : FC2_ENC_REGS)));
}
// one warp tile of the lane-per-group encoder: tile index t in the tile
// numbering of shape LPG (32 / LPG groups per tile)
template <int B, bool SR, int G, int LPG>
__device__ __forceinline__ void encode_grp_tile(const EncBatch& b, int64_t t, uint8_t* in0, uint32_t* tms) {
  constexpr int GPT = 32 / LPG;  // groups per warp tile
  const int lane = (int)lane_id();
  const EncJob& jb = b.j[find_job(b, t)];  // one lookup per tile
  __syncwarp();  // previous tile fully consumed
  issue_grp_tile<G, LPG>(jb, t, in0, b.row_len);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  const int64_t ngroups = jb.n / G;
  const int64_t tg0 = (t - jb.t0) * GPT;
  const int64_t gabs = tg0 + lane / LPG;
  const int ng = (int)min((int64_t)GPT, ngroups - tg0);
  EncCtx cx;
  cx.n = jb.n;
  cx.meta_off = jb.n * B / 8;
  cx.intlog = b.intlog;
  cx.theta = b.theta;
  cx.lut = b.lut;
  cx.err = b.err;
  encode_tile_bf16<B, SR, G, LPG>(in0, tms, gabs < ngroups, gabs, cx, jb.out, tg0, ng);
}

template <int B, bool SR, int G, int WARPS, int LPG>
__global__ void __launch_bounds__(WARPS * 32, enc_min_ctas(B, WARPS)) k_encode_grp(const __grid_constant__ EncBatch b) {
  pdl_enter();
  using IT = GTile<__nv_bfloat16, G, LPG>;
  constexpr int IN_BYTES = IT::IN_BYTES / LPG;
  constexpr int TIE_BYTES = G / LPG * 4;               // one 32-bit tie mask per run per lane
  constexpr int PER_WARP = IN_BYTES + TIE_BYTES;       // plane words go straight to global
  extern __shared__ __align__(16) uint8_t smem[];
  const int warp = (int)(threadIdx.x >> 5);
  uint8_t* in0 = smem + warp * PER_WARP;
  uint32_t* tms = reinterpret_cast<uint32_t*>(in0 + IN_BYTES);
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  for (int64_t t = (int64_t)blockIdx.x * WARPS + warp; t < b.total; t += nw)
    encode_grp_tile<B, SR, G, LPG>(b, t, in0, tms);
}

#ifndef FC2_ENC_WARPS
#define FC2_ENC_WARPS 1  // one-warp CTAs: finest block-scheduling grain for the last wave
#endif
#ifndef FC2_ENC_CTAS_PER_SM
#define FC2_ENC_CTAS_PER_SM 128
#endif

template <int B, bool SR, int G>
struct EncGrp {
  static constexpr int WARPS = FC2_ENC_WARPS;
  // the launcher picked b.lpg: enc_lpg(G) for bandwidth, enc_lpg_small(G)
  // (one 32-element run per lane; ~2x the instructions per element, 4x the
  // warps at g = 128) for chunks smaller than a wave
  static int go(const EncBatch& b, cudaStream_t st) {
    constexpr int S = enc_lpg_small(G), L = enc_lpg(G);
    if (b.lpg == S && S != L) return run<S>(b, st);
    return run<L>(b, st);
  }
  template <int LPG>
  static int run(const EncBatch& b, cudaStream_t st) {
    constexpr int SMEM = WARPS * (GTile<__nv_bfloat16, G>::IN_BYTES / LPG + G / LPG * 4);
    constexpr auto kern = k_encode_grp<B, SR, G, WARPS, LPG>;
    smem_attr<kern>(SMEM);
    int64_t blocks = (b.total + WARPS - 1) / WARPS;
    int64_t cap = (int64_t)num_sms() * FC2_ENC_CTAS_PER_SM;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    launch_pdl(kern, (unsigned)blocks, WARPS * 32, SMEM, st, b);
    return cuda_check("k_encode_grp");
  }
};

// ---------------------------------------------------------------------------
// generic encoder: warp per group, exact float64
// ---------------------------------------------------------------------------

template <typename T>
struct PlainLoader {
  const T* x;
  int64_t nv;
  __device__ double operator()(int64_t i) const { return load_elem<T>(x, i, nv); }
};

// gathered rows (MoE token dispatch): element i of the chunk is
// x[rows[i / H] * H + i % H]; zero past n_valid (the chunk's padding)
template <typename T>
struct RowLoader {
  const T* x;
  const int32_t* rows;
  int64_t nv, H;
  __device__ double operator()(int64_t i) const {
    if (i >= nv) return 0.0;
    const int64_t q = i / H;
    return load_elem<T>(x, (int64_t)__ldg(rows + q) * H + (i - q * H), INT64_MAX);
  }
};

template <typename T>
__global__ void __launch_bounds__(256) k_encode_gen(const __grid_constant__ EncBatch b) {
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < b.total; g += nw) {
    const int ji = find_job(b, g);
    const EncJob& jb = b.j[ji];
    EncCtx cx;
    cx.n = jb.n;
    cx.meta_off = jb.n * b.B / 8;
    cx.intlog = b.intlog;
    cx.theta = b.theta;
    cx.lut = b.lut;
    cx.err = b.err;
    OutList o;
    o.p[0] = jb.out;
    o.nd = 1;
    if (jb.rows) {
      RowLoader<T> ld{reinterpret_cast<const T*>(jb.x), jb.rows, jb.n_valid, b.row_len};
      generic_encode_group(ld, o, jb.n, g - jb.t0, b.B, b.G, b.sr != 0, cx);
    } else {
      PlainLoader<T> ld{reinterpret_cast<const T*>(jb.x), jb.n_valid};
      generic_encode_group(ld, o, jb.n, g - jb.t0, b.B, b.G, b.sr != 0, cx);
    }
  }
}

// ---------------------------------------------------------------------------
// decoders
// ---------------------------------------------------------------------------

template <typename OT>
__device__ __forceinline__ OT cvt_out(float v);
template <>
__device__ __forceinline__ float cvt_out<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(float v) {
  return __ushort_as_bfloat16((unsigned short)bf16_bits(v));  // bfloat16.py:16-25
}


// fast decode (G % 32 == 0): lane = 32 consecutive elements (one metadata
// record per lane), next tile's codes + record prefetched into registers,
// values staged in smem (swizzled) so the warp stores 16-byte chunks
// contiguously; reserved spikes are patched in the stage.
template <int B>
struct RunRegs {
  uint32_t w[B];   // packed code words of the 32-element run (unit 0 words first)
  uint32_t r[3];   // metadata record
};

// Decode v4: warp tile = 4096 elements, lane = 128 consecutive elements
// (4 runs of 32).  The tile's code planes are cp.async-staged (2 stages,
// XOR-swizzled per-lane words); the lane's metadata record(s) come straight
// from global (one record per lane when G >= 128); values are staged in smem
// and written back with coalesced 16-byte stores.  Requires G % 32 == 0.
#ifndef FC2_DEC_WARPS
#define FC2_DEC_WARPS 1  // one-warp CTAs (28 resident per SM by registers; finest tail grain)
#endif
constexpr int kDecWarps = FC2_DEC_WARPS;
constexpr int kDecElems = 128;            // elements per lane (4 runs of 32)
constexpr int kDecTile = 32 * kDecElems;  // elements per warp tile
#ifndef FC2_DEC_STAGES
#define FC2_DEC_STAGES 1  // the launch gives every warp one tile: a second input stage would sit idle
#endif
constexpr int kDecStages = FC2_DEC_STAGES;

template <int B>
struct DecIn {
  // unit u of the tile: kDecTile*W/8 bytes = per lane kDecElems*W/8 bytes
  __host__ __device__ static constexpr int off(int u) {
    return u == 0 ? 0 : off(u - 1) + kDecTile * unit_w(B, u - 1) / 8;
  }
  static constexpr int BYTES = kDecTile * B / 8;
  // lane l's bytes of unit u: [16*W*l, 16*W*(l+1)); chunk k of lane l (16 B):
  // swizzled slot so that both the coalesced fill and the per-lane reads are
  // bank-conflict free
  template <int W>
  __device__ static __forceinline__ int slot(int l, int k) {
    constexpr int CPL = W;  // 16*W bytes per lane = W chunks
    if constexpr (CPL == 1) return l;
    else return (l * CPL + k) ^ (((l * CPL + k) >> 3) & (CPL - 1));
  }
};

template <typename OT, int B>
__global__ void __launch_bounds__(kDecWarps * 32) k_decode_fast(const __grid_constant__ DecBatch b) {
  pdl_enter();
  constexpr int ESZ = (int)sizeof(OT);
  constexpr int OUT_BYTES = kDecTile / 2 * ESZ;  // half a tile: runs (0,1) then (2,3) of every lane
  constexpr int PER_WARP = kDecStages * DecIn<B>::BYTES + OUT_BYTES;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int warp = (int)(threadIdx.x >> 5), lane = (int)lane_id();
  uint8_t* in0 = dsm + warp * PER_WARP;
  uint8_t* ost = in0 + kDecStages * DecIn<B>::BYTES;
  const int64_t nw = (int64_t)gridDim.x * kDecWarps;
  const int rb = rec_bytes(b.sr, b.intlog);
  const int G = b.G;

  // cp.async the code planes of tile tt into stage buffer st (zero-fill past n)
  auto issue = [&](int64_t tt, uint8_t* st) {
    if (tt >= b.total) return;
    const DecJob& jb = b.j[find_job(b, tt)];
    const int64_t e0 = (tt - jb.t0) * kDecTile;
#pragma unroll
    for (int u = 0; u < n_units(B); ++u) {
      const int W = unit_w(B, u), O = unit_off(B, u);
      const uint8_t* src = jb.pay + (jb.n * O) / 8 + e0 * W / 8;
      const int64_t avail = (jb.n - e0) * W / 8;  // bytes of this plane left in the chunk
      const bool full = avail >= 512 * W;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const int c = lane + 32 * k;  // linear chunk of the tile segment
        const int l = c / W, kk = c % W;
        int bytes = 16;
        if (!full) {
          const int64_t v = avail - (int64_t)c * 16;
          bytes = v <= 0 ? 0 : (v >= 16 ? 16 : (int)v);
        }
        uint8_t* dst = st + DecIn<B>::off(u) + 16 * (W == 1 ? DecIn<B>::template slot<1>(l, kk)
                                                 : W == 2 ? DecIn<B>::template slot<2>(l, kk)
                                                 : W == 4 ? DecIn<B>::template slot<4>(l, kk)
                                                          : DecIn<B>::template slot<8>(l, kk));
        cp_async16(dst, bytes ? (const void*)(src + 16 * c) : (const void*)jb.pay, bytes);
      }
    }
  };

  int64_t t = (int64_t)blockIdx.x * kDecWarps + warp;
  issue(t, in0);
  cp_async_commit();
  int stage = 0;
  for (; t < b.total; t += nw) {
    const DecJob& jb = b.j[find_job(b, t)];
    const int64_t ebase = (t - jb.t0) * kDecTile;
    const int64_t e0 = ebase + (int64_t)lane * kDecElems;
    const uint8_t* st = in0 + stage * DecIn<B>::BYTES;
    // metadata record of this lane's first group (in flight with the codes)
    uint32_t rec[3] = {0, 0, 0};
    // group of the lane's first element; gin = offset inside it (no 64-bit division)
    int64_t grp;
    if ((G & (G - 1)) == 0) grp = e0 >> (__ffs(G) - 1);
    else if (e0 < 0x7fffffff) grp = (int64_t)((uint32_t)e0 / (uint32_t)G);
    else grp = e0 / G;
    int gin = (int)(e0 - grp * G);
    const bool live = e0 < jb.n;
    if (live) load_record(jb.pay + jb.n * B / 8 + grp * rb, rec, rb);
    if constexpr (kDecStages == 2) {  // prefetch this warp's next tile (grids that loop)
      issue(t + nw, in0 + (stage ^ 1) * DecIn<B>::BYTES);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    constexpr int CPR = 32 * (int)sizeof(OT) / 16;  // output chunks per run
    constexpr int CPH = 2 * CPR;                     // output chunks per lane per half
    GroupMeta m;
    {
      auto decode_meta = [&]() {
        m.imin = m.imax = -1;
        m.smin = m.smax = 0.f;
        m.s64 = 0.0; m.o64 = 0.0;
        if (!b.intlog) {
          m.s32 = bf16_val(rec[0] & 0xFFFFu);
          m.z32 = bf16_val(rec[0] >> 16);
          if (b.sr) {
            m.smin = bf16_val(rec[1] & 0xFFFFu);
            m.smax = bf16_val(rec[1] >> 16);
            const float fi = bf16_val(rec[2] & 0xFFFFu), fa = bf16_val(rec[2] >> 16);
            if ((fi > -1.0f) && (fi < (float)G) && (fa > -1.0f) && (fa < (float)G)) {
              m.imin = (int)fi; m.imax = (int)fa;
            } else {
              atomicOr(b.err, FC2_ERR_SPIKE_INDEX);
            }
          }
        } else {
          const int si = (int)(int8_t)(rec[0] & 0xFFu), zi = (int)(int8_t)((rec[0] >> 8) & 0xFFu);
          m.s64 = si == -128 ? 0.0 : b.lut[si + 128];
          m.o64 = __dmul_rn(-(double)zi, m.s64);
          m.s32 = 0.f; m.z32 = 0.f;
          if (b.sr) {
            m.smin = bf16_val(rec[0] >> 16);
            m.smax = bf16_val(rec[1] & 0xFFFFu);
            const int ii = (int)((rec[1] >> 16) & 0xFFu), ia = (int)(rec[1] >> 24);
            if (ii < G && ia < G) { m.imin = ii; m.imax = ia; }
            else atomicOr(b.err, FC2_ERR_SPIKE_INDEX);
          }
        }
      };
      // Reserved values of the current group: lane-relative positions (0..127,
      // else outside this lane's span) and their stage byte offsets, computed
      // once per group; patch_spikes(h) writes those in half h (the half now in
      // the stage), imin first, then imax (codec.py:559-561).
      int kmin = -1, kmax = -1, omin = 0, omax = 0;
      OT vmin{}, vmax{};
      auto spike_pos = [&]() {
        auto pos = [&](int idx, int& kk, int& off) {
          const int64_t k = grp * G + idx - e0;
          kk = (idx >= 0 && k >= 0 && k < kDecElems && grp * G + idx < jb.n) ? (int)k : -1;
          const int kh = kk & (kDecElems / 2 - 1);
          const int c = CPH * lane + kh / (16 / (int)sizeof(OT));
          off = 16 * (c ^ ((c >> 3) & 7)) + (kh % (16 / (int)sizeof(OT))) * (int)sizeof(OT);
        };
        pos(m.imin, kmin, omin);
        pos(m.imax, kmax, omax);
        float a = m.smin, z = m.smax;
        if (sizeof(OT) == 4 && b.round_bf16) { a = bf16_val(bf16_bits(a)); z = bf16_val(bf16_bits(z)); }
        vmin = cvt_out<OT>(a);
        vmax = cvt_out<OT>(z);
      };
      auto patch_spikes = [&](int h) {
        if (kmin >= 0 && (kmin >> 6) == h) *reinterpret_cast<OT*>(ost + omin) = vmin;
        if (kmax >= 0 && (kmax >> 6) == h) *reinterpret_cast<OT*>(ost + omax) = vmax;
      };
      if (live) {
        decode_meta();
        if (b.sr) spike_pos();
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
      if (live) {
#pragma unroll 1
      for (int r = 2 * h; r < 2 * h + 2; ++r) {
        const int64_t er = e0 + 32 * r;
        if (er >= jb.n) break;
        if (r > 0) gin += 32;
        if (gin >= G) {  // next group (G < 128): finish the previous one first
          if (b.sr) patch_spikes(h);
          gin -= G;
          grp += 1;
          load_record(jb.pay + jb.n * B / 8 + grp * rb, rec, rb);
          decode_meta();
          if (b.sr) spike_pos();
        }
        // ---- codes of this 32-element run from the stage
        RunRegs<B> rr;
#pragma unroll
        for (int u = 0; u < n_units(B); ++u) {
          const int W = unit_w(B, u), O = unit_off(B, u);
          const uint8_t* base = st + DecIn<B>::off(u);
          if (W == 8) {
            const int k0 = 2 * r;
            const uint4 q0 = *reinterpret_cast<const uint4*>(base + 16 * DecIn<B>::template slot<8>(lane, k0));
            const uint4 q1 = *reinterpret_cast<const uint4*>(base + 16 * DecIn<B>::template slot<8>(lane, k0 + 1));
            rr.w[O + 0] = q0.x; rr.w[O + 1] = q0.y; rr.w[O + 2] = q0.z; rr.w[O + 3] = q0.w;
            rr.w[O + 4] = q1.x; rr.w[O + 5] = q1.y; rr.w[O + 6] = q1.z; rr.w[O + 7] = q1.w;
          } else if (W == 4) {
            const uint4 q0 = *reinterpret_cast<const uint4*>(base + 16 * DecIn<B>::template slot<4>(lane, r));
            rr.w[O + 0] = q0.x; rr.w[O + 1] = q0.y; rr.w[O + 2] = q0.z; rr.w[O + 3] = q0.w;
          } else if (W == 2) {
            const uint2 q0 = *reinterpret_cast<const uint2*>(base + 16 * DecIn<B>::template slot<2>(lane, r >> 1) + 8 * (r & 1));
            rr.w[O + 0] = q0.x; rr.w[O + 1] = q0.y;
          } else {
            rr.w[O] = *reinterpret_cast<const uint32_t*>(base + 16 * DecIn<B>::template slot<1>(lane, 0) + 4 * r);
          }
        }
        // ---- codes -> exact floats (2^23 + code, as bit patterns)
        uint32_t cf[32];
        run_code_floats<B>(rr.w, cf);
        // ---- values
        float v[32];
        if (!b.intlog) {
#pragma unroll
          for (int k = 0; k < 32; k += 2) {
            float a0, a1;
            add2(a0, a1, __uint_as_float(cf[k]), __uint_as_float(cf[k + 1]), -8388608.0f, -8388608.0f);
            fma2(v[k], v[k + 1], a0, a1, m.s32, m.s32, m.z32, m.z32);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = dq32(cf[k] & 0xFFu, m, true);
        }
        if constexpr (sizeof(OT) == 4) {
          if (b.round_bf16) {
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = bf16_val(bf16_bits(v[k]));
          }
        }
        // ---- stage: this run's CPR chunks of the lane's half segment
        // (CPH is a multiple of 8, so (c >> 3) & 7 only sees the lane and the
        // chunk's 8-block: slot = c ^ sw)
        const int cbase = CPH * lane + CPR * (r & 1);
#pragma unroll
        for (int j = 0; j < CPR; ++j) {
          uint4 q;
          if constexpr (sizeof(OT) == 2) {
            __nv_bfloat162 h0 = __floats2bfloat162_rn(v[8 * j], v[8 * j + 1]);
            __nv_bfloat162 h1 = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
            __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]);
            __nv_bfloat162 h3 = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
            q = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                           *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
          } else {
            q = make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]), __float_as_uint(v[4 * j + 2]),
                           __float_as_uint(v[4 * j + 3]));
          }
          const int c = cbase + j;
          *reinterpret_cast<uint4*>(ost + 16 * (c ^ ((c >> 3) & 7))) = q;
        }
      }
      if (b.sr) patch_spikes(h);
      }
      __syncwarp();
      // ---- coalesced copy-out of half h, bounded by n_out: stage chunk q
      // (lane q / CPH, chunk q % CPH of its half) -> elements
      // 128 (q / CPH) + 64 h + EPC (q % CPH) of the tile; 32 consecutive q
      // cover whole 128-byte segments
      OT* y = reinterpret_cast<OT*>(jb.y) + ebase;
      const int64_t valid = jb.n_out - ebase;
      constexpr int EPC = 16 / ESZ;
      constexpr int NCH = kDecTile / 2 / EPC;
      if (valid >= kDecTile && (reinterpret_cast<uintptr_t>(y) & 15u) == 0) {
        // q = lane + 32 i: lane q / CPH = lane / CPH + (32 / CPH) i, chunk q % CPH = lane % CPH;
        // slot q ^ ((q >> 3) & 7) = 32 i + (lane ^ s_i), s_i = ((lane >> 3) + 4 i) & 7
        OT* yl = y + kDecElems * (lane / CPH) + 64 * h + EPC * (lane % CPH);
        const uint8_t* s0 = ost + 16 * (lane ^ ((lane >> 3) & 7));
        const uint8_t* s1 = ost + 16 * (lane ^ (((lane >> 3) + 4) & 7));
#pragma unroll
        for (int i = 0; i < NCH / 32; ++i)
          *reinterpret_cast<uint4*>(yl + (32 / CPH) * kDecElems * i) =
              *reinterpret_cast<const uint4*>((i & 1 ? s1 : s0) + 512 * i);
      } else {
        for (int i = lane; i < kDecTile / 2; i += 32) {
          const int q = i / EPC;
          const int64_t e = kDecElems * (q / CPH) + 64 * h + EPC * (q % CPH) + i % EPC;
          if (e < valid) y[e] = *reinterpret_cast<const OT*>(ost + 16 * (q ^ ((q >> 3) & 7)) + (i % EPC) * ESZ);
        }
      }
      __syncwarp();
      }
    }
    __syncwarp();
    if constexpr (kDecStages == 2) {
      stage ^= 1;
    } else if (t + nw < b.total) {  // single stage: refill it for the next tile
      issue(t + nw, in0);
      cp_async_commit();
    }
  }
  cp_async_wait<0>();
}

template <typename OT, int B>
int launch_decode_fast(const DecBatch& b, cudaStream_t st) {
  constexpr int SMEM = kDecWarps * (kDecStages * DecIn<B>::BYTES + kDecTile / 2 * (int)sizeof(OT));
  constexpr auto kern = k_decode_fast<OT, B>;
  smem_attr<kern>(SMEM);
  // one tile per warp: the block scheduler balances the tail (no persistent loop)
  int64_t blocks = (b.total + kDecWarps - 1) / kDecWarps;
  const int64_t cap = (int64_t)num_sms() * 64;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  launch_pdl(kern, (unsigned)blocks, kDecWarps * 32, SMEM, st, b);
  return cuda_check("k_decode_fast");
}

// generic decode: thread per element (any G, any output type)
template <typename OT>
__global__ void __launch_bounds__(256) k_decode_gen(const __grid_constant__ DecBatch b) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < b.total; t += stride) {
    const int ji = find_job(b, t);
    const DecJob& jb = b.j[ji];
    const int64_t e = t - jb.t0;
    if (e >= jb.n_out) continue;
    DecCtx c;
    c.n = jb.n; c.meta_off = jb.n * b.B / 8; c.B = b.B; c.G = b.G; c.sr = b.sr; c.intlog = b.intlog;
    c.theta = b.theta; c.lut = b.lut; c.err = b.err;
    OT* y = reinterpret_cast<OT*>(jb.y);
    if constexpr (sizeof(OT) == 8) {
      y[e] = decode_elem64(jb.pay, e, c);
    } else {
      float v = decode_elem32(jb.pay, e, c);
      if (b.round_bf16) v = bf16_val(bf16_bits(v));
      y[e] = cvt_out<OT>(v);
    }
  }
}

// ---------------------------------------------------------------------------
// reduce + requantize (two-step middle stage)
// ---------------------------------------------------------------------------

constexpr int kRedWarps = 4;

template <int B, bool SR, int G>
__global__ void __launch_bounds__(kRedWarps * 32) k_reduce_fast(const __grid_constant__ ReduceArgs a) {
  // per-lane spill region for the spike patch: 36 floats (padded, conflict-free)
  __shared__ __align__(16) float sp[kRedWarps * 32 * 36];
  const int warp = (int)(threadIdx.x >> 5), lane = (int)lane_id();
  float* mine = sp + (warp * 32 + lane) * 36;
  const int64_t nw = (int64_t)gridDim.x * kRedWarps;
  DecCtx dc;
  dc.n = a.n; dc.meta_off = a.n * B / 8; dc.B = B; dc.G = G; dc.sr = SR; dc.intlog = a.intlog;
  dc.theta = a.theta; dc.lut = a.lut; dc.err = a.err;
  EncCtx cx;
  cx.n = a.n; cx.meta_off = a.n * B / 8; cx.intlog = a.intlog; cx.theta = a.theta; cx.lut = a.lut;
  cx.err = a.err;
  for (int64_t t = (int64_t)blockIdx.x * kRedWarps + warp; t < a.total; t += nw) {
    const int64_t e0 = t * 1024 + lane * 32;
    const bool active = e0 < a.n;
    const int64_t ec = active ? e0 : 0;
    F32Vals acc;
    acc.st = nullptr;
    acc.spill = mine;
#pragma unroll
    for (int k = 0; k < 32; ++k) acc.f[k] = 0.0f;  // acc = zeros(float32) (collectives.py:293)
    const int64_t grp = ec / G;
    const int il = (int)(ec - grp * G);  // element offset of this lane inside its group
    for (int s = 0; s < a.nsrc; ++s) {
      GroupMeta m = read_meta(a.src[s], grp, dc);
      float d[32];
      dq_run32<B>(a.src[s], a.n, ec, m, a.intlog != 0, d);
      if constexpr (SR) {
        const bool hit_a = m.imin >= il && m.imin < il + 32;
        const bool hit_z = m.imax >= il && m.imax < il + 32;
        if (__any_sync(0xffffffffu, hit_a || hit_z)) {
#pragma unroll
          for (int k = 0; k < 32; k += 4) *reinterpret_cast<float4*>(mine + k) = make_float4(d[k], d[k + 1], d[k + 2], d[k + 3]);
          if (hit_a) mine[m.imin - il] = m.smin;
          if (hit_z) mine[m.imax - il] = m.smax;
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            float4 q = *reinterpret_cast<const float4*>(mine + k);
            d[k] = q.x; d[k + 1] = q.y; d[k + 2] = q.z; d[k + 3] = q.w;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) acc.f[k] = __fadd_rn(acc.f[k], d[k]);  // acc += dq (rank order)
    }
    auto store = [&](const uint32_t* w, int64_t e0_, bool meta, int64_t moff, const uint32_t* rec, int rb) {
      for (int dd = 0; dd < a.ndst; ++dd) {
        uint8_t* out = a.dst[dd];
#pragma unroll
        for (int u = 0; u < n_units(B); ++u) {
          const int W = unit_w(B, u), O = unit_off(B, u);
          uint8_t* p = out + (a.n * O) / 8 + (e0_ * W) / 8;
          if (W == 1) store_words<1>(p, w + LaneWords<B>::base(u));
          else if (W == 2) store_words<2>(p, w + LaneWords<B>::base(u));
          else if (W == 4) store_words<4>(p, w + LaneWords<B>::base(u));
          else store_words<8>(p, w + LaneWords<B>::base(u));
        }
        if (meta) store_record(out + cx.meta_off + moff, rec, rb);
      }
    };
#pragma unroll
    for (int k = 0; k < 32; k += 4)  // spill the sums for the rare exact path
      *reinterpret_cast<float4*>(mine + k) = make_float4(acc.f[k], acc.f[k + 1], acc.f[k + 2], acc.f[k + 3]);
    encode_lane<B, SR, G>(acc, active, e0, cx, store);
  }
}

}  // namespace fc2
#include "fc2_reduce_run.cuh"
namespace fc2 {

// ---------------------------------------------------------------------------
// template dispatch
// ---------------------------------------------------------------------------

template <int B, bool SR, int G>
struct EncFast {
  template <typename T>
  static int launch(const EncBatch& b, cudaStream_t st) {
    constexpr auto kern = k_encode_fast<T, B, SR, G>;
    const int smem = kEncWarps * kStages * Stage<T>::BYTES;
    smem_attr<kern>(smem);
    int64_t blocks = (b.total + kEncWarps - 1) / kEncWarps;
    int64_t cap = (int64_t)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, kEncWarps * 32, smem, st>>>(b);
    return cuda_check("k_encode_fast");
  }
};

#define FC2_G_CASES(BB, SS)                                              \
  switch (G) {                                                           \
    case 32: return F<BB, SS, 32>::go(std::forward<Args>(args)...);      \
    case 64: return F<BB, SS, 64>::go(std::forward<Args>(args)...);      \
    case 128: return F<BB, SS, 128>::go(std::forward<Args>(args)...);    \
    case 256: return F<BB, SS, 256>::go(std::forward<Args>(args)...);    \
  }                                                                      \
  break;
#define FC2_B_CASE(BB)                        \
  case BB:                                    \
    if (sr) { FC2_G_CASES(BB, true) }         \
    else { FC2_G_CASES(BB, false) }           \
    break;

// ---------------------------------------------------------------------------
// reduce + requantize, lane-per-group (fc2_reduce_group.cuh)
// ---------------------------------------------------------------------------

template <int B>
__device__ __forceinline__ void load_run_words(const uint8_t* pay, int64_t n, int64_t e, uint32_t* w) {
#pragma unroll
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u), O = unit_off(B, u);
    const uint8_t* p = pay + (n * O) / 8 + (e * W) / 8;
    if (W == 8) {
      const uint4 q0 = *reinterpret_cast<const uint4*>(p), q1 = *reinterpret_cast<const uint4*>(p + 16);
      w[O] = q0.x; w[O + 1] = q0.y; w[O + 2] = q0.z; w[O + 3] = q0.w;
      w[O + 4] = q1.x; w[O + 5] = q1.y; w[O + 6] = q1.z; w[O + 7] = q1.w;
    } else if (W == 4) {
      const uint4 q0 = *reinterpret_cast<const uint4*>(p);
      w[O] = q0.x; w[O + 1] = q0.y; w[O + 2] = q0.z; w[O + 3] = q0.w;
    } else if (W == 2) {
      const uint2 q0 = *reinterpret_cast<const uint2*>(p);
      w[O] = q0.x; w[O + 1] = q0.y;
    } else {
      w[O] = *reinterpret_cast<const uint32_t*>(p);
    }
  }
}

template <int B, bool SR, int G, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_reduce_grp(const __grid_constant__ ReduceArgs a) {
  using IT = GTile<float, G>;
  constexpr int RUNS = G / 32;
  constexpr int REC_BYTES = 32 * 3 * kRedMaxSrc * 4;  // per-lane metadata records of all sources
  constexpr int PER_WARP = IT::IN_BYTES + OutStage<B, G>::BYTES + REC_BYTES;
  constexpr int BATCH = 4;  // sources whose codes are in flight together
  extern __shared__ __align__(16) uint8_t rsm[];
  const int warp = (int)(threadIdx.x >> 5), lane = (int)lane_id();
  uint8_t* tile = rsm + warp * PER_WARP;
  uint8_t* ost = tile + IT::IN_BYTES;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  const int64_t ngroups = a.n / G;
  const int rb = rec_bytes(SR, a.intlog != 0);
  const int64_t meta_off = a.n * B / 8;
  EncCtx cx;
  cx.n = a.n; cx.meta_off = meta_off; cx.intlog = a.intlog; cx.theta = a.theta; cx.lut = a.lut; cx.err = a.err;
  for (int64_t t = (int64_t)blockIdx.x * WARPS + warp; t < a.total; t += nw) {
    const int64_t tg0 = t * 32, g = tg0 + lane;
    const bool active = g < ngroups;
    const int64_t gc = active ? g : 0;
    const int ng = (int)min((int64_t)32, ngroups - tg0);
    // raw metadata records of every source for this group (smem, so the
    // source loop can stay rolled without local-memory arrays)
    uint32_t* recs = reinterpret_cast<uint32_t*>(ost + OutStage<B, G>::BYTES) + lane * (3 * kRedMaxSrc);
#pragma unroll
    for (int s = 0; s < kRedMaxSrc; ++s)
      if (s < a.nsrc) {
        uint32_t rr[3];
        load_record(a.src[s] + meta_off + gc * rb, rr, rb);
        recs[3 * s] = rr[0]; recs[3 * s + 1] = rr[1]; recs[3 * s + 2] = rr[2];
      }
#pragma unroll 1
    for (int r = 0; r < RUNS; ++r) {
      const int64_t er = gc * G + 32 * r;
      float acc[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) acc[k] = 0.0f;  // acc = zeros(float32) (collectives.py:293)
#pragma unroll 1
      for (int s0 = 0; s0 < a.nsrc; s0 += BATCH) {
        uint32_t cw[BATCH][B];
#pragma unroll
        for (int i = 0; i < BATCH; ++i)
          if (s0 + i < a.nsrc) load_run_words<B>(a.src[s0 + i], a.n, er, cw[i]);
#pragma unroll
        for (int i = 0; i < BATCH; ++i) {
          const int s = s0 + i;
          if (s >= a.nsrc) break;
          const uint32_t rec0 = recs[3 * s], rec1 = recs[3 * s + 1], rec2 = recs[3 * s + 2];
          // metadata of source s (R10 layouts)
          float s32 = 0.f, z32 = 0.f, smin = 0.f, smax = 0.f;
          double s64 = 0.0, o64 = 0.0;
          int imin = -1, imax = -1;
          if (!a.intlog) {
            s32 = bf16_val(rec0 & 0xFFFFu);
            z32 = bf16_val(rec0 >> 16);
            if constexpr (SR) {
              smin = bf16_val(rec1 & 0xFFFFu);
              smax = bf16_val(rec1 >> 16);
              const float fi = bf16_val(rec2 & 0xFFFFu), fa = bf16_val(rec2 >> 16);
              if ((fi > -1.0f) && (fi < (float)G) && (fa > -1.0f) && (fa < (float)G)) {
                imin = (int)fi; imax = (int)fa;
              } else if (active && r == 0) {
                atomicOr(a.err, FC2_ERR_SPIKE_INDEX);
              }
            }
          } else {
            const int si = (int)(int8_t)(rec0 & 0xFFu), zi = (int)(int8_t)((rec0 >> 8) & 0xFFu);
            s64 = si == -128 ? 0.0 : a.lut[si + 128];
            o64 = __dmul_rn(-(double)zi, s64);
            if constexpr (SR) {
              smin = bf16_val(rec0 >> 16);
              smax = bf16_val(rec1 & 0xFFFFu);
              const int ii = (int)((rec1 >> 16) & 0xFFu), ia = (int)(rec1 >> 24);
              if (ii < G && ia < G) { imin = ii; imax = ia; }
              else if (active && r == 0) atomicOr(a.err, FC2_ERR_SPIKE_INDEX);
            }
          }
          uint32_t cf[32];
          run_code_floats<B>(cw[i], cf);
          float d[32];
          if (!a.intlog) {
#pragma unroll
            for (int k = 0; k < 32; k += 2) {
              float c0, c1;
              add2(c0, c1, __uint_as_float(cf[k]), __uint_as_float(cf[k + 1]), -8388608.0f, -8388608.0f);
              fma2(d[k], d[k + 1], c0, c1, s32, s32, z32, z32);
            }
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k)
              d[k] = __double2float_rn(__dadd_rn(__dmul_rn((double)(cf[k] & 0xFFu), s64), o64));
          }
          if constexpr (SR) {  // reserved values: imin then imax, via the lane's run region
            const int ka = imin - 32 * r, kz = imax - 32 * r;
            const bool ha = ka >= 0 && ka < 32, hz = kz >= 0 && kz < 32;
            if (__any_sync(0xffffffffu, ha || hz)) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<float4*>(tile + IT::in_pos(lane, 8 * r + j) * 16) =
                    make_float4(d[4 * j], d[4 * j + 1], d[4 * j + 2], d[4 * j + 3]);
              if (ha) *reinterpret_cast<float*>(tile + IT::in_pos(lane, 8 * r + (ka >> 2)) * 16 + (ka & 3) * 4) = smin;
              if (hz) *reinterpret_cast<float*>(tile + IT::in_pos(lane, 8 * r + (kz >> 2)) * 16 + (kz & 3) * 4) = smax;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 q = *reinterpret_cast<const float4*>(tile + IT::in_pos(lane, 8 * r + j) * 16);
                d[4 * j] = q.x; d[4 * j + 1] = q.y; d[4 * j + 2] = q.z; d[4 * j + 3] = q.w;
              }
            }
          }
#pragma unroll
          for (int k = 0; k < 32; k += 2) add2(acc[k], acc[k + 1], acc[k], acc[k + 1], d[k], d[k + 1]);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<float4*>(tile + IT::in_pos(lane, 8 * r + j) * 16) =
            make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    }
    __syncwarp();
    encode_tile_f32<B, SR, G>(tile, ost, active, g, cx, a.dst, a.ndst, tg0, ng);
  }
}


template <int B, bool SR, int G>
__global__ void __launch_bounds__(G) k_reduce_cta(const __grid_constant__ ReduceArgs a) {
  constexpr int LPG = G / 32;   // lanes per group in the encode phase (= warps per CTA)
  constexpr int GPW = 32 / LPG; // groups per warp in the encode phase
  constexpr int BATCH = 4;      // sources whose codes are in flight together
  extern __shared__ __align__(16) uint8_t csm[];
  uint8_t* tile = csm;
  uint8_t* ost = csm + RTile<G>::BYTES;
  const int w = (int)(threadIdx.x >> 5), lane = (int)lane_id();
  const int64_t ngroups = a.n / G;
  const int rb = rec_bytes(SR, a.intlog != 0);
  const int64_t meta_off = a.n * B / 8;
  EncCtx cx;
  cx.n = a.n; cx.meta_off = meta_off; cx.intlog = a.intlog; cx.theta = a.theta; cx.lut = a.lut; cx.err = a.err;
  const int64_t tps = (ngroups + 31) / 32;  // tiles per shard
  for (int64_t t = blockIdx.x; t < a.total; t += gridDim.x) {
    const int64_t sh = t / tps;
    const int64_t soff = sh * a.sstride, doff = sh * a.dstride;
    const int64_t tg0 = (t - sh * tps) * 32;
    const int ng = (int)min((int64_t)32, ngroups - tg0);
    // ---- accumulation: warp w = run w, lane = group
    {
      const int64_t g = tg0 + lane;
      const bool act = g < ngroups;
      const int64_t gc = act ? g : tg0;
      const int64_t er = gc * G + 32 * w;
      float acc[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) acc[k] = 0.0f;  // acc = zeros(float32) (collectives.py:293)
#pragma unroll 1
      for (int s0 = 0; s0 < a.nsrc; s0 += BATCH) {
        uint32_t cw[BATCH][B];
        uint32_t rec[BATCH][3];
#pragma unroll
        for (int i = 0; i < BATCH; ++i)
          if (s0 + i < a.nsrc) {
            load_run_words<B>(a.src[s0 + i] + soff, a.n, er, cw[i]);
            load_record(a.src[s0 + i] + soff + meta_off + gc * rb, rec[i], rb);
          }
#pragma unroll
        for (int i = 0; i < BATCH; ++i) {
          if (s0 + i >= a.nsrc) break;
          float s32 = 0.f, z32 = 0.f, smin = 0.f, smax = 0.f;
          double s64 = 0.0, o64 = 0.0;
          int imin = -1, imax = -1;
          if (!a.intlog) {
            s32 = bf16_val(rec[i][0] & 0xFFFFu);
            z32 = bf16_val(rec[i][0] >> 16);
            if constexpr (SR) {
              smin = bf16_val(rec[i][1] & 0xFFFFu);
              smax = bf16_val(rec[i][1] >> 16);
              const float fi = bf16_val(rec[i][2] & 0xFFFFu), fa = bf16_val(rec[i][2] >> 16);
              if ((fi > -1.0f) && (fi < (float)G) && (fa > -1.0f) && (fa < (float)G)) {
                imin = (int)fi; imax = (int)fa;
              } else if (act && w == 0) {
                atomicOr(a.err, FC2_ERR_SPIKE_INDEX);
              }
            }
          } else {
            const int si = (int)(int8_t)(rec[i][0] & 0xFFu), zi = (int)(int8_t)((rec[i][0] >> 8) & 0xFFu);
            s64 = si == -128 ? 0.0 : a.lut[si + 128];
            o64 = __dmul_rn(-(double)zi, s64);
            if constexpr (SR) {
              smin = bf16_val(rec[i][0] >> 16);
              smax = bf16_val(rec[i][1] & 0xFFFFu);
              const int ii = (int)((rec[i][1] >> 16) & 0xFFu), ia = (int)(rec[i][1] >> 24);
              if (ii < G && ia < G) { imin = ii; imax = ia; }
              else if (act && w == 0) atomicOr(a.err, FC2_ERR_SPIKE_INDEX);
            }
          }
          uint32_t cf[32];
          run_code_floats<B>(cw[i], cf);
          float d[32];
          if (!a.intlog) {
#pragma unroll
            for (int k = 0; k < 32; k += 2) {
              float c0, c1;
              add2(c0, c1, __uint_as_float(cf[k]), __uint_as_float(cf[k + 1]), -8388608.0f, -8388608.0f);
              fma2(d[k], d[k + 1], c0, c1, s32, s32, z32, z32);
            }
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k)
              d[k] = __double2float_rn(__dadd_rn(__dmul_rn((double)(cf[k] & 0xFFu), s64), o64));
          }
          if constexpr (SR) {  // reserved values (imin then imax) through the lane's tile region
            const int ka = imin - 32 * w, kz = imax - 32 * w;
            const bool ha = ka >= 0 && ka < 32, hz = kz >= 0 && kz < 32;
            if (__any_sync(0xffffffffu, ha || hz)) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<float4*>(tile + RTile<G>::pos(lane, 8 * w + j) * 16) =
                    make_float4(d[4 * j], d[4 * j + 1], d[4 * j + 2], d[4 * j + 3]);
              if (ha) *reinterpret_cast<float*>(tile + RTile<G>::pos(lane, 8 * w + (ka >> 2)) * 16 + (ka & 3) * 4) = smin;
              if (hz) *reinterpret_cast<float*>(tile + RTile<G>::pos(lane, 8 * w + (kz >> 2)) * 16 + (kz & 3) * 4) = smax;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 q = *reinterpret_cast<const float4*>(tile + RTile<G>::pos(lane, 8 * w + j) * 16);
                d[4 * j] = q.x; d[4 * j + 1] = q.y; d[4 * j + 2] = q.z; d[4 * j + 3] = q.w;
              }
            }
          }
#pragma unroll
          for (int k = 0; k < 32; k += 2) add2(acc[k], acc[k + 1], acc[k], acc[k + 1], d[k], d[k + 1]);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<float4*>(tile + RTile<G>::pos(lane, 8 * w + j) * 16) =
            make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    }
    __syncthreads();
    // ---- encode: LPG lanes per group, one run per lane
    {
      const int gl = w * GPW + lane / LPG, li = lane % LPG;
      const int64_t g_abs = tg0 + gl;
      encode_run_f32<B, SR, G>(tile, ost, gl, li, g_abs < ngroups, g_abs, cx, a.dst, a.ndst, doff);
    }
    __syncthreads();  // whole tile staged (runs of a group come from several warps... same warp here)
    // ---- copy-out: warp w writes groups [w*GPW, w*GPW + GPW) to every destination
    {
      const int first = w * GPW;
      const int cnt = max(0, min(GPW, ng - first));
      for (int dd = 0; dd < a.ndst; ++dd) {
#pragma unroll
        for (int u = 0; u < n_units(B); ++u) {
          const int W = unit_w(B, u), O = unit_off(B, u);
          const uint8_t* base = ost + OutStage<B, G>::off(u);
          uint8_t* dst = a.dst[dd] + doff + (a.n * O) / 8 + (tg0 + first) * (G * W / 8);
          if (W == 1) copy_out_groups<G, 1>(base, dst, first, cnt);
          else if (W == 2) copy_out_groups<G, 2>(base, dst, first, cnt);
          else if (W == 4) copy_out_groups<G, 4>(base, dst, first, cnt);
          else copy_out_groups<G, 8>(base, dst, first, cnt);
        }
      }
    }
    __syncthreads();
  }
}

template <int B, bool SR, int G>
struct RedCta {
  static constexpr int SMEM = RTile<G>::BYTES + OutStage<B, G>::BYTES;
  static int go(const ReduceArgs& a0, cudaStream_t st) {
    ReduceArgs a = a0;
    a.total = (a.n / G + 31) / 32 * a.nshard;
    constexpr auto kern = k_reduce_cta<B, SR, G>;
    smem_attr<kern>(SMEM);
    int64_t blocks = a.total;
    if (blocks < 1) blocks = 1;
    if (blocks > 65535LL * 16) blocks = 65535LL * 16;
    kern<<<(unsigned)blocks, G, SMEM, st>>>(a);
    return cuda_check("k_reduce_cta");
  }
};

template <int B, bool SR, int G>
struct RedGrp {
  static constexpr int WARPS = G <= 128 ? 4 : 2;
  static constexpr int SMEM = WARPS * (GTile<float, G>::IN_BYTES + OutStage<B, G>::BYTES + 32 * 3 * kRedMaxSrc * 4);
  static int go(const ReduceArgs& a0, cudaStream_t st) {
    ReduceArgs a = a0;
    a.total = (a.n / G + 31) / 32;
    constexpr auto kern = k_reduce_grp<B, SR, G, WARPS>;
    smem_attr<kern>(SMEM);
    int64_t blocks = (a.total + WARPS - 1) / WARPS;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, WARPS * 32, SMEM, st>>>(a);
    return cuda_check("k_reduce_grp");
  }
};

template <int B, bool SR, int G>
struct EncFastBf16 {
  static int go(const EncBatch& b, cudaStream_t st) { return EncFast<B, SR, G>::template launch<__nv_bfloat16>(b, st); }
};
template <int B, bool SR, int G>
struct EncFastF32 {
  static int go(const EncBatch& b, cudaStream_t st) { return EncFast<B, SR, G>::template launch<float>(b, st); }
};

template <int B, bool SR, int G>
struct RedFast {
  static int go(const ReduceArgs& a, cudaStream_t st) {
    int64_t blocks = (a.total + kRedWarps - 1) / kRedWarps;
    int64_t cap = (int64_t)num_sms() * 4;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k_reduce_fast<B, SR, G><<<(unsigned)blocks, kRedWarps * 32, 0, st>>>(a);
    return cuda_check("k_reduce_fast");
  }
};


// per-bitwidth launchers (defined in fc2_inst_b<B>.cu)
template <int B> int launch_enc_fast(int dtype, bool sr, int G, const EncBatch& b, cudaStream_t st);
template <int B> int launch_red_fast(bool sr, int G, const ReduceArgs& a, cudaStream_t st);
template <int B> int launch_dec_fast(int dtype, int64_t blocks, const DecBatch& b, cudaStream_t st);

template <int B>
struct Launchers {
  template <bool SR>
  static int enc(int dtype, int G, const EncBatch& b, cudaStream_t st) {
    switch (G) {
      case 32: return dtype == FC2_BF16 ? EncGrp<B, SR, 32>::go(b, st) : EncFastF32<B, SR, 32>::go(b, st);
      case 64: return dtype == FC2_BF16 ? EncGrp<B, SR, 64>::go(b, st) : EncFastF32<B, SR, 64>::go(b, st);
      case 128: return dtype == FC2_BF16 ? EncGrp<B, SR, 128>::go(b, st) : EncFastF32<B, SR, 128>::go(b, st);
      case 256: return dtype == FC2_BF16 ? EncGrp<B, SR, 256>::go(b, st) : EncFastF32<B, SR, 256>::go(b, st);
    }
    return set_err(FC2_ECONFIG, "no fast encoder for G=%d", G);
  }
  template <bool SR>
  static int red(int G, const ReduceArgs& a, cudaStream_t st) {
    bool grp = a.nsrc <= kRedMaxSrc;
    for (int s = 0; s < a.nsrc; ++s)
      if (reinterpret_cast<uintptr_t>(a.src[s]) & 15u) grp = false;
    if (grp && a.nshard > 1 && (a.sstride & 15)) grp = false;
    if (!grp && a.nshard > 1) {  // the other reducers take one shard per launch
      ReduceArgs one = a;
      one.nshard = 1;
      for (int64_t k = 0; k < a.nshard; ++k) {
        for (int s = 0; s < a.nsrc; ++s) one.src[s] = a.src[s] + k * a.sstride;
        for (int d = 0; d < a.ndst; ++d) one.dst[d] = a.dst[d] + k * a.dstride;
        int rc = red<SR>(G, one, st);
        if (rc) return rc;
      }
      return FC2_OK;
    }
    // default: bulk-copy staged tiles, sums in registers (k_reduce_run);
    // FC2_REDUCE=cta selects the round-1 CTA kernel (A/B measurements)
    static const bool use_cta = [] {
      const char* e = getenv("FC2_REDUCE");
      return e && e[0] == 'c';
    }();
    if (!use_cta) {
      switch (G) {
        case 32: if (RedRun<B, SR, 32>::ok(a)) return RedRun<B, SR, 32>::go(a, st); break;
        case 64: if (RedRun<B, SR, 64>::ok(a)) return RedRun<B, SR, 64>::go(a, st); break;
        case 128: if (RedRun<B, SR, 128>::ok(a)) return RedRun<B, SR, 128>::go(a, st); break;
        case 256: if (RedRun<B, SR, 256>::ok(a)) return RedRun<B, SR, 256>::go(a, st); break;
      }
    }
    if (grp) {
      switch (G) {
        case 32: return RedCta<B, SR, 32>::go(a, st);
        case 64: return RedCta<B, SR, 64>::go(a, st);
        case 128: return RedCta<B, SR, 128>::go(a, st);
        case 256: return RedCta<B, SR, 256>::go(a, st);
      }
    }
    switch (G) {
      case 32: return RedFast<B, SR, 32>::go(a, st);
      case 64: return RedFast<B, SR, 64>::go(a, st);
      case 128: return RedFast<B, SR, 128>::go(a, st);
      case 256: return RedFast<B, SR, 256>::go(a, st);
    }
    return set_err(FC2_ECONFIG, "no fast reducer for G=%d", G);
  }
};

#define FC2_INSTANTIATE_B(BB)                                                                  \
  template <> int launch_enc_fast<BB>(int dtype, bool sr, int G, const EncBatch& b, cudaStream_t st) { \
    return sr ? Launchers<BB>::enc<true>(dtype, G, b, st) : Launchers<BB>::enc<false>(dtype, G, b, st); \
  }                                                                                            \
  template <> int launch_red_fast<BB>(bool sr, int G, const ReduceArgs& a, cudaStream_t st) {  \
    return sr ? Launchers<BB>::red<true>(G, a, st) : Launchers<BB>::red<false>(G, a, st);     \
  }                                                                                            \
  template <> int launch_dec_fast<BB>(int dtype, int64_t blocks, const DecBatch& b, cudaStream_t st) { \
    (void)blocks;                                                                              \
    return dtype == FC2_BF16 ? launch_decode_fast<__nv_bfloat16, BB>(b, st)                     \
                             : launch_decode_fast<float, BB>(b, st);                            \
  }

}  // namespace fc2
