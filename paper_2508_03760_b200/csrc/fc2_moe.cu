// fc2_moe.cu -- MoE token routing around the quantized All2All (BASELINE
// configs[3]; the codec fused into token dispatch/combine).
//
// The reference's All2All (collectives.py:428-482) moves block (src, dst) of a
// flat payload: one chunk per block, zero-padded to a group multiple, QDQ'd,
// the diagonal exact.  For MoE the block (src, dst) is the rows of the
// tokens of rank src that route to at least one expert on rank dst (one copy
// per distinct destination rank, token order).  This file holds the pieces
// around the codec:
//
//   k_moe_route     top-k expert ids -> per-destination token lists (rows),
//                   per-token positions in them (pos) and the counts; one
//                   CTA, ballot + per-warp prefix, token order preserved
//   k_gather_rows   the diagonal block: exact gather-copy of token rows with
//                   the payload finiteness check (collectives.py:152-164)
//   k_moe_combine   out[t] = sum over destination ranks d in rank order of
//                   block(d -> me)[pos[t][d]] in fp32 from +0.0 (the QDQ'd
//                   expert outputs, exact on the diagonal)
//
// The gather itself is fused into the encoders (EncJob.rows): the packed
// block is produced straight from the token rows, no gathered copy in HBM.
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "../../include/fc2.h"
#include "fc2_common.cuh"
#include "fc2_decode.cuh"

namespace fc2 {
int set_err(int code, const char* fmt, ...);
int cuda_check(const char* what);
int num_sms();
const double* lut_for_cfg(const fc2_config* c, int* rc);
}  // namespace fc2

using namespace fc2;

#define FC2_MOE_MAX_WORLD 16

namespace {

// destination-rank mask of token t (bit d: one of its experts lives on rank d);
// the token's K ids are loaded before any is used (up to 16 in flight)
__device__ __forceinline__ uint32_t route_mask(const void* ids, int idx64, int64_t t, int K, int per,
                                               int n_experts, int32_t* err) {
  uint32_t m = 0;
  for (int k0 = 0; k0 < K; k0 += 16) {
    int64_t e[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      e[k] = k0 + k >= K ? 0
                         : (idx64 ? __ldg(reinterpret_cast<const long long*>(ids) + t * K + k0 + k)
                                  : (int64_t)__ldg(reinterpret_cast<const int32_t*>(ids) + t * K + k0 + k));
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k0 + k >= K) break;
      if (e[k] < 0 || e[k] >= n_experts) {
        atomicOr(err, FC2_ERR_EXPERT_RANGE);
        continue;
      }
      m |= 1u << ((int)e[k] / per);  // 32-bit division: a validated expert id
    }
  }
  return m;
}

#ifndef FC2_COMBINE_MINB
#define FC2_COMBINE_MINB 2
#endif
constexpr int kRouteChunk = 8192;  // tokens whose masks the routing CTA stages at once (32 KB of smem)

// pass 1, all SMs: mask of every token, parked in pos[t * world] (pass 2
// reads a chunk's masks into shared memory before it writes that chunk's pos)
__global__ void k_moe_masks(const void* ids, int idx64, int64_t T, int K, int per, int n_experts, int world,
                            int32_t* pos, int32_t* err) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) pos[t * world] = (int32_t)route_mask(ids, idx64, t, K, per, n_experts, err);
}

// One CTA of 1024 threads walks the tokens in rounds of 1024 (thread = token).
// Positions inside a destination list follow token order: ballot rank inside
// the warp + the warp's offset (scanned by thread d) + the running base.
__global__ void __launch_bounds__(1024) k_moe_route(const void* ids, int idx64, int64_t T, int K, int per,
                                                   int n_experts, int world, int32_t* counts, int32_t* rows,
                                                   int32_t* pos, int32_t* err) {
  __shared__ int32_t woff[32][FC2_MOE_MAX_WORLD];
  __shared__ int32_t base[FC2_MOE_MAX_WORLD];
  pdl_enter();
  __shared__ uint32_t masks[kRouteChunk];
  const int lane = (int)(threadIdx.x & 31), warp = (int)(threadIdx.x >> 5);
  const uint32_t lt = (1u << lane) - 1u;
  if (threadIdx.x < (unsigned)world) base[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t t0 = 0; t0 < T; t0 += blockDim.x) {
    if ((t0 % kRouteChunk) == 0) {  // the next chunk's masks (pass 1), all loads in flight together
      __syncthreads();
      uint32_t mk[kRouteChunk / 1024];
#pragma unroll
      for (int j = 0; j < kRouteChunk / 1024; ++j) {
        const int64_t tt = t0 + threadIdx.x + 1024 * j;
        mk[j] = tt < T ? (uint32_t)__ldcg(pos + tt * world) : 0u;
      }
#pragma unroll
      for (int j = 0; j < kRouteChunk / 1024; ++j) masks[threadIdx.x + 1024 * j] = mk[j];
      __syncthreads();
    }
    const int64_t t = t0 + threadIdx.x;
    const uint32_t m = masks[(t0 % kRouteChunk) + threadIdx.x];
    for (int d = 0; d < world; ++d) {
      const uint32_t bal = __ballot_sync(0xffffffffu, (m >> d) & 1u);
      if (lane == 0) woff[warp][d] = __popc(bal);
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)world) {  // exclusive scan over the warps, per destination
      const int d = (int)threadIdx.x;
      int run = base[d];
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        const int c = woff[w][d];
        woff[w][d] = run;
        run += c;
      }
      base[d] = run;
    }
    __syncthreads();
    // the token's pos row is built in registers and stored with 16-byte
    // stores (scattered 4-byte stores from one SM were the kernel's bottleneck)
    int32_t pv[FC2_MOE_MAX_WORLD];
#pragma unroll
    for (int d = 0; d < FC2_MOE_MAX_WORLD; ++d) {
      if (d >= world) break;
      const uint32_t bal = __ballot_sync(0xffffffffu, (m >> d) & 1u);
      pv[d] = -1;
      if (t < T && ((m >> d) & 1u)) {
        pv[d] = woff[warp][d] + __popc(bal & lt);
        rows[(int64_t)d * T + pv[d]] = (int32_t)t;
      }
    }
    if (t < T) {
      int32_t* pr = pos + t * world;
      if ((world & 3) == 0) {
#pragma unroll
        for (int d = 0; d < FC2_MOE_MAX_WORLD; d += 4)
          if (d < world) *reinterpret_cast<int4*>(pr + d) = make_int4(pv[d], pv[d + 1], pv[d + 2], pv[d + 3]);
      } else {
#pragma unroll
        for (int d = 0; d < FC2_MOE_MAX_WORLD; ++d)
          if (d < world) pr[d] = pv[d];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < (unsigned)world) counts[threadIdx.x] = base[threadIdx.x];
}

template <typename T>
__device__ __forceinline__ void load8(const T* p, float* v);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float* v) {
  const uint4 q = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float* v) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

__device__ __forceinline__ void load8_any(const void* p, int dt, int64_t i, float* v) {
  if (dt == FC2_BF16) load8<__nv_bfloat16>(reinterpret_cast<const __nv_bfloat16*>(p) + i, v);
  else load8<float>(reinterpret_cast<const float*>(p) + i, v);
}

__device__ __forceinline__ void store8_any(void* p, int dt, int64_t i, const float* v) {
  if (dt == FC2_BF16) {
    // RNE, as bf16_bits for every finite value (the sums here are finite or flagged)
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
      w[k] = *reinterpret_cast<const uint32_t*>(&h2);
    }
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p) + i) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    float* q = reinterpret_cast<float*>(p) + i;
    *reinterpret_cast<float4*>(q) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(q + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
}

// y[r * H + h] = x[rows[r] * H + h], 8 elements per thread-iteration
__global__ void k_gather_rows(const void* x, int xdt, const int32_t* rows, int64_t nrows, int64_t H, void* y,
                              int ydt, int32_t* err) {
  const int64_t n8 = nrows * H / 8;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = 8 * i, r = e / H, h = e - r * H;
    float v[8];
    load8_any(x, xdt, (int64_t)rows[r] * H + h, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) bad |= !isfinite(v[k]);
    store8_any(y, ydt, e, v);
  }
  if (bad) atomicOr(err, FC2_ERR_NONFINITE);
}

struct CombineArgs {
  const void* src[FC2_MOE_MAX_WORLD];  // block (d -> me), rows in pos order
  int dt[FC2_MOE_MAX_WORLD];
  int check[FC2_MOE_MAX_WORLD];        // exact (diagonal) blocks: flag non-finite values
  const int32_t* pos;                  // [T][world], -1: token not routed to d
  int64_t T, H;
  int world, odt;
  void* out;
  int32_t* err;
};

__global__ void k_moe_combine(const __grid_constant__ CombineArgs a) {
  const int64_t n8 = a.T * a.H / 8;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = 8 * i, t = e / a.H, h = e - t * a.H;
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0f;  // fp32 from +0.0, destination ranks in order
    for (int d = 0; d < a.world; ++d) {
      const int p = __ldg(a.pos + t * a.world + d);
      if (p < 0) continue;
      float v[8];
      load8_any(a.src[d], a.dt[d], (int64_t)p * a.H + h, v);
      if (a.check[d]) {
#pragma unroll
        for (int k = 0; k < 8; ++k) bad |= !isfinite(v[k]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = __fadd_rn(acc[k], v[k]);
    }
    store8_any(a.out, a.odt, e, acc);
  }
  if (bad) atomicOr(a.err, FC2_ERR_NONFINITE);
}

// Fused combine: the returned blocks are read in their packed form (no float32
// round trip through HBM).  Warp = one 1024-element segment of one token,
// lane = one 32-element run; per source rank d in order, the lane decodes
// its run of row pos[t][d] of block d (codes + the group's record, reserved
// spikes patched through a per-lane smem row) or reads the exact row of its
// own block, and adds in fp32.  Needs G % 32 == 0 and H % 32 == 0.
struct CombineQArgs {
  const uint8_t* pay[FC2_MOE_MAX_WORLD];  // block (d -> me), packed; unused for d == me
  int64_t n[FC2_MOE_MAX_WORLD];           // its chunk length (padded to a group multiple)
  const void* exact;                      // my own block's rows (d == me), dtype edt
  int edt;
  int me, world, B, G, sr, intlog, theta;
  int gshift;                             // log2(G) when G is a power of two, else -1
  const double* lut;
  const int32_t* pos;                     // [T][world]
  int64_t T, H;
  void* out;
  int odt;
  int32_t* err;
};

// the lane's 32-element run of a packed block: plane words (unit-major) with
// vector loads -- slots are 16-byte aligned and chunk lengths multiples of 32,
// so unit u's 4W bytes are 4W-aligned
template <int B>
__device__ __forceinline__ void load_run_words(const uint8_t* P, int64_t nd, int64_t e0, uint32_t (&w)[B]) {
#pragma unroll
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u), O = unit_off(B, u);
    const uint8_t* q = P + nd * O / 8 + e0 * W / 8;
    if (W == 8) {
      const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(q)), q1 = __ldg(reinterpret_cast<const uint4*>(q + 16));
      w[O] = q0.x; w[O + 1] = q0.y; w[O + 2] = q0.z; w[O + 3] = q0.w;
      w[O + 4] = q1.x; w[O + 5] = q1.y; w[O + 6] = q1.z; w[O + 7] = q1.w;
    } else if (W == 4) {
      const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(q));
      w[O] = q0.x; w[O + 1] = q0.y; w[O + 2] = q0.z; w[O + 3] = q0.w;
    } else if (W == 2) {
      const uint2 q0 = __ldg(reinterpret_cast<const uint2*>(q));
      w[O] = q0.x; w[O + 1] = q0.y;
    } else {
      w[O] = __ldg(reinterpret_cast<const uint32_t*>(q));
    }
  }
}

// operands of one source rank's run, loaded one source ahead of their use
template <int B>
struct CombineSrc {
  uint32_t w[B];    // plane words (packed block)
  uint32_t rec[3];  // the group's record (my own block's row is read at use)
};

template <int B>
__global__ void __launch_bounds__(256, FC2_COMBINE_MINB) k_moe_combine_q(const __grid_constant__ CombineQArgs a) {
  __shared__ __align__(16) float spill_all[8][32][36];
  const int warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
  float* spill = spill_all[warp][lane];
  // 32-bit task / position arithmetic (the launcher checks T * segments and
  // H against INT32_MAX): no 64-bit division per task
  const int H = (int)a.H;
  const int segs = (H + 1023) / 1024;
  const int tasks = (int)a.T * segs;
  const int nw = (int)gridDim.x * (int)(blockDim.x >> 5);
  const int rb = rec_bytes(a.sr != 0, a.intlog != 0);
  bool bad = false;
  for (int w = (int)blockIdx.x * (int)(blockDim.x >> 5) + warp; w < tasks; w += nw) {
    const int t = w / segs;
    const int h = (w - t * segs) * 1024 + 32 * lane;
    const bool on = h < H;
    // the token's row index in every source block: one load per lane, then shuffles
    const int mypos = lane < a.world ? __ldg(a.pos + (int64_t)t * a.world + lane) : -1;
    uint32_t todo = __ballot_sync(0xffffffffu, mypos >= 0);  // source ranks in order
    float acc[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) acc[k] = 0.0f;  // fp32 from +0.0, source ranks in order
    auto load = [&](int d, int64_t e0, CombineSrc<B>& o) {
      if (!on) return;
      if (d != a.me) {
        load_run_words<B>(a.pay[d], a.n[d], e0, o.w);
        const int64_t grp = a.gshift >= 0 ? e0 >> a.gshift : e0 / a.G;  // no 64-bit division per run
        load_record(a.pay[d] + a.n[d] * B / 8 + grp * rb, o.rec, rb);
      }
    };
    CombineSrc<B> cur, nxt;
    int dc = -1;
    int64_t ec = 0;
    if (todo) {
      dc = __ffs(todo) - 1;
      todo &= todo - 1;
      ec = (int64_t)__shfl_sync(0xffffffffu, mypos, dc) * H + h;
      load(dc, ec, cur);
    }
    while (dc >= 0) {  // warp-uniform
      int dn = -1;
      int64_t en = 0;
      if (todo) {  // next source's loads go out before this one is decoded
        dn = __ffs(todo) - 1;
        todo &= todo - 1;
        en = (int64_t)__shfl_sync(0xffffffffu, mypos, dn) * H + h;
        load(dn, en, nxt);
      }
      float v[32];
      if (dc == a.me) {
        if (on) {
#pragma unroll
          for (int k = 0; k < 32; k += 8) load8_any(a.exact, a.edt, ec + k, v + k);
#pragma unroll
          for (int k = 0; k < 32; ++k) bad |= !isfinite(v[k]);
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = 0.f;
        }
      } else {
        DecCtx c;
        c.n = a.n[dc];
        c.meta_off = a.n[dc] * B / 8;
        c.B = B; c.G = a.G; c.sr = a.sr != 0; c.intlog = a.intlog != 0; c.theta = a.theta;
        c.lut = a.lut; c.err = on ? a.err : nullptr;
        const GroupMeta m = meta_from_record(cur.rec, c);
        uint32_t cf[32];
        run_code_floats<B>(cur.w, cf);
        if (!c.intlog) {
#pragma unroll
          for (int k = 0; k < 32; k += 2) {
            float c0, c1;
            add2(c0, c1, __uint_as_float(cf[k]), __uint_as_float(cf[k + 1]), -8388608.0f, -8388608.0f);
            fma2(v[k], v[k + 1], c0, c1, m.s32, m.s32, m.z32, m.z32);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k)
            v[k] = __double2float_rn(__dadd_rn(__dmul_rn((double)(cf[k] & 0xFFu), m.s64), m.o64));
        }
        if (c.sr) {  // reserved values, imin then imax (codec.py:559-561)
          const int base = (int)(ec & (a.G - 1));
          const int ka = m.imin - (a.gshift >= 0 ? base : (int)(ec % a.G)), kz = m.imax - (a.gshift >= 0 ? base : (int)(ec % a.G));
          const bool ha = on && m.imin >= 0 && (unsigned)ka < 32u, hz = on && m.imax >= 0 && (unsigned)kz < 32u;
          // per-quad round trip at b4 / b8 as in k_reduce_run (configs[3] b4 SR: 85.7 -> 84.2 us)
          if (ha || hz) subst_reserved<B == 4 || B == 8>(v, spill, ha, ka, m.smin, hz, kz, m.smax);
        }
      }
#pragma unroll
      for (int k = 0; k < 32; k += 2) add2(acc[k], acc[k + 1], acc[k], acc[k + 1], v[k], v[k + 1]);
      dc = dn;
      ec = en;
      cur = nxt;
    }
    if (on) {
#pragma unroll
      for (int k = 0; k < 32; k += 8) store8_any(a.out, a.odt, (int64_t)t * H + h + k, acc + k);
    }
  }
  if (bad) atomicOr(a.err, FC2_ERR_NONFINITE);
}

int grid_for(int64_t n8, int threads) {
  int64_t blocks = (n8 + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  return (int)(blocks < 1 ? 1 : blocks);
}

}  // namespace

extern "C" {

int fc2_moe_route(const void* topk_ids, int32_t ids_are_int64, int64_t tokens, int32_t topk, int32_t n_experts,
                  int32_t world, int32_t* counts, int32_t* rows, int32_t* pos, int32_t* dev_err, void* stream) {
  if (world < 1 || world > FC2_MOE_MAX_WORLD) return set_err(FC2_ECONFIG, "world %d outside [1, 16]", world);
  if (n_experts < world || n_experts % world)
    return set_err(FC2_ECONFIG, "%d experts do not split evenly over %d ranks", n_experts, world);
  if (topk < 1 || tokens < 0 || tokens > INT32_MAX) return set_err(FC2_ECONFIG, "bad routing shape");
  if (tokens == 0) return cudaMemsetAsync(counts, 0, sizeof(int32_t) * world, (cudaStream_t)stream) == cudaSuccess
                              ? FC2_OK
                              : set_err(FC2_ECUDA, "cudaMemsetAsync failed");
  const int per = n_experts / world;
  k_moe_masks<<<(unsigned)((tokens + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      topk_ids, ids_are_int64 ? 1 : 0, tokens, topk, per, n_experts, world, pos, dev_err);
  int rc = cuda_check("k_moe_masks");
  if (rc) return rc;
  launch_pdl(k_moe_route, 1, 1024, 0, (cudaStream_t)stream, topk_ids, ids_are_int64 ? 1 : 0, tokens, topk, per,
             n_experts, world, counts, rows, pos, dev_err);
  return cuda_check("k_moe_route");
}

int fc2_gather_rows_check(const void* x, int32_t x_dtype, const int32_t* rows, int64_t nrows, int64_t row_len,
                          void* y, int32_t y_dtype, int32_t* dev_err, void* stream) {
  if (nrows <= 0) return FC2_OK;
  if (row_len <= 0 || row_len % 8) return set_err(FC2_ECONFIG, "row length must be a positive multiple of 8");
  if ((x_dtype != FC2_BF16 && x_dtype != FC2_F32) || (y_dtype != FC2_BF16 && y_dtype != FC2_F32))
    return set_err(FC2_ECONFIG, "gather supports bf16 / f32");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15u)
    return set_err(FC2_ECONFIG, "gather needs 16-byte aligned buffers");
  const int64_t n8 = nrows * row_len / 8;
  k_gather_rows<<<grid_for(n8, 256), 256, 0, (cudaStream_t)stream>>>(x, x_dtype, rows, nrows, row_len, y, y_dtype,
                                                                   dev_err);
  return cuda_check("k_gather_rows");
}

int fc2_moe_combine_sum(int32_t world, const void* const* srcs, const int32_t* src_dtypes,
                        const int32_t* check_finite, const int32_t* pos, int64_t tokens, int64_t row_len, void* out,
                        int32_t out_dtype, int32_t* dev_err, void* stream) {
  if (world < 1 || world > FC2_MOE_MAX_WORLD) return set_err(FC2_ECONFIG, "world %d outside [1, 16]", world);
  if (tokens <= 0) return FC2_OK;
  if (row_len <= 0 || row_len % 8) return set_err(FC2_ECONFIG, "row length must be a positive multiple of 8");
  if (out_dtype != FC2_BF16 && out_dtype != FC2_F32) return set_err(FC2_ECONFIG, "combine output is bf16 / f32");
  CombineArgs a;
  for (int d = 0; d < world; ++d) {
    if (src_dtypes[d] != FC2_BF16 && src_dtypes[d] != FC2_F32) return set_err(FC2_ECONFIG, "combine source dtype");
    if (reinterpret_cast<uintptr_t>(srcs[d]) & 15u) return set_err(FC2_ECONFIG, "combine sources must be 16-byte aligned");
    a.src[d] = srcs[d];
    a.dt[d] = src_dtypes[d];
    a.check[d] = check_finite ? check_finite[d] : 0;
  }
  if (reinterpret_cast<uintptr_t>(out) & 15u) return set_err(FC2_ECONFIG, "combine output must be 16-byte aligned");
  a.pos = pos;
  a.T = tokens;
  a.H = row_len;
  a.world = world;
  a.odt = out_dtype;
  a.out = out;
  a.err = dev_err;
  const int64_t n8 = tokens * row_len / 8;
  k_moe_combine<<<grid_for(n8, 256), 256, 0, (cudaStream_t)stream>>>(a);
  return cuda_check("k_moe_combine");
}

int fc2_moe_combine_q(const fc2_config* cfg, int32_t world, int32_t me, const void* const* payloads,
                      const int64_t* chunk_n, const void* exact, int32_t exact_dtype, const int32_t* pos,
                      int64_t tokens, int64_t row_len, void* out, int32_t out_dtype, int32_t* dev_err, void* stream) {
  int rc = fc2_check_config(cfg);
  if (rc) return rc;
  if (world < 1 || world > FC2_MOE_MAX_WORLD || me < 0 || me >= world)
    return set_err(FC2_ECONFIG, "bad rank %d / world %d", me, world);
  if (tokens <= 0) return FC2_OK;
  if (cfg->group_size % 32 || row_len <= 0 || row_len % 32)
    return set_err(FC2_ENOTAPPLICABLE, "fused combine needs group_size and row length multiples of 32");
  const double* lut = lut_for_cfg(cfg, &rc);
  if (rc) return rc;
  if ((exact_dtype != FC2_BF16 && exact_dtype != FC2_F32) || (out_dtype != FC2_BF16 && out_dtype != FC2_F32))
    return set_err(FC2_ECONFIG, "combine rows are bf16 / f32");
  if ((reinterpret_cast<uintptr_t>(exact) | reinterpret_cast<uintptr_t>(out)) & 15u)
    return set_err(FC2_ECONFIG, "combine buffers must be 16-byte aligned");
  CombineQArgs a;
  for (int d = 0; d < world; ++d) {
    a.pay[d] = (const uint8_t*)payloads[d];
    a.n[d] = chunk_n[d];
    if (d != me && payloads[d] && (reinterpret_cast<uintptr_t>(payloads[d]) & 3u))
      return set_err(FC2_ECONFIG, "payloads must be 4-byte aligned");
  }
  a.exact = exact;
  a.edt = exact_dtype;
  a.me = me; a.world = world;
  a.B = cfg->bitwidth; a.G = cfg->group_size; a.sr = cfg->scheme; a.intlog = cfg->scale_encoding; a.theta = cfg->theta;
  a.gshift = -1;
  for (int sh = 0; sh < 16; ++sh)
    if ((1 << sh) == a.G) a.gshift = sh;
  a.lut = lut;
  a.pos = pos; a.T = tokens; a.H = row_len; a.out = out; a.odt = out_dtype; a.err = dev_err;
  const int64_t tasks = tokens * ((row_len + 1023) / 1024);
  if (tasks > INT32_MAX || row_len > INT32_MAX - 1024)
    return set_err(FC2_ECONFIG, "combine of %lld tokens x %lld is too large", (long long)tokens, (long long)row_len);
  int64_t blocks = (tasks + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  cudaStream_t st = (cudaStream_t)stream;
  switch (cfg->bitwidth) {
    case 2: k_moe_combine_q<2><<<(unsigned)blocks, 256, 0, st>>>(a); break;
    case 3: k_moe_combine_q<3><<<(unsigned)blocks, 256, 0, st>>>(a); break;
    case 4: k_moe_combine_q<4><<<(unsigned)blocks, 256, 0, st>>>(a); break;
    case 5: k_moe_combine_q<5><<<(unsigned)blocks, 256, 0, st>>>(a); break;
    case 6: k_moe_combine_q<6><<<(unsigned)blocks, 256, 0, st>>>(a); break;
    case 7: k_moe_combine_q<7><<<(unsigned)blocks, 256, 0, st>>>(a); break;
    default: k_moe_combine_q<8><<<(unsigned)blocks, 256, 0, st>>>(a); break;
  }
  return cuda_check("k_moe_combine_q");
}

}  // extern "C"
