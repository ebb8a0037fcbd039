// fc2_comm.cu -- one-process-per-GPU communicator for the quantized collectives.
//
// Every rank owns one symmetric device buffer (cudaMalloc, exported with
// cudaIpcGetMemHandle, opened by every peer).  Layout of each buffer:
//
//   [0, 16384)                     flag page: uint32 arrive[FC2_COMM_MAX] at 0;
//                                  [1024, 3072): small all-gather area [parity][rank][16];
//                                  [4096, 6144): pipelined two-step flags [stage][src][chunk]
//   [4096, 4096 + N*slot)          landing slots  land[src]   (stage 1, my shard)
//   [.., + N*slot)                 gather slots   gath[owner] (stage 2)
//   [.., + a2a_bytes)              All2All receive region
//   [.., + (2N^2 + N)*slot_os)     one-shot region (landing[parity][src][shard], results)
//
// Two-step AllReduce on rank r (collectives.py:263-315, one call):
//   1. one batched encode launch quantizes shard j of x straight into
//      peer j's land[r] (NVLink peer stores from the kernel's copy-out);
//   2. barrier;
//   3. k_reduce decodes land[0..N-1] (local), sums in fp32 in rank order,
//      re-encodes and stores the packed shard into every peer's gath[r];
//   4. barrier;
//   5. decode gath[0..N-1] (local) into the bf16/f32 output.
// Buffer reuse across calls is safe with the two barriers.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <algorithm>
#include <vector>

#include "../../include/fc2.h"
#include "fc2_common.cuh"
#include "fc2_decode.cuh"
#include "fc2_encode.cuh"

namespace fc2 {
int set_err(int code, const char* fmt, ...);
int cuda_check(const char* what);
int decode_batch_grid(const fc2_config* cfg, int32_t y_dtype, int32_t njobs, const void* const* payloads,
                      const int64_t* n, void* const* ys, const int64_t* n_out, int32_t* dev_err, void* stream);
const double* lut_for_cfg(const fc2_config* c, int* rc);
int num_sms();
}  // namespace fc2

using namespace fc2;

#define FC2_COMM_MAX 16
#define FC2_FLAG_BYTES 16384
#define FC2_PIPE_FLAGS 4096   // flag page: pipelined two-step flags [stage][src][chunk]
#define FC2_PIPE_MAXK 16
#define FC2_FUSED_CTR 8192    // flag page: the fused one-shot's grid-barrier counter (local)

struct fc2_comm {
  int rank, world, device;
  int64_t bytes;
  uint8_t* local;
  uint8_t* peer[FC2_COMM_MAX];
  bool opened[FC2_COMM_MAX];
  uint32_t epoch;
  uint32_t oneshot_calls;  // parity selects the one-shot landing buffer
  uint32_t fused_arrivals; // fused one-shot: CTAs that have reached its grid barrier so far
  uint32_t ag_calls;       // parity selects the small all-gather area
  uint32_t pipe_epoch;     // pipelined two-step: flag value of the current call (parity: buffer set)
  cudaStream_t s_red, s_gat;  // pipelined two-step: reduce / gather-decode streams (lazy)
  cudaEvent_t ev_start, ev_red, ev_gat;
};

namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct BarrierArgs {
  uint32_t* mine;                    // my arrive[] array
  uint32_t* peers[FC2_COMM_MAX];     // peer p's arrive[] array (mapped)
  int rank, world;
  uint32_t epoch;
  int32_t* err;
  long long timeout_cycles;
};

// One thread per peer: publish "rank reached epoch" to peer p, then wait for
// peer p's arrival in my array.  fence.sys first: every store this device made
// before this kernel (earlier kernels on the stream) is ordered before the flag.
__global__ void k_barrier(const __grid_constant__ BarrierArgs a) {
  pdl_wait_only();
  const int p = threadIdx.x;
  if (p >= a.world) return;
  __threadfence_system();
  st_release_sys(a.peers[p] + a.rank, a.epoch);
  const long long t0 = clock64();
  while ((int32_t)(ld_acquire_sys(a.mine + p) - a.epoch) < 0) {
    if (clock64() - t0 > a.timeout_cycles) {
      atomicOr(a.err, FC2_ERR_TIMEOUT);
      break;
    }
    __nanosleep(256);
  }
  __threadfence_system();
}

// Pipelined two-step flags.  Signal: thread p publishes "my chunk is in
// place" into peer p's flag word (fence.sys first, so the payload stores of
// the kernels before it on this stream are ordered before the flag).  Wait:
// thread s spins until source s's flag reaches the call's epoch.
struct FlagArgs {
  uint32_t* words[FC2_COMM_MAX];  // signal: flag word in peer p; wait: my flag word for source s
  int world;
  uint32_t epoch;
  int32_t* err;
  long long timeout_cycles;
};

__global__ void k_flag_signal(const __grid_constant__ FlagArgs a) {
  pdl_wait_only();
  const int p = threadIdx.x;
  if (p >= a.world) return;
  __threadfence_system();
  st_release_sys(a.words[p], a.epoch);
}

__global__ void k_flag_wait(const __grid_constant__ FlagArgs a) {
  pdl_wait_only();
  const int s = threadIdx.x;
  if (s >= a.world) return;
  const long long t0 = clock64();
  while ((int32_t)(ld_acquire_sys(a.words[s]) - a.epoch) < 0) {
    if (clock64() - t0 > a.timeout_cycles) {
      atomicOr(a.err, FC2_ERR_TIMEOUT);
      break;
    }
    __nanosleep(128);
  }
  __threadfence_system();
}

// Plain device copy, 16 bytes per thread-iteration; dst may be a peer
// buffer mapped through CUDA IPC (NVLink stores): the packed-bytes move of
// the collectives and the NVLink peak probe of bench.py.
__global__ void __launch_bounds__(512) k_copy_bytes(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                                    int64_t nbytes) {
  const int64_t n16 = nbytes >> 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  const int64_t tail = nbytes & 15;
  if (blockIdx.x == 0 && (int64_t)threadIdx.x < tail) dst[(n16 << 4) + threadIdx.x] = src[(n16 << 4) + threadIdx.x];
}

}  // namespace

// ---------------------------------------------------------------------------
// Fused one-shot AllReduce ("a fused single-kernel two-step
// with in-kernel flags"): one cooperative launch does what
// fc2_allreduce_oneshot does in four (encode -> barrier -> reduce+requant ->
// decode).  Warp = one group, float64-exact generic codec throughout (the
// same bits as the fast kernels; this path is for latency-bound sizes):
//   phase 1  group g of shard j of x -> packed, stored once per peer into
//            landing[par][me][j] of every rank (up to 8 destinations per store);
//   barrier  every CTA bumps a local counter; CTA 0 waits for all of them,
//            then publishes "rank r reached epoch" to every peer (the
//            k_barrier protocol) and every CTA waits for all peers' flags;
//   phase 2  group g of shard j: the N landed sources decoded and summed in
//            fp32 in rank order from +0.0, requantized into the local result
//            slot, decoded back to the bf16 grid straight into y.
// The landing parity alternates with fc2_allreduce_oneshot's, so mixed calls
// stay safe without a trailing barrier.
// ---------------------------------------------------------------------------
namespace {

struct FusedArgs {
  const void* x;
  int xdt;
  void* y;
  int ydt;
  int64_t n, S;             // elements, shard length (padded / N)
  int N, r, par;
  uint8_t* base[FC2_COMM_MAX];  // every rank's symmetric buffer (this process' mapping) + flag page
  int64_t region_off, slot;
  uint32_t* arrive_mine;
  uint32_t* arrive_peer[FC2_COMM_MAX];
  uint32_t epoch;
  uint32_t* gctr;
  uint32_t gtarget;
  int B, G, sr, intlog, theta;
  const double* lut;
  int32_t* err;
  long long timeout_cycles;
};

constexpr int kFusedMaxG = 256;  // largest group the fused kernel stages (8 warps x 1 KB of smem)

// element i of the chunk from the warp's staged group (floats, exact for bf16 /
// f32 input and for fp32 sums); g0 = first element of the group
struct StagedGroup {
  const float* v;
  int64_t g0;
  __device__ double operator()(int64_t i) const { return (double)v[i - g0]; }
};

__device__ __forceinline__ uint8_t* fused_land(const FusedArgs& a, int dst, int src, int shard) {
  return a.base[dst] + a.region_off + ((int64_t)a.par * a.N * a.N + (int64_t)src * a.N + shard) * a.slot;
}

__device__ bool spin_until(const uint32_t* p, uint32_t target, const FusedArgs& a) {
  const long long t0 = clock64();
  while ((int32_t)(ld_acquire_sys(p) - target) < 0) {
    if (clock64() - t0 > a.timeout_cycles) {
      atomicOr(a.err, FC2_ERR_TIMEOUT);
      return false;
    }
    __nanosleep(128);
  }
  return true;
}

__global__ void __launch_bounds__(256) k_allreduce_fused(const __grid_constant__ FusedArgs a) {
  const int warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
  const int64_t gps = a.S / a.G;            // groups per shard
  const int64_t total = gps * a.N;          // groups of the padded tensor
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  EncCtx cx;
  cx.n = a.S; cx.meta_off = a.S * a.B / 8; cx.intlog = a.intlog; cx.theta = a.theta; cx.lut = a.lut;
  cx.err = a.err;
  // ---- phase 1: my shards, packed, into every rank's landing row for me.
  // The group is staged in shared memory first (coalesced loads, one round
  // trip) so the float64 encoder's two passes over it never touch global memory.
  __shared__ float stage[8][kFusedMaxG];
  float* sg = stage[warp];
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; w < total; w += nw) {
    const int j = (int)(w / gps);
    const int64_t gl = w - (int64_t)j * gps;
    const int64_t e0 = (int64_t)j * a.S + gl * a.G;  // element of x
    for (int e = lane; e < a.G; e += 32) {
      const int64_t idx = e0 + e;
      float v = 0.0f;  // zero padding past n (collectives.py:167-172)
      if (idx < a.n && (int64_t)gl * a.G + e < a.S)
        v = a.xdt == FC2_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.x)[idx])
                              : reinterpret_cast<const float*>(a.x)[idx];
      sg[e] = v;
    }
    __syncwarp();
    const StagedGroup ld{sg, gl * a.G};
    for (int d0 = 0; d0 < a.N; d0 += 8) {  // OutList carries up to 8 destinations
      OutList o;
      o.nd = a.N - d0 < 8 ? a.N - d0 : 8;
      for (int d = 0; d < o.nd; ++d) o.p[d] = fused_land(a, d0 + d, a.r, j);
      generic_encode_group(ld, o, a.S, gl, a.B, a.G, a.sr != 0, cx, true);
    }
    __syncwarp();
  }
  // ---- grid barrier (co-resident CTAs: cooperative launch), then the peers
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    atomicAdd(a.gctr, 1u);
    if (blockIdx.x == 0 && spin_until(a.gctr, a.gtarget, a)) {
      __threadfence_system();
      for (int p = 0; p < a.N; ++p) st_release_sys(a.arrive_peer[p] + a.r, a.epoch);
    }
    for (int p = 0; p < a.N; ++p)
      if (!spin_until(a.arrive_mine + p, a.epoch, a)) break;
    __threadfence_system();
  }
  __syncthreads();
  // ---- phase 2: every shard reduced, requantized and decoded locally
  uint8_t* result = a.base[a.r] + a.region_off + (int64_t)2 * a.N * a.N * a.slot;
  DecCtx dc;
  dc.n = a.S; dc.meta_off = a.S * a.B / 8; dc.B = a.B; dc.G = a.G; dc.sr = a.sr != 0; dc.intlog = a.intlog != 0;
  dc.theta = a.theta; dc.lut = a.lut; dc.err = a.err;
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; w < total; w += nw) {
    const int j = (int)(w / gps);
    const int64_t gl = w - (int64_t)j * gps;
    const int64_t g0 = gl * a.G;  // group start inside the shard
    // every source's record first (independent loads), then its codes: sums in
    // fp32 from +0.0 in rank order, lane = elements lane, lane + 32, ...
    float acc[kFusedMaxG / 32];
#pragma unroll
    for (int k = 0; k < kFusedMaxG / 32; ++k) acc[k] = 0.0f;
    for (int s0 = 0; s0 < a.N; s0 += 8) {
      const int ns = a.N - s0 < 8 ? a.N - s0 : 8;
      GroupMeta m[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < ns) m[q] = read_meta(fused_land(a, a.r, s0 + q, j), gl, dc);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q >= ns) break;
        const uint8_t* P = fused_land(a, a.r, s0 + q, j);
#pragma unroll
        for (int k = 0; k < kFusedMaxG / 32; ++k) {
          const int e = lane + 32 * k;
          if (e >= a.G) break;
          float v;
          if (dc.sr && e == m[q].imax) v = m[q].smax;  // imax written last (codec.py:559-561)
          else if (dc.sr && e == m[q].imin) v = m[q].smin;
          else v = dq32(load_code1(P, a.S, g0 + e, a.B), m[q], dc.intlog);
          acc[k] = __fadd_rn(acc[k], v);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kFusedMaxG / 32; ++k)
      if (lane + 32 * k < a.G) sg[lane + 32 * k] = acc[k];
    __syncwarp();
    OutList o;
    o.nd = 1;
    o.p[0] = result + (int64_t)j * a.slot;
    generic_encode_group(StagedGroup{sg, g0}, o, a.S, gl, a.B, a.G, a.sr != 0, cx, true);
    __syncwarp();  // the group's planes and record, written by the warp, before the warp reads them back
    const GroupMeta mr = read_meta(o.p[0], gl, dc);
    for (int e = lane; e < a.G; e += 32) {
      const int64_t idx = (int64_t)j * a.S + g0 + e;
      if (idx >= a.n) break;
      float v;
      if (dc.sr && e == mr.imax) v = mr.smax;
      else if (dc.sr && e == mr.imin) v = mr.smin;
      else v = dq32(load_code1(o.p[0], a.S, g0 + e, a.B), mr, dc.intlog);
      const uint32_t bits = bf16_bits(v);  // the bf16 grid (collectives.py:185-186)
      if (a.ydt == FC2_BF16) reinterpret_cast<uint16_t*>(a.y)[idx] = (uint16_t)bits;
      else reinterpret_cast<float*>(a.y)[idx] = bf16_val(bits);
    }
    __syncwarp();
  }
}

}  // namespace

extern "C" {

int fc2_copy_bytes(void* dst, const void* src, int64_t nbytes, int32_t ctas, void* stream) {
  if (nbytes <= 0) return FC2_OK;
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u)
    return set_err(FC2_ECONFIG, "fc2_copy_bytes needs 16-byte aligned buffers");
  int64_t blocks = ((nbytes >> 4) + 511) / 512;
  const int64_t cap = ctas > 0 ? ctas : 148 * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_copy_bytes<<<(unsigned)blocks, 512, 0, (cudaStream_t)stream>>>((uint8_t*)dst, (const uint8_t*)src, nbytes);
  return cuda_check("k_copy_bytes");
}

int fc2_comm_create(int32_t rank, int32_t world, int64_t bytes, fc2_comm** out, void* handle_out) {
  if (world < 1 || world > FC2_COMM_MAX || rank < 0 || rank >= world)
    return set_err(FC2_ECONFIG, "bad rank/world %d/%d (max %d ranks)", rank, world, FC2_COMM_MAX);
  fc2_comm* c = new fc2_comm();
  memset(c, 0, sizeof(*c));
  c->rank = rank;
  c->world = world;
  cudaGetDevice(&c->device);
  c->bytes = bytes + FC2_FLAG_BYTES;
  if (cudaMalloc(&c->local, c->bytes) != cudaSuccess) {
    delete c;
    return set_err(FC2_ECUDA, "cudaMalloc(%lld) failed", (long long)c->bytes);
  }
  cudaMemset(c->local, 0, FC2_FLAG_BYTES);
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, c->local) != cudaSuccess) {
    cudaFree(c->local);
    delete c;
    return set_err(FC2_ECUDA, "cudaIpcGetMemHandle failed");
  }
  memcpy(handle_out, &h, sizeof(h));
  c->peer[rank] = c->local;
  c->opened[rank] = false;
  cudaDeviceSynchronize();
  *out = c;
  return FC2_OK;
}

int fc2_comm_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

int fc2_comm_open_peers(fc2_comm* c, const void* handles) {
  const uint8_t* hs = (const uint8_t*)handles;
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, hs + (size_t)p * sizeof(h), sizeof(h));
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return set_err(FC2_ECUDA, "cudaIpcOpenMemHandle(peer %d): %s", p, cudaGetErrorString(e));
    c->peer[p] = (uint8_t*)ptr;
    c->opened[p] = true;
  }
  return FC2_OK;
}

int fc2_comm_destroy(fc2_comm* c) {
  if (!c) return FC2_OK;
  cudaDeviceSynchronize();
  if (c->s_red) {
    cudaStreamDestroy(c->s_red);
    cudaStreamDestroy(c->s_gat);
    cudaEventDestroy(c->ev_start);
    cudaEventDestroy(c->ev_red);
    cudaEventDestroy(c->ev_gat);
  }
  for (int p = 0; p < c->world; ++p)
    if (c->opened[p]) cudaIpcCloseMemHandle(c->peer[p]);
  cudaFree(c->local);
  delete c;
  return FC2_OK;
}

void* fc2_comm_buffer(fc2_comm* c, int32_t peer) {
  if (!c || peer < 0 || peer >= c->world) return nullptr;
  return c->peer[peer] + FC2_FLAG_BYTES;
}

int fc2_comm_barrier(fc2_comm* c, int32_t* dev_err, double timeout_s, void* stream) {
  BarrierArgs a;
  a.mine = (uint32_t*)c->local;
  for (int p = 0; p < c->world; ++p) a.peers[p] = (uint32_t*)c->peer[p];
  a.rank = c->rank;
  a.world = c->world;
  a.epoch = ++c->epoch;
  a.err = dev_err;
  a.timeout_cycles = (long long)(timeout_s * 2.0e9);
  launch_pdl(k_barrier, 1, 32, 0, (cudaStream_t)stream, a);
  return cuda_check("k_barrier");
}

int fc2_allreduce_2step(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, void* y,
                        int32_t y_dtype, int64_t n, int64_t slot_bytes, int32_t* dev_err, double timeout_s,
                        void* stream) {
  const int N = c->world, r = c->rank;
  int rc = fc2_check_config(cfg);
  if (rc) return rc;
  const int64_t mult = (int64_t)N * cfg->group_size;
  const int64_t padded = (n + mult - 1) / mult * mult;
  const int64_t S = padded / N;
  int64_t F = 0;
  rc = fc2_footprint(cfg, S, &F);
  if (rc) return rc;
  if (F > slot_bytes || (slot_bytes & 15)) return set_err(FC2_ECONFIG, "slot too small for shard footprint");
  if ((int64_t)2 * N * slot_bytes > c->bytes - FC2_FLAG_BYTES)
    return set_err(FC2_ECONFIG, "communicator buffer too small");
  const int esz = x_dtype == FC2_BF16 ? 2 : (x_dtype == FC2_F32 ? 4 : 8);
  auto land = [&](int dst, int src) { return (void*)(c->peer[dst] + FC2_FLAG_BYTES + (int64_t)src * slot_bytes); };
  auto gath = [&](int dst, int owner) {
    return (void*)(c->peer[dst] + FC2_FLAG_BYTES + (int64_t)(N + owner) * slot_bytes);
  };
  // 1. quantize my N shards straight into the owners' landing slots
  std::vector<const void*> xs(N);
  std::vector<int64_t> nv(N), ns(N);
  std::vector<void*> outs(N);
  for (int j = 0; j < N; ++j) {
    const int64_t valid = n - (int64_t)j * S;
    nv[j] = valid < 0 ? 0 : (valid > S ? S : valid);
    ns[j] = S;
    xs[j] = nv[j] ? (const uint8_t*)x + (int64_t)j * S * esz : x;
    outs[j] = land(j, r);
  }
  rc = fc2_encode_batch(cfg, x_dtype, N, xs.data(), nv.data(), ns.data(), outs.data(), dev_err, stream);
  if (rc) return rc;
  rc = fc2_comm_barrier(c, dev_err, timeout_s, stream);
  if (rc) return rc;
  // 3. reduce my shard from the N landing slots, push the packed result to everyone
  std::vector<const void*> srcs(N);
  std::vector<void*> dsts(N);
  for (int s = 0; s < N; ++s) srcs[s] = land(r, s);
  for (int p = 0; p < N; ++p) dsts[p] = gath(p, r);
  rc = fc2_reduce_requant(cfg, N, srcs.data(), S, N, dsts.data(), dev_err, stream);
  if (rc) return rc;
  rc = fc2_comm_barrier(c, dev_err, timeout_s, stream);
  if (rc) return rc;
  // 5. decode every owner's shard into the output (padding stripped)
  std::vector<const void*> gs(N);
  for (int o = 0; o < N; ++o) gs[o] = gath(r, o);
  return fc2_gather_decode(cfg, N, gs.data(), S, y, y_dtype, n, dev_err, stream);
}

// One-shot AllReduce: same arithmetic as the two-step
// (collectives.py:263-315), one exchange.  Region layout at region_off:
//   landing[parity][src][shard]  2 * N * N slots
//   result[shard]                N slots (this rank's requantized shards)
int fc2_allreduce_oneshot(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, void* y,
                          int32_t y_dtype, int64_t n, int64_t slot_bytes, int64_t region_off, int32_t* dev_err,
                          double timeout_s, void* stream) {
  const int N = c->world, r = c->rank;
  int rc = fc2_check_config(cfg);
  if (rc) return rc;
  const int64_t mult = (int64_t)N * cfg->group_size;
  const int64_t padded = (n + mult - 1) / mult * mult;
  const int64_t S = padded / N;
  int64_t F = 0;
  rc = fc2_footprint(cfg, S, &F);
  if (rc) return rc;
  if (F > slot_bytes || (slot_bytes & 15)) return set_err(FC2_ECONFIG, "slot too small for shard footprint");
  if (region_off < 0 || (region_off & 15) ||
      region_off + (int64_t)(2 * N * N + N) * slot_bytes > c->bytes - FC2_FLAG_BYTES)
    return set_err(FC2_ECONFIG, "communicator buffer too small for the one-shot region");
  if (N * N > FC2_MAX_JOBS) return set_err(FC2_ECONFIG, "one-shot supports world <= 16");
  const int esz = x_dtype == FC2_BF16 ? 2 : (x_dtype == FC2_F32 ? 4 : 8);
  const int par = (int)(c->oneshot_calls++ & 1u);
  auto land = [&](int dst, int src, int shard) {
    return (uint8_t*)c->peer[dst] + FC2_FLAG_BYTES + region_off +
           ((int64_t)par * N * N + (int64_t)src * N + shard) * slot_bytes;
  };
  uint8_t* result = c->local + FC2_FLAG_BYTES + region_off + (int64_t)2 * N * N * slot_bytes;
  // 1. my N shards, packed, into every rank's landing row for me (one launch)
  std::vector<const void*> xs(N * N);
  std::vector<int64_t> nv(N * N), ns(N * N);
  std::vector<void*> outs(N * N);
  for (int d = 0; d < N; ++d)
    for (int j = 0; j < N; ++j) {
      const int64_t valid = n - (int64_t)j * S;
      const int k = d * N + j;
      nv[k] = valid < 0 ? 0 : (valid > S ? S : valid);
      ns[k] = S;
      xs[k] = nv[k] ? (const uint8_t*)x + (int64_t)j * S * esz : x;
      outs[k] = land(d, r, j);
    }
  rc = fc2_encode_batch(cfg, x_dtype, N * N, xs.data(), nv.data(), ns.data(), outs.data(), dev_err, stream);
  if (rc) return rc;
  rc = fc2_comm_barrier(c, dev_err, timeout_s, stream);
  if (rc) return rc;
  // 2. reduce + requantize every shard locally (sources: landing[par][s][*])
  std::vector<const void*> srcs(N);
  for (int s2 = 0; s2 < N; ++s2) srcs[s2] = land(r, s2, 0);
  void* dst = result;
  rc = fc2_reduce_requant_batch(cfg, N, srcs.data(), S, N, slot_bytes, 1, &dst, slot_bytes, dev_err, stream);
  if (rc) return rc;
  // 3. decode all shards (padding stripped, bf16 grid)
  std::vector<const void*> gs(N);
  for (int o = 0; o < N; ++o) gs[o] = result + (int64_t)o * slot_bytes;
  return fc2_gather_decode(cfg, N, gs.data(), S, y, y_dtype, n, dev_err, stream);
}

// Fused one-shot AllReduce: same region, same result bits as
// fc2_allreduce_oneshot, one cooperative kernel (see k_allreduce_fused).
int fc2_allreduce_fused(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, void* y,
                        int32_t y_dtype, int64_t n, int64_t slot_bytes, int64_t region_off, int32_t* dev_err,
                        double timeout_s, void* stream) {
  const int N = c->world, r = c->rank;
  int rc = fc2_check_config(cfg);
  if (rc) return rc;
  if ((x_dtype != FC2_BF16 && x_dtype != FC2_F32) || (y_dtype != FC2_BF16 && y_dtype != FC2_F32))
    return set_err(FC2_ECONFIG, "the fused one-shot takes bf16 / f32 tensors");
  if (cfg->group_size > kFusedMaxG)
    return set_err(FC2_ECONFIG, "the fused one-shot stages groups of at most %d elements", kFusedMaxG);
  const int64_t mult = (int64_t)N * cfg->group_size;
  const int64_t padded = (n + mult - 1) / mult * mult;
  const int64_t S = padded / N;
  int64_t F = 0;
  rc = fc2_footprint(cfg, S, &F);
  if (rc) return rc;
  if (F > slot_bytes || (slot_bytes & 15)) return set_err(FC2_ECONFIG, "slot too small for shard footprint");
  if (region_off < 0 || (region_off & 15) ||
      region_off + (int64_t)(2 * N * N + N) * slot_bytes > c->bytes - FC2_FLAG_BYTES)
    return set_err(FC2_ECONFIG, "communicator buffer too small for the one-shot region");
  const double* lut = lut_for_cfg(cfg, &rc);
  if (rc) return rc;
  if (n == 0) return FC2_OK;
  FusedArgs a;
  memset(&a, 0, sizeof(a));
  a.x = x; a.xdt = x_dtype; a.y = y; a.ydt = y_dtype; a.n = n; a.S = S; a.N = N; a.r = r;
  a.par = (int)(c->oneshot_calls++ & 1u);
  for (int p = 0; p < N; ++p) {
    a.base[p] = c->peer[p] + FC2_FLAG_BYTES;
    a.arrive_peer[p] = (uint32_t*)c->peer[p];
  }
  a.region_off = region_off; a.slot = slot_bytes;
  a.arrive_mine = (uint32_t*)c->local;
  a.epoch = ++c->epoch;
  a.gctr = (uint32_t*)(c->local + FC2_FUSED_CTR);
  a.B = cfg->bitwidth; a.G = cfg->group_size; a.sr = cfg->scheme; a.intlog = cfg->scale_encoding;
  a.theta = cfg->theta; a.lut = lut; a.err = dev_err;
  a.timeout_cycles = (long long)(timeout_s * 2.0e9);
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_allreduce_fused, 256, 0);
    if (per_sm < 1) per_sm = 1;
  }
  const int64_t groups = padded / cfg->group_size;
  int64_t grid = (groups + 7) / 8;
  const int64_t cap = (int64_t)per_sm * num_sms();
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  a.gtarget = c->fused_arrivals + (uint32_t)grid;  // committed only once the launch is accepted
  void* args[] = {&a};
  if (cudaLaunchCooperativeKernel((const void*)k_allreduce_fused, dim3((unsigned)grid), dim3(256), args, 0,
                                  (cudaStream_t)stream) != cudaSuccess)
    return cuda_check("k_allreduce_fused (cooperative launch)");
  c->fused_arrivals = a.gtarget;
  return cuda_check("k_allreduce_fused");
}

// Pipelined two-step (the NVSwitch form of the reference's
// microchunked HierPP schedule, scheduling.py:119-156): the shard is cut into
// K microchunks of whole groups (groups are independent, so the result is the
// two-step's bit for bit) and the three stages run on three streams,
// synchronised per chunk by release/acquire flags in peer memory instead of
// two device-wide barriers:
//   caller stream   encode chunk k of my N shards -> peers' land[r][k]; signal F1[r][k]
//   s_red           wait F1[*][k]; reduce + requantize chunk k -> peers' gath[r][k]; signal F2[r][k]
//   s_gat           wait F2[*][k]; decode chunk k of the N shards into y
// so chunk k + 1's encode overlaps chunk k's reduce and chunk k - 1's decode.
// Buffers are double-buffered by call parity (region_off: 2 sets of land +
// gath slots, chunk_bytes each), which with the flag waits makes back-to-back
// calls safe without a trailing barrier.
int fc2_allreduce_2step_pipe(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, void* y,
                             int32_t y_dtype, int64_t n, int32_t chunks, int64_t chunk_bytes, int64_t region_off,
                             int64_t region_bytes, int32_t* dev_err, double timeout_s, void* stream) {
  NoPdl no_pdl;  // three streams joined by events: plain launches
  const int N = c->world, r = c->rank;
  int rc = fc2_check_config(cfg);
  if (rc) return rc;
  if (chunks < 1 || chunks > FC2_PIPE_MAXK) return set_err(FC2_ECONFIG, "chunks must be in [1, %d]", FC2_PIPE_MAXK);
  const int64_t G = cfg->group_size;
  const int64_t mult = (int64_t)N * G;
  const int64_t padded = (n + mult - 1) / mult * mult;
  const int64_t S = padded / N;
  // microchunk length: whole groups, a multiple of 1024 elements (aligned planes)
  int64_t q = 1024;
  while (q % G) q += 1024;
  int64_t Sk = (S + chunks - 1) / chunks;
  Sk = (Sk + q - 1) / q * q;
  const int K = S == 0 ? 0 : (int)((S + Sk - 1) / Sk);
  int64_t F = 0;
  rc = fc2_footprint(cfg, Sk, &F);
  if (rc) return rc;
  if (F > chunk_bytes || (chunk_bytes & 15)) return set_err(FC2_ECONFIG, "chunk slot too small for the microchunk");
  const int64_t set_bytes = (int64_t)2 * N * chunks * chunk_bytes;  // land + gath of one parity
  if (region_off < 0 || (region_off & 15) || 2 * set_bytes > region_bytes ||
      region_off + region_bytes + FC2_FLAG_BYTES > c->bytes)
    return set_err(FC2_ECONFIG, "communicator buffer too small for the pipelined region");
  if (n == 0) return FC2_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (!c->s_red) {
    if (cudaStreamCreateWithFlags(&c->s_red, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->s_gat, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_red, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_gat, cudaEventDisableTiming) != cudaSuccess)
      return set_err(FC2_ECUDA, "stream/event creation failed");
  }
  const uint32_t epoch = ++c->pipe_epoch;
  const int par = (int)(epoch & 1u);
  const int esz = x_dtype == FC2_BF16 ? 2 : (x_dtype == FC2_F32 ? 4 : 8);
  const int ysz = y_dtype == FC2_BF16 ? 2 : (y_dtype == FC2_F32 ? 4 : 8);
  auto base = [&](int peer) { return c->peer[peer] + FC2_FLAG_BYTES + region_off + (int64_t)par * set_bytes; };
  auto land = [&](int peer, int src, int k) { return (void*)(base(peer) + ((int64_t)src * chunks + k) * chunk_bytes); };
  auto gath = [&](int peer, int own, int k) {
    return (void*)(base(peer) + ((int64_t)(N + own) * chunks + k) * chunk_bytes);
  };
  auto flag = [&](int peer, int stage, int src, int k) {
    return reinterpret_cast<uint32_t*>(c->peer[peer] + FC2_PIPE_FLAGS) + (stage * FC2_COMM_MAX + src) * FC2_PIPE_MAXK + k;
  };
  const long long tmo = (long long)(timeout_s * 2.0e9);
  auto signal = [&](int stage, int k, cudaStream_t s) {
    FlagArgs a;
    for (int p = 0; p < N; ++p) a.words[p] = flag(p, stage, r, k);
    a.world = N; a.epoch = epoch; a.err = dev_err; a.timeout_cycles = tmo;
    launch_pdl(k_flag_signal, 1, 32, 0, s, a);
    return cuda_check("k_flag_signal");
  };
  auto wait = [&](int stage, int k, cudaStream_t s) {
    FlagArgs a;
    for (int p = 0; p < N; ++p) a.words[p] = flag(r, stage, p, k);
    a.world = N; a.epoch = epoch; a.err = dev_err; a.timeout_cycles = tmo;
    launch_pdl(k_flag_wait, 1, 32, 0, s, a);
    return cuda_check("k_flag_wait");
  };
  // the side streams start where the caller's stream is now
  cudaEventRecord(c->ev_start, st);
  cudaStreamWaitEvent(c->s_red, c->ev_start, 0);
  cudaStreamWaitEvent(c->s_gat, c->ev_start, 0);
  for (int k = 0; k < K; ++k) {
    const int64_t e0 = (int64_t)k * Sk, len = std::min<int64_t>(Sk, S - e0);
    // 1. encode chunk k of my N shards into the owners' landing slots
    std::vector<const void*> xs(N);
    std::vector<int64_t> nv(N), ns(N);
    std::vector<void*> outs(N);
    for (int j = 0; j < N; ++j) {
      const int64_t at = (int64_t)j * S + e0;
      const int64_t valid = n - at;
      nv[j] = valid < 0 ? 0 : (valid > len ? len : valid);
      ns[j] = len;
      xs[j] = nv[j] ? (const uint8_t*)x + at * esz : x;
      outs[j] = land(j, r, k);
    }
    if ((rc = fc2_encode_batch(cfg, x_dtype, N, xs.data(), nv.data(), ns.data(), outs.data(), dev_err, st))) return rc;
    if ((rc = signal(0, k, st))) return rc;
    // 2. reduce chunk k of my shard once every source has landed it
    if ((rc = wait(0, k, c->s_red))) return rc;
    std::vector<const void*> srcs(N);
    std::vector<void*> dsts(N);
    for (int s2 = 0; s2 < N; ++s2) srcs[s2] = land(r, s2, k);
    for (int p = 0; p < N; ++p) dsts[p] = gath(p, r, k);
    if ((rc = fc2_reduce_requant(cfg, N, srcs.data(), len, N, dsts.data(), dev_err, c->s_red))) return rc;
    if ((rc = signal(1, k, c->s_red))) return rc;
    // 3. decode chunk k of every owner's shard
    if ((rc = wait(1, k, c->s_gat))) return rc;
    std::vector<const void*> gs(N);
    std::vector<int64_t> gn(N), go(N);
    std::vector<void*> ys(N);
    for (int o = 0; o < N; ++o) {
      const int64_t at = (int64_t)o * S + e0;
      const int64_t rem = n - at;
      gs[o] = gath(r, o, k);
      gn[o] = len;
      go[o] = rem < 0 ? 0 : (rem > len ? len : rem);
      ys[o] = (uint8_t*)y + (go[o] ? at : 0) * ysz;
    }
    if ((rc = decode_batch_grid(cfg, y_dtype, N, gs.data(), gn.data(), ys.data(), go.data(), dev_err, c->s_gat)))
      return rc;
  }
  // the caller's stream continues after both side streams
  cudaEventRecord(c->ev_red, c->s_red);
  cudaEventRecord(c->ev_gat, c->s_gat);
  cudaStreamWaitEvent(st, c->ev_red, 0);
  cudaStreamWaitEvent(st, c->ev_gat, 0);
  return cuda_check("pipelined two-step");
}

}  // extern "C"

namespace {

// Quantized All2All over the symmetric buffers (collectives.py:428-482 for
// dispatch; combine = the same exchange with the transposed matrix).
// m: host int64[N*N], m[src*N + dst] = elements rank src sends to dst.
// x: this rank's payload, blocks for dst = 0..N-1 back to back -- or, with
//    rows != nullptr (MoE token dispatch), token rows: block dst is the
//    rows rows[dst * rows_stride + i] of x (row_len elements each), gathered
//    inside the encoder.
// y: this rank's receive buffer, blocks from src = 0..N-1 back to back
//    (y_dtype F32 or BF16).  The diagonal block is an exact (gather-)copy when
//    copy_diag, else left untouched.  region_off: byte offset of the All2All
//    region.
// byte offset of the block src -> dst inside dst's All2All region (blocks of
// sources 0..N-1 back to back, 16-byte aligned slots; the diagonal and empty
// blocks take no space); *F_out = the block's payload bytes
int64_t a2a_slot(const fc2_config* cfg, const int64_t* m, int N, int dst, int src, int64_t* F_out) {
  const int64_t G = cfg->group_size;
  int64_t off = 0;
  for (int s = 0; s <= src; ++s) {
    const int64_t v = m[(int64_t)s * N + dst];
    int64_t F = 0;
    if (s != dst && v > 0) fc2_footprint(cfg, (v + G - 1) / G * G, &F);
    if (s == src) { *F_out = F; return off; }
    off += (F + 15) / 16 * 16;
  }
  return off;
}

// decode_recv = false: the received blocks stay packed in the region (the
// fused MoE combine reads them there) and the trailing barrier is the
// caller's, after it has consumed them.
int a2a_core(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, const int64_t* m,
             const int32_t* rows, int64_t rows_stride, int64_t row_len, void* y, int32_t y_dtype, bool copy_diag,
             int64_t region_off, int64_t region_bytes, int32_t* dev_err, double timeout_s, void* stream,
             bool decode_recv = true) {
  const int N = c->world, r = c->rank;
  int rc = fc2_check_config(cfg);
  if (rc) return rc;
  const int64_t G = cfg->group_size;
  const int esz = x_dtype == FC2_BF16 ? 2 : (x_dtype == FC2_F32 ? 4 : 8);
  const int ysz = y_dtype == FC2_BF16 ? 2 : (y_dtype == FC2_F32 ? 4 : 8);
  auto slot_off = [&](int dst, int src, int64_t* F_out) -> int64_t { return a2a_slot(cfg, m, N, dst, src, F_out); };
  if (region_off < 0 || region_bytes < 0 || region_off + region_bytes + FC2_FLAG_BYTES > c->bytes)
    return set_err(FC2_ECONFIG, "a2a region [%lld, +%lld) outside the communicator buffer", (long long)region_off,
                   (long long)region_bytes);
  for (int d = 0; d < N; ++d) {  // every receiver's blocks must fit the All2All region itself
    int64_t F = 0;
    int64_t end = slot_off(d, N - 1, &F) + F;
    if (end > region_bytes)
      return set_err(FC2_ECONFIG, "All2All blocks for rank %d need %lld bytes; the All2All region holds %lld", d,
                     (long long)end, (long long)region_bytes);
  }
  std::vector<const void*> xs;
  std::vector<const int32_t*> rs;
  std::vector<int64_t> nv, ns;
  std::vector<void*> outs;
  int64_t soff = 0;
  for (int d = 0; d < N; ++d) {
    const int64_t v = m[(int64_t)r * N + d];
    if (d != r && v > 0) {
      int64_t F = 0;
      const int64_t o = slot_off(d, r, &F);
      xs.push_back((const uint8_t*)x + soff * esz);
      rs.push_back(rows ? rows + (int64_t)d * rows_stride : nullptr);
      nv.push_back(v);
      ns.push_back((v + G - 1) / G * G);
      outs.push_back(c->peer[d] + FC2_FLAG_BYTES + region_off + o);
    }
    soff += v;
  }
  for (size_t i = 0; i < xs.size(); i += FC2_MAX_JOBS) {
    const int nj = (int)std::min<size_t>(FC2_MAX_JOBS, xs.size() - i);
    rc = rows ? fc2_encode_batch_rows(cfg, x_dtype, nj, x, rs.data() + i, row_len, nv.data() + i, ns.data() + i,
                                      outs.data() + i, dev_err, stream)
              : fc2_encode_batch(cfg, x_dtype, nj, xs.data() + i, nv.data() + i, ns.data() + i, outs.data() + i,
                                 dev_err, stream);
    if (rc) return rc;
  }
  rc = fc2_comm_barrier(c, dev_err, timeout_s, stream);
  if (rc || !decode_recv) return rc;
  std::vector<const void*> ps;
  std::vector<int64_t> pn, po;
  std::vector<void*> ys;
  int64_t roff = 0;
  for (int s = 0; s < N; ++s) {
    const int64_t v = m[(int64_t)s * N + r];
    if (s != r && v > 0) {
      int64_t F = 0;
      const int64_t o = slot_off(r, s, &F);
      ps.push_back(c->local + FC2_FLAG_BYTES + region_off + o);
      pn.push_back((v + G - 1) / G * G);
      ys.push_back((uint8_t*)y + roff * ysz);
      po.push_back(v);
    }
    roff += v;
  }
  for (size_t i = 0; i < ps.size(); i += FC2_MAX_JOBS) {
    const int nj = (int)std::min<size_t>(FC2_MAX_JOBS, ps.size() - i);
    rc = fc2_decode_batch(cfg, y_dtype, nj, ps.data() + i, pn.data() + i, ys.data() + i, po.data() + i, dev_err,
                          stream);
    if (rc) return rc;
  }
  // diagonal block: exact copy, non-finite values flagged (collectives.py:152-164, 466-468)
  if (copy_diag) {
    int64_t so = 0, ro = 0;
    for (int d = 0; d < r; ++d) so += m[(int64_t)r * N + d];
    for (int s = 0; s < r; ++s) ro += m[(int64_t)s * N + r];
    const int64_t v = m[(int64_t)r * N + r];
    if (v > 0) {
      rc = rows ? fc2_gather_rows_check(x, x_dtype, rows + (int64_t)r * rows_stride, v / row_len, row_len,
                                        (uint8_t*)y + ro * ysz, y_dtype, dev_err, stream)
                : fc2_copy_check((const uint8_t*)x + so * esz, x_dtype, (uint8_t*)y + ro * ysz, y_dtype, v, dev_err,
                                 stream);
      if (rc) return rc;
    }
  }
  // everyone has consumed its region before anyone writes the next call's blocks
  return fc2_comm_barrier(c, dev_err, timeout_s, stream);
}

// plain stores of my n values into every peer's small all-gather area
__global__ void k_put_small(const int32_t* __restrict__ mine, int n, int rank, int world,
                            const __grid_constant__ BarrierArgs peers, int64_t area_off) {
  const int i = (int)threadIdx.x;
  if (i >= n * world) return;
  const int p = i / n, k = i % n;
  int32_t* dst = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(peers.peers[p]) + area_off) + rank * 16 + k;
  *dst = mine[k];
}

}  // namespace

extern "C" {

int fc2_a2a_q(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, const int64_t* matrix,
              void* y, int32_t y_dtype, int64_t region_off, int64_t region_bytes, int32_t* dev_err,
              double timeout_s, void* stream) {
  return a2a_core(c, cfg, x, x_dtype, matrix, nullptr, 0, 0, y, y_dtype, true, region_off, region_bytes, dev_err,
                  timeout_s, stream);
}

// Small all-gather through the flag page (the MoE token counts): rank r's n
// (<= 16) int32 values land in every peer's area at [call parity][r]; after
// the barrier all_out[p * n + k] = value k of rank p.  The parity double
// buffer keeps a fast peer's next call from overwriting values not yet read.
int fc2_comm_allgather_i32(fc2_comm* c, const int32_t* mine, int32_t n, int32_t* all_out, int32_t* dev_err,
                           double timeout_s, void* stream) {
  if (n < 1 || n > 16) return set_err(FC2_ECONFIG, "small all-gather takes 1..16 values");
  const int N = c->world;
  const int par = (int)(c->ag_calls++ & 1u);
  const int64_t area = 1024 + (int64_t)par * FC2_COMM_MAX * 16 * 4;
  BarrierArgs pa;
  for (int p = 0; p < N; ++p) pa.peers[p] = (uint32_t*)c->peer[p];
  k_put_small<<<1, 256, 0, (cudaStream_t)stream>>>(mine, n, c->rank, N, pa, area);
  int rc = cuda_check("k_put_small");
  if (rc) return rc;
  rc = fc2_comm_barrier(c, dev_err, timeout_s, stream);
  if (rc) return rc;
  if (cudaMemcpy2DAsync(all_out, n * sizeof(int32_t), c->local + area, 16 * sizeof(int32_t), n * sizeof(int32_t),
                        N, cudaMemcpyDeviceToDevice, (cudaStream_t)stream) != cudaSuccess)
    return set_err(FC2_ECUDA, "cudaMemcpy2DAsync failed");
  return FC2_OK;
}

// MoE token dispatch (BASELINE configs[3]): token_matrix[s*N + d] = rows rank
// s sends to rank d (every rank knows it, e.g. from fc2_moe_route counts and
// fc2_comm_allgather_i32); rows_dev: this rank's fc2_moe_route lists (dst d
// at rows_dev + d * tokens).  y receives, per source rank in order, the
// QDQ'd rows (exact on the diagonal).
int fc2_moe_dispatch(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, int64_t tokens,
                     int64_t row_len, const int32_t* rows_dev, const int64_t* token_matrix, void* y, int32_t y_dtype,
                     int64_t region_off, int64_t region_bytes, int32_t* dev_err, double timeout_s, void* stream) {
  const int N = c->world;
  if (row_len <= 0 || row_len % 8) return set_err(FC2_ECONFIG, "row length must be a positive multiple of 8");
  std::vector<int64_t> m((size_t)N * N);
  for (int i = 0; i < N * N; ++i) {
    if (token_matrix[i] < 0 || token_matrix[i] > tokens) return set_err(FC2_ECONFIG, "token matrix entry out of range");
    m[i] = token_matrix[i] * row_len;
  }
  return a2a_core(c, cfg, x, x_dtype, m.data(), rows_dev, tokens, row_len, y, y_dtype, true, region_off,
                  region_bytes, dev_err, timeout_s, stream);
}

// MoE combine: the expert rank returns, to every source rank s, the rows it
// received from s (y holds them in dispatch order), quantized like dispatch;
// the source rank then sums, per token, the returned rows in destination-rank
// order in fp32 (exact rows for its own rank): out[t] = sum_d block(d)[pos[t][d]].
// scratch: float32 rows for every block this rank receives back (the sum of
// token_matrix[rank][*] rows; the diagonal's share is left unused).
int fc2_moe_combine(fc2_comm* c, const fc2_config* cfg, const void* y, int32_t y_dtype, int64_t tokens,
                    int64_t row_len, const int64_t* token_matrix, const int32_t* pos_dev, float* scratch, void* out,
                    int32_t out_dtype, int64_t region_off, int64_t region_bytes, int32_t* dev_err,
                    double timeout_s, void* stream) {
  const int N = c->world, r = c->rank;
  if (row_len <= 0 || row_len % 8) return set_err(FC2_ECONFIG, "row length must be a positive multiple of 8");
  std::vector<int64_t> mt((size_t)N * N);  // transposed: expert rank e returns token_matrix[s][e] rows to s
  for (int s = 0; s < N; ++s)
    for (int e = 0; e < N; ++e) mt[(size_t)e * N + s] = token_matrix[(size_t)s * N + e] * row_len;
  const bool fused = cfg->group_size % 32 == 0 && row_len % 32 == 0;
  int rc = a2a_core(c, cfg, y, y_dtype, mt.data(), nullptr, 0, 0, scratch, FC2_F32, false, region_off, region_bytes,
                    dev_err, timeout_s, stream, !fused);
  if (rc) return rc;
  if (fused) {  // read the returned blocks packed, straight from the region
    const void* pays[FC2_COMM_MAX];
    int64_t ns[FC2_COMM_MAX];
    int64_t yoff = 0;
    for (int s = 0; s < r; ++s) yoff += token_matrix[(size_t)s * N + r];
    for (int d = 0; d < N; ++d) {
      int64_t F = 0;
      const int64_t v = mt[(size_t)d * N + r];
      pays[d] = c->local + FC2_FLAG_BYTES + region_off + a2a_slot(cfg, mt.data(), N, r, d, &F);
      ns[d] = (v + cfg->group_size - 1) / cfg->group_size * cfg->group_size;
    }
    rc = fc2_moe_combine_q(cfg, N, r, pays, ns, (const uint8_t*)y + yoff * row_len * (y_dtype == FC2_BF16 ? 2 : 4),
                           y_dtype, pos_dev, tokens, row_len, out, out_dtype, dev_err, stream);
    if (rc) return rc;
    // everyone has consumed its region before anyone writes the next call's blocks
    return fc2_comm_barrier(c, dev_err, timeout_s, stream);
  }
  const void* srcs[FC2_COMM_MAX];
  int32_t dts[FC2_COMM_MAX], chk[FC2_COMM_MAX];
  int64_t off = 0, yoff = 0;
  for (int s = 0; s < r; ++s) yoff += token_matrix[(size_t)s * N + r];  // my own tokens' rows inside y
  for (int d = 0; d < N; ++d) {
    if (d == r) {
      srcs[d] = (const uint8_t*)y + yoff * row_len * (y_dtype == FC2_BF16 ? 2 : 4);
      dts[d] = y_dtype;
      chk[d] = 1;
    } else {
      srcs[d] = scratch + off * row_len;
      dts[d] = FC2_F32;
      chk[d] = 0;
    }
    off += token_matrix[(size_t)r * N + d];
  }
  return fc2_moe_combine_sum(N, srcs, dts, chk, pos_dev, tokens, row_len, out, out_dtype, dev_err, stream);
}

}  // extern "C"
