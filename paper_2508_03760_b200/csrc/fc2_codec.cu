// fc2_codec.cu -- host side of the C ABI for the codec hot path (kernels in
// fc2_kernels.cuh, instantiated per bit width in fc2_inst_b<B>.cu).
//
//   k_encode_grp    encode_chunk (codec.py:477-519) for bf16 input, G in
//                   {32,64,128,256}: lane-per-group warp tiles, payload words
//                   stored straight from registers (fc2_encode_group.cuh).
//   k_encode_fast   the same for f32 input: warp tile = 1024 elements.
//   k_encode_gen    the same contract for any G (multiple of 8) and f64 input,
//                   warp-per-group, exact float64.
//   k_decode_fast   decode_chunk (codec.py:522-563), G % 32 == 0: lane = 128
//                   elements, smem-staged coalesced stores.
//   k_decode_gen    elementwise decode for any G.
//   k_reduce_cta    two-step middle stage (collectives.py:291-311): decode N
//                   sources, fp32 rank-order accumulate, re-encode, push to up
//                   to 16 destinations; several shards per launch (one-shot).
//   k_reduce_fast / k_reduce_grp / k_reduce_gen   fallbacks (misaligned
//                   sources, > 16 sources, any G).
//   k_pack / k_unpack / bf16 casts / group and int-log helpers: codec.py:204-238,
//                   278-392, bfloat16.py:16-36.
// Host-resident chunks (fc2_*_host) are sliced and pipelined over internal
// streams (see host_pipeline below).
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <utility>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "fc2_kernels.cuh"

namespace fc2 {

// ---------------------------------------------------------------------------
// library state
// ---------------------------------------------------------------------------

thread_local std::string g_err;
static int64_t g_launches = 0;
static std::mutex g_mu;
constexpr int kMaxDev = 64;
static double* g_lut[kMaxDev] = {nullptr};   // per device: 255 thetas x 256 entries
static bool g_lut_ok[kMaxDev][256] = {{false}};

int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(FC2_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED);
  return FC2_OK;
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}


#define FC2_BSWITCH(EXPR)                                                   \
  switch (B) {                                                              \
    case 2: return EXPR(2); case 3: return EXPR(3); case 4: return EXPR(4);  \
    case 5: return EXPR(5); case 6: return EXPR(6); case 7: return EXPR(7);  \
    case 8: return EXPR(8);                                                 \
  }                                                                         \
  return set_err(FC2_ECONFIG, "bad bitwidth %d", B);

struct SumLoader {
  const ReduceArgs* a;
  DecCtx c;
  __device__ double operator()(int64_t i) const {
    float s = 0.0f;
    for (int k = 0; k < a->nsrc; ++k) s = __fadd_rn(s, decode_elem32(a->src[k], i, c));
    return (double)s;
  }
};

__global__ void __launch_bounds__(256) k_reduce_gen(const __grid_constant__ ReduceArgs a) {
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  SumLoader ld;
  ld.a = &a;
  ld.c.n = a.n; ld.c.meta_off = a.n * a.B / 8; ld.c.B = a.B; ld.c.G = a.G; ld.c.sr = a.sr;
  ld.c.intlog = a.intlog; ld.c.theta = a.theta; ld.c.lut = a.lut; ld.c.err = a.err;
  EncCtx cx;
  cx.n = a.n; cx.meta_off = a.n * a.B / 8; cx.intlog = a.intlog; cx.theta = a.theta; cx.lut = a.lut;
  cx.err = a.err;
  OutList o;
  o.nd = a.ndst < 8 ? a.ndst : 8;
  for (int d = 0; d < o.nd; ++d) o.p[d] = a.dst[d];
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < a.total; g += nw)
    generic_encode_group(ld, o, a.n, g, a.B, a.G, a.sr != 0, cx);
}

// ---------------------------------------------------------------------------
// pack / unpack (codec.py:204-238) and bf16 casts (bfloat16.py:16-31)
// ---------------------------------------------------------------------------

__global__ void k_pack(const int64_t* codes, int64_t n, int B, uint8_t* planes, int32_t* err) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // run of 8 codes
  if (r * 8 >= n) return;
  uint32_t c[8];
  bool bad = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int64_t v = codes[r * 8 + j];
    if (v < 0 || v >= (1ll << B)) bad = true;
    c[j] = (uint32_t)v;
  }
  if (bad) atomicOr(err, FC2_ERR_CODE_RANGE);
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u), O = unit_off(B, u);
    uint64_t bits = 0;
    for (int j = 0; j < 8; ++j) bits |= (uint64_t)((c[j] >> O) & ((1u << W) - 1u)) << (j * W);
    uint8_t* p = planes + (n * O) / 8 + r * W;
    for (int i = 0; i < W; ++i) p[i] = (uint8_t)(bits >> (8 * i));
  }
}

__global__ void k_unpack(const uint8_t* planes, int64_t n, int B, uint8_t* codes) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r * 8 >= n) return;
  uint32_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u), O = unit_off(B, u);
    const uint8_t* p = planes + (n * O) / 8 + r * W;
    uint64_t bits = 0;
    for (int i = 0; i < W; ++i) bits |= (uint64_t)p[i] << (8 * i);
    for (int j = 0; j < 8; ++j) c[j] |= (uint32_t)((bits >> (j * W)) & ((1u << W) - 1u)) << O;
  }
  for (int j = 0; j < 8; ++j) codes[r * 8 + j] = (uint8_t)c[j];
}

__global__ void k_f32_to_bf16(const float* x, int64_t n, uint16_t* y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (uint16_t)bf16_bits(x[i]);
}
__global__ void k_bf16_to_f32(const uint16_t* x, int64_t n, float* y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = bf16_val(x[i]);
}

// exact block copy with the collectives' float32 staging (collectives.py:160:
// every payload is cast to float32 first, then checked for non-finite values,
// :162-163) -- the All2All diagonal block (:466-468), which never crosses a wire
__device__ __forceinline__ float cc_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float cc_f32(float v) { return v; }
__device__ __forceinline__ float cc_f32(double v) { return __double2float_rn(v); }
__device__ __forceinline__ void cc_put(__nv_bfloat16* y, float v) { *y = __ushort_as_bfloat16((unsigned short)bf16_bits(v)); }
__device__ __forceinline__ void cc_put(float* y, float v) { *y = v; }
__device__ __forceinline__ void cc_put(double* y, float v) { *y = (double)v; }

template <typename TI, typename TO>
__global__ void k_copy_check(const TI* __restrict__ x, TO* __restrict__ y, int64_t n, int32_t* err) {
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = cc_f32(x[i]);
    bad |= !isfinite(v);
    cc_put(y + i, v);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, FC2_ERR_NONFINITE);
}

template <typename TI>
static int launch_copy_check(const void* x, void* y, int32_t y_dtype, int64_t n, int32_t* err, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  const TI* xi = (const TI*)x;
  if (y_dtype == FC2_BF16) k_copy_check<<<(unsigned)blocks, 256, 0, st>>>(xi, (__nv_bfloat16*)y, n, err);
  else if (y_dtype == FC2_F32) k_copy_check<<<(unsigned)blocks, 256, 0, st>>>(xi, (float*)y, n, err);
  else k_copy_check<<<(unsigned)blocks, 256, 0, st>>>(xi, (double*)y, n, err);
  return cuda_check("k_copy_check");
}

// ---------------------------------------------------------------------------
// per-group scalar API (codec.py:278-343) and int-log scales (codec.py:366-392)
// ---------------------------------------------------------------------------

// one warp: exact float64 group statistics + codes for an arbitrary-length group
__global__ void k_group_raw(const double* v, int64_t n, int B, int sr, uint8_t* codes, double* params,
                            int32_t* idx, int32_t* err) {
  const int lane = (int)lane_id();
  const int L = (1 << B) - 1;
  double mn1 = INFINITY, mn2 = INFINITY, mx1 = -INFINITY, mx2 = -INFINITY;
  int i1 = 1 << 30, j1 = 1 << 30;
  bool bad = false;
  for (int64_t e = lane; e < n; e += 32) {
    const double x = v[e];
    if (!isfinite(x)) bad = true;
    merge_min(mn1, i1, mn2, x, (int)e, INFINITY);
    merge_max(mx1, j1, mx2, x, (int)e, -INFINITY);
  }
  for (int o = 16; o >= 1; o >>= 1) {
    double a1 = __shfl_xor_sync(0xffffffffu, mn1, o), a2 = __shfl_xor_sync(0xffffffffu, mn2, o);
    int ai = __shfl_xor_sync(0xffffffffu, i1, o);
    double b1 = __shfl_xor_sync(0xffffffffu, mx1, o), b2 = __shfl_xor_sync(0xffffffffu, mx2, o);
    int bi = __shfl_xor_sync(0xffffffffu, j1, o);
    merge_min(mn1, i1, mn2, a1, ai, a2);
    merge_max(mx1, j1, mx2, b1, bi, b2);
  }
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0) atomicOr(err, FC2_ERR_NONFINITE);
    return;
  }
  double zero = mn1, vmax = mx1;
  int imin = 0, imax = 1;
  if (sr) {
    imin = i1; imax = j1;
    if (imin == imax) { imin = 0; imax = 1; }
    zero = mn2; vmax = mx2;  // shrunk range (codec.py:269-275)
  }
  const double scale = __ddiv_rn(__dsub_rn(vmax, zero), (double)L);
  for (int64_t e = lane; e < n; e += 32) {
    const double x = (sr && (e == imin || e == imax)) ? 0.0 : v[e];  // reserved slots quantized as 0.0
    codes[e] = (uint8_t)exact_code(x, zero, scale, L);
  }
  if (lane == 0) {
    params[0] = scale;
    params[1] = zero;
    if (sr) {
      params[2] = (double)bf16_val(bf16_bits(__double2float_rn(v[imin])));
      params[3] = (double)bf16_val(bf16_bits(__double2float_rn(v[imax])));
      idx[0] = imin;
      idx[1] = imax;
    }
  }
}

__global__ void k_group_decode_raw(const uint8_t* codes, int64_t n, double scale, double zero, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __dadd_rn(__dmul_rn((double)codes[i], scale), zero);  // codes * scale + zero (codec.py:295)
}

__global__ void k_scale_to_int(const double* s, int64_t n, int theta, int8_t* out, int32_t* err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = s[i];
    if (x < 0.0) atomicOr(err, FC2_ERR_NEGATIVE);
    int si = -128;
    if (x > 0.0) {
      const double t = __dmul_rn(log2(x), (double)theta);
      const double ft = fabs(t) - floor(fabs(t));
      if (fabs(ft - 0.5) < 1e-9) atomicOr(err, FC2_ERR_LOG2_TIE);
      double r = rha(t);
      r = r < -128.0 ? -128.0 : (r > 127.0 ? 127.0 : r);
      si = (int)r;
    }
    out[i] = (int8_t)si;
  }
}

__global__ void k_int_to_scale(const double* si, int64_t n, int theta, const double* lut, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = si[i];
    double r;
    if (v == -128.0) r = 0.0;
    else if (v == floor(v) && v >= -128.0 && v <= 127.0) r = lut[(int)v + 128];  // numpy's own values
    else r = exp2(__ddiv_rn(v, (double)theta));
    out[i] = r;
  }
}

static int enc_fast(int B, int dtype, bool sr, int G, const EncBatch& b, cudaStream_t st) {
#define E(BB) launch_enc_fast<BB>(dtype, sr, G, b, st)
  FC2_BSWITCH(E)
#undef E
}
static int red_fast(int B, bool sr, int G, const ReduceArgs& a, cudaStream_t st) {
#define E(BB) launch_red_fast<BB>(sr, G, a, st)
  FC2_BSWITCH(E)
#undef E
}
static int dec_fast(int B, int dtype, int64_t blocks, const DecBatch& b, cudaStream_t st) {
#define E(BB) launch_dec_fast<BB>(dtype, blocks, b, st)
  FC2_BSWITCH(E)
#undef E
}

static bool fast_group(int G) { return G == 32 || G == 64 || G == 128 || G == 256; }

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------

static int check_cfg(const fc2_config* c) {
  if (!c) return set_err(FC2_ECONFIG, "null config");
  if (c->bitwidth < 2 || c->bitwidth > 8) return set_err(FC2_ECONFIG, "bitwidth must be in [2, 8], got %d", c->bitwidth);
  if (c->group_size <= 0 || c->group_size % 8) return set_err(FC2_ECONFIG, "group_size must be a positive multiple of 8, got %d", c->group_size);
  if (c->scheme == 1 && (c->group_size < 4 || c->group_size > 256))
    return set_err(FC2_ECONFIG, "spike reserving needs 4 <= group_size <= 256, got %d", c->group_size);
  if (c->scheme != 0 && c->scheme != 1) return set_err(FC2_ECONFIG, "bad scheme %d", c->scheme);
  if (c->scale_encoding != 0 && c->scale_encoding != 1) return set_err(FC2_ECONFIG, "bad scale encoding %d", c->scale_encoding);
  if (c->theta < 1 || c->theta > 255) return set_err(FC2_ECONFIG, "theta must be in [1, 255], got %d", c->theta);
  return FC2_OK;
}

static const double* lut_for(const fc2_config* c, int* rc) {
  *rc = FC2_OK;
  if (c->scale_encoding != 1) return nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev || !g_lut[dev] || !g_lut_ok[dev][c->theta]) {
    *rc = set_err(FC2_ECONFIG, "INT_LOG table for theta=%d not loaded (call fc2_set_intlog_table)", c->theta);
    return nullptr;
  }
  return g_lut[dev] + (size_t)(c->theta - 1) * 256;
}

// for the other translation units (fc2_moe.cu)
const double* lut_for_cfg(const fc2_config* c, int* rc) { return lut_for(c, rc); }

static int64_t rec_nb(const fc2_config* c) { return rec_bytes(c->scheme == 1, c->scale_encoding == 1); }

}  // namespace fc2

using namespace fc2;

// ===========================================================================
// C ABI
// ===========================================================================

extern "C" {

int fc2_version(void) { return 1; }
const char* fc2_last_error(void) { return g_err.c_str(); }
int64_t fc2_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int fc2_check_config(const fc2_config* cfg) { return check_cfg(cfg); }

int fc2_footprint(const fc2_config* cfg, int64_t n, int64_t* nbytes) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (n < 0 || n % cfg->group_size) return set_err(FC2_ECONFIG, "element count %lld not a multiple of group_size %d", (long long)n, cfg->group_size);
  *nbytes = n * cfg->bitwidth / 8 + (n / cfg->group_size) * rec_nb(cfg);
  return FC2_OK;
}

int64_t fc2_plane_offset(const fc2_config* cfg, int64_t n, int32_t unit) {
  if (check_cfg(cfg) || unit < 0 || unit >= n_units(cfg->bitwidth)) return -1;
  return n * unit_off(cfg->bitwidth, unit) / 8;
}
int64_t fc2_meta_offset(const fc2_config* cfg, int64_t n) {
  if (check_cfg(cfg)) return -1;
  return n * cfg->bitwidth / 8;
}

int fc2_set_intlog_table(int32_t theta, const double* table256) {
  if (theta < 1 || theta > 255 || !table256) return set_err(FC2_ECONFIG, "bad theta/table");
  std::lock_guard<std::mutex> lk(g_mu);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) return set_err(FC2_ECUDA, "device %d out of range", dev);
  if (!g_lut[dev] && cudaMalloc(&g_lut[dev], sizeof(double) * 255 * 256) != cudaSuccess)
    return set_err(FC2_ECUDA, "cudaMalloc lut failed");
  if (cudaMemcpy(g_lut[dev] + (size_t)(theta - 1) * 256, table256, 256 * sizeof(double), cudaMemcpyHostToDevice) !=
      cudaSuccess)
    return set_err(FC2_ECUDA, "lut upload failed");
  g_lut_ok[dev][theta] = true;
  return FC2_OK;
}

}  // extern "C"

namespace fc2 {
// Encode tile granularity of a job (elements): the unit a sub-range launch
// must start on.  Fast bf16: one warp tile of 32 / LPG groups; fast f32: 1024;
// generic: one group.
static int64_t enc_unit(const fc2_config* cfg, int32_t x_dtype, const void* x, int64_t n_valid, int lpg) {
  const int G = cfg->group_size;
  const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15u) == 0 || n_valid == 0;
  if (!(fast_group(G) && x_dtype != FC2_F64 && aligned)) return G;
  return x_dtype == FC2_BF16 ? 32 / lpg * (int64_t)G : 1024;
}

// e_begin / e_end (nullable): encode only elements [e_begin, e_end) of each
// chunk (e_begin a multiple of enc_unit); the job's tile numbering is shifted
// with a negative t0 so the kernels see absolute tile indices.
static int encode_batch_impl(const fc2_config* cfg, int32_t x_dtype, int32_t njobs, const void* const* xs,
                             const int64_t* n_valid, const int64_t* n, void* const* payloads, int32_t* dev_err,
                             void* stream, const int64_t* e_begin, const int64_t* e_end,
                             const int32_t* const* rows = nullptr, int64_t row_len = 0) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (rows) {
    if (row_len <= 0 || row_len % 8 || row_len > INT32_MAX)
      return set_err(FC2_ECONFIG, "gathered rows need a row length that is a positive multiple of 8 (got %lld)",
                     (long long)row_len);
    for (int i = 0; i < njobs; ++i)
      if (n[i] > INT32_MAX) return set_err(FC2_ECONFIG, "gathered chunk of %lld elements is too long", (long long)n[i]);
  }
  if (njobs < 0 || njobs > FC2_MAX_JOBS) return set_err(FC2_ECONFIG, "njobs %d out of range", njobs);
  if ((e_begin || e_end) && njobs != 1) return set_err(FC2_ECONFIG, "sub-range encode takes one job");
  if (x_dtype < 0 || x_dtype > 2) return set_err(FC2_ECONFIG, "bad dtype %d", x_dtype);
  const double* lut = lut_for(cfg, &rc);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int B = cfg->bitwidth, G = cfg->group_size;
  const bool sr = cfg->scheme == 1;
  const int esz = x_dtype == FC2_BF16 ? 2 : (x_dtype == FC2_F32 ? 4 : 8);
  // shape of the bf16 lane-per-group encoder: bandwidth tiles, or one run
  // per lane when the whole launch is smaller than a wave of them
  int64_t elems = 0;
  for (int i = 0; i < njobs; ++i)
    elems += (e_end ? e_end[i] : n[i]) - (e_begin ? e_begin[i] : 0);
  const int lpg = elems < (int64_t)FC2_ENC_SMALL_TILES * (32 / enc_lpg(G)) * G ? enc_lpg_small(G) : enc_lpg(G);
  EncBatch fast, gen;
  for (EncBatch* b : {&fast, &gen}) {
    b->nj = 0; b->B = B; b->G = G; b->sr = sr; b->intlog = cfg->scale_encoding; b->theta = cfg->theta;
    b->lpg = lpg; b->row_len = (int)row_len; b->total = 0; b->lut = lut; b->err = dev_err;
  }
  auto launch_gen = [&]() -> int {
    int64_t blocks = (gen.total + 7) / 8;
    int64_t cap = (int64_t)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    if (x_dtype == FC2_BF16) k_encode_gen<__nv_bfloat16><<<(unsigned)blocks, 256, 0, st>>>(gen);
    else if (x_dtype == FC2_F32) k_encode_gen<float><<<(unsigned)blocks, 256, 0, st>>>(gen);
    else k_encode_gen<double><<<(unsigned)blocks, 256, 0, st>>>(gen);
    return cuda_check("k_encode_gen");
  };
  // one launch per FC2_KERNEL_JOBS jobs of a kind (small kernel parameters)
  auto flush = [&](EncBatch& b) -> int {
    if (!b.nj) return FC2_OK;
    const int r = &b == &fast ? enc_fast(B, x_dtype, sr, G, fast, st) : launch_gen();
    b.nj = 0;
    b.total = 0;
    return r;
  };
  for (int i = 0; i < njobs; ++i) {
    if (n[i] < 0 || n[i] % G) return set_err(FC2_ECONFIG, "chunk %lld not a multiple of group_size %d", (long long)n[i], G);
    if (n_valid[i] < 0 || n_valid[i] > n[i]) return set_err(FC2_EDATA, "n_valid %lld outside [0, %lld]", (long long)n_valid[i], (long long)n[i]);
    if (n[i] == 0) continue;
    if (reinterpret_cast<uintptr_t>(payloads[i]) & 3u) return set_err(FC2_ECONFIG, "payload must be 4-byte aligned");
    const bool aligned = (reinterpret_cast<uintptr_t>(xs[i]) & 15u) == 0 || n_valid[i] == 0;
    const bool use_fast = fast_group(G) && x_dtype != FC2_F64 && aligned;
    EncBatch* b = use_fast ? &fast : &gen;
    if (b->nj == FC2_KERNEL_JOBS && (rc = flush(*b))) return rc;
    EncJob& j = b->j[b->nj++];
    j.x = xs[i] ? xs[i] : payloads[i];
    j.out = (uint8_t*)payloads[i];
    j.rows = rows ? rows[i] : nullptr;
    j.n_valid = n_valid[i];
    j.n = n[i];
    // fast tiles: bf16 -> 32 / LPG groups per warp tile; f32 -> 1024 elements; generic: groups
    const int64_t tile = enc_unit(cfg, x_dtype, xs[i], n_valid[i], lpg);
    const int64_t eb = e_begin ? e_begin[i] : 0, ee = e_end ? e_end[i] : n[i];
    if (eb % tile || eb < 0 || ee > n[i] || ee < eb)
      return set_err(FC2_ECONFIG, "encode range [%lld, %lld) not on a %lld-element boundary", (long long)eb,
                     (long long)ee, (long long)tile);
    const int64_t first = eb / tile, last = (ee + tile - 1) / tile;
    if (last <= first) { b->nj--; continue; }
    j.t0 = b->total - first;
    b->total += last - first;
    (void)esz;
  }
  if ((rc = flush(fast))) return rc;
  return flush(gen);
}

}  // namespace fc2

extern "C" {

int fc2_encode_batch(const fc2_config* cfg, int32_t x_dtype, int32_t njobs, const void* const* xs,
                     const int64_t* n_valid, const int64_t* n, void* const* payloads, int32_t* dev_err,
                     void* stream) {
  return encode_batch_impl(cfg, x_dtype, njobs, xs, n_valid, n, payloads, dev_err, stream, nullptr, nullptr);
}

int fc2_encode_batch_rows(const fc2_config* cfg, int32_t x_dtype, int32_t njobs, const void* x,
                          const int32_t* const* rows, int64_t row_len, const int64_t* n_valid, const int64_t* n,
                          void* const* payloads, int32_t* dev_err, void* stream) {
  if (njobs < 0 || njobs > FC2_MAX_JOBS) return set_err(FC2_ECONFIG, "njobs %d out of range", njobs);
  std::vector<const void*> xs(njobs > 0 ? njobs : 1, x);
  return encode_batch_impl(cfg, x_dtype, njobs, xs.data(), n_valid, n, payloads, dev_err, stream, nullptr, nullptr,
                           rows, row_len);
}

int fc2_encode(const fc2_config* cfg, const void* x, int32_t x_dtype, int64_t n_valid, int64_t n, void* payload,
               int32_t* dev_err, void* stream) {
  return fc2_encode_batch(cfg, x_dtype, 1, &x, &n_valid, &n, &payload, dev_err, stream);
}

static int decode_batch_impl(const fc2_config* cfg, int32_t y_dtype, int32_t njobs, const void* const* payloads,
                             const int64_t* n, void* const* ys, const int64_t* n_out, int32_t* dev_err,
                             void* stream, int round_bf16, const int64_t* e_begin = nullptr,
                             const int64_t* e_end = nullptr);

int fc2_decode_batch(const fc2_config* cfg, int32_t y_dtype, int32_t njobs, const void* const* payloads,
                     const int64_t* n, void* const* ys, const int64_t* n_out, int32_t* dev_err, void* stream) {
  return decode_batch_impl(cfg, y_dtype, njobs, payloads, n, ys, n_out, dev_err, stream, 0);
}

static int decode_batch_impl(const fc2_config* cfg, int32_t y_dtype, int32_t njobs, const void* const* payloads,
                             const int64_t* n, void* const* ys, const int64_t* n_out, int32_t* dev_err,
                             void* stream, int round_bf16, const int64_t* e_begin, const int64_t* e_end) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (njobs < 0 || njobs > FC2_MAX_JOBS) return set_err(FC2_ECONFIG, "njobs %d out of range", njobs);
  if ((e_begin || e_end) && njobs != 1) return set_err(FC2_ECONFIG, "sub-range decode takes one job");
  if (y_dtype < 0 || y_dtype > 2) return set_err(FC2_ECONFIG, "bad dtype %d", y_dtype);
  const double* lut = lut_for(cfg, &rc);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int B = cfg->bitwidth, G = cfg->group_size;
  // fast decode: G % 32 == 0, bf16/f32 output, payloads 16-byte aligned
  bool fastG = y_dtype != FC2_F64 && G % 32 == 0;
  for (int i = 0; i < njobs; ++i) {
    if (reinterpret_cast<uintptr_t>(payloads[i]) & 15u) fastG = false;
    // the fast decoder cp.asyncs 16-byte chunks of every plane: each plane's
    // offset n * unit_off / 8 must be 16-byte aligned too (B = 3, 7 with
    // n % 64 != 0, e.g. G = 32 and an odd group count, is not)
    for (int u = 1; u < n_units(B); ++u)
      if ((n[i] * unit_off(B, u) / 8) & 15) fastG = false;
  }
  DecBatch b;
  b.round_bf16 = round_bf16;
  b.nj = 0; b.B = B; b.G = G; b.sr = cfg->scheme == 1; b.intlog = cfg->scale_encoding; b.theta = cfg->theta;
  b.total = 0; b.lut = lut; b.err = dev_err;
  // one launch per FC2_KERNEL_JOBS jobs (small kernel parameters)
  auto flush = [&]() -> int {
    if (!b.nj) return FC2_OK;
    int r;
    if (fastG) {
      r = dec_fast(B, y_dtype, 0, b, st);
    } else {
      int64_t blocks = (b.total + 255) / 256;
      int64_t cap = (int64_t)num_sms() * 16;
      if (blocks > cap) blocks = cap;
      if (y_dtype == FC2_BF16) k_decode_gen<__nv_bfloat16><<<(unsigned)blocks, 256, 0, st>>>(b);
      else if (y_dtype == FC2_F32) k_decode_gen<float><<<(unsigned)blocks, 256, 0, st>>>(b);
      else k_decode_gen<double><<<(unsigned)blocks, 256, 0, st>>>(b);
      r = cuda_check("k_decode_gen");
    }
    b.nj = 0;
    b.total = 0;
    return r;
  };
  for (int i = 0; i < njobs; ++i) {
    if (n[i] < 0 || n[i] % G) return set_err(FC2_ECONFIG, "chunk %lld not a multiple of group_size %d", (long long)n[i], G);
    if (n_out[i] < 0 || n_out[i] > n[i]) return set_err(FC2_ECONFIG, "n_out out of range");
    if (n[i] == 0 || n_out[i] == 0) continue;
    if (b.nj == FC2_KERNEL_JOBS && (rc = flush())) return rc;
    DecJob& j = b.j[b.nj++];
    j.pay = (const uint8_t*)payloads[i];
    j.y = ys[i];
    j.n = n[i];
    j.n_out = n_out[i];
    // sub-range [e_begin, e_end): fast tiles are 4096 elements, generic units one element
    const int64_t unit = fastG ? 4096 : 1;
    const int64_t eb = e_begin ? e_begin[i] : 0;
    const int64_t ee = e_end ? (e_end[i] < n_out[i] ? e_end[i] : n_out[i]) : n_out[i];
    if (eb % unit || eb < 0) return set_err(FC2_ECONFIG, "decode range start %lld not on a %lld-element boundary",
                                             (long long)eb, (long long)unit);
    const int64_t first = eb / unit, last = (ee + unit - 1) / unit;
    if (last <= first) { b.nj--; continue; }
    j.t0 = b.total - first;
    b.total += last - first;
  }
  return flush();
}

int fc2_decode(const fc2_config* cfg, const void* payload, int64_t n, void* y, int32_t y_dtype, int64_t n_out,
               int32_t* dev_err, void* stream) {
  return fc2_decode_batch(cfg, y_dtype, 1, &payload, &n, &y, &n_out, dev_err, stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// host-buffer pipeline: encode_chunk / decode_chunk / their round trip with
// the chunk in host memory.  The chunk is cut into slices on tile boundaries;
// slice k goes
//   H2D(x slice) -> encode(slice) [-> decode(slice)] -> D2H(plane + meta
//   segments of the slice) [+ D2H(y slice)]
//   (decode only: H2D(payload segments) -> decode(slice) -> D2H(y slice))
// with all uploads on one stream, all downloads on another and the kernels on
// two more, joined by per-slice events, so PCIe traffic in both directions
// overlaps the kernels and each other.
// Stream-ordered with respect to the caller's stream (event fork / join).
// ---------------------------------------------------------------------------

namespace fc2 {

#ifndef FC2_PIPE_STREAMS
#define FC2_PIPE_STREAMS 4
#endif
constexpr int kPipeStreams = FC2_PIPE_STREAMS;  // s[0]: uploads; s[1]: downloads; s[2..]: kernels
static_assert(kPipeStreams >= 3, "host pipeline needs an upload, a download and a kernel stream");
constexpr int kPipeEvents = 8;
#ifndef FC2_PIPE_PAYLOAD_LAST
#define FC2_PIPE_PAYLOAD_LAST 1
#endif
#ifndef FC2_PIPE_TRACE
#define FC2_PIPE_TRACE 0  // dev builds: print a timing-event timeline of every host pipeline call
#endif
struct PipeTrace {
  std::vector<std::pair<cudaEvent_t, std::string>> ev;
  std::vector<double> host_us;
  void mark(cudaStream_t s, const char* what, int64_t k) {
    if (!FC2_PIPE_TRACE) return;
    host_us.push_back(std::chrono::duration<double, std::micro>(
        std::chrono::steady_clock::now().time_since_epoch()).count());
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.emplace_back(e, std::string(what) + " " + std::to_string(k));
  }
  void dump(cudaStream_t st) {
    if (!FC2_PIPE_TRACE || ev.empty()) return;
    cudaStreamSynchronize(st);
    for (size_t i = 0; i < ev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[0].first, ev[i].first);
      fprintf(stderr, "[pipe] gpu %8.1f us  host %8.1f us  %s\n", ms * 1e3f, host_us[i] - host_us[0],
              ev[i].second.c_str());
    }
    for (auto& x : ev) cudaEventDestroy(x.first);
  }
};
struct HostPipe {
  cudaStream_t s[kPipeStreams];
  cudaEvent_t fork, join[kPipeStreams], up[kPipeEvents], dn[kPipeEvents];
};

static HostPipe* host_pipe(int* rc) {
  static HostPipe pipes[64];
  static bool made[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) { *rc = set_err(FC2_ECUDA, "device %d out of range", dev); return nullptr; }
  std::lock_guard<std::mutex> lk(g_mu);
  if (!made[dev]) {
    HostPipe& p = pipes[dev];
    for (int i = 0; i < kPipeStreams; ++i) {
      if (cudaStreamCreateWithFlags(&p.s[i], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&p.join[i], cudaEventDisableTiming) != cudaSuccess) {
        *rc = set_err(FC2_ECUDA, "host pipeline stream/event creation failed");
        return nullptr;
      }
    }
    bool ok = cudaEventCreateWithFlags(&p.fork, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < kPipeEvents; ++i)
      ok = ok && cudaEventCreateWithFlags(&p.up[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&p.dn[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
      *rc = set_err(FC2_ECUDA, "host pipeline event creation failed");
      return nullptr;
    }
    made[dev] = true;
  }
  *rc = FC2_OK;
  return &pipes[dev];
}

static int esize(int32_t dt) { return dt == FC2_BF16 ? 2 : (dt == FC2_F32 ? 4 : (dt == FC2_F64 ? 8 : 0)); }

// copy the payload bytes of elements [e0, e1) (one segment per plane + the
// metadata segment) between host and device
static int copy_payload_slice(const fc2_config* cfg, int64_t n, int64_t e0, int64_t e1, void* dev, void* host,
                              cudaMemcpyKind kind, cudaStream_t st) {
  const int B = cfg->bitwidth, G = cfg->group_size;
  for (int u = 0; u < n_units(B); ++u) {
    const int W = unit_w(B, u);
    const int64_t off = n * unit_off(B, u) / 8 + e0 * W / 8, len = (e1 - e0) * W / 8;
    uint8_t* d = (uint8_t*)dev + off;
    uint8_t* h = (uint8_t*)host + off;
    if (cudaMemcpyAsync(kind == cudaMemcpyHostToDevice ? (void*)d : (void*)h,
                        kind == cudaMemcpyHostToDevice ? (const void*)h : (const void*)d, len, kind, st) != cudaSuccess)
      return set_err(FC2_ECUDA, "payload plane copy failed");
  }
  const int64_t rb = rec_nb(cfg), off = n * B / 8 + e0 / G * rb, len = (e1 - e0) / G * rb;
  uint8_t* d = (uint8_t*)dev + off;
  uint8_t* h = (uint8_t*)host + off;
  if (cudaMemcpyAsync(kind == cudaMemcpyHostToDevice ? (void*)d : (void*)h,
                      kind == cudaMemcpyHostToDevice ? (const void*)h : (const void*)d, len, kind, st) != cudaSuccess)
    return set_err(FC2_ECUDA, "payload meta copy failed");
  return FC2_OK;
}

// mode bit 1: x_host -> encode; 2: payload -> payload_host; 4: payload_host -> device;
// 8: decode -> y_host
static int host_pipeline(int mode, const fc2_config* cfg, const void* x_host, int32_t x_dtype, int64_t n,
                         void* x_dev, void* pay_dev, void* y_dev, int32_t y_dtype, void* pay_host, void* y_host,
                         int64_t slice, int32_t* dev_err, void* stream) {
  int rc = check_cfg(cfg);
  if (rc) return rc;
  const int G = cfg->group_size;
  if (n < 0 || n % G) return set_err(FC2_ECONFIG, "chunk %lld not a multiple of group_size %d", (long long)n, G);
  if (n == 0) return FC2_OK;
  if ((mode & 1) && (!x_host || !x_dev || !esize(x_dtype))) return set_err(FC2_ECONFIG, "encode needs x buffers");
  if ((mode & 8) && (!y_host || !y_dev || !esize(y_dtype))) return set_err(FC2_ECONFIG, "decode needs y buffers");
  if ((mode & 6) && !pay_host) return set_err(FC2_ECONFIG, "payload host buffer missing");
  if (!pay_dev) return set_err(FC2_ECONFIG, "payload device buffer missing");
  // slice: a multiple of every tile unit (encode <= 8192 elements or one
  // group; decode 4096) and of the group size
  int64_t unit = 32768;
  while (unit % G) unit += 32768;
  if (slice <= 0) slice = (int64_t)1 << 22;
  slice = (slice + unit - 1) / unit * unit;
  HostPipe* hp = host_pipe(&rc);
  if (rc) return rc;
  NoPdl no_pdl;  // kernels here follow cross-stream event waits
  // the per-device pipeline streams and events are shared: one host thread
  // enqueues a pipeline at a time (the enqueue is short; the work stays async)
  static std::mutex pipe_mu;
  std::lock_guard<std::mutex> pipe_lk(pipe_mu);
  cudaStream_t st = (cudaStream_t)stream;
  PipeTrace tr;
  tr.mark(st, "fork", 0);
  if (cudaEventRecord(hp->fork, st) != cudaSuccess) return set_err(FC2_ECUDA, "fork event failed");
  for (int i = 0; i < kPipeStreams; ++i) cudaStreamWaitEvent(hp->s[i], hp->fork, 0);
  const int xs = esize(x_dtype), ys = esize(y_dtype);
  // s[0]: uploads, back to back; s[1]: downloads, in slice order; slice k's
  // kernels on s[2 + k % 2] between its upload event and its download event.
  // One stream per copy direction keeps each direction on its own copy engine.
  cudaStream_t up = hp->s[0], down = hp->s[1];
  int64_t k = 0;
  for (int64_t e0 = 0; e0 < n; e0 += slice, ++k) {
    const int64_t e1 = e0 + slice < n ? e0 + slice : n;
    cudaStream_t s = hp->s[2 + k % (kPipeStreams - 2)];
    if (mode & 5) {
      if (mode & 1) {
        if (cudaMemcpyAsync((uint8_t*)x_dev + e0 * xs, (const uint8_t*)x_host + e0 * xs, (e1 - e0) * xs,
                            cudaMemcpyHostToDevice, up) != cudaSuccess)
          return set_err(FC2_ECUDA, "x slice copy failed");
      } else {
        rc = copy_payload_slice(cfg, n, e0, e1, pay_dev, pay_host, cudaMemcpyHostToDevice, up);
        if (rc) return rc;
      }
      tr.mark(up, "up_done", k);
      cudaEvent_t ev = hp->up[k % kPipeEvents];
      if (cudaEventRecord(ev, up) != cudaSuccess || cudaStreamWaitEvent(s, ev, 0) != cudaSuccess)
        return set_err(FC2_ECUDA, "upload event failed");
    }
    tr.mark(s, "kern_start", k);
    if (mode & 1) {
      rc = encode_batch_impl(cfg, x_dtype, 1, &x_dev, &n, &n, &pay_dev, dev_err, s, &e0, &e1);
      if (rc) return rc;
      tr.mark(s, "enc_done", k);
    }
    if (mode & 8) {
      const void* pd = pay_dev;
      rc = decode_batch_impl(cfg, y_dtype, 1, &pd, &n, &y_dev, &n, dev_err, s, 0, &e0, &e1);
      if (rc) return rc;
    }
    if (mode & 10) {
      tr.mark(s, "kern_done", k);
      cudaEvent_t ev = hp->dn[k % kPipeEvents];
      if (cudaEventRecord(ev, s) != cudaSuccess || cudaStreamWaitEvent(down, ev, 0) != cudaSuccess)
        return set_err(FC2_ECUDA, "download event failed");
      if ((mode & 2) && !(FC2_PIPE_PAYLOAD_LAST && (mode & 8))) {
        rc = copy_payload_slice(cfg, n, e0, e1, pay_dev, pay_host, cudaMemcpyDeviceToHost, down);
        if (rc) return rc;
      }
      if ((mode & 8) && cudaMemcpyAsync((uint8_t*)y_host + e0 * ys, (const uint8_t*)y_dev + e0 * ys,
                                        (e1 - e0) * ys, cudaMemcpyDeviceToHost, down) != cudaSuccess)
        return set_err(FC2_ECUDA, "y slice copy failed");
      tr.mark(down, "down_done", k);
    }
  }
  // round trip: the payload comes back in one copy per plane + one for the
  // metadata after the last slice (fewer, larger DMA transfers)
  if (FC2_PIPE_PAYLOAD_LAST && (mode & 2) && (mode & 8)) {
    rc = copy_payload_slice(cfg, n, 0, n, pay_dev, pay_host, cudaMemcpyDeviceToHost, down);
    if (rc) return rc;
    tr.mark(down, "payload_done", 0);
  }
  for (int i = 0; i < kPipeStreams; ++i) {
    cudaEventRecord(hp->join[i], hp->s[i]);
    cudaStreamWaitEvent(st, hp->join[i], 0);
  }
  tr.mark(st, "join", 0);
  tr.dump(st);
  return cuda_check("host pipeline");
}

}  // namespace fc2

extern "C" {

int fc2_encode_host(const fc2_config* cfg, const void* x_host, int32_t x_dtype, int64_t n, void* x_dev,
                    void* payload_dev, void* payload_host, int64_t slice, int32_t* dev_err, void* stream) {
  return host_pipeline(1 | 2, cfg, x_host, x_dtype, n, x_dev, payload_dev, nullptr, 0, payload_host, nullptr, slice,
                       dev_err, stream);
}

int fc2_decode_host(const fc2_config* cfg, const void* payload_host, int64_t n, void* payload_dev, void* y_dev,
                    int32_t y_dtype, void* y_host, int64_t slice, int32_t* dev_err, void* stream) {
  return host_pipeline(4 | 8, cfg, nullptr, 0, n, nullptr, payload_dev, y_dev, y_dtype,
                       const_cast<void*>(payload_host), y_host, slice, dev_err, stream);
}

int fc2_roundtrip_host(const fc2_config* cfg, const void* x_host, int32_t x_dtype, int64_t n, void* x_dev,
                       void* payload_dev, void* y_dev, int32_t y_dtype, void* payload_host, void* y_host,
                       int64_t slice, int32_t* dev_err, void* stream) {
  return host_pipeline(1 | (payload_host ? 2 : 0) | 8, cfg, x_host, x_dtype, n, x_dev, payload_dev, y_dev, y_dtype,
                       payload_host, y_host, slice, dev_err, stream);
}

int fc2_gather_decode(const fc2_config* cfg, int32_t nshards, const void* const* shard_payloads, int64_t shard_len,
                      void* y, int32_t y_dtype, int64_t n_out, int32_t* dev_err, void* stream) {
  if (nshards < 0 || nshards > FC2_MAX_JOBS) return set_err(FC2_ECONFIG, "nshards out of range");
  const int esz = y_dtype == FC2_BF16 ? 2 : (y_dtype == FC2_F32 ? 4 : 8);
  int64_t ns[FC2_MAX_JOBS], no[FC2_MAX_JOBS];
  void* ys[FC2_MAX_JOBS];
  for (int i = 0; i < nshards; ++i) {
    ns[i] = shard_len;
    int64_t rem = n_out - (int64_t)i * shard_len;
    no[i] = rem < 0 ? 0 : (rem > shard_len ? shard_len : rem);
    ys[i] = (uint8_t*)y + (size_t)i * shard_len * esz;
  }
  return decode_batch_impl(cfg, y_dtype, nshards, shard_payloads, ns, ys, no, dev_err, stream, 1);
}

int fc2_reduce_requant(const fc2_config* cfg, int32_t nsrc, const void* const* src_payloads, int64_t n, int32_t ndst,
                       void* const* dst_payloads, int32_t* dev_err, void* stream) {
  return fc2_reduce_requant_batch(cfg, nsrc, src_payloads, n, 1, 0, ndst, dst_payloads, 0, dev_err, stream);
}

int fc2_reduce_requant_batch(const fc2_config* cfg, int32_t nsrc, const void* const* src_payloads, int64_t n,
                             int32_t nshard, int64_t src_stride, int32_t ndst, void* const* dst_payloads,
                             int64_t dst_stride, int32_t* dev_err, void* stream) {
  int rc = check_cfg(cfg);
  if (nshard < 1) return set_err(FC2_ECONFIG, "nshard must be >= 1");
  if (rc) return rc;
  if (nsrc < 1 || nsrc > FC2_MAX_PEERS || ndst < 1 || ndst > FC2_MAX_PEERS)
    return set_err(FC2_ECONFIG, "nsrc/ndst out of range");
  if (n < 0 || n % cfg->group_size) return set_err(FC2_ECONFIG, "shard not a multiple of group_size");
  if (n == 0) return FC2_OK;
  const double* lut = lut_for(cfg, &rc);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  ReduceArgs a;
  a.nsrc = nsrc; a.ndst = ndst; a.B = cfg->bitwidth; a.G = cfg->group_size; a.sr = cfg->scheme == 1;
  a.intlog = cfg->scale_encoding; a.theta = cfg->theta; a.n = n; a.lut = lut; a.err = dev_err;
  a.nshard = nshard; a.sstride = src_stride; a.dstride = dst_stride;
  for (int i = 0; i < nsrc; ++i) a.src[i] = (const uint8_t*)src_payloads[i];
  for (int i = 0; i < ndst; ++i) a.dst[i] = (uint8_t*)dst_payloads[i];
  if (fast_group(a.G)) {
    a.total = (n + 1023) / 1024;
    return red_fast(a.B, a.sr != 0, a.G, a, st);
  }
  if (ndst > 8) return set_err(FC2_ECONFIG, "generic reduce supports <= 8 destinations");
  if (nshard > 1) {  // the generic reducer takes one shard per launch
    std::vector<const void*> s1(nsrc);
    std::vector<void*> d1(ndst);
    for (int64_t k = 0; k < nshard; ++k) {
      for (int i = 0; i < nsrc; ++i) s1[i] = (const uint8_t*)src_payloads[i] + k * src_stride;
      for (int i = 0; i < ndst; ++i) d1[i] = (uint8_t*)dst_payloads[i] + k * dst_stride;
      rc = fc2_reduce_requant_batch(cfg, nsrc, s1.data(), n, 1, 0, ndst, d1.data(), 0, dev_err, stream);
      if (rc) return rc;
    }
    return FC2_OK;
  }
  a.total = n / a.G;
  int64_t blocks = (a.total + 7) / 8;
  int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  k_reduce_gen<<<(unsigned)blocks, 256, 0, st>>>(a);
  return cuda_check("k_reduce_gen");
}

int fc2_pack_codes(const int64_t* codes, int64_t n, int32_t bitwidth, uint8_t* planes, int32_t* dev_err,
                   void* stream) {
  if (bitwidth < 2 || bitwidth > 8) return set_err(FC2_ECONFIG, "bitwidth must be in [2, 8], got %d", bitwidth);
  if (n < 0 || n % 8) return set_err(FC2_EDATA, "code count %lld must be a multiple of 8", (long long)n);
  if (n == 0) return FC2_OK;
  int64_t runs = n / 8;
  k_pack<<<(unsigned)((runs + 255) / 256), 256, 0, (cudaStream_t)stream>>>(codes, n, bitwidth, planes, dev_err);
  return cuda_check("k_pack");
}

int fc2_unpack_codes(const uint8_t* planes, int64_t n, int32_t bitwidth, uint8_t* codes, void* stream) {
  if (bitwidth < 2 || bitwidth > 8) return set_err(FC2_ECONFIG, "bitwidth must be in [2, 8], got %d", bitwidth);
  if (n < 0 || n % 8) return set_err(FC2_EDATA, "code count must be a multiple of 8");
  if (n == 0) return FC2_OK;
  int64_t runs = n / 8;
  k_unpack<<<(unsigned)((runs + 255) / 256), 256, 0, (cudaStream_t)stream>>>(planes, n, bitwidth, codes);
  return cuda_check("k_unpack");
}

int fc2_f32_to_bf16_bits(const float* x, int64_t n, uint16_t* out, void* stream) {
  if (n <= 0) return FC2_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  k_f32_to_bf16<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, n, out);
  return cuda_check("k_f32_to_bf16");
}

int fc2_copy_check(const void* x, int32_t x_dtype, void* y, int32_t y_dtype, int64_t n, int32_t* dev_err,
                   void* stream) {
  if (x_dtype < 0 || x_dtype > 2 || y_dtype < 0 || y_dtype > 2) return set_err(FC2_ECONFIG, "bad dtype");
  if (n <= 0) return FC2_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (x_dtype == FC2_BF16) return launch_copy_check<__nv_bfloat16>(x, y, y_dtype, n, dev_err, st);
  if (x_dtype == FC2_F32) return launch_copy_check<float>(x, y, y_dtype, n, dev_err, st);
  return launch_copy_check<double>(x, y, y_dtype, n, dev_err, st);
}

int fc2_bf16_bits_to_f32(const uint16_t* x, int64_t n, float* out, void* stream) {
  if (n <= 0) return FC2_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  k_bf16_to_f32<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, n, out);
  return cuda_check("k_bf16_to_f32");
}

int fc2_group_encode_raw(const double* v, int64_t n, int32_t bitwidth, int32_t sr, uint8_t* codes, double* params,
                         int32_t* idx, int32_t* dev_err, void* stream) {
  if (bitwidth < 2 || bitwidth > 8) return set_err(FC2_ECONFIG, "bitwidth must be in [2, 8], got %d", bitwidth);
  if (n < 1 || n > (1 << 30)) return set_err(FC2_EDATA, "group must be a non-empty one-dimensional vector");
  if (sr && n < 4) return set_err(FC2_ECONFIG, "spike reserving needs at least 4 elements, got %lld", (long long)n);
  k_group_raw<<<1, 32, 0, (cudaStream_t)stream>>>(v, n, bitwidth, sr, codes, params, idx, dev_err);
  return cuda_check("k_group_raw");
}

int fc2_group_decode_raw(const uint8_t* codes, int64_t n, double scale, double zero, double* out, void* stream) {
  if (n <= 0) return FC2_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  k_group_decode_raw<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(codes, n, scale, zero, out);
  return cuda_check("k_group_decode_raw");
}

int fc2_scale_to_int(const double* s, int64_t n, int32_t theta, int8_t* out, int32_t* dev_err, void* stream) {
  if (theta < 1 || theta > 255) return set_err(FC2_ECONFIG, "theta must be in [1, 255], got %d", theta);
  if (n <= 0) return FC2_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  k_scale_to_int<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(s, n, theta, out, dev_err);
  return cuda_check("k_scale_to_int");
}

int fc2_int_to_scale(const double* si, int64_t n, int32_t theta, double* out, void* stream) {
  fc2_config c = {4, 32, 0, 1, theta};
  int rc = FC2_OK;
  const double* lut = lut_for(&c, &rc);
  if (rc) return rc;
  if (n <= 0) return FC2_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  k_int_to_scale<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(si, n, theta, lut, out);
  return cuda_check("k_int_to_scale");
}

}  // extern "C"

namespace fc2 {
// batched decode whose float32 output is snapped to the bf16 grid (the
// AllReduce output, collectives.py:185-186, 313-314), for fc2_comm.cu
int decode_batch_grid(const fc2_config* cfg, int32_t y_dtype, int32_t njobs, const void* const* payloads,
                      const int64_t* n, void* const* ys, const int64_t* n_out, int32_t* dev_err, void* stream) {
  return decode_batch_impl(cfg, y_dtype, njobs, payloads, n, ys, n_out, dev_err, stream, 1);
}
}  // namespace fc2
