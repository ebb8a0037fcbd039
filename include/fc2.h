/*
 * fc2.h -- C ABI of the B200-native FlashCommunication-V2 hot path.
 *
 * Plain C: pointers, sizes and int status codes; no torch / C++ types.  All
 * compute entry points are asynchronous on the caller's CUDA stream (passed
 * as `void* stream`, a cudaStream_t), never allocate, never synchronize, and
 * report data-dependent errors through a caller-owned device int32 word
 * (`dev_err`, bit mask FC2_ERR_*) that the host checks when it wants to.
 *
 * Threading: the codec entry points may be called from several host threads
 * (the host-resident pipelines serialize their enqueues internally).  A
 * communicator (fc2_comm) is driven by one host thread, and every rank must
 * issue the same sequence of collective calls on it (ranks synchronize through
 * flags in each other's buffers).
 *
 * Each entry point names the reference interface it replaces (paths relative
 * to /root/reference/pkg/src/qcomm).  The reference is a pure Python+numpy
 * package with no FFI; the binding a maintainer would add is the ctypes stub
 * in INTEGRATION.md, which is exactly what paper_2508_03760_b200/_lib.py does.
 */
#ifndef FC2_H
#define FC2_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map onto errors.py:4-21) ---------------------------- */
#define FC2_OK              0
#define FC2_ECONFIG        -1  /* ConfigError      */
#define FC2_EDATA          -2  /* DataError        */
#define FC2_EFORMAT        -3  /* DecodeFormatError */
#define FC2_ENOTAPPLICABLE -4  /* NotApplicableError */
#define FC2_ECUDA          -5  /* CUDA runtime failure (fc2_last_error has text) */

/* ---- device error word bits (dev_err) ---------------------------------- */
#define FC2_ERR_NONFINITE   1  /* encode saw NaN/inf    -> DataError (codec.py:482-483) */
#define FC2_ERR_SPIKE_INDEX 2  /* decode spike index out of range -> DecodeFormatError (codec.py:555-558) */
#define FC2_ERR_LOG2_TIE    4  /* INT_LOG: log2(scale)*theta within 1e-9 of a .5 tie (parity warning) */
#define FC2_ERR_TIMEOUT     8  /* cross-rank flag wait timed out */
#define FC2_ERR_CODE_RANGE 16  /* pack: code outside [0, 2^bits) -> CodeRangeError (codec.py:216-217) */
#define FC2_ERR_NEGATIVE   32  /* scale_to_int: negative scale -> DataError (codec.py:373-374) */
#define FC2_ERR_EXPERT_RANGE 64 /* MoE routing: expert id outside [0, n_experts) -> ConfigError */

/* ---- element types ----------------------------------------------------- */
#define FC2_BF16 0
#define FC2_F32  1
#define FC2_F64  2

/* QuantConfig (codec.py:55-90).  scheme: 0 RTN, 1 SPIKE_RESERVING.
 * scale_encoding: 0 BF16, 1 INT_LOG.  chunk_size is a host-side notion: every
 * call below passes the chunk length `n` explicitly. */
typedef struct fc2_config {
    int32_t bitwidth;
    int32_t group_size;
    int32_t scheme;
    int32_t scale_encoding;
    int32_t theta;
} fc2_config;

/* Validate a config (codec.py:71-86).  Returns FC2_OK or FC2_ECONFIG. */
int fc2_check_config(const fc2_config* cfg);

/* Payload bytes for n elements: planes + metadata (codec.py:428-432). */
int fc2_footprint(const fc2_config* cfg, int64_t n, int64_t* nbytes);

/* Byte offset of bit-split plane u / of the metadata section inside one
 * chunk payload of n elements (R9-R11; codec.py:129,518). */
int64_t fc2_plane_offset(const fc2_config* cfg, int64_t n, int32_t unit);
int64_t fc2_meta_offset(const fc2_config* cfg, int64_t n);

/* Must be called once per process before INT_LOG work: the 256-entry table
 * exp2(si/theta), si = -128..127, computed on the host by numpy so the
 * device scale values are bit-identical to codec.py:468,542. */
int fc2_set_intlog_table(int32_t theta, const double* table256);

/* encode_chunk (codec.py:477-519) on device memory.
 * x: n_valid elements of x_dtype; elements [n_valid, n) are encoded as +0.0
 * (the zero padding of collectives.py:167-172).  n % group_size == 0.
 * payload: fc2_footprint(n) bytes, 4-byte aligned (16 for full speed). */
int fc2_encode(const fc2_config* cfg, const void* x, int32_t x_dtype, int64_t n_valid,
               int64_t n, void* payload, int32_t* dev_err, void* stream);

/* Batched encode: njobs independent chunks in one launch (the per-(src,shard)
 * loop of collectives.py:280-290 and the per-block loop of :462-480).
 * Host arrays of length njobs; njobs <= FC2_MAX_JOBS. */
#define FC2_MAX_JOBS 256
int fc2_encode_batch(const fc2_config* cfg, int32_t x_dtype, int32_t njobs,
                     const void* const* xs, const int64_t* n_valid, const int64_t* n,
                     void* const* payloads, int32_t* dev_err, void* stream);

/* Batched encode with the token-row gather fused in (MoE dispatch): chunk i
 * is the rows rows[i][0..n_valid[i] / row_len) of x (row_len elements each,
 * row_len % 8 == 0), i.e. element e is x[rows[i][e / row_len] * row_len +
 * e % row_len]; the encoders read the rows directly, nothing is gathered
 * into HBM first.  Same payload bytes as fc2_encode_batch on the gathered
 * block (collectives.py:462-480 on the block of routed tokens). */
int fc2_encode_batch_rows(const fc2_config* cfg, int32_t x_dtype, int32_t njobs, const void* x,
                          const int32_t* const* rows, int64_t row_len, const int64_t* n_valid, const int64_t* n,
                          void* const* payloads, int32_t* dev_err, void* stream);

/* decode_chunk (codec.py:522-563): payload of n elements -> y (y_dtype).
 * Only the first n_out <= n values are written (padding strip,
 * collectives.py:185-186, :480).  FC2_F64 output is bit-identical to the
 * reference's float64 result; FC2_F32 to its .astype(float32)
 * (collectives.py:182); FC2_BF16 to bf16_round of that (:185-186). */
int fc2_decode(const fc2_config* cfg, const void* payload, int64_t n, void* y,
               int32_t y_dtype, int64_t n_out, int32_t* dev_err, void* stream);

int fc2_decode_batch(const fc2_config* cfg, int32_t y_dtype, int32_t njobs,
                     const void* const* payloads, const int64_t* n, void* const* ys,
                     const int64_t* n_out, int32_t* dev_err, void* stream);

/* Two-step AllReduce middle stage (collectives.py:291-311): decode nsrc
 * payloads of the same shard (n elements each), accumulate in fp32 in source
 * order from +0.0, re-encode the sum, and store the packed result to every
 * one of ndst destinations (local buffer and/or peer pointers). */
int fc2_reduce_requant(const fc2_config* cfg, int32_t nsrc, const void* const* src_payloads,
                       int64_t n, int32_t ndst, void* const* dst_payloads, int32_t* dev_err,
                       void* stream);

/* The same for nshard independent shards in one launch: shard k's sources are
 * src_payloads[s] + k * src_stride and its destinations dst_payloads[d] +
 * k * dst_stride (the one-shot AllReduce reduces every shard on every rank). */
int fc2_reduce_requant_batch(const fc2_config* cfg, int32_t nsrc, const void* const* src_payloads,
                             int64_t n, int32_t nshard, int64_t src_stride, int32_t ndst,
                             void* const* dst_payloads, int64_t dst_stride, int32_t* dev_err,
                             void* stream);

/* Decode the N gathered shard payloads of a two-step AllReduce straight into
 * the bf16/f32 output on the bf16 grid, stripping padding (collectives.py:313-314,
 * 185-186). */
int fc2_gather_decode(const fc2_config* cfg, int32_t nshards, const void* const* shard_payloads,
                      int64_t shard_len, void* y, int32_t y_dtype, int64_t n_out,
                      int32_t* dev_err, void* stream);

/* Host-resident chunks (the reference's encode_chunk / decode_chunk take and
 * return host arrays and bytes: codec.py:477-519, 522-563).  The chunk of n
 * elements lives in host memory (pin it for overlap); the caller supplies the
 * device staging buffers (x_dev: n elements, payload_dev: fc2_footprint(n)
 * bytes, y_dev: n elements) so nothing is allocated per call.  The chunk is
 * processed in slices of `slice` elements (rounded up to a multiple of 32768
 * and of group_size; <= 0: 4 Mi) on internal streams so host<->device copies
 * in both directions overlap the kernels; stream-ordered with respect to
 * `stream`.  payload_host holds the exact payload bytes (planes, then
 * metadata; R9-R11).  Round trip = encode then decode of the same chunk, the
 * QDQ of collectives.py:179-182 (_encode_once); payload_host may be NULL
 * there when only the decoded values are wanted. */
int fc2_encode_host(const fc2_config* cfg, const void* x_host, int32_t x_dtype, int64_t n,
                    void* x_dev, void* payload_dev, void* payload_host, int64_t slice,
                    int32_t* dev_err, void* stream);
int fc2_decode_host(const fc2_config* cfg, const void* payload_host, int64_t n, void* payload_dev,
                    void* y_dev, int32_t y_dtype, void* y_host, int64_t slice, int32_t* dev_err,
                    void* stream);
int fc2_roundtrip_host(const fc2_config* cfg, const void* x_host, int32_t x_dtype, int64_t n,
                       void* x_dev, void* payload_dev, void* y_dev, int32_t y_dtype,
                       void* payload_host, void* y_host, int64_t slice, int32_t* dev_err,
                       void* stream);

/* pack_codes / unpack_codes (codec.py:204-238): codes are int64 (range
 * checked on device, FC2_ERR_CODE_RANGE), n % 8 == 0; planes is one
 * contiguous buffer (plane 0, plane 1, ...). */
int fc2_pack_codes(const int64_t* codes, int64_t n, int32_t bitwidth, uint8_t* planes,
                   int32_t* dev_err, void* stream);
int fc2_unpack_codes(const uint8_t* planes, int64_t n, int32_t bitwidth, uint8_t* codes,
                     void* stream);

/* Per-group scalar API (codec.py:278-343): one group of any length n >= 1
 * (>= 4 with spike reserving), float64 values, exact float64 arithmetic.
 * Outputs: codes[n]; params = {scale, zero, spike_min_value, spike_max_value}
 * (float64, spikes only when sr); idx = {spike_min_index, spike_max_index}. */
int fc2_group_encode_raw(const double* v, int64_t n, int32_t bitwidth, int32_t sr, uint8_t* codes,
                         double* params, int32_t* idx, int32_t* dev_err, void* stream);
/* codes * scale + zero in float64 (codec.py:293-295). */
int fc2_group_decode_raw(const uint8_t* codes, int64_t n, double scale, double zero, double* out, void* stream);

/* Integer log scales (codec.py:366-392): round-half-away(log2(s) * theta)
 * clipped to int8 (0 -> -128 sentinel; negative -> FC2_ERR_NEGATIVE), and the
 * inverse exp2(si / theta) (integers in [-128, 127] from the host table). */
int fc2_scale_to_int(const double* s, int64_t n, int32_t theta, int8_t* out, int32_t* dev_err, void* stream);
int fc2_int_to_scale(const double* si, int64_t n, int32_t theta, double* out, void* stream);

/* Exact copy of n elements with the collectives' float32 staging
 * (collectives.py:160: cast to float32; :162-163: non-finite -> DataError via
 * FC2_ERR_NONFINITE in dev_err): the All2All diagonal block, which never
 * crosses a wire (collectives.py:466-468).  Output bf16 is the RNE rounding of
 * the float32 value (exact for bf16 input). */
int fc2_copy_check(const void* x, int32_t x_dtype, void* y, int32_t y_dtype, int64_t n, int32_t* dev_err,
                   void* stream);

/* bfloat16.py:16-36 on device arrays. */
int fc2_f32_to_bf16_bits(const float* x, int64_t n, uint16_t* out, void* stream);
int fc2_bf16_bits_to_f32(const uint16_t* x, int64_t n, float* out, void* stream);

/* ---- one-process-per-GPU communicator (CUDA IPC symmetric buffers) ------ */
typedef struct fc2_comm fc2_comm;

/* Bytes of one IPC handle (cudaIpcMemHandle_t). */
int fc2_comm_handle_bytes(void);
/* Allocate this rank's symmetric buffer (`bytes` usable + 4 KB of barrier
 * flags) on the current device and export its IPC handle into handle_out. */
int fc2_comm_create(int32_t rank, int32_t world, int64_t bytes, fc2_comm** out, void* handle_out);
/* Map every peer's buffer; handles = world * fc2_comm_handle_bytes() bytes
 * (all ranks' handles in rank order, e.g. from an all_gather). */
int fc2_comm_open_peers(fc2_comm* c, const void* handles);
int fc2_comm_destroy(fc2_comm* c);
/* Device pointer of peer's usable buffer (peer == own rank: local). */
void* fc2_comm_buffer(fc2_comm* c, int32_t peer);
/* Stream-ordered device barrier over all ranks (release/acquire system-scope
 * flags in peer memory); on timeout sets FC2_ERR_TIMEOUT in dev_err. */
int fc2_comm_barrier(fc2_comm* c, int32_t* dev_err, double timeout_s, void* stream);

/* Two-step quantized AllReduce of n elements per rank (collectives.py:263-315)
 * with the exchanges done as NVLink peer stores from the codec kernels.
 * slot_bytes: per-shard slot size (>= footprint of the shard, multiple of 16);
 * the buffer must hold 2 * world * slot_bytes. */
int fc2_allreduce_2step(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, void* y,
                        int32_t y_dtype, int64_t n, int64_t slot_bytes, int32_t* dev_err, double timeout_s,
                        void* stream);

/* One-shot variant for small messages (latency-bound sizes), same result bit
 * for bit: every rank stores all N of its packed shards into every peer (one
 * all-gather of packed bytes instead of the two-step's two exchanges), one
 * device barrier, then each rank reduces + requantizes every shard itself
 * (deterministic, so all ranks agree) and decodes.  Uses the region at
 * region_off of the symmetric buffer: 2 * world * world + world slots of
 * slot_bytes (double-buffered by call parity, so no trailing barrier). */
int fc2_allreduce_oneshot(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, void* y,
                          int32_t y_dtype, int64_t n, int64_t slot_bytes, int64_t region_off,
                          int32_t* dev_err, double timeout_s, void* stream);
/* Fused one-shot AllReduce ("a fused single-kernel two-step
 * with in-kernel flags"): the result of fc2_allreduce_oneshot -- same region,
 * same bits -- from one cooperative kernel: pack + peer stores, an in-kernel
 * grid barrier and cross-rank flags, then reduce + requantize + decode of every
 * shard.  bf16 / f32 tensors; float64-exact generic codec (latency regime). */
int fc2_allreduce_fused(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, void* y,
                        int32_t y_dtype, int64_t n, int64_t slot_bytes, int64_t region_off, int32_t* dev_err,
                        double timeout_s, void* stream);

/* Pipelined two-step (the NVSwitch form of the reference's microchunked
 * schedule, scheduling.py:119-156 over collectives.py:263-315): the shard is
 * cut into `chunks` (<= 16) microchunks of whole groups and encode/scatter,
 * reduce/requantize and gather/decode of successive microchunks overlap on
 * three streams, synchronised per chunk by release/acquire flags in peer
 * memory (no device-wide barrier).  Same result as fc2_allreduce_2step bit for
 * bit.  region_off / region_bytes: 4 * world * chunks * chunk_bytes bytes of
 * the symmetric buffer (two parity sets of landing + gather slots);
 * chunk_bytes >= footprint of one microchunk, a multiple of 16. */
int fc2_allreduce_2step_pipe(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, void* y,
                             int32_t y_dtype, int64_t n, int32_t chunks, int64_t chunk_bytes, int64_t region_off,
                             int64_t region_bytes, int32_t* dev_err, double timeout_s, void* stream);

/* Quantized All2All (dispatch, collectives.py:428-482; combine = transposed
 * matrix).  matrix: host int64[world*world] element counts.  Remote blocks are
 * encoded straight into the receiver's All2All region [region_off,
 * region_off + region_bytes) of the symmetric buffer (FC2_ECONFIG when they do
 * not fit it); the diagonal block is an exact copy (collectives.py:466-468)
 * whose non-finite values are flagged like the encoder's (:152-164). */
int fc2_a2a_q(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, const int64_t* matrix,
              void* y, int32_t y_dtype, int64_t region_off, int64_t region_bytes, int32_t* dev_err,
              double timeout_s, void* stream);

/* ---- MoE token dispatch / combine (BASELINE configs[3]; the reference's
 * block All2All, collectives.py:428-482, applied to routed token rows) ----- */

/* Routing: topk_ids [tokens][topk] (int32, or int64 when ids_are_int64),
 * experts split contiguously over world ranks (n_experts / world each).  A
 * token goes once to every rank holding at least one of its experts.
 * counts[d]: tokens for rank d; rows[d * tokens + i]: the i-th such token
 * (ascending); pos[t * world + d]: its index in that list or -1.  Expert ids
 * outside [0, n_experts) set FC2_ERR_EXPERT_RANGE. */
int fc2_moe_route(const void* topk_ids, int32_t ids_are_int64, int64_t tokens, int32_t topk, int32_t n_experts,
                  int32_t world, int32_t* counts, int32_t* rows, int32_t* pos, int32_t* dev_err, void* stream);
/* y[i] = x[rows[i]] for nrows rows of row_len elements (bf16/f32, 16-byte
 * aligned); non-finite values set FC2_ERR_NONFINITE (the diagonal block). */
int fc2_gather_rows_check(const void* x, int32_t x_dtype, const int32_t* rows, int64_t nrows, int64_t row_len,
                          void* y, int32_t y_dtype, int32_t* dev_err, void* stream);
/* Combine reduction: out[t] = sum over d = 0..world-1 with pos[t*world+d] >= 0
 * of srcs[d][pos[t*world+d]] (rows of row_len, dtype src_dtypes[d]), fp32 from
 * +0.0 in rank order; check_finite[d] flags non-finite rows of source d. */
int fc2_moe_combine_sum(int32_t world, const void* const* srcs, const int32_t* src_dtypes,
                        const int32_t* check_finite, const int32_t* pos, int64_t tokens, int64_t row_len, void* out,
                        int32_t out_dtype, int32_t* dev_err, void* stream);
/* Fused combine straight from the packed returned blocks: payloads[d] holds
 * block (d -> me) as one chunk of chunk_n[d] elements (d != me); exact: my own
 * block's rows (dtype exact_dtype).  Same result as decoding every block to
 * float32 and calling fc2_moe_combine_sum, without the float32 round trip.
 * Needs group_size % 32 == 0 and row_len % 32 == 0 (else FC2_ENOTAPPLICABLE). */
int fc2_moe_combine_q(const fc2_config* cfg, int32_t world, int32_t me, const void* const* payloads,
                      const int64_t* chunk_n, const void* exact, int32_t exact_dtype, const int32_t* pos,
                      int64_t tokens, int64_t row_len, void* out, int32_t out_dtype, int32_t* dev_err, void* stream);
/* Small all-gather of n <= 16 int32 values per rank through the communicator
 * (the token counts): all_out[p * n + k] = value k of rank p (device). */
int fc2_comm_allgather_i32(fc2_comm* c, const int32_t* mine, int32_t n, int32_t* all_out, int32_t* dev_err,
                           double timeout_s, void* stream);
/* SPMD dispatch: token_matrix[s*world + d] = rows rank s sends to d (host,
 * same on all ranks); rows_dev from fc2_moe_route.  y: the received rows,
 * per source rank in order (QDQ'd; exact for the rank's own tokens). */
int fc2_moe_dispatch(fc2_comm* c, const fc2_config* cfg, const void* x, int32_t x_dtype, int64_t tokens,
                     int64_t row_len, const int32_t* rows_dev, const int64_t* token_matrix, void* y, int32_t y_dtype,
                     int64_t region_off, int64_t region_bytes, int32_t* dev_err, double timeout_s, void* stream);
/* SPMD combine: y = the expert outputs in dispatch order; every block goes
 * back to its source rank with the same codec, and the source sums, per
 * token, the returned rows in rank order (fc2_moe_combine_sum) into out
 * [tokens][row_len].  scratch: float32, sum_d token_matrix[rank*world+d] rows. */
int fc2_moe_combine(fc2_comm* c, const fc2_config* cfg, const void* y, int32_t y_dtype, int64_t tokens,
                    int64_t row_len, const int64_t* token_matrix, const int32_t* pos_dev, float* scratch, void* out,
                    int32_t out_dtype, int64_t region_off, int64_t region_bytes, int32_t* dev_err,
                    double timeout_s, void* stream);

/* Device copy of nbytes (16-byte aligned buffers) with at most `ctas` CTAs
 * (<= 0: 4 per SM); dst may be a peer's symmetric buffer (fc2_comm_buffer), so
 * this is also the NVLink store-bandwidth probe. */
int fc2_copy_bytes(void* dst, const void* src, int64_t nbytes, int32_t ctas, void* stream);

/* Diagnostics. */
const char* fc2_last_error(void);
int64_t fc2_launch_count(void);   /* kernels launched by this library so far */
int fc2_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FC2_H */
