/* hsz_b200.h -- C ABI of the B200-native HoSZp hot path (sm_100a).
 *
 * Drop-in boundary for the reference package `hoszp` 0.1.0
 * (arxiv 2408.11971).  The reference is pure Python/numpy and has no FFI;
 * its operator API is the module surface listed in SURVEY.md §8(b).  Each
 * entry point below names the reference function it replaces (file:line
 * relative to /root/reference/pkg/src/hoszp/).  The Python mirror of that
 * API (paper_2408_11971_b200/codec.py, ops.py) binds these symbols through
 * ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - every pointer argument is DEVICE memory unless stated; the caller owns
 *    all buffers (torch tensors or cudaMalloc) and passes a cudaStream_t as
 *    `void* stream` (NULL = legacy default stream);
 *  - all calls are asynchronous on `stream`; data-dependent failures are
 *    OR-ed into the device error word `*err` (HSZ_ERR_* bits) and surface
 *    after the caller synchronizes -- the Python layer maps them onto the
 *    reference's exception classes (errors.py:4-45);
 *  - the return value reports argument / launch errors only (HSZ_OK = 0);
 *  - a stream is described by four section buffers exactly as in
 *    pkg/FORMAT.md:24-37 -- widths u8[B], outliers i32[B], sign planes,
 *    payload -- plus a tile-offset cache: u64[2*(T+1)] holding the exclusive
 *    (sign, payload) byte offset of every tile of HSZ_TILE_BLOCKS blocks,
 *    T = hsz_tile_count(n, block_len); entry T is the section totals;
 *  - section buffers must have HSZ_SECTION_SLACK zero bytes of slack past
 *    their capacity (kernels read/write whole 32-bit words at the end);
 *  - `ws` is a per-stream workspace of hsz_workspace_size() bytes, zeroed
 *    once with hsz_workspace_init(); it is reused across calls on the same
 *    CUDA stream (never concurrently from two streams).  Encoders tag their
 *    look-back words with 24 bits of a launch epoch kept in the workspace:
 *    re-initialise it at least every 2^23 calls (the Python layer does so
 *    every 2^22).
 */
#ifndef HSZ_B200_H
#define HSZ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HSZ_TILE_BLOCKS 128
#define HSZ_SECTION_SLACK 16

/* raw element type codes (FORMAT.md header byte 5) */
#define HSZ_F32 0
#define HSZ_F64 1

/* decode output kinds */
#define HSZ_OUT_F32 0   /* float32 values   (codec.py:112-115, f32 streams)   */
#define HSZ_OUT_F64 1   /* float64 grid     (codec.py:107-109, 511-513)       */
#define HSZ_OUT_BINS 2  /* int64 bins       (codec.py:517-520 decode_to_quant) */
#define HSZ_OUT_BINS_ADD 3  /* out[i] += bin_i (int64, modulo 2^64): N-way folds  */
#define HSZ_OUT_BINS_SUB 4  /* out[i] -= bin_i (distsim.py:80-103)                 */

/* return codes */
#define HSZ_OK 0
#define HSZ_EINVAL (-1)
#define HSZ_ECUDA (-2)
#define HSZ_ETIMEDOUT (-3) /* a host-side wait on the stream exceeded its bound */

/* device error-word bits */
#define HSZ_ERR_NONFINITE (1u << 0)         /* ValueError      codec.py:52-53   */
#define HSZ_ERR_QUANT_OVERFLOW (1u << 1)    /* QuantOverflow   codec.py:136-137 */
#define HSZ_ERR_QUANT_RESOLUTION (1u << 2)  /* QuantOverflow   codec.py:150-154 */
#define HSZ_ERR_PREFIX_OVERFLOW (1u << 3)   /* QuantOverflow   codec.py:259-260 */
#define HSZ_ERR_RESCALE_OVERFLOW (1u << 4)  /* QuantOverflow   ops.py:201-202   */
#define HSZ_ERR_OUTLIER_OVERFLOW (1u << 5)  /* OutlierOverflow model.py:182-191 */
#define HSZ_ERR_CAPACITY (1u << 6)          /* output section buffer too small  */
#define HSZ_ERR_OUTPUT_NONFINITE (1u << 7)  /* ValueError on decoded RawArray   */
#define HSZ_ERR_BAD_WIDTH (1u << 8)         /* GeometryMismatch model.py:217    */
#define HSZ_ERR_LOOKBACK_TIMEOUT (1u << 9)  /* encoder look-back watchdog fired:
                                               offsets undefined (DeviceTimeout);
                                               re-initialise the workspace      */

/* ---- geometry / workspace ------------------------------------------------ */

/* number of tiles of HSZ_TILE_BLOCKS blocks (QuantParams.block_count, model.py:81-84) */
uint64_t hsz_tile_count(uint64_t n, uint32_t block_len);
/* worst-case section sizes (bytes) for n elements: sign planes, payload */
uint64_t hsz_sign_bound(uint64_t n, uint32_t block_len);
uint64_t hsz_payload_bound(uint64_t n, uint32_t block_len);
uint64_t hsz_workspace_size(uint64_t n, uint32_t block_len);
int hsz_workspace_init(void* ws, uint64_t ws_bytes, void* stream);
/* scratch (device bytes) hsz_scalar_mul needs besides ws (0 for block_len 32) */
uint64_t hsz_scalar_mul_scratch_size(uint64_t n, uint32_t block_len);

/* ---- K0: value range + finiteness -----------------------------------------
 * Replaces the RawArray finite check (codec.py:52-53) and the two reductions
 * of resolve_eps(mode="rel") (codec.py:96-99).  minmax = device double[2]
 * (exact: every f32 widens exactly). */
int hsz_minmax(const void* x, int dtype, uint64_t n, double* minmax, uint32_t* err,
               void* ws, uint64_t ws_bytes, void* stream);

/* ---- K1: compress ----------------------------------------------------------
 * Replaces codec.compress (codec.py:495-498) = quantize (codec.py:118-155)
 * + _split_residuals/_block_widths/_pack_stream (codec.py:178-225,393-416).
 * Single pass: the input is read once, sections are placed by decoupled
 * look-back.  tile_offsets[2*T], [2*T+1] receive the section totals.  If a
 * section outgrows its capacity HSZ_ERR_CAPACITY is set (totals still valid)
 * and the caller retries with exact capacities. */
int hsz_compress(const void* x, int dtype, uint64_t n, uint32_t block_len, double eps,
                 uint8_t* widths, int32_t* outliers, uint8_t* signs, uint64_t sign_cap,
                 uint8_t* payload, uint64_t payload_cap, uint64_t* tile_offsets,
                 uint32_t* err, void* ws, uint64_t ws_bytes, void* stream);

/* Replaces codec.encode_from_quant (codec.py:523-525): int64 bins -> stream. */
int hsz_encode_bins(const int64_t* bins, uint64_t n, uint32_t block_len, uint8_t* widths,
                    int32_t* outliers, uint8_t* signs, uint64_t sign_cap, uint8_t* payload,
                    uint64_t payload_cap, uint64_t* tile_offsets, uint32_t* err, void* ws,
                    uint64_t ws_bytes, void* stream);

/* Replaces codec.quantize (codec.py:118-155): raw values -> int64 bins. */
int hsz_quantize(const void* x, int dtype, uint64_t n, double eps, int64_t* bins,
                 uint32_t* err, void* stream);

/* Replaces codec.dequantize (codec.py:158-160): int64 bins -> values
 * (out_kind HSZ_OUT_F32 / HSZ_OUT_F64). */
int hsz_dequantize(const int64_t* bins, uint64_t n, double eps, int out_kind, void* out,
                   uint32_t* err, void* stream);

/* ---- K2: tile offsets (section offsets of codec.py:298-301, per tile) ---- */
int hsz_tile_offsets(const uint8_t* widths, uint64_t n, uint32_t block_len,
                     uint64_t* tile_offsets, uint32_t* err, void* ws, uint64_t ws_bytes,
                     void* stream);

/* ---- K3: decode ------------------------------------------------------------
 * Replaces codec.decompress (codec.py:501-514) and decode_to_quant
 * (codec.py:517-520): unpack (codec.py:350-441) + prefix rebuild
 * (codec.py:228-262) + dequantize (codec.py:107-115).  out_kind HSZ_OUT_*. */
int hsz_decode(const uint8_t* widths, const int32_t* outliers, const uint8_t* signs,
               const uint8_t* payload, const uint64_t* tile_offsets, uint64_t n,
               uint32_t block_len, double eps, int out_kind, void* out, uint32_t* err,
               void* stream);

/* ---- K4: negate (ops.py:88-109) --------------------------------------------
 * Flips every stored sign bit (padding untouched) and negates the outliers.
 * widths / payload / tile offsets are shared with the input, as in the
 * reference.  The sign-section length is read from tile_offsets[2*T]. */
int hsz_negate(const uint8_t* widths, const int32_t* outliers_in, int32_t* outliers_out,
               const uint8_t* signs_in, uint8_t* signs_out, const uint64_t* tile_offsets,
               uint64_t n, uint32_t block_len, uint32_t* err, void* stream);

/* ---- K5: scalar add / sub (ops.py:112-125): outliers + rs, int32 guard --- */
int hsz_scalar_add(const int32_t* outliers_in, int32_t* outliers_out, uint64_t nblocks,
                   int64_t rs, uint32_t* err, void* stream);

/* ---- K6: scalar multiply (ops.py:199-225) ----------------------------------
 * decode -> p = bin * rs (exact) -> RN(2eps * f64(p)) -> round half away ->
 * re-encode, fused and placed by look-back.  `scratch` as sized by
 * hsz_scalar_mul_scratch_size (may be NULL when that is 0). */
int hsz_scalar_mul(const uint8_t* widths, const int32_t* outliers, const uint8_t* signs,
                   const uint8_t* payload, const uint64_t* tile_offsets, uint64_t n,
                   uint32_t block_len, double eps, int64_t rs, uint8_t* out_widths,
                   int32_t* out_outliers, uint8_t* out_signs, uint64_t sign_cap,
                   uint8_t* out_payload, uint64_t payload_cap, uint64_t* out_tile_offsets,
                   void* scratch, uint32_t* err, void* ws, uint64_t ws_bytes, void* stream);

/* ---- K8: element-wise add / sub of two streams (ops.py:163-192) ----------
 * out = a + b (sub = 0) or a - b (sub = 1); a and b share n / block_len /
 * eps (the caller checks the params, ops.py:77-81).  Outliers combine in
 * int64 under the int32 guard (HSZ_ERR_OUTLIER_OVERFLOW), signed residuals
 * combine element by element, the result is re-encoded and placed by
 * look-back.  `scratch` as sized by hsz_elementwise_scratch_size. */
uint64_t hsz_elementwise_scratch_size(uint64_t n, uint32_t block_len);
int hsz_elementwise(const uint8_t* a_widths, const int32_t* a_outliers, const uint8_t* a_signs,
                    const uint8_t* a_payload, const uint64_t* a_tile_offsets,
                    const uint8_t* b_widths, const int32_t* b_outliers, const uint8_t* b_signs,
                    const uint8_t* b_payload, const uint64_t* b_tile_offsets, uint64_t n,
                    uint32_t block_len, int sub, uint8_t* out_widths, int32_t* out_outliers,
                    uint8_t* out_signs, uint64_t sign_cap, uint8_t* out_payload,
                    uint64_t payload_cap, uint64_t* out_tile_offsets, void* scratch, uint32_t* err,
                    void* ws, uint64_t ws_bytes, void* stream);

/* ---- bivariate quantized-domain operations (ops.py:226-240, 400-513) and
 * per-block means (ops.py:366-379): the operands decode to int64 bins in
 * `scratch` (hsz_bivariate_scratch_size bytes), then
 *   hsz_hadamard    bins = round-half-away(RN(2eps * RN(a*b))), re-encoded;
 *   hsz_pair_stats  exact sums for covariance / ssim_global into out
 *                   (u64[52]: 24 carry-save counters of 32-bit chunks, two
 *                   words each -- SA+ SA- SB+ SB- (2 chunks), QA QB SAB+ SAB-
 *                   (4 chunks) -- then min a, max a, min b, max b as int64);
 *   hsz_block_means out (device f64[B]) = 2eps * sum(block bins) / length. */
uint64_t hsz_bivariate_scratch_size(uint64_t n, uint32_t block_len);
int hsz_hadamard(const uint8_t* a_widths, const int32_t* a_outliers, const uint8_t* a_signs,
                 const uint8_t* a_payload, const uint64_t* a_tile_offsets, const uint8_t* b_widths,
                 const int32_t* b_outliers, const uint8_t* b_signs, const uint8_t* b_payload,
                 const uint64_t* b_tile_offsets, uint64_t n, uint32_t block_len, double eps,
                 uint8_t* out_widths, int32_t* out_outliers, uint8_t* out_signs, uint64_t sign_cap,
                 uint8_t* out_payload, uint64_t payload_cap, uint64_t* out_tile_offsets,
                 void* scratch, uint32_t* err, void* ws, uint64_t ws_bytes, void* stream);
int hsz_pair_stats(const uint8_t* a_widths, const int32_t* a_outliers, const uint8_t* a_signs,
                   const uint8_t* a_payload, const uint64_t* a_tile_offsets,
                   const uint8_t* b_widths, const int32_t* b_outliers, const uint8_t* b_signs,
                   const uint8_t* b_payload, const uint64_t* b_tile_offsets, uint64_t n,
                   uint32_t block_len, uint64_t* out, void* scratch, uint32_t* err, void* stream);
int hsz_block_means(const uint8_t* widths, const int32_t* outliers, const uint8_t* signs,
                    const uint8_t* payload, const uint64_t* tile_offsets, uint64_t n,
                    uint32_t block_len, double eps, double* out, void* scratch, uint32_t* err,
                    void* stream);

/* ---- K7: exact moments (ops.py:249-357) -------------------------------------
 * out (device u64[5]) = S as signed 128-bit (lo, hi) and, if want_sq,
 * Q = sum(bins^2) as unsigned 192-bit (limb0, limb1, limb2).  The host
 * finishes mean (ops.py:363) / variance (ops.py:386,393) with exact ints. */
int hsz_moments(const uint8_t* widths, const int32_t* outliers, const uint8_t* signs,
                const uint8_t* payload, const uint64_t* tile_offsets, uint64_t n,
                uint32_t block_len, int want_sq, uint64_t* out, uint32_t* err, void* ws,
                uint64_t ws_bytes, void* stream);

/* ---- host plumbing for the Python layer ------------------------------------
 * hsz_copy_d2h: asynchronous device -> host copy on `stream` (host should be
 * pinned for a truly asynchronous copy); hsz_stream_sync: wait for `stream`.
 * Used to fetch a reduction's limbs and the error word in one round trip. */
int hsz_copy_d2h(void* host, const void* dev, uint64_t bytes, void* stream);
int hsz_stream_sync(void* stream);
/* copy + wait in one call: the round trip of a reduction whose result and
 * error word share one small device record */
int hsz_fetch(void* host, const void* dev, uint64_t bytes, void* stream);

/* Host-mapped mailbox variants of the two reductions the host waits on:
 * `mailbox` = pinned host memory (u64[8], device-accessible through UVA);
 * the kernel's last CTA writes [1..nres] = the result words (minmax: 2 f64
 * bit patterns, moments: the 5 u64 limbs), [1 + nres] = the error word, then
 * [0] = seq.  hsz_mailbox_wait polls word 0 for `seq`; it returns HSZ_OK,
 * HSZ_ECUDA (the stream faulted) or HSZ_EINVAL (the stream drained without
 * a post -- fetch with hsz_fetch instead). */
int hsz_minmax_mb(const void* x, int dtype, uint64_t n, double* minmax, uint32_t* err, void* ws,
                  uint64_t ws_bytes, uint64_t* mailbox, uint64_t seq, void* stream);
int hsz_moments_mb(const uint8_t* widths, const int32_t* outliers, const uint8_t* signs,
                   const uint8_t* payload, const uint64_t* tile_offsets, uint64_t n,
                   uint32_t block_len, int want_sq, uint64_t* out, uint32_t* err, void* ws,
                   uint64_t ws_bytes, uint64_t* mailbox, uint64_t seq, void* stream);
int hsz_mailbox_wait(const uint64_t* mailbox, uint64_t seq, void* stream);

/* ---- node-local host all-gather (multi-GPU plumbing) -----------------------
 * The small per-step exchanges of sharding.Collectives (C1 value range, C2
 * section sizes, C3 moment limbs) between the one-process-
 * per-GPU ranks of ONE node, through a shared memory segment of
 * hsz_hostcoll_bytes(world) zeroed bytes every rank maps.  Round r (1, 2,
 * ...; the same on every rank) publishes nvals (<= 40) int64 words of this
 * rank and gathers world * nvals words in rank order into out.  Returns
 * HSZ_ECUDA when a peer has not published within timeout_s (> 0). */
uint64_t hsz_hostcoll_bytes(int world);
int hsz_hostcoll_allgather(void* shm, int rank, int world, uint64_t round, const int64_t* vals,
                           int nvals, int64_t* out, double timeout_s);

/* Bound (seconds, default 600) of every host-side wait of this library
 * (hsz_stream_sync, hsz_fetch, hsz_mailbox_wait): past it they return
 * HSZ_ETIMEDOUT instead of blocking forever on a hung kernel.  seconds <= 0
 * leaves it unchanged; returns the previous bound. */
double hsz_set_host_wait_timeout(double seconds);

/* library identification (for the loader's sanity check) */
const char* hsz_version(void);

/* Look-back watchdog of the encoders: how many back-offs a warp waiting for
 * a predecessor tile's offsets takes before it gives up and sets
 * HSZ_ERR_LOOKBACK_TIMEOUT (0 = leave unchanged).  Returns the previous
 * bound.  Default 2^23 (seconds of waiting; no legitimate wait comes close). */
unsigned int hsz_set_lookback_watchdog(unsigned int max_sleeps);

/* debug builds (-DHSZ_TRACE): copy out per-CTA phase timestamps; -1 otherwise */
int hsz_trace_read(unsigned long long* host, int cap, int reset);
/* debug builds: look-back (rounds, sleeps, resolves) since the last call; -1 otherwise */
int hsz_trace_lookback(unsigned int* out3);

#ifdef __cplusplus
}
#endif

#endif /* HSZ_B200_H */
