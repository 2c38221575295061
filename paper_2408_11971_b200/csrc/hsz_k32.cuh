// block_len == 32 fast path: one warp per block, one lane per element.
//
// A 32-element block is the reference default (model.py:58) and every
// BASELINE config.  With 32 lanes per block:
//   * the sign plane of a full block is exactly one word:
//       big-endian bytes of __brev(__ballot(resid < 0))        (FORMAT.md:30-32)
//   * the payload of a full block is exactly `w` 32-bit words of
//     element-major, MSB-first w-bit fields                     (FORMAT.md:33-37)
//   * every block section starts 4-byte aligned (only the global tail block,
//     always last, has a byte-granular size)
//
// Encode kernels (compress / encode_bins / scalar_mul) are single pass: the
// CTA stages its tile's input in shared memory with one TMA bulk copy,
// builds the packed sign words / payload words in shared memory, learns its
// global byte offsets by decoupled look-back (hsz_common.cuh) and streams
// the sections out.  Decode kernels (decompress / moments / the front half
// of scalar_mul) stage a tile's sign + payload bytes with bulk copies and
// rebuild bins with a warp inclusive scan.
#pragma once

#include "hsz_common.cuh"
#include "hsz_quant.cuh"

namespace hsz {
namespace k32 {

constexpr int K = 32;
constexpr int TB = kTileBlocks;          // blocks per tile (128)
constexpr int BPW = kBlocksPerWarp;      // blocks per warp (16)
constexpr int kThreads = kCtaWarps * 32;
constexpr int kPayWordsPerWarp = BPW * 64;    // worst case w = 64
constexpr int kTileElems = TB * K;

// ---------------------------------------------------------------------------
// packing of one block's magnitudes into `w` big-endian payload words

// w <= 32: every lane's field touches at most two words.  The word a field
// starts in is OR-reduced over its lanes by a segmented doubling shuffle;
// the (single) lane straddling into the next word hands its low part to the
// next segment's head.  Heads (lanes whose field starts a new word) store.
__device__ __forceinline__ void pack_narrow(uint32_t* dst, uint32_t mag, int w, int lane) {
  const uint32_t start = lane * w;
  const uint32_t a = start >> 5, o = start & 31;
  const uint32_t top = (w == 32) ? mag : (mag << (32 - w));   // left-aligned field
  uint32_t hi = top >> o;
  const uint32_t lo = (o + w > 32) ? (top << (32 - o)) : 0u;
  const uint32_t rem = 32 - o;              // bits of word `a` at or after my start
  // segment length <= ceil(32 / w); doubling steps while d*w < 32
  for (uint32_t d = 1, dw = w; dw < 32; d <<= 1, dw <<= 1) {
    const uint32_t v = __shfl_down_sync(kFull, hi, d);
    if (dw < rem && lane + d < 32) hi |= v;
  }
  const uint32_t carry = __shfl_up_sync(kFull, lo, 1);
  if (o < static_cast<uint32_t>(w)) {       // head of word a
    const uint32_t word = hi | (lane ? carry : 0u);
    if (a < static_cast<uint32_t>(w)) dst[a] = bswap32(word);
  }
}

// 32 < w <= 64: up to three words per field; zero then OR in shared memory.
__device__ __forceinline__ void pack_wide(uint32_t* dst, uint64_t mag, int w, int lane) {
  for (int t = lane; t < w; t += 32) dst[t] = 0u;
  __syncwarp();
  const uint32_t start = lane * w;
  const uint32_t a = start >> 5, o = start & 31;
  const unsigned __int128 win = static_cast<unsigned __int128>(mag) << (128 - w - o);
  const uint32_t w0 = static_cast<uint32_t>(win >> 96);
  const uint32_t w1 = static_cast<uint32_t>(win >> 64);
  const uint32_t w2 = static_cast<uint32_t>(win >> 32);
  if (w0) atomicOr(&dst[a], bswap32(w0));
  if (w1) atomicOr(&dst[a + 1], bswap32(w1));
  if (w2) atomicOr(&dst[a + 2], bswap32(w2));
  __syncwarp();
}

// ---------------------------------------------------------------------------
// bin sources for the encoder.  stage() runs with all CTA threads after the
// ticket is known; bin() returns lane's bin of tile-local block `lb`.

// copy `bytes` (multiple of 4) of a contiguous global range into smem with a
// TMA bulk copy when both ends are 16-byte aligned, else plain loads
__device__ __forceinline__ void stage_contig(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar, bool use_bulk) {
  if (use_bulk) {
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(bar, bytes);
      bulk_g2s(dst, src, bytes, bar);
    }
    __syncthreads();
    mbar_wait_parity(bar, 0);
  } else {
    const uint32_t* s = static_cast<const uint32_t*>(src);
    uint32_t* d = static_cast<uint32_t*>(dst);
    for (uint32_t i = threadIdx.x; i < bytes / 4; i += blockDim.x) d[i] = __ldg(s + i);
    __syncthreads();
  }
}

template <typename T>
struct SrcQuant {
  const T* x;
  uint64_t n;
  QuantConst c;
  static constexpr uint32_t kStageBytes = kTileElems * sizeof(T);

  __device__ __forceinline__ void stage(uint64_t tile, unsigned char* sm, uint64_t* bar) const {
    const uint64_t e0 = tile * kTileElems;
    const uint64_t cnt = (n - e0 < (uint64_t)kTileElems) ? (n - e0) : (uint64_t)kTileElems;
    const bool full = cnt == (uint64_t)kTileElems;
    const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
    if (full) {
      stage_contig(sm, x + e0, kStageBytes, bar, aligned);
    } else {
      T* d = reinterpret_cast<T*>(sm);
      for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) d[i] = x[e0 + i];
      __syncthreads();
    }
  }
  __device__ __forceinline__ int64_t bin(const unsigned char* sm, int lb, int lane, uint64_t,
                                         uint32_t* flags) const {
    const T v = reinterpret_cast<const T*>(sm)[lb * K + lane];
    return quantize1(static_cast<double>(v), c, flags);
  }
};

struct SrcBins {
  const int64_t* bins;
  uint64_t n;
  static constexpr uint32_t kStageBytes = kTileElems * 8;

  __device__ __forceinline__ void stage(uint64_t tile, unsigned char* sm, uint64_t* bar) const {
    const uint64_t e0 = tile * kTileElems;
    const uint64_t cnt = (n - e0 < (uint64_t)kTileElems) ? (n - e0) : (uint64_t)kTileElems;
    const bool aligned = (reinterpret_cast<uintptr_t>(bins) & 15u) == 0;
    if (cnt == (uint64_t)kTileElems) {
      stage_contig(sm, bins + e0, kStageBytes, bar, aligned);
    } else {
      int64_t* d = reinterpret_cast<int64_t*>(sm);
      for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) d[i] = bins[e0 + i];
      __syncthreads();
    }
  }
  __device__ __forceinline__ int64_t bin(const unsigned char* sm, int lb, int lane, uint64_t,
                                         uint32_t* flags) const {
    const int64_t v = reinterpret_cast<const int64_t*>(sm)[lb * K + lane];
    if (v == INT64_MIN) *flags |= HSZ_ERR_RESCALE_OVERFLOW;   // QuantArray guard model.py:124-128
    return v;
  }
};

// ---------------------------------------------------------------------------
// decode side: per-warp block metadata + tile staging of sign/payload bytes

struct StreamIn {
  const uint8_t* widths;
  const int32_t* outliers;
  const uint8_t* signs;
  const uint8_t* payload;
  const uint64_t* toff;
  uint64_t n;
  uint64_t nblocks;
  uint32_t tail_len;   // length of the last block (1..32)
};

// shared-memory image of one tile of an input stream
struct TileIn {
  static constexpr uint32_t kSignCap = TB * 4 + 32;
  static constexpr uint32_t kPayCap = TB * 256 + 32;
  static constexpr uint32_t kBytes = kSignCap + kPayCap;
  // per-warp block metadata, lane j (< BPW) holds block j
  uint32_t w;
  int32_t o;
  uint32_t soff;   // offsets into the staged tile images (bytes)
  uint32_t poff;
  const unsigned char* sgn;   // staged sign bytes (4-aligned view of the tile)
  const unsigned char* pay;
};

// Stage the sign and payload bytes of `tile` and compute, for the calling
// warp, the per-block metadata of its BPW blocks.  All CTA threads call.
__device__ __forceinline__ TileIn stage_tile_in(const StreamIn& s, uint64_t tile,
                                                unsigned char* sm, uint64_t* bar,
                                                uint32_t* s_wtot /* [2*kCtaWarps] */,
                                                uint32_t* flags) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t b = tile * TB + warp * BPW + lane;
  uint32_t w = 0;
  int32_t o = 0;
  uint32_t len = K;
  if (lane < BPW && b < s.nblocks) {
    w = s.widths[b];
    o = s.outliers[b];
    if (b == s.nblocks - 1) len = s.tail_len;
  }
  if (w > 64) {
    *flags |= HSZ_ERR_BAD_WIDTH;
    w = 0;
  }
  const uint32_t sb = w ? (len + 7) / 8 : 0;
  const uint32_t pb = (len * w + 7) / 8;
  // round to words: every block but the last one has word-multiple sizes
  uint32_t ss = sb, ps = pb;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t vs = __shfl_up_sync(kFull, ss, d);
    const uint32_t vp = __shfl_up_sync(kFull, ps, d);
    if (lane >= d) {
      ss += vs;
      ps += vp;
    }
  }
  // ss/ps are inclusive within the warp; lane 31 holds the warp totals
  if (lane == 31) {
    s_wtot[warp] = ss;
    s_wtot[kCtaWarps + warp] = ps;
  }
  const uint64_t g_s0 = s.toff[2 * tile], g_p0 = s.toff[2 * tile + 1];
  const uint64_t g_s1 = s.toff[2 * tile + 2], g_p1 = s.toff[2 * tile + 3];
  // stage [floor16(g0), ceil16(g1)) of both sections
  const uint64_t s_lo = g_s0 & ~15ull, s_hi = (g_s1 + 15) & ~15ull;
  const uint64_t p_lo = g_p0 & ~15ull, p_hi = (g_p1 + 15) & ~15ull;
  unsigned char* sm_sign = sm;
  unsigned char* sm_pay = sm + TileIn::kSignCap;
  const uint32_t sbytes = static_cast<uint32_t>(s_hi - s_lo);
  const uint32_t pbytes = static_cast<uint32_t>(p_hi - p_lo);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, sbytes + pbytes);
    if (sbytes) bulk_g2s(sm_sign, s.signs + s_lo, sbytes, bar);
    if (pbytes) bulk_g2s(sm_pay, s.payload + p_lo, pbytes, bar);
  }
  __syncthreads();
  uint32_t base_s = static_cast<uint32_t>(g_s0 - s_lo), base_p = static_cast<uint32_t>(g_p0 - p_lo);
  for (int i = 0; i < warp; ++i) {
    base_s += s_wtot[i];
    base_p += s_wtot[kCtaWarps + i];
  }
  TileIn t;
  t.w = w;
  t.o = o;
  t.soff = base_s + ss - sb;   // exclusive
  t.poff = base_p + ps - pb;
  t.sgn = sm_sign;
  t.pay = sm_pay;
  mbar_wait_parity(bar, 0);
  return t;
}

// Decode lane's bin of a block given its (warp-uniform) metadata.  The bins
// are O + inclusive prefix of signed residuals (slot 0 is ignored, as in
// codec.py:241 / 256-258).  Flags prefix overflow beyond +-(2^63-1).
__device__ __forceinline__ int64_t decode_block(const unsigned char* sgn, const unsigned char* pay,
                                                uint32_t w, int64_t o, uint32_t soff,
                                                uint32_t poff, int len, int lane,
                                                uint32_t* flags) {
  if (w == 0) return o;
  const uint32_t sw = bswap32(*reinterpret_cast<const uint32_t*>(sgn + soff));
  const bool neg = (__brev(sw) >> lane) & 1u;
  const uint32_t* pw = reinterpret_cast<const uint32_t*>(pay + poff);
  const uint32_t start = lane * w;
  const uint32_t a = start >> 5, sh = start & 31;
  const bool live = lane > 0 && lane < len;
  if (w <= 26) {
    // |resid| < 2^26: the 31-term prefix fits int32, bins fit int64 trivially
    const uint32_t w0 = bswap32(pw[a]);
    const uint32_t w1 = (sh + w > 32) ? bswap32(pw[a + 1]) : 0u;
    const uint64_t cat = (static_cast<uint64_t>(w0) << 32) | w1;
    const uint32_t mag = static_cast<uint32_t>((cat << sh) >> (64 - w));
    int32_t r = live ? (neg ? -static_cast<int32_t>(mag) : static_cast<int32_t>(mag)) : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t v = __shfl_up_sync(kFull, r, d);
      if (lane >= d) r += v;
    }
    return o + static_cast<int64_t>(r);
  }
  // wide residuals: exact 128-bit prefix with the reference's overflow rule
  uint64_t mag;
  {
    const uint32_t w0 = bswap32(pw[a]);
    const uint32_t w1 = bswap32(pw[a + 1]);
    const uint32_t w2 = (sh + w > 64) ? bswap32(pw[a + 2]) : 0u;
    const unsigned __int128 cat = (static_cast<unsigned __int128>(w0) << 64) |
                                  (static_cast<unsigned __int128>(w1) << 32) | w2;
    mag = static_cast<uint64_t>((cat << (32 + sh)) >> (128 - w));
  }
  __int128 r = live ? (neg ? -static_cast<__int128>(mag) : static_cast<__int128>(mag)) : 0;
  if (lane == 0) r = o;
  // the reference checks every running prefix; an inclusive scan yields all
  // of them (lanes past len repeat the last one)
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t vlo = __shfl_up_sync(kFull, static_cast<uint64_t>(r), d);
    const uint64_t vhi = __shfl_up_sync(kFull, static_cast<uint64_t>(r >> 64), d);
    if (lane >= d) r += (static_cast<__int128>(static_cast<int64_t>(vhi)) << 64) | vlo;
  }
  const __int128 lim = static_cast<__int128>(INT64_MAX);
  if (r > lim || r < -lim) {
    *flags |= HSZ_ERR_PREFIX_OVERFLOW;
    return 0;
  }
  return static_cast<int64_t>(r);
}

// ---------------------------------------------------------------------------
// smul source: decode the input stream tile, rescale (ops.py:199-225)

struct SrcSmul {
  StreamIn in;
  int64_t rs;
  double d;
  static constexpr uint32_t kStageBytes = TileIn::kBytes;
  // per-thread decode metadata built in stage()
  TileIn t;

  __device__ __forceinline__ void stage(uint64_t tile, unsigned char* sm, uint64_t* bar,
                                        uint32_t* s_wtot, uint32_t* flags) {
    t = stage_tile_in(in, tile, sm, bar, s_wtot, flags);
  }
  __device__ __forceinline__ int64_t bin(int j, int lane, int len, uint32_t* flags) {
    const uint32_t w = __shfl_sync(kFull, t.w, j);
    const int64_t o = __shfl_sync(kFull, t.o, j);
    const uint32_t so = __shfl_sync(kFull, t.soff, j);
    const uint32_t po = __shfl_sync(kFull, t.poff, j);
    uint32_t f = 0;
    const int64_t q = decode_block(t.sgn, t.pay, w, o, so, po, len, lane, &f);
    *flags |= f;
    if (f) return 0;
    return rescale1(product_rn(q, rs), d, flags);
  }
};

// ---------------------------------------------------------------------------
// the encoder kernel

struct EncodeOut {
  uint8_t* widths;
  int32_t* outliers;
  uint8_t* signs;
  uint64_t sign_cap;
  uint8_t* payload;
  uint64_t payload_cap;
  uint64_t* toff;
  uint32_t* err;
  void* ws;
};

template <class Src>
struct EncodeSmem {
  static constexpr uint32_t kStage = (Src::kStageBytes + 15) & ~15u;
  static constexpr uint32_t kSign = TB * 4;
  static constexpr uint32_t kPay = kCtaWarps * kPayWordsPerWarp * 4;
  static constexpr uint32_t kBytes = kStage + kSign + kPay;
};

template <class Src, bool kDecodes>
__global__ void __launch_bounds__(kThreads) encode_kernel(Src src, EncodeOut out,
                                                          uint64_t nblocks, uint64_t ntiles,
                                                          uint32_t tail_len) {
  extern __shared__ __align__(16) unsigned char sm[];
  using L = EncodeSmem<Src>;
  uint32_t* sm_sign = reinterpret_cast<uint32_t*>(sm + L::kStage);
  uint32_t* sm_pay = reinterpret_cast<uint32_t*>(sm + L::kStage + L::kSign);
  __shared__ uint64_t s_bar;
  __shared__ uint64_t s_tile, s_epoch, s_excl_s, s_excl_p;
  __shared__ uint32_t s_wtot[2 * kCtaWarps];
  __shared__ uint32_t s_wsb[kCtaWarps], s_wpb[kCtaWarps];
  __shared__ uint32_t s_err;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  LookbackWs lw = LookbackWs::bind(out.ws, ntiles);
  if (threadIdx.x == 0) {
    uint64_t t, e;
    draw_ticket(lw, ntiles, &t, &e);
    s_tile = t;
    s_epoch = e;
    s_err = 0;
  }
  __syncthreads();
  const uint64_t tile = s_tile;
  uint32_t flags = 0;
  if constexpr (kDecodes) {
    src.stage(tile, sm, &s_bar, s_wtot, &flags);
  } else {
    src.stage(tile, sm, &s_bar);
  }

  const uint64_t blk0 = tile * TB + warp * BPW;
  uint32_t* wsgn = sm_sign + warp * BPW;
  uint32_t* wpay = sm_pay + warp * kPayWordsPerWarp;
  uint32_t nsw = 0, npw = 0;          // staged sign words / payload words
  uint32_t sbytes = 0, pbytes = 0;    // exact section bytes of this warp
  uint32_t my_w = 0;
  int64_t my_o = 0;

  for (int j = 0; j < BPW; ++j) {
    const uint64_t b = blk0 + j;
    if (b >= nblocks) break;
    const int len = (b == nblocks - 1) ? static_cast<int>(tail_len) : K;
    int64_t q = 0;
    if constexpr (kDecodes) {
      q = src.bin(j, lane, len, &flags);
    } else {
      if (lane < len) q = src.bin(sm, warp * BPW + j, lane, b, &flags);
    }
    const int64_t first = __shfl_sync(kFull, q, 0);
    const int64_t prev = __shfl_up_sync(kFull, q, 1);
    bool neg = false;
    uint64_t mag = 0;
    if (lane > 0 && lane < len) mag = absdiff64(q, prev, &neg);
    const unsigned sbits = __ballot_sync(kFull, neg);
    const int wl = mag ? 64 - __clzll(static_cast<long long>(mag)) : 0;
    const int w = __reduce_max_sync(kFull, wl);
    if (lane == j) {
      my_w = w;
      my_o = first;
    }
    if (w) {
      if (lane == 0) wsgn[nsw] = bswap32(__brev(sbits));
      nsw += 1;
      sbytes += (len + 7) >> 3;
      if (w <= 32) {
        pack_narrow(wpay + npw, static_cast<uint32_t>(mag), w, lane);
      } else {
        pack_wide(wpay + npw, mag, w, lane);
      }
      npw += (len * w + 31) >> 5;
      pbytes += (len * w + 7) >> 3;
    }
  }
  // widths / outliers go straight to their fixed positions
  if (lane < BPW && blk0 + lane < nblocks) {
    out.widths[blk0 + lane] = static_cast<uint8_t>(my_w);
    if (my_o < INT32_MIN || my_o > INT32_MAX) flags |= HSZ_ERR_OUTLIER_OVERFLOW;
    out.outliers[blk0 + lane] = static_cast<int32_t>(my_o);
  }
  if (lane == 0) {
    s_wsb[warp] = sbytes;
    s_wpb[warp] = pbytes;
  }
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(&s_err, flags);
  __syncthreads();

  if (warp == 0) {
    uint32_t vs = lane < kCtaWarps ? s_wsb[lane] : 0u;
    uint32_t vp = lane < kCtaWarps ? s_wpb[lane] : 0u;
    uint64_t agg_s = __reduce_add_sync(kFull, vs);
    uint64_t agg_p = __reduce_add_sync(kFull, vp);
    uint64_t es, ep;
    lookback(lw, tile, s_epoch, agg_s, agg_p, &es, &ep);
    if (lane == 0) {
      s_excl_s = es;
      s_excl_p = ep;
      out.toff[2 * tile] = es;
      out.toff[2 * tile + 1] = ep;
      if (tile == ntiles - 1) {
        out.toff[2 * ntiles] = es + agg_s;
        out.toff[2 * ntiles + 1] = ep + agg_p;
      }
      uint32_t e = s_err;
      if (es + agg_s > out.sign_cap || ep + agg_p > out.payload_cap) e |= HSZ_ERR_CAPACITY;
      s_err = e;
      if (e) atomicOr(out.err, e);
    }
  }
  __syncthreads();
  if (s_err & HSZ_ERR_CAPACITY) return;
  uint64_t gs = s_excl_s, gp = s_excl_p;
  for (int i = 0; i < warp; ++i) {
    gs += s_wsb[i];
    gp += s_wpb[i];
  }
  // sections start 4-byte aligned (see header comment)
  uint32_t* dsg = reinterpret_cast<uint32_t*>(out.signs + gs);
  for (uint32_t i = lane; i < nsw; i += 32) dsg[i] = wsgn[i];
  uint32_t* dpy = reinterpret_cast<uint32_t*>(out.payload + gp);
  if (((gp & 15) == 0) && npw >= 4) {
    const uint32_t nv = npw >> 2;
    uint4* dv = reinterpret_cast<uint4*>(dpy);
    const uint4* sv = reinterpret_cast<const uint4*>(wpay);
    for (uint32_t i = lane; i < nv; i += 32) dv[i] = sv[i];
    for (uint32_t i = (nv << 2) + lane; i < npw; i += 32) dpy[i] = wpay[i];
  } else {
    for (uint32_t i = lane; i < npw; i += 32) dpy[i] = wpay[i];
  }
}

// ---------------------------------------------------------------------------
// decode kernels (grid = tiles, no look-back: offsets come from the cache)

struct SinkF32 {
  float* out;
  double d;
  __device__ __forceinline__ void put(uint64_t e, int64_t bin, uint32_t* flags) const {
    const float v = __double2float_rn(grid1(bin, d));
    if (!isfinite(v)) *flags |= HSZ_ERR_OUTPUT_NONFINITE;
    out[e] = v;
  }
};
struct SinkF64 {
  double* out;
  double d;
  __device__ __forceinline__ void put(uint64_t e, int64_t bin, uint32_t* flags) const {
    const double v = grid1(bin, d);
    if (!isfinite(v)) *flags |= HSZ_ERR_OUTPUT_NONFINITE;
    out[e] = v;
  }
};
struct SinkBins {
  int64_t* out;
  __device__ __forceinline__ void put(uint64_t e, int64_t bin, uint32_t*) const { out[e] = bin; }
};

template <class Sink>
__global__ void __launch_bounds__(kThreads) decode_kernel(StreamIn s, Sink sink, uint32_t* err) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint64_t s_bar;
  __shared__ uint32_t s_wtot[2 * kCtaWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t tile = blockIdx.x;
  uint32_t flags = 0;
  const TileIn t = stage_tile_in(s, tile, sm, &s_bar, s_wtot, &flags);
  const uint64_t blk0 = tile * TB + warp * BPW;
#pragma unroll 2
  for (int j = 0; j < BPW; ++j) {
    const uint64_t b = blk0 + j;
    if (b >= s.nblocks) break;
    const int len = (b == s.nblocks - 1) ? static_cast<int>(s.tail_len) : K;
    const uint32_t w = __shfl_sync(kFull, t.w, j);
    const int64_t o = __shfl_sync(kFull, t.o, j);
    const uint32_t so = __shfl_sync(kFull, t.soff, j);
    const uint32_t po = __shfl_sync(kFull, t.poff, j);
    const int64_t q = decode_block(t.sgn, t.pay, w, o, so, po, len, lane, &flags);
    if (lane < len) sink.put(b * K + lane, q, &flags);
  }
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(err, flags);
}

// exact moments: per lane S (int128) and Q (unsigned 192-bit)
struct Acc {
  __int128 s;
  unsigned __int128 q;
  uint64_t q2;
  __device__ __forceinline__ void add(int64_t bin, bool want_sq) {
    s += bin;
    if (want_sq) {
      const uint64_t m = bin < 0 ? static_cast<uint64_t>(-(bin + 1)) + 1u : static_cast<uint64_t>(bin);
      const unsigned __int128 sq = static_cast<unsigned __int128>(m) * m;
      const unsigned __int128 nq = q + sq;
      q2 += (nq < q) ? 1u : 0u;
      q = nq;
    }
  }
  __device__ __forceinline__ void merge(const Acc& o) {
    s += o.s;
    const unsigned __int128 nq = q + o.q;
    q2 += o.q2 + ((nq < q) ? 1u : 0u);
    q = nq;
  }
};

__device__ __forceinline__ Acc shfl_xor_acc(const Acc& a, int m) {
  Acc r;
  const uint64_t s0 = __shfl_xor_sync(kFull, static_cast<uint64_t>(a.s), m);
  const uint64_t s1 = __shfl_xor_sync(kFull, static_cast<uint64_t>(static_cast<unsigned __int128>(a.s) >> 64), m);
  const uint64_t q0 = __shfl_xor_sync(kFull, static_cast<uint64_t>(a.q), m);
  const uint64_t q1 = __shfl_xor_sync(kFull, static_cast<uint64_t>(a.q >> 64), m);
  r.q2 = __shfl_xor_sync(kFull, a.q2, m);
  r.s = static_cast<__int128>((static_cast<unsigned __int128>(s1) << 64) | s0);
  r.q = (static_cast<unsigned __int128>(q1) << 64) | q0;
  return r;
}

// Partials live in the workspace "vals" area: 6 u64 per tile.  The last CTA
// to finish (done counter) reduces them and writes out[5].
__device__ __forceinline__ void finish_moments(Acc acc, uint64_t ntiles, void* ws,
                                               uint64_t* out) {
  __shared__ Acc s_acc[kCtaWarps];
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int m = 16; m > 0; m >>= 1) acc.merge(shfl_xor_acc(acc, m));
  if (lane == 0) s_acc[warp] = acc;
  __syncthreads();
  uint64_t* base = static_cast<uint64_t*>(ws);
  uint64_t* done = base + 2;
  uint64_t* part = base + kWsFlagsOff + ntiles;   // vals area
  const int nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    Acc t = s_acc[0];
    for (int i = 1; i < nw; ++i) t.merge(s_acc[i]);
    uint64_t* p = part + 6 * blockIdx.x;
    p[0] = static_cast<uint64_t>(t.s);
    p[1] = static_cast<uint64_t>(static_cast<unsigned __int128>(t.s) >> 64);
    p[2] = static_cast<uint64_t>(t.q);
    p[3] = static_cast<uint64_t>(t.q >> 64);
    p[4] = t.q2;
    __threadfence();
    const uint64_t prev = atom_add_acq_rel(done, 1);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  Acc tot;
  tot.s = 0;
  tot.q = 0;
  tot.q2 = 0;
  for (uint64_t i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
    const uint64_t* p = part + 6 * i;
    Acc a;
    a.s = static_cast<__int128>((static_cast<unsigned __int128>(ld_relaxed(p + 1)) << 64) | ld_relaxed(p));
    a.q = (static_cast<unsigned __int128>(ld_relaxed(p + 3)) << 64) | ld_relaxed(p + 2);
    a.q2 = ld_relaxed(p + 4);
    tot.merge(a);
  }
  for (int m = 16; m > 0; m >>= 1) tot.merge(shfl_xor_acc(tot, m));
  __syncthreads();
  if (lane == 0) s_acc[warp] = tot;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc t = s_acc[0];
    for (int i = 1; i < nw; ++i) t.merge(s_acc[i]);
    out[0] = static_cast<uint64_t>(t.s);
    out[1] = static_cast<uint64_t>(static_cast<unsigned __int128>(t.s) >> 64);
    out[2] = static_cast<uint64_t>(t.q);
    out[3] = static_cast<uint64_t>(t.q >> 64);
    out[4] = t.q2;
    st_relaxed(done, 0);   // rearm for the next launch on this workspace
  }
}

template <bool kWantSq>
__global__ void __launch_bounds__(kThreads) moments_kernel(StreamIn s, uint64_t* out,
                                                           uint32_t* err, void* ws) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint64_t s_bar;
  __shared__ uint32_t s_wtot[2 * kCtaWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t tile = blockIdx.x;
  uint32_t flags = 0;
  const TileIn t = stage_tile_in(s, tile, sm, &s_bar, s_wtot, &flags);
  const uint64_t blk0 = tile * TB + warp * BPW;
  Acc acc;
  acc.s = 0;
  acc.q = 0;
  acc.q2 = 0;
  for (int j = 0; j < BPW; ++j) {
    const uint64_t b = blk0 + j;
    if (b >= s.nblocks) break;
    const int len = (b == s.nblocks - 1) ? static_cast<int>(s.tail_len) : K;
    const uint32_t w = __shfl_sync(kFull, t.w, j);
    const int64_t o = __shfl_sync(kFull, t.o, j);
    const uint32_t so = __shfl_sync(kFull, t.soff, j);
    const uint32_t po = __shfl_sync(kFull, t.poff, j);
    const int64_t q = decode_block(t.sgn, t.pay, w, o, so, po, len, lane, &flags);
    if (lane < len) acc.add(q, kWantSq);
  }
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(err, flags);
  const uint64_t ntiles = gridDim.x;
  finish_moments(acc, ntiles, ws, out);
}

}  // namespace k32
}  // namespace hsz
