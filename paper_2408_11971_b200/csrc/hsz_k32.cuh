// block_len == 32 kernels (the reference default, model.py:58, and every
// BASELINE config).  One CTA of 128 threads owns one tile of 128 blocks
// (4096 elements).
//
// Fast path (every tile whose bins fit 30 bits / whose residual widths are
// <= 26 bits -- all realistic data):
//   * element-parallel phase: quantize (or decode) with coalesced shared
//     memory access into a tile of int32 bin rows, row stride 33 words so
//     that a thread walking "its" row never bank-conflicts with its warp;
//   * thread-per-block phase: each thread walks one 32-element row serially
//     -- Lorenzo residuals, OR-reduced width, sign word, MSB-first bit
//     packing through a 64-bit shift register -- no shuffles, no ballots,
//     every instruction works for 32 blocks at once.
// Fallback (a tile with wider values): one warp per block, one lane per
// element, exact 64/128-bit arithmetic for widths up to 64.  Both produce
// identical bytes; the choice is per tile (CTA-uniform).
//
// Encoders (compress / encode_bins / scalar_mul) are single pass: the input
// tile is staged in shared memory with one TMA bulk copy, the packed sign
// words / payload words are built in shared memory, the tile's global byte
// offsets come from the decoupled look-back of hsz_common.cuh and the
// sections are streamed out with coalesced (16-byte when aligned) stores.
// Decoders (decompress / moments / the front of scalar_mul) stage the tile's
// sign + payload bytes with bulk copies and locate every block from the
// tile-offset cache plus a CTA scan of the widths.
//
// Stream layout facts used throughout (FORMAT.md:24-37, block_len 32): the
// sign plane of a full block is one big-endian word, the payload of a full
// block is exactly `w` big-endian words, so every section offset except the
// one after the global tail block is 4-byte aligned.
#pragma once

#include "hsz_common.cuh"
#include "hsz_quant.cuh"

namespace hsz {
namespace k32 {

constexpr int K = 32;
constexpr int TB = kTileBlocks;               // 128 blocks per tile
constexpr int BPW = kBlocksPerWarp;           // 32 blocks per warp (fallback path)
constexpr int kThreads = kCtaWarps * 32;      // 128
constexpr int kTileElems = TB * K;            // 4096
constexpr int kWideLimit = 1 << 30;           // fast path: |bin| < 2^30
constexpr int kRow = 33;                      // padded row stride: conflict-free row walks

static_assert(kThreads == TB, "fast path maps one thread to one block");

// ---------------------------------------------------------------------------
// CTA-wide exclusive scan of two u32 (blockDim == 128)

__device__ __forceinline__ void scan2(uint32_t a, uint32_t b, uint32_t* ea, uint32_t* eb,
                                      uint32_t* ta, uint32_t* tb, uint32_t* s_tmp /*[8]*/) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t ia = a, ib = b;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t va = __shfl_up_sync(kFull, ia, d);
    const uint32_t vb = __shfl_up_sync(kFull, ib, d);
    if (lane >= d) {
      ia += va;
      ib += vb;
    }
  }
  if (lane == 31) {
    s_tmp[warp] = ia;
    s_tmp[4 + warp] = ib;
  }
  __syncthreads();
  uint32_t pa = 0, pb = 0, sa = 0, sb = 0;
#pragma unroll
  for (int i = 0; i < kCtaWarps; ++i) {
    const uint32_t xa = s_tmp[i], xb = s_tmp[4 + i];
    if (i < warp) {
      pa += xa;
      pb += xb;
    }
    sa += xa;
    sb += xb;
  }
  *ea = pa + ia - a;
  *eb = pb + ib - b;
  *ta = sa;
  *tb = sb;
}

// ---------------------------------------------------------------------------
// TMA staging helpers

// copy `bytes` (multiple of 16) of a contiguous, 16-byte aligned global
// range into smem with one bulk copy (thread 0 issues; everyone waits)
__device__ __forceinline__ void stage_bulk(void* dst, const void* src, uint32_t bytes,
                                           uint64_t* bar) {
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(dst, src, bytes, bar);
  }
  __syncthreads();
  mbar_wait_parity(bar, 0);
}

template <typename T>
__device__ __forceinline__ void stage_elems(T* dst, const T* src, uint64_t e0, uint64_t n,
                                            uint64_t* bar) {
  const uint64_t cnt = (n - e0 < (uint64_t)kTileElems) ? (n - e0) : (uint64_t)kTileElems;
  const bool aligned = (reinterpret_cast<uintptr_t>(src) & 15u) == 0;
  if (cnt == (uint64_t)kTileElems && aligned) {
    stage_bulk(dst, src + e0, kTileElems * sizeof(T), bar);
  } else {
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) dst[i] = src[e0 + i];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// input stream tile (decode side)

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

constexpr int kFastW = 26;                                  // fast decode: widths <= 26
constexpr uint32_t kStageSign = TB * 4 + 32;                // staged sign bytes (+ align slack)
constexpr uint32_t kStagePay = TB * kFastW * 4 + 32;        // staged payload of a fast tile
constexpr uint32_t kStageFast = kStageSign + kStagePay;     // 13888 bytes

// element (b, i) of a padded tile image: row walks (thread b, i = 0..31) and
// element-order sweeps (e = j*128 + tid) are both bank-conflict free, and
// both use immediate offsets
__device__ __forceinline__ int pad(int b, int i) { return b * kRow + i; }
// element e = j * 128 + threadIdx.x of the tile, padded
__device__ __forceinline__ int pad_sweep_base() { return (threadIdx.x >> 5) * kRow + (threadIdx.x & 31); }
constexpr int kSweepStride = 4 * kRow;   // += per j

// One tile of an input stream as seen by thread b (= block b of the tile).
// Fast tiles (every width <= 26) are staged in shared memory by TMA bulk
// copies; other tiles are read in place from global memory.
struct TileIn {
  uint32_t w;      // width of this thread's block
  int32_t o;       // its outlier
  int len;         // its length (0 past the end of the stream)
  uint64_t soff;   // byte offsets relative to sgn / pay
  uint64_t poff;
  const unsigned char* sgn;
  const unsigned char* pay;
  bool fast;       // CTA-uniform
};

__device__ __forceinline__ void stage_tile_in(const StreamIn& s, uint64_t tile, unsigned char* sm,
                                              uint64_t* bar, uint32_t* s_tmp, TileIn* t,
                                              uint32_t* flags) {
  const uint64_t b = tile * TB + threadIdx.x;
  uint32_t w = 0;
  int32_t o = 0;
  int len = 0;
  if (b < s.nblocks) {
    w = s.widths[b];
    o = s.outliers[b];
    len = (b == s.nblocks - 1) ? static_cast<int>(s.tail_len) : K;
  }
  if (w > 64) {
    *flags |= HSZ_ERR_BAD_WIDTH;
    w = 0;
  }
  const uint32_t sb = w ? (len + 7) / 8 : 0;
  const uint32_t pb = (len * w + 7) / 8;
  uint32_t es, ep, ts, tp;
  scan2(sb, pb, &es, &ep, &ts, &tp, s_tmp);
  const uint64_t g_s0 = s.toff[2 * tile], g_p0 = s.toff[2 * tile + 1];
  const bool fast = __syncthreads_and(w <= kFastW) != 0;   // also orders s_tmp reuse
  t->w = w;
  t->o = o;
  t->len = len;
  t->fast = fast;
  if (fast) {
    const uint64_t s_lo = g_s0 & ~15ull, s_hi = (g_s0 + ts + 15) & ~15ull;
    const uint64_t p_lo = g_p0 & ~15ull, p_hi = (g_p0 + tp + 15) & ~15ull;
    const uint32_t sbytes = static_cast<uint32_t>(s_hi - s_lo);
    const uint32_t pbytes = static_cast<uint32_t>(p_hi - p_lo);
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(bar, sbytes + pbytes);
      if (sbytes) bulk_g2s(sm, s.signs + s_lo, sbytes, bar);
      if (pbytes) bulk_g2s(sm + kStageSign, s.payload + p_lo, pbytes, bar);
    }
    t->sgn = sm;
    t->pay = sm + kStageSign;
    t->soff = (g_s0 - s_lo) + es;
    t->poff = (g_p0 - p_lo) + ep;
    __syncthreads();
    mbar_wait_parity(bar, 0);
  } else {
    t->sgn = s.signs;
    t->pay = s.payload;
    t->soff = g_s0 + es;
    t->poff = g_p0 + ep;
  }
}

// Fast decode of this thread's block (w <= 26): calls emit(i, P) for every
// element i < 32 with P = prefix sum of signed residuals (P = 0 at i = 0);
// the bin is t.o + P.  |P| < 2^31.
template <class Emit>
__device__ __forceinline__ void decode_row_fast(const TileIn& t, Emit&& emit) {
  const uint32_t w = t.w;
  if (w == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) emit(i, 0);
    return;
  }
  const uint32_t sw = bswap32(*reinterpret_cast<const uint32_t*>(t.sgn + t.soff));
  const uint32_t* pw = reinterpret_cast<const uint32_t*>(t.pay + t.poff);
  const uint32_t mask = (1u << w) - 1u;
  uint64_t acc = 0;
  int nb = 0, wi = 0;
  int32_t P = 0;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    if (nb < static_cast<int>(w)) {
      acc = (acc << 32) | bswap32(pw[wi++]);
      nb += 32;
    }
    nb -= w;
    const int32_t mag = static_cast<int32_t>(static_cast<uint32_t>(acc >> nb) & mask);
    if (i > 0 && i < t.len) P += ((sw >> (31 - i)) & 1u) ? -mag : mag;
    emit(i, P);
  }
}

// Decode lane's bin of one block (fallback: warp per block, lane per
// element, exact for widths up to 64).  Bins = O + inclusive prefix of signed
// residuals (slot 0 is ignored, codec.py:241 / 256-258); flags a prefix
// beyond +-(2^63 - 1) (codec.py:259-260).
__device__ __forceinline__ int64_t decode_lane(const unsigned char* sgn, const unsigned char* pay,
                                               uint32_t w, int64_t o, uint64_t soff,
                                               uint64_t poff, int len, int lane, uint32_t* flags) {
  if (w == 0) return o;
  const uint32_t sw = bswap32(*reinterpret_cast<const uint32_t*>(sgn + soff));
  const bool neg = (__brev(sw) >> lane) & 1u;
  const uint32_t* pw = reinterpret_cast<const uint32_t*>(pay + poff);
  const uint32_t start = lane * w;
  const uint32_t a = start >> 5, sh = start & 31;
  const bool live = lane > 0 && lane < len;
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

// fallback helper: broadcast block j's metadata (held by lane j) to the warp
struct LaneBlock {
  uint32_t w;
  int64_t o;
  uint64_t soff, poff;
  int len;
};
__device__ __forceinline__ LaneBlock lane_block(const TileIn& t, int j) {
  LaneBlock r;
  r.w = __shfl_sync(kFull, t.w, j);
  r.o = __shfl_sync(kFull, t.o, j);
  r.soff = __shfl_sync(kFull, t.soff, j);
  r.poff = __shfl_sync(kFull, t.poff, j);
  r.len = __shfl_sync(kFull, t.len, j);
  return r;
}

// ---------------------------------------------------------------------------
// bin sources of the encoder
//
//   stage(tile, sm, bar, s_tmp, flags)  -- all threads: stage the tile input
//   rows(rows, flags) -> bool            -- quantize/decode into registers; if
//        the whole tile fits the fast path, write int32 bin rows in place
//        (padded, see pad) and return true.  CTA-uniform.
//   lane_bin(lb, lane, len, flags)       -- fallback: lane's bin of tile block lb

template <typename T>
struct SrcQuant {
  const T* x;
  uint64_t n;
  QuantConst c;
  uint64_t tile;
  const T* xs;   // staged tile
  static constexpr uint32_t kStageBytes = kTileElems * sizeof(T);
  static constexpr int kMinBlocks = 8;   // <= 64 registers

  __device__ __forceinline__ void stage(uint64_t t, unsigned char* sm, uint64_t* bar, uint32_t*,
                                        uint32_t*) {
    tile = t;
    xs = reinterpret_cast<const T*>(sm);
    stage_elems(reinterpret_cast<T*>(sm), x, t * kTileElems, n, bar);
  }
  // element-parallel quantize straight into the (separate) bin rows; the
  // staged input stays intact for the fallback
  __device__ __forceinline__ bool rows(int32_t* rows, uint32_t* flags) {
    const uint64_t e0 = tile * kTileElems;
    const uint32_t cnt = static_cast<uint32_t>((n - e0 < (uint64_t)kTileElems) ? (n - e0) : kTileElems);
    bool ok = true;
    const int base = pad_sweep_base();
    if (cnt == kTileElems) {
      // full tile: groups of 4 elements, one vote per group
#pragma unroll 1
      for (int j0 = 0; j0 < K; j0 += 4) {
        int32_t v[4];
        double xd[4];
        unsigned bad = 0;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          xd[jj] = static_cast<double>(xs[(j0 + jj) * kThreads + threadIdx.x]);
          bad |= quantize_fast(xd[jj], c, &v[jj]) ? 0u : (1u << jj);
        }
        if (__any_sync(kFull, bad != 0)) {   // rare: near a bin edge or out of range
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            if (bad & (1u << jj)) {
              const int64_t q = quantize1(xd[jj], c, flags);
              ok &= (q > -kWideLimit) & (q < kWideLimit);
              v[jj] = static_cast<int32_t>(q);
            }
          }
        }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) rows[base + (j0 + jj) * kSweepStride] = v[jj];
      }
    } else {
      for (int j = 0; j < K; ++j) {
        const uint32_t e = j * kThreads + threadIdx.x;
        int32_t v = 0;
        if (e < cnt) {
          const int64_t q = quantize1(static_cast<double>(xs[e]), c, flags);
          ok &= (q > -kWideLimit) & (q < kWideLimit);
          v = static_cast<int32_t>(q);
        }
        rows[base + j * kSweepStride] = v;
      }
    }
    return __syncthreads_and(ok) != 0;
  }
  __device__ __forceinline__ int64_t lane_bin(int lb, int lane, int len, uint32_t* flags) {
    if (lane >= len) return 0;
    return quantize1(static_cast<double>(xs[lb * K + lane]), c, flags);
  }
};

struct SrcBins {
  const int64_t* bins;
  uint64_t n;
  uint64_t tile;
  const int64_t* bs;
  static constexpr uint32_t kStageBytes = kTileElems * 8;
  static constexpr int kMinBlocks = 6;

  __device__ __forceinline__ void stage(uint64_t t, unsigned char* sm, uint64_t* bar, uint32_t*,
                                        uint32_t*) {
    tile = t;
    bs = reinterpret_cast<const int64_t*>(sm);
    stage_elems(reinterpret_cast<int64_t*>(sm), bins, t * kTileElems, n, bar);
  }
  __device__ __forceinline__ bool rows(int32_t* rows, uint32_t* flags) {
    const uint64_t e0 = tile * kTileElems;
    const uint32_t cnt = static_cast<uint32_t>((n - e0 < (uint64_t)kTileElems) ? (n - e0) : kTileElems);
    bool ok = true;
    const int base = pad_sweep_base();
#pragma unroll 8
    for (int j = 0; j < K; ++j) {
      const uint32_t e = j * kThreads + threadIdx.x;
      int32_t v = 0;
      if (e < cnt) {
        const int64_t q = bs[e];
        ok &= (q > -kWideLimit) & (q < kWideLimit);
        v = static_cast<int32_t>(q);
      }
      rows[base + j * kSweepStride] = v;
    }
    return __syncthreads_and(ok) != 0;
  }
  __device__ __forceinline__ int64_t lane_bin(int lb, int lane, int len, uint32_t* flags) {
    if (lane >= len) return 0;
    const int64_t v = bs[lb * K + lane];
    if (v == INT64_MIN) *flags |= HSZ_ERR_RESCALE_OVERFLOW;   // QuantArray guard model.py:124-128
    return v;
  }
};

// scalar multiply: decode the input stream tile, rescale (ops.py:199-225)
struct SrcSmul {
  StreamIn in;
  int64_t rs;
  double d;
  TileIn t;
  static constexpr uint32_t kStageBytes = kStageFast;
  static constexpr int kMinBlocks = 4;

  __device__ __forceinline__ void stage(uint64_t tile, unsigned char* sm, uint64_t* bar,
                                        uint32_t* s_tmp, uint32_t* flags) {
    stage_tile_in(in, tile, sm, bar, s_tmp, &t, flags);
  }
  __device__ __forceinline__ bool rows(int32_t* rows, uint32_t* flags) {
    if (!t.fast) return false;      // CTA-uniform
    bool ok = true;
    const int64_t o = t.o;
    uint32_t f = 0;
    int32_t* row = rows + threadIdx.x * kRow;
    decode_row_fast(t, [&](int i, int32_t P) {
      const int64_t v = rescale1(product_rn(o + P, rs), d, &f);
      ok &= (v > -kWideLimit) & (v < kWideLimit);
      row[i] = static_cast<int32_t>(v);
    });
    *flags |= f;
    return __syncthreads_and(ok) != 0;
  }
  __device__ __forceinline__ int64_t lane_bin(int lb, int lane, int len, uint32_t* flags) {
    const LaneBlock m = lane_block(t, lb & (BPW - 1));
    uint32_t f = 0;
    const int64_t q = decode_lane(t.sgn, t.pay, m.w, m.o, m.soff, m.poff, len, lane, &f);
    *flags |= f;
    if (f || lane >= len) return 0;
    return rescale1(product_rn(q, rs), d, flags);
  }
};

// ---------------------------------------------------------------------------
// packing of one block's residual magnitudes (fallback path, lane per element)

// w <= 32: segmented doubling OR-reduce of the word each field starts in;
// the lane straddling into the next word hands its low part over.
__device__ __forceinline__ void pack_narrow(uint32_t* dst, uint32_t mag, int w, int lane) {
  const uint32_t start = lane * w;
  const uint32_t a = start >> 5, o = start & 31;
  const uint32_t top = (w == 32) ? mag : (mag << (32 - w));
  uint32_t hi = top >> o;
  const uint32_t lo = (o + w > 32) ? (top << (32 - o)) : 0u;
  const uint32_t rem = 32 - o;
  for (uint32_t d = 1, dw = w; dw < 32; d <<= 1, dw <<= 1) {
    const uint32_t v = __shfl_down_sync(kFull, hi, d);
    if (dw < rem && lane + d < 32) hi |= v;
  }
  const uint32_t carry = __shfl_up_sync(kFull, lo, 1);
  if (o < static_cast<uint32_t>(w)) {
    const uint32_t word = hi | (lane ? carry : 0u);
    if (a < static_cast<uint32_t>(w)) dst[a] = bswap32(word);
  }
}

// 32 < w <= 64: up to three words per field; zero then OR in shared memory
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
  // [staged input | int32 bin rows | packed sign words | fallback scratch];
  // once the rows are built the fast path packs payload words over the
  // staged input (<= 31 words per block fits the 16 KB f32 stage)
  static constexpr uint32_t kStage = ((Src::kStageBytes > TB * 31 * 4 ? Src::kStageBytes : TB * 31 * 4) + 15) & ~15u;
  static constexpr uint32_t kRows = TB * kRow * 4;
  static constexpr uint32_t kSign = TB * 4;
  static constexpr uint32_t kScratch = kCtaWarps * 64 * 4;   // fallback: one block's words per warp
  static constexpr uint32_t kBytes = kStage + kRows + kSign + kScratch;
};

template <class Src>
__global__ void __launch_bounds__(kThreads, Src::kMinBlocks) encode_kernel(Src src, EncodeOut out,
                                                          uint64_t nblocks, uint64_t ntiles,
                                                          uint32_t tail_len) {
  extern __shared__ __align__(16) unsigned char sm[];
  using L = EncodeSmem<Src>;
  uint32_t* words = reinterpret_cast<uint32_t*>(sm);          // packed payload (fast path)
  int32_t* rows = reinterpret_cast<int32_t*>(sm + L::kStage);
  uint32_t* sm_sign = reinterpret_cast<uint32_t*>(sm + L::kStage + L::kRows);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(sm + L::kStage + L::kRows + L::kSign);
  __shared__ uint64_t s_bar;
  __shared__ uint64_t s_tile, s_epoch, s_excl_s, s_excl_p;
  __shared__ uint32_t s_tmp[8];
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
  src.stage(tile, sm, &s_bar, s_tmp, &flags);
  const bool fast = src.rows(rows, &flags);        // CTA-uniform

  uint32_t tile_s = 0, tile_p = 0;                 // fast path: tile section bytes
  if (fast) {
    // ---- thread-per-block: residuals, width, sign word ------------------
    const int b = threadIdx.x;
    const uint64_t gb = tile * TB + b;
    const bool active = gb < nblocks;
    const int len = active ? ((gb == nblocks - 1) ? static_cast<int>(tail_len) : K) : 0;
    const int32_t* row = rows + b * kRow;
    uint32_t mx = 0, sbits = 0;
    const int32_t first = row[0];
    {
      int32_t prev = first;
#pragma unroll
      for (int i = 1; i < K; ++i) {
        const int32_t q = row[i];
        const int32_t dlt = q - prev;      // |q| < 2^30: no overflow
        prev = q;
        const bool live = i < len;
        mx |= live ? static_cast<uint32_t>(dlt < 0 ? -dlt : dlt) : 0u;   // bit length of OR == of max
        sbits |= (live && dlt < 0) ? (1u << (31 - i)) : 0u;
      }
    }
    const uint32_t w = mx ? 32 - __clz(mx) : 0;
    const uint32_t sb = (active && w) ? (len + 7) >> 3 : 0;
    const uint32_t pb = active ? (len * w + 7) >> 3 : 0;
    uint32_t es, ep;
    scan2(sb, pb, &es, &ep, &tile_s, &tile_p, s_tmp);
    // publish the tile aggregate now; successors can start summing it while
    // this CTA packs
    if (threadIdx.x == 0) publish_aggregate(lw, tile, s_epoch, tile_s, tile_p);
    if (w) {
      // second walk: MSB-first w-bit fields through a 64-bit shift register,
      // packed over the (consumed) staged input
      sm_sign[es >> 2] = bswap32(sbits);
      uint32_t* dst = words + (ep >> 2);
      uint64_t acc = 0;
      int nb = w, wi = 0;                  // slot 0: a zero field
      int32_t prev = first;
#pragma unroll
      for (int i = 1; i < K; ++i) {
        const int32_t q = row[i];
        const int32_t dlt = q - prev;
        prev = q;
        const uint32_t m = (i < len) ? static_cast<uint32_t>(dlt < 0 ? -dlt : dlt) : 0u;
        acc = (acc << w) | m;
        nb += w;
        if (nb >= 32) {
          nb -= 32;
          dst[wi++] = bswap32(static_cast<uint32_t>(acc >> nb));
        }
      }
      if (nb > 0) dst[wi] = bswap32(static_cast<uint32_t>(acc << (32 - nb)));   // tail block only
    }
    if (active) {
      out.widths[gb] = static_cast<uint8_t>(w);
      out.outliers[gb] = first;
    }
  } else {
    // ---- fallback pass 1: one warp per block, sizes only -----------------
    const uint64_t blk0 = tile * TB + warp * BPW;
    uint32_t sbytes = 0, pbytes = 0, my_w = 0;
    int64_t my_o = 0;
    for (int j = 0; j < BPW; ++j) {
      const uint64_t b = blk0 + j;
      if (b >= nblocks) break;
      const int len = (b == nblocks - 1) ? static_cast<int>(tail_len) : K;
      const int64_t q = src.lane_bin(warp * BPW + j, lane, len, &flags);
      const int64_t first = __shfl_sync(kFull, q, 0);
      const int64_t prev = __shfl_up_sync(kFull, q, 1);
      bool neg = false;
      uint64_t mag = 0;
      if (lane > 0 && lane < len) mag = absdiff64(q, prev, &neg);
      const int wl = mag ? 64 - __clzll(static_cast<long long>(mag)) : 0;
      const int w = __reduce_max_sync(kFull, wl);
      if (lane == j) {
        my_w = w;
        my_o = first;
      }
      if (w) sbytes += (len + 7) >> 3;
      pbytes += (len * w + 7) >> 3;
    }
    if (blk0 + lane < nblocks) {
      out.widths[blk0 + lane] = static_cast<uint8_t>(my_w);
      if (my_o < INT32_MIN || my_o > INT32_MAX) flags |= HSZ_ERR_OUTLIER_OVERFLOW;
      out.outliers[blk0 + lane] = static_cast<int32_t>(my_o);
    }
    if (lane == 0) {
      s_wsb[warp] = sbytes;
      s_wpb[warp] = pbytes;
    }
  }
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(&s_err, flags);
  __syncthreads();

  if (warp == 0) {
    uint64_t agg_s = tile_s, agg_p = tile_p;
    if (!fast) {
      agg_s = __reduce_add_sync(kFull, lane < kCtaWarps ? s_wsb[lane] : 0u);
      agg_p = __reduce_add_sync(kFull, lane < kCtaWarps ? s_wpb[lane] : 0u);
    }
    uint64_t es, ep;
    if (fast) {
      resolve_prefix(lw, tile, s_epoch, agg_s, agg_p, &es, &ep);
    } else {
      lookback(lw, tile, s_epoch, agg_s, agg_p, &es, &ep);
    }
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

  if (fast) {
    // ---- stream the packed tile out (coalesced; 16-byte when aligned) ---
    const uint64_t gs = s_excl_s, gp = s_excl_p;
    uint32_t* dsg = reinterpret_cast<uint32_t*>(out.signs + gs);
    const uint32_t nsw = (tile_s + 3) >> 2, npw = (tile_p + 3) >> 2;
    for (uint32_t i = threadIdx.x; i < nsw; i += kThreads) dsg[i] = sm_sign[i];
    uint32_t* dpy = reinterpret_cast<uint32_t*>(out.payload + gp);
    uint32_t head = 0;
    if ((gp & 15) == 0) {
      const uint32_t nv = npw >> 2;
      uint4* dv = reinterpret_cast<uint4*>(dpy);
      const uint4* sv = reinterpret_cast<const uint4*>(words);
      for (uint32_t i = threadIdx.x; i < nv; i += kThreads) dv[i] = sv[i];
      head = nv << 2;
    }
    for (uint32_t i = head + threadIdx.x; i < npw; i += kThreads) dpy[i] = words[i];
    return;
  }
  // ---- fallback pass 2: recompute each block, pack, write at its offset --
  uint64_t gs = s_excl_s, gp = s_excl_p;
  for (int i = 0; i < warp; ++i) {
    gs += s_wsb[i];
    gp += s_wpb[i];
  }
  uint32_t* wscr = scratch + warp * 64;
  const uint64_t blk0 = tile * TB + warp * BPW;
  for (int j = 0; j < BPW; ++j) {
    const uint64_t b = blk0 + j;
    if (b >= nblocks) break;
    const int len = (b == nblocks - 1) ? static_cast<int>(tail_len) : K;
    uint32_t f = 0;
    const int64_t q = src.lane_bin(warp * BPW + j, lane, len, &f);
    const int64_t prev = __shfl_up_sync(kFull, q, 1);
    bool neg = false;
    uint64_t mag = 0;
    if (lane > 0 && lane < len) mag = absdiff64(q, prev, &neg);
    const unsigned sbits = __ballot_sync(kFull, neg);
    const int wl = mag ? 64 - __clzll(static_cast<long long>(mag)) : 0;
    const int w = __reduce_max_sync(kFull, wl);
    if (w == 0) continue;
    if (lane == 0) *reinterpret_cast<uint32_t*>(out.signs + gs) = bswap32(__brev(sbits));
    gs += (len + 7) >> 3;
    if (w <= 32) {
      pack_narrow(wscr, static_cast<uint32_t>(mag), w, lane);
    } else {
      pack_wide(wscr, mag, w, lane);
    }
    __syncwarp();
    const int nw = (len * w + 31) >> 5;
    uint32_t* dpy = reinterpret_cast<uint32_t*>(out.payload + gp);
    for (int t = lane; t < nw; t += 32) dpy[t] = wscr[t];
    __syncwarp();
    gp += (len * w + 7) >> 3;
  }
}

// ---------------------------------------------------------------------------
// decode kernels (grid = tiles, offsets from the cache, no look-back)

struct SinkF32 {
  float* out;
  double d;
  bool may_overflow;   // d * 2^33 can exceed FLT_MAX (host-computed)
  using T = float;
  static constexpr int kMinBlocks = 8;
  __device__ __forceinline__ float value(int64_t bin, uint32_t* flags) const {
    const float v = __double2float_rn(grid1(bin, d));
    if (!isfinite(v)) *flags |= HSZ_ERR_OUTPUT_NONFINITE;
    return v;
  }
  // fast path: bin = o + P, exact as a double (|o|, |P| < 2^31)
  __device__ __forceinline__ float value2(double od, int32_t P, uint32_t* flags) const {
    const float v = __double2float_rn(__dmul_rn(d, __dadd_rn(od, i32_to_double(P))));
    if (may_overflow && !isfinite(v)) *flags |= HSZ_ERR_OUTPUT_NONFINITE;
    return v;
  }
  __device__ __forceinline__ void put(uint64_t e, int64_t bin, uint32_t* flags) const {
    out[e] = value(bin, flags);
  }
  __device__ __forceinline__ T* base() const { return out; }
};
struct SinkF64 {
  double* out;
  double d;
  bool may_overflow;
  using T = double;
  static constexpr int kMinBlocks = 4;
  __device__ __forceinline__ double value(int64_t bin, uint32_t* flags) const {
    const double v = grid1(bin, d);
    if (!isfinite(v)) *flags |= HSZ_ERR_OUTPUT_NONFINITE;
    return v;
  }
  __device__ __forceinline__ double value2(double od, int32_t P, uint32_t* flags) const {
    const double v = __dmul_rn(d, __dadd_rn(od, i32_to_double(P)));
    if (may_overflow && !isfinite(v)) *flags |= HSZ_ERR_OUTPUT_NONFINITE;
    return v;
  }
  __device__ __forceinline__ void put(uint64_t e, int64_t bin, uint32_t* flags) const {
    out[e] = value(bin, flags);
  }
  __device__ __forceinline__ T* base() const { return out; }
};
struct SinkBins {
  int64_t* out;
  using T = int64_t;
  static constexpr int kMinBlocks = 4;
  __device__ __forceinline__ int64_t value(int64_t bin, uint32_t*) const { return bin; }
  __device__ __forceinline__ void put(uint64_t e, int64_t bin, uint32_t*) const { out[e] = bin; }
  __device__ __forceinline__ T* base() const { return out; }
};

template <class Sink>
struct DecodeSmem {
  static constexpr uint32_t kOut = TB * kRow * sizeof(typename Sink::T);
  static constexpr uint32_t kBytes = kStageFast > kOut ? kStageFast : kOut;
};

template <class Sink>
__global__ void __launch_bounds__(kThreads, Sink::kMinBlocks) decode_kernel(StreamIn s, Sink sink, uint32_t* err) {
  extern __shared__ __align__(16) unsigned char sm[];
  using T = typename Sink::T;
  __shared__ uint64_t s_bar;
  __shared__ uint32_t s_tmp[8];
  T* ot = reinterpret_cast<T*>(sm);     // output tile, written over the staged input
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t tile = blockIdx.x;
  uint32_t flags = 0;
  TileIn t;
  stage_tile_in(s, tile, sm, &s_bar, s_tmp, &t, &flags);
  if (t.fast) {
    T v[K];
    if constexpr (std::is_same<T, int64_t>::value) {
      const int64_t o = t.o;
      decode_row_fast(t, [&](int i, int32_t P) { v[i] = o + P; });
    } else {
      const double od = static_cast<double>(t.o);
      decode_row_fast(t, [&](int i, int32_t P) { v[i] = sink.value2(od, P, &flags); });
    }
    __syncthreads();                    // the staged bytes are consumed
#pragma unroll
    for (int i = 0; i < K; ++i) ot[pad(threadIdx.x, i)] = v[i];
  } else {
    for (int j = 0; j < BPW; ++j) {
      const int lb = warp * BPW + j;
      const LaneBlock m = lane_block(t, j);
      if (m.len == 0) break;
      const int64_t q = decode_lane(t.sgn, t.pay, m.w, m.o, m.soff, m.poff, m.len, lane, &flags);
      ot[pad(lb, lane)] = sink.value(q, &flags);
    }
  }
  __syncthreads();
  // coalesced store of the tile
  const uint64_t e0 = tile * kTileElems;
  const uint64_t cnt = (s.n - e0 < (uint64_t)kTileElems) ? (s.n - e0) : (uint64_t)kTileElems;
  T* g = sink.base() + e0;
  const int base = pad_sweep_base();
  if (cnt == kTileElems) {
#pragma unroll 8
    for (int j = 0; j < K; ++j) g[j * kThreads + threadIdx.x] = ot[base + j * kSweepStride];
  } else {
    for (int j = 0; j < K; ++j) {
      const uint32_t e = j * kThreads + threadIdx.x;
      if (e < cnt) g[e] = ot[base + j * kSweepStride];
    }
  }
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(err, flags);
}

// exact moments: per thread S (int128) and Q (unsigned 192-bit)
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

// Partials live in the workspace "vals" area: 6 u64 per CTA.  The last CTA
// to finish (done counter) reduces them and writes out[5].
__device__ __forceinline__ void finish_moments(Acc acc, uint64_t ntiles, void* ws,
                                               uint64_t* out) {
  __shared__ Acc s_acc[32];
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int m = 16; m > 0; m >>= 1) acc.merge(shfl_xor_acc(acc, m));
  if (lane == 0) s_acc[warp] = acc;
  __syncthreads();
  uint64_t* base = static_cast<uint64_t*>(ws);
  uint64_t* done = base + 2;
  uint64_t* part = base + kWsFlagsOff + ntiles;   // vals area
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
  __shared__ uint32_t s_tmp[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t tile = blockIdx.x;
  uint32_t flags = 0;
  TileIn t;
  stage_tile_in(s, tile, sm, &s_bar, s_tmp, &t, &flags);
  Acc acc;
  acc.s = 0;
  acc.q = 0;
  acc.q2 = 0;
  if (t.fast) {
    // block: S_b = len*O + sum P_i ; Q_b = len*O^2 + 2*O*sum P_i + sum P_i^2
    int64_t sp = 0;       // |sum P| < 32 * 2^31
    uint64_t sp2 = 0;     // sum P^2 < 32 * 2^62: 67 bits, carry kept in sp2_hi
    uint64_t sp2_hi = 0;
    const int len = t.len;
    decode_row_fast(t, [&](int i, int32_t P) {
      if (i < len) {
        sp += P;
        if (kWantSq) {
          const uint64_t p2 = static_cast<uint64_t>(static_cast<int64_t>(P) * P);
          const uint64_t n2 = sp2 + p2;
          sp2_hi += n2 < sp2 ? 1u : 0u;
          sp2 = n2;
        }
      }
    });
    const __int128 o = t.o;
    acc.s = o * len + sp;
    if (kWantSq) {
      const unsigned __int128 psq = (static_cast<unsigned __int128>(sp2_hi) << 64) | sp2;
      const __int128 tot = o * o * len + 2 * o * sp + static_cast<__int128>(psq);  // = sum bin^2 >= 0
      acc.q = static_cast<unsigned __int128>(tot);
    }
  } else {
    for (int j = 0; j < BPW; ++j) {
      const LaneBlock m = lane_block(t, j);
      if (m.len == 0) break;
      const int64_t q = decode_lane(t.sgn, t.pay, m.w, m.o, m.soff, m.poff, m.len, lane, &flags);
      if (lane < m.len) acc.add(q, kWantSq);
    }
  }
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(err, flags);
  (void)warp;
  finish_moments(acc, gridDim.x, ws, out);
}

}  // namespace k32
}  // namespace hsz
