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
  grp_sync();
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
  uint32_t sh[8];   // PRMT sign replication: element i's sign from sh[i % 8]
#pragma unroll
  for (int k = 0; k < 8; ++k) sh[k] = sw << k;
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
    const int32_t neg = static_cast<int32_t>(prmt_sign(sh[i & 7], 3 - (i >> 3)));
    if (i > 0 && i < t.len) P += (mag ^ neg) - neg;
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

// the lane's signed residual (lane 0: the outlier; 0 past len) without the
// prefix sum -- the residual-domain element-wise ops combine streams here
// (ops.py:163-182), so operands whose BINS would leave int64 (widths 62-64)
// are combined exactly, like the reference's Python-int path
__device__ __forceinline__ __int128 decode_lane_resid(const unsigned char* sgn,
                                                      const unsigned char* pay, uint32_t w,
                                                      int64_t o, uint64_t soff, uint64_t poff,
                                                      int len, int lane) {
  if (lane == 0) return o;
  if (w == 0 || lane >= len) return 0;
  const uint32_t sw = bswap32(*reinterpret_cast<const uint32_t*>(sgn + soff));
  const bool neg = (__brev(sw) >> lane) & 1u;
  const uint32_t* pw = reinterpret_cast<const uint32_t*>(pay + poff);
  const uint32_t start = lane * w;
  const uint32_t a = start >> 5, sh = start & 31;
  const uint32_t w0 = bswap32(pw[a]);
  const uint32_t w1 = bswap32(pw[a + 1]);
  const uint32_t w2 = (sh + w > 64) ? bswap32(pw[a + 2]) : 0u;
  const unsigned __int128 cat = (static_cast<unsigned __int128>(w0) << 64) |
                                (static_cast<unsigned __int128>(w1) << 32) | w2;
  const uint64_t mag = static_cast<uint64_t>((cat << (32 + sh)) >> (128 - w));
  return neg ? -static_cast<__int128>(mag) : static_cast<__int128>(mag);
}

// sources that deliver residuals (lane_resid) instead of bins (lane_bin)
template <class S, class = void>
struct ResidSrc : std::false_type {};
template <class S>
struct ResidSrc<S, std::void_t<decltype(S::kResid)>> : std::bool_constant<S::kResid> {};

// (first = outlier of the block, neg / mag = this lane's residual) from a
// source of either kind; residual magnitudes of 2^64 or more are flagged
template <class Src>
__device__ __forceinline__ void lane_code(Src& src, int lb, int lane, int len, uint32_t* flags,
                                          int64_t* first, bool* neg, uint64_t* mag) {
  if constexpr (ResidSrc<Src>::value) {
    const __int128 r = src.lane_resid(lb, lane, len, flags);
    const uint64_t lo = static_cast<uint64_t>(r);
    *first = static_cast<int64_t>(__shfl_sync(kFull, lo, 0));
    *neg = false;
    *mag = 0;
    if (lane > 0 && lane < len) {
      *neg = r < 0;
      const unsigned __int128 u = *neg ? static_cast<unsigned __int128>(-r)
                                       : static_cast<unsigned __int128>(r);
      if (u >> 64) *flags |= HSZ_ERR_PREFIX_OVERFLOW;   // beyond the 64-bit field width
      *mag = static_cast<uint64_t>(u);
    }
  } else {
    const int64_t q = src.lane_bin(lb, lane, len, flags);
    *first = __shfl_sync(kFull, q, 0);
    const int64_t prev = __shfl_up_sync(kFull, q, 1);
    *neg = false;
    *mag = 0;
    if (lane > 0 && lane < len) *mag = absdiff64(q, prev, neg);
  }
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
// staging with a reusable mbarrier (persistent CTAs): thread 0 issues TMA bulk
// copies and arms the barrier; everybody waits on the current phase parity.

struct Stager {
  uint64_t* bar;
  uint32_t phase;   // parity of the next completion (flips on every bulk use)
  bool bulk;        // the current tile was staged with a bulk copy
  __device__ __forceinline__ void init(uint64_t* b) {
    bar = b;
    phase = 0;
    bulk = false;
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
    }
  }
  // thread 0: make prior generic-proxy accesses of the buffer visible before
  // the async proxy overwrites it, then arm + issue
  __device__ __forceinline__ void arm(uint32_t bytes) const {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(bar, bytes);
  }
  __device__ __forceinline__ void wait() {
    if (bulk) {
      mbar_wait_parity(bar, phase);
      phase ^= 1u;
    }
  }
};

// ---------------------------------------------------------------------------
// bin sources of the encoder (all calls are CTA-uniform)
//
//   issue(tile, stage, st, s_tmp, flags) -- start staging `tile` (async when
//                                           possible; the stage buffer is free)
//   rows(stage, st, rows, flags) -> bool  -- wait for the staged tile, build the
//        int32 bin rows (padded, see pad) and report whether the whole tile is
//        on the fast path
//   lane_bin(lb, lane, len, flags)        -- fallback: lane's exact bin of tile
//        block lb, read from global memory (the stage may be reused)

template <typename T>
struct SrcQuant {
  const T* x;
  uint64_t n;
  QuantConst c;
  uint64_t tile;
  static constexpr uint32_t kStageBytes = kTileElems * sizeof(T);
  static constexpr int kMinBlocks = 4;

  __device__ __forceinline__ void issue(uint64_t t, unsigned char* stage, Stager& st, uint32_t*,
                                        uint32_t*) {
    tile = t;
    const uint64_t e0 = t * kTileElems;
    const uint64_t cnt = (n - e0 < (uint64_t)kTileElems) ? (n - e0) : (uint64_t)kTileElems;
    st.bulk = cnt == (uint64_t)kTileElems && (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
    if (st.bulk) {
      if (threadIdx.x == 0) {
        st.arm(kStageBytes);
        bulk_g2s(stage, x + e0, kStageBytes, st.bar);
      }
    } else {
      T* d = reinterpret_cast<T*>(stage);
      for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) d[i] = x[e0 + i];
      grp_sync();
    }
  }
  __device__ __forceinline__ bool rows(const unsigned char* stage, Stager& st, int32_t* rows,
                                       uint32_t* flags) {
    st.wait();
    const T* xs = reinterpret_cast<const T*>(stage);
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
    return grp_and(ok);
  }
  __device__ __forceinline__ int64_t lane_bin(int lb, int lane, int len, uint32_t* flags) {
    if (lane >= len) return 0;
    return quantize1(static_cast<double>(x[tile * kTileElems + lb * K + lane]), c, flags);
  }
};

struct SrcBins {
  const int64_t* bins;
  uint64_t n;
  uint64_t tile;
  static constexpr uint32_t kStageBytes = kTileElems * 8;
  static constexpr int kMinBlocks = 4;

  __device__ __forceinline__ void issue(uint64_t t, unsigned char* stage, Stager& st, uint32_t*,
                                        uint32_t*) {
    tile = t;
    const uint64_t e0 = t * kTileElems;
    const uint64_t cnt = (n - e0 < (uint64_t)kTileElems) ? (n - e0) : (uint64_t)kTileElems;
    st.bulk = cnt == (uint64_t)kTileElems && (reinterpret_cast<uintptr_t>(bins) & 15u) == 0;
    if (st.bulk) {
      if (threadIdx.x == 0) {
        st.arm(kStageBytes);
        bulk_g2s(stage, bins + e0, kStageBytes, st.bar);
      }
    } else {
      int64_t* d = reinterpret_cast<int64_t*>(stage);
      for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) d[i] = bins[e0 + i];
      grp_sync();
    }
  }
  __device__ __forceinline__ bool rows(const unsigned char* stage, Stager& st, int32_t* rows,
                                       uint32_t*) {
    st.wait();
    const int64_t* bs = reinterpret_cast<const int64_t*>(stage);
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
    return grp_and(ok);
  }
  __device__ __forceinline__ int64_t lane_bin(int lb, int lane, int len, uint32_t* flags) {
    if (lane >= len) return 0;
    const int64_t v = bins[tile * kTileElems + lb * K + lane];
    if (v == INT64_MIN) *flags |= HSZ_ERR_RESCALE_OVERFLOW;   // QuantArray guard model.py:124-128
    return v;
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

// Fallback encoder (a tile with a bin beyond 2^30, or a stream tile wider than
// 26 bits): one warp per block, exact 64-bit residuals, widths up to 64.
// Pass 1 computes sizes (and writes widths / outliers); after the look-back,
// pass 2 recomputes each block and writes it at its final offset.  Out of
// line so that the fast path's register budget is not set by it.
template <class Src>
__device__ __noinline__ uint32_t fallback_sizes(Src src, EncodeOut out, uint64_t tile,
                                                 uint64_t nblocks, uint32_t tail_len,
                                                 uint32_t* s_wsb, uint32_t* s_wpb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t flags = 0;
  const uint64_t blk0 = tile * TB + warp * BPW;
  uint32_t sbytes = 0, pbytes = 0, my_w = 0;
  int64_t my_o = 0;
  for (int j = 0; j < BPW; ++j) {
    const uint64_t b = blk0 + j;
    if (b >= nblocks) break;
    const int len = (b == nblocks - 1) ? static_cast<int>(tail_len) : K;
    int64_t first;
    bool neg;
    uint64_t mag;
    lane_code(src, warp * BPW + j, lane, len, &flags, &first, &neg, &mag);
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
  return flags;
}

template <class Src>
__device__ __noinline__ void fallback_pack(Src src, EncodeOut out, uint64_t tile,
                                           uint64_t nblocks, uint32_t tail_len, uint64_t gs,
                                           uint64_t gp, uint32_t* wscr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t blk0 = tile * TB + warp * BPW;
  for (int j = 0; j < BPW; ++j) {
    const uint64_t b = blk0 + j;
    if (b >= nblocks) break;
    const int len = (b == nblocks - 1) ? static_cast<int>(tail_len) : K;
    uint32_t f = 0;
    int64_t first;
    bool neg;
    uint64_t mag;
    lane_code(src, warp * BPW + j, lane, len, &f, &first, &neg, &mag);
    (void)first;
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

template <class Src>
struct EncodeSmem {
  // [staged input | int32 bin rows | 2 x (packed payload | sign words) | fallback scratch]
  static constexpr uint32_t kStage = (Src::kStageBytes + 15) & ~15u;
  static constexpr uint32_t kRows = TB * kRow * 4;
  static constexpr uint32_t kPackedCap = 8192;              // payload bytes per staged tile
  static constexpr uint32_t kBuf = kPackedCap + TB * 4;     // + sign words
  static constexpr uint32_t kScratch = kCtaWarps * 64 * 4;  // fallback: one block per warp
  static constexpr uint32_t kBytes = kStage + kRows + 2 * kBuf + kScratch;
};

// Persistent, warp-specialised single-pass encoder.  A CTA = 4 compute warps
// (one thread per block of a 128-block tile) + 1 store warp.  Compute warps
// loop over tiles drawn from the ticket counter (always one ticket ahead):
//   rows(t) [TMA-staged input, prefetched during the previous iteration]
//   -> issue the TMA prefetch of the next tile into the freed stage
//   -> widths / outliers / sizes of t, CTA scan, publish t's aggregate
//   -> pack t into one of two staging buffers and hand it to the store warp.
// The store warp resolves each handed-over tile's look-back prefix and
// streams its sections out (16-byte stores), then releases the buffer -- the
// look-back latency overlaps the next tile's compute.  Tiles whose packed
// payload exceeds a staging buffer, and exact-path (fallback) tiles, are
// resolved and written by the compute warps themselves.
constexpr int kEncThreads = kThreads + 32;

template <class Src>
__global__ void __launch_bounds__(kEncThreads, Src::kMinBlocks) encode_kernel(Src src, EncodeOut out,
                                                                              uint64_t nblocks,
                                                                              uint64_t ntiles,
                                                                              uint32_t tail_len) {
  extern __shared__ __align__(16) unsigned char sm[];
  using L = EncodeSmem<Src>;
  unsigned char* stage = sm;
  int32_t* rows = reinterpret_cast<int32_t*>(sm + L::kStage);
  unsigned char* bufs = sm + L::kStage + L::kRows;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(sm + L::kStage + L::kRows + 2 * L::kBuf);
  __shared__ uint64_t s_bar, s_full[2], s_empty[2];
  __shared__ uint64_t s_next, s_epoch, s_excl_s, s_excl_p;
  __shared__ uint64_t s_hand_tile[2];           // handed-over tile (~0 = stop)
  __shared__ uint32_t s_hand_s[2], s_hand_p[2];
  __shared__ uint32_t s_tmp[8];
  __shared__ uint32_t s_wsb[kCtaWarps], s_wpb[kCtaWarps];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  LookbackWs lw = LookbackWs::bind(out.ws, ntiles);
  const uint64_t last_draw = ntiles + gridDim.x - 1;   // every CTA draws once past the end
  Stager st;
  st.init(&s_bar);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 1);
    }
    fence_mbar_init();
    const uint64_t e = ld_acquire(lw.epoch);
    const uint64_t t = atom_add_acq_rel(lw.ticket, 1);
    if (t == last_draw) {
      st_relaxed(lw.ticket, 0);
      st_release(lw.epoch, e + 1);
    }
    s_next = t;
    s_epoch = e;
  }
  __syncthreads();
  const uint64_t epoch = s_epoch;

  if (warp == kCtaWarps) {
    // ===================== store warp =====================
    uint32_t fp[2] = {0, 0};
    for (int b = 0;; b ^= 1) {
      mbar_wait_parity(&s_full[b], fp[b]);
      fp[b] ^= 1u;
      const uint64_t t = s_hand_tile[b];
      if (t == ~0ull) break;
      const uint32_t ts = s_hand_s[b], tp = s_hand_p[b];
      const uint32_t* packed = reinterpret_cast<const uint32_t*>(bufs + b * L::kBuf);
      const uint32_t* sgn = reinterpret_cast<const uint32_t*>(bufs + b * L::kBuf + L::kPackedCap);
      uint64_t es, ep;
      resolve_prefix(lw, t, epoch, ts, tp, &es, &ep, out.err);
      const bool fits = es + ts <= out.sign_cap && ep + tp <= out.payload_cap;
      if (lane == 0) {
        out.toff[2 * t] = es;
        out.toff[2 * t + 1] = ep;
        if (t == ntiles - 1) {
          out.toff[2 * ntiles] = es + ts;
          out.toff[2 * ntiles + 1] = ep + tp;
        }
        if (!fits) atomicOr(out.err, HSZ_ERR_CAPACITY);
      }
      if (fits) {
        uint32_t* dsg = reinterpret_cast<uint32_t*>(out.signs + es);
        const uint32_t nsw = (ts + 3) >> 2, npw = (tp + 3) >> 2;
        for (uint32_t i = lane; i < nsw; i += 32) dsg[i] = sgn[i];
        uint32_t* dpy = reinterpret_cast<uint32_t*>(out.payload + ep);
        uint32_t head = static_cast<uint32_t>(((16 - (ep & 15)) & 15) >> 2);
        head = head < npw ? head : npw;
        for (uint32_t i = lane; i < head; i += 32) dpy[i] = packed[i];
        // 16-byte stores from the first 16-byte aligned global word on
        const uint32_t nv = (npw - head) >> 2;
        uint4* dv = reinterpret_cast<uint4*>(dpy + head);
        for (uint32_t i = lane; i < nv; i += 32) {
          const uint32_t k = head + 4 * i;
          dv[i] = make_uint4(packed[k], packed[k + 1], packed[k + 2], packed[k + 3]);
        }
        for (uint32_t i = head + 4 * nv + lane; i < npw; i += 32) dpy[i] = packed[i];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);
    }
    return;
  }

  // ===================== compute warps =====================
  uint64_t tile = s_next;
  uint32_t flags = 0;
  uint32_t ep_parity[2] = {1, 1};               // both staging buffers start empty
  int buf = 0;
  if (tile < ntiles) src.issue(tile, stage, st, s_tmp, &flags);
  // one ticket ahead: thread 0 fetches the ticket after `tile` now
  uint64_t ahead = 0;
  if (threadIdx.x == 0 && tile < ntiles) ahead = atom_add_acq_rel(lw.ticket, 1);

  // resolve a tile in place (compute warps) and return its exclusive offsets
  auto resolve_here = [&](uint64_t t, uint32_t agg_s, uint32_t agg_p, bool published) -> bool {
    if (warp == 0) {
      uint64_t es, ep;
      if (published) {
        resolve_prefix(lw, t, epoch, agg_s, agg_p, &es, &ep, out.err);
      } else {
        lookback(lw, t, epoch, agg_s, agg_p, &es, &ep, out.err);
      }
      if (lane == 0) {
        s_excl_s = es;
        s_excl_p = ep;
        out.toff[2 * t] = es;
        out.toff[2 * t + 1] = ep;
        if (t == ntiles - 1) {
          out.toff[2 * ntiles] = es + agg_s;
          out.toff[2 * ntiles + 1] = ep + agg_p;
        }
        if (es + agg_s > out.sign_cap || ep + agg_p > out.payload_cap) {
          atomicOr(out.err, HSZ_ERR_CAPACITY);
          s_excl_s = ~0ull;
        }
      }
    }
    grp_sync();
    return s_excl_s != ~0ull;
  };

  while (tile < ntiles) {
    trace(1);
    const bool fast = src.rows(stage, st, rows, &flags);   // CTA-uniform, ends with a barrier
    trace(2);
    // the ticket drawn one iteration ago becomes `next`; draw the one after
    if (threadIdx.x == 0) {
      if (ahead == last_draw) {
        st_relaxed(lw.ticket, 0);
        st_release(lw.epoch, epoch + 1);
      }
      s_next = ahead;
    }
    grp_sync();
    const uint64_t next = s_next;
    if (threadIdx.x == 0 && next < ntiles) ahead = atom_add_acq_rel(lw.ticket, 1);
    if (fast) {
      if (next < ntiles) src.issue(next, stage, st, s_tmp, &flags);   // prefetch
      // ---- thread-per-block: residuals, width, sign word -----------------
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
          mx |= live ? static_cast<uint32_t>(dlt < 0 ? -dlt : dlt) : 0u;   // bitlen(OR) == bitlen(max)
          sbits |= (live && dlt < 0) ? (1u << (31 - i)) : 0u;
        }
      }
      const uint32_t w = mx ? 32 - __clz(mx) : 0;
      const uint32_t sb = (active && w) ? (len + 7) >> 3 : 0;
      const uint32_t pb = active ? (len * w + 7) >> 3 : 0;
      uint32_t es, ep, tile_s, tile_p;
      scan2(sb, pb, &es, &ep, &tile_s, &tile_p, s_tmp);
      if (threadIdx.x == 0) publish_aggregate(lw, tile, epoch, tile_s, tile_p);
      if (active) {
        out.widths[gb] = static_cast<uint8_t>(w);
        out.outliers[gb] = first;
      }
      trace(3);
      const bool staged = tile_p <= L::kPackedCap;   // CTA-uniform
      uint32_t* dst;
      uint32_t* sgn;
      if (staged) {
        mbar_wait_parity(&s_empty[buf], ep_parity[buf]);   // buffer streamed out
        ep_parity[buf] ^= 1u;
        dst = reinterpret_cast<uint32_t*>(bufs + buf * L::kBuf) + (ep >> 2);
        sgn = reinterpret_cast<uint32_t*>(bufs + buf * L::kBuf + L::kPackedCap);
      } else {
        // rare: a very wide tile -- resolve here, pack straight to global
        const bool ok = resolve_here(tile, tile_s, tile_p, true);
        dst = ok ? reinterpret_cast<uint32_t*>(out.payload + s_excl_p + ep) : nullptr;
        sgn = ok ? reinterpret_cast<uint32_t*>(out.signs + s_excl_s) : nullptr;
      }
      trace(4);
      if (w && dst) {
        // second walk: MSB-first w-bit fields through a 64-bit shift register
        sgn[es >> 2] = bswap32(sbits);
        uint64_t acc = 0;
        int nb = w, wi = 0;                // slot 0: a zero field
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
      }
      grp_sync();                           // packed tile complete; rows free
      trace(5);
      if (staged && threadIdx.x == 0) {
        s_hand_tile[buf] = tile;
        s_hand_s[buf] = tile_s;
        s_hand_p[buf] = tile_p;
        mbar_arrive(&s_full[buf]);
      }
      if (staged) buf ^= 1;
    } else {
      // ---- fallback tile: exact path, resolved here ------------------------
      flags |= fallback_sizes(src, out, tile, nblocks, tail_len, s_wsb, s_wpb);
      grp_sync();
      const uint32_t agg_s = s_wsb[0] + s_wsb[1] + s_wsb[2] + s_wsb[3];
      const uint32_t agg_p = s_wpb[0] + s_wpb[1] + s_wpb[2] + s_wpb[3];
      if (resolve_here(tile, agg_s, agg_p, false)) {
        uint64_t gs = s_excl_s, gp = s_excl_p;
        for (int i = 0; i < warp; ++i) {
          gs += s_wsb[i];
          gp += s_wpb[i];
        }
        fallback_pack(src, out, tile, nblocks, tail_len, gs, gp, scratch + warp * 64);
      }
      grp_sync();
      if (next < ntiles) src.issue(next, stage, st, s_tmp, &flags);
    }
    tile = next;
  }
  // stop the store warp after it has drained both buffers
  for (int i = 0; i < 2; ++i) {
    mbar_wait_parity(&s_empty[buf], ep_parity[buf]);
    ep_parity[buf] ^= 1u;
    if (i == 0) {
      grp_sync();
      if (threadIdx.x == 0) {
        s_hand_tile[buf] = ~0ull;
        mbar_arrive(&s_full[buf]);
      }
    }
    buf ^= 1;
  }
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(out.err, flags);
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

template <class Sink, typename T>
__device__ __noinline__ uint32_t fallback_decode(TileIn t, Sink sink, T* ot) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t flags = 0;
  for (int j = 0; j < BPW; ++j) {
    const int lb = warp * BPW + j;
    const LaneBlock m = lane_block(t, j);
    if (m.len == 0) break;
    const int64_t q = decode_lane(t.sgn, t.pay, m.w, m.o, m.soff, m.poff, m.len, lane, &flags);
    ot[pad(lb, lane)] = sink.value(q, &flags);
  }
  return flags;
}

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
    flags |= fallback_decode(t, sink, ot);
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

// Cross-CTA reduction without a serial tail: every CTA adds its S (int128,
// two's complement) and Q (uint192) as 32-bit chunks into ten u64
// carry-save counters in the workspace (ws[8..18); a chunk < 2^32, so 2^32
// CTAs cannot overflow a counter).  The last CTA to finish folds the
// counters into exact 128/192-bit values, writes out[5] and re-zeroes them.
__device__ __forceinline__ void add_shifted(uint64_t* L, int nl, uint64_t c, int bit) {
  // L (nl little-endian u64 limbs) += c << bit
  const int li = bit >> 6, sh = bit & 63;
  unsigned __int128 v = static_cast<unsigned __int128>(c) << sh;
  for (int i = li; i < nl && v; ++i) {
    const unsigned __int128 sum = static_cast<unsigned __int128>(L[i]) + static_cast<uint64_t>(v);
    L[i] = static_cast<uint64_t>(sum);
    v = (v >> 64) + (sum >> 64);
  }
}

__device__ __forceinline__ void finish_moments(Acc acc, uint64_t, void* ws, uint64_t* out) {
  __shared__ Acc s_acc[32];
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int m = 16; m > 0; m >>= 1) acc.merge(shfl_xor_acc(acc, m));
  if (lane == 0) s_acc[warp] = acc;
  __syncthreads();
  uint64_t* base = static_cast<uint64_t*>(ws);
  uint64_t* done = base + 2;
  uint64_t* cs = base + 8;
  if (threadIdx.x == 0) {
    Acc t = s_acc[0];
    for (int i = 1; i < nw; ++i) t.merge(s_acc[i]);
    const unsigned __int128 su = static_cast<unsigned __int128>(t.s);
    for (int k = 0; k < 4; ++k) {
      const uint64_t ch = static_cast<uint64_t>(su >> (32 * k)) & 0xffffffffull;
      if (ch) atomicAdd(reinterpret_cast<unsigned long long*>(cs + k), ch);
    }
    for (int k = 0; k < 6; ++k) {
      const uint64_t ch = (k < 4) ? static_cast<uint64_t>(t.q >> (32 * k)) & 0xffffffffull
                                  : (t.q2 >> (32 * (k - 4))) & 0xffffffffull;
      if (ch) atomicAdd(reinterpret_cast<unsigned long long*>(cs + 4 + k), ch);
    }
    __threadfence();
    s_last = atom_add_acq_rel(done, 1) == gridDim.x - 1;
    if (s_last) {
      __threadfence();
      uint64_t S[2] = {0, 0}, Q[4] = {0, 0, 0, 0};
      for (int k = 0; k < 4; ++k) add_shifted(S, 2, ld_relaxed(cs + k), 32 * k);
      for (int k = 0; k < 6; ++k) add_shifted(Q, 4, ld_relaxed(cs + 4 + k), 32 * k);
      out[0] = S[0];
      out[1] = S[1];
      out[2] = Q[0];
      out[3] = Q[1];
      out[4] = Q[2];
      for (int k = 0; k < 10; ++k) st_relaxed(cs + k, 0);
      st_relaxed(done, 0);   // rearm for the next launch on this workspace
    }
  }
}

}  // namespace k32
}  // namespace hsz
