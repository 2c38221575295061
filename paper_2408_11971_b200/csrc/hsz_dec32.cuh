// Stream-tile front end for block_len 32 (decode side) and the register-
// resident scalar multiply.
//
// A tile = 128 blocks.  The TMA warp stages one input tile per mbarrier phase:
//   * its widths / outliers with plain loads by the 32 lanes (640 bytes);
//   * its sign bytes and payload bytes with two cp.async.bulk copies
//     (UBLKCP), located by the input stream's tile-offset cache
//     (toff[2t], toff[2t+1] .. toff[2t+2], toff[2t+3]);
//   * a tile whose payload does not fit the staging buffer is read in place.
// Compute thread b then decodes block b into 32 registers (prefix sums of
// the signed residuals seeded with the outlier, codec.py:228-262).
//
// scalar_mul (ops.py:199-225) = this front + the exact rescale
// t = RN(2eps * RN(bin * rs)), bin' = round-half-away(t) + the encoder back
// half of hsz_enc32.cuh (code, scan, publish, pack, placement warp).
#pragma once

#include "hsz_enc32.cuh"

namespace hsz {
namespace d32 {

constexpr int K = 32;
constexpr int TB = kTileBlocks;
constexpr int kCompute = e32::kCompute;
constexpr uint32_t kSignCap = TB * 4 + 32;   // staged sign bytes (+ 16-byte alignment slack)
#ifndef HSZ_PAYCAP
#define HSZ_PAYCAP 16384
#endif
constexpr uint32_t kPayCap = HSZ_PAYCAP;     // staged payload bytes
constexpr int kFastW = 24;                   // register decode: widths <= 24, |outlier| < 2^29

struct StreamIn {
  const uint8_t* widths;
  const int32_t* outliers;
  const uint8_t* signs;
  const uint8_t* payload;
  const uint64_t* toff;
  uint64_t n;
  uint64_t nblocks;
  uint64_t ntiles;
  uint32_t tail_len;
};

template <uint32_t kCap>
struct InTileT {
  static constexpr uint32_t kPayBytes = kCap;
  alignas(16) unsigned char sgn[kSignCap];
  alignas(16) unsigned char pay[kCap];
  alignas(16) int32_t o[TB];
  alignas(16) uint8_t w[TB];
  uint64_t tile;       // >= ntiles: no more tiles
  uint64_t gs0, gp0;   // global offsets of the tile's first sign / payload byte
  uint32_t soff;       // offset of that sign byte within sgn[]
  uint32_t poff;       // offset of that payload byte within pay[] (staged tiles)
  uint32_t staged;     // payload staged (else read in place from global memory)
};
using InTile = InTileT<kPayCap>;

__device__ __forceinline__ void bulk_g2s_(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMA warp (all 32 lanes): the tile-offset entries of tile t (lanes 0-3 hold
// toff[2t + lane]); issued a tile ahead so their latency is hidden.
__device__ __forceinline__ uint64_t prefetch_toff(const StreamIn& s, uint64_t t) {
  const int lane = threadIdx.x & 31;
  return (lane < 4 && t < s.ntiles) ? s.toff[2 * t + lane] : 0ull;
}

// TMA warp (all 32 lanes): stage tile t (or "no more tiles") into `it`,
// completing one phase of `bar` (count 1: lane 0's arrive).  `tv` = the
// prefetched tile-offset entries.  Full tiles arrive by four bulk copies
// (widths, outliers, sign bytes, payload bytes); the stream's last tile
// loads its widths / outliers with plain loads.
template <class IT>
__device__ __forceinline__ void stage_tile(const StreamIn& s, uint64_t t, uint64_t tv, IT& it,
                                           uint64_t* bar) {
  const int lane = threadIdx.x & 31;
  if (t >= s.ntiles) {
    if (lane == 0) {
      it.tile = t;
      mbar_arrive(bar);
    }
    __syncwarp();
    return;
  }
  const uint64_t s0 = __shfl_sync(kFull, tv, 0), p0 = __shfl_sync(kFull, tv, 1);
  const uint64_t s1 = __shfl_sync(kFull, tv, 2), p1 = __shfl_sync(kFull, tv, 3);
  const bool full = (t + 1) * TB <= s.nblocks &&
                    ((reinterpret_cast<uintptr_t>(s.widths) | reinterpret_cast<uintptr_t>(s.outliers)) & 15u) == 0;
  if (!full) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t lb = 4 * lane + j;
      const uint64_t b = t * TB + lb;
      uint8_t w = 0;
      int32_t o = 0;
      if (b < s.nblocks) {
        w = s.widths[b];
        o = s.outliers[b];
      }
      it.w[lb] = w;
      it.o[lb] = o;
    }
  }
  __syncwarp();
  if (lane == 0) {
    const uint64_t s_lo = s0 & ~15ull, s_hi = (s1 + 15) & ~15ull;
    const uint64_t p_lo = p0 & ~15ull, p_hi = (p1 + 15) & ~15ull;
    const uint32_t sbytes = static_cast<uint32_t>(s_hi - s_lo);
    const uint32_t pbytes = static_cast<uint32_t>(p_hi - p_lo);
    const bool staged = pbytes <= IT::kPayBytes && sbytes <= kSignCap;
    it.tile = t;
    it.gs0 = s0;
    it.gp0 = p0;
    it.soff = static_cast<uint32_t>(s0 - s_lo);
    it.poff = static_cast<uint32_t>(p0 - p_lo);
    it.staged = staged ? 1u : 0u;
    const uint32_t bytes = (full ? TB * 5u : 0u) + (staged ? sbytes + pbytes : 0u);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (bytes) {
      mbar_arrive_expect_tx(bar, bytes);
      if (full) {
        bulk_g2s_(it.w, s.widths + t * TB, TB, bar);
        bulk_g2s_(it.o, s.outliers + t * TB, TB * 4, bar);
      }
      if (staged && sbytes) bulk_g2s_(it.sgn, s.signs + s_lo, sbytes, bar);
      if (staged && pbytes) bulk_g2s_(it.pay, s.payload + p_lo, pbytes, bar);
    } else {
      mbar_arrive(bar);
    }
  }
  __syncwarp();
}

// Register decode of this thread's block (w <= kFastW, |o| < 2^29): bins as
// int32 (|bin| < 2^30).  kFull: a full block (len == 32, no tail checks);
// otherwise elements past `len` replicate the last live bin (kResid: their
// residuals are 0).  Fields are read G at a time (G * w <= 32): one window
// refill check per G fields.
#ifndef HSZ_REFILL_AHEAD
#define HSZ_REFILL_AHEAD 1
#endif

// next big-endian payload word of a staged block: a shared-memory load
// through a running 32-bit address (an index into a generic pointer costs two
// more instructions a refill: the multiply-add for the address and a move
// for the predicated increment)
#ifndef HSZ_REFILL_PTR
#define HSZ_REFILL_PTR 1
#endif
__device__ __forceinline__ uint32_t next_word(uint32_t& pa) {
  uint32_t x;
  asm("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(pa));
  pa += 4;
  return bswap32(x);
}

// kAcc: 0 q[i] = bin_i, 1 q[i] += bin_i, 2 q[i] -= bin_i (modulo 2^32)
template <int kAcc>
__device__ __forceinline__ void put_bin(int32_t& qi, int32_t v) {
  if (kAcc == 0) qi = v;
  else if (kAcc == 1) qi = static_cast<int32_t>(static_cast<uint32_t>(qi) + static_cast<uint32_t>(v));
  else qi = static_cast<int32_t>(static_cast<uint32_t>(qi) - static_cast<uint32_t>(v));
}

// kResid: q[i] receives the signed residual d_i (q[0] the outlier) instead of
// the bin -- the element-wise ops combine streams in the residual domain
// (ops.py:171-176), so they need no prefix sums on the way in
template <bool kFull, int G, int kAcc = 0, bool kResid = false>
__device__ __forceinline__ void decode_block_t(const unsigned char* sgn, const unsigned char* pay,
                                               uint32_t w, int32_t o, int len, int32_t (&q)[K]) {
  const uint32_t sw = bswap32(*reinterpret_cast<const uint32_t*>(sgn));
  // sign of element i = bit 31 - i of sw = the top bit of byte 3 - i/8 of
  // (sw << i%8): one PRMT with sign replication per element
  uint32_t sh[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) sh[k] = sw << k;
  const uint32_t* pw = reinterpret_cast<const uint32_t*>(pay);
  const uint32_t mask = (1u << w) - 1u;
  const int wg = G * static_cast<int>(w);
  uint64_t win = 0;
  int nb = 0;   // valid bits at the bottom of win
  // software-pipelined refill: the next payload word is loaded one refill
  // ahead, so its shared-memory latency overlaps the fields extracted in
  // between instead of stalling the chain (the read may run one word past
  // the block -- still inside the staging buffer)
  // (indexed loads here: the running-address form of decode_sum_t / decode_f32_t
  // measured 2% slower in the recode kernels)
#if HSZ_REFILL_AHEAD
  uint32_t nxt = pw[0];
  int wi = 1;
#else
  int wi = 0;
#endif
  int32_t P = o;
  put_bin<kAcc>(q[0], o);
#pragma unroll
  for (int c = 0; c < (K + G - 1) / G; ++c) {
    if (nb < wg) {
#if HSZ_REFILL_AHEAD
      win = (win << 32) | bswap32(nxt);
      nxt = pw[wi++];
#else
      win = (win << 32) | bswap32(pw[wi++]);
#endif
      nb += 32;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int i = c * G + g;
      if (i >= K) break;
      nb -= static_cast<int>(w);
      if (i == 0) continue;   // slot 0: the outlier's zero field
      const int32_t mag = static_cast<int32_t>(static_cast<uint32_t>(win >> nb) & mask);
      const int32_t neg = static_cast<int32_t>(prmt_sign(sh[i & 7], 3 - (i >> 3)));
      int32_t d = (mag ^ neg) - neg;
      if (!kFull) d = (i < len) ? d : 0;
      if constexpr (kResid) {
        put_bin<kAcc>(q[i], d);
      } else {
        P += d;
        put_bin<kAcc>(q[i], P);
      }
    }
  }
}

// all 32 lanes of the warp call this (the field grouping is warp-uniform)
template <int kAcc = 0, bool kResid = false>
__device__ __forceinline__ void decode_block(const unsigned char* sgn, const unsigned char* pay,
                                             uint32_t w, int32_t o, int len, int32_t (&q)[K]) {
  const uint32_t wmax = __reduce_max_sync(kFull, w);
  if (w == 0) {
    put_bin<kAcc>(q[0], o);
#pragma unroll
    for (int i = 1; i < K; ++i) put_bin<kAcc>(q[i], kResid ? 0 : o);
    return;
  }
  if (len != K) {
    decode_block_t<false, 1, kAcc, kResid>(sgn, pay, w, o, len, q);
  } else if (wmax <= 8) {
    decode_block_t<true, 4, kAcc, kResid>(sgn, pay, w, o, len, q);
  } else if (wmax <= 10) {
    decode_block_t<true, 3, kAcc, kResid>(sgn, pay, w, o, len, q);
  } else if (wmax <= 16) {
    decode_block_t<true, 2, kAcc, kResid>(sgn, pay, w, o, len, q);
  } else {
    decode_block_t<true, 1, kAcc, kResid>(sgn, pay, w, o, len, q);
  }
}

// Register-light block sums for the moment kernels: the same field walk as
// decode_block_t, but the prefix sums P_i are accumulated on the fly
// (sum P_i, and sum P_i^2 for kSq) instead of being kept as 32 bins.
#ifndef HSZ_SUM_V2
#define HSZ_SUM_V2 1
#endif

template <bool kFull, int G, bool kSq>
__device__ __forceinline__ void decode_sum_t(const unsigned char* sgn, const unsigned char* pay,
                                             uint32_t w, int len, int64_t* sp_out, uint64_t* sp2_out) {
  const uint32_t sw = bswap32(*reinterpret_cast<const uint32_t*>(sgn));
#if HSZ_SUM_V2
  uint32_t sh[8];   // sign of element i: PRMT sign replication (see decode_block_t)
#pragma unroll
  for (int k = 0; k < 8; ++k) sh[k] = sw << k;
#endif
  const uint32_t* pw = reinterpret_cast<const uint32_t*>(pay);
#if HSZ_REFILL_PTR
  uint32_t pa = smem_u32(pay);
  (void)pw;
#endif
  const uint32_t mask = (1u << w) - 1u;
  const int wg = G * static_cast<int>(w);
  uint64_t win = 0;
  int nb = 0;
  int wi = 0;
  int32_t P = 0;      // |P| <= 31 * (2^w - 1) < 2^29
  // sum P <= 496 * (2^w - 1): int32 holds it up to w = 22 (G >= 2 means
  // w <= 16); the one-field-per-step path serves widths up to kFastW = 24
  using SumT = std::conditional_t<(G >= 2), int32_t, int64_t>;
  SumT sp = 0;
  // sum P^2 < 32 * 2^58; with w <= 8 (G = 4) sum_i (255 i)^2 < 6.8e8 fits 32 bits
  using SqT = std::conditional_t<(HSZ_SUM_V2 && G >= 4), uint32_t, uint64_t>;
  SqT sp2 = 0;
#pragma unroll
  for (int c = 0; c < (K + G - 1) / G; ++c) {
    if (nb < wg) {
#if HSZ_REFILL_PTR
      win = (win << 32) | next_word(pa);
      (void)wi;
#else
      win = (win << 32) | bswap32(pw[wi++]);
#endif
      nb += 32;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int i = c * G + g;
      if (i >= K) break;
      nb -= static_cast<int>(w);
      if (i == 0) continue;
      const int32_t mag = static_cast<int32_t>(static_cast<uint32_t>(win >> nb) & mask);
#if HSZ_SUM_V2
      const int32_t neg = static_cast<int32_t>(prmt_sign(sh[i & 7], 3 - (i >> 3)));
#else
      const int32_t neg = static_cast<int32_t>(sw << i) >> 31;
#endif
      int32_t d = (mag ^ neg) - neg;
      if (!kFull) d = (i < len) ? d : 0;
      if (HSZ_SUM_V2 && kFull && !kSq) {
        // sum_i P_i = sum_j (K - j) d_j: one multiply-add per element and no
        // serial prefix chain (the same exact integer)
        sp += static_cast<SumT>(K - i) * d;
        continue;
      }
      P += d;
      if (kFull || i < len) {
        sp += P;
        if (kSq) {
          if constexpr (sizeof(SqT) == 4)
            sp2 += static_cast<uint32_t>(P * P);
          else
            sp2 += static_cast<uint64_t>(static_cast<int64_t>(P) * P);
        }
      }
    }
  }
  *sp_out = sp;
  *sp2_out = sp2;
}

template <bool kSq>
__device__ __forceinline__ void decode_sum(const unsigned char* sgn, const unsigned char* pay,
                                           uint32_t w, int len, int64_t* sp, uint64_t* sp2) {
  const uint32_t wmax = __reduce_max_sync(kFull, w);
  *sp = 0;
  *sp2 = 0;
  if (w == 0) return;
  if (len != K) {
    decode_sum_t<false, 1, kSq>(sgn, pay, w, len, sp, sp2);
  } else if (wmax <= 8) {
    decode_sum_t<true, 4, kSq>(sgn, pay, w, len, sp, sp2);
  } else if (wmax <= 10) {
    decode_sum_t<true, 3, kSq>(sgn, pay, w, len, sp, sp2);
  } else if (wmax <= 16) {
    decode_sum_t<true, 2, kSq>(sgn, pay, w, len, sp, sp2);
  } else {
    decode_sum_t<true, 1, kSq>(sgn, pay, w, len, sp, sp2);
  }
}

// Decompress without keeping the block's bins: every value is converted as
// soon as its bin is known (RN32(RN64(2eps * bin)), codec.py:107-115) and
// written four at a time into the block's swizzled 128-byte row.
template <bool kFull, int G>
__device__ __forceinline__ void decode_f32_t(const unsigned char* sgn, const unsigned char* pay,
                                             uint32_t w, int32_t o, int len, double dd,
                                             unsigned char* row, uint32_t rsw, bool may_overflow,
                                             uint32_t* flags) {
  // a constant block has no sign bytes: its offset may be unaligned (after
  // the stream's partial last block), so the word is read only when w > 0
  const uint32_t sw = w ? bswap32(*reinterpret_cast<const uint32_t*>(sgn)) : 0u;
#if HSZ_SUM_V2
  uint32_t sh[8];   // PRMT sign replication, as in decode_block_t
#pragma unroll
  for (int k = 0; k < 8; ++k) sh[k] = sw << k;
#endif
  const uint32_t* pw = reinterpret_cast<const uint32_t*>(pay);
#if HSZ_REFILL_PTR
  uint32_t pa = smem_u32(pay);
  (void)pw;
#endif
  const uint32_t mask = (1u << w) - 1u;
  const int wg = G * static_cast<int>(w);
  uint64_t win = 0;
  int nb = 0;
  int wi = 0;
  int32_t P = o;
  float v[4];
  bool bad = false;
#pragma unroll
  for (int c = 0; c < (K + G - 1) / G; ++c) {
    if (w && nb < wg) {
#if HSZ_REFILL_PTR
      win = (win << 32) | next_word(pa);
      (void)wi;
#else
      win = (win << 32) | bswap32(pw[wi++]);
#endif
      nb += 32;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int i = c * G + g;
      if (i >= K) break;
      nb -= static_cast<int>(w);
      if (i > 0 && w) {
        const int32_t mag = static_cast<int32_t>(static_cast<uint32_t>(win >> nb) & mask);
#if HSZ_SUM_V2
        const int32_t neg = static_cast<int32_t>(prmt_sign(sh[i & 7], 3 - (i >> 3)));
#else
        const int32_t neg = static_cast<int32_t>(sw << i) >> 31;
#endif
        int32_t d = (mag ^ neg) - neg;
        if (!kFull) d = (i < len) ? d : 0;
        P += d;
      }
      v[i & 3] = __double2float_rn(__dmul_rn(dd, i32_to_double(P)));
      if (may_overflow) bad |= !isfinite(v[i & 3]);
      if ((i & 3) == 3)
        *reinterpret_cast<float4*>(row + (((i >> 2) ^ rsw) << 4)) = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
  if (bad) *flags |= HSZ_ERR_OUTPUT_NONFINITE;
}

__device__ __forceinline__ void decode_f32(const unsigned char* sgn, const unsigned char* pay,
                                           uint32_t w, int32_t o, int len, double dd,
                                           unsigned char* row, uint32_t rsw, bool may_overflow,
                                           uint32_t* flags) {
  const uint32_t wmax = __reduce_max_sync(kFull, w);
  if (len != K) {
    decode_f32_t<false, 1>(sgn, pay, w, o, len, dd, row, rsw, may_overflow, flags);
  } else if (wmax <= 8) {
    decode_f32_t<true, 4>(sgn, pay, w, o, len, dd, row, rsw, may_overflow, flags);
  } else if (wmax <= 10) {
    decode_f32_t<true, 3>(sgn, pay, w, o, len, dd, row, rsw, may_overflow, flags);
  } else if (wmax <= 16) {
    decode_f32_t<true, 2>(sgn, pay, w, o, len, dd, row, rsw, may_overflow, flags);
  } else {
    decode_f32_t<true, 1>(sgn, pay, w, o, len, dd, row, rsw, may_overflow, flags);
  }
}

// ---------------------------------------------------------------------------
// re-encoding operations: scalar multiply (kOp 0) and element-wise add / sub
// of two streams (kOp 1 / 2, ops.py:163-192) share one persistent kernel --
// decode front (one or two staged input tiles), per-element transform in
// registers, the encoder back half of hsz_enc32.cuh.

constexpr int kOpSmul = 0, kOpAdd = 1, kOpSub = 2;
constexpr uint32_t kEwPayCap = 8192;   // per operand (two staged tiles: 4 CTAs per SM)

struct EmptyTile {};

template <int kOp>
struct RecodeSmem {
  static constexpr bool kTwo = kOp != kOpSmul;
  using Tile = InTileT<kTwo ? kEwPayCap : kPayCap>;
  Tile in;
  std::conditional_t<kTwo, Tile, EmptyTile> in2;   // second operand (element-wise ops)
  alignas(16) unsigned char pk[2][e32::kBufBytes];
  alignas(16) uint32_t sgn[2][TB];
  uint32_t bes[TB], bep[TB];      // per-block offsets within the input tile (exact path)
  uint32_t bes2[kTwo ? TB : 1], bep2[kTwo ? TB : 1];
  uint64_t bar, in_empty, st_full[2], st_empty[2];
  uint64_t excl_s[2], excl_p[2];
  uint32_t agg_ts[2], agg_tp[2];
  uint64_t tile_of[2];
  uint64_t epoch;
  // scalar_mul releases S.in right after the decode; a tile that then turns
  // out to need the exact path (a rescaled bin beyond 2^30) re-decodes from
  // global memory and finds its block headers here
  uint64_t xgs0, xgp0;
  int32_t xo[TB];
  uint8_t xw[TB];
  // three scan buffers: the two operands' in-tile offset scans run back to
  // back with no barrier between the first one's reads and the second one's
  // writes, so they must not share one (a shared buffer let a fast warp
  // overwrite a total a slow warp had not read yet: wrong offsets)
  alignas(16) uint32_t scan[4], scan_in[4], scan_in2[4];
  uint32_t wsb[4], wpb[4];
};
using SmulSmem = RecodeSmem<kOpSmul>;

// exact (64/128-bit) bins of the output for the warp-per-block fallback: the
// input block is decoded from global memory
struct SrcSmulExact {
  StreamIn in;
  const SmulSmem* S;
  int64_t rs;
  double d;
  __device__ __forceinline__ int64_t lane_bin(int lb, int lane, int len, uint32_t* flags) {
    uint32_t f = 0;
    const int64_t q = k32::decode_lane(in.signs, in.payload, S->xw[lb], S->xo[lb],
                                       S->xgs0 + S->bes[lb], S->xgp0 + S->bep[lb], len, lane, &f);
    *flags |= f;
    if (f || lane >= len) return 0;
    return rescale1(product_rn(q, rs), d, flags);
  }
};

// element-wise: residual_a (+|-) residual_b exactly in 128 bits, outliers
// o_a (+|-) o_b -- the reference's residual-domain fold (ops.py:163-182): no
// bins are formed, so operands of any width up to 64 combine exactly (a
// combined magnitude of 2^64 or more is flagged, where the reference's
// uint64 conversion fails)
template <int kOp>
struct SrcEwExact {
  static constexpr bool kResid = true;
  StreamIn a, b;
  const RecodeSmem<kOp>* S;
  __device__ __forceinline__ __int128 lane_resid(int lb, int lane, int len, uint32_t* flags) {
    (void)flags;
    const __int128 ra = k32::decode_lane_resid(a.signs, a.payload, S->in.w[lb], S->in.o[lb],
                                               S->in.gs0 + S->bes[lb], S->in.gp0 + S->bep[lb], len,
                                               lane);
    const __int128 rb = k32::decode_lane_resid(b.signs, b.payload, S->in2.w[lb], S->in2.o[lb],
                                               S->in2.gs0 + S->bes2[lb], S->in2.gp0 + S->bep2[lb],
                                               len, lane);
    return kOp == kOpSub ? ra - rb : ra + rb;
  }
};

template <class SM>
__device__ __forceinline__ void smul_copy_staged(SM& S, const k32::EncodeOut& out,
                                                 uint32_t ts, uint32_t tp, int par, uint32_t rank,
                                                 uint32_t nthr) {
  const uint64_t es = S.excl_s[par], ep = S.excl_p[par];
  if (es == ~0ull) return;
  uint32_t* dsg = reinterpret_cast<uint32_t*>(out.signs + es);
  for (uint32_t i = rank; i < ((ts + 3u) >> 2); i += nthr) dsg[i] = S.sgn[par][i];
  const uint32_t* pbuf = reinterpret_cast<const uint32_t*>(S.pk[par]);
  uint32_t* dst = reinterpret_cast<uint32_t*>(out.payload + ep);
  const uint32_t nw = (tp + 3u) >> 2;
  uint32_t head = static_cast<uint32_t>(((16u - (ep & 15u)) & 15u) >> 2);
  head = head < nw ? head : nw;
  if (rank < head) dst[rank] = pbuf[e32::swz_word(rank)];
  const uint32_t nv = (nw - head) >> 2;
  uint4* dv = reinterpret_cast<uint4*>(dst + head);
  for (uint32_t i = rank; i < nv; i += nthr) {
    const uint32_t k = head + 4u * i;
    dv[i] = make_uint4(pbuf[e32::swz_word(k)], pbuf[e32::swz_word(k + 1)],
                       pbuf[e32::swz_word(k + 2)], pbuf[e32::swz_word(k + 3)]);
  }
  const uint32_t rest = head + 4u * nv + rank;
  if (rest < nw) dst[rest] = pbuf[e32::swz_word(rest)];
}

template <class SM>
__device__ __forceinline__ void smul_resolve(SM& S, const k32::EncodeOut& out, uint64_t tile,
                                             uint64_t epoch, uint64_t ntiles, uint32_t ts,
                                             uint32_t tp, int par) {
  const int lane = threadIdx.x & 31;
  uint64_t es, ep;
  lb_resolve(lb_words(out.ws), tile, epoch, ts, tp, &es, &ep, out.err);
  if (lane == 0) {
    out.toff[2 * tile] = es;
    out.toff[2 * tile + 1] = ep;
    if (tile == ntiles - 1) {
      out.toff[2 * ntiles] = es + ts;
      out.toff[2 * ntiles + 1] = ep + tp;
    }
    const bool fits = es + ts <= out.sign_cap && ep + tp <= out.payload_cap;
    if (!fits) atomicOr(out.err, HSZ_ERR_CAPACITY);
    S.excl_s[par] = fits ? es : ~0ull;
    S.excl_p[par] = ep;
  }
}

struct SmulParams {
  int64_t rs;
  double d;      // 2 eps
  double rsd;    // (double) rs
  int small_rs;  // |rs| < 2^23: every register-path product is exact in float64
};

// in-tile (sign, payload) byte offsets of this thread's block: one CTA scan
__device__ __forceinline__ void block_offsets(uint32_t w, int len, uint32_t* scan, uint32_t* es,
                                              uint32_t* ep) {
  const uint32_t isb = w ? ((static_cast<uint32_t>(len) + 7u) >> 3) : 0u;
  const uint32_t ipb = (static_cast<uint32_t>(len) * w + 7u) >> 3;
  uint32_t itot;
  const uint32_t iex = e32::cta_scan(isb | (ipb << 10), scan, &itot);
  *es = iex & 1023u;
  *ep = iex >> 10;
}
// ... with a CTA-wide OR of `flag` on the same barrier
__device__ __forceinline__ bool block_offsets_or(uint32_t w, int len, bool flag, uint32_t* scan,
                                                 uint32_t* es, uint32_t* ep) {
  const uint32_t isb = w ? ((static_cast<uint32_t>(len) + 7u) >> 3) : 0u;
  const uint32_t ipb = (static_cast<uint32_t>(len) * w + 7u) >> 3;
  uint32_t itot;
  bool any;
  const uint32_t iex = e32::cta_scan_or(isb | (ipb << 10), flag, scan, &itot, &any);
  *es = iex & 1023u;
  *ep = iex >> 10;
  return any;
}

// Persistent, warp-specialised like the compressor: warps 0-3 decode +
// transform + code + pack, warp 4 stages input tiles (both operands' for the
// element-wise ops, on one mbarrier), warp 5 places output tiles
// (look-back + copy).
template <int kOp>
__global__ void __launch_bounds__(e32::kThreadsWS, HSZ_ENC_CTAS)
    recode_kernel(StreamIn in, StreamIn in2, SmulParams sp, k32::EncodeOut out) {
  constexpr bool kTwo = kOp != kOpSmul;
  using SM = RecodeSmem<kOp>;
  extern __shared__ unsigned char smraw[];
  const uint32_t a0 = smem_u32(smraw);
  SM& S = *reinterpret_cast<SM*>(smraw + (((a0 + 1023u) & ~1023u) - a0));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t ntiles = in.ntiles, nblocks = in.nblocks;
  LookbackWs lw = LookbackWs::bind(out.ws, ntiles);
  const uint64_t last_draw = ntiles + gridDim.x - 1;
  if (tid == kCompute) {
    mbar_init(&S.bar, kTwo ? 2 : 1);
    mbar_init(&S.in_empty, kCompute / 32);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&S.st_full[b], kCompute / 32);
      mbar_init(&S.st_empty[b], 1);
    }
    fence_mbar_init();
    S.epoch = ld_acquire(lw.epoch);
  }
  __syncthreads();
  const uint64_t epoch = S.epoch;
  auto draw = [&]() -> uint64_t {
    const uint64_t t = atom_add_relaxed(lw.ticket, 1);
    if (t == last_draw) {
      st_relaxed(lw.ticket, 0);
      st_release(lw.epoch, epoch + 1);
    }
    return t;
  };

  if (warp == kCompute / 32) {
    // ============================ TMA warp ==============================
    uint64_t t = 0, ahead = 0;
    if (lane == 0) {
      t = draw();
      if (t < ntiles) ahead = draw();
    }
    t = __shfl_sync(kFull, t, 0);
    ahead = __shfl_sync(kFull, ahead, 0);
    stage_tile(in, t, prefetch_toff(in, t), S.in, &S.bar);
    if constexpr (kTwo) stage_tile(in2, t, prefetch_toff(in2, t), S.in2, &S.bar);
    uint64_t tv = prefetch_toff(in, ahead);
    uint64_t tv2 = kTwo ? prefetch_toff(in2, ahead) : 0ull;
    for (uint32_t k = 0; t < ntiles; ++k) {
      const uint64_t nx = ahead;
      mbar_wait_parity_sleep(&S.in_empty, k & 1u);
      stage_tile(in, nx, tv, S.in, &S.bar);
      if constexpr (kTwo) stage_tile(in2, nx, tv2, S.in2, &S.bar);
      // draw the ticket after the wait, not before it: a tile period less
      // between a ticket and its tile's aggregate, so fewer look-backs find a
      // predecessor that has not published yet
      if (lane == 0 && nx < ntiles) ahead = draw();
      ahead = __shfl_sync(kFull, ahead, 0);
      tv = prefetch_toff(in, ahead);
      if (kTwo) tv2 = prefetch_toff(in2, ahead);
      t = nx;
    }
    return;
  }

  if (warp == kCompute / 32 + 1) {
    // =========================== placement warp ===========================
    for (uint32_t kk = 0;; ++kk) {
      const int b = kk & 1;
      mbar_wait_parity_sleep(&S.st_full[b], (kk >> 1) & 1u);
      const uint32_t pts = S.agg_ts[b], ptp = S.agg_tp[b];
      if (pts == e32::kDone) break;
      if (pts != e32::kSelfPlaced) {
        trace_tile(S.tile_of[b], 7);
        smul_resolve(S, out, S.tile_of[b], epoch, ntiles, pts, ptp, b);
        __syncwarp();
        smul_copy_staged(S, out, pts, ptp, b, lane, 32);
        trace_tile(S.tile_of[b], 8);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.st_empty[b]);
    }
    return;
  }

  // =========================== compute warps ===========================
  uint32_t phase = 0, flags = 0;
  int par = 0, k = 0;
  while (true) {
    mbar_wait_parity(&S.bar, phase);
    phase ^= 1u;
    const uint64_t cur = S.in.tile;
    if (cur < ntiles) trace_tile(cur, 1);
    if (cur >= ntiles) {
      if (k >= 2) mbar_wait_parity(&S.st_empty[par], ((k >> 1) - 1) & 1u);
      if (tid == 0) S.agg_ts[par] = e32::kDone;
      mbar_arrive_warp(&S.st_full[par]);
      break;
    }
    // ---- locate and decode this thread's block -------------------------------
    const uint64_t gb = cur * TB + tid;
    const bool active = gb < nblocks;
    const int len = !active ? 0 : (gb == nblocks - 1 ? static_cast<int>(in.tail_len) : K);
    uint32_t w = S.in.w[tid];
    const int32_t o = S.in.o[tid];
    if (w > 64) {
      flags |= HSZ_ERR_BAD_WIDTH;
      w = 0;
    }
    if constexpr (!kTwo) {
      S.xw[tid] = static_cast<uint8_t>(w);
      S.xo[tid] = o;
      if (tid == 0) {
        S.xgs0 = S.in.gs0;
        S.xgp0 = S.in.gp0;
      }
    }
    uint32_t ies, iep;
    bool fast_in = S.in.staged && w <= static_cast<uint32_t>(kFastW) && o > -(1 << 29) && o < (1 << 29);
    bool exact;
    if constexpr (!kTwo) {
      // the CTA-uniform path choice rides on the offset scan's barrier
      exact = block_offsets_or(w, len, !fast_in || !sp.small_rs, S.scan_in, &ies, &iep);
    } else
    {
      block_offsets(w, len, S.scan_in, &ies, &iep);
    }
    S.bes[tid] = ies;
    S.bep[tid] = iep;
    uint32_t w2 = 0, ies2 = 0, iep2 = 0;
    int32_t o2 = 0;
    if constexpr (kTwo) {
      w2 = S.in2.w[tid];
      o2 = S.in2.o[tid];
      if (w2 > 64) {
        flags |= HSZ_ERR_BAD_WIDTH;
        w2 = 0;
      }
      fast_in = fast_in && S.in2.staged && w2 <= static_cast<uint32_t>(kFastW) && o2 > -(1 << 29) &&
                o2 < (1 << 29);
      exact = block_offsets_or(w2, len, !fast_in, S.scan_in2, &ies2, &iep2);
      S.bes2[tid] = ies2;
      S.bep2[tid] = iep2;
    }
    // CTA-uniform: the register decode is warp-collective (decode_block)
    trace_tile(cur, 2);
    uint32_t qb[K];
    bool released = false;   // this warp's in_empty arrival of the tile is done
    bool over = false;       // scalar_mul: a rescaled bin beyond the register path
    if (!exact) {
      int32_t q[K];
      decode_block<0, kTwo>(S.in.sgn + S.in.soff + ies, S.in.pay + S.in.poff + iep, w, o, len, q);
      if constexpr (kOp == kOpSmul) {
        // this warp is done with the staged tile: the next one may load (a
        // tile that still turns out exact re-decodes from the header copies)
        mbar_arrive_warp(&S.in_empty);
        released = true;
        // rescale: |bin| < 2^30, |rs| < 2^23 -> bin * rs exact in float64;
        // then ops.py:199-208 verbatim
#pragma unroll
        for (int i = 0; i < K; ++i) {
          // int -> double by the conversion unit, then the exact product
          // (|bin * rs| < 2^53)
          const double pd = __dmul_rn(__int2double_rn(q[i]), sp.rsd);
          const double tt = __dmul_rn(sp.d, pd);
          // floor(RN(|t| + 1/2)): RN(|t| + 1/2) is exact here (|t| < 2^31), and
          // adding 2^52 rounding toward -inf leaves floor() in the low word
          const uint32_t mi = static_cast<uint32_t>(
              __double2loint(__dadd_rd(__dadd_rn(fabs(tt), 0.5), 4503599627370496.0)));
          over |= mi >= 1073741823u;
          qb[i] = tt < 0.0 ? 0u - mi : mi;
        }
      } else {
        // residual domain (ops.py:171-176): outlier sums |o_a +- o_b| < 2^30
        // and residual sums < 2^25 (the encoder's register path)
        decode_block<kOp == kOpSub ? 2 : 1, true>(S.in2.sgn + S.in2.soff + ies2,
                                             S.in2.pay + S.in2.poff + iep2, w2, o2, len, q);
#pragma unroll
        for (int i = 0; i < K; ++i) qb[i] = static_cast<uint32_t>(q[i]);
      }
    }
    trace_tile(cur, 3);
    uint32_t ts = 0, tp = 0;
    bool do_exact = exact;   // CTA-uniform
    if (!exact) {
      if (!released) {       // (per warp: in_empty counts warps, no CTA barrier needed)
        mbar_arrive_warp(&S.in_empty);
        released = true;
      }
      e32::BlockCode bc;
      if constexpr (kTwo)
        e32::block_code_resid(qb, bc);   // qb already holds the outlier and residuals
      else
        e32::block_code(qb, len, bc);
      const uint32_t wmax = __reduce_max_sync(kFull, bc.w);
      const uint32_t sb = (bc.w && active) ? ((static_cast<uint32_t>(len) + 7u) >> 3) : 0u;
      const uint32_t pb = (static_cast<uint32_t>(len) * bc.w + 7u) >> 3;
      uint32_t tot, ex;
      if constexpr (kOp == kOpSmul) {
        // the overflow report rides on the output scan's barrier
        ex = e32::cta_scan_or(sb | (pb << 10), over, S.scan, &tot, &do_exact);
      } else {
        ex = e32::cta_scan(sb | (pb << 10), S.scan, &tot);
      }
      if (k >= 2) mbar_wait_parity(&S.st_empty[par], ((k >> 1) - 1) & 1u);
      if (!do_exact) {
        const uint32_t es = ex & 1023u, ep = ex >> 10;
        ts = tot & 1023u;
        tp = tot >> 10;
        if (tid == 0) {
          lb_publish(lb_words(out.ws), cur, epoch, ts, tp);
          S.agg_ts[par] = ts;
          S.agg_tp[par] = tp;
          S.tile_of[par] = cur;
        }
        if (active) {
          out.widths[gb] = static_cast<uint8_t>(bc.w);
          out.outliers[gb] = static_cast<int32_t>(qb[0]);
        }
        if (sb) S.sgn[par][es >> 2] = bswap32(bc.sg);
        trace_tile(cur, 4);
        e32::pack_block<true>(bc, wmax, ep >> 2, reinterpret_cast<uint32_t*>(S.pk[par]));
        trace_tile(cur, 5);
      }
    } else {
      if (k >= 2) mbar_wait_parity(&S.st_empty[par], ((k >> 1) - 1) & 1u);
    }
    if (do_exact) {
      // exact warp-per-block path, decoding from global memory; places itself
      if constexpr (kOp == kOpSmul) {
        SrcSmulExact src{in, &S, sp.rs, sp.d};
        flags |= k32::fallback_sizes(src, out, cur, nblocks, in.tail_len, S.wsb, S.wpb);
      } else {
        SrcEwExact<kOp> src{in, in2, &S};
        flags |= k32::fallback_sizes(src, out, cur, nblocks, in.tail_len, S.wsb, S.wpb);
      }
      e32::bar_sync_n(1, kCompute);
      ts = S.wsb[0] + S.wsb[1] + S.wsb[2] + S.wsb[3];
      tp = S.wpb[0] + S.wpb[1] + S.wpb[2] + S.wpb[3];
      if (warp == 0) {
        if (lane == 0) {
          lb_publish(lb_words(out.ws), cur, epoch, ts, tp);
          S.agg_ts[par] = e32::kSelfPlaced;
        }
        __syncwarp();
        smul_resolve(S, out, cur, epoch, ntiles, ts, tp, par);
      }
      e32::bar_sync_n(1, kCompute);
      if (S.excl_s[par] != ~0ull) {
        uint64_t gs = S.excl_s[par], gp = S.excl_p[par];
        for (int i = 0; i < warp; ++i) {
          gs += S.wsb[i];
          gp += S.wpb[i];
        }
        if constexpr (kOp == kOpSmul) {
          SrcSmulExact src{in, &S, sp.rs, sp.d};
          k32::fallback_pack(src, out, cur, nblocks, in.tail_len, gs, gp,
                             reinterpret_cast<uint32_t*>(S.pk[par]) + warp * 64);
        } else {
          SrcEwExact<kOp> src{in, in2, &S};
          k32::fallback_pack(src, out, cur, nblocks, in.tail_len, gs, gp,
                             reinterpret_cast<uint32_t*>(S.pk[par]) + warp * 64);
        }
      }
      e32::bar_sync_n(1, kCompute);
      // the per-block offsets in S.bes/bep are no longer needed
      if (!released) mbar_arrive_warp(&S.in_empty);
    }
    mbar_arrive_warp(&S.st_full[par]);
    par ^= 1;
    ++k;
  }
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(out.err, flags);
}

template <int kOp>
constexpr uint32_t recode_smem_bytes() { return sizeof(RecodeSmem<kOp>) + 1024; }
constexpr uint32_t kSmulSmemBytes = recode_smem_bytes<kOpSmul>();

// ---------------------------------------------------------------------------
// Decode pipeline (moments, decompress to float32): persistent CTAs of 4
// compute warps + 1 TMA warp; tiles by grid stride (no ordering needed),
// input double-buffered.

// the moment kernels keep no bins in registers (decode_sum below), so they
// fit more CTAs per SM; their staging is sized for widths <= 16 (8 KB per
// tile, wider tiles take the in-place exact path)
#ifndef HSZ_F32_STREAM
#define HSZ_F32_STREAM 1
#endif
#ifndef HSZ_F32_PAYCAP
#define HSZ_F32_PAYCAP 8192
#endif
#ifndef HSZ_SUM_PAYCAP
#define HSZ_SUM_PAYCAP 8192
#endif
#ifndef HSZ_SUM_CTAS
#define HSZ_SUM_CTAS 8
#endif
#ifndef HSZ_DEC_SCAN_OR
#define HSZ_DEC_SCAN_OR 0
#endif
#ifndef HSZ_ACC64
#define HSZ_ACC64 1
#endif

// staged input tiles in flight per CTA (the moment kernels hold 8 KB of
// payload per tile: 3 buffers still fit 8 CTAs per SM)
#ifndef HSZ_SUM_NBUF
#define HSZ_SUM_NBUF 2
#endif
#ifndef HSZ_F32_NBUF
#define HSZ_F32_NBUF 2
#endif
template <int kMode>
struct DecSmem {
  static constexpr int kNB = kMode == 2 ? HSZ_F32_NBUF : HSZ_SUM_NBUF;
  using Tile = InTileT<kMode == 2 ? HSZ_F32_PAYCAP : HSZ_SUM_PAYCAP>;
  Tile in[kNB];
  alignas(1024) unsigned char out[kMode == 2 ? e32::kBufBytes : 16];   // decompress: value tile
  uint64_t full[kNB], empty[kNB];
  alignas(16) uint32_t scan[2][4];   // by tile parity: one CTA barrier per tile (cta_scan_or)
};
template <int kMode>
constexpr uint32_t dec_smem_bytes() { return sizeof(DecSmem<kMode>) + 1024; }
constexpr int kDecThreads = kCompute + 32;

// the 32-lane exact decode of one tile's blocks (any width up to 64, any
// outlier), reading the sections in place; calls f(local block, lane, bin,
// live) for every element
template <class IT, class F>
__device__ __forceinline__ uint32_t exact_tile(const StreamIn& in, const IT& it, uint32_t es,
                                               uint32_t ep, uint32_t w, int32_t o, int len, F&& f) {
  k32::TileIn t;
  t.w = w;
  t.o = o;
  t.len = len;
  t.soff = it.gs0 + es;
  t.poff = it.gp0 + ep;
  t.sgn = in.signs;
  t.pay = in.payload;
  t.fast = false;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t flags = 0;
  for (int j = 0; j < 32; ++j) {
    const k32::LaneBlock m = k32::lane_block(t, j);
    if (m.len == 0) break;
    const int64_t q = k32::decode_lane(t.sgn, t.pay, m.w, m.o, m.soff, m.poff, m.len, lane, &flags);
    f(warp * 32 + j, lane, q, lane < m.len);
  }
  return flags;
}

// exact moments of this CTA's compute threads -> the carry-save counters
// (same protocol as k32::finish_moments, over the 128 compute threads)
__device__ __forceinline__ void finish_moments_compute(k32::Acc acc, void* ws, uint64_t* out,
                                                       const Mailbox& mb, const uint32_t* err) {
  __shared__ k32::Acc s_acc[4];
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int m = 16; m > 0; m >>= 1) acc.merge(k32::shfl_xor_acc(acc, m));
  if (lane == 0) s_acc[warp] = acc;
  e32::bar_sync_n(1, kCompute);
  uint64_t* base = static_cast<uint64_t*>(ws);
  uint64_t* done = base + 2;
  uint64_t* cs = base + 8;
  if (threadIdx.x == 0) {
    k32::Acc t = s_acc[0];
    for (int i = 1; i < 4; ++i) t.merge(s_acc[i]);
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
      for (int k = 0; k < 4; ++k) k32::add_shifted(S, 2, ld_relaxed(cs + k), 32 * k);
      for (int k = 0; k < 6; ++k) k32::add_shifted(Q, 4, ld_relaxed(cs + 4 + k), 32 * k);
      out[0] = S[0];
      out[1] = S[1];
      out[2] = Q[0];
      out[3] = Q[1];
      out[4] = Q[2];
      for (int k = 0; k < 10; ++k) st_relaxed(cs + k, 0);
      st_relaxed(done, 0);
      const uint64_t res[5] = {S[0], S[1], Q[0], Q[1], Q[2]};
      mailbox_post(mb, res, 5, err);
    }
  }
}

struct MomentsSink {
  uint64_t* out;
  void* ws;
  Mailbox mb;
};
struct DecF32Sink {
  float* out;
  double d;
  bool may_overflow;
};

template <class Sink>
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

// kMode 0: mean (S), 1: variance (S, Q), 2: decompress to float32
template <int kMode>
#ifndef HSZ_DEC_CTAS
#define HSZ_DEC_CTAS 6
#endif
__global__ void __launch_bounds__(kDecThreads, kMode == 2 ? HSZ_DEC_CTAS : HSZ_SUM_CTAS)
    decode_pipe_kernel(const __grid_constant__ CUtensorMap omap, StreamIn in, DecF32Sink fs,
                       MomentsSink ms, int use_tma, uint32_t* err) {
  extern __shared__ unsigned char smraw[];
  const uint32_t a0 = smem_u32(smraw);
  DecSmem<kMode>& S = *reinterpret_cast<DecSmem<kMode>*>(smraw + (((a0 + 1023u) & ~1023u) - a0));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t ntiles = in.ntiles, nblocks = in.nblocks;
  constexpr int kNB = DecSmem<kMode>::kNB;
  if (tid == kCompute) {
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&S.full[b], 1);
      mbar_init(&S.empty[b], kCompute / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == kCompute / 32) {
    // ============================ TMA warp ==============================
    uint32_t i = 0;
    uint64_t tv = prefetch_toff(in, blockIdx.x);
    for (uint64_t t = blockIdx.x;; t += gridDim.x, ++i) {
      const int b = i % kNB;
      const uint64_t tvn = prefetch_toff(in, t + gridDim.x);   // consumed next iteration
      if (i >= kNB) mbar_wait_parity_sleep(&S.empty[b], ((i / kNB) - 1) & 1u);
      stage_tile(in, t, tv, S.in[b], &S.full[b]);
      if (t >= ntiles) break;
      tv = tvn;
    }
    return;
  }
  // =========================== compute warps ===========================
  uint32_t flags = 0;
  k32::Acc acc;
  acc.s = 0;
  acc.q = 0;
  acc.q2 = 0;
  uint32_t i = 0;
  for (;; ++i) {
    const int b = i % kNB;
    mbar_wait_parity(&S.full[b], (i / kNB) & 1u);
    const auto& it = S.in[b];
    const uint64_t cur = it.tile;
    if (cur >= ntiles) break;
    const uint64_t gb = cur * TB + tid;
    const bool active = gb < nblocks;
    const int len = !active ? 0 : (gb == nblocks - 1 ? static_cast<int>(in.tail_len) : K);
    uint32_t w = it.w[tid];
    const int32_t o = it.o[tid];
    if (w > 64) {
      flags |= HSZ_ERR_BAD_WIDTH;
      w = 0;
    }
    const uint32_t isb = w ? ((static_cast<uint32_t>(len) + 7u) >> 3) : 0u;
    const uint32_t ipb = (static_cast<uint32_t>(len) * w + 7u) >> 3;
    uint32_t itot;
    const bool slow = !(it.staged && w <= static_cast<uint32_t>(kFastW) && o > -(1 << 29) && o < (1 << 29));
#if HSZ_DEC_SCAN_OR
    // the in-tile offsets and the CTA-uniform path choice on ONE barrier
    // (measured: no gain for the moment kernels, 3-4% slower for variance and
    // decompress on config 4 -- off by default)
    bool any_slow;
    const uint32_t iex = e32::cta_scan_or(isb | (ipb << 10), slow, S.scan[i & 1u], &itot, &any_slow);
    const bool fast = !any_slow;
#else
    const uint32_t iex = e32::cta_scan(isb | (ipb << 10), S.scan[0], &itot);
    const bool fast = e32::bar_or_compute(slow) == false;
#endif
    const uint32_t ies = iex & 1023u, iep = iex >> 10;
    if (kMode == 2 && i > 0 && tid == 0) {
      // the previous tile's TMA store has finished reading S.out
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    if (kMode == 2) e32::bar_sync_n(1, kCompute);
    if (fast && kMode != 2) {
      int64_t sp;
      uint64_t sp2;
      decode_sum<kMode == 1>(it.sgn + it.soff + ies, it.pay + it.poff + iep, w, len, &sp, &sp2);
      mbar_arrive_warp(&S.empty[b]);          // staged bytes consumed
      if (len > 0) {
#if HSZ_ACC64
        // block sums in 64 bits where they provably fit (|o| < 2^29 on this
        // path): S_b = len o + sum P, |S_b| < 2^36; and for widths <= 16
        // (|P| < 2^21, |sum P| < 2^26) Q_b = sum (o + P)^2 <= 32 (2^29 + 2^21)^2
        // < 2^64, so its three terms add exactly modulo 2^64.  The 128-bit
        // products cost ~40 instructions a block.
        acc.s += static_cast<int64_t>(o) * len + sp;
        if (kMode == 1) {
          unsigned __int128 tot;
          if (w <= 16u) {
            const uint64_t o2 = static_cast<uint64_t>(static_cast<int64_t>(o) * o);
            tot = o2 * static_cast<uint64_t>(len) +
                  static_cast<uint64_t>(2 * static_cast<int64_t>(o) * sp) + sp2;
          } else {
            const __int128 oo = o;
            tot = static_cast<unsigned __int128>(oo * oo * len + 2 * oo * sp + static_cast<__int128>(sp2));
          }
          const unsigned __int128 nq = acc.q + tot;
          acc.q2 += nq < acc.q ? 1u : 0u;
          acc.q = nq;
        }
#else
        const __int128 oo = o;
        acc.s += oo * len + sp;
        if (kMode == 1) {
          const __int128 tot = oo * oo * len + 2 * oo * sp + static_cast<__int128>(sp2);
          const unsigned __int128 nq = acc.q + static_cast<unsigned __int128>(tot);
          acc.q2 += nq < acc.q ? 1u : 0u;
          acc.q = nq;
        }
#endif
      }
    } else if (fast && HSZ_F32_STREAM) {
      decode_f32(it.sgn + it.soff + ies, it.pay + it.poff + iep, w, o, len, fs.d, S.out + tid * 128,
                 static_cast<uint32_t>(tid & 7), fs.may_overflow, &flags);
      mbar_arrive_warp(&S.empty[b]);          // staged bytes consumed
    } else if (fast) {
      int32_t q[K];
      decode_block(it.sgn + it.soff + ies, it.pay + it.poff + iep, w, o, len, q);
      mbar_arrive_warp(&S.empty[b]);          // staged bytes consumed
      if (kMode == 2) {
        // f32 values = RN32(RN64(2eps * bin)) (codec.py:107-115), into the
        // swizzled 128-byte row of this block
        float v[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          v[k] = __double2float_rn(__dmul_rn(fs.d, i32_to_double(q[k])));
          if (fs.may_overflow && !isfinite(v[k])) flags |= HSZ_ERR_OUTPUT_NONFINITE;
        }
        unsigned char* row = S.out + tid * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(row + ((j ^ (tid & 7)) << 4)) =
              make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      } else if (len > 0) {
        // block sums: S_b = sum bin, Q_b = sum bin^2 with bin = o + P_i
        int64_t sp = 0;
        uint64_t sp2 = 0;
        if (len == K) {
          int64_t sp32 = 0;   // sum P reaches 496 * 2^24 > 2^31
#pragma unroll
          for (int k = 1; k < K; ++k) {
            const int32_t P = q[k] - o;   // |P| < 2^29
            sp32 += P;
            if (kMode == 1) sp2 += static_cast<uint64_t>(static_cast<int64_t>(P) * P);
          }
          sp = sp32;
        } else {
#pragma unroll
          for (int k = 1; k < K; ++k) {
            const int32_t P = q[k] - o;
            if (k < len) {
              sp += P;
              if (kMode == 1) sp2 += static_cast<uint64_t>(static_cast<int64_t>(P) * P);
            }
          }
        }
        const __int128 oo = o;
        acc.s += oo * len + sp;
        if (kMode == 1) {
          const __int128 tot = oo * oo * len + 2 * oo * sp + static_cast<__int128>(sp2);
          const unsigned __int128 nq = acc.q + static_cast<unsigned __int128>(tot);
          acc.q2 += nq < acc.q ? 1u : 0u;
          acc.q = nq;
        }
      }
    } else {
      // exact lane-per-element path, sections read in place
      if (kMode == 2) {
        flags |= exact_tile(in, it, ies, iep, w, o, len, [&](int lb, int ln, int64_t q, bool live) {
          if (live) {
            const float v = __double2float_rn(grid1(q, fs.d));
            if (!isfinite(v)) flags |= HSZ_ERR_OUTPUT_NONFINITE;
            fs.out[(cur * TB + lb) * K + ln] = v;
          }
        });
      } else {
        flags |= exact_tile(in, it, ies, iep, w, o, len, [&](int, int, int64_t q, bool live) {
          if (live) acc.add(q, kMode == 1);
        });
      }
      mbar_arrive_warp(&S.empty[b]);
    }
    if (kMode == 2) {
      // one TMA tensor store of the whole tile (the stream's partial last
      // block and rows past the end are written by plain stores / clipped)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      e32::bar_sync_n(1, kCompute);
      if (fast) {
        const uint64_t full_rows = in.n / K;
        const uint64_t row0 = cur * TB;
        if (use_tma) {
          if (tid == 0) {
            tma_store_2d<DecF32Sink>(&omap, S.out, 0, static_cast<int>(row0));
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else {
          for (uint32_t e = tid; e < TB * K; e += kCompute) {
            const uint64_t g = row0 * K + e;
            if (g < full_rows * K) fs.out[g] = *reinterpret_cast<const float*>(S.out + e32::swz_elem(e >> 5, e & 31u));
          }
        }
        if ((in.n % K) != 0 && full_rows >= row0 && full_rows < row0 + TB && tid < static_cast<int>(in.n % K)) {
          const uint32_t r = static_cast<uint32_t>(full_rows - row0);
          fs.out[full_rows * K + tid] = *reinterpret_cast<const float*>(S.out + e32::swz_elem(r, tid));
        }
      }
    }
  }
  if (kMode == 2 && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(err, flags);   // before the completion count: the last CTA reports it
  if (kMode != 2) finish_moments_compute(acc, ms.ws, ms.out, ms.mb, err);
}

}  // namespace d32
}  // namespace hsz
