// Register-resident block_len-32 encoder (compress of float32 fields).
//
// A tile = 128 blocks (4096 elements); a CTA of 128 threads works on one tile
// at a time and thread b owns block b, keeping its 32 bins in registers from
// quantization to bit packing:
//
//   1. the tile (16 KB) arrives in shared memory by one TMA 2-D tensor load
//      with the 128-byte swizzle, so thread b's eight 16-byte reads of its
//      own 128-byte row hit eight different bank groups (conflict free);
//      as soon as the registers hold it, the next tile's load is issued
//      into the same buffer;
//   2. certified float32 quantization (quant_f32 below) -- bit-identical to
//      the reference's float64 floor((x + eps) / 2eps) + repair pass
//      (codec.py:118-155) whenever its certificate holds, the exact float64
//      path (hsz_quant.cuh quantize1) for the ~2^-20 of elements where it
//      does not;
//   3. Lorenzo residuals, OR-reduced width and the big-endian sign word
//      (one funnel shift per element) in registers (codec.py:178-225);
//   4. one 32-bit CTA scan of the (sign bytes, payload bytes) of the 128
//      blocks; the tile aggregate is published for the decoupled look-back
//      at once (fence-free tagged words, hsz_common.cuh lb_*);
//   5. the PREVIOUS tile of this CTA is placed: warp 0 resolves its global
//      offsets (its predecessors had a whole iteration to publish theirs, so
//      the look-back rarely waits) and the CTA streams its staged sign words
//      and payload out with 16-byte stores;
//   6. MSB-first element-major packing (codec.py:280-286) of the current
//      tile -- G = 4 / 2 / 1 fields combined per IMAD step, G chosen per warp
//      from its widest block -- into the staging buffer (row-XOR swizzle).
//
// The grid is persistent (every CTA resident); tiles are handed out in order
// by an atomic ticket drawn one tile ahead, so every wait of the look-back is
// on a lower ticket whose owner can always progress.
//
// Tiles holding a bin with |bin| >= 2^30 (only possible for eps tiny against
// the data) fall back to the exact warp-per-block encoder of hsz_k32.cuh.
#pragma once

#include <cuda.h>

#include "hsz_common.cuh"
#include "hsz_k32.cuh"
#include "hsz_quant.cuh"

namespace hsz {
namespace e32 {

constexpr int K = 32;
constexpr int TB = kTileBlocks;                  // 128 blocks per tile
constexpr int kThreads = TB;                     // one thread per block
constexpr uint32_t kBufBytes = TB * K * 4;       // 16 KB: input tile, then packed payload
constexpr uint32_t kMagicBits = 0x4B400000u;     // bits of 1.5 * 2^23
constexpr float kMagicF = 12582912.0f;           // 1.5 * 2^23
constexpr int64_t kWide = 1ll << 30;             // register path: |bin| < 2^30

static_assert(kThreads == 128, "the CTA scan assumes 4 warps");

// ---------------------------------------------------------------------------
// certified float32 quantizer
//
// t = x/d + 1/2 (d = 2 eps); the reference returns floor(RN(RN(x + eps) / d))
// (+ a repair pass).  With R = RN64(1/d) split as rh + rl (two floats):
//   p = RN(x*rh), e = x*rh - p (exact FMA), m = floor(p), f = p - m,
//   c = RN(x*rl + e), v = RN(RN(f - 1/2) + c)  ~  t - m - 1
// |v - (t - m - 1)| < 2^-23 for |p| < 2^21 (error analysis in DESIGN.md), so
// if |v| > 2^-21 then t is at least 2^-22 away from the integer m + 1,
// floor(t) = m + [v >= 0] equals the reference's floor (whose own error is
// below 2^-31 here), and |x - d q| <= eps - d 2^-22 proves that the repair
// pass of codec.py:140-154 does not fire.  Returns the bin offset by the
// magic constant: bits(m + 1.5*2^23) + [v >= 0] = 0x4B400000 + floor(t).
// (A round-to-nearest variant without FRND was tried: products that are
// exact half-integers, 2^-10 of them at |p| ~ 2^13, land on its certificate
// boundary and push whole warps into the slow path -- 40% slower.)
struct QuantF32 {
  float rh, rl;
  float delta;   // > 0 enables the fast path (else every element takes quantize1)
};

__host__ inline QuantF32 make_quant_f32(const QuantConst& c) {
  QuantF32 q;
  const double R = 1.0 / c.d;
  q.rh = static_cast<float>(R);
  q.rl = static_cast<float>(R - static_cast<double>(q.rh));
  const bool ok = c.d >= 0x1p-60 && c.d <= 0x1p+60;
  q.delta = ok ? 0x1p-21f : -1.0f;
  return q;
}

__device__ __forceinline__ uint32_t quant_f32(float x, const QuantF32& qf, bool& bad) {
  const float p = __fmul_rn(x, qf.rh);
  const float e = __fmaf_rn(x, qf.rh, -p);
  const float m = floorf(p);
  const float f = __fsub_rn(p, m);
  const float c = __fmaf_rn(x, qf.rl, e);
  const float v = __fadd_rn(__fsub_rn(f, 0.5f), c);
  bad |= !((fabsf(v) > qf.delta) & (fabsf(p) < 2097152.0f) & (qf.delta > 0.0f));
  const uint32_t mb = __float_as_uint(__fadd_rn(m, kMagicF));
  return mb + 1u + static_cast<uint32_t>(__float_as_int(v) >> 31);
}

// The same quantizer for the hot loop: the certificate of a whole row is
// tested once, on the smallest |v| and the largest |p| of its 32 elements --
// a three-input FMNMX3 folds two elements' magnitudes per instruction, where
// the per-element form spends two FSETP and half a PLOP3 (48 instructions a
// block less).  The maximum propagates NaN (a NaN or infinite x fails the
// test like before; v is only non-finite when p is).
__device__ __forceinline__ float max3_nan_abs(float a, float b, float c) {
  float r;
  asm("{\n\t.reg .f32 x, y;\n\tabs.f32 x, %2;\n\tabs.f32 y, %3;\n\tmax.NaN.f32 %0, %1, x, y;\n}"
      : "=f"(r)
      : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ uint32_t quant_f32m(float x, const QuantF32& qf, float& vmin, float& pout) {
  const float p = __fmul_rn(x, qf.rh);
  const float e = __fmaf_rn(x, qf.rh, -p);
  const float m = floorf(p);
  const float f = __fsub_rn(p, m);
  const float c = __fmaf_rn(x, qf.rl, e);
  const float v = __fadd_rn(__fsub_rn(f, 0.5f), c);
  vmin = fminf(vmin, fabsf(v));
  pout = p;
  const uint32_t mb = __float_as_uint(__fadd_rn(m, kMagicF));
  return mb + 1u + static_cast<uint32_t>(__float_as_int(v) >> 31);
}

struct ExactQ {
  int64_t q;
  uint32_t flags;
};

__device__ __noinline__ ExactQ quant_exact(float x, QuantConst c) {
  ExactQ r;
  r.flags = 0;
  r.q = quantize1(static_cast<double>(x), c, &r.flags);
  return r;
}

// ---------------------------------------------------------------------------
// shared memory

struct Smem {
  unsigned char in[kBufBytes];    // input tile (TMA 128B swizzle; 1024-aligned)
  unsigned char pk[2][kBufBytes]; // packed payload of the staged tiles (word swizzle; by parity)
  alignas(16) uint32_t sgn[2][TB];  // their sign words (compacted)
  uint64_t bar;                   // input full (TMA or "no more tiles")
  uint64_t in_empty;              // compute warps consumed S.in        (128 arrivals)
  uint64_t st_full[2];            // tile staged in pk[b]                (128 arrivals)
  uint64_t st_empty[2];           // pk[b] copied out by the copy warp      (1 arrival)
  uint64_t tile_of[2];            // tile id staged in pk[b]
  uint64_t cur, epoch;
  uint64_t excl_s[2], excl_p[2];  // resolved offsets of the staged tile (service warp; by parity)
  uint32_t agg_ts[2], agg_tp[2];  // aggregate of the current tile (compute warps; by parity)
  uint32_t scan[4];
  uint32_t wsb[4], wpb[4];
};
constexpr uint32_t kSmemBytes = sizeof(Smem) + 1024;   // + alignment slack

__device__ __forceinline__ Smem& smem_at(unsigned char* raw) {
  const uint32_t a = smem_u32(raw);
  return *reinterpret_cast<Smem*>(raw + (((a + 1023u) & ~1023u) - a));
}

// element i of tile row r in the 128B-swizzled tile image
__device__ __forceinline__ uint32_t swz_elem(uint32_t r, uint32_t i) {
  return r * 128u + ((((i >> 2) ^ (r & 7u)) << 4) | ((i & 3u) << 2));
}

// payload staging: logical word a at a ^ row(a) within its 32-word row
__device__ __forceinline__ uint32_t swz_word(uint32_t a) { return a ^ ((a >> 5) & 31u); }

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// named barriers: 1 = the 128 compute threads, 2 = "input consumed"
// (compute arrive, service sync), 3 = "offsets ready" (all 160 threads)
constexpr int kCompute = 128;
constexpr int kThreadsWS = kCompute + 64;   // + TMA warp (tickets, loads) + placement warp
#ifndef HSZ_ENC_CTAS
#define HSZ_ENC_CTAS 4   // CTAs per SM the register budget is sized for
#endif
__device__ __forceinline__ void bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ bool bar_or_compute(bool p) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred q, o;\n\tsetp.ne.u32 q, %1, 0;\n\t"
      "bar.red.or.pred o, 1, 128, q;\n\tselp.u32 %0, 1, 0, o;\n}"
      : "=r"(r)
      : "r"(static_cast<uint32_t>(p))
      : "memory");
  return r != 0;
}

// exclusive scan of one u32 over the 128 compute threads; *total = sum
__device__ __forceinline__ uint32_t cta_scan(uint32_t v, uint32_t* s_scan, uint32_t* total) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(kFull, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) s_scan[warp] = inc;
  bar_sync_n(1, kCompute);
  const uint32_t a0 = s_scan[0], a1 = s_scan[1], a2 = s_scan[2], a3 = s_scan[3];
  const uint32_t pre = (warp > 0 ? a0 : 0u) + (warp > 1 ? a1 : 0u) + (warp > 2 ? a2 : 0u);
  *total = a0 + a1 + a2 + a3;
  return pre + inc - v;
}

// the same scan with a CTA-wide OR of `flag` riding on its one barrier: each
// warp's total carries any(flag) of the warp in bit 31 (the sums stay below
// 2^26).  Callers whose next use of `s_scan` is not separated from this one
// by another barrier alternate between two buffers.
__device__ __forceinline__ uint32_t cta_scan_or(uint32_t v, bool flag, uint32_t* s_scan,
                                                uint32_t* total, bool* any) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(kFull, inc, d);
    if (lane >= d) inc += o;
  }
  const bool wany = __any_sync(kFull, flag);
  if (lane == 31) s_scan[warp] = inc | (wany ? 0x80000000u : 0u);
  bar_sync_n(1, kCompute);
  const uint4 a = *reinterpret_cast<const uint4*>(s_scan);
  *any = ((a.x | a.y | a.z | a.w) >> 31) != 0;
  const uint32_t a0 = a.x & 0x7fffffffu, a1 = a.y & 0x7fffffffu, a2 = a.z & 0x7fffffffu,
                 a3 = a.w & 0x7fffffffu;
  const uint32_t pre = (warp > 0 ? a0 : 0u) + (warp > 1 ? a1 : 0u) + (warp > 2 ? a2 : 0u);
  *total = a0 + a1 + a2 + a3;
  return pre + inc - v;
}

// ---------------------------------------------------------------------------
// per-thread block encoding

struct BlockCode {
  uint32_t mg[K];   // residual magnitudes (mg[0] = 0: slot 0 holds the outlier)
  uint32_t sg;      // sign bits, element i at bit 31 - i
  uint32_t w;       // width
};

// residuals (codec.py:178-212), width (codec.py:215-225), sign word
__device__ __forceinline__ void block_code(uint32_t (&qb)[K], int len, BlockCode& bc) {
  if (len < K) {   // the stream's tail block (or no block): replicate the last live bin
#pragma unroll
    for (int i = 1; i < K; ++i) qb[i] = (i < len) ? qb[i] : qb[i - 1];
  }
  uint32_t mx = 0, sg = 0;
  bc.mg[0] = 0;
#pragma unroll
  for (int i = 1; i < K; ++i) {
    const int32_t d = static_cast<int32_t>(qb[i] - qb[i - 1]);
    sg = __funnelshift_l(static_cast<uint32_t>(d), sg, 1);
    bc.mg[i] = static_cast<uint32_t>(d < 0 ? -d : d);
    mx |= bc.mg[i];
  }
  bc.sg = sg;
  bc.w = 32u - __clz(mx);
}

// the same from signed residuals (qb[0] = the outlier, qb[i] = d_i; zero past
// a tail block's length)
__device__ __forceinline__ void block_code_resid(const uint32_t (&qb)[K], BlockCode& bc) {
  uint32_t mx = 0, sg = 0;
  bc.mg[0] = 0;
#pragma unroll
  for (int i = 1; i < K; ++i) {
    const int32_t d = static_cast<int32_t>(qb[i]);
    sg = __funnelshift_l(static_cast<uint32_t>(d), sg, 1);
    bc.mg[i] = static_cast<uint32_t>(d < 0 ? -d : d);
    mx |= bc.mg[i];
  }
  bc.sg = sg;
  bc.w = 32u - __clz(mx);
}

#ifndef HSZ_PACK_G3
#define HSZ_PACK_G3 0
#endif
#ifndef HSZ_QUANT_MINMAX
#define HSZ_QUANT_MINMAX 1
#endif

// MSB-first w-bit fields, G fields combined per step (G * w < 32)
template <int G>
__device__ __forceinline__ void pack_fields(const BlockCode& bc, uint32_t a, uint32_t* pbuf) {
  const uint32_t w = bc.w;
  const uint32_t pw = 1u << w, pg = 1u << (G * w);
  uint32_t acc = 0;
  int nbm = -32;   // pending bits - 32
#pragma unroll
  for (int c = 0; c < (K + G - 1) / G; ++c) {
    constexpr int kLast = K - ((K + G - 1) / G - 1) * G;   // fields in the last group
    const int gn = (c == (K + G - 1) / G - 1) ? kLast : G;
    uint32_t chunk = bc.mg[c * G];
#pragma unroll
    for (int g = 1; g < G; ++g)
      if (g < gn) chunk = chunk * pw + bc.mg[c * G + g];
    const uint64_t t = static_cast<uint64_t>(acc) * (gn == G ? pg : (1u << (gn * w))) + chunk;
    nbm += gn * static_cast<int>(w);
    if (nbm >= 0) {
      pbuf[swz_word(a)] = bswap32(static_cast<uint32_t>(t >> nbm));
      ++a;
      nbm -= 32;
    }
    acc = static_cast<uint32_t>(t);
  }
  if (nbm > -32) pbuf[swz_word(a)] = bswap32(acc << (-nbm));   // partial tail block
}

// wmax = __reduce_max_sync over the warp (warp-uniform grouping; computed by
// the caller early so its latency overlaps other work).  kG3: three-field
// groups for widths 8-10 -- the recode kernels gain 2-4% from them (their
// outputs are a few bits wider than a compressor's), the compressor, at its
// register limit, loses 1%
template <bool kG3 = (HSZ_PACK_G3 != 0)>
__device__ __forceinline__ void pack_block(const BlockCode& bc, uint32_t wmax, uint32_t a,
                                           uint32_t* pbuf) {
  if (bc.w == 0) return;
  if (wmax <= 7) {
    pack_fields<4>(bc, a, pbuf);
  } else if (kG3 && wmax <= 10) {
    pack_fields<3>(bc, a, pbuf);
  } else if (wmax <= 15) {
    pack_fields<2>(bc, a, pbuf);
  } else {
    pack_fields<1>(bc, a, pbuf);
  }
}

// ---------------------------------------------------------------------------
// placement of the staged tile (compute threads; offsets from the service warp)

constexpr uint32_t kSelfPlaced = 0xFFFFFFFFu;   // agg_ts marker: exact-path tile placed itself
constexpr uint32_t kDone = 0xFFFFFFFEu;         // agg_ts marker: no more tiles (copy warp exits)

// copy a staged tile to its resolved offsets; `rank`/`nthr` = this thread's
// index among the threads sharing the copy
__device__ __forceinline__ void copy_staged(Smem& S, const k32::EncodeOut& out, uint32_t ts,
                                            uint32_t tp, int par, uint32_t rank, uint32_t nthr) {
  const uint64_t es = S.excl_s[par], ep = S.excl_p[par];
  if (es == ~0ull) return;   // capacity exceeded (flagged)
  // sign words: offsets are multiples of 4 (the stream's tail block is last)
  uint32_t* dsg = reinterpret_cast<uint32_t*>(out.signs + es);
  for (uint32_t i = rank; i < ((ts + 3u) >> 2); i += nthr) dsg[i] = S.sgn[par][i];
  // payload: 16-byte stores from the first 16-byte aligned destination word
  const uint32_t* pbuf = reinterpret_cast<const uint32_t*>(S.pk[par]);
  uint32_t* dst = reinterpret_cast<uint32_t*>(out.payload + ep);
  const uint32_t nw = (tp + 3u) >> 2;
  uint32_t head = static_cast<uint32_t>(((16u - (ep & 15u)) & 15u) >> 2);
  head = head < nw ? head : nw;
  if (rank < head) dst[rank] = pbuf[swz_word(rank)];
  const uint32_t nv = (nw - head) >> 2;
  uint4* dv = reinterpret_cast<uint4*>(dst + head);
  for (uint32_t i = rank; i < nv; i += nthr) {
    const uint32_t k = head + 4u * i;
    dv[i] = make_uint4(pbuf[swz_word(k)], pbuf[swz_word(k + 1)], pbuf[swz_word(k + 2)],
                       pbuf[swz_word(k + 3)]);
  }
  const uint32_t rest = head + 4u * nv + rank;
  if (rest < nw) dst[rest] = pbuf[swz_word(rest)];
}

// one warp: resolve `tile` and record its offsets (+ the tile-offset cache)
__device__ __forceinline__ void resolve_tile(Smem& S, const k32::EncodeOut& out, uint64_t tile,
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

// ---------------------------------------------------------------------------
// compress, float32 input, block_len 32
//
// Persistent, warp-specialised: warps 0-3 compute (thread b = block b of the
// current tile), warp 4 issues the TMA tile loads (tickets drawn one ahead),
// warp 5 places staged tiles (look-back + copy-out).  Per tile k:
//
//   compute:   wait full[k&1] | quantize | arrive in_empty[k&1] | code, scan,
//              publish | claim slot k%4 and ring space | pack into the ring
//              | arrive st_full[slot]
//   TMA:       wait in_empty (tile k-1's buffer) | TMA(tile k+1) | draw
//   placement: wait st_full[slot] | resolve | copy out | free ring space
//              | arrive st_empty[slot]
//
// Input tiles are double-buffered (the next load overlaps a whole tile of
// compute); staged payloads live in a 16 KB byte ring sized by the actual
// payload (4-5 KB typical, 15.9 KB worst case), so up to 4 tiles can wait
// for their offsets without stalling the compute warps.

#ifndef HSZ_RING_BYTES
#define HSZ_RING_BYTES 16384
#endif
constexpr uint32_t kRingBytes = HSZ_RING_BYTES;
#ifndef HSZ_RING_SLOTS
#define HSZ_RING_SLOTS 4
#endif
constexpr int kSlots = HSZ_RING_SLOTS;

struct RingRec {
  uint64_t tile;
  uint64_t end;    // ring bytes allocated up to and including this tile
  uint32_t ts, tp;
  uint32_t off;    // byte offset of the tile's payload in the ring (128-aligned)
  uint32_t pad;
};

struct Smem6 {
  unsigned char in[2][kBufBytes];   // input tiles (TMA 128B swizzle; 1024-aligned)
  unsigned char ring[kRingBytes];   // staged payloads (row-XOR word swizzle per 128 B row)
  alignas(16) uint32_t sgn[kSlots][TB];
  uint64_t full[2], in_empty[2];
  uint64_t st_full[kSlots], st_empty[kSlots];
  uint64_t cur[2];
  uint64_t excl_s[kSlots], excl_p[kSlots];
  RingRec rec[kSlots];
  volatile uint64_t ring_tail;      // bytes of the ring freed (placement warp)
  uint64_t epoch;
  uint32_t alloc_off;
  uint32_t scan[4];
  uint32_t wsb[4], wpb[4];
  uint32_t xscratch[4][64];         // exact path: one block's packed words per warp
};
constexpr uint32_t kSmem6Bytes = sizeof(Smem6) + 1024;

__device__ __forceinline__ void copy_ring(const uint32_t* sgn, const unsigned char* ring,
                                          const k32::EncodeOut& out, const RingRec& r, uint64_t es,
                                          uint64_t ep) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t* dsg = reinterpret_cast<uint32_t*>(out.signs + es);
  for (uint32_t i = lane; i < ((r.ts + 3u) >> 2); i += 32) dsg[i] = sgn[i];
  const uint32_t* pbuf = reinterpret_cast<const uint32_t*>(ring + r.off);
  uint32_t* dst = reinterpret_cast<uint32_t*>(out.payload + ep);
  const uint32_t nw = (r.tp + 3u) >> 2;
  uint32_t head = static_cast<uint32_t>(((16u - (ep & 15u)) & 15u) >> 2);
  head = head < nw ? head : nw;
  if (lane < head) dst[lane] = pbuf[swz_word(lane)];
  const uint32_t nv = (nw - head) >> 2;
  uint4* dv = reinterpret_cast<uint4*>(dst + head);
  for (uint32_t i = lane; i < nv; i += 32) {
    const uint32_t k = head + 4u * i;
    dv[i] = make_uint4(pbuf[swz_word(k)], pbuf[swz_word(k + 1)], pbuf[swz_word(k + 2)],
                       pbuf[swz_word(k + 3)]);
  }
  const uint32_t rest = head + 4u * nv + lane;
  if (rest < nw) dst[rest] = pbuf[swz_word(rest)];
}

// one warp: resolve `tile`; returns the offsets (~0 sign offset: over capacity)
__device__ __forceinline__ void resolve6(const k32::EncodeOut& out, uint64_t tile, uint64_t epoch,
                                         uint64_t ntiles, uint32_t ts, uint32_t tp, uint64_t* es_out,
                                         uint64_t* ep_out) {
  const int lane = threadIdx.x & 31;
  uint64_t es, ep;
  lb_resolve(lb_words(out.ws), tile, epoch, ts, tp, &es, &ep, out.err);
  const bool fits = es + ts <= out.sign_cap && ep + tp <= out.payload_cap;
  if (lane == 0) {
    out.toff[2 * tile] = es;
    out.toff[2 * tile + 1] = ep;
    if (tile == ntiles - 1) {
      out.toff[2 * ntiles] = es + ts;
      out.toff[2 * ntiles + 1] = ep + tp;
    }
    if (!fits) atomicOr(out.err, HSZ_ERR_CAPACITY);
  }
  *es_out = fits ? es : ~0ull;
  *ep_out = ep;
}

// v7: 4 compute warps + 1 placement warp (160 threads, 4 CTAs per SM).  The
// compute warps' thread 0 issues the next tile's TMA load as soon as the CTA
// has read the current tile (single input buffer) and draws tickets one tile
// ahead; placement and the staging ring are as described above.
constexpr int kThreadsC = kCompute + 32;
// (4 CTAs per SM at 96 registers, no spills: 178 us on config 4 against 183
// at 5 CTAs / 72 registers with ~100 B of spills, 195 at 3)
#ifndef HSZ_CMP_CTAS
#define HSZ_CMP_CTAS 4
#endif

template <uint32_t kInBytes>
struct Smem7T {
  unsigned char in[kInBytes];       // input tile (TMA 128B swizzle; 1024-aligned)
  unsigned char ring[kRingBytes];   // staged payloads (row-XOR word swizzle per 128 B row)
  alignas(16) uint32_t sgn[kSlots][TB];
  uint64_t full;
  uint64_t st_full[kSlots], st_empty[kSlots];
  uint64_t cur;
  uint64_t excl_s[kSlots], excl_p[kSlots];
  RingRec rec[kSlots];
  volatile uint64_t ring_tail;      // bytes of the ring freed (placement warp)
  uint64_t epoch;
  uint32_t alloc_off;
  alignas(16) uint32_t scan[4];
  uint32_t wsb[4], wpb[4];
  uint32_t xscratch[4][64];         // exact path: one block's packed words per warp
};
using Smem7 = Smem7T<kBufBytes>;
constexpr uint32_t kSmem7Bytes = sizeof(Smem7) + 1024;
// encode_from_quant: an int64 bin tile is 32 KB
using Smem7Bins = Smem7T<2 * kBufBytes>;
constexpr uint32_t kSmem7BinsBytes = sizeof(Smem7Bins) + 1024;
#ifndef HSZ_BINS_CTAS
#define HSZ_BINS_CTAS 4
#endif

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

template <class Src>
__device__ __forceinline__ Src make_exact_src(const float* x, const int64_t* xb, uint64_t n,
                                              const QuantConst& qc, uint64_t tile) {
  if constexpr (std::is_same_v<Src, k32::SrcBins>) {
    (void)x;
    (void)qc;
    return k32::SrcBins{xb, n, tile};
  } else {
    (void)xb;
    return Src{x, n, qc, tile};
  }
}

// byte offset of bin i of tile block r in the staged int64 tile: the TMA
// view is [half][block][16 bins] (3-D map, dims reordered), 128-byte rows
// swizzled by (row & 7) = (block & 7), so the 8 threads of a wavefront read
// 8 distinct bank groups
__device__ __forceinline__ uint32_t bins_off(uint32_t r, uint32_t i) {
  const uint32_t h = i >> 4, e = i & 15u;
  return (h * TB + r) * 128u + ((((e >> 1) ^ (r & 7u)) << 4) | ((e & 1u) << 3));
}

// kBins = false: compress of a float32 field (codec.py:495-498);
// kBins = true:  encode_from_quant of int64 bins (codec.py:523-525) -- the
// same encoder with the bins staged by a 3-D TMA load instead of quantized
template <bool kTma, bool kBins = false>
__global__ void __launch_bounds__(kThreadsC, kBins ? HSZ_BINS_CTAS : HSZ_CMP_CTAS)
    compress_f32_kernel(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ x,
                        uint64_t n, QuantF32 qf, QuantConst qc, k32::EncodeOut out,
                        uint64_t nblocks, uint64_t ntiles, uint32_t tail_len,
                        const int64_t* __restrict__ xb = nullptr) {
  using SM = std::conditional_t<kBins, Smem7Bins, Smem7>;
  extern __shared__ unsigned char smraw[];
  const uint32_t a0 = smem_u32(smraw);
  SM& S = *reinterpret_cast<SM*>(smraw + (((a0 + 1023u) & ~1023u) - a0));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  LookbackWs lw = LookbackWs::bind(out.ws, ntiles);
  const uint64_t last_draw = ntiles + gridDim.x - 1;   // every CTA draws once past the end
  const uint64_t full_rows = n / K;
  if (tid == 0) {
    mbar_init(&S.full, 1);
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&S.st_full[i], kCompute / 32);
      mbar_init(&S.st_empty[i], 1);
    }
    S.ring_tail = 0;
    fence_mbar_init();
    S.epoch = ld_acquire(lw.epoch);
  }
  __syncthreads();
  const uint64_t epoch = S.epoch;

  if (warp == kCompute / 32) {
    // =========================== placement warp ===========================
    for (uint32_t kk = 0;; ++kk) {
      const int slot = kk % kSlots;
      mbar_wait_parity_sleep(&S.st_full[slot], (kk / kSlots) & 1u);
      const RingRec r = S.rec[slot];
      if (r.ts == kDone) break;
      if (r.ts != kSelfPlaced) {
        uint64_t es, ep;
        resolve6(out, r.tile, epoch, ntiles, r.ts, r.tp, &es, &ep);
        if (es != ~0ull) copy_ring(S.sgn[slot], S.ring, out, r, es, ep);
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();   // the ring reads complete before the space is reused
        S.ring_tail = r.end;
        mbar_arrive(&S.st_empty[slot]);
      }
    }
    return;
  }

  // =========================== compute warps ===========================
  // thread 0: tickets and TMA issue
  auto draw_raw = [&]() -> uint64_t { return atom_add_relaxed(lw.ticket, 1); };
  auto consume = [&](uint64_t t) {   // a drawn ticket: the CTA drawing the last one re-arms
    if (t == last_draw) {
      st_relaxed(lw.ticket, 0);
      st_release(lw.epoch, epoch + 1);
    }
  };
  auto issue = [&](uint64_t t) {     // tile t into S.in (or "no more tiles")
    S.cur = t;
    if (t < ntiles && kTma) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if constexpr (kBins) {
        mbar_arrive_expect_tx(&S.full, 2 * kBufBytes);
        tma_load_3d(S.in, &tmap, 0, static_cast<int>(t * TB), 0, &S.full);
      } else {
        mbar_arrive_expect_tx(&S.full, kBufBytes);
        tma_load_2d(S.in, &tmap, 0, static_cast<int>(t * TB), &S.full);
      }
    } else {
      mbar_arrive(&S.full);
    }
  };
  // warp 1 lane 0 (thread kTmaThread) owns tickets and TMA issue, thread 0 the
  // aggregate publication and ring claims: the serial work of a tile is spread
  constexpr int kTmaThread = 32;
  uint64_t ahead = ~0ull;   // ticket in flight
  if (tid == kTmaThread) {
    const uint64_t t = draw_raw();
    consume(t);
    issue(t);
    if (t < ntiles) ahead = draw_raw();
  }
  uint32_t flags = 0;
  uint64_t head = 0;   // ring bytes allocated (identical in every compute thread)
  for (uint32_t k = 0;; ++k) {
    const int slot = k % kSlots;
    mbar_wait_parity(&S.full, k & 1u);
    const uint64_t cur = S.cur;
    if (cur >= ntiles) {
      // stop the placement warp
      if (k >= kSlots) mbar_wait_parity(&S.st_empty[slot], ((k / kSlots) - 1) & 1u);
      if (tid == 0) {
        S.rec[slot].ts = kDone;
        S.rec[slot].end = head;
      }
      mbar_arrive_warp(&S.st_full[slot]);
      break;
    }
    unsigned char* in = S.in;
    bool wide = false;
    uint32_t qb[K];
    const uint64_t row0 = cur * TB;
    if (kTma) {
      // the partial last block is not covered by the tensor map (zero-filled)
      if ((n % K) != 0 && full_rows >= row0 && full_rows < row0 + TB) {
        if (tid < K) {
          const uint32_t r = static_cast<uint32_t>(n % K);
          const uint32_t rr = static_cast<uint32_t>(full_rows - row0);
          if constexpr (kBins) {
            const int64_t v = static_cast<uint32_t>(tid) < r ? xb[full_rows * K + tid] : 0;
            *reinterpret_cast<int64_t*>(in + bins_off(rr, tid)) = v;
          } else {
            const float v = static_cast<uint32_t>(tid) < r ? x[full_rows * K + tid] : 0.0f;
            *reinterpret_cast<float*>(in + swz_elem(rr, tid)) = v;
          }
        }
        bar_sync_n(1, kCompute);
      }
    } else if constexpr (kBins) {
      __trap();                        // the host launches the bins variant with TMA only
    } else {
      const uint64_t e0 = row0 * K;
      for (uint32_t i = tid; i < TB * K; i += kCompute) {
        const uint64_t e = e0 + i;
        const float v = e < n ? x[e] : 0.0f;
        *reinterpret_cast<float*>(in + swz_elem(i >> 5, i & 31u)) = v;
      }
      bar_sync_n(1, kCompute);
    }
    if constexpr (kBins) {
      // ---- this thread's 32 bins: the register path needs |bin| < 2^30 ------
      bool big = false;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(
              in + (h * TB + tid) * 128 + ((j ^ (tid & 7)) << 4));
          big |= (v.x + static_cast<uint64_t>(kWide) >= 2ull * kWide) |
                 (v.y + static_cast<uint64_t>(kWide) >= 2ull * kWide);
          qb[16 * h + 2 * j] = static_cast<uint32_t>(v.x) + kMagicBits;
          qb[16 * h + 2 * j + 1] = static_cast<uint32_t>(v.y) + kMagicBits;
        }
      }
      wide = bar_or_compute(big);     // ... and every read of the input buffer is done
      if (tid == kTmaThread) {        // refill it: the next tile's load overlaps this tile
        const uint64_t nx = ahead;
        consume(nx);
        issue(nx);
        if (nx < ntiles) ahead = draw_raw();
      }
    } else
    // ---- quantize this thread's row ----------------------------------------
    {
      const unsigned char* row = in + tid * 128;
#if HSZ_QUANT_MINMAX
      float vmin = 1.0f, pmax = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 v = *reinterpret_cast<const float4*>(row + ((j ^ (tid & 7)) << 4));
        float p0, p1, p2, p3;
        qb[4 * j + 0] = quant_f32m(v.x, qf, vmin, p0);
        qb[4 * j + 1] = quant_f32m(v.y, qf, vmin, p1);
        qb[4 * j + 2] = quant_f32m(v.z, qf, vmin, p2);
        qb[4 * j + 3] = quant_f32m(v.w, qf, vmin, p3);
        pmax = max3_nan_abs(pmax, p0, p1);
        pmax = max3_nan_abs(pmax, p2, p3);
      }
      bool bad = !((vmin > qf.delta) & (pmax < 2097152.0f) & (qf.delta > 0.0f));
#else
      bool bad = false;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 v = *reinterpret_cast<const float4*>(row + ((j ^ (tid & 7)) << 4));
        qb[4 * j + 0] = quant_f32(v.x, qf, bad);
        qb[4 * j + 1] = quant_f32(v.y, qf, bad);
        qb[4 * j + 2] = quant_f32(v.z, qf, bad);
        qb[4 * j + 3] = quant_f32(v.w, qf, bad);
      }
#endif
      if (__any_sync(kFull, bad)) {   // rare: an element inside the certificate margin
        uint32_t mask = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          float* pi = reinterpret_cast<float*>(in + swz_elem(tid, i));
          bool bb = false;
          (void)quant_f32(*pi, qf, bb);
          mask |= (bb ? 1u : 0u) << i;
          if (!bb) *reinterpret_cast<uint32_t*>(pi) = qb[i];
        }
#pragma unroll 1
        for (int i = 0; i < K; ++i) {
          if ((mask >> i) & 1u) {
            uint32_t* pi = reinterpret_cast<uint32_t*>(in + swz_elem(tid, i));
            const ExactQ r = quant_exact(__uint_as_float(*pi), qc);
            flags |= r.flags;
            wide |= !((r.q > -kWide) & (r.q < kWide));
            *pi = static_cast<uint32_t>(static_cast<uint64_t>(r.q) + kMagicBits);
          }
        }
#pragma unroll
        for (int i = 0; i < K; ++i) qb[i] = *reinterpret_cast<const uint32_t*>(in + swz_elem(tid, i));
      }
      wide = bar_or_compute(wide);    // ... and every read of the input buffer is done
      if (tid == kTmaThread) {        // refill it: the next tile's load overlaps this tile
        const uint64_t nx = ahead;
        consume(nx);
        issue(nx);
        if (nx < ntiles) ahead = draw_raw();
      }
    }
    if (!wide) {
      const uint64_t gb = cur * TB + tid;
      const bool active = gb < nblocks;
      const int len = !active ? 0 : (gb == nblocks - 1 ? static_cast<int>(tail_len) : K);
      BlockCode bc;
      block_code(qb, len, bc);
      const uint32_t wmax = __reduce_max_sync(kFull, bc.w);
      const uint32_t sb = (bc.w && active) ? ((static_cast<uint32_t>(len) + 7u) >> 3) : 0u;
      const uint32_t pb = (static_cast<uint32_t>(len) * bc.w + 7u) >> 3;
      uint32_t tot;
      const uint32_t ex = cta_scan(sb | (pb << 10), S.scan, &tot);   // sb <= 512, pb <= 15872
      const uint32_t es = ex & 1023u, ep = ex >> 10;
      const uint32_t ts = tot & 1023u, tp = tot >> 10;
      if (tid == 0) lb_publish(lb_words(out.ws), cur, epoch, ts, tp);
      if (active) {
        out.widths[gb] = static_cast<uint8_t>(bc.w);
        out.outliers[gb] = static_cast<int32_t>(qb[0] - kMagicBits);
      }
      // claim metadata slot k%4 and ring space for the packed payload; every
      // thread tracks the ring head itself (same tp on all threads), so no
      // broadcast barrier is needed
      if (k >= kSlots) mbar_wait_parity(&S.st_empty[slot], ((k / kSlots) - 1) & 1u);
      const uint32_t need = (tp + 127u) & ~127u;
      uint32_t pos = static_cast<uint32_t>(head % kRingBytes);
      const uint64_t prev_end = head;   // end of the last tile this CTA allocated
      if (pos + need > kRingBytes) {   // no wrap inside a tile: skip to the ring start
        head += kRingBytes - pos;
        pos = 0;
      }
      // [head, head + need) must be free.  The skipped bytes belong to no tile,
      // so ring_tail (the end of the last PLACED tile) never covers them: once
      // every earlier tile is placed (tail == prev_end) the ring is empty and the
      // tile fits -- without this test a skip of more than kRingBytes - need
      // bytes (a small tile followed by a large one) waited forever.
      for (unsigned ns = 32;;) {
        const uint64_t tail = S.ring_tail;
        if (tail >= prev_end || head + need - tail <= kRingBytes) break;
        __nanosleep(ns);
        ns = ns < 256 ? ns * 2 : 256;
      }
      head += need;
      if (tid == 0) {
        S.rec[slot].tile = cur;
        S.rec[slot].end = head;
        S.rec[slot].ts = ts;
        S.rec[slot].tp = tp;
        S.rec[slot].off = pos;
      }
      if (sb) S.sgn[slot][es >> 2] = bswap32(bc.sg);
      pack_block(bc, wmax, ep >> 2, reinterpret_cast<uint32_t*>(S.ring + pos));
      mbar_arrive_warp(&S.st_full[slot]);
    } else {
      // exact path: sizes and publish first; the tile then resolves and
      // places itself (the placement warp resolves the previous tiles)
      using Src = std::conditional_t<kBins, k32::SrcBins, k32::SrcQuant<float>>;
      Src src = make_exact_src<Src>(x, xb, n, qc, cur);
      flags |= k32::fallback_sizes(src, out, cur, nblocks, tail_len, S.wsb, S.wpb);
      bar_sync_n(1, kCompute);
      const uint32_t ts = S.wsb[0] + S.wsb[1] + S.wsb[2] + S.wsb[3];
      const uint32_t tp = S.wpb[0] + S.wpb[1] + S.wpb[2] + S.wpb[3];
      if (tid == 0) lb_publish(lb_words(out.ws), cur, epoch, ts, tp);
      if (k >= kSlots) mbar_wait_parity(&S.st_empty[slot], ((k / kSlots) - 1) & 1u);
      if (tid == 0) {
        S.rec[slot].tile = cur;
        S.rec[slot].end = head;
        S.rec[slot].ts = kSelfPlaced;
      }
      mbar_arrive_warp(&S.st_full[slot]);
      if (warp == 0) {
        uint64_t es, ep;
        resolve6(out, cur, epoch, ntiles, ts, tp, &es, &ep);
        if (lane == 0) {
          S.excl_s[slot] = es;
          S.excl_p[slot] = ep;
        }
      }
      bar_sync_n(1, kCompute);
      if (S.excl_s[slot] != ~0ull) {
        uint64_t gs = S.excl_s[slot], gp = S.excl_p[slot];
        for (int i = 0; i < warp; ++i) {
          gs += S.wsb[i];
          gp += S.wpb[i];
        }
        k32::fallback_pack(src, out, cur, nblocks, tail_len, gs, gp, S.xscratch[warp]);
      }
      bar_sync_n(1, kCompute);
    }
  }
  flags = __reduce_or_sync(kFull, flags);
  if (lane == 0 && flags) atomicOr(out.err, flags);
}

}  // namespace e32
}  // namespace hsz
