// Generic block_len path (any k != 32): one thread per block.
//
// The reference accepts any block_len >= 1 (model.py:69-70) and its tests
// use 1, 3, 4, 8, 33, 128 (conftest.py:35, test_codec.py:353,
// test_acceptance.py:201).  None of the BASELINE configs do, so this path
// favours simplicity over speed: encode is three kernels (widths/outliers,
// tile offsets by look-back, packing with byte stores) and decode walks a
// block's bits serially.  Results are bit-identical to the k=32 kernels'
// contract.
#pragma once

#include "hsz_common.cuh"
#include "hsz_quant.cuh"

namespace hsz {

// CTA-wide exclusive scan of two u32 values (blockDim.x <= 1024)
__device__ __forceinline__ void cta_excl_scan2(uint32_t a, uint32_t b, uint32_t* ea,
                                               uint32_t* eb, uint32_t* ta, uint32_t* tb) {
  __shared__ uint32_t s_a[32], s_b[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = (blockDim.x + 31) >> 5;
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
    s_a[warp] = ia;
    s_b[warp] = ib;
  }
  __syncthreads();
  uint32_t pa = 0, pb = 0, sa = 0, sb = 0;
  for (int i = 0; i < nw; ++i) {
    if (i < warp) {
      pa += s_a[i];
      pb += s_b[i];
    }
    sa += s_a[i];
    sb += s_b[i];
  }
  *ea = pa + ia - a;
  *eb = pb + ib - b;
  *ta = sa;
  *tb = sb;
  __syncthreads();
}

__device__ __forceinline__ uint32_t block_len_of(uint64_t b, uint64_t n, uint32_t k) {
  const uint64_t e0 = b * k;
  const uint64_t r = n - e0;
  return r < k ? static_cast<uint32_t>(r) : k;
}

namespace gen {

constexpr int kThreads = kTileBlocks;   // one tile per CTA, one block per thread

template <typename T>
struct GQuant {
  const T* x;
  QuantConst c;
  __device__ __forceinline__ int64_t get(uint64_t e, uint32_t* f) const {
    return quantize1(static_cast<double>(x[e]), c, f);
  }
};

struct GBins {
  const int64_t* b;
  __device__ __forceinline__ int64_t get(uint64_t e, uint32_t* f) const {
    const int64_t v = b[e];
    if (v == INT64_MIN) *f |= HSZ_ERR_RESCALE_OVERFLOW;
    return v;
  }
};

template <class G>
__global__ void __launch_bounds__(kThreads) widths_kernel(G src, uint64_t n, uint32_t k,
                                                          uint64_t nblocks, uint8_t* widths,
                                                          int32_t* outliers, uint32_t* err) {
  const uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  const uint32_t len = block_len_of(b, n, k);
  const uint64_t e0 = b * k;
  uint32_t flags = 0;
  const int64_t first = src.get(e0, &flags);
  int64_t prev = first;
  uint64_t mx = 0;
  for (uint32_t i = 1; i < len; ++i) {
    const int64_t q = src.get(e0 + i, &flags);
    bool neg;
    const uint64_t m = absdiff64(q, prev, &neg);
    mx = m > mx ? m : mx;
    prev = q;
  }
  widths[b] = static_cast<uint8_t>(mx ? 64 - __clzll(static_cast<long long>(mx)) : 0);
  if (first < INT32_MIN || first > INT32_MAX) flags |= HSZ_ERR_OUTLIER_OVERFLOW;
  outliers[b] = static_cast<int32_t>(first);
  if (flags) atomicOr(err, flags);
}

struct ByteWriter {
  uint8_t* p;
  uint64_t acc;
  int nbits;
  __device__ __forceinline__ void push(uint64_t v, int w) {   // w <= 64, MSB first
    while (w > 0) {
      const int take = w > 32 ? 32 : w;
      const uint64_t chunk = (v >> (w - take)) & ((1ull << take) - 1ull);
      acc = (acc << take) | chunk;
      nbits += take;
      w -= take;
      while (nbits >= 8) {
        *p++ = static_cast<uint8_t>(acc >> (nbits - 8));
        nbits -= 8;
      }
    }
  }
  __device__ __forceinline__ void flush() {
    if (nbits > 0) *p++ = static_cast<uint8_t>(acc << (8 - nbits));
    nbits = 0;
  }
};

template <class G>
__global__ void __launch_bounds__(kThreads) pack_kernel(G src, uint64_t n, uint32_t k,
                                                        uint64_t nblocks, uint64_t ntiles,
                                                        const uint8_t* widths,
                                                        const uint64_t* toff, uint8_t* signs,
                                                        uint64_t sign_cap, uint8_t* payload,
                                                        uint64_t pay_cap, uint32_t* err) {
  const uint64_t tile = blockIdx.x;
  const uint64_t b = tile * kThreads + threadIdx.x;
  uint32_t w = 0, len = 0;
  if (b < nblocks) {
    w = widths[b];
    len = block_len_of(b, n, k);
  }
  const uint32_t sb = w ? (len + 7) / 8 : 0;
  const uint32_t pb = static_cast<uint32_t>((static_cast<uint64_t>(len) * w + 7) / 8);
  uint32_t es, ep, ts, tp;
  cta_excl_scan2(sb, pb, &es, &ep, &ts, &tp);
  if (toff[2 * ntiles] > sign_cap || toff[2 * ntiles + 1] > pay_cap) {
    if (threadIdx.x == 0 && tile == 0) atomicOr(err, HSZ_ERR_CAPACITY);
    return;
  }
  if (w == 0) return;
  uint32_t flags = 0;
  const uint64_t e0 = b * k;
  ByteWriter sw{signs + toff[2 * tile] + es, 0, 0};
  ByteWriter pw{payload + toff[2 * tile + 1] + ep, 0, 0};
  int64_t prev = src.get(e0, &flags);
  sw.push(0, 1);   // slot 0 carries the outlier
  pw.push(0, w);
  for (uint32_t i = 1; i < len; ++i) {
    const int64_t q = src.get(e0 + i, &flags);
    bool neg;
    const uint64_t m = absdiff64(q, prev, &neg);
    sw.push(neg ? 1 : 0, 1);
    pw.push(m, w);
    prev = q;
  }
  sw.flush();
  pw.flush();
  (void)flags;   // already reported by widths_kernel
}

// read `w` (<= 64) bits MSB-first starting at bit `pos` of byte string p
__device__ __forceinline__ uint64_t read_bits(const uint8_t* p, uint64_t pos, int w) {
  const uint64_t byte = pos >> 3;
  const int off = static_cast<int>(pos & 7);
  const int nb = (off + w + 7) >> 3;   // <= 9
  unsigned __int128 acc = 0;
  for (int i = 0; i < nb; ++i) acc = (acc << 8) | p[byte + i];
  const int total = nb * 8;
  acc >>= (total - off - w);
  return static_cast<uint64_t>(acc & ((static_cast<unsigned __int128>(1) << w) - 1u));
}

struct GStream {
  const uint8_t* widths;
  const int32_t* outliers;
  const uint8_t* signs;
  const uint8_t* payload;
  const uint64_t* toff;
  uint64_t n;
  uint32_t k;
  uint64_t nblocks;
};

// Serial per-block decode; calls sink.put(e, bin, flags) for each element.
template <class Sink>
__device__ __forceinline__ void decode_one_block(const GStream& s, uint64_t tile, uint64_t b,
                                                 Sink& sink, uint32_t* flags) {
  uint32_t w = 0, len = 0;
  if (b < s.nblocks) {
    w = s.widths[b];
    len = block_len_of(b, s.n, s.k);
  }
  if (w > 64) {
    *flags |= HSZ_ERR_BAD_WIDTH;
    w = 0;
  }
  const uint32_t sb = w ? (len + 7) / 8 : 0;
  const uint32_t pb = static_cast<uint32_t>((static_cast<uint64_t>(len) * w + 7) / 8);
  uint32_t es, ep, ts, tp;
  cta_excl_scan2(sb, pb, &es, &ep, &ts, &tp);
  if (b >= s.nblocks) return;
  const uint64_t e0 = b * s.k;
  const int64_t o = s.outliers[b];
  sink.put(e0, o, flags);
  if (w == 0) {
    for (uint32_t i = 1; i < len; ++i) sink.put(e0 + i, o, flags);
    return;
  }
  const uint8_t* sg = s.signs + s.toff[2 * tile] + es;
  const uint8_t* py = s.payload + s.toff[2 * tile + 1] + ep;
  __int128 acc = o;
  const __int128 lim = static_cast<__int128>(INT64_MAX);
  for (uint32_t i = 1; i < len; ++i) {
    const bool neg = (sg[i >> 3] >> (7 - (i & 7))) & 1u;
    const uint64_t m = read_bits(py, static_cast<uint64_t>(i) * w, static_cast<int>(w));
    acc += neg ? -static_cast<__int128>(m) : static_cast<__int128>(m);
    if (acc > lim || acc < -lim) {
      *flags |= HSZ_ERR_PREFIX_OVERFLOW;
      return;
    }
    sink.put(e0 + i, static_cast<int64_t>(acc), flags);
  }
}

template <class Sink>
__global__ void __launch_bounds__(kThreads) decode_kernel(GStream s, Sink sink, uint32_t* err) {
  uint32_t flags = 0;
  const uint64_t tile = blockIdx.x;
  decode_one_block(s, tile, tile * kThreads + threadIdx.x, sink, &flags);
  if (flags) atomicOr(err, flags);
}

// rescaled-product sink for the generic scalar multiply
struct SinkSmul {
  int64_t* out;
  int64_t rs;
  double d;
  __device__ __forceinline__ void put(uint64_t e, int64_t bin, uint32_t* flags) const {
    out[e] = rescale1(product_rn(bin, rs), d, flags);
  }
};

// tile-offset scan of an existing widths section (any k), by look-back
__global__ void __launch_bounds__(kThreads) tile_offsets_kernel(const uint8_t* widths, uint64_t n,
                                                                uint32_t k, uint64_t nblocks,
                                                                uint64_t ntiles, uint64_t* toff,
                                                                uint32_t* err, void* ws) {
  __shared__ uint64_t s_tile, s_epoch;
  LookbackWs lw = LookbackWs::bind(ws, ntiles);
  if (threadIdx.x == 0) {
    uint64_t t, e;
    draw_ticket(lw, ntiles, &t, &e);
    s_tile = t;
    s_epoch = e;
  }
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t b = tile * kThreads + threadIdx.x;
  uint32_t w = 0, len = 0;
  if (b < nblocks) {
    w = widths[b];
    len = block_len_of(b, n, k);
  }
  if (w > 64) {
    atomicOr(err, HSZ_ERR_BAD_WIDTH);
    w = 0;
  }
  const uint32_t sb = w ? (len + 7) / 8 : 0;
  const uint32_t pb = static_cast<uint32_t>((static_cast<uint64_t>(len) * w + 7) / 8);
  uint32_t es, ep, ts, tp;
  cta_excl_scan2(sb, pb, &es, &ep, &ts, &tp);
  if (threadIdx.x < 32) {
    uint64_t xs, xp;
    lookback(lw, tile, s_epoch, ts, tp, &xs, &xp, err);
    if (threadIdx.x == 0) {
      toff[2 * tile] = xs;
      toff[2 * tile + 1] = xp;
      if (tile == ntiles - 1) {
        toff[2 * ntiles] = xs + ts;
        toff[2 * ntiles + 1] = xp + tp;
      }
    }
  }
}

}  // namespace gen
}  // namespace hsz
