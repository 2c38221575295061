// Bivariate quantized-domain operations and per-block reductions (SURVEY.md
// §8(f) row 3): hadamard (ops.py:226-240), the exact pair statistics behind
// covariance / ssim_global (ops.py:400-513) and block_means (ops.py:366-379).
//
// All three run on the operands' int64 bins (decoded by the stream decoders
// into scratch) with grid-stride kernels; the results are exact integers
// (carry-save 32-bit chunk counters) or the reference's own float64 steps.
#pragma once

#include "hsz_common.cuh"
#include "hsz_quant.cuh"

namespace hsz {
namespace bv {

constexpr int kThreads = 256;

// pair-statistics counters (u64 each, carry-save: counter j of a bank holds
// 32-bit chunks of weight 2^(32 j)):
//   SA+ [0,2)  SA- [2,4)   SB+ [4,6)  SB- [6,8)      sums of bins (|bin| < 2^63)
//   QA  [8,12) QB  [12,16)                            sums of squares (< 2^126)
//   SAB+ [16,20) SAB- [20,24)                         sums of products
//   min a, max a, min b, max b [24,28)                 (signed, atomics)
constexpr int kPairWords = 28;

__device__ __forceinline__ void put_chunks(uint64_t* c, unsigned __int128 v, int nchunks) {
  for (int j = 0; j < nchunks; ++j) c[j] += static_cast<uint64_t>(v >> (32 * j)) & 0xffffffffull;
}

__device__ __forceinline__ unsigned __int128 uabs128(__int128 v) {
  return v < 0 ? static_cast<unsigned __int128>(-(v + 1)) + 1u : static_cast<unsigned __int128>(v);
}

__global__ void __launch_bounds__(kThreads) pair_stats_kernel(const int64_t* a, const int64_t* b,
                                                             uint64_t n, uint64_t* out) {
  uint64_t c[24];
#pragma unroll
  for (int j = 0; j < 24; ++j) c[j] = 0;
  int64_t mna = INT64_MAX, mxa = INT64_MIN, mnb = INT64_MAX, mxb = INT64_MIN;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t x = a[i], y = b[i];
    const __int128 xw = x, yw = y;
    put_chunks(c + (x < 0 ? 2 : 0), uabs128(xw), 2);
    put_chunks(c + (y < 0 ? 6 : 4), uabs128(yw), 2);
    put_chunks(c + 8, uabs128(xw * xw), 4);
    put_chunks(c + 12, uabs128(yw * yw), 4);
    const __int128 p = xw * yw;
    put_chunks(c + (p < 0 ? 20 : 16), uabs128(p), 4);
    mna = x < mna ? x : mna;
    mxa = x > mxa ? x : mxa;
    mnb = y < mnb ? y : mnb;
    mxb = y > mxb ? y : mxb;
  }
  __shared__ unsigned long long s[kPairWords];
  if (threadIdx.x < 24) s[threadIdx.x] = 0;
  else if (threadIdx.x < kPairWords)
    s[threadIdx.x] = (threadIdx.x & 1) ? static_cast<unsigned long long>(INT64_MIN)
                                       : static_cast<unsigned long long>(INT64_MAX);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 24; ++j) {
    uint64_t v = c[j];
    for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(kFull, v, m);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s[j], static_cast<unsigned long long>(v));
  }
  for (int m = 16; m > 0; m >>= 1) {
    const int64_t t0 = __shfl_xor_sync(kFull, mna, m), t1 = __shfl_xor_sync(kFull, mxa, m);
    const int64_t t2 = __shfl_xor_sync(kFull, mnb, m), t3 = __shfl_xor_sync(kFull, mxb, m);
    mna = t0 < mna ? t0 : mna;
    mxa = t1 > mxa ? t1 : mxa;
    mnb = t2 < mnb ? t2 : mnb;
    mxb = t3 > mxb ? t3 : mxb;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(reinterpret_cast<long long*>(&s[24]), static_cast<long long>(mna));
    atomicMax(reinterpret_cast<long long*>(&s[25]), static_cast<long long>(mxa));
    atomicMin(reinterpret_cast<long long*>(&s[26]), static_cast<long long>(mnb));
    atomicMax(reinterpret_cast<long long*>(&s[27]), static_cast<long long>(mxb));
  }
  __syncthreads();
  if (threadIdx.x < 24) {
    // carry-save into the global counters: the block sum's low and high
    // 32-bit halves go to chunk j and j + 1 of the same bank
    const uint64_t v = s[threadIdx.x];
    const int j = threadIdx.x;
    atomicAdd(reinterpret_cast<unsigned long long*>(out + 2 * j), v & 0xffffffffull);
    atomicAdd(reinterpret_cast<unsigned long long*>(out + 2 * j + 1), v >> 32);
  } else if (threadIdx.x < kPairWords) {
    long long* o = reinterpret_cast<long long*>(out + 48 + (threadIdx.x - 24));
    const long long v = static_cast<long long>(s[threadIdx.x]);
    if (threadIdx.x & 1) atomicMax(o, v);
    else atomicMin(o, v);
  }
}

// the min/max slots start at +inf / -inf; the rest at 0
__global__ void pair_stats_init(uint64_t* out) {
  const int t = threadIdx.x;
  if (t < 48) out[t] = 0;
  else if (t < 52) out[t] = (t & 1) ? static_cast<uint64_t>(INT64_MIN) : static_cast<uint64_t>(INT64_MAX);
}

// hadamard (ops.py:226-240): bins = round-half-away(RN(2eps * RN(a * b)))
__global__ void __launch_bounds__(kThreads) hadamard_kernel(int64_t* a, const int64_t* b, uint64_t n,
                                                           double d, uint32_t* err) {
  uint32_t flags = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    a[i] = rescale1(product_rn(a[i], b[i]), d, &flags);
  if (flags) atomicOr(err, flags);
}

// numpy's float64 pairwise sum (the inner loop of ``ndarray.sum(dtype=
// np.float64)`` on a contiguous int64 row): sequential from 0 below 8
// elements, 8 interleaved partial sums up to 128, halves (multiples of 8)
// above -- so block_means matches the reference bit for bit even when the
// float sums are inexact
__device__ double np_pairwise_sum(const int64_t* a, uint64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (uint64_t i = 0; i < n; ++i) r = __dadd_rn(r, __ll2double_rn(a[i]));
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = __ll2double_rn(a[j]);
    uint64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __ll2double_rn(a[i + j]));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, __ll2double_rn(a[i]));
    return res;
  }
  uint64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_sum(a, n2), np_pairwise_sum(a + n2, n - n2));
}

// block_means (ops.py:366-379): (2 eps * sum) / length with the reference's
// sums -- len * outlier (exact integer, then float64) for constant blocks,
// numpy's float64 row sum of the bins otherwise
__global__ void __launch_bounds__(kThreads) block_means_kernel(const int64_t* bins, const uint8_t* widths,
                                                              const int32_t* outliers, uint64_t n,
                                                              uint32_t k, uint64_t nblocks, double d,
                                                              double* out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t blk = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; blk < nblocks;
       blk += stride) {
    const uint64_t e0 = blk * k;
    const uint64_t len = (e0 + k < n ? e0 + k : n) - e0;
    const double sf = widths[blk] == 0
                          ? __ll2double_rn(static_cast<int64_t>(len) * outliers[blk])
                          : np_pairwise_sum(bins + e0, len);
    out[blk] = __ddiv_rn(__dmul_rn(d, sf), static_cast<double>(len));
  }
}

}  // namespace bv
}  // namespace hsz
