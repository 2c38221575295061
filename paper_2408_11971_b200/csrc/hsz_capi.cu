// C ABI of the B200 hot path (see include/hsz_b200.h) + the streaming ops
// (value range, negate, scalar add) that need no block decoding.
//
// Build (done by __graft_entry__.build / paper_2408_11971_b200/build.py):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared
//        -Xcompiler -fPIC -o paper_2408_11971_b200/_lib/libhsz_b200.so hsz_capi.cu

#include <cstdio>
#include <ctime>
#include <cstring>

#include <cudaTypedefs.h>

#include "hsz_common.cuh"
#include "hsz_dec32.cuh"
#include "hsz_bivar.cuh"
#include "hsz_enc32.cuh"
#include "hsz_generic.cuh"
#include "hsz_k32.cuh"
#include "hsz_quant.cuh"

namespace hsz {
namespace ops {

constexpr int kThreads = 256;
constexpr int kMinmaxCtas = static_cast<int>(kMinmaxCtasMax);

// ---- K0: min / max / finiteness (codec.py:52-53, 96-99) -------------------
template <typename T>
__global__ void __launch_bounds__(kThreads) minmax_kernel(const T* x, uint64_t n, double* out,
                                                          uint32_t* err, void* ws) {
  double lo = INFINITY, hi = -INFINITY;
  bool bad = false;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if constexpr (sizeof(T) == 4) {
    const bool vec = (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
    const uint64_t nv = vec ? n / 4 : 0;
    const float4* xv = reinterpret_cast<const float4*>(x);
    float flo = INFINITY, fhi = -INFINITY;
    uint64_t i = tid;
    for (; i + 3 * stride < nv; i += 4 * stride) {   // 4 independent 16-byte loads in flight
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(xv + i + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        bad |= !isfinite(v[u].x) | !isfinite(v[u].y) | !isfinite(v[u].z) | !isfinite(v[u].w);
        flo = fminf(fminf(flo, v[u].x), fminf(fminf(v[u].y, v[u].z), v[u].w));
        fhi = fmaxf(fmaxf(fhi, v[u].x), fmaxf(fmaxf(v[u].y, v[u].z), v[u].w));
      }
    }
    for (; i < nv; i += stride) {
      const float4 v = __ldcs(xv + i);
      bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
      flo = fminf(fminf(flo, v.x), fminf(fminf(v.y, v.z), v.w));
      fhi = fmaxf(fmaxf(fhi, v.x), fmaxf(fmaxf(v.y, v.z), v.w));
    }
    for (uint64_t i = nv * 4 + tid; i < n; i += stride) {
      const float v = x[i];
      bad |= !isfinite(v);
      flo = fminf(flo, v);
      fhi = fmaxf(fhi, v);
    }
    lo = flo;
    hi = fhi;
  } else {
    for (uint64_t i = tid; i < n; i += stride) {
      const double v = x[i];
      bad |= !isfinite(v);
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
  }
  for (int m = 16; m > 0; m >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(kFull, lo, m));
    hi = fmax(hi, __shfl_xor_sync(kFull, hi, m));
  }
  if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(err, HSZ_ERR_NONFINITE);
  __shared__ double s_lo[kThreads / 32], s_hi[kThreads / 32];
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_lo[warp] = lo;
    s_hi[warp] = hi;
  }
  __syncthreads();
  uint64_t* base = static_cast<uint64_t*>(ws);
  uint64_t* done = base + 3;
  double* part = reinterpret_cast<double*>(base + kWsMinmaxOff);
  if (threadIdx.x == 0) {
    for (int i = 1; i < kThreads / 32; ++i) {
      lo = fmin(lo, s_lo[i]);
      hi = fmax(hi, s_hi[i]);
    }
    part[2 * blockIdx.x] = lo;
    part[2 * blockIdx.x + 1] = hi;
    __threadfence();
    s_last = atom_add_acq_rel(done, 1) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // the last CTA folds every CTA's partial in parallel
  lo = INFINITY;
  hi = -INFINITY;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
    lo = fmin(lo, __longlong_as_double(ld_relaxed(reinterpret_cast<uint64_t*>(part + 2 * i))));
    hi = fmax(hi, __longlong_as_double(ld_relaxed(reinterpret_cast<uint64_t*>(part + 2 * i + 1))));
  }
  for (int m = 16; m > 0; m >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(kFull, lo, m));
    hi = fmax(hi, __shfl_xor_sync(kFull, hi, m));
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    s_lo[warp] = lo;
    s_hi[warp] = hi;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = 1; i < kThreads / 32; ++i) {
    lo = fmin(lo, s_lo[i]);
    hi = fmax(hi, s_hi[i]);
  }
  out[0] = lo;
  out[1] = hi;
  st_relaxed(done, 0);
}

// ---- K0 for float32: 8 independent 16-byte loads in flight per thread -------
#ifndef HSZ_MM_LOAD
#define HSZ_MM_LOAD __ldcs
#endif
#ifndef HSZ_MM_THREADS
#define HSZ_MM_THREADS 256
#endif
constexpr int kMmThreads = HSZ_MM_THREADS;
__global__ void __launch_bounds__(kMmThreads) minmax_f32_kernel(const float* __restrict__ x, uint64_t n,
                                                                double* out, uint32_t* err, void* ws,
                                                                Mailbox mb) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nv = n / 4;
  const float4* xv = reinterpret_cast<const float4*>(x);
  float flo = INFINITY, fhi = -INFINITY;
  bool bad = false;
  uint64_t i = tid;
  for (; i + 7 * stride < nv; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = HSZ_MM_LOAD(xv + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      bad |= !isfinite(v[u].x) | !isfinite(v[u].y) | !isfinite(v[u].z) | !isfinite(v[u].w);
      flo = fminf(fminf(flo, v[u].x), fminf(fminf(v[u].y, v[u].z), v[u].w));
      fhi = fmaxf(fmaxf(fhi, v[u].x), fmaxf(fmaxf(v[u].y, v[u].z), v[u].w));
    }
  }
  for (; i < nv; i += stride) {
    const float4 v = __ldcs(xv + i);
    bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
    flo = fminf(fminf(flo, v.x), fminf(fminf(v.y, v.z), v.w));
    fhi = fmaxf(fmaxf(fhi, v.x), fmaxf(fmaxf(v.y, v.z), v.w));
  }
  for (uint64_t j = nv * 4 + tid; j < n; j += stride) {
    const float v = x[j];
    bad |= !isfinite(v);
    flo = fminf(flo, v);
    fhi = fmaxf(fhi, v);
  }
  double lo = flo, hi = fhi;
  for (int m = 16; m > 0; m >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(kFull, lo, m));
    hi = fmax(hi, __shfl_xor_sync(kFull, hi, m));
  }
  if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(err, HSZ_ERR_NONFINITE);
  __shared__ double s_lo[kMmThreads / 32], s_hi[kMmThreads / 32];
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_lo[warp] = lo;
    s_hi[warp] = hi;
  }
  __syncthreads();
  uint64_t* base = static_cast<uint64_t*>(ws);
  uint64_t* done = base + 3;
  double* part = reinterpret_cast<double*>(base + kWsMinmaxOff);
  if (threadIdx.x == 0) {
    for (int k = 1; k < kMmThreads / 32; ++k) {
      lo = fmin(lo, s_lo[k]);
      hi = fmax(hi, s_hi[k]);
    }
    part[2 * blockIdx.x] = lo;
    part[2 * blockIdx.x + 1] = hi;
    __threadfence();
    s_last = atom_add_acq_rel(done, 1) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  lo = INFINITY;
  hi = -INFINITY;
  for (unsigned k = threadIdx.x; k < gridDim.x; k += blockDim.x) {
    lo = fmin(lo, __longlong_as_double(ld_relaxed(reinterpret_cast<uint64_t*>(part + 2 * k))));
    hi = fmax(hi, __longlong_as_double(ld_relaxed(reinterpret_cast<uint64_t*>(part + 2 * k + 1))));
  }
  for (int m = 16; m > 0; m >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(kFull, lo, m));
    hi = fmax(hi, __shfl_xor_sync(kFull, hi, m));
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    s_lo[warp] = lo;
    s_hi[warp] = hi;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int k = 1; k < kMmThreads / 32; ++k) {
    lo = fmin(lo, s_lo[k]);
    hi = fmax(hi, s_hi[k]);
  }
  out[0] = lo;
  out[1] = hi;
  st_relaxed(done, 0);
  const uint64_t res[2] = {static_cast<uint64_t>(__double_as_longlong(lo)),
                           static_cast<uint64_t>(__double_as_longlong(hi))};
  mailbox_post(mb, res, 2, err);
}

// ---- K4 for block_len 32: every stored sign byte flips (full blocks have 4
// sign bytes, all bits live); only the partial tail block's last byte keeps
// its zero padding (ops.py:88-109).  One wave of CTAs (SMs x 8); per round a
// thread issues ALL its loads -- kStreamU 16-byte outlier chunks and
// kStreamU 16-byte sign chunks -- before it computes or stores anything, so
// a round costs one DRAM round trip (the arrays are 10s of MB: latency, not
// bandwidth, is what a naive grid-stride loop pays).
constexpr int kStreamU = 4;
constexpr int kStreamThreads = 256;

__device__ __forceinline__ int4 neg4(int4 v, uint32_t& flags) {
  flags |= (v.x == INT32_MIN) | (v.y == INT32_MIN) | (v.z == INT32_MIN) | (v.w == INT32_MIN)
               ? HSZ_ERR_OUTLIER_OVERFLOW : 0u;
  return make_int4(-v.x, -v.y, -v.z, -v.w);
}

__global__ void __launch_bounds__(kStreamThreads) negate32_kernel(
    const uint8_t* __restrict__ widths, const int32_t* __restrict__ oin, int32_t* __restrict__ oout,
    const uint8_t* __restrict__ sin, uint8_t* __restrict__ sout, const uint64_t* __restrict__ toff,
    uint64_t ntiles, uint64_t n, uint64_t nblocks, uint64_t sign_chunks_max, uint32_t* err) {
  const uint64_t S = __ldg(toff + 2 * ntiles);          // issued first: the sign bound
  const uint64_t noc = nblocks / 4;                    // full outlier chunks
  const uint32_t r = static_cast<uint32_t>(n % 32);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int4* oin4 = reinterpret_cast<const int4*>(oin);
  int4* oout4 = reinterpret_cast<int4*>(oout);
  const uint4* sin4 = reinterpret_cast<const uint4*>(sin);
  uint4* sout4 = reinterpret_cast<uint4*>(sout);
  uint32_t flags = 0;
  (void)sign_chunks_max;
  for (uint64_t c0 = tid;; c0 += kStreamU * stride) {
    const uint64_t nsc = (S + 15) / 16;                // sign chunks in use
    if (c0 >= noc && c0 >= nsc) break;
    int4 ov[kStreamU];
    uint4 sv[kStreamU];
#pragma unroll
    for (int u = 0; u < kStreamU; ++u) {
      const uint64_t c = c0 + u * stride;
      if (c < noc) ov[u] = __ldcs(oin4 + c);
    }
#pragma unroll
    for (int u = 0; u < kStreamU; ++u) {
      const uint64_t c = c0 + u * stride;
      if (c < nsc) sv[u] = __ldcs(sin4 + c);
    }
#pragma unroll
    for (int u = 0; u < kStreamU; ++u) {
      const uint64_t c = c0 + u * stride;
      if (c < noc) oout4[c] = neg4(ov[u], flags);
    }
#pragma unroll
    for (int u = 0; u < kStreamU; ++u) {
      const uint64_t c = c0 + u * stride;
      if (c < nsc) {
        uint4 v = make_uint4(~sv[u].x, ~sv[u].y, ~sv[u].z, ~sv[u].w);
        if (c == nsc - 1 && (r & 7u) != 0 && widths[nblocks - 1] > 0) {
          // the tail block's last sign byte: its padding bits stay zero
          const uint32_t j = static_cast<uint32_t>((S - 1) & 15u);
          const uint32_t tmask = (0xFFu << (8 - (r & 7u))) & 0xFFu;
          reinterpret_cast<uint32_t*>(&v)[j >> 2] ^= (0xFFu ^ tmask) << (8 * (j & 3u));
        }
        sout4[c] = v;
      }
    }
  }

  for (uint64_t b = noc * 4 + tid; b < nblocks; b += stride) {   // the last < 4 outliers
    const int32_t v = oin[b];
    if (v == INT32_MIN) flags |= HSZ_ERR_OUTLIER_OVERFLOW;
    oout[b] = -v;
  }
  if (flags) atomicOr(err, flags);
}

// ---- K4: negate (ops.py:88-109) --------------------------------------------
// Every stored sign bit flips; padding bits of a block's last sign byte stay
// 0.  Full non-constant blocks all contribute sk = ceil(k/8) bytes, so the
// mask of byte j depends only on j % sk -- except for a partial tail block,
// which always sits at the very end of the section.
__global__ void __launch_bounds__(kThreads) negate_kernel(
    const uint8_t* widths, const int32_t* oin, int32_t* oout, const uint8_t* sin, uint8_t* sout,
    const uint64_t* toff, uint64_t ntiles, uint64_t n, uint32_t k, uint64_t nblocks,
    uint32_t* err) {
  const uint64_t S = toff[2 * ntiles];
  const uint32_t r = static_cast<uint32_t>(n % k);
  const bool tail_part = r != 0 && widths[nblocks - 1] > 0;
  const uint64_t tail_bytes = tail_part ? (r + 7) / 8 : 0;
  const uint64_t per_end = S - tail_bytes;
  const uint32_t sk = (k + 7) / 8, kr = k & 7;
  const uint8_t kmask = static_cast<uint8_t>((0xFFu << (8 - kr)) & 0xFFu);
  const uint8_t tmask = static_cast<uint8_t>((0xFFu << (8 - (r & 7))) & 0xFFu);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  // sign planes, 16 bytes per thread step
  const uint64_t nchunks = (S + 15) / 16;
  for (uint64_t c = tid; c < nchunks; c += stride) {
    const uint64_t j0 = c * 16;
    if (kr == 0 && j0 + 16 <= per_end) {
      uint4 v = *reinterpret_cast<const uint4*>(sin + j0);
      v.x = ~v.x;
      v.y = ~v.y;
      v.z = ~v.z;
      v.w = ~v.w;
      *reinterpret_cast<uint4*>(sout + j0) = v;
      continue;
    }
    const uint64_t j1 = (j0 + 16 < S) ? j0 + 16 : S;
    for (uint64_t j = j0; j < j1; ++j) {
      uint8_t m = 0xFF;
      if (j < per_end) {
        if (kr && (j % sk) == sk - 1) m = kmask;
      } else if (j == S - 1 && (r & 7)) {
        m = tmask;
      }
      sout[j] = sin[j] ^ m;
    }
  }
  // outliers
  uint32_t flags = 0;
  for (uint64_t i = tid; i < nblocks; i += stride) {
    const int64_t v = -static_cast<int64_t>(oin[i]);
    if (v > INT32_MAX) flags |= HSZ_ERR_OUTLIER_OVERFLOW;
    oout[i] = static_cast<int32_t>(v);
  }
  if (flags) atomicOr(err, flags);
}

// ---- K5: scalar add (ops.py:112-118) -----------------------------------------
// outlier + rs in int64 (numpy wraps), then the int32 guard (model.py:182-191).
// A wrapped int64 sum can never land back inside int32 (|rs| < 2^63), so the
// guard on the wrapped value is the exact test.  kSmall (rs fits int32): the
// same result from a 32-bit add, overflow iff the operands agree in sign and
// the sum does not -- 3 instructions an element instead of ~30 for the int128
// form, which made this streaming kernel issue-bound.
template <bool kSmall>
__device__ __forceinline__ int32_t sadd1(int32_t o, int64_t rs, uint32_t& bad) {
  if constexpr (kSmall) {
    const int32_t r = static_cast<int32_t>(rs);
    const int32_t v = static_cast<int32_t>(static_cast<uint32_t>(o) + static_cast<uint32_t>(r));
    bad |= static_cast<uint32_t>((o ^ v) & (r ^ v));          // sign bit: signed overflow
    return v;
  } else {
    const int64_t v = static_cast<int64_t>(static_cast<uint64_t>(static_cast<int64_t>(o)) +
                                           static_cast<uint64_t>(rs));
    bad |= (static_cast<uint64_t>(v) + 0x80000000ull) > 0xFFFFFFFFull ? 0x80000000u : 0u;
    return static_cast<int32_t>(v);
  }
}

template <bool kSmall>
__global__ void __launch_bounds__(kStreamThreads) sadd_kernel(const int32_t* oin, int32_t* oout,
                                                              uint64_t nblocks, int64_t rs,
                                                              uint32_t* err) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t bad = 0;
  const bool vec = ((reinterpret_cast<uintptr_t>(oin) | reinterpret_cast<uintptr_t>(oout)) & 15u) == 0;
  const uint64_t nv = vec ? nblocks / 4 : 0;
  const int4* in4 = reinterpret_cast<const int4*>(oin);
  int4* out4 = reinterpret_cast<int4*>(oout);
  // one DRAM round trip per round: all kStreamU loads issued before any store
  for (uint64_t c0 = tid; c0 < nv; c0 += kStreamU * stride) {
    int4 v[kStreamU];
#pragma unroll
    for (int u = 0; u < kStreamU; ++u) {
      const uint64_t c = c0 + u * stride;
      if (c < nv) v[u] = __ldcs(in4 + c);
    }
#pragma unroll
    for (int u = 0; u < kStreamU; ++u) {
      const uint64_t c = c0 + u * stride;
      if (c < nv)
        out4[c] = make_int4(sadd1<kSmall>(v[u].x, rs, bad), sadd1<kSmall>(v[u].y, rs, bad),
                            sadd1<kSmall>(v[u].z, rs, bad), sadd1<kSmall>(v[u].w, rs, bad));
    }
  }
  for (uint64_t j = nv * 4 + tid; j < nblocks; j += stride) oout[j] = sadd1<kSmall>(oin[j], rs, bad);
  if (__any_sync(kFull, (bad >> 31) != 0) && (threadIdx.x & 31) == 0)
    atomicOr(err, HSZ_ERR_OUTLIER_OVERFLOW);
}

}  // namespace ops

// ---------------------------------------------------------------------------
// launch helpers

static inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

static inline int launch_status() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "hsz_b200: CUDA launch failed: %s\n", cudaGetErrorString(e));
    return HSZ_ECUDA;
  }
  return HSZ_OK;
}

template <typename Kern>
static inline void allow_smem(Kern kern, int bytes) {
  static int configured_device = -1;   // one static per kernel instantiation
  int dev = 0;
  cudaGetDevice(&dev);
  if (bytes > 48 * 1024 && configured_device != dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    configured_device = dev;
  }
}

static inline uint64_t grid_for(uint64_t items, uint64_t per_thread, int threads, uint64_t cap) {
  uint64_t g = ceil_div(ceil_div(items, per_thread), threads);
  if (g < 1) g = 1;
  return g < cap ? g : cap;
}

// one resident wave of 256-thread streaming CTAs: SMs x 8
static inline uint64_t stream_wave() {
  static int sms = 0, dev_cached = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev_cached != dev) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    dev_cached = dev;
  }
  return static_cast<uint64_t>(sms > 0 ? sms : 148) * 8;
}

static inline uint32_t tail_len_of(uint64_t n, uint32_t k) {
  const uint32_t r = static_cast<uint32_t>(n % k);
  return r ? r : k;
}

template <class Src>
static int launch_encode32(Src src, const k32::EncodeOut& out, uint64_t n, cudaStream_t st) {
  const uint64_t nb = ceil_div(n, 32);
  const uint64_t nt = ceil_div(nb, kTileBlocks);
  auto kern = k32::encode_kernel<Src>;
  constexpr int smem = k32::EncodeSmem<Src>::kBytes;
  allow_smem(kern, smem);
  // persistent: as many CTAs as can be co-resident, each looping over tickets
  static int resident = 0, resident_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (resident_dev != dev) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, k32::kEncThreads, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    resident = per_sm > 0 ? per_sm * sms : sms;
    resident_dev = dev;
  }
  const uint64_t grid = nt < static_cast<uint64_t>(resident) ? nt : static_cast<uint64_t>(resident);
  kern<<<static_cast<unsigned>(grid), k32::kEncThreads, smem, st>>>(src, out, nb, nt, tail_len_of(n, 32));
  return launch_status();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D tensor map over a float32 field viewed as rows of 32 values (one block
// per row), 128-row boxes, 128-byte swizzle; false if the field does not allow it
static bool make_rows_map_f32_uncached(const float* x, uint64_t n, CUtensorMap* map);

// the encoded maps of the last few (pointer, length) pairs, per host thread:
// a chain of ops on the same buffers skips cuTensorMapEncodeTiled
static bool make_rows_map_f32(const float* x, uint64_t n, CUtensorMap* map) {
  struct Entry {
    const float* x;
    uint64_t n;
    bool ok;
    CUtensorMap map;
  };
  static thread_local Entry cache[4] = {};
  static thread_local int next = 0;
  for (const Entry& e : cache)
    if (e.x == x && e.n == n && x) {
      *map = e.map;
      return e.ok;
    }
  const bool ok = make_rows_map_f32_uncached(x, n, map);
  Entry& e = cache[next];
  next = (next + 1) & 3;
  e.x = x;
  e.n = n;
  e.ok = ok;
  e.map = *map;
  return ok;
}

static bool make_rows_map_f32_uncached(const float* x, uint64_t n, CUtensorMap* map) {
  std::memset(map, 0, sizeof(*map));
  const uint64_t rows = n / 32;
  if ((reinterpret_cast<uintptr_t>(x) & 15u) != 0 || rows < static_cast<uint64_t>(kTileBlocks) ||
      rows >= (1ull << 31))
    return false;
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {32, rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {32, static_cast<cuuint32_t>(kTileBlocks)};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D tensor map over int64 bins viewed as [half][block][16 bins] (dims
// reordered: the block stride is 256 B, the half stride 128 B), 128-row boxes
// of both halves, 128-byte swizzle -- the staged image puts block r's two
// 128-byte rows at r and 128 + r, so the swizzle spreads a wavefront's 8
// threads over 8 bank groups (e32::bins_off)
static bool make_bins_map(const int64_t* b, uint64_t n, CUtensorMap* map) {
  std::memset(map, 0, sizeof(*map));
  const uint64_t rows = n / 32;
  if ((reinterpret_cast<uintptr_t>(b) & 15u) != 0 || rows < static_cast<uint64_t>(kTileBlocks) ||
      rows >= (1ull << 31))
    return false;
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {16, rows, 2};
  cuuint64_t strides[2] = {256, 128};
  cuuint32_t box[3] = {16, static_cast<cuuint32_t>(kTileBlocks), 2};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, const_cast<int64_t*>(b), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int kMode>
static int launch_decode_pipe(const d32::StreamIn& in, float* out, double d, uint64_t* mout,
                              void* ws, uint32_t* err, cudaStream_t st, Mailbox mb = Mailbox{nullptr, 0}) {
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  int use_tma = 0;
  if (kMode == 2) use_tma = make_rows_map_f32(out, in.n, &map) ? 1 : 0;
  constexpr int smem = static_cast<int>(d32::dec_smem_bytes<kMode>());
  auto kern = d32::decode_pipe_kernel<kMode>;
  static int resident = 0, resident_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (resident_dev != dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, d32::kDecThreads, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    resident = (per_sm > 0 ? per_sm : 1) * sms;
    resident_dev = dev;
  }
  const uint64_t grid = in.ntiles < static_cast<uint64_t>(resident) ? in.ntiles : static_cast<uint64_t>(resident);
  const d32::DecF32Sink fs{out, d, d * 0x1p33 >= 3.4028234663852886e38};
  const d32::MomentsSink ms{mout, ws, mb};
  kern<<<static_cast<unsigned>(grid), d32::kDecThreads, smem, st>>>(map, in, fs, ms, use_tma, err);
  return launch_status();
}

// compress of a float32 field, block_len 32: register-resident encoder with
// a swizzled 2-D TMA tile load when the field allows it
static int launch_compress_f32(const float* x, uint64_t n, const QuantConst& c,
                               const k32::EncodeOut& out, cudaStream_t st) {
  const uint64_t nb = ceil_div(n, 32);
  const uint64_t nt = ceil_div(nb, kTileBlocks);
  const e32::QuantF32 qf = e32::make_quant_f32(c);
  CUtensorMap map;
  const bool tma = make_rows_map_f32(x, n, &map);
  constexpr int smem = static_cast<int>(e32::kSmem7Bytes);
  auto kern = tma ? e32::compress_f32_kernel<true> : e32::compress_f32_kernel<false>;
  // persistent grid: every CTA resident (the look-back relies on it)
  static int resident[2] = {0, 0}, resident_dev[2] = {-1, -1};
  int dev = 0;
  cudaGetDevice(&dev);
  if (resident_dev[tma] != dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, e32::kThreadsC, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    resident[tma] = (per_sm > 0 ? per_sm : 1) * sms;
    resident_dev[tma] = dev;
  }
  const uint64_t grid = nt < static_cast<uint64_t>(resident[tma]) ? nt : static_cast<uint64_t>(resident[tma]);
  kern<<<static_cast<unsigned>(grid), e32::kThreadsC, smem, st>>>(map, x, n, qf, c, out, nb, nt,
                                                                tail_len_of(n, 32), nullptr);
  return launch_status();
}

// encode_from_quant, block_len 32: the compressor's register-resident
// encoder fed by a 3-D TMA tile of int64 bins; false if the bins do not allow
// the tensor map (the caller then takes the first-generation encoder)
static bool launch_encode_bins32(const int64_t* bins, uint64_t n, const k32::EncodeOut& out,
                                 cudaStream_t st, int* rc) {
  CUtensorMap map;
  if (!make_bins_map(bins, n, &map)) return false;
  const uint64_t nb = ceil_div(n, 32);
  const uint64_t nt = ceil_div(nb, kTileBlocks);
  constexpr int smem = static_cast<int>(e32::kSmem7BinsBytes);
  auto kern = e32::compress_f32_kernel<true, true>;
  static int resident = 0, resident_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (resident_dev != dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, e32::kThreadsC, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    resident = (per_sm > 0 ? per_sm : 1) * sms;
    resident_dev = dev;
  }
  const uint64_t grid = nt < static_cast<uint64_t>(resident) ? nt : static_cast<uint64_t>(resident);
  const e32::QuantF32 qf{0.f, 0.f, -1.f};
  const QuantConst qc = make_quant_const(1.0);
  kern<<<static_cast<unsigned>(grid), e32::kThreadsC, smem, st>>>(map, nullptr, n, qf, qc, out, nb, nt,
                                                                tail_len_of(n, 32), bins);
  *rc = launch_status();
  return true;
}

template <class G>
static int launch_encode_generic(G src, uint64_t n, uint32_t k, uint8_t* widths,
                                 int32_t* outliers, uint8_t* signs, uint64_t sign_cap,
                                 uint8_t* payload, uint64_t payload_cap, uint64_t* toff,
                                 uint32_t* err, void* ws, cudaStream_t st) {
  const uint64_t nb = ceil_div(n, k);
  const uint64_t nt = ceil_div(nb, kTileBlocks);
  gen::widths_kernel<G><<<static_cast<unsigned>(ceil_div(nb, gen::kThreads)), gen::kThreads, 0, st>>>(
      src, n, k, nb, widths, outliers, err);
  gen::tile_offsets_kernel<<<static_cast<unsigned>(nt), gen::kThreads, 0, st>>>(widths, n, k, nb, nt,
                                                                               toff, err, ws);
  gen::pack_kernel<G><<<static_cast<unsigned>(nt), gen::kThreads, 0, st>>>(
      src, n, k, nb, nt, widths, toff, signs, sign_cap, payload, payload_cap, err);
  return launch_status();
}

namespace ops {
template <typename T>
__global__ void quantize_kernel(const T* x, uint64_t n, QuantConst c, int64_t* bins, uint32_t* err) {
  uint32_t flags = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    bins[i] = quantize1(static_cast<double>(x[i]), c, &flags);
  if (flags) atomicOr(err, flags);
}
}  // namespace ops

namespace ops {
// element-wise combination sink: acc[e] = acc[e] (+|-) bin, modulo 2^64 --
// the re-encoder's residuals bin[i] - bin[i-1] are then exactly the sums of
// the operands' residuals (ops.py:171-176) whenever those fit 63 bits
struct SinkCombineBins {
  int64_t* acc;
  int sub;
  __device__ __forceinline__ void put(uint64_t e, int64_t bin, uint32_t*) const {
    const uint64_t a = static_cast<uint64_t>(acc[e]);
    acc[e] = static_cast<int64_t>(sub ? a - static_cast<uint64_t>(bin) : a + static_cast<uint64_t>(bin));
  }
};
}  // namespace ops

namespace ops {
struct SinkAcc {
  k32::Acc acc;
  bool want_sq;
  __device__ __forceinline__ void put(uint64_t, int64_t bin, uint32_t*) { acc.add(bin, want_sq); }
};

__global__ void __launch_bounds__(gen::kThreads) gen_moments_kernel(gen::GStream s, int want_sq,
                                                                    uint64_t* out, uint32_t* err,
                                                                    void* ws) {
  uint32_t flags = 0;
  SinkAcc sink;
  sink.acc.s = 0;
  sink.acc.q = 0;
  sink.acc.q2 = 0;
  sink.want_sq = want_sq != 0;
  const uint64_t tile = blockIdx.x;
  gen::decode_one_block(s, tile, tile * gen::kThreads + threadIdx.x, sink, &flags);
  if (flags) atomicOr(err, flags);
  k32::finish_moments(sink.acc, gridDim.x, ws, out);
}
}  // namespace ops

namespace ops {
template <class Sink>
__global__ void dequant_kernel(const int64_t* bins, uint64_t n, Sink sink, uint32_t* err) {
  uint32_t flags = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    sink.put(i, bins[i], &flags);
  if (flags) atomicOr(err, flags);
}
}  // namespace ops

}  // namespace hsz

using namespace hsz;

// ===========================================================================
// persistent re-encoding kernel (scalar multiply, element-wise add / sub):
// one CTA per resident slot, tiles by ticket
template <int kOp>
static int launch_recode(const d32::StreamIn& a, const d32::StreamIn& b, const d32::SmulParams& sp,
                         const k32::EncodeOut& out, uint64_t nt, cudaStream_t st) {
  constexpr int smem = static_cast<int>(d32::recode_smem_bytes<kOp>());
  auto kern = d32::recode_kernel<kOp>;
  static int resident = 0, resident_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (resident_dev != dev) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, e32::kThreadsWS, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    #ifdef HSZ_RECODE_CTAS_CAP
    if (per_sm > HSZ_RECODE_CTAS_CAP) per_sm = HSZ_RECODE_CTAS_CAP;
#endif
    resident = (per_sm > 0 ? per_sm : 1) * sms;
    resident_dev = dev;
  }
  const uint64_t grid = nt < static_cast<uint64_t>(resident) ? nt : static_cast<uint64_t>(resident);
  kern<<<static_cast<unsigned>(grid), e32::kThreadsWS, smem, st>>>(a, b, sp, out);
  return launch_status();
}

#ifndef HSZ_BINS_REGISTER_PATH
#define HSZ_BINS_REGISTER_PATH 1
#endif

namespace hsz {
namespace ops {
// mailbox post for reduction paths that do not post in-kernel
__global__ void mailbox_post_kernel(Mailbox mb, const uint64_t* res, int nres, const uint32_t* err) {
  uint64_t r[5];
  for (int i = 0; i < nres; ++i) r[i] = res[i];
  mailbox_post(mb, r, nres, err);
}
}  // namespace ops
}  // namespace hsz

extern "C" {

const char* hsz_version(void) { return "hsz_b200 1.1 sm_100a"; }

unsigned int hsz_set_lookback_watchdog(unsigned int max_sleeps) {
  unsigned int old = 0;
  if (cudaMemcpyFromSymbol(&old, hsz::g_lb_max_sleeps, sizeof(old)) != cudaSuccess) return 0;
  if (max_sleeps) cudaMemcpyToSymbol(hsz::g_lb_max_sleeps, &max_sleeps, sizeof(max_sleeps));
  return old;
}

// debug: copy out phase-trace records (only in -DHSZ_TRACE builds; returns count)
int hsz_trace_read(unsigned long long* host, int cap, int reset) {
#ifdef HSZ_TRACE
  unsigned int n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, g_trace_n, sizeof(n));
  if (n > static_cast<unsigned>(kTraceCap)) n = kTraceCap;
  if (static_cast<int>(n) > cap) n = cap;
  if (host && n) cudaMemcpyFromSymbol(host, g_trace, n * sizeof(unsigned long long));
  if (reset) {
    unsigned int z = 0;
    cudaMemcpyToSymbol(g_trace_n, &z, sizeof(z));
  }
  return static_cast<int>(n);
#else
  (void)host; (void)cap; (void)reset;
  return -1;
#endif
}

// debug: look-back statistics since the last call (rounds, sleeps, resolves)
int hsz_trace_lookback(unsigned int* out3) {
#ifdef HSZ_TRACE
  cudaDeviceSynchronize();
  {
    unsigned long long c[2] = {0, 0};
    cudaMemcpyFromSymbol(&c[0], g_lb_cycles_round, 8);
    cudaMemcpyFromSymbol(&c[1], g_lb_cycles_total, 8);
    unsigned int calls = 0;
    cudaMemcpyFromSymbol(&calls, g_lb_calls, 4);
    if (calls) fprintf(stderr, "lookback cycles: round-load %.0f total %.0f per resolve\n",
                       double(c[0]) / calls, double(c[1]) / calls);
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(g_lb_cycles_round, &z, 8);
    cudaMemcpyToSymbol(g_lb_cycles_total, &z, 8);
  }
  unsigned int v[3] = {0, 0, 0};
  cudaMemcpyFromSymbol(&v[0], g_lb_rounds, sizeof(unsigned));
  cudaMemcpyFromSymbol(&v[1], g_lb_sleeps, sizeof(unsigned));
  cudaMemcpyFromSymbol(&v[2], g_lb_calls, sizeof(unsigned));
  const unsigned int z = 0;
  cudaMemcpyToSymbol(g_lb_rounds, &z, sizeof(z));
  cudaMemcpyToSymbol(g_lb_sleeps, &z, sizeof(z));
  cudaMemcpyToSymbol(g_lb_calls, &z, sizeof(z));
  if (out3) for (int i = 0; i < 3; ++i) out3[i] = v[i];
  return 3;
#else
  (void)out3;
  return -1;
#endif
}

int hsz_copy_d2h(void* host, const void* dev, uint64_t bytes, void* stream) {
  if (!host || !dev) return HSZ_EINVAL;
  return cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess
             ? HSZ_OK
             : HSZ_ECUDA;
}

// Host-side waits are bounded: a kernel that never finishes (a GPU-side hang)
// turns into HSZ_ETIMEDOUT after g_host_wait_s seconds instead of blocking the
// calling thread forever (which no Python-level timeout could interrupt).
static double g_host_wait_s = 600.0;

static inline double wall_s() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<double>(ts.tv_sec) + 1e-9 * static_cast<double>(ts.tv_nsec);
}

static int bounded_sync(cudaStream_t st) {
  cudaError_t e = cudaStreamQuery(st);
  if (e == cudaSuccess) return HSZ_OK;
  const double t0 = wall_s();
  for (uint64_t it = 1;; ++it) {
    if (e == cudaSuccess) return HSZ_OK;
    if (e != cudaErrorNotReady) return HSZ_ECUDA;
    if ((it & 1023u) == 0 && wall_s() - t0 > g_host_wait_s) return HSZ_ETIMEDOUT;
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
    e = cudaStreamQuery(st);
  }
}

double hsz_set_host_wait_timeout(double seconds) {
  const double old = g_host_wait_s;
  if (seconds > 0) g_host_wait_s = seconds;
  return old;
}

int hsz_fetch(void* host, const void* dev, uint64_t bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess) return HSZ_ECUDA;
  return bounded_sync(st);
}

int hsz_stream_sync(void* stream) { return bounded_sync(static_cast<cudaStream_t>(stream)); }

uint64_t hsz_tile_count(uint64_t n, uint32_t k) {
  if (k == 0) return 0;
  return ceil_div(ceil_div(n, k), kTileBlocks);
}

uint64_t hsz_sign_bound(uint64_t n, uint32_t k) {
  if (k == 0) return 0;
  return ceil_div(n, k) * ((k + 7) / 8);
}

uint64_t hsz_payload_bound(uint64_t n, uint32_t k) {
  if (k == 0) return 0;
  return ceil_div(n, k) * (static_cast<uint64_t>(k) * 8);
}

uint64_t hsz_workspace_size(uint64_t n, uint32_t k) {
  const uint64_t nt = hsz_tile_count(n, k);
  // header + minmax partials, then 8 words per tile: the look-back records
  // (kLbStride words) or the flag/value protocol (7 words)
  return 8 * (kWsFlagsOff + 8 * (nt + 1));
}

int hsz_workspace_init(void* ws, uint64_t ws_bytes, void* stream) {
  if (!ws) return HSZ_EINVAL;
  return cudaMemsetAsync(ws, 0, ws_bytes, static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? HSZ_OK
             : HSZ_ECUDA;
}

uint64_t hsz_scalar_mul_scratch_size(uint64_t n, uint32_t k) { return k == 32 ? 0 : 8 * n; }

int hsz_minmax_mb(const void* x, int dtype, uint64_t n, double* minmax, uint32_t* err, void* ws,
                  uint64_t ws_bytes, uint64_t* mailbox, uint64_t seq, void* stream) {
  if (!x || !minmax || !err || !ws || n == 0) return HSZ_EINVAL;
  if (ws_bytes < 8 * kWsFlagsOff) return HSZ_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned g = static_cast<unsigned>(grid_for(n, dtype == HSZ_F32 ? 16 : 8, ops::kThreads, ops::kMinmaxCtas));
  if (dtype == HSZ_F32 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0) {
    const unsigned g2 = static_cast<unsigned>(grid_for(n, 32, ops::kMmThreads, ops::kMinmaxCtas));
    ops::minmax_f32_kernel<<<g2, ops::kMmThreads, 0, st>>>(static_cast<const float*>(x), n, minmax, err, ws,
                                                           Mailbox{mailbox, seq});
  } else {
    if (dtype == HSZ_F32)
      ops::minmax_kernel<float><<<g, ops::kThreads, 0, st>>>(static_cast<const float*>(x), n, minmax, err, ws);
    else if (dtype == HSZ_F64)
      ops::minmax_kernel<double><<<g, ops::kThreads, 0, st>>>(static_cast<const double*>(x), n, minmax, err, ws);
    else
      return HSZ_EINVAL;
    if (mailbox)
      ops::mailbox_post_kernel<<<1, 1, 0, st>>>(Mailbox{mailbox, seq},
                                                reinterpret_cast<const uint64_t*>(minmax), 2, err);
  }
  return launch_status();
}

int hsz_minmax(const void* x, int dtype, uint64_t n, double* minmax, uint32_t* err, void* ws,
               uint64_t ws_bytes, void* stream) {
  return hsz_minmax_mb(x, dtype, n, minmax, err, ws, ws_bytes, nullptr, 0, stream);
}

int hsz_compress(const void* x, int dtype, uint64_t n, uint32_t k, double eps, uint8_t* widths,
                 int32_t* outliers, uint8_t* signs, uint64_t sign_cap, uint8_t* payload,
                 uint64_t payload_cap, uint64_t* toff, uint32_t* err, void* ws,
                 uint64_t ws_bytes, void* stream) {
  if (!x || !widths || !outliers || !signs || !payload || !toff || !err || !ws || n == 0 || k == 0)
    return HSZ_EINVAL;
  if (ws_bytes < hsz_workspace_size(n, k)) return HSZ_EINVAL;
  if (dtype != HSZ_F32 && dtype != HSZ_F64) return HSZ_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const QuantConst c = make_quant_const(eps);
  if (k == 32) {
    const k32::EncodeOut out{widths, outliers, signs, sign_cap, payload, payload_cap, toff, err, ws};
    if (dtype == HSZ_F32) return launch_compress_f32(static_cast<const float*>(x), n, c, out, st);
    return launch_encode32(k32::SrcQuant<double>{static_cast<const double*>(x), n, c}, out, n, st);
  }
  if (dtype == HSZ_F32)
    return launch_encode_generic(gen::GQuant<float>{static_cast<const float*>(x), c}, n, k, widths, outliers,
                                 signs, sign_cap, payload, payload_cap, toff, err, ws, st);
  return launch_encode_generic(gen::GQuant<double>{static_cast<const double*>(x), c}, n, k, widths, outliers,
                               signs, sign_cap, payload, payload_cap, toff, err, ws, st);
}

int hsz_encode_bins(const int64_t* bins, uint64_t n, uint32_t k, uint8_t* widths, int32_t* outliers,
                    uint8_t* signs, uint64_t sign_cap, uint8_t* payload, uint64_t payload_cap,
                    uint64_t* toff, uint32_t* err, void* ws, uint64_t ws_bytes, void* stream) {
  if (!bins || !widths || !outliers || !signs || !payload || !toff || !err || !ws || n == 0 || k == 0)
    return HSZ_EINVAL;
  if (ws_bytes < hsz_workspace_size(n, k)) return HSZ_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (k == 32) {
    const k32::EncodeOut out{widths, outliers, signs, sign_cap, payload, payload_cap, toff, err, ws};
#if HSZ_BINS_REGISTER_PATH
    int rc = HSZ_OK;
    if (launch_encode_bins32(bins, n, out, st, &rc)) return rc;
#endif
    return launch_encode32(k32::SrcBins{bins, n}, out, n, st);
  }
  return launch_encode_generic(gen::GBins{bins}, n, k, widths, outliers, signs, sign_cap, payload,
                               payload_cap, toff, err, ws, st);
}


int hsz_quantize(const void* x, int dtype, uint64_t n, double eps, int64_t* bins, uint32_t* err,
                 void* stream) {
  if (!x || !bins || !err || n == 0) return HSZ_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const QuantConst c = make_quant_const(eps);
  const unsigned g = static_cast<unsigned>(grid_for(n, 4, 256, 148 * 16));
  if (dtype == HSZ_F32)
    ops::quantize_kernel<float><<<g, 256, 0, st>>>(static_cast<const float*>(x), n, c, bins, err);
  else if (dtype == HSZ_F64)
    ops::quantize_kernel<double><<<g, 256, 0, st>>>(static_cast<const double*>(x), n, c, bins, err);
  else
    return HSZ_EINVAL;
  return launch_status();
}

int hsz_dequantize(const int64_t* bins, uint64_t n, double eps, int out_kind, void* out,
                   uint32_t* err, void* stream) {
  if (!bins || !out || !err || n == 0) return HSZ_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned g = static_cast<unsigned>(grid_for(n, 4, 256, 148 * 16));
  const double d = 2.0 * eps;
  if (out_kind == HSZ_OUT_F32)
    ops::dequant_kernel<<<g, 256, 0, st>>>(bins, n, k32::SinkF32{static_cast<float*>(out), d, d * 0x1p33 >= 3.4028234663852886e38}, err);
  else if (out_kind == HSZ_OUT_F64)
    ops::dequant_kernel<<<g, 256, 0, st>>>(bins, n, k32::SinkF64{static_cast<double*>(out), d, d * 0x1p33 >= 1.7976931348623157e308}, err);
  else
    return HSZ_EINVAL;
  return launch_status();
}

int hsz_tile_offsets(const uint8_t* widths, uint64_t n, uint32_t k, uint64_t* toff, uint32_t* err,
                     void* ws, uint64_t ws_bytes, void* stream) {
  if (!widths || !toff || !err || !ws || n == 0 || k == 0) return HSZ_EINVAL;
  if (ws_bytes < hsz_workspace_size(n, k)) return HSZ_EINVAL;
  const uint64_t nb = ceil_div(n, k);
  const uint64_t nt = ceil_div(nb, kTileBlocks);
  gen::tile_offsets_kernel<<<static_cast<unsigned>(nt), gen::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      widths, n, k, nb, nt, toff, err, ws);
  return launch_status();
}

int hsz_decode(const uint8_t* widths, const int32_t* outliers, const uint8_t* signs,
               const uint8_t* payload, const uint64_t* toff, uint64_t n, uint32_t k, double eps,
               int out_kind, void* out, uint32_t* err, void* stream) {
  if (!widths || !outliers || !signs || !payload || !toff || !out || !err || n == 0 || k == 0)
    return HSZ_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t nb = ceil_div(n, k);
  const uint64_t nt = ceil_div(nb, kTileBlocks);
  const double d = 2.0 * eps;
  if (out_kind == HSZ_OUT_BINS_ADD || out_kind == HSZ_OUT_BINS_SUB) {
    // accumulate into existing int64 bins (folds of several streams)
    const gen::GStream s{widths, outliers, signs, payload, toff, n, k, nb};
    gen::decode_kernel<ops::SinkCombineBins><<<static_cast<unsigned>(nt), gen::kThreads, 0, st>>>(
        s, ops::SinkCombineBins{static_cast<int64_t*>(out), out_kind == HSZ_OUT_BINS_SUB ? 1 : 0}, err);
    return launch_status();
  }
  if (k == 32) {
    const k32::StreamIn s{widths, outliers, signs, payload, toff, n, nb, tail_len_of(n, 32)};
    const unsigned g = static_cast<unsigned>(nt);
    switch (out_kind) {
      case HSZ_OUT_F32: {
        const d32::StreamIn in{widths, outliers, signs, payload, toff, n, nb, nt, tail_len_of(n, 32)};
        return launch_decode_pipe<2>(in, static_cast<float*>(out), d, nullptr, nullptr, err, st);
      }
      case HSZ_OUT_F64: {
        constexpr int smem = k32::DecodeSmem<k32::SinkF64>::kBytes;
        allow_smem(k32::decode_kernel<k32::SinkF64>, smem);
        k32::decode_kernel<k32::SinkF64><<<g, k32::kThreads, smem, st>>>(
            s, k32::SinkF64{static_cast<double*>(out), d, d * 0x1p33 >= 1.7976931348623157e308}, err);
        break;
      }
      case HSZ_OUT_BINS: {
        constexpr int smem = k32::DecodeSmem<k32::SinkBins>::kBytes;
        allow_smem(k32::decode_kernel<k32::SinkBins>, smem);
        k32::decode_kernel<k32::SinkBins><<<g, k32::kThreads, smem, st>>>(
            s, k32::SinkBins{static_cast<int64_t*>(out)}, err);
        break;
      }
      default:
        return HSZ_EINVAL;
    }
    return launch_status();
  }
  const gen::GStream s{widths, outliers, signs, payload, toff, n, k, nb};
  switch (out_kind) {
    case HSZ_OUT_F32:
      gen::decode_kernel<k32::SinkF32><<<static_cast<unsigned>(nt), gen::kThreads, 0, st>>>(
          s, k32::SinkF32{static_cast<float*>(out), d, d * 0x1p33 >= 3.4028234663852886e38}, err);
      break;
    case HSZ_OUT_F64:
      gen::decode_kernel<k32::SinkF64><<<static_cast<unsigned>(nt), gen::kThreads, 0, st>>>(
          s, k32::SinkF64{static_cast<double*>(out), d, d * 0x1p33 >= 1.7976931348623157e308}, err);
      break;
    case HSZ_OUT_BINS:
      gen::decode_kernel<k32::SinkBins><<<static_cast<unsigned>(nt), gen::kThreads, 0, st>>>(
          s, k32::SinkBins{static_cast<int64_t*>(out)}, err);
      break;
    default:
      return HSZ_EINVAL;
  }
  return launch_status();
}

int hsz_negate(const uint8_t* widths, const int32_t* oin, int32_t* oout, const uint8_t* sin,
               uint8_t* sout, const uint64_t* toff, uint64_t n, uint32_t k, uint32_t* err,
               void* stream) {
  if (!widths || !oin || !oout || !sin || !sout || !toff || !err || n == 0 || k == 0) return HSZ_EINVAL;
  const uint64_t nb = ceil_div(n, k);
  const uint64_t nt = ceil_div(nb, kTileBlocks);
  const uint64_t sign_bound = hsz_sign_bound(n, k);
  const bool aligned = ((reinterpret_cast<uintptr_t>(oin) | reinterpret_cast<uintptr_t>(oout) |
                         reinterpret_cast<uintptr_t>(sin) | reinterpret_cast<uintptr_t>(sout)) & 15u) == 0;
  if (k == 32 && aligned) {
    const uint64_t items = nb / 4 > sign_bound / 16 ? nb / 4 : sign_bound / 16;
    const unsigned g = static_cast<unsigned>(
        grid_for(items, ops::kStreamU, ops::kStreamThreads, stream_wave()));
    ops::negate32_kernel<<<g, ops::kStreamThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        widths, oin, oout, sin, sout, toff, nt, n, nb, sign_bound / 16, err);
    return launch_status();
  }
  const uint64_t items = (sign_bound / 16 > nb) ? sign_bound / 16 : nb;
  const unsigned g = static_cast<unsigned>(grid_for(items, 2, ops::kThreads, 148 * 16));
  ops::negate_kernel<<<g, ops::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      widths, oin, oout, sin, sout, toff, nt, n, k, nb, err);
  return launch_status();
}

int hsz_scalar_add(const int32_t* oin, int32_t* oout, uint64_t nblocks, int64_t rs, uint32_t* err,
                   void* stream) {
  if (!oin || !oout || !err || nblocks == 0) return HSZ_EINVAL;
  const unsigned g = static_cast<unsigned>(
      grid_for(nblocks, 4 * ops::kStreamU, ops::kStreamThreads, stream_wave()));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rs >= INT32_MIN && rs <= INT32_MAX)
    ops::sadd_kernel<true><<<g, ops::kStreamThreads, 0, st>>>(oin, oout, nblocks, rs, err);
  else
    ops::sadd_kernel<false><<<g, ops::kStreamThreads, 0, st>>>(oin, oout, nblocks, rs, err);
  return launch_status();
}

int hsz_scalar_mul(const uint8_t* widths, const int32_t* outliers, const uint8_t* signs,
                   const uint8_t* payload, const uint64_t* toff, uint64_t n, uint32_t k, double eps,
                   int64_t rs, uint8_t* ow, int32_t* oo, uint8_t* os, uint64_t sign_cap, uint8_t* op,
                   uint64_t payload_cap, uint64_t* otoff, void* scratch, uint32_t* err, void* ws,
                   uint64_t ws_bytes, void* stream) {
  if (!widths || !outliers || !signs || !payload || !toff || !ow || !oo || !os || !op || !otoff ||
      !err || !ws || n == 0 || k == 0)
    return HSZ_EINVAL;
  if (ws_bytes < hsz_workspace_size(n, k)) return HSZ_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t nb = ceil_div(n, k);
  const uint64_t nt = ceil_div(nb, kTileBlocks);
  const double d = 2.0 * eps;
  if (k == 32) {
    const d32::StreamIn in{widths, outliers, signs, payload, toff, n, nb, nt, tail_len_of(n, 32)};
    d32::SmulParams sp;
    sp.rs = rs;
    sp.d = d;
    sp.rsd = static_cast<double>(rs);
    sp.small_rs = (rs > -(1ll << 23) && rs < (1ll << 23)) ? 1 : 0;
    const k32::EncodeOut out{ow, oo, os, sign_cap, op, payload_cap, otoff, err, ws};
    return launch_recode<d32::kOpSmul>(in, in, sp, out, nt, st);
  }
  if (!scratch) return HSZ_EINVAL;
  int64_t* bins = static_cast<int64_t*>(scratch);
  const gen::GStream s{widths, outliers, signs, payload, toff, n, k, nb};
  gen::decode_kernel<gen::SinkSmul><<<static_cast<unsigned>(nt), gen::kThreads, 0, st>>>(
      s, gen::SinkSmul{bins, rs, d}, err);
  return launch_encode_generic(gen::GBins{bins}, n, k, ow, oo, os, sign_cap, op, payload_cap, otoff,
                               err, ws, st);
}

uint64_t hsz_elementwise_scratch_size(uint64_t n, uint32_t k) { return (k && k != 32) ? 8 * n : 0; }

int hsz_elementwise(const uint8_t* wa, const int32_t* oa, const uint8_t* sa, const uint8_t* pa,
                    const uint64_t* ta, const uint8_t* wb, const int32_t* ob, const uint8_t* sb,
                    const uint8_t* pb, const uint64_t* tb, uint64_t n, uint32_t k, int sub,
                    uint8_t* ow, int32_t* oo, uint8_t* os, uint64_t sign_cap, uint8_t* op,
                    uint64_t payload_cap, uint64_t* otoff, void* scratch, uint32_t* err, void* ws,
                    uint64_t ws_bytes, void* stream) {
  if (!wa || !oa || !sa || !pa || !ta || !wb || !ob || !sb || !pb || !tb || !ow || !oo || !os ||
      !op || !otoff || !err || !ws || n == 0 || k == 0)
    return HSZ_EINVAL;
  if (ws_bytes < hsz_workspace_size(n, k)) return HSZ_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t nb = ceil_div(n, k);
  const uint64_t nt = ceil_div(nb, kTileBlocks);
  if (k == 32) {
    // one fused pass: both operands' tiles staged, decoded into the same
    // registers, re-encoded and placed by look-back
    const uint32_t tl = tail_len_of(n, 32);
    const d32::StreamIn A{wa, oa, sa, pa, ta, n, nb, nt, tl};
    const d32::StreamIn B{wb, ob, sb, pb, tb, n, nb, nt, tl};
    const d32::SmulParams sp{0, 0.0, 0.0, 0};
    const k32::EncodeOut out{ow, oo, os, sign_cap, op, payload_cap, otoff, err, ws};
    return sub ? launch_recode<d32::kOpSub>(A, B, sp, out, nt, st)
               : launch_recode<d32::kOpAdd>(A, B, sp, out, nt, st);
  }
  if (!scratch) return HSZ_EINVAL;
  int64_t* bins = static_cast<int64_t*>(scratch);
  // bins(a) (+|-) bins(b) modulo 2^64, then one re-encode: outliers a0 (+|-) b0
  // under the int32 guard, residuals ra (+|-) rb
  const gen::GStream A{wa, oa, sa, pa, ta, n, k, nb};
  const gen::GStream B{wb, ob, sb, pb, tb, n, k, nb};
  gen::decode_kernel<k32::SinkBins><<<static_cast<unsigned>(nt), gen::kThreads, 0, st>>>(
      A, k32::SinkBins{bins}, err);
  gen::decode_kernel<ops::SinkCombineBins><<<static_cast<unsigned>(nt), gen::kThreads, 0, st>>>(
      B, ops::SinkCombineBins{bins, sub}, err);
  // (k == 32 returned above through the fused recode kernel)
  return launch_encode_generic(gen::GBins{bins}, n, k, ow, oo, os, sign_cap, op, payload_cap, otoff,
                               err, ws, st);
}

uint64_t hsz_bivariate_scratch_size(uint64_t n, uint32_t k) { return k ? 16 * n : 0; }

// decode both operands to int64 bins: a -> bins[0, n), b -> bins[n, 2n)
static int decode_pair_bins(const uint8_t* wa, const int32_t* oa, const uint8_t* sa,
                            const uint8_t* pa, const uint64_t* ta, const uint8_t* wb,
                            const int32_t* ob, const uint8_t* sb, const uint8_t* pb,
                            const uint64_t* tb, uint64_t n, uint32_t k, int64_t* bins,
                            uint32_t* err, void* stream) {
  int rc = hsz_decode(wa, oa, sa, pa, ta, n, k, 1.0, HSZ_OUT_BINS, bins, err, stream);
  if (rc != HSZ_OK) return rc;
  return hsz_decode(wb, ob, sb, pb, tb, n, k, 1.0, HSZ_OUT_BINS, bins + n, err, stream);
}

static unsigned bv_grid(uint64_t items) {
  const uint64_t g = ceil_div(items, bv::kThreads);
  return static_cast<unsigned>(g < 148 * 8 ? (g ? g : 1) : 148 * 8);
}

int hsz_hadamard(const uint8_t* wa, const int32_t* oa, const uint8_t* sa, const uint8_t* pa,
                 const uint64_t* ta, const uint8_t* wb, const int32_t* ob, const uint8_t* sb,
                 const uint8_t* pb, const uint64_t* tb, uint64_t n, uint32_t k, double eps,
                 uint8_t* ow, int32_t* oo, uint8_t* os, uint64_t sign_cap, uint8_t* op,
                 uint64_t payload_cap, uint64_t* otoff, void* scratch, uint32_t* err, void* ws,
                 uint64_t ws_bytes, void* stream) {
  if (!scratch || !err || !ws || n == 0 || k == 0) return HSZ_EINVAL;
  if (ws_bytes < hsz_workspace_size(n, k)) return HSZ_EINVAL;
  int64_t* bins = static_cast<int64_t*>(scratch);
  int rc = decode_pair_bins(wa, oa, sa, pa, ta, wb, ob, sb, pb, tb, n, k, bins, err, stream);
  if (rc != HSZ_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  bv::hadamard_kernel<<<bv_grid(n), bv::kThreads, 0, st>>>(bins, bins + n, n, 2.0 * eps, err);
  rc = launch_status();
  if (rc != HSZ_OK) return rc;
  return hsz_encode_bins(bins, n, k, ow, oo, os, sign_cap, op, payload_cap, otoff, err, ws,
                         ws_bytes, stream);
}

int hsz_pair_stats(const uint8_t* wa, const int32_t* oa, const uint8_t* sa, const uint8_t* pa,
                   const uint64_t* ta, const uint8_t* wb, const int32_t* ob, const uint8_t* sb,
                   const uint8_t* pb, const uint64_t* tb, uint64_t n, uint32_t k, uint64_t* out,
                   void* scratch, uint32_t* err, void* stream) {
  if (!out || !scratch || !err || n == 0 || k == 0) return HSZ_EINVAL;
  if (n >= (1ull << 32)) return HSZ_EINVAL;   // carry-save counter headroom
  int64_t* bins = static_cast<int64_t*>(scratch);
  int rc = decode_pair_bins(wa, oa, sa, pa, ta, wb, ob, sb, pb, tb, n, k, bins, err, stream);
  if (rc != HSZ_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  bv::pair_stats_init<<<1, 64, 0, st>>>(out);
  bv::pair_stats_kernel<<<bv_grid(n), bv::kThreads, 0, st>>>(bins, bins + n, n, out);
  return launch_status();
}

int hsz_block_means(const uint8_t* widths, const int32_t* outliers, const uint8_t* signs,
                    const uint8_t* payload, const uint64_t* toff, uint64_t n, uint32_t k,
                    double eps, double* out, void* scratch, uint32_t* err, void* stream) {
  if (!out || !scratch || !err || n == 0 || k == 0) return HSZ_EINVAL;
  int64_t* bins = static_cast<int64_t*>(scratch);
  int rc = hsz_decode(widths, outliers, signs, payload, toff, n, k, 1.0, HSZ_OUT_BINS, bins, err, stream);
  if (rc != HSZ_OK) return rc;
  const uint64_t nb = ceil_div(n, k);
  bv::block_means_kernel<<<bv_grid(nb), bv::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      bins, widths, outliers, n, k, nb, 2.0 * eps, out);
  return launch_status();
}

int hsz_moments_mb(const uint8_t* widths, const int32_t* outliers, const uint8_t* signs,
                   const uint8_t* payload, const uint64_t* toff, uint64_t n, uint32_t k, int want_sq,
                   uint64_t* out, uint32_t* err, void* ws, uint64_t ws_bytes, uint64_t* mailbox,
                   uint64_t seq, void* stream) {
  if (!widths || !outliers || !signs || !payload || !toff || !out || !err || !ws || n == 0 || k == 0)
    return HSZ_EINVAL;
  if (ws_bytes < hsz_workspace_size(n, k)) return HSZ_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t nb = ceil_div(n, k);
  const uint64_t nt = ceil_div(nb, kTileBlocks);
  if (k == 32) {
    const d32::StreamIn in{widths, outliers, signs, payload, toff, n, nb, nt, tail_len_of(n, 32)};
    const Mailbox mb{mailbox, seq};
    if (want_sq) return launch_decode_pipe<1>(in, nullptr, 0.0, out, ws, err, st, mb);
    return launch_decode_pipe<0>(in, nullptr, 0.0, out, ws, err, st, mb);
  }
  const gen::GStream s{widths, outliers, signs, payload, toff, n, k, nb};
  ops::gen_moments_kernel<<<static_cast<unsigned>(nt), gen::kThreads, 0, st>>>(s, want_sq, out, err, ws);
  if (mailbox) ops::mailbox_post_kernel<<<1, 1, 0, st>>>(Mailbox{mailbox, seq}, out, 5, err);
  return launch_status();
}

int hsz_moments(const uint8_t* widths, const int32_t* outliers, const uint8_t* signs,
                const uint8_t* payload, const uint64_t* toff, uint64_t n, uint32_t k, int want_sq,
                uint64_t* out, uint32_t* err, void* ws, uint64_t ws_bytes, void* stream) {
  return hsz_moments_mb(widths, outliers, signs, payload, toff, n, k, want_sq, out, err, ws, ws_bytes,
                        nullptr, 0, stream);
}

int hsz_mailbox_wait(const uint64_t* mailbox, uint64_t seq, void* stream) {
  // poll the host word the kernel posts; every 4096 polls ask whether the
  // stream died (error) or drained without posting (caller falls back)
  const volatile uint64_t* w = mailbox;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double t0 = -1.0;
  for (uint64_t it = 1;; ++it) {
    if (*w == seq) {
      __atomic_thread_fence(__ATOMIC_ACQUIRE);
      return HSZ_OK;
    }
    if ((it & 4095u) == 0) {
      const double now = wall_s();
      if (t0 < 0) t0 = now;
      else if (now - t0 > g_host_wait_s) return HSZ_ETIMEDOUT;
      const cudaError_t e = cudaStreamQuery(st);
      if (e == cudaSuccess) {
        if (*w == seq) {
          __atomic_thread_fence(__ATOMIC_ACQUIRE);
          return HSZ_OK;
        }
        return HSZ_EINVAL;   // drained without a post: fall back to a copy
      }
      if (e != cudaErrorNotReady) return HSZ_ECUDA;
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
}

// ---------------------------------------------------------------------------
// node-local host all-gather of a few int64 words per rank through a shared
// memory segment every rank maps (one process per GPU on one node).  The C1
// value range, C2 section sizes and C3 moment limbs are host scalars already
// (they come back through the mailbox); exchanging them here costs a few
// microseconds instead of an NCCL round trip plus two host<->device copies.
// Slot r (kHcSlot bytes): [0] seq (release-stored), two value buffers of
// kHcMaxVals words at +64 and +64 + 8 * kHcMaxVals selected by round parity
// -- a rank can only reach round + 2 (and
// overwrite this round's buffer) after every rank published round + 1, i.e.
// finished reading round.
namespace {
constexpr int kHcMaxVals = 40;
constexpr uint64_t kHcSlot = 64 + 2 * 8 * kHcMaxVals;   // 704: a multiple of 64
inline double hc_now() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}
}  // namespace

uint64_t hsz_hostcoll_bytes(int world) { return world > 0 ? kHcSlot * world : 0; }

int hsz_hostcoll_allgather(void* shm, int rank, int world, uint64_t round, const int64_t* vals,
                           int nvals, int64_t* out, double timeout_s) {
  if (!shm || world <= 0 || rank < 0 || rank >= world || round == 0 || nvals < 0 ||
      nvals > kHcMaxVals || (nvals && (!vals || !out)))
    return HSZ_EINVAL;
  unsigned char* base = static_cast<unsigned char*>(shm);
  const uint64_t buf_off = 64 + 8 * kHcMaxVals * (round & 1u);
  unsigned char* mine = base + kHcSlot * rank;
  std::memcpy(mine + buf_off, vals, sizeof(int64_t) * nvals);
  __atomic_store_n(reinterpret_cast<uint64_t*>(mine), round, __ATOMIC_RELEASE);
  const double t0 = timeout_s > 0 ? hc_now() : 0.0;
  for (int r = 0; r < world; ++r) {
    const unsigned char* slot = base + kHcSlot * r;
    const uint64_t* seq = reinterpret_cast<const uint64_t*>(slot);
    for (uint64_t it = 1; __atomic_load_n(seq, __ATOMIC_ACQUIRE) < round; ++it) {
      if (timeout_s > 0 && (it & 4095u) == 0 && hc_now() - t0 > timeout_s) return HSZ_ECUDA;
#if defined(__x86_64__)
      __builtin_ia32_pause();
#endif
    }
    std::memcpy(out + static_cast<size_t>(r) * nvals, slot + buf_off, sizeof(int64_t) * nvals);
  }
  return HSZ_OK;
}

}  // extern "C"
