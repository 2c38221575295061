// Shared device helpers for the HoSZp B200 hot path (sm_100a).
//
// * error word bits (HSZ_ERR_*, same values as include/hsz_b200.h)
// * big-endian / bit-reversal helpers for the MSB-first sign planes and
//   element-major payload fields of pkg/FORMAT.md:24-37
// * TMA bulk copy (cp.async.bulk) + mbarrier wrappers
// * the single-pass decoupled look-back used to place variable-length
//   blocks (sign planes, payload) at their global byte offsets
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "../../include/hsz_b200.h"

namespace hsz {

// Optional phase tracing (compile with -DHSZ_TRACE): thread 0 of each CTA
// appends (tag, globaltimer) records; read with hsz_trace_read().
#ifdef HSZ_TRACE
constexpr int kTraceCap = 1 << 20;
__device__ unsigned long long g_trace[kTraceCap];
__device__ unsigned int g_trace_n;
__device__ __forceinline__ void trace(uint32_t tag) {
  if (threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned i = atomicAdd(&g_trace_n, 1u);
    if (i < kTraceCap) g_trace[i] = (static_cast<unsigned long long>(blockIdx.x) << 48) |
                                    (static_cast<unsigned long long>(tag) << 40) | (t & ((1ull << 40) - 1));
  }
}
// per-tile record: (tile << 40) | (tag << 32) | low 32 bits of globaltimer (ns)
__device__ __forceinline__ void trace_tile(uint64_t tile, uint32_t tag) {
  if (threadIdx.x == 0 || threadIdx.x == 128) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned i = atomicAdd(&g_trace_n, 1u);
    if (i < kTraceCap) g_trace[i] = (tile << 40) | (static_cast<unsigned long long>(tag) << 32) | (t & 0xffffffffull);
  }
}
#else
__device__ __forceinline__ void trace(uint32_t) {}
__device__ __forceinline__ void trace_tile(uint64_t, uint32_t) {}
#endif

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// Tile geometry shared by every kernel and by the tile-offset cache of a
// device stream: a tile is kTileBlocks consecutive blocks.
constexpr int kTileBlocks = HSZ_TILE_BLOCKS;   // 128
constexpr int kCtaWarps = 4;                    // 128-thread CTAs (one thread per block of a tile)
constexpr int kBlocksPerWarp = kTileBlocks / kCtaWarps;  // 32

static_assert(kTileBlocks % kCtaWarps == 0, "tile must split evenly over warps");

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

// 0xFFFFFFFF if the top bit of byte b of x is set, else 0 (PRMT sign mode)
__device__ __forceinline__ uint32_t prmt_sign(uint32_t x, int b) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(x), "r"((8 + b) * 0x1111));
  return r;
}

__device__ __forceinline__ void set_err(uint32_t* err, uint32_t bits) {
  if (bits) atomicOr(err, bits);
}

// ---------------------------------------------------------------------------
// shared-memory addresses, mbarrier and bulk async copy (TMA engine)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

#ifndef HSZ_CMP_SLEEP_MAX
#define HSZ_CMP_SLEEP_MAX 0
#endif
__device__ __forceinline__ bool mbar_test_parity(uint64_t* bar, uint32_t parity);
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
#if HSZ_CMP_SLEEP_MAX > 0
  if (mbar_test_parity(bar, parity)) return;
  unsigned ns = 16;
  while (!mbar_test_parity(bar, parity)) {
    __nanosleep(ns);
    ns = ns < HSZ_CMP_SLEEP_MAX ? 2 * ns : HSZ_CMP_SLEEP_MAX;
  }
  return;
#endif
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// non-blocking probe of a phase
__device__ __forceinline__ bool mbar_test_parity(uint64_t* bar, uint32_t parity) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(r)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return r != 0;
}

// service-warp wait (TMA issue, placement): poll with an exponential
// nanosleep back-off.  A parked try_wait is woken by every mbarrier event of
// the SM, so a waiting producer would otherwise spin through hundreds of
// wake-ups per tile and steal issue slots from the compute warps.
#ifndef HSZ_SVC_SLEEP_MAX
#define HSZ_SVC_SLEEP_MAX 0
#endif
__device__ __forceinline__ void mbar_wait_parity_sleep(uint64_t* bar, uint32_t parity) {
#if HSZ_SVC_SLEEP_MAX > 0
  if (mbar_test_parity(bar, parity)) return;
  unsigned ns = 32;
  while (!mbar_test_parity(bar, parity)) {
    __nanosleep(ns);
    ns = ns < HSZ_SVC_SLEEP_MAX ? 2 * ns : HSZ_SVC_SLEEP_MAX;
  }
#else
  mbar_wait_parity(bar, parity);
#endif
}

// global -> shared bulk copy; dst/src 16-byte aligned, bytes % 16 == 0
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// named barrier 1 over the 128 compute threads (warps 0-3) of a CTA that may
// also contain a specialised store warp; equivalent to __syncthreads() in
// 128-thread CTAs
__device__ __forceinline__ void grp_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ bool grp_and(bool p) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred q, o;\n\tsetp.ne.u32 q, %1, 0;\n\t"
      "bar.red.and.pred o, 1, 128, q;\n\tselp.u32 %0, 1, 0, o;\n}"
      : "=r"(r)
      : "r"(static_cast<uint32_t>(p))
      : "memory");
  return r != 0;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// one arrival per warp (barriers initialised with the number of warps): the
// warp's prior shared-memory writes are ordered before lane 0's arrive
__device__ __forceinline__ void mbar_arrive_warp(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}

// ---------------------------------------------------------------------------
// gpu-scope acquire / release accesses for the look-back protocol

__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t atom_add_relaxed(uint64_t* p, uint64_t v) {
  uint64_t old;
  asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ uint64_t atom_add_acq_rel(uint64_t* p, uint64_t v) {
  uint64_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v)
               : "memory");
  return old;
}

// Workspace layout (u64 words; see hsz_workspace_size):
//   [0]      ticket          [1] epoch       [2] moments done-counter
//   [3]      minmax done-counter             [8..18) moments carry-save counters
//   [64 .. 64 + 2*kMinmaxCtasMax)            minmax per-CTA partials
//   flags[ntiles]   at kWsFlagsOff            (epoch << 2 | state)
//   vals[ntiles][6] right after the flags     (agg_sign, agg_pay, inc_sign,
//                                              inc_pay | moments partials)
constexpr uint64_t kMinmaxCtasMax = 148 * 4;
constexpr uint64_t kWsMinmaxOff = 64;
constexpr uint64_t kWsFlagsOff = kWsMinmaxOff + 2 * kMinmaxCtasMax;

// Host-mapped mailbox of a reduction (pinned host memory, UVA): the
// kernel's last CTA writes the result words and a snapshot of the error word
// straight into host memory, then (after a system-scope fence) the sequence
// number in word 0 -- the host polls word 0 instead of a D2H copy + stream
// synchronisation.  Layout (u64): [0] seq, [1..] results, [1 + nres] error word.
struct Mailbox {
  uint64_t* host;   // nullptr: no mailbox
  uint64_t seq;
};

__device__ __forceinline__ void mailbox_post(const Mailbox& mb, const uint64_t* res, int nres,
                                             const uint32_t* err) {
  if (!mb.host) return;
  for (int i = 0; i < nres; ++i) mb.host[1 + i] = res[i];
  mb.host[1 + nres] = *reinterpret_cast<const volatile uint32_t*>(err);
  __threadfence_system();
  *reinterpret_cast<volatile uint64_t*>(mb.host) = mb.seq;
}

struct LookbackWs {
  uint64_t* ticket;
  uint64_t* epoch;
  uint64_t* flags;
  uint64_t* vals;
  __device__ static LookbackWs bind(void* ws, uint64_t ntiles) {
    LookbackWs w;
    uint64_t* base = static_cast<uint64_t*>(ws);
    w.ticket = base;
    w.epoch = base + 1;
    w.flags = base + kWsFlagsOff;
    w.vals = base + kWsFlagsOff + ntiles;
    return w;
  }
};

constexpr uint64_t kStAgg = 1, kStInc = 2;

// Look-back watchdog: a warp that has backed off this many times waiting for
// a predecessor tile gives up, sets HSZ_ERR_LOOKBACK_TIMEOUT and publishes
// what it has (the offsets of that tile and its successors are then wrong,
// and flagged), so a protocol failure -- e.g. a workspace left inconsistent
// by an aborted launch -- raises on the host instead of hanging the GPU.
// Each back-off is >= 16-128 ns plus an L2 round trip: the default bound is
// several seconds, far above any legitimate wait (tickets are drawn in
// order, so every awaited predecessor is resident and progressing).
// Settable through hsz_set_lookback_watchdog().
__device__ unsigned int g_lb_max_sleeps = 1u << 23;

// Called by thread 0: draw the launch epoch and a tile ticket (tickets are
// handed out in order, so every predecessor of a tile is resident or done,
// which makes the spin in lookback() deadlock-free).  The CTA drawing the
// last ticket rearms the counter and advances the epoch for the next launch.
__device__ __forceinline__ void draw_ticket(LookbackWs& w, uint64_t ntiles, uint64_t* tile,
                                            uint64_t* epoch) {
  uint64_t e = ld_acquire(w.epoch);
  uint64_t t = atom_add_acq_rel(w.ticket, 1);
  if (t == ntiles - 1) {
    st_relaxed(w.ticket, 0);
    st_release(w.epoch, e + 1);
  }
  *tile = t;
  *epoch = e;
}

// Decoupled look-back over (sign bytes, payload bytes), in two steps so the
// CTA can do useful work in between:
//   publish_aggregate -- lane 0 publishes the tile's aggregate (tile 0: its
//                        inclusive prefix) as soon as the tile sizes are known;
//   resolve_prefix    -- one full warp sums predecessors (32 at a time) until
//                        an inclusive prefix is found, publishes this tile's
//                        inclusive prefix and returns the exclusive one.
__device__ __forceinline__ void publish_aggregate(LookbackWs& w, uint64_t tile, uint64_t epoch,
                                                  uint64_t agg_s, uint64_t agg_p) {
  const uint64_t tag = epoch << 2;
  if (tile == 0) {
    w.vals[2] = agg_s;   // inclusive slots of tile 0
    w.vals[3] = agg_p;
    st_release(&w.flags[0], tag | kStInc);
  } else {
    w.vals[tile * 4 + 0] = agg_s;
    w.vals[tile * 4 + 1] = agg_p;
    st_release(&w.flags[tile], tag | kStAgg);
  }
}

__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Each lane inspects kLbPerLane consecutive predecessors, so one round trip
// covers 32 * kLbPerLane tiles: with hundreds of tiles in flight, the nearest
// published inclusive prefix is usually found in one or two rounds.
#ifndef HSZ_LB_PER_LANE
#define HSZ_LB_PER_LANE 1
#endif
constexpr int kLbPerLane = HSZ_LB_PER_LANE;

__device__ __forceinline__ void resolve_prefix(LookbackWs& w, uint64_t tile, uint64_t epoch,
                                               uint64_t agg_s, uint64_t agg_p, uint64_t* excl_s,
                                               uint64_t* excl_p, uint32_t* err) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    *excl_s = 0;
    *excl_p = 0;
    return;
  }
  uint64_t sum_s = 0, sum_p = 0;
  int64_t base = static_cast<int64_t>(tile) - 1;
  unsigned backoff = 32;
  const unsigned max_sleeps = g_lb_max_sleeps;
  unsigned sleeps = 0;
  while (true) {
    // relaxed flag loads (all in flight together), then one acquire fence
    uint32_t stj[kLbPerLane];
#pragma unroll
    for (int j = 0; j < kLbPerLane; ++j) {
      const int64_t idx = base - (lane * kLbPerLane + j);
      uint32_t st = kStInc;       // virtual inclusive zero before tile 0
      if (idx >= 0) {
        const uint64_t f = ld_relaxed(&w.flags[idx]);
        st = ((f >> 2) == epoch) ? static_cast<uint32_t>(f & 3) : 0u;
      }
      stj[j] = st;
    }
    fence_acq_rel_gpu();
    int fj = kLbPerLane;                 // first inclusive in my run
    bool inv_all = false, inv_pre = false;
#pragma unroll
    for (int j = kLbPerLane - 1; j >= 0; --j) {
      if (stj[j] == kStInc) fj = j;
      inv_all |= stj[j] == 0;
    }
#pragma unroll
    for (int j = 0; j < kLbPerLane; ++j) inv_pre |= (j <= fj) && (stj[j] == 0);
    const unsigned inc = __ballot_sync(kFull, fj < kLbPerLane);
    const int first = inc ? (__ffs(inc) - 1) : 32;
    const bool bad = (lane < first && inv_all) || (lane == first && inv_pre);
    if (__any_sync(kFull, bad)) {        // a needed predecessor has not published yet
      if (++sleeps > max_sleeps) {       // watchdog (warp-uniform)
        if (lane == 0) atomicOr(err, HSZ_ERR_LOOKBACK_TIMEOUT);
        break;
      }
      __nanosleep(backoff);
      backoff = backoff < 256 ? backoff * 2 : 256;
      continue;
    }
    uint64_t vs = 0, vp = 0;
    if (lane <= first) {
      const int stop = (lane < first) ? kLbPerLane : fj;
#pragma unroll
      for (int j = 0; j < kLbPerLane; ++j) {
        const int64_t idx = base - (lane * kLbPerLane + j);
        if (idx >= 0 && j <= stop && j < kLbPerLane) {
          if (j < stop) {
            vs += ld_relaxed(&w.vals[idx * 4 + 0]);
            vp += ld_relaxed(&w.vals[idx * 4 + 1]);
          } else {
            vs += ld_relaxed(&w.vals[idx * 4 + 2]);
            vp += ld_relaxed(&w.vals[idx * 4 + 3]);
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      vs += __shfl_xor_sync(kFull, vs, o);
      vp += __shfl_xor_sync(kFull, vp, o);
    }
    sum_s += vs;
    sum_p += vp;
    if (first < 32) break;
    base -= 32 * kLbPerLane;
  }
  if (lane == 0) {
    w.vals[tile * 4 + 2] = sum_s + agg_s;
    w.vals[tile * 4 + 3] = sum_p + agg_p;
    st_release(&w.flags[tile], (epoch << 2) | kStInc);
  }
  *excl_s = sum_s;
  *excl_p = sum_p;
}

// both steps back to back (callers with nothing to overlap)
__device__ __forceinline__ void lookback(LookbackWs& w, uint64_t tile, uint64_t epoch,
                                         uint64_t agg_s, uint64_t agg_p, uint64_t* excl_s,
                                         uint64_t* excl_p, uint32_t* err) {
  if ((threadIdx.x & 31) == 0) publish_aggregate(w, tile, epoch, agg_s, agg_p);
  __syncwarp();
  resolve_prefix(w, tile, epoch, agg_s, agg_p, excl_s, excl_p, err);
}

// ---------------------------------------------------------------------------
// Fence-free decoupled look-back (register-resident encoders).
//
// One 16-byte record per tile in the workspace, {sign, payload}, written with
// a single 16-byte store; each 8-byte half is self-validating:
//   bit 63 = 1, bit 62 = inclusive (else aggregate), bits 61..39 = the low 23
//   bits of the launch epoch, bits 38..0 = the value.
// A reader accepts a record only if both halves carry the current epoch and
// the same state, so it needs no acquire fence between a flag and its value.
// (Words of the flag/value protocol above never have bit 63 set.  The epoch
// tag repeats after 2^23 launches on one workspace: the host re-initialises
// the workspace before that, see hsz_workspace_init.)
constexpr int kLbValBits = 39;
constexpr uint64_t kLbValMask = (1ull << kLbValBits) - 1;
constexpr int kLbStride = 2;   // u64 words per tile record

__device__ __forceinline__ uint64_t lb_tag(uint64_t epoch) {   // bits 63..39 of an aggregate
  return (1ull << 24) | (epoch & 0x7FFFFFull);
}
constexpr uint64_t kLbIncBit = 1ull << 23;                      // in the tag: inclusive

__device__ __forceinline__ void st_relaxed_v2(uint64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_relaxed_v2(const uint64_t* p, uint64_t* a, uint64_t* b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(*a), "=l"(*b) : "l"(p) : "memory");
}

__device__ __forceinline__ uint64_t* lb_words(void* ws) {
  return static_cast<uint64_t*>(ws) + kWsFlagsOff;
}

// one thread: the tile's aggregate (tile 0: its inclusive prefix)
__device__ __forceinline__ void lb_publish(uint64_t* words, uint64_t tile, uint64_t epoch,
                                           uint64_t agg_s, uint64_t agg_p) {
  const uint64_t t = (lb_tag(epoch) | (tile == 0 ? kLbIncBit : 0)) << kLbValBits;
  st_relaxed_v2(words + kLbStride * tile, t | agg_s, t | agg_p);
}

#ifndef HSZ_LB2_PER_LANE
#define HSZ_LB2_PER_LANE 1
#endif

#ifdef HSZ_TRACE
__device__ unsigned int g_lb_rounds, g_lb_sleeps, g_lb_calls;
__device__ unsigned long long g_lb_cycles_round, g_lb_cycles_total;
#endif

// one full warp: exclusive prefix of `tile` (its aggregate already published);
// publishes the tile's inclusive prefix.
//
// Each round lane i reads the record of tile base - i (one L2 round trip for
// the warp) and the warp accepts the records from the nearest one up to the
// first inclusive prefix -- or up to the first record that is not published
// yet, in which case the next round resumes AT that record (no re-read of
// what was accepted, the window slides 32 tiles further back behind it).
// Accepted values stay in per-lane partial sums; the one cross-lane
// reduction happens at the end.  (The placement warp of a CTA spends most of
// a tile period here, competing for issue slots with the compute warps: the
// round is ~30 instructions instead of the ~100 of the reduce-every-round
// form, which measured 3.8 us per resolve on config 4.)
#if HSZ_LB2_PER_LANE != 1
#error "lb_resolve reads one record per lane"
#endif
__device__ __forceinline__ void lb_resolve(uint64_t* words, uint64_t tile, uint64_t epoch,
                                           uint64_t agg_s, uint64_t agg_p, uint64_t* excl_s,
                                           uint64_t* excl_p, uint32_t* err) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    *excl_s = 0;
    *excl_p = 0;
    return;
  }
  const uint64_t tag = lb_tag(epoch);
  uint64_t acc_s = 0, acc_p = 0;   // this lane's accepted records
  int64_t base = static_cast<int64_t>(tile) - 1;
  unsigned backoff = 16;
  const unsigned max_sleeps = g_lb_max_sleeps;
  unsigned nsleep = 0;
#ifdef HSZ_TRACE
  unsigned rounds = 0, sleeps = 0;
  const long long c_start = clock64();
  long long c_round = 0;
#endif
  while (true) {
#ifdef HSZ_TRACE
    ++rounds;
    const long long c0 = clock64();
#endif
    const int64_t idx = base - lane;
    const bool real = idx >= 0;      // else: the virtual inclusive 0 before tile 0
    uint64_t ra, rb;
    ld_relaxed_v2(words + kLbStride * (real ? idx : 0), &ra, &rb);
    const uint64_t ta = ra >> kLbValBits, tb = rb >> kLbValBits;
    const bool ok = !real || ((ta == tb) & ((ta & ~kLbIncBit) == tag));
    const bool inc = !real || (ta & kLbIncBit) != 0;
    const unsigned fm = __ballot_sync(kFull, ok & inc);   // inclusive prefixes
    const unsigned vm = __ballot_sync(kFull, !ok);        // not published yet
#ifdef HSZ_TRACE
    c_round += clock64() - c0;
#endif
    const int first = fm ? (__ffs(fm) - 1) : 32;          // nearest inclusive prefix
    const int hole = vm ? (__ffs(vm) - 1) : 32;           // nearest unpublished record
    const int take = hole < first ? hole : first + 1;     // lanes [0, take) are accepted
    if (lane < take && real) {
      acc_s += ra & kLbValMask;
      acc_p += rb & kLbValMask;
    }
    if (hole > first) break;        // reached an inclusive prefix with no hole before it
    if (hole == 32) {               // 32 aggregates, no inclusive prefix yet: further back
      base -= 32;
      continue;
    }
    base -= hole;                   // resume at the unpublished record
    if (hole == 0) {                // no progress this round: back off
      if (++nsleep > max_sleeps) {  // watchdog (warp-uniform): give up, flagged
        if (lane == 0) atomicOr(err, HSZ_ERR_LOOKBACK_TIMEOUT);
        break;
      }
      __nanosleep(backoff);
      backoff = backoff < 128 ? backoff * 2 : 128;
#ifdef HSZ_TRACE
      ++sleeps;
#endif
    } else {
      backoff = 16;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc_s += __shfl_xor_sync(kFull, acc_s, o);
    acc_p += __shfl_xor_sync(kFull, acc_p, o);
  }
  if (lane == 0) {
    const uint64_t t = (tag | kLbIncBit) << kLbValBits;
    st_relaxed_v2(words + kLbStride * tile, t | (acc_s + agg_s), t | (acc_p + agg_p));
#ifdef HSZ_TRACE
    atomicAdd(&g_lb_rounds, rounds);
    atomicAdd(&g_lb_sleeps, sleeps);
    atomicAdd(&g_lb_calls, 1u);
    atomicAdd(&g_lb_cycles_round, static_cast<unsigned long long>(c_round));
    atomicAdd(&g_lb_cycles_total, static_cast<unsigned long long>(clock64() - c_start));
#endif
  }
  *excl_s = acc_s;
  *excl_p = acc_p;
}

// ---------------------------------------------------------------------------
// exact integer helpers

// 64-bit signed difference a - b as (magnitude, negative) -- exact for any
// pair with |a|,|b| <= 2^63 - 1 (magnitude < 2^64).
__device__ __forceinline__ uint64_t absdiff64(int64_t a, int64_t b, bool* neg) {
  *neg = a < b;
  return a >= b ? static_cast<uint64_t>(a) - static_cast<uint64_t>(b)
                : static_cast<uint64_t>(b) - static_cast<uint64_t>(a);
}

// Round-to-nearest-even conversion of a signed 128-bit integer to double
// (what numpy / CPython do for the exact product p = bin * rs).
__device__ __forceinline__ double i128_to_double_rn(__int128 v) {
  const bool neg = v < 0;
  unsigned __int128 m = neg ? (unsigned __int128)(-(v + 1)) + 1u : (unsigned __int128)v;
  const uint64_t hi = static_cast<uint64_t>(m >> 64);
  double r;
  if (hi == 0) {
    r = __ull2double_rn(static_cast<uint64_t>(m));
  } else {
    const int lz = __clzll(hi);            // 0..63
    const int sh = 64 - lz;                // bits to drop so the value fits 64 bits
    const uint64_t top = static_cast<uint64_t>(m >> sh);
    const bool sticky = (m & ((((unsigned __int128)1) << sh) - 1u)) != 0;
    // the sticky bit sits far below the rounding position of a 53-bit
    // mantissa, so RN of (top | sticky) equals RN of the full value
    r = ldexp(__ull2double_rn(top | (sticky ? 1u : 0u)), sh);
  }
  return neg ? -r : r;
}

}  // namespace hsz
