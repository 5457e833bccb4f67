// bx_launch.cuh -- host-side launch geometry and the per-Q launcher template.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <cuda_runtime.h>

#include "bx_core.cuh"

namespace bx {

struct LaunchCfg {
  int tpb_log2 = 0;
  int tile = 0;       // blocks per CTA
  int staged = 1;
  int threads = 256;
  int stage_words = 0;
  int stages = 2;     // TMA kernel input stages
  int tile0 = 0;      // TMA: the tile choose_launch planned (before the stage budget)
  size_t smem = 0;
  int64_t grid = 0;
  int family = 0;     // 0 diag, 1 holes
  int direct = 0;     // 1: eq_direct_kernel (aligned fast path)
  int tma = 0;        // 1: eq_tma_kernel (persistent, cp.async.bulk double buffer)
  int units = 0;      // direct: 128-bit units per block
};

inline bool period_enabled() {
  static const bool on = [] {
    const char* e = getenv("BX_PERIOD");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// q with an aligned one-thread-per-block kernel: powers of two
// (eq_direct_kernel) and q = 24, 40, 48, 56 (eq_period_kernel; BX_PERIOD=0
// sends those to the TMA kernel, for A/B runs)
inline bool direct_q(int q) {
  return q == 1 || q == 2 || q == 4 || q == 8 || q == 16 || q == 32 || q == 64 || q == 128 ||
         (period_q(q) && period_enabled());
}

// Aligned fast path eligibility (see eq_direct_kernel).
inline bool direct_ok(int q, int n, int64_t x_bit0, int64_t y_bit0, int64_t out_bit0,
                      const void* x, const void* y) {
  const int64_t B = (int64_t)q * n;
  return direct_q(q) && B % 128 == 0 && x_bit0 % 128 == 0 && y_bit0 % 128 == 0 &&
         out_bit0 % 32 == 0 && (((uintptr_t)x | (uintptr_t)y) & 15) == 0;
}

// 256-bit loads in the q = 32 direct kernel (BX_WIDE32=0/1 for A/B runs)
#ifndef BX_WIDE32_DEFAULT
#define BX_WIDE32_DEFAULT 0
#endif
inline bool wide32_enabled() {
  static const int v = [] {
    const char* e = getenv("BX_WIDE32");
    return e ? atoi(e) : BX_WIDE32_DEFAULT;
  }();
  return v != 0;
}

// 256-bit loads in the q = 16 and q = 128 direct kernels (BX_WIDE=0 disables, for A/B runs).
inline bool wide_loads_enabled() {
  static const bool on = [] {
    const char* e = getenv("BX_WIDE");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

constexpr size_t kStageBudget = 96 * 1024;    // preferred smem per CTA
constexpr size_t kStageMax = 200 * 1024;      // hard cap before going direct

inline LaunchCfg choose_launch(int q, int n, int64_t nblocks) {
  LaunchCfg c;
  c.family = q <= kDiagMaxQ ? 0 : 1;
  const int64_t B = (int64_t)q * n;
  int64_t units, target;
  // elements (word chunks for the diag family) a thread should own before a
  // block is split over another thread: BX_TPB_TARGET overrides (A/B runs)
  static const int env_target = [] {
    const char* e = getenv("BX_TPB_TARGET");
    return e ? atoi(e) : 0;
  }();
  if (c.family == 0) {
    units = cdiv(n, 32 / q);
    target = 8;
  } else {
    units = n;
    // amortise the per-thread Karatsuba recombination; the dot form accumulates
    // four elements per step and recombines twice the accumulators, so it
    // wants 16 (c4p 2.20 -> 2.05 ms, q=37 n=50 -13%, q=20 n=60 -16%; the IMAD
    // form at q = 80 is 2% slower with 16 -- profiles/r02/dp2a_sweep.txt, sweep 10)
    target = (BX_DP2A_TILE != 0 && cdiv(q, 16) <= BX_DOT_TILE_MAX_HALVES) ? 16 : 8;
  }
  if (env_target > 0) target = env_target;
  int tpb = 1;
  while (tpb < 32 && units / (2 * tpb) >= target) tpb *= 2;
  c.tpb_log2 = 0;
  while ((1 << c.tpb_log2) < tpb) c.tpb_log2++;
  int T = 256 / tpb;
  auto stage_words = [&](int t) { return (int)(((31 + (int64_t)t * B + 31) >> 5) + 2); };
  auto out_words = [&](int t) { return (int)(((31 + (int64_t)t * q + 31) >> 5) + 2); };
  auto bytes = [&](int t) { return (size_t)(2 * (int64_t)stage_words(t) + out_words(t)) * 4; };
  const int Tmin = 32 / tpb > 0 ? 32 / tpb : 1;
  while (bytes(T) > kStageBudget && T > Tmin) T /= 2;
  c.tile = T;
  c.threads = T * tpb;
  if (bytes(T) <= kStageMax) {
    c.staged = 1;
    c.stage_words = stage_words(T);
    c.smem = bytes(T);
  } else {
    c.staged = 0;
    c.stage_words = 0;
    c.smem = (size_t)out_words(T) * 4;
  }
  c.grid = (nblocks + T - 1) / T;
  return c;
}

inline int sm_count();

inline LaunchCfg choose_direct(int q, int n, int64_t nblocks) {
  LaunchCfg c;
  c.family = q <= kDiagMaxQ ? 0 : 1;
  c.direct = 1;
  c.tpb_log2 = 0;
  // small runs: narrower CTAs so the blocks spread over more SMs
  int threads = period_q(q) ? BX_PERIOD_THREADS : direct_threads(q);
  while (threads > 64 && (nblocks + threads - 1) / threads < 2 * (int64_t)sm_count()) threads /= 2;
  c.tile = threads;
  c.threads = threads;
  c.staged = 0;
  c.smem = 0;
  c.units = (int)((int64_t)q * n / 128);
  const int bpt = direct_bpt(q, c.units);
  c.grid = (nblocks + (int64_t)threads * bpt - 1) / ((int64_t)threads * bpt);
  return c;
}

// Persistent TMA-bulk variant of a staged configuration: two stages of both
// windows (16-byte padded) plus two output tiles; grid = resident CTAs.
inline int sm_count() {
  // per device (the library may drive several GPUs from one process)
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v;
  }
  return cache[dev];
}

// Shared memory per TMA CTA: two stages of both windows; kept small enough for
// three resident CTAs per SM (228 KB) so tile loads of one CTA overlap the
// integer work of the others.
// Shared-memory budget for one TMA stage pair: 72 KB, 96 KB for q >= 64
// (paper q=80: 0.365 vs 0.372 ms; c4p q=58 unchanged at 72-96 KB and 10-18%
// slower below 72 -- profiles/r02/tma_budget_sweep.txt).  BX_TMA_BUDGET_KB
// overrides.
inline size_t tma_budget(int q) {
  static const int env = [] {
    const char* e = getenv("BX_TMA_BUDGET_KB");
    return e ? atoi(e) : 0;
  }();
  return (size_t)(env > 0 ? env : (q >= 64 ? 96 : 72)) * 1024;
}

// Raise a kernel's MaxDynamicSharedMemorySize to at least `smem` (per device).
// The attribute is per function and shared by every launch configuration and
// host thread, so it only ever grows: lowering it for a smaller tile would make
// a concurrent or later launch of a larger tile fail with cudaErrorInvalidValue.
inline cudaError_t raise_smem_limit(const void* k, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  struct Lim {
    int dev;
    const void* k;
    size_t smem;
  };
  static std::mutex mu;
  static std::vector<Lim> lims;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  for (Lim& l : lims)
    if (l.dev == dev && l.k == k) {
      if (l.smem >= smem) return cudaSuccess;
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess) l.smem = smem;
      return e;
    }
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) lims.push_back(Lim{dev, k, smem});
  return e;
}

// Occupancy of a TMA kernel configuration (raising its dynamic shared memory
// limit first), memoised per (device, Q, threads, smem).  The kernel's limit
// is a per-function attribute shared by every configuration of that Q, so it
// only ever grows: lowering it for a smaller tile would make a later launch of
// a memoised larger tile fail with cudaErrorInvalidValue.
inline cudaError_t tma_occupancy(const void* k, int q, int threads, size_t smem, int* occ) {
  struct Entry {
    int dev, q, threads;
    size_t smem;
    int occ;
  };
  static std::mutex mu;
  static std::vector<Entry> memo;
  int dev = 0;
  cudaGetDevice(&dev);
  // every launch: the limit may not cover this smem yet on this device
  if (cudaError_t e = raise_smem_limit(k, smem); e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> g(mu);
    for (const Entry& e : memo)
      if (e.dev == dev && e.q == q && e.threads == threads && e.smem == smem) {
        *occ = e.occ;
        return cudaSuccess;
      }
  }
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k, threads, smem);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  memo.push_back(Entry{dev, q, threads, smem, *occ});
  return cudaSuccess;
}

// Input stages of the TMA kernel: 2 = double buffer (the planned geometry,
// what bx_launch_info reports), 1 = one buffer per CTA, i.e. twice the tile (or
// twice the CTAs) in the same shared memory.  Unset: launch_eq picks per
// launch from the occupancy of both (see tma_pick_stages); BX_TMA_STAGES=1/2
// forces one, for A/B runs.
inline int tma_stages_env() {
  static const int v = [] {
    const char* e = getenv("BX_TMA_STAGES");
    const int s = e ? atoi(e) : 0;
    return s == 1 || s == 2 ? s : 0;
  }();
  return v;
}

inline void make_tma(LaunchCfg& c, int q, int n, int64_t nblocks, int S = 0) {
  const size_t kTmaBudget = tma_budget(q);
  const int64_t B = (int64_t)q * n;
  if (S == 0) S = tma_stages_env() == 1 ? 1 : 2;
  auto words = [&](int t) { return (int)((((((int64_t)t * B + 7) >> 3) + 4 + 32) + 15) / 16 * 4); };
  auto outw = [&](int t) { return (int)((31 + (int64_t)t * q + 31) >> 5) + 2; };
  auto bytes = [&](int t) { return (size_t)(2 * S * (int64_t)words(t) + 2 * outw(t)) * 4; };
  if (!c.tma) c.tile0 = c.tile;     // the tile before any TMA budget cut
  int T = c.tile0;
  const int Tmin = 32 >> c.tpb_log2 > 0 ? 32 >> c.tpb_log2 : 1;
  while (bytes(T) > kTmaBudget && T > Tmin) T /= 2;
  if (bytes(T) > 200 * 1024) return;  // keep the non-pipelined configuration
  c.tma = 1;
  c.staged = 1;
  c.tile = T;
  c.threads = T << c.tpb_log2;
  c.stage_words = words(T);
  c.stages = S;
  c.smem = bytes(T);
  const int64_t ntiles = (nblocks + T - 1) / T;
  const int per_sm = (int)((200 * 1024) / c.smem) > 0 ? (int)((200 * 1024) / c.smem) : 1;
  const int64_t resident = (int64_t)sm_count() * (per_sm < 4 ? per_sm : 4);
  c.grid = ntiles < resident ? ntiles : resident;
}

template <int Q>
cudaError_t launch_eq(const EqArgs& a, const LaunchCfg& c, cudaStream_t s) {
  if (c.tma) {
    auto k = eq_tma_kernel<Q>;
    // persistent: exactly the CTAs that can be resident at once.  The
    // attribute and occupancy queries cost microseconds; they are cached per
    // (device, threads, smem) so small launches stay launch-latency bound.
    int occ = 0;
    cudaError_t e = tma_occupancy(reinterpret_cast<const void*>(k), Q, c.threads, c.smem, &occ);
    if (e != cudaSuccess) return e;
    if (c.stages == 2 && tma_stages_env() == 0) {
      // Single-stage twin of the planned geometry: the same shared memory holds
      // twice the tile, so a CTA has twice the threads.  It wins where the
      // double-buffered plan leaves the SM short of warps -- the 128-register
      // dot kernels at 32 < q <= 64 run 256 threads per SM with two stages and
      // 512 with one (c4p -6%, q=52 n=100 -18%, q=64 n=31 -27%) -- and loses
      // where registers already cap the resident threads or fewer than three
      // CTAs would share an SM (nothing then overlaps a CTA's only load):
      // q=33 n=120 +8%, q=20 n=60 +8% (profiles/r02/dp2a_sweep.txt, sweeps 17-18).
      LaunchCfg alt = c;
      make_tma(alt, Q, a.n, a.nblocks, 1);
      int occ1 = 0;
      if (alt.tma && alt.stages == 1 &&
          tma_occupancy(reinterpret_cast<const void*>(k), Q, alt.threads, alt.smem, &occ1) == cudaSuccess &&
          occ1 >= 3 && 2 * (int64_t)occ1 * alt.threads >= 3 * (int64_t)occ * c.threads) {
        EqArgs a1 = a;
        a1.tile_blocks = alt.tile;
        a1.stage_words = alt.stage_words;
        a1.stages = 1;
        return launch_eq<Q>(a1, alt, s);
      }
    }
    const int64_t ntiles = (a.nblocks + c.tile - 1) / c.tile;
    const int64_t resident = (int64_t)sm_count() * (occ > 0 ? occ : 1);
    const int64_t grid = ntiles < resident ? ntiles : resident;
#if BX_PDL
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(c.threads);
    cfg.dynamicSmemBytes = c.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, a);
#else
    k<<<(unsigned)grid, c.threads, c.smem, s>>>(a);
    return cudaGetLastError();
#endif
  }
  if constexpr (Q == 1 || Q == 2 || Q == 4 || Q == 8 || Q == 16 || Q == 32 || Q == 64 || Q == 128 ||
                period_q(Q)) {
    if (c.direct) {
      DirectArgs d;
      d.x = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(a.x) + a.x_bit0 / 8);
      d.y = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(a.y) + a.y_bit0 / 8);
      d.nblocks = a.nblocks;
      d.out = a.out + a.out_bit0 / 32;
      d.units = c.units;
      // 256-bit loads (two units per load; sweeps C, P, T): q = 8, 16, 128 at
      // any even unit count; q <= 4 from 8 units per block up (the fully
      // unrolled 128-bit form of those is register-bound: q=4 n=256 +57%)
      d.wide = ((Q == 8 || Q == 16 || Q == 128 || (Q == 32 && wide32_enabled()) ||
                 (Q <= 4 && c.units >= 8)) && c.units % 2 == 0 &&
                wide_loads_enabled() &&
                ((reinterpret_cast<uintptr_t>(d.x) | reinterpret_cast<uintptr_t>(d.y)) & 31) == 0)
                   ? 1 : 0;
      d.x_limit = a.x_limit / 4 - a.x_bit0 / 128;
      d.y_limit = a.y_limit / 4 - a.y_bit0 / 128;
      d.out_words = a.out_words - a.out_bit0 / 32;
      const dim3 g((unsigned)c.grid), b(c.threads);
#if BX_PDL
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = g;
      cfg.blockDim = b;
      cfg.dynamicSmemBytes = 0;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if constexpr (period_q(Q)) return cudaLaunchKernelEx(&cfg, eq_period_kernel<Q>, d);
      switch (c.units) {
        case 1: return cudaLaunchKernelEx(&cfg, eq_direct_kernel<Q, 1>, d);
        case 2: return cudaLaunchKernelEx(&cfg, eq_direct_kernel<Q, 2>, d);
        case 4: return cudaLaunchKernelEx(&cfg, eq_direct_kernel<Q, 4>, d);
        case 8: return cudaLaunchKernelEx(&cfg, eq_direct_kernel<Q, 8>, d);
        default: return cudaLaunchKernelEx(&cfg, eq_direct_kernel<Q, 0>, d);
      }
#else
      if constexpr (period_q(Q)) {
        eq_period_kernel<Q><<<g, b, 0, s>>>(d);
        return cudaGetLastError();
      }
      switch (c.units) {
        case 1: eq_direct_kernel<Q, 1><<<g, b, 0, s>>>(d); break;
        case 2: eq_direct_kernel<Q, 2><<<g, b, 0, s>>>(d); break;
        case 4: eq_direct_kernel<Q, 4><<<g, b, 0, s>>>(d); break;
        case 8: eq_direct_kernel<Q, 8><<<g, b, 0, s>>>(d); break;
        default: eq_direct_kernel<Q, 0><<<g, b, 0, s>>>(d); break;
      }
      return cudaGetLastError();
#endif
    }
  }
  if (c.staged) {
    auto k = eq_kernel<Q, true>;
    if (cudaError_t e = raise_smem_limit(reinterpret_cast<const void*>(k), c.smem); e != cudaSuccess)
      return e;
    k<<<(unsigned)c.grid, c.threads, c.smem, s>>>(a);
  } else {
    auto k = eq_kernel<Q, false>;
    k<<<(unsigned)c.grid, c.threads, c.smem, s>>>(a);
  }
  return cudaGetLastError();
}

using LaunchFn = cudaError_t (*)(const EqArgs&, const LaunchCfg&, cudaStream_t);

}  // namespace bx
