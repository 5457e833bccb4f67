// bx_launch.cuh -- host-side launch geometry and the per-Q launcher template.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "bx_core.cuh"

namespace bx {

struct LaunchCfg {
  int tpb_log2 = 0;
  int tile = 0;       // blocks per CTA
  int staged = 1;
  int threads = 256;
  int stage_words = 0;
  size_t smem = 0;
  int64_t grid = 0;
  int family = 0;     // 0 diag, 1 holes
};

constexpr size_t kStageBudget = 96 * 1024;    // preferred smem per CTA
constexpr size_t kStageMax = 200 * 1024;      // hard cap before going direct

inline LaunchCfg choose_launch(int q, int n, int64_t nblocks) {
  LaunchCfg c;
  c.family = q <= kDiagMaxQ ? 0 : 1;
  const int64_t B = (int64_t)q * n;
  int64_t units, target;
  if (c.family == 0) {
    units = cdiv(n, 32 / q);
    target = 8;
  } else {
    units = n;
    target = q <= 32 ? 4 : 2;
  }
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

template <int Q>
cudaError_t launch_eq(const EqArgs& a, const LaunchCfg& c, cudaStream_t s) {
  if (c.staged) {
    auto k = eq_kernel<Q, true>;
    if (c.smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
      if (e != cudaSuccess) return e;
    }
    k<<<(unsigned)c.grid, c.threads, c.smem, s>>>(a);
  } else {
    auto k = eq_kernel<Q, false>;
    k<<<(unsigned)c.grid, c.threads, c.smem, s>>>(a);
  }
  return cudaGetLastError();
}

using LaunchFn = cudaError_t (*)(const EqArgs&, const LaunchCfg&, cudaStream_t);

}  // namespace bx
