// bx_host.cu -- one-call extraction from host memory (the real-time small-run
// path: one call per capture chunk, reference extractor.py:264-279 through
// bitio.py:16-64).
//
// bx_extract_eq_host stages both windows into a per-device cached pinned
// buffer, moves them with ONE H2D, runs bx_extract_eq, brings the packed output
// back with one D2H and synchronises: three stream operations (the zeroed
// output region rides in the H2D) and no
// allocation after the first call, so a config-1 run (2 x 128 KiB) costs the
// copies plus a few microseconds of API time instead of a Python/torch
// orchestration of each step.
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include <cuda_runtime.h>

#include "../../include/blockext_b200.h"

namespace bx {
int set_error(int code, const std::string& msg);   // bx_abi.cu
}

namespace {

struct HostCtx {
  std::mutex m;
  cudaStream_t st = nullptr;
  uint8_t* h = nullptr;   // pinned staging: x | y | out
  size_t hcap = 0;
  uint8_t* d = nullptr;   // device: x | y | out
  size_t dcap = 0;
};

constexpr int kMaxDev = 64;
std::mutex g_ctx_m;
std::unique_ptr<HostCtx> g_ctx[kMaxDev];

HostCtx* ctx_for(int dev) {
  std::lock_guard<std::mutex> l(g_ctx_m);
  if (!g_ctx[dev]) g_ctx[dev].reset(new HostCtx);
  return g_ctx[dev].get();
}

int64_t padded(int64_t bytes) { return ((bytes + 15) / 16) * 16 + 16; }

int cuda_fail(const char* what, cudaError_t e) {
  return bx::set_error(BX_ECUDA, std::string("bx_extract_eq_host: ") + what + ": " +
                                     cudaGetErrorString(e));
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" int bx_extract_eq_host(const void* x, int64_t x_bytes, int64_t x_bit0, const void* y,
                                  int64_t y_bytes, int64_t y_bit0, int q, int n, int64_t nblocks,
                                  void* out, int device) {
  if (q < 1 || q > 128) return bx::set_error(BX_ERANGE, "field width outside 1..128");
  if (n < 1 || nblocks < 0 || x_bytes < 0 || y_bytes < 0 || x_bit0 < 0 || y_bit0 < 0)
    return bx::set_error(BX_EINVAL, "bx_extract_eq_host: bad shape");
  if (nblocks == 0) return BX_OK;
  if (!x || !y || !out) return bx::set_error(BX_EINVAL, "bx_extract_eq_host: null buffer");
  if (device < 0 || device >= kMaxDev) return bx::set_error(BX_EINVAL, "bx_extract_eq_host: bad device");
  const int64_t B = (int64_t)q * n;
  if (nblocks > (INT64_MAX / 2 - x_bit0) / B || nblocks > (INT64_MAX / 2 - y_bit0) / B)
    return bx::set_error(BX_EINVAL, "bx_extract_eq_host: block range overflows");
  // only the bytes the run reads cross the link
  const int64_t xn = (x_bit0 + nblocks * B + 7) / 8, yn = (y_bit0 + nblocks * B + 7) / 8;
  if (xn > x_bytes || yn > y_bytes)
    return bx::set_error(BX_EINVAL, "bx_extract_eq_host: stream shorter than the block range");
  const int64_t ob = (nblocks * q + 7) / 8;
  const int64_t px = padded(xn), py = padded(yn), po = padded(ob);
  const size_t need = (size_t)(px + py + po);
  HostCtx* c = ctx_for(device);
  std::lock_guard<std::mutex> l(c->m);
  DevGuard g(device);
  cudaError_t e;
  if (!c->st && (e = cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_fail("stream", e);
  if (c->hcap < need) {
    cudaFreeHost(c->h);
    c->h = nullptr;
    c->hcap = 0;
    const size_t cap = need > (1u << 20) ? need : (1u << 20);
    if ((e = cudaMallocHost(&c->h, cap)) != cudaSuccess) return cuda_fail("pinned staging", e);
    c->hcap = cap;
  }
  if (c->dcap < need) {
    cudaFree(c->d);
    c->d = nullptr;
    c->dcap = 0;
    const size_t cap = need > (1u << 20) ? need : (1u << 20);
    if ((e = cudaMalloc(&c->d, cap)) != cudaSuccess) return cuda_fail("device buffer", e);
    c->dcap = cap;
  }
  uint8_t* h = c->h;
  std::memcpy(h, x, (size_t)xn);
  std::memset(h + xn, 0, (size_t)(px - xn));
  std::memcpy(h + px, y, (size_t)yn);
  std::memset(h + px + yn, 0, (size_t)(py - yn));
  std::memset(h + px + py, 0, (size_t)po);   // the zeroed output rides along in the one H2D
  uint8_t* d = c->d;
  if ((e = cudaMemcpyAsync(d, h, (size_t)(px + py + po), cudaMemcpyHostToDevice, c->st)) != cudaSuccess)
    return cuda_fail("H2D", e);
  const int rc = bx_extract_eq(d, xn, x_bit0, d + px, yn, y_bit0, q, n, nblocks, d + px + py, 0, c->st);
  if (rc) return rc;
  if ((e = cudaMemcpyAsync(h + px + py, d + px + py, (size_t)ob, cudaMemcpyDeviceToHost, c->st)) !=
      cudaSuccess)
    return cuda_fail("D2H", e);
  if ((e = cudaStreamSynchronize(c->st)) != cudaSuccess) return cuda_fail("synchronize", e);
  std::memcpy(out, h + px + py, (size_t)ob);
  return BX_OK;
}
