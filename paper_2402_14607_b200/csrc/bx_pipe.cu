// bx_pipe.cu -- native streaming ingestion.
//
// A push-based pipeline for producers that live outside Python (an ADC /
// FPGA capture loop in C or C++): the caller hands over host bytes of both
// streams as they arrive; the pipe stages them through pinned buffers, copies
// them to the device on two copy streams (x and y in parallel), extracts every
// block that is complete, and returns the packed output bytes.  Incomplete
// trailing blocks are carried, byte-granular, into the next push (their bit
// offset is handed to the kernels as x_bit0 / y_bit0), and so is the last
// partial output byte (merged by the kernels' boundary handling), so any
// sequence of push sizes yields exactly the bytes of one equal-width run over
// the concatenated streams (reference extractor.py:182-208, bitio.py:74-88).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>

#include <cuda_runtime.h>

#include "../../include/blockext_b200.h"

struct bx_pipe {
  int q = 0, n = 0, device = 0;
  int64_t B = 0;               // bits per block per stream
  int64_t cap = 0;             // device stream capacity (bytes)
  int64_t chunk = 0;           // max new bytes per push per stream
  uint8_t* dx = nullptr;       // device streams: [carried bytes | new bytes | guard]
  uint8_t* dy = nullptr;
  uint8_t* dx2 = nullptr;      // ping-pong partners for moving the carried tail
  uint8_t* dy2 = nullptr;
  uint8_t* dout = nullptr;     // device output (packed bits of this push + carried byte)
  uint8_t* hx = nullptr;       // pinned staging
  uint8_t* hy = nullptr;
  uint8_t* hout = nullptr;
  int64_t carry_bytes = 0;     // carried input bytes at the front of dx / dy
  int carry_bit0 = 0;          // bit offset of the first unprocessed bit in them
  uint8_t out_carry = 0;       // partial output byte not yet returned
  int out_carry_bits = 0;
  int64_t blocks_done = 0;
  cudaStream_t cx = nullptr, cy = nullptr, comp = nullptr;
  cudaEvent_t ex = nullptr, ey = nullptr;
};

namespace {

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

int64_t padded(int64_t bytes) { return ((bytes + 15) / 16) * 16 + 16; }

}  // namespace

extern "C" {

bx_pipe* bx_pipe_create(int q, int n, int64_t chunk_bytes, int device) {
  if (q < 1 || q > 128 || n < 1 || chunk_bytes < 1) return nullptr;
  bx_pipe* p = new (std::nothrow) bx_pipe;
  if (!p) return nullptr;
  p->q = q;
  p->n = n;
  p->device = device;
  p->B = (int64_t)q * n;
  p->chunk = chunk_bytes;
  p->cap = chunk_bytes + (p->B + 7) / 8 + 1;          // new bytes + the carried partial block
  const int64_t max_out = (8 * p->cap / p->B) * q / 8 + 2;
  DevGuard g(device);
  bool ok = cudaMalloc(&p->dx, padded(p->cap)) == cudaSuccess &&
            cudaMalloc(&p->dy, padded(p->cap)) == cudaSuccess &&
            cudaMalloc(&p->dx2, padded(p->cap)) == cudaSuccess &&
            cudaMalloc(&p->dy2, padded(p->cap)) == cudaSuccess &&
            cudaMalloc(&p->dout, padded(max_out)) == cudaSuccess &&
            cudaMallocHost(&p->hx, chunk_bytes) == cudaSuccess &&
            cudaMallocHost(&p->hy, chunk_bytes) == cudaSuccess &&
            cudaMallocHost(&p->hout, padded(max_out)) == cudaSuccess &&
            cudaStreamCreateWithFlags(&p->cx, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&p->cy, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&p->ex, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&p->ey, cudaEventDisableTiming) == cudaSuccess;
  if (ok) ok = cudaMemset(p->dx, 0, padded(p->cap)) == cudaSuccess &&
               cudaMemset(p->dy, 0, padded(p->cap)) == cudaSuccess &&
               cudaMemset(p->dx2, 0, padded(p->cap)) == cudaSuccess &&
               cudaMemset(p->dy2, 0, padded(p->cap)) == cudaSuccess;
  if (!ok) {
    bx_pipe_destroy(p);
    return nullptr;
  }
  return p;
}

void bx_pipe_destroy(bx_pipe* p) {
  if (!p) return;
  DevGuard g(p->device);
  cudaFree(p->dx);
  cudaFree(p->dy);
  cudaFree(p->dx2);
  cudaFree(p->dy2);
  cudaFree(p->dout);
  cudaFreeHost(p->hx);
  cudaFreeHost(p->hy);
  cudaFreeHost(p->hout);
  if (p->cx) cudaStreamDestroy(p->cx);
  if (p->cy) cudaStreamDestroy(p->cy);
  if (p->comp) cudaStreamDestroy(p->comp);
  if (p->ex) cudaEventDestroy(p->ex);
  if (p->ey) cudaEventDestroy(p->ey);
  delete p;
}

int bx_pipe_push(bx_pipe* p, const void* x, const void* y, int64_t nbytes, void* out,
                 int64_t out_cap, int64_t* out_bytes) {
  if (!p || nbytes < 0 || nbytes > p->chunk || (!x && nbytes) || (!y && nbytes) || !out_bytes)
    return BX_EINVAL;
  *out_bytes = 0;
  DevGuard g(p->device);
  // stage and copy the new bytes behind the carried ones
  if (nbytes) {
    std::memcpy(p->hx, x, (size_t)nbytes);
    cudaMemcpyAsync(p->dx + p->carry_bytes, p->hx, nbytes, cudaMemcpyHostToDevice, p->cx);
    cudaEventRecord(p->ex, p->cx);
    std::memcpy(p->hy, y, (size_t)nbytes);
    cudaMemcpyAsync(p->dy + p->carry_bytes, p->hy, nbytes, cudaMemcpyHostToDevice, p->cy);
    cudaEventRecord(p->ey, p->cy);
    cudaStreamWaitEvent(p->comp, p->ex, 0);
    cudaStreamWaitEvent(p->comp, p->ey, 0);
  }
  const int64_t have = p->carry_bytes + nbytes;
  const int64_t avail_bits = 8 * have - p->carry_bit0;
  const int64_t k = avail_bits / p->B;                 // complete blocks
  const int64_t out_bits = k * p->q;
  const int64_t total_bits = p->out_carry_bits + out_bits;
  const int64_t whole = total_bits / 8;
  if (whole > out_cap) return BX_EINVAL;
  if (k > 0) {
    // the carried partial output byte goes in first; the kernel merges after it
    cudaMemcpyAsync(p->dout, &p->out_carry, 1, cudaMemcpyHostToDevice, p->comp);
    const int rc = bx_extract_eq(p->dx, have, p->carry_bit0, p->dy, have, p->carry_bit0, p->q, p->n,
                                 k, p->dout, p->out_carry_bits, p->comp);
    if (rc) return rc;
    cudaMemcpyAsync(p->hout, p->dout, (total_bits + 7) / 8, cudaMemcpyDeviceToHost, p->comp);
  }
  if (cudaStreamSynchronize(p->comp) != cudaSuccess || cudaStreamSynchronize(p->cx) != cudaSuccess ||
      cudaStreamSynchronize(p->cy) != cudaSuccess)
    return BX_ECUDA;
  if (k > 0) {
    std::memcpy(out, p->hout, (size_t)whole);
    p->out_carry_bits = (int)(total_bits % 8);
    p->out_carry = p->out_carry_bits ? (uint8_t)(p->hout[whole] & ((1u << p->out_carry_bits) - 1)) : 0;
    *out_bytes = whole;
  }
  // carry the unused tail bytes to the front of the device streams
  const int64_t used_bits = p->carry_bit0 + k * p->B;
  const int64_t first = used_bits / 8;
  const int64_t rest = have - first;
  if (first > 0 && rest > 0) {
    // source and destination would overlap in place: move into the partner
    // buffers and swap
    cudaMemcpyAsync(p->dx2, p->dx + first, rest, cudaMemcpyDeviceToDevice, p->comp);
    cudaMemcpyAsync(p->dy2, p->dy + first, rest, cudaMemcpyDeviceToDevice, p->comp);
    if (cudaStreamSynchronize(p->comp) != cudaSuccess) return BX_ECUDA;
    std::swap(p->dx, p->dx2);
    std::swap(p->dy, p->dy2);
  }
  p->carry_bytes = rest;
  p->carry_bit0 = (int)(used_bits % 8);
  p->blocks_done += k;
  return BX_OK;
}

int bx_pipe_flush(bx_pipe* p, void* out, int64_t* out_bytes) {
  if (!p || !out || !out_bytes) return BX_EINVAL;
  *out_bytes = 0;
  if (p->out_carry_bits) {
    static_cast<uint8_t*>(out)[0] = p->out_carry;   // zero-padded final byte (bitio.py:84-88)
    *out_bytes = 1;
    p->out_carry = 0;
    p->out_carry_bits = 0;
  }
  return BX_OK;
}

int64_t bx_pipe_blocks(const bx_pipe* p) { return p ? p->blocks_done : -1; }

}  // extern "C"
