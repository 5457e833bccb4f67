// bx_pipe.cu -- native streaming ingestion.
//
// A push-based pipeline for producers that live outside Python (an ADC /
// FPGA capture loop in C or C++): the caller hands over host bytes of both
// streams as they arrive and gets back the packed output bytes of completed
// blocks.  Incomplete trailing blocks are carried, byte-granular, into the
// next push (their bit offset is handed to the kernels as x_bit0 / y_bit0),
// and so is the last partial output byte (merged by the kernels' boundary
// handling), so any sequence of push sizes yields exactly the bytes of one
// equal-width run over the concatenated streams (reference
// extractor.py:182-208, bitio.py:74-88).
//
// The block arithmetic of a push (complete blocks, carried bytes, output
// bits) depends only on byte counts, so the host never waits for the device
// to plan the next push.  Each push owns one of `depth` slots (pinned
// staging, device windows, device/pinned output):
//
//   host:  memcpy x, y -> pinned slot s
//   cx/cy: carried tail  slot s-1 -> slot s (D2D), new bytes pinned -> slot s (H2D)
//   comp:  wait cx, cy; carried output byte -> dout[s][0]; bx_extract_eq;
//          last partial output byte -> dcarry; whole bytes dout[s] -> hout[s]
//
// and the call returns the output of the oldest push once more than depth-1
// pushes are in flight.  With depth 2, push k+1's host copy and H2D overlap
// push k's kernel and D2H; depth 1 is the synchronous pipe (every push
// returns its own output).  bx_pipe_drain retires everything in flight.
#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/blockext_b200.h"

namespace bx {
int set_error(int code, const std::string& msg);   // bx_abi.cu
}

namespace {

constexpr int kMaxDepth = 4;

struct Slot {
  uint8_t* dx = nullptr;     // device windows: [carried bytes | new bytes | guard]
  uint8_t* dy = nullptr;
  uint8_t* dout = nullptr;   // device output: [carried partial byte | this push's bits]
  uint8_t* hx = nullptr;     // pinned staging
  uint8_t* hy = nullptr;
  uint8_t* hout = nullptr;   // pinned output (whole bytes)
  cudaEvent_t ex = nullptr, ey = nullptr, done = nullptr;
  int64_t whole = 0;         // output bytes this push returns
  int64_t have = 0;          // valid input bytes in dx / dy
};

int64_t padded(int64_t bytes) { return ((bytes + 15) / 16) * 16 + 16; }

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

// Host copy workers: the staging memcpy (caller memory -> pinned slot) is
// host-memory bound at ~10 GB/s per thread, so each push splits its x and y
// copies into pieces run by a few persistent threads (BX_PIPE_THREADS,
// default 4) plus the calling thread.
class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 0; i < n; i++) th_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> l(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // copies every (dst, src, len) job; returns when all are done
  void run(const std::vector<std::tuple<uint8_t*, const uint8_t*, size_t>>& jobs) {
    {
      std::lock_guard<std::mutex> l(m_);
      jobs_ = &jobs;
      next_ = 0;
      left_ = jobs.size();
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [this] { return left_ == 0; });
    jobs_ = nullptr;
  }

 private:
  bool take(size_t* i) {
    std::lock_guard<std::mutex> l(m_);
    if (!jobs_ || next_ >= jobs_->size()) return false;
    *i = next_++;
    return true;
  }
  void work() {
    size_t i;
    while (take(&i)) {
      auto [d, s, n] = (*jobs_)[i];
      std::memcpy(d, s, n);
      std::lock_guard<std::mutex> l(m_);
      if (--left_ == 0) done_.notify_all();
    }
  }
  void loop() {
    for (;;) {
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [this] { return stop_ || (jobs_ && next_ < jobs_->size()); });
        if (stop_) return;
      }
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::vector<std::tuple<uint8_t*, const uint8_t*, size_t>>* jobs_ = nullptr;
  size_t next_ = 0, left_ = 0;
  bool stop_ = false;
};

int pipe_threads() {
  const char* e = std::getenv("BX_PIPE_THREADS");
  const int n = e ? std::atoi(e) : 4;
  return std::max(0, std::min(n, 32));
}

int cuda_fail(const char* what, cudaError_t e) {
  return bx::set_error(BX_ECUDA, std::string("bx_pipe: ") + what + ": " + cudaGetErrorString(e));
}

}  // namespace

struct bx_pipe {
  int q = 0, n = 0, device = 0, depth = 1;
  int nslots = 2;              // max(depth, 2): the carried tail moves between slots
  int64_t B = 0;               // bits per block per stream
  int64_t cap = 0;             // device window capacity (bytes)
  int64_t chunk = 0;           // max new bytes per push per stream
  int64_t max_out = 0;         // max whole output bytes of one push
  Slot slot[kMaxDepth];
  uint8_t* dcarry = nullptr;   // device: the partial output byte not yet returned
  int64_t pushes = 0;          // pushes enqueued
  int64_t retired = 0;         // pushes whose output was returned
  int cur = -1;                // slot of the newest push (holds the carried input tail)
  int64_t carry_bytes = 0;     // carried input bytes (front of the next push's windows)
  int64_t carry_first = 0;     // ... their offset in slot `cur`'s windows
  int carry_bit0 = 0;          // bit offset of the first unprocessed bit in them
  int out_carry_bits = 0;      // valid bits in dcarry
  int64_t blocks_done = 0;
  cudaStream_t cx = nullptr, cy = nullptr, comp = nullptr;
  CopyPool* pool = nullptr;
};

namespace {

void release(bx_pipe* p) {
  for (Slot& s : p->slot) {
    cudaFree(s.dx);
    cudaFree(s.dy);
    cudaFree(s.dout);
    cudaFreeHost(s.hx);
    cudaFreeHost(s.hy);
    cudaFreeHost(s.hout);
    if (s.ex) cudaEventDestroy(s.ex);
    if (s.ey) cudaEventDestroy(s.ey);
    if (s.done) cudaEventDestroy(s.done);
  }
  delete p->pool;
  p->pool = nullptr;
  cudaFree(p->dcarry);
  if (p->cx) cudaStreamDestroy(p->cx);
  if (p->cy) cudaStreamDestroy(p->cy);
  if (p->comp) cudaStreamDestroy(p->comp);
}

// wait for the oldest in-flight push and append its output to out
int retire_one(bx_pipe* p, uint8_t* out, int64_t* written) {
  Slot& s = p->slot[p->retired % p->nslots];
  cudaError_t e = cudaEventSynchronize(s.done);
  if (e != cudaSuccess) return cuda_fail("output of a push", e);
  if (s.whole) std::memcpy(out + *written, s.hout, (size_t)s.whole);
  *written += s.whole;
  p->retired++;
  return BX_OK;
}

int64_t pending_bytes(const bx_pipe* p, int64_t keep) {
  int64_t tot = 0;
  for (int64_t k = p->retired; k + keep < p->pushes; k++) tot += p->slot[k % p->nslots].whole;
  return tot;
}

}  // namespace

extern "C" {

bx_pipe* bx_pipe_create_async(int q, int n, int64_t chunk_bytes, int device, int depth) {
  if (q < 1 || q > 128 || n < 1 || chunk_bytes < 1 || depth < 1 || depth > kMaxDepth) {
    bx::set_error(BX_EINVAL, "bx_pipe_create: need 1 <= q <= 128, n >= 1, chunk_bytes >= 1, "
                             "1 <= depth <= 4");
    return nullptr;
  }
  bx_pipe* p = new (std::nothrow) bx_pipe;
  if (!p) {
    bx::set_error(BX_ECUDA, "bx_pipe_create: out of host memory");
    return nullptr;
  }
  p->q = q;
  p->n = n;
  p->device = device;
  p->depth = depth;
  p->nslots = std::max(depth, 2);
  p->B = (int64_t)q * n;
  p->chunk = chunk_bytes;
  p->cap = chunk_bytes + (p->B + 7) / 8 + 1;           // new bytes + the carried partial block
  p->max_out = (8 * p->cap / p->B) * q / 8 + 2;
  DevGuard g(device);
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t r) {
    if (e == cudaSuccess) e = r;
    return e == cudaSuccess;
  };
  for (int i = 0; i < p->nslots && e == cudaSuccess; i++) {
    Slot& s = p->slot[i];
    ok(cudaMalloc(&s.dx, padded(p->cap))) && ok(cudaMalloc(&s.dy, padded(p->cap))) &&
        ok(cudaMalloc(&s.dout, padded(p->max_out))) && ok(cudaMallocHost(&s.hx, chunk_bytes)) &&
        ok(cudaMallocHost(&s.hy, chunk_bytes)) && ok(cudaMallocHost(&s.hout, padded(p->max_out))) &&
        ok(cudaEventCreateWithFlags(&s.ex, cudaEventDisableTiming)) &&
        ok(cudaEventCreateWithFlags(&s.ey, cudaEventDisableTiming)) &&
        ok(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming)) &&
        ok(cudaMemset(s.dx, 0, padded(p->cap))) && ok(cudaMemset(s.dy, 0, padded(p->cap)));
  }
  ok(cudaMalloc(&p->dcarry, 16)) && ok(cudaMemset(p->dcarry, 0, 16)) &&
      ok(cudaStreamCreateWithFlags(&p->cx, cudaStreamNonBlocking)) &&
      ok(cudaStreamCreateWithFlags(&p->cy, cudaStreamNonBlocking)) &&
      ok(cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking));
  if (e == cudaSuccess) {
    const int nt = pipe_threads();
    if (nt > 0) p->pool = new (std::nothrow) CopyPool(nt);
  }
  if (e != cudaSuccess) {
    cuda_fail("create", e);
    release(p);
    delete p;
    return nullptr;
  }
  return p;
}

bx_pipe* bx_pipe_create(int q, int n, int64_t chunk_bytes, int device) {
  return bx_pipe_create_async(q, n, chunk_bytes, device, 1);
}

int64_t bx_pipe_max_output(const bx_pipe* p) { return p ? p->max_out : -1; }

int bx_pipe_push(bx_pipe* p, const void* x, const void* y, int64_t nbytes, void* out,
                 int64_t out_cap, int64_t* out_bytes) {
  if (!p || !out_bytes) return bx::set_error(BX_EINVAL, "bx_pipe_push: null pipe or out_bytes");
  *out_bytes = 0;
  if (nbytes < 0 || nbytes > p->chunk)
    return bx::set_error(BX_EINVAL, "bx_pipe_push: nbytes outside 0..chunk_bytes");
  if ((!x || !y) && nbytes) return bx::set_error(BX_EINVAL, "bx_pipe_push: null input");
  // block arithmetic of this push (host only)
  const int64_t have = p->carry_bytes + nbytes;
  const int64_t k = (8 * have - p->carry_bit0) / p->B;            // complete blocks
  const int64_t total_bits = p->out_carry_bits + k * p->q;
  const int64_t whole = total_bits / 8;
  // outputs this call returns: the oldest pushes, this one included, until
  // depth-1 stay in flight
  int64_t need = 0;
  for (int64_t idx = p->retired; idx + p->depth - 1 <= p->pushes; idx++)
    need += idx == p->pushes ? whole : p->slot[idx % p->nslots].whole;
  if (need > out_cap) return bx::set_error(BX_EINVAL, "bx_pipe_push: out_cap too small for the "
                                                      "output this push returns");
  if (need && !out) return bx::set_error(BX_EINVAL, "bx_pipe_push: null out");
  DevGuard g(p->device);
  const int si = (int)(p->pushes % p->nslots);
  Slot& s = p->slot[si];
  // slot si was last used by push (pushes - nslots), which has been retired
  // (synchronised), so its buffers are free; the carried tail comes from the
  // previous push's slot, never this one (nslots >= 2)
  cudaError_t e;
  const int64_t rest = p->carry_bytes;
  if (nbytes) {
    // stage both streams into the slot's pinned buffers: pieces of >= 1 MiB
    // over the copy workers
    std::vector<std::tuple<uint8_t*, const uint8_t*, size_t>> jobs;
    const int64_t piece = std::max<int64_t>(1 << 20, nbytes / (2 * (p->pool ? 5 : 1)) + 1);
    for (int side = 0; side < 2; side++) {
      uint8_t* h = side ? s.hy : s.hx;
      const uint8_t* src = static_cast<const uint8_t*>(side ? y : x);
      for (int64_t o = 0; o < nbytes; o += piece)
        jobs.emplace_back(h + o, src + o, (size_t)std::min(piece, nbytes - o));
    }
    if (p->pool && jobs.size() > 1) {
      p->pool->run(jobs);
    } else {
      for (auto& [d, src, len] : jobs) std::memcpy(d, src, len);
    }
  }
  for (int side = 0; side < 2; side++) {
    uint8_t* dst = side ? s.dy : s.dx;
    uint8_t* h = side ? s.hy : s.hx;
    cudaStream_t st = side ? p->cy : p->cx;
    if (rest > 0) {
      const uint8_t* src = (side ? p->slot[p->cur].dy : p->slot[p->cur].dx) + p->carry_first;
      if ((e = cudaMemcpyAsync(dst, src, rest, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return cuda_fail("carry tail", e);
    }
    if (nbytes) {
      if ((e = cudaMemcpyAsync(dst + rest, h, nbytes, cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return cuda_fail("H2D", e);
    }
    if ((e = cudaEventRecord(side ? s.ey : s.ex, st)) != cudaSuccess) return cuda_fail("event", e);
  }
  if ((e = cudaStreamWaitEvent(p->comp, s.ex, 0)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(p->comp, s.ey, 0)) != cudaSuccess)
    return cuda_fail("stream wait", e);
  if (k > 0) {
    // the carried partial output byte goes in first; the kernel merges after it
    if (p->out_carry_bits &&
        (e = cudaMemcpyAsync(s.dout, p->dcarry, 1, cudaMemcpyDeviceToDevice, p->comp)) != cudaSuccess)
      return cuda_fail("output carry", e);
    const int rc = bx_extract_eq(s.dx, have, p->carry_bit0, s.dy, have, p->carry_bit0, p->q, p->n, k,
                                 s.dout, p->out_carry_bits, p->comp);
    if (rc) return rc;
    if (total_bits % 8 &&
        (e = cudaMemcpyAsync(p->dcarry, s.dout + whole, 1, cudaMemcpyDeviceToDevice, p->comp)) !=
            cudaSuccess)
      return cuda_fail("output carry", e);
    if (whole && (e = cudaMemcpyAsync(s.hout, s.dout, whole, cudaMemcpyDeviceToHost, p->comp)) !=
                     cudaSuccess)
      return cuda_fail("D2H", e);
  }
  if ((e = cudaEventRecord(s.done, p->comp)) != cudaSuccess) return cuda_fail("event", e);
  s.whole = whole;
  s.have = have;
  // the unused tail stays in this slot's windows and moves with the next push
  const int64_t used_bits = p->carry_bit0 + k * p->B;
  p->carry_first = used_bits / 8;
  p->carry_bytes = have - p->carry_first;
  p->carry_bit0 = (int)(used_bits % 8);
  if (k > 0) p->out_carry_bits = (int)(total_bits % 8);
  p->blocks_done += k;
  p->cur = si;
  p->pushes++;
  // the next push reads the carried tail from slot si on cx / cy, ordered
  // behind this push's H2D
  int64_t written = 0;
  while (p->pushes - p->retired > p->depth - 1) {
    const int rc = retire_one(p, static_cast<uint8_t*>(out), &written);
    if (rc) return rc;
  }
  *out_bytes = written;
  return BX_OK;
}

int bx_pipe_drain(bx_pipe* p, void* out, int64_t out_cap, int64_t* out_bytes) {
  if (!p || !out_bytes) return bx::set_error(BX_EINVAL, "bx_pipe_drain: null pipe or out_bytes");
  *out_bytes = 0;
  const int64_t need = pending_bytes(p, 0);
  if (need > out_cap) return bx::set_error(BX_EINVAL, "bx_pipe_drain: out_cap too small");
  if (need && !out) return bx::set_error(BX_EINVAL, "bx_pipe_drain: null out");
  DevGuard g(p->device);
  int64_t written = 0;
  while (p->retired < p->pushes) {
    const int rc = retire_one(p, static_cast<uint8_t*>(out), &written);
    if (rc) return rc;
  }
  *out_bytes = written;
  return BX_OK;
}

int bx_pipe_flush(bx_pipe* p, void* out, int64_t* out_bytes) {
  if (!p || !out || !out_bytes) return bx::set_error(BX_EINVAL, "bx_pipe_flush: null argument");
  *out_bytes = 0;
  if (p->retired < p->pushes)
    return bx::set_error(BX_EINVAL, "bx_pipe_flush: pushes still in flight (bx_pipe_drain first)");
  if (p->out_carry_bits) {
    DevGuard g(p->device);
    uint8_t b = 0;
    cudaError_t e = cudaMemcpy(&b, p->dcarry, 1, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail("flush", e);
    // zero-padded final byte (bitio.py:84-88)
    static_cast<uint8_t*>(out)[0] = (uint8_t)(b & ((1u << p->out_carry_bits) - 1));
    *out_bytes = 1;
    p->out_carry_bits = 0;
    if ((e = cudaMemset(p->dcarry, 0, 1)) != cudaSuccess) return cuda_fail("flush", e);
  }
  return BX_OK;
}

int64_t bx_pipe_blocks(const bx_pipe* p) { return p ? p->blocks_done : -1; }

void bx_pipe_destroy(bx_pipe* p) {
  if (!p) return;
  DevGuard g(p->device);
  cudaStreamSynchronize(p->cx);
  cudaStreamSynchronize(p->cy);
  cudaStreamSynchronize(p->comp);
  release(p);
  delete p;
}

}  // extern "C"
