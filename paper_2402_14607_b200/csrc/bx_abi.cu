// bx_abi.cu -- the extern "C" boundary (include/blockext_b200.h).
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>

#include <cuda_runtime.h>

#include "../../include/blockext_b200.h"
#include "bx_launch.cuh"

namespace bx {
cudaError_t launch_pack(const void*, int, int, int64_t, void*, int64_t, cudaStream_t, int*);
cudaError_t launch_bernoulli(uint32_t*, int64_t, uint64_t, int64_t, double, cudaStream_t);
int64_t xor_scan_scratch_words(int64_t, int);
cudaError_t launch_xor_scan(uint32_t*, int64_t, int, uint32_t*, cudaStream_t);
int64_t markov_scratch_ints(int64_t, int);
cudaError_t launch_markov(const double*, int64_t, const double*, int, int, uint16_t*, int*,
                          cudaStream_t);
cudaError_t launch_ip_table(int, uint32_t, int, uint32_t, uint32_t, uint16_t*, cudaStream_t);
cudaError_t launch_ip_hist(int, uint32_t, int, uint32_t, uint32_t, uint32_t*, cudaStream_t);
cudaError_t launch_rows_uniform(const uint32_t*, uint32_t, uint32_t, uint32_t, uint8_t*,
                                cudaStream_t);
cudaError_t launch_wide256(const void*, const void*, int, int64_t, void*, cudaStream_t);
cudaError_t launch_gf_pow(int, const uint32_t*, const uint32_t*, const uint32_t*, int64_t, uint32_t*,
                          cudaStream_t);
cudaError_t launch_gf_ip_generic(int, const uint32_t*, const uint32_t*, const uint32_t*, int, int64_t,
                                 uint32_t*, cudaStream_t);

#define BX_EXTERN_Q(Q) extern template cudaError_t launch_eq<Q>(const EqArgs&, const LaunchCfg&, cudaStream_t);
#define BX_X8(b) BX_EXTERN_Q(b + 1) BX_EXTERN_Q(b + 2) BX_EXTERN_Q(b + 3) BX_EXTERN_Q(b + 4) \
                 BX_EXTERN_Q(b + 5) BX_EXTERN_Q(b + 6) BX_EXTERN_Q(b + 7) BX_EXTERN_Q(b + 8)
BX_X8(0) BX_X8(8) BX_X8(16) BX_X8(24) BX_X8(32) BX_X8(40) BX_X8(48) BX_X8(56)
BX_X8(64) BX_X8(72) BX_X8(80) BX_X8(88) BX_X8(96) BX_X8(104) BX_X8(112) BX_X8(120)

template <int... Is>
constexpr auto make_table(std::integer_sequence<int, Is...>) {
  return std::array<LaunchFn, sizeof...(Is)>{{&launch_eq<Is + 1>...}};
}
}  // namespace bx

#include <array>

#ifdef BX_CHECKED
namespace bx {
__device__ unsigned long long g_violations = 0;
__device__ long long g_first_violation[3] = {0, 0, 0};
}  // namespace bx
#endif

namespace {
thread_local std::string g_err;

// The library links its own (static) CUDA runtime, whose per-thread current
// device is independent of the caller's runtime (e.g. torch's).  Every entry
// point therefore switches, for the duration of the call, to the device the
// work runs on: the device of the caller's stream when one is given, else the
// device that owns the call's INPUT (x / samples / counts).  Never the output:
// an output may be a peer GPU's buffer mapped into this process (CUDA IPC,
// distributed_extract(gather="peer")), and choosing its device would size the
// grid for, and launch on, the wrong GPU with a stream that is not its own.
int device_of(const void* p) {
  cudaPointerAttributes at;
  if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) return -1;
  return at.device;
}

struct DeviceScope {
  int prev = -1;
  int dev = -1;   // device the call's kernels run on
  DeviceScope(const void* input, void* stream) {
    int d = -1;
    if (stream && cudaStreamGetDevice(static_cast<cudaStream_t>(stream), &d) != cudaSuccess) {
      cudaGetLastError();
      d = -1;
    }
    if (d < 0) d = device_of(input);
    int cur = 0;
    if (cudaGetDevice(&cur) != cudaSuccess) cur = 0;
    dev = d < 0 ? cur : d;
    if (cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  // true if a kernel on `dev` may dereference p: host/unregistered pointers
  // are left to the caller (UVA host memory), device memory must be local or
  // on a peer this device can access
  bool reaches(const void* p) const {
    const int d = device_of(p);
    if (d < 0 || d == dev) return true;
    static std::atomic<int> memo[64][64];   // 0 unknown, 1 yes, 2 no
    if (dev >= 64 || d >= 64) return true;
    int m = memo[dev][d].load(std::memory_order_acquire);
    if (!m) {
      int ok = 0;
      if (cudaDeviceCanAccessPeer(&ok, dev, d) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
      }
      if (ok) {
        // Capability is not access: a buffer another process exported over
        // CUDA IPC is mapped in ITS device's context here (torch opens the
        // handle under that device), so `dev` -- current for this scope --
        // must enable peer access to d itself.  The setting belongs to the
        // primary contexts, shared with the caller's runtime; "already
        // enabled" (by torch or NCCL) is success.
        const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
        if (e != cudaSuccess) {
          cudaGetLastError();
          if (e != cudaErrorPeerAccessAlreadyEnabled) ok = 0;
        }
      }
      m = ok ? 1 : 2;
      memo[dev][d].store(m, std::memory_order_release);
    }
    return m == 1;
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};
std::atomic<int64_t> g_launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

namespace bx {
// error reporting for the other translation units (bx_pipe.cu)
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace bx

namespace {
const std::array<bx::LaunchFn, 128>& table() {
  static const auto t = bx::make_table(std::make_integer_sequence<int, 128>{});
  return t;
}
}  // namespace

extern "C" {

int bx_version(void) { return 100; }

const char* bx_last_error(void) { return g_err.c_str(); }

int bx_modulus_exponents(int q, int* exps) {
  if (q < 1 || q > 128) return fail(BX_ERANGE, "field width outside 1..128");
  const bx::ModRow& r = bx::kModulus[q];
  for (int i = 0; i < 5; i++) exps[i] = i < r.count ? r.e[i] : 0;
  return r.count;
}

int bx_launch_info(int q, int n, int64_t nblocks, int* tpb, int* tile, int* staged,
                   int* threads, int* smem_bytes, int64_t* grid, int* family) {
  if (q < 1 || q > 128) return fail(BX_ERANGE, "field width outside 1..128");
  if (n < 1 || nblocks < 0) return fail(BX_EINVAL, "n must be >= 1 and nblocks >= 0");
  // geometry for 16-byte aligned buffers starting at bit 0
  const void* al = reinterpret_cast<const void*>(uintptr_t(256));
  bx::LaunchCfg c = bx::direct_ok(q, n, 0, 0, 0, al, al) ? bx::choose_direct(q, n, nblocks)
                                                         : bx::choose_launch(q, n, nblocks);
  if (!c.direct && c.staged) bx::make_tma(c, q, n, nblocks);
  if (tpb) *tpb = 1 << c.tpb_log2;
  if (tile) *tile = c.tile;
  if (staged) *staged = c.staged;
  if (threads) *threads = c.threads;
  if (smem_bytes) *smem_bytes = (int)c.smem;
  if (grid) *grid = c.grid;
  if (family) *family = c.family + (c.direct ? 2 : 0) + (c.tma ? 4 : 0);
  return BX_OK;
}

int bx_extract_eq(const void* x, int64_t x_bytes, int64_t x_bit0, const void* y, int64_t y_bytes,
                  int64_t y_bit0, int q, int n, int64_t nblocks, void* out, int64_t out_bit0,
                  void* stream) {
  if (q < 1 || q > 128) return fail(BX_ERANGE, "field width outside 1..128");
  if (n < 1) return fail(BX_EINVAL, "vec_len must be >= 1");
  if (nblocks < 0 || x_bit0 < 0 || y_bit0 < 0 || out_bit0 < 0 || x_bytes < 0 || y_bytes < 0)
    return fail(BX_EINVAL, "negative size or offset");
  if (nblocks == 0) return BX_OK;
  if (!x || !y || !out) return fail(BX_EINVAL, "null buffer");
  if (((uintptr_t)x | (uintptr_t)y | (uintptr_t)out) & 3)
    return fail(BX_EINVAL, "buffers must be 4-byte aligned");
  const DeviceScope scope(x, stream);
  if (!scope.reaches(y) || !scope.reaches(out))
    return fail(BX_EINVAL, "y or out lives on a GPU the compute device (x's / the stream's) cannot reach");
  const int64_t B = (int64_t)q * n;
  if (nblocks > (INT64_MAX - x_bit0) / B || nblocks > (INT64_MAX - y_bit0) / B)
    return fail(BX_EINVAL, "block range overflows");
  if (x_bit0 + nblocks * B > 8 * x_bytes) return fail(BX_EINVAL, "x stream shorter than the block range");
  if (y_bit0 + nblocks * B > 8 * y_bytes) return fail(BX_EINVAL, "y stream shorter than the block range");
  bx::LaunchCfg c = bx::direct_ok(q, n, x_bit0, y_bit0, out_bit0, x, y)
                        ? bx::choose_direct(q, n, nblocks)
                        : bx::choose_launch(q, n, nblocks);
  if (!c.direct && c.staged && ((((uintptr_t)x) | ((uintptr_t)y)) & 15) == 0)
    bx::make_tma(c, q, n, nblocks);
  if (c.grid > 0x7FFFFFFF) return fail(BX_EINVAL, "too many blocks for one launch");
  bx::EqArgs a;
  a.x = static_cast<const uint32_t*>(x);
  a.y = static_cast<const uint32_t*>(y);
  a.x_bit0 = x_bit0;
  a.y_bit0 = y_bit0;
  a.x_words = (x_bytes + 3) / 4;
  a.y_words = (y_bytes + 3) / 4;
  a.nblocks = nblocks;
  a.out = static_cast<uint32_t*>(out);
  a.out_bit0 = out_bit0;
  a.n = n;
  a.tpb_log2 = c.tpb_log2;
  a.tile_blocks = c.tile;
  a.stage_words = c.stage_words;
  a.stages = c.stages;
  // ABI guarantee: readable through round_up(bytes, 16) + 16
  a.x_limit = ((x_bytes + 15) / 16) * 4 + 4;
  a.y_limit = ((y_bytes + 15) / 16) * 4 + 4;
  a.out_words = (out_bit0 + nblocks * q + 31) / 32;
#ifdef BX_CHECKED
  // self-test of the checker: under-report the output bound by one word so
  // the last store of the run must be flagged
  if (getenv("BX_CHECK_SELFTEST")) a.out_words -= 1;
#endif
  cudaError_t e = table()[q - 1](a, c, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(BX_ECUDA, std::string("bx_extract_eq: ") + cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return BX_OK;
}

int bx_extract_neq(const void* x, int64_t x_bytes, const void* y, int64_t y_bytes, int q1,
                   int step, int n, int64_t nblocks, void* out, void* stream) {
  if (n < 1 || nblocks < 0 || q1 < 1 || step < 0) return fail(BX_EINVAL, "bad neq schedule");
  if (nblocks == 0) return BX_OK;
  const int64_t qlast = (int64_t)q1 + (nblocks - 1) * (int64_t)step;
  if (qlast > 128) return fail(BX_ERANGE, "block width beyond 128 (reference width-cap)");
  int64_t in_off = 0, out_off = 0;
  int64_t k = 0;
  while (k < nblocks) {
    // runs of equal width (step == 0: the whole schedule) go out as one launch
    const int q = (int)(q1 + k * (int64_t)step);
    const int64_t run = step == 0 ? nblocks : 1;
    const int rc = bx_extract_eq(x, x_bytes, in_off, y, y_bytes, in_off, q, n, run, out, out_off,
                                 stream);
    if (rc) return rc;
    in_off += run * (int64_t)q * n;
    out_off += run * q;
    k += run;
  }
  return BX_OK;
}

int bx_pack(const void* samples, int elem_bytes, int b, int64_t count, void* out, int64_t out_bit0,
            void* stream) {
  if (!(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8))
    return fail(BX_EINVAL, "elem_bytes must be 1, 2, 4 or 8");
  if (b < 1 || b > 8 * elem_bytes) return fail(BX_EINVAL, "bits per sample outside 1..8*elem_bytes");
  if (count < 0 || out_bit0 < 0) return fail(BX_EINVAL, "negative count or offset");
  if (count == 0) return BX_OK;
  if (!samples || !out) return fail(BX_EINVAL, "null buffer");
  if ((uintptr_t)out & 3) return fail(BX_EINVAL, "out must be 4-byte aligned");
  const DeviceScope scope(samples, stream);
  if (!scope.reaches(out)) return fail(BX_EINVAL, "out lives on a GPU the samples' device cannot reach");
  int launched = 0;
  cudaError_t e = bx::launch_pack(samples, elem_bytes, b, count, out, out_bit0,
                                  static_cast<cudaStream_t>(stream), &launched);
  if (e != cudaSuccess) return fail(BX_ECUDA, std::string("bx_pack: ") + cudaGetErrorString(e));
  g_launches.fetch_add(launched, std::memory_order_relaxed);
  return BX_OK;
}

int bx_bernoulli_bits(void* out, int64_t nbits, double p, uint64_t seed, int64_t bit0,
                      void* stream) {
  if (nbits < 0 || bit0 < 0 || !(p >= 0.0 && p <= 1.0)) return fail(BX_EINVAL, "bad Bernoulli request");
  if (nbits == 0) return BX_OK;
  if (!out || ((uintptr_t)out & 3)) return fail(BX_EINVAL, "out must be a 4-byte aligned buffer");
  const DeviceScope scope(out, stream);
  cudaError_t e = bx::launch_bernoulli(static_cast<uint32_t*>(out), nbits, seed, bit0, p,
                                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(BX_ECUDA, std::string("bx_bernoulli_bits: ") + cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return BX_OK;
}

int64_t bx_xor_scan_scratch_bytes(int64_t rows, int row_words) {
  if (rows < 0 || row_words < 1) return fail(BX_EINVAL, "bad matrix shape");
  return 4 * bx::xor_scan_scratch_words(rows, row_words);
}

int bx_xor_scan_rows(void* matrix, int64_t rows, int row_words, void* scratch, void* stream) {
  if (rows < 0 || row_words < 1) return fail(BX_EINVAL, "bad matrix shape");
  if (rows <= 1) return BX_OK;
  if (!matrix || !scratch || ((uintptr_t)matrix & 3) || ((uintptr_t)scratch & 3))
    return fail(BX_EINVAL, "matrix and scratch must be 4-byte aligned device buffers");
  const DeviceScope scope(matrix, stream);
  cudaError_t e = bx::launch_xor_scan(static_cast<uint32_t*>(matrix), rows, row_words,
                                      static_cast<uint32_t*>(scratch), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(BX_ECUDA, std::string("bx_xor_scan_rows: ") + cudaGetErrorString(e));
  g_launches.fetch_add(3, std::memory_order_relaxed);
  return BX_OK;
}

int64_t bx_markov_scratch_bytes(int64_t count, int b) {
  if (count < 0 || b < 1 || b > 16) return fail(BX_EINVAL, "bad markov shape");
  return 4 * bx::markov_scratch_ints(count, b);
}

int bx_markov_chain(const void* u, int64_t count, const void* cum, int b, int start_state,
                    void* values, void* scratch, void* stream) {
  if (count < 0 || b < 1 || b > 16) return fail(BX_EINVAL, "bits per sample outside 1..16");
  if (start_state < 0 || start_state >= (1 << b)) return fail(BX_EINVAL, "start state out of range");
  if (count == 0) return BX_OK;
  if (!u || !cum || !values || !scratch) return fail(BX_EINVAL, "null buffer");
  const DeviceScope scope(u, stream);
  if (!scope.reaches(values) || !scope.reaches(cum) || !scope.reaches(scratch))
    return fail(BX_EINVAL, "markov buffers live on a GPU the compute device cannot reach");
  cudaError_t e = bx::launch_markov(static_cast<const double*>(u), count, static_cast<const double*>(cum),
                                    b, start_state, static_cast<uint16_t*>(values),
                                    static_cast<int*>(scratch), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(BX_ECUDA, std::string("bx_markov_chain: ") + cudaGetErrorString(e));
  g_launches.fetch_add(3, std::memory_order_relaxed);
  return BX_OK;
}

static uint32_t modulus_low(int q) {
  uint32_t low = 0;
  const bx::ModRow& r = bx::kModulus[q];
  for (int i = 0; i < r.count; i++)
    if (r.e[i] != q) low |= 1u << r.e[i];
  return low;
}

int bx_ip_table(int q, int n, uint32_t x0, uint32_t nx, void* out, void* stream) {
  if (q < 1 || n < 1 || q * n > 16) return fail(BX_EINVAL, "ip table needs q*n <= 16");
  if (nx == 0) return BX_OK;
  if ((uint64_t)x0 + nx > (1ull << (q * n))) return fail(BX_EINVAL, "x range beyond 2^(q*n)");
  if (!out || ((uintptr_t)out & 1)) return fail(BX_EINVAL, "out must be a 2-byte aligned buffer");
  const DeviceScope scope(out, stream);
  cudaError_t e = bx::launch_ip_table(q, modulus_low(q), n, x0, nx, static_cast<uint16_t*>(out),
                                      static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(BX_ECUDA, std::string("bx_ip_table: ") + cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return BX_OK;
}

int bx_ip_histograms(int q, int n, uint32_t d0, uint32_t nd, void* counts, void* stream) {
  if (q < 1 || n < 1 || q * n > 16) return fail(BX_EINVAL, "histograms need q*n <= 16");
  if (nd == 0) return BX_OK;
  if ((uint64_t)d0 + nd > (1ull << (q * n))) return fail(BX_EINVAL, "d range beyond 2^(q*n)");
  if (!counts || ((uintptr_t)counts & 3)) return fail(BX_EINVAL, "counts must be 4-byte aligned");
  const DeviceScope scope(counts, stream);
  cudaError_t e = bx::launch_ip_hist(q, modulus_low(q), n, d0, nd, static_cast<uint32_t*>(counts),
                                     static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(BX_ECUDA, std::string("bx_ip_histograms: ") + cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return BX_OK;
}

int bx_rows_uniform(const void* counts, uint32_t nrows, uint32_t bins, uint32_t expected,
                    void* flags, void* stream) {
  if (nrows == 0) return BX_OK;
  if (!counts || !flags) return fail(BX_EINVAL, "null buffer");
  const DeviceScope scope(counts, stream);
  if (!scope.reaches(flags)) return fail(BX_EINVAL, "flags live on a GPU the counts' device cannot reach");
  cudaError_t e = bx::launch_rows_uniform(static_cast<const uint32_t*>(counts), nrows, bins, expected,
                                          static_cast<uint8_t*>(flags), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(BX_ECUDA, std::string("bx_rows_uniform: ") + cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return BX_OK;
}

int bx_extract_eq_wide(const void* x, int64_t x_bytes, const void* y, int64_t y_bytes, int q, int n,
                       int64_t nblocks, void* out, int64_t out_word0, void* stream) {
  if (q != 256) return fail(BX_ERANGE, "wide extraction supports q = 256");
  if (n < 1 || nblocks < 0 || x_bytes < 0 || y_bytes < 0 || out_word0 < 0)
    return fail(BX_EINVAL, "bad wide shape");
  if (nblocks == 0) return BX_OK;
  if (!x || !y || !out) return fail(BX_EINVAL, "null buffer");
  if ((((uintptr_t)x) | ((uintptr_t)y)) & 15) return fail(BX_EINVAL, "x and y must be 16-byte aligned");
  if ((((uintptr_t)out) + 4 * out_word0) & 15)
    return fail(BX_EINVAL, "out + 4*out_word0 must be 16-byte aligned");
  if (nblocks > INT64_MAX / (32 * (int64_t)n)) return fail(BX_EINVAL, "block range overflows");
  const int64_t need = nblocks * 32 * (int64_t)n;
  if (need > x_bytes || need > y_bytes) return fail(BX_EINVAL, "stream shorter than the block range");
  const DeviceScope scope(x, stream);
  if (!scope.reaches(y) || !scope.reaches(out))
    return fail(BX_EINVAL, "y or out lives on a GPU x's device cannot reach");
  cudaError_t e = bx::launch_wide256(x, y, n, nblocks, static_cast<uint32_t*>(out) + out_word0,
                                     static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(BX_ECUDA, std::string("bx_extract_eq_wide: ") + cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return BX_OK;
}

int bx_gf_pow(int q, const void* modulus_low, const void* x, const void* e, int64_t count, void* out,
              void* stream) {
  if (q < 1 || q > 128) return fail(BX_ERANGE, "field width outside 1..128");
  if (count < 0) return fail(BX_EINVAL, "count must be >= 0");
  if (count == 0) return BX_OK;
  if (!modulus_low || !x || !e || !out) return fail(BX_EINVAL, "null buffer");
  const DeviceScope scope(x, stream);
  if (!scope.reaches(e) || !scope.reaches(out) || !scope.reaches(modulus_low))
    return fail(BX_EINVAL, "e, modulus or out lives on a GPU x's device cannot reach");
  cudaError_t err = bx::launch_gf_pow(q, static_cast<const uint32_t*>(modulus_low),
                                      static_cast<const uint32_t*>(x), static_cast<const uint32_t*>(e),
                                      count, static_cast<uint32_t*>(out),
                                      static_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return fail(BX_ECUDA, std::string("bx_gf_pow: ") + cudaGetErrorString(err));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return BX_OK;
}

int bx_gf_ip_generic(int q, const void* modulus_low, const void* x, const void* y, int n,
                     int64_t nvec, void* out, void* stream) {
  if (q < 1 || q > 128) return fail(BX_ERANGE, "field width outside 1..128");
  if (n < 1 || nvec < 0) return fail(BX_EINVAL, "n must be >= 1 and nvec >= 0");
  if (nvec == 0) return BX_OK;
  if (!modulus_low || !x || !y || !out) return fail(BX_EINVAL, "null buffer");
  const DeviceScope scope(x, stream);
  if (!scope.reaches(y) || !scope.reaches(out) || !scope.reaches(modulus_low))
    return fail(BX_EINVAL, "y, modulus or out lives on a GPU x's device cannot reach");
  cudaError_t e = bx::launch_gf_ip_generic(q, static_cast<const uint32_t*>(modulus_low),
                                           static_cast<const uint32_t*>(x), static_cast<const uint32_t*>(y),
                                           n, nvec, static_cast<uint32_t*>(out),
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(BX_ECUDA, std::string("bx_gf_ip_generic: ") + cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return BX_OK;
}

int64_t bx_checked_violations(int reset, int64_t* first) {
#ifdef BX_CHECKED
  unsigned long long v = 0;
  long long f[3] = {0, 0, 0};
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&v, bx::g_violations, sizeof v);
  cudaMemcpyFromSymbol(f, bx::g_first_violation, sizeof f);
  if (first) for (int i = 0; i < 3; i++) first[i] = f[i];
  if (reset) {
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(bx::g_violations, &z, sizeof z);
  }
  return (int64_t)v;
#else
  (void)reset;
  (void)first;
  return -1;  // not a checked build
#endif
}

int64_t bx_launch_count(int reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}

}  // extern "C"
