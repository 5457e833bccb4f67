// bx_pack.cu -- raw-sample packer (reference sources._pack_samples,
// pkg/src/blockext/sources.py:116-121): the low b bits of sample i become
// stream bits [out_bit0 + i*b, out_bit0 + (i+1)*b), LSB-first.
//
// Fast path (pack_tile_kernel<T, B>, T the narrowest type holding B bits):
// a warp owns a tile of 1024 samples, which is exactly 32*B output words.
// Lane l reads its 32 consecutive samples with 256-bit loads (32*sizeof(T)
// bytes: every load is one whole 32-byte sector), merges narrow samples
// SWAR-style, and folds them -- shift amounts are compile-time constants --
// into B words held in registers; they pass through a per-warp shared-memory
// stage (conflict-free / 2-way) so the warp stores 32 consecutive words per
// instruction.  The next tile's loads are issued before the current tile
// folds (software pipeline).  When the stream does not start on a word, words
// are funnel-shifted by out_bit0 % 32; only words shared with the neighbouring
// tiles or with bits outside the range are merged with atomicAnd/Or.  No
// division on the data path; HBM traffic = samples in + packed bits out.
//
// B == 8*sizeof(T) with a byte-aligned destination is a plain D2D copy (the
// packed stream IS the little-endian sample array); other shapes (unaligned
// sample pointers, a type wider than B needs) use pack_generic_kernel.
#include <array>
#include <cstdint>
#include <utility>

#include <cuda_runtime.h>

namespace bx {

namespace {

constexpr int kTile = 1024;   // samples per warp tile (32 lanes x 32 samples)

__device__ __forceinline__ void ldg256(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}

// Bit accumulator whose fill level is a compile-time constant once the
// caller's loop is unrolled; full words land in the lane's register array.
template <int NW>
struct Acc {
  uint32_t cur = 0;
  int nb = 0;
  int wi = 0;
  uint32_t (&o)[NW];
  __device__ __forceinline__ explicit Acc(uint32_t (&r)[NW]) : o(r) {}
  // v holds exactly `width` (1..32) significant low bits
  __device__ __forceinline__ void push(uint32_t v, int width) {
    cur |= v << nb;
    if (nb + width >= 32) {
      o[wi++] = cur;
      cur = nb == 0 ? 0u : (v >> (32 - nb));
      nb = nb + width - 32;
    } else {
      nb += width;
    }
  }
};

template <typename T>
constexpr int kWords = 8 * (int)sizeof(T);   // raw 32-bit words per lane (32 samples)

template <int B>
constexpr uint32_t lowmask() { return B >= 32 ? 0xFFFFFFFFu : ((1u << B) - 1u); }

// Fold a lane's 32 raw samples into its B packed words.  Narrow samples are
// merged SWAR-style first (4 bytes -> one 4B-bit field, 2 halves -> one
// 2B-bit field), so the accumulator sees 8 or 16 pushes instead of 32.
template <typename T, int B>
__device__ __forceinline__ void fold(const uint32_t (&w)[kWords<T>], uint32_t (&o)[B]) {
  Acc<B> a(o);
  if constexpr (sizeof(T) == 1 && B == 1) {
    // 4 samples per multiply: bytes' low bits gathered into the top nibble
    // (0x10204080 places byte k's bit 0 at bit 28+k; cross terms stay < 2^24)
#pragma unroll
    for (int i = 0; i < 8; i++) a.push(((w[i] & 0x01010101u) * 0x10204080u) >> 28, 4);
  } else if constexpr (sizeof(T) == 1) {
    constexpr uint32_t m1 = lowmask<B>() * 0x00010001u;           // bytes 0, 2
    constexpr uint32_t m2 = lowmask<2 * B>();
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const uint32_t t = (w[i] & m1) | ((w[i] >> (8 - B)) & (m1 << B));   // 2B bits per half
      const uint32_t u = (t & m2) | ((t >> (16 - 2 * B)) & (m2 << (2 * B)));
      a.push(u, 4 * B);
    }
  } else if constexpr (sizeof(T) == 2) {
#pragma unroll
    for (int i = 0; i < 16; i++)
      a.push((w[i] & lowmask<B>()) | ((w[i] >> (16 - B)) & (lowmask<B>() << B)), 2 * B);
  } else if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int k = 0; k < 32; k++) a.push(w[k] & lowmask<B>(), B);
  } else {
#pragma unroll
    for (int k = 0; k < 32; k++) {
      if constexpr (B <= 32) {
        a.push(w[2 * k] & lowmask<B>(), B);
      } else {
        a.push(w[2 * k], 32);
        a.push(w[2 * k + 1] & lowmask<B - 32>(), B - 32);
      }
    }
  }
}

template <typename T>
constexpr int pack_warps() { return sizeof(T) == 8 ? 4 : 8; }

// Shared-memory slot of tile word i: odd B writes (lane stride B) are
// conflict-free as is; even B gets one pad word per 32 (<= 2-way writes).
// Reads of 32 consecutive words are conflict-free either way.
template <int B>
__device__ __forceinline__ int sidx(int i) { return (B & 1) ? i : i + (i >> 5); }
template <int B>
constexpr int stage_words() { return (B & 1) ? 32 * B : 33 * B; }

template <typename T>
__device__ __forceinline__ void load_full(const T* p, uint32_t (&w)[kWords<T>]) {
#pragma unroll
  for (int i = 0; i < (int)sizeof(T); i++) {
    uint32_t r[8];
    ldg256(p + i * (32 / (int)sizeof(T)), r);
#pragma unroll
    for (int j = 0; j < 8; j++) w[8 * i + j] = r[j];
  }
}

template <typename T, int B>
__global__ void __launch_bounds__(32 * pack_warps<T>())
    pack_tile_kernel(const T* __restrict__ s, int64_t count, uint32_t* __restrict__ out,
                     int64_t out_bit0) {
  constexpr int W = pack_warps<T>();
  __shared__ uint32_t stage_all[W][stage_words<B>()];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* stage = stage_all[warp];
  const int off = (int)(out_bit0 & 31);
  const int64_t full = count / kTile;                   // whole tiles
  const int64_t stride = (int64_t)gridDim.x * W;
  uint32_t* const base = out + (out_bit0 >> 5);
  int64_t t = (int64_t)blockIdx.x * W + warp;
  // software pipeline: the next tile's samples are in flight while this one folds
  uint32_t wn[kWords<T>];
  if (t < full) load_full(s + t * kTile + lane * 32, wn);
  for (; t <= full; t += stride) {
    const int64_t s0 = t * kTile;
    const int64_t nt = t < full ? kTile : count - s0;
    if (nt <= 0) break;
    uint32_t w[kWords<T>];
    if (t < full) {
#pragma unroll
      for (int i = 0; i < kWords<T>; i++) w[i] = wn[i];
      if (t + stride < full) load_full(s + (t + stride) * kTile + lane * 32, wn);
    } else {   // the job's last, partial tile: guarded element loads, zero fill
      const T* p = s + s0 + lane * 32;
#pragma unroll
      for (int i = 0; i < kWords<T>; i++) w[i] = 0;
#pragma unroll
      for (int k = 0; k < 32; k++) {
        const uint64_t v = (lane * 32 + k < nt) ? (uint64_t)p[k] : 0ull;
        constexpr int E = (int)sizeof(T);
        const int bit = (k * E * 8) & 31, word = (k * E * 8) >> 5;
        w[word] |= (uint32_t)v << bit;
        if (E == 8) w[word + 1] = (uint32_t)(v >> 32);
      }
    }
    uint32_t o[B];
    fold<T, B>(w, o);
    // lane l's words are tile words [l*B, l*B + B); through shared memory so
    // the warp stores 32 consecutive words per instruction
#pragma unroll
    for (int j = 0; j < B; j++) stage[sidx<B>(lane * B + j)] = o[j];
    __syncwarp();
    uint32_t* dst = base + s0 * B / 32;                 // s0*B is a multiple of 32
    if (off == 0 && nt == kTile) {
#pragma unroll
      for (int r = 0; r < B; r++) dst[32 * r + lane] = stage[sidx<B>(32 * r + lane)];
    } else {
      // shifted by out_bit0 % 32 and/or partial: words shared with the
      // neighbouring tiles or with bits outside the range merge atomically
      const int64_t tbits = nt * B;
      const int nw = (int)((off + tbits + 31) >> 5);
      for (int g = lane; g < nw; g += 32) {
        const uint32_t cur = g < 32 * B ? stage[sidx<B>(g)] : 0u;
        uint32_t val = cur;
        if (off) {
          const uint32_t prev = g ? stage[sidx<B>(g - 1)] : 0u;
          val = (cur << off) | (prev >> (32 - off));
        }
        const int lo = g == 0 ? off : 0;
        const int64_t hi64 = off + tbits - 32 * (int64_t)g;
        const int hi = hi64 > 32 ? 32 : (int)hi64;
        if (lo == 0 && hi == 32) {
          dst[g] = val;
        } else {
          const uint32_t mask = (hi == 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u)) & (0xFFFFFFFFu << lo);
          atomicAnd(&dst[g], ~mask);
          atomicOr(&dst[g], val & mask);
        }
      }
    }
    __syncwarp();
  }
}

// Any element type / alignment: one thread per output word gathers the
// samples overlapping it.
template <typename T>
__global__ void __launch_bounds__(256) pack_generic_kernel(const T* __restrict__ s, int b,
                                                           int64_t count, uint32_t* __restrict__ out,
                                                           int64_t out_bit0, int64_t nwords) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nwords) return;
  const int64_t gw = (out_bit0 >> 5) + i;
  const int64_t lo = gw * 32;             // absolute stream bit of word start
  const int64_t begin = out_bit0, end = out_bit0 + count * (int64_t)b;
  const int64_t r0 = lo - begin;          // relative bit of word start
  int64_t k0 = r0 > 0 ? r0 / b : 0;
  int64_t k1 = (r0 + 31) / b;
  if (k1 > count - 1) k1 = count - 1;
  const uint64_t vmask = b >= 64 ? ~0ull : ((1ull << b) - 1ull);
  uint32_t word = 0;
  for (int64_t k = k0; k <= k1; k++) {
    const uint64_t v = (uint64_t)s[k] & vmask;
    const int64_t p = k * b - r0;         // sample position relative to word start
    uint64_t part;
    if (p >= 0) part = p >= 64 ? 0ull : (v << p);
    else part = -p >= 64 ? 0ull : (v >> -p);
    word |= (uint32_t)part;
  }
  const int64_t s_ = lo > begin ? lo : begin;
  const int64_t e_ = lo + 32 < end ? lo + 32 : end;
  if (s_ == lo && e_ == lo + 32) {
    out[gw] = word;
  } else {
    const int nbits = (int)(e_ - s_), off = (int)(s_ - lo);
    const uint32_t mask = (nbits >= 32 ? 0xFFFFFFFFu : ((1u << nbits) - 1u)) << off;
    atomicAnd(&out[gw], ~mask);
    atomicOr(&out[gw], word & mask);
  }
}

template <typename T, int B>
cudaError_t launch_tile(const T* s, int64_t count, uint32_t* out, int64_t out_bit0,
                        cudaStream_t st) {
  constexpr int W = pack_warps<T>();
  const int64_t ntiles = (count + kTile - 1) / kTile;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pack_tile_kernel<T, B>, 32 * W, 0);
  if (per_sm < 1) per_sm = 1;
  const int64_t want = (ntiles + W - 1) / W;
  const int64_t cap = (int64_t)sms * per_sm;
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  pack_tile_kernel<T, B><<<grid, 32 * W, 0, st>>>(s, count, out, out_bit0);
  return cudaGetLastError();
}

using TileFn = cudaError_t (*)(const void*, int64_t, uint32_t*, int64_t, cudaStream_t);

template <typename T, int B>
cudaError_t tile_entry(const void* s, int64_t count, uint32_t* out, int64_t out_bit0,
                       cudaStream_t st) {
  return launch_tile<T, B>(static_cast<const T*>(s), count, out, out_bit0, st);
}

// B in (4*sizeof(T), 8*sizeof(T)) -- T is the narrowest type holding B bits
// -- plus B < 8 for uint16 (the device Markov chain emits int16 states).
template <typename T, int LO, int... Is>
constexpr auto tile_table(std::integer_sequence<int, Is...>) {
  return std::array<TileFn, sizeof...(Is)>{{&tile_entry<T, LO + Is>...}};
}

}  // namespace


// entry for (elem_bytes, b) with a fast tile kernel, else nullptr
static TileFn tile_fn(int elem, int b) {
  static const auto t8 = tile_table<uint8_t, 1>(std::make_integer_sequence<int, 7>{});     // 1..7
  static const auto t16 = tile_table<uint16_t, 1>(std::make_integer_sequence<int, 15>{});  // 1..15
  static const auto t32 = tile_table<uint32_t, 17>(std::make_integer_sequence<int, 15>{}); // 17..31
  static const auto t64 = tile_table<uint64_t, 33>(std::make_integer_sequence<int, 31>{}); // 33..63
  switch (elem) {
    case 1: return b >= 1 && b <= 7 ? t8[b - 1] : nullptr;
    case 2: return b >= 1 && b <= 15 ? t16[b - 1] : nullptr;
    case 4: return b >= 17 && b <= 31 ? t32[b - 17] : nullptr;
    case 8: return b >= 33 && b <= 63 ? t64[b - 33] : nullptr;
    default: return nullptr;
  }
}

// *kernel_launched = 0 when the call was served by a copy (or had no work).
cudaError_t launch_pack(const void* samples, int elem_bytes, int b, int64_t count, void* out,
                        int64_t out_bit0, cudaStream_t st, int* kernel_launched) {
  *kernel_launched = 0;
  const int64_t end = out_bit0 + count * (int64_t)b;
  const int64_t nwords = ((end + 31) >> 5) - (out_bit0 >> 5);
  if (nwords <= 0) return cudaSuccess;
  uint32_t* o = static_cast<uint32_t*>(out);
  if (b == 8 * elem_bytes && (out_bit0 & 7) == 0) {
    // full-width samples: the packed stream is the sample array itself
    return cudaMemcpyAsync(static_cast<uint8_t*>(out) + (out_bit0 >> 3), samples,
                           (size_t)count * elem_bytes, cudaMemcpyDeviceToDevice, st);
  }
  *kernel_launched = 1;
  if (((uintptr_t)samples & 31) == 0) {
    if (TileFn f = tile_fn(elem_bytes, b)) return f(samples, count, o, out_bit0, st);
  }
  const unsigned grid = (unsigned)((nwords + 255) / 256);
  switch (elem_bytes) {
    case 1: pack_generic_kernel<uint8_t><<<grid, 256, 0, st>>>((const uint8_t*)samples, b, count, o, out_bit0, nwords); break;
    case 2: pack_generic_kernel<uint16_t><<<grid, 256, 0, st>>>((const uint16_t*)samples, b, count, o, out_bit0, nwords); break;
    case 4: pack_generic_kernel<uint32_t><<<grid, 256, 0, st>>>((const uint32_t*)samples, b, count, o, out_bit0, nwords); break;
    default: pack_generic_kernel<uint64_t><<<grid, 256, 0, st>>>((const uint64_t*)samples, b, count, o, out_bit0, nwords); break;
  }
  return cudaGetLastError();
}

}  // namespace bx
