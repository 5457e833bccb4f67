// bx_pack.cu -- raw-sample packer (reference sources._pack_samples,
// pkg/src/blockext/sources.py:116-121): the low b bits of sample i become
// stream bits [out_bit0 + i*b, out_bit0 + (i+1)*b), LSB-first.
//
// One thread per output 32-bit word gathers the (at most 32/b + 2) samples
// overlapping it; full words are stored, the (<= 2) boundary words are merged
// with atomicAnd/atomicOr so bits outside the range survive.
#include <cstdint>
#include <cuda_runtime.h>

namespace bx {

template <typename T>
__global__ void __launch_bounds__(256) pack_kernel(const T* __restrict__ s, int b, int64_t count,
                                                   uint32_t* __restrict__ out, int64_t out_bit0,
                                                   int64_t nwords) {
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

cudaError_t launch_pack(const void* samples, int elem_bytes, int b, int64_t count, void* out,
                        int64_t out_bit0, cudaStream_t st) {
  const int64_t end = out_bit0 + count * (int64_t)b;
  const int64_t nwords = ((end + 31) >> 5) - (out_bit0 >> 5);
  if (nwords <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)((nwords + 255) / 256);
  uint32_t* o = static_cast<uint32_t*>(out);
  switch (elem_bytes) {
    case 1: pack_kernel<uint8_t><<<grid, 256, 0, st>>>((const uint8_t*)samples, b, count, o, out_bit0, nwords); break;
    case 2: pack_kernel<uint16_t><<<grid, 256, 0, st>>>((const uint16_t*)samples, b, count, o, out_bit0, nwords); break;
    case 4: pack_kernel<uint32_t><<<grid, 256, 0, st>>>((const uint32_t*)samples, b, count, o, out_bit0, nwords); break;
    default: pack_kernel<uint64_t><<<grid, 256, 0, st>>>((const uint64_t*)samples, b, count, o, out_bit0, nwords); break;
  }
  return cudaGetLastError();
}

}  // namespace bx
