// bx_wide.cu -- GF(2^256) block inner products: config 3 as BASELINE states it
// (1024-bit blocks, m = 256 output bits per block).  The reference caps fields
// at q = 128 (gf2q.py:20, 111-112: CapacityError), so this is an opt-in
// extension beyond the drop-in API (paper_2402_14607_b200.wide), built from the
// same pieces as the q <= 128 kernels:
//
//   z_l = reduce_P256( XOR_j x_lj * y_lj ),  P256 = x^256 + x^10 + x^5 + x^2 + 1
//
// (the first irreducible of the reference modulus scan, _moduli.py:1-11 /
// tools/gen_moduli.py, extended to q = 256).  One thread per block.  The
// 256x256 carry-less products are split with two Karatsuba levels taken
// OUTSIDE the element loop: 128-bit halves (L, H, M = lo^hi) and, inside each,
// 64-bit halves -- nine passes over the block, each accumulating one 64x64
// sub-product over all elements with the holes IMAD kernel (Holes<64>: nine
// 16-bit leaves, 27 accumulators).  Sums over j commute with the linear
// Karatsuba recombination, so each pass's unreduced 127-bit sum is XORed
// straight into the 511-bit result at its combined offset; one reduction per
// block.  Passes 2..9 re-read the block's 2 x 32n bytes from L1.
#include <cstdint>

#include <cuda_runtime.h>

#include "bx_core.cuh"

namespace bx {

namespace {

// 64-bit operand of pass (A, B) from one 256-bit element w[0..7]:
// A selects the 128-bit half (0 lo, 1 hi, 2 lo^hi), B the 64-bit half of it.
template <int A, int B>
__device__ __forceinline__ void wide_part(const uint4& u0, const uint4& u1, uint32_t (&o)[2]) {
  uint32_t h[4];
  if constexpr (A == 0) {
    h[0] = u0.x; h[1] = u0.y; h[2] = u0.z; h[3] = u0.w;
  } else if constexpr (A == 1) {
    h[0] = u1.x; h[1] = u1.y; h[2] = u1.z; h[3] = u1.w;
  } else {
    h[0] = u0.x ^ u1.x; h[1] = u0.y ^ u1.y; h[2] = u0.z ^ u1.z; h[3] = u0.w ^ u1.w;
  }
  if constexpr (B == 0) {
    o[0] = h[0]; o[1] = h[1];
  } else if constexpr (B == 1) {
    o[0] = h[2]; o[1] = h[3];
  } else {
    o[0] = h[0] ^ h[2]; o[1] = h[1] ^ h[3];
  }
}

// Karatsuba placement of a sub-product: L at 0 and h, H at 2h and h, M at h
// (h = half width), as XOR-sets of word offsets for 64-bit (2-word) and
// 128-bit (4-word) halves.
template <int B>
constexpr int offs64() { return B == 0 ? 0b011 : (B == 1 ? 0b110 : 0b010); }   // bits: 0, 2, 4 words
template <int A>
constexpr int offs128() { return A == 0 ? 0b011 : (A == 1 ? 0b110 : 0b010); }  // bits: 0, 4, 8 words

template <int A, int B>
__device__ __forceinline__ void wide_pass(const uint4* xp, const uint4* yp, int n, uint32_t (&c)[16]) {
  Holes<64> acc;
  acc.init();
  int j = 0;
#pragma unroll 1
  for (; j + 1 < n; j += 2) {
    uint32_t a[2], b[2], a2[2], b2[2];
    wide_part<A, B>(__ldg(xp + 2 * j), __ldg(xp + 2 * j + 1), a);
    wide_part<A, B>(__ldg(yp + 2 * j), __ldg(yp + 2 * j + 1), b);
    wide_part<A, B>(__ldg(xp + 2 * j + 2), __ldg(xp + 2 * j + 3), a2);
    wide_part<A, B>(__ldg(yp + 2 * j + 2), __ldg(yp + 2 * j + 3), b2);
    acc.add2(a, b, a2, b2);
  }
  if (j < n) {
    uint32_t a[2], b[2];
    wide_part<A, B>(__ldg(xp + 2 * j), __ldg(xp + 2 * j + 1), a);
    wide_part<A, B>(__ldg(yp + 2 * j), __ldg(yp + 2 * j + 1), b);
    acc.add(a, b);
  }
  const Wide<4> p = acc.unreduced();   // 127-bit sum of 64x64 products
#pragma unroll
  for (int s128 = 0; s128 < 3; s128++) {
    if (!((offs128<A>() >> s128) & 1)) continue;
#pragma unroll
    for (int s64 = 0; s64 < 3; s64++) {
      if (!((offs64<B>() >> s64) & 1)) continue;
      const int w0 = 4 * s128 + 2 * s64;
#pragma unroll
      for (int i = 0; i < 4; i++)
        if (w0 + i < 16) c[w0 + i] ^= p.w[i];
    }
  }
}

// c (511 bits) mod x^256 + x^10 + x^5 + x^2 + 1 -> z (256 bits)
__device__ __forceinline__ void reduce256(const uint32_t (&c)[16], uint32_t (&z)[8]) {
  uint32_t h[9];   // high part c >> 256 (255 bits), then the overflow of one fold
#pragma unroll
  for (int i = 0; i < 8; i++) {
    z[i] = c[i];
    h[i] = c[8 + i];
  }
  h[8] = 0;
  // z ^= h * (1 + x^2 + x^5 + x^10); the shifted copies spill up to 10 bits
  // past bit 256: collect them and fold once more (degree <= 9 + 10 < 256)
  constexpr int kS[4] = {0, 2, 5, 10};
  uint32_t spill = 0;
#pragma unroll
  for (int t = 0; t < 4; t++) {
    const int s = kS[t];
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const uint32_t lo = h[i] << s | (i > 0 && s ? h[i - 1] >> (32 - s) : 0u);
      z[i] ^= s ? lo : h[i];
    }
    if (s) spill ^= h[7] >> (32 - s);
  }
#pragma unroll
  for (int t = 0; t < 4; t++) z[0] ^= spill << kS[t];
  // spill < 2^10, so spill << 10 < 2^20: no further overflow
}

#ifndef BX_WIDE_MINB
#define BX_WIDE_MINB 1
#endif

__global__ void __launch_bounds__(128, BX_WIDE_MINB) eq_wide256_kernel(const uint4* __restrict__ x,
                                                         const uint4* __restrict__ y, int n,
                                                         int64_t nblocks, uint32_t* __restrict__ out) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nblocks) return;
  const uint4* xp = x + l * 2 * n;   // 32 bytes = 2 units per element
  const uint4* yp = y + l * 2 * n;
  uint32_t c[16];
#pragma unroll
  for (int i = 0; i < 16; i++) c[i] = 0u;
  wide_pass<0, 0>(xp, yp, n, c);
  wide_pass<0, 1>(xp, yp, n, c);
  wide_pass<0, 2>(xp, yp, n, c);
  wide_pass<1, 0>(xp, yp, n, c);
  wide_pass<1, 1>(xp, yp, n, c);
  wide_pass<1, 2>(xp, yp, n, c);
  wide_pass<2, 0>(xp, yp, n, c);
  wide_pass<2, 1>(xp, yp, n, c);
  wide_pass<2, 2>(xp, yp, n, c);
  uint32_t z[8];
  reduce256(c, z);
  uint4* o = reinterpret_cast<uint4*>(out + l * 8);
  o[0] = make_uint4(z[0], z[1], z[2], z[3]);
  o[1] = make_uint4(z[4], z[5], z[6], z[7]);
}

}  // namespace

cudaError_t launch_wide256(const void* x, const void* y, int n, int64_t nblocks, void* out,
                           cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  const int64_t grid = (nblocks + 127) / 128;
  eq_wide256_kernel<<<(unsigned)grid, 128, 0, st>>>(static_cast<const uint4*>(x),
                                                    static_cast<const uint4*>(y), n, nblocks,
                                                    static_cast<uint32_t*>(out));
  return cudaGetLastError();
}

}  // namespace bx
