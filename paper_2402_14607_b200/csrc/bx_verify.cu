// bx_verify.cu -- exhaustive small-instance kernels for the verification
// suites (reference pkg/src/blockext/verify.py).
//
// Instances have t = q*n <= 16 input bits per source, so every vector fits a
// 32-bit word and an inner product <x, y> = sum_j x_j * y_j over GF(2^q)
// (reference extractor.py:77-87) is evaluated per thread: carry-less products
// accumulated unreduced (degree <= 2q-2 < 32) and one reduction by the
// modulus's low part (fold per set high bit, reference gf2q.py:156-169).
//
//  * ip_table_kernel:   z[x][y] = <x, y> for x in [x0, x0+nx), all y
//                       (reference ip_value_table, verify.py:200-207)
//  * ip_hist_kernel:    counts[d][v] = #{y : <d, y> = v} for d in [d0, d0+nd)
//                       (the histograms of _hadamard_counts, verify.py:262-297)
//  * rows_uniform:      flag[d] = all counts[d][.] == expected
#include <cstdint>
#include <cuda_runtime.h>

#include "bx_core.cuh"

namespace bx {

struct SmallField {
  int q;
  uint32_t mask;
  uint32_t low;  // modulus without x^q
};

__device__ __forceinline__ uint32_t clmul_small(uint32_t a, uint32_t b) {
  uint32_t r = 0;
  while (a) {
    const int i = __ffs(a) - 1;
    r ^= b << i;
    a &= a - 1;
  }
  return r;
}

__device__ __forceinline__ uint32_t reduce_small(const SmallField& f, uint32_t c) {
  // c has degree <= 2q-2; fold the high part bit by bit from the top
  for (int i = 2 * f.q - 2; i >= f.q; i--) {
    if ((c >> i) & 1u) c ^= (1u << i) ^ (f.low << (i - f.q));
  }
  return c & f.mask;
}

__device__ __forceinline__ uint32_t ip_small(const SmallField& f, int n, uint32_t x, uint32_t y) {
  uint32_t c = 0;
  for (int j = 0; j < n; j++) {
    const uint32_t xj = (x >> (j * f.q)) & f.mask, yj = (y >> (j * f.q)) & f.mask;
    c ^= clmul_small(xj, yj);
  }
  return reduce_small(f, c);
}

__global__ void ip_table_kernel(SmallField f, int n, uint32_t x0, uint32_t nx, uint16_t* out) {
  const int t = f.q * n;
  const uint64_t ny = 1ull << t;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (uint64_t)nx * ny) return;
  const uint32_t x = x0 + (uint32_t)(i >> t), y = (uint32_t)(i & (ny - 1));
  out[i] = (uint16_t)ip_small(f, n, x, y);
}

// One CTA per d; y strided over the CTA; histogram in shared memory when 2^q
// bins fit, else global atomics on this d's row.
__global__ void ip_hist_kernel(SmallField f, int n, uint32_t d0, uint32_t* counts) {
  extern __shared__ uint32_t hist[];
  const int t = f.q * n;
  const uint32_t d = d0 + blockIdx.x;
  const uint32_t bins = 1u << f.q;
  const bool in_smem = bins <= 8192;
  uint32_t* row = counts + (uint64_t)blockIdx.x * bins;
  if (in_smem) {
    for (uint32_t v = threadIdx.x; v < bins; v += blockDim.x) hist[v] = 0;
    __syncthreads();
  }
  for (uint32_t y = threadIdx.x; y < (1u << t); y += blockDim.x) {
    const uint32_t v = ip_small(f, n, d, y);
    atomicAdd(in_smem ? &hist[v] : &row[v], 1u);
  }
  if (in_smem) {
    __syncthreads();
    for (uint32_t v = threadIdx.x; v < bins; v += blockDim.x) row[v] = hist[v];
  }
}

__global__ void rows_uniform_kernel(const uint32_t* counts, uint32_t nrows, uint32_t bins,
                                    uint32_t expected, uint8_t* flags) {
  const uint32_t r = blockIdx.x;
  if (r >= nrows) return;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (uint32_t v = threadIdx.x; v < bins; v += blockDim.x)
    if (counts[(uint64_t)r * bins + v] != expected) bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) flags[r] = bad ? 0 : 1;
}

cudaError_t launch_ip_table(int q, uint32_t low, int n, uint32_t x0, uint32_t nx, uint16_t* out,
                            cudaStream_t st) {
  SmallField f{q, (1u << q) - 1u, low};
  const uint64_t total = (uint64_t)nx << (q * n);
  ip_table_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(f, n, x0, nx, out);
  return cudaGetLastError();
}

cudaError_t launch_ip_hist(int q, uint32_t low, int n, uint32_t d0, uint32_t nd, uint32_t* counts,
                           cudaStream_t st) {
  SmallField f{q, (1u << q) - 1u, low};
  const uint32_t bins = 1u << q;
  if (bins > 8192) cudaMemsetAsync(counts, 0, (size_t)nd * bins * 4, st);
  const size_t smem = bins <= 8192 ? bins * 4 : 0;
  ip_hist_kernel<<<nd, 256, smem, st>>>(f, n, d0, counts);
  return cudaGetLastError();
}

cudaError_t launch_rows_uniform(const uint32_t* counts, uint32_t nrows, uint32_t bins,
                                uint32_t expected, uint8_t* flags, cudaStream_t st) {
  rows_uniform_kernel<<<nrows, 256, 0, st>>>(counts, nrows, bins, expected, flags);
  return cudaGetLastError();
}

}  // namespace bx

// ---------------------------------------------------------------------------
// Runtime-modulus field arithmetic (GFContext with a caller-chosen irreducible
// modulus, reference gf2q.py:99-189 allows any; and pow / inv for every
// modulus).  Not the extraction path: one thread per vector or element,
// 128-bit operands, carry-less products with the holes kernel (Holes<128>),
// reduction through a per-CTA fold table of the modulus.
namespace bx {

// Fold table of a runtime modulus: R[i] = x^(q+i) mod P for i in [0, q)
// (reference gf2q.py:124-133), 4 words per entry, built once per CTA.
__device__ void fold_table128(int q, const uint32_t (&m)[4], uint32_t (*R)[4]) {
  uint32_t t[4] = {m[0], m[1], m[2], m[3]};   // x^q mod P = P - x^q
  for (int i = 0; i < q; i++) {
#pragma unroll
    for (int w = 0; w < 4; w++) R[i][w] = t[w];
    // t <<= 1; if bit q set: t ^= x^q + m (clears bit q, adds the low part)
    const uint32_t top = (t[(q - 1) >> 5] >> ((q - 1) & 31)) & 1u;
    t[3] = (t[3] << 1) | (t[2] >> 31);
    t[2] = (t[2] << 1) | (t[1] >> 31);
    t[1] = (t[1] << 1) | (t[0] >> 31);
    t[0] <<= 1;
    if (q < 128) t[q >> 5] &= ~(1u << (q & 31));
    if (top) {
#pragma unroll
      for (int w = 0; w < 4; w++) t[w] ^= m[w];
    }
  }
}

__device__ __forceinline__ void reduce_runtime(int q, const uint32_t (*R)[4], const Wide<8>& c,
                                               uint32_t (&r)[4]);

// r = a * b mod P for q-bit a, b: the 255-bit carry-less product with the
// holes kernel (Holes<128>: Karatsuba over 16-bit halves, IMAD products),
// then the high part folded with R.  All register-resident; the bit scan of
// the high part is unrolled over static word/bit positions.
__device__ __forceinline__ void mulmod128(int q, const uint32_t (*R)[4], const uint32_t (&a)[4],
                                          const uint32_t (&b)[4], uint32_t (&r)[4]) {
  Holes<128> h;
  h.init();
  h.add(a, b);
  reduce_runtime(q, R, h.unreduced(), r);
}

// z = c mod P (runtime modulus through the fold table R)
__device__ __forceinline__ void reduce_runtime(int q, const uint32_t (*R)[4], const Wide<8>& c,
                                               uint32_t (&r)[4]) {
  uint32_t z[4];
#pragma unroll
  for (int w = 0; w < 4; w++) {
    const int lo = 32 * w;
    uint32_t val = c.w[w];
    if (lo >= q) val = 0;
    else if (q - lo < 32) val &= (1u << (q - lo)) - 1u;
    z[w] = val;
  }
#pragma unroll
  for (int w = 0; w < 8; w++) {
    uint32_t word = c.w[w];
    // bits of this word at positions >= q
    const int lo = 32 * w;
    if (lo + 31 < q) continue;
    if (lo < q) word &= ~((q - lo) >= 32 ? 0xFFFFFFFFu : ((1u << (q - lo)) - 1u));
    while (word) {
      const int bit = __ffs(word) - 1;
      word &= word - 1u;
      const uint32_t* f = R[lo + bit - q];
#pragma unroll
      for (int k = 0; k < 4; k++) z[k] ^= f[k];
    }
  }
#pragma unroll
  for (int w = 0; w < 4; w++) r[w] = z[w];
}

// Inner products under a runtime modulus (GFContext(q, modulus).mul / ext_ip,
// reference gf2q.py:99-169): the unreduced products of a vector are summed
// with the holes kernel (Holes<128>) and reduced once with the CTA's fold
// table of the modulus.
__global__ void __launch_bounds__(128) gf_ip_generic_kernel(int q, const uint32_t* modulus,
                                                            const uint32_t* x, const uint32_t* y,
                                                            int n, int64_t nvec, uint32_t* out) {
  __shared__ uint32_t R[128][4];
  const uint32_t m[4] = {modulus[0], modulus[1], modulus[2], modulus[3]};
  if (threadIdx.x == 0) fold_table128(q, m, R);
  __syncthreads();
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nvec) return;
  Holes<128> h;
  h.init();
  for (int j = 0; j < n; j++) {
    const uint4 a = reinterpret_cast<const uint4*>(x)[v * n + j];
    const uint4 b = reinterpret_cast<const uint4*>(y)[v * n + j];
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
    h.add(aw, bw);
  }
  uint32_t z[4];
  reduce_runtime(q, R, h.unreduced(), z);
#pragma unroll
  for (int w = 0; w < 4; w++) out[v * 4 + w] = z[w];
}

// out[v] = x[v]^e[v] by square-and-multiply over the exponent's bits, LSB
// first (the reference GFContext.pow loop, gf2q.py:171-182), one thread per
// element; 128-bit little-endian operands.
__global__ void __launch_bounds__(128) gf_pow_kernel(int q, const uint32_t* modulus,
                                                     const uint32_t* x, const uint32_t* e,
                                                     int64_t count, uint32_t* out) {
  __shared__ uint32_t R[128][4];
  const uint32_t m[4] = {modulus[0], modulus[1], modulus[2], modulus[3]};
  if (threadIdx.x == 0) fold_table128(q, m, R);
  __syncthreads();
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= count) return;
  uint32_t b[4] = {x[v * 4], x[v * 4 + 1], x[v * 4 + 2], x[v * 4 + 3]};
  uint32_t r[4] = {1u, 0u, 0u, 0u};
  const uint32_t ew[4] = {e[v * 4], e[v * 4 + 1], e[v * 4 + 2], e[v * 4 + 3]};
  int top = -1;
#pragma unroll
  for (int w = 3; w >= 0; w--)
    if (top < 0 && ew[w]) top = 32 * w + 31 - __clz(ew[w]);
  for (int i = 0; i <= top; i++) {
    uint32_t t[4];
    if ((ew[i >> 5] >> (i & 31)) & 1u) {
      mulmod128(q, R, r, b, t);
#pragma unroll
      for (int w = 0; w < 4; w++) r[w] = t[w];
    }
    if (i < top) {
      mulmod128(q, R, b, b, t);
#pragma unroll
      for (int w = 0; w < 4; w++) b[w] = t[w];
    }
  }
#pragma unroll
  for (int w = 0; w < 4; w++) out[v * 4 + w] = r[w];
}

cudaError_t launch_gf_pow(int q, const uint32_t* modulus, const uint32_t* x, const uint32_t* e,
                          int64_t count, uint32_t* out, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  gf_pow_kernel<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(q, modulus, x, e, count, out);
  return cudaGetLastError();
}

cudaError_t launch_gf_ip_generic(int q, const uint32_t* modulus, const uint32_t* x, const uint32_t* y,
                                 int n, int64_t nvec, uint32_t* out, cudaStream_t st) {
  if (nvec <= 0) return cudaSuccess;
  gf_ip_generic_kernel<<<(unsigned)((nvec + 127) / 128), 128, 0, st>>>(q, modulus, x, y, n, nvec, out);
  return cudaGetLastError();
}

}  // namespace bx
