// bx_core.cuh -- GF(2^q) block inner-product kernels for sm_100a.
//
// One block l of an equal-width run reads q*n bits of each stream,
// x_l = bits [x_bit0 + l*q*n, ...), y_l likewise, splits them into n q-bit
// elements LSB-first (reference extractor.py:182-208, bitio.py:45-60) and emits
//
//     z_l = reduce_P( XOR_j clmul(x_lj, y_lj) )                       (*)
//
// at output bits [out_bit0 + l*q, ...) (reference bitio.py:74-88).  (*) equals
// the reference's XOR of reduced products (extractor.py:77-87 with
// gf2q.py:156-169) because reduction mod P is GF(2)-linear; the carry-less
// products are therefore accumulated UNREDUCED over the block and reduced once.
//
// There is no carry-less multiply instruction on the GPU.  Three integer-pipe
// formulations are used, chosen at compile time by Q:
//
//  * Diag (Q <= 8): a 32-bit chunk holds E = 32/Q elements.  For every shift
//    d in [0, Q): acc_d ^= (X & (Y << d)) ^ ((X << d) & Y).  Bit jQ+p of acc_d
//    (p >= d) holds the two products x_{j,a} y_{j,b} with a + b = 2p - d and
//    |a - b| = d; at the end
//        c_k = XOR over elements and d of bit (k+d)/2 of acc_d,
//    formed by a fold over elements and a bit spread (Q = 4, 8) or masked
//    parities.  Cost: 2Q-1 LOP3 (ALU) + 2Q-2 left shifts (IMAD.SHL, FMA pipe)
//    per chunk.
//
//  * Holes (Q >= 9): elements are cut into 16-bit halves; a 16x16 carry-less
//    product is formed with nine 32-bit IMADs on "holed" operands
//    (bits = i mod 3 of each half).  In each integer product all set
//    coefficients sit at positions = (i+k) mod 3 and each coefficient count is
//    <= 6 < 8, so no carry reaches the next same-residue position: bit p of the
//    product is the parity of the count, i.e. the carry-less coefficient.
//    Halves are combined with Karatsuba (K(8) = 27 half products for q=128
//    instead of 64); leaf products are XOR-accumulated per residue over the
//    whole block and recombined and masked once per block.
//    IMAD.WIDE is avoided: it issues at 1/3 the rate of IMAD on sm_100a
//    (profiles/r01_pipes_microbench.txt).
//
//  * Dot (Q >= 9, up to four halves; the q = 16 / 32 direct kernels, the tile
//    and period kernels up to q = 64): the same holes with IDP.2A, a two-term
//    16x8 dot product at IMAD's rate -- two elements' halves per operand, one
//    LOP3 masking two halves or four bytes (see "dot-product holes" below).
//    Same product count, about a quarter fewer ALU operations.
//
// Reduction mod P uses the shipped sparse modulus (bx_moduli.h) with all shift
// amounts compile-time constants.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "bx_moduli.h"

namespace bx {

// ---------------------------------------------------------- checked builds
// With -DBX_CHECKED (libbx_b200_checked.so) every shared / global index is
// compared with its bound and violations are counted in g_violations (the
// first one's tag and index are kept) instead of trapping, so a bad access is
// reported without faulting the GPU.  Normal builds compile the checks away.
#ifdef BX_CHECKED
extern __device__ unsigned long long g_violations;
extern __device__ long long g_first_violation[3];
__device__ __noinline__ inline void violation(int tag, long long idx, long long bound) {
  if (atomicAdd(&g_violations, 1ull) == 0ull) {
    g_first_violation[0] = tag;
    g_first_violation[1] = idx;
    g_first_violation[2] = bound;
  }
}
#define BX_CHECK(idx, bound, tag)                                              \
  do {                                                                          \
    const long long bx_i_ = (long long)(idx), bx_b_ = (long long)(bound);       \
    if (bx_i_ < 0 || bx_i_ >= bx_b_) ::bx::violation((tag), bx_i_, bx_b_);      \
  } while (0)
#else
#define BX_CHECK(idx, bound, tag) \
  do {                            \
  } while (0)
#endif

constexpr int kDiagMaxQ = 8;

__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }

// ----------------------------------------------------------- multiword values

template <int N>
struct Wide {
  uint32_t w[N];
};

template <int N>
__device__ __forceinline__ uint32_t at(const Wide<N>& a, int i) {
  return (i >= 0 && i < N) ? a.w[i] : 0u;
}

template <int N>
__device__ __forceinline__ Wide<N> wzero() {
  Wide<N> r;
#pragma unroll
  for (int i = 0; i < N; i++) r.w[i] = 0u;
  return r;
}

// r = a >> S, truncated to M words
template <int S, int M, int N>
__device__ __forceinline__ Wide<M> wshr(const Wide<N>& a) {
  Wide<M> r;
  constexpr int ws = S / 32, bs = S % 32;
#pragma unroll
  for (int i = 0; i < M; i++) {
    const uint32_t lo = at(a, i + ws), hi = at(a, i + ws + 1);
    r.w[i] = bs ? __funnelshift_r(lo, hi, bs) : lo;
  }
  return r;
}

// r ^= a << S (r has M words, bits shifted past M words are dropped)
template <int S, int M, int N>
__device__ __forceinline__ void wxor_shl(Wide<M>& r, const Wide<N>& a) {
  constexpr int ws = S / 32, bs = S % 32;
#pragma unroll
  for (int i = 0; i < M; i++) {
    const uint32_t hi = at(a, i - ws), lo = at(a, i - ws - 1);
    r.w[i] ^= bs ? __funnelshift_l(lo, hi, bs) : hi;
  }
}

// low Q bits of a, as cdiv(Q,32) words
template <int Q, int N>
__device__ __forceinline__ Wide<cdiv(Q, 32)> wlow(const Wide<N>& a) {
  constexpr int M = cdiv(Q, 32);
  Wide<M> r;
#pragma unroll
  for (int i = 0; i < M; i++) r.w[i] = at(a, i);
  if constexpr (Q % 32) r.w[M - 1] &= (1u << (Q % 32)) - 1u;
  return r;
}

// ------------------------------------------------------- reduction mod P(Q)

__host__ __device__ constexpr int fold_rounds(int q) {
  // c has degree <= 2q-2, so its high part (c >> q) has degree <= q-2.  One
  // fold maps a high part of degree d to one of degree d + e_max - q.
  int emax = 0;
  for (int i = 1; i < kModulus[q].count; i++)
    if (kModulus[q].e[i] > emax) emax = kModulus[q].e[i];
  int d = q - 2, f = 0;
  while (d >= 0) {
    d += emax - q;
    f++;
  }
  return f;
}

template <int Q, int I, int CW>
__device__ __forceinline__ void fold_terms(Wide<CW>& t, const Wide<CW>& hi) {
  if constexpr (I < kModulus[Q].count) {
    constexpr int e = kModulus[Q].e[I];
    if constexpr (e != Q) wxor_shl<e>(t, hi);
    fold_terms<Q, I + 1, CW>(t, hi);
  }
}

// z = c mod P, c of degree <= 2Q-2 held in CW words
template <int Q, int CW>
__device__ __forceinline__ Wide<cdiv(Q, 32)> reduce(const Wide<CW>& c) {
  Wide<cdiv(Q, 32)> lo = wlow<Q>(c);
  Wide<CW> hi = wshr<Q, CW>(c);
  constexpr int F = fold_rounds(Q);
#pragma unroll
  for (int f = 0; f < F; f++) {
    Wide<CW> t = wzero<CW>();
    fold_terms<Q, 0, CW>(t, hi);
    const Wide<cdiv(Q, 32)> tl = wlow<Q>(t);
#pragma unroll
    for (int i = 0; i < cdiv(Q, 32); i++) lo.w[i] ^= tl.w[i];
    hi = wshr<Q, CW>(t);
  }
  return lo;
}

// --------------------------------------------------------------- bit access

// 32 bits of an LSB-first word stream starting at bit `off` (word off>>5 + 1
// must be readable).  T: int64_t for global streams, uint32_t for shared-memory
// tiles (32-bit index math).
template <typename T>
__device__ __forceinline__ uint32_t read32(const uint32_t* src, T off, int64_t lim) {
  const T w = off >> 5;
  BX_CHECK(w + 1, lim, 1);
  return __funnelshift_r(src[w], src[w + 1], (uint32_t)(off & 31));
}

// ------------------------------------------------------------- diag (Q<=8)

// Merged diagonal accumulators (explicit LOP3s) for q = 4: c2 +3.5%, c5 n=256
// +5%; q = 8 loses 13% (two dependent LOP3s per accumulator and word), q = 2
// 1% -- profiles/r01_direct_sweep.txt R.  BX_DIAG_MERGED=0 turns it off.
#ifndef BX_DIAG_MERGED
#define BX_DIAG_MERGED 1
#endif

template <int Q>
struct Diag {
  static constexpr bool kMerged = BX_DIAG_MERGED && Q == 4;
  static constexpr int E = 32 / Q;   // elements per 32-bit chunk
  static constexpr int EB = E * Q;   // bits per chunk
  // acc(d) is the sum of the two diagonals at distance d:
  //   X & (Y << d)   bit jQ+p holds x_{j,p}   y_{j,p-d}
  //   (X << d) & Y   bit jQ+p holds x_{j,p-d} y_{j,p}
  // both valid for p >= d and both contributing to c_{2p-d}, so they share one
  // register.  Only left shifts, so the compiler issues them as IMAD.SHL on the
  // FMA pipe and the ALU pipe carries just the 2Q-1 LOP3s per chunk.
  // The two diagonals are kept in separate registers during the block (pos,
  // neg: one a ^ (b & c) LOP3 each; a merged register makes the compiler
  // build (X & Y<<d) ^ (X<<d & Y) trees, +25% LOP3) and merged at the end.
  uint32_t pos[Q];
  uint32_t neg[Q];

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int d = 0; d < Q; d++) pos[d] = neg[d] = 0u;
  }

  __device__ __forceinline__ void add(uint32_t X, uint32_t Y) {
    if constexpr (kMerged) {
      // one accumulator per d, updated by two explicit a ^ (b & c) LOP3s (ptxas
      // cannot re-associate inline lop3 into AND/XOR trees): the same 2Q-1 LOP3
      // per word pair, Q-1 fewer registers, no pos ^ neg merge per block
#pragma unroll
      for (int d = 0; d < Q; d++) {
        asm("lop3.b32 %0, %0, %1, %2, 0x78;" : "+r"(pos[d]) : "r"(X), "r"(Y << d));
        if (d) asm("lop3.b32 %0, %0, %1, %2, 0x78;" : "+r"(pos[d]) : "r"(X << d), "r"(Y));
      }
    } else {
#pragma unroll
      for (int d = 0; d < Q; d++) pos[d] ^= X & (Y << d);
#pragma unroll
      for (int d = 1; d < Q; d++) neg[d] ^= (X << d) & Y;
    }
  }

  __device__ __forceinline__ uint32_t acc(int d) const {
    if constexpr (kMerged) return pos[d];
    else return d ? pos[d] ^ neg[d] : pos[0];
  }

  static __host__ __device__ constexpr uint32_t mask_b(int b) {   // bit b of every element
    uint32_t m = 0;
    for (int j = 0; j < E; j++) m |= 1u << (j * Q + b);
    return m;
  }
  static __host__ __device__ constexpr uint32_t mask_ge(int d) {  // bits >= d of every element
    uint32_t m = 0;
    for (int b = d; b < Q; b++) m |= mask_b(b);
    return m;
  }

  // unreduced c (2Q-1 <= 15 bits), c_k = XOR over elements and d of the valid
  // bits p = (k+d)/2 of acc[d].
  __device__ __forceinline__ uint32_t unreduced() const {
    if constexpr (Q == 4 || Q == 8) {
      // Fold/spread form (~28 ops at Q=8 instead of ~Q^2 LOP3 + 2Q-1 POPC):
      // for d = 2e (2e+1) the valid bits shifted down by e go to A (B); bit p'
      // of the element-fold of A (B) then belongs at c_{2p'} (c_{2p'-1}), so
      // c = spread(fold A) ^ (spread(fold B) >> 1), spread: bit p -> bit 2p.
      // The right shift by e <= d only pulls in masked (zero) bits.
      uint32_t A = 0u, B = 0u;
#pragma unroll
      for (int d = 0; d < Q; d++) {
        const uint32_t t = (acc(d) >> (d >> 1)) & (mask_ge(d) >> (d >> 1));
        if (d & 1) B ^= t;
        else A ^= t;
      }
      A ^= A >> 16;                                  // 2 elements per 16-bit lane left
      B ^= B >> 16;
      uint32_t v = __byte_perm(A, B, 0x5410);        // A lane in bits 0-15, B lane in 16-31
      constexpr uint32_t lane = (1u << Q) - 1u;
#pragma unroll
      for (int s = 8; s > Q; s >>= 1) v ^= v >> s;
      v = (v ^ (v >> Q)) & (lane | (lane << 16));    // each lane: Q-bit fold at its bit 0
      if constexpr (Q == 8) v = (v | (v << 4)) & 0x0F0F0F0Fu;
      v = (v | (v << 2)) & 0x33333333u;
      v = (v | (v << 1)) & 0x55555555u;
      return (v & 0xFFFFu) ^ (v >> 17);
    } else {
      // c_k = parity(XOR_d acc[d] & M_{(k+d)/2}): one LOP3 per (k, d) pair and
      // one POPC per k
      uint32_t c = 0;
#pragma unroll
      for (int k = 0; k < 2 * Q - 1; k++) {
        uint32_t t = 0;
#pragma unroll
        for (int d = 0; d < Q; d++) {
          if ((k + d) & 1) continue;
          const int p = (k + d) >> 1;
          if (p < d || p >= Q) continue;
          t ^= acc(d) & mask_b(p);
        }
        c |= (uint32_t)(__popc(t) & 1) << k;
      }
      return c;
    }
  }
};

// ---------------------------------------------------------- holes (Q >= 9)

// A 16-bit half split into its three residue classes (bits = r mod 3).
struct Parts {
  uint32_t p[3];
};

__device__ __forceinline__ Parts split_lo(uint32_t w) {  // low half of w
  return Parts{{w & 0x9249u, w & 0x2492u, w & 0x4924u}};
}

#ifndef BX_SPLIT_IMAD
#define BX_SPLIT_IMAD 0
#endif
#if BX_SPLIT_IMAD
// -1 from the constant bank: ptxas cannot fold it, so h - p0 - p1 stays two
// IMADs on the FMA pipe instead of becoming an IADD3 on the ALU pipe
__constant__ uint32_t kMinusOne = 0xFFFFFFFFu;
#endif

// A 16-bit half with no bits above bit 15 (e.g. w >> 16): the third residue
// class is h - p0 - p1 (disjoint bits, no borrows), moved to the FMA pipe
// when BX_SPLIT_IMAD is set.
__device__ __forceinline__ Parts split_clean(uint32_t h) {
#if BX_SPLIT_IMAD
  const uint32_t p0 = h & 0x9249u, p1 = h & 0x2492u;
  uint32_t p2;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(p2) : "r"(p1), "r"(kMinusOne), "r"(h));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(p2) : "r"(p0), "r"(kMinusOne), "r"(p2));
  return Parts{{p0, p1, p2}};
#else
  return Parts{{h & 0x9249u, h & 0x2492u, h & 0x4924u}};
#endif
}

__device__ __forceinline__ Parts pxor(const Parts& a, const Parts& b) {
  return Parts{{a.p[0] ^ b.p[0], a.p[1] ^ b.p[1], a.p[2] ^ b.p[2]}};
}

// One 16x16 carry-less half product with nine 32-bit IMADs on holed operands,
// XOR-accumulated per residue class (see the header comment).
__device__ __forceinline__ void holes16(const Parts& x, const Parts& y, uint32_t (&acc)[3]) {
  acc[0] ^= (x.p[0] * y.p[0]) ^ (x.p[1] * y.p[2]) ^ (x.p[2] * y.p[1]);
  acc[1] ^= (x.p[0] * y.p[1]) ^ (x.p[1] * y.p[0]) ^ (x.p[2] * y.p[2]);
  acc[2] ^= (x.p[0] * y.p[2]) ^ (x.p[1] * y.p[1]) ^ (x.p[2] * y.p[0]);
}

// Two element pairs at once: 18 products into 3 accumulators with 3 three-input
// LOP3s per residue (instead of 4).
__device__ __forceinline__ void holes16x2(const Parts& xa, const Parts& ya, const Parts& xb,
                                          const Parts& yb, uint32_t (&acc)[3]) {
  acc[0] ^= (xa.p[0] * ya.p[0]) ^ (xa.p[1] * ya.p[2]) ^ (xa.p[2] * ya.p[1]) ^
            (xb.p[0] * yb.p[0]) ^ (xb.p[1] * yb.p[2]) ^ (xb.p[2] * yb.p[1]);
  acc[1] ^= (xa.p[0] * ya.p[1]) ^ (xa.p[1] * ya.p[0]) ^ (xa.p[2] * ya.p[2]) ^
            (xb.p[0] * yb.p[1]) ^ (xb.p[1] * yb.p[0]) ^ (xb.p[2] * yb.p[2]);
  acc[2] ^= (xa.p[0] * ya.p[2]) ^ (xa.p[1] * ya.p[1]) ^ (xa.p[2] * ya.p[0]) ^
            (xb.p[0] * yb.p[2]) ^ (xb.p[1] * yb.p[1]) ^ (xb.p[2] * yb.p[0]);
}

// Karatsuba over 16-bit halves.  A size-M operand pair splits into
// L = x_L*y_L, H = x_H*y_H and Mid = (x_L+x_H)(y_L+y_H); in GF(2)[t]
//     x*y = L (1 + t^h) + Mid t^h + H (t^h + t^2h),   t = x^16, h = ceil(M/2).
// Leaves are single half products; they are accumulated over the whole block
// (all j) and recombined once per block -- the sum over j commutes with the
// linear recombination, so Karatsuba's extra additions are paid per block,
// not per element.  Halves are split into residue classes once, and the
// Mid operands are formed by XOR on the split parts (masking commutes with
// XOR).  Leaves per size: K(1)=1, K(m)=2K(ceil(m/2))+K(floor(m/2))
// (K(2)=3, K(4)=9, K(8)=27 vs 4, 16, 64 half products for schoolbook).
__host__ __device__ constexpr int kara_leaves(int m) {
  return m <= 1 ? 1 : 2 * kara_leaves((m + 1) / 2) + kara_leaves(m / 2);
}

template <int M, int L0, int K>
__device__ __forceinline__ void kara_acc(const Parts* xo, const Parts* yo, uint32_t (&acc)[K][3]) {
  if constexpr (M == 1) {
    holes16(xo[0], yo[0], acc[L0]);
  } else {
    constexpr int h = (M + 1) / 2;
    kara_acc<h, L0, K>(xo, yo, acc);
    kara_acc<M - h, L0 + kara_leaves(h), K>(xo + h, yo + h, acc);
    Parts xm[h], ym[h];
#pragma unroll
    for (int i = 0; i < h; i++) {
      xm[i] = (i + h < M) ? pxor(xo[i], xo[i + h]) : xo[i];
      ym[i] = (i + h < M) ? pxor(yo[i], yo[i + h]) : yo[i];
    }
    kara_acc<h, L0 + kara_leaves(h) + kara_leaves(M - h), K>(xm, ym, acc);
  }
}

template <int M, int L0, int K>
__device__ __forceinline__ void kara_acc2(const Parts* xa, const Parts* ya, const Parts* xb,
                                          const Parts* yb, uint32_t (&acc)[K][3]) {
  if constexpr (M == 1) {
    holes16x2(xa[0], ya[0], xb[0], yb[0], acc[L0]);
  } else {
    constexpr int h = (M + 1) / 2;
    kara_acc2<h, L0, K>(xa, ya, xb, yb, acc);
    kara_acc2<M - h, L0 + kara_leaves(h), K>(xa + h, ya + h, xb + h, yb + h, acc);
    Parts xam[h], yam[h], xbm[h], ybm[h];
#pragma unroll
    for (int i = 0; i < h; i++) {
      xam[i] = (i + h < M) ? pxor(xa[i], xa[i + h]) : xa[i];
      yam[i] = (i + h < M) ? pxor(ya[i], ya[i + h]) : ya[i];
      xbm[i] = (i + h < M) ? pxor(xb[i], xb[i + h]) : xb[i];
      ybm[i] = (i + h < M) ? pxor(yb[i], yb[i + h]) : yb[i];
    }
    kara_acc2<h, L0 + kara_leaves(h) + kara_leaves(M - h), K>(xam, yam, xbm, ybm, acc);
  }
}

// Residue-class parts of every 16-bit half of a q-bit element held in EW words
// (one SHF per word for the high half, three LOP3 per half).
template <int NH, int EW>
__device__ __forceinline__ void split_halves(const uint32_t (&w)[EW], Parts (&o)[NH]) {
#pragma unroll
  for (int u = 0; u < NH; u++) o[u] = split_lo((u & 1) ? (w[u >> 1] >> 16) : w[u >> 1]);
}

template <int CW>
__device__ __forceinline__ void placed_xor(Wide<CW>& c, uint32_t cs, int s) {
  // c ^= cs << (16*s); s is a compile-time constant after unrolling
  const int w = (16 * s) >> 5;
  if ((s & 1) == 0) {
    if (w < CW) c.w[w] ^= cs;
  } else {
    if (w < CW) c.w[w] ^= cs << 16;
    if (w + 1 < CW) c.w[w + 1] ^= cs >> 16;
  }
}

// Recombine leaf values P into c; OFFS is the XOR-set of slot offsets (bit o =
// offset 16*o) at which the current node's product is added.
template <int M, int L0, uint32_t OFFS, int K, int CW>
__device__ __forceinline__ void kara_fin(const uint32_t (&P)[K], Wide<CW>& c) {
  if constexpr (M == 1) {
#pragma unroll
    for (int o = 0; o < 16; o++)
      if ((OFFS >> o) & 1u) placed_xor(c, P[L0], o);
  } else {
    constexpr int h = (M + 1) / 2;
    kara_fin<h, L0, OFFS ^ (OFFS << h), K, CW>(P, c);
    kara_fin<M - h, L0 + kara_leaves(h), (OFFS << h) ^ (OFFS << (2 * h)), K, CW>(P, c);
    kara_fin<h, L0 + kara_leaves(h) + kara_leaves(M - h), (OFFS << h), K, CW>(P, c);
  }
}

#ifndef BX_KPAIR_MAX_HALVES
#define BX_KPAIR_MAX_HALVES 6   // pair two elements per accumulate step up to this many halves
#endif

template <int Q>
struct Holes {
  static constexpr int EW = cdiv(Q, 32);       // 32-bit words per element
  static constexpr int NH = cdiv(Q, 16);       // 16-bit halves per element
  static constexpr int K = kara_leaves(NH);    // leaf half products per element
  static constexpr int CW = cdiv(2 * Q - 1, 32);
  // pairing two elements per accumulate step saves a LOP3 per residue but
  // doubles the live operand parts: +3-6% up to 6 halves (q <= 96; measured
  // profiles/r01_direct_sweep.txt H), none at 7-8 halves, where the register
  // cap is the limit (an uncapped 255-register q=128 variant was 13% slower).
  static constexpr bool kPair = NH <= BX_KPAIR_MAX_HALVES;
  uint32_t acc[K][3];

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int s = 0; s < K; s++) acc[s][0] = acc[s][1] = acc[s][2] = 0u;
  }

  __device__ __forceinline__ void add(const uint32_t (&xw)[EW], const uint32_t (&yw)[EW]) {
    Parts xo[NH], yo[NH];
    split_halves<NH>(xw, xo);
    split_halves<NH>(yw, yo);
    kara_acc<NH, 0, K>(xo, yo, acc);
  }

  // one 16-bit element per operand, both with no bits above bit 15
  __device__ __forceinline__ void add_clean(uint32_t x, uint32_t y) {
    static_assert(NH == 1, "add_clean is for q <= 16");
    holes16(split_clean(x), split_clean(y), acc[0]);
  }

  __device__ __forceinline__ void add2(const uint32_t (&xa)[EW], const uint32_t (&ya)[EW],
                                       const uint32_t (&xb)[EW], const uint32_t (&yb)[EW]) {
    Parts pxa[NH], pya[NH], pxb[NH], pyb[NH];
    split_halves<NH>(xa, pxa);
    split_halves<NH>(ya, pya);
    split_halves<NH>(xb, pxb);
    split_halves<NH>(yb, pyb);
    kara_acc2<NH, 0, K>(pxa, pya, pxb, pyb, acc);
  }

  __device__ __forceinline__ Wide<CW> unreduced() const {
    uint32_t P[K];
#pragma unroll
    for (int s = 0; s < K; s++)
      P[s] = (acc[s][0] & 0x49249249u) | (acc[s][1] & 0x92492492u) | (acc[s][2] & 0x24924924u);
    Wide<CW> c = wzero<CW>();
    kara_fin<NH, 0, 1u, K, CW>(P, c);
    return c;
  }
};

// ------------------------------------------ dot-product holes (IDP.2A, q >= 9)
//
// The same residue-class trick with sm_100a's full-rate 16x8 two-term dot
// product (dp2a -> IDP.2A, 64/clk/SM on the FMA pipe like IMAD, co-issues with
// LOP3: tools/microbench/idp.cu): a = [h1 : h0] holds the same 16-bit half of
// TWO consecutive elements, b = bytes [h1.b1, h0.b1, h1.b0, h0.b0] of the other
// operand's halves, and
//     dp2a.lo(a & MX_r, b & MY_s) = h0_r (x) h0.b0_s + h1_r (x) h1.b0_s
// (dp2a.hi the same with the high bytes).  A holed 16-bit half has <= 6 bits,
// a holed byte <= 3, so a coefficient counts <= 3 products per term and <= 6
// per instruction: still no carry into the next same-residue position.  One
// LOP3 now masks two halves (or four bytes) at once, and the high halves need
// no shift (one PRMT packs two elements): 11 instead of 20 ALU operations per
// q = 32 element pair in front of the same 27 FMA-pipe products, 3.5 instead
// of 7 at q = 16.  The high-byte products are accumulated apart and shifted by
// 8 once per block.
#ifndef BX_DP2A
#define BX_DP2A 1
#endif
// the tile / period kernels (any q >= 9) with the dot-product form
#ifndef BX_DP2A_TILE
#define BX_DP2A_TILE 1
#endif
// widest element (16-bit halves) the tile / period kernels take in the dot form:
// its K(NH) x 6 accumulators must fit the kernels' register caps
#ifndef BX_DOT_TILE_MAX_HALVES
#define BX_DOT_TILE_MAX_HALVES 4
#endif
#ifndef BX_DOT_QUAD_MAX_HALVES
#define BX_DOT_QUAD_MAX_HALVES 8
#endif

__device__ __forceinline__ Parts dsplit_x(uint32_t w) {   // two 16-bit halves
  return Parts{{w & 0x92499249u, w & 0x24922492u, w & 0x49244924u}};
}
__device__ __forceinline__ Parts dsplit_y(uint32_t w) {   // four bytes, in-byte residues
  return Parts{{w & 0x49494949u, w & 0x92929292u, w & 0x24242424u}};
}

struct DotAcc {
  uint32_t lo[3], hi[3];
};

// one packed pair (two elements' halves): 18 IDP.2A into 6 accumulators
__device__ __forceinline__ void dot16(const Parts& x, const Parts& y, DotAcc& A) {
#pragma unroll
  for (int c = 0; c < 3; c++) {
    uint32_t l = 0u, h = 0u;
#pragma unroll
    for (int r = 0; r < 3; r++) {
      const int s = (c + 3 - r) % 3;
      l ^= __dp2a_lo(x.p[r], y.p[s], 0u);
      h ^= __dp2a_hi(x.p[r], y.p[s], 0u);
    }
    A.lo[c] ^= l;
    A.hi[c] ^= h;
  }
}

// two packed pairs (four elements): 6 products + the accumulator = three
// 3-input LOP3 per accumulator instead of four
__device__ __forceinline__ void dot16x2(const Parts& xa, const Parts& ya, const Parts& xb,
                                        const Parts& yb, DotAcc& A) {
#pragma unroll
  for (int c = 0; c < 3; c++) {
    uint32_t l = 0u, h = 0u;
#pragma unroll
    for (int r = 0; r < 3; r++) {
      const int s = (c + 3 - r) % 3;
      l ^= __dp2a_lo(xa.p[r], ya.p[s], 0u) ^ __dp2a_lo(xb.p[r], yb.p[s], 0u);
      h ^= __dp2a_hi(xa.p[r], ya.p[s], 0u) ^ __dp2a_hi(xb.p[r], yb.p[s], 0u);
    }
    A.lo[c] ^= l;
    A.hi[c] ^= h;
  }
}

template <int M, int L0, int K>
__device__ __forceinline__ void dkara_acc(const Parts* xo, const Parts* yo, DotAcc (&acc)[K]) {
  if constexpr (M == 1) {
    dot16(xo[0], yo[0], acc[L0]);
  } else {
    constexpr int h = (M + 1) / 2;
    dkara_acc<h, L0, K>(xo, yo, acc);
    dkara_acc<M - h, L0 + kara_leaves(h), K>(xo + h, yo + h, acc);
    Parts xm[h], ym[h];
#pragma unroll
    for (int i = 0; i < h; i++) {
      xm[i] = (i + h < M) ? pxor(xo[i], xo[i + h]) : xo[i];
      ym[i] = (i + h < M) ? pxor(yo[i], yo[i + h]) : yo[i];
    }
    dkara_acc<h, L0 + kara_leaves(h) + kara_leaves(M - h), K>(xm, ym, acc);
  }
}

template <int M, int L0, int K>
__device__ __forceinline__ void dkara_acc2(const Parts* xa, const Parts* ya, const Parts* xb,
                                           const Parts* yb, DotAcc (&acc)[K]) {
  if constexpr (M == 1) {
    dot16x2(xa[0], ya[0], xb[0], yb[0], acc[L0]);
  } else {
    constexpr int h = (M + 1) / 2;
    dkara_acc2<h, L0, K>(xa, ya, xb, yb, acc);
    dkara_acc2<M - h, L0 + kara_leaves(h), K>(xa + h, ya + h, xb + h, yb + h, acc);
    Parts xam[h], yam[h], xbm[h], ybm[h];
#pragma unroll
    for (int i = 0; i < h; i++) {
      xam[i] = (i + h < M) ? pxor(xa[i], xa[i + h]) : xa[i];
      yam[i] = (i + h < M) ? pxor(ya[i], ya[i + h]) : ya[i];
      xbm[i] = (i + h < M) ? pxor(xb[i], xb[i + h]) : xb[i];
      ybm[i] = (i + h < M) ? pxor(yb[i], yb[i + h]) : yb[i];
    }
    dkara_acc2<h, L0 + kara_leaves(h) + kara_leaves(M - h), K>(xam, yam, xbm, ybm, acc);
  }
}

template <int Q>
struct Dot {
  static constexpr int EW = cdiv(Q, 32);
  static constexpr int NH = cdiv(Q, 16);
  static constexpr int K = kara_leaves(NH);
  static constexpr int CW = cdiv(2 * Q - 1, 32);
  DotAcc acc[K];

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int s = 0; s < K; s++)
#pragma unroll
      for (int c = 0; c < 3; c++) acc[s].lo[c] = acc[s].hi[c] = 0u;
  }

  // Residue parts of two elements a, b packed half by half: x side
  // [b.half_u : a.half_u], y side [b.half_u.b1, a.half_u.b1, b.half_u.b0, a.half_u.b0].
  static __device__ __forceinline__ void pack_x(const uint32_t (&a)[EW], const uint32_t (&b)[EW],
                                                Parts (&o)[NH]) {
#pragma unroll
    for (int u = 0; u < NH; u++)
      o[u] = dsplit_x(__byte_perm(a[u >> 1], b[u >> 1], (u & 1) ? 0x7632u : 0x5410u));
  }
  static __device__ __forceinline__ void pack_y(const uint32_t (&a)[EW], const uint32_t (&b)[EW],
                                                Parts (&o)[NH]) {
#pragma unroll
    for (int u = 0; u < NH; u++)
      o[u] = dsplit_y(__byte_perm(a[u >> 1], b[u >> 1], (u & 1) ? 0x7362u : 0x5140u));
  }

  static constexpr bool kPair = true;
  // four elements per accumulate step (three 3-input LOP3 per accumulator and
  // four elements instead of two per two) while the operand parts fit
  static constexpr bool kQuad = NH <= BX_DOT_QUAD_MAX_HALVES;

  // a single element (tails): its partner is zero
  __device__ __forceinline__ void add(const uint32_t (&xa)[EW], const uint32_t (&ya)[EW]) {
    uint32_t z[EW];
#pragma unroll
    for (int i = 0; i < EW; i++) z[i] = 0u;
    add2(xa, ya, z, z);
  }

  // two elements
  __device__ __forceinline__ void add2(const uint32_t (&xa)[EW], const uint32_t (&ya)[EW],
                                       const uint32_t (&xb)[EW], const uint32_t (&yb)[EW]) {
    Parts px[NH], py[NH];
    pack_x(xa, xb, px);
    pack_y(ya, yb, py);
    dkara_acc<NH, 0, K>(px, py, acc);
  }

  // four elements
  __device__ __forceinline__ void add4(const uint32_t (&xa)[EW], const uint32_t (&ya)[EW],
                                       const uint32_t (&xb)[EW], const uint32_t (&yb)[EW],
                                       const uint32_t (&xc)[EW], const uint32_t (&yc)[EW],
                                       const uint32_t (&xd)[EW], const uint32_t (&yd)[EW]) {
    Parts px0[NH], py0[NH], px1[NH], py1[NH];
    pack_x(xa, xb, px0);
    pack_y(ya, yb, py0);
    pack_x(xc, xd, px1);
    pack_y(yc, yd, py1);
    dkara_acc2<NH, 0, K>(px0, py0, px1, py1, acc);
  }

  // q = 16: a stream word already holds two elements' (only) halves
  __device__ __forceinline__ void add_words2(uint32_t x0, uint32_t y0, uint32_t x1, uint32_t y1) {
    static_assert(NH == 1, "add_words2 is for q = 16");
    dot16x2(dsplit_x(x0), dsplit_y(__byte_perm(y0, 0u, 0x3120u)), dsplit_x(x1),
            dsplit_y(__byte_perm(y1, 0u, 0x3120u)), acc[0]);
  }

  __device__ __forceinline__ Wide<CW> unreduced() const {
    uint32_t P[K];
#pragma unroll
    for (int s = 0; s < K; s++) {
      const uint32_t l = (acc[s].lo[0] & 0x49249249u) | (acc[s].lo[1] & 0x92492492u) |
                         (acc[s].lo[2] & 0x24924924u);
      const uint32_t h = (acc[s].hi[0] & 0x49249249u) | (acc[s].hi[1] & 0x92492492u) |
                         (acc[s].hi[2] & 0x24924924u);
      P[s] = l ^ (h << 8);
    }
    Wide<CW> c = wzero<CW>();
    kara_fin<NH, 0, 1u, K, CW>(P, c);
    return c;
  }
};

// Dot form with the high-byte sums folded into the low-byte accumulators at
// every step (h << 8 moves class c + 1 onto class c; bits shifted out are
// count garbage): three accumulators per leaf like the IMAD form, for elements
// of five to eight halves, whose 6 x K(NH) split accumulators do not fit.
// Costs one SHF and a wider XOR per class and step; pairs only.
__device__ __forceinline__ void dotm16(const Parts& x, const Parts& y, uint32_t (&acc)[3]) {
  uint32_t l[3], h[3];
#pragma unroll
  for (int c = 0; c < 3; c++) {
    l[c] = 0u;
    h[c] = 0u;
#pragma unroll
    for (int r = 0; r < 3; r++) {
      const int s = (c + 3 - r) % 3;
      l[c] ^= __dp2a_lo(x.p[r], y.p[s], 0u);
      h[c] ^= __dp2a_hi(x.p[r], y.p[s], 0u);
    }
  }
#pragma unroll
  for (int c = 0; c < 3; c++) acc[c] ^= l[c] ^ (h[(c + 1) % 3] << 8);
}

template <int M, int L0, int K>
__device__ __forceinline__ void mkara_acc(const Parts* xo, const Parts* yo, uint32_t (&acc)[K][3]) {
  if constexpr (M == 1) {
    dotm16(xo[0], yo[0], acc[L0]);
  } else {
    constexpr int h = (M + 1) / 2;
    mkara_acc<h, L0, K>(xo, yo, acc);
    mkara_acc<M - h, L0 + kara_leaves(h), K>(xo + h, yo + h, acc);
    Parts xm[h], ym[h];
#pragma unroll
    for (int i = 0; i < h; i++) {
      xm[i] = (i + h < M) ? pxor(xo[i], xo[i + h]) : xo[i];
      ym[i] = (i + h < M) ? pxor(yo[i], yo[i + h]) : yo[i];
    }
    mkara_acc<h, L0 + kara_leaves(h) + kara_leaves(M - h), K>(xm, ym, acc);
  }
}

template <int Q>
struct DotM {
  static constexpr int EW = cdiv(Q, 32);
  static constexpr int NH = cdiv(Q, 16);
  static constexpr int K = kara_leaves(NH);
  static constexpr int CW = cdiv(2 * Q - 1, 32);
  static constexpr bool kPair = true;
  uint32_t acc[K][3];

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int s = 0; s < K; s++) acc[s][0] = acc[s][1] = acc[s][2] = 0u;
  }
  __device__ __forceinline__ void add2(const uint32_t (&xa)[EW], const uint32_t (&ya)[EW],
                                       const uint32_t (&xb)[EW], const uint32_t (&yb)[EW]) {
    Parts px[NH], py[NH];
    Dot<Q>::pack_x(xa, xb, px);
    Dot<Q>::pack_y(ya, yb, py);
    mkara_acc<NH, 0, K>(px, py, acc);
  }
  __device__ __forceinline__ void add(const uint32_t (&xa)[EW], const uint32_t (&ya)[EW]) {
    uint32_t z[EW];
#pragma unroll
    for (int i = 0; i < EW; i++) z[i] = 0u;
    add2(xa, ya, z, z);
  }
  __device__ __forceinline__ Wide<CW> unreduced() const {
    uint32_t P[K];
#pragma unroll
    for (int s = 0; s < K; s++)
      P[s] = (acc[s][0] & 0x49249249u) | (acc[s][1] & 0x92492492u) | (acc[s][2] & 0x24924924u);
    Wide<CW> c = wzero<CW>();
    kara_fin<NH, 0, 1u, K, CW>(P, c);
    return c;
  }
};

// widest element the tile kernels take in the merged form (0: off): -3..-12%
// against the IMAD form from 16 elements per block up, +3..7% at n <= 9
// (profiles/r02/dp2a_sweep.txt, sweep 23)
#ifndef BX_DOTM_MAX_HALVES
#define BX_DOTM_MAX_HALVES 8
#endif

// accumulator of the direct kernels' holes widths
// the q = 64 direct kernel in the dot form (four elements per step): q=64 n=50
// 0.367 -> 0.311 ms, n=64 / n=8 -9% (profiles/r02/dp2a_sweep.txt, sweep 16)
#ifndef BX_DP2A_Q64
#define BX_DP2A_Q64 1
#endif
__host__ __device__ constexpr bool dot_direct_q(int q) {
  return BX_DP2A && (q == 16 || q == 32 || (q == 64 && BX_DP2A_Q64));
}
// accumulator of the tile and period kernels
template <int Q>
using TileHoles = typename std::conditional<
    (BX_DP2A_TILE != 0 && cdiv(Q, 16) <= BX_DOT_TILE_MAX_HALVES), Dot<Q>,
    typename std::conditional<(BX_DP2A_TILE != 0 && cdiv(Q, 16) <= BX_DOTM_MAX_HALVES), DotM<Q>,
                              Holes<Q>>::type>::type;
template <typename H>
struct has_quad { static constexpr bool value = false; };
template <int Q>
struct has_quad<Dot<Q>> { static constexpr bool value = Dot<Q>::kQuad; };

// ----------------------------------------------------------------- kernel

struct EqArgs {
  const uint32_t* x;
  const uint32_t* y;
  int64_t x_bit0;
  int64_t y_bit0;
  int64_t x_words;     // readable words of x (bounds for staging)
  int64_t y_words;
  int64_t nblocks;
  uint32_t* out;
  int64_t out_bit0;
  int n;
  int tpb_log2;        // threads per block = 1 << tpb_log2 (<= 32)
  int tile_blocks;     // blocks per CTA
  int stage_words;     // smem words per source (STAGED only)
  int stages;          // TMA kernel: input stages per CTA (2: double buffer, 1: single)
  int64_t x_limit;     // words of x the ABI guarantees readable (checked builds)
  int64_t y_limit;
  int64_t out_words;   // words of out the run may touch (checked builds)
};

// One q-bit element at bit `off`: the EW + 1 covering words are loaded once and
// funnel-shifted (word (off>>5) + EW must be readable).
template <int Q, int EW, typename T>
__device__ __forceinline__ void read_elem(const uint32_t* src, T off, int64_t lim,
                                          uint32_t (&w)[EW]) {
  const T w0 = off >> 5;
  const uint32_t sh = (uint32_t)(off & 31);
  BX_CHECK(w0 + EW, lim, 1);
  uint32_t r[EW + 1];
#pragma unroll
  for (int i = 0; i <= EW; i++) r[i] = src[w0 + i];
#pragma unroll
  for (int i = 0; i < EW; i++) w[i] = __funnelshift_r(r[i], r[i + 1], sh);
  if constexpr (Q % 32) w[EW - 1] &= (1u << (Q % 32)) - 1u;
}

// Blocks [tile0, tile0 + nb) of a tile: each group of tpb threads computes one
// block from the word arrays sx / sy (shared or global memory) whose block 0
// starts at bit xbase / ybase, and ORs its q-bit output into `so` at bit
// obase + grp*Q (so must be zeroed).  xlim / ylim / olim are the word bounds of
// sx / sy / so (checked builds).  Ends with the caller's __syncthreads.
template <int Q, typename T = int64_t>
__device__ __forceinline__ void tile_compute(const EqArgs& a, const uint32_t* sx, const uint32_t* sy,
                                             int64_t xbase, int64_t ybase, uint32_t* so,
                                             int64_t obase, int nb, int64_t xlim, int64_t ylim,
                                             int64_t olim) {
  constexpr int EW = cdiv(Q, 32);
  constexpr int CW = cdiv(2 * Q - 1, 32);
  const int tpb = 1 << a.tpb_log2;
  const int64_t B = (int64_t)Q * a.n;
  const int tid = threadIdx.x;
  const int grp = tid >> a.tpb_log2, sub = tid & (tpb - 1);
  Wide<CW> c = wzero<CW>();
  if (grp < nb) {
    const T xo = (T)xbase + (T)grp * (T)B, yo = (T)ybase + (T)grp * (T)B;
    if constexpr (Q <= kDiagMaxQ) {
      using D = Diag<Q>;
      D acc;
      acc.init();
      const int nch = cdiv(a.n, D::E);
      for (int ch = sub; ch < nch; ch += tpb) {
        const T off = (T)ch * (T)D::EB;
        const int valid = min(D::E, a.n - ch * D::E) * Q;
        const uint32_t m = valid >= 32 ? 0xFFFFFFFFu : ((1u << valid) - 1u);
        acc.add(read32(sx, xo + off, xlim) & m, read32(sy, yo + off, ylim));
      }
      c.w[0] = acc.unreduced();
    } else {
      using H = TileHoles<Q>;
      H acc;
      acc.init();
      int j = sub;
      if constexpr (has_quad<H>::value) {
        for (; j + 3 * tpb < a.n; j += 4 * tpb) {
          uint32_t xw[4][EW], yw[4][EW];
#pragma unroll
          for (int k = 0; k < 4; k++) {
            read_elem<Q>(sx, xo + (T)(j + k * tpb) * (T)Q, xlim, xw[k]);
            read_elem<Q>(sy, yo + (T)(j + k * tpb) * (T)Q, ylim, yw[k]);
          }
          acc.add4(xw[0], yw[0], xw[1], yw[1], xw[2], yw[2], xw[3], yw[3]);
        }
      }
      for (; H::kPair && j + tpb < a.n; j += 2 * tpb) {
        uint32_t xw[EW], yw[EW], xw2[EW], yw2[EW];
        read_elem<Q>(sx, xo + (T)j * (T)Q, xlim, xw);
        read_elem<Q>(sy, yo + (T)j * (T)Q, ylim, yw);
        read_elem<Q>(sx, xo + (T)(j + tpb) * (T)Q, xlim, xw2);
        read_elem<Q>(sy, yo + (T)(j + tpb) * (T)Q, ylim, yw2);
        acc.add2(xw, yw, xw2, yw2);
      }
      for (; j < a.n; j += tpb) {
        uint32_t xw[EW], yw[EW];
        read_elem<Q>(sx, xo + (T)j * (T)Q, xlim, xw);
        read_elem<Q>(sy, yo + (T)j * (T)Q, ylim, yw);
        acc.add(xw, yw);
      }
      c = acc.unreduced();
    }
  }
  for (int m = 1; m < tpb; m <<= 1) {
#pragma unroll
    for (int i = 0; i < CW; i++) c.w[i] ^= __shfl_xor_sync(0xFFFFFFFFu, c.w[i], m);
  }
  if (grp < nb && sub == 0) {
    const Wide<EW> z = reduce<Q>(c);
    const int64_t ob = obase + (int64_t)grp * Q;
    const int w0 = (int)(ob >> 5);
    const uint32_t sh = (uint32_t)(ob & 31);
#pragma unroll
    for (int i = 0; i <= EW; i++) {
      const uint32_t lo = at(z, i - 1), hi = at(z, i);
      const uint32_t v = sh ? __funnelshift_l(lo, hi, sh) : hi;
      if (v) {
        BX_CHECK(w0 + i, olim, 2);
        atomicOr(&so[w0 + i], v);
      }
    }
  }
}

// Store the assembled output words of one tile: interior words plainly, the
// (<= 2) boundary words merged atomically so bits outside the run survive.
// CLEAR: leave the tile's words of `so` zeroed for the buffer's next use (every
// word a tile's blocks can touch lies in [0, ow)).
template <bool CLEAR = false>
__device__ __forceinline__ void tile_store(uint32_t* out, uint32_t* so, int64_t ostart,
                                           int64_t oend, int64_t out_words) {
  const int64_t gw0 = ostart >> 5;
  const int ow = (int)(((oend + 31) >> 5) - gw0);
  for (int i = threadIdx.x; i < ow; i += blockDim.x) {
    const int64_t lo = (gw0 + i) * 32, hi = lo + 32;
    const uint32_t v = so[i];
    if constexpr (CLEAR) so[i] = 0u;
    BX_CHECK(gw0 + i, out_words, 3);
    if (lo >= ostart && hi <= oend) {
      out[gw0 + i] = v;
    } else {
      const int64_t s = lo > ostart ? lo : ostart;
      const int64_t e = hi < oend ? hi : oend;
      const int nbits = (int)(e - s), off = (int)(s - lo);
      const uint32_t mask = (nbits >= 32 ? 0xFFFFFFFFu : ((1u << nbits) - 1u)) << off;
      atomicAnd(&out[gw0 + i], ~mask);
      atomicOr(&out[gw0 + i], v & mask);
    }
  }
}

template <int Q, bool STAGED>
__global__ void __launch_bounds__(256, (Q > 32 ? 2 : 1)) eq_kernel(const EqArgs a) {
  extern __shared__ uint32_t smem[];
  const int T = a.tile_blocks;
  const int64_t B = (int64_t)Q * a.n;
  const int64_t tile0 = (int64_t)blockIdx.x * T;
  const int nb = (int)((a.nblocks - tile0) < T ? (a.nblocks - tile0) : T);
  const int tid = threadIdx.x, nthr = blockDim.x;

  const uint32_t* sx;
  const uint32_t* sy;
  uint32_t* so;
  int64_t xbase, ybase;
  if constexpr (STAGED) {
    const int sw = a.stage_words;
    const int64_t xs = a.x_bit0 + tile0 * B, ys = a.y_bit0 + tile0 * B;
    const int64_t xw0 = xs >> 5, yw0 = ys >> 5;
    const int nwx = (int)((((xs & 31) + nb * B + 31) >> 5) + 1);
    const int nwy = (int)((((ys & 31) + nb * B + 31) >> 5) + 1);
    BX_CHECK(nwx - 1, sw, 4);
    BX_CHECK(nwy - 1, sw, 4);
    for (int i = tid; i < nwx; i += nthr)
      smem[i] = (xw0 + i < a.x_words) ? __ldg(a.x + xw0 + i) : 0u;
    for (int i = tid; i < nwy; i += nthr)
      smem[sw + i] = (yw0 + i < a.y_words) ? __ldg(a.y + yw0 + i) : 0u;
    sx = smem;
    sy = smem + sw;
    so = smem + 2 * sw;
    xbase = xs & 31;
    ybase = ys & 31;
  } else {
    sx = a.x;
    sy = a.y;
    so = smem;
    xbase = a.x_bit0 + tile0 * B;
    ybase = a.y_bit0 + tile0 * B;
  }
  const int64_t ostart = a.out_bit0 + tile0 * Q;
  const int ow = (int)((((ostart & 31) + (int64_t)nb * Q + 31) >> 5));
  for (int i = tid; i < ow + 1; i += nthr) so[i] = 0u;
  __syncthreads();
  const int64_t xlim = STAGED ? a.stage_words : a.x_limit;
  const int64_t ylim = STAGED ? a.stage_words : a.y_limit;
  if constexpr (STAGED)
    tile_compute<Q, uint32_t>(a, sx, sy, xbase, ybase, so, ostart & 31, nb, xlim, ylim, ow + 1);
  else
    tile_compute<Q, int64_t>(a, sx, sy, xbase, ybase, so, ostart & 31, nb, xlim, ylim, ow + 1);
  __syncthreads();
  tile_store(a.out, so, ostart, ostart + (int64_t)nb * Q, a.out_words);
}

// ------------------------------------------------- TMA-bulk pipelined kernel
//
// Persistent CTAs walk tiles t = blockIdx.x, += gridDim.x.  Each tile's two
// input windows are brought into shared memory with one cp.async.bulk per
// stream (the TMA engine, completion counted on an mbarrier), double
// buffered: while the CTA computes tile t from one buffer, tile t + gridDim.x
// is already landing in the other.  Requires 16-byte aligned stream bases and
// streams readable through round_up(bytes, 16) + 16.

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

struct TileWin {
  int64_t lo;      // first byte copied (16-aligned)
  uint32_t bytes;  // bytes copied (multiple of 16)
  int64_t bit0;    // bit of block 0 relative to the copied bytes
};

__device__ __forceinline__ TileWin tile_window(int64_t bit_start, int64_t nbits) {
  TileWin w;
  w.lo = (bit_start >> 3) & ~(int64_t)15;
  const int64_t hi = ((((bit_start + nbits + 7) >> 3) + 4 + 15) & ~(int64_t)15);
  w.bytes = (uint32_t)(hi - w.lo);
  w.bit0 = bit_start - 8 * w.lo;
  return w;
}

#ifndef BX_PDL
#define BX_PDL 1   // programmatic dependent launch for the direct and TMA kernels (0: plain, A/B)
#endif

// Programmatic dependent launch: allow the next launch in the stream to be
// scheduled as this grid drains; wait for the previous grid (complete, memory
// visible) before touching global memory.
__device__ __forceinline__ void pdl_entry() {
#if BX_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// Resident CTAs the TMA kernel's registers are capped for at 32 < q <= 64: the
// dot form keeps 6 accumulators per leaf (36 / 54 for 3 / 4 halves), which
// spills under the 85-register cap of three CTAs (c4p 2.66 ms) and runs in
// 128 registers with two (c4p 2.19 ms; the IMAD form with three: 2.38 ms --
// profiles/r02/dp2a_sweep.txt).
#ifndef BX_TMA_MINB_Q64
#define BX_TMA_MINB_Q64 2
#endif
#ifndef BX_TMA_MINB_Q128
#define BX_TMA_MINB_Q128 2
#endif
template <int Q>
__global__ void __launch_bounds__(256, (Q > 64 ? BX_TMA_MINB_Q128 : (Q > 32 ? BX_TMA_MINB_Q64 : 2))) eq_tma_kernel(const EqArgs a) {
  pdl_entry();
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ __align__(8) uint64_t bars[2];
  const int T = a.tile_blocks;
  const int sw = a.stage_words;  // words per source buffer (multiple of 4)
  const int64_t B = (int64_t)Q * a.n;
  const int64_t ntiles = (a.nblocks + T - 1) / T;
  const int ow_max = (int)((31 + (int64_t)T * Q + 31) >> 5) + 2;
  const int S = a.stages;                         // input stages (1 or 2)
  uint32_t* bufs = smem;                          // [stage][x|y][sw]
  uint32_t* outs = smem + 2 * S * sw;             // [2][ow_max]
  const char* xg = reinterpret_cast<const char*>(a.x);
  const char* yg = reinterpret_cast<const char*>(a.y);

  auto issue = [&](int64_t t, int st) {
    const int64_t tile0 = t * T;
    const int64_t nb = (a.nblocks - tile0) < T ? (a.nblocks - tile0) : T;
    const TileWin wx = tile_window(a.x_bit0 + tile0 * B, nb * B);
    const TileWin wy = tile_window(a.y_bit0 + tile0 * B, nb * B);
    BX_CHECK((int64_t)wx.bytes / 4 - 1, sw, 5);
    BX_CHECK((int64_t)wy.bytes / 4 - 1, sw, 5);
    BX_CHECK((wx.lo + wx.bytes) / 4 - 1, a.x_limit, 6);
    BX_CHECK((wy.lo + wy.bytes) / 4 - 1, a.y_limit, 6);
    mbar_expect_tx(&bars[st], wx.bytes + wy.bytes);
    bulk_g2s(bufs + (2 * st) * sw, xg + wx.lo, wx.bytes, &bars[st]);
    bulk_g2s(bufs + (2 * st + 1) * sw, yg + wy.lo, wy.bytes, &bars[st]);
  };

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // both output tiles start zeroed; afterwards tile_store<true> re-zeroes the
  // words it consumed, so a tile needs no zeroing pass (and no barrier) before
  // its blocks OR their outputs in
  for (int i = threadIdx.x; i < 2 * ow_max; i += blockDim.x) outs[i] = 0u;
  __syncthreads();
  int64_t t = blockIdx.x;
  if (threadIdx.x == 0 && t < ntiles) issue(t, 0);
  uint32_t phase[2] = {0u, 0u};
  int st = 0, ost = 0;
  for (; t < ntiles; t += gridDim.x, ost ^= 1) {
    const int64_t tn = t + gridDim.x;
    if (S == 2 && threadIdx.x == 0 && tn < ntiles) {
      // the buffer being refilled was last read through the generic proxy
      // (before the previous iteration's __syncthreads); order those reads
      // before the async-proxy (TMA) writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tn, st ^ 1);
    }
    const int64_t tile0 = t * T;
    const int nb = (int)((a.nblocks - tile0) < T ? (a.nblocks - tile0) : T);
    const int64_t ostart = a.out_bit0 + tile0 * Q;
    uint32_t* so = outs + ost * ow_max;
    const TileWin wx = tile_window(a.x_bit0 + tile0 * B, (int64_t)nb * B);
    const TileWin wy = tile_window(a.y_bit0 + tile0 * B, (int64_t)nb * B);
    // every thread observes the phase flip itself, which makes the bulk copy's
    // bytes visible to it: no CTA barrier before the compute
    mbar_wait(&bars[st], phase[st]);
    phase[st] ^= 1u;
    tile_compute<Q, uint32_t>(a, bufs + (2 * st) * sw, bufs + (2 * st + 1) * sw, wx.bit0, wy.bit0, so,
                    ostart & 31, nb, sw, sw, ow_max);
    // all of this tile's output bits are in `so` and all reads of this input
    // buffer are done (thread 0 refills it next iteration)
    __syncthreads();
    if (S == 1) {
      // single stage: the only input buffer is free now; its refill overlaps
      // this tile's store and the other resident CTAs' compute (half the
      // shared memory per CTA, twice the resident warps)
      if (threadIdx.x == 0 && tn < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(tn, 0);
      }
    } else {
      st ^= 1;
    }
    tile_store<true>(a.out, so, ostart, ostart + (int64_t)nb * Q, a.out_words);
  }
}

// ------------------------------------------------------- direct kernel
//
// Aligned fast path: Q in {1,2,4,8,16,32,64,128}, q*n a multiple of 128 bits,
// 16-byte aligned stream starts, word-aligned output.  One thread per block;
// the block's windows are read with 128-bit loads straight from HBM (each
// 128-bit unit holds 128/Q whole elements), no shared-memory staging.  The
// outputs of a warp's 32 consecutive blocks are OR-combined with shuffles
// into whole 32-bit words (Q < 32) or stored directly (Q >= 32).
struct DirectArgs {
  const uint4* x;      // 16-byte aligned start of block 0's window
  const uint4* y;
  int64_t nblocks;
  uint32_t* out;       // word holding output bit 0 of block 0
  int units;           // 128-bit units per block (q*n/128)
  int wide;            // 1: x, y 32-byte aligned and units even -> 256-bit loads
  int64_t x_limit;     // readable 16-byte units from x / y (checked builds)
  int64_t y_limit;
  int64_t out_words;   // writable words from out (checked builds)
};

// Pairing two elements per accumulate step (Holes::add2): same LOP3 count
// after ptxas re-associates the XOR trees, but a different schedule.  At
// q = 16 the unpaired order is 5% faster; at q = 32 / 64 the paired one is
// equal / 3-5% faster (profiles/r01_direct_sweep.txt J).
#ifndef BX_DIRECT_PAIR
#define BX_DIRECT_PAIR 1
#endif
#ifndef BX_DIRECT_PAIR16
#define BX_DIRECT_PAIR16 0
#endif

template <int Q>
using DirectHoles = typename std::conditional<dot_direct_q(Q), Dot<Q>, Holes<Q>>::type;

template <int Q>
__device__ __forceinline__ void direct_unit(const uint4& X, const uint4& Y, void* accp) {
  if constexpr (Q <= kDiagMaxQ) {
    Diag<Q>& acc = *static_cast<Diag<Q>*>(accp);
    acc.add(X.x, Y.x);
    acc.add(X.y, Y.y);
    acc.add(X.z, Y.z);
    acc.add(X.w, Y.w);
  } else if constexpr (dot_direct_q(Q)) {
    Dot<Q>& acc = *static_cast<Dot<Q>*>(accp);
    if constexpr (Q == 16) {
      acc.add_words2(X.x, Y.x, X.y, Y.y);
      acc.add_words2(X.z, Y.z, X.w, Y.w);
    } else if constexpr (Q == 64) {     // one unit = two elements
      const uint32_t xa[2] = {X.x, X.y}, xb[2] = {X.z, X.w};
      const uint32_t ya[2] = {Y.x, Y.y}, yb[2] = {Y.z, Y.w};
      acc.add2(xa, ya, xb, yb);
    } else {
      const uint32_t xa[1] = {X.x}, xb[1] = {X.y}, xc[1] = {X.z}, xd[1] = {X.w};
      const uint32_t ya[1] = {Y.x}, yb[1] = {Y.y}, yc[1] = {Y.z}, yd[1] = {Y.w};
      acc.add4(xa, ya, xb, yb, xc, yc, xd, yd);
    }
  } else {
    Holes<Q>& acc = *static_cast<Holes<Q>*>(accp);
    constexpr int EW = cdiv(Q, 32);
    const uint32_t xs[4] = {X.x, X.y, X.z, X.w};
    const uint32_t ys[4] = {Y.x, Y.y, Y.z, Y.w};
    if constexpr (Q == 16) {
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const uint32_t a0[1] = {xs[i]}, b0[1] = {ys[i]};          // low half (split masks it)
        const uint32_t a1[1] = {xs[i] >> 16}, b1[1] = {ys[i] >> 16};
#if BX_DIRECT_PAIR16
        acc.add2(a0, b0, a1, b1);
#else
        acc.add(a0, b0);
        acc.add_clean(a1[0], b1[0]);   // high halves: no bits above 15 after the shift
#endif
      }
    } else if constexpr (4 / EW >= 2 && Holes<Q>::kPair && BX_DIRECT_PAIR) {
#pragma unroll
      for (int e = 0; e < 4 / EW; e += 2) {
        uint32_t a[EW], b[EW], c2[EW], d2[EW];
#pragma unroll
        for (int i = 0; i < EW; i++) {
          a[i] = xs[e * EW + i];
          b[i] = ys[e * EW + i];
          c2[i] = xs[(e + 1) * EW + i];
          d2[i] = ys[(e + 1) * EW + i];
        }
        acc.add2(a, b, c2, d2);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4 / EW; e++) {          // every element of the unit
        uint32_t a[EW], b[EW];
#pragma unroll
        for (int i = 0; i < EW; i++) {
          a[i] = xs[e * EW + i];
          b[i] = ys[e * EW + i];
        }
        acc.add(a, b);
      }
    }
  }
}

// Two consecutive 128-bit units with one 256-bit load (LDG.E.ENL2.256 on
// sm_100a): a whole 32-byte sector per thread per instruction.  Threads of a
// warp read windows q*n/8 bytes apart, so every load touches 32 lines; at
// q = 16 the 128-bit-load kernel is L1-throughput bound and the 256-bit loads
// halve its L1 requests (+8%, profiles/r01_direct_sweep.txt).
#ifndef BX_L2_HINT
#define BX_L2_HINT 0
#endif
#if BX_L2_HINT == 256
#define BX_LD_HINT ".L2::256B"
#elif BX_L2_HINT == 128
#define BX_LD_HINT ".L2::128B"
#elif BX_L2_HINT == 64
#define BX_LD_HINT ".L2::64B"
#else
#define BX_LD_HINT ""
#endif

// 128-bit read-only load of a stream unit (with the L2 sector-promotion hint
// BX_L2_HINT when set)
__device__ __forceinline__ uint4 ldg128(const uint4* p) {
#if BX_L2_HINT
  uint4 a;
  asm volatile("ld.global.nc" BX_LD_HINT ".v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w)
               : "l"(p));
  return a;
#else
  return __ldg(p);
#endif
}

__device__ __forceinline__ void ldg256(const uint4* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc" BX_LD_HINT ".v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

// Register double buffer of the next 256-bit unit pair in the q = 16 wide loop,
// with the q = 16 kernel capped at 64 registers (4 CTAs/SM): c5 n=1024 3.37 vs
// 3.41 ms; uncapped (81 registers, 3 CTAs) it is 5% slower, and the same
// prefetch for q = 17..32 is 4% slower (profiles/r02/direct_prefetch_sweep.txt).
#ifndef BX_PREFETCH_WIDE
#define BX_PREFETCH_WIDE 1
#endif
#ifndef BX_PREFETCH_Q32
#define BX_PREFETCH_Q32 0
#endif

// Unreduced inner product of one block's windows with 256-bit loads (units
// even, xp / yp 32-byte aligned).
template <int Q>
__device__ __forceinline__ Wide<cdiv(2 * Q - 1, 32)> direct_block_wide(const uint4* xp, const uint4* yp,
                                                                       int units) {
  Wide<cdiv(2 * Q - 1, 32)> c;
  if constexpr (Q <= kDiagMaxQ) {
    Diag<Q> acc;
    acc.init();
#pragma unroll 2
    for (int u = 0; u < units; u += 2) {
      uint4 X0, X1, Y0, Y1;
      ldg256(xp + u, X0, X1);
      ldg256(yp + u, Y0, Y1);
      direct_unit<Q>(X0, Y0, &acc);
      direct_unit<Q>(X1, Y1, &acc);
    }
    c.w[0] = acc.unreduced();
  } else {
    DirectHoles<Q> acc;
    acc.init();
#if BX_PREFETCH_WIDE
    // register double buffer: the next unit pair is in flight while this one
    // multiplies (ncu: long_scoreboard was the top stall of the q = 16 loop)
    uint4 X0, X1, Y0, Y1;
    ldg256(xp, X0, X1);
    ldg256(yp, Y0, Y1);
#pragma unroll 1
    for (int u = 0; u < units; u += 2) {
      uint4 N0 = X0, N1 = X1, M0 = Y0, M1 = Y1;
      if (u + 2 < units) {
        ldg256(xp + u + 2, N0, N1);
        ldg256(yp + u + 2, M0, M1);
      }
      direct_unit<Q>(X0, Y0, &acc);
      direct_unit<Q>(X1, Y1, &acc);
      X0 = N0; X1 = N1; Y0 = M0; Y1 = M1;
    }
#else
#pragma unroll 1
    for (int u = 0; u < units; u += 2) {
      uint4 X0, X1, Y0, Y1;
      ldg256(xp + u, X0, X1);
      ldg256(yp + u, Y0, Y1);
      direct_unit<Q>(X0, Y0, &acc);
      direct_unit<Q>(X1, Y1, &acc);
    }
#endif
    c = acc.unreduced();
  }
  return c;
}

// Min resident CTAs for the q = 17..32 direct kernels: 3 caps them at 85
// registers (127 uncapped, 2 CTAs/SM) without spills: +9% at q = 32
// (profiles/r01_direct_sweep.txt K).
// q = 128 in three passes over the block (BX_Q128_PASSES=0: one pass).  The
// top Karatsuba level (64-bit halves) is taken outside the element loop:
//     x*y = L + (L + H + M) t^64 + H t^128,  L = lo*lo, H = hi*hi, M = (lo^hi)*(hi^lo),
// each summed over the block's elements by its own pass, so only one 64-bit
// sub-product's 27 accumulators are live (the one-pass form keeps 81, which
// forbids element pairing under the 128-register cap).  The block's 2 x 256
// bytes are re-read from L1/L2 by passes 2 and 3.
#ifndef BX_Q128_PASSES
#define BX_Q128_PASSES 1
#endif

// q = 128 passes with the dot-product accumulator (0: IMAD holes, 1: pairs,
// 2: four elements per step)
#ifndef BX_Q128_DOT
#define BX_Q128_DOT 0
#endif

template <int P>
__device__ __forceinline__ void q128_part(const uint4& v, uint32_t (&o)[2]) {
  if constexpr (P == 0) {
    o[0] = v.x;
    o[1] = v.y;
  } else if constexpr (P == 1) {
    o[0] = v.z;
    o[1] = v.w;
  } else {
    o[0] = v.x ^ v.z;
    o[1] = v.y ^ v.w;
  }
}

template <int P>
__device__ __forceinline__ void q128_pass(const uint4* xp, const uint4* yp, int units, bool wide,
                                          Wide<8>& c) {
  typename std::conditional<(BX_Q128_DOT != 0), Dot<64>, Holes<64>>::type acc;
  acc.init();
  int u = 0;
#if BX_Q128_DOT == 2
#pragma unroll 1
  for (; u + 3 < units; u += 4) {     // four elements per accumulate step
    uint4 X[4], Y[4];
    if (wide) {
      ldg256(xp + u, X[0], X[1]);
      ldg256(yp + u, Y[0], Y[1]);
      ldg256(xp + u + 2, X[2], X[3]);
      ldg256(yp + u + 2, Y[2], Y[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; k++) {
        X[k] = ldg128(xp + u + k);
        Y[k] = ldg128(yp + u + k);
      }
    }
    uint32_t a[4][2], b[4][2];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      q128_part<P>(X[k], a[k]);
      q128_part<P>(Y[k], b[k]);
    }
    acc.add4(a[0], b[0], a[1], b[1], a[2], b[2], a[3], b[3]);
  }
#endif
#pragma unroll 1
  for (; u + 1 < units; u += 2) {
    uint4 X0, X1, Y0, Y1;
    if (wide) {            // the passes re-read the block: halve the L1 requests
      ldg256(xp + u, X0, X1);
      ldg256(yp + u, Y0, Y1);
    } else {
      X0 = ldg128(xp + u);
      Y0 = ldg128(yp + u);
      X1 = ldg128(xp + u + 1);
      Y1 = ldg128(yp + u + 1);
    }
    uint32_t a[2], b[2], a2[2], b2[2];
    q128_part<P>(X0, a);
    q128_part<P>(Y0, b);
    q128_part<P>(X1, a2);
    q128_part<P>(Y1, b2);
    acc.add2(a, b, a2, b2);
  }
  if (u < units) {
    uint32_t a[2], b[2];
    q128_part<P>(ldg128(xp + u), a);
    q128_part<P>(ldg128(yp + u), b);
    acc.add(a, b);
  }
  const Wide<4> p = acc.unreduced();
#pragma unroll
  for (int i = 0; i < 4; i++) {
    if constexpr (P == 0) c.w[i] ^= p.w[i];          // L at t^0
    if constexpr (P == 1) c.w[i + 4] ^= p.w[i];      // H at t^128
    c.w[i + 2] ^= p.w[i];                            // L, H, M at t^64
  }
}

__device__ __forceinline__ Wide<8> direct_block_q128(const uint4* xp, const uint4* yp, int units,
                                                     bool wide) {
  Wide<8> c = wzero<8>();
  q128_pass<0>(xp, yp, units, wide, c);
  q128_pass<1>(xp, yp, units, wide, c);
  q128_pass<2>(xp, yp, units, wide, c);
  return c;
}

#ifndef BX_Q32_UNROLL
#define BX_Q32_UNROLL 2
#endif
constexpr int kQ32Unroll = BX_Q32_UNROLL;
#ifndef BX_DIRECT_MINB_Q32
#define BX_DIRECT_MINB_Q32 3
#endif
#ifndef BX_DIRECT_MINB_Q16
#define BX_DIRECT_MINB_Q16 4
#endif
#ifndef BX_DIRECT_MINB_Q8
#define BX_DIRECT_MINB_Q8 1
#endif

// q = 128 (three passes): 3 CTAs/SM (80 registers) for 8 or more units per
// block (c3 n=8: +4% over one pass), 2 below (n=4: 3 CTAs cost 13%, 2 gain
// 12%) -- profiles/r01_direct_sweep.txt L.
#ifndef BX_DIRECT_MINB_Q128
#define BX_DIRECT_MINB_Q128(U) ((U) == 0 || (U) >= 8 ? 3 : 2)
#endif

// CTA size of the direct kernel: 128 threads (twice the CTAs per SM, same
// registers) for q >= 32, where it gains 3% (q = 32, 128); 256 below, where
// blocks are small and 128-thread CTAs hit the CTA launch rate (q = 2: -42%)
// -- profiles/r01_direct_sweep.txt O.
__host__ __device__ constexpr int direct_threads(int q) { return q >= 32 ? 128 : 256; }

// Blocks per thread of the direct kernel for small blocks at q <= 4: one-unit
// blocks (c5 n = 128) take BX_DIRECT_BPT1, two-unit blocks (c5 n = 256, c2)
// BX_DIRECT_BPT2 blocks per thread, one grid stride apart.  2 and 2: c5 n=128
// 2.53 -> 2.39 ms, n=256 2.43 -> 2.39 ms (7.25 TB/s read, 1.11 x the copy
// peak); 4 per thread is flat at n=128 and 5% slower at n=256, 8 is 38% slower
// (profiles/r02/direct_prefetch_sweep.txt).
#ifndef BX_DIRECT_BPT1
#define BX_DIRECT_BPT1 2
#endif
#ifndef BX_DIRECT_BPT2
#define BX_DIRECT_BPT2 2
#endif
#ifndef BX_DIRECT_BPT8
#define BX_DIRECT_BPT8 1
#endif
__host__ __device__ constexpr int direct_bpt(int q, int u) {
  return q == 8 && u == 4 ? BX_DIRECT_BPT8
                          : (q > 4 ? 1 : (u == 1 ? BX_DIRECT_BPT1 : (u == 2 ? BX_DIRECT_BPT2 : 1)));
}

// Store block l's output z: for q < 32, 32/q consecutive blocks (lanes) share
// one output word, assembled with shuffles (every lane of the warp must call);
// the run's last partial word is merged atomically.
template <int Q>
__device__ __forceinline__ void direct_store(const DirectArgs& a, int64_t l, const Wide<cdiv(Q, 32)>& z,
                                             int lane) {
  constexpr int EW = cdiv(Q, 32);
  if constexpr (Q < 32) {
    // 32/Q consecutive blocks share one output word
    constexpr int G = 32 / Q;
    uint32_t v = z.w[0] << ((lane % G) * Q);
#pragma unroll
    for (int m = 1; m < G; m <<= 1) v |= __shfl_xor_sync(0xFFFFFFFFu, v, m);
    const int64_t first = l - (lane % G);      // first block of this word
    if ((lane % G) == 0 && first < a.nblocks) {
      const int64_t w = first * Q / 32;
      const int64_t valid = (a.nblocks - first) * Q;
      BX_CHECK(w, a.out_words, 8);
      if (valid >= 32) {
        a.out[w] = v;
      } else {
        const uint32_t mask = (1u << valid) - 1u;
        atomicAnd(&a.out[w], ~mask);
        atomicOr(&a.out[w], v & mask);
      }
    }
  } else {
    if (l < a.nblocks) {
#pragma unroll
      for (int i = 0; i < EW; i++) {
        BX_CHECK(l * EW + i, a.out_words, 8);
        a.out[l * EW + i] = z.w[i];
      }
    }
  }
}

template <int Q, int U>
__global__ void __launch_bounds__(direct_threads(Q),
                                  (256 / direct_threads(Q)) *
                                      (Q == 128 ? BX_DIRECT_MINB_Q128(U)
                                                : (Q > 32 ? 2 : (Q > 16 ? BX_DIRECT_MINB_Q32
                                                                        : (Q > 8 ? BX_DIRECT_MINB_Q16
                                                                                 : (Q > 4 ? BX_DIRECT_MINB_Q8 : 1))))))
    eq_direct_kernel(const DirectArgs a) {
  constexpr int EW = cdiv(Q, 32);
  constexpr int CW = cdiv(2 * Q - 1, 32);
  pdl_entry();
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if constexpr (Q <= 4 && direct_bpt(Q, U) > 1) {
    // small blocks (q <= 4, one or two units): each thread takes BPT blocks one
    // grid stride apart and issues all their loads before computing (more
    // bytes in flight per thread, BPT x fewer CTAs to launch)
    constexpr int BPT = direct_bpt(Q, U);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    uint4 X[BPT][U], Y[BPT][U];
#pragma unroll
    for (int k = 0; k < BPT; k++) {
      const int64_t lk = l + k * stride;
      if (lk < a.nblocks) {
        BX_CHECK((lk + 1) * U - 1, a.x_limit, 7);
        BX_CHECK((lk + 1) * U - 1, a.y_limit, 7);
#pragma unroll
        for (int u = 0; u < U; u++) {
          X[k][u] = ldg128(a.x + lk * U + u);
          Y[k][u] = ldg128(a.y + lk * U + u);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < BPT; k++) {
      const int64_t lk = l + k * stride;
      Wide<EW> zk = wzero<EW>();
      if (lk < a.nblocks) {
        Diag<Q> acc;
        acc.init();
#pragma unroll
        for (int u = 0; u < U; u++) direct_unit<Q>(X[k][u], Y[k][u], &acc);
        Wide<CW> c;
        c.w[0] = acc.unreduced();
        zk = reduce<Q>(c);
      }
      direct_store<Q>(a, lk, zk, lane);
    }
    return;
  }
  if constexpr (Q == 8 && U == 4 && BX_DIRECT_BPT8 > 1) {
    // q = 8, four units per block (c5 n = 512): the next block's 2 x 64 bytes
    // are loaded (256-bit loads when aligned) while this block multiplies
    constexpr int BPT = BX_DIRECT_BPT8;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    uint4 X[2][4], Y[2][4];
    auto load = [&](int64_t lk, uint4 (&xs)[4], uint4 (&ys)[4]) {
      const uint4* xp = a.x + lk * 4;
      const uint4* yp = a.y + lk * 4;
      if (a.wide) {
        ldg256(xp, xs[0], xs[1]);
        ldg256(xp + 2, xs[2], xs[3]);
        ldg256(yp, ys[0], ys[1]);
        ldg256(yp + 2, ys[2], ys[3]);
      } else {
#pragma unroll
        for (int u = 0; u < 4; u++) {
          xs[u] = ldg128(xp + u);
          ys[u] = ldg128(yp + u);
        }
      }
    };
    if (l < a.nblocks) load(l, X[0], Y[0]);
#pragma unroll
    for (int k = 0; k < BPT; k++) {
      const int64_t lk = l + k * stride;
      if (k + 1 < BPT && lk + stride < a.nblocks) load(lk + stride, X[(k + 1) & 1], Y[(k + 1) & 1]);
      Wide<EW> zk = wzero<EW>();
      if (lk < a.nblocks) {
        BX_CHECK((lk + 1) * 4 - 1, a.x_limit, 7);
        BX_CHECK((lk + 1) * 4 - 1, a.y_limit, 7);
        Diag<Q> acc;
        acc.init();
#pragma unroll
        for (int u = 0; u < 4; u++) direct_unit<Q>(X[k & 1][u], Y[k & 1][u], &acc);
        Wide<CW> c;
        c.w[0] = acc.unreduced();
        zk = reduce<Q>(c);
      }
      direct_store<Q>(a, lk, zk, lane);
    }
    return;
  }
  Wide<EW> z = wzero<EW>();
  if (l < a.nblocks) {
    const uint4* xp = a.x + l * a.units;
    const uint4* yp = a.y + l * a.units;
    BX_CHECK((l + 1) * (U > 0 ? U : a.units) - 1, a.x_limit, 7);
    BX_CHECK((l + 1) * (U > 0 ? U : a.units) - 1, a.y_limit, 7);
    // U > 0: the unit count is a compile-time constant (fully unrolled,
    // all loads issued up front); U == 0: runtime count.
    const int units = U > 0 ? U : a.units;
    if ((Q <= 16 || Q == 32) && a.wide) {
      z = reduce<Q>(direct_block_wide<Q>(xp, yp, units));
    } else {
      Wide<CW> c;
      if constexpr (Q <= kDiagMaxQ) {
        Diag<Q> acc;
        acc.init();
#pragma unroll 4
        for (int u = 0; u < units; u++) direct_unit<Q>(ldg128(xp + u), ldg128(yp + u), &acc);
        c.w[0] = acc.unreduced();
      } else {
        if constexpr (Q == 128 && BX_Q128_PASSES) {
          c = direct_block_q128(xp, yp, units, a.wide);
        } else {
          DirectHoles<Q> acc;
          acc.init();
          if constexpr (Q == 64 && dot_direct_q(Q)) {
            int u = 0;
#pragma unroll 1
            for (; u + 1 < units; u += 2) {     // four elements per accumulate step
              const uint4 X0 = ldg128(xp + u), Y0 = ldg128(yp + u);
              const uint4 X1 = ldg128(xp + u + 1), Y1 = ldg128(yp + u + 1);
              const uint32_t xa[2] = {X0.x, X0.y}, xb[2] = {X0.z, X0.w};
              const uint32_t xc[2] = {X1.x, X1.y}, xd[2] = {X1.z, X1.w};
              const uint32_t ya[2] = {Y0.x, Y0.y}, yb[2] = {Y0.z, Y0.w};
              const uint32_t yc[2] = {Y1.x, Y1.y}, yd[2] = {Y1.z, Y1.w};
              acc.add4(xa, ya, xb, yb, xc, yc, xd, yd);
            }
            if (u < units) direct_unit<Q>(ldg128(xp + u), ldg128(yp + u), &acc);
          } else if constexpr (Q > 32) {
#pragma unroll 1
            for (int u = 0; u < units; u++) direct_unit<Q>(ldg128(xp + u), ldg128(yp + u), &acc);
          } else {
#if BX_PREFETCH_Q32
            // register double buffer of one unit (q = 17..32)
            uint4 X = ldg128(xp), Y = ldg128(yp);
#pragma unroll 2
            for (int u = 0; u < units; u++) {
              uint4 NX = X, NY = Y;
              if (u + 1 < units) {
                NX = ldg128(xp + u + 1);
                NY = ldg128(yp + u + 1);
              }
              direct_unit<Q>(X, Y, &acc);
              X = NX;
              Y = NY;
            }
#else
#pragma unroll kQ32Unroll
            for (int u = 0; u < units; u++) direct_unit<Q>(ldg128(xp + u), ldg128(yp + u), &acc);
#endif
          }
          c = acc.unreduced();
        }
      }
      z = reduce<Q>(c);
    }
  }
  direct_store<Q>(a, l, z, lane);
}

// ------------------------------------------------------- period kernel
//
// Aligned fast path for q = 24, 40, 48, 56 (multiples of 8 that are not powers
// of two; q*n a multiple of 128, 16-byte aligned windows, word-aligned output):
// element starts repeat every lcm(q, 128) bits, a "period" of q/g 128-bit units
// holding 128/g elements (g = gcd(q, 128); q = 56: 7 units, 16 elements).  One
// thread per block loads a period's units straight from HBM and extracts every
// element with compile-time funnel shifts -- no shared-memory staging, no
// runtime bit offsets, no tile barriers (what the TMA kernel pays for arbitrary
// offsets).  A warp's 32 consecutive outputs are 32*q bits = q whole words,
// assembled in a per-warp shared buffer.
__host__ __device__ constexpr int cgcd(int a, int b) { return b ? cgcd(b, a % b) : a; }

__host__ __device__ constexpr bool period_q(int q) {
  return q == 24 || q == 40 || q == 48 || q == 56;
}

#ifndef BX_PERIOD_MINB
#define BX_PERIOD_MINB 4
#endif
#ifndef BX_PERIOD_PAIR
#define BX_PERIOD_PAIR 1
#endif

#ifndef BX_PERIOD_QUADLOOP
#define BX_PERIOD_QUADLOOP 1
#endif
#ifndef BX_PERIOD_QUAD_PREFETCH
#define BX_PERIOD_QUAD_PREFETCH 0
#endif
#ifndef BX_PERIOD_QUAD_UNROLL
#define BX_PERIOD_QUAD_UNROLL 1
#endif
constexpr int kPeriodQuadUnroll = BX_PERIOD_QUAD_UNROLL;

#ifndef BX_PERIOD_THREADS
#define BX_PERIOD_THREADS 128
#endif

template <int Q>
__global__ void __launch_bounds__(BX_PERIOD_THREADS, BX_PERIOD_MINB) eq_period_kernel(const DirectArgs a) {
  constexpr int EW = cdiv(Q, 32);
  constexpr int G = cgcd(Q, 128);
  constexpr int UNITS = Q / G;          // 128-bit units per period
  constexpr int ELEMS = 128 / G;        // elements per period (even)
  constexpr int WORDS = 4 * UNITS;
  __shared__ uint32_t sout[BX_PERIOD_THREADS / 32][Q + 1];
  pdl_entry();
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Wide<EW> z = wzero<EW>();
  if (l < a.nblocks) {
    const uint4* xp = a.x + l * a.units;
    const uint4* yp = a.y + l * a.units;
    BX_CHECK((l + 1) * a.units - 1, a.x_limit, 7);
    BX_CHECK((l + 1) * a.units - 1, a.y_limit, 7);
    using H = TileHoles<Q>;
    H acc;
    acc.init();
    if constexpr (BX_PERIOD_QUADLOOP && has_quad<H>::value && Q == 56) {
      // Four elements are Q/8 whole words and the shift pattern repeats with
      // them, so the loop runs over quads with 32-bit loads: a body of one quad
      // (650 instructions at q = 56) instead of a whole period (2,562, which
      // missed the instruction cache: ncu no_instruction 0.57 warps per issue).
      // c2p 0.270 -> 0.261 ms; at q = 24 / 40 / 48 the 32-bit loads make the
      // kernel L1-wavefront bound (-35% / -6% / -60%), so only q = 56 takes it
      // (profiles/r02/dp2a_sweep.txt, sweep 8).
      constexpr int WP = Q / 8;
      const uint32_t* xq = reinterpret_cast<const uint32_t*>(xp);
      const uint32_t* yq = reinterpret_cast<const uint32_t*>(yp);
      const int quads = a.units * 32 / Q;
#if BX_PERIOD_QUAD_PREFETCH
      uint32_t nx[WP], ny[WP];
#pragma unroll
      for (int i = 0; i < WP; i++) {
        nx[i] = __ldg(xq + i);
        ny[i] = __ldg(yq + i);
      }
#endif
#pragma unroll kPeriodQuadUnroll
      for (int k = 0; k < quads; k++) {
        uint32_t xw[WP], yw[WP];
#if BX_PERIOD_QUAD_PREFETCH
        // register double buffer: the next quad's words are in flight while
        // this one multiplies
#pragma unroll
        for (int i = 0; i < WP; i++) {
          xw[i] = nx[i];
          yw[i] = ny[i];
        }
        if (k + 1 < quads) {
#pragma unroll
          for (int i = 0; i < WP; i++) {
            nx[i] = __ldg(xq + (k + 1) * WP + i);
            ny[i] = __ldg(yq + (k + 1) * WP + i);
          }
        }
#else
#pragma unroll
        for (int i = 0; i < WP; i++) {
          xw[i] = __ldg(xq + k * WP + i);
          yw[i] = __ldg(yq + k * WP + i);
        }
#endif
        uint32_t xe[4][EW], ye[4][EW];
#pragma unroll
        for (int e = 0; e < 4; e++) {
#pragma unroll
          for (int i = 0; i < EW; i++) {
            const int o = e * Q + 32 * i;
            const int w = o >> 5, sh = o & 31;
            const uint32_t x1 = w + 1 < WP ? xw[w + 1 < WP ? w + 1 : 0] : 0u;
            const uint32_t y1 = w + 1 < WP ? yw[w + 1 < WP ? w + 1 : 0] : 0u;
            xe[e][i] = sh ? __funnelshift_r(xw[w], x1, sh) : xw[w];
            ye[e][i] = sh ? __funnelshift_r(yw[w], y1, sh) : yw[w];
          }
          if constexpr (Q % 32) {
            constexpr uint32_t m = (1u << (Q % 32)) - 1u;
            xe[e][EW - 1] &= m; ye[e][EW - 1] &= m;
          }
        }
        acc.add4(xe[0], ye[0], xe[1], ye[1], xe[2], ye[2], xe[3], ye[3]);
      }
      z = reduce<Q>(acc.unreduced());
    } else {
    const int periods = a.units / UNITS;
#pragma unroll 1
    for (int p = 0; p < periods; p++) {
      uint32_t xw[WORDS], yw[WORDS];
#pragma unroll
      for (int u = 0; u < UNITS; u++) {
        const uint4 X = ldg128(xp + p * UNITS + u), Y = ldg128(yp + p * UNITS + u);
        xw[4 * u] = X.x; xw[4 * u + 1] = X.y; xw[4 * u + 2] = X.z; xw[4 * u + 3] = X.w;
        yw[4 * u] = Y.x; yw[4 * u + 1] = Y.y; yw[4 * u + 2] = Y.z; yw[4 * u + 3] = Y.w;
      }
      // element e of the period: compile-time funnel shifts
      auto elem = [&](int e, uint32_t (&xe)[EW], uint32_t (&ye)[EW]) {
#pragma unroll
        for (int i = 0; i < EW; i++) {
          const int o = e * Q + 32 * i;
          const int w = o >> 5, sh = o & 31;
          const uint32_t x1 = w + 1 < WORDS ? xw[w + 1] : 0u, y1 = w + 1 < WORDS ? yw[w + 1] : 0u;
          xe[i] = sh ? __funnelshift_r(xw[w], x1, sh) : xw[w];
          ye[i] = sh ? __funnelshift_r(yw[w], y1, sh) : yw[w];
        }
        if constexpr (Q % 32) {
          constexpr uint32_t m = (1u << (Q % 32)) - 1u;
          xe[EW - 1] &= m; ye[EW - 1] &= m;
        }
      };
      if constexpr (has_quad<H>::value && ELEMS % 4 == 0) {
#pragma unroll
        for (int e = 0; e < ELEMS; e += 4) {
          uint32_t xe[4][EW], ye[4][EW];
#pragma unroll
          for (int k = 0; k < 4; k++) elem(e + k, xe[k], ye[k]);
          acc.add4(xe[0], ye[0], xe[1], ye[1], xe[2], ye[2], xe[3], ye[3]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < ELEMS; e += 2) {
          uint32_t xa[EW], ya[EW], xb[EW], yb[EW];
          elem(e, xa, ya);
          elem(e + 1, xb, yb);
#if BX_PERIOD_PAIR
          acc.add2(xa, ya, xb, yb);
#else
          acc.add(xa, ya);
          acc.add(xb, yb);
#endif
        }
      }
    }
    z = reduce<Q>(acc.unreduced());
    }
  }
  // the warp's 32 blocks own output words [first*Q/32, first*Q/32 + Q)
  uint32_t* so = sout[warp];
  for (int i = lane; i <= Q; i += 32) so[i] = 0u;
  __syncwarp();
  if (l < a.nblocks) {
    const int bit = lane * Q, w0 = bit >> 5, sh = bit & 31;
#pragma unroll
    for (int i = 0; i <= EW; i++) {
      const uint32_t lo = at(z, i - 1), hi = at(z, i);
      const uint32_t v = sh ? __funnelshift_l(lo, hi, sh) : hi;
      if (v) atomicOr(&so[w0 + i], v);
    }
  }
  __syncwarp();
  const int64_t first = l - lane;
  if (first < a.nblocks) {
    const int64_t nv = (a.nblocks - first) < 32 ? (a.nblocks - first) : 32;
    const int64_t bits = nv * Q;
    const int words = (int)((bits + 31) >> 5);
    for (int i = lane; i < words; i += 32) {
      const int64_t gw = first / 32 * Q + i;
      BX_CHECK(gw, a.out_words, 8);
      if ((int64_t)(i + 1) * 32 <= bits) {
        a.out[gw] = so[i];
      } else {
        const uint32_t mask = (1u << (bits & 31)) - 1u;
        atomicAnd(&a.out[gw], ~mask);
        atomicOr(&a.out[gw], so[i] & mask);
      }
    }
  }
}

}  // namespace bx
