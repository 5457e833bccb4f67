// bx_sources.cu -- device source simulators.
//
//  * bernoulli_bits: counter-based Bernoulli(p) bit stream (SplitMix64 of the
//    bit index), packed LSB-first; defines the builder's block-Markov source
//    of config 4 together with
//  * xor_scan_rows: in-place inclusive prefix XOR down the rows of a
//    row-major word matrix (block k := block k-1 XOR mask_k);
//  * markov_chain: the reference `markov` model's sample path
//    (pkg/src/blockext/sources.py:141-152): state_i = min(searchsorted(
//    cum[state_{i-1}], u_i, side='right'), 2^b - 1) for host-drawn u_i,
//    computed with a segmented parallel walk -- every segment is simulated
//    from every possible entry state, the entry states are chained on one
//    thread, and the segments are replayed from their true entry states.
#include <cstdint>
#include <cuda_runtime.h>

namespace bx {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// bit i = (splitmix64(seed_mix + i) >> 11) < threshold53, i in [bit0, bit0 + 32*nwords)
__global__ void __launch_bounds__(256) bernoulli_bits_kernel(uint32_t* out, int64_t nbits,
                                                             uint64_t seed_mix, int64_t bit0,
                                                             uint64_t threshold53) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w * 32 >= nbits) return;
  uint32_t word = 0;
  const uint64_t base = seed_mix + (uint64_t)(bit0 + 32 * w);
#pragma unroll 8
  for (int k = 0; k < 32; k++) word |= (uint32_t)((splitmix64(base + k) >> 11) < threshold53) << k;
  const int64_t left = nbits - 32 * w;
  if (left < 32) word &= (1u << left) - 1u;
  out[w] = word;
}

// Pass 1: XOR of each column over each segment of `seg` rows.
__global__ void xor_scan_totals(const uint32_t* m, int64_t rows, int cols, int64_t seg,
                                uint32_t* totals) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nseg = (rows + seg - 1) / seg;
  if (t >= nseg * cols) return;
  const int64_t s = t / cols;
  const int c = (int)(t % cols);
  const int64_t r1 = (s + 1) * seg < rows ? (s + 1) * seg : rows;
  uint32_t acc = 0;
  for (int64_t r = s * seg; r < r1; r++) acc ^= m[r * cols + c];
  totals[t] = acc;
}

// Pass 3: replay each segment from its exclusive prefix (totals now hold the
// exclusive prefix of every segment).
__global__ void xor_scan_apply(uint32_t* m, int64_t rows, int cols, int64_t seg,
                               const uint32_t* prefix) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nseg = (rows + seg - 1) / seg;
  if (t >= nseg * cols) return;
  const int64_t s = t / cols;
  const int c = (int)(t % cols);
  const int64_t r1 = (s + 1) * seg < rows ? (s + 1) * seg : rows;
  uint32_t acc = prefix[t];
  for (int64_t r = s * seg; r < r1; r++) {
    acc ^= m[r * cols + c];
    m[r * cols + c] = acc;
  }
}

// Exclusive prefix XOR of a small (nseg x cols) matrix, one thread per column.
__global__ void xor_scan_serial_exclusive(uint32_t* t, int64_t nseg, int cols) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  uint32_t acc = 0;
  for (int64_t s = 0; s < nseg; s++) {
    const uint32_t v = t[s * cols + c];
    t[s * cols + c] = acc;
    acc ^= v;
  }
}

// ---------------------------------------------------------------- markov

__device__ __forceinline__ int markov_step(const double* cum, int size, int s, double u) {
  // searchsorted(cum[s], u, side='right'): first index with cum[s][i] > u
  const double* row = cum + (int64_t)s * size;
  int lo = 0, hi = size;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (row[mid] <= u) lo = mid + 1;
    else hi = mid;
  }
  return lo < size - 1 ? lo : size - 1;
}

// ends[seg * size + c] = state after walking segment seg from entry state c
__global__ void markov_segment_ends(const double* u, int64_t count, const double* cum, int size,
                                    int64_t seg, int* ends) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nseg = (count + seg - 1) / seg;
  if (t >= nseg * size) return;
  const int64_t sg = t / size;
  int s = (int)(t % size);
  const int64_t i1 = (sg + 1) * seg < count ? (sg + 1) * seg : count;
  for (int64_t i = sg * seg; i < i1; i++) s = markov_step(cum, size, s, u[i]);
  ends[t] = s;
}

__global__ void markov_chain_entries(const int* ends, int64_t nseg, int size, int start,
                                     int* entry) {
  if (blockIdx.x | threadIdx.x) return;
  int s = start;
  for (int64_t sg = 0; sg < nseg; sg++) {
    entry[sg] = s;
    s = ends[sg * size + s];
  }
}

__global__ void markov_replay(const double* u, int64_t count, const double* cum, int size,
                              int64_t seg, const int* entry, uint16_t* values) {
  const int64_t sg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nseg = (count + seg - 1) / seg;
  if (sg >= nseg) return;
  int s = entry[sg];
  const int64_t i1 = (sg + 1) * seg < count ? (sg + 1) * seg : count;
  for (int64_t i = sg * seg; i < i1; i++) {
    s = markov_step(cum, size, s, u[i]);
    values[i] = (uint16_t)s;
  }
}

// ----------------------------------------------------------------- launch

static unsigned blocks_for(int64_t n) { return (unsigned)((n + 255) / 256); }

cudaError_t launch_bernoulli(uint32_t* out, int64_t nbits, uint64_t seed, int64_t bit0, double p,
                             cudaStream_t st) {
  if (nbits <= 0) return cudaSuccess;
  const int64_t nwords = (nbits + 31) / 32;
  double t = p * 9007199254740992.0;  // 2^53
  const uint64_t thr = t >= 9007199254740992.0 ? (1ull << 53) : (t <= 0 ? 0ull : (uint64_t)t);
  const uint64_t mix = seed * 0xD1B54A32D192ED03ull;
  bernoulli_bits_kernel<<<blocks_for(nwords), 256, 0, st>>>(out, nbits, mix, bit0, thr);
  return cudaGetLastError();
}

// Segments are sized so there are at most kScanSegs of them: the serial
// exclusive pass over segment totals stays short and the scratch small.
constexpr int64_t kScanSegs = 4096;

int64_t xor_scan_scratch_words(int64_t rows, int cols) {
  int64_t seg = (rows + kScanSegs - 1) / kScanSegs;
  if (seg < 64) seg = 64;
  return ((rows + seg - 1) / seg) * cols;
}

cudaError_t launch_xor_scan(uint32_t* m, int64_t rows, int cols, uint32_t* scratch,
                            cudaStream_t st) {
  if (rows <= 1) return cudaSuccess;
  int64_t seg = (rows + kScanSegs - 1) / kScanSegs;
  if (seg < 64) seg = 64;
  const int64_t nseg = (rows + seg - 1) / seg;
  const int64_t n = nseg * cols;
  xor_scan_totals<<<blocks_for(n), 256, 0, st>>>(m, rows, cols, seg, scratch);
  xor_scan_serial_exclusive<<<(unsigned)((cols + 127) / 128), 128, 0, st>>>(scratch, nseg, cols);
  xor_scan_apply<<<blocks_for(n), 256, 0, st>>>(m, rows, cols, seg, scratch);
  return cudaGetLastError();
}

int64_t markov_scratch_ints(int64_t count, int b) {
  int64_t seg = (count + kScanSegs - 1) / kScanSegs;
  if (seg < 64) seg = 64;
  return ((count + seg - 1) / seg) * ((1 << b) + 1);
}

cudaError_t launch_markov(const double* u, int64_t count, const double* cum, int b, int start,
                          uint16_t* values, int* scratch, cudaStream_t st) {
  const int size = 1 << b;
  if (count <= 0) return cudaSuccess;
  // segment ends table (nseg * size ints) followed by the nseg entry states
  int64_t seg = (count + kScanSegs - 1) / kScanSegs;
  if (seg < 64) seg = 64;
  const int64_t nseg = (count + seg - 1) / seg;
  int* ends = scratch;
  int* entry = scratch + nseg * size;
  markov_segment_ends<<<blocks_for(nseg * size), 256, 0, st>>>(u, count, cum, size, seg, ends);
  markov_chain_entries<<<1, 32, 0, st>>>(ends, nseg, size, start, entry);
  markov_replay<<<blocks_for(nseg), 256, 0, st>>>(u, count, cum, size, seg, entry, values);
  return cudaGetLastError();
}

}  // namespace bx
