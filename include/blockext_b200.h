/*
 * blockext_b200.h -- C ABI of the B200 block extractor (libbx_b200.so).
 *
 * Plain pointers and sizes only.  Every compute entry point is asynchronous on
 * the given cudaStream_t (passed as void*, NULL = legacy default stream) and
 * returns 0 on success or a negative BX_E* code; bx_last_error() then holds a
 * thread-local message.  All buffers are device buffers owned by the caller;
 * the library keeps no allocations between calls.
 *
 * The reference (`blockext`, pure Python) has no FFI; these entry points
 * replace the compute of its Python functions, which the package
 * paper_2402_14607_b200 re-exposes with the reference's signatures:
 *
 *   bx_extract_eq   <- Extraction._blocks + run_parallel + ext_ip + GFContext.mul
 *                      + BitWriter      (pkg/src/blockext/extractor.py:182-208,
 *                      :94-130, :77-87; gf2q.py:156-169; bitio.py:67-88)
 *   bx_pack         <- sources._pack_samples (pkg/src/blockext/sources.py:116-121)
 *                      and the bit packing inside generate() (:133-140)
 *   bx_modulus_exponents <- _moduli.MODULUS_EXPONENTS / modulus_int
 *                      (pkg/src/blockext/_moduli.py:13-151)
 */
#ifndef BLOCKEXT_B200_H
#define BLOCKEXT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BX_OK 0
#define BX_EINVAL -1   /* bad argument (message says which)            */
#define BX_ECUDA -2    /* CUDA launch/runtime error                      */
#define BX_ERANGE -3   /* field width outside 1..128 (reference CapacityError) */

/* ABI version (major*100 + minor). */
int bx_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char* bx_last_error(void);

/* Default modulus of GF(2^q): writes its exponents, highest first, to exps[5]
 * and returns how many there are (2, 3 or 5); BX_ERANGE for q outside 1..128. */
int bx_modulus_exponents(int q, int* exps);

/*
 * Equal-width two-source extraction of `nblocks` blocks.
 *
 * Block l reads bits [x_bit0 + l*q*n, x_bit0 + (l+1)*q*n) of the LSB-first bit
 * stream at x (and likewise y), splits them into n q-bit elements and writes
 *   z_l = sum_j x_{l,j} * y_{l,j}  in GF(2^q) (default modulus)
 * to bits [out_bit0 + l*q, out_bit0 + (l+1)*q) of out.  Other bits of out are
 * preserved (boundary words are updated atomically).
 *
 * x, y, out: device pointers, 4-byte aligned; the kernels run on the device
 * of `stream` (non-NULL) or else the device that owns x -- never out's: out may
 * be memory of a peer GPU mapped into this process
 * (CUDA IPC / peer access: the outputs are then stored over NVLink -- how
 * sharding.distributed_extract(gather="peer") gathers ranks' ranges into rank
 * 0's buffer).  x_bytes / y_bytes: bytes of
 * valid stream data; the buffers must stay readable up to round_up(x_bytes, 16)
 * + 16 bytes (the TMA-bulk path copies whole 16-byte granules).  16-byte
 * aligned x and y select the aligned kernels (direct, or persistent TMA-bulk).
 * Requires x_bit0 + nblocks*q*n <= 8*x_bytes (same for y).  y and out must be
 * local to the compute device or on a peer it can access (else BX_EINVAL).
 */
int bx_extract_eq(const void* x, int64_t x_bytes, int64_t x_bit0,
                  const void* y, int64_t y_bytes, int64_t y_bit0,
                  int q, int n, int64_t nblocks,
                  void* out, int64_t out_bit0, void* stream);

/*
 * Incremental-width extraction (extract_neq): block k (0-based) has width
 * q1 + k*step (all <= 128) and reads the next (q1 + k*step)*n bits of each
 * stream, starting at bit 0; outputs are concatenated from bit 0 of out.
 * Replaces the neq schedule of Extraction._blocks (extractor.py:170-173,
 * 188-205).  One launch per distinct width.
 */
int bx_extract_neq(const void* x, int64_t x_bytes, const void* y, int64_t y_bytes, int q1,
                   int step, int n, int64_t nblocks, void* out, void* stream);

/*
 * Launch geometry bx_extract_eq would use (for tests, benches and profiling):
 * threads per block-pair group, blocks per CTA tile, staged (1) or direct (0),
 * CTA threads, dynamic shared memory bytes, grid size, and kernel family
 * (bit 0: 0 = diag, 1 = holes; bit 1: aligned direct kernel; bit 2:
 * persistent TMA-bulk staged kernel), for
 * 16-byte aligned buffers starting at bit 0.  Any output pointer may be NULL.
 */
int bx_launch_info(int q, int n, int64_t nblocks, int* tpb, int* tile, int* staged,
                   int* threads, int* smem_bytes, int64_t* grid, int* family);

/*
 * One-call extraction of a short run from HOST memory (the real-time path:
 * one call per capture chunk): reads bytes [0, ceil((x_bit0 + nblocks*q*n)/8))
 * of x (x_bytes = what the caller can provide; must cover that) and likewise
 * y, stages both through a per-device cached pinned buffer, copies them to
 * `device` with one H2D, runs bx_extract_eq and writes the packed output --
 * ceil(nblocks*q/8) bytes, last byte zero-padded -- to host memory `out`.
 * Synchronous; thread-safe (calls on one device are serialised).  For long
 * runs use bx_extract_eq on device buffers with your own copy pipeline.
 */
int bx_extract_eq_host(const void* x, int64_t x_bytes, int64_t x_bit0, const void* y,
                       int64_t y_bytes, int64_t y_bit0, int q, int n, int64_t nblocks,
                       void* out, int device);

/*
 * Extension beyond the reference's q <= 128 cap (its GFContext raises
 * CapacityError above 128, gf2q.py:111-112): equal-width blocks over
 * GF(2^256) with P = x^256 + x^10 + x^5 + x^2 + 1 (the first irreducible of
 * the reference's modulus scan order, _moduli.py:1-11), for BASELINE config 3
 * as stated (1024-bit blocks -> 256 output bits: q = 256, n = 4).  Block l
 * reads bytes [32*n*l, 32*n*(l+1)) of x and y (16-byte aligned) and writes
 * words [out_word0 + 8*l, +8) of out (whole 32-bit words; out + 4*out_word0
 * 16-byte aligned).  q must be 256 (BX_ERANGE otherwise).
 */
int bx_extract_eq_wide(const void* x, int64_t x_bytes, const void* y, int64_t y_bytes, int q,
                       int n, int64_t nblocks, void* out, int64_t out_word0, void* stream);

/*
 * Sample packer: the low b bits of sample i go to stream bits
 * [out_bit0 + i*b, out_bit0 + (i+1)*b).  samples: `count` little-endian
 * unsigned integers of elem_bytes (1, 2, 4 or 8) each; b in 1..8*elem_bytes.
 * Bits of out outside the written range are preserved; out must be 4-byte
 * aligned.
 */
int bx_pack(const void* samples, int elem_bytes, int b, int64_t count,
            void* out, int64_t out_bit0, void* stream);

/*
 * Inner products over GF(2^q) with a caller-chosen modulus (GFContext(q,
 * modulus), reference gf2q.py:99-183): out[v] = sum_j x[v][j] * y[v][j] for
 * nvec vectors of n elements.  Elements, the modulus's low part (modulus minus
 * x^q) and outputs are 128-bit little-endian (4 uint32 words each), device
 * memory.  A simple per-vector kernel for API calls, not the extraction path.
 */
int bx_gf_ip_generic(int q, const void* modulus_low, const void* x, const void* y, int n,
                     int64_t nvec, void* out, void* stream);

/*
 * Powers over GF(2^q) with a caller-chosen modulus (GFContext.pow / inv,
 * reference gf2q.py:171-189): out[v] = x[v]^e[v], square-and-multiply over
 * e's bits in one launch (one thread per element).  x, e, out: count 128-bit
 * little-endian values; modulus_low as for bx_gf_ip_generic.  Callers reduce
 * e modulo 2^q - 1 for nonzero x (the multiplicative group's order).
 */
int bx_gf_pow(int q, const void* modulus_low, const void* x, const void* e, int64_t count,
              void* out, void* stream);

/* ---- native streaming pipeline ----------------- */

/*
 * Push-based equal-width extraction for producers outside Python.  Each push
 * hands over the next nbytes (<= chunk_bytes) of both streams from host
 * memory (copied before the call returns, so the caller may reuse them);
 * every block completed by the bytes so far is extracted on `device`.
 * Partial blocks and the last partial output byte carry over, so the
 * concatenated outputs of any push sequence (then drain, then flush) equal
 * one run over the concatenated streams (reference extractor.py:182-208,
 * bitio.py:74-88; replaces the reference CLI's file loop, cli.py:88-129).
 *
 * bx_pipe_create: synchronous pipe -- each push returns its own output.
 * bx_pipe_create_async: `depth` (1..4) pushes in flight; a push enqueues its
 *   host copy, H2D, kernel and D2H and returns the output of the pushes
 *   older than the newest depth-1 (depth 2: push k returns push k-1's bytes,
 *   and push k's copies overlap push k-1's kernel and D2H).
 * The whole output bytes returned by a call are written to out (capacity
 * out_cap; bx_pipe_max_output(p) bytes per retired push suffice),
 * *out_bytes = count.  Errors set bx_last_error(); after a BX_ECUDA the pipe
 * must be destroyed.
 */
typedef struct bx_pipe bx_pipe;
bx_pipe* bx_pipe_create(int q, int n, int64_t chunk_bytes, int device);
bx_pipe* bx_pipe_create_async(int q, int n, int64_t chunk_bytes, int device, int depth);
int bx_pipe_push(bx_pipe* p, const void* x, const void* y, int64_t nbytes, void* out,
                 int64_t out_cap, int64_t* out_bytes);
/* Waits for every push in flight and writes their output (async pipes). */
int bx_pipe_drain(bx_pipe* p, void* out, int64_t out_cap, int64_t* out_bytes);
/* Emits the carried partial output byte (zero padded), if any; requires
 * nothing in flight (drain first). */
int bx_pipe_flush(bx_pipe* p, void* out, int64_t* out_bytes);
/* Largest output one push (or one retired push in a drain) can produce. */
int64_t bx_pipe_max_output(const bx_pipe* p);
/* Blocks extracted so far (or -1 for NULL). */
int64_t bx_pipe_blocks(const bx_pipe* p);
void bx_pipe_destroy(bx_pipe* p);

/* ---- device source simulators ---------------- */

/*
 * Counter-based Bernoulli(p) bits: stream bit i (i = bit0 .. bit0+nbits-1) is
 * 1 iff (splitmix64(seed*0xD1B54A32D192ED03 + i) >> 11) < p*2^53.  Writes
 * ceil(nbits/32) words at out (LSB-first), zero past nbits.  Builder-defined
 * generator of the config-4 block-Markov masks (no reference counterpart).
 */
int bx_bernoulli_bits(void* out, int64_t nbits, double p, uint64_t seed, int64_t bit0,
                      void* stream);

/* In-place inclusive prefix XOR down the rows of a row-major uint32 matrix
 * (rows x row_words): row r := row 0 ^ ... ^ row r.  scratch: device buffer of
 * bx_xor_scan_scratch_bytes(rows, row_words) bytes. */
int64_t bx_xor_scan_scratch_bytes(int64_t rows, int row_words);
int bx_xor_scan_rows(void* matrix, int64_t rows, int row_words, void* scratch, void* stream);

/*
 * Sample path of the reference `markov` source (pkg/src/blockext/sources.py:
 * 141-152): with cum = row-wise cumulative transition table (2^b x 2^b
 * doubles, last column forced to 1.0) and host-drawn uniforms u[0..count),
 * state_i = min(searchsorted(cum[state_{i-1}], u_i, right), 2^b - 1) from
 * start_state; values (uint16) receive state_1 .. state_count.  Segmented
 * parallel walk; scratch: bx_markov_scratch_bytes(count, b) bytes.
 */
int64_t bx_markov_scratch_bytes(int64_t count, int b);
int bx_markov_chain(const void* u, int64_t count, const void* cum, int b, int start_state,
                    void* values, void* scratch, void* stream);

/* ---- exhaustive verification kernels --------- */

/* z[i*2^t + y] = <x0+i, y> over GF(2^q) (default modulus), t = q*n <= 16, for
 * i < nx and all y < 2^t; out: uint16.  Replaces the dense inner-product table
 * of the reference verify.ip_value_table (pkg/src/blockext/verify.py:200-207). */
int bx_ip_table(int q, int n, uint32_t x0, uint32_t nx, void* out, void* stream);

/* counts[i*2^q + v] = #{y < 2^t : <d0+i, y> = v} for i < nd (uint32); the
 * histograms of verify._hadamard_counts (verify.py:262-297). */
int bx_ip_histograms(int q, int n, uint32_t d0, uint32_t nd, void* counts, void* stream);

/* flags[r] = 1 iff counts[r*bins + v] == expected for every v (uint8). */
int bx_rows_uniform(const void* counts, uint32_t nrows, uint32_t bins, uint32_t expected,
                    void* flags, void* stream);

/* Bounds-check violations recorded by a BX_CHECKED build of the library
 * (libbx_b200_checked.so): synchronises the device, returns the count and
 * writes (tag, index, bound) of the first one to first[3] if non-NULL;
 * returns -1 in normal builds. */
int64_t bx_checked_violations(int reset, int64_t* first);

/* Number of kernel launches issued by this process (all threads, all devices)
 * since the last reset (reset != 0 returns the count and zeroes it). */
int64_t bx_launch_count(int reset);

#ifdef __cplusplus
}
#endif

#endif /* BLOCKEXT_B200_H */
