/* Plain-C consumer of the C ABI (include/blockext_b200.h): no Python, no torch.
 * Allocates device buffers with the CUDA runtime, extracts random blocks for a
 * few shapes and compares with the CPU oracle library (oracle/_build). */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>

#include "blockext_b200.h"

int bxo_extract_eq(const uint8_t*, int64_t, const uint8_t*, int64_t, int, int, int64_t, const int*,
                   int, uint8_t*, int64_t, int, int);

static uint64_t rng = 88172645463325252ull;
static uint8_t rb(void) {
  rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
  return (uint8_t)rng;
}

int main(void) {
  const int shapes[][3] = {{4, 64, 5000}, {128, 8, 700}, {56, 48, 333}, {13, 7, 999}, {1, 24, 64}};
  int fails = 0;
  for (unsigned s = 0; s < sizeof shapes / sizeof shapes[0]; s++) {
    const int q = shapes[s][0], n = shapes[s][1];
    const int64_t k = shapes[s][2];
    const int64_t bytes = (k * q * n + 7) / 8;
    const int64_t alloc = ((bytes + 15) / 16) * 16 + 16;
    const int64_t obytes = (k * q + 7) / 8;
    uint8_t *hx = calloc(alloc, 1), *hy = calloc(alloc, 1), *ho = calloc(obytes + 16, 1),
            *want = calloc(obytes + 16, 1);
    for (int64_t i = 0; i < bytes; i++) { hx[i] = rb(); hy[i] = rb(); }
    void *dx, *dy, *dout;
    cudaMalloc(&dx, alloc); cudaMalloc(&dy, alloc); cudaMalloc(&dout, obytes + 16);
    cudaMemcpy(dx, hx, alloc, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, hy, alloc, cudaMemcpyHostToDevice);
    cudaMemset(dout, 0, obytes + 16);
    int rc = bx_extract_eq(dx, bytes, 0, dy, bytes, 0, q, n, k, dout, 0, NULL);
    if (rc) { printf("q=%d n=%d: rc=%d %s\n", q, n, rc, bx_last_error()); fails++; continue; }
    cudaMemcpy(ho, dout, obytes, cudaMemcpyDeviceToHost);
    int exps[5];
    int ne = bx_modulus_exponents(q, exps);
    bxo_extract_eq(hx, 0, hy, 0, q, n, k, exps, ne, want, 0, 1, 1);
    int ok = memcmp(ho, want, obytes) == 0;
    printf("q=%d n=%d blocks=%lld: %s\n", q, n, (long long)k, ok ? "ok" : "MISMATCH");
    fails += !ok;
    cudaFree(dx); cudaFree(dy); cudaFree(dout);
    free(hx); free(hy); free(ho); free(want);
  }
  /* native streaming pipeline: uneven pushes == one run over the concatenation */
  {
    const int q = 4, n = 64;
    const int64_t total = 3000017, chunk = 1 << 20;
    uint8_t *hx = malloc(total), *hy = malloc(total), *got = calloc(total, 1), *want = calloc(total, 1);
    for (int64_t i = 0; i < total; i++) { hx[i] = rb(); hy[i] = rb(); }
    bx_pipe* p = bx_pipe_create(q, n, chunk, 0);
    int64_t pos = 0, outpos = 0, got_bytes = 0;
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0); cudaEventCreate(&t1);
    cudaEventRecord(t0, 0);
    while (pos < total) {
      int64_t step = (pos / 7919) % 3 == 0 ? 12345 : chunk;
      if (step > total - pos) step = total - pos;
      if (bx_pipe_push(p, hx + pos, hy + pos, step, got + outpos, total - outpos, &got_bytes)) { fails++; break; }
      pos += step; outpos += got_bytes;
    }
    bx_pipe_flush(p, got + outpos, &got_bytes); outpos += got_bytes;
    cudaEventRecord(t1, 0); cudaEventSynchronize(t1);
    float ms = 0; cudaEventElapsedTime(&ms, t0, t1);
    const int64_t k = bx_pipe_blocks(p);
    int exps[5];
    int ne = bx_modulus_exponents(q, exps);
    bxo_extract_eq(hx, 0, hy, 0, q, n, k, exps, ne, want, 0, 1, 1);
    const int ok = k == total * 8 / (q * n) && outpos == (k * q + 7) / 8 && memcmp(got, want, outpos) == 0;
    printf("pipe q=%d n=%d blocks=%lld: %s (%.1f Gbit/s raw, synchronous pushes)\n", q, n, (long long)k,
           ok ? "ok" : "MISMATCH", 2.0 * 8 * total / (ms * 1e-3) / 1e9);
    fails += !ok;
    bx_pipe_destroy(p);
    free(hx); free(hy); free(got); free(want);
  }
  /* async pipe (2 pushes in flight) + drain + flush: same bytes as one run */
  {
    const int q = 16, n = 64;
    const int64_t total = 2000003, chunk = 1 << 19;
    uint8_t *hx = malloc(total), *hy = malloc(total), *want = calloc(total, 1);
    for (int64_t i = 0; i < total; i++) { hx[i] = rb(); hy[i] = rb(); }
    bx_pipe* p = bx_pipe_create_async(q, n, chunk, 0, 2);
    const int64_t cap = 2 * bx_pipe_max_output(p);
    uint8_t* got = calloc(total + cap, 1);
    int64_t pos = 0, outpos = 0, got_bytes = 0;
    while (pos < total) {
      int64_t step = (pos / 4099) % 2 ? 7777 : chunk;
      if (step > total - pos) step = total - pos;
      if (bx_pipe_push(p, hx + pos, hy + pos, step, got + outpos, cap, &got_bytes)) {
        printf("async push: %s\n", bx_last_error()); fails++; break;
      }
      pos += step; outpos += got_bytes;
    }
    if (bx_pipe_drain(p, got + outpos, cap, &got_bytes)) fails++;
    outpos += got_bytes;
    bx_pipe_flush(p, got + outpos, &got_bytes); outpos += got_bytes;
    const int64_t k = bx_pipe_blocks(p);
    int exps[5];
    int ne = bx_modulus_exponents(q, exps);
    bxo_extract_eq(hx, 0, hy, 0, q, n, k, exps, ne, want, 0, 1, 1);
    const int ok = k == total * 8 / (q * n) && outpos == (k * q + 7) / 8 && memcmp(got, want, outpos) == 0;
    printf("async pipe q=%d n=%d blocks=%lld: %s\n", q, n, (long long)k, ok ? "ok" : "MISMATCH");
    fails += !ok;
    bx_pipe_destroy(p);
    free(hx); free(hy); free(got); free(want);
  }
  /* one-call host extraction at a bit offset (config-1 shape) */
  {
    const int q = 32, n = 4;
    const int64_t k = 8192, bit0 = 5;
    const int64_t bytes = (bit0 + k * q * n + 7) / 8;
    uint8_t *hx = malloc(bytes), *hy = malloc(bytes), *got = calloc(k * q / 8, 1), *want = calloc(k * q / 8 + 16, 1);
    for (int64_t i = 0; i < bytes; i++) { hx[i] = rb(); hy[i] = rb(); }
    int rc = bx_extract_eq_host(hx, bytes, bit0, hy, bytes, bit0, q, n, k, got, 0);
    int exps[5];
    int ne = bx_modulus_exponents(q, exps);
    bxo_extract_eq(hx, bit0, hy, bit0, q, n, k, exps, ne, want, 0, 1, 1);
    const int ok = rc == 0 && memcmp(got, want, k * q / 8) == 0;
    printf("host one-call q=%d n=%d blocks=%lld: %s\n", q, n, (long long)k, ok ? "ok" : "MISMATCH");
    fails += !ok;
    if (bx_extract_eq_host(hx, bytes - 1, bit0, hy, bytes, bit0, q, n, k, got, 0) != BX_EINVAL) fails++;
    free(hx); free(hy); free(got); free(want);
  }
  /* error path: field width beyond the cap */
  if (bx_extract_eq(NULL, 0, 0, NULL, 0, 0, 200, 4, 1, NULL, 0, NULL) != BX_ERANGE) fails++;
  printf("launches=%lld version=%d fails=%d\n", (long long)bx_launch_count(0), bx_version(), fails);
  return fails != 0;
}
