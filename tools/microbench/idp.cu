// IDP.2A / IDP.4A issue-rate microbenchmark for sm_100a: is the 16x8 two-term
// dot product (dp2a) a full-rate instruction, which pipe does it occupy, and does
// it co-issue with LOP3 the way IMAD does?  (Feeds the q = 16 / 32 "dot-product
// holes" kernels: one IDP.2A multiplies two holed 16-bit halves by two holed
// bytes and adds the two products.)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define ILP 8

#define CHAIN_KERNEL(NAME, ASM)                                                 \
  __global__ void NAME(uint32_t* out, uint32_t s) {                            \
    uint32_t a[ILP], b = s * 2654435761u + threadIdx.x, c = s ^ 0x9e3779b9u;    \
    for (int i = 0; i < ILP; i++) a[i] = threadIdx.x * (i + 1) + s;            \
    for (int it = 0; it < ITERS; it++) {                                       \
      _Pragma("unroll") for (int i = 0; i < ILP; i++) {                        \
        asm volatile(ASM : "+r"(a[i]) : "r"(b), "r"(c));                       \
      }                                                                        \
    }                                                                          \
    uint32_t r = 0;                                                            \
    for (int i = 0; i < ILP; i++) r ^= a[i];                                   \
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;                            \
  }

CHAIN_KERNEL(k_imad, "mad.lo.u32 %0, %0, %1, %2;")
CHAIN_KERNEL(k_dp2a_lo, "dp2a.lo.u32.u32 %0, %0, %1, %2;")
CHAIN_KERNEL(k_dp2a_hi, "dp2a.hi.u32.u32 %0, %0, %1, %2;")
CHAIN_KERNEL(k_dp2a_z, "dp2a.lo.u32.u32 %0, %0, %1, 0;")
CHAIN_KERNEL(k_dp4a, "dp4a.u32.u32 %0, %0, %1, %2;")

#define MIX_KERNEL(NAME, ASM_A, ASM_L, NL)                                      \
  __global__ void NAME(uint32_t* out, uint32_t s) {                            \
    uint32_t a[ILP], l[ILP];                                                   \
    uint32_t b = s * 2654435761u + threadIdx.x, c = s ^ 0x9e3779b9u;            \
    for (int i = 0; i < ILP; i++) { a[i] = threadIdx.x * (i + 1) + s; l[i] = a[i] * 3u; } \
    for (int it = 0; it < ITERS; it++) {                                       \
      _Pragma("unroll") for (int i = 0; i < ILP; i++) {                        \
        asm volatile(ASM_A : "+r"(a[i]) : "r"(b), "r"(c));                     \
        _Pragma("unroll") for (int k = 0; k < NL; k++)                         \
          asm volatile(ASM_L : "+r"(l[i]) : "r"(b), "r"(c));                   \
      }                                                                        \
    }                                                                          \
    uint32_t r = 0;                                                            \
    for (int i = 0; i < ILP; i++) r ^= a[i] ^ l[i];                            \
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;                            \
  }

MIX_KERNEL(k_imad_lop, "mad.lo.u32 %0, %0, %1, %2;", "lop3.b32 %0, %0, %1, %2, 0x78;", 1)
MIX_KERNEL(k_dp2a_lop, "dp2a.lo.u32.u32 %0, %0, %1, %2;", "lop3.b32 %0, %0, %1, %2, 0x78;", 1)
MIX_KERNEL(k_dp2a_imad, "dp2a.lo.u32.u32 %0, %0, %1, %2;", "mad.lo.u32 %0, %0, %1, %2;", 1)
MIX_KERNEL(k_dp2a_ffma, "dp2a.lo.u32.u32 %0, %0, %1, %2;", "fma.rn.f32 %0, %0, %1, %2;", 1)
MIX_KERNEL(k_dp4a_lop, "dp4a.u32.u32 %0, %0, %1, %2;", "lop3.b32 %0, %0, %1, %2, 0x78;", 1)

typedef void (*kfn)(uint32_t*, uint32_t);

static void run(const char* name, kfn f, double ops_per_step, int sms, int clk_khz) {
  int threads = 256, blocks = sms * 8;
  uint32_t* out; cudaMalloc(&out, sizeof(uint32_t) * threads * blocks);
  f<<<blocks, threads>>>(out, 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) f<<<blocks, threads>>>(out, r + 2);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 5.0 * threads * blocks * (double)ITERS * ILP * ops_per_step;
  double tops = ops / (ms * 1e-3) / 1e12;
  printf("%-12s %8.3f ms  %8.2f T thread-ops/s  (%.1f ops/clk/SM at max clock %d MHz)\n",
         name, ms, tops, tops * 1e12 / (sms * (double)clk_khz * 1e3), clk_khz / 1000);
  cudaFree(out);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, clk);
  int n = p.multiProcessorCount;
  run("imad", k_imad, 1, n, clk);
  run("dp2a.lo", k_dp2a_lo, 1, n, clk);
  run("dp2a.hi", k_dp2a_hi, 1, n, clk);
  run("dp2a.lo+0", k_dp2a_z, 1, n, clk);
  run("dp4a", k_dp4a, 1, n, clk);
  run("imad+lop3", k_imad_lop, 2, n, clk);
  run("dp2a+lop3", k_dp2a_lop, 2, n, clk);
  run("dp2a+imad", k_dp2a_imad, 2, n, clk);
  run("dp2a+ffma", k_dp2a_ffma, 2, n, clk);
  run("dp4a+lop3", k_dp4a_lop, 2, n, clk);
  return 0;
}
