// Integer-pipe issue-rate microbenchmark for sm_100a: LOP3, SHF, IMAD, IMAD.WIDE
// and a LOP3+IMAD.WIDE mix.  Reports thread-ops per clock per SM and T ops/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define ILP 8

__global__ void k_lop3(uint32_t* out, uint32_t s) {
  uint32_t a[ILP], b = s * 2654435761u + threadIdx.x, c = s ^ 0x9e3779b9u;
  for (int i = 0; i < ILP; i++) a[i] = threadIdx.x * (i + 1) + s;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x78;" : "+r"(a[i]) : "r"(b), "r"(c));
    }
  }
  uint32_t r = 0;
  for (int i = 0; i < ILP; i++) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_shf(uint32_t* out, uint32_t s) {
  uint32_t a[ILP], b = s * 2654435761u + threadIdx.x;
  for (int i = 0; i < ILP; i++) a[i] = threadIdx.x * (i + 1) + s;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(a[i]) : "r"(b));
    }
  }
  uint32_t r = 0;
  for (int i = 0; i < ILP; i++) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_imad(uint32_t* out, uint32_t s) {
  uint32_t a[ILP], b = s * 2654435761u + threadIdx.x, c = s ^ 0x9e3779b9u;
  for (int i = 0; i < ILP; i++) a[i] = threadIdx.x * (i + 1) + s;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
    }
  }
  uint32_t r = 0;
  for (int i = 0; i < ILP; i++) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_imadwide(uint32_t* out, uint32_t s) {
  uint64_t a[ILP];
  uint32_t b = s * 2654435761u + threadIdx.x;
  uint32_t x[ILP];
  for (int i = 0; i < ILP; i++) { a[i] = threadIdx.x * (i + 1) + s; x[i] = s + i * 77u + threadIdx.x; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      asm volatile("{ .reg .u32 lo; cvt.u32.u64 lo, %0; mad.wide.u32 %0, lo, %1, %0; }" : "+l"(a[i]) : "r"(b));
    }
  }
  uint64_t r = x[0];
  for (int i = 0; i < ILP; i++) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)(r ^ (r >> 32));
}

// 1 IMAD.WIDE + 1 LOP3 per step (the holes-clmul inner mix)
__global__ void k_mix(uint32_t* out, uint32_t s) {
  uint64_t a[ILP];
  uint32_t b = s * 2654435761u + threadIdx.x, c = s ^ 0x9e3779b9u;
  uint32_t x[ILP], l[ILP];
  for (int i = 0; i < ILP; i++) { a[i] = threadIdx.x * (i + 1) + s; x[i] = s + i * 77u + threadIdx.x; l[i] = x[i] * 3u; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      asm volatile("{ .reg .u32 lo; cvt.u32.u64 lo, %0; mad.wide.u32 %0, lo, %1, %0; }" : "+l"(a[i]) : "r"(b));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x78;" : "+r"(l[i]) : "r"(b), "r"(c));
    }
  }
  uint64_t r = 0;
  for (int i = 0; i < ILP; i++) r ^= a[i] ^ l[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)(r ^ (r >> 32));
}

// 1 IMAD (32-bit) + 1 LOP3 per step
__global__ void k_mix32(uint32_t* out, uint32_t s) {
  uint32_t a[ILP], l[ILP];
  uint32_t b = s * 2654435761u + threadIdx.x, c = s ^ 0x9e3779b9u;
  for (int i = 0; i < ILP; i++) { a[i] = threadIdx.x * (i + 1) + s; l[i] = a[i] * 3u; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x78;" : "+r"(l[i]) : "r"(b), "r"(c));
    }
  }
  uint32_t r = 0;
  for (int i = 0; i < ILP; i++) r ^= a[i] ^ l[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}


#define CHAIN_KERNEL(NAME, ASM, ...)                                            \
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

// 2-register IMAD (a*b + RZ), IMAD with immediate multiplier, IMAD.HI,
// LOP3 with an immediate operand, PRMT, IADD3, FFMA (3-reg and immediate),
// HFMA2, POPC.  "%1, %2" are registers; the chains keep a[i] dependent.
CHAIN_KERNEL(k_mul2, "mul.lo.u32 %0, %0, %1;")
CHAIN_KERNEL(k_imadimm, "mad.lo.u32 %0, %0, 0x9249, %2;")
CHAIN_KERNEL(k_mulhi, "mul.hi.u32 %0, %0, %1;")
CHAIN_KERNEL(k_lop3imm, "lop3.b32 %0, %0, 0x92492492, %2, 0x78;")
CHAIN_KERNEL(k_lop3imm2, "and.b32 %0, %0, 0x92492492;")
CHAIN_KERNEL(k_prmt, "prmt.b32 %0, %0, %1, 0x5410;")
CHAIN_KERNEL(k_iadd3, "add.u32 %0, %0, %1;")
CHAIN_KERNEL(k_ffma, "fma.rn.f32 %0, %0, %1, %2;")
CHAIN_KERNEL(k_ffmaimm, "fma.rn.f32 %0, %0, 0f3F800001, %2;")
CHAIN_KERNEL(k_hfma2, "fma.rn.f16x2 %0, %0, %1, %2;")
CHAIN_KERNEL(k_popc, "popc.b32 %0, %0;")
CHAIN_KERNEL(k_shl_imad, "shl.b32 %0, %0, 3;")

// mixes: one 2-reg IMAD + one 3-reg LOP3; two LOP3 + one IMAD
__global__ void k_mix_mul2_lop(uint32_t* out, uint32_t s) {
  uint32_t a[ILP], l[ILP];
  uint32_t b = s * 2654435761u + threadIdx.x, c = s ^ 0x9e3779b9u;
  for (int i = 0; i < ILP; i++) { a[i] = threadIdx.x * (i + 1) + s; l[i] = a[i] * 3u; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x78;" : "+r"(l[i]) : "r"(b), "r"(c));
    }
  }
  uint32_t r = 0;
  for (int i = 0; i < ILP; i++) r ^= a[i] ^ l[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}


// FP64 pipe: DFMA chain, and a 3-way mix DFMA + IMAD + LOP3 (is fp64 a third pipe?)
__global__ void k_dfma(uint32_t* out, uint32_t s) {
  double a[ILP], b = 1.0000001 + s * 1e-9, c = 1e-7;
  for (int i = 0; i < ILP; i++) a[i] = threadIdx.x * (i + 1) + s;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[i]) : "d"(b), "d"(c));
  }
  double r = 0; for (int i = 0; i < ILP; i++) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)r;
}
__global__ void k_mix3(uint32_t* out, uint32_t s) {
  double d[ILP], b = 1.0000001 + s * 1e-9, c = 1e-7;
  uint32_t m[ILP], l[ILP], bb = s * 2654435761u + threadIdx.x, cc = s ^ 0x9e3779b9u;
  for (int i = 0; i < ILP; i++) { d[i] = threadIdx.x * (i + 1) + s; m[i] = threadIdx.x + i; l[i] = m[i] * 3u; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(b), "d"(c));
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(m[i]) : "r"(bb), "r"(cc));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x78;" : "+r"(l[i]) : "r"(bb), "r"(cc));
    }
  }
  double r = 0; uint32_t q = 0; for (int i = 0; i < ILP; i++) { r += d[i]; q ^= m[i] ^ l[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)r ^ q;
}

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
  printf("%-10s %8.3f ms  %8.2f T thread-ops/s  (%.1f ops/clk/SM at max clock %d MHz)\n",
         name, ms, tops, tops * 1e12 / (sms * (double)clk_khz * 1e3), clk_khz / 1000);
  cudaFree(out);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, clk);
  run("lop3", k_lop3, 1, p.multiProcessorCount, clk);
  run("shf", k_shf, 1, p.multiProcessorCount, clk);
  run("imad", k_imad, 1, p.multiProcessorCount, clk);
  run("imad.wide", k_imadwide, 1, p.multiProcessorCount, clk);
  run("mix_wide", k_mix, 2, p.multiProcessorCount, clk);
  run("mix32", k_mix32, 2, p.multiProcessorCount, clk);
  run("mul2", k_mul2, 1, p.multiProcessorCount, clk);
  run("imad_imm", k_imadimm, 1, p.multiProcessorCount, clk);
  run("mul.hi", k_mulhi, 1, p.multiProcessorCount, clk);
  run("lop3_imm", k_lop3imm, 1, p.multiProcessorCount, clk);
  run("and_imm", k_lop3imm2, 1, p.multiProcessorCount, clk);
  run("prmt", k_prmt, 1, p.multiProcessorCount, clk);
  run("iadd", k_iadd3, 1, p.multiProcessorCount, clk);
  run("ffma", k_ffma, 1, p.multiProcessorCount, clk);
  run("ffma_imm", k_ffmaimm, 1, p.multiProcessorCount, clk);
  run("hfma2", k_hfma2, 1, p.multiProcessorCount, clk);
  run("popc", k_popc, 1, p.multiProcessorCount, clk);
  run("shl_imm", k_shl_imad, 1, p.multiProcessorCount, clk);
  run("mul2+lop3", k_mix_mul2_lop, 2, p.multiProcessorCount, clk);
  run("dfma", k_dfma, 1, p.multiProcessorCount, clk);
  run("dfma+imad+lop3", k_mix3, 3, p.multiProcessorCount, clk);
  return 0;
}
