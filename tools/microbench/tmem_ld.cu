// TMEM -> register read throughput on sm_100a (tcgen05.ld), the number the
// DESIGN.md tensor-core rejection rests on (a Gram-matrix formulation must
// read q x q int32 accumulators per block back out of TMEM).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld tmem_ld.cu && ./tmem_ld
//
// Every CTA (4 warps = the 4 TMEM lane quarters) allocates COLS columns and
// each warp repeatedly loads its 32 lanes x X columns (32x32b.xX shape:
// X registers per thread), waiting after each load (the epilogue pattern:
// the values are consumed before the next load).  Reported: bytes moved per
// SM clock, for 1..4 resident CTAs per SM and two load widths.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CHECK(x)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));            \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

constexpr int COLS = 128;

template <int X>
__device__ __forceinline__ void tmem_ld(uint32_t addr, uint32_t (&v)[X]);

template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}

template <>
__device__ __forceinline__ void tmem_ld<64>(uint32_t addr, uint32_t (&v)[64]) {
#pragma unroll
  for (int h = 0; h < 4; h++) {
    uint32_t (&w)[16] = *reinterpret_cast<uint32_t(*)[16]>(&v[16 * h]);
    tmem_ld<16>(addr + 16 * h, w);
  }
}

template <int X>
__global__ void __launch_bounds__(128) k_tmem(uint32_t* out, int iters) {
  __shared__ uint32_t base_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&base_s)), "n"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = base_s + ((uint32_t)(32 * warp) << 16);
  uint32_t acc = 0;
  for (int it = 0; it < iters; it++) {
    uint32_t v[X];
    tmem_ld<X>(base + (uint32_t)((it * X) % COLS), v);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int i = 0; i < X; i++) acc ^= v[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(base_s), "n"(COLS));
}

template <int X>
int run(int sms, int clock_khz, uint32_t* d) {
  const int iters = 4096;
  cudaEvent_t a, b;
  CHECK(cudaEventCreate(&a));
  CHECK(cudaEventCreate(&b));
  for (int per_sm = 1; per_sm <= 4; per_sm++) {
    const int grid = sms * per_sm;
    k_tmem<X><<<grid, 128>>>(d, 64);     // warm-up
    CHECK(cudaDeviceSynchronize());
    CHECK(cudaEventRecord(a));
    k_tmem<X><<<grid, 128>>>(d, iters);
    CHECK(cudaEventRecord(b));
    CHECK(cudaEventSynchronize(b));
    CHECK(cudaGetLastError());
    float ms = 0;
    CHECK(cudaEventElapsedTime(&ms, a, b));
    const double bytes = (double)grid * 128 * iters * X * 4;
    const double per_sm_clk = bytes / (ms * 1e-3) / sms / (clock_khz * 1e3);
    printf("tcgen05.ld 32x32b.x%-2d  CTAs/SM=%d  %8.3f ms  %8.1f GB/s  %6.1f B/clk/SM (at %d MHz)\n", X,
           per_sm, ms, bytes / (ms * 1e-3) / 1e9, per_sm_clk, clock_khz / 1000);
  }
  return 0;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CHECK(cudaGetDevice(&dev));
  CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CHECK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  uint32_t* d = nullptr;
  CHECK(cudaMalloc(&d, (size_t)sms * 4 * 128 * 4));
  printf("SMs=%d clock=%d kHz\n", sms, clk);
  if (run<16>(sms, clk, d)) return 1;
  if (run<64>(sms, clk, d)) return 1;
  return 0;
}
