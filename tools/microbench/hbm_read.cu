// Read-only HBM streaming rate on this B200 (the extraction kernels only read
// their inputs, so a copy-test peak -- read + write -- is not their ceiling).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_read hbm_read.cu && ./hbm_read
//
// Grid-stride XOR reduction over a 16 GiB buffer with 256-bit loads
// (ld.global.nc.v8.u32, one sector per thread per load), 2 and 4 loads in
// flight per thread; and a copy kernel for comparison.  Best of 10 launches.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CHECK(x)                                                              \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));        \
      return 1;                                                               \
    }                                                                         \
  } while (0)

__device__ __forceinline__ void ld256(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}

template <int ILP>
__global__ void __launch_bounds__(256) k_read(const uint8_t* __restrict__ p, int64_t n32,
                                              uint32_t* out) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i = tid; i < n32; i += stride * ILP) {
    uint32_t r[ILP][8];
#pragma unroll
    for (int k = 0; k < ILP; k++)
      if (i + k * stride < n32) ld256(p + 32 * (i + k * stride), r[k]);
      else
#pragma unroll
        for (int j = 0; j < 8; j++) r[k][j] = 0;
#pragma unroll
    for (int k = 0; k < ILP; k++)
#pragma unroll
      for (int j = 0; j < 8; j++) acc ^= r[k][j];
  }
  if (acc == 0x12345678u) out[0] = acc;   // keep the loads alive
}

__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, int64_t n16) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <typename F>
float best_ms(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0, dev = 0;
  CHECK(cudaGetDevice(&dev));
  CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t bytes = 16ll << 30;
  uint8_t *p = nullptr, *q = nullptr;
  uint32_t* out = nullptr;
  CHECK(cudaMalloc(&p, bytes));
  CHECK(cudaMalloc(&q, bytes / 2));
  CHECK(cudaMalloc(&out, 4));
  CHECK(cudaMemset(p, 1, bytes));
  const int64_t n32 = bytes / 32;
  for (int per_sm : {4, 8, 16}) {
    const int grid = sms * per_sm;
    const float m2 = best_ms([&] { k_read<2><<<grid, 256>>>(p, n32, out); }, 10);
    const float m4 = best_ms([&] { k_read<4><<<grid, 256>>>(p, n32, out); }, 10);
    CHECK(cudaGetLastError());
    printf("read-only 256-bit, %2d CTAs/SM x 256: ILP2 %.1f GB/s  ILP4 %.1f GB/s\n", per_sm,
           bytes / (m2 * 1e-3) / 1e9, bytes / (m4 * 1e-3) / 1e9);
  }
  const int64_t half = bytes / 2;
  const float mc = best_ms([&] { k_copy<<<sms * 16, 256>>>((const uint4*)p, (uint4*)q, half / 16); }, 10);
  CHECK(cudaGetLastError());
  printf("copy (read + write, 8 GiB each way): %.1f GB/s of traffic\n", 2 * half / (mc * 1e-3) / 1e9);
  return 0;
}
