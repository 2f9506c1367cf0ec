// Integer-issue microbenchmark for sm_100a: measures LOP3 / PRMT / SHF / IMAD lane-op
// throughput per SM per clock (fixes R_int of the roofline).
// Many independent dependency chains per thread so the pipes, not latency, bind.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 8
#define ITERS 4096

template <int KIND>
__global__ void k_issue(uint32_t* out, uint32_t seed) {
  uint32_t a[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; i++) a[i] = seed ^ (threadIdx.x * 2654435761u + i);
  uint32_t b = seed * 7u + threadIdx.x, c = seed * 13u + blockIdx.x;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CHAINS; i++) {
      if (KIND == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));
      if (KIND == 1) asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
      if (KIND == 2) asm volatile("shf.l.wrap.b32 %0, %0, %0, %1;" : "+r"(a[i]) : "r"(b));
      if (KIND == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
      if (KIND == 4) {  // half LOP3, half IMAD (dual-pipe issue test)
        if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
        else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b), "r"(c));
      }
      if (KIND == 5) asm volatile("xor.b32 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) r ^= a[i];
  if (r == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_copy(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) out[i] = in[i];
}

template <int KIND>
double run(int sms, int threads, int blocks_per_sm) {
  uint32_t* out; cudaMalloc(&out, 1 << 24);
  int grid = sms * blocks_per_sm;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_issue<KIND><<<grid, threads>>>(out, 1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) k_issue<KIND><<<grid, threads>>>(out, r + 2);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 5.0 * grid * threads * (double)ITERS * CHAINS;
  cudaFree(out);
  return ops / (ms * 1e-3);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s sms=%d clock_attr_mhz=%.0f smem_per_sm=%zu regs_per_sm=%d l2=%d\n", p.name,
         p.multiProcessorCount, clk_khz / 1e3, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor, p.l2CacheSize);
  int sms = p.multiProcessorCount;
  const char* names[] = {"lop3", "prmt", "shf", "imad", "lop3+imad", "xor"};
  for (int rep = 0; rep < 2; rep++) {
    double r[6];
    r[0] = run<0>(sms, 512, 4); r[1] = run<1>(sms, 512, 4); r[2] = run<2>(sms, 512, 4);
    r[3] = run<3>(sms, 512, 4); r[4] = run<4>(sms, 512, 4); r[5] = run<5>(sms, 512, 4);
    for (int i = 0; i < 6; i++)
      printf("%-10s %.3f T lane-ops/s  = %.1f lanes/clk/SM at %.0f MHz (max clock)\n", names[i], r[i] / 1e12,
             r[i] / (sms * 1965e6), 1965.0);
  }
  // HBM copy
  size_t n = (size_t)1 << 30;  // 1 GiB each way
  uint4 *a, *b; cudaMalloc(&a, n); cudaMalloc(&b, n); cudaMemset(a, 1, n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bps : {2, 4, 8}) for (int th : {256, 512}) {
    k_copy<<<sms * bps, th>>>(a, b, n / 16);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; r++) k_copy<<<sms * bps, th>>>(a, b, n / 16);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy grid=%dx%d: %.1f GB/s (read+write)\n", sms * bps, th, 10.0 * 2 * n / (ms * 1e-3) / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
