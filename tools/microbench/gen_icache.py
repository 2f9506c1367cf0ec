#!/usr/bin/env python3
"""Generate icache.cu: the I-cache microbenchmark of DESIGN.md §5 ("Instruction supply").

Each kernel kN runs a loop whose body is N 3-input LOP3s over 16 registers (N * 16 bytes of
SASS), so bodies above the 32 KB instruction cache show the fetch stalls the generated
per-coefficient kernels hit.  The generated source is not committed (it is ~32k lines):

    python tools/microbench/gen_icache.py > /tmp/icache.cu
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/icache /tmp/icache.cu && /tmp/icache
"""
import random
import sys

SIZES = (256, 1024, 2048, 4096, 8192, 16384)


def kernel(n, rnd):
    regs = ", ".join("r%d = threadIdx.x * %du" % (i, i + 1) for i in range(16))
    out = ["__global__ void k%d(uint32_t* out, int iters, int sync) {" % n, "  uint32_t %s;" % regs,
           "  for (int it = 0; it < iters; it++) {", "   if (sync) __syncthreads();"]
    for i in range(n):
        d = i % 16
        a, b = rnd.sample([r for r in range(16) if r != d], 2)
        out.append('    asm volatile("lop3.b32 %%0, %%0, %%1, %%2, 0x96;" : "+r"(r%d) : "r"(r%d), "r"(r%d));'
                   % (d, a, b))
    out += ["  }", "  uint32_t x = " + "^".join("r%d" % i for i in range(16)) + ";",
            "  if (x == 0x1234567u) out[threadIdx.x] = x;", "}"]
    return "\n".join(out)


def main():
    rnd = random.Random(1)
    src = ["#include <cstdio>", "#include <cstdint>", "#include <cuda_runtime.h>"]
    src += [kernel(n, rnd) for n in SIZES]
    src.append("""
template <typename K> void run(const char* name, K kern, int N, int tpb, int sync) {
  uint32_t* out; cudaMalloc(&out, 4096);
  int iters = (1 << 24) / N; if (iters < 4) iters = 4;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<148, tpb>>>(out, 2, sync);
  cudaEventRecord(e0); kern<<<148, tpb>>>(out, iters, sync); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 148.0 * tpb * (double)iters * N;
  printf("%s body=%6d B tpb=%4d sync=%d: %.1f lanes/clk/SM (at 1965 MHz), IPC/SM=%.2f\\n", name, N * 16, tpb, sync,
         ops / (ms * 1e-3) / 148 / 1965e6, ops / 32 / (ms * 1e-3) / 148 / 1965e6);
  cudaFree(out);
}
int main() {""")
    for n in SIZES:
        for tpb in (256, 512):
            for sync in (0, 1):
                src.append('  run("k%d", k%d, %d, %d, %d);' % (n, n, n, tpb, sync))
    src.append('  printf("err=%s\\n", cudaGetErrorString(cudaGetLastError())); return 0; }')
    sys.stdout.write("\n".join(src) + "\n")


if __name__ == "__main__":
    main()
