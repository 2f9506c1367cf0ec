// Seeded input generator: host and device fills of the counter-based stream in pmrc_inputs.h.
// No method arithmetic lives here.
#include "pmrc_inputs.h"
#include <cuda_runtime.h>

__host__ __device__ static inline uint8_t gen_byte(uint64_t key, uint64_t o, uint64_t real_len) {
  if (o >= real_len) return 0;
  return (uint8_t)(pmrc_splitmix64(key ^ (o >> 3)) >> (8 * (o & 7)));
}

extern "C" void pmrc_inputs_fill_host(uint8_t *dst, size_t len, uint64_t seed, uint64_t offset,
                                      uint64_t real_len) {
  uint64_t key = pmrc_splitmix64(seed);
  size_t i = 0;
  // head until 8-aligned global offset
  while (i < len && ((offset + i) & 7)) { dst[i] = gen_byte(key, offset + i, real_len); i++; }
  for (; i + 8 <= len; i += 8) {
    uint64_t o = offset + i;
    if (o + 8 <= real_len) {
      uint64_t w = pmrc_splitmix64(key ^ (o >> 3));
      for (int b = 0; b < 8; b++) dst[i + b] = (uint8_t)(w >> (8 * b));
    } else {
      for (int b = 0; b < 8; b++) dst[i + b] = gen_byte(key, o + b, real_len);
    }
  }
  for (; i < len; i++) dst[i] = gen_byte(key, offset + i, real_len);
}

__global__ void k_fill(uint8_t *dst, size_t len, uint64_t key, uint64_t offset, uint64_t real_len) {
  // one thread per 8 destination bytes (dst-aligned); generic byte path keeps it simple and exact
  size_t stride = (size_t)gridDim.x * blockDim.x * 8;
  for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < len; i += stride) {
    uint64_t o = offset + i;
    if (((o & 7) == 0) && (i + 8 <= len) && (o + 8 <= real_len) && ((((uintptr_t)(dst + i)) & 7) == 0)) {
      *(uint64_t *)(dst + i) = pmrc_splitmix64(key ^ (o >> 3));  // little-endian byte order
    } else {
      for (int b = 0; b < 8 && i + b < len; b++) dst[i + b] = gen_byte(key, o + b, real_len);
    }
  }
}

extern "C" int pmrc_inputs_fill_device(void *dst, size_t len, uint64_t seed, uint64_t offset,
                                       uint64_t real_len, void *stream) {
  if (len == 0) return 0;
  uint64_t key = pmrc_splitmix64(seed);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  size_t words = (len + 7) / 8;
  size_t blocks = (words + 255) / 256;
  if (blocks > (size_t)sms * 16) blocks = (size_t)sms * 16;
  k_fill<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((uint8_t *)dst, len, key, offset, real_len);
  return (int)cudaGetLastError();
}
