/* pmrc_inputs.h — seeded synthetic input generator shared by the oracle side and the CUDA side.
 *
 * This module holds NO arithmetic of the method (no GF(2^8), no coding); it only produces the
 * uniform-random source bytes the paper's workloads use ("uniform random data", BASELINE.json
 * configs; PAPER.md:214-216 measure on synthetic blocks).  Both sides regenerate any byte from
 * its global offset, so the oracle never needs a device->host copy of the inputs.
 *
 * Definition (counter based):
 *   key      = splitmix64(seed)
 *   word(w)  = splitmix64(key ^ w)                      (w = o >> 3)
 *   byte(o)  = o < real_len ? (word(o>>3) >> (8*(o&7))) & 0xFF : 0     (zero padding, R11)
 * where o is the global source offset  t*B*S + c*S + p  (stripe t, block c, byte p).
 */
#ifndef PMRC_INPUTS_H
#define PMRC_INPUTS_H
#include <stddef.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define PMRC_INPUTS_HD __host__ __device__ __forceinline__
#else
#define PMRC_INPUTS_HD static inline
#endif

PMRC_INPUTS_HD uint64_t pmrc_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

#ifdef __cplusplus
extern "C" {
#endif
/* Fill dst[0..len) with bytes for global offsets [offset, offset+len). Host memory. */
void pmrc_inputs_fill_host(uint8_t *dst, size_t len, uint64_t seed, uint64_t offset, uint64_t real_len);
/* Same, for the layout [stripes][blocks][S] starting at global stripe t0: byte (t,c,p) gets
 * offset (t0+t)*blocks*S + c*S + p.  (Equivalent to one contiguous fill; kept for clarity.) */
/* Device fill (dst is a device pointer; stream is a cudaStream_t or NULL).  Returns 0 or a CUDA
 * error code. */
int pmrc_inputs_fill_device(void *dst, size_t len, uint64_t seed, uint64_t offset, uint64_t real_len,
                            void *stream);
#ifdef __cplusplus
}
#endif
#endif
