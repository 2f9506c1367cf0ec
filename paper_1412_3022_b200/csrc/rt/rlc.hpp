// Runtime-coefficient region-linear-combination kernel (csrc/rt/rlc.cu): plan blob format and
// launch interface shared by the host (rlc_host.cpp) and the device code.  No torch types.
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace pmrc_rt {

// Plan blob (u32 words).  Offsets are in words.  The first smem_words words (header, term and
// wiring tables, masks, and -- when they fit -- the coefficient tables) are copied into shared
// memory; tables of plans too large for shared memory (flags & kRlcGlobalTables) are read from the
// blob in device memory (L1-resident: a pass touches G R rows of them).
//   ttabA[4 q], ttabB[q]: PRMT tables of term q's coefficient (derived inputs, rlc.cu)
//   terms[2 q]     = slot | (last-term-of-its-input << 30) | (plain, coefficient 1 << 31)
//   terms[2 q + 1] = blk  | (input index << 16)
//   outs[2 r]      = slot,  outs[2 r + 1] = blk
//   masks[i * n_rb + b] = bit j set iff A[b R + j][i] != 0     (row blocks of R rows)
//   tabA[4 (i n_out + r)] = (T0a, T0b, T1a, T1b) of A[r][i], tabB[i n_out + r] = T2  (last in the blob)
//   pstart[p] .. pstart[p + 1]: the pass-p slice of seq; seq[e] = the terms pass p streams (every term
//     of each input that some row of the pass reads, in input order: a pass skips inputs its G R
//     rows do not use, e.g. the other symbol groups' inputs of an MBR encode)
struct RlcHdr {
  uint32_t magic;  // kRlcMagic
  uint32_t words;  // total blob words
  uint32_t n_in, n_out, n_terms, R, n_rb, flags;   // n_rb = ceil(n_out / R) row blocks
  uint32_t off_tabA, off_tabB, off_ttabA, off_ttabB, off_terms, off_outs, off_masks, smem_words;
  uint32_t G, n_pass, off_pstart, off_seq;         // n_pass = ceil(n_rb / G); seq_len = pstart[n_pass]
  uint32_t seq_len, pad0, pad1, pad2;
};
constexpr uint32_t kRlcGlobalTables = 1u;  // flags: coefficient tables stay in device memory
constexpr uint32_t kRlcDirect = 2u;        // flags: every input is one plain term (no derived inputs)
constexpr uint32_t kRlcNoPlain = 4u;       // flags: no term has coefficient 1
constexpr uint32_t kRlcMagic = 0x524C4331u;  // "RLC1"
constexpr int kRlcMaxPlanWords = 40 * 1024;  // shared-memory plan budget (160 KB); larger tables stay global

constexpr int kRlcMaxSlots = 48;              // node / buffer regions a launch can address

struct RlcArgs {
  const uint32_t *plan0;              // device: the plan of every stripe when stripe_plan == NULL
  const unsigned long long *plan_ptrs; // device: blob address of plan p (batch launches)
  const uint16_t *stripe_plan;        // device: plan index of stripe t, or NULL
  const unsigned long long *item_bounds;  // device: CTA b walks items [item_bounds[b], item_bounds[b+1]),
                                          // or NULL (equal item counts per CTA)
  unsigned long long S;               // block bytes (multiple of 16)
  unsigned long long stripes;
  unsigned max_words;                 // largest smem_words of the launch's plans (shared-memory plan area)
  unsigned n_slots;
  unsigned sh3, sh6, sh12;            // 2^29, 2^26, 2^20: shift multipliers passed at run time so
                                      // the shifts stay IMAD.HI on the FMA pipe (a literal power
                                      // of two becomes LEA.HI on the ALU pipe the PRMTs need)
  unsigned long long slot_ptr[kRlcMaxSlots];     // base address of slot s (stripe 0)
  unsigned long long slot_stride[kRlcMaxSlots];  // bytes between consecutive stripes of slot s
};

// Launch shape: R rows x V 32-bit words of accumulators per thread, G row groups of GT consumer
// threads per CTA (+ one producer warp); a tile is GT V 4 bytes of every block, a pass covers G R
// rows; tg: coefficient tables read from device memory (plans above the shared-memory budget).
// Instantiated: (8,4,1,256) and (8,4,2,256), each with tg = 0 / 1.
struct RlcShape {
  int R, V, G, GT;
  bool tg;
};
bool rlc_shape_ok(const RlcShape &sh);
// Returns 0, -1 (CUDA error: cudaGetLastError has it), -2 (no such instantiation).
int rlc_launch(const RlcArgs &a, const RlcShape &sh, int grid, void *stream);
// Shared memory the launch needs (bytes) and the CTAs per SM it allows (occupancy).
size_t rlc_smem_bytes(int V, int GT, unsigned max_words);
int rlc_ctas_per_sm(const RlcShape &sh, unsigned max_words);

}  // namespace pmrc_rt
