/*
 * pmrc.h — C ABI of libpmrc: B200-native (sm_100a) product-matrix regenerating codes
 * (Rashmi et al. MSR/MBR) made fast as in arxiv 1412.3022, "Fast Product-Matrix Regenerating
 * Codes" (Le Scouarnec).  Citations: P:L = PAPER.md line L, S:L = SPEC.md line L; readings R1..R14
 * are listed in DESIGN.md §3.
 *
 * Field: GF(2^8), primitive polynomial 0x11D, g = 2 (R1).  Symbols are bytes; a "block"
 * (the paper's block) is S bytes; a "stripe" is one codeword: B data blocks encoded
 * into n*alpha blocks, alpha per node.  Node ids are 0-based here (the paper is
 * 1-based): nodes 0..k-1 are systematic, k..n-1 parity.
 *
 * Memory layouts (all buffers are caller-owned DEVICE memory on the device the code was created
 * on, except pmrc_encode_host which takes pinned or pageable HOST memory):
 *   data    [stripes][B][S]            block c of stripe t at data + t*B*S + c*S
 *   parity  [stripes][(n-k)*alpha][S]  parity node p (p >= k), symbol j at
 *                                       parity + t*P*S + ((p-k)*alpha + j)*S,  P = (n-k)*alpha
 *   piece   a node's alpha blocks of one stripe, contiguous: [alpha][S]; a pmrc_region gives
 *           the piece of stripe 0 (ptr) and the distance between consecutive stripes' pieces.
 *   For MSR/RS, systematic node i's piece is the data view data + t*B*S + i*alpha*S
 *   (stripe_stride B*S); parity node p's piece is the parity view above (stripe_stride P*S).
 *   For MBR (R6), systematic node i stores row i of the message matrix M(X): symbol j
 *   is data block L_{i,j}; such pieces must be materialised by the caller (pmrc_layout gives L).
 *
 * Alignment (GPU-path restriction, not the paper's): S % 16 == 0, every block address 16-byte
 * aligned (ptr and stripe_stride multiples of 16).  Violations return PMRC_EALIGN.
 *
 * All data-path calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default
 * stream) and never synchronise.  They return synchronously-detected errors only; faults of
 * earlier launches surface as PMRC_ECUDA on a later call.  A handle may be used from one host
 * thread at a time.
 */
#ifndef PMRC_H
#define PMRC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pmrc_code pmrc_code;

/* code kinds */
enum {
  PMRC_MSR_SPARSE = 0,       /* the paper's sparse MSR: Phi = [I; Cauchy], Lambda Moebius */
  PMRC_MSR_VANILLA = 1,      /* Rashmi et al. Vandermonde MSR */
  PMRC_MBR = 2,              /* systematic MBR, Psi = [I_k 0; Cauchy] (R5) */
  PMRC_RS_VANDERMONDE = 3,   /* systematic Vandermonde Reed-Solomon baseline (R12); d = k */
  PMRC_MSR_SPARSE_N2K = 4    /* EXTENSION, not the paper's: the sparse Phi = [I; Cauchy] with Lambda
                                chosen greedily (R15) so that every d-row subset of Psi is
                                invertible at n = 2k too: repair never returns PMRC_ESINGULAR
                                (SURVEY §8(c) A7, §8(f) NEXT-4); n <= 41 */
};

/* error codes */
enum {
  PMRC_OK = 0,
  PMRC_EINVAL = -1,       /* null pointer, id out of range / duplicated, wrong counts */
  PMRC_EUNSUPPORTED = -2, /* w not in {8, 16} (w = 16: sparse MSR only, and not for pmrc_apply /
                             the split repair calls); MSR with d != 2k-2; field too small;
                             invalid construction */
  PMRC_ESINGULAR = -3,    /* survivors do not span the data / helper matrix Psi_H singular (R10) */
  PMRC_EALIGN = -4,       /* S % 16 != 0 or a block address not 16-byte aligned */
  PMRC_ENOMEM = -5,       /* host or device allocation failed */
  PMRC_ECUDA = -6,        /* CUDA runtime / driver error (details in pmrc_last_error) */
  PMRC_EJIT = -7          /* kernel generation or NVRTC compilation failed */
};

/* A node piece region: piece of stripe t starts at ptr + t*stripe_stride (bytes). */
typedef struct {
  const void *ptr;
  size_t stripe_stride;
} pmrc_cregion;
typedef struct {
  void *ptr;
  size_t stripe_stride;
} pmrc_region;

typedef struct {
  int kind, n, k, d, w;
  int alpha;           /* blocks per node */
  int B;               /* data blocks per stripe, k*Delta */
  int parity_rows;     /* (n-k)*alpha: rows of G'' */
  int nnz;             /* nonzeros of G'' (the multiply-XORs per byte position) */
  double zero_pct;     /* 100 * zeros / size of G'' (Table 1) */
  int repair_complete; /* 1 if every d-subset of rows of Psi is invertible, so every
                          (lost, helpers) repair succeeds; 0 for sparse MSR at n >= 2k (R10) */
  long xor_ops;        /* LOP3 lane-ops per 32 byte positions of the encode XOR program
                          (after common-subexpression elimination), 0 before generation */
  long xor_ops_naive;  /* the naive bit-matrix count W of SURVEY §8(d) (roofline term) */
} pmrc_info_t;

/* Build the code: Psi, L, G, G' = G Gtilde^{-1}, G''; generate and compile the encode
 * kernel for the CUDA device current at the call (the paper's "initialization").
 * w = 8 (GF(2^8), every operation), or w = 16 for the sparse MSR code (GF(2^16), polynomial 0x1100B,
 * little-endian byte-pair symbols; encode, decode and fused repair).  For RS d is ignored (taken = k).  *out receives a handle to free with
 * pmrc_destroy. */
int pmrc_create(pmrc_code **out, int kind, int k, int d, int n, int w);
void pmrc_destroy(pmrc_code *c);
int pmrc_info(const pmrc_code *c, pmrc_info_t *out);

/* Copy matrices out (host memory).  which: 0 = Psi (n x d; RS n x k), 1 = G (n alpha x B),
 * 2 = G' (n alpha x B), 3 = G'' (parity_rows x B), 4 = lambda (n), 5 = Gtilde^{-1} (B x B, the
 * precode of P:112; MSR / RS only, PMRC_EUNSUPPORTED for MBR).  rows/cols receive the shape;
 * buf may be NULL to query the shape; otherwise it must hold rows*cols bytes. */
int pmrc_matrix(const pmrc_code *c, int which, uint8_t *buf, int *rows, int *cols);
/* Index matrix L, 1-based data indices, 0 = structural zero: MSR d x alpha, MBR d x d,
 * RS: k x 1 (identity layout).  buf may be NULL to query the shape. */
int pmrc_layout(const pmrc_code *c, int *buf, int *rows, int *cols);

/* Systematic encode: parity = G'' data for `stripes` stripes of B blocks of S bytes.
 * Zero coefficients are skipped at kernel-generation time. */
int pmrc_encode(pmrc_code *c, const void *data, void *parity, size_t S, size_t stripes, void *stream);

/* Same computation from HOST buffers (pinned memory recommended): the library stages chunks of
 * stripes through a ring of 3 device buffers it owns, overlapping H2D, the encode kernel and D2H on
 * 3 internal streams ordered after `stream`.  Synchronises before returning. */
int pmrc_encode_host(pmrc_code *c, const void *data_host, void *parity_host, size_t S, size_t stripes,
                     void *stream);

/* Lazy linear decode: given n_surv >= k surviving node ids and their pieces,
 * write the data blocks that are NOT held by a surviving systematic node into data_out
 * ([stripes][B][S]; other blocks are left untouched, so passing the data buffer itself completes
 * it in place).  Rows of G' are chosen systematic-first, then ascending id (R13); the B x B
 * inversion is done once per survivor set and cached.  *n_written (may be NULL) receives
 * the number of data blocks written per stripe.  PMRC_ESINGULAR if the survivors do not span B. */
int pmrc_decode(pmrc_code *c, const int *surv_ids, int n_surv, const pmrc_cregion *pieces, void *data_out,
                size_t S, size_t stripes, int *n_written, void *stream);

/* Exact repair of node lost_id from d helpers (RS: k), P:53 footnote: helper h
 * contributes beta_h = mu . piece_h (mu = phi_f for MSR, psi_f for MBR; only blocks with nonzero
 * mu are read); the newcomer solves Psi_H z = beta (cached d x d inversion) and forms its
 * alpha blocks (MSR: z_a + lambda_f z_{alpha+a}; MBR: z).  One fused launch.  out_piece receives
 * the lost node's piece.  PMRC_ESINGULAR when Psi_H is singular (R10). */
int pmrc_repair(pmrc_code *c, int lost_id, const int *helper_ids, int n_helpers, const pmrc_cregion *helper_pieces,
                pmrc_region out_piece, size_t S, size_t stripes, void *stream);

/* The two halves of repair as separate calls (the helper side and the newcomer side, which in a
 * storage system run on different machines):  beta (one block per stripe) = mu . piece. */
int pmrc_repair_project(pmrc_code *c, int lost_id, pmrc_cregion piece, pmrc_region beta, size_t S, size_t stripes,
                        void *stream);
/* newcomer: out_piece from the d helpers' betas (betas[i] belongs to helper_ids[i]). */
int pmrc_repair_combine(pmrc_code *c, int lost_id, const int *helper_ids, int n_helpers, const pmrc_cregion *betas,
                        pmrc_region out_piece, size_t S, size_t stripes, void *stream);

/* General region linear combination on the same generated kernels: for every stripe t and byte
 * position, out block r = XOR_c A[r][c] * in block c (GF(2^8), r < rows, c < cols), with input
 * block c of stripe t at in + t*in_stride + c*S and output block r at out + t*out_stride + r*S.
 * A: rows x cols, row-major, host memory; zero coefficients are skipped at generation time.  The
 * kernel is generated per matrix and cached on the handle (keyed by shape + coefficient hash).
 * Used for the paper's comparison paths (non-systematic encode Y = G Z, precode Z = Gtilde^{-1} X
 * then parity = G_parity Z).  PMRC_EINVAL for an all-zero A. */
int pmrc_apply(pmrc_code *c, const uint8_t *A, int rows, int cols, const void *in, size_t in_stride, void *out,
               size_t out_stride, size_t S, size_t stripes, void *stream);

/* Engine policy.  Every call runs a plan (a coefficient matrix + its wiring) on one
 * of two sm_100a kernels:
 *   PMRC_PLAN_JIT      the plan's generated bitsliced kernel (GF(2) XOR network per coefficient
 *                      matrix, zero coefficients skipped at generation time): the fastest
 *                      for a hot pattern; the first use of a new pattern generates and NVRTC-
 *                      compiles it (seconds) unless the in-tree kernel cache has it
 *   PMRC_PLAN_RUNTIME  the precompiled runtime-coefficient kernel (PRMT 3-3-2 table lookups,
 *                      coefficients as data): a new pattern costs only the host inversion and a
 *                      table fill (P:216's per-pattern initialisation, well under a millisecond)
 *   PMRC_PLAN_AUTO     (default) JIT for the encode (built at pmrc_create) and for plans whose JIT
 *                      kernel is already loaded on the handle (pmrc_plan_prepare, a call made
 *                      under PMRC_PLAN_JIT, or automatic promotion: pmrc_set_auto_promotion); the
 *                      runtime kernel for every other GF(2^8) plan.
 * GF(2^16) codes always use JIT.  Results are bit-identical under every policy. */
enum { PMRC_PLAN_AUTO = 0, PMRC_PLAN_JIT = 1, PMRC_PLAN_RUNTIME = 2 };
int pmrc_set_plan_policy(pmrc_code *c, int policy);
int pmrc_get_plan_policy(const pmrc_code *c);
/* JIT-compile (or load from the kernel cache) and keep on the handle the generated kernel of a
 * decode (op 0, ids = survivors) or repair (op 1, lost_id, ids = helpers) pattern, so that later
 * calls with this pattern run it under PMRC_PLAN_AUTO (hot-pattern promotion).  Errors as
 * pmrc_decode / pmrc_repair. */
int pmrc_plan_prepare(pmrc_code *c, int op, int lost_id, const int *ids, int n_ids);
/* Automatic promotion under PMRC_PLAN_AUTO (a pattern's initialisation is reused across the
 * stripes that follow): once a decode / repair pattern has moved `bytes` of plan traffic (S x
 * stripes x (input blocks + output blocks), summed over its single calls) on the runtime kernel, a
 * host thread generates and NVRTC-compiles its kernel into the in-tree kernel cache while the calls
 * keep running on the runtime kernel; the first call after that loads the cubin (milliseconds) and
 * the pattern runs its generated kernel from then on.  Default 1 GiB; 0 disables.  Needs the kernel
 * cache (PMRC_KCACHE not "off").  Batch calls use promoted patterns but do not count traffic.
 * pmrc_destroy waits for compilations in flight (so that no library thread outlives the handle). */
int pmrc_set_auto_promotion(pmrc_code *c, unsigned long long bytes);
/* Engine state of a decode (op 0) / repair (op 1) pattern on this handle: 0 runtime kernel (no
 * generated kernel loaded), 1 promotion compiling, 2 promotion compiled (loaded by the next call),
 * 3 generated kernel loaded.  Negative: error code. */
int pmrc_plan_state(pmrc_code *c, int op, int lost_id, const int *ids, int n_ids);

/* The runtime-coefficient kernel's plan blob (u32 words; layout: csrc/rt/rlc.hpp RlcHdr) of a decode
 * (op 0, ids = survivors), repair (op 1, lost_id, ids = helpers) or encode (op 2) plan, built on the
 * host without a GPU (slots: survivor / helper index in ascending id order, then the output).
 * *n_words receives the length; buf (may be NULL) receives the words when cap >= *n_words. */
int pmrc_rt_plan_blob(pmrc_code *c, int op, int lost_id, const int *ids, int n_ids, uint32_t *buf, size_t cap,
                      size_t *n_words);

/* Per-stripe failure patterns in ONE launch (config 4 as BASELINE.json states it; the
 * initialisation "depends on the failure pattern but can be reused across stripes"): stripe t has
 * its own pattern, run by the runtime-coefficient kernel (GF(2^8) codes).  Under PMRC_PLAN_AUTO a
 * stripe whose pattern has its generated kernel loaded (pmrc_plan_prepare) runs that kernel instead
 * (one launch per run of consecutive stripes with that pattern, before the runtime launch of the
 * rest); PMRC_PLAN_RUNTIME keeps every stripe on the runtime kernel.  nodes[i] (i < n) is node
 * i's piece region (stripe 0 + stripe stride, as pmrc_cregion elsewhere); only the regions a
 * stripe's pattern reads are touched (and validated).  Patterns are cached on the handle by id set.
 *
 * decode: surv_ids[t * n_surv + q] = survivor q of stripe t (any order); data_out [stripes][B][S]
 * receives, per stripe, the data blocks no surviving systematic node of that stripe holds (others
 * untouched); n_written (may be NULL) receives stripes counts.  PMRC_ESINGULAR (detail names the
 * stripe) if a stripe's survivors do not span the data. */
int pmrc_decode_batch(pmrc_code *c, const int *surv_ids, int n_surv, const pmrc_cregion *nodes, void *data_out,
                      size_t S, size_t stripes, int *n_written, void *stream);
/* repair: lost_ids[t] and helper_ids[t * n_helpers + h] (n_helpers = d; RS: k) per stripe; out_piece
 * receives stripe t's repaired piece (alpha blocks) at out_piece.ptr + t * stripe_stride.
 * PMRC_ESINGULAR (detail names the stripe) for a singular (lost, helpers) pair (R10). */
int pmrc_repair_batch(pmrc_code *c, const int *lost_ids, const int *helper_ids, int n_helpers, const pmrc_cregion *nodes,
                      pmrc_region out_piece, size_t S, size_t stripes, void *stream);

/* The paper's "specific" product-matrix decoders, for the
 * linear-vs-specific comparison: from exactly k survivors, MSR codes run the
 * symmetric-matrix method (A = C_DC Phi_DC^t; P, Q from its off-diagonal pairs; U = P/Q rows times
 * the other survivors' (Phi^t)^-1; S1, S2 = Phi_sel^-1 U_sel; the message Z through L) and then the
 * systematic data X_miss = Gtilde[miss] Z; MBR codes run T = Phi_DC^-1 R_right,
 * W = R_left + Delta_DC T^t, S = Phi_DC^-1 W, X through L.  Each step is one launch of a region
 * linear combination (on the engine pmrc_set_plan_policy selects) with its blocks in `scratch`
 * (device memory of at least pmrc_decode_specific_scratch bytes, caller-owned).  Output contract as
 * pmrc_decode: only the data blocks no surviving systematic node holds are written, and the result
 * equals pmrc_decode's (the decoded data is unique).  PMRC_EINVAL unless n_surv == k;
 * PMRC_EUNSUPPORTED for RS and GF(2^16) codes; PMRC_ESINGULAR for a singular submatrix. */
int pmrc_decode_specific_scratch(pmrc_code *c, size_t S, size_t stripes, size_t *bytes);
int pmrc_decode_specific(pmrc_code *c, const int *surv_ids, int n_surv, const pmrc_cregion *pieces, void *data_out,
                         void *scratch, size_t scratch_bytes, size_t S, size_t stripes, int *n_written, void *stream);

/* Cap the grid of every launch on this handle at max_ctas CTAs (0 = default: one full wave, one
 * persistent CTA per SM).  With a cap, small launches issued on several streams (e.g. config 4's
 * per-stripe failure patterns, one plan per stripe) run side by side on disjoint SMs instead of
 * each paying a full-GPU ramp and tail. */
int pmrc_set_max_ctas(pmrc_code *c, int max_ctas);

/* on = 1: the caller guarantees that consecutive launches of this handle on a stream are
 * independent (none reads or writes what the preceding one writes, e.g. config 4's per-stripe
 * repairs / decodes of different stripes when issued one launch per stripe).  Kernels are then
 * launched with programmatic dependent launch (cuLaunchKernelEx, PROGRAMMATIC_STREAM_SERIALIZATION)
 * and trigger their dependents on entry without waiting for their predecessor, so the next
 * launch's CTAs start as this launch's CTAs retire and a small launch does not pay a full-GPU
 * ramp and tail (measured config-4 per-stripe repair 0.517 -> 0.348 ms).
 * Ordering contract: the launch is ordered after a preceding kernel of another library only if
 * that kernel does NOT itself trigger programmatic completion early (griddepcontrol.launch_dependents
 * / cudaTriggerProgrammaticLaunchCompletion before its last store); kernels without such a trigger
 * (the default for every non-PDL kernel) complete before the launch starts.  When the preceding
 * work may trigger early (another handle with independent launches on, a PDL-enabled library
 * kernel), separate the two with an event wait or a non-PDL launch.  The batch calls
 * (pmrc_decode_batch / pmrc_repair_batch) run the non-promoted per-stripe patterns in ONE launch
 * and need none of this.  on = 0 (default): ordinary stream order.  Synchronises the device and drops the handle's
 * built kernels (rebuilt on next use).  PMRC_EINVAL for other values. */
int pmrc_set_independent_launches(pmrc_code *c, int on);

/* Blocks each helper reads to repair lost_id: nnz(phi_f) (MSR: 1 if f < alpha else alpha,
 * P:209), nnz(psi_f) for MBR, 1 for RS. */
int pmrc_read_cost(const pmrc_code *c, int lost_id, int *blocks_per_helper);

/* Generate the encode kernel and NVRTC-compile it (sm_100a) into the in-tree kernel cache
 * (paper_1412_3022_b200/kcache, or $PMRC_KCACHE) without loading it: needs no GPU.  build() uses it
 * so that pmrc_create on the GPU box loads a cached cubin instead of compiling. */
int pmrc_precompile(const pmrc_code *c);

/* The generated CUDA source of the encode kernel (for inspection / offline nvcc builds).  Writes
 * up to cap bytes (NUL-terminated if room) and the full length to *len. */
int pmrc_encode_source(const pmrc_code *c, char *buf, size_t cap, size_t *len);

/* The generated CUDA source of a decode (op 0: ids = survivors) or repair (op 1: lost_id, ids =
 * helpers) plan, without a GPU and without launching; compile != 0 also NVRTC-compiles it into
 * the kernel cache (so build() can pre-compile plans of known failure patterns).  Errors as
 * pmrc_decode / pmrc_repair (e.g. PMRC_ESINGULAR); PMRC_EINVAL if the plan computes nothing
 * (all data survives).  Output convention as pmrc_encode_source. */
int pmrc_plan_source(pmrc_code *c, int op, int lost_id, const int *ids, int n_ids, int compile, char *buf, size_t cap,
                     size_t *len);

/* Work of a plan (op 0 decode, 1 repair as in pmrc_plan_source; op 2 encode, ids ignored), per
 * stripe and per 32 byte positions of every block, for roofline accounting:
 * in_blocks / out_blocks = distinct blocks read / written per stripe (algorithmic HBM bytes =
 * (in_blocks + out_blocks) * S per stripe); naive_lop3 = SURVEY §8(d)'s W (3-input XORs of the
 * GF(2) expansion with zero coefficients skipped); xor2 = 2-input XORs of the emitted networks;
 * transposes = 8x8 bit transposes (24 LOP3 each).  No GPU needed. */
typedef struct {
  int groups, in_blocks, out_blocks;
  long long naive_lop3, xor2;
  int transposes;
} pmrc_plan_stats_t;
int pmrc_plan_stats(pmrc_code *c, int op, int lost_id, const int *ids, int n_ids, pmrc_plan_stats_t *out);
/* The same for the plan pmrc_apply would run for matrix A (rows x cols). */
int pmrc_apply_stats(pmrc_code *c, const uint8_t *A, int rows, int cols, pmrc_plan_stats_t *out);

/* Diagnostics of CTA pacing / timing (group-specialised layouts) of the last launched kernel that
 * has counters (PMRC_GEN=trace=1 or pace_lag): copies the device counter area (5 x E u64: progress
 * counters, then per-(CTA, team) start / end globaltimer ns, ns spent pacing and (group << 32 |
 * pacing timeouts)) to host[0..cap) and its length to *n (0 if no launched kernel has counters).
 * Synchronous (cudaMemcpy); not part of the data path. */
int pmrc_debug_counters(const pmrc_code *c, unsigned long long *host, size_t cap, size_t *n);

/* Number of kernels this library launched since load (for the bench's gpu_launches claim). */
unsigned long long pmrc_launch_count(void);

const char *pmrc_strerror(int err);
/* Thread-local detail string of the last error raised on this thread. */
const char *pmrc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* PMRC_H */
