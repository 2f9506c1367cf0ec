// Region-linear-combination plans and their bitsliced sm_100a kernels.
//
// A plan computes, for every stripe t and byte position p,
//     out_r[t][p] = XOR_c A[r][c] * in_c[t][p]          over GF(2^8)
// where every input / output is a block addressed as  slot_ptr[slot] + t*slot_stride[slot]
// + blk*S.  Encode (G''), decode (rows of Gtilde^{-1}) and repair (projection + newcomer) are all
// plans; only the coefficient matrix and the slot wiring differ (north star: "reuse the same
// region-linear-combination kernel").  An input may itself be a small combination of blocks
// ("derived" input, used by the fused repair: beta_h = phi_f . piece_h).
#pragma once
#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "gf256.hpp"
#include "xorprog.hpp"

namespace pmrc {

struct Term {
  int slot, blk;
  uint16_t coef;  // GF(2^8) or, for w = 16 plans, GF(2^16)
};
struct InputDesc {
  std::vector<Term> terms;  // one term with coef 1 = plain block
};
struct OutputDesc {
  int slot, blk;
};

struct PlanSpec {
  int n_slots = 0;
  std::vector<InputDesc> inputs;
  std::vector<OutputDesc> outputs;
  Mat A;  // outputs x inputs (w = 16: nonzero pattern only, coefficients in A16)
  int w = 8;                   // symbol width: GF(2^8) bytes or GF(2^16) little-endian byte pairs
  std::vector<uint16_t> A16;   // w = 16: outputs x inputs coefficients, row-major
  uint32_t coef(int r, int c) const { return w == 16 ? A16[(size_t)r * A.c + c] : A.at(r, c); }
};

struct GenOptions {
  int max_rows = 8;      // output blocks per group (8 planes each in registers)
  int in_block = 16;     // max loaded blocks per stage (shared-memory buffer of in_block KiB, x2)
  bool stage_even = true;  // split a group's inputs into equal stages of <= in_block blocks
  int warps = 0;         // warps per CTA (0 = auto: 12; 16 for wide decode plans; capped by smem)
  int tpb = 256;         // (derived) threads per CTA
  bool cse = true;       // Paar CSE (false: naive per-row XOR chains)
  bool sync_groups = true;  // __syncthreads() before each group: warps of a CTA execute the same code
  int dyn = -1;             // layout 1: dynamic chunk schedule (per-group counters) instead of static
                            // ranges; 2: teams then help the other groups (-1 auto: 2 for clustered
                            // plans, i.e. decode, else 0)
  int pdl = 0;               // programmatic dependent launch: 1 overlap launch only (wait for the
                            // predecessor's memory first), 2 fully overlapped (independent launches)
  int smem_kib = 0;          // shared-memory budget per CTA for the warp count (0 = 220 KiB)
  int dyn_static = 0;        // dyn >= 2: per mille of the chunks in static ranges (the rest: the counters)
  int cta_sync = 0;         // layout 1: all teams of a CTA start every item together (CTA barrier):
                            // the teams then fetch the same instructions at about the same time
  int chunk_loop = 24;      // chunks per team per group (loop: instruction reuse)
  int team = 2;             // warps sharing one chunk's stage buffer (each computes 1/team of the rows)
  int ld_hint = 1;
  bool fold = true;         // eager-fold emission of XOR networks (low register pressure)
  int layout = -1;          // 0: every CTA walks all groups; 1: group-specialised CTAs; 2: same, CTAs
                            // apportioned by group cost; -1: auto
  int grid_ctas = 148;      // layout 2: CTAs the apportionment table is made for (one per SM)
  bool tr_balance = false;   // split a stage's loads + transposes over team ranks by network cost
                             // (measured: config-4 decode 0.647 -> 0.680 ms: off)
  bool balance_ranks = false; // reorder a group's rows to balance estimated work per team rank
                             // (measured: decode 0.651 -> 0.663 ms, encode 0.528 -> 0.532: off)
  bool cluster_wide = false; // clustering ties -> the widest row (dense and sparse decode rows in
                             // different groups; measured 0.651 -> 0.734 ms: the groups' fronts drift
                             // apart and the shared inputs are read from DRAM twice)
  bool even_groups = false; // clustered plans: equal group sizes instead of max_rows-sized groups
  bool auto_wide16 = true;   // resolve_options: group-specialised CTAs (layout 1, stealing schedule)
                             // for many groups whose supports have >= 16 rows (k = 16 encode)
  bool auto_wide = true;    // resolve_options: 16-row groups on 4-warp teams for wide multi-stage plans
  int enc_restarts = 4;     // CSE restarts for the encode plan (built once per code; capi.cpp)
  int cse_restarts = 1;     // CSE runs per network (seeded near-tie randomisation), keep the cheapest
  bool sched = false;       // register-pressure-aware temp order (emit_slp_sched) instead of CSE order
  int l2_shared = 0;        // layouts 1/2: L2 policy of blocks read by >1 group (-1 static last-read rule, 0 normal, 2 evict_last)
  int ws_prod = 1;          // producer warps per warp-specialised team
  bool ws = false;          // warp-specialised teams (producer transposes, consumers run networks)
  bool own_first = false;   // sub-networks over a warp's own transposed blocks before the team barrier
  int nbuf = 2;             // stage buffers per team (layouts 1/2): prefetch nbuf-1 stages ahead
  int tr_unroll = 1;        // unroll factor of the in-place input transpose loop
  bool fence = true;        // register fence after every (sub-)network (see codegen.cpp)
  bool net_even = true;     // split a stage into equal sub-networks (<= net_in inputs each)
  int net_in = 7;           // inputs per CSE sub-network within a stage (0 = the whole stage)
  bool trace = false;       // layout 1 diagnostics: per-team start/end/wait times (pmrc_debug_counters)
  int pace_lag = 0;         // layout 1: max chunks a team runs ahead of its peers (0 = no pacing)
  int rt_groups = 0;        // runtime-coefficient kernel (rtplan.hpp): row groups per CTA (0 = auto)
  int rt_rows = 0;          // runtime-coefficient kernel: rows per thread, 7 or 8 (0 = auto)
  int part_search = 0;      // evaluations of the input / row partition search per single-stage group (codegen.cpp)
  int enc_part_search = 200; // part_search of the encode plan (built once per code; capi.cpp)
  bool auto_nbuf = true;    // resolve_options: a 3-deep stage ring for multi-group plans when it still fits 16 warps (k = 4 codes)
};

constexpr int kDynSlots = 64;  // counter slots of the dynamic schedule (launches in flight per plan)

struct GenStats {
  int groups = 0;
  long xor2 = 0;         // 2-input XORs of the emitted network
  long naive_lop3 = 0;   // W of SURVEY §8(d) (per 32 byte positions)
  long xor2_naive = 0;   // 2-input XORs without CSE
  int transposes = 0;    // 8x8 bit transposes per 32 byte positions (in + out)
  long loads = 0;        // 16-B vector loads per lane per item sum
  int smem_per_warp = 0; // bytes of shared memory (transposed input planes) per warp
  int max_stages = 0;    // most shared-memory stages of any group
  int max_support_rows = 0;  // most output rows sharing one support (before the max_rows split)
  bool clustered = false;  // rows had distinct supports and were clustered greedily
  double group_cost_ratio = 1;  // max / min estimated group cost (loaded blocks + outputs)
};

// Generate CUDA C++ source of the bitsliced kernel `pmrc_kernel` for a plan.
std::string generate_source(const PlanSpec &p, const GenOptions &o, GenStats &st);

// Compiled kernel (driver-API module) bound to the device current at compile time.
struct Kernel {
  void *module = nullptr;    // CUmodule
  void *function = nullptr;  // CUfunction
  int n_slots = 0;
  int n_groups = 0;
  int tpb = 256;
  int chunk_loop = 1;
  int layout = 0;
  int w = 8;                 // symbol width: chunk = 128 w bytes of every block per warp
  int grid_ctas = 148;
  int teams = 1;
  void *pace = nullptr;             // layout 1: per-(CTA, team) progress counters (device)
  size_t pace_entries = 0;
  void *dyn = nullptr;              // layout 1 dynamic schedule: kDynSlots x n_groups x 2 u32 counters
  bool dyn_on = false;
  bool dyn_full = false;
  bool pdl = false;                 // launched with programmatic stream serialization            // stealing schedule: launched on the full grid (not G x spg)
  mutable uint32_t epoch = 0;       // launch epoch (counters carry it, so they never need a reset)
  size_t smem = 0;
  int blocks_per_sm = 1;
  int sms = 148;
  int regs = 0;
  GenStats stats;
  std::string source;
  double compile_ms = 0;
  bool from_cache = false;
};

// Generate + NVRTC-compile + load.  Returns 0 or PMRC_E*; err gets the log on failure.
int build_kernel(const PlanSpec &p, const GenOptions &o, Kernel &k, std::string &err);
void free_kernel(Kernel &k);
// Source of the kernel build_kernel would compile (options resolved).
std::string plan_source(const PlanSpec &p, const GenOptions &o, GenStats &st);
// Generate + NVRTC-compile into the kernel cache only (no GPU needed).
int precompile_kernel(const PlanSpec &p, const GenOptions &o, std::string &err);
// True when the kernel cache is enabled and its plan index holds this plan (same spec, options and
// library build) with its cubin: build_kernel then loads it without generation or NVRTC.
bool plan_indexed(const PlanSpec &p, const GenOptions &o);
bool kernel_cache_enabled();

// Launch over `stripes` stripes of S-byte blocks.  ptrs/strides: n_slots entries.
int launch_kernel(const Kernel &k, const uint64_t *ptrs, const uint64_t *strides, size_t S, size_t stripes,
                  void *stream, std::string &err, int max_ctas = 0);  // max_ctas: grid cap (0 = one wave)

std::atomic<unsigned long long> &launch_counter();

}  // namespace pmrc
