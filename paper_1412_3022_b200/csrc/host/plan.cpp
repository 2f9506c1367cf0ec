// NVRTC JIT + launcher of the generated bitsliced kernels (see plan.hpp; generator in codegen.cpp).
#include "plan.hpp"

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <dlfcn.h>
#include <sys/stat.h>

#include <algorithm>
#include <atomic>
#include <fstream>
#include <chrono>
#include <unistd.h>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>

#include "../../../include/pmrc.h"
#include "cudrv.hpp"

namespace pmrc {

std::atomic<unsigned long long> &launch_counter() {
  static std::atomic<unsigned long long> c{0};
  return c;
}

namespace {
std::string cu_err(CUresult r) {
  const char *s = nullptr;
  if (drv().GetErrorString) drv().GetErrorString(r, &s);
  return s ? s : "unknown CUDA driver error";
}
}  // namespace

// Compiled-kernel cache: cubins keyed by a hash of the generated source, stored in-tree next to
// libpmrc.so (kcache/) so build() can pre-compile the standard plans on a machine without a GPU
// and the GPU box loads them without NVRTC.  PMRC_KCACHE overrides the directory; "off" disables.
static std::string cache_dir() {
  if (const char *e = getenv("PMRC_KCACHE")) return std::string(e) == "off" ? "" : std::string(e);
  Dl_info info;
  if (dladdr((void *)&cache_dir, &info) && info.dli_fname) {
    std::string so = info.dli_fname;
    size_t sl = so.rfind('/');
    return (sl == std::string::npos ? std::string(".") : so.substr(0, sl)) + "/kcache";
  }
  return "";
}

static std::string source_key(const std::string &src) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char ch : src) h = (h ^ ch) * 1099511628211ull;
  char buf[64];
  snprintf(buf, sizeof buf, "%016llx_%zu", (unsigned long long)h, src.size());
  return buf;
}

// Plan index: kcache/<plan key>.meta maps (plan, generator options, library build) to the source key
// of the plan's cubin plus the generator's statistics and resolved launch options, so that a plan
// built before loads its cubin without generating its source again (generation is the seconds of a
// plan build; NVRTC is skipped by the cubin cache).  The build id is part of the key: a rebuilt
// library never reuses another build's index (its cubins, keyed by source, stay valid).
static const char kBuildId[] = __DATE__ " " __TIME__;

#define PMRC_GEN_FIELDS(X)                                                                                     \
  X(max_rows) X(in_block) X(stage_even) X(warps) X(tpb) X(cse) X(sync_groups) X(dyn) X(pdl) X(smem_kib)         \
  X(dyn_static) X(cta_sync) X(chunk_loop) X(team) X(ld_hint) X(fold) X(layout) X(grid_ctas) X(tr_balance)       \
  X(balance_ranks) X(cluster_wide) X(even_groups) X(auto_wide16) X(auto_wide) X(enc_restarts) X(cse_restarts)   \
  X(sched) X(l2_shared) X(ws_prod) X(ws) X(own_first) X(nbuf) X(tr_unroll) X(fence) X(net_even) X(net_in)       \
  X(trace) X(pace_lag) X(rt_groups) X(rt_rows) X(part_search) X(enc_part_search) X(auto_nbuf)
#define PMRC_COUNT(m) +1
static_assert(0 PMRC_GEN_FIELDS(PMRC_COUNT) == 43 && sizeof(GenOptions) == 144,
              "GenOptions changed: list every field in PMRC_GEN_FIELDS (the plan index key)");
#undef PMRC_COUNT

namespace {
struct Fnv {
  uint64_t h = 1469598103934665603ull;
  void add(const void *p, size_t n) {
    const unsigned char *b = (const unsigned char *)p;
    for (size_t i = 0; i < n; i++) h = (h ^ b[i]) * 1099511628211ull;
  }
  template <class T>
  void v(T x) {
    add(&x, sizeof x);
  }
};
}  // namespace

static std::string plan_key(const PlanSpec &p, const GenOptions &o) {
  Fnv f;
  f.add(kBuildId, sizeof kBuildId);
  f.v(p.n_slots);
  f.v(p.w);
  f.v(p.inputs.size());
  for (const auto &in : p.inputs) {
    f.v(in.terms.size());
    for (const auto &t : in.terms) {
      f.v(t.slot);
      f.v(t.blk);
      f.v(t.coef);
    }
  }
  f.v(p.outputs.size());
  for (const auto &out : p.outputs) {
    f.v(out.slot);
    f.v(out.blk);
  }
  f.v(p.A.r);
  f.v(p.A.c);
  f.add(p.A.a.data(), p.A.a.size());
  f.v(p.A16.size());
  f.add(p.A16.data(), p.A16.size() * sizeof(uint16_t));
#define X(m) f.v(o.m);
  PMRC_GEN_FIELDS(X)
#undef X
  char buf[40];
  snprintf(buf, sizeof buf, "%016llx", (unsigned long long)f.h);
  return buf;
}

struct PlanMeta {
  std::string src_key;
  GenStats st;
  GenOptions oo;  // resolved: tpb, chunk_loop, layout, grid_ctas, warps, team, pdl are read back
  bool dyn_on = false, dyn_full = false;
};

static void write_meta(const std::string &dir, const std::string &key, const PlanMeta &m) {
  if (dir.empty()) return;
  mkdir(dir.c_str(), 0755);
  const std::string path = dir + "/" + key + ".meta", tmp = path + ".tmp" + std::to_string((long)getpid());
  {
    std::ofstream f(tmp);
    const GenStats &t = m.st;
    const GenOptions &o = m.oo;
    f << "pmrc-plan-meta 1\n"
      << m.src_key << "\n"
      << t.groups << " " << t.xor2 << " " << t.naive_lop3 << " " << t.xor2_naive << " " << t.transposes << " "
      << t.loads << " " << t.smem_per_warp << " " << t.max_stages << " " << t.max_support_rows << " "
      << (int)t.clustered << " " << std::hexfloat << t.group_cost_ratio << std::defaultfloat << "\n"
      << o.tpb << " " << o.chunk_loop << " " << o.layout << " " << o.grid_ctas << " " << o.warps << " " << o.team
      << " " << o.pdl << " " << (int)m.dyn_on << " " << (int)m.dyn_full << "\n";
    if (!f) {
      remove(tmp.c_str());
      return;
    }
  }
  rename(tmp.c_str(), path.c_str());
}

static bool read_meta(const std::string &dir, const std::string &key, PlanMeta &m) {
  if (dir.empty()) return false;
  std::ifstream f(dir + "/" + key + ".meta");
  std::string tag;
  int ver = 0, cl = 0, don = 0, dfull = 0;
  if (!(f >> tag >> ver) || tag != "pmrc-plan-meta" || ver != 1) return false;
  GenStats &t = m.st;
  GenOptions &o = m.oo;
  std::string ratio;
  if (!(f >> m.src_key >> t.groups >> t.xor2 >> t.naive_lop3 >> t.xor2_naive >> t.transposes >> t.loads >>
        t.smem_per_warp >> t.max_stages >> t.max_support_rows >> cl >> ratio))
    return false;
  t.clustered = cl != 0;
  t.group_cost_ratio = strtod(ratio.c_str(), nullptr);
  if (!(f >> o.tpb >> o.chunk_loop >> o.layout >> o.grid_ctas >> o.warps >> o.team >> o.pdl >> don >> dfull)) return false;
  m.dyn_on = don != 0;
  m.dyn_full = dfull != 0;
  return true;
}

// Structure statistics for resolve_options (groups, stages, supports, clustering, group costs,
// shared memory per warp): none depends on the XOR networks' common-subexpression elimination, so
// the probes generate without it (the expensive part of a generation)
static void probe(const PlanSpec &p, GenOptions o, GenStats &st) {
  o.cse = false;
  o.cse_restarts = 1;
  o.enc_restarts = 1;
  o.part_search = 0;
  o.enc_part_search = 0;
  (void)generate_source(p, o, st);
}

static GenOptions resolve_options(const PlanSpec &p, const GenOptions &o) {
  GenOptions oo = o;
  {
    // wide plans whose rows have distinct supports (decode: rows of G~^-1 over all B inputs, more
    // than 8 outputs, >= 3 stages): groups of 16 rows on teams of 4 warps (2 rows each) halve the
    // input transposes per output (measured: config-4 decode 1.14 -> 1.30 TB/s, profiles/r01d)
    GenOptions p0 = oo;
    if (p0.layout < 0) p0.layout = 0;
    GenStats w0;
    probe(p, p0, w0);
    if (o.auto_wide && p.w != 16 && w0.clustered && w0.max_stages >= 3 && p.outputs.size() > 8 && oo.team == 2 &&
        oo.max_rows == 8) {
      oo.max_rows = 16;
      oo.team = 4;
      if (oo.warps <= 0) oo.warps = 16;
    } else if (o.auto_wide16 && p.w != 16 && !w0.clustered && w0.max_support_rows >= 16 && w0.groups > 16 &&
               oo.team == 2 && oo.max_rows == 8 && oo.layout < 0) {
      // many groups whose supports have >= 16 rows (k = 16 encode: 30 / 60 groups of 8 rows, two per
      // support): group-specialised CTAs (8-row groups on 2-warp teams) with the stealing schedule
      // (dyn = 2 below: the 148 % G SMs left over visit other groups), so every SM streams one
      // group's network code for all its chunks.  Measured at config 5's 8 GiB per GPU against the
      // previous default (16-row groups on 4-warp teams walking all groups in layout 0, which had
      // beaten layout 0 with 8-row groups: 869 -> 901 GB/s at 1 GiB): MSR k=16 843-858 -> 883 GB/s,
      // MBR k=16 726-771 -> 868-870 (profiles/r02/k16_layout.jsonl); 16-row groups in layout 1
      // measure 782 / 670.  Stages of <= 10 blocks (30 inputs: 3 x 10, 16 inputs: 2 x 8) fit 16 warps
      // in the shared-memory budget where 15-block stages fit 14: MSR 884 -> 935 GB/s, MBR 867 -> 882
      // (with the encode's best-of-4 CSE, capi.cpp: 950 / 909; profiles/r02/k16_knobs.jsonl)
      oo.layout = 1;
      if (oo.in_block == 16) oo.in_block = 10;
    }
    // One group of 9-16 rows -- decode rows clustered into a single group (two missing systematic
    // nodes), or rows sharing one support (the fused repair of an MBR node: alpha = d = 14 rows,
    // which 8-row groups split in two, each re-reading every helper block): 8 rows per warp on
    // 2-warp teams, 8 warps (half the warps meeting at each team barrier), and a 3-deep stage ring
    // when the group has >= 3 stages.  Measured (profiles/r02/decode_shapes.jsonl,
    // repair_shapes.jsonl): config-3 MBR decode 0.252 -> 0.222 ms, MSR decode of 14 rows 0.302 ->
    // 0.275, MBR repair of a parity node 0.562 -> 0.454-0.460, of a systematic node 0.089 -> 0.076;
    // 7-row MSR repairs (<= 8 rows) and decodes of > 16 rows keep their shapes (slower this way).
    // ALU-heavy plans (decodes) run 12 warps (6 teams; 158-164 registers fit the 170 of 384 threads,
    // so the stage ring stays 2 deep in the shared-memory budget) with sub-networks of 8 inputs (16-
    // block stages as 8 + 8 instead of 6 + 5 + 5: -7.5% XORs, no spills): ncu of the 8-warp shape
    // showed nothing saturated (ALU 60%, shared memory 39%, DRAM 49%) and fixed-latency `wait`
    // stalls on top with 2 warps per SMSP.  Measured (profiles/r02/dec3_shapes.txt): config-3 MBR
    // decode 0.221 -> 0.204 ms, MSR 14-row decode 0.277 -> 0.246; the MBR fused repair keeps 8
    // warps and the 3-deep ring (0.459 vs 0.493 ms with 12 warps)
    const size_t nout = p.outputs.size();
    if (p.w != 16 && nout > 8 && nout <= 16 && (w0.clustered || w0.max_support_rows >= (int)nout) &&
        o.team == 2 && o.max_rows == 8 && o.warps <= 0 && o.nbuf == 2 && o.in_block == 16) {
      oo.max_rows = 16;
      oo.team = 2;
      // ALU-heavy plans (>= 40 naive LOP3 per 32 positions of each block read or written: these
      // decodes 62-79; the MBR parity-node repair, 196 helper blocks, 19) take the 12-warp shape
      long blocks = (long)nout;
      for (const auto &in : p.inputs) blocks += (long)in.terms.size();
      if (w0.naive_lop3 >= 40L * blocks) {
        oo.warps = 12;
        if (o.net_in == 7) oo.net_in = 8;
      } else if (w0.max_stages >= 3) {
        // light multi-stage plans (the MBR parity-node repair: 14 stages of one helper's 14 blocks):
        // with 8 warps and a 3-deep ring the kernel time depends on the helper set -- 0.46 ms when
        // all k systematic nodes help, 0.70-0.72 ms when one of them is the node left out (8 of the
        // 15 choices of 14 helpers; no generator knob at 8 warps moves it: fence, net_in, nbuf 4,
        // static ranges) -- while 12 warps with the 2-deep ring run both at 0.49 ms
        // (profiles/r02/mbr_repair_patterns*.jsonl)
        oo.warps = 12;
      } else {
        oo.warps = 8;
      }
    }
  }
  if (oo.dyn < 0) {
    // dynamic chunk schedule, with teams moving on to other groups' chunks when theirs are done,
    // for clustered plans (decode: rows of G~^-1): measured config-4 decode 0.873 -> 0.681 ms
    // (static ranges left whole TPCs finishing 35% late); the encode keeps static ranges (0.528 vs
    // 0.542 / 0.548 ms with dyn = 1 / 2)
    GenOptions p1 = oo;
    if (p1.layout < 0) p1.layout = 0;
    GenStats w1;
    probe(p, p1, w1);
    if (w1.clustered) oo.dyn = 2;
  }
  if (p.w == 16) {  // 16 planes per row: groups of 4 rows (2 per warp), stages of <= 8 blocks of 2 KiB
    if (oo.team == 2 && oo.max_rows == 8) oo.max_rows = 4;      // measured: k=8 0.54 -> 0.74 TB/s
    if (oo.in_block == 16) oo.in_block = 8;
  }
  if (oo.layout < 0) {
    // group-specialised CTAs when the groups tile the 148 SMs with <= 10% left idle
    GenStats g0;
    oo.layout = 0;
    probe(p, oo, g0);
    const int G = std::max(1, g0.groups), sms = 148;
    oo.layout = (G <= sms && (sms % G) * 10 <= sms) ? 1 : 0;
    // unequal groups: apportion CTAs by cost (layout 2), unless the dynamic schedule balances them
    if (oo.layout == 1 && g0.group_cost_ratio > 1.2 && oo.dyn <= 0) oo.layout = 2;
  }
  if (oo.dyn < 0) {
    // group-specialised plans whose groups leave >= 4 SMs without a group (G x spg < 148): the
    // stealing schedule puts those SMs to work as visitors (GF(2^16) k=8 encode, 14 groups:
    // 767 -> 822 GB/s); with <= 3 idle SMs static ranges measured better (GF(2^8) k=8: 7 groups)
    GenStats g2;
    probe(p, oo, g2);
    // ... and single-group plans of >= 3 stages (parity-node repair, 98 blocks in 7 stages: 0.405 ->
    // 0.387 ms; one-stage single-group plans, RS encode and systematic-node repair, measured slower)
    oo.dyn = (oo.layout == 1 && ((g2.groups > 1 && 148 % g2.groups >= 4) || (g2.groups == 1 && g2.max_stages >= 3)))
                 ? 2 : 0;
  }
  if (oo.ws) {  // ws_prod producers + 2 consumers per team, <= 4 teams (4 named barriers each), 2 buffers
    oo.team = std::max(1, oo.ws_prod) + 2;
    oo.warps = oo.team * std::min(4, 12 / oo.team);
    oo.nbuf = 2;
  }
  // A 3-deep stage ring when it still fits 16 warps (stages of <= 9 blocks: the k = 4 codes):
  // these plans are HBM-bound and latency-limited, and prefetching two items ahead lifts the MSR
  // k = 4 encode from 0.391 to 0.366 ms (0.84 -> 0.90 of HBM; 24 warps: 0.362, but they cost MBR
  // k = 4 30%); MBR k = 4 is unchanged (0.459 / 0.458) (profiles/r02/k4_knobs.jsonl)
  if (o.auto_nbuf && oo.nbuf == 2 && oo.layout >= 1 && !oo.ws && p.w != 16 && (oo.warps <= 0 || oo.warps == 16)) {
    GenOptions o3 = oo;
    o3.nbuf = 3;
    GenStats p3;
    probe(p, o3, p3);
    const int budget3 = o.smem_kib > 0 ? o.smem_kib * 1024 : 225 * 1024;
    // (plans of several groups only: the one-group RS encode measured 0.337 -> 0.360 ms with it)
    if (p3.groups > 1 && p3.smem_per_warp > 0 && budget3 / p3.smem_per_warp >= 16) oo.nbuf = 3;
  }
  // warps per CTA from the shared-memory budget (2 stage buffers of in_block KiB per team)
  GenStats pr;
  probe(p, oo, pr);
  // 225 KiB of stage buffers (+ 1 KiB alignment reservation + the schedule slots <= 227 KiB): 16 warps
  // (8 teams of 2) with the k=8 encode's 14-block stages (224 KiB)
  int budget = o.smem_kib > 0 ? o.smem_kib * 1024 : 225 * 1024;
  int w = std::max(1, std::min(32, budget / std::max(1, pr.smem_per_warp)));
  // 16 warps when they fit: measured against 12 (the previous default, whose 220 KiB budget left the
  // encode at 12): MSR k=8 encode 0.528 -> 0.501 ms, MBR k=8 0.597 -> 0.568, parity-node repair
  // 0.387 -> 0.358, GF(2^16) k=8 1.359 -> 1.218, RS 0.345 -> 0.340; MSR k=4 and vanilla unchanged;
  // 14 warps measured worse (0.571)
  int want = oo.warps;
  if (want <= 0) want = 16;
  w = std::min(w, want);
  w = std::max(oo.team, w - w % std::max(1, oo.team));  // whole teams
  oo.warps = w;
  oo.tpb = 32 * oo.warps;
  return oo;
}

// NVRTC compile (no GPU needed) with the on-disk cache; returns the cubin.
static bool cached_cubin(const std::string &dir, const std::string &src_key, std::vector<char> &cubin) {
  if (dir.empty()) return false;
  std::ifstream f(dir + "/" + src_key + ".cubin", std::ios::binary);
  if (!f) return false;
  cubin.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
  return !cubin.empty();
}

static int compile_cubin(const std::string &src, std::vector<char> &cubin, bool &from_cache, std::string &err) {
  from_cache = false;
  const std::string dir = cache_dir();
  const std::string path = dir.empty() ? "" : dir + "/" + source_key(src) + ".cubin";
  if (cached_cubin(dir, source_key(src), cubin)) {
    from_cache = true;
    return PMRC_OK;
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "pmrc_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    err = "nvrtcCreateProgram failed";
    return PMRC_EJIT;
  }
  const char *opts[] = {"-arch=sm_100a", "-lineinfo", "-default-device", "--std=c++17"};
  nvrtcResult rc = nvrtcCompileProgram(prog, 4, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    err = std::string("NVRTC: ") + nvrtcGetErrorString(rc) + "\n" + log.substr(0, 4000);
    nvrtcDestroyProgram(&prog);
    return PMRC_EJIT;
  }
  size_t nc = 0;
  nvrtcGetCUBINSize(prog, &nc);
  cubin.resize(nc);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  if (!path.empty()) {
    mkdir(dir.c_str(), 0755);
    std::string tmp = path + ".tmp" + std::to_string((long)getpid());
    std::ofstream f(tmp, std::ios::binary);
    if (f.write(cubin.data(), (std::streamsize)cubin.size())) {
      f.close();
      rename(tmp.c_str(), path.c_str());
    } else {
      remove(tmp.c_str());
    }
  }
  return PMRC_OK;
}

std::string plan_source(const PlanSpec &p, const GenOptions &o, GenStats &st) {
  return generate_source(p, resolve_options(p, o), st);
}

bool kernel_cache_enabled() { return !cache_dir().empty(); }

bool plan_indexed(const PlanSpec &p, const GenOptions &o) {
  const std::string dir = cache_dir();
  PlanMeta m;
  return read_meta(dir, plan_key(p, o), m) && access((dir + "/" + m.src_key + ".cubin").c_str(), R_OK) == 0;
}

static bool dyn_on_of(const std::string &src) { return src.find("u32 *__restrict__ dyn)") != std::string::npos; }
static bool dyn_full_of(const std::string &src) { return src.find("for (u32 hop = 0;") != std::string::npos; }

int precompile_kernel(const PlanSpec &p, const GenOptions &o, std::string &err) {
  const std::string dir = cache_dir(), key = plan_key(p, o);
  PlanMeta m;
  std::vector<char> cubin;
  if (read_meta(dir, key, m) && cached_cubin(dir, m.src_key, cubin)) return PMRC_OK;
  m.oo = resolve_options(p, o);
  std::string src = generate_source(p, m.oo, m.st);
  bool cached = false;
  int rc = compile_cubin(src, cubin, cached, err);
  if (rc) return rc;
  m.src_key = source_key(src);
  m.dyn_on = dyn_on_of(src);
  m.dyn_full = dyn_full_of(src);
  write_meta(dir, key, m);
  return PMRC_OK;
}

int build_kernel(const PlanSpec &p, const GenOptions &o, Kernel &k, std::string &err) {
  auto t0 = std::chrono::steady_clock::now();
  k = Kernel();
  const std::string dir = cache_dir(), key = plan_key(p, o);
  PlanMeta m;
  std::vector<char> cubin;
  bool cached = false;
  // a plan built before (same spec, options, library build): cubin and launch parameters from the
  // index, no generation (diagnostic builds, PMRC_DUMP / trace / pacing, always generate)
  const bool diag = getenv("PMRC_DUMP") || o.trace || o.pace_lag > 0;
  GenOptions oo;
  if (!diag && read_meta(dir, key, m) && cached_cubin(dir, m.src_key, cubin)) {
    cached = true;
    oo = o;
    oo.tpb = m.oo.tpb;
    oo.chunk_loop = m.oo.chunk_loop;
    oo.layout = m.oo.layout;
    oo.grid_ctas = m.oo.grid_ctas;
    oo.warps = m.oo.warps;
    oo.team = m.oo.team;
    oo.pdl = m.oo.pdl;
    k.stats = m.st;
  } else {
    oo = resolve_options(p, o);
    k.source = generate_source(p, oo, k.stats);
    if (const char *dd = getenv("PMRC_DUMP")) {  // diagnostics: keep the generated source of every plan
      std::ofstream(std::string(dd) + "/" + source_key(k.source) + ".cu") << k.source;
    }
    int crc = compile_cubin(k.source, cubin, cached, err);
    if (crc) return crc;
    m.src_key = source_key(k.source);
    m.st = k.stats;
    m.oo = oo;
    m.dyn_on = dyn_on_of(k.source);
    m.dyn_full = dyn_full_of(k.source);
    if (!diag) write_meta(dir, key, m);
  }
  k.n_slots = std::max(1, p.n_slots);
  k.n_groups = std::max(1, k.stats.groups);
  k.tpb = oo.tpb;
  k.chunk_loop = oo.chunk_loop;
  k.layout = oo.layout;
  k.w = p.w == 16 ? 16 : 8;
  k.grid_ctas = oo.grid_ctas;
  k.teams = std::max(1, oo.warps / std::max(1, oo.team));
  k.pdl = oo.pdl > 0;
  k.smem = (size_t)k.stats.smem_per_warp * oo.warps;
  auto t1 = std::chrono::steady_clock::now();
  k.compile_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  k.from_cache = cached;

  // load into the current context (the runtime's primary context for the current device)
  if (cudaFree(0) != cudaSuccess) {
    err = "no usable CUDA device";
    cudaGetLastError();
    return PMRC_ECUDA;
  }
  const Drv &D = drv();
  if (!D.ok) { err = "CUDA driver (libcuda.so.1) not available"; return PMRC_ECUDA; }
  CUmodule mod;
  CUresult cr = D.ModuleLoadData(&mod, cubin.data());
  if (cr != CUDA_SUCCESS) { err = "cuModuleLoadData: " + cu_err(cr); return PMRC_ECUDA; }
  CUfunction fn;
  cr = D.ModuleGetFunction(&fn, mod, "pmrc_kernel");
  if (cr != CUDA_SUCCESS) { D.ModuleUnload(mod); err = "cuModuleGetFunction: " + cu_err(cr); return PMRC_ECUDA; }
  k.module = mod;
  k.function = fn;
  int regs = 0;
  D.FuncGetAttribute(&regs, CU_FUNC_ATTRIBUTE_NUM_REGS, fn);
  k.regs = regs;
  int static_smem = 0;  // e.g. the dynamic schedule's per-team slots
  D.FuncGetAttribute(&static_smem, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, fn);
  if (k.smem + (size_t)static_smem > 48 * 1024) {
    cr = D.FuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)k.smem);
    if (cr != CUDA_SUCCESS) { D.ModuleUnload(mod); err = "cuFuncSetAttribute(smem): " + cu_err(cr); return PMRC_ECUDA; }
  }
  int nb = 1;
  D.OccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, k.tpb, k.smem);
  k.blocks_per_sm = std::max(1, nb);
  CUdevice dev;
  D.CtxGetDevice(&dev);
  int sms = 148;
  D.DeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev);
  k.sms = sms;
  if ((k.layout == 1 && oo.pace_lag > 0) || (k.layout >= 1 && oo.trace)) {
    k.pace_entries = 4096;  // per field; 5 fields (progress, then trace: start, end, wait, timeouts)
    if (cudaMalloc(&k.pace, k.pace_entries * 8 * 6) != cudaSuccess ||
        cudaMemset(k.pace, 0, k.pace_entries * 8 * 6) != cudaSuccess) {
      cudaGetLastError();
      free_kernel(k);
      err = "cudaMalloc(pace counters)";
      return PMRC_ENOMEM;
    }
  }
  if (m.dyn_on) {
    // dynamic schedule: a ring of counter slots, one per launch (the last team of a group resets
    // its slot), so launches of this plan on different streams do not share counters
    const size_t bytes = (size_t)kDynSlots * 2 * k.n_groups * sizeof(uint32_t);
    if (cudaMalloc(&k.dyn, bytes) != cudaSuccess || cudaMemset(k.dyn, 0, bytes) != cudaSuccess) {
      cudaGetLastError();
      free_kernel(k);
      err = "cudaMalloc(schedule counters)";
      return PMRC_ENOMEM;
    }
    k.dyn_on = true;
    k.dyn_full = m.dyn_full;
  }
  return PMRC_OK;
}

void free_kernel(Kernel &k) {
  if (k.pace) cudaFree(k.pace);
  k.pace = nullptr;
  if (k.dyn) cudaFree(k.dyn);
  k.dyn = nullptr;
  k.dyn_on = false;
  k.dyn_full = false;
  if (k.module && drv().ok) drv().ModuleUnload((CUmodule)k.module);
  k.module = nullptr;
  k.function = nullptr;
}

static int oo_grid(const Kernel &k) { return k.grid_ctas; }

int launch_kernel(const Kernel &k, const uint64_t *ptrs, const uint64_t *strides, size_t S, size_t stripes,
                  void *stream, std::string &err, int max_ctas) {
  if (S == 0 || stripes == 0) return PMRC_OK;
  const uint64_t cb = 128ull * (uint64_t)k.w;  // chunk bytes per block
  const uint64_t chunks64 = (S + cb - 1) / cb;
  if (chunks64 > 0xFFFFFFFFull) { err = "S too large"; return PMRC_EINVAL; }
  const uint32_t chunks = (uint32_t)chunks64;
  // items = stripes * chunks * groups must fit in 32 bits: split launches over stripe ranges
  const uint64_t per_stripe = (uint64_t)chunks;
  const uint64_t max_stripes = std::max<uint64_t>(1, 0xFFFFFFF0ull / per_stripe);
  std::vector<uint64_t> buf(2 * k.n_slots);
  for (size_t s0 = 0; s0 < stripes; s0 += max_stripes) {
    const uint32_t ns = (uint32_t)std::min<uint64_t>(max_stripes, stripes - s0);
    for (int i = 0; i < k.n_slots; i++) {
      buf[i] = ptrs[i] + s0 * strides[i];
      buf[k.n_slots + i] = strides[i];
    }
    uint64_t S64 = S;
    // the kernel splits the ns * chunks chunk range evenly over the CTAs
    uint64_t grid = (uint64_t)k.sms * k.blocks_per_sm;
    // a grid cap lets several small launches (per-stripe failure patterns) share the GPU
    if (max_ctas > 0) grid = std::min<uint64_t>(grid, (uint64_t)max_ctas);
    if (k.layout == 2) {
      grid = max_ctas > 0 ? std::min<uint64_t>((uint64_t)oo_grid(k), grid) : (uint64_t)oo_grid(k);  // equal-cost slices
    } else if (k.layout == 1) {
      // group-specialised: G groups x spg chunk ranges (grid must be a multiple of G)
      const uint64_t G = (uint64_t)k.n_groups;
      uint64_t spg = std::max<uint64_t>(1, grid / G);
      spg = std::min<uint64_t>(spg, (uint64_t)ns * chunks);
      // (the stealing schedule also uses the grid % G CTAs beyond G x spg, as visitors)
      grid = k.dyn_full && grid >= G ? std::min<uint64_t>(grid, G * spg + G - 1) : G * spg;
    } else {
      grid = std::min<uint64_t>(grid, (uint64_t)ns * chunks);
      grid = std::max<uint64_t>(grid, 1);
    }
    // pacing only when every CTA has its counters and can be co-resident
    void *pace = (k.pace && grid * k.teams <= k.pace_entries) ? k.pace : nullptr;
    const uint32_t epoch = ++k.epoch;
    void *dyn = k.dyn_on ? (void *)((uint32_t *)k.dyn + (size_t)(epoch % kDynSlots) * 2 * k.n_groups) : nullptr;
    void *args[] = {buf.data(), &S64, (void *)&ns, (void *)&chunks, &pace, (void *)&epoch, &dyn};
    CUresult cr;
    if (k.pdl && drv().LaunchKernelEx) {
      CUlaunchAttribute at[1];
      at[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
      at[0].value.programmaticStreamSerializationAllowed = 1;
      CUlaunchConfig cfg = {};
      cfg.gridDimX = (unsigned)grid; cfg.gridDimY = 1; cfg.gridDimZ = 1;
      cfg.blockDimX = (unsigned)k.tpb; cfg.blockDimY = 1; cfg.blockDimZ = 1;
      cfg.sharedMemBytes = (unsigned)k.smem;
      cfg.hStream = (CUstream)stream;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cr = drv().LaunchKernelEx(&cfg, (CUfunction)k.function, args, nullptr);
    } else {
      cr = drv().LaunchKernel((CUfunction)k.function, (unsigned)grid, 1, 1, k.tpb, 1, 1, (unsigned)k.smem, (CUstream)stream,
                              args, nullptr);
    }
    if (cr != CUDA_SUCCESS) { err = "cuLaunchKernel: " + cu_err(cr); return PMRC_ECUDA; }
    launch_counter()++;
  }
  return PMRC_OK;
}

}  // namespace pmrc
