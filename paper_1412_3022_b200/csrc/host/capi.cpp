// C ABI of libpmrc (include/pmrc.h): code handles, plan caches, and the data-path entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/pmrc.h"
#include "../rt/rlc.hpp"
#include "construct.hpp"
#include "plan.hpp"
#include "rtplan.hpp"

using namespace pmrc;

namespace {
thread_local std::string g_last_error;

int fail(int rc, const std::string &msg) {
  g_last_error = msg;
  return rc;
}

constexpr int kHostBufs = 3;  // staging ring: H2D of chunk i+1/i+2 overlaps compute and D2H of chunk i
struct HostStage {
  size_t data_bytes = 0;  // allocated size of each d_data[i] (bytes, not stripes: S may change
  size_t par_bytes = 0;   //   between calls on one handle) / of each d_par[i]
  void *d_data[kHostBufs] = {};
  void *d_par[kHostBufs] = {};
  cudaStream_t st[kHostBufs] = {};
  cudaEvent_t ev_start = nullptr;
};
}  // namespace

struct pmrc_code {
  CodeDef def;
  int device = -1;
  GenOptions gen;
  PlanSpec enc_spec;
  Kernel enc;
  bool enc_built = false;
  mutable GenStats enc_stats;       // XOR-program statistics of the encode (pmrc_info; computed on first use)
  mutable bool enc_stats_ok = false;
  std::map<std::string, std::unique_ptr<Kernel>> plans;  // decode / repair / project / combine
  std::map<std::string, int> plan_err;                   // cached failures (ESINGULAR)
  std::map<std::string, int> plan_meta;                  // e.g. blocks written by a decode plan
  HostStage hs;
  int w = 8;                   // symbol width (16: GF(2^16) encode, decode, repair)
  std::vector<uint16_t> psi16, lam16;  // w = 16: Psi (n x d) and Lambda (n)
  const Kernel *traced = nullptr;  // the last launched kernel with pacing / trace counters
  int max_ctas = 0;            // pmrc_set_max_ctas: grid cap for every launch (0 = one full wave)
  std::string *dry = nullptr;  // pmrc_plan_source: get_kernel stores the generated source here instead
  PlanSpec dry_spec;           //   and the plan
  GenStats dry_stats;
  bool dry_compile = false;    //   (and NVRTC-compiles it into the kernel cache if set)
  int policy = PMRC_PLAN_AUTO; // engine choice (pmrc_set_plan_policy)
  std::map<std::string, std::unique_ptr<PlanSpec>> specs;  // plan specs by key (null: nothing to compute)
  std::map<std::string, std::unique_ptr<RtPlan>> rt_plans; // runtime-coefficient plans by key + shape
  bool no_evict = false;       // a batch call holds pointers into the caches: no eviction meanwhile
  // AUTO promotion of hot patterns (pmrc_set_auto_promotion): plan traffic run on the runtime
  // kernel per single-call plan key; past promote_bytes a host thread compiles the pattern's
  // generated kernel into the kernel cache, and the next call after it finished loads and runs it
  unsigned long long promote_bytes = 1ull << 30;
  std::map<std::string, unsigned long long> rt_traffic;
  struct Promotion {
    std::thread th;
    std::atomic<int> state{1};  // 1 compiling, 2 compiled into the cache, 3 failed
  };
  std::map<std::string, std::unique_ptr<Promotion>> promos;
  ~pmrc_code() {
    for (auto &kv : promos)
      if (kv.second->th.joinable()) kv.second->th.join();
  }
};

namespace {

bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }

int check_region(const void *p, size_t stride, size_t stripes) {
  if (!p) return PMRC_EINVAL;
  if (!aligned16(p) || (stripes > 1 && (stride & 15))) return PMRC_EALIGN;
  return PMRC_OK;
}

int ensure_device(pmrc_code *c) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return fail(PMRC_ECUDA, "no CUDA device available (the GPU path has no CPU fallback)");
  }
  if (c->device < 0) c->device = dev;
  if (dev != c->device) return fail(PMRC_EINVAL, "handle was created for another CUDA device");
  return PMRC_OK;
}

constexpr int kDryRun = 1;  // internal: plan generated for pmrc_plan_source, nothing launched

int get_kernel(pmrc_code *c, const std::string &key, const PlanSpec &spec, Kernel **out) {
  if (c->dry) {
    GenStats st;
    *c->dry = plan_source(spec, c->gen, st);
    c->dry_spec = spec;
    c->dry_stats = st;
    if (c->dry_compile) {
      std::string err;
      int rc = precompile_kernel(spec, c->gen, err);
      if (rc) return fail(rc, err);
    }
    return kDryRun;
  }
  auto it = c->plans.find(key);
  if (it != c->plans.end()) {
    *out = it->second.get();
    return PMRC_OK;
  }
  int rc = ensure_device(c);
  if (rc) return rc;
  auto k = std::make_unique<Kernel>();
  std::string err;
  rc = build_kernel(spec, c->gen, *k, err);
  if (rc) return fail(rc, err);
  *out = k.get();
  c->plans[key] = std::move(k);
  return PMRC_OK;
}

// the encode plan is built once per code: CSE restarts with randomised near-ties (keep the cheapest
// network) are worth their host time there (config 2: 12,362 -> 12,305 XORs, 0.501 -> 0.491 ms;
// k = 16 at config 5's size: MSR 935 -> 950 GB/s, MBR 882 -> 909, for ~1-3 s more of host time)
GenOptions enc_gen(const pmrc_code *c) {
  GenOptions g = c->gen;
  if (c->w == 8) g.cse_restarts = std::max(g.cse_restarts, g.enc_restarts);
  if (c->w == 8 && g.part_search == 0) g.part_search = g.enc_part_search;
  return g;
}

int build_encode(pmrc_code *c) {
  if (c->enc_built) return PMRC_OK;
  int rc = ensure_device(c);
  if (rc) return rc;
  std::string err;
  rc = build_kernel(c->enc_spec, enc_gen(c), c->enc, err);
  if (rc) return fail(rc, err);
  c->enc_built = true;
  return PMRC_OK;
}

std::string ids_key(const char *tag, const int *ids, int n, int extra) {
  std::string k = tag;
  k += ":" + std::to_string(extra);
  for (int i = 0; i < n; i++) k += "," + std::to_string(ids[i]);
  return k;
}

int check_ids(const CodeDef &d, const int *ids, int n) {
  for (int i = 0; i < n; i++) {
    if (ids[i] < 0 || ids[i] >= d.n) return PMRC_EINVAL;
    for (int j = 0; j < i; j++)
      if (ids[i] == ids[j]) return PMRC_EINVAL;
  }
  return PMRC_OK;
}

// repair coefficient vector mu of lost node f (MSR: phi_f; MBR: psi_f; RS: [1])
std::vector<uint8_t> repair_mu(const CodeDef &d, int f) {
  if (d.kind == KIND_RS) return {1};
  int m = (d.kind == KIND_MBR) ? d.d : d.alpha;
  std::vector<uint8_t> mu(m);
  for (int t = 0; t < m; t++) mu[t] = d.psi.at(f, t);
  return mu;
}

// newcomer matrix R: out_a = sum_h R[a][h] beta_h  (alpha x n_helpers).  false if singular.
bool repair_matrix(const CodeDef &d, int f, const int *H, Mat &R) {
  if (d.kind == KIND_RS) {
    // lost = G'_f (G'_H)^{-1} [c_h]
    Mat GH(d.k, d.k), GHi;
    for (int a = 0; a < d.k; a++)
      for (int j = 0; j < d.k; j++) GH.at(a, j) = d.Gsys.at(H[a], j);
    if (!invert(GH, GHi)) return false;
    Mat row(1, d.k);
    for (int j = 0; j < d.k; j++) row.at(0, j) = d.Gsys.at(f, j);
    R = matmul(row, GHi);
    return true;
  }
  Mat PH(d.d, d.d), PHi;
  for (int a = 0; a < d.d; a++)
    for (int j = 0; j < d.d; j++) PH.at(a, j) = d.psi.at(H[a], j);
  if (!invert(PH, PHi)) return false;  // R10: predicted singular sets at n >= 2k
  if (d.kind == KIND_MBR) {
    R = PHi;  // piece = z = Psi_H^{-1} beta (M symmetric)
    return true;
  }
  // MSR: piece_a = z_a + lambda_f z_{alpha+a}
  Mat sel(d.alpha, d.d);
  for (int a = 0; a < d.alpha; a++) {
    sel.at(a, a) = 1;
    sel.at(a, d.alpha + a) = d.lambda[f];
  }
  R = matmul(sel, PHi);
  return true;
}

// (id, region) pairs sorted by id: plans and their cache keys depend on id sets, not orders
void canonical_order(const int *ids, const pmrc_cregion *regs, int n, std::vector<int> &ids_out,
                     std::vector<pmrc_cregion> &regs_out) {
  std::vector<int> perm(n);
  for (int i = 0; i < n; i++) perm[i] = i;
  std::sort(perm.begin(), perm.end(), [&](int a, int b) { return ids[a] < ids[b]; });
  ids_out.resize(n);
  regs_out.resize(n);
  for (int i = 0; i < n; i++) {
    ids_out[i] = ids[perm[i]];
    regs_out[i] = regs[perm[i]];
  }
}

// PMRC_GEN parser (see pmrc_create).  Only result-preserving generator options are accepted.
int apply_gen_knobs(const std::string &s, GenOptions &G, std::string &err) {
  struct Knob {
    const char *key;
    int min;
    void (*set)(GenOptions &, int);
  };
  static const Knob knobs[] = {
      {"max_rows", 1, [](GenOptions &o, int v) { o.max_rows = v; }},
      {"in_block", 1, [](GenOptions &o, int v) { o.in_block = v; }},
      {"warps", 1, [](GenOptions &o, int v) { o.warps = v; }},
      {"cse", 0, [](GenOptions &o, int v) { o.cse = v != 0; }},
      {"sync_groups", 0, [](GenOptions &o, int v) { o.sync_groups = v != 0; }},
      {"cta_sync", 0, [](GenOptions &o, int v) { o.cta_sync = v; }},
      {"dyn", -1, [](GenOptions &o, int v) { o.dyn = v; }},
      {"enc_restarts", 1, [](GenOptions &o, int v) { o.enc_restarts = v; }},
      {"part_search", -100000, [](GenOptions &o, int v) { o.part_search = v; }},
      {"enc_part_search", 0, [](GenOptions &o, int v) { o.enc_part_search = v; }},
      {"auto_nbuf", 0, [](GenOptions &o, int v) { o.auto_nbuf = v != 0; }},
      {"smem_kib", 0, [](GenOptions &o, int v) { o.smem_kib = v; }},
      {"pdl", 0, [](GenOptions &o, int v) { o.pdl = v; }},
      {"auto_wide16", 0, [](GenOptions &o, int v) { o.auto_wide16 = v != 0; }},
      {"dyn_static", 0, [](GenOptions &o, int v) { o.dyn_static = v; }},
      {"even_groups", 0, [](GenOptions &o, int v) { o.even_groups = v != 0; }},
      {"tr_balance", 0, [](GenOptions &o, int v) { o.tr_balance = v != 0; }},
      {"cluster_wide", 0, [](GenOptions &o, int v) { o.cluster_wide = v != 0; }},
      {"balance_ranks", 0, [](GenOptions &o, int v) { o.balance_ranks = v != 0; }},
      {"ld_hint", 0, [](GenOptions &o, int v) { o.ld_hint = v; }},
      {"chunk_loop", 1, [](GenOptions &o, int v) { o.chunk_loop = v; }},
      {"team", 1, [](GenOptions &o, int v) { o.team = v; }},
      {"fold", 0, [](GenOptions &o, int v) { o.fold = v != 0; }},
      {"layout", -1, [](GenOptions &o, int v) { o.layout = v; }},
      {"pace_lag", 0, [](GenOptions &o, int v) { o.pace_lag = v; }},
      {"trace", 0, [](GenOptions &o, int v) { o.trace = v != 0; }},
      {"net_in", 0, [](GenOptions &o, int v) { o.net_in = v; }},
      {"net_even", 0, [](GenOptions &o, int v) { o.net_even = v != 0; }},
      {"stage_even", 0, [](GenOptions &o, int v) { o.stage_even = v != 0; }},
      {"fence", 0, [](GenOptions &o, int v) { o.fence = v != 0; }},
      {"tr_unroll", 1, [](GenOptions &o, int v) { o.tr_unroll = v; }},
      {"sched", 0, [](GenOptions &o, int v) { o.sched = v != 0; }},
      {"cse_restarts", 1, [](GenOptions &o, int v) { o.cse_restarts = v; }},
      {"auto_wide", 0, [](GenOptions &o, int v) { o.auto_wide = v != 0; }},
      {"nbuf", 2, [](GenOptions &o, int v) { o.nbuf = v; }},
      {"own_first", 0, [](GenOptions &o, int v) { o.own_first = v != 0; }},
      {"l2_shared", -1, [](GenOptions &o, int v) { o.l2_shared = v; }},
      {"ws", 0, [](GenOptions &o, int v) { o.ws = v != 0; }},
      {"ws_prod", 1, [](GenOptions &o, int v) { o.ws_prod = v; }},
      {"grid_ctas", 1, [](GenOptions &o, int v) { o.grid_ctas = v; }},
      {"rt_groups", 0, [](GenOptions &o, int v) { o.rt_groups = v; }},
      {"rt_rows", 0, [](GenOptions &o, int v) { o.rt_rows = v; }},
  };
  std::string applied;
  size_t pos = 0;
  while (pos < s.size()) {
    size_t e = s.find(',', pos);
    if (e == std::string::npos) e = s.size();
    const std::string kv = s.substr(pos, e - pos);
    pos = e + 1;
    if (kv.empty()) continue;
    const size_t eq = kv.find('=');
    char *end = nullptr;
    const long v = eq == std::string::npos ? 0 : strtol(kv.c_str() + eq + 1, &end, 10);
    if (eq == std::string::npos || end == kv.c_str() + eq + 1 || *end) {
      err = "PMRC_GEN: malformed entry '" + kv + "' (want key=integer)";
      return PMRC_EINVAL;
    }
    const std::string key = kv.substr(0, eq);
    const Knob *k = nullptr;
    for (const Knob &kn : knobs)
      if (key == kn.key) k = &kn;
    if (!k) {
      err = "PMRC_GEN: unknown generator knob '" + key + "'";
      return PMRC_EINVAL;
    }
    if (v < k->min || v > (1 << 20)) {
      err = "PMRC_GEN: value out of range in '" + kv + "'";
      return PMRC_EINVAL;
    }
    k->set(G, (int)v);
    applied += (applied.empty() ? "" : ",") + kv;
  }
  err = "PMRC_GEN applied: " + applied;
  return PMRC_OK;
}

}  // namespace

static int get_rt_plan(pmrc_code *c, const std::string &key, const PlanSpec &spec, int R, int G, RtPlan **out);

extern "C" {

const char *pmrc_strerror(int err) {
  switch (err) {
    case PMRC_OK: return "ok";
    case PMRC_EINVAL: return "invalid argument";
    case PMRC_EUNSUPPORTED: return "unsupported parameters";
    case PMRC_ESINGULAR: return "singular (not decodable / repairable from this set)";
    case PMRC_EALIGN: return "misaligned buffer or block size (GPU path needs S % 16 == 0, 16-B aligned blocks)";
    case PMRC_ENOMEM: return "out of memory";
    case PMRC_ECUDA: return "CUDA error";
    case PMRC_EJIT: return "kernel generation / NVRTC compilation failed";
    default: return "unknown error";
  }
}

const char *pmrc_last_error(void) { return g_last_error.c_str(); }

unsigned long long pmrc_launch_count(void) { return launch_counter().load(); }

int pmrc_create(pmrc_code **out, int kind, int k, int d, int n, int w) {
  if (!out) return fail(PMRC_EINVAL, "out is NULL");
  *out = nullptr;
  std::unique_ptr<pmrc_code> c(new (std::nothrow) pmrc_code());
  if (!c) return fail(PMRC_ENOMEM, "host allocation");
  std::string err;
  if (kind == KIND_RS) d = k;
  // generator tuning knobs (experiments only): PMRC_GEN="max_rows=8,in_block=16,warps=16".  Every
  // knob selects among code-generation strategies that compute the same result (the bitsliced
  // networks are exact whatever the grouping, staging, schedule or warp count); an unknown key or
  // a malformed entry fails pmrc_create with PMRC_EINVAL, so a typo or a stale knob cannot pass
  // silently.  The applied knobs are readable through pmrc_last_error() right after pmrc_create.
  if (const char *g = getenv("PMRC_GEN")) {
    int rc0 = apply_gen_knobs(g, c->gen, err);
    if (rc0) return fail(rc0, err);
    g_last_error = err;
  }
  int rc;
  if (w == 16) {
    // GF(2^16): sparse MSR encode only; the symbols are little-endian byte pairs
    if (kind != KIND_MSR_SPARSE) return fail(PMRC_EUNSUPPORTED, "w = 16: only the sparse MSR code (kind 0)");
    int alpha = 0, B = 0;
    std::vector<uint16_t> gpp;
    rc = build_gpp16(k, d, n, alpha, B, gpp, err, &c->psi16, &c->lam16);
    if (rc) return fail(rc, err);
    CodeDef &D = c->def;
    D.kind = kind; D.n = n; D.k = k; D.d = d; D.alpha = alpha; D.B = B; D.P = (n - k) * alpha;
    D.repair_complete = false;
    c->w = 16;
    c->enc_spec.w = 16;
    c->enc_spec.A16 = gpp;
    c->enc_spec.A = Mat(D.P, D.B);
    for (size_t i = 0; i < gpp.size(); i++) c->enc_spec.A.a[i] = gpp[i] ? 1 : 0;
  } else {
    rc = build_code(kind, k, d, n, w, c->def, err);
    if (rc) return fail(rc, err);
    c->enc_spec.A = c->def.Gpp;
  }
  // encode plan: inputs = data blocks (slot 0), outputs = parity rows (slot 1), A = G''
  const CodeDef &D = c->def;
  c->enc_spec.n_slots = 2;
  for (int i = 0; i < D.B; i++) c->enc_spec.inputs.push_back({{{0, i, 1}}});
  for (int r = 0; r < D.P; r++) c->enc_spec.outputs.push_back({1, r});
  // compile now if a device is present (the paper's initialization); else on first use
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0) {
    rc = build_encode(c.get());
    if (rc) return rc;
  } else {
    cudaGetLastError();
  }
  *out = c.release();
  return PMRC_OK;
}

void pmrc_destroy(pmrc_code *c) {
  if (!c) return;
  int cur = -1;
  bool have = cudaGetDevice(&cur) == cudaSuccess;
  if (c->device >= 0 && have) cudaSetDevice(c->device);
  free_kernel(c->enc);
  for (auto &kv : c->plans) free_kernel(*kv.second);
  for (auto &kv : c->rt_plans) rt_free(*kv.second);
  for (int i = 0; i < kHostBufs; i++) {
    if (c->hs.d_data[i]) cudaFree(c->hs.d_data[i]);
    if (c->hs.d_par[i]) cudaFree(c->hs.d_par[i]);
    if (c->hs.st[i]) cudaStreamDestroy(c->hs.st[i]);
  }
  if (c->hs.ev_start) cudaEventDestroy(c->hs.ev_start);
  if (have && cur >= 0) cudaSetDevice(cur);
  cudaGetLastError();
  delete c;
}

int pmrc_info(const pmrc_code *c, pmrc_info_t *o) {
  if (!c || !o) return fail(PMRC_EINVAL, "NULL argument");
  const CodeDef &D = c->def;
  memset(o, 0, sizeof(*o));
  o->kind = D.kind; o->n = D.n; o->k = D.k; o->d = D.d; o->w = 8;
  o->alpha = D.alpha; o->B = D.B; o->parity_rows = D.P;
  o->w = c->w;
  const Mat &Apat = c->enc_spec.A;  // G'' (w = 16: its nonzero pattern)
  long nnz = 0;
  for (uint8_t v : Apat.a) nnz += v != 0;
  o->nnz = (int)nnz;
  o->zero_pct = Apat.a.empty() ? 0.0 : 100.0 * (double)(Apat.a.size() - nnz) / (double)Apat.a.size();
  o->repair_complete = D.repair_complete ? 1 : 0;
  if (!c->enc_stats_ok) {
    (void)generate_source(c->enc_spec, enc_gen(c), c->enc_stats);
    c->enc_stats_ok = true;
  }
  o->xor_ops = c->enc_stats.xor2;
  o->xor_ops_naive = c->enc_stats.naive_lop3;
  return PMRC_OK;
}

int pmrc_precompile(const pmrc_code *c) {
  if (!c) return fail(PMRC_EINVAL, "NULL handle");
  std::string err;
  int rc = precompile_kernel(c->enc_spec, enc_gen(c), err);
  if (rc) return fail(rc, err);
  return PMRC_OK;
}

int pmrc_debug_counters(const pmrc_code *c, unsigned long long *host, size_t cap, size_t *n) {
  if (!c || !n) return fail(PMRC_EINVAL, "NULL argument");
  *n = 0;
  const Kernel *K = c->traced;  // the last launched kernel that has counters
  if (!K) return PMRC_OK;
  const size_t total = K->pace_entries * 6;
  *n = total;
  if (!host || cap < total) return PMRC_OK;
  if (cudaMemcpy(host, K->pace, total * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return fail(PMRC_ECUDA, "cudaMemcpy(pace counters)");
  }
  return PMRC_OK;
}

int pmrc_plan_source(pmrc_code *c, int op, int lost_id, const int *ids, int n_ids, int compile, char *buf, size_t cap,
                     size_t *len) {
  if (!c || !ids) return fail(PMRC_EINVAL, "NULL argument");
  std::string src;
  c->dry = &src;
  c->dry_compile = compile != 0;
  std::vector<pmrc_cregion> pieces(std::max(1, n_ids), pmrc_cregion{(const void *)(uintptr_t)4096, 0});
  int rc;
  if (op == 0) {
    int nw = 0;
    rc = pmrc_decode(c, ids, n_ids, pieces.data(), (void *)(uintptr_t)4096, 16, 0, &nw, nullptr);
  } else {
    rc = pmrc_repair(c, lost_id, ids, n_ids, pieces.data(), pmrc_region{(void *)(uintptr_t)4096, 0}, 16, 0, nullptr);
  }
  c->dry = nullptr;
  c->dry_compile = false;
  if (rc != kDryRun) return rc ? rc : fail(PMRC_EINVAL, "no kernel for this plan (nothing to compute)");
  if (len) *len = src.size();
  if (buf && cap) {
    size_t n = std::min(cap - 1, src.size());
    memcpy(buf, src.data(), n);
    buf[n] = 0;
  }
  return PMRC_OK;
}

static void fill_stats(const PlanSpec &spec, const GenStats &st, pmrc_plan_stats_t *out);

int pmrc_apply_stats(pmrc_code *c, const uint8_t *A, int rows, int cols, pmrc_plan_stats_t *out) {
  if (!c || !out || !A) return fail(PMRC_EINVAL, "NULL argument");
  memset(out, 0, sizeof(*out));
  std::string src;
  c->dry = &src;
  int rc = pmrc_apply(c, A, rows, cols, (const void *)(uintptr_t)4096, 0, (void *)(uintptr_t)4096, 0, 16, 0, nullptr);
  c->dry = nullptr;
  if (rc != kDryRun) return rc ? rc : fail(PMRC_EINVAL, "no kernel for this matrix");
  fill_stats(c->dry_spec, c->dry_stats, out);
  return PMRC_OK;
}

int pmrc_plan_stats(pmrc_code *c, int op, int lost_id, const int *ids, int n_ids, pmrc_plan_stats_t *out) {
  if (!c || !out) return fail(PMRC_EINVAL, "NULL argument");
  memset(out, 0, sizeof(*out));
  GenStats st;
  PlanSpec spec;
  if (op == 2) {
    (void)plan_source(c->enc_spec, enc_gen(c), st);
    spec = c->enc_spec;
  } else {
    int rc = pmrc_plan_source(c, op, lost_id, ids, n_ids, 0, nullptr, 0, nullptr);
    if (rc) return rc;
    st = c->dry_stats;
    spec = c->dry_spec;
  }
  fill_stats(spec, st, out);
  return PMRC_OK;
}

static void fill_stats(const PlanSpec &spec, const GenStats &st, pmrc_plan_stats_t *out) {
  std::vector<std::pair<int, int>> blocks;
  for (auto &in : spec.inputs)
    for (auto &t : in.terms) blocks.push_back({t.slot, t.blk});
  std::sort(blocks.begin(), blocks.end());
  blocks.erase(std::unique(blocks.begin(), blocks.end()), blocks.end());
  out->groups = st.groups;
  out->in_blocks = (int)blocks.size();
  out->out_blocks = (int)spec.outputs.size();
  out->naive_lop3 = st.naive_lop3;
  out->xor2 = st.xor2;
  out->transposes = st.transposes;
}

int pmrc_encode_source(const pmrc_code *c, char *buf, size_t cap, size_t *len) {
  if (!c) return fail(PMRC_EINVAL, "NULL handle");
  GenStats st;
  std::string src = plan_source(c->enc_spec, enc_gen(c), st);
  if (len) *len = src.size();
  if (buf && cap) {
    size_t n = std::min(cap - 1, src.size());
    memcpy(buf, src.data(), n);
    buf[n] = 0;
  }
  return PMRC_OK;
}

int pmrc_matrix(const pmrc_code *c, int which, uint8_t *buf, int *rows, int *cols) {
  if (c && c->w != 8) return fail(PMRC_EUNSUPPORTED, "w = 16 codes support encode, decode and repair (SURVEY NEXT-4)");
  if (!c || !rows || !cols) return fail(PMRC_EINVAL, "NULL argument");
  const CodeDef &D = c->def;
  const Mat *M = nullptr;
  Mat lam;
  switch (which) {
    case 0: M = &D.psi; break;
    case 1: M = &D.G; break;
    case 2: M = &D.Gsys; break;
    case 3: M = &D.Gpp; break;
    case 5:
      if (D.Gti.r == 0) return fail(PMRC_EUNSUPPORTED, "MBR has no precode matrix (its systematic rows are unit rows)");
      M = &D.Gti;
      break;
    case 4:
      lam = Mat(1, D.n);
      for (int i = 0; i < D.n && i < (int)D.lambda.size(); i++) lam.at(0, i) = D.lambda[i];
      M = &lam;
      break;
    default: return fail(PMRC_EINVAL, "unknown matrix id");
  }
  *rows = M->r;
  *cols = M->c;
  if (buf) memcpy(buf, M->a.data(), M->a.size());
  return PMRC_OK;
}

int pmrc_layout(const pmrc_code *c, int *buf, int *rows, int *cols) {
  if (c && c->w != 8) return fail(PMRC_EUNSUPPORTED, "w = 16 codes support encode, decode and repair (SURVEY NEXT-4)");
  if (!c || !rows || !cols) return fail(PMRC_EINVAL, "NULL argument");
  *rows = c->def.Lrows;
  *cols = c->def.Lcols;
  if (buf) memcpy(buf, c->def.Lidx.data(), sizeof(int) * c->def.Lidx.size());
  return PMRC_OK;
}

int pmrc_encode(pmrc_code *c, const void *data, void *parity, size_t S, size_t stripes, void *stream) {
  if (!c) return fail(PMRC_EINVAL, "NULL handle");
  if (S == 0 || stripes == 0) return PMRC_OK;
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  const CodeDef &D = c->def;
  int rc = check_region(data, (size_t)D.B * S, stripes);
  if (!rc) rc = check_region(parity, (size_t)D.P * S, stripes);
  if (rc) return fail(rc, "bad data/parity pointer");
  uint64_t ptrs[2] = {(uint64_t)(uintptr_t)data, (uint64_t)(uintptr_t)parity};
  uint64_t strides[2] = {(uint64_t)D.B * S, (uint64_t)D.P * S};
  std::string err;
  if (c->policy == PMRC_PLAN_RUNTIME && c->w == 8) {
    // the same G'' on the runtime-coefficient kernel (the formulation comparison of DESIGN.md)
    const pmrc_rt::RlcShape sh = rt_shape(D.P, c->gen);
    RtPlan *P = nullptr;
    rc = get_rt_plan(c, "enc", c->enc_spec, sh.R, sh.G, &P);
    if (rc) return rc;
    rc = ensure_device(c);
    if (rc) return rc;
    rc = rt_launch({P}, nullptr, ptrs, strides, 2, S, stripes, sh, stream, c->max_ctas, err);
    if (rc) return fail(rc, err);
    return PMRC_OK;
  }
  rc = build_encode(c);
  if (rc) return rc;
  if (c->enc.pace) c->traced = &c->enc;
  rc = launch_kernel(c->enc, ptrs, strides, S, stripes, stream, err, c->max_ctas);
  if (rc) return fail(rc, err);
  return PMRC_OK;
}

int pmrc_encode_host(pmrc_code *c, const void *data_host, void *parity_host, size_t S, size_t stripes, void *stream) {
  if (!c || !data_host || !parity_host) return fail(PMRC_EINVAL, "NULL argument");
  if (S == 0 || stripes == 0) return PMRC_OK;
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  int rc = build_encode(c);
  if (rc) return rc;
  const CodeDef &D = c->def;
  HostStage &h = c->hs;
  const size_t in_b = (size_t)D.B * S, out_b = (size_t)D.P * S;
  // chunks of ~64 MiB of source data, a ring of kHostBufs buffers / streams
  size_t chunk = std::max<size_t>(1, ((size_t)64 << 20) / in_b);
  chunk = std::min(chunk, stripes);
  if (h.data_bytes < chunk * in_b || h.par_bytes < chunk * out_b) {
    // (re)allocate by byte size: a later call with a larger S must not reuse smaller buffers
    for (int i = 0; i < kHostBufs; i++) {
      if (h.d_data[i] && cudaStreamSynchronize(h.st[i]) != cudaSuccess) cudaGetLastError();
      if (h.d_data[i]) cudaFree(h.d_data[i]);
      if (h.d_par[i]) cudaFree(h.d_par[i]);
      h.d_data[i] = h.d_par[i] = nullptr;
    }
    h.data_bytes = h.par_bytes = 0;
    const size_t nd = std::max(h.data_bytes, chunk * in_b), np = std::max(h.par_bytes, chunk * out_b);
    for (int i = 0; i < kHostBufs; i++) {
      if (cudaMalloc(&h.d_data[i], nd) != cudaSuccess || cudaMalloc(&h.d_par[i], np) != cudaSuccess) {
        cudaGetLastError();
        for (int j = 0; j <= i; j++) {
          if (h.d_data[j]) cudaFree(h.d_data[j]);
          if (h.d_par[j]) cudaFree(h.d_par[j]);
          h.d_data[j] = h.d_par[j] = nullptr;
        }
        return fail(PMRC_ENOMEM, "staging buffers");
      }
    }
    h.data_bytes = nd;
    h.par_bytes = np;
  }
  for (int i = 0; i < kHostBufs; i++)
    if (!h.st[i] && cudaStreamCreateWithFlags(&h.st[i], cudaStreamNonBlocking) != cudaSuccess)
      return fail(PMRC_ECUDA, "stream create");
  if (!h.ev_start && cudaEventCreateWithFlags(&h.ev_start, cudaEventDisableTiming) != cudaSuccess)
    return fail(PMRC_ECUDA, "event create");
  // order after the caller's stream
  cudaEventRecord(h.ev_start, (cudaStream_t)stream);
  for (int i = 0; i < kHostBufs; i++) cudaStreamWaitEvent(h.st[i], h.ev_start, 0);
  size_t idx = 0;
  for (size_t s0 = 0; s0 < stripes; s0 += chunk, idx++) {
    const size_t ns = std::min(chunk, stripes - s0);
    const int b = (int)(idx % kHostBufs);
    cudaStream_t st = h.st[b];
    if (cudaMemcpyAsync(h.d_data[b], (const uint8_t *)data_host + s0 * in_b, ns * in_b, cudaMemcpyHostToDevice, st) !=
        cudaSuccess)
      return fail(PMRC_ECUDA, "H2D copy");
    uint64_t ptrs[2] = {(uint64_t)(uintptr_t)h.d_data[b], (uint64_t)(uintptr_t)h.d_par[b]};
    uint64_t strides[2] = {in_b, out_b};
    std::string err;
    if (c->enc.pace) c->traced = &c->enc;
  rc = launch_kernel(c->enc, ptrs, strides, S, ns, st, err, c->max_ctas);
    if (rc) return fail(rc, err);
    if (cudaMemcpyAsync((uint8_t *)parity_host + s0 * out_b, h.d_par[b], ns * out_b, cudaMemcpyDeviceToHost, st) !=
        cudaSuccess)
      return fail(PMRC_ECUDA, "D2H copy");
  }
  for (int i = 0; i < kHostBufs; i++)
    if (cudaStreamSynchronize(h.st[i]) != cudaSuccess) return fail(PMRC_ECUDA, cudaGetErrorString(cudaGetLastError()));
  return PMRC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// Plan specs of decode and repair.  slot_of[q] is the slot that survivor / helper q's piece is
// read from (single calls: q; batch calls: the node id), out_slot the output region's slot.
// Each returns PMRC_OK, PMRC_ESINGULAR, or kNothing (no block to compute).
// ---------------------------------------------------------------------------------------------
constexpr int kNothing = 1;

// GF(2^16) decode plan (w = 16): the same rule as the GF(2^8) plan (R13): greedy B
// independent rows of G' = [I_B; G''], systematic survivors first, then the inverse's rows of the
// data blocks no surviving systematic node holds.
static int decode_spec16(const pmrc_code *c, const int *surv_ids, int n_surv, const int *slot_of, int out_slot,
                         int n_slots, PlanSpec &spec) {
  const CodeDef &D = c->def;
  const GF65536 &F = gf16();
  const int B = D.B, a = D.alpha;
  const std::vector<uint16_t> &Gpp = c->enc_spec.A16;
  auto row_of = [&](int node, int j, std::vector<uint16_t> &row) {
    row.assign(B, 0);
    if (node < D.k) row[node * a + j] = 1;
    else for (int x = 0; x < B; x++) row[x] = Gpp[(size_t)((node - D.k) * a + j) * B + x];
  };
  std::vector<int> order;
  for (int pass = 0; pass < 2; pass++)
    for (int id = 0; id < D.n; id++) {
      if ((pass == 0) != (id < D.k)) continue;
      for (int q = 0; q < n_surv; q++)
        if (surv_ids[q] == id) order.push_back(q);
    }
  std::vector<std::vector<uint16_t>> basis, selrows;
  std::vector<int> pivcol;
  std::vector<std::pair<int, int>> sel;
  std::vector<uint16_t> row;
  for (int q : order)
    for (int j = 0; j < a && (int)sel.size() < B; j++) {
      row_of(surv_ids[q], j, row);
      std::vector<uint16_t> red = row;
      for (size_t bi = 0; bi < basis.size(); bi++) {
        const uint16_t f = red[pivcol[bi]];
        if (!f) continue;
        for (int x = 0; x < B; x++) red[x] ^= F.mul(f, basis[bi][x]);
      }
      int pc = -1;
      for (int x = 0; x < B; x++)
        if (red[x]) { pc = x; break; }
      if (pc < 0) continue;
      const uint16_t sc = F.inv(red[pc]);
      for (int x = 0; x < B; x++) red[x] = F.mul(red[x], sc);
      for (size_t bi = 0; bi < basis.size(); bi++) {
        const uint16_t f = basis[bi][pc];
        if (!f) continue;
        for (int x = 0; x < B; x++) basis[bi][x] ^= F.mul(f, red[x]);
      }
      basis.push_back(red);
      pivcol.push_back(pc);
      selrows.push_back(row);
      sel.push_back({q, j});
    }
  if ((int)sel.size() < B) return PMRC_ESINGULAR;
  // invert the selected rows (Gauss-Jordan)
  std::vector<uint16_t> Wm((size_t)B * B), Inv((size_t)B * B, 0);
  for (int r = 0; r < B; r++) {
    for (int x = 0; x < B; x++) Wm[(size_t)r * B + x] = selrows[r][x];
    Inv[(size_t)r * B + r] = 1;
  }
  for (int col = 0; col < B; col++) {
    int piv = -1;
    for (int r = col; r < B; r++)
      if (Wm[(size_t)r * B + col]) { piv = r; break; }
    if (piv < 0) return PMRC_ESINGULAR;
    if (piv != col)
      for (int x = 0; x < B; x++) {
        std::swap(Wm[(size_t)piv * B + x], Wm[(size_t)col * B + x]);
        std::swap(Inv[(size_t)piv * B + x], Inv[(size_t)col * B + x]);
      }
    const uint16_t sc = F.inv(Wm[(size_t)col * B + col]);
    for (int x = 0; x < B; x++) {
      Wm[(size_t)col * B + x] = F.mul(Wm[(size_t)col * B + x], sc);
      Inv[(size_t)col * B + x] = F.mul(Inv[(size_t)col * B + x], sc);
    }
    for (int r = 0; r < B; r++) {
      const uint16_t f = r == col ? 0 : Wm[(size_t)r * B + col];
      if (!f) continue;
      for (int x = 0; x < B; x++) {
        Wm[(size_t)r * B + x] ^= F.mul(f, Wm[(size_t)col * B + x]);
        Inv[(size_t)r * B + x] ^= F.mul(f, Inv[(size_t)col * B + x]);
      }
    }
  }
  std::vector<char> held(B, 0);
  for (int q = 0; q < n_surv; q++)
    if (surv_ids[q] < D.k)
      for (int j = 0; j < a; j++) held[surv_ids[q] * a + j] = 1;
  std::vector<int> missing, used;
  for (int x = 0; x < B; x++)
    if (!held[x]) missing.push_back(x);
  if (missing.empty()) return kNothing;
  for (int x = 0; x < B; x++) {
    bool nz = false;
    for (int m : missing) nz |= Inv[(size_t)m * B + x] != 0;
    if (nz) used.push_back(x);
  }
  spec = PlanSpec();
  spec.n_slots = n_slots;
  spec.w = 16;
  for (int x : used) spec.inputs.push_back({{{slot_of[sel[x].first], sel[x].second, 1}}});
  for (int m : missing) spec.outputs.push_back({out_slot, m});
  spec.A = Mat((int)missing.size(), (int)used.size());
  spec.A16.assign(missing.size() * used.size(), 0);
  for (size_t r = 0; r < missing.size(); r++)
    for (size_t x = 0; x < used.size(); x++) {
      const uint16_t v = Inv[(size_t)missing[r] * B + used[x]];
      spec.A16[r * used.size() + x] = v;
      spec.A.at((int)r, (int)x) = v ? 1 : 0;
    }
  return PMRC_OK;
}

// GF(2^8) decode plan (R13): greedy B independent rows of G', systematic survivors
// first, then ascending id; invert; keep the rows of the data blocks no surviving systematic node
// holds, over the columns they use (the lazy decode of P:106: only missing blocks are computed).
static int decode_spec8(const pmrc_code *c, const int *surv_ids, int n_surv, const int *slot_of, int out_slot,
                        int n_slots, PlanSpec &spec) {
  const CodeDef &D = c->def;
  std::vector<int> order;
  for (int pass = 0; pass < 2; pass++)
    for (int id = 0; id < D.n; id++) {
      if ((pass == 0) != (id < D.k)) continue;
      for (int a = 0; a < n_surv; a++)
        if (surv_ids[a] == id) order.push_back(a);
    }
  std::vector<std::vector<uint8_t>> basis;  // reduced rows (incremental elimination)
  std::vector<int> pivcol;
  std::vector<std::pair<int, int>> sel;  // (survivor index, symbol)
  Mat Sel(D.B, D.B);
  const GF256 &F = gf();
  for (int a : order) {
    for (int j = 0; j < D.alpha && (int)sel.size() < D.B; j++) {
      std::vector<uint8_t> row(D.B);
      for (int x = 0; x < D.B; x++) row[x] = D.Gsys.at(surv_ids[a] * D.alpha + j, x);
      std::vector<uint8_t> red = row;
      for (size_t bi = 0; bi < basis.size(); bi++) {
        uint8_t f = red[pivcol[bi]];
        if (!f) continue;
        for (int x = 0; x < D.B; x++) red[x] ^= F.mul(f, basis[bi][x]);
      }
      int pc = -1;
      for (int x = 0; x < D.B; x++)
        if (red[x]) { pc = x; break; }
      if (pc < 0) continue;
      uint8_t s = F.inv(red[pc]);
      for (int x = 0; x < D.B; x++) red[x] = F.mul(red[x], s);
      for (size_t bi = 0; bi < basis.size(); bi++) {
        uint8_t f = basis[bi][pc];
        if (!f) continue;
        for (int x = 0; x < D.B; x++) basis[bi][x] ^= F.mul(f, red[x]);
      }
      basis.push_back(red);
      pivcol.push_back(pc);
      for (int x = 0; x < D.B; x++) Sel.at((int)sel.size(), x) = row[x];
      sel.push_back({a, j});
    }
  }
  if ((int)sel.size() < D.B) return PMRC_ESINGULAR;
  Mat Inv;
  if (!invert(Sel, Inv)) return PMRC_ESINGULAR;
  std::vector<char> held(D.B, 0);
  for (int a = 0; a < n_surv; a++)
    if (surv_ids[a] < D.k)
      for (int j = 0; j < D.alpha; j++) held[D.sys_block(surv_ids[a], j)] = 1;
  std::vector<int> missing;
  for (int x = 0; x < D.B; x++)
    if (!held[x]) missing.push_back(x);
  if (missing.empty()) return kNothing;
  spec = PlanSpec();
  spec.n_slots = n_slots;
  std::vector<int> used_cols;
  for (int x = 0; x < D.B; x++) {
    bool nz = false;
    for (int m : missing) nz |= Inv.at(m, x) != 0;
    if (nz) used_cols.push_back(x);
  }
  for (int x : used_cols) spec.inputs.push_back({{{slot_of[sel[x].first], sel[x].second, 1}}});
  for (int m : missing) spec.outputs.push_back({out_slot, m});
  spec.A = Mat((int)missing.size(), (int)used_cols.size());
  for (size_t r = 0; r < missing.size(); r++)
    for (size_t x = 0; x < used_cols.size(); x++) spec.A.at((int)r, (int)x) = Inv.at(missing[r], used_cols[x]);
  return PMRC_OK;
}

static int decode_spec(const pmrc_code *c, const int *surv, int n_surv, const int *slot_of, int out_slot, int n_slots,
                       PlanSpec &spec) {
  return c->w == 16 ? decode_spec16(c, surv, n_surv, slot_of, out_slot, n_slots, spec)
                    : decode_spec8(c, surv, n_surv, slot_of, out_slot, n_slots, spec);
}

// Fused repair plan (P:53 footnote): input h = beta_h = mu . piece_h (derived; only
// the blocks with a nonzero mu are read), outputs = the alpha blocks of the lost piece,
// A = R (the newcomer's matrix: MSR [I | lambda_f I] Psi_H^{-1}, MBR Psi_H^{-1}, RS G'_f (G'_H)^{-1}).
static int repair_spec(const pmrc_code *c, int f, const int *H, int nh, const int *slot_of, int out_slot, int n_slots,
                       PlanSpec &spec) {
  const CodeDef &D = c->def;
  spec = PlanSpec();
  spec.n_slots = n_slots;
  if (c->w == 16) {
    const GF65536 &F = gf16();
    const int dd = D.d, a = D.alpha;
    std::vector<uint16_t> Wm((size_t)dd * dd), Inv((size_t)dd * dd, 0);
    for (int r = 0; r < dd; r++) {
      for (int x = 0; x < dd; x++) Wm[(size_t)r * dd + x] = c->psi16[(size_t)H[r] * dd + x];
      Inv[(size_t)r * dd + r] = 1;
    }
    for (int col = 0; col < dd; col++) {
      int piv = -1;
      for (int r = col; r < dd; r++)
        if (Wm[(size_t)r * dd + col]) { piv = r; break; }
      if (piv < 0) return PMRC_ESINGULAR;
      if (piv != col)
        for (int x = 0; x < dd; x++) {
          std::swap(Wm[(size_t)piv * dd + x], Wm[(size_t)col * dd + x]);
          std::swap(Inv[(size_t)piv * dd + x], Inv[(size_t)col * dd + x]);
        }
      const uint16_t sc = F.inv(Wm[(size_t)col * dd + col]);
      for (int x = 0; x < dd; x++) {
        Wm[(size_t)col * dd + x] = F.mul(Wm[(size_t)col * dd + x], sc);
        Inv[(size_t)col * dd + x] = F.mul(Inv[(size_t)col * dd + x], sc);
      }
      for (int r = 0; r < dd; r++) {
        const uint16_t g = r == col ? 0 : Wm[(size_t)r * dd + col];
        if (!g) continue;
        for (int x = 0; x < dd; x++) {
          Wm[(size_t)r * dd + x] ^= F.mul(g, Wm[(size_t)col * dd + x]);
          Inv[(size_t)r * dd + x] ^= F.mul(g, Inv[(size_t)col * dd + x]);
        }
      }
    }
    const uint16_t lf = c->lam16[f];
    spec.w = 16;
    for (int h = 0; h < nh; h++) {
      InputDesc in;
      for (int b = 0; b < a; b++) {
        const uint16_t mu = c->psi16[(size_t)f * dd + b];
        if (mu) in.terms.push_back({slot_of[h], b, mu});
      }
      spec.inputs.push_back(in);
    }
    for (int q = 0; q < a; q++) spec.outputs.push_back({out_slot, q});
    spec.A = Mat(a, nh);
    spec.A16.assign((size_t)a * nh, 0);
    for (int q = 0; q < a; q++)
      for (int h = 0; h < nh; h++) {
        const uint16_t v = Inv[(size_t)q * dd + h] ^ F.mul(lf, Inv[(size_t)(a + q) * dd + h]);
        spec.A16[(size_t)q * nh + h] = v;
        spec.A.at(q, h) = v ? 1 : 0;
      }
    return PMRC_OK;
  }
  Mat R;
  if (!repair_matrix(D, f, H, R)) return PMRC_ESINGULAR;  // R10: predicted singular sets at n >= 2k
  std::vector<uint8_t> mu = repair_mu(D, f);
  for (int h = 0; h < nh; h++) {
    InputDesc in;
    for (size_t b = 0; b < mu.size(); b++)
      if (mu[b]) in.terms.push_back({slot_of[h], (int)b, mu[b]});
    spec.inputs.push_back(in);
  }
  for (int a = 0; a < D.alpha; a++) spec.outputs.push_back({out_slot, a});
  spec.A = R;
  return PMRC_OK;
}

// ---------------------------------------------------------------------------------------------
// Engines.  Every data-path call runs a plan on one of two kernels:
//   JIT      the generated bitsliced kernel of the plan (codegen.cpp; NVRTC on first use unless
//            the in-tree cache has it): the fastest, but the first contact with a new failure
//            pattern costs kernel generation + NVRTC (seconds)
//   RUNTIME  the precompiled runtime-coefficient kernel (csrc/rt/rlc.cu): coefficients are data,
//            a new pattern costs the host inversion + table fill (P:216's initialisation)
// Policy PMRC_PLAN_AUTO (default): JIT for the encode (compiled at pmrc_create) and for plans whose
// JIT kernel is already loaded on the handle (pmrc_plan_prepare / earlier JIT calls / a finished
// background promotion, maybe_promote), RUNTIME for every other plan; GF(2^16) plans always use JIT.
// ---------------------------------------------------------------------------------------------
static bool use_runtime(const pmrc_code *c, const std::string &key) {
  if (c->w != 8) return false;
  if (c->policy == PMRC_PLAN_JIT) return false;
  if (c->policy == PMRC_PLAN_RUNTIME) return true;
  return !c->plans.count(key);
}

constexpr size_t kMaxRtPlans = 1024;  // runtime plans cached per handle (<= ~160 KB device memory each)
constexpr size_t kMaxSpecs = 8192;     // plan specs cached per handle

static std::string rt_key(const std::string &key, int R, int G) {
  return key + "#rt" + std::to_string(R) + "x" + std::to_string(G);
}

// runtime plan of `spec` for R-row blocks and G row groups, cached on the handle under `key`
static int get_rt_plan(pmrc_code *c, const std::string &key, const PlanSpec &spec, int R, int G, RtPlan **out) {
  const std::string k = rt_key(key, R, G);
  auto it = c->rt_plans.find(k);
  if (it != c->rt_plans.end()) {
    *out = it->second.get();
    return PMRC_OK;
  }
  if (c->rt_plans.size() >= kMaxRtPlans && !c->no_evict) {
    // bounded cache (a batch of many patterns per call can add thousands): the device copies may
    // still be read by launches in flight, so drop them only after the device is idle
    if (cudaDeviceSynchronize() != cudaSuccess) {
      cudaGetLastError();
      return fail(PMRC_ECUDA, "cudaDeviceSynchronize (plan cache eviction)");
    }
    for (auto &kv : c->rt_plans) rt_free(*kv.second);
    c->rt_plans.clear();
  }
  auto p = std::make_unique<RtPlan>();
  std::string err;
  int rc = rt_build(spec, R, G, *p, err);
  if (rc) return fail(rc, err);
  *out = p.get();
  c->rt_plans[k] = std::move(p);
  return PMRC_OK;
}

// The plan cache: key -> spec (built once; nullptr-equivalent when the plan computes nothing),
// cached failures (ESINGULAR) in plan_err, number of outputs in plan_meta.
template <class Make>
static int get_spec(pmrc_code *c, const std::string &key, Make make, const PlanSpec **out) {
  *out = nullptr;
  auto fe = c->plan_err.find(key);
  if (fe != c->plan_err.end())
    return fail(fe->second, fe->second == PMRC_ESINGULAR ? "singular (cached): survivors do not span the data / "
                                                           "Psi_H singular (DESIGN.md R10)"
                                                         : "plan failed (cached)");
  auto it = c->specs.find(key);
  if (it == c->specs.end() && c->specs.size() >= kMaxSpecs && !c->no_evict) {
    // bounded host cache of plan specs (only referenced during a call); loaded JIT kernels and
    // runtime plans keep their own caches
    c->specs.clear();
    c->plan_meta.clear();
    it = c->specs.end();
  }
  if (it == c->specs.end() || c->dry) {
    auto sp = std::make_unique<PlanSpec>();
    const int rc = make(*sp);
    if (rc == PMRC_ESINGULAR) {
      c->plan_err[key] = rc;
      return fail(rc, "singular: survivors do not span the data / Psi_H singular for this (lost, helpers) pair "
                      "(DESIGN.md R10)");
    }
    if (rc && rc != kNothing) return rc;
    c->plan_meta[key] = rc == kNothing ? 0 : (int)sp->outputs.size();
    if (rc == kNothing) sp.reset();
    it = c->specs.insert_or_assign(key, std::move(sp)).first;
  }
  *out = it->second.get();
  return PMRC_OK;
}

// Hot-pattern promotion under AUTO.  Traffic of a plan = S x stripes x (distinct input blocks +
// outputs).  Once a pattern's runtime-kernel traffic reaches promote_bytes, a host thread
// generates and NVRTC-compiles its kernel into the kernel cache (the calls keep running on the
// runtime kernel meanwhile); the first call after that loads the cubin through the plan index
// (milliseconds) and runs the generated kernel from then on.  Needs the kernel cache.
static void maybe_promote(pmrc_code *c, const std::string &key, const PlanSpec &spec, unsigned long long cols) {
  if (!c->promote_bytes || c->promos.count(key) || !kernel_cache_enabled()) return;
  if (c->rt_traffic.size() > kMaxSpecs) c->rt_traffic.clear();
  std::vector<std::pair<int, int>> blocks;
  for (const auto &in : spec.inputs)
    for (const auto &t : in.terms) blocks.push_back({t.slot, t.blk});
  std::sort(blocks.begin(), blocks.end());
  blocks.erase(std::unique(blocks.begin(), blocks.end()), blocks.end());
  unsigned long long &tr = c->rt_traffic[key];
  tr += cols * (unsigned long long)(blocks.size() + spec.outputs.size());
  if (tr < c->promote_bytes) return;
  auto pr = std::make_unique<pmrc_code::Promotion>();
  pmrc_code::Promotion *pp = pr.get();
  pr->th = std::thread([pp, sp = spec, g = c->gen]() {
    std::string err;
    pp->state = precompile_kernel(sp, g, err) == PMRC_OK ? 2 : 3;
  });
  c->promos[key] = std::move(pr);
}

// true when the pattern's promotion finished and its kernel is in the cache's plan index for the
// handle's current options (then get_kernel loads it without generation or NVRTC)
static bool promotion_done(pmrc_code *c, const std::string &key, const PlanSpec &spec) {
  auto it = c->promos.find(key);
  if (it == c->promos.end() || it->second->state.load() == 1) return false;
  it->second->th.join();
  const bool ok = it->second->state.load() == 2 && plan_indexed(spec, c->gen);
  if (!ok) {
    c->promos.erase(it);  // failed, or compiled for options changed since: account afresh
    c->rt_traffic.erase(key);
    return false;
  }
  c->promos.erase(it);
  Kernel *K = nullptr;
  return get_kernel(c, key, spec, &K) == PMRC_OK;
}

// Run a single plan over `stripes` stripes (slots of stripe 0 in ptrs, their strides).
static int run_plan(pmrc_code *c, const std::string &key, const PlanSpec &spec, const uint64_t *ptrs,
                    const uint64_t *strides, size_t S, size_t stripes, void *stream) {
  std::string err;
  if (c->dry) {
    Kernel *K = nullptr;
    return get_kernel(c, key, spec, &K);  // kDryRun (source / stats only)
  }
  bool rt = use_runtime(c, key);
  if (rt && c->policy == PMRC_PLAN_AUTO && promotion_done(c, key, spec)) rt = false;
  if (rt) {
    const pmrc_rt::RlcShape sh = rt_shape((int)spec.outputs.size(), c->gen);
    RtPlan *P = nullptr;
    int rc = get_rt_plan(c, key, spec, sh.R, sh.G, &P);
    if (rc == PMRC_OK) {
      if (!stripes || !S) return PMRC_OK;
      rc = ensure_device(c);
      if (rc) return rc;
      rc = rt_launch({P}, nullptr, ptrs, strides, spec.n_slots, S, stripes, sh, stream, c->max_ctas, err);
      if (rc) return fail(rc, err);
      if (c->policy == PMRC_PLAN_AUTO) maybe_promote(c, key, spec, (unsigned long long)S * stripes);
      return PMRC_OK;
    }
    if (!(rc == PMRC_EUNSUPPORTED && c->policy == PMRC_PLAN_AUTO)) return rc;
    // AUTO: plans the runtime kernel cannot hold (wiring and masks above its shared-memory budget,
    // more than kRlcMaxSlots regions) use JIT
  }
  Kernel *K = nullptr;
  int rc = get_kernel(c, key, spec, &K);
  if (rc) return rc;
  if (!stripes || !S) return PMRC_OK;
  if (K->pace) c->traced = K;
  rc = launch_kernel(*K, ptrs, strides, S, stripes, stream, err, c->max_ctas);
  if (rc) return fail(rc, err);
  return PMRC_OK;
}

extern "C" {

int pmrc_decode(pmrc_code *c, const int *surv_ids_in, int n_surv, const pmrc_cregion *pieces_in, void *data_out,
                size_t S, size_t stripes, int *n_written, void *stream) {
  if (n_written) *n_written = 0;
  if (!c || !surv_ids_in || !pieces_in || !data_out) return fail(PMRC_EINVAL, "NULL argument");
  const CodeDef &D = c->def;
  if (n_surv < 1 || n_surv > D.n || check_ids(D, surv_ids_in, n_surv)) return fail(PMRC_EINVAL, "bad survivor ids");
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  // canonical order: the plan (and its cache key) depends on the survivor SET only; the pieces are
  // permuted with the ids (the decoded data is unique, so the order cannot change it)
  std::vector<int> surv;
  std::vector<pmrc_cregion> pieces;
  canonical_order(surv_ids_in, pieces_in, n_surv, surv, pieces);
  const std::string key = ids_key("dec", surv.data(), n_surv, 0);
  std::vector<int> slot_of(n_surv);
  for (int q = 0; q < n_surv; q++) slot_of[q] = q;
  const PlanSpec *spec = nullptr;
  int rc = get_spec(c, key, [&](PlanSpec &sp) { return decode_spec(c, surv.data(), n_surv, slot_of.data(), n_surv,
                                                                    n_surv + 1, sp); },
                    &spec);
  if (rc) return rc;
  const int written = c->plan_meta[key];
  if (n_written) *n_written = written;
  if (!spec) return PMRC_OK;  // every data block survives on a systematic node
  std::vector<uint64_t> ptrs(n_surv + 1), strides(n_surv + 1);
  if (!c->dry && stripes && S) {
    for (int a = 0; a < n_surv; a++) {
      rc = check_region(pieces[a].ptr, pieces[a].stripe_stride, stripes);
      if (rc) return fail(rc, "bad survivor piece region");
    }
    rc = check_region(data_out, (size_t)D.B * S, stripes);
    if (rc) return fail(rc, "bad data_out");
  }
  for (int a = 0; a < n_surv; a++) {
    ptrs[a] = (uint64_t)(uintptr_t)pieces[a].ptr;
    strides[a] = pieces[a].stripe_stride;
  }
  ptrs[n_surv] = (uint64_t)(uintptr_t)data_out;
  strides[n_surv] = (uint64_t)D.B * S;
  return run_plan(c, key, *spec, ptrs.data(), strides.data(), S, stripes, stream);
}

int pmrc_apply(pmrc_code *c, const uint8_t *A, int rows, int cols, const void *in, size_t in_stride, void *out,
               size_t out_stride, size_t S, size_t stripes, void *stream) {
  if (c && c->w != 8) return fail(PMRC_EUNSUPPORTED, "w = 16 codes support encode, decode and repair (SURVEY NEXT-4)");
  if (!c || !A || !in || !out) return fail(PMRC_EINVAL, "NULL argument");
  if (rows < 1 || cols < 1 || rows > 4096 || cols > 4096) return fail(PMRC_EINVAL, "bad matrix shape");
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  // plan key: shape + FNV-1a of the coefficients (the matrix defines the kernel)
  uint64_t h = 1469598103934665603ull;
  for (long i = 0; i < (long)rows * cols; i++) h = (h ^ A[i]) * 1099511628211ull;
  char kb[96];
  snprintf(kb, sizeof kb, "apply:%dx%d:%016llx", rows, cols, (unsigned long long)h);
  const std::string key = kb;
  bool any = false;
  for (long i = 0; i < (long)rows * cols; i++) any |= A[i] != 0;
  if (!any) return fail(PMRC_EINVAL, "all-zero matrix (nothing to compute)");
  const PlanSpec *spec = nullptr;
  int rc = get_spec(c, key, [&](PlanSpec &sp) {
    sp.n_slots = 2;
    for (int x = 0; x < cols; x++) sp.inputs.push_back({{{0, x, 1}}});
    for (int r = 0; r < rows; r++) sp.outputs.push_back({1, r});
    sp.A = Mat(rows, cols);
    memcpy(sp.A.a.data(), A, (size_t)rows * cols);
    return PMRC_OK;
  }, &spec);
  if (rc) return rc;
  if (!c->dry && stripes && S) {
    rc = check_region(in, in_stride, stripes);
    if (!rc) rc = check_region(out, out_stride, stripes);
    if (rc) return fail(rc, "bad in/out region");
  }
  uint64_t ptrs[2] = {(uint64_t)(uintptr_t)in, (uint64_t)(uintptr_t)out};
  uint64_t strides[2] = {(uint64_t)in_stride, (uint64_t)out_stride};
  return run_plan(c, key, *spec, ptrs, strides, S, stripes, stream);
}

int pmrc_set_max_ctas(pmrc_code *c, int max_ctas) {
  if (!c || max_ctas < 0) return fail(PMRC_EINVAL, "bad argument");
  c->max_ctas = max_ctas;
  return PMRC_OK;
}

int pmrc_set_plan_policy(pmrc_code *c, int policy) {
  if (!c || policy < PMRC_PLAN_AUTO || policy > PMRC_PLAN_RUNTIME) return fail(PMRC_EINVAL, "bad argument");
  c->policy = policy;
  return PMRC_OK;
}

int pmrc_get_plan_policy(const pmrc_code *c) { return c ? c->policy : PMRC_EINVAL; }

int pmrc_set_independent_launches(pmrc_code *c, int on) {
  if (!c || on < 0 || on > 1) return fail(PMRC_EINVAL, "bad argument");
  const int want = on ? 2 : 0;
  if (c->gen.pdl == want) return PMRC_OK;
  // the kernels are generated with or without the PDL prologue: drop the built ones (they are
  // rebuilt on next use, from the in-tree cubin cache when present) after the device is idle
  if ((c->enc_built || !c->plans.empty()) && cudaDeviceSynchronize() != cudaSuccess) {
    cudaGetLastError();
    return fail(PMRC_ECUDA, "cudaDeviceSynchronize");
  }
  c->gen.pdl = want;
  free_kernel(c->enc);
  c->enc = Kernel();
  c->enc_built = false;
  for (auto &kv : c->plans) free_kernel(*kv.second);
  c->plans.clear();
  c->traced = nullptr;
  return PMRC_OK;
}

int pmrc_read_cost(const pmrc_code *c, int lost_id, int *blocks) {
  if (c && c->w != 8) return fail(PMRC_EUNSUPPORTED, "w = 16 codes support encode, decode and repair (SURVEY NEXT-4)");
  if (!c || !blocks) return fail(PMRC_EINVAL, "NULL argument");
  if (lost_id < 0 || lost_id >= c->def.n) return fail(PMRC_EINVAL, "bad lost id");
  int cnt = 0;
  for (uint8_t v : repair_mu(c->def, lost_id)) cnt += v != 0;
  *blocks = cnt;
  return PMRC_OK;
}

static int repair_common(pmrc_code *c, int lost_id, const int *helper_ids, int n_helpers, int *need) {
  const CodeDef &D = c->def;
  *need = (D.kind == KIND_RS) ? D.k : D.d;
  if (lost_id < 0 || lost_id >= D.n) return fail(PMRC_EINVAL, "bad lost id");
  if (n_helpers != *need) return fail(PMRC_EINVAL, "repair needs exactly d helpers (RS: k)");
  if (check_ids(D, helper_ids, n_helpers)) return fail(PMRC_EINVAL, "bad helper ids");
  for (int i = 0; i < n_helpers; i++)
    if (helper_ids[i] == lost_id) return fail(PMRC_EINVAL, "lost node among helpers");
  return PMRC_OK;
}

int pmrc_repair(pmrc_code *c, int lost_id, const int *helper_ids_in, int n_helpers,
                const pmrc_cregion *helper_pieces_in, pmrc_region out_piece, size_t S, size_t stripes, void *stream) {
  if (!c || !helper_ids_in || !helper_pieces_in) return fail(PMRC_EINVAL, "NULL argument");
  int need = 0;
  int rc = repair_common(c, lost_id, helper_ids_in, n_helpers, &need);
  if (rc) return rc;
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  // canonical helper order (the plan depends on the helper SET; the repaired piece is unique)
  std::vector<int> H;
  std::vector<pmrc_cregion> hp;
  canonical_order(helper_ids_in, helper_pieces_in, n_helpers, H, hp);
  const std::string key = ids_key("rep", H.data(), n_helpers, lost_id);
  std::vector<int> slot_of(n_helpers);
  for (int q = 0; q < n_helpers; q++) slot_of[q] = q;
  const PlanSpec *spec = nullptr;
  rc = get_spec(c, key, [&](PlanSpec &sp) {
    return repair_spec(c, lost_id, H.data(), n_helpers, slot_of.data(), n_helpers, n_helpers + 1, sp);
  }, &spec);
  if (rc) return rc;
  std::vector<uint64_t> ptrs(n_helpers + 1), strides(n_helpers + 1);
  if (!c->dry && stripes && S) {
    for (int h = 0; h < n_helpers; h++) {
      rc = check_region(hp[h].ptr, hp[h].stripe_stride, stripes);
      if (rc) return fail(rc, "bad helper piece region");
    }
    rc = check_region(out_piece.ptr, out_piece.stripe_stride, stripes);
    if (rc) return fail(rc, "bad output piece region");
  }
  for (int h = 0; h < n_helpers; h++) {
    ptrs[h] = (uint64_t)(uintptr_t)hp[h].ptr;
    strides[h] = hp[h].stripe_stride;
  }
  ptrs[n_helpers] = (uint64_t)(uintptr_t)out_piece.ptr;
  strides[n_helpers] = out_piece.stripe_stride;
  return run_plan(c, key, *spec, ptrs.data(), strides.data(), S, stripes, stream);
}

int pmrc_repair_project(pmrc_code *c, int lost_id, pmrc_cregion piece, pmrc_region beta, size_t S, size_t stripes,
                        void *stream) {
  if (c && c->w != 8) return fail(PMRC_EUNSUPPORTED, "w = 16 codes support encode, decode and repair (SURVEY NEXT-4)");
  if (!c) return fail(PMRC_EINVAL, "NULL handle");
  const CodeDef &D = c->def;
  if (lost_id < 0 || lost_id >= D.n) return fail(PMRC_EINVAL, "bad lost id");
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  const std::string key = "proj:" + std::to_string(lost_id);
  const PlanSpec *spec = nullptr;
  int rc = get_spec(c, key, [&](PlanSpec &sp) {
    std::vector<uint8_t> mu = repair_mu(D, lost_id);
    sp.n_slots = 2;
    std::vector<int> cols;
    for (size_t b = 0; b < mu.size(); b++)
      if (mu[b]) {
        sp.inputs.push_back({{{0, (int)b, 1}}});  // only blocks with nonzero mu are read
        cols.push_back((int)b);
      }
    sp.outputs.push_back({1, 0});
    sp.A = Mat(1, (int)cols.size());
    for (size_t x = 0; x < cols.size(); x++) sp.A.at(0, (int)x) = mu[cols[x]];
    return PMRC_OK;
  }, &spec);
  if (rc) return rc;
  if (!c->dry && stripes && S) {
    rc = check_region(piece.ptr, piece.stripe_stride, stripes);
    if (!rc) rc = check_region(beta.ptr, beta.stripe_stride, stripes);
    if (rc) return fail(rc, "bad piece/beta region");
  }
  uint64_t ptrs[2] = {(uint64_t)(uintptr_t)piece.ptr, (uint64_t)(uintptr_t)beta.ptr};
  uint64_t strides[2] = {piece.stripe_stride, beta.stripe_stride};
  return run_plan(c, key, *spec, ptrs, strides, S, stripes, stream);
}

int pmrc_repair_combine(pmrc_code *c, int lost_id, const int *helper_ids_in, int n_helpers,
                        const pmrc_cregion *betas_in, pmrc_region out_piece, size_t S, size_t stripes, void *stream) {
  if (c && c->w != 8) return fail(PMRC_EUNSUPPORTED, "w = 16 codes support encode, decode and repair (SURVEY NEXT-4)");
  if (!c || !helper_ids_in || !betas_in) return fail(PMRC_EINVAL, "NULL argument");
  int need = 0;
  int rc = repair_common(c, lost_id, helper_ids_in, n_helpers, &need);
  if (rc) return rc;
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  std::vector<int> H;
  std::vector<pmrc_cregion> betas;
  canonical_order(helper_ids_in, betas_in, n_helpers, H, betas);
  const CodeDef &D = c->def;
  const std::string key = ids_key("comb", H.data(), n_helpers, lost_id);
  const PlanSpec *spec = nullptr;
  rc = get_spec(c, key, [&](PlanSpec &sp) {
    Mat R;
    if (!repair_matrix(D, lost_id, H.data(), R)) return PMRC_ESINGULAR;
    sp.n_slots = n_helpers + 1;
    for (int h = 0; h < n_helpers; h++) sp.inputs.push_back({{{h, 0, 1}}});
    for (int a = 0; a < D.alpha; a++) sp.outputs.push_back({n_helpers, a});
    sp.A = R;
    return PMRC_OK;
  }, &spec);
  if (rc) return rc;
  std::vector<uint64_t> ptrs(n_helpers + 1), strides(n_helpers + 1);
  if (!c->dry && stripes && S) {
    for (int h = 0; h < n_helpers; h++) {
      rc = check_region(betas[h].ptr, betas[h].stripe_stride, stripes);
      if (rc) return fail(rc, "bad beta region");
    }
    rc = check_region(out_piece.ptr, out_piece.stripe_stride, stripes);
    if (rc) return fail(rc, "bad output piece region");
  }
  for (int h = 0; h < n_helpers; h++) {
    ptrs[h] = (uint64_t)(uintptr_t)betas[h].ptr;
    strides[h] = betas[h].stripe_stride;
  }
  ptrs[n_helpers] = (uint64_t)(uintptr_t)out_piece.ptr;
  strides[n_helpers] = out_piece.stripe_stride;
  return run_plan(c, key, *spec, ptrs.data(), strides.data(), S, stripes, stream);
}

// ---------------------------------------------------------------------------------------------
// Batch calls: per-stripe failure patterns in ONE launch of the runtime-coefficient kernel
// (config 4 as BASELINE.json states it).  Slots 0..n-1 are the nodes' piece regions, slot n the
// output region; stripe t runs the plan of its own pattern.
// ---------------------------------------------------------------------------------------------
static int check_node_regions(const pmrc_code *c, const pmrc_cregion *nodes, const std::vector<char> &used,
                              size_t stripes) {
  for (int i = 0; i < c->def.n; i++) {
    if (!used[i]) continue;
    const int rc = check_region(nodes[i].ptr, nodes[i].stripe_stride, stripes);
    if (rc) return fail(rc, "bad node piece region " + std::to_string(i));
  }
  return PMRC_OK;
}

// shared tail of the batch calls: per-stripe keys -> specs -> runtime plans of one shape -> launch
// jkeys[t] / jids[t]: the single-call plan key of stripe t's pattern and its node ids in slot order
// (sorted); under PMRC_PLAN_AUTO a stripe whose pattern has a loaded JIT kernel (pmrc_plan_prepare,
// earlier single calls under JIT) runs that kernel (runs of consecutive stripes of one pattern in
// one launch, the node regions offset to the run's first stripe), the rest one runtime launch.
static int run_batch(pmrc_code *c, const std::vector<std::string> &keys, const std::vector<const PlanSpec *> &specs,
                     const std::vector<std::string> &jkeys, const std::vector<std::vector<int>> &jids,
                     const pmrc_cregion *nodes, uint64_t out_ptr, uint64_t out_stride, size_t S, size_t stripes,
                     void *stream) {
  const int n = c->def.n;
  std::vector<char> jit(stripes, 0);
  if (c->policy == PMRC_PLAN_AUTO && !c->dry)
    for (size_t t = 0; t < stripes; t++) jit[t] = specs[t] && c->plans.count(jkeys[t]);
  int max_out = 0;
  for (size_t t = 0; t < stripes; t++)
    if (specs[t] && !jit[t]) max_out = std::max(max_out, (int)specs[t]->outputs.size());
  const bool any_jit = std::find(jit.begin(), jit.end(), 1) != jit.end();
  if (!S || (!max_out && !any_jit)) return PMRC_OK;  // nothing to compute in any stripe
  int rc = ensure_device(c);
  if (rc) return rc;
  std::string err;
  for (size_t t0 = 0; t0 < stripes;) {
    if (!jit[t0]) {
      t0++;
      continue;
    }
    size_t t1 = t0 + 1;
    while (t1 < stripes && jit[t1] && jkeys[t1] == jkeys[t0]) t1++;
    Kernel *K = c->plans[jkeys[t0]].get();
    const std::vector<int> &ids = jids[t0];
    std::vector<uint64_t> ptrs(ids.size() + 1), strides(ids.size() + 1);
    for (size_t q = 0; q < ids.size(); q++) {
      ptrs[q] = (uint64_t)(uintptr_t)nodes[ids[q]].ptr + t0 * nodes[ids[q]].stripe_stride;
      strides[q] = nodes[ids[q]].stripe_stride;
    }
    ptrs[ids.size()] = out_ptr + t0 * out_stride;
    strides[ids.size()] = out_stride;
    if (K->pace) c->traced = K;
    rc = launch_kernel(*K, ptrs.data(), strides.data(), S, t1 - t0, stream, err, c->max_ctas);
    if (rc) return fail(rc, err);
    t0 = t1;
  }
  if (!max_out) return PMRC_OK;  // nothing left for the runtime kernel
  const pmrc_rt::RlcShape sh = rt_shape(max_out, c->gen);
  std::vector<RtPlan *> plans;
  std::map<std::string, uint16_t> idx;
  std::vector<uint16_t> stripe_plan(stripes);
  for (size_t t = 0; t < stripes; t++) {
    if (!specs[t] || jit[t]) {
      stripe_plan[t] = 0xFFFF;  // nothing to compute in this stripe (or done by its JIT kernel)
      continue;
    }
    auto it = idx.find(keys[t]);
    if (it == idx.end()) {
      if (plans.size() >= 0xFFFF) return fail(PMRC_EUNSUPPORTED, "too many distinct patterns in one batch");
      RtPlan *P = nullptr;
      int rc = get_rt_plan(c, keys[t], *specs[t], sh.R, sh.G, &P);
      if (rc) return rc;
      it = idx.insert({keys[t], (uint16_t)plans.size()}).first;
      plans.push_back(P);
    }
    stripe_plan[t] = it->second;
  }
  std::vector<uint64_t> ptrs(n + 1), strides(n + 1);
  for (int i = 0; i < n; i++) {
    ptrs[i] = (uint64_t)(uintptr_t)nodes[i].ptr;
    strides[i] = nodes[i].stripe_stride;
  }
  ptrs[n] = out_ptr;
  strides[n] = out_stride;
  rc = rt_launch(plans, stripe_plan.data(), ptrs.data(), strides.data(), n + 1, S, stripes, sh, stream, c->max_ctas,
                 err);
  if (rc) return fail(rc, err);
  return PMRC_OK;
}

int pmrc_decode_batch(pmrc_code *c, const int *surv_ids, int n_surv, const pmrc_cregion *nodes, void *data_out,
                      size_t S, size_t stripes, int *n_written, void *stream) {
  if (!c || !surv_ids || !nodes || !data_out) return fail(PMRC_EINVAL, "NULL argument");
  if (c->w != 8) return fail(PMRC_EUNSUPPORTED, "batch calls: GF(2^8) codes only");
  const CodeDef &D = c->def;
  if (n_surv < 1 || n_surv > D.n) return fail(PMRC_EINVAL, "bad survivor count");
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  if (D.n + 1 > pmrc_rt::kRlcMaxSlots) return fail(PMRC_EUNSUPPORTED, "too many nodes for a batch launch");
  // the caches are bounded; evict up front, never while this call holds pointers into them
  if (c->specs.size() + stripes > kMaxSpecs) {
    c->specs.clear();
    c->plan_meta.clear();
  }
  if (c->rt_plans.size() + stripes > kMaxRtPlans) {
    if (cudaDeviceSynchronize() != cudaSuccess) {
      cudaGetLastError();
      return fail(PMRC_ECUDA, "cudaDeviceSynchronize (plan cache eviction)");
    }
    for (auto &kv : c->rt_plans) rt_free(*kv.second);
    c->rt_plans.clear();
  }
  struct NoEvict {
    pmrc_code *c;
    ~NoEvict() { c->no_evict = false; }
  } guard{c};
  c->no_evict = true;
  std::vector<std::string> keys(stripes), jkeys(stripes);
  std::vector<std::vector<int>> jids(stripes);
  std::vector<const PlanSpec *> specs(stripes);
  std::vector<char> used(D.n, 0);
  std::vector<int> slot_of(D.n);
  for (int i = 0; i < D.n; i++) slot_of[i] = i;
  for (size_t t = 0; t < stripes; t++) {
    const int *ids = surv_ids + t * (size_t)n_surv;
    if (check_ids(D, ids, n_surv)) return fail(PMRC_EINVAL, "bad survivor ids in stripe " + std::to_string(t));
    std::vector<int> s(ids, ids + n_surv);
    std::sort(s.begin(), s.end());
    keys[t] = ids_key("decn", s.data(), n_surv, 0);
    jkeys[t] = ids_key("dec", s.data(), n_surv, 0);  // pmrc_decode's plan of this survivor set
    jids[t] = s;
    std::vector<int> so(n_surv);
    for (int q = 0; q < n_surv; q++) so[q] = s[q];  // slot = node id
    int rc = get_spec(c, keys[t], [&](PlanSpec &sp) { return decode_spec(c, s.data(), n_surv, so.data(), D.n, D.n + 1,
                                                                          sp); },
                      &specs[t]);
    if (rc) return fail(rc, std::string(pmrc_last_error()) + " (stripe " + std::to_string(t) + ")");
    if (n_written) n_written[t] = c->plan_meta[keys[t]];
    if (specs[t])
      for (const auto &in : specs[t]->inputs)
        for (const auto &tm : in.terms) used[tm.slot] = 1;
  }
  int rc = check_node_regions(c, nodes, used, stripes);
  if (!rc) rc = check_region(data_out, (size_t)D.B * S, stripes);
  if (rc) return fail(rc, "bad region");
  return run_batch(c, keys, specs, jkeys, jids, nodes, (uint64_t)(uintptr_t)data_out, (uint64_t)D.B * S, S, stripes,
                   stream);
}

int pmrc_repair_batch(pmrc_code *c, const int *lost_ids, const int *helper_ids, int n_helpers, const pmrc_cregion *nodes,
                      pmrc_region out_piece, size_t S, size_t stripes, void *stream) {
  if (!c || !lost_ids || !helper_ids || !nodes) return fail(PMRC_EINVAL, "NULL argument");
  if (c->w != 8) return fail(PMRC_EUNSUPPORTED, "batch calls: GF(2^8) codes only");
  const CodeDef &D = c->def;
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  if (D.n + 1 > pmrc_rt::kRlcMaxSlots) return fail(PMRC_EUNSUPPORTED, "too many nodes for a batch launch");
  // the caches are bounded; evict up front, never while this call holds pointers into them
  if (c->specs.size() + stripes > kMaxSpecs) {
    c->specs.clear();
    c->plan_meta.clear();
  }
  if (c->rt_plans.size() + stripes > kMaxRtPlans) {
    if (cudaDeviceSynchronize() != cudaSuccess) {
      cudaGetLastError();
      return fail(PMRC_ECUDA, "cudaDeviceSynchronize (plan cache eviction)");
    }
    for (auto &kv : c->rt_plans) rt_free(*kv.second);
    c->rt_plans.clear();
  }
  struct NoEvict {
    pmrc_code *c;
    ~NoEvict() { c->no_evict = false; }
  } guard{c};
  c->no_evict = true;
  std::vector<std::string> keys(stripes), jkeys(stripes);
  std::vector<std::vector<int>> jids(stripes);
  std::vector<const PlanSpec *> specs(stripes);
  std::vector<char> used(D.n, 0);
  for (size_t t = 0; t < stripes; t++) {
    const int f = lost_ids[t];
    const int *ids = helper_ids + t * (size_t)n_helpers;
    int need = 0;
    int rc = repair_common(c, f, ids, n_helpers, &need);
    if (rc) return fail(rc, std::string(pmrc_last_error()) + " (stripe " + std::to_string(t) + ")");
    std::vector<int> H(ids, ids + n_helpers);
    std::sort(H.begin(), H.end());
    keys[t] = ids_key("repn", H.data(), n_helpers, f);
    jkeys[t] = ids_key("rep", H.data(), n_helpers, f);  // pmrc_repair's plan of this (f, H)
    jids[t] = H;
    rc = get_spec(c, keys[t], [&](PlanSpec &sp) {
      return repair_spec(c, f, H.data(), n_helpers, H.data(), D.n, D.n + 1, sp);  // slot = node id
    }, &specs[t]);
    if (rc) return fail(rc, std::string(pmrc_last_error()) + " (stripe " + std::to_string(t) + ")");
    for (const auto &in : specs[t]->inputs)
      for (const auto &tm : in.terms) used[tm.slot] = 1;
  }
  int rc = check_node_regions(c, nodes, used, stripes);
  if (!rc) rc = check_region(out_piece.ptr, out_piece.stripe_stride, stripes);
  if (rc) return fail(rc, "bad region");
  return run_batch(c, keys, specs, jkeys, jids, nodes, (uint64_t)(uintptr_t)out_piece.ptr, out_piece.stripe_stride, S,
                   stripes, stream);
}

// ---------------------------------------------------------------------------------------------
// The paper's "specific" product-matrix decoders (NEXT-2) on the
// GPU: each algebraic step is one region linear combination (a plan on the same engines), with the
// intermediate blocks in caller scratch.  Exactly k survivors (the decoders' data collector).
//   MSR:  A = C_DC Phi_DC^t;  Q_ij = (A_ij + A_ji)/(l_i + l_j),  P_ij = A_ij + l_i Q_ij
//                 (i != j);  U1_i = (P row i, off-diagonal) (Phi_others(i)^t)^-1, U2_i likewise
//                 from Q;  S1 = Phi_sel^-1 U1_sel,  S2 = Phi_sel^-1 U2_sel  (sel = first alpha
//                 survivors);  Z through L;  systematic data  X_miss = Gtilde[miss] Z
//   MBR:  T = Phi_DC^-1 R_right;  W = R_left + Delta_DC T^t;  S = Phi_DC^-1 W;  X through
//                 L (only the blocks no surviving systematic node holds are written)
// Slots: 0..k-1 survivor pieces, k.. scratch stage buffers, last = data_out.
// ---------------------------------------------------------------------------------------------
namespace {

struct SpecStages {
  std::vector<PlanSpec> stages;
  std::vector<int> scratch_blocks;  // blocks per stripe of each scratch buffer (slot k + b)
  int written = 0;                  // data blocks written per stripe
};

int msr_specific_stages(const pmrc_code *c, const int *ids, SpecStages &out) {
  const CodeDef &D = c->def;
  const GF256 &F = gf();
  const int k = D.k, a = D.alpha, d = D.d, B = D.B;
  if (k - 1 != a) return PMRC_EUNSUPPORTED;
  auto phi = [&](int node, int t) { return D.psi.at(node, t); };
  for (int x = 0; x < k; x++)
    for (int y = 0; y < x; y++)
      if (D.lambda[ids[x]] == D.lambda[ids[y]]) return PMRC_ESINGULAR;
  // per-survivor inverse of the other survivors' Phi^t, and Phi_sel^-1
  std::vector<Mat> oth(k);
  for (int i = 0; i < k; i++) {
    Mat M(a, a);
    int r = 0;
    for (int j = 0; j < k; j++) {
      if (j == i) continue;
      for (int t = 0; t < a; t++) M.at(t, r) = phi(ids[j], t);
      r++;
    }
    if (!invert(M, oth[i])) return PMRC_ESINGULAR;
  }
  Mat Sel(a, a), SelInv;
  for (int x = 0; x < a; x++)
    for (int t = 0; t < a; t++) Sel.at(x, t) = phi(ids[x], t);
  if (!invert(Sel, SelInv)) return PMRC_ESINGULAR;
  const int sA = k, sPQ = k + 1, sU = k + 2, sZ = k + 3, sOut = k + 4, nslots = k + 5;
  out.scratch_blocks = {k * k, 2 * k * k, 2 * k * a, B};
  // stage 1: A_ij = sum_t phi_j[t] C_i[t]
  PlanSpec s1;
  s1.n_slots = nslots;
  for (int i = 0; i < k; i++)
    for (int t = 0; t < a; t++) s1.inputs.push_back({{{i, t, 1}}});
  for (int i = 0; i < k; i++)
    for (int j = 0; j < k; j++) s1.outputs.push_back({sA, i * k + j});
  s1.A = Mat(k * k, k * a);
  for (int i = 0; i < k; i++)
    for (int j = 0; j < k; j++)
      for (int t = 0; t < a; t++) s1.A.at(i * k + j, i * a + t) = phi(ids[j], t);
  // stage 2: P_ij, Q_ij (i != j) from A_ij, A_ji
  PlanSpec s2;
  s2.n_slots = nslots;
  for (int e = 0; e < k * k; e++) s2.inputs.push_back({{{sA, e, 1}}});
  std::vector<std::pair<int, int>> offd;
  for (int i = 0; i < k; i++)
    for (int j = 0; j < k; j++)
      if (i != j) offd.push_back({i, j});
  s2.A = Mat(2 * (int)offd.size(), k * k);
  for (size_t q = 0; q < offd.size(); q++) {
    const int i = offd[q].first, j = offd[q].second;
    const uint8_t li = D.lambda[ids[i]], lj = D.lambda[ids[j]];
    const uint8_t cq = F.inv(li ^ lj);
    s2.outputs.push_back({sPQ, 2 * (i * k + j)});      // P_ij
    s2.outputs.push_back({sPQ, 2 * (i * k + j) + 1});  // Q_ij
    const uint8_t lc = F.mul(li, cq);
    s2.A.at(2 * (int)q, i * k + j) = 1 ^ lc;           // P_ij = (1 + l_i c) A_ij + l_i c A_ji
    s2.A.at(2 * (int)q, j * k + i) = lc;
    s2.A.at(2 * (int)q + 1, i * k + j) = cq;           // Q_ij = c (A_ij + A_ji)
    s2.A.at(2 * (int)q + 1, j * k + i) = cq;
  }
  // stage 3: U1_i = P_i,others . oth_i, U2_i = Q_i,others . oth_i
  PlanSpec s3;
  s3.n_slots = nslots;
  for (int e = 0; e < 2 * k * k; e++) s3.inputs.push_back({{{sPQ, e, 1}}});
  s3.A = Mat(2 * k * a, 2 * k * k);
  for (int w = 0; w < 2; w++)
    for (int i = 0; i < k; i++)
      for (int cc = 0; cc < a; cc++) {
        const int row = w * k * a + i * a + cc;
        s3.outputs.push_back({sU, row});
        int r = 0;
        for (int j = 0; j < k; j++) {
          if (j == i) continue;
          s3.A.at(row, 2 * (i * k + j) + w) = oth[i].at(r, cc);
          r++;
        }
      }
  // stage 4: S1 = SelInv U1_sel, S2 = SelInv U2_sel, written as Z through L (each index once)
  PlanSpec s4;
  s4.n_slots = nslots;
  for (int e = 0; e < 2 * k * a; e++) s4.inputs.push_back({{{sU, e, 1}}});
  std::vector<char> done(B + 1, 0);
  std::vector<std::vector<uint8_t>> rows4;
  for (int l = 0; l < d; l++)
    for (int j = 0; j < a; j++) {
      const int idx = D.Lidx[(size_t)l * D.Lcols + j];
      if (idx <= 0 || done[idx]) continue;
      done[idx] = 1;
      const int w = l < a ? 0 : 1, rr = l < a ? l : l - a;  // S_w[rr][j]
      std::vector<uint8_t> row(2 * k * a, 0);
      for (int t = 0; t < a; t++) row[w * k * a + t * a + j] = SelInv.at(rr, t);
      s4.outputs.push_back({sZ, idx - 1});
      rows4.push_back(row);
    }
  s4.A = Mat((int)rows4.size(), 2 * k * a);
  for (size_t r = 0; r < rows4.size(); r++) memcpy(&s4.A.a[r * 2 * k * a], rows4[r].data(), 2 * k * a);
  // stage 5: X_miss = Gtilde[miss] Z  (Gtilde = G's first B rows)
  std::vector<char> held(B, 0);
  for (int x = 0; x < k; x++)
    if (ids[x] < k)
      for (int j = 0; j < a; j++) held[D.sys_block(ids[x], j)] = 1;
  std::vector<int> miss;
  for (int m = 0; m < B; m++)
    if (!held[m]) miss.push_back(m);
  out.written = (int)miss.size();
  out.stages = {s1, s2, s3, s4};
  if (miss.empty()) return PMRC_OK;
  PlanSpec s5;
  s5.n_slots = nslots;
  std::vector<int> used;
  for (int z = 0; z < B; z++) {
    bool nz = false;
    for (int m : miss) nz |= D.G.at(m, z) != 0;
    if (nz) used.push_back(z);
  }
  for (int z : used) s5.inputs.push_back({{{sZ, z, 1}}});
  for (int m : miss) s5.outputs.push_back({sOut, m});
  s5.A = Mat((int)miss.size(), (int)used.size());
  for (size_t r = 0; r < miss.size(); r++)
    for (size_t x = 0; x < used.size(); x++) s5.A.at((int)r, (int)x) = D.G.at(miss[r], used[x]);
  out.stages.push_back(s5);
  return PMRC_OK;
}

int mbr_specific_stages(const pmrc_code *c, const int *ids, SpecStages &out) {
  const CodeDef &D = c->def;
  const int k = D.k, d = D.d, B = D.B, dk = d - k;
  Mat Phi(k, k), PhiInv;
  for (int x = 0; x < k; x++)
    for (int t = 0; t < k; t++) Phi.at(x, t) = D.psi.at(ids[x], t);
  if (!invert(Phi, PhiInv)) return PMRC_ESINGULAR;
  const int sT = k, sW = k + 1, sOut = k + 2, nslots = k + 3;
  out.scratch_blocks = {std::max(1, k * dk), k * k};
  std::vector<PlanSpec> st;
  // stage 1: T[r][cc] = sum_t PhiInv[r][t] R[t][k + cc]
  if (dk > 0) {
    PlanSpec s1;
    s1.n_slots = nslots;
    for (int t = 0; t < k; t++)
      for (int cc = 0; cc < dk; cc++) s1.inputs.push_back({{{t, k + cc, 1}}});
    s1.A = Mat(k * dk, k * dk);
    for (int r = 0; r < k; r++)
      for (int cc = 0; cc < dk; cc++) {
        s1.outputs.push_back({sT, r * dk + cc});
        for (int t = 0; t < k; t++) s1.A.at(r * dk + cc, t * dk + cc) = PhiInv.at(r, t);
      }
    st.push_back(s1);
  }
  // stage 2: W[x][cc] = R[x][cc] + sum_t Delta[x][t] T[cc][t]
  PlanSpec s2;
  s2.n_slots = nslots;
  for (int x = 0; x < k; x++)
    for (int cc = 0; cc < k; cc++) s2.inputs.push_back({{{x, cc, 1}}});
  for (int e = 0; e < k * dk; e++) s2.inputs.push_back({{{sT, e, 1}}});
  s2.A = Mat(k * k, k * k + k * dk);
  for (int x = 0; x < k; x++)
    for (int cc = 0; cc < k; cc++) {
      s2.outputs.push_back({sW, x * k + cc});
      s2.A.at(x * k + cc, x * k + cc) = 1;
      for (int t = 0; t < dk; t++) s2.A.at(x * k + cc, k * k + cc * dk + t) = D.psi.at(ids[x], k + t);
    }
  st.push_back(s2);
  // stage 3: S = PhiInv W (missing blocks only), T entries of missing blocks copied from T
  std::vector<char> held(B, 0);
  for (int x = 0; x < k; x++)
    if (ids[x] < k)
      for (int j = 0; j < d; j++) held[D.sys_block(ids[x], j)] = 1;
  PlanSpec s3;
  s3.n_slots = nslots;
  for (int e = 0; e < k * k; e++) s3.inputs.push_back({{{sW, e, 1}}});
  for (int e = 0; e < k * dk; e++) s3.inputs.push_back({{{sT, e, 1}}});
  std::vector<char> done(B + 1, 0);
  std::vector<std::vector<uint8_t>> rows3;
  for (int r = 0; r < k; r++)
    for (int cc = 0; cc < d; cc++) {
      const int idx = D.Lidx[(size_t)r * D.Lcols + cc];
      if (idx <= 0 || done[idx] || held[idx - 1]) continue;
      done[idx] = 1;
      std::vector<uint8_t> row(k * k + k * dk, 0);
      if (cc < k) {
        for (int t = 0; t < k; t++) row[t * k + cc] = PhiInv.at(r, t);  // S[r][cc]
      } else {
        row[k * k + r * dk + (cc - k)] = 1;                             // T[r][cc - k]
      }
      s3.outputs.push_back({sOut, idx - 1});
      rows3.push_back(row);
    }
  out.written = (int)rows3.size();
  if (!rows3.empty()) {
    s3.A = Mat((int)rows3.size(), k * k + k * dk);
    for (size_t r = 0; r < rows3.size(); r++) memcpy(&s3.A.a[r * (k * k + k * dk)], rows3[r].data(), k * k + k * dk);
    st.push_back(s3);
  }
  out.stages = st;
  return PMRC_OK;
}

int specific_stages(const pmrc_code *c, const int *ids, SpecStages &out) {
  if (c->w != 8) return PMRC_EUNSUPPORTED;
  const int kind = c->def.kind;
  if (kind == KIND_MBR) return mbr_specific_stages(c, ids, out);
  if (kind == KIND_RS) return PMRC_EUNSUPPORTED;
  return msr_specific_stages(c, ids, out);
}

size_t scratch_bytes_of(const SpecStages &ss, size_t S, size_t stripes) {
  size_t t = 0;
  for (int b : ss.scratch_blocks) t += (size_t)b * S * stripes;
  return t;
}

}  // namespace

int pmrc_decode_specific_scratch(pmrc_code *c, size_t S, size_t stripes, size_t *bytes) {
  if (!c || !bytes) return fail(PMRC_EINVAL, "NULL argument");
  const CodeDef &D = c->def;
  std::vector<int> ids(D.k);
  for (int i = 0; i < D.k; i++) ids[i] = D.n - D.k + i;  // shape only (any k-set has the same buffers)
  SpecStages ss;
  int rc = specific_stages(c, ids.data(), ss);
  if (rc == PMRC_ESINGULAR) {  // the scratch shape does not depend on the set: use the first k nodes
    for (int i = 0; i < D.k; i++) ids[i] = i;
    rc = specific_stages(c, ids.data(), ss);
  }
  if (rc) return fail(rc, "specific decoder: unsupported code");
  *bytes = scratch_bytes_of(ss, S, stripes);
  return PMRC_OK;
}

int pmrc_decode_specific(pmrc_code *c, const int *surv_ids_in, int n_surv, const pmrc_cregion *pieces_in,
                         void *data_out, void *scratch, size_t scratch_bytes, size_t S, size_t stripes,
                         int *n_written, void *stream) {
  if (n_written) *n_written = 0;
  if (!c || !surv_ids_in || !pieces_in || !data_out || !scratch) return fail(PMRC_EINVAL, "NULL argument");
  const CodeDef &D = c->def;
  if (n_surv != D.k || check_ids(D, surv_ids_in, n_surv)) return fail(PMRC_EINVAL, "specific decode needs exactly k distinct survivors");
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  std::vector<int> surv;
  std::vector<pmrc_cregion> pieces;
  canonical_order(surv_ids_in, pieces_in, n_surv, surv, pieces);
  SpecStages ss;
  int rc = specific_stages(c, surv.data(), ss);
  if (rc) return fail(rc, rc == PMRC_ESINGULAR ? "specific decoder: singular submatrix for this survivor set"
                                               : "specific decoder: unsupported code (MSR / MBR over GF(2^8))");
  if (n_written) *n_written = ss.written;
  if (!stripes || !S) return PMRC_OK;
  if (scratch_bytes < scratch_bytes_of(ss, S, stripes)) return fail(PMRC_EINVAL, "scratch too small");
  const int k = D.k, nb = (int)ss.scratch_blocks.size(), nslots = k + nb + 1;
  std::vector<uint64_t> ptrs(nslots), strides(nslots);
  for (int a = 0; a < k; a++) {
    rc = check_region(pieces[a].ptr, pieces[a].stripe_stride, stripes);
    if (rc) return fail(rc, "bad survivor piece region");
    ptrs[a] = (uint64_t)(uintptr_t)pieces[a].ptr;
    strides[a] = pieces[a].stripe_stride;
  }
  rc = check_region(scratch, 16, stripes);
  if (!rc) rc = check_region(data_out, (size_t)D.B * S, stripes);
  if (rc) return fail(rc, "bad scratch / data_out");
  uint64_t off = (uint64_t)(uintptr_t)scratch;
  for (int b = 0; b < nb; b++) {
    ptrs[k + b] = off;
    strides[k + b] = (uint64_t)ss.scratch_blocks[b] * S;
    off += (uint64_t)ss.scratch_blocks[b] * S * stripes;
  }
  ptrs[k + nb] = (uint64_t)(uintptr_t)data_out;
  strides[k + nb] = (uint64_t)D.B * S;
  const std::string base = ids_key("spec", surv.data(), n_surv, 0);
  for (size_t q = 0; q < ss.stages.size(); q++) {
    const std::string key = base + ":" + std::to_string(q);
    const PlanSpec *sp = nullptr;
    rc = get_spec(c, key, [&](PlanSpec &x) {
      x = ss.stages[q];
      return PMRC_OK;
    }, &sp);
    if (rc) return rc;
    rc = run_plan(c, key, *sp, ptrs.data(), strides.data(), S, stripes, stream);
    if (rc) return rc;
  }
  return PMRC_OK;
}

int pmrc_rt_plan_blob(pmrc_code *c, int op, int lost_id, const int *ids_in, int n_ids, uint32_t *buf, size_t cap,
                      size_t *n_words) {
  // the runtime-coefficient kernel's plan blob for a pattern, built on the host (no GPU): for
  // inspection and for the CPU tier's emulation of the kernel (tests/test_rt_plan.py)
  if (!c || !n_words) return fail(PMRC_EINVAL, "NULL argument");
  *n_words = 0;
  if (c->w != 8) return fail(PMRC_EUNSUPPORTED, "runtime-coefficient plans are GF(2^8) only");
  const CodeDef &D = c->def;
  PlanSpec spec;
  int rc = PMRC_OK;
  if (op == 2) {
    spec = c->enc_spec;
  } else if (op == 0 || op == 1) {
    if (!ids_in || n_ids < 1 || n_ids > D.n || check_ids(D, ids_in, n_ids)) return fail(PMRC_EINVAL, "bad ids");
    std::vector<int> ids(ids_in, ids_in + n_ids), slot_of(n_ids);
    std::sort(ids.begin(), ids.end());
    for (int q = 0; q < n_ids; q++) slot_of[q] = q;
    if (op == 0) {
      rc = decode_spec(c, ids.data(), n_ids, slot_of.data(), n_ids, n_ids + 1, spec);
      if (rc == kNothing) return fail(PMRC_EINVAL, "no data block is missing (nothing to compute)");
    } else {
      int need = 0;
      rc = repair_common(c, lost_id, ids.data(), n_ids, &need);
      if (!rc) rc = repair_spec(c, lost_id, ids.data(), n_ids, slot_of.data(), n_ids, n_ids + 1, spec);
    }
    if (rc) return rc == PMRC_ESINGULAR ? fail(rc, "singular pattern") : rc;
  } else {
    return fail(PMRC_EINVAL, "op must be 0 (decode), 1 (repair) or 2 (encode)");
  }
  const pmrc_rt::RlcShape sh = rt_shape((int)spec.outputs.size(), c->gen);
  RtPlan P;
  std::string err;
  rc = rt_build(spec, sh.R, sh.G, P, err);
  if (rc) return fail(rc, err);
  *n_words = P.blob.size();
  if (buf && cap >= P.blob.size()) memcpy(buf, P.blob.data(), P.blob.size() * 4);
  return PMRC_OK;
}

int pmrc_set_auto_promotion(pmrc_code *c, unsigned long long bytes) {
  if (!c) return fail(PMRC_EINVAL, "NULL handle");
  c->promote_bytes = bytes;
  return PMRC_OK;
}

int pmrc_plan_state(pmrc_code *c, int op, int lost_id, const int *ids, int n_ids) {
  // 0: no generated kernel loaded (runtime kernel under AUTO), 1: promotion compiling,
  // 2: promotion compiled (loaded at the next call), 3: generated kernel loaded
  if (!c || !ids) return fail(PMRC_EINVAL, "NULL argument");
  if (op != 0 && op != 1) return fail(PMRC_EINVAL, "op must be 0 (decode) or 1 (repair)");
  std::vector<int> s(ids, ids + n_ids);
  std::sort(s.begin(), s.end());
  const std::string key = op == 0 ? ids_key("dec", s.data(), n_ids, 0) : ids_key("rep", s.data(), n_ids, lost_id);
  if (c->plans.count(key)) return 3;
  auto it = c->promos.find(key);
  if (it == c->promos.end()) return 0;
  return it->second->state.load() == 1 ? 1 : 2;
}

int pmrc_plan_prepare(pmrc_code *c, int op, int lost_id, const int *ids, int n_ids) {
  // promote a (hot) failure pattern to its generated bitsliced kernel: build + NVRTC-compile (or
  // load from the kernel cache) now, so later calls with this pattern run the JIT kernel under
  // PMRC_PLAN_AUTO
  if (!c || !ids) return fail(PMRC_EINVAL, "NULL argument");
  const int saved = c->policy;
  c->policy = PMRC_PLAN_JIT;
  std::vector<pmrc_cregion> pieces(std::max(1, n_ids), pmrc_cregion{(const void *)(uintptr_t)4096, 0});
  int rc;
  if (op == 0) {
    int nw = 0;
    rc = pmrc_decode(c, ids, n_ids, pieces.data(), (void *)(uintptr_t)4096, 16, 0, &nw, nullptr);
  } else if (op == 1) {
    rc = pmrc_repair(c, lost_id, ids, n_ids, pieces.data(), pmrc_region{(void *)(uintptr_t)4096, 0}, 16, 0, nullptr);
  } else {
    rc = fail(PMRC_EINVAL, "op must be 0 (decode) or 1 (repair)");
  }
  c->policy = saved;
  return rc;
}

}  // extern "C"
