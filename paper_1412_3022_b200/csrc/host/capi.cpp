// C ABI of libpmrc (include/pmrc.h): code handles, plan caches, and the data-path entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../../include/pmrc.h"
#include "construct.hpp"
#include "plan.hpp"

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
  GenStats enc_stats;
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
// network) are worth their host time there (config 2: 12,362 -> 12,305 XORs, 0.501 -> 0.491 ms)
GenOptions enc_gen(const pmrc_code *c) {
  GenOptions g = c->gen;
  if (c->w == 8 && c->def.k <= 8) g.cse_restarts = std::max(g.cse_restarts, g.enc_restarts);  // (k=16: minutes)
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
  (void)generate_source(c->enc_spec, enc_gen(c.get()), c->enc_stats);  // XOR-program statistics
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
  rc = build_encode(c);
  if (rc) return rc;
  uint64_t ptrs[2] = {(uint64_t)(uintptr_t)data, (uint64_t)(uintptr_t)parity};
  uint64_t strides[2] = {(uint64_t)D.B * S, (uint64_t)D.P * S};
  std::string err;
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

// GF(2^16) decode plan (w = 16): the same rule as the GF(2^8) plan in pmrc_decode (R13):
// greedy B independent rows of G' = [I_B; G''], systematic survivors first, then the inverse's
// rows of the data blocks no surviving systematic node holds.  Returns 0, PMRC_ESINGULAR, or 1 if
// nothing is missing.
static int decode_spec16(const pmrc_code *c, const int *surv_ids, int n_surv, PlanSpec &spec) {
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
  if (missing.empty()) return 1;
  for (int x = 0; x < B; x++) {
    bool nz = false;
    for (int m : missing) nz |= Inv[(size_t)m * B + x] != 0;
    if (nz) used.push_back(x);
  }
  spec = PlanSpec();
  spec.n_slots = n_surv + 1;
  spec.w = 16;
  for (int x : used) spec.inputs.push_back({{{sel[x].first, sel[x].second, 1}}});
  for (int m : missing) spec.outputs.push_back({n_surv, m});
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

int pmrc_decode(pmrc_code *c, const int *surv_ids_in, int n_surv, const pmrc_cregion *pieces_in, void *data_out,
                size_t S, size_t stripes, int *n_written, void *stream) {
  if (n_written) *n_written = 0;
  if (!c || !surv_ids_in || !pieces_in || !data_out) return fail(PMRC_EINVAL, "NULL argument");
  const CodeDef &D = c->def;
  if (n_surv < 1 || n_surv > D.n || check_ids(D, surv_ids_in, n_surv)) return fail(PMRC_EINVAL, "bad survivor ids");
  // canonical order: the plan (and its cache key) depends on the survivor SET only; the pieces are
  // permuted with the ids (the decoded data is unique, so the order cannot change it)
  std::vector<int> surv_v;
  std::vector<pmrc_cregion> pieces_v;
  canonical_order(surv_ids_in, pieces_in, n_surv, surv_v, pieces_v);
  const int *surv_ids = surv_v.data();
  const pmrc_cregion *pieces = pieces_v.data();
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  const std::string key = ids_key("dec", surv_ids, n_surv, 0);
  auto fe = c->plan_err.find(key);
  if (fe != c->plan_err.end()) return fail(fe->second, "survivors do not span the data (cached)");
  if (c->w == 16 && (c->dry || !c->plan_meta.count(key))) {
    PlanSpec spec;
    const int r16 = decode_spec16(c, surv_ids, n_surv, spec);
    if (r16 == PMRC_ESINGULAR) {
      c->plan_err[key] = PMRC_ESINGULAR;
      return fail(PMRC_ESINGULAR, "survivors do not span the data");
    }
    if (r16 == 1) {
      c->plan_meta[key] = 0;
      return PMRC_OK;
    }
    Kernel *Kb = nullptr;
    int rc = get_kernel(c, key, spec, &Kb);
    if (rc) return rc;
    c->plan_meta[key] = (int)spec.outputs.size();
  } else if (c->dry || !c->plan_meta.count(key)) {
    PlanSpec spec;
    {
      // ---- plan (R13): greedy B independent rows of G', systematic survivors first ----
      std::vector<int> order;
      for (int pass = 0; pass < 2; pass++)
        for (int id = 0; id < D.n; id++) {
          if ((pass == 0) != (id < D.k)) continue;
          for (int a = 0; a < n_surv; a++)
            if (surv_ids[a] == id) order.push_back(a);
        }
      // incremental elimination to test independence
      std::vector<std::vector<uint8_t>> basis;  // reduced rows
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
          // keep basis fully reduced on pivot columns
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
      if ((int)sel.size() < D.B) {
        c->plan_err[key] = PMRC_ESINGULAR;
        return fail(PMRC_ESINGULAR, "survivors do not span the data");
      }
      Mat Inv;
      if (!invert(Sel, Inv)) return fail(PMRC_ESINGULAR, "selected rows singular");
      // missing data blocks: not held by a surviving systematic node
      std::vector<char> held(D.B, 0);
      for (int a = 0; a < n_surv; a++)
        if (surv_ids[a] < D.k)
          for (int j = 0; j < D.alpha; j++) held[D.sys_block(surv_ids[a], j)] = 1;
      std::vector<int> missing;
      for (int x = 0; x < D.B; x++)
        if (!held[x]) missing.push_back(x);
      if (missing.empty()) {
        c->plan_meta[key] = 0;
        return PMRC_OK;
      }
      spec.n_slots = n_surv + 1;
      std::vector<int> used_cols;
      for (int x = 0; x < D.B; x++) {
        bool nz = false;
        for (int m : missing) nz |= Inv.at(m, x) != 0;
        if (nz) used_cols.push_back(x);
      }
      for (int x : used_cols) spec.inputs.push_back({{{sel[x].first, sel[x].second, 1}}});
      for (int m : missing) spec.outputs.push_back({n_surv, m});
      spec.A = Mat((int)missing.size(), (int)used_cols.size());
      for (size_t r = 0; r < missing.size(); r++)
        for (size_t x = 0; x < used_cols.size(); x++) spec.A.at((int)r, (int)x) = Inv.at(missing[r], used_cols[x]);
    }
    Kernel *Kb = nullptr;
    int rc = get_kernel(c, key, spec, &Kb);
    if (rc) return rc;
    c->plan_meta[key] = (int)spec.outputs.size();
  }
  const int written = c->plan_meta[key];
  Kernel *K = written ? c->plans[key].get() : nullptr;
  if (n_written) *n_written = written;
  if (!written || !stripes || !S) return PMRC_OK;
  std::vector<uint64_t> ptrs(n_surv + 1), strides(n_surv + 1);
  for (int a = 0; a < n_surv; a++) {
    int rc = check_region(pieces[a].ptr, pieces[a].stripe_stride, stripes);
    if (rc) return fail(rc, "bad survivor piece region");
    ptrs[a] = (uint64_t)(uintptr_t)pieces[a].ptr;
    strides[a] = pieces[a].stripe_stride;
  }
  int rc = check_region(data_out, (size_t)D.B * S, stripes);
  if (rc) return fail(rc, "bad data_out");
  ptrs[n_surv] = (uint64_t)(uintptr_t)data_out;
  strides[n_surv] = (uint64_t)D.B * S;
  std::string err;
  if (K->pace) c->traced = K;
  rc = launch_kernel(*K, ptrs.data(), strides.data(), S, stripes, stream, err, c->max_ctas);
  if (rc) return fail(rc, err);
  return PMRC_OK;
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
  Kernel *K = nullptr;
  auto it = c->plans.find(key);
  if (c->dry || it == c->plans.end()) {
    PlanSpec spec;
    spec.n_slots = 2;
    for (int x = 0; x < cols; x++) spec.inputs.push_back({{{0, x, 1}}});
    for (int r = 0; r < rows; r++) spec.outputs.push_back({1, r});
    spec.A = Mat(rows, cols);
    memcpy(spec.A.a.data(), A, (size_t)rows * cols);
    bool any = false;
    for (uint8_t v : spec.A.a) any |= v != 0;
    if (!any) return fail(PMRC_EINVAL, "all-zero matrix (nothing to compute)");
    int rc = get_kernel(c, key, spec, &K);
    if (rc) return rc;
  } else {
    K = it->second.get();
  }
  if (!stripes || !S) return PMRC_OK;
  int rc = check_region(in, in_stride, stripes);
  if (!rc) rc = check_region(out, out_stride, stripes);
  if (rc) return fail(rc, "bad in/out region");
  uint64_t ptrs[2] = {(uint64_t)(uintptr_t)in, (uint64_t)(uintptr_t)out};
  uint64_t strides[2] = {(uint64_t)in_stride, (uint64_t)out_stride};
  std::string err;
  if (K->pace) c->traced = K;
  rc = launch_kernel(*K, ptrs, strides, S, stripes, stream, err, c->max_ctas);
  if (rc) return fail(rc, err);
  return PMRC_OK;
}

int pmrc_set_max_ctas(pmrc_code *c, int max_ctas) {
  if (!c || max_ctas < 0) return fail(PMRC_EINVAL, "bad argument");
  c->max_ctas = max_ctas;
  return PMRC_OK;
}

int pmrc_set_independent_launches(pmrc_code *c, int on) {
  if (!c || on < 0 || on > 1) return fail(PMRC_EINVAL, "bad argument");
  const int want = on ? 2 : 0;
  if (c->gen.pdl == want) return PMRC_OK;
  // the kernels are generated with or without griddepcontrol.wait: drop the built ones (they are
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
  c->plan_meta.clear();
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
  // canonical helper order (the plan depends on the helper SET; the repaired piece is unique)
  std::vector<int> help_v;
  std::vector<pmrc_cregion> hp_v;
  canonical_order(helper_ids_in, helper_pieces_in, n_helpers, help_v, hp_v);
  const int *helper_ids = help_v.data();
  const pmrc_cregion *helper_pieces = hp_v.data();
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  const CodeDef &D = c->def;
  const std::string key = ids_key("rep", helper_ids, n_helpers, lost_id);
  auto fe = c->plan_err.find(key);
  if (fe != c->plan_err.end()) return fail(fe->second, "helper matrix singular (cached)");
  Kernel *K = nullptr;
  if (c->w == 16 && (c->dry || !c->plans.count(key))) {
    // GF(2^16) (w = 16): mu = phi_f (P:53 footnote), R = [I_alpha | lambda_f I_alpha] Psi_H^{-1}
    const GF65536 &F = gf16();
    const int dd = D.d, a = D.alpha;
    std::vector<uint16_t> Wm((size_t)dd * dd), Inv((size_t)dd * dd, 0);
    for (int r = 0; r < dd; r++) {
      for (int x = 0; x < dd; x++) Wm[(size_t)r * dd + x] = c->psi16[(size_t)helper_ids[r] * dd + x];
      Inv[(size_t)r * dd + r] = 1;
    }
    for (int col = 0; col < dd; col++) {
      int piv = -1;
      for (int r = col; r < dd; r++)
        if (Wm[(size_t)r * dd + col]) { piv = r; break; }
      if (piv < 0) {
        c->plan_err[key] = PMRC_ESINGULAR;
        return fail(PMRC_ESINGULAR, "Psi_H singular for this (lost, helpers) pair (DESIGN.md R10)");
      }
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
        const uint16_t f = r == col ? 0 : Wm[(size_t)r * dd + col];
        if (!f) continue;
        for (int x = 0; x < dd; x++) {
          Wm[(size_t)r * dd + x] ^= F.mul(f, Wm[(size_t)col * dd + x]);
          Inv[(size_t)r * dd + x] ^= F.mul(f, Inv[(size_t)col * dd + x]);
        }
      }
    }
    const uint16_t lf = c->lam16[lost_id];
    PlanSpec spec;
    spec.w = 16;
    spec.n_slots = n_helpers + 1;
    for (int h = 0; h < n_helpers; h++) {
      InputDesc in;
      for (int b = 0; b < a; b++) {
        const uint16_t mu = c->psi16[(size_t)lost_id * dd + b];
        if (mu) in.terms.push_back({h, b, mu});
      }
      spec.inputs.push_back(in);
    }
    for (int q = 0; q < a; q++) spec.outputs.push_back({n_helpers, q});
    spec.A = Mat(a, n_helpers);
    spec.A16.assign((size_t)a * n_helpers, 0);
    for (int q = 0; q < a; q++)
      for (int h = 0; h < n_helpers; h++) {
        const uint16_t v = Inv[(size_t)q * dd + h] ^ F.mul(lf, Inv[(size_t)(a + q) * dd + h]);
        spec.A16[(size_t)q * n_helpers + h] = v;
        spec.A.at(q, h) = v ? 1 : 0;
      }
    rc = get_kernel(c, key, spec, &K);
    if (rc) return rc;
  } else if (c->dry || !c->plans.count(key)) {
    Mat R;
    if (!repair_matrix(D, lost_id, helper_ids, R)) {
      c->plan_err[key] = PMRC_ESINGULAR;
      return fail(PMRC_ESINGULAR, "Psi_H singular for this (lost, helpers) pair (DESIGN.md R10)");
    }
    // fused plan: input h = beta_h = mu . piece_h (derived), outputs = alpha blocks
    std::vector<uint8_t> mu = repair_mu(D, lost_id);
    PlanSpec spec;
    spec.n_slots = n_helpers + 1;
    for (int h = 0; h < n_helpers; h++) {
      InputDesc in;
      for (size_t b = 0; b < mu.size(); b++)
        if (mu[b]) in.terms.push_back({h, (int)b, mu[b]});
      spec.inputs.push_back(in);
    }
    for (int a = 0; a < D.alpha; a++) spec.outputs.push_back({n_helpers, a});
    spec.A = R;
    rc = get_kernel(c, key, spec, &K);
    if (rc) return rc;
  } else {
    K = c->plans[key].get();
  }
  if (!stripes || !S) return PMRC_OK;
  std::vector<uint64_t> ptrs(n_helpers + 1), strides(n_helpers + 1);
  for (int h = 0; h < n_helpers; h++) {
    rc = check_region(helper_pieces[h].ptr, helper_pieces[h].stripe_stride, stripes);
    if (rc) return fail(rc, "bad helper piece region");
    ptrs[h] = (uint64_t)(uintptr_t)helper_pieces[h].ptr;
    strides[h] = helper_pieces[h].stripe_stride;
  }
  rc = check_region(out_piece.ptr, out_piece.stripe_stride, stripes);
  if (rc) return fail(rc, "bad output piece region");
  ptrs[n_helpers] = (uint64_t)(uintptr_t)out_piece.ptr;
  strides[n_helpers] = out_piece.stripe_stride;
  std::string err;
  if (K->pace) c->traced = K;
  rc = launch_kernel(*K, ptrs.data(), strides.data(), S, stripes, stream, err, c->max_ctas);
  if (rc) return fail(rc, err);
  return PMRC_OK;
}

int pmrc_repair_project(pmrc_code *c, int lost_id, pmrc_cregion piece, pmrc_region beta, size_t S, size_t stripes,
                        void *stream) {
  if (c && c->w != 8) return fail(PMRC_EUNSUPPORTED, "w = 16 codes support encode, decode and repair (SURVEY NEXT-4)");
  if (!c) return fail(PMRC_EINVAL, "NULL handle");
  const CodeDef &D = c->def;
  if (lost_id < 0 || lost_id >= D.n) return fail(PMRC_EINVAL, "bad lost id");
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  const std::string key = "proj:" + std::to_string(lost_id);
  Kernel *K = nullptr;
  if (!c->plans.count(key)) {
    std::vector<uint8_t> mu = repair_mu(D, lost_id);
    PlanSpec spec;
    spec.n_slots = 2;
    std::vector<int> cols;
    for (size_t b = 0; b < mu.size(); b++)
      if (mu[b]) {
        spec.inputs.push_back({{{0, (int)b, 1}}});  // only blocks with nonzero mu are read
        cols.push_back((int)b);
      }
    spec.outputs.push_back({1, 0});
    spec.A = Mat(1, (int)cols.size());
    for (size_t x = 0; x < cols.size(); x++) spec.A.at(0, (int)x) = mu[cols[x]];
    int rc = get_kernel(c, key, spec, &K);
    if (rc) return rc;
  } else {
    K = c->plans[key].get();
  }
  if (!stripes || !S) return PMRC_OK;
  int rc = check_region(piece.ptr, piece.stripe_stride, stripes);
  if (!rc) rc = check_region(beta.ptr, beta.stripe_stride, stripes);
  if (rc) return fail(rc, "bad piece/beta region");
  uint64_t ptrs[2] = {(uint64_t)(uintptr_t)piece.ptr, (uint64_t)(uintptr_t)beta.ptr};
  uint64_t strides[2] = {piece.stripe_stride, beta.stripe_stride};
  std::string err;
  if (K->pace) c->traced = K;
  rc = launch_kernel(*K, ptrs, strides, S, stripes, stream, err, c->max_ctas);
  if (rc) return fail(rc, err);
  return PMRC_OK;
}

int pmrc_repair_combine(pmrc_code *c, int lost_id, const int *helper_ids_in, int n_helpers,
                        const pmrc_cregion *betas_in, pmrc_region out_piece, size_t S, size_t stripes, void *stream) {
  if (c && c->w != 8) return fail(PMRC_EUNSUPPORTED, "w = 16 codes support encode, decode and repair (SURVEY NEXT-4)");
  if (!c || !helper_ids_in || !betas_in) return fail(PMRC_EINVAL, "NULL argument");
  int need = 0;
  int rc = repair_common(c, lost_id, helper_ids_in, n_helpers, &need);
  if (rc) return rc;
  std::vector<int> help_v;
  std::vector<pmrc_cregion> b_v;
  canonical_order(helper_ids_in, betas_in, n_helpers, help_v, b_v);
  const int *helper_ids = help_v.data();
  const pmrc_cregion *betas = b_v.data();
  if (S % 16) return fail(PMRC_EALIGN, "S must be a multiple of 16");
  const CodeDef &D = c->def;
  const std::string key = ids_key("comb", helper_ids, n_helpers, lost_id);
  auto fe = c->plan_err.find(key);
  if (fe != c->plan_err.end()) return fail(fe->second, "helper matrix singular (cached)");
  Kernel *K = nullptr;
  if (c->dry || !c->plans.count(key)) {
    Mat R;
    if (!repair_matrix(D, lost_id, helper_ids, R)) {
      c->plan_err[key] = PMRC_ESINGULAR;
      return fail(PMRC_ESINGULAR, "Psi_H singular for this (lost, helpers) pair (DESIGN.md R10)");
    }
    PlanSpec spec;
    spec.n_slots = n_helpers + 1;
    for (int h = 0; h < n_helpers; h++) spec.inputs.push_back({{{h, 0, 1}}});
    for (int a = 0; a < D.alpha; a++) spec.outputs.push_back({n_helpers, a});
    spec.A = R;
    rc = get_kernel(c, key, spec, &K);
    if (rc) return rc;
  } else {
    K = c->plans[key].get();
  }
  if (!stripes || !S) return PMRC_OK;
  std::vector<uint64_t> ptrs(n_helpers + 1), strides(n_helpers + 1);
  for (int h = 0; h < n_helpers; h++) {
    rc = check_region(betas[h].ptr, betas[h].stripe_stride, stripes);
    if (rc) return fail(rc, "bad beta region");
    ptrs[h] = (uint64_t)(uintptr_t)betas[h].ptr;
    strides[h] = betas[h].stripe_stride;
  }
  rc = check_region(out_piece.ptr, out_piece.stripe_stride, stripes);
  if (rc) return fail(rc, "bad output piece region");
  ptrs[n_helpers] = (uint64_t)(uintptr_t)out_piece.ptr;
  strides[n_helpers] = out_piece.stripe_stride;
  std::string err;
  if (K->pace) c->traced = K;
  rc = launch_kernel(*K, ptrs.data(), strides.data(), S, stripes, stream, err, c->max_ctas);
  if (rc) return fail(rc, err);
  return PMRC_OK;
}

}  // extern "C"
