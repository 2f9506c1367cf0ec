#include <cmath>
#include <cstdio>
#include <cstdlib>
// Generator of the bitsliced sm_100a region-linear-combination kernels.
//
// Kernel design, driven by what the B200 measurements showed:
//   * A group = output blocks that read the same inputs (sparse MSR encode: the n-k parity symbols
//     of one PM symbol index j read the same d inputs).  Its GF(2^8) coefficients, expanded to
//     8x8 GF(2) matrices with zero coefficients skipped, form one XOR network, shortened by
//     Paar CSE and emitted as straight-line code: the only coefficient-specific code.
//   * Work unit = one warp x one 1 KiB chunk (32 lanes x 32 byte positions).  Lane l owns bytes
//     [16l,16l+16) and [512+16l,512+16l+16) of every block of the chunk.
//   * Instruction supply is the first-order constraint (profiles/r01): straight-line code that is
//     not re-executed starves the SM.  So all warps of a CTA execute the same group at the same
//     time, everything except the XOR networks is a loop, and per-group code stays ~20 KB.
//   * Memory: each team of warps runs a 2-stage pipeline: while a stage computes, every lane issues
//     16-B cp.async.cg copies (zero-fill via src-size at ragged ends) of the next stage's 1 KiB
//     input blocks into the other shared-memory buffer.  (A lane-0 TMA 1-D bulk-copy variant with
//     mbarrier complete_tx measured slower, profiles/r01/README.md v4 -> v5.)  Blocks read by a
//     single group and all parity stores carry an L2 evict-first policy.
//   * Each lane transposes its 32 bytes per block in place in shared memory (3 delta-swap stages,
//     LOP3 mux + IMAD shifts) into 8 bit planes; the XOR network reads planes with LDS.128, keeps
//     the group's 8 x 8 output planes in registers, then transposes back and stores 16-B vectors.
#include <algorithm>
#include <atomic>
#include <functional>
#include <map>
#include <sstream>
#include <thread>

#include "plan.hpp"

namespace pmrc {

namespace {

const char *kHeader = R"CUDA(
typedef unsigned int u32;
typedef unsigned long long u64;
// one delta-swap stage of an 8x8 bit transpose (per byte lane):
//   a' = m ? a : (b << s);  b' = m ? (a >> s) : b   -- LOP3 mux; shifts as IMAD / IMAD.HI (FMA pipe)
static __device__ __forceinline__ void pm_sw(u32 &a, u32 &b, const int s, const u32 m) {
  u32 bs, ar, na, nb;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(bs) : "r"(b), "r"(1u << s));
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(ar) : "r"(a), "r"(1u << (32 - s)));
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(na) : "r"(a), "r"(bs), "r"(m));
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(nb) : "r"(ar), "r"(b), "r"(m));
  a = na;
  b = nb;
}
// 8 words (32 bytes) <-> 8 bit planes (plane b = bit b of the 32 bytes); an involution
static __device__ __forceinline__ void pm_tr8(u32 &w0, u32 &w1, u32 &w2, u32 &w3, u32 &w4, u32 &w5, u32 &w6, u32 &w7) {
  pm_sw(w0, w4, 4, 0x0F0F0F0Fu); pm_sw(w1, w5, 4, 0x0F0F0F0Fu); pm_sw(w2, w6, 4, 0x0F0F0F0Fu); pm_sw(w3, w7, 4, 0x0F0F0F0Fu);
  pm_sw(w0, w2, 2, 0x33333333u); pm_sw(w1, w3, 2, 0x33333333u); pm_sw(w4, w6, 2, 0x33333333u); pm_sw(w5, w7, 2, 0x33333333u);
  pm_sw(w0, w1, 1, 0x55555555u); pm_sw(w2, w3, 1, 0x55555555u); pm_sw(w4, w5, 1, 0x55555555u); pm_sw(w6, w7, 1, 0x55555555u);
}
static __device__ __forceinline__ u32 pm_saddr(const void *p) { return (u32)__cvta_generic_to_shared(p); }
static __device__ __forceinline__ u64 pm_policy_ef() {
  u64 p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
static __device__ __forceinline__ void pm_st(unsigned char *p, bool v, u32 a, u32 b, u32 c, u32 d, u64 pol) {
  if (v) asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;"
                      :: "l"(p), "r"(a), "r"(b), "r"(c), "r"(d), "l"(pol) : "memory");
}
static __device__ __forceinline__ uint4 pm_lds(u32 a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
static __device__ __forceinline__ void pm_sts(u32 a, u32 x, u32 y, u32 z, u32 w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" :: "r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
// 16-B async copy global -> shared with an L2 cache policy; src_size 0 zero-fills (no branch)
static __device__ __forceinline__ void pm_cp16(u32 dst, const void *src, u32 src_size, u64 pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;"
               :: "r"(dst), "l"(src), "r"(src_size), "l"(pol) : "memory");
}
static __device__ __forceinline__ u64 pm_policy_el() {
  u64 p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
static __device__ __forceinline__ u64 pm_policy_en() {
  u64 p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
static __device__ __forceinline__ void pm_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> static __device__ __forceinline__ void pm_cp_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }
static __device__ __forceinline__ void pm_team_sync(u32 id, u32 n) { asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory"); }
static __device__ __forceinline__ void pm_team_arrive(u32 id, u32 n) { asm volatile("bar.arrive %0, %1;" :: "r"(id), "r"(n) : "memory"); }
// pacing of group-specialised CTAs (layout 1): wait until the n peer counters p[i * stride] reach
// `want`; bounded (a peer that is not resident must never deadlock us): after a timeout the caller
// stops pacing for the rest of the launch.  Counters are (epoch << 32 | chunks done).
static __device__ __forceinline__ bool pm_pace(const u64 *p, u32 stride, u32 n, u64 want, u32 lane) {
  for (u32 spin = 0; spin < 2048u; spin++) {
    bool ok = true;
    for (u32 i = lane; i < n; i += 32u) {
      u64 v;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p + (u64)i * stride) : "memory");
      ok = ok && v >= want;
    }
    if (__all_sync(0xffffffffu, ok)) return true;
    __nanosleep(128);
  }
  return false;
}
// n / d by multiply-high (Granlund-Montgomery): magic from pm_udiv_setup(d) once per thread
static __device__ __forceinline__ void pm_udiv_setup(u32 d, u32 &m, u32 &s1, u32 &s2) {
  const u32 l = d > 1u ? 32u - __clz(d - 1u) : 0u;
  m = (u32)(((1ull << 32) * ((1ull << l) - d)) / d) + 1u;
  s1 = l < 1u ? l : 1u;
  s2 = l > 0u ? l - 1u : 0u;
}
static __device__ __forceinline__ u32 pm_udiv(u32 n, u32 m, u32 s1, u32 s2) {
  const u32 t = __umulhi(m, n);
  return (t + ((n - t) >> s1)) >> s2;
}
static __device__ __forceinline__ u64 pm_gtime() {
  u64 t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
static __device__ __forceinline__ void pm_pace_post(u64 *p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
)CUDA";

void coef_rows(uint8_t c, uint8_t rows[8]) { gf().bitmatrix(c, rows); }
// W x W GF(2) matrix of "multiply by c" in GF(2^W) (W = 8 or 16), rows as masks over input bits
void coef_rows_w(int W, uint32_t c, uint32_t rows[16]) {
  if (W == 8) {
    uint8_t r8[8];
    gf().bitmatrix((uint8_t)c, r8);
    for (int b = 0; b < 8; b++) rows[b] = r8[b];
    return;
  }
  gf16().bitmatrix((uint16_t)c, rows);
}

// Emit an XOR program: base signal i is named base[i]; outputs into outs (assign or accumulate).
// Statements (temps and output rows) are emitted by a greedy register-pressure-aware list
// scheduler: among the statements whose temp operands exist, pick the one that minimises
// (new live values) - (operands that die here), so temps are consumed soon after they are made.
// need(name) is called before a statement for every base operand it reads (lazy plane loads).
template <class Need>
void emit_slp_lazy(std::ostringstream &s, const Slp &p, const std::vector<std::string> &base,
                   const std::vector<std::string> &outs, bool accumulate, const std::string &tpref, Need need) {
  const int nin = p.n_in, nt = (int)p.tmp.size(), nr = (int)p.rows.size();
  const int nst = nt + nr;
  std::vector<std::vector<int>> ops(nst);
  for (int i = 0; i < nt; i++) ops[i] = p.tmp[i];
  for (int r = 0; r < nr; r++) ops[nt + r] = p.rows[r];
  std::vector<int> uses(nin + nt, 0);
  for (auto &o : ops)
    for (int x : o) uses[x]++;
  std::vector<char> done(nst, 0), have(nin + nt, 0);
  for (int i = 0; i < nin; i++) have[i] = 1;
  // base signals come in quads (one LDS.128 = 4 registers, live until all 4 planes are done)
  std::vector<int> quad_uses((nin + 3) / 4, 0);
  std::vector<char> quad_live((nin + 3) / 4, 0);
  for (auto &o : ops)
    for (int x : o)
      if (x < nin) quad_uses[x / 4]++;
  auto nm = [&](int sig) -> std::string {
    if (sig < nin) {
      need(base[sig]);
      return base[sig];
    }
    return tpref + std::to_string(sig - nin);
  };
  auto ready = [&](int st) {
    for (int x : ops[st])
      if (!have[x]) return false;
    return true;
  };
  std::vector<int> qcount((nin + 3) / 4, 0);
  for (int step = 0; step < nst; step++) {
    int best = -1, bestscore = 1 << 30;
    for (int st = 0; st < nst; st++) {
      if (done[st] || !ready(st)) continue;
      int sc = 0;
      if (st < nt) sc += 1;                                   // defines a temp
      else if (!accumulate && !ops[st].empty()) sc += 1;      // defines an output (stays live)
      for (int x : ops[st]) {
        if (x >= nin && uses[x] == 1) sc -= 1;                // a temp's last use
        if (x < nin) qcount[x / 4]++;
      }
      for (int x : ops[st]) {
        if (x >= nin) continue;
        const int q = x / 4;
        if (!qcount[q]) continue;
        if (!quad_live[q]) sc += 4;                           // loads a quad
        if (quad_uses[q] == qcount[q]) sc -= 4;               // the quad's last use
        qcount[q] = 0;
      }
      if (sc < bestscore || (sc == bestscore && st < best)) { bestscore = sc; best = st; }
    }
    const int st = best;
    done[st] = 1;
    for (int x : ops[st]) {
      uses[x]--;
      if (x < nin) {
        quad_uses[x / 4]--;
        quad_live[x / 4] = quad_uses[x / 4] > 0;
      }
    }
    if (st < nt) {
      std::vector<std::string> on;
      for (int x : ops[st]) on.push_back(nm(x));
      s << "    const u32 " << tpref << st << " = ";
      for (size_t j = 0; j < on.size(); j++) s << (j ? " ^ " : "") << on[j];
      s << ";\n";
      have[nin + st] = 1;
    } else {
      const int r = st - nt;
      if (ops[st].empty()) {
        if (!accumulate) s << "    " << outs[r] << " = 0u;\n";
        continue;
      }
      std::vector<std::string> on;
      for (int x : ops[st]) on.push_back(nm(x));
      // balanced ternary XOR tree (3-input LOP3 per node): depth log3(k) instead of k/2
      while (on.size() > 3) {
        std::vector<std::string> nx;
        for (size_t j = 0; j < on.size(); j += 3) {
          if (j + 1 >= on.size()) nx.push_back(on[j]);
          else if (j + 2 >= on.size()) nx.push_back("(" + on[j] + " ^ " + on[j + 1] + ")");
          else nx.push_back("(" + on[j] + " ^ " + on[j + 1] + " ^ " + on[j + 2] + ")");
        }
        on.swap(nx);
      }
      s << "    " << outs[r] << (accumulate ? " ^= " : " = ");
      for (size_t j = 0; j < on.size(); j++) s << (j ? " ^ " : "") << on[j];
      s << ";\n";
    }
  }
}
// Eager-fold emission: temps in creation order; every operand that becomes available (a temp when
// created, a plane quad when loaded) is folded into the rows that use it as soon as a row has two
// pending operands (o ^= a ^ b: one 3-input LOP3), so temps and plane quads die right after their
// last consumer instead of living until a row's single big expression.
template <class Need>
void emit_slp_fold(std::ostringstream &s, const Slp &p, const std::vector<std::string> &base,
                   const std::vector<std::string> &outs, bool accumulate, const std::string &tpref, Need need) {
  const int nin = p.n_in, nt = (int)p.tmp.size(), nr = (int)p.rows.size();
  std::vector<std::vector<int>> rows_of(nin + nt);
  for (int r = 0; r < nr; r++)
    for (int x : p.rows[r]) rows_of[x].push_back(r);
  std::vector<std::vector<int>> pending(nr);
  std::vector<char> started(nr, accumulate ? 1 : 0), quad_done((nin + 3) / 4, 0);
  auto name = [&](int sig) { return sig < nin ? base[sig] : tpref + std::to_string(sig - nin); };
  auto try_fold = [&](int r) {
    auto &pd = pending[r];
    if (!started[r]) {
      if (pd.size() < 3) return;
      s << "    " << outs[r] << " = " << name(pd[0]) << " ^ " << name(pd[1]) << " ^ " << name(pd[2]) << ";\n";
      pd.erase(pd.begin(), pd.begin() + 3);
      started[r] = 1;
    }
    while (pd.size() >= 2) {
      s << "    " << outs[r] << " ^= " << name(pd[0]) << " ^ " << name(pd[1]) << ";\n";
      pd.erase(pd.begin(), pd.begin() + 2);
    }
  };
  auto make_available = [&](int sig) {
    for (int r : rows_of[sig]) {
      pending[r].push_back(sig);
      try_fold(r);
    }
  };
  auto load_quad = [&](int q) {
    if (quad_done[q]) return;
    quad_done[q] = 1;
    need(base[4 * q]);
    for (int x = 4 * q; x < std::min(nin, 4 * q + 4); x++) make_available(x);
  };
  for (int i = 0; i < nt; i++) {
    for (int x : p.tmp[i])
      if (x < nin) load_quad(x / 4);
    s << "    const u32 " << tpref << i << " = ";
    for (size_t j = 0; j < p.tmp[i].size(); j++) s << (j ? " ^ " : "") << name(p.tmp[i][j]);
    s << ";\n";
    make_available(nin + i);
  }
  for (int r = 0; r < nr; r++)
    for (int x : p.rows[r])
      if (x < nin) load_quad(x / 4);
  for (int r = 0; r < nr; r++) {
    auto &pd = pending[r];
    if (!started[r]) {
      s << "    " << outs[r] << " = ";
      if (pd.empty()) s << "0u";
      for (size_t j = 0; j < pd.size(); j++) s << (j ? " ^ " : "") << name(pd[j]);
      s << ";\n";
    } else if (!pd.empty()) {
      s << "    " << outs[r] << " ^= " << name(pd[0]) << ";\n";
    }
    pd.clear();
  }
}

// Register-pressure-aware eager-fold emission: the same fold mechanics as emit_slp_fold, but the
// next temp is chosen greedily (instead of in CSE creation order) to minimise the growth of live
// values: loading a plane quad costs 4 registers, a new temp 1, and every operand (temp or quad)
// whose last consumer this temp is frees its registers.  Ties: CSE order.
template <class Need>
void emit_slp_sched(std::ostringstream &s, const Slp &p, const std::vector<std::string> &base,
                    const std::vector<std::string> &outs, bool accumulate, const std::string &tpref, Need need) {
  const int nin = p.n_in, nt = (int)p.tmp.size(), nr = (int)p.rows.size();
  const int nq = (nin + 3) / 4;
  std::vector<std::vector<int>> rows_of(nin + nt), tmps_of(nin + nt);
  for (int r = 0; r < nr; r++)
    for (int x : p.rows[r]) rows_of[x].push_back(r);
  for (int i = 0; i < nt; i++)
    for (int x : p.tmp[i]) tmps_of[x].push_back(i);
  // remaining temp consumers of each signal, and of each quad (sum over its planes)
  std::vector<int> tleft(nin + nt, 0), qleft(nq, 0);
  for (int i = 0; i < nt; i++)
    for (int x : p.tmp[i]) {
      tleft[x]++;
      if (x < nin) qleft[x / 4]++;
    }
  std::vector<std::vector<int>> pending(nr);
  std::vector<char> started(nr, accumulate ? 1 : 0), quad_done(nq, 0), made(nt, 0);
  auto name = [&](int sig) { return sig < nin ? base[sig] : tpref + std::to_string(sig - nin); };
  auto try_fold = [&](int r) {
    auto &pd = pending[r];
    if (!started[r]) {
      if (pd.size() < 3) return;
      s << "    " << outs[r] << " = " << name(pd[0]) << " ^ " << name(pd[1]) << " ^ " << name(pd[2]) << ";\n";
      pd.erase(pd.begin(), pd.begin() + 3);
      started[r] = 1;
    }
    while (pd.size() >= 2) {
      s << "    " << outs[r] << " ^= " << name(pd[0]) << " ^ " << name(pd[1]) << ";\n";
      pd.erase(pd.begin(), pd.begin() + 2);
    }
  };
  auto make_available = [&](int sig) {
    for (int r : rows_of[sig]) {
      pending[r].push_back(sig);
      try_fold(r);
    }
  };
  auto load_quad = [&](int q) {
    if (quad_done[q]) return;
    quad_done[q] = 1;
    need(base[4 * q]);
    for (int x = 4 * q; x < std::min(nin, 4 * q + 4); x++) make_available(x);
  };
  for (int step = 0; step < nt; step++) {
    int best = -1, bscore = 1 << 30;
    for (int i = 0; i < nt; i++) {
      if (made[i]) continue;
      bool ready = true;
      for (int x : p.tmp[i])
        if (x >= nin && !made[x - nin]) ready = false;
      if (!ready) continue;
      int sc = 1;
      int qs[3] = {-1, -1, -1}, nqs = 0;
      for (int x : p.tmp[i]) {
        if (x >= nin) {
          if (tleft[x] == 1) sc -= 1;
        } else {
          const int q = x / 4;
          bool seen = false;
          for (int k = 0; k < nqs; k++) seen |= qs[k] == q;
          if (seen) continue;
          qs[nqs++] = q;
          int use = 0;
          for (int y : p.tmp[i])
            if (y < nin && y / 4 == q) use++;
          if (!quad_done[q]) sc += 4;
          if (qleft[q] == use) sc -= 4;
        }
      }
      if (sc < bscore) { bscore = sc; best = i; }
    }
    const int i = best;
    for (int x : p.tmp[i])
      if (x < nin) load_quad(x / 4);
    s << "    const u32 " << tpref << i << " = ";
    for (size_t j = 0; j < p.tmp[i].size(); j++) s << (j ? " ^ " : "") << name(p.tmp[i][j]);
    s << ";\n";
    made[i] = 1;
    for (int x : p.tmp[i]) {
      tleft[x]--;
      if (x < nin) qleft[x / 4]--;
    }
    make_available(nin + i);
  }
  for (int r = 0; r < nr; r++)
    for (int x : p.rows[r])
      if (x < nin) load_quad(x / 4);
  for (int r = 0; r < nr; r++) {
    auto &pd = pending[r];
    if (!started[r]) {
      s << "    " << outs[r] << " = ";
      if (pd.empty()) s << "0u";
      for (size_t j = 0; j < pd.size(); j++) s << (j ? " ^ " : "") << name(pd[j]);
      s << ";\n";
    } else if (!pd.empty()) {
      s << "    " << outs[r] << " ^= " << name(pd[0]) << ";\n";
    }
    pd.clear();
  }
}

void emit_slp(std::ostringstream &s, const Slp &p, const std::vector<std::string> &base,
              const std::vector<std::string> &outs, bool accumulate, const std::string &tpref) {
  emit_slp_lazy(s, p, base, outs, accumulate, tpref, [](const std::string &) {});
}

Slp make_slp(int n_in, const std::vector<std::vector<int>> &rows, bool cse, int restarts = 1) {
  if (cse) {
    Slp best = cse3(n_in, rows, 0);
    long bc = best.lop3();
    for (int r = 1; r < restarts; r++) {
      Slp t = cse3(n_in, rows, (uint32_t)r);
      const long c = t.lop3();
      if (c < bc) { bc = c; best = std::move(t); }
    }
    return best;
  }
  Slp s;
  s.n_in = n_in;
  s.rows = rows;
  return s;
}

struct Group {
  std::vector<int> rows, cols;
};
struct Stage {
  int g = 0;
  std::vector<int> cols;  // inputs (plan columns) computed in this stage
  std::vector<std::pair<int, int>> blocks;  // loaded (slot, blk), in smem slot order
  std::vector<int> first_block;             // per col: index of its first loaded block
  std::vector<char> ef;                     // per loaded block: last read -> evict-first
};

bool is_plain(const InputDesc &in) { return in.terms.size() == 1 && in.terms[0].coef == 1; }

}  // namespace

std::string generate_source(const PlanSpec &p, const GenOptions &o, GenStats &st) {
  st = GenStats();
  // symbol width: W bit planes per symbol; a warp handles a chunk of CB = 128 W bytes of every
  // block (32 lanes x 32 symbols), a lane's 32 symbols are NSEG 16-byte segments 512 B apart
  const int W = p.w == 16 ? 16 : 8;
  const int CB = 128 * W, NSEG = W / 4;
  const int R = (int)p.outputs.size();
  const int C = (int)p.inputs.size();
  // ---- groups: output rows with identical support, split into chunks of max_rows ----
  std::map<std::vector<int>, std::vector<int>> by_support;
  for (int r = 0; r < R; r++) {
    std::vector<int> sup;
    for (int c = 0; c < C; c++)
      if (p.A.at(r, c)) sup.push_back(c);
    by_support[sup].push_back(r);
  }
  std::vector<Group> groups;
  for (auto &kv : by_support) st.max_support_rows = std::max(st.max_support_rows, (int)kv.second.size());
  for (auto &kv : by_support)
    for (size_t i = 0; i < kv.second.size(); i += o.max_rows) {
      Group g;
      g.cols = kv.first;
      for (size_t j = i; j < std::min(kv.second.size(), i + (size_t)o.max_rows); j++) g.rows.push_back(kv.second[j]);
      groups.push_back(g);
    }
  // Rows with (nearly) all-distinct supports (decode: rows of G~^-1) would make one group per row,
  // each loading and transposing its own inputs.  Then cluster rows greedily instead: seed with the
  // widest remaining row, add the rows that grow the union support least, up to max_rows; a zero
  // coefficient inside a group's union costs a load but no XOR (skipped when the network is built).
  const size_t min_groups = (R + o.max_rows - 1) / std::max(1, o.max_rows);
  if (R > 0 && groups.size() > min_groups + min_groups / 2) {
    std::vector<std::vector<char>> sup(R, std::vector<char>(C, 0));
    std::vector<int> w(R, 0);
    for (int r = 0; r < R; r++)
      for (int c = 0; c < C; c++)
        if (p.A.at(r, c)) sup[r][c] = 1, w[r]++;
    std::vector<char> left(R, 1);
    int nleft = R;
    groups.clear();
    st.clustered = true;
    // even_groups: equal group sizes (28 rows, max 16 -> 14 + 14, not 16 + 12), for static equal
    // chunk ranges; with the dynamic schedule 16 + 12 is better: 4 + 4 + 4 + 4 and 3 + 3 + 3 + 3 rows
    // per team rank keep the team barriers balanced (14 rows: 3 + 4 + 3 + 4)
    const int cap = o.even_groups ? (int)((R + min_groups - 1) / min_groups) : o.max_rows;
    while (nleft > 0) {
      int seed = -1;
      for (int r = 0; r < R; r++)
        if (left[r] && (seed < 0 || w[r] > w[seed])) seed = r;
      Group g;
      std::vector<char> U = sup[seed];
      g.rows.push_back(seed);
      left[seed] = 0;
      nleft--;
      while ((int)g.rows.size() < cap && nleft > 0) {
        int best = -1, bgrow = 1 << 30;
        for (int r = 0; r < R; r++) {
          if (!left[r]) continue;
          int grow = 0;
          for (int c = 0; c < C; c++) grow += sup[r][c] && !U[c];
          // ties (typically 0: the seed already reads every input): the widest row, so that
          // rows of similar weight share a group (decode: dense rows of lost data vs sparse ones)
          if (grow < bgrow || (o.cluster_wide && grow == bgrow && w[r] > w[best])) { bgrow = grow; best = r; }
        }
        g.rows.push_back(best);
        left[best] = 0;
        nleft--;
        for (int c = 0; c < C; c++) U[c] |= sup[best][c];
      }
      std::sort(g.rows.begin(), g.rows.end());
      for (int c = 0; c < C; c++)
        if (U[c]) g.cols.push_back(c);
      groups.push_back(g);
    }
  }
  st.groups = (int)groups.size();
  {
    long mn = 1L << 40, mx = 0;
    for (auto &g : groups) {
      long c = (long)g.rows.size();
      for (int col : g.cols) c += (long)p.inputs[col].terms.size();
      mn = std::min(mn, c);
      mx = std::max(mx, c);
    }
    st.group_cost_ratio = groups.empty() ? 1.0 : (double)mx / (double)std::max(1L, mn);
  }
  // ---- partition search (part_search != 0): a group of plain inputs is computed as T ranks (row
  // shares) x stages x sub-networks (input shares), each (rank, sub-network) with its own CSE.  Which inputs share
  // a sub-network and which rows share a warp is free: hill-climb over swaps of two inputs between
  // sub-networks / two rows between ranks, minimising the slower rank's LOP3 count (the ranks meet
  // at a barrier), then the total.  Deterministic (fixed seeds); the groups search in parallel.
  // part_search > 0 searches plans of unequal groups only, < 0 every plan.  Measured (200 and 600
  // evaluations, profiles/r02/part_search.jsonl): MBR k = 8 encode (14- and 8-input groups) 19,960 ->
  // 19,700 XORs, 0.573 -> 0.559 ms; the MSR k = 8 encode's equal groups lose 1.5% of their XORs
  // (12,305 -> 12,122) but run 0.8% slower (0.491 -> 0.495 ms), MSR k = 4 is unchanged.
  if (o.part_search != 0 && (o.part_search < 0 || st.group_cost_ratio > 1.2) && o.cse && W == 8 && !st.clustered &&
      !(o.ws && o.layout >= 1)) {
    const int evals = std::abs(o.part_search);
    const int TT = std::max(1, o.team);
    auto search = [&](Group &G, uint32_t seed) {
      for (int c : G.cols)
        if (p.inputs[c].terms.size() != 1) return;
      const int ncols = (int)G.cols.size(), mall = (int)G.rows.size();
      // segments: the stages the inputs are packed into (the rule of the stage loop below), each
      // cut into sub-networks (the rule of the network emission); seg0[q] = first input of segment q
      const int IB = std::max(1, o.in_block);
      int cap = IB;
      if (o.stage_even) {
        const int nst = std::max(1, (ncols + IB - 1) / IB);
        cap = std::min(IB, (ncols + nst - 1) / nst);
      }
      std::vector<int> seg0;
      for (int s0 = 0; s0 < ncols; s0 += cap) {
        const int ncs = std::min(cap, ncols - s0);
        int sub = o.net_in > 0 ? o.net_in : ncs;
        if (o.net_even && sub < ncs) {
          const int nsub = (ncs + sub - 1) / sub;
          sub = (ncs + nsub - 1) / nsub;
        }
        for (int c0 = 0; c0 < ncs; c0 += sub) seg0.push_back(s0 + c0);
      }
      const int nseg = (int)seg0.size();
      // multi-stage groups (k = 16: 30 inputs in 3 stages) only on request (part_search < 0): the
      // search shortens their networks by 1.4% but the kernels measure 0.2-0.7% slower
      // (profiles/r02/part_search_k16.jsonl)
      if (ncols > cap && o.part_search > 0) return;
      seg0.push_back(ncols);
      std::vector<int> seg_of(ncols);
      for (int q = 0; q < nseg; q++)
        for (int ci = seg0[q]; ci < seg0[q + 1]; ci++) seg_of[ci] = q;
      const bool col_moves = nseg >= 2, row_moves = TT >= 2 && mall >= 2 * TT;
      if (!col_moves && !row_moves) return;
      auto net = [&](const std::vector<int> &rw, const std::vector<int> &cl, int rk, int q) {
        const int r0 = mall * rk / TT, m = mall * (rk + 1) / TT - r0, c0 = seg0[q], c1 = seg0[q + 1];
        std::vector<std::vector<int>> sr(W * m);
        for (int r = 0; r < m; r++)
          for (int ci = c0; ci < c1; ci++) {
            const uint32_t cf = p.coef(rw[r0 + r], cl[ci]);
            if (!cf) continue;
            uint32_t br[16];
            coef_rows_w(W, cf, br);
            for (int b = 0; b < W; b++)
              for (int bp = 0; bp < W; bp++)
                if ((br[b] >> bp) & 1) sr[r * W + b].push_back((ci - c0) * W + bp);
          }
        return cse3(W * (c1 - c0), sr, 0).lop3();
      };
      auto score = [&](const std::vector<long> &c) {  // c[rk * nseg + q]
        long worst = 0, total = 0;
        for (int rk = 0; rk < TT; rk++) {
          long mine = 0;
          for (int q = 0; q < nseg; q++) mine += c[rk * nseg + q];
          worst = std::max(worst, mine);
          total += mine;
        }
        return worst * 1000000 + total;
      };
      std::vector<int> rw = G.rows, cl = G.cols;
      std::vector<long> cc(TT * nseg);
      for (int rk = 0; rk < TT; rk++)
        for (int q = 0; q < nseg; q++) cc[rk * nseg + q] = net(rw, cl, rk, q);
      long cur = score(cc);
      uint32_t x = seed * 2654435761u + 12345u;
      auto rnd = [&](int n) {
        x ^= x << 13, x ^= x >> 17, x ^= x << 5;
        return (int)(x % (uint32_t)n);
      };
      for (int it = 0; it < evals; it++) {
        std::vector<int> r2 = rw, c2 = cl;
        std::vector<long> n2 = cc;
        if (row_moves && (!col_moves || it % 3 == 2)) {
          const int a = rnd(TT), b = (a + 1 + rnd(TT - 1)) % TT;
          const int ia = mall * a / TT + rnd(mall * (a + 1) / TT - mall * a / TT);
          const int ib = mall * b / TT + rnd(mall * (b + 1) / TT - mall * b / TT);
          std::swap(r2[ia], r2[ib]);
          for (int q = 0; q < nseg; q++) n2[a * nseg + q] = net(r2, c2, a, q), n2[b * nseg + q] = net(r2, c2, b, q);
        } else {
          const int ia = rnd(ncols);
          int ib = rnd(ncols);
          for (int tries = 0; seg_of[ia] == seg_of[ib] && tries < 64; tries++) ib = rnd(ncols);
          if (seg_of[ia] == seg_of[ib]) continue;
          std::swap(c2[ia], c2[ib]);
          for (int rk = 0; rk < TT; rk++)
            for (int q : {seg_of[ia], seg_of[ib]}) n2[rk * nseg + q] = net(r2, c2, rk, q);
        }
        const long c = score(n2);
        if (c <= cur) cur = c, rw.swap(r2), cl.swap(c2), cc.swap(n2);
      }
      G.rows = rw;
      G.cols = cl;
    };
    std::vector<std::thread> th;
    const size_t nth = std::min<size_t>(groups.size(), std::max(1u, std::thread::hardware_concurrency()));
    std::atomic<size_t> next{0};
    for (size_t t = 0; t < nth; t++)
      th.emplace_back([&] {
        for (size_t g = next++; g < groups.size(); g = next++) search(groups[g], (uint32_t)g + 1);
      });
    for (auto &t : th) t.join();
  }

  // ---- stages: each group's inputs packed into shared-memory buffers of <= IB loaded blocks ----
  const int IB = std::max(1, o.in_block);
  std::vector<Stage> stages;
  std::vector<std::vector<int>> gstages(groups.size());
  for (size_t g = 0; g < groups.size(); g++) {
    Stage cur;
    cur.g = (int)g;
    // balanced stages: as few as IB allows, of equal size (30 inputs -> 15 + 15, not 14 + 14 + 2)
    int cap = IB;
    if (o.stage_even) {
      int tot = 0;
      for (int c : groups[g].cols) tot += (int)p.inputs[c].terms.size();
      const int nst = std::max(1, (tot + IB - 1) / IB);
      cap = std::min(IB, (tot + nst - 1) / nst);
    }
    for (int c : groups[g].cols) {
      const InputDesc &in = p.inputs[c];
      int need = (int)in.terms.size();
      if (!cur.cols.empty() && (int)cur.blocks.size() + need > cap) {
        gstages[g].push_back((int)stages.size());
        stages.push_back(cur);
        cur = Stage();
        cur.g = (int)g;
      }
      cur.first_block.push_back((int)cur.blocks.size());
      cur.cols.push_back(c);
      for (auto &t : in.terms) cur.blocks.push_back({t.slot, t.blk});
    }
    if (!cur.cols.empty()) {
      gstages[g].push_back((int)stages.size());
      stages.push_back(cur);
    }
  }
  int qmax = 1;
  for (auto &sg : stages) qmax = std::max(qmax, (int)sg.blocks.size());
  // ---- per-stage split of the loaded blocks over the team ranks: rank rk loads (cp.async) and
  // transposes blocks [tsplit[si][rk], tsplit[si][rk + 1]) of stage si (a warp can only wait for its
  // own copies, so loads and transposes split alike).  Default: equal shares.  tr_balance: shares
  // that equalise each rank's (XOR network + transposes) per item, from the networks' LOP3 counts,
  // since the ranks meet at a barrier every stage (decode rows differ 4x in XOR work).
  std::vector<std::vector<int>> tsplit(stages.size());
  {
    const int TT = std::max(1, o.team);
    const bool ws_on = o.ws && o.layout >= 1 && TT >= 2;
    const int NPk = ws_on ? std::max(1, std::min(TT - 1, o.ws_prod)) : 0;
    for (size_t si = 0; si < stages.size(); si++) {
      const int n = (int)stages[si].blocks.size(), parts = ws_on ? NPk : TT;
      for (int rk = 0; rk <= parts; rk++) tsplit[si].push_back(n * rk / parts);
    }
    if (o.tr_balance && TT >= 2 && !ws_on) {
      const int sub_in = o.net_in > 0 ? (W == 16 ? (o.net_in + 1) / 2 : o.net_in) : 0;
      for (size_t g = 0; g < groups.size(); g++) {
        const Group &G = groups[g];
        const int mall = (int)G.rows.size();
        std::vector<double> net(TT, 0.0);
        int n_in = 0;
        for (int si : gstages[g]) n_in += (int)stages[si].blocks.size();
        for (int rk = 0; rk < TT; rk++) {
          const int r0 = mall * rk / TT, m = mall * (rk + 1) / TT - r0;
          net[rk] += 24.0 * m;  // output transposes
          for (int si : gstages[g]) {
            const Stage &sg = stages[si];
            std::vector<std::vector<int>> rows(W * m);
            for (int r = 0; r < m; r++)
              for (size_t ci = 0; ci < sg.cols.size(); ci++) {
                const uint32_t cf = p.coef(G.rows[r0 + r], sg.cols[ci]);
                if (!cf) continue;
                uint32_t br[16];
                coef_rows_w(W, cf, br);
                for (int b = 0; b < W; b++)
                  for (int bp = 0; bp < W; bp++)
                    if ((br[b] >> bp) & 1) rows[r * W + b].push_back((int)ci * W + bp);
              }
            const int ncols = (int)sg.cols.size();
            int sub = sub_in > 0 ? sub_in : ncols;
            if (o.net_even && sub < ncols) {
              const int nsub = (ncols + sub - 1) / sub;
              sub = (ncols + nsub - 1) / nsub;
            }
            for (int c0 = 0; c0 < ncols; c0 += sub) {
              const int c1 = std::min(ncols, c0 + sub);
              std::vector<std::vector<int>> sr(rows.size());
              for (size_t r = 0; r < rows.size(); r++)
                for (int x : rows[r])
                  if (x >= W * c0 && x < W * c1) sr[r].push_back(x - W * c0);
              net[rk] += (double)make_slp(W * (c1 - c0), sr, o.cse, o.cse_restarts).lop3() + 0.5 * W * m;
            }
          }
        }
        // water-fill the group's n_in input transposes (24 LOP3-equivalents each) over the ranks
        std::vector<int> x(TT, 0);
        for (int k = 0; k < n_in; k++) {
          int best = 0;
          for (int rk = 1; rk < TT; rk++)
            if (net[rk] + 24.0 * x[rk] < net[best] + 24.0 * x[best]) best = rk;
          x[best]++;
        }
        // per stage: cumulative rounding of the shares x[rk] / n_in
        std::vector<double> cum(TT + 1, 0.0);
        for (int rk = 0; rk < TT; rk++) cum[rk + 1] = cum[rk] + x[rk];
        for (int si : gstages[g]) {
          const int n = (int)stages[si].blocks.size();
          for (int rk = 0; rk <= TT; rk++)
            tsplit[si][rk] = n_in ? (int)std::lround(cum[rk] * n / n_in) : n * rk / TT;
        }
      }
    }
  }
  // ---- rows -> team ranks: rank rk computes rows [m*rk/T, m*(rk+1)/T) of its group's row list and
  // transposes blocks [n*rk/T, n*(rk+1)/T) of every stage; the ranks meet at a barrier per stage, so
  // reorder the rows to balance (XOR work + transposes) per rank (longest-processing-time greedy).
  // (Option, off by default: measured slower for decode and encode.)
  if (o.balance_ranks && o.team >= 2 && !(o.ws && o.layout >= 1)) {
    const int TT = o.team;
    for (size_t g = 0; g < groups.size(); g++) {
      Group &G = groups[g];
      const int mall = (int)G.rows.size();
      if (mall < 2) continue;
      std::vector<double> load(TT, 0.0);
      std::vector<int> room(TT);
      for (int rk = 0; rk < TT; rk++) {
        room[rk] = mall * (rk + 1) / TT - mall * rk / TT;
        for (int si : gstages[g]) {
          const int nb = (int)stages[si].blocks.size();
          load[rk] += 44.0 * (nb * (rk + 1) / TT - nb * rk / TT);  // a transpose ~ 44 XOR2 of issue
        }
        load[rk] += 44.0 * room[rk];  // output transposes
      }
      std::vector<std::pair<double, int>> cost;
      for (int r : G.rows) {
        long ones = 0;
        for (int c : G.cols)
          if (const uint32_t cf = p.coef(r, c)) {
            uint32_t br[16];
            coef_rows_w(W, cf, br);
            for (int b = 0; b < W; b++) ones += __builtin_popcount(br[b]);
          }
        cost.push_back({0.55 * (double)ones, r});  // ~ XOR2 after CSE
      }
      double lo = 1e300, hi = 0;
      for (auto &cr : cost) lo = std::min(lo, cr.first), hi = std::max(hi, cr.first);
      if (hi <= 1.1 * lo) continue;  // rows alike: keep the order
      std::stable_sort(cost.begin(), cost.end(), [](const std::pair<double, int> &a, const std::pair<double, int> &b) {
        return a.first > b.first;
      });
      std::vector<std::vector<int>> lists(TT);
      for (auto &cr : cost) {
        int best = -1;
        for (int rk = 0; rk < TT; rk++)
          if ((int)lists[rk].size() < room[rk] && (best < 0 || load[rk] < load[best])) best = rk;
        lists[best].push_back(cr.second);
        load[best] += cr.first;
      }
      // pairwise swaps between ranks while they lower the larger of the two loads (the fixed row
      // counts per rank keep LPT alone from balancing rows of similar cost)
      std::map<int, double> rc;
      for (auto &cr : cost) rc[cr.second] = cr.first;
      for (int it = 0; it < 64; it++) {
        double gain = 0;
        int ba = -1, bb = -1, bi = -1, bj = -1;
        for (int a = 0; a < TT; a++)
          for (int b = 0; b < TT; b++) {
            if (load[a] <= load[b]) continue;
            for (size_t i = 0; i < lists[a].size(); i++)
              for (size_t j = 0; j < lists[b].size(); j++) {
                const double d = rc[lists[a][i]] - rc[lists[b][j]];
                if (d <= 0) continue;
                const double nm = std::max(load[a] - d, load[b] + d), g0 = load[a] - nm;
                if (g0 > gain) gain = g0, ba = a, bb = b, bi = (int)i, bj = (int)j;
              }
          }
        if (ba < 0) break;
        const double d = rc[lists[ba][bi]] - rc[lists[bb][bj]];
        std::swap(lists[ba][bi], lists[bb][bj]);
        load[ba] -= d;
        load[bb] += d;
      }
      if (getenv("PMRC_DEBUG_BAL"))
        for (int rk = 0; rk < TT; rk++) {
          fprintf(stderr, "group %zu rank %d load %.0f rows", g, rk, load[rk]);
          for (int r : lists[rk]) fprintf(stderr, " %d:%.0f", r, rc[r]);
          fprintf(stderr, "\n");
        }
      G.rows.clear();
      for (auto &l : lists) {
        std::sort(l.begin(), l.end());
        G.rows.insert(G.rows.end(), l.begin(), l.end());
      }
    }
  }
  // L2 policy: a loaded block keeps normal priority if a later stage of the tile loads it again
  {
    std::map<std::pair<int, int>, std::pair<int, int>> last;  // block -> (stage, index) of last read
    for (size_t g = 0; g < groups.size(); g++)
      for (int si : gstages[g])
        for (size_t i = 0; i < stages[si].blocks.size(); i++) last[stages[si].blocks[i]] = {si, (int)i};
    // layouts 1/2 run the groups concurrently on different SMs, so "the last read" is not known
    // statically there: a block loaded by more than one group gets policy o.l2_shared (0 normal,
    // 2 evict_last), a block loaded by one group only is streamed with evict_first
    std::map<std::pair<int, int>, int> readers;
    for (size_t g = 0; g < groups.size(); g++) {
      std::map<std::pair<int, int>, bool> seen;
      for (int si : gstages[g])
        for (auto &b : stages[si].blocks) seen[b] = true;
      for (auto &kv : seen) readers[kv.first]++;
    }
    for (size_t si = 0; si < stages.size(); si++) {
      stages[si].ef.assign(stages[si].blocks.size(), 0);
      for (size_t i = 0; i < stages[si].blocks.size(); i++) {
        // (a block that every group reads -- decode plans -- keeps the static rule: measured
        // 0.858 vs 0.976 ms for the config-4 decode)
        const int nr = readers[stages[si].blocks[i]];
        if (o.layout >= 1 && o.l2_shared >= 0 && (nr == 1 || nr < (int)groups.size())) {
          stages[si].ef[i] = nr > 1 ? (o.l2_shared == 2 ? 2 : 0) : 1;
          continue;
        }
        auto l = last[stages[si].blocks[i]];
        stages[si].ef[i] = (l.first == (int)si && l.second == (int)i) ? 1 : 0;
      }
    }
  }

  const int M = std::max(1, o.chunk_loop);
  // stage-buffer ring per team: NB buffers, prefetch distance D = NB - 1 stages (layouts 1/2)
  // The dynamic chunk schedule knows a team's next item one item ahead, so with it the prefetch
  // distance may not reach past the next item: every group must have >= D stages (else 2 buffers).
  int min_ns = 1 << 30;
  for (auto &gs : gstages)
    if (!gs.empty()) min_ns = std::min(min_ns, (int)gs.size());
  int NB = (o.layout == 0 || (o.ws && o.team >= 2)) ? 2 : std::max(2, o.nbuf);
  if (NB > 2 && o.dyn > 0 && o.layout == 1 && NB - 1 > min_ns) NB = 2;
  const int D = NB - 1;
  const int T = std::max(1, o.team);  // warps sharing one chunk's stage buffer
  // warp-specialised teams (o.ws, layouts 1/2): rank 0 loads and transposes every block of a
  // stage (producer), ranks 1..T-1 run the XOR networks (consumers); named barriers FULL/EMPTY per
  // stage buffer replace the team barrier (4 ids per team: teams <= 4, two buffers)
  const bool WS = o.ws && o.layout >= 1 && T >= 2;
  const int NP = WS ? std::max(1, std::min(T - 1, o.ws_prod)) : 0;  // producer warps per team
  std::ostringstream s;
  s << "// generated by libpmrc (codegen.cpp) — bitsliced GF(2^8) region linear combination\n";
  s << kHeader;
  if (W == 16)
    s << R"CUDA(// 16 words (32 GF(2^16) symbols, little-endian) <-> 16 bit planes; an involution (4 delta-swap stages)
static __device__ __forceinline__ void pm_tr16(u32 *w) {
  #pragma unroll
  for (int i = 0; i < 8; i++) pm_sw(w[i], w[i + 8], 8, 0x00FF00FFu);
  #pragma unroll
  for (int h = 0; h < 16; h += 8)
    #pragma unroll
    for (int i = 0; i < 4; i++) pm_sw(w[h + i], w[h + i + 4], 4, 0x0F0F0F0Fu);
  #pragma unroll
  for (int h = 0; h < 16; h += 4)
    #pragma unroll
    for (int i = 0; i < 2; i++) pm_sw(w[h + i], w[h + i + 2], 2, 0x33333333u);
  #pragma unroll
  for (int h = 0; h < 16; h += 2) pm_sw(w[h], w[h + 1], 1, 0x55555555u);
}
)CUDA";
  s << "struct Slots { u64 ptr[" << std::max(1, p.n_slots) << "]; u64 stride[" << std::max(1, p.n_slots) << "]; };\n";
  s << "#define PM_QMAX " << qmax << "u\n";
  s << "#define PM_T " << T << "u\n";
  size_t nb_total = 0;
  for (auto &sg : stages) nb_total += sg.blocks.size();
  // loaded blocks: (slot << 16 | blk), bit 31 = last read (evict-first)
  s << "__constant__ u32 pm_blk[" << std::max<size_t>(1, nb_total) << "] = {";
  {
    size_t k = 0;
    for (auto &sg : stages)
      for (size_t i = 0; i < sg.blocks.size(); i++, k++)
        s << (k ? ", " : "") << ((sg.ef[i] ? 0x80000000u : 0u) | ((uint32_t)sg.blocks[i].first << 16) |
                                 (uint32_t)sg.blocks[i].second) << "u";
    if (!nb_total) s << "0u";
  }
  s << "};\n";
  s << "__constant__ u32 pm_stage_off[" << stages.size() + 1 << "] = {";
  {
    size_t off = 0;
    for (size_t si = 0; si <= stages.size(); si++) {
      s << (si ? ", " : "") << off << "u";
      if (si < stages.size()) off += stages[si].blocks.size();
    }
  }
  s << "};\n";
  std::vector<uint32_t> seq;
  for (size_t g = 0; g < groups.size(); g++)
    for (int m = 0; m < M; m++)
      for (int si : gstages[g]) seq.push_back(((uint32_t)si << 8) | (uint32_t)m);
  const size_t L = seq.size();
  s << "#define PM_L " << L << "u\n";
  s << "__constant__ u32 pm_seq[" << std::max<size_t>(1, L) << "] = {";
  for (size_t i = 0; i < L; i++) s << (i ? ", " : "") << seq[i] << "u";
  if (!L) s << "0u";
  s << "};\n";

  s << "\n// in-place 8x8 bit transpose of this lane's 32 bytes of blocks [lo, hi) of a stage buffer\n"
       "static __device__ __forceinline__ void pm_transpose_in(const u32 buf, const u32 lo, const u32 hi) {\n"
       "  #pragma unroll " << std::max(1, o.tr_unroll) << "\n";
  if (W == 8)
  s << R"CUDA(  for (u32 i = lo; i < hi; i++) {
    const u32 a0 = buf + i * 1024u, a1 = a0 + 512u;
    const uint4 a = pm_lds(a0), b = pm_lds(a1);
    u32 w0 = a.x, w1 = a.y, w2 = a.z, w3 = a.w, w4 = b.x, w5 = b.y, w6 = b.z, w7 = b.w;
    pm_tr8(w0, w1, w2, w3, w4, w5, w6, w7);
    pm_sts(a0, w0, w1, w2, w3);
    pm_sts(a1, w4, w5, w6, w7);
  }
}
)CUDA";
  else
  s << R"CUDA(  for (u32 i = lo; i < hi; i++) {
    const u32 a0 = buf + i * 2048u;
    u32 w[16];
    #pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint4 v = pm_lds(a0 + 512u * q);
      w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
    pm_tr16(w);
    #pragma unroll
    for (int q = 0; q < 4; q++) pm_sts(a0 + 512u * q, w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
  }
}
)CUDA";

  static const char *comp[4] = {"x", "y", "z", "w"};
  // ---- prefetch code for a stage (static block list; runtime stripe tt, chunk qq, buffer bb) ----
  auto emit_issue = [&](std::ostringstream &o2, int sid, const std::string &gi, const std::string &valid,
                        const std::string &bb, const std::string &ind) {
    const Stage &sg = stages[sid];
    const int n = (int)sg.blocks.size();
    o2 << ind << "{ const u32 gq = " << gi << ";\n";
    o2 << ind << "  const u64 tt = pm_udiv(gq, dv_m, dv_s1, dv_s2);\n";
    o2 << ind << "  const u64 qo = (u64)(gq - (u32)tt * chunks) * " << CB << "u + lane * 16u;\n";
    o2 << ind << "  const bool okq = " << valid << ";\n";
    if (NSEG == 2)
      o2 << ind << "  const u32 z0 = (okq && qo < S) ? 16u : 0u, z1 = (okq && qo + 512u < S) ? 16u : 0u;\n";
    else
      for (int g4 = 0; g4 < NSEG; g4++)
        o2 << ind << "  const u32 z" << g4 << " = (okq && qo + " << 512 * g4 << "u < S) ? 16u : 0u;\n";
    o2 << ind << "  const u32 dst = sbuf + (" << bb << ") * (PM_QMAX * " << CB << "u) + lane * 16u;\n";
    o2 << ind << "  switch (rank) {\n";
    for (int rk = 0; rk < (WS ? NP : T); rk++) {
      const int lo = tsplit[sid][rk], hi = tsplit[sid][rk + 1];
      o2 << ind << "  case " << rk << ": {\n";
      std::map<int, bool> slots;
      for (int i = lo; i < hi; i++) slots[sg.blocks[i].first] = true;
      for (auto &kv : slots)
        o2 << ind << "    const u64 sb" << kv.first << " = R.ptr[" << kv.first << "] + tt * R.stride[" << kv.first
           << "] + qo;\n";
      for (int i = lo; i < hi; i++) {
        const auto &bk = sg.blocks[i];
        o2 << ind << "    { const u64 a = sb" << bk.first << " + (u64)" << bk.second << "u * S;\n";
        // src_size 0 (chunk beyond S) zero-fills without reading the source
        const char *pol = sg.ef[i] == 1 ? "pol_ef" : (sg.ef[i] == 2 ? "pol_el" : "pol_en");
        o2 << ind << "      pm_cp16(dst + " << i * CB << "u, (const void *)a, z0, " << pol
           << ");\n";
        for (int g4 = 1; g4 < NSEG; g4++)
          o2 << ind << "      pm_cp16(dst + " << i * CB + 512 * g4 << "u, (const void *)(a + " << 512 * g4 << "u), z" << g4
             << ", " << pol << ")" << (g4 + 1 == NSEG ? "; }" : ";") << "\n";
      }
      o2 << ind << "  } break;\n";
    }
    o2 << ind << "  default: break;\n" << ind << "  }\n" << ind << "}\n";
  };

  if (o.layout == 2) {
    // layout 2: groups of unequal cost (MBR: d- and k-input groups).  The (group, chunk) work is
    // laid out group-major with an estimated cost per chunk of each group, and every CTA takes an
    // equal-cost slice: at most two groups per CTA, run one after the other (so each SM still
    // executes one group's code at a time), and all CTAs finish together.
    std::vector<long> cw(groups.size() + 1, 0);
    for (size_t g = 0; g < groups.size(); g++) {
      long ones = 0;
      for (int r : groups[g].rows)
        for (int c : groups[g].cols)
          if (const uint32_t cf = p.coef(r, c)) {
            uint32_t br[16];
            coef_rows_w(W, cf, br);
            for (int b = 0; b < W; b++) ones += __builtin_popcount(br[b]);
          }
      long nblk = 0;
      for (int c : groups[g].cols) nblk += (long)p.inputs[c].terms.size();
      // per-chunk cost: transposes (48 instructions per block), XOR work, fixed per-item overhead
      const long w = 6L * W * (nblk + (long)groups[g].rows.size()) + (3 * ones) / 10 + 300;
      cw[g + 1] = cw[g] + w;
    }
    s << "__constant__ unsigned int pm_cw[" << cw.size() << "] = {";
    for (size_t g = 0; g < cw.size(); g++) s << (g ? ", " : "") << cw[g] << "u";
    s << "};\n";
  }
  const int TPB = 32 * std::max(T, o.warps);
  const int teams = TPB / 32 / T;
  // dynamic chunk schedule (layout 1): teams take their next chunk from a per-group counter
  const bool DYN = o.dyn > 0 && o.layout == 1 && !WS && o.pace_lag == 0 && o.cta_sync == 0;
  const bool HYB = DYN && o.dyn >= 2 && groups.size() > 1 && o.dyn_static > 0;  // static ranges + pool
  // layout 0 with dynamic tiles: a CTA takes its next tile of teams x chunk_loop chunks from a counter
  const bool DYN0 = o.dyn > 0 && o.layout == 0 && o.sync_groups;
  s << "extern \"C\" __global__ void __launch_bounds__(" << TPB << ", 1) pmrc_kernel(const __grid_constant__ Slots R, "
       "const u64 S, const u32 stripes, const u32 chunks, u64 *__restrict__ pace, const u32 epoch"
    << ((DYN || DYN0) ? ", u32 *__restrict__ dyn" : "") << ") {\n";
  s << "  extern __shared__ __align__(1024) unsigned char pm_smem[];\n";
  if (o.pdl > 0) {
    // programmatic dependent launch: let the next launch's CTAs be scheduled as this kernel's CTAs
    // retire; pdl = 1 also waits for the preceding kernel's memory before touching global memory
    s << "  asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");\n";
    if (o.pdl == 1) s << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
  }
  s << "  const u32 lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, team = warp / PM_T, rank = warp - team * PM_T;\n";
  s << "  u32 dv_m, dv_s1, dv_s2;\n  pm_udiv_setup(chunks, dv_m, dv_s1, dv_s2);\n";
  int first_sid = -1;
  for (size_t g = 0; g < groups.size() && first_sid < 0; g++)
    if (!gstages[g].empty()) first_sid = gstages[g][0];
  // the work of one (group, chunk) item: per stage wait -> transpose -> team sync -> prefetch(g, sj)
  // -> XOR network; then transpose back and store.  Needs gi, t, q, o0, o1, v0, v1 in scope.
  auto emit_body = [&](size_t g, const std::function<void(size_t, size_t)> &prefetch) {
    const Group &G = groups[g];
    const int mall = (int)G.rows.size();
    s << "      switch (rank) {\n";
    for (int rk = 0; rk < T; rk++) {
      const int r0 = WS ? (rk < NP ? 0 : mall * (rk - NP) / (T - NP)) : mall * rk / T;
      const int r1 = WS ? (rk < NP ? 0 : mall * (rk - NP + 1) / (T - NP)) : mall * (rk + 1) / T;
      const int m = r1 - r0;
      s << "      case " << rk << ": {\n";
      std::vector<std::string> outs;
      for (int r = 0; r < m; r++)
        for (int b = 0; b < W; b++) outs.push_back("o" + std::to_string(r) + "_" + std::to_string(b));
      if (!outs.empty()) {
        s << "        u32 ";
        for (size_t i = 0; i < outs.size(); i++) s << (i ? ", " : "") << outs[i];
        s << ";\n";
      }
      if (gstages[g].empty())
        for (auto &nn : outs) s << "        " << nn << " = 0u;\n";
      bool first = true;
      for (size_t sj = 0; sj < gstages[g].size(); sj++) {
        const int si = gstages[g][sj];
        const Stage &sg = stages[si];
        const int nblk = (int)sg.blocks.size();
        s << "        {\n";
        if (WS) {
          s << "          const u32 buf = sbuf + pb * (PM_QMAX * " << CB << "u);\n";
          if (rk < NP) {
            // producer: data landed -> transpose its share of the blocks -> FULL; wait until the
            // consumers released the other buffer (EMPTY) before loading the successor stage
            s << "          pm_cp_wait<0>();\n";
            s << "          pm_transpose_in(buf + lane * 16u, " << tsplit[si][rk] << "u, " << tsplit[si][rk + 1] << "u);\n";
            s << "          pm_team_arrive(4u * team + pb, PM_T * 32u);\n";
            s << "          if (kk != 0u" << (sj ? " || true" : "") << ") pm_team_sync(4u * team + 2u + (pb ^ 1u), PM_T * 32u);\n";
            prefetch(g, sj);
            s << "          pm_cp_commit();\n";
          } else {
            s << "          pm_team_sync(4u * team + pb, PM_T * 32u);\n";
            s << "          const u32 pl = buf + lane * 16u;\n";
          }
        } else {
        // consume: own copies landed -> transpose own share -> team barrier
        s << "          pm_cp_wait<" << (D - 1) << ">();\n";
        s << "          const u32 buf = sbuf + pb * (PM_QMAX * " << CB << "u);\n";
        s << "          pm_transpose_in(buf + lane * 16u, " << tsplit[si][rk] << "u, " << tsplit[si][rk + 1] << "u);\n";
        s << "          const u32 pl = buf + lane * 16u;\n";
        }
        // the team barrier + the prefetch of the successor stage into the other buffer; emitted
        // after the sub-networks that read only this warp's own transposed blocks (below)
        auto emit_sync = [&]() {
          if (WS) return;  // producer / consumer barriers instead
          s << "          " << (T > 1 ? "pm_team_sync(1u + team, PM_T * 32u);" : "__syncwarp();") << "\n";
          prefetch(g, sj);
          s << "          pm_cp_commit();\n";
        };
        if (m == 0) emit_sync();
        if (m > 0) {
          std::vector<std::string> base;
          std::vector<char> used_half(NSEG * nblk, 0);
          std::ostringstream body;
          for (size_t ci = 0; ci < sg.cols.size(); ci++) {
            const InputDesc &in = p.inputs[sg.cols[ci]];
            const int fb = sg.first_block[ci];
            if (is_plain(in)) {
              for (int b = 0; b < W; b++) base.push_back("P" + std::to_string(NSEG * fb + b / 4) + "." + comp[b % 4]);
              continue;
            }
            std::string nm = "d" + std::to_string(ci);
            std::vector<std::string> dbase;
            std::vector<std::vector<int>> drows(W);
            for (size_t u = 0; u < in.terms.size(); u++) {
              const int bi = fb + (int)u;
              uint32_t br[16];
              coef_rows_w(W, in.terms[u].coef, br);
              for (int bb = 0; bb < W; bb++) {
                dbase.push_back("P" + std::to_string(NSEG * bi + bb / 4) + "." + comp[bb % 4]);
                for (int bp = 0; bp < W; bp++)
                  if ((br[bb] >> bp) & 1) drows[bb].push_back((int)u * W + bp);
              }
            }
            Slp ds = make_slp((int)dbase.size(), drows, o.cse, o.cse_restarts);
            if (rk == 0) {
              st.xor2 += ds.xor2();
              st.naive_lop3 += naive_lop3(drows);
              st.xor2_naive += make_slp((int)dbase.size(), drows, false).xor2();
            }
            body << "          u32 ";
            for (int bb = 0; bb < W; bb++) body << (bb ? ", " : "") << nm << "_" << bb;
            body << ";\n";
            std::vector<std::string> dout;
            for (int bb = 0; bb < W; bb++) dout.push_back(nm + "_" + std::to_string(bb));
            emit_slp(body, ds, dbase, dout, false, nm + "t");
            for (size_t u = 0; u < in.terms.size(); u++)
              for (int g4 = 0; g4 < NSEG; g4++) used_half[NSEG * (fb + u) + g4] = 1;
            for (int b = 0; b < W; b++) base.push_back(nm + "_" + std::to_string(b));
          }
          std::vector<std::vector<int>> rows(W * m);
          for (int r = 0; r < m; r++)
            for (size_t ci = 0; ci < sg.cols.size(); ci++) {
              const uint32_t cf = p.coef(G.rows[r0 + r], sg.cols[ci]);
              if (!cf) continue;
              uint32_t br[16];
              coef_rows_w(W, cf, br);
              for (int b = 0; b < W; b++)
                for (int bp = 0; bp < W; bp++)
                  if ((br[b] >> bp) & 1) rows[r * W + b].push_back((int)ci * W + bp);
            }
          // the stage's network, optionally cut into sub-networks over net_in inputs each (CSE
          // within a sub-network only): temps and plane quads then die at sub-network boundaries,
          // which bounds register pressure for wide plans (decode) at the price of some sharing
          const int ncols = (int)sg.cols.size();
          // equal-sized sub-networks of at most net_in inputs (14 -> 7 + 7, 8 -> 4 + 4, not 7 + 1)
          // (net_in counts GF(2^8) inputs: a GF(2^16) input has twice the planes)
          int sub = o.net_in > 0 ? (W == 16 ? (o.net_in + 1) / 2 : o.net_in) : ncols;
          if (o.net_even && sub < ncols) {
            const int nsub = (ncols + sub - 1) / sub;
            sub = (ncols + nsub - 1) / nsub;
          }
          std::vector<Slp> subs;
          std::vector<std::vector<std::string>> sub_base;
          for (int c0 = 0; c0 < ncols; c0 += sub) {
            const int c1 = std::min(ncols, c0 + sub);
            std::vector<std::vector<int>> sr(rows.size());
            for (size_t r = 0; r < rows.size(); r++)
              for (int x : rows[r])
                if (x >= W * c0 && x < W * c1) sr[r].push_back(x - W * c0);
            subs.push_back(make_slp(W * (c1 - c0), sr, o.cse, o.cse_restarts));
            sub_base.emplace_back(base.begin() + W * c0, base.begin() + W * c1);
            const bool acc = !(first && c0 == 0);
            st.xor2 += subs.back().xor2() + (acc ? W * m : 0);
            st.xor2_naive += make_slp(W * (c1 - c0), sr, false).xor2() + (acc ? W * m : 0);
          }
          st.naive_lop3 += naive_lop3(rows);
          // sub-networks whose inputs are all plain blocks this warp transposed itself run before
          // the team barrier (their planes are already in place), the rest after it
          const int own_lo = tsplit[si][rk], own_hi = tsplit[si][rk + 1];
          std::vector<int> order_pre, order_post;
          for (size_t si2 = 0; si2 < subs.size(); si2++) {
            bool own = T > 1 && o.own_first && !WS;
            const int cc0 = (int)si2 * sub, cc1 = std::min(ncols, cc0 + sub);
            for (int ci = cc0; ci < cc1 && own; ci++) {
              const InputDesc &in = p.inputs[sg.cols[ci]];
              const int fb = sg.first_block[ci];
              own = is_plain(in) && fb >= own_lo && fb < own_hi;
            }
            (own ? order_pre : order_post).push_back((int)si2);
          }
          std::vector<char> loaded(NSEG * nblk, 0);
          int emitted = 0;
          auto emit_sub = [&](int si2) {
            std::ostringstream net;
            auto need = [&](const std::string &nmb) {
              if (nmb[0] != 'P') return;
              int h = std::stoi(nmb.substr(1, nmb.find('.') - 1));
              if (loaded[h]) return;
              loaded[h] = 1;
              net << "          const uint4 P" << h << " = pm_lds(pl + " << (h / NSEG) * CB + (h % NSEG) * 512 << "u);\n";
            };
            const bool acc = !(first && emitted == 0);
            emitted++;
            const std::string tp = subs.size() > 1 ? "t" + std::to_string(si2) + "_" : "t";
            if (subs.size() > 1) net << "          {\n";
            if (o.fold && o.sched)
              emit_slp_sched(net, subs[si2], sub_base[si2], outs, acc, tp, need);
            else if (o.fold)
              emit_slp_fold(net, subs[si2], sub_base[si2], outs, acc, tp, need);
            else
              emit_slp_lazy(net, subs[si2], sub_base[si2], outs, acc, tp, need);
            if (subs.size() > 1) net << "          }\n";
            if (o.fence) {
              // register fence: the accumulators pass through an empty volatile asm, so ptxas
              // cannot interleave (and keep live together) the networks of consecutive stages
              for (size_t f0 = 0; f0 < outs.size(); f0 += 8) {
                net << "          asm volatile(\"\" :";
                for (size_t f = f0; f < std::min(outs.size(), f0 + 8); f++)
                  net << (f > f0 ? ", " : " ") << "\"+r\"(" << outs[f] << ")";
                net << ");\n";
              }
            }
            s << net.str();
          };
          for (int si2 : order_pre) emit_sub(si2);
          emit_sync();
          {
            // planes of derived inputs (fused repair projections) after the barrier
            std::ostringstream pre;
            for (int h = 0; h < NSEG * nblk; h++)
              if (used_half[h] && !loaded[h]) {
                loaded[h] = 1;
                pre << "          const uint4 P" << h << " = pm_lds(pl + " << (h / NSEG) * CB + (h % NSEG) * 512 << "u);\n";
              }
            s << pre.str() << body.str();
          }
          for (int si2 : order_post) emit_sub(si2);
          first = false;
        }
        if (WS && rk >= NP) s << "          pm_team_arrive(4u * team + 2u + pb, PM_T * 32u);\n";
        s << (NB == 2 ? "          pb ^= 1u;\n" : "          pb = pb + 1u == " + std::to_string(NB) + "u ? 0u : pb + 1u;\n");
        s << "        }\n";
        if (rk == 0) {
          st.loads += nblk;
          st.transposes += nblk;
        }
      }
      // transpose back and store (evict-first: parity is not re-read)
      std::map<int, bool> oslots;
      for (int r = 0; r < m; r++) oslots[p.outputs[G.rows[r0 + r]].slot] = true;
      for (auto &kv : oslots)
        s << "        const u64 ob" << kv.first << " = R.ptr[" << kv.first << "] + t * R.stride[" << kv.first << "];\n";
      for (int r = 0; r < m; r++) {
        const OutputDesc &od = p.outputs[G.rows[r0 + r]];
        std::string n = "o" + std::to_string(r);
        if (W == 8) {
        s << "        pm_tr8(" << n << "_0, " << n << "_1, " << n << "_2, " << n << "_3, " << n << "_4, " << n << "_5, "
          << n << "_6, " << n << "_7);\n";
        s << "        { unsigned char *pp = (unsigned char *)(ob" << od.slot << " + (u64)" << od.blk << "u * S);\n";
        s << "          pm_st(pp + o0, v0, " << n << "_0, " << n << "_1, " << n << "_2, " << n << "_3, pol_ef);\n";
        s << "          pm_st(pp + o1, v1, " << n << "_4, " << n << "_5, " << n << "_6, " << n << "_7, pol_ef); }\n";
        } else {
          s << "        { u32 wv[16] = {";
          for (int b = 0; b < 16; b++) s << (b ? ", " : "") << n << "_" << b;
          s << "};\n";
          s << "          pm_tr16(wv);\n";
          s << "          unsigned char *pp = (unsigned char *)(ob" << od.slot << " + (u64)" << od.blk << "u * S);\n";
          for (int q4 = 0; q4 < 4; q4++)
            s << "          pm_st(pp + o" << q4 << ", v" << q4 << ", wv[" << 4 * q4 << "], wv[" << 4 * q4 + 1 << "], wv["
              << 4 * q4 + 2 << "], wv[" << 4 * q4 + 3 << "], pol_ef);\n";
          s << "        }\n";
        }
        st.transposes++;
      }
      s << "      } break;\n";
    }
    s << "      default: break;\n      }\n";
  };
  if (o.layout == 0) {
  // layout 0: CTA b owns the contiguous global chunk range [c0, c1) (chunk index t * chunks + q
  // across stripes), processed in steps of teams x chunk_loop chunks, all groups in turn; a step's
  // chunks are split evenly over the teams, so the last (short) step costs ~1 chunk, not a tile.
  s << "  const u32 teams = " << teams << "u, per = " << teams << "u * " << M << "u;\n";
  s << "  const u32 total = stripes * chunks;\n";
  if (DYN0) {
    // tiles of `per` chunks: CTA b starts with tile b, then takes gridDim.x + atomicAdd (thread 0,
    // one tile ahead, published through shared memory behind a CTA barrier)
    s << "  const u32 ntiles = (total + per - 1u) / per;\n";
    s << "  __shared__ u32 pm_nt[2];\n";
    s << "  u32 tile = blockIdx.x, nxt_tile = threadIdx.x == 0u ? gridDim.x + atomicAdd(dyn, 1u) : 0u;\n";
    s << "  const u32 c0 = min(total, tile * per), c1 = min(total, c0 + per);\n";
  } else {
  s << "  const u32 per_cta = (total + gridDim.x - 1u) / gridDim.x;\n";
  s << "  const u32 c0 = blockIdx.x * per_cta, c1 = min(total, c0 + per_cta);\n";
  }
  s << "  const u32 sbuf = pm_saddr(pm_smem) + team * (" << NB << "u * PM_QMAX * " << CB << "u);\n";
  s << "  const u64 pol_ef = pm_policy_ef(), pol_en = pm_policy_en(), pol_el = pm_policy_el();\n";
  s << "  u32 pb = 0u;\n";
  if (first_sid >= 0) {
    s << "  if (c0 < c1) {\n";
    s << "    const u32 n0 = min(per, c1 - c0), mt0 = (n0 + teams - 1u) / teams;\n";
    emit_issue(s, first_sid, "c0 + team * mt0", "team * mt0 < n0", "0u", "    ");
    s << "  }\n";
  }
  s << "  pm_cp_commit();\n";
  if (DYN0) {
    s << "  for (u32 it = 0; tile < ntiles; it++) {\n";
    s << "    const u32 base = tile * per;\n";
    s << "    const u32 n = min(per, total - base), mt = (n + teams - 1u) / teams;\n";
    s << "    const u32 tb = base + team * mt;\n";
    s << "    const u32 cnt = team * mt < n ? min(mt, n - team * mt) : 0u;\n";
    s << "    if (threadIdx.x == 0u) { pm_nt[it & 1u] = nxt_tile; nxt_tile = gridDim.x + atomicAdd(dyn, 1u); }\n";
    s << "    __syncthreads();\n";
    s << "    const u32 ntile = pm_nt[it & 1u];\n";
    s << "    const u32 nbase = ntile * per;\n";
    s << "    const u32 nn = ntile < ntiles ? min(per, total - nbase) : 0u, nmt = (nn + teams - 1u) / teams;\n";
  } else {
  s << "  for (u32 base = c0; base < c1; base += per) {\n";
  s << "    const u32 n = min(per, c1 - base), mt = (n + teams - 1u) / teams;\n";
  s << "    const u32 tb = base + team * mt;\n";
  s << "    const u32 cnt = team * mt < n ? min(mt, n - team * mt) : 0u;\n";
  s << "    const u32 nbase = base + per;\n";
  s << "    const u32 nn = nbase < c1 ? min(per, c1 - nbase) : 0u, nmt = (nn + teams - 1u) / teams;\n";
  }
  for (size_t g = 0; g < groups.size(); g++) {
    // successor group with stages (for the prefetch after this group's last stage at m = M-1)
    int next_g = -1;
    for (size_t g2 = g + 1; g2 < groups.size(); g2++)
      if (!gstages[g2].empty()) { next_g = (int)g2; break; }
    if (o.sync_groups) s << "    __syncthreads();\n";
    s << "    #pragma unroll 1\n";
    s << "    for (u32 m = 0; m < cnt; m++) {\n";
    s << "      const u32 gi = tb + m;\n";
    s << "      const u64 t = pm_udiv(gi, dv_m, dv_s1, dv_s2);\n";
    s << "      const u32 q = gi - (u32)t * chunks;\n";
    if (W == 8) {
      s << "      const u64 o0 = (u64)q * 1024u + lane * 16u, o1 = o0 + 512u;\n";
      s << "      const bool v0 = o0 < S, v1 = o1 < S;\n";
    } else {
      s << "      const u64 o0 = (u64)q * " << CB << "u + lane * 16u, o1 = o0 + 512u, o2 = o0 + 1024u, o3 = o0 + 1536u;\n";
      s << "      const bool v0 = o0 < S, v1 = o1 < S, v2 = o2 < S, v3 = o3 < S;\n";
    }
    emit_body(g, [&](size_t gg, size_t sj) {
      if (sj + 1 < gstages[gg].size()) {
        emit_issue(s, gstages[gg][sj + 1], "gi", "true", "pb ^ 1u", "          ");
        return;
      }
      s << "          if (m + 1u < cnt) {\n";
      emit_issue(s, gstages[gg][0], "gi + 1u", "true", "pb ^ 1u", "            ");
      s << "          } else {\n";
      if (next_g >= 0) {
        emit_issue(s, gstages[next_g][0], "tb", "true", "pb ^ 1u", "            ");
      } else if (first_sid >= 0) {
        s << "            if (team * nmt < nn) {\n";
        emit_issue(s, first_sid, "nbase + team * nmt", "true", "pb ^ 1u", "              ");
        s << "            }\n";
      }
      s << "          }\n";
    });
    s << "    }\n";
  }
  if (DYN0) {
    s << "    tile = ntile;\n  }\n";
    s << "  if (threadIdx.x == 0u) { __threadfence(); if (atomicAdd(dyn + 1, 1u) == gridDim.x - 1u) "
         "{ atomicExch(dyn, 0u); atomicExch(dyn + 1, 0u); } }\n}\n";
  } else
  s << "  }\n}\n";
  } else {
  // layout 1 (group-specialised CTAs): CTA b computes group g = b / spg only, over chunk range
  // r = b % spg of the global chunk index; the spg ranges are the same for every group, so the
  // CTAs of different groups that read a shared input block do so at about the same time (the
  // second read hits L2) and each SM only ever executes one group's code (instruction cache).
  // Teams interleave over the range (team, team + teams, ...) so all groups advance in step.
  s << "  const u32 teams = " << teams << "u;\n";
  s << "  const u32 sbuf = pm_saddr(pm_smem) + team * (" << NB << "u * PM_QMAX * " << CB << "u);\n";
  s << "  const u64 pol_ef = pm_policy_ef(), pol_en = pm_policy_en(), pol_el = pm_policy_el();\n";
  s << "  u32 pb = 0u;\n";
  s << "  bool pacing = pace != 0;\n";
  if (o.trace) s << "  const u64 tr_t0 = pm_gtime(); u64 tr_wait = 0; u32 tr_fail = 0;\n";
  if (o.layout == 2) {
    const size_t G = groups.size();
    s << "  const u32 r = 0u, spg = 1u;  // (pacing is layout-1 only)\n";
    s << "  const u64 Ct = (u64)stripes * chunks, Wt = Ct * " << "pm_cw[" << G << "];\n";
    s << "  const u64 x0 = Wt * blockIdx.x / gridDim.x, x1 = Wt * (blockIdx.x + 1u) / gridDim.x;\n";
    s << "  u32 g = 0u;\n";
    s << "  for (u32 gs = 0; gs < " << G << "u; gs++) {\n";
    s << "  const u64 s0 = Ct * pm_cw[gs], s1 = Ct * pm_cw[gs + 1u];\n";
    s << "  if (s1 <= x0 || s0 >= x1) continue;\n";
    s << "  const u64 wg = pm_cw[gs + 1u] - pm_cw[gs];\n";
    s << "  const u64 lo = (x0 > s0 ? x0 : s0) - s0, hi = (x1 < s1 ? x1 : s1) - s0;\n";
    s << "  const u32 c0 = (u32)((lo + wg - 1u) / wg), c1 = (u32)((hi + wg - 1u) / wg);\n";
    s << "  g = gs;\n  pb = 0u;\n";
  } else {
    if (DYN && o.dyn >= 2 && groups.size() > 1) {
      // steal mode runs on the full grid: the gridDim.x % G CTAs beyond G x spg start as visitors
      s << "  const u32 spg = gridDim.x / " << groups.size() << "u;\n";
      s << "  u32 g = blockIdx.x / spg, r = blockIdx.x - g * spg;\n";
      s << "  if (blockIdx.x >= " << groups.size() << "u * spg) { g = blockIdx.x - " << groups.size() << "u * spg; r = spg; }\n";
    } else
    s << "  const u32 spg = gridDim.x / " << groups.size() << "u, g = blockIdx.x / spg, r = blockIdx.x - g * spg;\n";
    s << "  const u32 total = stripes * chunks;\n";
    if (HYB) {
      // hybrid: static equal ranges over the first dyn_static / 1000 of the chunks, the rest is a pool
      // handed out by the per-group counters (the slow-TPC tail is absorbed there)
      s << "  const u32 P0 = (u32)((u64)total * " << o.dyn_static << "u / 1000u);\n";
      s << "  const u32 c0 = (u32)((u64)P0 * r / spg), c1 = (u32)((u64)P0 * (r + 1u) / spg);\n";
    } else
    s << "  const u32 c0 = (u32)((u64)total * r / spg), c1 = (u32)((u64)total * (r + 1u) / spg);\n";
    if (DYN) s << "  __shared__ u32 pm_nx[" << 4 * teams << "];\n";
  }
  // dyn = 2 (steal): a team whose group has no chunks left goes on to the other groups' counters
  const bool STEAL = DYN && o.dyn >= 2 && groups.size() > 1;
  if (STEAL)
    s << "  for (u32 hop = 0; hop < " << groups.size() << "u; hop++) {\n"
      << "  const u32 gh = g + hop < " << groups.size() << "u ? g + hop : g + hop - " << groups.size() << "u;\n"
      << "  switch (gh) {\n";
  else
  s << "  switch (g) {\n";
  for (size_t g = 0; g < groups.size(); g++) {
    s << "  case " << g << ": {\n";
    if (DYN) {
      // team tau = r * teams + team of the group's NT teams starts at chunk tau; every further
      // chunk comes from the group's counter (NT + atomicAdd), taken by rank 0 at the start of an
      // item and passed to the team through shared memory (read after the item's first barrier)
      s << "    const u32 NT = spg * teams;\n";
      s << "    u32 *const dctr = dyn + 2u * " << g << "u;\n";
      if (HYB) {
        // own group: the static range first (sn = next static chunk), then the pool; other groups
        // (hop != 0) and the visitor CTAs: the pool only.  First chunk: static, else from the
        // counter, broadcast through the team barrier (slots double-buffered by hop)
        s << "    pb = 0u;\n";
        s << "    const u32 cl = hop == 0u ? c1 : 0u;\n";
        s << "    u32 sn = c0 + team, tau;\n";
        s << "    if (sn < cl) { tau = sn; sn += teams; } else {\n";
        s << "      const u32 hs = 2u * teams + 2u * team + (hop & 1u);\n";
        s << "      if (rank == 0u && lane == 0u) pm_nx[hs] = P0 + atomicAdd(dctr, 1u);\n";
        s << "      " << (T > 1 ? "pm_team_sync(1u + team, PM_T * 32u);" : "__syncwarp();") << "\n";
        s << "      tau = pm_nx[hs];\n";
        s << "    }\n";
      } else if (STEAL) {
        // a visiting team starts from the counter too (broadcast through the team barrier, which
        // also keeps the team's last buffer from being overwritten while a rank still reads it)
        s << "    pb = 0u;\n";
        s << "    u32 tau = r * teams + team;\n";
        s << "    if (hop != 0u || r >= spg) {\n";
        // (own slots, double-buffered by hop: a rank may still read the loop slots or the previous
        // hop's slot when rank 0 gets here)
        s << "      const u32 hs = 2u * teams + 2u * team + (hop & 1u);\n";
        s << "      if (rank == 0u && lane == 0u) pm_nx[hs] = NT + atomicAdd(dctr, 1u);\n";
        s << "      " << (T > 1 ? "pm_team_sync(1u + team, PM_T * 32u);" : "__syncwarp();") << "\n";
        s << "      tau = pm_nx[hs];\n";
        s << "    }\n";
      } else
        s << "    const u32 tau = r * teams + team;\n";
      // the first D stages of the first item (D <= the group's stage count, see NB)
      for (int pp = 0; pp < D; pp++) {
        if (pp < (int)gstages[g].size()) {
          s << "    if (tau < total) {\n";
          emit_issue(s, gstages[g][pp], "tau", "true", std::to_string(pp) + "u", "      ");
          s << "    }\n";
        }
        s << "    pm_cp_commit();\n";
      }
    } else {
      const int ns = (int)gstages[g].size();
      for (int pp = 0; pp < D; pp++) {
        if (ns) {
          const int di = pp / ns, sid = gstages[g][pp % ns];
          const std::string it = "c0 + team + " + std::to_string(di) + "u * teams";
          s << "    if (" << it << " < c1) {\n";
          emit_issue(s, sid, it, "true", std::to_string(pp % NB) + "u", "      ");
          s << "    }\n";
        }
        s << "    pm_cp_commit();\n";
      }
    }
    s << "    #pragma unroll 1\n";
    const bool csync = o.cta_sync > 0 && o.layout == 1 && !WS;
    if (csync) {
      // every team runs the same number of iterations (the last one possibly idle) so that the
      // CTA barrier at the top of each item is reached by all warps
      s << "    for (u32 gb = c0, kk = 0; gb < c1; gb += teams, kk++) {\n";
      s << "      const u32 gi = gb + team;\n";
      s << "      __syncthreads();\n";
      s << "      if (gi >= c1) continue;\n";
    } else if (DYN) {
      // rank 0 takes its counter value one item ahead (the atomic's L2 round trip overlaps a whole
      // item): item kk publishes the value taken during item kk - 1
      const std::string take = HYB ? "(sn < cl ? (sn += teams) - teams : P0 + atomicAdd(dctr, 1u))"
                                   : "NT + atomicAdd(dctr, 1u)";
      s << "    u32 nxt = (rank == 0u && lane == 0u) ? " << take << " : 0u;\n";
      s << "    for (u32 gi = tau, kk = 0; gi < total; kk++) {\n";
      s << "      if (rank == 0u && lane == 0u) { pm_nx[2u * team + (kk & 1u)] = nxt; nxt = " << take << "; }\n";
    } else
    s << "    for (u32 gi = c0 + team, kk = 0; gi < c1; gi += teams, kk++) {\n";
    const int pace_lag = o.layout == 1 ? o.pace_lag : 0;  // pacing assumes aligned (layout 1) ranges
    const bool pace_async = pace_lag > 0 && groups.size() <= 32;
    if (pace_lag > 0) {
      // stay within pace_lag chunks of the slowest CTA of the same range (all groups).  Only rank 0
      // paces (rank 1 meets it at the team barrier).  The peers' counters for the next iteration
      // are loaded here and tested after this iteration's work, so the L2 round trip (several us
      // under full HBM load) overlaps the XOR network instead of stalling the team.
      if (o.trace)
        s << "      if (r == 0u && team == 0u && rank == 0u && lane == 0u && kk < 256u) pace[5u * 4096u + g * 256u + kk] = pm_gtime();\n";
      if (pace_async) {
        s << "      u64 pv = ~0ull;\n";
        s << "      if (pacing && rank == 0u && lane < " << groups.size() << "u)\n";
        s << "        asm volatile(\"ld.relaxed.gpu.global.u64 %0, [%1];\" : \"=l\"(pv) : \"l\"(pace + (r + lane * spg) * teams + team));\n";
      } else {
        s << "      if (pacing && rank == 0u && kk > " << pace_lag << "u) {\n";
        if (o.trace) s << "        const u64 tw = pm_gtime();\n";
        s << "        pacing = pm_pace(pace + r * teams + team, spg * teams, " << groups.size()
          << "u, ((u64)epoch << 32) | (kk - " << pace_lag << "u), lane);\n";
        if (o.trace) s << "        tr_wait += pm_gtime() - tw; tr_fail += pacing ? 0u : 1u;\n";
        s << "      }\n";
      }
    }
    s << "      const u64 t = pm_udiv(gi, dv_m, dv_s1, dv_s2);\n";
    s << "      const u32 q = gi - (u32)t * chunks;\n";
    if (W == 8) {
      s << "      const u64 o0 = (u64)q * 1024u + lane * 16u, o1 = o0 + 512u;\n";
      s << "      const bool v0 = o0 < S, v1 = o1 < S;\n";
    } else {
      s << "      const u64 o0 = (u64)q * " << CB << "u + lane * 16u, o1 = o0 + 512u, o2 = o0 + 1024u, o3 = o0 + 1536u;\n";
      s << "      const bool v0 = o0 < S, v1 = o1 < S, v2 = o2 < S, v3 = o3 < S;\n";
    }
    emit_body(g, [&](size_t gg, size_t sj) {
      const int ns = (int)gstages[gg].size();
      const int di = ((int)sj + D) / ns, sid = gstages[gg][((int)sj + D) % ns];
      const std::string bb = NB == 2 ? std::string("pb ^ 1u")
                                     : "(pb + " + std::to_string(D) + "u) % " + std::to_string(NB) + "u";
      if (di == 0) {
        emit_issue(s, sid, "gi", "true", bb, "          ");
        return;
      }
      if (DYN) {
        s << "          { const u32 nx = pm_nx[2u * team + (kk & 1u)];\n";
        s << "          if (nx < total) {\n";
        emit_issue(s, sid, "nx", "true", bb, "            ");
        s << "          } }\n";
        return;
      }
      const std::string it = "gi + " + std::to_string(di) + "u * teams";
      s << "          if (" << it << " < c1) {\n";
      emit_issue(s, sid, it, "true", bb, "            ");
      s << "          }\n";
    });
    if (DYN) s << "      gi = pm_nx[2u * team + (kk & 1u)];\n";
    if (pace_lag > 0)
      s << "      if (pace && rank == 0u && lane == 0u) pm_pace_post(pace + blockIdx.x * teams + team, ((u64)epoch << 32) | (kk + 1u));\n";
    if (pace_async) {
      s << "      if (pacing && rank == 0u && kk + 1u > " << pace_lag << "u) {\n";
      s << "        const u64 want = ((u64)epoch << 32) | (kk + 1u - " << pace_lag << "u);\n";
      s << "        if (!__all_sync(0xffffffffu, pv >= want)) {\n";
      if (o.trace) s << "          const u64 tw = pm_gtime();\n";
      s << "          pacing = pm_pace(pace + r * teams + team, spg * teams, " << groups.size() << "u, want, lane);\n";
      if (o.trace) s << "          tr_wait += pm_gtime() - tw; tr_fail += pacing ? 0u : 1u;\n";
      s << "        }\n      }\n";
    }
    s << "    }\n";
    if (DYN)  // the group's last team to finish resets its counters for a later launch (slot ring)
      s << "    if (rank == 0u && lane == 0u) { __threadfence(); if (atomicAdd(dctr + 1, 1u) == "
        << (STEAL ? "gridDim.x * teams" : "NT") << " - 1u) { atomicExch(dctr, 0u); atomicExch(dctr + 1, 0u); } }\n";
    if (WS)  // balance the last EMPTY arrival of the consumers (the producer's final wait)
      s << "    if (rank < " << NP << "u && c0 + team < c1) pm_team_sync(4u * team + 2u + (pb ^ 1u), PM_T * 32u);\n";
    s << "  } break;\n";
  }
  s << "  default: break;\n  }\n";
  if (STEAL) s << "  }\n";  // hop loop
  if (o.layout == 2) s << "  }\n";  // segment loop
  if (o.trace) {
    // diagnostics (E = 4096 entries per field, plan.cpp): [E + i] start, [2E + i] end (globaltimer ns),
    // [3E + i] ns spent pacing, [4E + i] = smid << 48 | group << 32 | pacing timeouts
    s << "  if (pace && rank == 0u && lane == 0u) {\n";
    s << "    const u32 E = 4096u, i = blockIdx.x * teams + team;\n";
    s << "    pace[E + i] = tr_t0; pace[2u * E + i] = pm_gtime(); pace[3u * E + i] = tr_wait; u32 smid; asm volatile(\"mov.u32 %0, %%smid;\" : \"=r\"(smid)); pace[4u * E + i] = ((u64)smid << 48) | ((u64)g << 32) | tr_fail;\n";
    s << "  }\n";
  }
  s << "}\n";
  }
  st.smem_per_warp = (NB * qmax * CB + T - 1) / T;
  for (auto &gs : gstages) st.max_stages = std::max(st.max_stages, (int)gs.size());
  return s.str();
}

}  // namespace pmrc
