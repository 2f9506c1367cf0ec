#include "construct.hpp"

#include "../../../include/pmrc.h"

namespace pmrc {

int CodeDef::sys_block(int i, int j) const {
  if (kind == KIND_MBR) return Lidx[(size_t)i * Lcols + j] - 1;
  return i * alpha + j;
}

namespace {

// index matrix: symmetric blocks numbered row-major over the upper triangle (R4)
void number_symmetric(std::vector<int> &L, int cols, int r0, int c0, int m, int &next) {
  for (int a = 0; a < m; a++)
    for (int b = a; b < m; b++) {
      L[(size_t)(r0 + a) * cols + c0 + b] = next;
      L[(size_t)(r0 + b) * cols + c0 + a] = next;
      next++;
    }
}

// C(n, r) capped
double n_choose(int n, int r) {
  double v = 1;
  for (int i = 0; i < r; i++) v = v * (n - i) / (i + 1);
  return v;
}

bool all_subsets_full_rank(const Mat &psi, int rsel, int cols) {
  int n = psi.r;
  std::vector<int> c(rsel);
  for (int i = 0; i < rsel; i++) c[i] = i;
  Mat M(rsel, cols);
  for (;;) {
    for (int a = 0; a < rsel; a++)
      for (int t = 0; t < cols; t++) M.at(a, t) = psi.at(c[a], t);
    if (rank(M) < rsel) return false;
    int i = rsel - 1;
    while (i >= 0 && c[i] == n - rsel + i) i--;
    if (i < 0) return true;
    c[i]++;
    for (int j = i + 1; j < rsel; j++) c[j] = c[j - 1] + 1;
  }
}

// Extension (not the paper's, R10b): the sparse Phi = [I; Cauchy] with
// Lambda chosen greedily so that Psi stays valid at n = 2k: for nodes i = 0..n-1 in order,
// lambda_i = g^e with the smallest e >= 0 such that lambda_i differs from the earlier lambdas and
// every d-row subset of rows 0..i that contains row i has full rank.  Returns false if no e works.
bool greedy_lambda(const Mat &phi, int n, int a, int d, Mat &psi, std::vector<uint8_t> &lambda) {
  const GF256 &F = gf();
  psi = Mat(n, d);
  lambda.assign(n, 0);
  Mat M(d, d);
  for (int i = 0; i < n; i++) {
    bool placed = false;
    for (int e = 0; e < 255 && !placed; e++) {
      const uint8_t lam = F.gexp(e);
      bool clash = false;
      for (int j = 0; j < i; j++) clash |= lambda[j] == lam;
      if (clash) continue;
      for (int t = 0; t < a; t++) {
        psi.at(i, t) = phi.at(i, t);
        psi.at(i, a + t) = F.mul(lam, phi.at(i, t));
      }
      bool ok = true;
      if (i + 1 >= d) {
        // subsets = row i plus every (d-1)-subset of rows 0..i-1
        std::vector<int> c(d - 1);
        for (int q = 0; q < d - 1; q++) c[q] = q;
        for (;;) {
          for (int q = 0; q < d - 1; q++)
            for (int t = 0; t < d; t++) M.at(q, t) = psi.at(c[q], t);
          for (int t = 0; t < d; t++) M.at(d - 1, t) = psi.at(i, t);
          if (rank(M) < d) { ok = false; break; }
          int q = d - 2;
          while (q >= 0 && c[q] == i - (d - 1) + q) q--;
          if (q < 0) break;
          c[q]++;
          for (int r = q + 1; r < d - 1; r++) c[r] = c[r - 1] + 1;
        }
      }
      if (ok) {
        lambda[i] = lam;
        placed = true;
      }
    }
    if (!placed) return false;
  }
  return true;
}

}  // namespace

int build_code(int kind, int k, int d, int n, int w, CodeDef &o, std::string &err) {
  const GF256 &F = gf();
  if (w != 8) { err = "only w = 8 (GF(2^8)) is supported"; return PMRC_EUNSUPPORTED; }
  if (k < 1 || n < 2 || n > 255) { err = "bad n/k"; return PMRC_EINVAL; }
  o = CodeDef();
  o.kind = kind; o.n = n; o.k = k;
  switch (kind) {
    case KIND_MSR_SPARSE:
    case KIND_MSR_VANILLA:
    case KIND_MSR_SPARSE_N2K:
      // alpha = Delta = d - k + 1; PM-MSR needs d = 2k - 2 (R7)
      if (k < 2 || d != 2 * k - 2) { err = "MSR requires k >= 2 and d = 2k-2"; return PMRC_EUNSUPPORTED; }
      if (n <= d) { err = "MSR requires n > d"; return PMRC_EINVAL; }
      o.d = d; o.alpha = k - 1; o.B = k * o.alpha;
      break;
    case KIND_MBR:
      // alpha = d, Delta = (2d - k + 1)/2
      if (k < 2 || d < k || n <= d) { err = "MBR requires 2 <= k <= d < n"; return PMRC_EINVAL; }
      o.d = d; o.alpha = d; o.B = k * (2 * d - k + 1) / 2;
      break;
    case KIND_RS:
      if (n <= k) { err = "RS requires n > k"; return PMRC_EINVAL; }
      o.d = k; o.alpha = 1; o.B = k;
      break;
    default: err = "unknown kind"; return PMRC_EINVAL;
  }
  const int a = o.alpha;
  o.P = (n - k) * a;

  // ---- Psi (and lambda) ----
  if (kind == KIND_RS) {
    o.psi = Mat(n, k);  // R12: V_ij = g^{(i-1)(j-1)}
    for (int i = 0; i < n; i++)
      for (int j = 0; j < k; j++) o.psi.at(i, j) = F.gexp((long)i * j);
  } else {
    o.psi = Mat(n, o.d);
    o.lambda.assign(n, 0);
    if (kind == KIND_MSR_VANILLA) {
      // Phi_ij = g^{(i-1)(j-1)}, Lambda_ii = g^{(i-1) alpha}, Psi = [Phi  Lambda Phi]
      for (int i = 0; i < n; i++) {
        o.lambda[i] = F.gexp((long)i * a);
        for (int j = 0; j < a; j++) {
          uint8_t phi = F.gexp((long)i * j);
          o.psi.at(i, j) = phi;
          o.psi.at(i, a + j) = F.mul(o.lambda[i], phi);
        }
      }
      for (int i = 0; i < n; i++)
        for (int i2 = 0; i2 < i; i2++)
          if (o.lambda[i] == o.lambda[i2]) {
            err = "vanilla MSR: Lambda values collide (n > 255/gcd(alpha,255), R8)";
            return PMRC_EUNSUPPORTED;
          }
    } else if (kind == KIND_MSR_SPARSE_N2K) {
      // extension: the paper's sparse Phi, greedy Lambda valid at n = 2k (greedy_lambda above)
      if (n + a > 254) { err = "sparse MSR needs n + alpha <= 254 in GF(2^8)"; return PMRC_EUNSUPPORTED; }
      if (n - 1 > 40) { err = "n=2k-valid sparse MSR: greedy Lambda search limited to n <= 41"; return PMRC_EUNSUPPORTED; }
      Mat phi(n, a);
      for (int i = 0; i < n; i++) {
        uint8_t x = F.gexp(i + 1 + a);
        for (int j = 0; j < a; j++) phi.at(i, j) = (i < a) ? (uint8_t)(i == j) : F.inv(x ^ F.gexp(j));
      }
      if (!greedy_lambda(phi, n, a, o.d, o.psi, o.lambda)) {
        err = "n=2k-valid sparse MSR: no Lambda keeps every d-row subset invertible";
        return PMRC_EUNSUPPORTED;
      }
    } else if (kind == KIND_MSR_SPARSE) {
      // x_i = g^{i+alpha} (1-based i, R2); Phi = [I_alpha; 1/(x_i - y_j)], y_j = g^{j-1};
      // Lambda_ii = (x_i - 1)/(x_i - g^alpha)
      if (n + a > 254) { err = "sparse MSR needs n + alpha <= 254 in GF(2^8)"; return PMRC_EUNSUPPORTED; }
      for (int i = 0; i < n; i++) {
        uint8_t x = F.gexp(i + 1 + a);
        o.lambda[i] = F.div(x ^ 1, x ^ F.gexp(a));
        for (int j = 0; j < a; j++) {
          uint8_t phi = (i < a) ? (uint8_t)(i == j) : F.inv(x ^ F.gexp(j));
          o.psi.at(i, j) = phi;
          o.psi.at(i, a + j) = F.mul(o.lambda[i], phi);
        }
      }
      for (int i = 0; i < n; i++)
        for (int i2 = 0; i2 < i; i2++)
          if (o.lambda[i] == o.lambda[i2]) { err = "sparse MSR: Lambda values collide"; return PMRC_EUNSUPPORTED; }
    } else {
      // MBR (R5): rows 1..k = [I_k 0], rows i = k+1..n: 1/(g^{d+i} - g^{j-1})
      if (n + o.d > 254) { err = "MBR needs n + d <= 254 in GF(2^8)"; return PMRC_EUNSUPPORTED; }
      for (int i = 0; i < n; i++)
        for (int j = 0; j < o.d; j++)
          o.psi.at(i, j) = (i < k) ? (uint8_t)(i == j) : F.inv(F.gexp(o.d + i + 1) ^ F.gexp(j));
    }
  }

  // ---- index matrix L ----
  if (kind == KIND_RS) {
    o.Lrows = k; o.Lcols = 1;
    o.Lidx.resize(k);
    for (int i = 0; i < k; i++) o.Lidx[i] = i + 1;
  } else if (kind == KIND_MBR) {
    o.Lrows = o.d; o.Lcols = o.d;
    o.Lidx.assign((size_t)o.d * o.d, 0);
    int next = 1;
    number_symmetric(o.Lidx, o.d, 0, 0, k, next);  // S
    for (int r = 0; r < k; r++)                    // T and T^t
      for (int c = k; c < o.d; c++) {
        o.Lidx[(size_t)r * o.d + c] = next;
        o.Lidx[(size_t)c * o.d + r] = next;
        next++;
      }
  } else {
    o.Lrows = o.d; o.Lcols = a;
    o.Lidx.assign((size_t)o.d * a, 0);
    int next = 1;
    number_symmetric(o.Lidx, a, 0, 0, a, next);  // S1
    number_symmetric(o.Lidx, a, a, 0, a, next);  // S2
  }

  // ---- G: G_{alpha i + j, L_{l,j}} = Psi_{i,l} ----
  o.G = Mat(n * a, o.B);
  if (kind == KIND_RS) {
    o.G = o.psi;
  } else {
    for (int i = 0; i < n; i++)
      for (int j = 0; j < a; j++)
        for (int l = 0; l < o.d; l++) {
          int idx = o.Lidx[(size_t)l * o.Lcols + j];
          if (idx) o.G.at(i * a + j, idx - 1) = o.psi.at(i, l);
        }
  }

  // ---- G' ----
  if (kind == KIND_MBR) {
    o.Gsys = o.G;  // R6: systematic rows are unit rows already
  } else {
    Mat Gt(o.B, o.B), Gti;
    for (int r = 0; r < o.B; r++)
      for (int c2 = 0; c2 < o.B; c2++) Gt.at(r, c2) = o.G.at(r, c2);
    if (!invert(Gt, Gti)) { err = "Gtilde (first B rows of G) is singular"; return PMRC_EUNSUPPORTED; }
    o.Gsys = matmul(o.G, Gti);
    o.Gti = Gti;
  }
  o.Gpp = Mat(o.P, o.B);
  for (int r = 0; r < o.P; r++)
    for (int c2 = 0; c2 < o.B; c2++) o.Gpp.at(r, c2) = o.Gsys.at(k * a + r, c2);

  // ---- repair completeness: every d rows of Psi independent ----
  if (kind != KIND_RS) {
    if (n_choose(n, o.d) <= 20000)
      o.repair_complete = all_subsets_full_rank(o.psi, o.d, o.d);
    else
      o.repair_complete = (n == o.d + 1) ? all_subsets_full_rank(o.psi, o.d, o.d) : false;
  }
  return PMRC_OK;
}

}  // namespace pmrc

namespace pmrc {

// GF(2^16) sparse PM-MSR, systematic parity part only (P:163-187 with the field of
// reading R1b): the same Psi / L / G / G' = G Gtilde^{-1} pipeline as build_code, on 16-bit symbols.
int build_gpp16(int k, int d, int n, int &alpha, int &B, std::vector<uint16_t> &gpp, std::string &err,
                std::vector<uint16_t> *psi_out, std::vector<uint16_t> *lam_out) {
  const GF65536 &F = gf16();
  if (k < 2 || d != 2 * k - 2) { err = "MSR requires k >= 2 and d = 2k-2"; return PMRC_EUNSUPPORTED; }
  if (n <= d || n > 4096) { err = "MSR requires d < n <= 4096"; return PMRC_EINVAL; }
  const int a = k - 1;
  alpha = a;
  B = k * a;
  // Psi: x_i = g^{i+alpha} (1-based i), Phi = [I_alpha; 1/(x_i - y_j)], y_j = g^{j-1};
  // Lambda_ii = (x_i - 1)/(x_i - g^alpha)
  std::vector<uint16_t> psi((size_t)n * d), lam(n);
  for (int i = 0; i < n; i++) {
    const uint16_t x = F.gexp(i + 1 + a);
    lam[i] = F.div(x ^ 1, x ^ F.gexp(a));
    for (int j = 0; j < a; j++) {
      const uint16_t phi = (i < a) ? (uint16_t)(i == j) : F.inv(x ^ F.gexp(j));
      psi[(size_t)i * d + j] = phi;
      psi[(size_t)i * d + a + j] = F.mul(lam[i], phi);
    }
  }
  for (int i = 0; i < n; i++)
    for (int i2 = 0; i2 < i; i2++)
      if (lam[i] == lam[i2]) { err = "sparse MSR (GF(2^16)): Lambda values collide"; return PMRC_EUNSUPPORTED; }
  if (psi_out) *psi_out = psi;
  if (lam_out) *lam_out = lam;
  // L: S1 then S2, row-major over each upper triangle (R4)
  std::vector<int> L((size_t)d * a, 0);
  int next = 1;
  number_symmetric(L, a, 0, 0, a, next);
  number_symmetric(L, a, a, 0, a, next);
  // G (n alpha x B): G_{alpha i + j, L_{l,j}} = Psi_{i,l}
  std::vector<uint16_t> G((size_t)n * a * B, 0);
  for (int i = 0; i < n; i++)
    for (int j = 0; j < a; j++)
      for (int l = 0; l < d; l++) {
        const int idx = L[(size_t)l * a + j];
        if (idx) G[((size_t)i * a + j) * B + idx - 1] = psi[(size_t)i * d + l];
      }
  // Gtilde^{-1} by Gauss-Jordan
  std::vector<uint16_t> Wm(G.begin(), G.begin() + (size_t)B * B), Inv((size_t)B * B, 0);
  for (int i = 0; i < B; i++) Inv[(size_t)i * B + i] = 1;
  for (int col = 0; col < B; col++) {
    int piv = -1;
    for (int r = col; r < B; r++)
      if (Wm[(size_t)r * B + col]) { piv = r; break; }
    if (piv < 0) { err = "Gtilde singular (GF(2^16))"; return PMRC_EUNSUPPORTED; }
    if (piv != col)
      for (int c = 0; c < B; c++) {
        std::swap(Wm[(size_t)piv * B + c], Wm[(size_t)col * B + c]);
        std::swap(Inv[(size_t)piv * B + c], Inv[(size_t)col * B + c]);
      }
    const uint16_t s = F.inv(Wm[(size_t)col * B + col]);
    for (int c = 0; c < B; c++) {
      Wm[(size_t)col * B + c] = F.mul(Wm[(size_t)col * B + c], s);
      Inv[(size_t)col * B + c] = F.mul(Inv[(size_t)col * B + c], s);
    }
    for (int r = 0; r < B; r++) {
      const uint16_t f = r == col ? 0 : Wm[(size_t)r * B + col];
      if (!f) continue;
      for (int c = 0; c < B; c++) {
        Wm[(size_t)r * B + c] ^= F.mul(f, Wm[(size_t)col * B + c]);
        Inv[(size_t)r * B + c] ^= F.mul(f, Inv[(size_t)col * B + c]);
      }
    }
  }
  // G'' = (parity rows of G) Gtilde^{-1}
  const int P = (n - k) * a;
  gpp.assign((size_t)P * B, 0);
  for (int r = 0; r < P; r++)
    for (int t = 0; t < B; t++) {
      const uint16_t g = G[((size_t)k * a + r) * B + t];
      if (!g) continue;
      for (int c = 0; c < B; c++) gpp[(size_t)r * B + c] ^= F.mul(g, Inv[(size_t)t * B + c]);
    }
  return PMRC_OK;
}

}  // namespace pmrc
