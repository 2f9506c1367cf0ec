/*
 * pmrc_oracle.c — plain, slow, obviously-correct CPU oracle for the product-matrix
 * regenerating-code hot path of arxiv 1412.3022 ("Fast Product-Matrix Regenerating Codes").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke(), bench.py's cpu_baseline /
 * --impl reference legs and the sampled correctness checks of tools/sweep.py may load this library.  The product (paper_1412_3022_b200/, include/)
 * shares no code with it and never calls it.
 *
 * Citations:  P:L = /root/reference/PAPER.md line L (section), S:L = SPEC.md line L.
 * Readings of silent/ambiguous passages are numbered R1..R14 in DESIGN.md §3.
 *
 * Everything is scalar GF(2^8) arithmetic over log/antilog tables (R1: primitive polynomial
 * 0x11D, generator g = 2), byte position by byte position, in the paper's order and notation:
 *   - parameters                      P:51            (MSR alpha=Delta=d-k+1; MBR alpha=d, Delta=(2d-k+1)/2)
 *   - index matrix L                  P:75-83         (message matrix M_{i,j} = X_{L_{i,j}})
 *   - encoding matrix Psi             P:121-158 (vanilla), P:163-187 (sparse), P:115 + R5 (MBR)
 *   - linearisation G                 P:95-104        (G_{alpha i+j, L_{l,j}} = Psi_{i,l})
 *   - systematic G' = G Gtilde^-1
 *   - encode Y = G''X, zeros skipped
 *   - specific encode C = Psi M
 *   - linear (lazy) decode
 *   - specific MSR / MBR decode       S:406-423 (reconstructed; the paper defers to Rashmi2011)
 *   - exact repair                    P:53 footnote
 *   - construction validation
 * Parity of every function is pinned by tests/test_oracle_*.py against values the paper prints,
 * closed forms, cross-paths and brute force.
 *
 * Return codes: 0 ok, -1 invalid argument, -2 unsupported parameters, -3 singular.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL -1
#define OR_EUNSUP -2
#define OR_ESING -3

enum { OR_MSR_SPARSE = 0, OR_MSR_VANILLA = 1, OR_MBR = 2, OR_RS = 3, OR_MSR_N2K = 4 };
/* kind 4 is an EXTENSION, not the paper's construction (R15): the sparse Phi with a
 * Lambda chosen greedily so that the code is valid at n = 2k.  It is an MSR code in every other
 * respect (parameters, L, linearisation, decode, repair). */
#define OR_IS_MSR(kind) ((kind) == OR_MSR_SPARSE || (kind) == OR_MSR_VANILLA || (kind) == OR_MSR_N2K)

/* ------------------------------------------------------------------ GF(2^8), R1 */
static uint8_t EXPT[512];
static int LOGT[256];
static int gf_ready = 0;

void or_init(void) {
  if (gf_ready) return;
  unsigned x = 1;
  for (int e = 0; e < 255; e++) {
    EXPT[e] = (uint8_t)x;
    LOGT[x] = e;
    x <<= 1; /* multiply by g = 2 */
    if (x & 0x100) x ^= 0x11D;
  }
  for (int e = 255; e < 512; e++) EXPT[e] = EXPT[e - 255];
  LOGT[0] = -1;
  gf_ready = 1;
}

uint8_t or_gf_mul(uint8_t a, uint8_t b) {
  if (a == 0 || b == 0) return 0;
  return EXPT[LOGT[a] + LOGT[b]];
}
uint8_t or_gf_inv(uint8_t a) { return a ? EXPT[(255 - LOGT[a]) % 255] : 0; }
uint8_t or_gf_div(uint8_t a, uint8_t b) { return or_gf_mul(a, or_gf_inv(b)); }
/* g^e for any integer e >= 0 (exponent reduced mod 255) */
uint8_t or_gf_exp(long e) { return EXPT[((e % 255) + 255) % 255]; }
int or_gf_log(uint8_t a) { return LOGT[a]; }

/* ------------------------------------------------------------------ small matrices */
/* C (r x c) = A (r x m) * B (m x c), row-major */
void or_mat_mul(const uint8_t *A, const uint8_t *B, uint8_t *C, int r, int m, int c) {
  for (int i = 0; i < r; i++)
    for (int j = 0; j < c; j++) {
      uint8_t s = 0;
      for (int t = 0; t < m; t++) s ^= or_gf_mul(A[i * m + t], B[t * c + j]);
      C[i * c + j] = s;
    }
}

/* Gauss-Jordan inverse (first nonzero pivot). Returns OR_ESING if singular. */
int or_mat_inv(const uint8_t *A, uint8_t *Ainv, int m) {
  uint8_t *W = (uint8_t *)malloc((size_t)m * 2 * m);
  if (!W) return OR_EINVAL;
  for (int i = 0; i < m; i++) {
    for (int j = 0; j < m; j++) W[i * 2 * m + j] = A[i * m + j];
    for (int j = 0; j < m; j++) W[i * 2 * m + m + j] = (uint8_t)(i == j);
  }
  for (int col = 0; col < m; col++) {
    int piv = -1;
    for (int r = col; r < m; r++)
      if (W[r * 2 * m + col]) { piv = r; break; }
    if (piv < 0) { free(W); return OR_ESING; }
    if (piv != col)
      for (int j = 0; j < 2 * m; j++) {
        uint8_t t = W[col * 2 * m + j];
        W[col * 2 * m + j] = W[piv * 2 * m + j];
        W[piv * 2 * m + j] = t;
      }
    uint8_t inv = or_gf_inv(W[col * 2 * m + col]);
    for (int j = 0; j < 2 * m; j++) W[col * 2 * m + j] = or_gf_mul(W[col * 2 * m + j], inv);
    for (int r = 0; r < m; r++) {
      if (r == col) continue;
      uint8_t f = W[r * 2 * m + col];
      if (!f) continue;
      for (int j = 0; j < 2 * m; j++) W[r * 2 * m + j] ^= or_gf_mul(f, W[col * 2 * m + j]);
    }
  }
  for (int i = 0; i < m; i++)
    for (int j = 0; j < m; j++) Ainv[i * m + j] = W[i * 2 * m + m + j];
  free(W);
  return OR_OK;
}

/* row rank by elimination */
int or_mat_rank(const uint8_t *A, int r, int c) {
  uint8_t *W = (uint8_t *)malloc((size_t)r * c + 1);
  memcpy(W, A, (size_t)r * c);
  int rank = 0;
  for (int col = 0; col < c && rank < r; col++) {
    int piv = -1;
    for (int i = rank; i < r; i++)
      if (W[i * c + col]) { piv = i; break; }
    if (piv < 0) continue;
    for (int j = 0; j < c; j++) {
      uint8_t t = W[rank * c + j];
      W[rank * c + j] = W[piv * c + j];
      W[piv * c + j] = t;
    }
    uint8_t inv = or_gf_inv(W[rank * c + col]);
    for (int i = 0; i < r; i++) {
      if (i == rank || !W[i * c + col]) continue;
      uint8_t f = or_gf_mul(W[i * c + col], inv);
      for (int j = 0; j < c; j++) W[i * c + j] ^= or_gf_mul(f, W[rank * c + j]);
    }
    rank++;
  }
  free(W);
  return rank;
}

/* ------------------------------------------------------------------ parameters */
int or_params(int kind, int n, int k, int d, int *alpha, int *B) {
  if (k < 1 || n < 1) return OR_EINVAL;
  if (OR_IS_MSR(kind)) {
    /* MSR: alpha = Delta = d - k + 1; the PM construction needs d = 2k-2 (R7) */
    if (k < 2 || d != 2 * k - 2 || n <= d) return OR_EUNSUP;
    *alpha = d - k + 1;
    *B = k * (*alpha); /* B = k Delta */
    return OR_OK;
  }
  if (kind == OR_MBR) {
    /* MBR: alpha = d, Delta = (2d-k+1)/2, B = k Delta */
    if (k < 2 || d < k || n <= d) return OR_EUNSUP;
    *alpha = d;
    *B = k * (2 * d - k + 1) / 2;
    return OR_OK;
  }
  if (kind == OR_RS) {
    /* Reed-Solomon baseline: alpha = 1, B = k; d is taken equal to k (R12) */
    if (k < 1 || n <= k || n > 255) return OR_EUNSUP;
    *alpha = 1;
    *B = k;
    return OR_OK;
  }
  return OR_EINVAL;
}

/* ------------------------------------------------------------------ index matrix L */
/* L is d x alpha (MSR: [S1;S2]) or d x d (MBR: [[S,T],[T^t,0]]), 1-based data indices, 0 = zero.
 * Symmetric blocks are numbered row-major over their upper triangle (R4, reproduces P:77-83). */
int or_index_matrix(int kind, int k, int d, int *L) {
  int alpha, B;
  if (OR_IS_MSR(kind)) {
    int rc = or_params(kind, d + 1, k, d, &alpha, &B);
    if (rc) return rc;
    int v = 1;
    for (int blk = 0; blk < 2; blk++) /* S1 then S2 */
      for (int r = 0; r < alpha; r++)
        for (int c = r; c < alpha; c++) {
          L[(blk * alpha + r) * alpha + c] = v;
          L[(blk * alpha + c) * alpha + r] = v;
          v++;
        }
    return OR_OK;
  }
  if (kind == OR_MBR) {
    int rc = or_params(kind, d + 1, k, d, &alpha, &B);
    if (rc) return rc;
    memset(L, 0, sizeof(int) * d * d);
    int v = 1;
    for (int r = 0; r < k; r++) /* S: k x k symmetric */
      for (int c = r; c < k; c++) {
        L[r * d + c] = v;
        L[c * d + r] = v;
        v++;
      }
    for (int r = 0; r < k; r++) /* T: k x (d-k), and T^t below */
      for (int c = k; c < d; c++) {
        L[r * d + c] = v;
        L[c * d + r] = v;
        v++;
      }
    return OR_OK;
  }
  return OR_EINVAL;
}

/* ------------------------------------------------------------------ encoding matrix Psi */
/* psi: n x d (RS: n x k Vandermonde V), lambda: n (MSR only; may be NULL). */
int or_psi(int kind, int n, int k, int d, uint8_t *psi, uint8_t *lambda) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  if (kind == OR_MSR_VANILLA) {
    /* Phi_{i,j} = g^{(i-1)(j-1)};  P:143-148: Lambda_{i,i} = g^{(i-1) alpha};
       P:123: Psi = [Phi  Lambda Phi].  The matrix is built even when lambdas collide (R8:
       n > 255/gcd(alpha,255), e.g. Table 1's k=16 column); or_validate reports the collision. */
    if (n > 255) return OR_EUNSUP;
    for (int i = 1; i <= n; i++) {
      uint8_t lam = or_gf_exp((long)(i - 1) * alpha);
      if (lambda) lambda[i - 1] = lam;
      for (int j = 1; j <= alpha; j++) {
        uint8_t phi = or_gf_exp((long)(i - 1) * (j - 1));
        psi[(i - 1) * d + (j - 1)] = phi;
        psi[(i - 1) * d + alpha + (j - 1)] = or_gf_mul(lam, phi);
      }
    }
    return OR_OK;
  }
  if (kind == OR_MSR_SPARSE) {
    /* Phi = [I_alpha ; Cauchy], Phi_{i,j} = (g^{i+alpha} - g^{j-1})^{-1} for i > alpha;
       Lambda_{i,i} = (g^{i+alpha} - g^0) / (g^{i+alpha} - g^alpha);  Psi = [Phi  Lambda Phi].
       1-based i, j (R2, pinned by the display P:168-181).  Points must stay distinct: n+alpha <= 254. */
    if (n + alpha > 254) return OR_EUNSUP;
    for (int i = 1; i <= n; i++) {
      uint8_t xi = or_gf_exp(i + alpha);
      uint8_t lam = or_gf_div(xi ^ or_gf_exp(0), xi ^ or_gf_exp(alpha));
      if (lambda) lambda[i - 1] = lam;
      for (int j = 1; j <= alpha; j++) {
        uint8_t phi;
        if (i <= alpha)
          phi = (uint8_t)(i == j);
        else
          phi = or_gf_inv(xi ^ or_gf_exp(j - 1));
        psi[(i - 1) * d + (j - 1)] = phi;
        psi[(i - 1) * d + alpha + (j - 1)] = or_gf_mul(lam, phi);
      }
    }
    return OR_OK;
  }
  if (kind == OR_MSR_N2K) {
    /* R15 (extension): Phi as in the sparse code; for i = 1..n in order, Lambda_{i,i} =
       g^e with the smallest e >= 0 such that it differs from Lambda_{1..i-1} and every d-row
       subset of Psi's rows 1..i that contains row i has rank d. */
    if (n + alpha > 254 || n > 41) return OR_EUNSUP;
    uint8_t *lam = (uint8_t *)malloc(n), *M = (uint8_t *)malloc((size_t)d * d);
    int *c = (int *)malloc(sizeof(int) * (d > 1 ? d : 1));
    for (int i = 1; i <= n; i++) {
      uint8_t xi = or_gf_exp(i + alpha);
      int found = 0;
      for (int e = 0; e < 255 && !found; e++) {
        uint8_t l = or_gf_exp(e);
        int clash = 0;
        for (int j = 1; j < i; j++)
          if (lam[j - 1] == l) clash = 1;
        if (clash) continue;
        for (int j = 1; j <= alpha; j++) {
          uint8_t phi = (i <= alpha) ? (uint8_t)(i == j) : or_gf_inv(xi ^ or_gf_exp(j - 1));
          psi[(i - 1) * d + (j - 1)] = phi;
          psi[(i - 1) * d + alpha + (j - 1)] = or_gf_mul(l, phi);
        }
        int ok = 1;
        if (i >= d) {
          /* every choice of d-1 rows among rows 1..i-1, plus row i */
          for (int q = 0; q < d - 1; q++) c[q] = q;
          for (;;) {
            for (int q = 0; q < d - 1; q++) memcpy(M + (size_t)q * d, psi + (size_t)c[q] * d, d);
            memcpy(M + (size_t)(d - 1) * d, psi + (size_t)(i - 1) * d, d);
            if (or_mat_rank(M, d, d) < d) { ok = 0; break; }
            int q = d - 2;
            while (q >= 0 && c[q] == (i - 1) - (d - 1) + q) q--;
            if (q < 0) break;
            c[q]++;
            for (int r2 = q + 1; r2 < d - 1; r2++) c[r2] = c[r2 - 1] + 1;
          }
        }
        if (ok) { lam[i - 1] = l; found = 1; }
      }
      if (!found) { free(lam); free(M); free(c); return OR_EUNSUP; }
    }
    if (lambda) memcpy(lambda, lam, n);
    free(lam); free(M); free(c);
    return OR_OK;
  }
  if (kind == OR_MBR) {
    /* P:115 + R5: rows 1..k = [I_k 0]; rows k+1..n Cauchy (g^{d+i} - g^{j-1})^{-1}. */
    if (n + d > 254) return OR_EUNSUP;
    for (int i = 1; i <= n; i++)
      for (int j = 1; j <= d; j++) {
        uint8_t v;
        if (i <= k)
          v = (uint8_t)(i == j);
        else
          v = or_gf_inv(or_gf_exp(d + i) ^ or_gf_exp(j - 1));
        psi[(i - 1) * d + (j - 1)] = v;
      }
    if (lambda) memset(lambda, 0, n);
    return OR_OK;
  }
  if (kind == OR_RS) {
    /* R12: V_{i,j} = g^{(i-1)(j-1)}, n x k ("Vandermonde-based Reed-Solomon") */
    for (int i = 1; i <= n; i++)
      for (int j = 1; j <= k; j++) psi[(i - 1) * k + (j - 1)] = or_gf_exp((long)(i - 1) * (j - 1));
    if (lambda) memset(lambda, 0, n);
    return OR_OK;
  }
  return OR_EINVAL;
}

/* ------------------------------------------------------------------ linearisation */
/* G: (n alpha) x B, G_{alpha(i-1)+j, L_{l,j}} = Psi_{i,l} (R3: node-major row index). */
int or_generator(int kind, int n, int k, int d, uint8_t *G) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  if (kind == OR_RS) return or_psi(kind, n, k, d, G, NULL); /* G = V directly */
  int dd = (kind == OR_MBR) ? d : alpha;                     /* columns of L */
  int *L = (int *)malloc(sizeof(int) * d * dd);
  uint8_t *psi = (uint8_t *)malloc((size_t)n * d);
  rc = or_index_matrix(kind, k, d, L);
  if (!rc) rc = or_psi(kind, n, k, d, psi, NULL);
  if (!rc) {
    memset(G, 0, (size_t)n * alpha * B);
    for (int i = 1; i <= n; i++)
      for (int j = 1; j <= alpha; j++)
        for (int l = 1; l <= d; l++) {
          int lp = L[(l - 1) * dd + (j - 1)];
          if (lp == 0) continue; /* structural zero of M contributes nothing */
          G[((size_t)alpha * (i - 1) + (j - 1)) * B + (lp - 1)] = psi[(i - 1) * d + (l - 1)];
        }
  }
  free(L);
  free(psi);
  return rc;
}

/* ------------------------------------------------------------------ systematic form */
/* Gp = G' (n alpha x B).  MSR / RS: G' = G Gtilde^{-1} with Gtilde the first B rows.
 * MBR (R6): the systematic rows of G are already unit rows (Psi = [I 0; Psi'']); G' = G. */
int or_systematic(int kind, int n, int k, int d, uint8_t *Gp) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  size_t R = (size_t)n * alpha;
  uint8_t *G = (uint8_t *)malloc(R * B);
  rc = or_generator(kind, n, k, d, G);
  if (rc) { free(G); return rc; }
  if (kind == OR_MBR) {
    memcpy(Gp, G, R * B);
    free(G);
    return OR_OK;
  }
  uint8_t *Ginv = (uint8_t *)malloc((size_t)B * B);
  rc = or_mat_inv(G, Ginv, B); /* Gtilde = first B rows of G */
  if (!rc) or_mat_mul(G, Ginv, Gp, (int)R, B, B);
  free(Ginv);
  free(G);
  return rc;
}

/* parity part G'' = rows k alpha .. n alpha - 1 of G' ((n-k) alpha x B) */
int or_parity_matrix(int kind, int n, int k, int d, uint8_t *Gpp) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  uint8_t *Gp = (uint8_t *)malloc((size_t)n * alpha * B);
  rc = or_systematic(kind, n, k, d, Gp);
  if (!rc) memcpy(Gpp, Gp + (size_t)k * alpha * B, (size_t)(n - k) * alpha * B);
  free(Gp);
  return rc;
}

/* ------------------------------------------------------------------ region linear combination */
/* out_r = XOR_c A_{r,c} * in_c, byte by byte (P:40 Y = GX).  skip_zeros: multiplications by zero
 * coefficients are skipped; skip_zeros = 0 multiplies densely (the north-star pin
 * "sparsified and dense generators give identical codewords"). */
void or_apply(const uint8_t *A, int R, int C, const uint8_t *const *in, uint8_t *const *out, size_t S,
              int skip_zeros) {
  for (int r = 0; r < R; r++) {
    uint8_t *o = out[r];
    memset(o, 0, S);
    for (int c = 0; c < C; c++) {
      uint8_t a = A[(size_t)r * C + c];
      if (skip_zeros && a == 0) continue;
      const uint8_t *x = in[c];
      for (size_t p = 0; p < S; p++) o[p] ^= or_gf_mul(a, x[p]);
    }
  }
}

/* contiguous convenience: A (R x C), in = C blocks of S bytes, out = R blocks of S bytes */
void or_apply_flat(const uint8_t *A, int R, int C, const uint8_t *in, uint8_t *out, size_t S,
                   int skip_zeros) {
  const uint8_t **ip = (const uint8_t **)malloc(sizeof(void *) * (C ? C : 1));
  uint8_t **op = (uint8_t **)malloc(sizeof(void *) * (R ? R : 1));
  for (int c = 0; c < C; c++) ip[c] = in + (size_t)c * S;
  for (int r = 0; r < R; r++) op[r] = out + (size_t)r * S;
  or_apply(A, R, C, ip, op, S, skip_zeros);
  free(ip);
  free(op);
}

/* ------------------------------------------------------------------ systematic linear encode */
/* data: stripes x [B][S]; parity: stripes x [(n-k) alpha][S].  Y_parity = G'' X. */
int or_encode(int kind, int n, int k, int d, const uint8_t *data, uint8_t *parity, size_t S,
              size_t stripes) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  int P = (n - k) * alpha;
  uint8_t *Gpp = (uint8_t *)malloc((size_t)P * B);
  rc = or_parity_matrix(kind, n, k, d, Gpp);
  if (!rc)
    for (size_t t = 0; t < stripes; t++)
      or_apply_flat(Gpp, P, B, data + t * (size_t)B * S, parity + t * (size_t)P * S, S, 1);
  free(Gpp);
  return rc;
}

/* ------------------------------------------------------------------ specific encode */
/* code (n alpha blocks, node-major) = Psi M(Z) with M_{l,j} = Z_{L_{l,j}} (0 if L = 0).
 * For RS this is V Z.  Z has B blocks. */
int or_encode_specific(int kind, int n, int k, int d, const uint8_t *Z, uint8_t *code, size_t S) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  if (kind == OR_RS) {
    uint8_t *V = (uint8_t *)malloc((size_t)n * k);
    or_psi(kind, n, k, d, V, NULL);
    or_apply_flat(V, n, k, Z, code, S, 1);
    free(V);
    return OR_OK;
  }
  int dd = (kind == OR_MBR) ? d : alpha;
  int *L = (int *)malloc(sizeof(int) * d * dd);
  uint8_t *psi = (uint8_t *)malloc((size_t)n * d);
  or_index_matrix(kind, k, d, L);
  or_psi(kind, n, k, d, psi, NULL);
  for (int i = 0; i < n; i++)
    for (int j = 0; j < alpha; j++) {
      uint8_t *o = code + ((size_t)i * alpha + j) * S;
      memset(o, 0, S);
      for (int l = 0; l < d; l++) { /* C_{i,j} = sum_l Psi_{i,l} M_{l,j} */
        int lp = L[l * dd + j];
        uint8_t a = psi[i * d + l];
        if (lp == 0 || a == 0) continue;
        const uint8_t *x = Z + (size_t)(lp - 1) * S;
        for (size_t p = 0; p < S; p++) o[p] ^= or_gf_mul(a, x[p]);
      }
    }
  free(L);
  free(psi);
  return OR_OK;
}

/* ------------------------------------------------------------------ linear (lazy) decode */
/* ids: n_ids distinct node ids (0-based), pieces: n_ids x [alpha][S].  X (B blocks) = Gtilde^{-1}
 * Ytilde where the B rows are taken greedily from the survivors' rows of G':
 * systematic survivors first, then the rest, each in ascending id, symbols in order (R13).
 * Returns OR_ESING if the survivors do not span B independent rows. */
int or_decode_linear(int kind, int n, int k, int d, const int *ids, int n_ids, const uint8_t *pieces,
                     uint8_t *X, size_t S) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  for (int a = 0; a < n_ids; a++) {
    if (ids[a] < 0 || ids[a] >= n) return OR_EINVAL;
    for (int b = 0; b < a; b++)
      if (ids[a] == ids[b]) return OR_EINVAL;
  }
  uint8_t *Gp = (uint8_t *)malloc((size_t)n * alpha * B);
  rc = or_systematic(kind, n, k, d, Gp);
  if (rc) { free(Gp); return rc; }
  /* candidate order */
  int *order = (int *)malloc(sizeof(int) * (n_ids ? n_ids : 1));
  int no = 0;
  for (int pass = 0; pass < 2; pass++)
    for (int id = 0; id < n; id++) {
      if ((pass == 0) != (id < k)) continue;
      for (int a = 0; a < n_ids; a++)
        if (ids[a] == id) order[no++] = a;
    }
  uint8_t *Sel = (uint8_t *)malloc((size_t)B * B);
  const uint8_t **Ysel = (const uint8_t **)malloc(sizeof(void *) * B);
  int nsel = 0;
  for (int o = 0; o < no && nsel < B; o++) {
    int a = order[o];
    for (int j = 0; j < alpha && nsel < B; j++) {
      memcpy(Sel + (size_t)nsel * B, Gp + ((size_t)ids[a] * alpha + j) * B, B);
      if (or_mat_rank(Sel, nsel + 1, B) == nsel + 1) { /* greedy: keep independent rows */
        Ysel[nsel] = pieces + ((size_t)a * alpha + j) * S;
        nsel++;
      }
    }
  }
  if (nsel < B) rc = OR_ESING;
  if (!rc) {
    uint8_t *Inv = (uint8_t *)malloc((size_t)B * B);
    rc = or_mat_inv(Sel, Inv, B);
    if (!rc) {
      uint8_t **Xo = (uint8_t **)malloc(sizeof(void *) * B);
      for (int c = 0; c < B; c++) Xo[c] = X + (size_t)c * S;
      or_apply(Inv, B, B, Ysel, Xo, S, 1);
      free(Xo);
    }
    free(Inv);
  }
  free(Sel);
  free(Ysel);
  free(order);
  free(Gp);
  return rc;
}

/* ------------------------------------------------------------------ specific MSR decode */
/* From exactly k distinct nodes (pieces k x [alpha][S]) of the PM code C = Psi M(Z), recover the
 * message Z (B blocks) with the symmetric-matrix method: A = C_DC Phi_DC^t = P + Lambda_DC Q,
 * Q_ij = (A_ij - A_ji)/(lambda_i - lambda_j), P_ij = A_ij - lambda_i Q_ij (i != j); for each i the
 * alpha off-diagonal entries of row i give phi_i S1 (resp. phi_i S2) through the alpha x alpha
 * matrix of the other nodes' phi rows; S1, S2 follow from alpha of those rows. */
int or_decode_msr_specific_Z(int kind, int n, int k, int d, const int *ids, const uint8_t *pieces,
                             uint8_t *Z, size_t S) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  if (!OR_IS_MSR(kind)) return OR_EINVAL;
  for (int a = 0; a < k; a++) {
    if (ids[a] < 0 || ids[a] >= n) return OR_EINVAL;
    for (int b = 0; b < a; b++)
      if (ids[a] == ids[b]) return OR_EINVAL;
  }
  uint8_t *psi = (uint8_t *)malloc((size_t)n * d), *lam = (uint8_t *)malloc(n);
  int *L = (int *)malloc(sizeof(int) * d * alpha);
  or_psi(kind, n, k, d, psi, lam);
  or_index_matrix(kind, k, d, L);
  /* phi rows of DC: Phi_DC[a][t] = psi[ids[a]][t], t < alpha */
  /* per-node inverse of the other nodes' Phi^t (alpha x alpha) */
  uint8_t *OthInv = (uint8_t *)malloc((size_t)k * alpha * alpha);
  uint8_t *Mtx = (uint8_t *)malloc((size_t)alpha * alpha);
  for (int i = 0; i < k && !rc; i++) {
    int r = 0;
    for (int j = 0; j < k; j++) {
      if (j == i) continue;
      /* column r of Phi_{others}^t = phi_j */
      for (int t = 0; t < alpha; t++) Mtx[t * alpha + r] = psi[ids[j] * d + t];
      r++;
    }
    rc = or_mat_inv(Mtx, OthInv + (size_t)i * alpha * alpha, alpha);
  }
  /* first alpha nodes of DC for the final solve */
  uint8_t *SelInv = (uint8_t *)malloc((size_t)alpha * alpha);
  if (!rc) {
    for (int a = 0; a < alpha; a++)
      for (int t = 0; t < alpha; t++) Mtx[a * alpha + t] = psi[ids[a] * d + t];
    rc = or_mat_inv(Mtx, SelInv, alpha);
  }
  for (int a = 0; a < k && !rc; a++)
    for (int b = 0; b < a; b++)
      if (lam[ids[a]] == lam[ids[b]]) rc = OR_EUNSUP;
  uint8_t *A = (uint8_t *)malloc((size_t)k * k), *Pm = (uint8_t *)malloc((size_t)k * k),
          *Qm = (uint8_t *)malloc((size_t)k * k);
  uint8_t *U1 = (uint8_t *)malloc((size_t)k * alpha), *U2 = (uint8_t *)malloc((size_t)k * alpha);
  uint8_t *S1 = (uint8_t *)malloc((size_t)alpha * alpha), *S2 = (uint8_t *)malloc((size_t)alpha * alpha);
  uint8_t *vec = (uint8_t *)malloc(alpha);
  for (size_t p = 0; p < S && !rc; p++) {
    /* A = C_DC Phi_DC^t */
    for (int i = 0; i < k; i++)
      for (int j = 0; j < k; j++) {
        uint8_t s = 0;
        for (int t = 0; t < alpha; t++)
          s ^= or_gf_mul(pieces[((size_t)i * alpha + t) * S + p], psi[ids[j] * d + t]);
        A[i * k + j] = s;
      }
    for (int i = 0; i < k; i++)
      for (int j = 0; j < k; j++) {
        if (i == j) continue;
        uint8_t li = lam[ids[i]], lj = lam[ids[j]];
        uint8_t q = or_gf_div(A[i * k + j] ^ A[j * k + i], li ^ lj);
        Qm[i * k + j] = q;
        Pm[i * k + j] = A[i * k + j] ^ or_gf_mul(li, q);
      }
    /* u_i = (off-diagonal row i) * (Phi_others^t)^{-1} */
    for (int i = 0; i < k; i++) {
      const uint8_t *Inv = OthInv + (size_t)i * alpha * alpha;
      for (int which = 0; which < 2; which++) {
        const uint8_t *Src = which ? Qm : Pm;
        uint8_t *U = which ? U2 : U1;
        int r = 0;
        for (int j = 0; j < k; j++)
          if (j != i) vec[r++] = Src[i * k + j];
        for (int c = 0; c < alpha; c++) {
          uint8_t s = 0;
          for (int t = 0; t < alpha; t++) s ^= or_gf_mul(vec[t], Inv[t * alpha + c]);
          U[i * alpha + c] = s;
        }
      }
    }
    /* S = Phi_sel^{-1} U_sel, sel = first alpha nodes of DC */
    or_mat_mul(SelInv, U1, S1, alpha, alpha, alpha);
    or_mat_mul(SelInv, U2, S2, alpha, alpha, alpha);
    /* read Z out through L = [S1; S2] */
    for (int l = 0; l < d; l++)
      for (int j = 0; j < alpha; j++) {
        int lp = L[l * alpha + j];
        uint8_t v = (l < alpha) ? S1[l * alpha + j] : S2[(l - alpha) * alpha + j];
        Z[(size_t)(lp - 1) * S + p] = v;
      }
  }
  free(psi); free(lam); free(L); free(OthInv); free(Mtx); free(SelInv);
  free(A); free(Pm); free(Qm); free(U1); free(U2); free(S1); free(S2); free(vec);
  return rc;
}

/* ------------------------------------------------------------------ specific MBR decode */
/* From exactly k nodes (pieces k x [d][S]) of C = Psi M(X): with Psi_DC = [Phi_DC Delta_DC],
 * T = Phi_DC^{-1} R_right, S = Phi_DC^{-1} (R_left - Delta_DC T^t); X read out through L. */
int or_decode_mbr_specific(int n, int k, int d, const int *ids, const uint8_t *pieces, uint8_t *X,
                           size_t S) {
  int alpha, B;
  int rc = or_params(OR_MBR, n, k, d, &alpha, &B);
  if (rc) return rc;
  for (int a = 0; a < k; a++) {
    if (ids[a] < 0 || ids[a] >= n) return OR_EINVAL;
    for (int b = 0; b < a; b++)
      if (ids[a] == ids[b]) return OR_EINVAL;
  }
  uint8_t *psi = (uint8_t *)malloc((size_t)n * d);
  int *L = (int *)malloc(sizeof(int) * d * d);
  or_psi(OR_MBR, n, k, d, psi, NULL);
  or_index_matrix(OR_MBR, k, d, L);
  uint8_t *Phi = (uint8_t *)malloc((size_t)k * k), *PhiInv = (uint8_t *)malloc((size_t)k * k);
  for (int a = 0; a < k; a++)
    for (int t = 0; t < k; t++) Phi[a * k + t] = psi[ids[a] * d + t];
  rc = or_mat_inv(Phi, PhiInv, k);
  int dk = d - k;
  uint8_t *R = (uint8_t *)malloc((size_t)k * d), *T = (uint8_t *)malloc((size_t)k * (dk ? dk : 1));
  uint8_t *Sm = (uint8_t *)malloc((size_t)k * k), *W = (uint8_t *)malloc((size_t)k * k);
  for (size_t p = 0; p < S && !rc; p++) {
    for (int a = 0; a < k; a++)
      for (int l = 0; l < d; l++) R[a * d + l] = pieces[((size_t)a * d + l) * S + p];
    /* T = Phi^{-1} R_right  (k x (d-k)) */
    for (int r = 0; r < k; r++)
      for (int c = 0; c < dk; c++) {
        uint8_t s = 0;
        for (int t = 0; t < k; t++) s ^= or_gf_mul(PhiInv[r * k + t], R[t * d + k + c]);
        T[r * dk + c] = s;
      }
    /* W = R_left - Delta_DC T^t (k x k) */
    for (int a = 0; a < k; a++)
      for (int c = 0; c < k; c++) {
        uint8_t s = R[a * d + c];
        for (int t = 0; t < dk; t++) s ^= or_gf_mul(psi[ids[a] * d + k + t], T[c * dk + t]);
        W[a * k + c] = s;
      }
    or_mat_mul(PhiInv, W, Sm, k, k, k);
    for (int r = 0; r < k; r++)
      for (int c = 0; c < d; c++) {
        int lp = L[r * d + c];
        uint8_t v = (c < k) ? Sm[r * k + c] : T[r * dk + (c - k)];
        X[(size_t)(lp - 1) * S + p] = v;
      }
  }
  free(psi); free(L); free(Phi); free(PhiInv); free(R); free(T); free(Sm); free(W);
  return rc;
}

/* ------------------------------------------------------------------ repair, P:53 fn */
/* repair coefficient vector mu of the lost node f: MSR phi_f (alpha entries), MBR psi_f (d entries),
 * RS [1].  Reads per helper = number of nonzero entries. */
int or_repair_mu(int kind, int n, int k, int d, int f, uint8_t *mu, int *len) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  if (f < 0 || f >= n) return OR_EINVAL;
  if (kind == OR_RS) { mu[0] = 1; *len = 1; return OR_OK; }
  uint8_t *psi = (uint8_t *)malloc((size_t)n * d);
  or_psi(kind, n, k, d, psi, NULL);
  int m = (kind == OR_MBR) ? d : alpha;
  for (int t = 0; t < m; t++) mu[t] = psi[f * d + t];
  *len = m;
  free(psi);
  return OR_OK;
}

int or_repair_reads(int kind, int n, int k, int d, int f) {
  uint8_t mu[256];
  int len = 0;
  if (or_repair_mu(kind, n, k, d, f, mu, &len)) return -1;
  int c = 0;
  for (int t = 0; t < len; t++) c += mu[t] != 0;
  return c;
}

/* Helper projection: beta = sum_a mu_a C_h[a], reading only blocks with mu_a != 0. */
int or_repair_project(int kind, int n, int k, int d, int f, const uint8_t *piece, uint8_t *beta,
                      size_t S) {
  uint8_t mu[256];
  int len = 0;
  int rc = or_repair_mu(kind, n, k, d, f, mu, &len);
  if (rc) return rc;
  memset(beta, 0, S);
  for (int a = 0; a < len; a++) {
    if (!mu[a]) continue;
    for (size_t p = 0; p < S; p++) beta[p] ^= or_gf_mul(mu[a], piece[(size_t)a * S + p]);
  }
  return OR_OK;
}

/* Newcomer: solve Psi_H z = beta (d x d); MSR piece_a = z_a + lambda_f z_{alpha+a};
 * MBR piece = z (M symmetric).  RS (alpha=1, d=k): lost = G'_f (G'_H)^{-1} beta.
 * Returns OR_ESING when Psi_H is singular (R10: predicted set at n = 2k). */
int or_repair_combine(int kind, int n, int k, int d, int f, const int *H, const uint8_t *betas,
                      uint8_t *out, size_t S) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  int nh = (kind == OR_RS) ? k : d;
  if (f < 0 || f >= n) return OR_EINVAL;
  for (int a = 0; a < nh; a++) {
    if (H[a] < 0 || H[a] >= n || H[a] == f) return OR_EINVAL;
    for (int b = 0; b < a; b++)
      if (H[a] == H[b]) return OR_EINVAL;
  }
  if (kind == OR_RS) {
    uint8_t *Gp = (uint8_t *)malloc((size_t)n * k), *GH = (uint8_t *)malloc((size_t)k * k),
            *GHi = (uint8_t *)malloc((size_t)k * k), *row = (uint8_t *)malloc(k);
    or_systematic(kind, n, k, d, Gp);
    for (int a = 0; a < k; a++) memcpy(GH + a * k, Gp + (size_t)H[a] * k, k);
    rc = or_mat_inv(GH, GHi, k);
    if (!rc) {
      or_mat_mul(Gp + (size_t)f * k, GHi, row, 1, k, k);
      or_apply_flat(row, 1, k, betas, out, S, 1);
    }
    free(Gp); free(GH); free(GHi); free(row);
    return rc;
  }
  uint8_t *psi = (uint8_t *)malloc((size_t)n * d), *lam = (uint8_t *)malloc(n);
  uint8_t *PH = (uint8_t *)malloc((size_t)d * d), *PHi = (uint8_t *)malloc((size_t)d * d);
  or_psi(kind, n, k, d, psi, lam);
  for (int a = 0; a < d; a++) memcpy(PH + a * d, psi + (size_t)H[a] * d, d);
  rc = or_mat_inv(PH, PHi, d);
  if (!rc) {
    uint8_t *z = (uint8_t *)malloc((size_t)d * S);
    or_apply_flat(PHi, d, d, betas, z, S, 1); /* z = Psi_H^{-1} beta */
    if (kind == OR_MBR) {
      memcpy(out, z, (size_t)d * S);
    } else {
      uint8_t lf = lam[f];
      for (int a = 0; a < alpha; a++)
        for (size_t p = 0; p < S; p++)
          out[(size_t)a * S + p] = z[(size_t)a * S + p] ^ or_gf_mul(lf, z[(size_t)(alpha + a) * S + p]);
    }
    free(z);
  }
  free(psi); free(lam); free(PH); free(PHi);
  return rc;
}

/* Full repair: pieces = helpers' pieces (nh x [alpha][S]) -> out (alpha blocks). */
int or_repair(int kind, int n, int k, int d, int f, const int *H, const uint8_t *pieces, uint8_t *out,
              size_t S) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  int nh = (kind == OR_RS) ? k : d;
  uint8_t *betas = (uint8_t *)malloc((size_t)nh * S + 1);
  for (int a = 0; a < nh && !rc; a++)
    rc = or_repair_project(kind, n, k, d, f, pieces + (size_t)a * alpha * S, betas + (size_t)a * S, S);
  if (!rc) rc = or_repair_combine(kind, n, k, d, f, H, betas, out, S);
  free(betas);
  return rc;
}

/* ------------------------------------------------------------------ validation */
static int next_comb(int *c, int r, int n) {
  int i = r - 1;
  while (i >= 0 && c[i] == n - r + i) i--;
  if (i < 0) return 0;
  c[i]++;
  for (int j = i + 1; j < r; j++) c[j] = c[j - 1] + 1;
  return 1;
}

/* Checks the constraints of P:121-127: flags |= 1 lambda values not distinct (MSR); 2 some d rows
 * of Psi dependent; 4 some alpha rows of Phi dependent (MSR; MBR: k rows of Phi); 8 a check was
 * skipped because it has more than max_subsets subsets.  check_phi = 0 skips the Phi check (P:189:
 * "by construction, any k rows of Phi are invertible").  witness (may be NULL) receives the first
 * failing d-row subset of Psi. */
int or_validate(int kind, int n, int k, int d, long max_subsets, int check_phi, int *witness) {
  int alpha, B;
  int rc = or_params(kind, n, k, d, &alpha, &B);
  if (rc) return rc;
  uint8_t *psi = (uint8_t *)malloc((size_t)n * d), *lam = (uint8_t *)malloc(n);
  rc = or_psi(kind, n, k, d, psi, lam);
  if (rc) { free(psi); free(lam); return rc; }
  int flags = 0;
  if (OR_IS_MSR(kind))
    for (int a = 0; a < n; a++)
      for (int b = 0; b < a; b++)
        if (lam[a] == lam[b]) flags |= 1;
  /* number of d-subsets */
  double cnt = 1;
  for (int i = 0; i < d; i++) cnt = cnt * (n - i) / (i + 1);
  int c[256];
  uint8_t *M = (uint8_t *)malloc((size_t)d * d);
  if (cnt > (double)max_subsets) {
    flags |= 8;
  } else {
    for (int i = 0; i < d; i++) c[i] = i;
    do {
      for (int a = 0; a < d; a++) memcpy(M + a * d, psi + (size_t)c[a] * d, d);
      if (or_mat_rank(M, d, d) < d) {
        if (!(flags & 2) && witness)
          for (int a = 0; a < d; a++) witness[a] = c[a];
        flags |= 2;
        break;
      }
    } while (next_comb(c, d, n));
  }
  if (check_phi && kind != OR_RS) {
    int r = (kind == OR_MBR) ? k : alpha;
    double cnt2 = 1;
    for (int i = 0; i < r; i++) cnt2 = cnt2 * (n - i) / (i + 1);
    if (cnt2 > (double)max_subsets) {
      flags |= 8;
    } else {
      for (int i = 0; i < r; i++) c[i] = i;
      do {
        for (int a = 0; a < r; a++)
          for (int t = 0; t < r; t++) M[a * r + t] = psi[(size_t)c[a] * d + t];
        if (or_mat_rank(M, r, r) < r) { flags |= 4; break; }
      } while (next_comb(c, r, n));
    }
  }
  free(M);
  free(psi);
  free(lam);
  return flags;
}

/* ------------------------------------------------------------------ GF(2^16) validity */
/* P:189's second claim: the sparse construction is valid for k in {2..64} in GF(2^16).  Reading
 * R1 extended to w = 16 (GF-Complete's default, as for w = 8): primitive polynomial
 * x^16+x^12+x^3+x+1 (0x1100B), g = 2.  The sparse Psi (same formulas and 1-based indices as
 * or_psi) at n = d+1, checked like P:189 describes: Lambda distinct, and all n d x d submatrices
 * of Psi invertible.  Returns flags as or_validate (1 lambda collision, 2 singular submatrix). */
static uint16_t EXP16[2 * 65535];
static int LOG16[65536];
static int gf16_ready = 0;
static void gf16_init(void) {
  if (gf16_ready) return;
  unsigned x = 1;
  for (int e = 0; e < 65535; e++) {
    EXP16[e] = (uint16_t)x;
    LOG16[x] = e;
    x <<= 1;
    if (x & 0x10000) x ^= 0x1100B;
  }
  for (int e = 65535; e < 2 * 65535; e++) EXP16[e] = EXP16[e - 65535];
  LOG16[0] = -1;
  gf16_ready = 1;
}
static uint16_t gf16_mul(uint16_t a, uint16_t b) {
  if (!a || !b) return 0;
  return EXP16[LOG16[a] + LOG16[b]];
}
static uint16_t gf16_inv(uint16_t a) { return EXP16[(65535 - LOG16[a]) % 65535]; }
static uint16_t gf16_exp(long e) { return EXP16[((e % 65535) + 65535) % 65535]; }
static int gf16_rank(uint16_t *W, int r, int c) {
  int rank = 0;
  for (int col = 0; col < c && rank < r; col++) {
    int piv = -1;
    for (int i = rank; i < r; i++)
      if (W[i * c + col]) { piv = i; break; }
    if (piv < 0) continue;
    if (piv != rank)
      for (int j = 0; j < c; j++) { uint16_t t = W[piv * c + j]; W[piv * c + j] = W[rank * c + j]; W[rank * c + j] = t; }
    uint16_t inv = gf16_inv(W[rank * c + col]);
    for (int i = 0; i < r; i++) {
      if (i == rank || !W[i * c + col]) continue;
      uint16_t f = gf16_mul(W[i * c + col], inv);
      for (int j = 0; j < c; j++) W[i * c + j] ^= gf16_mul(f, W[rank * c + j]);
    }
    rank++;
  }
  return rank;
}
uint16_t or_gf16_mul(uint16_t a, uint16_t b) { gf16_init(); return gf16_mul(a, b); }

/* P:189 validity check of the sparse MSR code over GF(2^16) at n = d+1 (the n d-subsets the paper
 * checks) -- or, through or_validate16_sparse_n, at n = d+1 or d+2 over EVERY d-row subset (all
 * rows but one / but two), counting the singular ones (SURVEY §8(c) A7 predicts exactly the
 * C(alpha, 2) subsets that omit two identity rows at n = 2k, k >= 3). */
int or_validate16_sparse_n(int k, int n, int *flags_out, int *n_singular);
int or_validate16_sparse(int k, int *flags_out) { return or_validate16_sparse_n(k, 2 * k - 1, flags_out, 0); }

int or_validate16_sparse_n(int k, int n, int *flags_out, int *n_singular) {
  gf16_init();
  if (k < 2 || k > 200) return OR_EINVAL;
  const int alpha = k - 1, d = 2 * k - 2;
  if (n < d + 1 || n > d + 2) return OR_EINVAL;
  uint16_t *psi = (uint16_t *)malloc(sizeof(uint16_t) * n * d), *lam = (uint16_t *)malloc(sizeof(uint16_t) * n);
  uint16_t *M = (uint16_t *)malloc(sizeof(uint16_t) * d * d);
  for (int i = 1; i <= n; i++) {
    uint16_t xi = gf16_exp(i + alpha);
    uint16_t l = gf16_mul(xi ^ gf16_exp(0), gf16_inv(xi ^ gf16_exp(alpha)));
    lam[i - 1] = l;
    for (int j = 1; j <= alpha; j++) {
      uint16_t phi = (i <= alpha) ? (uint16_t)(i == j) : gf16_inv(xi ^ gf16_exp(j - 1));
      psi[(i - 1) * d + (j - 1)] = phi;
      psi[(i - 1) * d + alpha + (j - 1)] = gf16_mul(l, phi);
    }
  }
  int flags = 0;
  for (int a = 0; a < n; a++)
    for (int b = 0; b < a; b++)
      if (lam[a] == lam[b]) flags |= 1;
  int sing = 0;
  for (int s1 = 0; s1 < n; s1++) /* every d-subset: all rows but {s1} (n = d+1) or {s1, s2} (n = d+2) */
    for (int s2 = (n == d + 2 ? s1 + 1 : n); s2 <= n; s2++) {
      if (n == d + 2 && s2 == n) continue;
      int r = 0;
      for (int i = 0; i < n; i++)
        if (i != s1 && i != s2) memcpy(M + (size_t)(r++) * d, psi + (size_t)i * d, sizeof(uint16_t) * d);
      if (gf16_rank(M, d, d) < d) {
        flags |= 2;
        sing++;
      }
    }
  free(psi); free(lam); free(M);
  *flags_out = flags;
  if (n_singular) *n_singular = sing;
  return OR_OK;
}
