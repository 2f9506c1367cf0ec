#include "gf256.hpp"

namespace pmrc {

const GF256 &gf() {
  static const GF256 g;
  return g;
}

const GF65536 &gf16() {
  static const GF65536 g;
  return g;
}

Mat matmul(const Mat &A, const Mat &B) {
  const GF256 &F = gf();
  Mat C(A.r, B.c);
  for (int i = 0; i < A.r; i++)
    for (int t = 0; t < A.c; t++) {
      uint8_t a = A.at(i, t);
      if (!a) continue;
      const uint8_t *row = F.mul_t[a];
      for (int j = 0; j < B.c; j++) C.at(i, j) ^= row[B.at(t, j)];
    }
  return C;
}

bool invert(const Mat &A, Mat &out) {
  const GF256 &F = gf();
  int m = A.r;
  Mat W = A;
  out = Mat(m, m);
  for (int i = 0; i < m; i++) out.at(i, i) = 1;
  for (int col = 0; col < m; col++) {
    int piv = col;
    while (piv < m && !W.at(piv, col)) piv++;
    if (piv == m) return false;
    if (piv != col)
      for (int j = 0; j < m; j++) {
        std::swap(W.at(piv, j), W.at(col, j));
        std::swap(out.at(piv, j), out.at(col, j));
      }
    uint8_t s = F.inv(W.at(col, col));
    for (int j = 0; j < m; j++) {
      W.at(col, j) = F.mul(W.at(col, j), s);
      out.at(col, j) = F.mul(out.at(col, j), s);
    }
    for (int i = 0; i < m; i++) {
      uint8_t f = W.at(i, col);
      if (i == col || !f) continue;
      const uint8_t *row = F.mul_t[f];
      for (int j = 0; j < m; j++) {
        W.at(i, j) ^= row[W.at(col, j)];
        out.at(i, j) ^= row[out.at(col, j)];
      }
    }
  }
  return true;
}

int rank(const Mat &A) {
  const GF256 &F = gf();
  Mat W = A;
  int rk = 0;
  for (int col = 0; col < W.c && rk < W.r; col++) {
    int piv = rk;
    while (piv < W.r && !W.at(piv, col)) piv++;
    if (piv == W.r) continue;
    for (int j = 0; j < W.c; j++) std::swap(W.at(piv, j), W.at(rk, j));
    uint8_t s = F.inv(W.at(rk, col));
    for (int i = rk + 1; i < W.r; i++) {
      uint8_t f = F.mul(W.at(i, col), s);
      if (!f) continue;
      const uint8_t *row = F.mul_t[f];
      for (int j = 0; j < W.c; j++) W.at(i, j) ^= row[W.at(rk, j)];
    }
    rk++;
  }
  return rk;
}

}  // namespace pmrc
