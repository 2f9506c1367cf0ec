#include <cstdio>
#include <map>
#include <string>
#include <vector>
#include "construct.hpp"
#include "xorprog.hpp"
using namespace pmrc;
static long net_cost(const Mat &A, const std::vector<int> &rows, const std::vector<int> &cols) {
  std::vector<std::vector<int>> r(8 * rows.size());
  for (size_t i = 0; i < rows.size(); i++)
    for (size_t ci = 0; ci < cols.size(); ci++) {
      const uint8_t cf = A.at(rows[i], cols[ci]);
      if (!cf) continue;
      uint8_t br[8];
      gf().bitmatrix(cf, br);
      for (int b = 0; b < 8; b++)
        for (int bp = 0; bp < 8; bp++)
          if ((br[b] >> bp) & 1) r[i * 8 + b].push_back((int)ci * 8 + bp);
    }
  return cse3(8 * (int)cols.size(), r, 0).lop3();
}
int main() {
  CodeDef D; std::string err;
  build_code(KIND_MSR_SPARSE, 8, 14, 16, 8, D, err);
  const Mat &A = D.Gpp;
  std::map<std::vector<int>, std::vector<int>> g;
  for (int r = 0; r < A.r; r++) { std::vector<int> s; for (int c = 0; c < A.c; c++) if (A.at(r, c)) s.push_back(c); g[s].push_back(r); }
  for (auto &kv : g) {
    const auto &cols = kv.first; const auto &rows = kv.second;
    std::vector<int> c0(cols.begin(), cols.begin() + 7), c1(cols.begin() + 7, cols.end());
    std::vector<int> r0(rows.begin(), rows.begin() + 4), r1(rows.begin() + 4, rows.end());
    long a = net_cost(A, r0, c0) + net_cost(A, r0, c1) + net_cost(A, r1, c0) + net_cost(A, r1, c1);
    long b = net_cost(A, rows, c0) + net_cost(A, rows, c1);
    long w = net_cost(A, rows, cols);
    printf("4x(4 rows x 7 in) %ld   2x(8 rows x 7 in) %ld   1x(8x14) %ld\n", a, b, w);
  }
}
