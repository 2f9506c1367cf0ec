// Host-only probe: how much does the choice of which inputs share a CSE sub-network (and which
// rows share a warp) change the LOP3 count of the config-2 encode's XOR networks?
// Build: g++ -O2 -std=c++17 -I paper_1412_3022_b200/csrc/host tools/probe/partition_search.cpp \
//   paper_1412_3022_b200/csrc/host/{construct,gf256,xorprog}.cpp -o /dev/shm/partition_search
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "construct.hpp"
#include "xorprog.hpp"

using namespace pmrc;

static long net_cost(const Mat &A, const std::vector<int> &rows, const std::vector<int> &cols, int restarts) {
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
  long best = -1;
  for (int s = 0; s < restarts; s++) {
    const long c = cse3(8 * (int)cols.size(), r, (uint32_t)s).lop3();
    if (best < 0 || c < best) best = c;
  }
  return best;
}

int main(int argc, char **argv) {
  const int trials = argc > 1 ? atoi(argv[1]) : 40, restarts = argc > 2 ? atoi(argv[2]) : 4;
  CodeDef D;
  std::string err;
  if (build_code(KIND_MSR_SPARSE, 8, 14, 16, 8, D, err)) { printf("build: %s\n", err.c_str()); return 1; }
  const Mat &A = D.Gpp;
  std::map<std::vector<int>, std::vector<int>> by_support;
  for (int r = 0; r < A.r; r++) {
    std::vector<int> sup;
    for (int c = 0; c < A.c; c++) if (A.at(r, c)) sup.push_back(c);
    by_support[sup].push_back(r);
  }
  std::mt19937 rng(1);
  long tot_def = 0, tot_best = 0;
  for (auto &kv : by_support) {
    const std::vector<int> &cols = kv.first, &rows = kv.second;
    auto cost = [&](const std::vector<int> &rw, const std::vector<int> &cl) {
      long c = 0;
      const int hr = (int)rw.size() / 2, hc = (int)cl.size() / 2;
      for (int rk = 0; rk < 2; rk++) {
        std::vector<int> rr(rw.begin() + rk * hr, rk ? rw.end() : rw.begin() + hr);
        for (int sn = 0; sn < 2; sn++) {
          std::vector<int> cc(cl.begin() + sn * hc, sn ? cl.end() : cl.begin() + hc);
          c += net_cost(A, rr, cc, restarts) + 4 * (long)rr.size();  // + the accumulate XORs, as codegen counts
        }
      }
      return c;
    };
    const long def = cost(rows, cols);
    long best = def, worst = def;
    std::vector<int> rw = rows, cl = cols;
    if (getenv("HILL")) {
      // hill climb: swap one input between the two sub-networks or one row between the two warps
      long cur = def;
      for (int t = 0; t < trials; t++) {
        std::vector<int> r2 = rw, c2 = cl;
        if (t % 3 == 2) std::swap(r2[rng() % 4], r2[4 + rng() % 4]);
        else std::swap(c2[rng() % 7], c2[7 + rng() % 7]);
        const long c = cost(r2, c2);
        if (c <= cur) { cur = c; rw = r2; cl = c2; }
        worst = std::max(worst, c);
      }
      best = cur;
    } else
    for (int t = 0; t < trials; t++) {
      std::shuffle(cl.begin(), cl.end(), rng);
      if (t & 1) std::shuffle(rw.begin(), rw.end(), rng);
      const long c = cost(rw, cl);
      best = std::min(best, c);
      worst = std::max(worst, c);
    }
    printf("group rows %zu cols %zu: default %ld best %ld worst %ld\n", rows.size(), cols.size(), def, best, worst);
    tot_def += def;
    tot_best += best;
  }
  printf("total default %ld best-of-%d %ld (%.2f%%)\n", tot_def, trials, tot_best, 100.0 * (tot_def - tot_best) / tot_def);
  return 0;
}
