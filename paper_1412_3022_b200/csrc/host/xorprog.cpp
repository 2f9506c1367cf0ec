#include "xorprog.hpp"

#include <algorithm>
#include <queue>
#include <tuple>
#include <unordered_map>

namespace pmrc {

long Slp::xor2() const {
  long c = (long)tmp.size();
  for (auto &r : rows)
    if (r.size() > 1) c += (long)r.size() - 1;
  return c;
}

long naive_lop3(const std::vector<std::vector<int>> &rows) {
  long c = 0;
  for (auto &r : rows)
    if (r.size() > 1) c += ((long)r.size() - 1 + 1) / 2;
  return c;
}

namespace {
inline uint64_t pkey(int a, int b) {
  if (a > b) std::swap(a, b);
  return ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
}
}  // namespace

Slp paar(int n_in, const std::vector<std::vector<int>> &rows_in) {
  Slp s;
  s.n_in = n_in;
  s.rows = rows_in;
  for (auto &r : s.rows) std::sort(r.begin(), r.end());
  const int R = (int)s.rows.size();
  const int W = (R + 63) / 64;
  // sig_rows[sig] = bitset of rows containing sig
  std::vector<std::vector<uint64_t>> sig_rows(n_in, std::vector<uint64_t>(W, 0));
  for (int r = 0; r < R; r++)
    for (int x : s.rows[r]) sig_rows[x][r >> 6] |= 1ull << (r & 63);

  std::unordered_map<uint64_t, int> cnt;
  cnt.reserve(1 << 14);
  // heap of (count, -a, -b): max count first, then smallest (a, b) for determinism
  std::priority_queue<std::tuple<int, int, int>> heap;
  for (auto &r : s.rows)
    for (size_t i = 0; i < r.size(); i++)
      for (size_t j = i + 1; j < r.size(); j++) cnt[pkey(r[i], r[j])]++;
  for (auto &kv : cnt)
    if (kv.second >= 2) heap.emplace(kv.second, -(int)(kv.first >> 32), -(int)(uint32_t)kv.first);

  auto bump = [&](int a, int b, int delta) {
    int &c = cnt[pkey(a, b)];
    c += delta;
    if (c >= 2) heap.emplace(c, -std::min(a, b), -std::max(a, b));
  };

  while (!heap.empty()) {
    auto [c, na, nb] = heap.top();
    heap.pop();
    int a = -na, b = -nb;
    auto it = cnt.find(pkey(a, b));
    if (it == cnt.end() || it->second != c) continue;  // stale
    // materialise t = a ^ b
    int t = n_in + (int)s.tmp.size();
    s.tmp.push_back({a, b});
    sig_rows.emplace_back(W, 0);
    for (int w = 0; w < W; w++) {
      uint64_t both = sig_rows[a][w] & sig_rows[b][w];
      while (both) {
        int r = w * 64 + __builtin_ctzll(both);
        both &= both - 1;
        auto &row = s.rows[r];
        // remove a, b
        std::vector<int> nr;
        nr.reserve(row.size());
        for (int x : row)
          if (x != a && x != b) nr.push_back(x);
        for (int u : nr) {
          bump(a, u, -1);
          bump(b, u, -1);
          bump(t, u, +1);
        }
        cnt[pkey(a, b)]--;
        nr.push_back(t);  // t is the largest id: stays sorted
        row.swap(nr);
        sig_rows[a][r >> 6] &= ~(1ull << (r & 63));
        sig_rows[b][r >> 6] &= ~(1ull << (r & 63));
        sig_rows[t][r >> 6] |= 1ull << (r & 63);
      }
    }
  }
  return s;
}

}  // namespace pmrc
