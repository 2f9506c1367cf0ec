#include "xorprog.hpp"

#include <algorithm>
#include <queue>
#include <tuple>
#include <unordered_map>

namespace pmrc {

long Slp::xor2() const {
  long c = 0;
  for (auto &t : tmp) c += (long)t.size() - 1;
  for (auto &r : rows)
    if (r.size() > 1) c += (long)r.size() - 1;
  return c;
}

long Slp::lop3() const {
  long c = 0;
  for (auto &t : tmp) c += ((long)t.size() - 1 + 1) / 2;
  for (auto &r : rows)
    if (r.size() > 1) c += ((long)r.size() - 1 + 1) / 2;
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

Slp cse3(int n_in, const std::vector<std::vector<int>> &rows_in, uint32_t seed) {
  uint64_t rng = 0x9E3779B97F4A7C15ull * (seed + 1);
  auto noise = [&]() -> double {  // [0, 0.5): breaks ties / explores near-best choices (seed != 0)
    if (!seed) return 0.0;
    rng = rng * 6364136223846793005ull + 1442695040888963407ull;
    return (double)(rng >> 40) / (double)(1ull << 24) * 0.5;
  };
  Slp s;
  s.n_in = n_in;
  s.rows = rows_in;
  for (auto &r : s.rows) std::sort(r.begin(), r.end());
  const int R = (int)s.rows.size();
  const int W = (R + 63) / 64;
  std::vector<std::vector<uint64_t>> sig_rows(n_in, std::vector<uint64_t>(W, 0));
  for (int r = 0; r < R; r++)
    for (int x : s.rows[r]) sig_rows[x][r >> 6] |= 1ull << (r & 63);
  std::unordered_map<uint64_t, int> cnt;
  cnt.reserve(1 << 15);
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
  const int K = 24;  // candidate pairs extended to triples per step
  std::vector<int> freq;
  while (true) {
    // top-K valid, distinct pairs
    std::vector<std::tuple<int, int, int>> cand;
    std::vector<std::tuple<int, int, int>> keep;
    while (!heap.empty() && (int)cand.size() < K) {
      auto e = heap.top();
      heap.pop();
      int c = std::get<0>(e), a = -std::get<1>(e), b = -std::get<2>(e);
      auto it = cnt.find(pkey(a, b));
      if (it == cnt.end() || it->second != c) continue;  // stale
      bool dup = false;
      for (auto &x : cand)
        if (std::get<1>(x) == a && std::get<2>(x) == b) dup = true;
      if (dup) continue;
      cand.push_back({c, a, b});
    }
    for (auto &x : cand) heap.emplace(std::get<0>(x), -std::get<1>(x), -std::get<2>(x));
    if (cand.empty()) break;
    double best = 0;
    std::vector<int> bops;
    const int nsig = (int)sig_rows.size();
    for (auto &x : cand) {
      int c = std::get<0>(x), a = std::get<1>(x), b = std::get<2>(x);
      if (c >= 3 && c * 0.5 - 1 + noise() > best) { best = c * 0.5 - 1; bops = {a, b}; }
      // best third signal among the rows containing a and b
      freq.assign(nsig, 0);
      int bc = -1, bcnt = 0;
      for (int w = 0; w < W; w++) {
        uint64_t both = sig_rows[a][w] & sig_rows[b][w];
        while (both) {
          int r = w * 64 + __builtin_ctzll(both);
          both &= both - 1;
          for (int u : s.rows[r]) {
            if (u == a || u == b) continue;
            if (++freq[u] > bcnt || (freq[u] == bcnt && u < bc)) { bcnt = freq[u]; bc = u; }
          }
        }
      }
      if (bcnt >= 2 && bcnt - 1.0 + noise() > best) {
        best = bcnt - 1.0;
        bops = {a, b, bc};
      }
    }
    if (bops.empty() || best <= 0) break;
    std::sort(bops.begin(), bops.end());
    const int t = n_in + (int)s.tmp.size();
    s.tmp.push_back(bops);
    sig_rows.emplace_back(W, 0);
    for (int w = 0; w < W; w++) {
      uint64_t all = ~0ull;
      for (int o : bops) all &= sig_rows[o][w];
      while (all) {
        int r = w * 64 + __builtin_ctzll(all);
        all &= all - 1;
        auto &row = s.rows[r];
        std::vector<int> nr;
        nr.reserve(row.size());
        for (int x : row)
          if (std::find(bops.begin(), bops.end(), x) == bops.end()) nr.push_back(x);
        for (int u : nr) {
          for (int o : bops) bump(o, u, -1);
          bump(t, u, +1);
        }
        for (size_t i = 0; i < bops.size(); i++)
          for (size_t j = i + 1; j < bops.size(); j++) cnt[pkey(bops[i], bops[j])]--;
        nr.push_back(t);
        row.swap(nr);
        for (int o : bops) sig_rows[o][r >> 6] &= ~(1ull << (r & 63));
        sig_rows[t][r >> 6] |= 1ull << (r & 63);
      }
    }
  }
  return s;
}

}  // namespace pmrc
