// GF(2) straight-line XOR programs for bitsliced GF(2^8) region linear combinations.
//
// A GF(2^8) coefficient c acts on a byte as an 8x8 GF(2) matrix (column b' = c * 2^{b'}), so a
// group of m output blocks fed by q input blocks is a (8m) x (8q) bit matrix applied to bit planes
// (SURVEY §8(a) "bit-sliced" formulation).  Zero coefficients contribute no columns (the paper's
// sparsification, applied at kernel-generation time).  We shorten the XOR network with
// Paar's greedy common-subexpression elimination (repeatedly materialise the pair of signals that
// co-occurs in most rows); the result is exact (GF(2) identities), so outputs are bit-identical to
// the plain matrix product.
#pragma once
#include <array>
#include <cstdint>
#include <vector>

namespace pmrc {

struct Slp {
  int n_in = 0;                          // base signals 0..n_in-1
  std::vector<std::vector<int>> tmp;     // signal n_in+i = XOR of tmp[i] (2 or 3 signals)
  std::vector<std::vector<int>> rows;    // each output = XOR of these signals (empty = 0)
  long xor2() const;                     // 2-input XOR count
  long lop3() const;                     // 3-input LOP3 count (ternary trees)
};

// rows_in[r] = sorted list of base signals XORed into output r
Slp paar(int n_in, const std::vector<std::vector<int>> &rows_in);

// LOP3-aware CSE: greedily materialise the signal pair (used by >= 3 rows, saves ~r/2 - 1 LOP3) or
// triple (used by >= 2 rows, saves r - 1) with the best saving; triples are found by extending the
// top pairs with the best third signal among the rows that contain them.
// seed != 0 randomises near-ties (restarts: keep the cheapest of several seeds).
Slp cse3(int n_in, const std::vector<std::vector<int>> &rows_in, uint32_t seed = 0);

// naive 3-input-LOP3 count of a bit matrix row set: sum ceil((ones-1)/2)
long naive_lop3(const std::vector<std::vector<int>> &rows);

}  // namespace pmrc
