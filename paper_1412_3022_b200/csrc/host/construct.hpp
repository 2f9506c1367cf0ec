// Code construction on the host: parameters, index matrix L
// (P:75-83), encoding matrix Psi (R5, R12), linearised generator G,
// systematic G' = G Gtilde^{-1} and the parity part G''.
#pragma once
#include <string>
#include <vector>

#include "gf256.hpp"

namespace pmrc {

enum Kind { KIND_MSR_SPARSE = 0, KIND_MSR_VANILLA = 1, KIND_MBR = 2, KIND_RS = 3, KIND_MSR_SPARSE_N2K = 4 };

struct CodeDef {
  int kind = 0, n = 0, k = 0, d = 0, alpha = 0, B = 0, P = 0;
  Mat psi;                     // n x d (RS: n x k)
  std::vector<uint8_t> lambda; // n (MSR)
  Mat L;                       // index matrix stored in a byte-free int form below
  std::vector<int> Lidx;       // Lrows x Lcols, 1-based data index, 0 = structural zero
  int Lrows = 0, Lcols = 0;
  Mat G;     // n alpha x B
  Mat Gsys;  // G'
  Mat Gpp;   // P x B
  Mat Gti;   // Gtilde^{-1} (B x B; MSR / RS), the precode of P:112
  bool repair_complete = true;

  // data block held by systematic node i, symbol j (MSR/RS: i*alpha+j; MBR: L_{i,j}-1)
  int sys_block(int i, int j) const;
};

// returns 0 or a PMRC_E* code; err receives a description
int build_code(int kind, int k, int d, int n, int w, CodeDef &out, std::string &err);
// GF(2^16) sparse MSR (w = 16): alpha, B and the systematic parity matrix G'' ((n-k) alpha x B)
int build_gpp16(int k, int d, int n, int &alpha, int &B, std::vector<uint16_t> &gpp, std::string &err,
                std::vector<uint16_t> *psi_out = nullptr, std::vector<uint16_t> *lam_out = nullptr);

}  // namespace pmrc
