// GF(2^8) arithmetic for the host side of libpmrc (construction, inversion, plan building).
// Reading R1: primitive polynomial x^8+x^4+x^3+x^2+1 (0x11D), generator g = 2.
// Product tables are built from carry-less multiplication + reduction (independent of the
// oracle's log/antilog tables).
#pragma once
#include <cstdint>
#include <vector>

namespace pmrc {

struct GF256 {
  uint8_t mul_t[256][256];
  uint8_t inv_t[256];
  uint8_t pow_g[255];  // g^e, e in [0,255)

  GF256() {
    for (int a = 0; a < 256; a++)
      for (int b = 0; b < 256; b++) {
        unsigned r = 0;
        for (int i = 0; i < 8; i++)
          if ((b >> i) & 1) r ^= (unsigned)a << i;
        for (int bit = 14; bit >= 8; bit--)
          if ((r >> bit) & 1) r ^= 0x11Du << (bit - 8);
        mul_t[a][b] = (uint8_t)r;
      }
    inv_t[0] = 0;
    for (int a = 1; a < 256; a++)
      for (int b = 1; b < 256; b++)
        if (mul_t[a][b] == 1) { inv_t[a] = (uint8_t)b; break; }
    uint8_t x = 1;
    for (int e = 0; e < 255; e++) { pow_g[e] = x; x = mul_t[x][2]; }
  }
  uint8_t mul(uint8_t a, uint8_t b) const { return mul_t[a][b]; }
  uint8_t inv(uint8_t a) const { return inv_t[a]; }
  uint8_t div(uint8_t a, uint8_t b) const { return mul_t[a][inv_t[b]]; }
  uint8_t gexp(long e) const { return pow_g[((e % 255) + 255) % 255]; }
  // 8x8 GF(2) matrix of "multiply by c": bit b of (c * x) = XOR_{b'} M[b][b'] x_{b'};
  // column b' is c * 2^{b'}.  Returned as rows: row b is an 8-bit mask over b'.
  void bitmatrix(uint8_t c, uint8_t rows[8]) const {
    for (int b = 0; b < 8; b++) rows[b] = 0;
    for (int bp = 0; bp < 8; bp++) {
      uint8_t col = mul_t[c][1u << bp];
      for (int b = 0; b < 8; b++)
        if ((col >> b) & 1) rows[b] |= (uint8_t)(1u << bp);
    }
  }
};

const GF256 &gf();

// GF(2^16) for the w = 16 codes: x^16+x^12+x^3+x+1 (0x1100B), g = 2 (reading
// R1b).  Log/antilog tables built by shift-and-reduce (x * 2 each step).
struct GF65536 {
  std::vector<uint16_t> exp_t;  // 2 * 65535 entries
  std::vector<int> log_t;       // 65536 entries, log_t[0] = -1
  GF65536() : exp_t(2 * 65535), log_t(65536, -1) {
    uint32_t x = 1;
    for (int e = 0; e < 65535; e++) {
      exp_t[e] = (uint16_t)x;
      log_t[x] = e;
      x <<= 1;
      if (x & 0x10000u) x ^= 0x1100Bu;
    }
    for (int e = 65535; e < 2 * 65535; e++) exp_t[e] = exp_t[e - 65535];
  }
  uint16_t mul(uint16_t a, uint16_t b) const { return (a && b) ? exp_t[log_t[a] + log_t[b]] : 0; }
  uint16_t inv(uint16_t a) const { return exp_t[(65535 - log_t[a]) % 65535]; }
  uint16_t div(uint16_t a, uint16_t b) const { return mul(a, inv(b)); }
  uint16_t gexp(long e) const { return exp_t[((e % 65535) + 65535) % 65535]; }
  // 16x16 GF(2) matrix of "multiply by c": row b is a 16-bit mask over input bits b'
  void bitmatrix(uint16_t c, uint32_t rows[16]) const {
    for (int b = 0; b < 16; b++) rows[b] = 0;
    for (int bp = 0; bp < 16; bp++) {
      const uint16_t col = mul(c, (uint16_t)(1u << bp));
      for (int b = 0; b < 16; b++)
        if ((col >> b) & 1) rows[b] |= 1u << bp;
    }
  }
};
const GF65536 &gf16();

// dense byte matrix, row-major
struct Mat {
  int r = 0, c = 0;
  std::vector<uint8_t> a;
  Mat() {}
  Mat(int r_, int c_) : r(r_), c(c_), a((size_t)r_ * c_, 0) {}
  uint8_t &at(int i, int j) { return a[(size_t)i * c + j]; }
  uint8_t at(int i, int j) const { return a[(size_t)i * c + j]; }
};

Mat matmul(const Mat &A, const Mat &B);
// Gauss-Jordan inverse; returns false if singular.
bool invert(const Mat &A, Mat &out);
int rank(const Mat &A);

}  // namespace pmrc
