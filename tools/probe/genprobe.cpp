// Host-only probe: build a code, generate its encode kernel source, print XOR statistics.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include "../../paper_1412_3022_b200/csrc/host/construct.hpp"
#include "../../paper_1412_3022_b200/csrc/host/plan.hpp"
using namespace pmrc;
int main(int argc, char **argv) {
  int kind = argc > 1 ? atoi(argv[1]) : 0, k = argc > 2 ? atoi(argv[2]) : 8, n = argc > 3 ? atoi(argv[3]) : 16;
  int mr = argc > 4 ? atoi(argv[4]) : 8, ib = argc > 5 ? atoi(argv[5]) : 16, cse = argc > 6 ? atoi(argv[6]) : 1;
  int d = kind == 2 ? 2 * k - 2 : (kind == 3 ? k : 2 * k - 2);
  CodeDef c; std::string err;
  int rc = build_code(kind, k, d, n, 8, c, err);
  if (rc) { printf("build_code rc=%d %s\n", rc, err.c_str()); return 1; }
  PlanSpec p; p.n_slots = 2;
  for (int i = 0; i < c.B; i++) p.inputs.push_back({{{0, i, 1}}});
  for (int r = 0; r < c.P; r++) p.outputs.push_back({1, r});
  p.A = c.Gpp;
  GenOptions o; o.max_rows = mr; o.in_block = ib; o.cse = cse;
  if (argc > 7) {  // key=value,... (team, warps, chunk_loop)
    std::string g = argv[7]; size_t pos = 0;
    while (pos < g.size()) {
      size_t e = g.find(',', pos); if (e == std::string::npos) e = g.size();
      std::string kv = g.substr(pos, e - pos); size_t eq = kv.find('=');
      if (eq != std::string::npos) { std::string k = kv.substr(0, eq); int v = atoi(kv.c_str() + eq + 1);
        if (k == "team") o.team = v; if (k == "warps") o.warps = v; if (k == "chunk_loop") o.chunk_loop = v; }
      pos = e + 1;
    }
  }
  if (o.warps == 0) o.warps = 16;
  GenStats st;
  std::string src = generate_source(p, o, st);
  long nnz = 0; for (auto v : c.Gpp.a) nnz += v != 0;
  double srcB = 32.0 * c.B;  // source bytes per 32 positions
  printf("kind=%d k=%d n=%d B=%d P=%d nnz=%ld groups=%d naive_lop3=%ld (%.3f/B) xor2_naive=%ld xor2_cse=%ld (%.3f/B) transposes=%d (%.3f/B @24 ALU) repair_complete=%d\n",
         kind, k, n, c.B, c.P, nnz, st.groups, st.naive_lop3, st.naive_lop3 / srcB, st.xor2_naive, st.xor2, st.xor2 / srcB,
         st.transposes, st.transposes * 24 / srcB, (int)c.repair_complete);
  std::ofstream("/tmp/pmrc_gen.cu") << src;
  return 0;
}
