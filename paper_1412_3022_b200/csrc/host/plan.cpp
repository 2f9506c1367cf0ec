// Bitsliced sm_100a kernel generator + NVRTC JIT + launcher (see plan.hpp).
//
// Kernel shape:
//   * work item = (stripe t, 1024-byte chunk q, output group g); one warp per item, grid-stride
//     over items, adjacent warps of a CTA take the groups of the same chunk (their shared inputs
//     then hit L1/L2 instead of HBM);
//   * lane l owns byte positions [16l,16l+16) and [512+16l, 512+16l+16) of the chunk: two
//     coalesced 16-B vector loads per input block (a warp reads 1 KiB contiguous per block);
//   * the 8 words are transposed in registers (3 delta-swap stages, 8x8 bit transpose per byte
//     lane) into 8 bit planes, each holding bit b of 32 byte positions;
//   * GF(2^8) multiply-XOR = the group's GF(2) XOR network on planes (LOP3 after ptxas fusion),
//     generated with zero coefficients skipped and Paar CSE;
//   * output planes are transposed back and written with streaming 16-B stores.
#include "plan.hpp"

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>

#include "../../../include/pmrc.h"
#include "cudrv.hpp"

namespace pmrc {

unsigned long long &launch_counter() {
  static unsigned long long c = 0;
  return c;
}

namespace {

const char *kHeader = R"CUDA(
typedef unsigned int u32;
typedef unsigned long long u64;
// exchange the bits selected by ~m in a with the bits selected by m in b, shifted by s
// (one delta-swap stage of an 8x8 bit transpose, per byte lane)
static __device__ __forceinline__ void pm_sw(u32 &a, u32 &b, const int s, const u32 m) {
  // a' = m ? a : (b << s);  b' = m ? (a >> s) : b   -- one LOP3 mux each; the shifts are issued
  // as IMAD (left) and IMAD.HI (right) so they run on the FMA pipe, not the ALU pipe
  u32 bs, ar, na, nb;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(bs) : "r"(b), "r"(1u << s));
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(ar) : "r"(a), "r"(1u << (32 - s)));
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(na) : "r"(a), "r"(bs), "r"(m));
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(nb) : "r"(ar), "r"(b), "r"(m));
  a = na;
  b = nb;
}
// 8 words (32 bytes) <-> 8 bit planes; an involution
static __device__ __forceinline__ void pm_tr8(u32 &w0, u32 &w1, u32 &w2, u32 &w3, u32 &w4, u32 &w5, u32 &w6, u32 &w7) {
  pm_sw(w0, w4, 4, 0x0F0F0F0Fu); pm_sw(w1, w5, 4, 0x0F0F0F0Fu); pm_sw(w2, w6, 4, 0x0F0F0F0Fu); pm_sw(w3, w7, 4, 0x0F0F0F0Fu);
  pm_sw(w0, w2, 2, 0x33333333u); pm_sw(w1, w3, 2, 0x33333333u); pm_sw(w4, w6, 2, 0x33333333u); pm_sw(w5, w7, 2, 0x33333333u);
  pm_sw(w0, w1, 1, 0x55555555u); pm_sw(w2, w3, 1, 0x55555555u); pm_sw(w4, w5, 1, 0x55555555u); pm_sw(w6, w7, 1, 0x55555555u);
}
static __device__ __forceinline__ uint4 pm_ld(const unsigned char *p, bool v) {
  uint4 r = make_uint4(0u, 0u, 0u, 0u);
  if (v) r = __ldg(reinterpret_cast<const uint4 *>(p));
  return r;
}
static __device__ __forceinline__ void pm_st(unsigned char *p, bool v, u32 a, u32 b, u32 c, u32 d) {
  if (v) __stcs(reinterpret_cast<uint4 *>(p), make_uint4(a, b, c, d));
}
)CUDA";

struct Emitter {
  std::ostringstream s;
  int tmp_id = 0;
};

// bit rows of "multiply-accumulate coefficient c into the output": for output bit b, the set of
// input planes b' with M_c[b][b'] = 1
void coef_rows(uint8_t c, uint8_t rows[8]) { gf().bitmatrix(c, rows); }

std::string plane(const std::string &base, int b) { return base + "_" + std::to_string(b); }

// Emit loads + transposes of one plain input block into variables <name>_0..7
void emit_load(std::ostringstream &s, const std::string &name, int slot, int blk) {
  s << "    u32 " << name << "_0, " << name << "_1, " << name << "_2, " << name << "_3, " << name << "_4, "
    << name << "_5, " << name << "_6, " << name << "_7;\n";
  s << "    { const unsigned char *pp = (const unsigned char *)(R.ptr[" << slot << "] + t * R.stride[" << slot
    << "] + (u64)" << blk << " * S);\n";
  s << "      const uint4 va = pm_ld(pp + o0, v0), vb = pm_ld(pp + o1, v1);\n";
  s << "      " << name << "_0 = va.x; " << name << "_1 = va.y; " << name << "_2 = va.z; " << name << "_3 = va.w; "
    << name << "_4 = vb.x; " << name << "_5 = vb.y; " << name << "_6 = vb.z; " << name << "_7 = vb.w;\n";
  s << "      pm_tr8(" << name << "_0, " << name << "_1, " << name << "_2, " << name << "_3, " << name << "_4, "
    << name << "_5, " << name << "_6, " << name << "_7); }\n";
}

// Emit an XOR program: base signal i is named by base_names[i]; outputs into out_names (assign or
// accumulate).
void emit_slp(std::ostringstream &s, const Slp &p, const std::vector<std::string> &base_names,
              const std::vector<std::string> &out_names, bool accumulate, const std::string &tpref) {
  auto nm = [&](int sig) -> std::string {
    if (sig < p.n_in) return base_names[sig];
    return tpref + std::to_string(sig - p.n_in);
  };
  for (size_t i = 0; i < p.tmp.size(); i++)
    s << "    const u32 " << tpref << i << " = " << nm(p.tmp[i][0]) << " ^ " << nm(p.tmp[i][1]) << ";\n";
  for (size_t r = 0; r < p.rows.size(); r++) {
    const auto &row = p.rows[r];
    if (row.empty()) {
      if (!accumulate) s << "    " << out_names[r] << " = 0u;\n";
      continue;
    }
    s << "    " << out_names[r] << (accumulate ? " ^= " : " = ");
    for (size_t j = 0; j < row.size(); j++) s << (j ? " ^ " : "") << nm(row[j]);
    s << ";\n";
  }
}

Slp make_slp(int n_in, const std::vector<std::vector<int>> &rows, bool cse) {
  if (cse) return paar(n_in, rows);
  Slp s;
  s.n_in = n_in;
  s.rows = rows;
  return s;
}

}  // namespace

std::string generate_source(const PlanSpec &p, const GenOptions &o, GenStats &st) {
  st = GenStats();
  const int R = (int)p.outputs.size();
  const int C = (int)p.inputs.size();
  // ---- group output rows by support, then split into chunks of max_rows ----
  std::map<std::vector<int>, std::vector<int>> by_support;
  for (int r = 0; r < R; r++) {
    std::vector<int> sup;
    for (int c = 0; c < C; c++)
      if (p.A.at(r, c)) sup.push_back(c);
    by_support[sup].push_back(r);
  }
  struct Group {
    std::vector<int> rows, cols;
  };
  std::vector<Group> groups;
  for (auto &kv : by_support)
    for (size_t i = 0; i < kv.second.size(); i += o.max_rows) {
      Group g;
      g.cols = kv.first;
      for (size_t j = i; j < std::min(kv.second.size(), i + (size_t)o.max_rows); j++) g.rows.push_back(kv.second[j]);
      groups.push_back(g);
    }
  st.groups = (int)groups.size();

  std::ostringstream s;
  s << "// generated by libpmrc (plan.cpp) — bitsliced GF(2^8) region linear combination\n";
  s << kHeader;
  s << "struct Slots { u64 ptr[" << std::max(1, p.n_slots) << "]; u64 stride[" << std::max(1, p.n_slots) << "]; };\n";

  for (size_t g = 0; g < groups.size(); g++) {
    const Group &G = groups[g];
    const int m = (int)G.rows.size();
    s << "static __device__ __noinline__ void grp" << g
      << "(const Slots &R, const u64 S, const u64 t, const u64 o0, const u64 o1, const bool v0, const bool v1) {\n";
    std::vector<std::string> outs;
    for (int r = 0; r < m; r++)
      for (int b = 0; b < 8; b++) outs.push_back("o" + std::to_string(r) + "_" + std::to_string(b));
    s << "  u32 ";
    for (size_t i = 0; i < outs.size(); i++) s << (i ? ", " : "") << outs[i];
    s << ";\n";
    const int q = (int)G.cols.size();
    if (q == 0) {
      for (auto &n : outs) s << "  " << n << " = 0u;\n";
    }
    for (int b0 = 0; b0 < q; b0 += o.in_block) {
      const int b1 = std::min(q, b0 + o.in_block);
      s << "  {\n";
      std::vector<std::string> base;
      for (int ci = b0; ci < b1; ci++) {
        const int c = G.cols[ci];
        const InputDesc &in = p.inputs[c];
        std::string nm = "i" + std::to_string(c);
        if (in.terms.size() == 1 && in.terms[0].coef == 1) {
          emit_load(s, nm, in.terms[0].slot, in.terms[0].blk);
          st.loads += 2;
        } else {
          // derived input: x = sum_u coef_u * block_u (its own small XOR program)
          std::vector<std::string> dbase;
          std::vector<std::vector<int>> drows(8);
          for (size_t u = 0; u < in.terms.size(); u++) {
            std::string dn = nm + "d" + std::to_string(u);
            emit_load(s, dn, in.terms[u].slot, in.terms[u].blk);
            st.loads += 2;
            st.transposes++;
            uint8_t br[8];
            coef_rows(in.terms[u].coef, br);
            for (int bb = 0; bb < 8; bb++) {
              dbase.push_back(plane(dn, bb));
              for (int bp = 0; bp < 8; bp++)
                if ((br[bb] >> bp) & 1) drows[bb].push_back((int)u * 8 + bp);
            }
          }
          Slp ds = make_slp((int)dbase.size(), drows, o.cse);
          st.xor2 += ds.xor2();
          st.naive_lop3 += naive_lop3(drows);
          st.xor2_naive += make_slp((int)dbase.size(), drows, false).xor2();
          s << "    u32 " << nm << "_0, " << nm << "_1, " << nm << "_2, " << nm << "_3, " << nm << "_4, " << nm << "_5, "
            << nm << "_6, " << nm << "_7;\n";
          std::vector<std::string> dout;
          for (int bb = 0; bb < 8; bb++) dout.push_back(plane(nm, bb));
          emit_slp(s, ds, dbase, dout, false, nm + "t");
          st.transposes--;  // counted below once per input
        }
        st.transposes++;
        for (int b = 0; b < 8; b++) base.push_back(plane(nm, b));
      }
      // bit rows of this input block
      std::vector<std::vector<int>> rows(8 * m);
      for (int r = 0; r < m; r++)
        for (int ci = b0; ci < b1; ci++) {
          uint8_t c = p.A.at(G.rows[r], G.cols[ci]);
          if (!c) continue;
          uint8_t br[8];
          coef_rows(c, br);
          for (int b = 0; b < 8; b++)
            for (int bp = 0; bp < 8; bp++)
              if ((br[b] >> bp) & 1) rows[r * 8 + b].push_back((ci - b0) * 8 + bp);
        }
      Slp sl = make_slp((int)base.size(), rows, o.cse);
      st.xor2 += sl.xor2() + (b0 > 0 ? 8 * m : 0);
      st.naive_lop3 += naive_lop3(rows);
      st.xor2_naive += make_slp((int)base.size(), rows, false).xor2() + (b0 > 0 ? 8 * m : 0);
      emit_slp(s, sl, base, outs, b0 > 0, "t" + std::to_string(b0) + "_");
      s << "  }\n";
    }
    // transpose back and store
    for (int r = 0; r < m; r++) {
      const OutputDesc &od = p.outputs[G.rows[r]];
      std::string n = "o" + std::to_string(r);
      s << "  pm_tr8(" << n << "_0, " << n << "_1, " << n << "_2, " << n << "_3, " << n << "_4, " << n << "_5, " << n
        << "_6, " << n << "_7);\n";
      s << "  { unsigned char *pp = (unsigned char *)(R.ptr[" << od.slot << "] + t * R.stride[" << od.slot << "] + (u64)"
        << od.blk << " * S);\n";
      s << "    pm_st(pp + o0, v0, " << n << "_0, " << n << "_1, " << n << "_2, " << n << "_3);\n";
      s << "    pm_st(pp + o1, v1, " << n << "_4, " << n << "_5, " << n << "_6, " << n << "_7); }\n";
      st.transposes++;
    }
    s << "}\n";
  }
  const int NG = std::max(1, (int)groups.size());
  // Each CTA owns a tile of (warps per CTA) consecutive 1 KiB chunks of one stripe; every warp walks
  // all groups in the same order for its chunk, so the warps of an SM execute the same group code at
  // the same time (the straight-line XOR networks are large: instruction-cache reuse across warps
  // is what keeps the ALU fed) and a group's shared inputs were just read by the same warp (L1/L2).
  s << "extern \"C\" __global__ void __launch_bounds__(" << o.tpb << ", 1) pmrc_kernel(const __grid_constant__ Slots R, "
       "const u64 S, const u32 stripes, const u32 chunks) {\n";
  s << "  const u32 lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, W = blockDim.x >> 5;\n";
  s << "  const u32 tps = (chunks + W - 1) / W;\n";
  s << "  const u32 tiles = stripes * tps;\n";
  s << "  for (u32 tile = blockIdx.x; tile < tiles; tile += gridDim.x) {\n";
  s << "    const u64 t = tile / tps;\n";
  s << "    const u32 q = (tile - (u32)t * tps) * W + warp;\n";
  s << "    const u64 o0 = (u64)q * 1024u + lane * 16u, o1 = o0 + 512u;\n";
  s << "    const bool v0 = q < chunks && o0 < S, v1 = q < chunks && o1 < S;\n";
  for (size_t g = 0; g < groups.size(); g++) s << "    grp" << g << "(R, S, t, o0, o1, v0, v1);\n";
  s << "  }\n}\n";
  return s.str();
}

namespace {
std::string cu_err(CUresult r) {
  const char *s = nullptr;
  if (drv().GetErrorString) drv().GetErrorString(r, &s);
  return s ? s : "unknown CUDA driver error";
}
}  // namespace

int build_kernel(const PlanSpec &p, const GenOptions &o, Kernel &k, std::string &err) {
  auto t0 = std::chrono::steady_clock::now();
  k = Kernel();
  k.source = generate_source(p, o, k.stats);
  k.n_slots = std::max(1, p.n_slots);
  k.n_groups = std::max(1, k.stats.groups);
  k.tpb = o.tpb;
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, k.source.c_str(), "pmrc_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    err = "nvrtcCreateProgram failed";
    return PMRC_EJIT;
  }
  const char *opts[] = {"-arch=sm_100a", "-lineinfo", "-default-device", "--std=c++17"};
  nvrtcResult rc = nvrtcCompileProgram(prog, 4, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    err = std::string("NVRTC: ") + nvrtcGetErrorString(rc) + "\n" + log.substr(0, 4000);
    nvrtcDestroyProgram(&prog);
    return PMRC_EJIT;
  }
  size_t nc = 0;
  nvrtcGetCUBINSize(prog, &nc);
  std::vector<char> cubin(nc);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  auto t1 = std::chrono::steady_clock::now();
  k.compile_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();

  // load into the current context (the runtime's primary context for the current device)
  if (cudaFree(0) != cudaSuccess) {
    err = "no usable CUDA device";
    cudaGetLastError();
    return PMRC_ECUDA;
  }
  const Drv &D = drv();
  if (!D.ok) { err = "CUDA driver (libcuda.so.1) not available"; return PMRC_ECUDA; }
  CUmodule mod;
  CUresult cr = D.ModuleLoadData(&mod, cubin.data());
  if (cr != CUDA_SUCCESS) { err = "cuModuleLoadData: " + cu_err(cr); return PMRC_ECUDA; }
  CUfunction fn;
  cr = D.ModuleGetFunction(&fn, mod, "pmrc_kernel");
  if (cr != CUDA_SUCCESS) { D.ModuleUnload(mod); err = "cuModuleGetFunction: " + cu_err(cr); return PMRC_ECUDA; }
  k.module = mod;
  k.function = fn;
  int regs = 0;
  D.FuncGetAttribute(&regs, CU_FUNC_ATTRIBUTE_NUM_REGS, fn);
  k.regs = regs;
  int nb = 1;
  D.OccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, k.tpb, 0);
  k.blocks_per_sm = std::max(1, nb);
  CUdevice dev;
  D.CtxGetDevice(&dev);
  int sms = 148;
  D.DeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev);
  k.sms = sms;
  return PMRC_OK;
}

void free_kernel(Kernel &k) {
  if (k.module && drv().ok) drv().ModuleUnload((CUmodule)k.module);
  k.module = nullptr;
  k.function = nullptr;
}

int launch_kernel(const Kernel &k, const uint64_t *ptrs, const uint64_t *strides, size_t S, size_t stripes,
                  void *stream, std::string &err) {
  if (S == 0 || stripes == 0) return PMRC_OK;
  const uint64_t chunks64 = (S + 1023) / 1024;
  if (chunks64 > 0xFFFFFFFFull) { err = "S too large"; return PMRC_EINVAL; }
  const uint32_t chunks = (uint32_t)chunks64;
  // items = stripes * chunks * groups must fit in 32 bits: split launches over stripe ranges
  const uint64_t per_stripe = (uint64_t)chunks;
  const uint64_t max_stripes = std::max<uint64_t>(1, 0xFFFFFFF0ull / per_stripe);
  std::vector<uint64_t> buf(2 * k.n_slots);
  for (size_t s0 = 0; s0 < stripes; s0 += max_stripes) {
    const uint32_t ns = (uint32_t)std::min<uint64_t>(max_stripes, stripes - s0);
    for (int i = 0; i < k.n_slots; i++) {
      buf[i] = ptrs[i] + s0 * strides[i];
      buf[k.n_slots + i] = strides[i];
    }
    uint64_t S64 = S;
    void *args[] = {buf.data(), &S64, (void *)&ns, (void *)&chunks};
    const uint64_t warps_per_block = k.tpb / 32;
    const uint64_t tiles = (uint64_t)ns * ((chunks + warps_per_block - 1) / warps_per_block);
    uint64_t grid = (uint64_t)k.sms * k.blocks_per_sm;
    grid = std::min<uint64_t>(grid, tiles);
    grid = std::max<uint64_t>(grid, 1);
    CUresult cr = drv().LaunchKernel((CUfunction)k.function, (unsigned)grid, 1, 1, k.tpb, 1, 1, 0, (CUstream)stream, args,
                                 nullptr);
    if (cr != CUDA_SUCCESS) { err = "cuLaunchKernel: " + cu_err(cr); return PMRC_ECUDA; }
    launch_counter()++;
  }
  return PMRC_OK;
}

}  // namespace pmrc
