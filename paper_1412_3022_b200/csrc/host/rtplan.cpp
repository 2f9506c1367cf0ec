// Host side of the runtime-coefficient kernel (see rtplan.hpp and csrc/rt/rlc.cu).
#include "rtplan.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>

#include "../../../include/pmrc.h"
#include "../rt/rlc.hpp"

namespace pmrc {

using pmrc_rt::RlcArgs;
using pmrc_rt::RlcHdr;

pmrc_rt::RlcShape rt_shape(int n_out, const GenOptions &o) {
  // R rows x V words of accumulators per thread, G row groups of GT threads per CTA (a pass covers
  // G R rows; measured, profiles/r02):
  //   <= 8 rows (repair, projections, RS encode): (8, 4, 1, 256), two CTAs per SM
  //   more (decode, encode): (8, 4, 2, 256), 16 rows per pass (measured against it and slower:
  //   V = 2 with 3 or 7 groups -- twice the per-word overhead; 16 rows x 2 words in one group,
  //   which saves the second group's selectors: config-4 decode 2.58 -> 2.85 ms, repair 0.94 -> 1.37)
  // (rt_groups overrides for experiments; tg is set per launch from the plans)
  //   R = 7 or 8: the one with fewer passes, then fewer row slots (rows past n_out of a short last
  //   row block are computed and never stored); ties keep 8 (the k = 8 sparse-MSR encode's 8-row
  //   symbol groups fill 8-row blocks).  MSR k = 8 repair (7 rows) and config-4 decodes of 4
  //   missing nodes (28 rows) take R = 7.
  const int G = o.rt_groups == 1 || o.rt_groups == 2 ? o.rt_groups : (n_out <= 8 ? 1 : 2);
  auto cost = [&](int R) {
    const int blocks = (std::max(1, n_out) + R - 1) / R, passes = (blocks + G - 1) / G;
    return std::make_pair(passes, blocks * R);
  };
  int R = cost(7) < cost(8) ? 7 : 8;
  if (o.rt_rows == 7 || o.rt_rows == 8) R = o.rt_rows;
  return pmrc_rt::RlcShape{R, 4, G, 256, false};
}

// PRMT tables of coefficient c (rlc.cu): T0[j] = c*j, T1[j] = c*(j<<3) (j < 8), T2[j] = c*(j<<6) (j < 4),
// little-endian bytes: (T0a, T0b, T1a, T1b) and T2
static void tables(uint8_t c, uint32_t *a4, uint32_t *b1) {
  const GF256 &F = gf();
  uint8_t t0[8], t1[8], t2[4];
  for (int j = 0; j < 8; j++) {
    t0[j] = F.mul(c, (uint8_t)j);
    t1[j] = F.mul(c, (uint8_t)(j << 3));
  }
  for (int j = 0; j < 4; j++) t2[j] = F.mul(c, (uint8_t)(j << 6));
  auto pk = [](const uint8_t *b) {
    return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
  };
  a4[0] = pk(t0);
  a4[1] = pk(t0 + 4);
  a4[2] = pk(t1);
  a4[3] = pk(t1 + 4);
  *b1 = pk(t2);
}

int rt_build(const PlanSpec &p, int R, int G, RtPlan &out, std::string &err) {
  if (p.w != 8) {
    err = "runtime-coefficient kernel: GF(2^8) plans only";
    return PMRC_EUNSUPPORTED;
  }
  if (p.n_slots > pmrc_rt::kRlcMaxSlots) {
    err = "runtime-coefficient kernel: too many slots";
    return PMRC_EUNSUPPORTED;
  }
  const int n_in = (int)p.inputs.size(), n_out = (int)p.outputs.size();
  int n_terms = 0;
  for (const auto &in : p.inputs) n_terms += (int)in.terms.size();
  if (n_in == 0 || n_out == 0 || n_in > 65535 || n_terms > 65535) {
    err = "runtime-coefficient kernel: bad plan size";
    return PMRC_EUNSUPPORTED;
  }
  const int n_rb = (n_out + R - 1) / R;  // row blocks of R rows
  const int n_pass = (n_rb + G - 1) / G; // a pass runs G row blocks
  // row order: rows of equal support side by side, densest first (sparse MSR encode: the n-k rows
  // of a PM symbol index share their support, so every R-row block is all or nothing per input);
  // the kernel runs a block without per-row branches when every row of it reads the input
  std::vector<int> ord(n_out);
  for (int r = 0; r < n_out; r++) ord[r] = r;
  {
    std::vector<std::vector<uint8_t>> sup(n_out, std::vector<uint8_t>(n_in));
    std::vector<int> cnt(n_out, 0);
    for (int r = 0; r < n_out; r++)
      for (int i = 0; i < n_in; i++) cnt[r] += (sup[r][i] = p.A.at(r, i) != 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
      if (cnt[x] != cnt[y]) return cnt[x] > cnt[y];
      return sup[x] > sup[y];
    });
  }
  std::vector<uint32_t> masks((size_t)n_in * n_rb, 0u);
  long nnz = 0;
  for (int i = 0; i < n_in; i++)
    for (int r = 0; r < n_out; r++)
      if (p.A.at(ord[r], i)) {
        nnz++;
        masks[(size_t)i * n_rb + r / R] |= 1u << (r % R);
      }
  // pass sequences: pass pp streams every term of each input that a row of its G row blocks reads
  std::vector<int> tstart(n_in + 1, 0);
  for (int i = 0; i < n_in; i++) tstart[i + 1] = tstart[i] + (int)p.inputs[i].terms.size();
  std::vector<uint32_t> pstart(n_pass + 1, 0), seq;
  for (int pp = 0; pp < n_pass; pp++) {
    pstart[pp] = (uint32_t)seq.size();
    for (int i = 0; i < n_in; i++) {
      bool used = false;
      for (int rb = pp * G; rb < std::min(n_rb, pp * G + G); rb++) used |= masks[(size_t)i * n_rb + rb] != 0;
      if (used)
        for (int q = tstart[i]; q < tstart[i + 1]; q++) seq.push_back((uint32_t)q);
    }
  }
  pstart[n_pass] = (uint32_t)seq.size();
  // layout (words): header | ttabA 4*n_terms | ttabB n_terms | terms 2*n_terms | outs 2*n_out |
  //                 masks n_in*n_rb | pstart n_pass+1 | seq | (16-B aligned) tabA 4*n_in*n_out | tabB n_in*n_out
  RlcHdr h = {};
  h.magic = pmrc_rt::kRlcMagic;
  h.n_in = n_in;
  h.n_out = n_out;
  h.n_terms = n_terms;
  h.R = R;
  h.n_rb = n_rb;
  h.G = G;
  h.n_pass = n_pass;
  h.seq_len = (uint32_t)seq.size();
  uint32_t w = sizeof(RlcHdr) / 4;
  h.off_ttabA = w;
  w += 4u * n_terms;
  h.off_ttabB = w;
  w += n_terms;
  h.off_terms = w;
  w += 2u * n_terms;
  h.off_outs = w;
  w += 2u * n_out;
  h.off_masks = w;
  w += (uint32_t)masks.size();
  h.off_pstart = w;
  w += (uint32_t)pstart.size();
  h.off_seq = w;
  w += (uint32_t)seq.size();
  w = (w + 3u) & ~3u;  // tabA is read as uint4
  h.off_tabA = w;
  w += 4u * n_in * n_out;
  h.off_tabB = w;
  w += (uint32_t)n_in * n_out;
  h.words = w;
  h.smem_words = w;
  if (w > (uint32_t)pmrc_rt::kRlcMaxPlanWords) {
    // tables too large for shared memory: the kernel reads them from the blob in device memory
    h.flags |= pmrc_rt::kRlcGlobalTables;
    h.smem_words = h.off_tabA;
    if (h.smem_words > (uint32_t)pmrc_rt::kRlcMaxPlanWords) {
      err = "runtime-coefficient kernel: plan wiring too large (" + std::to_string(h.smem_words * 4) + " bytes)";
      return PMRC_EUNSUPPORTED;
    }
  }
  std::vector<uint32_t> b(w, 0u);
  for (int i = 0; i < n_in; i++)
    for (int r = 0; r < n_out; r++) {
      const uint8_t c = p.A.at(ord[r], i);
      if (c) tables(c, &b[h.off_tabA + 4 * ((size_t)i * n_out + r)], &b[h.off_tabB + (size_t)i * n_out + r]);
    }
  std::copy(masks.begin(), masks.end(), b.begin() + h.off_masks);
  std::copy(pstart.begin(), pstart.end(), b.begin() + h.off_pstart);
  std::copy(seq.begin(), seq.end(), b.begin() + h.off_seq);
  int q = 0, n_plain = 0;
  bool single = true;  // every input is one term
  for (int i = 0; i < n_in; i++) {
    const auto &terms = p.inputs[i].terms;
    single &= terms.size() == 1;
    for (size_t j = 0; j < terms.size(); j++, q++) {
      const Term &t = terms[j];
      if (t.slot < 0 || t.slot >= p.n_slots || t.blk < 0 || t.blk > 65535 || t.coef == 0 || t.coef > 255) {
        err = "runtime-coefficient kernel: bad term";
        return PMRC_EUNSUPPORTED;
      }
      uint32_t w0 = (uint32_t)t.slot;
      if (j + 1 == terms.size()) w0 |= 0x40000000u;
      if (t.coef == 1) {
        w0 |= 0x80000000u;
        n_plain++;
      } else tables((uint8_t)t.coef, &b[h.off_ttabA + 4 * q], &b[h.off_ttabB + q]);
      b[h.off_terms + 2 * q] = w0;
      b[h.off_terms + 2 * q + 1] = (uint32_t)t.blk | ((uint32_t)i << 16);
    }
  }
  // the kernel's loop for this term structure (rlc.cu)
  if (single && n_plain == n_terms) h.flags |= pmrc_rt::kRlcDirect;
  if (n_plain == 0) h.flags |= pmrc_rt::kRlcNoPlain;
  for (int r = 0; r < n_out; r++) {
    const OutputDesc &o = p.outputs[ord[r]];
    if (o.slot < 0 || o.slot >= p.n_slots || o.blk < 0) {
      err = "runtime-coefficient kernel: bad output";
      return PMRC_EUNSUPPORTED;
    }
    b[h.off_outs + 2 * r] = (uint32_t)o.slot;
    b[h.off_outs + 2 * r + 1] = (uint32_t)o.blk;
  }
  memcpy(b.data(), &h, sizeof h);
  rt_free(out);
  out.blob = std::move(b);
  out.R = R;
  out.G = G;
  out.n_in = n_in;
  out.n_out = n_out;
  out.n_terms = n_terms;
  out.nnz = nnz;
  return PMRC_OK;
}

void rt_free(RtPlan &p) {
  if (p.dev) cudaFree(p.dev);
  if (p.ready) cudaEventDestroy((cudaEvent_t)p.ready);
  p.dev = nullptr;
  p.ready = nullptr;
}

// estimated ALU work of one tile word of a plan (the batch launches balance CTAs by it): the
// selectors of every streamed input (per row group), the projections of coefficient terms (per row
// group), and the row MACs
double rt_cost(const RtPlan &p) {
  const uint32_t *b = p.blob.data();
  const RlcHdr *h = (const RlcHdr *)b;
  double c = 5.0 * (double)p.nnz;
  for (uint32_t e = 0; e < h->seq_len; e++) {
    const uint32_t j = b[h->off_seq + e], w0 = b[h->off_terms + 2 * j];
    if (!(w0 & 0x80000000u)) c += 8.0 * h->G;  // coefficient term: selectors + product
    if (w0 & 0x40000000u) c += 8.0 * h->G;     // input complete: its selectors
    c += 2.0;                                  // staging
  }
  return c;
}

static int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 148;
  }
  return n;
}

int rt_launch(const std::vector<RtPlan *> &plans, const uint16_t *stripe_plan, const uint64_t *ptrs,
              const uint64_t *strides, int n_slots, size_t S, size_t stripes, const pmrc_rt::RlcShape &sh,
              void *stream, int max_ctas, std::string &err) {
  if (S == 0 || stripes == 0) return PMRC_OK;
  if (plans.empty() || n_slots > pmrc_rt::kRlcMaxSlots) {
    err = "rt_launch: bad arguments";
    return PMRC_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  unsigned max_words = 0;
  bool tg = false;
  for (RtPlan *p : plans) {
    tg |= (p->blob[offsetof(RlcHdr, flags) / 4] & pmrc_rt::kRlcGlobalTables) != 0;
    if (p->R != sh.R || (int)p->blob[offsetof(RlcHdr, G) / 4] != sh.G) {
      err = "rt_launch: plans of one launch must share their shape";
      return PMRC_EINVAL;
    }
    max_words = std::max(max_words, p->blob[offsetof(RlcHdr, smem_words) / 4]);
    if (!p->dev) {
      const size_t nb = p->blob.size() * 4;
      if (cudaMalloc(&p->dev, nb) != cudaSuccess) {
        cudaGetLastError();
        p->dev = nullptr;
        err = "cudaMalloc(plan)";
        return PMRC_ENOMEM;
      }
      // the host blob lives in the cached plan, so the async copy's source outlives it; the event
      // orders later launches on other streams after the upload
      if (cudaMemcpyAsync(p->dev, p->blob.data(), nb, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaEventCreateWithFlags((cudaEvent_t *)&p->ready, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventRecord((cudaEvent_t)p->ready, st) != cudaSuccess) {
        err = std::string("plan upload: ") + cudaGetErrorString(cudaGetLastError());
        return PMRC_ECUDA;
      }
    } else if (p->ready && cudaStreamWaitEvent(st, (cudaEvent_t)p->ready, 0) != cudaSuccess) {
      err = std::string("plan upload wait: ") + cudaGetErrorString(cudaGetLastError());
      return PMRC_ECUDA;
    }
  }
  RlcArgs a;
  memset(&a, 0, sizeof a);
  a.S = S;
  a.stripes = stripes;
  a.max_words = max_words;
  a.n_slots = (unsigned)n_slots;
  a.sh3 = 1u << 29;
  a.sh6 = 1u << 26;
  a.sh12 = 1u << 20;
  for (int i = 0; i < n_slots; i++) {
    a.slot_ptr[i] = ptrs[i];
    a.slot_stride[i] = strides[i];
  }
  const uint64_t TP = (uint64_t)sh.GT * sh.V * 4;
  const uint64_t tiles = (S + TP - 1) / TP, items = tiles * (uint64_t)stripes;
  pmrc_rt::RlcShape shx = sh;
  shx.tg = tg;
  int per_sm = pmrc_rt::rlc_ctas_per_sm(shx, max_words);
  if (per_sm < 1) {
    err = "runtime-coefficient kernel does not fit on an SM (plan too large)";
    return PMRC_EUNSUPPORTED;
  }
  uint64_t grid = (uint64_t)sm_count() * per_sm;
  if (max_ctas > 0) grid = std::min<uint64_t>(grid, (uint64_t)max_ctas);
  grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, items));
  void *scratch = nullptr;
  if (stripe_plan) {
    const size_t np = plans.size();
    for (size_t t = 0; t < stripes; t++) {
      if (stripe_plan[t] >= np && stripe_plan[t] != 0xFFFF) {  // 0xFFFF: nothing to compute in stripe t
        err = "rt_launch: stripe plan index out of range";
        return PMRC_EINVAL;
      }
    }
    // CTA item ranges of equal estimated cost (ALU work per tile word of each stripe's plan)
    std::vector<double> pcost(np);
    for (size_t i = 0; i < np; i++) pcost[i] = rt_cost(*plans[i]);
    std::vector<uint64_t> bounds(grid + 1, items);
    double total = 0;
    for (size_t t = 0; t < stripes; t++) total += stripe_plan[t] == 0xFFFF ? 0.0 : pcost[stripe_plan[t]] * tiles;
    bounds[0] = 0;
    {
      // walk the stripes (O(stripes + grid)): boundary b goes after the first item at which the
      // cumulative cost reaches b / grid of the total; items of one stripe cost the same
      double cum = 0;
      uint64_t b = 1;
      for (size_t t = 0; t < stripes && b < grid; t++) {
        const double c = stripe_plan[t] == 0xFFFF ? 0.0 : pcost[stripe_plan[t]];
        if (c <= 0.0) continue;
        while (b < grid) {
          const double need = total * (double)b / (double)grid - cum;  // cost still missing for b
          const double jn = std::ceil(need / c - 1e-9);                   // items of stripe t it takes
          if (jn > (double)tiles) break;
          bounds[b++] = t * tiles + (uint64_t)std::max(1.0, jn);
        }
        cum += c * (double)tiles;
      }
    }
    // per-call launch tables in stream-ordered memory: plan addresses, the stripes' plan indices, the
    // CTA item bounds
    const size_t off_b = (np * 8 + stripes * 2 + 7) & ~(size_t)7, bytes = off_b + (grid + 1) * 8;
    std::vector<uint8_t> host(bytes, 0);
    for (size_t i = 0; i < np; i++) {
      const uint64_t d = (uint64_t)(uintptr_t)plans[i]->dev;
      memcpy(host.data() + 8 * i, &d, 8);
    }
    memcpy(host.data() + 8 * np, stripe_plan, stripes * 2);
    memcpy(host.data() + off_b, bounds.data(), (grid + 1) * 8);
    if (cudaMallocAsync(&scratch, bytes, st) != cudaSuccess) {
      cudaGetLastError();
      err = "cudaMallocAsync(launch tables)";
      return PMRC_ENOMEM;
    }
    // pageable source: staged before cudaMemcpyAsync returns, so `host` may go out of scope
    if (cudaMemcpyAsync(scratch, host.data(), bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) {
      err = std::string("launch tables: ") + cudaGetErrorString(cudaGetLastError());
      cudaFreeAsync(scratch, st);
      return PMRC_ECUDA;
    }
    a.plan_ptrs = (const unsigned long long *)scratch;
    a.stripe_plan = (const uint16_t *)((uint8_t *)scratch + 8 * np);
    a.item_bounds = (const unsigned long long *)((uint8_t *)scratch + off_b);
  } else {
    a.plan0 = (const uint32_t *)plans[0]->dev;
  }
  const int rc = pmrc_rt::rlc_launch(a, shx, (int)grid, stream);
  if (scratch) cudaFreeAsync(scratch, st);
  if (rc) {
    err = rc == -2 ? "runtime-coefficient kernel: no instantiation for this shape"
                   : std::string("runtime-coefficient launch: ") + cudaGetErrorString(cudaGetLastError());
    return rc == -2 ? PMRC_EUNSUPPORTED : PMRC_ECUDA;
  }
  launch_counter()++;
  return PMRC_OK;
}

}  // namespace pmrc
