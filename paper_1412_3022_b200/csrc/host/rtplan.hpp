// Host side of the runtime-coefficient kernel (csrc/rt/rlc.cu): turns a PlanSpec (plan.hpp) into
// the plan blob the kernel copies to shared memory (coefficients as PRMT tables), keeps it in
// device memory, and launches single-plan or per-stripe (batch) runs.  No NVRTC, no kernel
// generation: building a plan is O(rows x inputs) table fills after the host inversion.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../rt/rlc.hpp"
#include "plan.hpp"

namespace pmrc {

struct RtPlan {
  std::vector<uint32_t> blob;  // host copy (rlc.hpp RlcHdr layout)
  void *dev = nullptr;         // device copy (cudaMalloc), uploaded on first launch
  void *ready = nullptr;       // cudaEvent_t recorded after the upload (other streams wait on it)
  int R = 8, G = 1;            // rows per thread (row-block size of the masks), row groups per pass
  int n_in = 0, n_out = 0, n_terms = 0;
  long nnz = 0;                // nonzero A entries (MACs per 4 byte positions: nnz + derived terms)
};

// Launch shape for plans of up to n_out outputs (opts: rt_rows / rt_words / rt_groups /
// rt_group_threads, 0 = auto).
pmrc_rt::RlcShape rt_shape(int n_out, const GenOptions &o);
// Build the blob.  PMRC_EUNSUPPORTED if the plan does not fit the kernel (w != 8, > kRlcMaxSlots
// slots, block index >= 65536, tables above kRlcMaxPlanWords).
int rt_build(const PlanSpec &p, int R, int G, RtPlan &out, std::string &err);
void rt_free(RtPlan &p);
// estimated ALU work per tile word (batch launches split CTAs by it)
double rt_cost(const RtPlan &p);

// Launch: stripe_plan == nullptr -> plans[0] for every stripe; else plans[stripe_plan[t]] (0xFFFF:
// nothing to compute in stripe t).  All plans must be built for (sh.R, sh.G).  ptrs / strides: n_slots entries
// (slot s of stripe 0 and its stride).  max_ctas caps the grid (0 = one full wave).  Asynchronous.
int rt_launch(const std::vector<RtPlan *> &plans, const uint16_t *stripe_plan, const uint64_t *ptrs,
              const uint64_t *strides, int n_slots, size_t S, size_t stripes, const pmrc_rt::RlcShape &sh,
              void *stream, int max_ctas, std::string &err);

}  // namespace pmrc
