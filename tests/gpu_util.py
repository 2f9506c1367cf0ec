"""Helpers for the GPU parity tests: device buffers (torch, plumbing only), node piece views and
oracle comparisons.  Inputs come from the shared seeded generator (inputs/)."""
import numpy as np
import pytest
import torch

import inputs
import oracle as O
import paper_1412_3022_b200 as pm

DEV = torch.device("cuda:0")


class Stripes:
    """Data of `stripes` stripes on the device + its parity through the C ABI."""

    def __init__(self, kind, k, n, S, stripes, seed, device_fill=False, policy=None):
        self.kind, self.k, self.n, self.S, self.stripes = kind, k, n, S, stripes
        self.d = k if kind == pm.PMRC_RS_VANDERMONDE else 2 * k - 2
        self.code = pm.pmrc_create(kind, k, self.d, n)
        if policy is not None:
            pm.pmrc_set_plan_policy(self.code, policy)
        info = pm.pmrc_info(self.code)
        self.alpha, self.B, self.P = info["alpha"], info["B"], info["parity_rows"]
        self.seed = seed
        if device_fill:
            self.data = torch.empty((stripes, self.B, S), dtype=torch.uint8, device=DEV)
            inputs.fill_device(self.data.data_ptr(), self.data.numel(), seed,
                               stream=torch.cuda.current_stream().cuda_stream)
        else:
            self.data = torch.from_numpy(inputs.stripe_data(stripes, self.B, S, seed)).to(DEV)
        self.parity = torch.full((stripes, self.P, S), 0xEE, dtype=torch.uint8, device=DEV)
        self.stream = torch.cuda.current_stream().cuda_stream
        self.L = pm.pmrc_layout(self.code)
        self._mbr_sys = {}

    def close(self):
        pm.pmrc_destroy(self.code)

    def encode(self):
        pm.pmrc_encode(self.code, self.data.data_ptr(), self.parity.data_ptr(), self.S, self.stripes, self.stream)
        torch.cuda.synchronize()

    def host_data(self):
        return inputs.stripe_data(self.stripes, self.B, self.S, self.seed)

    def piece(self, i):
        """(ptr, stripe_stride) of node i's piece."""
        a, S = self.alpha, self.S
        if i >= self.k:
            return (self.parity.data_ptr() + (i - self.k) * a * S, self.P * S)
        if self.kind != pm.PMRC_MBR:
            return (self.data.data_ptr() + i * a * S, self.B * S)
        # MBR systematic node i stores row i of M(X): gather (R6)
        if i not in self._mbr_sys:
            idx = torch.tensor([int(v) - 1 for v in self.L[i]], device=DEV)
            self._mbr_sys[i] = self.data.index_select(1, idx).contiguous()
        t = self._mbr_sys[i]
        return (t.data_ptr(), a * S)

    def piece_tensor(self, i):
        a = self.alpha
        if i >= self.k:
            return self.parity[:, (i - self.k) * a:(i - self.k + 1) * a]
        if self.kind != pm.PMRC_MBR:
            return self.data[:, i * a:(i + 1) * a]
        self.piece(i)
        return self._mbr_sys[i]


    def nodes(self):
        """(ptr, stripe_stride) of every node's piece (the batch calls' node table)."""
        return [self.piece(i) for i in range(self.n)]


# both engines of every decode / repair / apply test (include/pmrc.h: results are bit-identical)
POLICIES = [pytest.param(pm.PMRC_PLAN_JIT, id="jit"), pytest.param(pm.PMRC_PLAN_RUNTIME, id="runtime")]


def oracle_kind(kind):
    return {pm.PMRC_MSR_SPARSE: O.MSR_SPARSE, pm.PMRC_MSR_VANILLA: O.MSR_VANILLA, pm.PMRC_MBR: O.MBR,
            pm.PMRC_RS_VANDERMONDE: O.RS, pm.PMRC_MSR_SPARSE_N2K: O.MSR_N2K}[kind]
