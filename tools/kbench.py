"""Kernel-only timing of the config-2 encode for generator variants (PMRC_GEN env), CUDA events."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import inputs
import paper_1412_3022_b200 as pm


def run(kind=0, k=8, n=16, S=1 << 20, real=1 << 30, steps=20):
    d = k if kind == 3 else 2 * k - 2
    t0 = time.time()
    code = pm.pmrc_create(kind, k, d, n)
    init = time.time() - t0
    info = pm.pmrc_info(code)
    B, P = info["B"], info["parity_rows"]
    stripes = -(-real // (B * S))
    data = torch.empty((stripes, B, S), dtype=torch.uint8, device="cuda")
    par = torch.empty((stripes, P, S), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    inputs.fill_device(data.data_ptr(), data.numel(), 1, stream=st.cuda_stream)
    for _ in range(3):
        pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    pm.pmrc_destroy(code)
    return {"gen": os.environ.get("PMRC_GEN", ""), "kind": kind, "k": k, "n": n, "S": S, "ms": round(ms, 4),
            "GBps_src": round(stripes * B * S / ms / 1e6, 1), "init_s": round(init, 2)}


if __name__ == "__main__":
    args = [int(a) for a in sys.argv[1:]]
    print(json.dumps(run(*args)))
