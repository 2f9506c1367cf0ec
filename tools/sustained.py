#!/usr/bin/env python3
"""Burst vs sustained kernel time of the config-2 encode for the generator options in PMRC_GEN:
20 launches after warm-up (burst), then ~2 s back to back (sustained: median of the last second),
with the SM clock and power NVML reports under that load.  One JSON line."""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
import torch

import inputs
import paper_1412_3022_b200 as pm


def main():
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    code = pm.pmrc_create(0, 8, 14, 16)
    S, stripes = 1 << 20, 19
    data = torch.empty((stripes, 56, S), dtype=torch.uint8, device="cuda")
    par = torch.empty_like(data)
    st = torch.cuda.current_stream()
    inputs.fill_device(data.data_ptr(), data.numel(), 1234, stream=st.cuda_stream)
    f = lambda: pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, st.cuda_stream)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    time.sleep(float(os.environ.get("COOL_S", "3")))      # let the power / clock state settle

    def run(n):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        ev[0].record(st)
        for i in range(n):
            f()
            ev[i + 1].record(st)
        torch.cuda.synchronize()
        return [ev[i].elapsed_time(ev[i + 1]) for i in range(n)]
    burst = sorted(run(20))
    samples, stop = [], [False]

    def samp():
        while not stop[0]:
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.02)
    th = threading.Thread(target=samp, daemon=True)
    th.start()
    per = run(4000)
    stop[0] = True
    th.join()
    tail = sorted(per[2000:])
    last = samples[len(samples) // 2:]
    print(json.dumps({"gen": os.environ.get("PMRC_GEN", ""), "burst_ms": round(burst[10], 4),
                      "sustained_ms": round(tail[len(tail) // 2], 4),
                      "sustained_GBps": round((1 << 30) / (tail[len(tail) // 2] * 1e-3) / 1e9, 1),
                      "sm_mhz": sorted(s[0] for s in last)[len(last) // 2] if last else None,
                      "power_w": round(sorted(s[1] for s in last)[len(last) // 2], 1) if last else None}))
    pm.pmrc_destroy(code)


if __name__ == "__main__":
    main()
