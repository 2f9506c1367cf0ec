#!/usr/bin/env python3
"""Sustained-load behaviour of the config-2 encode: 3000 back-to-back launches (1 GiB each) with
per-launch CUDA-event times (medians per 250 launches) and NVML samples of SM / memory clock,
temperature, power and clock-event reasons (profiles/r02/power_drift.txt)."""
import json, os, sys, time, threading
sys.path.insert(0, os.getcwd())
import torch, pynvml
import inputs, paper_1412_3022_b200 as pm
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
code = pm.pmrc_create(0, 8, 14, 16)
S = 1 << 20; stripes = 19
data = torch.empty((stripes, 56, S), dtype=torch.uint8, device="cuda"); par = torch.empty_like(data)
st = torch.cuda.current_stream()
inputs.fill_device(data.data_ptr(), data.numel(), 1234, stream=st.cuda_stream)
samples = []; stop = False
def samp():
    while not stop:
        try:
            samples.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                            pynvml.nvmlDeviceGetTemperature(h, 0), pynvml.nvmlDeviceGetPowerUsage(h) / 1000, pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        except Exception as e: samples.append(str(e))
        time.sleep(0.02)
th = threading.Thread(target=samp, daemon=True); th.start()
N = 3000
ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
ev[0].record(st)
for i in range(N):
    pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, st.cuda_stream)
    ev[i + 1].record(st)
torch.cuda.synchronize(); stop = True; th.join()
per = [ev[i].elapsed_time(ev[i + 1]) for i in range(N)]
for a in range(0, N, 250):
    seg = sorted(per[a:a + 250]); print("steps %4d-%4d median %.4f ms" % (a, a + 250, seg[len(seg) // 2]))
print("samples (t, sm, mem, temp, W, reasons):")
t0 = samples[0][0] if samples and not isinstance(samples[0], str) else 0
for s in samples[::max(1, len(samples) // 15)]:
    print(s if isinstance(s, str) else (round(s[0] - t0, 2),) + s[1:])
