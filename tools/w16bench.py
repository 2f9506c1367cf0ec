import sys, os, json, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import torch, inputs
import paper_1412_3022_b200 as pm
from sweep import timed
for k, n in ((8, 16), (4, 8)):
    c = pm.pmrc_create(0, k, 2 * k - 2, n, 16)
    info = pm.pmrc_info(c); B, P = info['B'], info['parity_rows']
    S = 1 << 20; stripes = -(-(1 << 30) // (B * S))
    data = torch.empty((stripes, B, S), dtype=torch.uint8, device='cuda'); par = torch.empty((stripes, P, S), dtype=torch.uint8, device='cuda')
    st = torch.cuda.current_stream().cuda_stream
    inputs.fill_device(data.data_ptr(), data.numel(), 3, stream=st)
    ms = timed(lambda: pm.pmrc_encode(c, data.data_ptr(), par.data_ptr(), S, stripes, st), 10)
    ps = pm.pmrc_plan_stats(c, 2)
    alu = ps['naive_lop3'] * (S // 64) * stripes / (148 * 64 * 1.965e9)
    print(json.dumps({'gen': os.environ.get('PMRC_GEN', ''), 'w': 16, 'k': k, 'n': n, 'ms': round(ms, 4), 'GBps': round(stripes * B * S / ms / 1e6, 1), 'alu_roof_frac': round(alu / (ms * 1e-3), 3)}))
    pm.pmrc_destroy(c)
