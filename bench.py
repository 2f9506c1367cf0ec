#!/usr/bin/env python3
"""bench.py — headline benchmark: MSR k=8, d=14, n=16 systematic sparse encode (BASELINE.json
config 2): 1 GiB of uniform random source data per GPU in 1 MiB sub-blocks (19 stripes of
56 x 1 MiB, the last zero padded, R11), GB/s of source data.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

One process per GPU (torchrun for N > 1, NCCL only for the barrier and the max-over-ranks
timing; stripes are independent so there is no data-path collective: weak scaling).  Rank 0
prints ONE JSON line.  ``--impl reference`` times the oracle (plain C, oracle/) on host cores on
a bounded sample of the same workload (rank 0 only).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

K_, D_, N_ = 8, 14, 16
S_ = 1 << 20
REAL = 1 << 30
METRIC = "MSR k=8,d=14,n=16 systematic encode GB/s per B200 & 8×B200; % roofline"
WORKLOAD = "config 2: MSR sparse systematic encode k=8 d=14 n=16, 1 GiB source per GPU, 1 MiB sub-blocks"
SMS, LANES_PER_CLK, SM_MAX_MHZ = 148, 64, 1965.0   # ALU-pipe issue rate (profiles/r01/int_issue_microbench.log)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, dev_index):
        self.samples, self.reasons, self.stop_flag = [], set(), False
        self.interval = float(os.environ.get("PMRC_CLOCK_INTERVAL", "0.005"))  # seconds between NVML samples
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self.stop_flag:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n_, bit in names.items():
                    if r & bit:
                        self.reasons.add(n_)
            except Exception:
                pass
            time.sleep(self.interval)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_flag = True
        if self.nv:
            self.t.join()

    def summary(self):
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz, "samples": len(s),
                "reasons": sorted(self.reasons)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(stripes_sample=4):
    """The oracle as it stands (plain C, scalar log/exp tables, never tuned) on the same workload's
    bytes (the shared seeded generator), on the box's host cores:
      * all cores: one host thread per core over the 19 stripes of the full 1 GiB job (ctypes
        releases the GIL inside the C call, so the threads run in parallel);
      * one core: the first `stripes_sample` stripes, the paper's own setting (one core)."""
    import concurrent.futures as cf
    import inputs
    import oracle as O
    B = 56
    stripes = -(-REAL // (B * S_))
    cores = os.cpu_count() or 1
    x1 = inputs.stripe_data(stripes_sample, B, S_, seed=1234, real_len=REAL)
    t0 = time.perf_counter()
    O.encode(O.MSR_SPARSE, N_, K_, D_, x1)
    dt1 = time.perf_counter() - t0
    del x1

    def one(t):
        x = inputs.stripe_data(1, B, S_, seed=1234, t0=t, real_len=REAL)
        t_ = time.perf_counter()
        O.encode(O.MSR_SPARSE, N_, K_, D_, x)
        return time.perf_counter() - t_
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=cores) as ex:
        list(ex.map(one, range(stripes)))
    dtn = time.perf_counter() - t0     # wall time of the parallel pass (includes host data generation)
    return {"value": REAL / dtn / 1e9, "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": "all %d stripes of the 1 GiB job (1064 MiB processed, R11), one host thread per core, "
                      "plain C scalar log/exp oracle" % stripes,
            "seconds": round(dtn, 2), "cpu_model": cpu_model(), "os_cpu_count": os.cpu_count(),
            "single_core": {"value": x_bytes(stripes_sample, B) / dt1 / 1e9, "unit": "GB/s", "cores": 1,
                            "sample": "%d of %d stripes (%d MiB of source), 1 thread (the paper's setting, P:214)" %
                                      (stripes_sample, stripes, x_bytes(stripes_sample, B) >> 20),
                            "seconds": round(dt1, 2)}}


def x_bytes(stripes, B):
    return stripes * B * S_


def bench_config(world):
    """The workload description both arms print (identical dicts: the driver compares them)."""
    B, P = 56, 56
    stripes = -(-REAL // (B * S_))
    return {"workload": WORKLOAD, "S": S_, "stripes_per_gpu": stripes, "real_bytes_per_gpu": REAL,
            "processed_bytes_per_gpu": stripes * B * S_, "parallelism": "stripes sharded by rank (dp%d)" % world,
            "l2": "inputs 1 GiB > 126 MB L2 (no flush needed)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps, warmup = args.steps, args.warmup
    import inputs
    import oracle as O
    B = 56
    x = inputs.stripe_data(1, B, S_, seed=1234, real_len=REAL)     # one stripe (56 MiB) per step
    for _ in range(max(0, min(warmup, 1))):
        O.encode(O.MSR_SPARSE, N_, K_, D_, x[:, :, : S_ // 16])
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.encode(O.MSR_SPARSE, N_, K_, D_, x)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    v = steps * x.size / tot / 1e9
    out = {"metric": METRIC, "value": v, "unit": "GB/s", "impl": "reference", "n_gpus": args.gpus, "steps": steps,
           "warmup": warmup, "ms_per_step": 1e3 * tot / steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded splitmix64 stream, inputs/)",
           "config": bench_config(int(os.environ.get("WORLD_SIZE", "1"))),
           "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle",
                            "sample": "1 of the 19 stripes (56 MiB of source) per step, plain C oracle, 1 thread"},
           "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def spawn_ranks(args):
    """`python bench.py --gpus N` outside torchrun: re-launch this script as N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1, exactly as the driver does, and return its
    exit code.  Inside torchrun (WORLD_SIZE set) the world size must equal --gpus."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def launch_check(args):
    """--launch-check: the multi-rank plumbing alone (gloo, CPU): every rank joins, rank 0 prints
    the world it saw.  Used by tests/test_bench_launcher.py to drive the launcher end to end."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([1.0])
    if world > 1:
        dist.all_reduce(t)
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "ranks_joined": int(t.item()),
                          "gpus_flag": args.gpus}))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="pmrc", choices=["pmrc", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--sustained-s", type=float, default=1.0, help="seconds of back-to-back launches for the "
                    "'sustained' figure (0 = skip)")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env != args.gpus:
        sys.stderr.write("bench.py: --gpus %d but WORLD_SIZE=%d: refusing to report a mismatched n_gpus\n"
                         % (args.gpus, world_env))
        return 2
    if args.launch_check:
        return launch_check(args)

    import torch
    import torch.distributed as dist

    import inputs
    import paper_1412_3022_b200 as pm
    from paper_1412_3022_b200 import build as pmbuild
    from paper_1412_3022_b200 import dist as pdist
    pmbuild.build_all(kernels=False)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    t_init0 = time.perf_counter()
    code = pm.pmrc_create(pm.PMRC_MSR_SPARSE, K_, D_, N_)
    init_s = time.perf_counter() - t_init0
    info = pm.pmrc_info(code)
    B, P = info["B"], info["parity_rows"]
    stripes = -(-REAL // (B * S_))                    # 19 (R11: last stripe zero padded)
    stream = torch.cuda.current_stream()
    data = torch.empty((stripes, B, S_), dtype=torch.uint8, device=dev)
    par = torch.empty((stripes, P, S_), dtype=torch.uint8, device=dev)
    # each rank encodes its own 1 GiB (distinct seeded bytes: global offset of rank r's stripes)
    inputs.fill_device(data.data_ptr(), data.numel(), 1234 + rank, real_len=REAL, stream=stream.cuda_stream)
    torch.cuda.synchronize()

    def step():
        pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S_, stripes, stream.cuda_stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    l0 = pm.pmrc_launch_count()
    with ClockSampler(local) as clk:
        ev[0].record(stream)
        for i in range(args.steps):
            step()
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
    launches = pm.pmrc_launch_count() - l0
    barrier()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    # max over ranks of the device-timed region, whole-job throughput (paper_1412_3022_b200/dist.py,
    # covered by the gloo world_size-2 test)
    total_ms = pdist.max_over_ranks(total_ms, dist if world > 1 else None, device=dev)
    ms_step = total_ms / args.steps
    value = pdist.aggregate_gbps(REAL, world, ms_step * 1e-3)

    # ---- roofline of the (only) kernel: pmrc_kernel, one launch per step ----
    pk = peaks()
    kern_ms = sorted(per)[len(per) // 2]
    processed = stripes * B * S_
    alg_bytes = processed + stripes * P * S_                 # data read + parity written
    W = info["xor_ops_naive"] * (S_ // 32) * stripes          # naive LOP3 lane-ops
    alu_peak = SMS * LANES_PER_CLK * SM_MAX_MHZ * 1e6 / 1e12  # T lane-ops/s
    t_hbm = alg_bytes / (pk["hbm_gbs"] * 1e9)
    t_issue = W / (alu_peak * 1e12)
    achieved_alu = W / (kern_ms * 1e-3) / 1e12
    achieved_hbm = alg_bytes / (kern_ms * 1e-3) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_encode_summary.json")))
        traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass
    bound = "alu" if t_issue >= t_hbm else "hbm"
    if bound == "alu":
        roof = {"bound": "alu", "achieved": achieved_alu, "peak": alu_peak, "unit": "T LOP3-lane-ops/s",
                "frac": achieved_alu / alu_peak, "traffic": traffic}
    else:
        roof = {"bound": "hbm", "achieved": achieved_hbm, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved_hbm / pk["hbm_gbs"], "traffic": traffic}
    roof.update({"kernel": "pmrc_kernel (JIT bitsliced encode)", "kernel_ms": kern_ms,
                 "peak_source": "alu: 148 SM x 64 lanes/clk (measured, profiles/r01) x 1965 MHz; hbm: MEASURED_PEAKS.json",
                 "hbm_achieved_gbs": achieved_hbm, "hbm_peak_gbs": pk["hbm_gbs"],
                 "hbm_frac": achieved_hbm / pk["hbm_gbs"], "t_roof_ms": 1e3 * max(t_hbm, t_issue),
                 "roof_frac": 1e3 * max(t_hbm, t_issue) / kern_ms,
                 "naive_lop3_per_32pos": info["xor_ops_naive"], "xor2_after_cse_per_32pos": info["xor_ops"]})

    # ---- sustained: the same launches back to back for ~1 s (outside the timed region).  Under
    # continuous load the B200 reaches its 1000 W power cap within ~0.1 s and lowers the SM clock
    # (profiles/r02/power_drift.txt); the K-step region above is the burst figure ----
    sus = None
    if args.sustained_s > 0:
        n_sus = max(20, int(args.sustained_s / max(1e-6, ms_step * 1e-3)))
        barrier()
        sev = [torch.cuda.Event(enable_timing=True) for _ in range(n_sus + 1)]
        with ClockSampler(local) as sclk:
            sev[0].record(stream)
            for i in range(n_sus):
                step()
                sev[i + 1].record(stream)
            torch.cuda.synchronize()
        tail = sorted(sev[i].elapsed_time(sev[i + 1]) for i in range(n_sus // 2, n_sus))
        sus_ms = pdist.max_over_ranks(tail[len(tail) // 2], dist if world > 1 else None, device=dev)
        sc = sclk.summary()
        mhz = sc["sm_mhz"] or SM_MAX_MHZ
        sus_peak = SMS * LANES_PER_CLK * mhz * 1e6 / 1e12
        sus = {"launches": n_sus, "ms_per_step": sus_ms, "value": pdist.aggregate_gbps(REAL, world, sus_ms * 1e-3),
               "unit": "GB/s", "clocks": sc,
               "alu_frac_at_clock": (W / (sus_ms * 1e-3) / 1e12) / sus_peak,
               "note": "median kernel time of the second half of ~%.1f s of back-to-back launches; ALU roof "
                       "at the SM clock measured under that load" % args.sustained_s}

    # ---- e2e: through the C ABI from pinned host buffers (H2D + encode + D2H per step) ----
    e2e = None
    if args.e2e_steps > 0:
        hd = torch.empty((stripes, B, S_), dtype=torch.uint8).pin_memory()
        hp = torch.empty((stripes, P, S_), dtype=torch.uint8).pin_memory()
        hd.copy_(data.cpu())
        pm.pmrc_encode_host(code, hd.data_ptr(), hp.data_ptr(), S_, stripes, stream.cuda_stream)  # warm
        barrier()
        times = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            pm.pmrc_encode_host(code, hd.data_ptr(), hp.data_ptr(), S_, stripes, stream.cuda_stream)
            times.append(time.perf_counter() - t0)
        tmax = pdist.max_over_ranks(sum(times) / len(times), dist if world > 1 else None, device=dev)
        e2e = {"value": pdist.aggregate_gbps(REAL, world, tmax), "unit": "GB/s",
               "h2d_bytes_per_step": stripes * B * S_, "d2h_bytes_per_step": stripes * P * S_,
               "api": "pmrc_encode_host (pinned host buffers, staged + overlapped copies)",
               "steps": len(times), "ms_per_step": 1e3 * sum(times) / len(times),
               "ms_per_step_median": 1e3 * sorted(times)[len(times) // 2],
               "note": "value = mean over the steps (host wall clock around the synchronous call); one run on a "
                       "busy host measured 31 GB/s where the same box gave 44.7 minutes later "
                       "(pinned-copy ceiling 50 GB/s each way, tools/pcie_bw.py)"}
        del hd, hp

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline()     # rank 0 only, after every rank's timed region

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded splitmix64 uniform bytes, inputs/)",
               "config": bench_config(world), "init_ms": round(init_s * 1e3, 1),
               "roofline": roof, "sustained": sus, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
               "clocks": clk.summary(),
               "paper_context": {"value": 0.79, "unit": "GB/s", "what": "1 core Xeon E5-2640, k=8, 16 KB blocks (P:329)"}}
        print(json.dumps(out))
    pm.pmrc_destroy(code)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
