#!/usr/bin/env python3
"""bench.py -- approximate GMAC/s (LUT lookups/s) of the AdaPT LUT layer hot path on B200.

One "step" is one pass of the whole hot path (plus a8 at N>1) over
one batch of BASELINE.json configs[2] (the approximate conv2d layer; DESIGN.md §6 says why
this config carries the headline number):
    amax(x) -> scale -> quantize NCHW fp32 -> NHWC int8 -> implicit-im2col LUT-conv with the
    dequantize epilogue -> fp32 NCHW y
Weights and the ACU table are prepared once, untimed (row a1/a2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload conv|linear]

Prints ONE JSON line (rank 0).  Multi-GPU: launched by torchrun, one rank per GPU over
NCCL; weak scaling (each rank runs its own batch; no data-path collective -- the batch is
the unit the method partitions); time = max over ranks of the CUDA-event time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

SM_COUNT_NOMINAL = 148
LANES = 32


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="conv", choices=["conv", "linear"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"sm_max_mhz": 1965.0, "hbm_gbs": 6650.0}, "fallback"


def committed_traffic(kernel_key: str):
    """dram bytes per launch from the committed ncu --set full summary (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(kernel_key)
    except Exception:
        return None


# ---------------------------------------------------------------------------------------
# clocks during the timed region (nvidia-smi sampler)
# ---------------------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons every few ms through NVML while
    the timed region runs; falls back to nvidia-smi polling."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []          # (sm_mhz, max_mhz, reason_bits)
        self._stop = threading.Event()
        self._t = None
        self._h = None
        self.src = "none"
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(device_index).uuid)
            try:
                self._h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid) if not uuid.startswith("GPU") else uuid)
            except Exception:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self._nv = pynvml
            self.src = "nvml"
        except Exception:
            self._h = None

    def _sample_nvml(self):
        nv = self._nv
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        return (float(sm), float(mx), int(rs))

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown")
        out = subprocess.run(["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + q,
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip().split(",")
        bits = 0
        for b, v in zip((0x4, 0x8, 0x20, 0x40), out[2:]):
            if v.strip().lower() == "active":
                bits |= b
        return (float(out[0]), float(out[1]), bits)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample_nvml() if self._h is not None else self._sample_smi())
                if self._h is None:
                    self.src = "nvidia-smi"
            except Exception:
                pass
            self._stop.wait(0.005 if self._h is not None else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.02)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({n for s in self.samples for b, n in self.REASONS.items() if s[2] & b})
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": self.src}


# ---------------------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------------------
def conv_workload(rank: int):
    import datagen
    c = datagen.config2()
    Nb, C, H, W = c.x.shape
    K, _, R, S = c.W.shape
    lookups = Nb * H * W * K * C * R * S          # stride 1, pad 1: Ho = H, Wo = W
    desc = {"workload": "BJ configs[2]: approximate conv2d, x fp32 [128,64,56,56] ReLU(N(0,1)), "
                        "W 64x64x3x3 Kaiming, stride 1 pad 1, int8 per-tensor max calibration, "
                        "randerr LUT (exact + U[-64,64]), implicit im2col, fp32 NCHW output",
            "lookups_per_step": lookups, "batch_per_gpu": Nb}
    return c, lookups, desc


def linear_workload(rank: int):
    import datagen
    c = datagen.config1()
    M, K = c.x.shape
    N = c.W.shape[0]
    desc = {"workload": "BJ configs[1]: approximate linear, x fp32 [256x1024], W [1024x1024], "
                        "trunc4 LUT, fp32 output", "lookups_per_step": M * N * K}
    return c, M * N * K, desc


# ---------------------------------------------------------------------------------------
# our implementation
# ---------------------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2203_04071_b200 as axq
    from paper_2203_04071_b200 import _lib as ax

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    if args.workload == "conv":
        c, lookups, desc = conv_workload(rank)
    else:
        c, lookups, desc = linear_workload(rank)
    bits = c.bits
    lut = axq.Lut(bits, c.lut)
    stream = torch.cuda.current_stream()

    if args.workload == "conv":
        from paper_2203_04071_b200.layers import ApproxConv2d
        layer = ApproxConv2d(torch.from_numpy(c.W).to(dev), None, lut, c.stride, c.pad)
        x_host = torch.from_numpy(c.x).pin_memory()
        x = x_host.to(dev)
        Nb, C, H, W = x.shape
        d = layer.desc(Nb, H, W)
        Ho, Wo = ax.axq_conv2d_out_hw(d)
        y = torch.empty(Nb, layer.Kout, Ho, Wo, device=dev)
        qx = torch.empty(Nb, H, W, C, dtype=torch.int8, device=dev)
        y_host = torch.empty(y.shape, dtype=torch.float32).pin_memory()

        def step(ev_pair=None):
            ax.axq_amax(x, layer.d_amax_a, stream)
            ax.axq_scale(layer.d_amax_a, bits, layer.d_scale_a, stream)
            ax.axq_quantize_nchw_to_nhwc(x, layer.d_scale_a, bits, qx, stream)
            if ev_pair:
                ev_pair[0].record(stream)
            ax.axq_lut_conv2d_dq(d, qx, layer.qw, lut, layer.d_scale_a, layer.d_scale_w, None,
                                 y, stream=stream)
            if ev_pair:
                ev_pair[1].record(stream)
        launches_per_step = 4       # amax, scale, quantize, LUT-conv(+dequant)
        in_bytes, out_bytes = x.numel() * 4, y.numel() * 4
    else:
        from paper_2203_04071_b200.layers import ApproxLinear
        layer = ApproxLinear(torch.from_numpy(c.W).to(dev), torch.from_numpy(c.b).to(dev), lut)
        x_host = torch.from_numpy(c.x).pin_memory()
        x = x_host.to(dev)
        M = x.shape[0]
        y = torch.empty(M, layer.N, device=dev)
        bufs = layer.buffers(M, dev)
        y_host = torch.empty(y.shape, dtype=torch.float32).pin_memory()

        def step(ev_pair=None):
            ax.axq_amax(x, layer.d_amax_a, stream)
            ax.axq_scale(layer.d_amax_a, bits, layer.d_scale_a, stream)
            ax.axq_quantize(x, layer.d_scale_a, bits, bufs["qa"], stream)
            if ev_pair:
                ev_pair[0].record(stream)
            ax.axq_lut_gemm_dq(bufs["qa"], layer.qw, lut, layer.d_scale_a, layer.d_scale_w,
                               layer.bias, y, workspace=bufs["ws"], stream=stream)
            if ev_pair:
                ev_pair[1].record(stream)
        launches_per_step = 6       # amax, scale, quantize, LUT-GEMM (split-K), dequant + memset
        in_bytes, out_bytes = x.numel() * 4, y.numel() * 4

    # L2 flush buffer (> 126 MB L2) written between timed steps, outside the timed region
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()

    step_ms, kern_ms = [], []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step((k0, k1))
            s1.record(stream)
            s1.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            kern_ms.append(k0.elapsed_time(k1))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = t.item()

    # e2e: the same step through the public API with HOST buffers (pinned), H2D of the
    # inputs and D2H of the result inside the timed region.
    e2e = None
    if not args.no_e2e:
        e_ms = []
        for _ in range(max(2, min(args.steps, 5))):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            x.copy_(x_host, non_blocking=True)
            step()
            y_host.copy_(y, non_blocking=True)
            b.record(stream)
            b.synchronize()
            e_ms.append(a.elapsed_time(b))
        e_tot = sum(e_ms)
        if dist:
            t = torch.tensor([e_tot], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_tot = t.item()
        e2e = {"value": world * lookups * len(e_ms) / (e_tot * 1e-3) / 1e9, "unit": "GMAC/s",
               "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": out_bytes,
               "ms_per_step": e_tot / len(e_ms)}

    result = None
    if rank == 0:
        peaks, peak_src = measured_peaks()
        sm = torch.cuda.get_device_properties(dev).multi_processor_count
        clocks = clk.summary()
        f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        roof_max = sm * LANES * f_max / 1e9                              # Glookups/s
        kmean = statistics.mean(kern_ms)
        achieved = lookups / (kmean * 1e-3) / 1e9
        value = world * lookups * args.steps / (total_ms * 1e-3) / 1e9
        f_meas = (clocks["sm_mhz"] or 0) * 1e6
        result = {
            "metric": "approximate GMAC/s (LUT lookups/s) per B200 and % of smem-lookup roofline",
            "value": round(value, 3), "unit": "GMAC/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic (seeded; DESIGN.md input recipe)",
            "config": dict(desc, parallelism="dp%d (batch-sharded replicas)" % world,
                           l2="flushed between timed steps (256 MiB write)",
                           lut_repr=lut.repr),
            "roofline": {"bound": "smem", "kernel": "lut_mm_kernel (axq_lut_conv2d_dq)"
                         if args.workload == "conv" else "lut_mm_kernel (axq_lut_gemm_dq)",
                         "achieved": round(achieved, 2), "peak": round(roof_max, 2),
                         "unit": "Glookup/s", "frac": round(achieved / roof_max, 4),
                         "peak_basis": "%d SMs x 32 lanes x %.0f MHz (%s sm_max_mhz); one "
                                       "shared-memory wavefront per SM clock" %
                                       (sm, f_max / 1e6, peak_src),
                         "frac_at_measured_clock": round(achieved / (sm * LANES * f_meas / 1e9), 4)
                         if f_meas else None,
                         "kernel_ms": round(kmean, 4),
                         "kernel_share_of_step": round(kmean / (total_ms / args.steps), 4),
                         "traffic": committed_traffic("lut_conv_c2" if args.workload == "conv"
                                                      else "lut_gemm_c1")},
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
        }
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return result


# ---------------------------------------------------------------------------------------
# oracle (CPU) timing: cpu_baseline leg and --impl reference
# ---------------------------------------------------------------------------------------
def oracle_conv_sample(c, n_img: int):
    import oracle
    t0 = time.perf_counter()
    sa = oracle.scale(oracle.amax(c.x), 8)               # full-tensor calibration, as the GPU
    qw, sw = oracle.quantize_tensor(c.W, 8)
    qx = oracle.quantize(c.x[:n_img], sa, 8)
    acc = oracle.lut_conv2d(qx, qw, c.lut, 8, c.stride, c.pad)
    oracle.dequantize(acc, sa, sw, None, 1)
    return time.perf_counter() - t0


def oracle_linear_sample(c, rows: int):
    import oracle
    t0 = time.perf_counter()
    sa = oracle.scale(oracle.amax(c.x), 8)
    qw, sw = oracle.quantize_tensor(c.W, 8)
    qa = oracle.quantize(c.x[:rows], sa, 8)
    acc = oracle.lut_gemm(qa, qw, c.lut, 8)
    oracle.dequantize(acc, sa, sw, c.b)
    return time.perf_counter() - t0


def cpu_baseline(args, budget_s: float = 12.0):
    import oracle
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    threads = oracle.max_threads()
    if args.workload == "conv":
        c, lookups, _ = conv_workload(0)
        per_img = lookups // c.x.shape[0]
        t1 = oracle_conv_sample(c, 1)
        n = int(max(1, min(c.x.shape[0], budget_s / max(t1, 1e-3))))
        t = oracle_conv_sample(c, n)
        return {"value": round(n * per_img / t / 1e9, 4), "unit": "GMAC/s", "cores": threads,
                "kind": "oracle",
                "sample": "%d of 128 images of the same workload (amax/quantize/LUT-conv/"
                          "dequant, OpenMP over (image, out-channel)), %.1f s" % (n, t)}
    c, lookups, _ = linear_workload(0)
    per_row = lookups // c.x.shape[0]
    t = oracle_linear_sample(c, c.x.shape[0])
    return {"value": round(lookups / t / 1e9, 4), "unit": "GMAC/s", "cores": threads,
            "kind": "oracle", "sample": "full workload (%.2f s)" % t}


def run_reference(args, rank):
    """--impl reference: the oracle as it stands, on the host cores, same metric/config."""
    if rank != 0:
        return None
    import oracle
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    threads = oracle.max_threads()
    if args.workload == "conv":
        c, lookups, desc = conv_workload(0)
        per_img = lookups // c.x.shape[0]
        unit_fn = lambda: oracle_conv_sample(c, 1)           # noqa: E731
        per_step_lookups = per_img
        sample = "1 of 128 images per step (bounded sample of the same workload)"
    else:
        c, lookups, desc = linear_workload(0)
        unit_fn = lambda: oracle_linear_sample(c, c.x.shape[0])  # noqa: E731
        per_step_lookups = lookups
        sample = "full workload per step"
    for _ in range(max(args.warmup, 0)):
        unit_fn()
    ts = [unit_fn() for _ in range(args.steps)]
    tot = sum(ts)
    value = per_step_lookups * args.steps / tot / 1e9
    return {"metric": "approximate GMAC/s (LUT lookups/s) per B200 and % of smem-lookup roofline",
            "impl": "reference", "value": round(value, 4), "unit": "GMAC/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic (seeded)", "config": dict(desc, parallelism="host cores"),
            "cpu_baseline": {"value": round(value, 4), "unit": "GMAC/s", "cores": threads,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 4), "unit": "GMAC/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        res = run_reference(args, rank)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    res = run_ours(args, rank, world, local_rank)
    if rank == 0 and res is not None:
        if world == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
