#!/usr/bin/env python3
"""bench.py -- approximate GMAC/s (LUT lookups/s) of the AdaPT LUT layer hot path on B200.

One "step" is one pass of the whole hot path over one batch of the
workload:
  resnet (default, BJ configs[3]): the ResNet-50-shaped approximate forward of the 256-image
      batch -- quantize the fp32 input, 54 LUT layers with fused dequant / residual / ReLU /
      requantize epilogues, int8 maxpool, avgpool, fc -- batch-sharded over the N GPUs
      (strong scaling: 256/N images per rank) with an NCCL all-gather of the logits (a8).
  conv (BJ configs[2]), linear (BJ configs[1]): one approximate layer (a3-a6).
  lstm (BJ configs[4]): the 128-step LSTM at b = 4, 6 and 8 (replicas at N > 1).
Weights, the ACU table and the static per-layer scales (calibration) are prepared once,
untimed (rows a1/a2, "learns offline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload resnet|conv|linear|lstm]

Prints ONE JSON line (rank 0).  Multi-GPU: launched by torchrun, one rank per GPU over NCCL;
time = max over ranks of the CUDA-event time.
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
QUANTIZER = "max"
LUT_KIND = "default"
DESIGN_LOOKUPS_PER_CLK = 1024.0 / 8.0    # issue bound of the P4W inner loop
DESIGN_BASIS = ("packed-table inner loop (r2, dp4a over 4-k byte transposes): per 1024 lookups "
                "of a warp 32 issued warp instructions (8 LDS, 14 ALU-pipe: code extracts + "
                "PRMT transposes, 10 FMA-pipe: row addresses + dp4a) at 4 issued per SM clock "
                "-> 128 lookups per SM clock; the ALU pipe alone (2 per SM clock) would allow "
                "146, shared memory at replay 1 (8 wavefronts) 128 (DESIGN.md 5.4)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet", choices=["resnet", "conv", "linear", "lstm", "gemm"])
    ap.add_argument("--quantizer", default="max", choices=["max", "paper"],
                    help="resnet only: 'paper' = per-channel weights + 99.9%% histogram "
                         "activations (NEXT-1, P:93-95) instead of BASELINE's per-tensor max")
    ap.add_argument("--lut", default="default", choices=["default", "err2000", "err1e5"],
                    help="conv only: 'err2000' = an ACU with a +-2000 error (beyond int8 E: the "
                         "packed int16-E kernel P4W16) instead of BJ configs[2]'s randerr table; "
                         "'err1e5' = a +-1e5-error ACU (beyond int16 E: the SM-resident int32 "
                         "table in two halves, lut_mm_kernel<REPR_I32>)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    a = ap.parse_args()
    if a.steps is None:
        a.steps = {"resnet": 10, "lstm": 5, "conv": 50, "linear": 200, "gemm": 200}[a.workload]
    return a


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
# workloads (ours)
# ---------------------------------------------------------------------------------------
class KernelTimer:
    """CUDA events around every LUT-kernel launch (on the launching stream)."""

    def __init__(self):
        self.enabled = False
        self.pairs = []

    def __call__(self, kind, stream):
        if not self.enabled:
            return
        import torch
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        if kind == "pre":
            self.pairs.append([ev, None])
        else:
            self.pairs[-1][1] = ev

    def total_ms(self):
        return sum(a.elapsed_time(b) for a, b in self.pairs)

    def reset(self):
        self.pairs = []


class ResNetWL:
    name = "resnet"
    scaling = "strong"
    pipelined_e2e = True

    def __init__(self, dev, rank, world, timer):
        import torch
        import datagen
        from paper_2203_04071_b200 import Lut
        from paper_2203_04071_b200.resnet import ApproxResNet, layer_specs
        from paper_2203_04071_b200.shard import shard_range
        self.dev, self.rank, self.world = dev, rank, world
        total = 256
        a, b = shard_range(total, world, rank)
        self.per = b - a
        self.total = total
        x_all = datagen.config3_images(total)
        self.x_host = torch.from_numpy(x_all[a:b]).pin_memory()
        self.x = self.x_host.to(dev)
        self.lut = Lut(8, datagen.lut_randerr(8, 0, 2))          # A15: c0's table
        self.quantizer = QUANTIZER
        self.net = ApproxResNet(datagen.network_weights(layer_specs(), 3), self.lut, dev,
                                quantizer=QUANTIZER)
        self.net.calibrate(torch.from_numpy(x_all[:8]).to(dev))   # static scales, untimed
        torch.cuda.synchronize()
        # every rank built the tables / weights / scales from the seed; confirm
        from paper_2203_04071_b200.shard import verify_replicas
        self.checksum = verify_replicas(self.net.replicated_state() +
                                        [torch.from_numpy(datagen.lut_randerr(8, 0, 2))],
                                        _dist_or_none(world), device=dev)
        self.net.timing_hook = timer
        self.lookups_rank = self.per * self.net.lookups_per_image()
        self.lookups_total = total * self.net.lookups_per_image()
        self.logits_all = torch.empty(total, 1000, device=dev)
        self.out_host = torch.empty(total, 1000).pin_memory()
        # 53 convs, stem im2col, fc (table build + GEMM when activation-specialised), quantize,
        # maxpool, avgpool (static fallback; the bench counts launches with CUPTI)
        fc_x = any("fc_xp" in b for b in self.net._bufs.values())
        self.launches = 53 + 1 + (3 if fc_x else 1) + 3
        self.in_bytes = self.x.numel() * 4
        self.out_bytes = self.logits_all.numel() * 4 if rank == 0 else 0
        self.desc = {"workload": "BJ configs[3]: ResNet-50-shaped approximate forward (53 convs + "
                                 "fc, every multiply a LUT lookup), x fp32 [256,3,224,224] N(0,1), "
                                 "Kaiming weights, randerr int8 LUT (c0's), static per-layer "
                                 + ("max calibration" if QUANTIZER == "max" else
                                    "99.9% histogram calibration with per-channel weight scales "
                                    "(the paper's quantizer, NEXT-1)") +
                                 " on images 0-7 (untimed)",
                     "global_batch": total, "batch_per_gpu": self.per,
                     "lookups_per_image": self.net.lookups_per_image()}

    def step(self, stream, dist):
        from paper_2203_04071_b200.shard import gather_rows
        lg = self.net.forward(self.x, stream)
        gather_rows(lg, self.logits_all, self.total, dist)      # a8: collect the outputs

    def h2d(self):
        self.x.copy_(self.x_host, non_blocking=True)

    def d2h(self):
        if self.rank == 0:
            self.out_host.copy_(self.logits_all, non_blocking=True)


class ConvWL:
    name = "conv"
    scaling = "strong"
    pipelined_e2e = True

    def __init__(self, dev, rank, world, timer):
        import torch
        import datagen
        from paper_2203_04071_b200 import Lut
        from paper_2203_04071_b200 import _lib as ax
        from paper_2203_04071_b200.layers import ApproxConv2d
        from paper_2203_04071_b200.shard import shard_range, verify_replicas
        self.ax = ax
        c = datagen.config2()
        if LUT_KIND == "err2000":
            c.lut = datagen.lut_bigerr(8, 2000, 8, 1)
        elif LUT_KIND == "err1e5":
            c.lut = datagen.lut_bigerr(8, 100_000, 8, 1)
        self.c = c
        self.lut = Lut(8, c.lut)
        self.world, self.rank = world, rank
        # BJ configs[2]'s input is ReLU(N(0,1)): non-negative codes (half-range packed tables)
        self.layer = ApproxConv2d(torch.from_numpy(c.W).to(dev), None, self.lut, c.stride, c.pad,
                                  a_nonneg=True)
        total = c.x.shape[0]
        a, b = shard_range(total, world, rank)        # images per rank
        self.total, self.per = total, b - a
        self.x_host = torch.from_numpy(c.x[a:b]).pin_memory()
        self.x = self.x_host.to(dev)
        Nb, C, H, W = self.x.shape
        self.d = self.layer.desc(Nb, H, W)
        Ho, Wo = ax.axq_conv2d_out_hw(self.d)
        self.y = torch.empty(Nb, self.layer.Kout, Ho, Wo, device=dev)
        self.y_all = torch.empty(total, self.layer.Kout, Ho, Wo, device=dev) if world > 1 else self.y
        self.qx = torch.empty(Nb, H, W, C, dtype=torch.int8, device=dev)
        self.pipelined_out = world == 1
        self.y_host = torch.empty(self.y_all.shape if rank == 0 else self.y.shape).pin_memory()
        self.timer = timer
        per_img = Ho * Wo * self.layer.Kout * C * 9
        self.lookups_rank = Nb * per_img
        self.lookups_total = total * per_img
        self.launches = 4
        self.in_bytes = self.x.numel() * 4
        self.out_bytes = self.y_host.numel() * 4
        self.checksum = verify_replicas([c.lut, self.layer.qw, self.layer.d_scale_w],
                                        _dist_or_none(world), device=dev)
        self.desc = {"workload": "BJ configs[2]: approximate conv2d, x fp32 [128,64,56,56] "
                                 "ReLU(N(0,1)), W 64x64x3x3 Kaiming, stride 1 pad 1, int8 dynamic "
                                 "per-tensor max calibration (N > 1: all_reduce(MAX) of the shard "
                                 "amax, then the same scale as one GPU), randerr LUT, implicit "
                                 "im2col, fp32 NCHW output (N > 1: all-gathered)" +
                                 {"err2000": " -- with a +-2000-error ACU instead (--lut err2000)",
                                  "err1e5": " -- with a +-1e5-error ACU instead (--lut err1e5, "
                                            "int32 table)"}.get(LUT_KIND, ""),
                     "global_batch": total, "batch_per_gpu": Nb}

    def step(self, stream, dist):
        from paper_2203_04071_b200.shard import all_reduce_max_, gather_rows
        ax, L = self.ax, self.layer
        ax.axq_amax(self.x, L.d_amax_a, stream)
        all_reduce_max_(L.d_amax_a, dist)             # G > 1 == G = 1 (reading A7)
        ax.axq_scale(L.d_amax_a, 8, L.d_scale_a, stream)
        ax.axq_quantize_nchw_to_nhwc(self.x, L.d_scale_a, 8, self.qx, stream)
        self.timer("pre", stream)
        L.conv_q(self.d, self.qx, L.d_scale_a, self.y, stream=stream)
        self.timer("post", stream)
        if self.world > 1:
            gather_rows(self.y, self.y_all, self.total, dist)   # a8: collect the outputs

    def h2d(self):
        self.x.copy_(self.x_host, non_blocking=True)

    def d2h(self):
        self.y_host.copy_(self.y_all if self.rank == 0 else self.y, non_blocking=True)


def _dist_or_none(world):
    if world <= 1:
        return None
    import torch.distributed as dist
    return dist


class LinearWL:
    name = "linear"
    scaling = "strong"
    pipelined_e2e = False   # 1 MB copies: the cross-stream waits cost more than the overlap saves

    def __init__(self, dev, rank, world, timer):
        import torch
        import datagen
        from paper_2203_04071_b200 import Lut
        from paper_2203_04071_b200 import _lib as ax
        from paper_2203_04071_b200.layers import ApproxLinear
        from paper_2203_04071_b200.shard import shard_range, verify_replicas
        self.ax = ax
        c = datagen.config1()
        self.lut = Lut(8, c.lut)
        self.world, self.rank = world, rank
        self.layer = ApproxLinear(torch.from_numpy(c.W).to(dev), torch.from_numpy(c.b).to(dev), self.lut)
        total = c.x.shape[0]
        a, b = shard_range(total, world, rank)        # rows per rank
        self.total = total
        self.x_host = torch.from_numpy(c.x[a:b]).pin_memory()
        self.x = self.x_host.to(dev)
        M = self.x.shape[0]
        self.y = torch.empty(M, self.layer.N, device=dev)
        self.y_all = torch.empty(total, self.layer.N, device=dev) if world > 1 else self.y
        self.bufs = self.layer.buffers(M, dev)
        self.y_host = torch.empty(self.y_all.shape if rank == 0 else self.y.shape).pin_memory()
        self.timer = timer
        self.lookups_rank = M * self.layer.N * self.layer.K
        self.lookups_total = total * self.layer.N * self.layer.K
        self.launches = 3 + (3 if self.layer.use_xspec(M) else 1)   # amax, scale, quantize + LUT
        self.in_bytes, self.out_bytes = self.x.numel() * 4, self.y_host.numel() * 4
        self.checksum = verify_replicas([c.lut, self.layer.qw, self.layer.d_scale_w, self.layer.bias],
                                        _dist_or_none(world), device=dev)
        self.desc = {"workload": "BJ configs[1]: approximate linear, x fp32 [256x1024] N(0,1), W "
                                 "[1024x1024] N(0,0.02), bias N(0,0.01), trunc4 LUT, fp32 output "
                                 "(N > 1: rows sharded, all_reduce(MAX) of the amax, outputs "
                                 "all-gathered)", "global_batch": total, "batch_per_gpu": M,
                     "kernel_path": {"xspec": "activation-specialised packed tables built per "
                                              "call (axq_wpack_repack) + 512-row P4W "
                                              "(axq_lut_gemm_xs)",
                                     "wpack": "weight-specialised packed tables + P4W",
                                     "gather": "per-row gather (v1)"}[self.layer.path(M)]}

    def step(self, stream, dist):
        from paper_2203_04071_b200.shard import all_reduce_max_, gather_rows
        ax, L = self.ax, self.layer
        ax.axq_amax(self.x, L.d_amax_a, stream)
        all_reduce_max_(L.d_amax_a, dist)             # G > 1 == G = 1 (reading A7)
        ax.axq_scale(L.d_amax_a, 8, L.d_scale_a, stream)
        ax.axq_quantize(self.x, L.d_scale_a, 8, self.bufs["qa"], stream)
        # LUT work = the per-call activation-table build + the packed-table GEMM (timed together)
        L.gemm_q(self.bufs["qa"], L.d_scale_a, self.y, stream, hook=self.timer)
        if self.world > 1:
            gather_rows(self.y, self.y_all, self.total, dist)

    def h2d(self):
        self.x.copy_(self.x_host, non_blocking=True)

    def d2h(self):
        self.y_host.copy_(self.y_all if self.rank == 0 else self.y, non_blocking=True)


class GemmWL:
    """BJ configs[0]: one raw LUT-GEMM (A int8 64x256, W int8 256x64, randerr LUT, int32 out).
    Latency-sized (1 M lookups): reported in microseconds; replicas at N > 1."""
    name = "gemm"
    scaling = "weak"
    pipelined_e2e = False

    def __init__(self, dev, rank, world, timer):
        import torch
        import datagen
        from paper_2203_04071_b200 import Lut
        from paper_2203_04071_b200 import _lib as ax
        self.ax = ax
        c = datagen.config0()
        self.lut = Lut(8, c.lut)
        self.A_host = torch.from_numpy(c.A).pin_memory()
        self.A = self.A_host.to(dev)
        self.W = torch.from_numpy(c.W).to(dev)
        self.C = torch.empty(64, 64, dtype=torch.int32, device=dev)
        self.C_host = torch.empty(64, 64, dtype=torch.int32).pin_memory()
        self.x, self.x_host = self.A, self.A_host
        self.timer = timer
        self.lookups_rank = 64 * 64 * 256
        self.lookups_total = self.lookups_rank * world
        self.launches = 1
        self.in_bytes, self.out_bytes = self.A.numel(), self.C.numel() * 4
        self.desc = {"workload": "BJ configs[0]: raw LUT-GEMM A int8 [64x256] x W int8 [256x64], "
                                 "randerr LUT (exact product + U[-64,64]), int32 output",
                     "global_batch": 64}

    def step(self, stream, dist):
        self.timer("pre", stream)
        self.ax.axq_lut_gemm(self.A, self.W, self.lut, self.C, stream)
        self.timer("post", stream)

    def h2d(self):
        self.A.copy_(self.A_host, non_blocking=True)

    def d2h(self):
        self.C_host.copy_(self.C, non_blocking=True)

    def extra(self):
        return {}


class LstmWL:
    name = "lstm"
    scaling = "weak"

    def __init__(self, dev, rank, world, timer):
        import torch
        import datagen
        from paper_2203_04071_b200 import Lut
        from paper_2203_04071_b200.lstm import ApproxLSTM
        c = datagen.config4()
        self.x_host = torch.from_numpy(c.x).pin_memory()
        self.x = self.x_host.to(dev)
        self.nets = {}
        self.replay = {}
        for b in (4, 6, 8):
            n = ApproxLSTM(c.W_ih, c.W_hh, c.b_ih, c.b_hh, Lut(b, c.luts[b]), dev)
            n.calibrate(self.x)
            self.replay[b] = n.capture(self.x)      # 128-step static forward as a CUDA graph
            self.nets[b] = n
        torch.cuda.synchronize()
        T, B, _ = self.x.shape
        per_b = self.nets[8].lookups(T, B)
        self.lookups_rank = 3 * per_b
        self.lookups_total = self.lookups_rank * world
        self.launches = 3 * 3   # per bit width: quantize x, ih GEMM, persistent recurrence
        self.in_bytes = self.x.numel() * 4
        self.out_bytes = 3 * T * B * 1024 * 4
        self.h_host = torch.empty(3, T, B, 1024).pin_memory()
        self.per_bit_ms = {}
        self.desc = {"workload": "BJ configs[4]: LSTM input 512, hidden 1024, seq 128, batch 64, "
                                 "approximate ih/hh gate GEMMs at b = 4, 6, 8 (randerr LUTs), "
                                 "static scales calibrated untimed; each forward replayed as one "
                                 "CUDA graph", "lookups_per_bitwidth": per_b}
        self.timer = timer

    def step(self, stream, dist):
        import torch
        for b, n in self.nets.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            self.timer("pre", stream)    # graph replay: the LUT-kernel time is bounded by the
            self.replay[b]()             # whole forward (GEMMs + cell kernels), conservative
            self.timer("post", stream)
            e1.record(stream)
            self.per_bit_ms.setdefault(b, []).append((e0, e1))

    def h2d(self):
        self.x.copy_(self.x_host, non_blocking=True)

    def d2h(self):
        for i, n in enumerate(self.nets.values()):
            hs, _ = n._bufs[(self.x.shape[0], self.x.shape[1])]["hs"], None
            self.h_host[i].copy_(hs, non_blocking=True)

    def extra(self):
        out = {}
        for b, ev in self.per_bit_ms.items():
            out["b%d_ms" % b] = round(statistics.median(a.elapsed_time(c) for a, c in ev), 3)
        if all(k in out for k in ("b4_ms", "b6_ms", "b8_ms")):
            out["ratio_b6_b4"] = round(out["b6_ms"] / out["b4_ms"], 3)
            out["ratio_b8_b6"] = round(out["b8_ms"] / out["b6_ms"], 3)
            out["paper_ratio_per_2_bits"] = "~2.1x (P:322, Xeon AVX2)"
        return out


WORKLOADS = {"resnet": ResNetWL, "conv": ConvWL, "linear": LinearWL, "lstm": LstmWL, "gemm": GemmWL}


def _time_ms(fn, stream, reps=20, warm=3, flush=None):
    """Median CUDA-event time of fn() on `stream` (L2 flushed before each rep when given)."""
    import torch
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def imma_reference(wl, stream, flush):
    """SURVEY §8(d) speed reference row: the EXACT int8 GEMM of the same shape on cuBLASLt IMMA
    (torch._int_mm), labelled as such -- it computes sum a*w, not the approximate sums.  c2 uses
    this library's im2col of the int8 codes + _int_mm (the explicit im2col GEMM of P:119)."""
    import torch
    from paper_2203_04071_b200 import _lib as ax
    dev = stream.device
    out = {"label": "exact int8 GEMM (cuBLASLt IMMA via torch._int_mm): a speed reference, NOT the "
                    "approximate path (no lookups)"}
    try:
        if wl.name == "gemm":
            A, W = wl.A, wl.W
            Wt = W.t().contiguous()
            ms = _time_ms(lambda: torch._int_mm(A, Wt), stream, flush=flush)
            out.update(shape="M64 N64 K256", ms=round(ms, 5), macs=64 * 64 * 256)
        elif wl.name == "linear":
            q = wl.bufs["qa"]
            Wt = wl.layer.qw.t().contiguous()
            ms = _time_ms(lambda: torch._int_mm(q, Wt), stream, flush=flush)
            M = q.shape[0]
            out.update(shape="M%d N1024 K1024" % M, ms=round(ms, 5), macs=M * 1024 * 1024)
        elif wl.name == "conv":
            Nb, H, W_, C = wl.qx.shape
            Ho, Wo = ax.axq_conv2d_out_hw(wl.d)
            cols = torch.empty(Nb * Ho * Wo, 576, dtype=torch.int8, device=dev)
            Wt = wl.layer.qw.reshape(wl.layer.Kout, -1).t().contiguous()
            im = lambda: ax.axq_im2col_nhwc_i8(wl.qx, 0, 3, 3, (1, 1), (1, 1), cols, stream)
            im()
            gm = lambda: torch._int_mm(cols, Wt)
            ms_g = _time_ms(gm, stream, flush=flush)
            ms_i = _time_ms(im, stream, flush=flush)
            out.update(shape="im2col [%d x 576] x [576 x 64]" % cols.shape[0], ms=round(ms_g + ms_i, 5),
                       gemm_ms=round(ms_g, 5), im2col_ms=round(ms_i, 5), macs=cols.shape[0] * 576 * 64)
        else:
            return None
        out["gmacs"] = round(out["macs"] / (out["ms"] * 1e-3) / 1e9, 2)
    except Exception as e:      # reported, never fatal: it is a reference row only
        out["error"] = repr(e)[:200]
    return out


def qdq_split(wl, stream, flush):
    """the unfused Q | GEMM | DQ split of c1 / c2 (the analogue of P:320's ~10 %
    quantize + dequantize share): amax + scale + quantize, the LUT kernel with raw int32
    output, and the stand-alone dequantize, each timed alone (L2 flushed), next to the fused
    step."""
    import torch
    from paper_2203_04071_b200 import _lib as ax
    L = wl.layer
    if wl.name == "conv":
        Nb, H, W_, C = wl.qx.shape
        Ho, Wo = ax.axq_conv2d_out_hw(wl.d)
        acc = torch.empty(Nb, Ho, Wo, L.Kout, dtype=torch.int32, device=wl.x.device)

        def q():
            ax.axq_amax(wl.x, L.d_amax_a, stream)
            ax.axq_scale(L.d_amax_a, 8, L.d_scale_a, stream)
            ax.axq_quantize_nchw_to_nhwc(wl.x, L.d_scale_a, 8, wl.qx, stream)

        def g():
            if L.wp is not None:
                ax.axq_lut_conv2d_wp(wl.d, wl.qx, L.wp, None, acc, stream)
            else:        # int32 table (--lut err1e5): the resident-table kernel, raw int32 out
                ax.axq_lut_conv2d(wl.d, wl.qx, L.qw, L.lut, acc, stream)

        def dq():
            ax.axq_dequantize_nhwc_to_nchw(acc, L.d_scale_a, L.d_scale_w, None, wl.y, stream)
    elif wl.name == "linear":
        qa = wl.bufs["qa"]
        acc = torch.empty(qa.shape[0], L.N, dtype=torch.int32, device=wl.x.device)

        def q():
            ax.axq_amax(wl.x, L.d_amax_a, stream)
            ax.axq_scale(L.d_amax_a, 8, L.d_scale_a, stream)
            ax.axq_quantize(wl.x, L.d_scale_a, 8, qa, stream)

        def g():   # raw int32 output: the per-row-gather kernel with its exact split-K
            ax.axq_lut_gemm(qa, L.qw, L.lut, acc, stream)

        def dq():
            ax.axq_dequantize(acc, L.d_scale_a, L.d_scale_w, L.bias, wl.y, stream)
    else:
        return None
    tq, tg, tdq = (_time_ms(f, stream, flush=flush) for f in (q, g, dq))
    tot = tq + tg + tdq
    return {"q_ms": round(tq, 5), "lut_gemm_ms": round(tg, 5), "dq_ms": round(tdq, 5),
            "qdq_share": round((tq + tdq) / tot, 4),
            "paper": "P:320: quantization + dequantization ~10 % of the time (Xeon, AVX2)",
            "note": "unfused pieces timed alone; the bench step fuses DQ (and for ResNet layers Q) "
                    "into the LUT kernel's epilogue"}


def count_launches(wl, stream, dist):
    """Kernels of this library (namespace axq::) one step launches, counted by the CUDA profiler
    (CUPTI activity records, graph replays included) over one untimed step; None when the
    profiler is unavailable (the workload's static count is reported instead)."""
    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            wl.step(stream, dist)
            torch.cuda.synchronize()
        n = sum(1 for e in prof.events() if "axq::" in e.name)
        return n if n > 0 else None
    except Exception:
        return None


def run_ours(args, rank, world, local_rank):
    import torch

    # AXQ_BENCH_ONE_GPU=1 (path check only, not a measurement): every rank on cuda:0 over gloo,
    # so the N > 1 code path can be exercised on a one-GPU box
    one_gpu = os.environ.get("AXQ_BENCH_ONE_GPU") == "1"
    dev = torch.device("cuda", 0 if one_gpu else local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    timer = KernelTimer()
    global QUANTIZER, LUT_KIND
    QUANTIZER = args.quantizer
    LUT_KIND = args.lut
    wl = WORKLOADS[args.workload](dev, rank, world, timer)
    stream = torch.cuda.current_stream()
    # L2 flush buffer (> 126 MB L2) written before every timed step, outside the timed region
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    for _ in range(max(args.warmup, 0)):
        wl.step(stream, dist)
    torch.cuda.synchronize()
    launches_step = count_launches(wl, stream, dist)
    torch.cuda.synchronize()
    if hasattr(wl, "per_bit_ms"):
        wl.per_bit_ms.clear()

    step_ms, kern_ms = [], []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            timer.reset()
            timer.enabled = True
            s0.record(stream)
            wl.step(stream, dist)
            s1.record(stream)
            s1.synchronize()
            timer.enabled = False
            step_ms.append(s0.elapsed_time(s1))
            kern_ms.append(timer.total_ms())
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    total_ms = sum(step_ms)
    per_rank_ms = [round(total_ms / args.steps, 4)]
    if dist:
        t = torch.tensor([total_ms], device=dev)
        parts = [torch.zeros(1, device=dev) for _ in range(world)]
        dist.all_gather(parts, t)
        per_rank_ms = [round(p.item() / args.steps, 4) for p in parts]
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = t.item()

    e2e = None
    if not args.no_e2e:
        pipelined = getattr(wl, "pipelined_e2e", False)
        n_e2e = max(2, min(args.steps, 10 if pipelined else 5))
        if pipelined:
            # double-buffered inputs: step i+1's H2D runs on a copy stream while step i computes;
            # every step still copies its own inputs in and its result out inside the timed region
            copy_s = torch.cuda.Stream(dev)
            bufs = [wl.x, torch.empty_like(wl.x)]
            copied = [torch.cuda.Event(), torch.cuda.Event()]
            free = [torch.cuda.Event(), torch.cuda.Event()]
            # large outputs (conv): double-buffered too, the D2H on its own stream (PCIe carries
            # both directions at once)
            out2 = getattr(wl, "pipelined_out", False)
            if out2:
                d2h_s = torch.cuda.Stream(dev)
                ybufs = [wl.y, torch.empty_like(wl.y)]
                done = [torch.cuda.Event(), torch.cuda.Event()]
                drained = [torch.cuda.Event(), torch.cuda.Event()]
            flush.fill_(1.0)
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            copy_s.wait_event(a)
            with torch.cuda.stream(copy_s):
                bufs[0].copy_(wl.x_host, non_blocking=True)
                copied[0].record(copy_s)
            for i in range(n_e2e):
                cur, nxt = i % 2, (i + 1) % 2
                stream.wait_event(copied[cur])
                if i + 1 < n_e2e:
                    if i >= 1:
                        copy_s.wait_event(free[nxt])          # step i-1 finished reading it
                    with torch.cuda.stream(copy_s):
                        bufs[nxt].copy_(wl.x_host, non_blocking=True)
                        copied[nxt].record(copy_s)
                wl.x = bufs[cur]
                if out2:
                    if i >= 2:
                        stream.wait_event(drained[cur])     # step i-2's result has left the device
                    wl.y = ybufs[cur]
                flush.fill_(1.0)      # L2 flushed before every step, inside the interval
                wl.step(stream, dist)
                free[cur].record(stream)
                if out2:
                    done[cur].record(stream)
                    d2h_s.wait_event(done[cur])
                    with torch.cuda.stream(d2h_s):
                        wl.d2h()
                        drained[cur].record(d2h_s)
                else:
                    wl.d2h()
            if out2:
                stream.wait_event(drained[(n_e2e - 1) % 2])
            b.record(stream)
            b.synchronize()
            wl.x = bufs[0]
            if out2:
                wl.y = ybufs[0]
            e_tot = a.elapsed_time(b)
            e_ms = [e_tot / n_e2e] * n_e2e
        else:
            e_ms = []
            for _ in range(n_e2e):
                flush.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                if dist:
                    dist.barrier()
                a.record(stream)
                wl.h2d()
                wl.step(stream, dist)
                wl.d2h()
                b.record(stream)
                b.synchronize()
                e_ms.append(a.elapsed_time(b))
        e_tot = sum(e_ms)
        if dist:
            t = torch.tensor([e_tot], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_tot = t.item()
        e2e = {"value": round(wl.lookups_total * len(e_ms) / (e_tot * 1e-3) / 1e9, 3),
               "unit": "GMAC/s", "h2d_bytes_per_step": wl.in_bytes,
               "d2h_bytes_per_step": wl.out_bytes, "ms_per_step": round(e_tot / len(e_ms), 4),
               "steps": len(e_ms),
               "overlap": ("double-buffered inputs: each step's H2D (pinned host -> device, on a "
                           "copy stream) overlaps the previous step's compute; the D2H of each "
                           "step's result follows it (double-buffered outputs on a D2H stream "
                           "when they are large); L2 flushed before every step inside the "
                           "interval; one CUDA-event interval over all steps") if pipelined else
                          "none: H2D, step, D2H serial per step (CUDA graph replay on fixed buffers)"}

    result = None
    if rank == 0:
        peaks, peak_src = measured_peaks()
        sm = torch.cuda.get_device_properties(dev).multi_processor_count
        clocks = clk.summary()
        f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        roof = sm * LANES * f_max / 1e9                                  # Glookups/s
        smem_peak = sm * 128 * f_max / 1e9                               # 1 B per lookup
        kmean = statistics.mean(kern_ms)
        achieved = wl.lookups_rank / (kmean * 1e-3) / 1e9
        value = wl.lookups_total * args.steps / (total_ms * 1e-3) / 1e9
        f_meas = (clocks.get("sm_mhz") or 0) * 1e6
        cfg = dict(wl.desc, parallelism="dp%d (%s)" % (world, "batch-sharded, NCCL all-gather "
                   "of logits" if wl.scaling == "strong" else "independent replicas"),
                   l2="flushed before every timed step (256 MiB write)", lut_repr=wl.lut.repr
                   if hasattr(wl, "lut") else "delta8")
        if hasattr(wl, "extra"):
            cfg.update(wl.extra())
        result = {
            "metric": "approximate GMAC/s (LUT lookups/s) per B200 and % of smem-lookup roofline",
            "value": round(value, 3), "unit": "GMAC/s", "n_gpus": world, "steps": args.steps,
            "per_rank_ms_per_step": per_rank_ms, "replica_checksum": getattr(wl, "checksum", None),
            "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
            "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None, "dtype": "int8",
            "data": "synthetic (seeded; DESIGN.md input recipe), random-init weights",
            "config": cfg,
            "roofline": {"bound": "smem", "kernel": "LUT kernels (lut_p4w_kernel packed-table "
                         "tcgen05 path in its 896- and 512-row shapes, p4_pack_tables_kernel for "
                         "per-call activation tables, lut_mm_kernel for small M, lstm_rec_kernel "
                         "for the LSTM recurrence: all LUT launches of the step, CUDA events "
                         "around each on the launching stream)",
                         "achieved": round(achieved, 2), "peak": round(smem_peak, 2),
                         "unit": "Glookup/s", "frac": round(achieved / smem_peak, 4),
                         "peak_basis": "shared-memory byte bound: %d SMs x 128 B per SM clock "
                                       "(32 banks x 4 B) x %.0f MHz (%s sm_max_mhz) at 1 table "
                                       "byte per lookup (int8 E entries) -- no table-lookup "
                                       "design can exceed it (DESIGN.md 5.4)"
                                       % (sm, f_max / 1e6, peak_src),
                         "frac_at_measured_clock": round(achieved / (sm * 128 * f_meas / 1e9), 4)
                         if f_meas else None,
                         "design_roofline": {
                             "bound": "issue", "peak": round(sm * f_max / 1e9 * DESIGN_LOOKUPS_PER_CLK, 2),
                             "unit": "Glookup/s",
                             "frac": round(achieved / (sm * f_max / 1e9 * DESIGN_LOOKUPS_PER_CLK), 4),
                             "basis": DESIGN_BASIS},
                         "metric_roofline": {
                             "peak": round(roof, 2), "unit": "Glookup/s", "frac": round(achieved / roof, 4),
                             "basis": "BASELINE metric's smem-lookup roofline: %d SMs x 32 lanes x "
                                      "%.0f MHz, one 32-lane wavefront per SM clock with one "
                                      "lookup per lane; the packed tables serve 4 lookups per "
                                      "lane per load, so this frac exceeds 1" % (sm, f_max / 1e6)},
                         "kernel_ms_per_step": round(kmean, 4),
                         "kernel_share_of_step": round(kmean / (total_ms / args.steps), 4),
                         "traffic": committed_traffic(wl.name),
                         "traffic_basis": "dram__bytes_read.sum + dram__bytes_write.sum summed "
                                          "over the step's LUT-kernel launches, one ncu capture "
                                          "(profiles/traffic.json); per step, like achieved"},
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": (launches_step if launches_step else wl.launches) * args.steps,
            "us_per_step": round(total_ms / args.steps * 1e3, 2) if wl.name == "gemm" else None,
            "gpu_launches_source": "CUPTI (torch.profiler) count of axq:: kernels in one untimed "
                                   "step x steps" if launches_step else "static per-step count x steps",
        }
    if rank == 0 and world == 1 and wl.name in ("gemm", "linear", "conv"):
        result["speed_reference_imma"] = imma_reference(wl, stream, flush)
        if wl.name in ("linear", "conv"):
            result["qdq_split"] = qdq_split(wl, stream, flush)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return result


# ---------------------------------------------------------------------------------------
# oracle (CPU) timing: cpu_baseline leg and --impl reference
# ---------------------------------------------------------------------------------------
class OracleSample:
    """A bounded sample of the workload run by the oracle as it stands (all host cores)."""

    def __init__(self, workload):
        import datagen
        import oracle
        self.o = oracle
        self.w = workload
        if workload == "resnet":
            from oracle import models
            self.lut = datagen.lut_randerr(8, 0, 2)
            self.net = models.ResNetOracle(self.lut, 8, config=3)
            self.x = datagen.config3_images(8)
            self.scales = self.net.calibrate(self.x[:1])      # untimed; values only
            self.per_unit = models.resnet_macs(self.net.layers)
            self.unit = "image"
        elif workload == "conv":
            self.c = datagen.config2()
            self.per_unit = self.c.x[0].size * 64 * 9
            self.unit = "image"
        elif workload == "linear":
            self.c = datagen.config1()
            self.per_unit = 256 * 1024 * 1024
            self.unit = "full layer"
        elif workload == "gemm":
            self.c = datagen.config0()
            self.per_unit = 64 * 64 * 256
            self.unit = "full GEMM"
        else:
            from oracle import models
            c = datagen.config4()
            self.lstm = models.LstmOracle(c, 8)
            self.T = c.x.shape[0]
            self.per_unit = c.x.shape[1] * 4096 * (512 + 1024)
            self.unit = "time step (b=8)"

    def run(self, n):
        o = self.o
        t0 = time.perf_counter()
        if self.w == "resnet":
            self.net.forward(self.x[:n], self.scales)
        elif self.w == "conv":
            c = self.c
            sa = o.scale(o.amax(c.x), 8)
            qw, sw = o.quantize_tensor(c.W, 8)
            acc = o.lut_conv2d(o.quantize(c.x[:n], sa, 8), qw, c.lut, 8, c.stride, c.pad)
            o.dequantize(acc, sa, sw, None, 1)
        elif self.w == "linear":
            for _ in range(n):
                o.linear(self.c.x, self.c.W, self.c.b, self.c.lut, 8)
        elif self.w == "gemm":
            for _ in range(n):
                o.lut_gemm(self.c.A, self.c.W, self.c.lut, 8)
        else:
            c = self.lstm.c
            keep = c.x
            c.x = keep[:n]
            try:
                self.lstm.run((o.scale(o.amax(keep), 8), np.float32(1.0 / 127)))
            finally:
                c.x = keep
        return time.perf_counter() - t0


def cpu_baseline(args, budget_s: float = 12.0):
    """The oracle as it stands on the host cores: all threads (the reported value) and one
    thread on the same sample, with the measured OpenMP speedup."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    s = OracleSample(args.workload)
    t1 = s.run(1)
    cap = {"resnet": 8, "conv": 128, "linear": 50, "lstm": 128, "gemm": 2000}[args.workload]
    n = int(max(1, min(cap, budget_s / max(t1, 1e-3))))
    t = s.run(n) if n > 1 else t1
    used = oracle.max_threads()
    # one thread on a smaller sample (about budget_s / 3 of work)
    oracle.set_threads(1)
    n1 = int(max(1, min(n, (budget_s / 3) / max(t1 * used, 1e-3))))
    ts = s.run(n1)
    oracle.set_threads(cores)
    v_all = n * s.per_unit / t / 1e9
    v_one = n1 * s.per_unit / ts / 1e9
    return {"value": round(v_all, 4), "unit": "GMAC/s", "cores": used, "kind": "oracle",
            "sample": "%d %s(s) of the same workload, %.1f s (OpenMP parallel-for over the "
                      "outermost loop, all host cores)" % (n, s.unit, t),
            "single_thread": {"value": round(v_one, 4), "unit": "GMAC/s", "cores": 1,
                              "sample": "%d %s(s), %.1f s" % (n1, s.unit, ts)},
            "omp_speedup": round(v_all / v_one, 2)}


def run_reference(args, rank):
    """--impl reference: the oracle as it stands, on the host cores, same metric/config."""
    if rank != 0:
        return None
    import oracle
    oracle.set_threads(len(os.sched_getaffinity(0)))
    s = OracleSample(args.workload)
    for _ in range(max(args.warmup, 0)):
        s.run(1)
    ts = [s.run(1) for _ in range(args.steps)]
    tot = sum(ts)
    value = s.per_unit * args.steps / tot / 1e9
    base = {"resnet": ("BJ configs[3] ResNet-50-shaped approximate forward", "strong"),
            "conv": ("BJ configs[2] approximate conv2d", "strong"),
            "linear": ("BJ configs[1] approximate linear", "strong"),
            "gemm": ("BJ configs[0] raw LUT-GEMM", "weak"),
            "lstm": ("BJ configs[4] LSTM, b=8", "weak")}[args.workload]
    sample = "1 %s per step (a bounded sample of the same workload)" % s.unit
    return {"metric": "approximate GMAC/s (LUT lookups/s) per B200 and % of smem-lookup roofline",
            "impl": "reference", "value": round(value, 4), "unit": "GMAC/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(tot / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": base[1], "vs_baseline": None, "dtype": "int8",
            "data": "synthetic (seeded)",
            "config": {"workload": base[0] + " (oracle on the host cores)",
                       "parallelism": "OpenMP, host cores"},
            "cpu_baseline": {"value": round(value, 4), "unit": "GMAC/s",
                             "cores": oracle.max_threads(), "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 4), "unit": "GMAC/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    args = parse()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` run directly: launch the N ranks (one per GPU, NCCL) ourselves,
        # exactly as the driver's torchrun command would
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE %d" % (args.gpus, world))
    if world > 1:
        # the communicator set-up lines (ranks, NVLink / NVLS transport) go to stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
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
