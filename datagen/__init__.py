"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no quantization, no LUT-GEMM, no
convolution, no dequantization).  It only draws the tensors BASELINE.json's configs name
and builds the approximate-multiplier tables (ACUs), which the method treats as black-box
inputs ("Any arbitrary ACU can be specified ... as long as the multiplier's output is
deterministic", §III.B).

Generator recipe:
  * numpy ``default_rng(seed)`` (PCG64), seed = 220304071 + 1000*config + tensor_index;
  * normals: ``standard_normal(dtype=float32)`` times an fp32 std;
  * uniforms: drawn in float64, cast to float32;
  * integers: ``integers(lo, hi, size, dtype=np.int64)`` then cast.

The paper's datasets (CIFAR10, ImageNet, IMDB, MNIST; Table I) and the
EvoApprox multipliers (mul8s_1L2H, mul12s_2KM; Table II) are not in the
container; these seeded tensors of the configs' shapes and distributions stand in for them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SEED_BASE = 220304071


def rng_for(config: int, tensor_index: int) -> np.random.Generator:
    return np.random.default_rng(SEED_BASE + 1000 * config + tensor_index)


def normal(config: int, idx: int, shape, std: float = 1.0) -> np.ndarray:
    x = rng_for(config, idx).standard_normal(size=shape, dtype=np.float32)
    if std != 1.0:
        x = x * np.float32(std)
    return x


def uniform(config: int, idx: int, shape, lo: float, hi: float) -> np.ndarray:
    return rng_for(config, idx).uniform(lo, hi, size=shape).astype(np.float32)


def int_uniform(config: int, idx: int, shape, lo: int, hi_excl: int) -> np.ndarray:
    return rng_for(config, idx).integers(lo, hi_excl, size=shape, dtype=np.int64)


# --------------------------------------------------------------------------------------
# ACU tables.  Host format: int32 array of length 2^(2b), entry index
# (ua << b) | uw, ua/uw the b-bit two's-complement patterns; first index = ACTIVATION.
# --------------------------------------------------------------------------------------

def signed_values(bits: int) -> np.ndarray:
    """sx(u) for u = 0 .. 2^b - 1 (two's-complement sign extension of the b-bit pattern)."""
    u = np.arange(1 << bits, dtype=np.int64)
    return np.where(u >= (1 << (bits - 1)), u - (1 << bits), u)


def lut_exact(bits: int) -> np.ndarray:
    """The exact multiplier: T[ua][uw] = sx(ua) * sx(uw)."""
    v = signed_values(bits)
    return np.outer(v, v).astype(np.int32).reshape(-1)


def lut_randerr(bits: int, config: int, idx: int) -> np.ndarray:
    """Exact product + seeded uniform integer error in [-2^(b-2), 2^(b-2)] (BJ:c0, BJ:c4),
    one ``integers(..., endpoint=True)`` draw of shape (2^b, 2^b) in index order (A9)."""
    e = 1 << (bits - 2)
    err = rng_for(config, idx).integers(-e, e, size=(1 << bits, 1 << bits), endpoint=True,
                                        dtype=np.int64)
    return (lut_exact(bits).astype(np.int64) + err.reshape(-1)).astype(np.int32)


def lut_bigerr(bits: int, err: int, config: int, idx: int) -> np.ndarray:
    """Exact product + seeded uniform integer error in [-err, err] (one endpoint-inclusive draw
    in index order, as lut_randerr): an ACU whose error does not fit int8 (e.g. err = 2000), the
    case the int8-E packed tables cannot hold (VERDICT r1 "fast-path cliff")."""
    e = rng_for(config, idx).integers(-err, err, size=(1 << bits, 1 << bits), endpoint=True,
                                      dtype=np.int64)
    return (lut_exact(bits).astype(np.int64) + e.reshape(-1)).astype(np.int32)


def lut_trunc4() -> np.ndarray:
    """BJ:c1 "exact product with low-bit truncation error (drop product bits 0-3)":
    p & ~0xF on the two's-complement product."""
    return (lut_exact(8).astype(np.int64) & ~np.int64(0xF)).astype(np.int32)


# --------------------------------------------------------------------------------------
# Configs (BASELINE.json configs[0..4]); SURVEY §8(d) "Synthetic inputs" table.
# --------------------------------------------------------------------------------------

@dataclass
class GemmCase:
    A: np.ndarray      # int8 [M][K] activations
    W: np.ndarray      # int8 [N][K] weights (y = x W^T)
    lut: np.ndarray    # int32 [2^(2b)]
    bits: int


def config0() -> GemmCase:
    """c0: A int8 [64x256], W int8 [256x64] (K x N) uniform on [-128,127]; randerr_8 LUT."""
    A = int_uniform(0, 0, (64, 256), -128, 128).astype(np.int8)
    Wkn = int_uniform(0, 1, (256, 64), -128, 128).astype(np.int8)
    W = np.ascontiguousarray(Wkn.T)          # A21: harness transposes to [N][K]
    return GemmCase(A=A, W=W, lut=lut_randerr(8, 0, 2), bits=8)


@dataclass
class LinearCase:
    x: np.ndarray      # fp32 [M][K]
    W: np.ndarray      # fp32 [N][K] ([out][in], A20)
    b: np.ndarray      # fp32 [N]
    lut: np.ndarray
    bits: int


def config1() -> LinearCase:
    x = normal(1, 0, (256, 1024))
    W = normal(1, 1, (1024, 1024), 0.02)
    b = normal(1, 2, (1024,), 0.01)
    return LinearCase(x=x, W=W, b=b, lut=lut_trunc4(), bits=8)


@dataclass
class ConvCase:
    x: np.ndarray      # fp32 NCHW
    W: np.ndarray      # fp32 [K][C][R][S] (PyTorch layout)
    bias: np.ndarray | None
    stride: tuple
    pad: tuple
    lut: np.ndarray
    bits: int


def config2(batch: int = 128) -> ConvCase:
    """c2: x = ReLU(N(0,1)) [128,64,56,56]; W = sqrt(2/576) N [64,64,3,3]; no bias;
    LUT = the identical array c0 uses (c0 seed, tensor index 2)."""
    x = normal(2, 0, (128, 64, 56, 56))
    if batch != 128:
        x = x[:batch]
    np.maximum(x, np.float32(0), out=x)
    W = normal(2, 1, (64, 64, 3, 3), math.sqrt(2.0 / 576.0))
    return ConvCase(x=np.ascontiguousarray(x), W=W, bias=None, stride=(1, 1), pad=(1, 1),
                    lut=lut_randerr(8, 0, 2), bits=8)


def random_int8(seed: int, shape, bits: int = 8, full_range: bool = True) -> np.ndarray:
    """Seeded b-bit operands for ragged-shape parity cases (tests only)."""
    lo = -(1 << (bits - 1)) if full_range else -((1 << (bits - 1)) - 1)
    return np.random.default_rng(seed).integers(lo, 1 << (bits - 1), size=shape,
                                                dtype=np.int64).astype(np.int8)


def random_int16(seed: int, shape, bits: int) -> np.ndarray:
    """Uniform b-bit signed codes in [-(2^(b-1) - 1), 2^(b-1) - 1] as int16 (NEXT-2 operands)."""
    q = (1 << (bits - 1)) - 1
    return np.random.default_rng(seed).integers(-q, q, size=shape, endpoint=True,
                                                dtype=np.int64).astype(np.int16)


def random_lut(seed: int, bits: int) -> np.ndarray:
    """A fully random ACU (no structure at all) for parity cases: every entry in
    [-2^(2b-2), 2^(2b-2)], so int16/int8 table representations are exercised where they fit."""
    lim = 1 << (2 * bits - 2)
    return np.random.default_rng(seed).integers(-lim, lim, size=1 << (2 * bits), endpoint=True,
                                                dtype=np.int64).astype(np.int32)


# --------------------------------------------------------------------------------------
# configs[3]: ResNet-50-shaped forward (weights are requested by each side with its own
# layer enumeration; tensor_index 0 = images, 1.. = weights in forward order, A16)
# --------------------------------------------------------------------------------------

def config3_images(batch: int = 256, start: int = 0) -> np.ndarray:
    """x ~ N(0,1) [256,3,224,224] fp32 (rows start..start+batch of the seeded batch)."""
    x = normal(3, 0, (256, 3, 224, 224))
    return np.ascontiguousarray(x[start:start + batch])


def kaiming_conv(config: int, idx: int, cout: int, cin: int, r: int, s: int) -> np.ndarray:
    """Kaiming-normal, fan_out mode: std = sqrt(2 / (Cout*R*S)) (A16)."""
    return normal(config, idx, (cout, cin, r, s), math.sqrt(2.0 / (cout * r * s)))


def kaiming_fc(config: int, idx: int, out_f: int, in_f: int) -> np.ndarray:
    """Kaiming-normal, fan_in mode: std = sqrt(2 / in) (A16)."""
    return normal(config, idx, (out_f, in_f), math.sqrt(2.0 / in_f))


def fc_bias(config: int, idx: int, out_f: int, in_f: int) -> np.ndarray:
    b = 1.0 / math.sqrt(in_f)
    return uniform(config, idx, (out_f,), -b, b)


# --------------------------------------------------------------------------------------
# configs[4]: LSTM (input 512, hidden 1024, seq 128, batch 64)
# --------------------------------------------------------------------------------------

@dataclass
class LstmCase:
    x: np.ndarray       # fp32 [T][B][I]
    W_ih: np.ndarray    # fp32 [4H][I]  gate order i, f, g, o
    W_hh: np.ndarray    # fp32 [4H][H]
    b_ih: np.ndarray
    b_hh: np.ndarray
    luts: dict          # bits -> int32 table


def config4(T: int = 128, B: int = 64, I: int = 512, H: int = 1024) -> LstmCase:
    s = 1.0 / 32.0
    x = normal(4, 0, (128, 64, 512))[:T, :B, :I]
    W_ih = uniform(4, 1, (4096, 512), -s, s)
    W_hh = uniform(4, 2, (4096, 1024), -s, s)
    b_ih = uniform(4, 3, (4096,), -s, s)
    b_hh = uniform(4, 4, (4096,), -s, s)
    if (I, H) != (512, 1024):   # reduced parity cases: sub-blocks of the same draws
        rows = np.concatenate([np.arange(g * 1024, g * 1024 + H) for g in range(4)])
        W_ih, W_hh = W_ih[rows][:, :I], W_hh[rows][:, :H]
        b_ih, b_hh = b_ih[rows], b_hh[rows]
    luts = {b: lut_randerr(b, 4, 10 + b) for b in (4, 6, 8)}
    return LstmCase(x=np.ascontiguousarray(x), W_ih=np.ascontiguousarray(W_ih),
                    W_hh=np.ascontiguousarray(W_hh), b_ih=np.ascontiguousarray(b_ih),
                    b_hh=np.ascontiguousarray(b_hh), luts=luts)


def network_weights(specs, config: int = 3) -> dict:
    """Weights for a layer list given as (name, kind, cout, cin, k, ...) tuples in forward
    order: tensor_index = position + 1; the fc bias takes the index after the fc weight."""
    W = {}
    for i, sp in enumerate(specs):
        name, kind, cout, cin, k = sp[:5]
        if kind == "conv":
            W[name] = kaiming_conv(config, i + 1, cout, cin, k, k)
        else:
            W[name] = kaiming_fc(config, i + 1, cout, cin)
            W[name + ".b"] = fc_bias(config, i + 2, cout, cin)
    return W
