"""Seeded SIREN-init T-MLP parameters and the canonical FP32 blob layout.

Init (BASELINE.json configs; SPEC S:129 init_params; readings R5/R6):
  layer 1 weights  W_1 ~ U(-1/3, 1/3)                (first SIREN layer, U(+-1/in_dim))
  hidden weights   W_i ~ U(-sqrt(6/H)/w0, +sqrt(6/H)/w0), i >= 2
  biases           b_i ~ U(-1/sqrt(fan_in), +1/sqrt(fan_in))
  tail weights     a_i (a_i0, a_i1) ~ same law as the hidden weights ("same init")
  tail biases      c_i (c_i0, c_i1) ~ same law as a hidden bias, U(+-1/sqrt(H))

Canonical blob order (include/sand.h, sand_load_weights):
  for i = 1..L: W_i [H][fan_in] row-major (fan_in = 3 if i == 1 else H), b_i [H]
  tails LINEAR: for i = 1..L: a_i [H], c_i
  tails MULT  : a_1 [H], c_1, then for i = 2..L: a_i0 [H], c_i0, a_i1 [H], c_i1
"""
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .rng import uniform

LINEAR = 0
MULT = 1


@dataclass
class TMlpSpec:
    L: int
    H: int
    omega0: float = 30.0
    tail: int = LINEAR  # 0 = LINEAR, 1 = MULT
    seed: int = 0


@dataclass
class TMlpParams:
    spec: TMlpSpec
    W: List[np.ndarray]            # W[i-1]: [H][fan_in] float32
    b: List[np.ndarray]            # b[i-1]: [H] float32
    a: List[np.ndarray]            # LINEAR tail weights (or a_i0 for MULT i>=2; a_1 always)
    c: List[float]                 # LINEAR tail biases (or c_i0)
    a1: List[np.ndarray] = field(default_factory=list)   # MULT only: a_i1 for i = 2..L (index i-2)
    c1: List[float] = field(default_factory=list)        # MULT only: c_i1


def _u32(seed, stream, n, bound):
    return uniform(seed, stream, n, -bound, bound).astype(np.float32)


def make_weights(spec: TMlpSpec) -> TMlpParams:
    L, H, w0, s = spec.L, spec.H, spec.omega0, spec.seed
    hid = np.sqrt(6.0 / H) / w0
    W, b, a, c, a1, c1 = [], [], [], [], [], []
    for i in range(1, L + 1):
        fan_in = 3 if i == 1 else H
        wb = (1.0 / 3.0) if i == 1 else hid
        W.append(_u32(s, 16 * i + 0, H * fan_in, wb).reshape(H, fan_in))
        b.append(_u32(s, 16 * i + 1, H, 1.0 / np.sqrt(fan_in)))
        a.append(_u32(s, 16 * i + 2, H, hid))
        c.append(float(_u32(s, 16 * i + 3, 1, 1.0 / np.sqrt(H))[0]))
        if spec.tail == MULT and i >= 2:
            a1.append(_u32(s, 16 * i + 4, H, hid))
            c1.append(float(_u32(s, 16 * i + 5, 1, 1.0 / np.sqrt(H))[0]))
    return TMlpParams(spec, W, b, a, c, a1, c1)


def blob_len(L: int, H: int, tail: int) -> int:
    n = 3 * H + H + (L - 1) * (H * H + H)
    if tail == LINEAR:
        n += L * (H + 1)
    else:
        n += (H + 1) + (L - 1) * 2 * (H + 1)
    return n


def pack_blob(p: TMlpParams) -> np.ndarray:
    L, H, tail = p.spec.L, p.spec.H, p.spec.tail
    parts = []
    for i in range(L):
        parts.append(p.W[i].reshape(-1))
        parts.append(p.b[i])
    if tail == LINEAR:
        for i in range(L):
            parts.append(p.a[i])
            parts.append(np.array([p.c[i]], np.float32))
    else:
        parts.append(p.a[0])
        parts.append(np.array([p.c[0]], np.float32))
        for i in range(1, L):
            parts.append(p.a[i])
            parts.append(np.array([p.c[i]], np.float32))
            parts.append(p.a1[i - 1])
            parts.append(np.array([p.c1[i - 1]], np.float32))
    out = np.concatenate(parts).astype(np.float32)
    assert out.size == blob_len(L, H, tail)
    return out


def unpack_blob(blob: np.ndarray, spec: TMlpSpec) -> TMlpParams:
    L, H, tail = spec.L, spec.H, spec.tail
    blob = np.asarray(blob, np.float32)
    assert blob.size == blob_len(L, H, tail)
    o = 0
    W, b, a, c, a1, c1 = [], [], [], [], [], []
    for i in range(L):
        fi = 3 if i == 0 else H
        W.append(blob[o:o + H * fi].reshape(H, fi).copy()); o += H * fi
        b.append(blob[o:o + H].copy()); o += H
    if tail == LINEAR:
        for i in range(L):
            a.append(blob[o:o + H].copy()); o += H
            c.append(float(blob[o])); o += 1
    else:
        a.append(blob[o:o + H].copy()); o += H
        c.append(float(blob[o])); o += 1
        for i in range(1, L):
            a.append(blob[o:o + H].copy()); o += H
            c.append(float(blob[o])); o += 1
            a1.append(blob[o:o + H].copy()); o += H
            c1.append(float(blob[o])); o += 1
    return TMlpParams(spec, W, b, a, c, a1, c1)
