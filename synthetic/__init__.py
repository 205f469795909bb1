"""Seeded synthetic gradient inputs shared by the oracle tests, the GPU parity
tests and bench.py.

This module holds NONE of the method's arithmetic: it only produces fp32
arrays (numpy, host memory) with the shapes, value distributions and edge
cases of the paper's workloads.  Both sides of every parity test consume the
same arrays.

Recipe ("Input recipe"):
  * SEED = 191108907.
  * Per-layer binade spread s_l ~ UniformInt[-24, -4] from
    default_rng([SEED, 999, l]) -- layers differ by many binades
    (Fig. `gradient_resnet50`).
  * g[r][l] = default_rng([SEED, r, l]).standard_normal(n_l, float32) * 2^s_l
    (bell-shaped, zero-mean histograms of Fig. `gradient_distribution`,
    P:137-157; a normal sample spans > 20 binades below its max).
  * 0.5 % exact zeros and one -0.0 per layer (A3 / A15 edge cases).
Shapes: torchvision ResNet-50 ``parameters()`` order (161 tensors,
25,557,032 elements) and HF ``BertModel`` bert-large (391 tensors,
335,141,888 elements), as recorded below.
"""
from __future__ import annotations

import numpy as np

SEED = 191108907

# torchvision.models.resnet50().parameters() numels, in order (161 tensors).
RESNET50_NUMELS = [
    9408, 64, 64, 4096, 64, 64, 36864, 64, 64, 16384, 256, 256, 16384, 256, 256, 16384, 64, 64,
    36864, 64, 64, 16384, 256, 256, 16384, 64, 64, 36864, 64, 64, 16384, 256, 256, 32768, 128,
    128, 147456, 128, 128, 65536, 512, 512, 131072, 512, 512, 65536, 128, 128, 147456, 128, 128,
    65536, 512, 512, 65536, 128, 128, 147456, 128, 128, 65536, 512, 512, 65536, 128, 128, 147456,
    128, 128, 65536, 512, 512, 131072, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 524288,
    1024, 1024, 262144, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 262144, 256, 256, 589824,
    256, 256, 262144, 1024, 1024, 262144, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 262144,
    256, 256, 589824, 256, 256, 262144, 1024, 1024, 262144, 256, 256, 589824, 256, 256, 262144,
    1024, 1024, 524288, 512, 512, 2359296, 512, 512, 1048576, 2048, 2048, 2097152, 2048, 2048,
    1048576, 512, 512, 2359296, 512, 512, 1048576, 2048, 2048, 1048576, 512, 512, 2359296, 512,
    512, 1048576, 2048, 2048, 2048000, 1000,
]
assert len(RESNET50_NUMELS) == 161 and sum(RESNET50_NUMELS) == 25_557_032


def bert_large_numels() -> list[int]:
    """HF BertModel(bert-large) ``parameters()`` numels in order (391 tensors)."""
    H, F, V, P, TT, L = 1024, 4096, 30522, 512, 2, 24
    out = [V * H, P * H, TT * H, H, H]                        # embeddings + LayerNorm
    for _ in range(L):
        out += [H * H, H, H * H, H, H * H, H]                 # q, k, v
        out += [H * H, H, H, H]                               # attn out dense + LayerNorm
        out += [F * H, F, H * F, H, H, H]                     # FFN in/out + LayerNorm
    out += [H * H, H]                                         # pooler
    return out


BERT_LARGE_NUMELS = bert_large_numels()
assert len(BERT_LARGE_NUMELS) == 391 and sum(BERT_LARGE_NUMELS) == 335_141_888

# Config 1 of BASELINE.json: "3 layers (4K, 64K, 256K fp32 grads) x 4 simulated ranks" (A18).
C1_NUMELS = [4096, 65536, 262144]

# The paper's own merged-layer workload: res5c_branch2a/2b/2c.
RES5C_NUMELS = [2048 * 512, 512 * 512 * 3 * 3, 512 * 2048]

# BASELINE.json configs as (name, numels, formats, ranks).
CONFIGS = {
    "c1": ("3 layers 4K/64K/256K, 4 simulated ranks, (5,2)", C1_NUMELS, [(5, 2)], [4]),
    "c2": ("ResNet-50 gradient shapes (161 tensors, 25.6M), (5,2)", RESNET50_NUMELS, [(5, 2)], [1, 2, 4, 8]),
    "c3": ("BERT-large gradient shapes (391 tensors, 335M), (4,3)", BERT_LARGE_NUMELS, [(4, 3)], [8]),
    "c4": ("format sweep on ResNet-50 shapes", RESNET50_NUMELS,
           [(3, 0), (5, 2), (4, 3), (5, 6), (5, 10)], [1, 8]),
}


def resnet50_hybrid_formats(low=(5, 2), last=(8, 23)) -> list[tuple[int, int]]:
    """Per-tensor formats of the paper's hybrid precision on ResNet-50 (P:545,
    Table last_layer_precision): the last (classification) layer --
    the fc weight and bias, the final two tensors -- in `last` (FP32 = (8, 23)),
    every other tensor in `low`."""
    n = len(RESNET50_NUMELS)
    return [tuple(low)] * (n - 2) + [tuple(last)] * 2


def layer_spread(l: int, seed: int = SEED) -> int:
    return int(np.random.default_rng([seed, 999, l]).integers(-24, -3))


def layer_grad(r: int, l: int, n: int, seed: int = SEED) -> np.ndarray:
    """Rank r's synthetic fp32 gradient for layer l with n elements."""
    rng = np.random.default_rng([seed, r, l])
    g = rng.standard_normal(n, dtype=np.float32)
    g *= np.float32(2.0 ** layer_spread(l, seed))
    zero = rng.random(n) < 0.005
    g[zero] = 0.0
    g[int(rng.integers(n))] = -0.0
    return g


def make_grads(numels, p: int, seed: int = SEED) -> list[list[np.ndarray]]:
    """grads[r][l] for p ranks."""
    return [[layer_grad(r, l, int(n), seed) for l, n in enumerate(numels)] for r in range(p)]


def edge_case_layers(p: int, seed: int = SEED) -> list[list[np.ndarray]]:
    """Edge-case suite: all-zero layer, 1-element layers,
    fp32 subnormals, an exact power-of-two max, a 1e+-30 range, all-equal-max
    adversarial inputs, ragged tails (not a multiple of 128 or 4)."""
    out = []
    for r in range(p):
        rng = np.random.default_rng([seed, 7777, r])
        layers = []
        layers.append(np.zeros(300, np.float32))                                   # all zero
        layers.append(np.array([rng.standard_normal()], np.float32))               # 1 element
        layers.append(np.array([0.0], np.float32) if r % 2 else np.array([-0.0], np.float32))
        sub = rng.integers(1, 2**23, 517).astype(np.uint32)
        sub |= rng.integers(0, 2, 517).astype(np.uint32) << np.uint32(31)
        layers.append(sub.view(np.float32))                                       # fp32 subnormals
        pw = rng.standard_normal(1000).astype(np.float32) * np.float32(0.25)
        pw[np.abs(pw) > 0.5] = 0.5
        pw[17] = 0.5 if r == 0 else -0.5                                           # max exactly 2^-1
        layers.append(pw)
        wide = (rng.standard_normal(4099) * 10.0 ** rng.uniform(-30, 30, 4099)).astype(np.float32)
        layers.append(wide)                                                        # 1e+-30
        layers.append(np.full(129, 3.0, np.float32))                               # all-equal max
        layers.append(np.full(131, -(2.0 ** -140), np.float32))                    # tiny, subnormal
        layers.append(rng.standard_normal(250).astype(np.float32) * np.float32(2.0 ** 100))
        out.append(layers)
    return out


def fp32_probe_patterns(n_random: int, seed: int = SEED) -> np.ndarray:
    """fp32 inputs for cast tests: random bit patterns plus every binade's
    edges (no NaN payload variety beyond a few)."""
    rng = np.random.default_rng([seed, 4242])
    bits = rng.integers(0, 2**32, n_random, dtype=np.uint64).astype(np.uint32)
    e = np.arange(256, dtype=np.uint32) << 23
    edges = np.concatenate([e, e + 1, e + 0x3FFFFF, e + 0x400000, e + 0x400001, e + 0x7FFFFF])
    edges = np.concatenate([edges, edges | np.uint32(0x80000000)])
    return np.concatenate([bits, edges]).view(np.float32)
