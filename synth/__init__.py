"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no smoothing, no quantization, no
products): it only draws random numbers and encodes them as bf16 bit patterns,
so that both sides of every parity test consume byte-identical inputs.

Recipe:
  * activations  x[t,i] = gamma_{m(t)} * c^{m(t)}_i * z[t,i], then bf16 RNE
      z ~ N(0,1); c^m_i = exp(N(0,1)) drawn independently per modality
      (per-channel dominance varies); 1% of channels (shared
      across modalities) boosted x10;
      gamma: text 1, image 20, audio 0.3 (20x gap PAPER.md:7, 10-100x
      PAPER.md:189, audio "smaller activation magnitudes" PAPER.md:405).
  * weights      W ~ N(0,1)/sqrt(d), bf16 RNE, layout [d x n]
      (the paper's W in R^{D_in x D_out}).
  * low-rank CMC factors L1^m [d x r], L2^m [r x n]:
      random Gaussian of the magnitude the correction has in practice (the
      correction carries most of the non-text output).
  * modality layout: contiguous spans per 1024-token sample (VQA-like),
      or an i.i.d.-shuffled variant for routing stress.
  * seed = 260304800 + 1000*config + 10*layer + input_index (numpy PCG64).
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 260304800
GAMMA = {0: 1.0, 1: 20.0, 2: 0.3}  # text, image, audio

# BASELINE.json configs; shapes per SURVEY.md §8(d) (public HF configs for the
# Qwen2.5 models, which the paper only names).
CONFIGS = {
    "c1": dict(T=256, d=64, n=128, n_mod=2, wbits=8, abits=8, r=16,
               pattern=[(0, 40), (1, 160), (0, 56)], repeat=1),
    "c2": dict(T=4096, d=2048, n=11008, n_mod=3, wbits=8, abits=8, r=0,
               pattern=[(0, 64), (1, 512), (2, 320), (0, 128)], repeat=4),
    "c3": dict(T=16384, d=3584, n=18944, n_mod=2, wbits=4, abits=8, r=64,
               pattern=[(0, 64), (1, 768), (0, 192)], repeat=16),
}
# Linear shapes of one decoder layer (fused qkv and gate+up).
LAYER_LINEARS = {
    "c2": [("qkv", 2048, 2560), ("o", 2048, 2048), ("gate_up", 2048, 22016), ("down", 11008, 2048)],
    "c3": [("qkv", 3584, 4608), ("o", 3584, 3584), ("gate_up", 3584, 37888), ("down", 18944, 3584)],
}


def seed_for(config_index: int, layer: int = 0, input_index: int = 0) -> int:
    return SEED_BASE + 1000 * config_index + 10 * layer + input_index


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even f32 -> bf16 bit pattern (finite inputs)."""
    # uint32 arithmetic cannot overflow for finite inputs (|bits| <= 0xFF7FFFFF, + <= 0x8000)
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    out = (b >> 16) & 1
    out += 0x7FFF
    out += b
    out >>= 16
    return out.astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def modality_ids(pattern, repeat: int = 1, T: int | None = None, shuffle_seed: int | None = None) -> np.ndarray:
    one = np.concatenate([np.full(cnt, m, dtype=np.uint8) for m, cnt in pattern])
    ids = np.tile(one, repeat)
    if T is not None:
        if T <= ids.size:
            ids = ids[:T]
        else:
            ids = np.tile(one, -(-T // one.size))[:T]
    if shuffle_seed is not None:
        rng = np.random.Generator(np.random.PCG64(shuffle_seed))
        ids = ids[rng.permutation(ids.size)]
    return np.ascontiguousarray(ids)


def activations(ids: np.ndarray, d: int, n_mod: int, seed: int, gamma=None,
                outlier_frac: float = 0.01, as_bf16: bool = True):
    """X [T x d]; returns bf16 bits (uint16) if as_bf16 else float32 values."""
    gamma = GAMMA if gamma is None else gamma
    rng = np.random.Generator(np.random.PCG64(seed))
    chan = np.exp(rng.standard_normal((n_mod, d))).astype(np.float32)
    n_out = max(1, int(round(outlier_frac * d)))
    out_idx = rng.choice(d, size=n_out, replace=False)
    chan[:, out_idx] *= 10.0
    g = np.array([gamma.get(m, 1.0) for m in range(n_mod)], dtype=np.float32)
    scale = g[:, None] * chan                                   # [M x d] f32
    x = rng.standard_normal((ids.size, d), dtype=np.float32)    # z
    idx = ids.astype(np.int64)
    for m in range(n_mod):                                      # x = scale[m(t)] * z, in place
        rows = np.nonzero(idx == m)[0]
        if rows.size:
            x[rows] *= scale[m]
    return f32_to_bf16_bits(x) if as_bf16 else x


def weight(d: int, n: int, seed: int) -> np.ndarray:
    """W [d x n] bf16 bits, N(0,1)/sqrt(d)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    w = rng.standard_normal((d, n), dtype=np.float32) * np.float32(1.0 / np.sqrt(d))
    return f32_to_bf16_bits(w)


def lowrank(d: int, n: int, r: int, n_mod: int, seed: int, gain: float = 4.0):
    """L1 [n_mod-1][d][r], L2 [n_mod-1][r][n] as bf16 bits.

    Magnitudes: L1 ~ N(0, 1/d)*sqrt(d/r)... chosen so that xs.L1.L2 has the size of
    gain * (xs . W) for unit-variance xs (the correction dominates non-text outputs).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    k = max(n_mod - 1, 0)
    l1 = rng.standard_normal((k, d, r), dtype=np.float32) * np.float32(1.0 / np.sqrt(d))
    l2 = rng.standard_normal((k, r, n), dtype=np.float32) * np.float32(gain / np.sqrt(r))
    return f32_to_bf16_bits(l1), f32_to_bf16_bits(l2)


def config_inputs(name: str, d: int | None = None, n: int | None = None, T: int | None = None,
                  layer: int = 0, shuffle: bool = False, r: int | None = None):
    """All inputs of one BASELINE config: dict with ids, X bits, W bits, L1/L2 bits."""
    cfg = dict(CONFIGS[name])
    ci = int(name[1:]) - 1
    d = cfg["d"] if d is None else d
    n = cfg["n"] if n is None else n
    r = cfg["r"] if r is None else r
    ids = modality_ids(cfg["pattern"], cfg["repeat"], T=T if T is not None else cfg["T"],
                       shuffle_seed=seed_for(ci, layer, 9) if shuffle else None)
    X = activations(ids, d, cfg["n_mod"], seed_for(ci, layer, 0))
    W = weight(d, n, seed_for(ci, layer, 1))
    L1, L2 = lowrank(d, n, r, cfg["n_mod"], seed_for(ci, layer, 2)) if r > 0 else (None, None)
    return dict(ids=ids, X=X, W=W, L1=L1, L2=L2, d=d, n=n, r=r, T=ids.size,
                n_mod=cfg["n_mod"], wbits=cfg["wbits"], abits=cfg["abits"])
