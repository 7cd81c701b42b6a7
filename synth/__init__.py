"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no diff, codec or packing). It
defines a counter-based generator (SplitMix64 finaliser) that is implemented
twice — here in numpy for the oracle/tests and in ``synth/gen.cu`` for the GPU —
plus the Qwen3 tensor manifests (public HF configs).

Recipe:
  h(stream, seed, t, i) = mix(mix(seed*256 + stream) ^ (t << 34) ^ i)
  old  = TABLE[h(VAL) >> 48]   (TABLE: 65536 bf16 RNE quantiles of N(0, 0.02))
         0x3F80 (1.0) for RMSNorm vectors
  mask U: (h(MASK) >> 32) < floor(rho * 2^32)
       R: row active iff (h(ROW, t, row) >> 32) < floor(q * 2^32), then rho/q inside
       E: expert (layer, e) active iff (h(EXP, layer, e) >> 32) < floor(f * 2^32), then rho/f inside
  new  = old ^ (1 + h(PERT) % 3) where mask
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

M64 = (1 << 64) - 1
S_VAL, S_MASK, S_PERT, S_ROW, S_EXP = 1, 2, 3, 4, 5
KIND_MATRIX, KIND_NORM = 0, 1
MASK_U, MASK_R, MASK_E = 0, 1, 2
ROW_Q = 0.10
EXPERT_F = 0.25
SIGMA = 0.02


def mix_int(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def mix_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z += np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def key(stream: int, seed: int, t: int) -> int:
    return mix_int((seed * 256 + stream) & M64) ^ ((t << 34) & M64)


def h(stream: int, seed: int, t: int, i: np.ndarray) -> np.ndarray:
    return mix_np(np.uint64(key(stream, seed, t)) ^ i.astype(np.uint64))


def threshold(p: float) -> int:
    """floor(p * 2^32) clamped to [0, 2^32]."""
    return max(0, min(1 << 32, int(math.floor(p * 4294967296.0))))


_TABLE = None


DTYPE_BF16, DTYPE_FP16, DTYPE_FP8 = 1, 2, 3
ONE = {DTYPE_BF16: 0x3F80, DTYPE_FP16: 0x3C00, DTYPE_FP8: 0x38}   # bit patterns of 1.0 (RMSNorm weights)
_TABLE16 = None
_TABLE8 = None


def fp8_table() -> np.ndarray:
    """65536 FP8 E4M3 bytes: torch's float8_e4m3fn cast (round to nearest even, saturating) of
    SIGMA * Phi^-1((k + 0.5) / 65536) — the same quantiles as the 16-bit tables, at 8-bit precision."""
    global _TABLE8
    if _TABLE8 is None:
        import torch
        from scipy.special import ndtri
        q = (np.arange(65536, dtype=np.float64) + 0.5) / 65536.0
        f32 = torch.from_numpy((SIGMA * ndtri(q)).astype(np.float32))
        _TABLE8 = f32.to(torch.float8_e4m3fn).view(torch.uint8).numpy().copy()
    return _TABLE8


def fp16_table() -> np.ndarray:
    """65536 fp16 bit patterns: RNE (numpy's float16 cast) of SIGMA * Phi^-1((k + 0.5) / 65536)."""
    global _TABLE16
    if _TABLE16 is None:
        from scipy.special import ndtri
        q = (np.arange(65536, dtype=np.float64) + 0.5) / 65536.0
        _TABLE16 = (SIGMA * ndtri(q)).astype(np.float32).astype(np.float16).view(np.uint16)
    return _TABLE16


def table(dtype: int = DTYPE_BF16) -> np.ndarray:
    if dtype == DTYPE_FP8:
        return fp8_table()
    return fp16_table() if dtype == DTYPE_FP16 else bf16_table()


def bf16_table() -> np.ndarray:
    """65536 bf16 bit patterns: RNE of SIGMA * Phi^-1((k + 0.5) / 65536), ascending k."""
    global _TABLE
    if _TABLE is None:
        from scipy.special import ndtri
        q = (np.arange(65536, dtype=np.float64) + 0.5) / 65536.0
        f32 = (SIGMA * ndtri(q)).astype(np.float32)
        u = f32.view(np.uint32).astype(np.uint64)
        # round-to-nearest-even to bf16 (finite inputs only)
        rnd = ((u >> np.uint64(16)) & np.uint64(1)) + np.uint64(0x7FFF)
        _TABLE = ((u + rnd) >> np.uint64(16)).astype(np.uint16)
    return _TABLE


@dataclass
class Tensor:
    name: str
    shape: tuple
    kind: int = KIND_MATRIX
    layer: int = -1
    expert: int = -1

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape)) if self.shape else 1

    @property
    def rows(self) -> int:
        return self.shape[0] if len(self.shape) == 2 else 1

    @property
    def cols(self) -> int:
        return self.shape[1] if len(self.shape) == 2 else self.numel


@dataclass
class Manifest:
    name: str
    tensors: list = field(default_factory=list)

    @property
    def numel(self) -> list:
        return [t.numel for t in self.tensors]

    @property
    def total(self) -> int:
        return sum(self.numel)

    def slice(self, lo: int, hi: int, name: str | None = None) -> "Manifest":
        return Manifest(name or f"{self.name}[{lo}:{hi}]", self.tensors[lo:hi])


def qwen3_manifest(name: str) -> Manifest:
    """Qwen3 tensor list in HF iteration order."""
    cfgs = {
        "qwen3-4b": dict(hid=2560, layers=36, heads=32, kv=8, hd=128, inter=9728, experts=0, moe=0,
                         vocab=151936, tied=True),
        "qwen3-30b-a3b": dict(hid=2048, layers=48, heads=32, kv=4, hd=128, inter=0, experts=128, moe=768,
                              vocab=151936, tied=False),
        "qwen3-235b-a22b": dict(hid=4096, layers=94, heads=64, kv=4, hd=128, inter=0, experts=128, moe=1536,
                                vocab=151936, tied=False),
    }
    c = cfgs[name]
    hid, hd = c["hid"], c["hd"]
    T = [Tensor("model.embed_tokens.weight", (c["vocab"], hid))]
    for l in range(c["layers"]):
        p = f"model.layers.{l}."
        T += [Tensor(p + "self_attn.q_proj.weight", (c["heads"] * hd, hid), layer=l),
              Tensor(p + "self_attn.k_proj.weight", (c["kv"] * hd, hid), layer=l),
              Tensor(p + "self_attn.v_proj.weight", (c["kv"] * hd, hid), layer=l),
              Tensor(p + "self_attn.o_proj.weight", (hid, c["heads"] * hd), layer=l),
              Tensor(p + "self_attn.q_norm.weight", (hd,), KIND_NORM, layer=l),
              Tensor(p + "self_attn.k_norm.weight", (hd,), KIND_NORM, layer=l)]
        if c["experts"]:
            T.append(Tensor(p + "mlp.gate.weight", (c["experts"], hid), layer=l))
            for e in range(c["experts"]):
                q = f"{p}mlp.experts.{e}."
                T += [Tensor(q + "gate_proj.weight", (c["moe"], hid), layer=l, expert=e),
                      Tensor(q + "up_proj.weight", (c["moe"], hid), layer=l, expert=e),
                      Tensor(q + "down_proj.weight", (hid, c["moe"]), layer=l, expert=e)]
        else:
            T += [Tensor(p + "mlp.gate_proj.weight", (c["inter"], hid), layer=l),
                  Tensor(p + "mlp.up_proj.weight", (c["inter"], hid), layer=l),
                  Tensor(p + "mlp.down_proj.weight", (hid, c["inter"]), layer=l)]
        T += [Tensor(p + "input_layernorm.weight", (hid,), KIND_NORM, layer=l),
              Tensor(p + "post_attention_layernorm.weight", (hid,), KIND_NORM, layer=l)]
    T.append(Tensor("model.norm.weight", (hid,), KIND_NORM))
    if not c["tied"]:
        T.append(Tensor("lm_head.weight", (c["vocab"], hid)))
    return Manifest(name, T)


def single_manifest(n: int, name: str = "single") -> Manifest:
    return Manifest(name, [Tensor("w", (n,))])


def shard(manifest: Manifest, rank: int, world: int) -> Manifest:
    """Contiguous, element-balanced tensor range for rank."""
    tot = manifest.total
    cum, lo, hi = 0, None, None
    for k, t in enumerate(manifest.tensors):
        owner = min(world - 1, (cum + t.numel // 2) * world // max(tot, 1))
        if owner == rank:
            lo = k if lo is None else lo
            hi = k + 1
        cum += t.numel
    if lo is None:
        return Manifest(f"{manifest.name}/r{rank}of{world}", [])
    return manifest.slice(lo, hi, f"{manifest.name}/r{rank}of{world}")


# ----------------------------------------------------------------------------- generation
def gen_old(t: Tensor, tid: int, seed: int, dtype: int = DTYPE_BF16) -> np.ndarray:
    if t.kind == KIND_NORM:
        return np.full(t.numel, ONE[dtype], np.uint8 if dtype == DTYPE_FP8 else np.uint16)
    i = np.arange(t.numel, dtype=np.uint64)
    return table(dtype)[(h(S_VAL, seed, tid, i) >> np.uint64(48)).astype(np.int64)]


def gen_mask(t: Tensor, tid: int, seed: int, rho: float, mask: int = MASK_U) -> np.ndarray:
    n = t.numel
    i = np.arange(n, dtype=np.uint64)
    hm = h(S_MASK, seed, tid, i) >> np.uint64(32)
    if mask == MASK_R and len(t.shape) == 2:
        rows = np.arange(t.rows, dtype=np.uint64)
        ract = (h(S_ROW, seed, tid, rows) >> np.uint64(32)) < np.uint64(threshold(ROW_Q))
        inside = hm < np.uint64(threshold(min(1.0, rho / ROW_Q)))
        return inside & np.repeat(ract, t.cols)
    if mask == MASK_E and t.expert >= 0:
        e = np.array([t.expert], np.uint64)
        act = bool((h(S_EXP, seed, t.layer, e) >> np.uint64(32))[0] < np.uint64(threshold(EXPERT_F)))
        if not act:
            return np.zeros(n, bool)
        return hm < np.uint64(threshold(min(1.0, rho / EXPERT_F)))
    return hm < np.uint64(threshold(rho))


def gen_new(old: np.ndarray, t: Tensor, tid: int, seed: int, rho: float, mask: int = MASK_U) -> np.ndarray:
    m = gen_mask(t, tid, seed, rho, mask)
    i = np.arange(t.numel, dtype=np.uint64)
    d = (np.uint64(1) + h(S_PERT, seed, tid, i) % np.uint64(3)).astype(old.dtype)
    return np.where(m, old ^ d, old).astype(old.dtype)


def generate(manifest: Manifest, seed: int = 0, rho: float = 0.01, mask: int = MASK_U, tid0: int = 0,
             dtype: int = DTYPE_BF16):
    """Lists (olds, news) of uint16 arrays; tensor ids start at tid0 (global manifest ids)."""
    olds, news = [], []
    for k, t in enumerate(manifest.tensors):
        o = gen_old(t, tid0 + k, seed, dtype)
        olds.append(o)
        news.append(gen_new(o, t, tid0 + k, seed, rho, mask))
    return olds, news
