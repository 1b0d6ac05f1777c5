"""Model shapes of the BASELINE configs and seeded device-side random init.

The reference has no model at all — only per-model calibration constants
(perf.py:281-326: Llama2-70B and BLOOM-176B presets, layers 80/70 at
cluster.py:115-117, KV bytes/token from ``2*layers*hidden*2`` at
perf.py:289-290).  The shapes below are the public decoder configs the
BASELINE names; ``tiny`` is this build's own correctness
model (the reference pkg has no demo model).

Weight layout per tensor-parallel rank (all bf16, K-major = [out, in]):
  embed [V, d], lm_head [V, d], final_norm [d]
  per layer: attn_norm [d], wqkv [(Hq/tp + 2 Hkv/tp) * dh, d],
             wo [d, Hq/tp * dh], mlp_norm [d],
             wgu [2 * ffn/tp, d] (gate/up interleaved in 128-row groups so the
             GEMM epilogue sees gate and up of the same features in one tile),
             wd [d, ffn/tp].
BLOOM (arch "bloom": LayerNorm with bias, ALiBi instead of RoPE, biased
linears, GELU MLP, tied embeddings, embedding LayerNorm):
  lm_head is embed; emb_norm/emb_norm_b, final_norm/final_norm_b [d]
  per layer adds attn_norm_b, mlp_norm_b [d], bqkv [(3 H/tp) dh] (sharded),
  bo, bd [d] (replicated: added once, by TP rank 0), bup [ffn/tp]; wgu is the
  plain up projection [ffn/tp, d] (no gate).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from .errors import ConfigurationError


@dataclass(frozen=True)
class ModelConfig:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    arch: str = "llama"          # "llama" (RMSNorm, RoPE, SwiGLU) or "bloom"
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    init_std: float = 0.02
    max_token_batch: int = 64    # reference max_token_batch (perf.py:303, :324)

    def kv_bytes_per_token(self, tp: int = 1) -> int:
        """K+V bytes per token per TP rank, bf16 (GQA-aware version of the
        reference's 2*layers*hidden*2, perf.py:289-290)."""
        return 2 * self.n_layers * (self.n_kv_heads // tp) * self.head_dim * 2

    def reference_mha_kv_bytes_per_token(self) -> int:
        """The reference's sizing formula verbatim (perf.py:289-290)."""
        return 2 * self.n_layers * self.d_model * 2

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def is_bloom(self) -> bool:
        return self.arch == "bloom"

    def params_nonembed(self) -> int:
        d, dh = self.d_model, self.head_dim
        per = d * self.n_heads * dh + 2 * d * self.n_kv_heads * dh + self.n_heads * dh * d
        per += (2 if self.is_bloom else 3) * d * self.ffn   # up+down vs gate+up+down
        return self.n_layers * per

    def weight_bytes(self, tp: int = 1) -> int:
        tables = 1 if self.is_bloom else 2                  # tied embeddings (BLOOM)
        return 2 * (self.params_nonembed() // tp + tables * self.vocab * self.d_model)

    def prefill_flops(self, S: int, tp: int = 1) -> float:
        """Algorithmic prefill FLOPs per TP rank for one S-token prompt
        (SURVEY §8(d)): linears + causal QK^T/PV + last-token LM head."""
        lin = 2.0 * S * self.params_nonembed()
        attn = 2.0 * self.n_layers * S * S * self.n_heads * self.head_dim  # causal half of 4*
        head = 2.0 * self.d_model * self.vocab
        return (lin + attn) / tp + head

    def decode_bytes(self, contexts, tp: int = 1) -> int:
        """Algorithmic HBM bytes of one decode step per TP rank: weights once
        + the KV of every context."""
        # LM head split by vocabulary rows across a TP pool (runner.vocab_parallel)
        head = self.vocab * self.d_model // (tp if self.vocab % tp == 0 else 1)
        w = 2 * (self.params_nonembed() // tp + head)
        kv = sum(contexts) * self.kv_bytes_per_token(tp)
        return w + kv

    def validate_tp(self, tp: int) -> None:
        if self.n_heads % tp or self.n_kv_heads % tp:
            raise ConfigurationError(f"{self.name}: heads not divisible by tp={tp}")
        if (self.ffn // tp) % 128 or self.ffn % tp:
            raise ConfigurationError(f"{self.name}: ffn/tp must be a multiple of 128")
        if self.head_dim != 128:
            raise ConfigurationError("kernels are specialised for head_dim 128")
        if self.arch not in ("llama", "bloom"):
            raise ConfigurationError(f"unknown arch {self.arch!r}")


PRESETS: dict[str, ModelConfig] = {
    # builder-defined correctness model (C1); GQA 4:2 to exercise grouping
    "tiny": ModelConfig("tiny", n_layers=4, d_model=512, n_heads=4, n_kv_heads=2,
                        head_dim=128, ffn=1536, vocab=2048),
    "llama2-7b": ModelConfig("llama2-7b", 32, 4096, 32, 32, 128, 11008, 32000),
    "llama2-70b": ModelConfig("llama2-70b", 80, 8192, 64, 8, 128, 28672, 32000),
    # MHA switch reproducing the reference's KV sizing (perf.py:289-290)
    "llama2-70b-mha": ModelConfig("llama2-70b-mha", 80, 8192, 64, 64, 128, 28672, 32000),
    "bloom-176b": ModelConfig("bloom-176b", 70, 14336, 112, 112, 128, 57344, 250880,
                              arch="bloom", max_token_batch=26),
    # builder-defined BLOOM-architecture correctness model (C5's kernels);
    # 6 heads exercise the non-power-of-two ALiBi slope rule like BLOOM's 112
    "bloom-tiny": ModelConfig("bloom-tiny", n_layers=3, d_model=768, n_heads=6, n_kv_heads=6,
                              head_dim=128, ffn=3072, vocab=2048, arch="bloom"),
    # TP=4-divisible variants for the 4-GPU pool checks (tools/tp_check.py)
    "tiny-tp4": ModelConfig("tiny-tp4", n_layers=4, d_model=1024, n_heads=8, n_kv_heads=4,
                            head_dim=128, ffn=2048, vocab=2048),
    "bloom-tiny-tp4": ModelConfig("bloom-tiny-tp4", n_layers=3, d_model=1024, n_heads=8,
                                  n_kv_heads=8, head_dim=128, ffn=4096, vocab=2048,
                                  arch="bloom"),
}


def alibi_slopes(n_heads: int) -> list[float]:
    """ALiBi head slopes as BLOOM defines them: a geometric sequence for the
    largest power of two <= n heads, then the odd powers of the next finer
    base for the remainder."""
    p2 = 2 ** math.floor(math.log2(n_heads))
    base = 2.0 ** (-(2.0 ** -(math.log2(p2) - 3)))
    slopes = [base ** i for i in range(1, p2 + 1)]
    if p2 != n_heads:
        extra = 2.0 ** (-(2.0 ** -(math.log2(2 * p2) - 3)))
        rem = min(p2, n_heads - p2)
        slopes += [extra ** i for i in range(1, 2 * rem, 2)]
    return slopes


def get_config(name: str) -> ModelConfig:
    if name not in PRESETS:
        raise ConfigurationError(f"unknown model {name!r}; have {sorted(PRESETS)}")
    return PRESETS[name]


def interleave_gate_up(gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
    """[f, d] x 2 -> [2f, d] in 128-row groups (g0..g127, u0..u127, g128..)."""
    f, d = gate.shape
    return torch.stack([gate.view(f // 128, 128, d), up.view(f // 128, 128, d)], 1).reshape(2 * f, d)


def split_gate_up(wgu: torch.Tensor):
    f2, d = wgu.shape
    v = wgu.view(f2 // 256, 2, 128, d)
    return v[:, 0].reshape(f2 // 2, d), v[:, 1].reshape(f2 // 2, d)


@dataclass
class LayerWeights:
    attn_norm: torch.Tensor
    wqkv: torch.Tensor
    wo: torch.Tensor
    mlp_norm: torch.Tensor
    wgu: torch.Tensor
    wd: torch.Tensor
    # BLOOM only
    attn_norm_b: torch.Tensor | None = None
    mlp_norm_b: torch.Tensor | None = None
    bqkv: torch.Tensor | None = None
    bo: torch.Tensor | None = None
    bup: torch.Tensor | None = None
    bd: torch.Tensor | None = None


@dataclass
class Weights:
    cfg: ModelConfig
    tp: int
    rank: int
    embed: torch.Tensor
    lm_head: torch.Tensor
    final_norm: torch.Tensor
    layers: list[LayerWeights] = field(default_factory=list)
    # BLOOM only
    final_norm_b: torch.Tensor | None = None
    emb_norm: torch.Tensor | None = None
    emb_norm_b: torch.Tensor | None = None
    alibi: torch.Tensor | None = None      # fp32 slopes of this rank's heads

    def nbytes(self) -> int:
        seen, n = set(), 0
        tensors = [self.embed, self.lm_head, self.final_norm]
        for lw in self.layers:
            tensors += [lw.attn_norm, lw.wqkv, lw.wo, lw.mlp_norm, lw.wgu, lw.wd]
        for t in tensors:
            if t.data_ptr() not in seen:      # tied embeddings count once
                seen.add(t.data_ptr())
                n += t.numel()
        return 2 * n


def _randn(gen, shape, std, device):
    t = torch.empty(shape, dtype=torch.bfloat16, device=device)
    t.normal_(0.0, std, generator=gen)
    return t


def init_weights(cfg: ModelConfig, seed: int = 0, tp: int = 1, rank: int = 0,
                 device: str | torch.device = "cuda") -> Weights:
    """Seeded random init directly on the device, one shard per TP rank.

    Every tensor draws from its own generator seeded by (seed, layer, tensor,
    rank), so a shard is reproducible in isolation and the logical model is
    the concatenation of the shards along the split dimension.  Replicated
    tensors (embeddings, norms) use rank 0's stream on every rank.
    """
    cfg.validate_tp(tp)
    dev = torch.device(device)
    gen = torch.Generator(device=dev)

    def g(layer, tag, shard):
        gen.manual_seed((seed * 1_000_003 + (layer + 1) * 7919 + tag * 131 + shard) & 0x7FFFFFFF)
        return gen

    std = cfg.init_std
    d, dh = cfg.d_model, cfg.head_dim
    hq, hkv, f = cfg.n_heads // tp, cfg.n_kv_heads // tp, cfg.ffn // tp

    def norm_w(layer, tag):
        return (1.0 + _randn(g(layer, tag, 0), (d,), std, dev).float()).bfloat16()

    embed = _randn(g(-1, 1, 0), (cfg.vocab, d), 1.0, dev)
    if cfg.is_bloom:
        lm_head = embed                                   # tied
        bloom = dict(final_norm_b=_randn(g(-1, 4, 0), (d,), std, dev),
                     emb_norm=norm_w(-1, 5), emb_norm_b=_randn(g(-1, 6, 0), (d,), std, dev),
                     alibi=torch.tensor(alibi_slopes(cfg.n_heads)[rank * hq:(rank + 1) * hq],
                                        dtype=torch.float32, device=dev))
    else:
        lm_head = _randn(g(-1, 2, 0), (cfg.vocab, d), std, dev)
        bloom = {}
    final_norm = norm_w(-1, 3)
    layers = []
    for layer in range(cfg.n_layers):
        lw = LayerWeights(
            attn_norm=norm_w(layer, 10),
            wqkv=_randn(g(layer, 11, rank), ((hq + 2 * hkv) * dh, d), std, dev),
            wo=_randn(g(layer, 12, rank), (d, hq * dh), std, dev),
            mlp_norm=norm_w(layer, 13),
            wgu=_randn(g(layer, 14, rank), ((1 if cfg.is_bloom else 2) * f, d), std, dev),
            wd=_randn(g(layer, 15, rank), (d, f), std, dev),
        )
        if cfg.is_bloom:
            lw.attn_norm_b = _randn(g(layer, 20, 0), (d,), std, dev)
            lw.mlp_norm_b = _randn(g(layer, 21, 0), (d,), std, dev)
            lw.bqkv = _randn(g(layer, 22, rank), ((hq + 2 * hkv) * dh,), std, dev)
            lw.bo = _randn(g(layer, 23, 0), (d,), std, dev)
            lw.bup = _randn(g(layer, 24, rank), (f,), std, dev)
            lw.bd = _randn(g(layer, 25, 0), (d,), std, dev)
        layers.append(lw)
    return Weights(cfg, tp, rank, embed, lm_head, final_norm, layers, **bloom)


def logical_layer_fp32(w: Weights, layer: int) -> dict:
    """Per-rank layer weights unpacked into logical fp32 CPU tensors for the
    oracle (q/k/v split, gate/up de-interleaved)."""
    cfg = w.cfg
    lw = w.layers[layer]
    hq, hkv, dh = cfg.n_heads // w.tp, cfg.n_kv_heads // w.tp, cfg.head_dim
    qkv = lw.wqkv.float().cpu()
    if cfg.is_bloom:
        f32 = lambda t: t.float().cpu()  # noqa: E731
        b = f32(lw.bqkv)
        return {
            "ln1_w": f32(lw.attn_norm), "ln1_b": f32(lw.attn_norm_b),
            "wq": qkv[:hq * dh], "wk": qkv[hq * dh:(hq + hkv) * dh], "wv": qkv[(hq + hkv) * dh:],
            "bq": b[:hq * dh], "bk": b[hq * dh:(hq + hkv) * dh], "bv": b[(hq + hkv) * dh:],
            "wo": f32(lw.wo), "bo": f32(lw.bo),
            "ln2_w": f32(lw.mlp_norm), "ln2_b": f32(lw.mlp_norm_b),
            "w_up": f32(lw.wgu), "b_up": f32(lw.bup), "wd": f32(lw.wd), "bd": f32(lw.bd),
        }
    gate, up = split_gate_up(lw.wgu.float().cpu())
    return {
        "attn_norm": lw.attn_norm.float().cpu(),
        "wq": qkv[:hq * dh], "wk": qkv[hq * dh:(hq + hkv) * dh], "wv": qkv[(hq + hkv) * dh:],
        "wo": lw.wo.float().cpu(), "mlp_norm": lw.mlp_norm.float().cpu(),
        "w_gate": gate, "w_up": up, "wd": lw.wd.float().cpu(),
    }
