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
"""

from __future__ import annotations

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

    def params_nonembed(self) -> int:
        d, dh = self.d_model, self.head_dim
        per = d * self.n_heads * dh + 2 * d * self.n_kv_heads * dh + self.n_heads * dh * d
        per += 3 * d * self.ffn
        return self.n_layers * per

    def weight_bytes(self, tp: int = 1) -> int:
        return 2 * (self.params_nonembed() // tp + 2 * self.vocab * self.d_model)

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
        w = 2 * (self.params_nonembed() // tp + self.vocab * self.d_model)
        kv = sum(contexts) * self.kv_bytes_per_token(tp)
        return w + kv

    def validate_tp(self, tp: int) -> None:
        if self.n_heads % tp or self.n_kv_heads % tp:
            raise ConfigurationError(f"{self.name}: heads not divisible by tp={tp}")
        if (self.ffn // tp) % 128 or self.ffn % tp:
            raise ConfigurationError(f"{self.name}: ffn/tp must be a multiple of 128")
        if self.head_dim != 128:
            raise ConfigurationError("kernels are specialised for head_dim 128")
        if self.arch != "llama":
            raise ConfigurationError(f"arch {self.arch!r} kernels not built in this round")


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
}


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


@dataclass
class Weights:
    cfg: ModelConfig
    tp: int
    rank: int
    embed: torch.Tensor
    lm_head: torch.Tensor
    final_norm: torch.Tensor
    layers: list[LayerWeights] = field(default_factory=list)

    def nbytes(self) -> int:
        n = self.embed.numel() + self.lm_head.numel() + self.final_norm.numel()
        for lw in self.layers:
            n += sum(t.numel() for t in (lw.attn_norm, lw.wqkv, lw.wo, lw.mlp_norm, lw.wgu, lw.wd))
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
    embed = _randn(g(-1, 1, 0), (cfg.vocab, d), 1.0, dev)
    lm_head = _randn(g(-1, 2, 0), (cfg.vocab, d), std, dev)
    final_norm = (1.0 + _randn(g(-1, 3, 0), (d,), std, dev).float()).bfloat16()
    layers = []
    for layer in range(cfg.n_layers):
        layers.append(LayerWeights(
            attn_norm=(1.0 + _randn(g(layer, 10, 0), (d,), std, dev).float()).bfloat16(),
            wqkv=_randn(g(layer, 11, rank), ((hq + 2 * hkv) * dh, d), std, dev),
            wo=_randn(g(layer, 12, rank), (d, hq * dh), std, dev),
            mlp_norm=(1.0 + _randn(g(layer, 13, 0), (d,), std, dev).float()).bfloat16(),
            wgu=_randn(g(layer, 14, rank), (2 * f, d), std, dev),
            wd=_randn(g(layer, 15, rank), (d, f), std, dev),
        ))
    return Weights(cfg, tp, rank, embed, lm_head, final_norm, layers)


def logical_layer_fp32(w: Weights, layer: int) -> dict:
    """Per-rank layer weights unpacked into logical fp32 CPU tensors for the
    oracle (q/k/v split, gate/up de-interleaved)."""
    cfg = w.cfg
    lw = w.layers[layer]
    hq, hkv, dh = cfg.n_heads // w.tp, cfg.n_kv_heads // w.tp, cfg.head_dim
    qkv = lw.wqkv.float().cpu()
    gate, up = split_gate_up(lw.wgu.float().cpu())
    return {
        "attn_norm": lw.attn_norm.float().cpu(),
        "wq": qkv[:hq * dh], "wk": qkv[hq * dh:(hq + hkv) * dh], "wv": qkv[(hq + hkv) * dh:],
        "wo": lw.wo.float().cpu(), "mlp_norm": lw.mlp_norm.float().cpu(),
        "w_gate": gate, "w_up": up, "wd": lw.wd.float().cpu(),
    }
