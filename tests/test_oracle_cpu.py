"""The fp32 CPU oracle itself (test infrastructure): paged decoding through
block tables equals contiguous decoding bit-for-bit, the CPU allocator is
lowest-free-first, RoPE is a rotation (norm-preserving, relative-position
invariant), and the greedy loop has the reference's phase structure (first
token from the prompt phase, out-1 from decode iterations)."""

import math

import torch

from oracle.decoder import LowestFreeAllocator, OracleDecoder, PagedKV, apply_rope, rope_tables


def _tiny_oracle(seed=0, layers=2, d=256, H=4, Hkv=2, dh=128, f=512, V=300):
    from paper_2311_18677_b200.model import ModelConfig
    cfg = ModelConfig("t", layers, d, H, Hkv, dh, f, V)
    g = torch.Generator().manual_seed(seed)

    def r(*s):
        return torch.randn(*s, generator=g) * 0.05
    lay = [{"attn_norm": 1 + r(d), "wq": r(H * dh, d), "wk": r(Hkv * dh, d),
            "wv": r(Hkv * dh, d), "wo": r(d, H * dh), "mlp_norm": 1 + r(d),
            "w_gate": r(f, d), "w_up": r(f, d), "wd": r(d, f)} for _ in range(layers)]
    return OracleDecoder(cfg, lay, torch.randn(V, d, generator=g), r(V, d), 1 + r(d))


def test_paged_equals_contiguous():
    orc = _tiny_oracle()
    prompt = list(range(5, 45))
    toks_c, log_c = orc.generate(prompt, 10)
    store = PagedKV(orc.cfg.n_layers, 32, orc.cfg.n_kv_heads, 16, orc.cfg.head_dim)
    store.reserve(7, 3)        # non-trivial table for seq 0
    store.reserve(0, len(prompt) + 10)
    toks_p, log_p = orc.paged_generate(prompt, 10, store, 0)
    assert toks_c == toks_p
    assert torch.equal(log_c, log_p)
    assert store.tables[0][0] == 1   # block 0 taken by seq 7


def test_lowest_free_first_allocator():
    a = LowestFreeAllocator(20)
    x = a.alloc(5)
    y = a.alloc(3)
    assert x == [0, 1, 2, 3, 4] and y == [5, 6, 7]
    a.free([1, 3])
    assert a.alloc(3) == [1, 3, 8]
    assert a.free_count == 20 - 9


def test_rope_is_rotation():
    x = torch.randn(6, 2, 128)
    cos, sin = rope_tables(torch.arange(100, 106), 128, 10000.0)
    y = apply_rope(x, cos, sin)
    assert torch.allclose(x.norm(dim=-1), y.norm(dim=-1), atol=1e-4)
    # <rope(q, m), rope(k, n)> depends only on m - n
    q, k = torch.randn(1, 1, 128), torch.randn(1, 1, 128)

    def dot(m, n):
        cm, sm = rope_tables(torch.tensor([m]), 128, 1e4)
        cn, sn = rope_tables(torch.tensor([n]), 128, 1e4)
        return (apply_rope(q, cm, sm) * apply_rope(k, cn, sn)).sum().item()
    assert math.isclose(dot(10, 3), dot(107, 100), rel_tol=1e-4)


def test_generate_phase_structure():
    orc = _tiny_oracle(seed=3)
    toks, logits = orc.generate([1, 2, 3, 4], 1)
    assert len(toks) == 1 and logits.shape[0] == 1      # out=1: no token phase
    toks, logits = orc.generate([1, 2, 3, 4], 6)
    assert len(toks) == 6 and logits.shape == (6, orc.cfg.vocab)
    # teacher forcing with the model's own tokens reproduces the free run
    toks2, logits2 = orc.generate([1, 2, 3, 4], 6, forced=toks[:-1])
    assert toks2 == toks and torch.equal(logits, logits2)


def _bloom_weights_cpu():
    from paper_2311_18677_b200.model import ModelConfig, init_weights
    # BLOOM shapes: d = H * dh, ffn = 4 d
    cfg = ModelConfig("bloom-t", 2, 768, 6, 6, 128, 3072, 300, arch="bloom", init_std=0.05)
    return cfg, init_weights(cfg, seed=3, device="cpu")


def test_bloom_oracle_matches_transformers_bloom():
    """The BLOOM restatement (LayerNorms, ALiBi, biases, tanh-GELU, tied
    head) equals transformers' BloomForCausalLM on the same weights."""
    from transformers import BloomConfig, BloomForCausalLM
    from paper_2311_18677_b200.model import logical_layer_fp32
    cfg, w = _bloom_weights_cpu()
    orc = OracleDecoder.from_weights(w)
    hf = BloomForCausalLM(BloomConfig(vocab_size=cfg.vocab, hidden_size=cfg.d_model,
                                      n_layer=cfg.n_layers, n_head=cfg.n_heads,
                                      layer_norm_epsilon=cfg.norm_eps, hidden_dropout=0.0,
                                      attention_dropout=0.0)).eval()
    H, dh = cfg.n_heads, cfg.head_dim
    sd = {"transformer.word_embeddings.weight": w.embed.float(),
          "transformer.word_embeddings_layernorm.weight": w.emb_norm.float(),
          "transformer.word_embeddings_layernorm.bias": w.emb_norm_b.float(),
          "transformer.ln_f.weight": w.final_norm.float(),
          "transformer.ln_f.bias": w.final_norm_b.float(),
          "lm_head.weight": w.embed.float()}
    for i in range(cfg.n_layers):
        L = logical_layer_fp32(w, i)
        p = f"transformer.h.{i}."
        # BLOOM's fused qkv is head-major [H][q|k|v][dh]
        wqkv = torch.stack([L["wq"].view(H, dh, -1), L["wk"].view(H, dh, -1),
                            L["wv"].view(H, dh, -1)], 1).reshape(3 * H * dh, -1)
        bqkv = torch.stack([L["bq"].view(H, dh), L["bk"].view(H, dh), L["bv"].view(H, dh)],
                           1).reshape(-1)
        sd.update({p + "input_layernorm.weight": L["ln1_w"], p + "input_layernorm.bias": L["ln1_b"],
                   p + "self_attention.query_key_value.weight": wqkv,
                   p + "self_attention.query_key_value.bias": bqkv,
                   p + "self_attention.dense.weight": L["wo"],
                   p + "self_attention.dense.bias": L["bo"],
                   p + "post_attention_layernorm.weight": L["ln2_w"],
                   p + "post_attention_layernorm.bias": L["ln2_b"],
                   p + "mlp.dense_h_to_4h.weight": L["w_up"], p + "mlp.dense_h_to_4h.bias": L["b_up"],
                   p + "mlp.dense_4h_to_h.weight": L["wd"], p + "mlp.dense_4h_to_h.bias": L["bd"]})
    missing, unexpected = hf.load_state_dict(sd, strict=False)
    assert not unexpected and all("lm_head" in m for m in missing), (missing, unexpected)
    hf.tie_weights()
    prompt = list(range(7, 47))
    toks, logits = orc.generate(prompt, 4)
    with torch.no_grad():
        ref = hf(torch.tensor([prompt + toks[:3]])).logits[0, len(prompt) - 1:].float()
    assert (logits - ref).abs().max().item() < 2e-4 * max(1.0, ref.abs().max().item())
