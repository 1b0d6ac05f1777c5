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
    # same arithmetic on gathered pages; CPU BLAS may block a reduction
    # differently from run to run (thread count under load), so not bitwise
    torch.testing.assert_close(log_p, log_c, rtol=1e-6, atol=1e-6)
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


def test_llama_oracle_matches_transformers_llama():
    """The Llama restatement (RMSNorm, half-split RoPE, GQA head grouping,
    SwiGLU, untied head) equals transformers' LlamaForCausalLM on the same
    weights — the independent pin of the branch C1-C4 run on."""
    from transformers import LlamaConfig, LlamaForCausalLM
    from paper_2311_18677_b200.model import ModelConfig, init_weights, logical_layer_fp32
    cfg = ModelConfig("llama-t", 2, 512, 4, 2, 128, 1024, 300, init_std=0.05)
    w = init_weights(cfg, seed=4, device="cpu")
    orc = OracleDecoder.from_weights(w)
    hf = LlamaForCausalLM(LlamaConfig(
        vocab_size=cfg.vocab, hidden_size=cfg.d_model, intermediate_size=cfg.ffn,
        num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_heads,
        num_key_value_heads=cfg.n_kv_heads, head_dim=cfg.head_dim, rms_norm_eps=cfg.norm_eps,
        rope_theta=cfg.rope_theta, max_position_embeddings=4096, tie_word_embeddings=False,
        attention_bias=False, mlp_bias=False)).eval()
    sd = {"model.embed_tokens.weight": w.embed.float(), "model.norm.weight": w.final_norm.float(),
          "lm_head.weight": w.lm_head.float()}
    for i in range(cfg.n_layers):
        L = logical_layer_fp32(w, i)
        p = f"model.layers.{i}."
        sd.update({p + "input_layernorm.weight": L["attn_norm"],
                   p + "self_attn.q_proj.weight": L["wq"], p + "self_attn.k_proj.weight": L["wk"],
                   p + "self_attn.v_proj.weight": L["wv"], p + "self_attn.o_proj.weight": L["wo"],
                   p + "post_attention_layernorm.weight": L["mlp_norm"],
                   p + "mlp.gate_proj.weight": L["w_gate"], p + "mlp.up_proj.weight": L["w_up"],
                   p + "mlp.down_proj.weight": L["wd"]})
    missing, unexpected = hf.load_state_dict(sd, strict=False)
    assert not unexpected and not [m for m in missing if "rotary" not in m], (missing, unexpected)
    # positions past the first few hundred exercise the RoPE angle tables
    prompt = torch.randint(0, cfg.vocab, (300,), generator=torch.Generator().manual_seed(2)).tolist()
    toks, logits = orc.generate(prompt, 5)
    with torch.no_grad():
        ref = hf(torch.tensor([prompt + toks[:4]])).logits[0, len(prompt) - 1:].float()
    err = (logits - ref).abs().max().item()
    assert err < 2e-4 * max(1.0, ref.abs().max().item()), err
    assert toks == ref.argmax(-1).tolist()
