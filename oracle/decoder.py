"""ORACLE — test infrastructure only (tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg).  Never imported by the
product package; the product path fails loudly without libswb200.so.

fp32 CPU restatement of the prefill -> KV hand-off -> decode arithmetic.

Parity status: the reference (splitsim) contains NO model arithmetic — its
prompt/token phases are latency lookups (reference perf.py:119-132) and KV is
a byte count (perf.py:134-141); SPEC.md:8/:173 put model math out of scope.
So the NUMERICS of this oracle are "parity unpinned" by the reference: it
follows the public Llama decoder definition (RMSNorm, RoPE half-split, GQA,
SwiGLU) and the public BLOOM definition (embedding LayerNorm, LayerNorm with
bias, ALiBi, biased linears, tanh-GELU, tied head) for the shapes in SURVEY
§8(c).  The BLOOM restatement is checked against transformers'
BloomForCausalLM on the same weights (tests/test_oracle_cpu.py).  What the reference DOES pin — the
phase semantics (the prompt phase produces the KV cache and the first token,
each token-phase iteration consumes the last token plus the KV,
PAPER.md:217-224; token task context = prompt+1, remaining = out-1,
engine.py:292-297) — is mirrored exactly: ``generate`` emits the first token
from the prompt phase and out-1 further tokens from decode iterations.

Also here: the deterministic lowest-free-first block allocator and a paged KV
store, so tests can check the device block tables bit-for-bit and that
decoding through block tables equals decoding over contiguous KV.
"""

from __future__ import annotations

import math

import torch


def _rmsnorm(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def _layernorm(x, w, b, eps):
    return torch.nn.functional.layer_norm(x, (x.shape[-1],), w, b, eps)


def _gelu_tanh(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * x * (1.0 + 0.044715 * x * x)))


def rope_tables(positions: torch.Tensor, dh: int, theta: float):
    half = dh // 2
    i = torch.arange(half, dtype=torch.float32)
    inv = torch.exp2(-math.log2(theta) * (2 * i) / dh)
    ang = positions.float()[:, None] * inv[None, :]
    return torch.cos(ang), torch.sin(ang)


def apply_rope(x, cos, sin):
    # x [S, heads, dh]
    half = x.shape[-1] // 2
    a, b = x[..., :half], x[..., half:]
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.cat([a * c - b * s, b * c + a * s], -1)


class LowestFreeAllocator:
    """CPU model of the device allocator (kvpool.cu): hands out the n lowest
    free block ids; freeing returns them.  Deterministic, so device tables
    must equal its tables bit-for-bit."""

    def __init__(self, num_blocks: int):
        self.num_blocks = num_blocks
        self.used = [False] * num_blocks

    @property
    def free_count(self):
        return self.used.count(False)

    def alloc(self, n: int) -> list[int]:
        if n > self.free_count:
            raise MemoryError(f"need {n} blocks, {self.free_count} free")
        out = []
        for b in range(self.num_blocks):
            if len(out) == n:
                break
            if not self.used[b]:
                self.used[b] = True
                out.append(b)
        return out

    def free(self, ids):
        for b in ids:
            self.used[b] = False


class PagedKV:
    """CPU paged KV store with the device layout [block][Hkv][bs][dh]."""

    def __init__(self, num_layers, num_blocks, n_kv_heads, block_size, head_dim):
        self.bs = block_size
        self.k = torch.zeros(num_layers, num_blocks, n_kv_heads, block_size, head_dim)
        self.v = torch.zeros_like(self.k)
        self.alloc = LowestFreeAllocator(num_blocks)
        self.tables: dict[int, list[int]] = {}

    def reserve(self, seq: int, tokens: int) -> list[int]:
        n = (tokens + self.bs - 1) // self.bs
        self.tables[seq] = self.alloc.alloc(n)
        return self.tables[seq]

    def release(self, seq: int):
        self.alloc.free(self.tables.pop(seq))

    def write(self, layer, seq, pos0, k, v):
        t = self.tables[seq]
        for i in range(k.shape[0]):
            p = pos0 + i
            self.k[layer, t[p // self.bs], :, p % self.bs] = k[i]
            self.v[layer, t[p // self.bs], :, p % self.bs] = v[i]

    def read(self, layer, seq, n):
        t = self.tables[seq]
        idx = torch.arange(n)
        blk = torch.tensor(t)[idx // self.bs]
        return self.k[layer, blk, :, idx % self.bs], self.v[layer, blk, :, idx % self.bs]


class OracleDecoder:
    """fp32 decoder over logical (unsharded, de-interleaved) weights: dict per
    layer with attn_norm, wq, wk, wv, wo, mlp_norm, w_gate, w_up, wd (Llama)
    or ln1_w/b, wq/k/v, bq/k/v, wo, bo, ln2_w/b, w_up, b_up, wd, bd (BLOOM,
    with ``extra`` = final_norm_b, emb_norm, emb_norm_b, alibi slopes)."""

    def __init__(self, cfg, layers, embed, lm_head, final_norm, threads: int | None = None,
                 extra: dict | None = None, emulate_bf16: bool = False):
        self.cfg = cfg
        # emulate_bf16: round every activation the device path stores in bf16
        # (GEMM inputs, q/k/v, attention output, MLP activation) — a
        # diagnostic twin that measures the error bf16 storage alone causes
        self.emulate_bf16 = emulate_bf16
        self.layers = layers
        self.embed = embed
        self.lm_head = lm_head
        self.final_norm = final_norm
        self.extra = extra or {}
        self.bloom = getattr(cfg, "arch", "llama") == "bloom"
        if threads:
            torch.set_num_threads(threads)

    @classmethod
    def from_weights(cls, w):
        """Build from a single-rank device ``Weights`` (copies to CPU fp32)."""
        from paper_2311_18677_b200.model import logical_layer_fp32
        assert w.tp == 1
        layers = [logical_layer_fp32(w, i) for i in range(w.cfg.n_layers)]
        extra = {}
        if w.cfg.arch == "bloom":
            extra = {k: getattr(w, k).float().cpu()
                     for k in ("final_norm_b", "emb_norm", "emb_norm_b", "alibi")}
        embed = w.embed.float().cpu()
        head = embed if w.lm_head.data_ptr() == w.embed.data_ptr() else w.lm_head.float().cpu()
        return cls(w.cfg, layers, embed, head, w.final_norm.float().cpu(), extra=extra)

    def _r(self, t):
        return t.bfloat16().float() if self.emulate_bf16 else t

    def _bloom_layer(self, li, x, pos0, kv_get, kv_put):
        """BLOOM block: pre-LayerNorm, fused biased qkv, ALiBi scores
        (slope * key position, as BLOOM builds its alibi tensor), biased
        dense, residual; LayerNorm, biased up, tanh-GELU, biased down."""
        cfg, L = self.cfg, self.layers[li]
        S = x.shape[0]
        H, dh, eps = cfg.n_heads, cfg.head_dim, cfg.norm_eps
        r = self._r
        h = r(_layernorm(x, L["ln1_w"], L["ln1_b"], eps))
        q = r(h @ L["wq"].t() + L["bq"]).view(S, H, dh)
        k = r(h @ L["wk"].t() + L["bk"]).view(S, H, dh)
        v = r(h @ L["wv"].t() + L["bv"]).view(S, H, dh)
        kv_put(li, pos0, k, v)
        K_all, V_all = kv_get(li, pos0 + S)
        n = pos0 + S
        s = torch.einsum("qhd,khd->hqk", q, K_all) / math.sqrt(dh)
        s = s + self.extra["alibi"][:, None, None] * torch.arange(n, dtype=torch.float32)
        qpos = torch.arange(pos0, pos0 + S)[:, None]
        kpos = torch.arange(n)[None, :]
        s = s.masked_fill((kpos > qpos)[None], float("-inf"))
        o = r(torch.einsum("hqk,khd->qhd", s.softmax(-1), V_all).reshape(S, H * dh))
        x = x + o @ L["wo"].t() + L["bo"]
        h2 = r(_layernorm(x, L["ln2_w"], L["ln2_b"], eps))
        a = r(_gelu_tanh(h2 @ L["w_up"].t() + L["b_up"]))
        return x + a @ L["wd"].t() + L["bd"]

    # -- one layer over S new tokens at positions pos0.. with cached K/V
    def _layer(self, li, x, pos0, kv_get, kv_put):
        if self.bloom:
            return self._bloom_layer(li, x, pos0, kv_get, kv_put)
        cfg, L = self.cfg, self.layers[li]
        S = x.shape[0]
        H, Hkv, dh = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
        r = self._r
        h = r(_rmsnorm(x, L["attn_norm"], cfg.norm_eps))
        q = r(h @ L["wq"].t()).view(S, H, dh)
        k = r(h @ L["wk"].t()).view(S, Hkv, dh)
        v = r(h @ L["wv"].t()).view(S, Hkv, dh)
        cos, sin = rope_tables(torch.arange(pos0, pos0 + S), dh, cfg.rope_theta)
        q, k = r(apply_rope(q, cos, sin)), r(apply_rope(k, cos, sin))
        kv_put(li, pos0, k, v)
        K_all, V_all = kv_get(li, pos0 + S)
        G = H // Hkv
        Kx, Vx = (K_all, V_all) if G == 1 else (K_all.repeat_interleave(G, 1),
                                                 V_all.repeat_interleave(G, 1))
        s = torch.einsum("qhd,khd->hqk", q, Kx) / math.sqrt(dh)
        qpos = torch.arange(pos0, pos0 + S)[:, None]
        kpos = torch.arange(pos0 + S)[None, :]
        s = s.masked_fill((kpos > qpos)[None], float("-inf"))
        o = r(torch.einsum("hqk,khd->qhd", s.softmax(-1), Vx).reshape(S, H * dh))
        x = x + o @ L["wo"].t()
        h2 = r(_rmsnorm(x, L["mlp_norm"], cfg.norm_eps))
        a = r(torch.nn.functional.silu(h2 @ L["w_gate"].t()) * (h2 @ L["w_up"].t()))
        return x + a @ L["wd"].t()

    def forward(self, tokens, pos0, kv_get, kv_put):
        x = self.embed[torch.as_tensor(tokens, dtype=torch.long)]
        eps = self.cfg.norm_eps
        if self.bloom:
            x = _layernorm(x, self.extra["emb_norm"], self.extra["emb_norm_b"], eps)
        for li in range(self.cfg.n_layers):
            x = self._layer(li, x, pos0, kv_get, kv_put)
        if self.bloom:
            h = _layernorm(x[-1:], self.final_norm, self.extra["final_norm_b"], eps)
        else:
            h = _rmsnorm(x[-1:], self.final_norm, eps)
        return (self._r(h) @ self.lm_head.t())[0]

    # -- contiguous KV (preallocated when the final length is known, so a
    #    decode step writes one row instead of re-concatenating the cache)
    def new_cache(self, max_len: int | None = None):
        c = {"k": [None] * self.cfg.n_layers, "v": [None] * self.cfg.n_layers, "cap": 0}
        if max_len:
            hkv, dh = self.cfg.n_kv_heads, self.cfg.head_dim
            c["k"] = [torch.empty(max_len, hkv, dh) for _ in range(self.cfg.n_layers)]
            c["v"] = [torch.empty(max_len, hkv, dh) for _ in range(self.cfg.n_layers)]
            c["cap"] = max_len
        return c

    def _contig(self, cache):
        def put(li, pos0, k, v):
            n = pos0 + k.shape[0]
            if n <= cache["cap"]:
                cache["k"][li][pos0:n] = k
                cache["v"][li][pos0:n] = v
            elif cache["k"][li] is None:
                cache["k"][li], cache["v"][li] = k, v
            else:
                cache["k"][li] = torch.cat([cache["k"][li][:pos0], k])
                cache["v"][li] = torch.cat([cache["v"][li][:pos0], v])

        def get(li, n):
            return cache["k"][li][:n], cache["v"][li][:n]
        return get, put

    def prefill(self, prompt, cache=None):
        cache = cache if cache is not None else self.new_cache()
        get, put = self._contig(cache)
        return self.forward(prompt, 0, get, put), cache

    def decode(self, tok, pos, cache):
        get, put = self._contig(cache)
        return self.forward([tok], pos, get, put)

    def generate(self, prompt, n_out, forced=None):
        """Greedy generation of n_out tokens (first from the prompt phase).
        ``forced`` teacher-forces the fed-back tokens (for comparing against a
        device run whose near-tie argmax may differ)."""
        logits, cache = self.prefill(prompt, self.new_cache(len(prompt) + n_out))
        toks, all_logits = [int(logits.argmax())], [logits]
        for i in range(1, n_out):
            feed = toks[-1] if forced is None else forced[i - 1]
            logits = self.decode(feed, len(prompt) + i - 1, cache)
            all_logits.append(logits)
            toks.append(int(logits.argmax()))
        return toks, torch.stack(all_logits)

    # -- paged KV (through block tables)
    def paged_generate(self, prompt, n_out, store: PagedKV, seq: int):
        def put(li, pos0, k, v):
            store.write(li, seq, pos0, k, v)

        def get(li, n):
            return store.read(li, seq, n)
        logits = self.forward(prompt, 0, get, put)
        toks, all_logits = [int(logits.argmax())], [logits]
        for i in range(1, n_out):
            logits = self.forward([toks[-1]], len(prompt) + i - 1, get, put)
            all_logits.append(logits)
            toks.append(int(logits.argmax()))
        return toks, torch.stack(all_logits)
