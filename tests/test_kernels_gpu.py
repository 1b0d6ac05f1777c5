"""Kernel-level numerics of libswb200 on the GPU, each against a plain
PyTorch fp32 reference of the same op (bf16 inputs upcast), and bit-exact
checks for the integer / byte paths (allocator, KV write, KV push)."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2311_18677_b200 import kernels
    torch.manual_seed(0)
    return kernels


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6)).item()


@pytest.mark.parametrize("M,N,K_", [(128, 256, 64), (1000, 768, 4096), (300, 12288, 4096),
                                    (129, 4096, 11008), (64, 96, 136), (2048, 512, 1024)])
def test_gemm_bf16(K, M, N, K_):
    a = torch.randn(M, K_, device="cuda").bfloat16()
    w = torch.randn(N, K_, device="cuda").bfloat16()
    ref = a.float() @ w.float().t()
    out = K.gemm(a, w, K.EPI_BF16)
    torch.cuda.synchronize()
    assert _rel(out, ref) < 1e-2
    out32 = K.gemm(a, w, K.EPI_F32)
    assert _rel(out32, ref) < 1e-4


def test_gemm_resid_and_swiglu(K):
    M, N, K_ = 300, 1024, 512
    a = torch.randn(M, K_, device="cuda").bfloat16()
    w = torch.randn(N, K_, device="cuda").bfloat16()
    res = torch.randn(M, N, device="cuda")
    ref = res + a.float() @ w.float().t()
    out = res.clone()
    K.gemm(a, w, K.EPI_RESID_F32, out=out, resid=out)
    assert _rel(out, ref) < 1e-4
    acc = a.float() @ w.float().t()
    g = acc.view(M, N // 256, 2, 128)[:, :, 0, :].reshape(M, N // 2)
    u = acc.view(M, N // 256, 2, 128)[:, :, 1, :].reshape(M, N // 2)
    ref_sw = torch.nn.functional.silu(g) * u
    out_sw = K.gemm(a, w, K.EPI_SWIGLU)
    assert _rel(out_sw, ref_sw) < 1e-2


@pytest.mark.parametrize("M", [1, 2, 3, 8, 16, 24, 32])
@pytest.mark.parametrize("N,K_", [(4096, 4096), (768, 256), (1000, 11008), (256, 14336),
                                  (250, 64)])
def test_gemv(K, M, N, K_):
    x = torch.randn(M, K_, device="cuda").bfloat16()
    w = torch.randn(N, K_, device="cuda").bfloat16()
    ref = x.float() @ w.float().t()
    assert _rel(K.gemv(x, w, K.EPI_F32), ref) < 1e-4
    assert _rel(K.gemv(x, w, K.EPI_BF16), ref) < 1e-2
    res = torch.randn(M, N, device="cuda")
    out = res.clone()
    K.gemv(x, w, K.EPI_RESID_F32, out=out, resid=out)
    assert _rel(out, res + ref) < 1e-4


@pytest.mark.parametrize("M", [1, 4, 20])
def test_gemv_swiglu(K, M):
    N, K_ = 2048, 1024
    x = torch.randn(M, K_, device="cuda").bfloat16()
    w = torch.randn(N, K_, device="cuda").bfloat16()
    acc = x.float() @ w.float().t()
    g = acc.view(M, N // 256, 2, 128)[:, :, 0, :].reshape(M, N // 2)
    u = acc.view(M, N // 256, 2, 128)[:, :, 1, :].reshape(M, N // 2)
    ref = torch.nn.functional.silu(g) * u
    assert _rel(K.gemv(x, w, K.EPI_SWIGLU), ref) < 1e-2


@pytest.mark.parametrize("M", [2, 8, 32])
def test_gemv_batched_deterministic(K, M):
    """The split-K tcgen05 GEMV reduces cluster partials in fixed rank order:
    repeated launches are bit-identical."""
    x = torch.randn(M, 11008, device="cuda").bfloat16()
    w = torch.randn(4096, 11008, device="cuda").bfloat16()
    a = K.gemv(x, w, K.EPI_F32)
    for _ in range(3):
        assert torch.equal(K.gemv(x, w, K.EPI_F32), a)


def test_embed_rmsnorm_argmax(K):
    V, d, rows = 1000, 4096, 37
    table = torch.randn(V, d, device="cuda").bfloat16()
    tok = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
    x = K.embed(tok, table)
    assert torch.equal(x, table[tok.long()].float())
    w = torch.randn(d, device="cuda").bfloat16()
    h = K.rmsnorm(x, w, 1e-5)
    ref = x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
    assert _rel(h, ref) < 1e-2
    idx = torch.tensor([3, 0, 36], device="cuda", dtype=torch.int32)
    h2 = K.rmsnorm(x, w, 1e-5, rows_index=idx)
    assert torch.equal(h2, h[idx.long()])
    logits = torch.randn(5, 32000, device="cuda")
    logits[2, 100] = 50.0
    logits[2, 7] = 50.0  # tie -> lowest index
    am = K.argmax(logits)
    ref_am = logits.argmax(-1).int()
    ref_am[2] = 7
    assert torch.equal(am, ref_am)


def _rope_ref(x, pos, theta):
    dh = x.shape[-1]
    half = dh // 2
    i = torch.arange(half, device=x.device, dtype=torch.float32)
    inv = torch.exp2(-math.log2(theta) * (2 * i) / dh)
    ang = pos.float()[:, None] * inv[None, :]
    c, s = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
    a, b = x[..., :half].float(), x[..., half:].float()
    return torch.cat([a * c - b * s, b * c + a * s], -1)


def test_rope_kv_write_bit_exact_pool(K):
    H, Hkv, dh, bs, rows = 8, 2, 128, 16, 50
    qkv = torch.randn(rows, (H + 2 * Hkv) * dh, device="cuda").bfloat16()
    pos = torch.arange(rows, device="cuda", dtype=torch.int32) + 1000
    nblk = 8
    kpool = torch.zeros(nblk, Hkv, bs, dh, device="cuda", dtype=torch.bfloat16)
    vpool = torch.zeros_like(kpool)
    table = torch.tensor([5, 2, 7, 0], device="cuda", dtype=torch.int32)
    p = torch.arange(rows, device="cuda")
    slots = (table[p // bs].long() * bs + p % bs).int()
    orig = qkv.clone()
    K.rope_kv_write(qkv, pos, H, Hkv, dh, 10000.0, kpool.data_ptr(), vpool.data_ptr(), slots, bs)
    q = orig[:, :H * dh].view(rows, H, dh)
    k = orig[:, H * dh:(H + Hkv) * dh].view(rows, Hkv, dh)
    v = orig[:, (H + Hkv) * dh:].view(rows, Hkv, dh)
    assert _rel(qkv[:, :H * dh].view(rows, H, dh), _rope_ref(q, pos, 1e4)) < 1e-2
    assert _rel(qkv[:, H * dh:(H + Hkv) * dh].view(rows, Hkv, dh), _rope_ref(k, pos, 1e4)) < 1e-2
    # pool holds exactly the rotated k and the untouched v (bitwise)
    kr = qkv[:, H * dh:(H + Hkv) * dh].view(rows, Hkv, dh)
    for r in range(rows):
        blk, off = int(slots[r]) // bs, int(slots[r]) % bs
        assert torch.equal(kpool[blk, :, off], kr[r])
        assert torch.equal(vpool[blk, :, off], v[r])


def _attn_ref(q, k, v, causal=True):
    # q [S,H,D], k/v [S,Hkv,D]
    S, H, D = q.shape
    G = H // k.shape[1]
    k = k.repeat_interleave(G, 1)
    v = v.repeat_interleave(G, 1)
    s = torch.einsum("qhd,khd->hqk", q.float(), k.float()) / math.sqrt(D)
    if causal:
        m = torch.ones(S, S, device=q.device, dtype=torch.bool).tril()
        s = s.masked_fill(~m, float("-inf"))
    p = s.softmax(-1)
    return torch.einsum("hqk,khd->qhd", p, v.float())


@pytest.mark.parametrize("impl", ["tc", "fa2"])
@pytest.mark.parametrize("H,Hkv,lens", [(4, 4, [1, 63, 64, 200, 130]),
                                        (8, 2, [1, 63, 64, 200, 130]),
                                        (4, 1, [129, 1024, 7, 256, 511])])
def test_attn_prefill_varlen(K, H, Hkv, lens, impl):
    dh = 128
    S = sum(lens)
    qkv = torch.randn(S, (H + 2 * Hkv) * dh, device="cuda").bfloat16()
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), device="cuda", dtype=torch.int32)
    out = K.attn_prefill(qkv, cu, len(lens), max(lens), H, Hkv, dh, 1 / math.sqrt(dh),
                         impl=impl)
    off = 0
    for L in lens:
        blk = qkv[off:off + L]
        q = blk[:, :H * dh].view(L, H, dh)
        k = blk[:, H * dh:(H + Hkv) * dh].view(L, Hkv, dh)
        v = blk[:, (H + Hkv) * dh:].view(L, Hkv, dh)
        ref = _attn_ref(q, k, v)
        got = out[off:off + L].view(L, H, dh)
        assert _rel(got, ref) < 2e-2, L
        off += L


@pytest.mark.parametrize("H,Hkv,part", [(32, 32, 128), (64, 8, 128), (32, 32, 32), (64, 8, 64)])
def test_attn_decode_paged(K, H, Hkv, part):
    dh, bs = 128, 16
    ctx = [1, 17, 300, 1100]
    B = len(ctx)
    maxb = 80
    nblk = 400
    kpool = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    vpool = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    perm = torch.randperm(nblk, device="cuda").int()
    tables = perm[:B * maxb].view(B, maxb).contiguous()
    qkv = torch.randn(B, (H + 2 * Hkv) * dh, device="cuda").bfloat16()
    lens = torch.tensor(ctx, device="cuda", dtype=torch.int32)
    wsb = K.attn_decode_workspace_bytes(B, H, 1200, part, dh)
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
    out = K.attn_decode(qkv, kpool.data_ptr(), vpool.data_ptr(), tables, lens, B, H, Hkv, dh, bs,
                        1 / math.sqrt(dh), 1200, part, ws)
    out2 = K.attn_decode(qkv, kpool.data_ptr(), vpool.data_ptr(), tables, lens, B, H, Hkv, dh,
                         bs, 1 / math.sqrt(dh), 1200, part, ws)   # tickets self-reset
    assert torch.equal(out, out2)
    for b in range(B):
        L = ctx[b]
        p = torch.arange(L, device="cuda")
        blk = tables[b][p // bs].long()
        k = kpool[blk, :, p % bs]  # [L,Hkv,dh]
        v = vpool[blk, :, p % bs]
        q = qkv[b, :H * dh].view(1, H, dh)
        G = H // Hkv
        s = torch.einsum("hd,lhd->hl", q[0].float(), k.repeat_interleave(G, 1).float()) / math.sqrt(dh)
        ref = torch.einsum("hl,lhd->hd", s.softmax(-1), v.repeat_interleave(G, 1).float())
        assert _rel(out[b].view(H, dh), ref) < 1e-2, b


def test_block_alloc_lowest_free_first(K):
    from paper_2311_18677_b200.kvcache import KVCacheManager
    from paper_2311_18677_b200.errors import CapacityError
    kv = KVCacheManager(num_layers=2, num_blocks=100, n_kv_heads=2, head_dim=128,
                        block_size=16, max_seqs=4, max_blocks_per_seq=40)
    s0 = kv.allocate(160)        # 10 blocks -> 0..9
    s1 = kv.allocate(80)         # 5 blocks  -> 10..14
    kv.release(s0)
    s2 = kv.allocate(180)        # 12 blocks -> 0..9, 15, 16 (lowest free first)
    torch.cuda.synchronize()
    t = kv.tables().cpu()
    assert t[s1, :5].tolist() == [10, 11, 12, 13, 14]
    assert t[s2, :12].tolist() == list(range(10)) + [15, 16]
    assert kv.free_blocks == 100 - 17
    with pytest.raises(CapacityError):
        kv.allocate(16 * 41)     # more than max_blocks_per_seq
    kv.close()


def test_kv_push_local_bit_exact(K):
    """Pack-and-push into a second pool on the same GPU: every pushed K/V
    byte must equal the source rows bitwise, at the slots of the table."""
    from paper_2311_18677_b200.kvcache import KVCacheManager
    H, Hkv, dh, bs, rows = 8, 2, 128, 16, 77
    dst = KVCacheManager(num_layers=3, num_blocks=64, n_kv_heads=Hkv, head_dim=dh,
                         block_size=bs, max_seqs=4, max_blocks_per_seq=16)
    dst.allocate(40)
    seq = dst.allocate(rows)
    qkv = torch.randn(rows, (H + 2 * Hkv) * dh, device="cuda").bfloat16()
    slots = torch.empty(rows, dtype=torch.int32, device="cuda")
    K.slots_from_table(dst.table_row_ptr(seq), 0, rows, bs, slots)
    K.kv_push_layer(qkv, rows, H, Hkv, dh, dst.k_layer_ptr(1), dst.v_layer_ptr(1), slots, bs,
                    num_ctas=8)
    torch.cuda.synchronize()
    kview, vview = dst.k_view(1), dst.v_view(1)
    table = dst.tables()[seq]
    p = torch.arange(rows, device="cuda")
    blk = table[p // bs].long()
    got_k = kview[blk, :, p % bs]
    got_v = vview[blk, :, p % bs]
    assert torch.equal(got_k, qkv[:, H * dh:(H + Hkv) * dh].view(rows, Hkv, dh))
    assert torch.equal(got_v, qkv[:, (H + Hkv) * dh:].view(rows, Hkv, dh))
    dst.close()


@pytest.mark.parametrize("M,d", [(1, 4096), (2, 4096), (3, 2048), (4, 4096), (8, 2048),
                                 (2, 8192)])
def test_gemv_rmsnorm_equals_rmsnorm_then_gemv(K, M, d):
    """The fused pre-norm GEMV sees exactly the bf16 h that swb_rmsnorm
    produces, so its outputs equal the two-kernel path: bitwise for the
    batched (mma.sync) kernel, which reduces rstd in swb_rmsnorm's order;
    fp32 tolerance for the M=1 kernel (h staged in 16 KB of smem)."""
    N = 3072
    x = torch.randn(M, d, device="cuda") * 3
    nw = (1 + 0.1 * torch.randn(d, device="cuda")).bfloat16()
    w = torch.randn(N, d, device="cuda").bfloat16()
    h = K.rmsnorm(x, nw, 1e-5)
    ref = K.gemv(h, w, K.EPI_F32)
    got = K.gemv_rmsnorm(x, nw, 1e-5, w, K.EPI_F32)
    wgu = torch.randn(2048, d, device="cuda").bfloat16()
    gu_f = K.gemv_rmsnorm(x, nw, 1e-5, wgu, K.EPI_SWIGLU)
    gu_r = K.gemv(h, wgu, K.EPI_SWIGLU)
    if M == 1:
        assert _rel(got, ref) < 1e-5
        assert _rel(gu_f, gu_r) < 1e-2
    else:
        assert torch.equal(got, ref)
        assert torch.equal(gu_f.view(torch.int16), gu_r.view(torch.int16))


def test_gemv_rmsnorm_rejects_oversized_stage(K):
    from paper_2311_18677_b200.errors import ValidationError
    nw = torch.ones(16384, device="cuda").bfloat16()
    w = torch.randn(256, 16384, device="cuda").bfloat16()
    with pytest.raises(ValidationError):       # M=1 stages h (K*2 bytes) in 16 KB
        K.gemv_rmsnorm(torch.randn(1, 16384, device="cuda"), nw, 1e-5, w, K.EPI_F32)
    with pytest.raises(ValidationError):       # batched variant: M <= 8, h <= 32 KB
        K.gemv_rmsnorm(torch.randn(9, 1024, device="cuda"), nw[:1024], 1e-5, w[:, :1024],
                       K.EPI_F32)
    with pytest.raises(ValidationError):
        K.gemv_rmsnorm(torch.randn(4, 8192, device="cuda"), nw[:8192], 1e-5, w[:, :8192],
                       K.EPI_F32)


@pytest.mark.parametrize("H,Hkv", [(32, 32), (64, 8)])
def test_attn_decode_fused_rope_append(K, H, Hkv):
    """Fused decode attention (RoPE + KV append of the current token inside
    the kernel) == rope_kv_write followed by plain paged attention, and the
    appended pool rows are bit-identical."""
    dh, bs, B = 128, 16, 3
    ctx = [5, 129, 700]          # tokens incl. the current one
    nblk = 200
    maxb = 48
    kp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    vp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    kp2, vp2 = kp.clone(), vp.clone()
    tables = torch.randperm(nblk, device="cuda").int()[:B * maxb].view(B, maxb).contiguous()
    lens = torch.tensor(ctx, device="cuda", dtype=torch.int32)
    pos = lens - 1
    slots = (tables[torch.arange(B, device="cuda"), (pos // bs).long()].long() * bs + pos % bs).int()
    qkv = torch.randn(B, (H + 2 * Hkv) * dh, device="cuda").bfloat16()
    qkv2 = qkv.clone()
    part = 128
    ws = torch.zeros(K.attn_decode_workspace_bytes(B, H, 768, part, dh), dtype=torch.uint8,
                     device="cuda")
    fused = K.attn_decode(qkv, kp.data_ptr(), vp.data_ptr(), tables, lens, B, H, Hkv, dh, bs,
                          1 / math.sqrt(dh), 768, part, ws, positions=pos, slots=slots,
                          theta=10000.0)
    K.rope_kv_write(qkv2, pos, H, Hkv, dh, 10000.0, kp2.data_ptr(), vp2.data_ptr(), slots, bs)
    ref = K.attn_decode(qkv2, kp2.data_ptr(), vp2.data_ptr(), tables, lens, B, H, Hkv, dh, bs,
                        1 / math.sqrt(dh), 768, part, ws)
    torch.cuda.synchronize()
    assert torch.equal(kp.view(torch.int16), kp2.view(torch.int16))
    assert torch.equal(vp.view(torch.int16), vp2.view(torch.int16))
    assert _rel(fused, ref) < 1e-3


@pytest.mark.parametrize("H,Hkv,part,alibi", [(32, 32, 64, False), (64, 8, 32, False),
                                              (16, 16, 128, True)])
def test_attn_decode_step_matches_explicit(K, H, Hkv, part, alibi):
    """Decode-graph attention (swb_attn_decode_step: position = ctx, slot from
    the block table, pages gathered before the PDL wait) equals the
    explicit-position split-K form: appended pool rows bit-identical; output
    within bf16 rounding (MHA runs the cluster-streaming kernel, whose online
    softmax sums in a different order)."""
    dh, bs, B = 128, 16, 4
    cached = [0, 15, 128, 1000]          # tokens already in the pool
    nblk, maxb = 400, 80
    kp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    vp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    kp2, vp2 = kp.clone(), vp.clone()
    tables = torch.randperm(nblk, device="cuda").int()[:B * maxb].view(B, maxb).contiguous()
    ctx = torch.tensor(cached, device="cuda", dtype=torch.int32)
    slots = (tables[torch.arange(B, device="cuda"), (ctx // bs).long()].long() * bs
             + ctx % bs).int()
    qkv = torch.randn(B, (H + 2 * Hkv) * dh, device="cuda").bfloat16()
    slopes = (torch.rand(H, device="cuda") * 0.5) if alibi else None
    max_ctx = 1024 + 64
    mk = lambda: torch.zeros(K.attn_decode_workspace_bytes(B, H, max_ctx, part, dh),  # noqa: E731
                             dtype=torch.uint8, device="cuda")
    out = torch.empty(B, H * dh, dtype=torch.bfloat16, device="cuda")
    K.attn_decode_step(qkv, kp.data_ptr(), vp.data_ptr(), tables, ctx, B, H, Hkv, dh, bs,
                       1 / math.sqrt(dh), max_ctx, part, mk(), out, theta=10000.0,
                       alibi=slopes)
    ref = K.attn_decode(qkv, kp2.data_ptr(), vp2.data_ptr(), tables, ctx + 1, B, H, Hkv, dh, bs,
                        1 / math.sqrt(dh), max_ctx, part, mk(), positions=ctx, slots=slots,
                        theta=10000.0, alibi=slopes)
    torch.cuda.synchronize()
    if H == Hkv:
        assert _rel(out, ref) < 4e-3
    else:
        assert torch.equal(out.view(torch.int16), ref.view(torch.int16))
    assert torch.equal(kp.view(torch.int16), kp2.view(torch.int16))
    assert torch.equal(vp.view(torch.int16), vp2.view(torch.int16))


@pytest.mark.parametrize("H,Hkv,alibi,cached,gqa", [
    (32, 32, False, [0, 15, 16, 130, 1000, 2047], "-"), (8, 4, False, [3, 700], "-"),
    (16, 16, True, [31, 1500], "-"), (32, 32, False, [8190], "-"),
    # B * heads * 8 > 444: the launcher picks 4-CTA clusters (7B B=2 shape)
    (32, 32, False, [1100, 1100], "-"), (16, 16, True, [31, 1500, 700, 0], "-"),
    (64, 8, False, [3, 1100], "cuda"), (16, 4, True, [500], "cuda"),
    (64, 8, False, [3, 1100], "mma"), (64, 8, False, [1900], "mma"), (16, 4, True, [500], "mma"),
    (64, 8, False, [5, 900, 40, 1023], "split")])
def test_attn_decode_cluster_kernel_vs_torch(K, H, Hkv, alibi, cached, gqa, monkeypatch):
    """Decode-graph attention — the cluster-streaming kernel for G = 1, 2 (and
    its head-split GQA mode), the tensor-core kernel for G = 4, 8 in its
    cluster (DSMEM merge) and split-K forms —
    against a plain torch fp32 attention over the gathered pages: the current
    token (position = ctx) is RoPE'd (or ALiBi-biased), appended to its
    block-table slot, and attends over positions 0..ctx; contexts from 1 token
    to 8191 (every CTA of the 8-CTA cluster empty, partial or full)."""
    from oracle.decoder import apply_rope, rope_tables
    # GQA path: the CUDA-core cluster kernel's head split ("cuda"), the
    # tensor-core cluster form ("mma", B <= 2) or the split-K MMA kernel
    monkeypatch.setenv("SWB_ATTN_CL_MAXB_GQA", "2" if gqa == "cuda" else "0")
    dh, bs, B = 128, 16, len(cached)
    maxb = (max(cached) + 1 + bs - 1) // bs + 1
    nblk = B * maxb + 8
    kp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    vp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    tables = torch.randperm(nblk, device="cuda").int()[:B * maxb].view(B, maxb).contiguous()
    ctx = torch.tensor(cached, device="cuda", dtype=torch.int32)
    qkv = torch.randn(B, (H + 2 * Hkv) * dh, device="cuda").bfloat16()
    slopes = (torch.rand(H, device="cuda") * 0.1) if alibi else None
    max_ctx = 16 * maxb
    ws = torch.zeros(K.attn_decode_workspace_bytes(B, H, max_ctx, 128, dh), dtype=torch.uint8,
                     device="cuda")
    out = torch.empty(B, H * dh, dtype=torch.bfloat16, device="cuda")
    kp0, vp0 = kp.clone(), vp.clone()
    K.attn_decode_step(qkv, kp.data_ptr(), vp.data_ptr(), tables, ctx, B, H, Hkv, dh, bs,
                       1 / math.sqrt(dh), max_ctx, 128, ws, out, theta=10000.0, alibi=slopes)
    torch.cuda.synchronize()
    G = H // Hkv
    for b, c in enumerate(cached):
        q = qkv[b, :H * dh].float().view(1, H, dh)
        k = qkv[b, H * dh:(H + Hkv) * dh].float().view(1, Hkv, dh)
        v = qkv[b, (H + Hkv) * dh:].float().view(1, Hkv, dh)
        if not alibi:
            cos, sin = rope_tables(torch.tensor([c]), dh, 10000.0)
            q = apply_rope(q.cpu(), cos, sin).bfloat16().float().cuda()
            k = apply_rope(k.cpu(), cos, sin).cuda()
        k = k.bfloat16()
        blk = tables[b, c // bs].long()
        assert _rel(kp[blk, :, c % bs], k[0]) < 1e-2              # RoPE'd k appended
        assert torch.equal(vp[blk, :, c % bs].view(torch.int16), v[0].bfloat16().view(torch.int16))
        pos = torch.arange(c + 1, device="cuda")
        Ks = kp0[tables[b, pos // bs].long(), :, pos % bs].float()
        Vs = vp0[tables[b, pos // bs].long(), :, pos % bs].float()
        Ks[c], Vs[c] = k[0].float(), v[0].bfloat16().float()
        Ks, Vs = Ks.repeat_interleave(G, 1), Vs.repeat_interleave(G, 1)
        s_ = torch.einsum("hd,thd->ht", q[0], Ks) / math.sqrt(dh)
        if alibi:
            s_ = s_ + slopes[:, None] * (pos - c)[None, :].float()
        ref = torch.einsum("ht,thd->hd", s_.softmax(-1), Vs).reshape(-1)
        assert _rel(out[b], ref) < 1e-2, (b, c)


@pytest.mark.parametrize("M", [1, 5, 300])
def test_bias_and_gelu_epilogues(K, M):
    """Biased linears (BLOOM): bf16 / GELU / residual epilogues with a bias
    against a torch fp32 reference, through the GEMV (M <= 16) and the
    tcgen05 GEMM (M > 16)."""
    N, Kd = 768, 512
    x = torch.randn(M, Kd, device="cuda").bfloat16()
    w = (torch.randn(N, Kd, device="cuda") * 0.05).bfloat16()
    b = torch.randn(N, device="cuda").bfloat16()
    ref = x.float() @ w.float().t() + b.float()
    assert _rel(K.linear(x, w, K.EPI_BF16, bias=b), ref) < 1e-2
    gelu = 0.5 * ref * (1 + torch.tanh(0.7978845608028654 * ref * (1 + 0.044715 * ref * ref)))
    assert _rel(K.linear(x, w, K.EPI_GELU, bias=b), gelu) < 1e-2
    r = torch.randn(M, N, device="cuda")
    res = r.clone()
    K.linear(x, w, K.EPI_RESID_F32, out=res, resid=res, bias=b)
    assert _rel(res, r + ref) < 1e-4


def test_layernorm(K):
    d = 1024
    x = torch.randn(7, d, device="cuda") * 3 + 1
    w = (1 + 0.1 * torch.randn(d, device="cuda")).bfloat16()
    b = (0.1 * torch.randn(d, device="cuda")).bfloat16()
    ref = torch.nn.functional.layer_norm(x, (d,), w.float(), b.float(), 1e-5)
    assert _rel(K.layernorm(x, w, b, 1e-5), ref) < 1e-2
    idx = torch.tensor([6, 0], device="cuda", dtype=torch.int32)
    assert _rel(K.layernorm(x, w, b, 1e-5, rows_index=idx), ref[[6, 0]]) < 1e-2
    y = x.clone()
    K.layernorm(y, w, b, 1e-5, out=y, out_f32=True)          # in place, fp32
    assert _rel(y, ref) < 1e-5


def _alibi_ref(q, k, v, slopes, q0=0):
    # q [S,H,dh] at positions q0.., k/v [T,H,dh] at 0..T-1; causal
    S, T = q.shape[0], k.shape[0]
    s = torch.einsum("qhd,khd->hqk", q.float(), k.float()) / math.sqrt(q.shape[-1])
    s = s + slopes[:, None, None] * torch.arange(T, device=q.device).float()
    qp = torch.arange(q0, q0 + S, device=q.device)[:, None]
    kp = torch.arange(T, device=q.device)[None, :]
    s = s.masked_fill((kp > qp)[None], float("-inf"))
    return torch.einsum("hqk,khd->qhd", s.softmax(-1), v.float())


def test_attn_prefill_alibi(K):
    from paper_2311_18677_b200.model import alibi_slopes
    H, dh = 6, 128
    lens = [1, 130, 300, 64]
    S = sum(lens)
    qkv = torch.randn(S, 3 * H * dh, device="cuda").bfloat16()
    slopes = torch.tensor(alibi_slopes(H), device="cuda")
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), device="cuda", dtype=torch.int32)
    out = K.attn_prefill(qkv, cu, len(lens), max(lens), H, H, dh, 1 / math.sqrt(dh),
                         alibi=slopes)
    off = 0
    for L in lens:
        blk = qkv[off:off + L]
        q, k, v = (blk[:, i * H * dh:(i + 1) * H * dh].view(L, H, dh) for i in range(3))
        assert _rel(out[off:off + L].view(L, H, dh), _alibi_ref(q, k, v, slopes)) < 2e-2, L
        off += L


def test_attn_decode_alibi_append(K):
    """ALiBi decode: no rotation, the current token's k/v are appended as is,
    scores carry slope * (key - query)."""
    from paper_2311_18677_b200.model import alibi_slopes
    H, dh, bs, B = 6, 128, 16, 3
    ctx = [1, 40, 333]
    nblk, maxb = 200, 32
    kp = torch.randn(nblk, H, bs, dh, device="cuda").bfloat16()
    vp = torch.randn(nblk, H, bs, dh, device="cuda").bfloat16()
    tables = torch.randperm(nblk, device="cuda").int()[:B * maxb].view(B, maxb).contiguous()
    lens = torch.tensor(ctx, device="cuda", dtype=torch.int32)
    pos = lens - 1
    slots = torch.stack([tables[b, int(pos[b]) // bs] * bs + int(pos[b]) % bs
                         for b in range(B)]).int()
    qkv = torch.randn(B, 3 * H * dh, device="cuda").bfloat16()
    slopes = torch.tensor(alibi_slopes(H), device="cuda")
    part = 128
    ws = torch.zeros(K.attn_decode_workspace_bytes(B, H, 384, part, dh), dtype=torch.uint8,
                     device="cuda")
    out = K.attn_decode(qkv, kp.data_ptr(), vp.data_ptr(), tables, lens, B, H, H, dh, bs,
                        1 / math.sqrt(dh), 384, part, ws, positions=pos.clone(),
                        slots=slots, alibi=slopes)
    for b in range(B):
        n = ctx[b]
        p = torch.arange(n, device="cuda")
        blocks = tables[b, p // bs].long()
        kk = kp[blocks, :, p % bs]                   # [n, H, dh]
        vv = vp[blocks, :, p % bs]
        cur_k = qkv[b, H * dh:2 * H * dh].view(H, dh)
        cur_v = qkv[b, 2 * H * dh:].view(H, dh)
        assert torch.equal(kk[-1], cur_k) and torch.equal(vv[-1], cur_v)   # appended as is
        q = qkv[b, :H * dh].view(1, H, dh)
        ref = _alibi_ref(q, kk, vv, slopes, q0=n - 1)[0]
        assert _rel(out[b].view(H, dh), ref) < 2e-2, b


@pytest.mark.parametrize("alibi", [False, True])
def test_attn_decode_step_large_batch(K, alibi):
    """Decode-graph attention at a batch that fills the GPU (B*Hkv = 320):
    output against a torch fp32 reference over the pool after the kernel
    appended the current token (RoPE'd at its position, or ALiBi), including
    contexts that end mid-page / mid-partition and the 0-cached case."""
    H = Hkv = 32
    dh, bs = 128, 16
    B = 10
    cached = [0, 1, 15, 16, 63, 64, 65, 700, 1000, 1500]
    maxb = 1600 // bs
    nblk = B * maxb + 8
    kp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    vp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    tables = torch.randperm(nblk, device="cuda").int()[:B * maxb].view(B, maxb).contiguous()
    ctx = torch.tensor(cached, device="cuda", dtype=torch.int32)
    qkv = torch.randn(B, 3 * H * dh, device="cuda").bfloat16()
    slopes = (torch.rand(H, device="cuda") * 0.1) if alibi else None
    out = torch.empty(B, H * dh, dtype=torch.bfloat16, device="cuda")
    ws = torch.zeros(K.attn_decode_workspace_bytes(B, H, 1664, 128, dh), dtype=torch.uint8,
                     device="cuda")
    K.attn_decode_step(qkv, kp.data_ptr(), vp.data_ptr(), tables, ctx, B, H, Hkv, dh, bs,
                       1 / math.sqrt(dh), 1664, 128, ws, out, theta=10000.0, alibi=slopes)
    torch.cuda.synchronize()
    for b in range(B):
        L = cached[b] + 1
        p = torch.arange(L, device="cuda")
        blk = tables[b][p // bs].long()
        k = kp[blk, :, p % bs].float()              # [L, H, dh] incl. the appended token
        v = vp[blk, :, p % bs].float()
        q = qkv[b, :H * dh].view(H, dh).float()
        if not alibi:   # the kernel rotates q at position cached[b]; use its appended k to check
            half = dh // 2
            inv = 10000.0 ** (-torch.arange(half, device="cuda", dtype=torch.float32) * 2 / dh)
            ang = cached[b] * inv
            c, s_ = torch.cos(ang), torch.sin(ang)
            q = torch.cat([q[:, :half] * c - q[:, half:] * s_, q[:, half:] * c + q[:, :half] * s_],
                          1).bfloat16().float()
        s = torch.einsum("hd,lhd->hl", q, k) / math.sqrt(dh)
        if alibi:
            s = s + slopes[:, None] * (p[None, :] - cached[b]).float()
        ref = torch.einsum("hl,lhd->hd", s.softmax(-1), v)
        assert _rel(out[b].view(H, dh), ref) < 1e-2, b


@pytest.mark.parametrize("M,bias,theta", [(100, False, 10000.0), (300, False, 10000.0),
                                          (300, True, 0.0), (1024, False, 500000.0)])
def test_gemm_qkv_rope_equals_gemm_then_rope(K, M, bias, theta):
    """The fused QKV-GEMM epilogue (RoPE + paged KV write) is bit-identical to
    the GEMM followed by swb_rope_kv_write: stored qkv and pool pages."""
    H, Hkv, dh, bs, d = 8, 2, 128, 16, 1024
    N = (H + 2 * Hkv) * dh
    a = torch.randn(M, d, device="cuda").bfloat16()
    w = (torch.randn(N, d, device="cuda") * 0.05).bfloat16()
    b = (torch.randn(N, device="cuda") * 0.1).bfloat16() if bias else None
    pos = torch.randint(0, 4000, (M,), device="cuda", dtype=torch.int32)
    nblk = (M + bs - 1) // bs + 4
    slots = torch.randperm(nblk * bs, device="cuda")[:M].int()
    k1 = torch.zeros(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    v1, k2, v2 = k1.clone(), k1.clone(), k1.clone()
    ref = K.gemm(a, w, K.EPI_BF16, bias=b)
    K.rope_kv_write(ref, pos, H, Hkv, dh, theta, k1.data_ptr(), v1.data_ptr(), slots, bs)
    for tab in (None, K.rope_table(theta, 2048) if theta > 1 else None):
        got = torch.empty_like(ref)
        k2.zero_(); v2.zero_()
        K.gemm_qkv_rope(a, w, got, pos, H, Hkv, theta, bias=b, k_layer=k2.data_ptr(),
                        v_layer=v2.data_ptr(), slots=slots, block_size=bs, rope_table=tab)
        torch.cuda.synchronize()   # positions >= 2048 fall back to computing the angles
        assert torch.equal(got.view(torch.int16), ref.view(torch.int16))
        assert torch.equal(k2.view(torch.int16), k1.view(torch.int16))
        assert torch.equal(v2.view(torch.int16), v1.view(torch.int16))


@pytest.mark.parametrize("H,Hkv,C,q0", [(4, 2, 64, 64), (4, 2, 64, 192), (4, 2, 1, 256),
                                        (4, 2, 44, 256), (8, 8, 128, 0), (32, 4, 100, 900)])
def test_attn_chunk_against_torch(K, H, Hkv, C, q0):
    """Chunk attention over the paged pool (keys 0..q0+C-1, causal per query
    row) against a torch fp32 reference."""
    dh, bs = 128, 16
    L = q0 + C
    maxb = (L + bs - 1) // bs + 2
    nblk = maxb + 4
    kp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    vp = torch.randn(nblk, Hkv, bs, dh, device="cuda").bfloat16()
    table = torch.randperm(nblk, device="cuda").int()[:maxb].contiguous()
    qkv = torch.randn(C, (H + 2 * Hkv) * dh, device="cuda").bfloat16()
    max_ctx = maxb * bs
    ws = torch.zeros(K.attn_chunk_workspace_bytes(C, H, max_ctx), dtype=torch.uint8, device="cuda")
    out = torch.empty(C, H * dh, dtype=torch.bfloat16, device="cuda")
    for _ in range(2):   # tickets self-reset
        K.attn_chunk(qkv, C, q0, kp.data_ptr(), vp.data_ptr(), table.data_ptr(), H, Hkv, dh, bs,
                     1 / math.sqrt(dh), max_ctx, ws, out)
    torch.cuda.synchronize()
    p = torch.arange(L, device="cuda")
    blk = table[p // bs].long()
    k = kp[blk, :, p % bs].float().repeat_interleave(H // Hkv, 1)    # [L, H, dh]
    v = vp[blk, :, p % bs].float().repeat_interleave(H // Hkv, 1)
    q = qkv[:, :H * dh].view(C, H, dh).float()
    s = torch.einsum("qhd,khd->hqk", q, k) / math.sqrt(dh)
    qpos = torch.arange(q0, q0 + C, device="cuda")
    s = s.masked_fill(p[None, None, :] > qpos[None, :, None], float("-inf"))
    ref = torch.einsum("hqk,khd->qhd", s.softmax(-1), v)
    assert _rel(out.view(C, H, dh), ref) < 1e-2


@pytest.mark.parametrize("bloom", [False, True])
def test_add_parts_norm_equals_sum_then_norm(K, bloom):
    """TP prefill exchange: the norm adds the ranks' bf16 partials (summed in
    fp32 in rank order) to the fp32 residual, bit-identical to adding the
    same sum first and normalising after."""
    T, d = 300, 1024
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(T, d, device="cuda", generator=g)
    parts = [torch.randn(T, d, device="cuda", generator=g).bfloat16() for _ in range(3)]
    w = (1 + 0.1 * torch.randn(d, device="cuda", generator=g)).bfloat16()
    b = (0.1 * torch.randn(d, device="cuda", generator=g)).bfloat16()
    s = parts[0].float() + parts[1].float() + parts[2].float()
    xr = x + s
    xa = x.clone()
    if bloom:
        got = K.layernorm(xa, w, b, 1e-5, addend=parts)
        ref = K.layernorm(xr, w, b, 1e-5)
    else:
        got = K.rmsnorm(xa, w, 1e-5, addend=parts)
        ref = K.rmsnorm(xr, w, 1e-5)
    torch.cuda.synchronize()
    assert torch.equal(xa, xr)
    assert torch.equal(got.view(torch.int16), ref.view(torch.int16))
