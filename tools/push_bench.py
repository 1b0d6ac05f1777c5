"""KV push bandwidth over NVLink: one layer's K/V rows of a prompt packed
from the prompt GPU's QKV buffer into the token GPU's paged pool (P2P
stores, kv_push_kernel), timed alone with CUDA events, vs a plain peer copy
of the same bytes (torch copy_, the driver's copy engines)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_18677_b200 import _abi
from paper_2311_18677_b200 import kernels as K
from paper_2311_18677_b200.kvcache import KVCacheManager

H = Hkv = 32; dh = 128; bs = 16
res = {}
with torch.cuda.device(1):
    kv = KVCacheManager(1, 4096, Hkv, dh, bs, 8, 256)
    seq = kv.allocate(4096)
    torch.cuda.synchronize()
with torch.cuda.device(0):
    _abi.call("swb_enable_peer", 1)
    for rows in (1024, 2048, 4096):
        qkv = torch.randn(rows, (H + 2 * Hkv) * dh, device="cuda:0").bfloat16()
        slots = torch.empty(rows, dtype=torch.int32, device="cuda:0")
        K.slots_from_table(kv.table_row_ptr(seq), 0, rows, bs, slots)
        nbytes = rows * 2 * Hkv * dh * 2
        for ctas in (32, 64, 148, 296, 592):
            f = lambda: K.kv_push_layer(qkv, rows, H, Hkv, dh, kv.k_layer_ptr(0), kv.v_layer_ptr(0),
                                        slots, bs, ctas)
            for _ in range(3): f()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(20): f()
            e.record(); torch.cuda.synchronize()
            ms = s.elapsed_time(e) / 20
            res[f"push_rows{rows}_ctas{ctas}_GBps"] = round(nbytes / ms / 1e6, 1)
        src = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda:0")
        dst = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda:1")
        for _ in range(3): dst.copy_(src)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20): dst.copy_(src)
        e.record(); torch.cuda.synchronize()
        res[f"peer_copy_{nbytes >> 20}MiB_GBps"] = round(nbytes / (s.elapsed_time(e) / 20) / 1e6, 1)
# correctness: pushed rows equal the source K/V
with torch.cuda.device(1):
    kt = kv.k_view(0); tbl = kv.tables()[seq].long()
    p = torch.arange(4096, device="cuda:1")
    got = kt[tbl[p // bs], :, p % bs].reshape(4096, Hkv * dh)
ref = qkv[:, H * dh:(H + Hkv) * dh].to("cuda:1")
res["bit_exact"] = bool(torch.equal(got.view(torch.int16), ref.view(torch.int16)))
print(json.dumps(res))
