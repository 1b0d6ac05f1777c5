"""Prefill attention A/B: tcgen05 kernel vs mma.sync FA2 kernel.

Prints per-shape time and causal-algorithmic TFLOP/s (4*S*S/2*H*dh per seq)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_18677_b200 import kernels as K  # noqa: E402


def bench(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    dh = 128
    for H, Hkv, lens in [(32, 32, [1024]), (32, 32, [4096]), (64, 8, [1024] * 2),
                         (32, 32, [512] * 8), (64, 8, [8192])]:
        S = sum(lens)
        qkv = torch.randn(S, (H + 2 * Hkv) * dh, device="cuda").bfloat16()
        cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), device="cuda",
                          dtype=torch.int32)
        flops = sum(2.0 * L * L * H * dh for L in lens)  # causal half of 4*L*L*H*dh
        res = {}
        outs = {}
        for impl in ("tc", "fa2"):
            out = torch.empty(S, H * dh, device="cuda", dtype=torch.bfloat16)
            ms = bench(lambda: K.attn_prefill(qkv, cu, len(lens), max(lens), H, Hkv, dh,
                                              1 / math.sqrt(dh), out=out, impl=impl))
            res[impl] = ms
            outs[impl] = out
        diff = (outs["tc"].float() - outs["fa2"].float()).abs().max().item()
        print(f"H={H} Hkv={Hkv} lens={lens[:2]}x{len(lens)}: "
              + "  ".join(f"{k} {v * 1e3:.1f}us {flops / v / 1e9:.0f}TF/s" for k, v in res.items())
              + f"  maxdiff={diff:.4f}", flush=True)


if __name__ == "__main__":
    main()
