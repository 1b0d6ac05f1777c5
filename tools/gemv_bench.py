"""Decode linear (GEMV) bandwidth across batch rows M and model shapes.

Usage: python tools/gemv_bench.py [--ms 1,2,4,8,16] [--ncu M]   (weights > L2)"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_18677_b200 import kernels as K  # noqa: E402

SHAPES = {  # name: (N, K, epilogue)
    "7b.qkv": (12288, 4096, K.EPI_BF16),
    "7b.gu": (22016, 4096, K.EPI_SWIGLU),
    "7b.down": (4096, 11008, K.EPI_RESID_F32),
    "70b-tp2.gu": (28672, 8192, K.EPI_SWIGLU),
    "70b-tp2.down": (8192, 14336, K.EPI_RESID_F32),
    "70b-tp4.qkv": (2560, 8192, K.EPI_BF16),
    "70b-tp4.o": (8192, 2048, K.EPI_RESID_F32),
    "70b-tp4.gu": (14336, 8192, K.EPI_SWIGLU),
    "70b-tp4.down": (8192, 7168, K.EPI_RESID_F32),
    "bloom-tp4.qkv": (10752, 14336, K.EPI_BF16),
    "bloom-tp4.o": (14336, 3584, K.EPI_RESID_F32),
    "bloom-tp4.up": (14336, 14336, K.EPI_GELU),
    "bloom-tp4.down": (14336, 14336, K.EPI_RESID_F32),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="1,2,4,8,16")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    ms = [int(v) for v in a.ms.split(",")]
    for name, (N, Kd, epi) in SHAPES.items():
        if a.only and a.only not in name:
            continue
        # several weight copies so consecutive launches never hit L2
        copies = max(2, int(2 * 126e6 // (N * Kd * 2)) + 1)
        ws = [torch.randn(N, Kd, device="cuda").bfloat16() for _ in range(copies)]
        row = []
        for M in ms:
            x = torch.randn(M, Kd, device="cuda").bfloat16()
            resid = torch.randn(M, N, device="cuda") if epi == K.EPI_RESID_F32 else None
            out = resid if resid is not None else None
            bias = torch.randn(N, device="cuda").bfloat16() if epi == K.EPI_GELU else None
            for i in range(3):
                K.gemv(x, ws[i % copies], epi, out=out, resid=resid, bias=bias)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for i in range(a.reps):
                K.gemv(x, ws[i % copies], epi, out=out, resid=resid, bias=bias)
            e.record()
            torch.cuda.synchronize()
            ms_ = s.elapsed_time(e) / a.reps
            row.append(f"M={M}: {ms_ * 1e3:6.1f}us {N * Kd * 2 / ms_ / 1e6:6.0f}GB/s")
        print(f"{name:16s} " + "  ".join(row), flush=True)
        del ws


if __name__ == "__main__":
    main()
