#!/usr/bin/env python
"""The paper's kernel benchmark grid on this GPU.

N in {512 .. 16384}, B = 16384 / N (16K tokens), d = 64 (H = 32) and d = 128 (H = 16), 0% and 25%
padding (every sequence n = 0.75 N), forward and backward timed separately with CUDA events.
TFLOPS on valid tokens: fwd 4 B H n^2 d, bwd 10 B H n^2 d.  Context column: torch SDPA
(softmax, flash / cuDNN backend, unpadded only) on the same box -- a comparison system, not a target.
usage: python scripts/kernel_grid.py [--iters 50] [--out profiles/r1_kernel_grid.txt]
"""
import argparse
import math
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27124_b200 as sa  # noqa: E402


def timeit(fn, iters):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    lines = []
    hdr = "%-5s %-6s %-4s %-4s %-5s | %9s %9s | %9s %9s | %9s" % (
        "d", "N", "B", "H", "pad", "fwd ms", "fwd TF", "bwd ms", "bwd TF", "sdpa f/b TF")
    lines.append(hdr)
    summary = {}
    for d, H in ((64, 32), (128, 16)):
        for N in (512, 1024, 2048, 4096, 8192, 16384):
            B = 16384 // N
            for pad in (0.0, 0.25):
                n = int(round(N * (1 - pad)))
                q, k, v, do = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(4))
                lens = torch.full((B,), n, dtype=torch.int32, device="cuda")
                ws = torch.empty(sa.bwd_workspace_bytes(B, H, N, N, d), dtype=torch.uint8, device="cuda")
                o = torch.empty_like(q)
                dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
                tf = timeit(lambda: sa.sigattn_fwd(q, k, v, lens, lens, out=o), a.iters)
                tb = timeit(lambda: sa.sigattn_bwd(q, k, v, do, lens, lens, dq=dq, dk=dk, dv=dv, workspace=ws), a.iters)
                ff = 4.0 * B * H * n * n * d
                sdpa = ""
                if pad == 0.0:
                    qq, kk, vv = (t.clone().requires_grad_(True) for t in (q, k, v))
                    ts_f = timeit(lambda: F.scaled_dot_product_attention(q, k, v), a.iters)
                    out = F.scaled_dot_product_attention(qq, kk, vv)
                    ts_b = timeit(lambda: torch.autograd.grad(out, (qq, kk, vv), do, retain_graph=True), a.iters)
                    sdpa = "%4.0f/%4.0f" % (ff / ts_f / 1e9, 2.5 * ff / ts_b / 1e9)
                fwd_tf, bwd_tf = ff / tf / 1e9, 2.5 * ff / tb / 1e9
                summary.setdefault((d, pad), []).append((fwd_tf, bwd_tf))
                lines.append("%-5d %-6d %-4d %-4d %-5s | %9.3f %9.1f | %9.3f %9.1f | %9s" % (
                    d, N, B, H, "%d%%" % int(pad * 100), tf, fwd_tf, tb, bwd_tf, sdpa))
                print(lines[-1], flush=True)
                del q, k, v, do, ws, o, dq, dk, dv
    lines.append("")
    for d in (64, 128):
        f0 = sum(x[0] for x in summary[(d, 0.0)]) / len(summary[(d, 0.0)])
        b0 = sum(x[1] for x in summary[(d, 0.0)]) / len(summary[(d, 0.0)])
        f1 = sum(x[0] for x in summary[(d, 0.25)]) / len(summary[(d, 0.25)])
        b1 = sum(x[1] for x in summary[(d, 0.25)]) / len(summary[(d, 0.25)])
        lines.append("d=%d mean over N: 0%% pad fwd %.1f bwd %.1f TFLOPS; 25%% pad fwd %.1f (%+.1f%%) bwd %.1f (%+.1f%%)" % (
            d, f0, b0, f1, 100 * (f1 / f0 - 1), b1, 100 * (b1 / b0 - 1)))
    lines.append("paper (H100, TritonSigmoid, mean over the grid): 0%->25% pad fwd 438.4->397.5, bwd 316.1->286.6 "
                 "TFLOPS (-9.3%, P:156-158); peak N=16K d=128 unpadded fwd 515.6 / bwd 373.5 (P:150)")
    text = "\n".join(lines)
    print("\n".join(lines[-4:]))
    if a.out:
        open(a.out, "w").write(text + "\n")


if __name__ == "__main__":
    main()
