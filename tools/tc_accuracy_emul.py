"""Emulate the tcgen05 3xTF32 accumulation schemes of dwm_gemm_tc.cu in NumPy
and report output MSE vs FP64 direct conv, relative to the reference DWM32.

Model (measured by tools/tc_accum_probe.cu / tc_probe.cu): operands are TF32
(V: hi = RNA-to-TF32 by the integer trick, lo = x - hi, truncated to TF32 by
the tensor core; U: hi/lo both RNA), the 8 products of one K=8 MMA step are
summed exactly, and the FP32 accumulator update truncates toward zero.

Schemes:
  chunk<S>  fresh accumulator per S channels (S a multiple of 32); per 32
            channels 8 correction steps, then 4 main steps; chunks summed in
            FP32 RN (chunk32: the shipped kernel for C = 64)
  cfirst<S> fresh accumulator per S channels: all 2S/8 correction steps,
            then the S/8 main steps
  split<K>  main (hi*hi) accumulator per K channels, one correction
            accumulator over all channels; mq = sum(main chunks) + corr
  long      one accumulator over all channels (corr first per 32 ch)
  <scheme>_tv  V's hi operand is raw V truncated by the tensor core (SS-mode A
            straight from the TMA stage) instead of the RN split
  pair<S>   main (hi*hi) and correction (hi*lo + lo*hi) in two accumulators,
            both fresh per S channels (one N=128 MMA [Uh;Ul] + one N=64
            MMA Vl*Uh per K step); chunk = main + corr, chunks summed in FP32

    python tools/tc_accuracy_emul.py [--workloads cfg4-7x7s1,...] [--filters 64]
"""

import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle.dwm_oracle import (direct_conv2d_f64, draw, dwm_conv2d_oracle, filter_transform_oracle,  # noqa: E402
                               input_transform_oracle, mse)
from paper_2002_00552_b200 import plan_decomposition  # noqa: E402
from paper_2002_00552_b200.configs import WORKLOADS  # noqa: E402
from paper_2002_00552_b200.transforms import to_float  # noqa: E402


def rna_tf32(x32):
    b = x32.view(np.uint32)
    return ((b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)


def trunc_tf32(x32):
    return (x32.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def rz32(x64):
    f = x64.astype(np.float32)
    over = np.abs(f.astype(np.float64)) > np.abs(x64)
    f[over] = np.nextafter(f[over], np.float32(0))
    return f


def step(acc, a, b, first):
    """One K=8 MMA step: acc (f32) + sum of 8 exact products, truncated."""
    p = np.einsum("qtc,qfc->qtf", a.astype(np.float64), b.astype(np.float64))
    return rz32(p) if first else rz32(acc.astype(np.float64) + p)


def contraction(V, U, scheme):
    Q, T, C = V.shape
    if scheme.endswith("_tv"):
        # raw V as the hi operand (the tensor core truncates it to TF32); lo = V - trunc(V)
        scheme = scheme[:-3]
        vh = trunc_tf32(V)
    else:
        vh = rna_tf32(V)
    vl = trunc_tf32((V - vh).astype(np.float32))
    uh = rna_tf32(U)
    ul = rna_tf32((U - uh).astype(np.float32))
    ks = [slice(8 * k, 8 * k + 8) for k in range(C // 8)]
    if scheme.startswith("chunk") or scheme == "long":
        span = int(scheme[len("chunk"):]) if scheme != "long" else C
        mq = None
        acc = None
        for c0 in range(0, C, 32):
            kk = ks[c0 // 8:c0 // 8 + 4]
            fresh = c0 % span == 0
            for i, k in enumerate(kk):
                acc = step(acc, vh[..., k], ul[..., k], fresh and i == 0)
                acc = step(acc, vl[..., k], uh[..., k], False)
            for k in kk:
                acc = step(acc, vh[..., k], uh[..., k], False)
            if scheme != "long" and (c0 + 32) % span == 0:
                mq = acc if mq is None else (mq + acc).astype(np.float32)
        return acc if scheme == "long" else mq
    if scheme.startswith("cfirst"):
        span = int(scheme[len("cfirst"):])
        mq = None
        for c0 in range(0, C, span):
            kk = ks[c0 // 8:(c0 + span) // 8]
            acc = None
            for i, k in enumerate(kk):
                acc = step(acc, vh[..., k], ul[..., k], i == 0)
                acc = step(acc, vl[..., k], uh[..., k], False)
            for k in kk:
                acc = step(acc, vh[..., k], uh[..., k], False)
            mq = acc if mq is None else (mq + acc).astype(np.float32)
        return mq
    if scheme.startswith("pairc"):
        # pair<S> plus a truncation-bias compensation: each of the S/8 main
        # steps truncates toward zero by ~0.5 ulp on average, so add back
        # alpha * steps * ulp(main) in the direction of main (scheme pairc<S>_<alpha*100>)
        span, alpha = scheme[len("pairc"):].split("_")
        span, alpha = int(span), int(alpha) / 100.0
        mq = None
        for c0 in range(0, C, span):
            kk = ks[c0 // 8:(c0 + span) // 8]
            acc = corr = None
            for i, k in enumerate(kk):
                acc = step(acc, vh[..., k], uh[..., k], i == 0)
                corr = step(corr, vh[..., k], ul[..., k], i == 0)
                corr = step(corr, vl[..., k], uh[..., k], False)
            e = np.floor(np.log2(np.maximum(np.abs(acc.astype(np.float64)), 1e-38)))
            ulp = np.exp2(e - 23).astype(np.float32)
            comp = (np.sign(acc) * np.float32(alpha * len(kk)) * ulp).astype(np.float32)
            chunk = ((acc + comp).astype(np.float32) + corr).astype(np.float32)
            mq = chunk if mq is None else (mq + chunk).astype(np.float32)
        return mq
    if scheme.startswith("pair"):
        span = int(scheme[len("pair"):])
        mq = None
        for c0 in range(0, C, span):
            kk = ks[c0 // 8:(c0 + span) // 8]
            acc = corr = None
            for i, k in enumerate(kk):
                acc = step(acc, vh[..., k], uh[..., k], i == 0)
                corr = step(corr, vh[..., k], ul[..., k], i == 0)
                corr = step(corr, vl[..., k], uh[..., k], False)
            chunk = (acc + corr).astype(np.float32)
            mq = chunk if mq is None else (mq + chunk).astype(np.float32)
        return mq
    kch = int(scheme[len("split"):])
    corr = None
    mq = None
    for c0 in range(0, C, kch):
        acc = None
        for i, k in enumerate(ks[c0 // 8:(c0 + kch) // 8]):
            acc = step(acc, vh[..., k], uh[..., k], i == 0)
            corr = step(corr, vh[..., k], ul[..., k], corr is None)
            corr = step(corr, vl[..., k], uh[..., k], False)
        mq = acc if mq is None else (mq + acc).astype(np.float32)
    return (mq + corr).astype(np.float32)


def output(M, spec, n, oh, ow):
    plan = plan_decomposition(spec)
    th, tw = -(-oh // 2), -(-ow // 2)
    F = M.shape[2]
    Y = np.zeros((4, M.shape[1], F), dtype=np.float32)
    q = 0
    for part in plan.parts:
        atr = to_float(part.transform_rows, np.float64)["a_t"]
        atc = to_float(part.transform_cols, np.float64)["a_t"]
        lr, lc = part.row.count + 1, part.col.count + 1
        for a in range(lr):
            for b in range(lc):
                for i in range(2):
                    for j in range(2):
                        cf = atr[i][a] * atc[j][b]
                        if cf > 0:
                            Y[2 * i + j] = (Y[2 * i + j] + M[q]).astype(np.float32)
                        elif cf < 0:
                            Y[2 * i + j] = (Y[2 * i + j] - M[q]).astype(np.float32)
                q += 1
    y = Y.reshape(2, 2, n, th, tw, F).transpose(2, 5, 3, 0, 4, 1).reshape(n, F, 2 * th, 2 * tw)
    return y[:, :, :oh, :ow]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="cfg4-3x3s1,cfg4-7x7s1,cfg5-5x5s2")
    ap.add_argument("--filters", type=int, default=64)
    ap.add_argument("--channels", type=int, default=0, help="override C_in (e.g. 64)")
    ap.add_argument("--schemes", default="chunk32,split64,split128,long")
    args = ap.parse_args()
    for name in args.workloads.split(","):
        wl = WORKLOADS[name]
        spec = wl.spec()
        c = args.channels or wl.c_in
        d, g = draw(1, (wl.kernel,) * 2, (wl.stride,) * 2, wl.hw, c, args.filters, 1)
        y64 = direct_conv2d_f64(d, g, spec)
        ref = mse(dwm_conv2d_oracle(d, g, spec, np.float32), y64)
        V = input_transform_oracle(d, spec, np.float32)
        U = filter_transform_oracle(g, spec, np.float32)
        oh, ow = y64.shape[2:]
        line = [f"{name} C={c} F={args.filters}: ref DWM32 MSE {ref:.3e}"]
        for sch in args.schemes.split(","):
            y = output(contraction(V, U, sch), spec, 1, oh, ow)
            line.append(f"{sch} {mse(y, y64) / ref:.3f}x")
        print(" | ".join(line), flush=True)


if __name__ == "__main__":
    main()
