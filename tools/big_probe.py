"""Probe: time the big-block spectra (A22 subspace iteration) and a pair batch
on full-size configs 3/4; compare a few blocks' top-r sigma against an fp64
eigh of the Gram (numpy).  Usage: python tools/big_probe.py config4 [iters]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2601_11626_b200 as cm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config4"
if len(sys.argv) > 2:
    os.environ["CMSVD_SUBSPACE_ITERS"] = sys.argv[2]
t = time.time()
col = synth.make_config(name)
print(f"{name}: N={col.N} m={col.m} n={col.n} r={col.r} gen {time.time() - t:.1f}s", flush=True)
cm.load()
blocks = torch.from_numpy(col.blocks).cuda()
with cm.Context(0, torch.cuda.current_stream().cuda_stream) as ctx:
    ctx.register(blocks)
    torch.cuda.synchronize()
    for rep in range(2):
        t = time.time()
        E, sig, rank = ctx.block_spectra(col.r)
        print(f"spectra {time.time() - t:.3f}s", flush=True)
    ctx.profile(True)
    ctx.register(blocks)
    ctx.block_spectra(col.r)
    prof = ctx.profile_read()
    ctx.profile(False)
    ems = prof["energy"][0]
    nbytes = col.blocks.nbytes
    print(f"S1 energy kernel: {ems:.3f} ms for {nbytes / 1e9:.2f} GB = {nbytes / (ems * 1e-3) / 1e9:.0f} GB/s; "
          f"S2 profile {prof}", flush=True)
    for i in [0, col.N - 1]:
        a = col.blocks[i].T.astype(np.float64)
        lam = np.linalg.eigvalsh(a @ a.T)[::-1][:col.r]
        ref = np.sqrt(np.maximum(lam, 0))
        rel = np.abs(sig[i] - ref) / ref
        print(f"block {i}: max rel sigma err {rel.max():.3e} (at l={rel.argmax()}), sigma_1 {ref[0]:.4g}, "
              f"sigma_r {ref[-1]:.4g}", flush=True)
    order = np.argsort(-E, kind="stable")
    pairs = synth.all_pairs_by_norm_order(order)
    if name == "config3":
        pairs = pairs[:2016]
    for rep in range(2):
        t = time.time()
        out = ctx.pair_errors(pairs, kinds=7, operand=cm.TRUNC)
        dt = time.time() - t
        print(f"pairs {len(pairs)}: {dt:.3f}s = {len(pairs) / dt:.1f} evals/s", flush=True)
    ctx.profile(True)
    out = ctx.pair_errors(pairs, kinds=7, operand=cm.TRUNC)
    print(ctx.profile_read(), flush=True)
    print("err2[:3]", out["err2"][:3], "total", out["total"][:3])
