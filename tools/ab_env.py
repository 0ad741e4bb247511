"""A/B probe: run config-2 all-pairs (all three estimators) in two contexts
created under different CMSVD_* environment settings and compare the outputs
bitwise, plus per-category kernel times.
Usage: python tools/ab_env.py CMSVD_ZZ_FUSED=0 CMSVD_ZZ_FUSED=1 [config]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2601_11626_b200 as cm  # noqa: E402

envA, envB = sys.argv[1], sys.argv[2]
name = sys.argv[3] if len(sys.argv) > 3 else "config2"
OPERAND = cm.TRUNC if name in ("config3", "config4") else cm.RAW
col = synth.make_config(name)
blocks = torch.from_numpy(col.blocks).cuda()
cm.load()


def run(env):
    k, v = env.split("=")
    old = os.environ.get(k)
    os.environ[k] = v
    try:
        with cm.Context(0, torch.cuda.current_stream().cuda_stream) as ctx:
            ctx.register(blocks)
            E, sig, rank = ctx.block_spectra(col.r)
            order = np.array(sorted(range(col.N), key=lambda i: (-E[i], i)))
            pairs = synth.all_pairs_by_norm_order(order)
            out = ctx.pair_errors(pairs, kinds=cm.ALL, operand=OPERAND)
            torch.cuda.synchronize()
            import time
            t0 = time.perf_counter()
            for _ in range(3):
                ctx.pair_errors(pairs, kinds=cm.ALL, operand=OPERAND)
            torch.cuda.synchronize()
            print(f"{env}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms per pass (host clock, 3 passes, host pairs in / results out)")
            ctx.profile(True)
            for _ in range(3):
                ctx.pair_errors(pairs, kinds=cm.ALL, operand=OPERAND)
            torch.cuda.synchronize()
            prof = ctx.profile_read()
            ctx.profile(False)
    finally:
        if old is None:
            del os.environ[k]
        else:
            os.environ[k] = old
    return out, {kk: round(vv[0] / max(vv[1], 1), 3) for kk, vv in prof.items() if vv[1]}


a, pa = run(envA)
b, pb = run(envB)
for key in a:
    x, y = np.asarray(a[key]), np.asarray(b[key])
    same = np.array_equal(x, y, equal_nan=True)
    rel = np.nanmax(np.abs(x - y) / np.maximum(np.abs(x), 1e-30)) if x.dtype.kind == "f" else float(not same)
    print(f"{key:12s} bitwise {'==' if same else '!='}  max rel diff {rel:.3e}")
print(f"{envA}: ms/launch {pa}")
print(f"{envB}: ms/launch {pb}")
