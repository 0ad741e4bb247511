"""A/B probe between two builds of libcmsvd.so: config-2 all-pairs outputs (bitwise comparison) and
per-category kernel times.  Usage: python tools/ab_lib.py <libA.so> <libB.so> [config]"""
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def child(lib, name, out):
    sys.path.insert(0, os.path.dirname(HERE))
    import torch
    import synth
    import paper_2601_11626_b200.cmsvd as cmb
    cmb.load(lib)
    import paper_2601_11626_b200 as cm
    col = synth.make_config(name)
    with cm.Context(0, torch.cuda.current_stream().cuda_stream) as ctx:
        ctx.register(torch.from_numpy(col.blocks).cuda())
        E, sig, rank = ctx.block_spectra(col.r)
        order = np.array(sorted(range(col.N), key=lambda i: (-E[i], i)))
        pairs = synth.all_pairs_by_norm_order(order)
        res = ctx.pair_errors(pairs)
        ctx.profile(True)
        for _ in range(3):
            ctx.pair_errors(pairs)
        torch.cuda.synchronize()
        prof = ctx.profile_read()
    np.savez(out, **{k: v for k, v in res.items() if v is not None})
    print({k: round(v[0] / max(v[1], 1), 3) for k, v in prof.items() if v[1]})


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3], sys.argv[4])
        sys.exit(0)
    a, b = sys.argv[1], sys.argv[2]
    name = sys.argv[3] if len(sys.argv) > 3 else "config2"
    outs = []
    for k, lib in enumerate((a, b)):
        o = f"/tmp/ab_lib_{k}.npz"
        r = subprocess.run([sys.executable, __file__, "--child", os.path.abspath(lib), name, o],
                           capture_output=True, text=True)
        print(os.path.basename(lib), r.stdout.strip(), r.stderr.strip()[-300:])
        outs.append(np.load(o))
    for key in outs[0].files:
        x, y = outs[0][key], outs[1][key]
        same = np.array_equal(x, y, equal_nan=True)
        rel = np.nanmax(np.abs(x - y) / np.maximum(np.abs(x), 1e-30))
        print(f"{key:12s} bitwise {'==' if same else '!='}  max rel diff {rel:.3e}")
