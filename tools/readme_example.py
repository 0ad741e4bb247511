import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch, synth
import paper_2601_11626_b200 as cm

col = synth.config2()
with cm.Context(0) as ctx:
    ctx.register(torch.from_numpy(col.blocks).cuda())
    E, sigma, rank = ctx.block_spectra(col.r)
    pairs = np.array([[0, 8], [0, 1]], np.int32)
    out = ctx.pair_errors(pairs)
    rel = np.sqrt(out["err2"] / out["total"][:, None])
    g = ctx.cluster(cm.ALG_APPROX, 0.05, sort=cm.SORT_RESIDUAL)
    v = ctx.cluster_verify(np.asarray(g["assign"], np.int32))
    s = ctx.sequence_errors([[0, 8, 16]])
    t = ctx.pair_errors_tight(pairs)
    print(rel, v["ratio"], s["err2"], t["err2x"])
