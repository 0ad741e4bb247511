import os, sys, subprocess, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
r = int(sys.argv[1]) if len(sys.argv) > 1 else 64
col = synth.config5(N=64, r=r)
sp = oracle.block_spectra(col.blocks)
order = np.array(sorted(range(col.N), key=lambda i: (-sp.E[i], i)))
pairs = synth.all_pairs_by_norm_order(order)[:12]
ref = oracle.pair_errors(sp, pairs, r, 7)
code = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import synth, paper_2601_11626_b200 as cm
col = synth.config5(N=64, r=int(sys.argv[2]))
ctx = cm.Context(0); ctx.register(col.blocks); ctx.block_spectra(col.r)
pairs = np.load(sys.argv[3])
out = ctx.pair_errors(pairs)
np.savez(sys.argv[4], **{k: v for k, v in out.items()})
'''
np.save("/tmp/pairs.npy", pairs)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for tag, env in [("tc", {}), ("simt", {"CMSVD_NO_TC": "1"})]:
    subprocess.run([sys.executable, "-c", code, root, str(r), "/tmp/pairs.npy", f"/tmp/{tag}.npz"], env=dict(os.environ, **env), check=True)
    o = np.load(f"/tmp/{tag}.npz")
    d = np.abs(o["sigma_tilde"] - ref.sigma_tilde)
    print(tag, "max |dsig~| =", d.max(), "at", np.unravel_index(d.argmax(), d.shape), "ref", ref.sigma_tilde[np.unravel_index(d.argmax(), d.shape)],
          " max rel err2 diff:", [float(np.max(np.abs(o["err2"][:, k] - ref.err2[:, k]) / ref.total)) for k in range(3)],
          " mu:", np.abs(o["mu"] - ref.mu).max())
