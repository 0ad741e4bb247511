"""The tcgen05 3xTF32 contraction path vs the SIMT path and the oracle (-m gpu)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import synth, paper_2601_11626_b200 as cm
name = sys.argv[2]
col = {"config1": synth.config1, "config2": synth.config2}[name]() if name != "config5" else synth.config5(N=256, r=int(sys.argv[3]))
ctx = cm.Context(0)
ctx.register(col.blocks)
E, sig, rank = ctx.block_spectra(col.r)
order = np.array(sorted(range(col.N), key=lambda i: (-E[i], i)))
pairs = synth.all_pairs_by_norm_order(order)[:2000]
out = ctx.pair_errors(pairs)
ctx.profile(True)
ctx.pair_errors(pairs[:64])
prof = ctx.profile_read()
np.savez(sys.argv[4], pairs=pairs, **{k: v for k, v in out.items()})
print(json.dumps({k: v[1] for k, v in prof.items() if v[1]}))
'''


def run(env_extra, name, r, path):
    env = dict(os.environ, **env_extra)
    res = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, name, str(r), path], env=env, capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    return res.stdout.strip().splitlines()[-1]


@pytest.mark.parametrize("name,r", [("config1", 8), ("config2", 32), ("config5", 16), ("config5", 64)])
def test_tc_matches_simt(tmp_path, name, r):
    a = str(tmp_path / "tc.npz")
    b = str(tmp_path / "simt.npz")
    prof_tc = run({}, name, r, a)
    prof_simt = run({"CMSVD_NO_TC": "1"}, name, r, b)
    assert "pair_tc" in prof_tc and "pair_tc" not in prof_simt
    A = np.load(a)
    B = np.load(b)
    tot = A["total"]
    for k in range(3):
        e1, e2 = A["err2"][:, k], B["err2"][:, k]
        assert np.all(np.abs(e1 - e2) <= 2e-3 * np.maximum(e1, e2) + 1e-7 * tot), (k, np.max(np.abs(e1 - e2) / tot))
    s1, s2 = A["sigma_tilde"], B["sigma_tilde"]
    assert np.all(np.abs(s1 - s2) <= 1e-4 * np.abs(s2) + 1e-6 * s2[:, :1])
