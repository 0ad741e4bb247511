"""Probe: phase split of the Rayleigh-Ritz eigen-solve of S2 (k_syev_ql, n = 512 in global memory).
Build a copy of the library with -DCMSVD_SYEV_PROF (tools/build_prof_lib.sh) and point CMSVD_LIB at it:
block 0's CTA prints the cycles of tridiagonalisation / QL / back-transformation.
Usage: [CMSVD_LIB=tools/libcmsvd_prof.so] [CMSVD_SYEV_COLBT=0] python tools/syev_phase.py [N]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2601_11626_b200 as cm  # noqa: E402
from paper_2601_11626_b200 import cmsvd as _b  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
col = synth.config4(N=N)
cm.load(os.environ.get("CMSVD_LIB", _b.LIB_PATH))
blocks = torch.from_numpy(col.blocks).cuda()
with cm.Context(0, torch.cuda.current_stream().cuda_stream) as ctx:
    ctx.register(blocks)
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.time()
        E, sig, rank = ctx.block_spectra(col.r)
        torch.cuda.synchronize()
        print(f"N={N} spectra {1e3 * (time.time() - t):.1f} ms  sigma[0][:3]={sig[0][:3]}  guard={ctx.spectra_diagnostics()}",
              flush=True)
