"""Run one small plan through the C ABI (debug helper for compute-sanitizer / ncu)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2502_07155_b200 import bnfft  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prec = sys.argv[2] if len(sys.argv) > 2 else "c64"
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cid = {1: 2, 2: 3, 3: 4}[d]
cfg = synth.CONFIGS[cid].scaled(M=32 if d > 1 else 1024, N=5000, batch=batch)
x = torch.from_numpy(synth.make_nodes(cfg)).cuda()
fh = torch.from_numpy(synth.make_spectrum(cfg, prec=prec)).cuda()
import os
p = bnfft.Plan(d, cfg.M, 2.0, 4, "sinh", prec, batch=batch, exact_taps=bool(int(os.environ.get("EXACT", "0"))))
print(p.info().tap_poly, p.info().nkeys, p.info().bin_log2[0])
p.set_nodes(x)
f = p.execute(fh)
torch.cuda.synchronize()
print("ok", f.shape, float(f.abs().max()))
